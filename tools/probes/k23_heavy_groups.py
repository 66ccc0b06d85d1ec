"""K2 on heavy-word pieces and K3 on document groups, small corpora with heavy
words (run under compute-sanitizer memcheck by tools/sanitize.sh)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1803_04631_b200 import synth, corpus as cp
from paper_1803_04631_b200.shard import DeviceShard
for (D, V, L, K) in [(2000, 500, 60.0, 64), (20000, 300, 80.0, 128)]:
    corp = synth.generate(D, V, L, seed=3)
    ch = cp.partition(corp, 1, K, 42)[0]
    with DeviceShard(K, V, 50.0 / K, 0.01, seed=7) as sh:
        sh.load(ch)
        print("loaded", D, flush=True)
        sh.rebuild_phi(); sh.synchronize(); print("K2 ok", flush=True)
        sh.prepare(); sh.synchronize(); print("prepare ok", flush=True)
        sh.rebuild_theta(); sh.synchronize(); print("K3 ok", flush=True)
        sh.check_errors()
