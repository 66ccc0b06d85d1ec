"""Draws of one K1 variant (GF_K1 env) on a fixed small state, saved to a
file: run twice with different GF_K1 and compare (the variants reorder work
only; every token keeps its Philox counter, so the draws must be identical)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1803_04631_b200 import corpus as cp, synth
from paper_1803_04631_b200.shard import DeviceShard
K = 1024
corp = synth.generate(40000, 20000, 90.0, seed=5)
ch = cp.partition(corp, 1, K, 9, device=0)[0]
with DeviceShard(K, corp.vocab_size, 50.0 / K, 0.01, seed=3) as sh:
    sh.load(ch)
    sh.initialize()
    out = []
    for it in range(3):
        sh.sample(it)
        out.append(sh.get_assignments().copy())
        out.append(np.array([sh.loglik_sum()]))
        sh.rebuild_phi(); sh.prepare(); sh.rebuild_theta(); sh.check_errors()
np.savez(sys.argv[1], *out)
