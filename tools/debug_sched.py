"""Debug: compare flat vs doc-blocked schedules step by step (GPU)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_04631_b200 import corpus as cp, synth
from paper_1803_04631_b200.shard import DeviceShard

K = 256
corp = synth.generate(1500, 3000, 250.0, seed=31)
ch = cp.partition(corp, 1, K, 7)[0]
a, b = 50.0 / K, 0.01

def run(kb, mr, iters):
    os.environ["GF_DOCBLOCK_KB"] = kb
    os.environ["GF_SLICE_MINRUNS"] = mr
    sh = DeviceShard(K, corp.vocab_size, a, b, seed=3).load(ch)
    sh.initialize()
    th0 = sh.get_theta()
    for it in range(iters):
        sh.sample(it)
        if it < iters - 1:
            sh.rebuild_phi(); sh.prepare(); sh.rebuild_theta()
    z = sh.get_assignments(); st = sh.stats(); ll = sh.loglik_sum()
    sh.close()
    return th0, z, st, ll

for iters in (1, 2):
    f = run("1000000", "1000000000", iters)
    for cfg in [("1000000", "1000000000"), ("256", "16"), ("100000", "16"), ("256", "100000")]:
        g = run(*cfg, iters)
        same_th = all((x == y).all() for x, y in zip(f[0], g[0]))
        d = np.flatnonzero(f[1] != g[1])
        print(iters, cfg, "theta0 same", same_th, "z diff", d.size, "slices", g[2]["slices"], "ctx", g[2]["word_contexts"],
              "blocks", g[2]["doc_blocks"], "ll", g[3] - f[3])
        if d.size:
            w = ch.word_ids[d]; dd = ch.doc_ids[d]
            print("   words", np.unique(w)[:10], "ndiff words", np.unique(w).size, "docs", np.unique(dd).size)
