"""K3 / K2 cost model (GPU box): time theta_rebuild and phi_rebuild alone on
corpora of (nearly) constant document length L, ~100M tokens, K=1024."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1803_04631_b200 import synth
from paper_1803_04631_b200.shard import DeviceShard
K = 1024
st = torch.cuda.current_stream()
def ev_time(fn, reps=5):
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(st); fn(); b.record(st); torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return float(np.median(out))
Ls = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "16,32,48,64,96,128,192,256,512".split(","))]
for L in Ls:
    D = 60_000_000 // L
    corp = synth.generate(D, 141_043, float(L), seed=5, sigma=1e-4)
    freq = np.bincount(corp.word_ids, minlength=corp.vocab_size).astype(np.int64)
    sh = DeviceShard(K, corp.vocab_size, 50.0 / K, 0.01, seed=42, global_word_freq=freq, stream=st)
    sh.load_tokens(0, corp.num_docs, corp.doc_ids, corp.word_ids, seed=42)
    sh.initialize()
    for it in range(3):
        sh.sample(it); sh.rebuild_phi(); sh.prepare(); sh.rebuild_theta()
    k3 = ev_time(sh.rebuild_theta)
    k2 = ev_time(sh.rebuild_phi)
    T = corp.num_tokens
    print(f"L={L:4d} D={D:9d} T={T/1e6:.1f}M  K3 {k3:.3f} ms = {k3*1e6/D:.2f} ns/doc {k3*1e6/T:.3f} ns/tok | K2 {k2:.3f} ms {T*2/k2/1e6:.0f} GB/s(z)", flush=True)
    sh.close()
