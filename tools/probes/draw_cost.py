"""K1 with and without its draws (gf_shard_evaluate = the same pass + loglik,
no draws) on a bench-like state: the draws' share of K1 time."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_1803_04631_b200 import _lib, synth
from paper_1803_04631_b200.shard import DeviceShard
wl = sys.argv[1] if len(sys.argv) > 1 else "pubmed"
K = 1024
shape = bench.SHAPES[wl]
corp = synth.generate(shape["num_docs"], shape["vocab_size"], shape["mean_len"], seed=bench.CORPUS_SEED)
freq = np.bincount(corp.word_ids, minlength=corp.vocab_size).astype(np.int64)
st = torch.cuda.current_stream()
sh = DeviceShard(K, corp.vocab_size, 50.0 / K, 0.01, seed=42, global_word_freq=freq, stream=st)
sh.load_tokens(0, corp.num_docs, corp.doc_ids, corp.word_ids, seed=42)
sh.initialize()
for it in range(8):                      # a bench-like (iteration ~8) state
    sh.sample(it); sh.rebuild_phi(); sh.prepare(); sh.rebuild_theta()
def t(fn, n=5):
    ms = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(st); fn(); b.record(st); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    return float(np.median(ms))
ev = t(lambda: _lib.check(_lib.lib().gf_shard_evaluate(sh._h)))
# sample the same state repeatedly: copy z so every launch starts from it
z0 = sh.get_assignments()
def samp():
    sh.sample(8)
smp = t(samp, 1)
print(f"{wl}: K1 sample {smp:.2f} ms, evaluate (no draws) {ev:.2f} ms -> draws ~{smp - ev:.2f} ms ({100 * (smp - ev) / smp:.1f}%)")
