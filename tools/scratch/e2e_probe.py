"""Where does the e2e step lose time against the resident step? PubMed-shape."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_1803_04631_b200.shard import DeviceShard
from paper_1803_04631_b200 import synth
K = 1024
shape = bench.SHAPES["pubmed"]
corp = synth.generate(shape["num_docs"], shape["vocab_size"], shape["mean_len"], seed=bench.CORPUS_SEED)
freq = np.bincount(corp.word_ids, minlength=corp.vocab_size).astype(np.int64)
st = torch.cuda.current_stream()
def make(phases):
    sh = DeviceShard(K, corp.vocab_size, 50.0 / K, 0.01, seed=42, global_word_freq=freq, stream=st, phases=phases)
    sh.load_tokens(0, corp.num_docs, corp.doc_ids, corp.word_ids, seed=42)
    sh.initialize()
    return sh
def ev_time(fn, reps=3):
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(st); fn(); b.record(st); torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return np.median(out)
it = [10]
def k1_all(sh):
    it[0] += 1; sh.sample(it[0])
sh1 = make(1)
for _ in range(3): k1_all(sh1)
print("K1 unphased ms", ev_time(lambda: k1_all(sh1)))
sh1.close()
for spec in ["geo:9", "geo:5", "4"]:
    if spec.startswith("geo:"):
        n = int(spec[4:]); cuts = [1.0 - 0.5 ** (p + 1) for p in range(n - 1)] + [1.0]
        sh = make(cuts)
    else:
        sh = make(int(spec))
    P = sh.num_phases
    def phased():
        it[0] += 1
        for p in range(P): sh.sample_phase(it[0], p)
    for _ in range(2): phased()
    print(spec, "K1 phased (one stream) ms", ev_time(phased))
    z = torch.empty(sh.num_tokens, dtype=torch.int16).pin_memory().numpy().view(np.uint16)
    z[:] = sh.get_assignments()
    def imp():
        sh.copy_assignments_async(z, 0, len(z), True); sh.assignments_imported()
    print(spec, "staged import (unchanged) ms", ev_time(imp))
    def counts():
        sh.rebuild_phi(); sh.prepare(); sh.rebuild_theta()
    print(spec, "counts serial ms", ev_time(counts))
    t0 = time.perf_counter(); ll = sh.loglik_sum(); print(spec, "loglik D2H ms", 1e3 * (time.perf_counter() - t0))
    sh.close()
