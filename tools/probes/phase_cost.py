"""Device-resident step (K1 + counts) with K1 unphased vs in word phases on two
alternating streams (the e2e schedule, no copies): python tools/probes/phase_cost.py nytimes geo:9"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_1803_04631_b200 import synth
from paper_1803_04631_b200.shard import DeviceShard
wl = sys.argv[1] if len(sys.argv) > 1 else "nytimes"
specs = sys.argv[2:] or ["geo:9"]
K = 1024
shape = bench.SHAPES[wl]
corp = synth.generate(shape["num_docs"], shape["vocab_size"], shape["mean_len"], seed=bench.CORPUS_SEED)
freq = np.bincount(corp.word_ids, minlength=corp.vocab_size).astype(np.int64)
st = torch.cuda.current_stream()
side, alt = torch.cuda.Stream(), torch.cuda.Stream()
def make(phases):
    sh = DeviceShard(K, corp.vocab_size, 50.0 / K, 0.01, seed=42, global_word_freq=freq, stream=st, phases=phases)
    sh.load_tokens(0, corp.num_docs, corp.doc_ids, corp.word_ids, seed=42)
    sh.initialize()
    return sh
def counts(sh):
    k = st.record_event(); side.wait_event(k)
    sh.set_stream(side); sh.rebuild_theta(); sh.set_stream(st)
    sh.rebuild_phi(); sh.prepare(); st.wait_stream(side)
def step_phased(sh, it, P):
    ready = st.record_event(); alt.wait_event(ready)
    done = [None, None]
    for p in range(P):
        ps = st if p % 2 == 0 else alt
        if p == P - 1 and done[1 - p % 2] is not None: ps.wait_event(done[1 - p % 2])
        sh.set_stream(ps); sh.sample_phase(it, p); done[p % 2] = ps.record_event()
    sh.set_stream(st); st.wait_stream(alt); counts(sh)
def timeit(fn, n=10):
    for i in range(3): fn(100 + i)
    torch.cuda.synchronize(); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for i in range(n): fn(200 + i)
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
sh = make(1)
print(wl, "unphased step ms", round(timeit(lambda it: (sh.sample(it), counts(sh))), 3))
sh.close()
for spec in specs:
    if spec.startswith("geo:"):
        n = int(spec[4:]); cuts = [1.0 - 0.5 ** (p + 1) for p in range(n - 1)] + [1.0]
    else:
        r, n = float(spec[1:].split(":")[0]), int(spec.split(":")[1]); cuts = [1.0 - r ** (p + 1) for p in range(n - 1)] + [1.0]
    sh = make(cuts); P = sh.num_phases
    print(wl, spec, "phased step ms", round(timeit(lambda it: step_phased(sh, it, P)), 3))
    sh.close()
