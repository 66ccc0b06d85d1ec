"""Where the e2e step loses time (GPU box): the bench step with K1 unphased,
K1 in geo:N phases on two alternating streams (the e2e schedule, no copies),
and the phased step plus the staged import of an unchanged z (H2D + diff)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_1803_04631_b200 import synth
from paper_1803_04631_b200.shard import DeviceShard
K = 1024
shape = bench.SHAPES["pubmed"]
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
def step_unphased(sh, it):
    sh.sample(it); counts(sh)
def step_phased(sh, it, P):
    ready = st.record_event(); alt.wait_event(ready)
    done = [None, None]
    for p in range(P):
        ps = st if p % 2 == 0 else alt
        if p == P - 1 and done[1 - p % 2] is not None: ps.wait_event(done[1 - p % 2])
        sh.set_stream(ps); sh.sample_phase(it, p); done[p % 2] = ps.record_event()
    sh.set_stream(st); st.wait_stream(alt); counts(sh)
def timeit(fn, n=8):
    for i in range(3): fn(100 + i)
    torch.cuda.synchronize(); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for i in range(n): fn(200 + i)
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
sh = make(1)
print("unphased step ms", timeit(lambda it: step_unphased(sh, it)))
sh.close()
for n in (9, 12):
    cuts = [1.0 - 0.5 ** (p + 1) for p in range(n - 1)] + [1.0]
    sh = make(cuts); P = sh.num_phases
    print(f"geo:{n} phased step ms", timeit(lambda it: step_phased(sh, it, P)))
    z = torch.empty(sh.num_tokens, dtype=torch.int16).pin_memory().numpy().view(np.uint16); z[:] = sh.get_assignments()
    def with_import(it):
        sh.copy_assignments_async(z, 0, len(z), True); sh.assignments_imported(); step_phased(sh, it, P)
    print(f"geo:{n} phased step + import ms", timeit(with_import))
    sh.close()
