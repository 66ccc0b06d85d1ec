"""Instrumented copy of bench.py's e2e loop (PubMed-shape, geo:9 phases):
CUDA events per segment to see where the e2e step loses time against the
device-resident step."""
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
device = 0
stream = torch.cuda.current_stream()
side = torch.cuda.Stream()
n = int(os.environ.get("PH", "9"))
cuts = [1.0 - 0.5 ** (p + 1) for p in range(n - 1)] + [1.0]
DOC = os.environ.get("ORDER", "word") == "doc"
sh = DeviceShard(K, corp.vocab_size, 50.0 / K, 0.01, seed=42, global_word_freq=freq, stream=stream,
                 phases=1 if DOC else cuts)
if DOC:
    sh.set_block_phases(cuts)
sh.load_tokens(0, corp.num_docs, corp.doc_ids, corp.word_ids, seed=42)
sh.initialize()
T_local = sh.num_tokens
z_in = torch.empty(T_local, dtype=torch.int16).pin_memory().numpy().view(np.uint16)
z_io = torch.empty(T_local, dtype=torch.int16).pin_memory().numpy().view(np.uint16)
copy = sh.copy_doc_assignments_async if DOC else sh.copy_assignments_async
imported = sh.doc_assignments_imported if DOC else sh.assignments_imported
if DOC:
    copy(z_in, 0, sh.num_tokens, False); sh.synchronize()
else:
    z_in[:] = sh.get_assignments()
nphase = sh.num_phases
ranges = [sh.phase_doc_range(p) if DOC else sh.phase_range(p) for p in range(nphase)]
print("ranges", [(b - a) / sh.num_tokens for a, b in ranges])
nchunk = max(nphase, 16)
target = max(1, T_local // nchunk)
pieces = []
for a0, b0 in ranges:
    per = max(1, int(round((b0 - a0) / target)))
    cut = np.linspace(a0, b0, per + 1).astype(np.int64)
    pieces.append([(int(x), int(y)) for x, y in zip(cut[:-1], cut[1:]) if y > x])
d2h_s, h2d_s, alt = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def upload(host):
    for ps in pieces:
        for x, y in ps:
            copy(host, x, y - x, True, h2d_s)
    return h2d_s.record_event()
def counts_from_z():
    k = stream.record_event(); side.wait_event(k)
    sh.set_stream(side); sh.rebuild_theta(); sh.set_stream(stream)
    sh.rebuild_phi(); sh.prepare(); stream.wait_stream(side)
E = lambda: torch.cuda.Event(enable_timing=True)
copy(z_in, 0, 1, True, h2d_s)
torch.cuda.synchronize()
steps = 8
it = 10
marks = []
t0 = time.perf_counter()
ev_in = upload(z_in)
for i in range(steps):
    m = {k: E() for k in ("start", "in_ready", "imported", "counts", "k1_end", "out_end")}
    m["start"].record(stream)
    stream.wait_event(ev_in)
    m["in_ready"].record(stream)
    imported()
    m["imported"].record(stream)
    counts_from_z()
    m["counts"].record(stream)
    last = i + 1 == steps
    ready = stream.record_event(); alt.wait_event(ready)
    done = [None, None]
    for p in range(nphase):
        ps = stream if p % 2 == 0 else alt
        if p == nphase - 1 and done[1 - p % 2] is not None: ps.wait_event(done[1 - p % 2])
        sh.set_stream(ps); sh.sample_phase(it, p); done[p % 2] = ps.record_event()
        pe = E(); pe.record(ps); m.setdefault("ph", []).append(pe)
        if DOC and p == 0: continue
        d2h_s.wait_event(done[p % 2])
        if DOC: d2h_s.wait_event(done[0])
        for x, y in pieces[p]:
            copy(z_io, x, y - x, False, d2h_s)
            if not last:
                h2d_s.wait_event(d2h_s.record_event())
                copy(z_io, x, y - x, True, h2d_s)
    sh.set_stream(stream); stream.wait_stream(alt)
    m["k1_end"].record(stream)
    it += 1
    ev_in = h2d_s.record_event()
    th = time.perf_counter()
    lls = sh.loglik_sum()
    m["host_wait_ms"] = 1e3 * (time.perf_counter() - th)
    m["out_end"].record(d2h_s)
    marks.append(m)
torch.cuda.synchronize()
el = time.perf_counter() - t0
print(f"phases {nphase}: e2e {T_local * steps / el / 1e9:.3f} G tokens/s, {1e3 * el / steps:.2f} ms/step (wall)")
for i, m in enumerate(marks):
    seg = lambda a, b: m[a].elapsed_time(m[b])
    nxt = marks[i + 1]["start"] if i + 1 < len(marks) else None
    gap = m["k1_end"].elapsed_time(nxt) if nxt else float("nan")
    if i == len(marks) - 1:
        print("phase ends (ms after counts):", [round(m["counts"].elapsed_time(e), 2) for e in m["ph"]])
    print(f"step {i}: wait-input {seg('start','in_ready'):6.2f} import {seg('in_ready','imported'):5.2f} counts {seg('imported','counts'):5.2f} "
          f"K1 phases {seg('counts','k1_end'):6.2f} | gap to next step {gap:6.2f} | host loglik wait {m['host_wait_ms']:6.2f}")
