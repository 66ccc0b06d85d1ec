"""K1 time under phase-major schedules (GPU box): one launch vs P sample_phase
launches for P in (1, 16) on WL=nytimes|pubmed, from the state after 3 iterations."""
import time, sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_1803_04631_b200 import synth, corpus as cp
from paper_1803_04631_b200.shard import DeviceShard
import os
corp = synth.shaped(os.environ.get("WL", "nytimes"), seed=20261017)
K = 1024
st = torch.cuda.current_stream()
z = None
for P in (1, 16):
    sh = DeviceShard(K, corp.vocab_size, 50.0 / K, 0.01, seed=42, stream=st, phases=P)
    sh.load_tokens(0, corp.num_docs, corp.doc_ids, corp.word_ids, seed=20261017, chunk_id=0)
    if z is None:
        sh.initialize()
        for it in range(3):
            sh.iterate(it)
        z = sh.get_assignments()
    sh.set_assignments(z); sh.initialize()
    for mode in ("one", "phases"):
        ts = []
        for rep in range(4):
            sh.set_assignments(z); sh.initialize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            if mode == "one": sh.sample(3)
            else:
                for p in range(P): sh.sample_phase(3, p)
            e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        print(f"P={P} {mode}: K1 {np.median(ts[1:]):.3f} ms  ranges={[sh.phase_range(p) for p in range(P)][:3]}")
    sh.close()
