"""PCIe microbenchmark (GPU box): pinned H2D, D2H, both directions at once and
the chunked D2H->H2D round trip bench.py's e2e leg uses, for a 199 MB buffer."""
import torch, time
n = 199 * 1024 * 1024 // 2
h1 = torch.empty(n, dtype=torch.int16).pin_memory(); h2 = torch.empty(n, dtype=torch.int16).pin_memory()
d1 = torch.empty(n, dtype=torch.int16, device="cuda"); d2 = torch.empty(n, dtype=torch.int16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
def chunked(nc=16):
    c = n // nc
    for i in range(nc):
        with torch.cuda.stream(s2): h2[i*c:(i+1)*c].copy_(d2[i*c:(i+1)*c], non_blocking=True)
        e = s2.record_event()
        s1.wait_event(e)
        with torch.cuda.stream(s1): d1[i*c:(i+1)*c].copy_(h2[i*c:(i+1)*c], non_blocking=True)
for name, f in [("h2d", h2d), ("d2h", d2h), ("both", both), ("chunked roundtrip", chunked)]:
    ms = t(f); print(f"{name}: {ms:.2f} ms  ({2*n/ms/1e6:.1f} GB/s per direction)")
