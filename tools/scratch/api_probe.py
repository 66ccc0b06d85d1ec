import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1803_04631_b200 import corpus as cp, synth, model as md
from paper_1803_04631_b200.shard import DeviceShard
def t(f, n=3):
    ts=[]
    for _ in range(n):
        torch.cuda.synchronize(); t0=time.perf_counter(); r=f(); torch.cuda.synchronize(); ts.append(time.perf_counter()-t0)
    return min(ts)*1e3, r
N=200*2**20
h=np.ones(N, np.uint8); d=torch.empty(N, dtype=torch.uint8, device='cuda'); p=torch.empty(N, dtype=torch.uint8).pin_memory()
print("pageable H2D GB/s", N/t(lambda: d.copy_(torch.from_numpy(h)))[0]/1e6)
print("pinned H2D GB/s", N/t(lambda: d.copy_(p, non_blocking=True))[0]/1e6)
print("pageable D2H GB/s", N/t(lambda: torch.from_numpy(h).copy_(d))[0]/1e6)
print("pinned D2H GB/s", N/t(lambda: p.copy_(d, non_blocking=True))[0]/1e6)
print("host memcpy GB/s", N/t(lambda: np.copyto(h, p.numpy()))[0]/1e6)
K=1024
corp=synth.shaped("nytimes"); ch=cp.partition(corp,1,K,42,device=0)[0]
sh=DeviceShard(K, corp.vocab_size, 50/K, 0.01, seed=42).load(ch); sh.initialize()
ms,th=t(sh.get_theta); print("get_theta ms", ms, "nnz", len(th[1]))
print("set_theta ms", t(lambda: sh.set_theta(*th))[0])
ms,ph=t(lambda: sh.get_phi(16)); print("get_phi16 ms", ms)
print("set_phi16 ms", t(lambda: sh.set_phi(ph[0], ph[1]))[0])
ms,ph32=t(lambda: sh.get_phi(32)); print("get_phi32 ms", ms)
print("set_phi32 ms", t(lambda: sh.set_phi(ph32[0], ph32[1]))[0])
ms,z=t(sh.get_assignments); print("get_z ms", ms)
print("set_z ms", t(lambda: sh.set_assignments(z))[0])
print("stage_z ms", t(lambda: (sh.copy_assignments_async(z,0,len(z),True), sh.assignments_imported()))[0])
print("rebuild_theta ms", t(sh.rebuild_theta)[0], "rebuild_phi ms", t(sh.rebuild_phi)[0])
print("prepare+sample ms", t(lambda: (sh.prepare(), sh.sample(3)))[0])
