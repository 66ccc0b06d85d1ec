"""Log-likelihood vs time at scale (BASELINE metric "log-likelihood vs time";
north star: "per-token log-likelihood must stay within 1% of the reference's
trajectory at matched iterations").

GPU: the device trainer on one shard, `--gpu-iters` deferred iterations; the
loglik of each iteration's starting model is fused into K1, time is the
cumulative CUDA-event time of the iterations.
CPU: the oracle (oracle/, the SPEC sampler in its thin form + the reference
rebuilds, OpenMP C on all host cores) from the same chunk and seed for
`--cpu-iters` iterations; its loglik is the O(T K_d) S + Q form of SPEC.md:405.

    python tools/trajectory.py [--workload nytimes] [--gpu-iters 100] [--cpu-iters 12]

Writes profiles/<tag>_loglik_<workload>.csv and .json.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="nytimes")
    ap.add_argument("--topics", type=int, default=1024)
    ap.add_argument("--gpu-iters", type=int, default=100)
    ap.add_argument("--cpu-iters", type=int, default=12)
    ap.add_argument("--seed", type=int, default=20261017)
    ap.add_argument("--tag", default="r1d")
    ap.add_argument("--out-dir", default="profiles")
    args = ap.parse_args()

    import torch

    import oracle
    from paper_1803_04631_b200 import corpus as cp
    from paper_1803_04631_b200 import synth
    from paper_1803_04631_b200.shard import DeviceShard

    K = args.topics
    a, b = 50.0 / K, 0.01
    corp = synth.shaped(args.workload, seed=args.seed)
    ch = cp.partition(corp, 1, K, args.seed)[0]
    T = corp.num_tokens

    # ---- GPU ----
    st = torch.cuda.current_stream()
    sh = DeviceShard(K, corp.vocab_size, a, b, seed=42, stream=st).load(ch)   # events bracket its kernels
    sh.initialize()
    gpu_ll, gpu_t = [], []
    acc = 0.0
    for it in range(args.gpu_iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        sh.sample(it)
        sh.rebuild_phi()
        sh.prepare()
        sh.rebuild_theta()
        e1.record(st)
        torch.cuda.synchronize()
        acc += e0.elapsed_time(e1) / 1e3
        gpu_ll.append(sh.loglik_sum() / T)
        gpu_t.append(acc)
    sh.check_errors()
    sh.close()

    # ---- CPU oracle (same chunk, same Philox stream) ----
    threads = os.cpu_count() or 1
    z = ch.assignments.copy()
    cpu_ll, cpu_t = [], []
    acc = 0.0
    for it in range(args.cpu_iters):
        t0 = time.perf_counter()
        rp, ids, cn = oracle.rebuild_theta(z, ch.dw_ptr, ch.dw_tok, 0, K)
        phi, tot = oracle.rebuild_phi(z, ch.word_ids, K, corp.vocab_size)
        phi = phi.astype(np.uint32)
        t_sample = time.perf_counter()
        z = oracle.sample_tokens(K, corp.vocab_size, a, b, 42, it, ch.doc_ids, ch.word_ids, z, 0, rp, ids, cn,
                                 phi, tot, nthreads=threads)
        acc += time.perf_counter() - t0                  # rebuild + sample (the iteration)
        cpu_t.append(acc)
        cpu_ll.append(oracle.loglik_sq(K, corp.vocab_size, a, b, ch.doc_ids, ch.word_ids, 0, rp, ids, cn,
                                       corp.doc_lengths, phi, tot, nthreads=threads))   # (not timed)
        print(f"cpu it {it}: loglik {cpu_ll[-1]:.6f} gpu {gpu_ll[it]:.6f} ({time.perf_counter() - t_sample:.1f} s)",
              flush=True)

    n = min(len(cpu_ll), len(gpu_ll))
    rel = [abs(gpu_ll[i] - cpu_ll[i]) / abs(cpu_ll[i]) for i in range(n)]
    out = os.path.join(ROOT, args.out_dir, f"{args.tag}_loglik_{args.workload}")
    with open(out + ".csv", "w") as fh:
        fh.write("iteration,gpu_elapsed_s,gpu_loglik_per_token,cpu_elapsed_s,cpu_loglik_per_token\n")
        for i in range(len(gpu_ll)):
            c = (f"{cpu_t[i]:.3f},{cpu_ll[i]:.8f}" if i < len(cpu_ll) else ",")
            fh.write(f"{i},{gpu_t[i]:.6f},{gpu_ll[i]:.8f},{c}\n")
    summary = {"workload": args.workload, "topics": K, "tokens": T, "gpu_iterations": len(gpu_ll),
               "cpu_iterations": len(cpu_ll), "cpu_threads": threads,
               "max_rel_diff_matched": max(rel) if rel else None, "rel_diff_matched": rel,
               "gpu_first_100_avg_tokens_per_s": T * len(gpu_ll) / gpu_t[-1],
               "cpu_tokens_per_s": T * len(cpu_ll) / cpu_t[-1] if cpu_t else None,
               "gpu_loglik_first_last": [gpu_ll[0], gpu_ll[-1]],
               "note": "loglik of each iteration's starting model; GPU time = CUDA events of the iterations, "
                       "CPU time = wall time of rebuild + sample (oracle, OpenMP C)"}
    with open(out + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "rel_diff_matched"}))


if __name__ == "__main__":
    main()
