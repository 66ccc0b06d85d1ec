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
    ap.add_argument("--cpu-seeds", default="42",
                    help="comma-separated Philox keys of the oracle chains (42 = the device's own uniforms; "
                         "others give independent chains from the same initial state)")
    ap.add_argument("--cpu-mode", default="direct", choices=["direct", "thin"])
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

    # ---- CPU oracle chains (same chunk and initial state; Philox key per chain) ----
    threads = os.cpu_count() or 1
    seeds = [int(x) for x in args.cpu_seeds.split(",") if x]
    chains = {}
    for seed in seeds:
        z = ch.assignments.copy()
        cpu_ll, cpu_t = [], []
        acc = 0.0
        for it in range(args.cpu_iters):
            t0 = time.perf_counter()
            rp, ids, cn = oracle.rebuild_theta(z, ch.dw_ptr, ch.dw_tok, 0, K)
            phi, tot = oracle.rebuild_phi(z, ch.word_ids, K, corp.vocab_size)
            phi = phi.astype(np.uint32)
            t_sample = time.perf_counter()
            z = oracle.sample_tokens(K, corp.vocab_size, a, b, seed, it, ch.doc_ids, ch.word_ids, z, 0, rp, ids,
                                     cn, phi, tot, nthreads=threads, mode=args.cpu_mode)
            acc += time.perf_counter() - t0              # rebuild + sample (the iteration)
            cpu_t.append(acc)
            cpu_ll.append(oracle.loglik_sq(K, corp.vocab_size, a, b, ch.doc_ids, ch.word_ids, 0, rp, ids, cn,
                                           corp.doc_lengths, phi, tot, nthreads=threads))   # (not timed)
            print(f"seed {seed} it {it}: loglik {cpu_ll[-1]:.6f} gpu {gpu_ll[it]:.6f} "
                  f"({time.perf_counter() - t_sample:.1f} s)", flush=True)
        chains[seed] = (cpu_ll, cpu_t)

    n = min(min(len(c[0]) for c in chains.values()), len(gpu_ll))
    band = np.array([chains[s_][0][:n] for s_ in seeds])
    lo, hi = band.min(axis=0), band.max(axis=0)
    g = np.array(gpu_ll[:n])
    outside = np.maximum(lo - g, 0) + np.maximum(g - hi, 0)
    rel_band = outside / np.abs(np.where(g < lo, lo, hi))
    rel_first = [abs(gpu_ll[i] - band[0][i]) / abs(band[0][i]) for i in range(n)]
    out = os.path.join(ROOT, args.out_dir, f"{args.tag}_loglik_{args.workload}")
    with open(out + ".csv", "w") as fh:
        fh.write("iteration,gpu_elapsed_s,gpu_loglik_per_token," +
                 ",".join(f"cpu{s_}_elapsed_s,cpu{s_}_loglik_per_token" for s_ in seeds) + "\n")
        for i in range(len(gpu_ll)):
            cols = [f"{chains[s_][1][i]:.3f},{chains[s_][0][i]:.8f}" if i < len(chains[s_][0]) else ","
                    for s_ in seeds]
            fh.write(f"{i},{gpu_t[i]:.6f},{gpu_ll[i]:.8f}," + ",".join(cols) + "\n")
    cpu_t0 = chains[seeds[0]][1]
    summary = {"workload": args.workload, "topics": K, "tokens": T, "gpu_iterations": len(gpu_ll),
               "cpu_iterations": n, "cpu_threads": threads, "cpu_mode": args.cpu_mode, "cpu_seeds": seeds,
               "gpu_seed": 42,
               "max_rel_outside_seed_band": float(rel_band.max()) if n else None,
               "rel_outside_seed_band": rel_band.tolist(),
               "band_width_rel_last": float((hi[-1] - lo[-1]) / abs(lo[-1])) if n else None,
               "max_rel_diff_vs_first_chain": max(rel_first) if rel_first else None,
               "gpu_first_100_avg_tokens_per_s": T * len(gpu_ll) / gpu_t[-1],
               "cpu_tokens_per_s": T * len(cpu_t0) / cpu_t0[-1] if cpu_t0 else None,
               "gpu_loglik_first_last": [gpu_ll[0], gpu_ll[-1]],
               "note": "loglik of each iteration's starting model; GPU time = CUDA events of the iterations, "
                       "CPU time = wall time of rebuild + sample (oracle, OpenMP C); the band = min/max over the "
                       "oracle chains at each matched iteration (0 when the GPU lies inside it)"}
    with open(out + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k not in ("rel_outside_seed_band",)}))


if __name__ == "__main__":
    main()
