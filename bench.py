"""Benchmark: sampled tokens/s of the B200 CuLDA_CGS hot path (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload pubmed|nytimes|z4shard|tiny] [--topics 1024]
                    [--scaling strong|weak] [--shard r/N]

A step is one full deferred training iteration (K1 sample + fused loglik, K2
phi rebuild, [phi allreduce], K3 theta rebuild, prepare) with every input
resident in HBM.  The default workload is the north star's headline: the
PubMed-shaped corpus (BASELINE.json configs[2]: 8.2M docs, V=141,043,
~738M tokens) at K=1024.  Under torchrun the SAME corpus is split over the N
ranks ("strong" scaling): rank r owns documents greedy_boundaries(doc
lengths, N)[r] (corpus.py:210-237, C = G) and generates only those, and the
phi replicas are summed with NCCL every iteration.  `--scaling weak` gives
every rank its own full-size corpus instead (z4shard is always weak: it is
one GPU's share of BASELINE configs[4]).

`--shard r/N` runs ONE rank's shard of an N-way split on one GPU (full
vocabulary, no collective): the per-rank step time of the N-GPU run, minus the
allreduce, measured on a single GPU.

`--impl reference` times the CPU implementation of the same path on the host
cores.  The reference package has no sampler, so each step is one deferred
iteration of the oracle port (oracle/: the SPEC sampler + rebuild_theta +
rebuild_phi, OpenMP C, all threads) over a bounded document sample of the
same corpus, which it generates with oracle/gf_synth_ref.c (identical to the
product generator, no product library) and partitions with the reference
package's own `partition` (baseline/_ref) when it is installed.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sampled tokens/sec"
UNIT = "tokens/s"

# BASELINE.json config shapes: docs, vocabulary, mean length
SHAPES = {
    "tiny": dict(num_docs=1_000, vocab_size=1_000, mean_len=100.0),
    "nytimes": dict(num_docs=299_752, vocab_size=101_636, mean_len=332.08),
    "pubmed": dict(num_docs=8_200_000, vocab_size=141_043, mean_len=89.98),
    "z4shard": dict(num_docs=5_000_000, vocab_size=1_000_000, mean_len=100.0),
}
CORPUS_SEED = 20261017
TRAIN_SEED = 42
# documents in the bounded CPU sample (about 9M tokens PubMed-shape, 6.6M NYTimes-shape)
CPU_SAMPLE_DOCS = {"tiny": 1_000, "nytimes": 20_000, "pubmed": 100_000, "z4shard": 100_000}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="pubmed", choices=sorted(SHAPES))
    ap.add_argument("--topics", type=int, default=None)
    ap.add_argument("--seed", type=int, default=CORPUS_SEED)
    ap.add_argument("--scaling", default=None, choices=["strong", "weak"],
                    help="N>1: split one corpus over the ranks (strong, default) or one corpus per rank (weak)")
    ap.add_argument("--shard", default=None, help="r/N: run rank r's shard of an N-way split on one GPU")
    ap.add_argument("--cpu-sample-docs", type=int, default=0, help="docs in the bounded CPU sample (0: auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--phi-sync", default="nccl", choices=["nccl", "peer"],
                    help="N>1: phi sum by all_reduce, or by the IPC peer-memory exchange kernel")
    a = ap.parse_args()
    if a.scaling is None:
        a.scaling = "weak" if a.workload == "z4shard" else "strong"
    return a


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def topics_of(args):
    return args.topics or (32 if args.workload == "tiny" else 1024)


def split_of(args, world, rank):
    """(parts, part): which greedy_boundaries split this process runs."""
    if args.shard:
        r, n = (int(x) for x in args.shard.split("/"))
        if not 0 <= r < n:
            raise SystemExit(f"--shard {args.shard}: need 0 <= r < N")
        return n, r
    if args.scaling == "strong":
        return world, rank
    return 1, 0


def make_config(args, world, tokens_total):
    """The `config` object: identical for both arms of the same command."""
    shape = SHAPES[args.workload]
    parts, part = split_of(args, world, 0)
    docs_total = shape["num_docs"] * (world if args.scaling == "weak" and not args.shard else 1)
    c = {
        "workload": f"{args.workload}-shaped synthetic LDA corpus, K={topics_of(args)}",
        "docs_total": docs_total, "vocab": shape["vocab_size"], "tokens_total": int(tokens_total),
        "topics": topics_of(args), "alpha": 50.0 / topics_of(args), "beta": 0.01,
        "iterations": [args.warmup, args.warmup + args.steps],
        "scaling": "shard-proxy" if args.shard else args.scaling,
        "parallelism": (f"rank {args.shard} of a doc-sharded dp{parts} (one GPU, no collective)" if args.shard else
                        (f"doc-shard dp{world} (greedy_boundaries) + phi allreduce" if world > 1 else "dp1")),
        "l2": "inputs larger than L2 (z 2T B, theta 4*NNZ B, phi >= 200 MB vs 126 MB L2)",
        "corpus_seed": args.seed, "train_seed": TRAIN_SEED,
    }
    return c


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region: NVML every
    ~2 ms (initialised up front, plus one sample at entry and exit so even a
    short region has readings; nvidia-smi as a fallback)."""

    def __init__(self, device):
        self.device = device
        self.rows = []                       # (sm_mhz, sm_max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._t = None
        self._nv = None
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            self._nv = lambda: (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), mx, reasons(h))
        except Exception:
            self._nv = None

    def _sample(self):
        if self._nv is not None:
            try:
                self.rows.append(self._nv())
            except Exception:
                pass
            return
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
        try:
            out = subprocess.run(["nvidia-smi", f"--id={self.device}", f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
            a, b, c = [x.strip() for x in out.stdout.strip().split(",")]
            self.rows.append((float(a), float(b), int(c, 16)))
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.002 if self._nv is not None else 0.1)

    def __enter__(self):
        self._sample()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        self._sample()

    # NVML clocks-event reason bits
    BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
            0x80: "hw_power_brake_slowdown"}

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for r in self.rows for bit, n in self.BITS.items() if r[2] & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(r[1] for r in self.rows)),
                "reasons": reasons, "samples": len(self.rows)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload, K):
    """DRAM read+write bytes per K1 launch from the committed `ncu --set full`
    capture of the same workload and K (None when there is none).  ncu cannot
    run inside the timed region, so this is a labelled lookup: the entry names
    its capture file and the iteration it profiled."""
    p = os.path.join(ROOT, "profiles", "sample_kernel_traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh).get(f"{workload}-{K}")
    except Exception:
        return None


# -------------------------------------------------------------- CPU side --
def cpu_sample_state(args, K, ndocs):
    """The first `ndocs` documents of the benchmark corpus, generated by the
    oracle's generator (no product library) and partitioned by the reference
    package's own partition() when it is installed (baseline/_ref), else by
    the oracle's restatement of it; the initial counts by the oracle."""
    import oracle

    shape = SHAPES[args.workload]
    corp = oracle.synth_generate(ndocs, shape["vocab_size"], shape["mean_len"], seed=args.seed)
    part_by = "oracle.partition (restatement of corpus.py:240-287)"
    ref = os.path.join(ROOT, "baseline", "_ref")
    chunk = None
    if os.path.isdir(os.path.join(ref, "gibbsflow")):
        try:
            import tempfile

            os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="gf_numba_"))
            sys.path.insert(0, ref)
            try:
                from gibbsflow import corpus as rc
            finally:
                sys.path.remove(ref)
            rcorp = rc.corpus_from_tokens(corp["doc_ids"], corp["word_ids"], corp["V"])
            c = rc.partition(rcorp, 1, K, TRAIN_SEED)[0]
            chunk = dict(doc_ids=c.doc_ids, word_ids=c.word_ids, assignments=c.assignments, dw_ptr=c.dw_ptr,
                         dw_tok=c.dw_tok)
            part_by = "gibbsflow.corpus.partition (the reference package, baseline/_ref)"
        except Exception as e:                                # noqa: BLE001 -- fall back to the restatement
            part_by = f"oracle.partition (reference package failed: {type(e).__name__})"
            chunk = None
    if chunk is None:
        chunk = oracle.partition(corp, 1, K, TRAIN_SEED)[0]
    z = np.ascontiguousarray(chunk["assignments"], dtype=np.uint16).copy()
    st = {"V": corp["V"], "T": corp["T"], "doc_ids": np.ascontiguousarray(chunk["doc_ids"], np.int32),
          "word_ids": np.ascontiguousarray(chunk["word_ids"], np.int32), "z": z,
          "dw_ptr": np.ascontiguousarray(chunk["dw_ptr"], np.int64),
          "dw_tok": np.ascontiguousarray(chunk["dw_tok"], np.int64), "partitioned_by": part_by}
    st["theta"] = oracle.rebuild_theta(z, st["dw_ptr"], st["dw_tok"], 0, K)
    phi, tot = oracle.rebuild_phi(z, st["word_ids"], K, st["V"])
    st["phi"] = (phi.astype(np.uint32), tot)
    return st


def cpu_iteration(st, K, iteration, threads):
    """One deferred iteration of the oracle port on the sample: sample (SPEC
    sampler, OpenMP) + theta rebuild + phi rebuild.  Returns seconds."""
    import oracle

    a, b = 50.0 / K, 0.01
    rp, ids, cn = st["theta"]
    phi, tot = st["phi"]
    t0 = time.perf_counter()
    z = oracle.sample_tokens(K, st["V"], a, b, TRAIN_SEED, iteration, st["doc_ids"], st["word_ids"], st["z"], 0,
                             rp, ids, cn, phi, tot, nthreads=threads)
    theta = oracle.rebuild_theta(z, st["dw_ptr"], st["dw_tok"], 0, K)
    phi2, tot2 = oracle.rebuild_phi(z, st["word_ids"], K, st["V"])
    dt = time.perf_counter() - t0
    st["z"], st["theta"], st["phi"] = z, theta, (phi2.astype(np.uint32), tot2)
    return dt


def cpu_sample_text(args, st, ndocs, threads):
    shape = SHAPES[args.workload]
    return (f"the first {ndocs} of the {shape['num_docs']} documents ({st['T']} tokens) of the same corpus, "
            f"K={topics_of(args)}; step = one deferred iteration (SPEC sampler + rebuild_theta + rebuild_phi) of "
            f"the oracle port (oracle/gf_oracle.c, OpenMP C, {threads} threads; the reference package has no "
            f"sampler); chunk from {st['partitioned_by']}")


def cpu_baseline(args, K, ndocs, iters=2):
    threads = os.cpu_count() or 1
    st = cpu_sample_state(args, K, ndocs)
    times = [cpu_iteration(st, K, it, threads) for it in range(iters)]
    return {"value": st["T"] / float(np.mean(times)), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": cpu_sample_text(args, st, ndocs, threads) + f"; mean of {iters} iterations"}


def reference_components(args, K, ndocs):
    """Time the UNMODIFIED reference package (baseline/_ref/gibbsflow, installed
    offline from /root/reference/pkg) on a document sample: its own
    partition (corpus.py:240-287), rebuild_theta (model.py:109-124) and
    rebuild_phi_replica (model.py:142-161), single-threaded numpy/numba as
    shipped -- the CPU counterparts of K4, K3 and K2."""
    import tempfile

    import oracle

    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "gibbsflow")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="gf_numba_"))
    sys.path.insert(0, ref)
    try:
        from gibbsflow import corpus as rc
        from gibbsflow import model as rm
    finally:
        sys.path.remove(ref)
    shape = SHAPES[args.workload]
    corp = oracle.synth_generate(ndocs, shape["vocab_size"], shape["mean_len"], seed=args.seed)
    rcorp = rc.corpus_from_tokens(corp["doc_ids"], corp["word_ids"], corp["V"])
    T = int(rcorp.num_tokens)
    rc.partition(rcorp, 1, K, TRAIN_SEED)                      # numba JIT outside the timing
    out = {"sample": f"{ndocs} docs ({T} tokens), K={K}, reference package as installed (single thread)"}
    t0 = time.perf_counter()
    chunk = rc.partition(rcorp, 1, K, TRAIN_SEED)[0]
    out["partition_tokens_per_s"] = T / (time.perf_counter() - t0)
    t0 = time.perf_counter()
    rm.rebuild_theta(chunk, K)
    out["rebuild_theta_tokens_per_s"] = T / (time.perf_counter() - t0)
    t0 = time.perf_counter()
    rm.rebuild_phi_replica(chunk, K, corp["V"])
    out["rebuild_phi_tokens_per_s"] = T / (time.perf_counter() - t0)
    return out


def corpus_tokens_total(args, world):
    """Tokens one step processes over the whole job, from the document lengths
    alone (the oracle's generator: the reference arm loads no product code)."""
    import oracle

    shape = SHAPES[args.workload]
    D = shape["num_docs"]
    if args.shard:
        parts, part = split_of(args, world, 0)
        L = oracle.synth_lengths(args.seed, D, shape["mean_len"])
        lo, hi = oracle.greedy_boundaries(L, parts)[part]
        return int(L[lo:hi].sum())
    if args.scaling == "weak" and world > 1:
        return sum(int(oracle.synth_lengths(args.seed, D, shape["mean_len"], doc_begin=r * D).sum())
                   for r in range(world))
    return int(oracle.synth_lengths(args.seed, D, shape["mean_len"]).sum())


def run_reference(args, world, rank):
    if rank != 0:
        return
    K = topics_of(args)
    ndocs = args.cpu_sample_docs or min(CPU_SAMPLE_DOCS[args.workload], SHAPES[args.workload]["num_docs"])
    threads = os.cpu_count() or 1
    st = cpu_sample_state(args, K, ndocs)
    it = 0
    for _ in range(args.warmup):
        cpu_iteration(st, K, it, threads)
        it += 1
    times = []
    for _ in range(args.steps):
        times.append(cpu_iteration(st, K, it, threads))
        it += 1
    v = st["T"] / float(np.mean(times))
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True,
        "scaling": "shard-proxy" if args.shard else args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": make_config(args, world, corpus_tokens_total(args, world)),
        "impl": "reference",
        "sample": {"docs": ndocs, "tokens": st["T"]},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": cpu_sample_text(args, st, ndocs, threads)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_components": reference_components(args, K, min(ndocs, 5000)),
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours ----
def rank_corpus(args, world, rank):
    """(corpus of this rank's documents with doc ids relative to lo, lo, T of the
    whole run): strong scaling and --shard split the global corpus with
    greedy_boundaries; weak scaling gives each rank its own full-size corpus."""
    from paper_1803_04631_b200 import corpus as cp
    from paper_1803_04631_b200 import synth

    shape = SHAPES[args.workload]
    D = shape["num_docs"]
    parts, part = split_of(args, world, rank)
    if parts == 1:
        lo = rank * D if (args.scaling == "weak" and world > 1) else 0
        corp = synth.generate(D, shape["vocab_size"], shape["mean_len"], seed=args.seed, doc_begin=lo)
        return corp, lo
    L = synth.doc_lengths(args.seed, D, shape["mean_len"])
    lo, hi = cp.greedy_boundaries(L, parts)[part]
    corp = synth.generate(hi - lo, shape["vocab_size"], shape["mean_len"], seed=args.seed, doc_begin=lo)
    return corp, lo


def global_word_freq(args, world):
    """Word frequencies of the whole corpus for --shard (the N-GPU run allreduces
    the ranks' counts; one GPU recounts the corpus in pieces)."""
    from paper_1803_04631_b200 import synth

    shape = SHAPES[args.workload]
    freq = np.zeros(shape["vocab_size"], np.int64)
    step = 1_000_000
    for b in range(0, shape["num_docs"], step):
        c = synth.generate(min(step, shape["num_docs"] - b), shape["vocab_size"], shape["mean_len"], seed=args.seed,
                           doc_begin=b)
        freq += np.bincount(c.word_ids, minlength=shape["vocab_size"])
    return freq


def kernel_block(name, ms, nbytes, peak):
    gbs = nbytes / (ms / 1e3) / 1e9 if ms > 0 else 0.0
    return {"kernel": name, "ms": ms, "algorithmic_bytes": int(nbytes), "achieved_gbs": gbs, "frac": gbs / peak}


def run_ours(args, world, rank, local):
    import torch

    from paper_1803_04631_b200.shard import DeviceShard

    dist = None
    # one rank per GPU; --dist-backend gloo (with more ranks than GPUs) is the
    # single-GPU smoke test of the multi-rank path -- NCCL refuses two ranks on
    # one device
    device = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(device)
    # GF_FORCE_DIST=1: run the distributed code path even with one rank (a
    # one-rank NCCL group exercises the sync-buffer allreduce on one GPU)
    if world > 1 or os.environ.get("GF_FORCE_DIST") == "1":
        import torch.distributed as dist

        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{device}"))
        else:
            dist.init_process_group(args.dist_backend)

    def ar(t, op=None, async_op=False):
        """all_reduce; gloo gets a host copy of device tensors (smoke path)"""
        op = dist.ReduceOp.SUM if op is None else op
        if args.dist_backend == "gloo" and t.is_cuda:
            c = t.cpu()
            dist.all_reduce(c, op=op)
            t.copy_(c)
            return None
        return dist.all_reduce(t, op=op, async_op=async_op)

    K = topics_of(args)
    corp, lo = rank_corpus(args, world, rank)
    freq = np.bincount(corp.word_ids, minlength=corp.vocab_size).astype(np.int64)
    T_local = corp.num_tokens
    T_all = T_local
    if args.shard:
        freq = global_word_freq(args, world)
    if dist:
        t = torch.as_tensor(freq).cuda()
        ar(t)
        freq = t.cpu().numpy()
        tt = torch.tensor([T_local], dtype=torch.int64, device="cuda")
        ar(tt)
        T_all = int(tt.item())
    stream = torch.cuda.current_stream(device)
    sh = DeviceShard(K, corp.vocab_size, 50.0 / K, 0.01, seed=TRAIN_SEED, device=device, global_word_freq=freq,
                     stream=stream)
    chunk_id = int(args.shard.split("/")[0]) if args.shard else rank
    # K4: partition (stable word sort, dw-map, splitmix64 z0) + shard layout on
    # the device, from the doc-major tokens of this rank's documents.  A small
    # warm-up load first, so one-time CUDA costs (lazy module loading, first
    # allocations) stay out of the preprocessing throughput
    nw = min(corp.num_docs, 2000)
    tw = int(np.searchsorted(corp.doc_ids, nw))
    with DeviceShard(K, corp.vocab_size, 50.0 / K, 0.01, seed=TRAIN_SEED, device=device, global_word_freq=freq,
                     stream=stream) as warm:
        warm.load_tokens(lo, lo + nw, corp.doc_ids[:tw] + lo, corp.word_ids[:tw], seed=TRAIN_SEED, chunk_id=chunk_id)
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    sh.load_tokens(lo, lo + corp.num_docs, corp.doc_ids + lo, corp.word_ids, seed=TRAIN_SEED, chunk_id=chunk_id)
    torch.cuda.synchronize(device)
    prep_s = time.perf_counter() - t0
    sync_t = sh.sync_tensor() if dist else None
    peer = bool(dist) and args.phi_sync == "peer"
    if peer:          # map every rank's sync buffer; the phi sum becomes one kernel (k_peer.cu)
        handles = [None] * world
        dist.all_gather_object(handles, sh.peer_handle())
        sh.peer_open(rank, world, handles)

    def allreduce_async():
        if peer:
            sh.peer_allreduce()               # stream-ordered on the compute stream
            return None
        return ar(sync_t, async_op=True) if dist else None

    # initial counts
    sh.rebuild_phi()
    w = allreduce_async()
    if w:
        w.wait()
    sh.prepare()
    sh.rebuild_theta()
    sh.check_errors()

    # per step: [0] step start, [1] K1 end, [2] K2 end, [3] allreduce + prepare end,
    # [4] step end (main stream); K3's own start / end on the side stream
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(7)] for _ in range(args.steps)]

    side = torch.cuda.Stream(device)

    def step(it, ev=None):
        """K1, then K3 (theta from zdoc) on a side stream concurrently with K2
        (phi from z) + [allreduce] + prepare on the main stream; K3 and K2 are
        independent (different inputs and outputs), the next K1 waits for both."""
        if ev:
            ev[0].record(stream)
        sh.sample(it)
        k1 = stream.record_event()
        if ev:
            ev[1].record(stream)
        side.wait_event(k1)
        sh.set_stream(side)
        if ev:
            ev[5].record(side)
        sh.rebuild_theta()                    # K3, concurrent with K2 / allreduce / prepare
        if ev:
            ev[6].record(side)
        sh.set_stream(stream)
        sh.rebuild_phi()
        if ev:
            ev[2].record(stream)
        work = allreduce_async()
        if work:
            work.wait()
        sh.prepare()
        if ev:
            ev[3].record(stream)
        stream.wait_stream(side)
        if ev:
            ev[4].record(stream)

    it = 0
    for _ in range(args.warmup):
        step(it)
        it += 1
    sh.check_errors()
    sh.reset_stats()

    def barrier():
        torch.cuda.synchronize(device)
        if dist:
            dist.barrier()
            torch.cuda.synchronize(device)

    # the e2e leg below replays the SAME iterations from the same state (the
    # sampler gets faster as theta sparsifies, so later iterations would
    # flatter it): keep the state the timed region starts from
    it_start = it
    z_start = sh.get_assignments() if not args.no_e2e else None
    clocks = ClockSampler(device)
    barrier()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clocks:
        start.record(stream)
        for i in range(args.steps):
            step(it, evs[i])                  # per-kernel events on the launching streams
            it += 1
        stop.record(stream)
        barrier()
    acc = np.zeros(5)
    for ev in evs:
        acc += [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]),
                ev[3].elapsed_time(ev[4]), ev[5].elapsed_time(ev[6])]
    acc /= args.steps
    ms_total = start.elapsed_time(stop)
    if dist:
        t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
        ar(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    T_step = T_local if args.shard else T_all
    value = T_step / (ms_step / 1e3)
    ll = sh.loglik_sum()
    if dist:
        t = torch.tensor([ll], dtype=torch.float64, device="cuda")
        ar(t)
        ll = float(t.item())
    ll /= T_step
    sh.check_errors()
    st = sh.stats()
    # own kernels per step: sample + ll_reduce, phi_rebuild, theta_rebuild,
    # prepare (+ context_kernel when some word is split into several slices)
    launches_per_step = 5 + (1 if st["word_contexts"] > 0 else 0) + (1 if peer else 0)
    k1_ms = acc[0]
    peak, peak_src = measured_peak()
    achieved = st["sample_bytes"] / (k1_ms / 1e3) / 1e9
    traffic = ncu_traffic(args.workload, K)

    # ---- end to end through the public API with host buffers (pinned) ----
    e2e = None
    if not args.no_e2e:
        # one step from host state: H2D of the input assignments (pinned), the
        # counts of that state (K2 [+ allreduce] + prepare + K3: a rebuild from z
        # needs no consistency validation), K1, D2H of the new assignments and of
        # the loglik.  The copies go in chunks on two copy streams: chunk c of
        # the step's output is read back and, as soon as it lands, sent as chunk
        # c of the next step's input, so the two PCIe directions run concurrently.
        z_in = torch.empty(T_local, dtype=torch.int16).pin_memory().numpy().view(np.uint16)
        z_io = torch.empty(T_local, dtype=torch.int16).pin_memory().numpy().view(np.uint16)
        # streamed sampling: the schedule is split into phases, so phase p's
        # assignments travel back (and out again as the next step's input)
        # while phases p+1.. sample; only the last phase's round trip is
        # exposed.  Word-group phases (halving sizes) and the word-group (chunk)
        # order by default; GF_E2E_ORDER=doc: document-block phases and the
        # shard's document-major order (no theta row streamed twice, but phase
        # 0 -- the words not cut at block boundaries, ~46% of K1 on
        # PubMed-shape -- must finish before any document range is final, so
        # the round trip starts too late: measured 8.9 vs 11.1 G).  Reload the
        # same tokens with the phased schedule; the state carries over through
        # z (the counts are rebuilt from it every step).
        order = os.environ.get("GF_E2E_ORDER", "word")
        doc = order == "doc"
        # phase sizes (measured): PubMed-shape (1.48 GB of z per step) r0.45:8
        # 11.22 / geo:9 11.08 G; NYTimes-shape (199 MB) geo:9 8.65 / r0.45:8
        # 8.15 G -- large steps prefer fewer, faster-shrinking phases
        spec = os.environ.get("GF_E2E_PHASES", "r0.45:8" if T_local >= 300_000_000 else "geo:9")
        if spec.startswith("geo:"):       # halving phase sizes: 1/2, 1/4, ..., last two equal
            n = int(spec[4:])
            cuts = [1.0 - 0.5 ** (p + 1) for p in range(n - 1)] + [1.0]
        elif spec.startswith("r"):        # "r0.4:7": each phase `ratio` of the previous one, n phases
            ratio, n = float(spec[1:].split(":")[0]), int(spec.split(":")[1])
            cuts = [1.0 - ratio ** (p + 1) for p in range(n - 1)] + [1.0]
        else:
            n = int(spec)
            cuts = [(p + 1) / n for p in range(n)]
        cuts[-1] = 1.0
        z_now = z_start                          # the timed region's starting state ...
        it = it_start                            # ... and iterations
        if doc:
            sh.set_block_phases(cuts)
        elif n > 1:
            sh.set_phases(cuts)
        sh.load_tokens(lo, lo + corp.num_docs, corp.doc_ids + lo, corp.word_ids, seed=TRAIN_SEED, chunk_id=chunk_id)
        sh.set_assignments(z_now)
        if peer:
            handles = [None] * world
            dist.all_gather_object(handles, sh.peer_handle())
            sh.peer_open(rank, world, handles)
        sync_t = sh.sync_tensor() if dist else None
        copy = sh.copy_doc_assignments_async if doc else sh.copy_assignments_async
        imported = sh.doc_assignments_imported if doc else sh.assignments_imported
        if doc:
            copy(z_in, 0, T_local, False)
            sh.synchronize()
        else:
            z_in[:] = z_now
        nphase = sh.num_phases
        ranges = [sh.phase_doc_range(p) if doc else sh.phase_range(p) for p in range(nphase)]
        nchunk = max(nphase, int(os.environ.get("GF_E2E_CHUNKS", "16")))
        target = max(1, T_local // nchunk)          # pieces of ~T/nchunk tokens inside each phase
        pieces = []
        for a0, b0 in ranges:
            per = max(1, int(round((b0 - a0) / target)))
            cut = np.linspace(a0, b0, per + 1).astype(np.int64)
            pieces.append([(int(x), int(y)) for x, y in zip(cut[:-1], cut[1:]) if y > x])
        d2h_s, h2d_s, alt = torch.cuda.Stream(device), torch.cuda.Stream(device), torch.cuda.Stream(device)

        def upload(host):
            for ps in pieces:
                for x, y in ps:
                    copy(host, x, y - x, True, h2d_s)
            return h2d_s.record_event()

        def counts_from_z():
            # K3 (theta from zdoc) on the side stream beside K2 [+ allreduce] + prepare
            k = stream.record_event()
            side.wait_event(k)
            sh.set_stream(side)
            sh.rebuild_theta()
            sh.set_stream(stream)
            sh.rebuild_phi()
            w = allreduce_async()
            if w:
                w.wait()
            sh.prepare()
            stream.wait_stream(side)

        copy(z_in, 0, 1, True, h2d_s)            # allocates the import staging buffer
        # each step's loglik is read back (D2H) without blocking the host, so
        # the host never waits for a step before enqueueing the next one
        ll_host = torch.zeros(2 * args.steps, dtype=torch.float64).pin_memory().numpy()
        torch.cuda.synchronize(device)
        barrier()
        t0 = time.perf_counter()
        ev_in = upload(z_in)
        for i in range(args.steps):
            stream.wait_event(ev_in)
            imported()
            counts_from_z()
            last = i + 1 == args.steps
            ready = stream.record_event()
            alt.wait_event(ready)
            done = [None, None]
            for p in range(nphase):
                # phases alternate between two streams (they are independent), so a
                # phase's tail CTAs overlap the next phase's start; the last phase
                # (it also reduces the loglik) waits for the other stream
                ps = stream if p % 2 == 0 else alt
                if p == nphase - 1 and done[1 - p % 2] is not None:
                    ps.wait_event(done[1 - p % 2])
                sh.set_stream(ps)
                sh.sample_phase(it, p)
                done[p % 2] = ps.record_event()
                if doc and p == 0:
                    continue                  # document ranges are final from phase 1 on
                d2h_s.wait_event(done[p % 2])
                if doc:                       # ... and need phase 0 too (other stream)
                    d2h_s.wait_event(done[0])
                for x, y in pieces[p]:
                    copy(z_io, x, y - x, False, d2h_s)
                    if not last:             # out again as the next step's input once it landed
                        h2d_s.wait_event(d2h_s.record_event())
                        copy(z_io, x, y - x, True, h2d_s)
            sh.set_stream(stream)
            stream.wait_stream(alt)
            it += 1
            ev_in = h2d_s.record_event()
            sh.loglik_sum_async(ll_host[2 * i: 2 * i + 2], stream)   # D2H of the step's loglik
        torch.cuda.synchronize(device)
        barrier()
        el = time.perf_counter() - t0
        lls = ll_host[0::2] - ll_host[1::2]
        if not np.all(np.isfinite(lls)) or not np.all(lls < 0):
            raise RuntimeError(f"e2e step logliks not finite / negative: {lls}")
        if dist:
            t = torch.tensor([el], dtype=torch.float64, device="cuda")
            ar(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        fn = "copy_doc_assignments_async" if doc else "copy_assignments_async"
        e2e = {"value": T_step * args.steps / el, "unit": UNIT, "h2d_bytes_per_step": 2 * T_local,
               "d2h_bytes_per_step": 2 * T_local + 8,
               "api": f"DeviceShard.{fn} (pinned host buffers, two copy streams; assignments in "
                      f"{'document-major' if doc else 'word-group'} order) + "
                      f"{'doc_' if doc else ''}assignments_imported, rebuild_phi/prepare/rebuild_theta, "
                      f"sample_phase x {nphase} ({'document-block' if doc else 'word-group'} phases; each "
                      f"phase's assignments copied back and out while later phases sample), "
                      f"loglik_sum_async (C ABI; every step's loglik read back, the host never blocks on a step)"}
        del lls

    # ---- after the timed regions: K2 and K3 each ALONE (the step runs them
    # concurrently), and the K5 conservation check's cost (debug mode) ----
    def alone(fn, reps=3):
        ms = []
        for _ in range(reps):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(device)
            a0.record(stream)
            fn()
            a1.record(stream)
            torch.cuda.synchronize(device)
            ms.append(a0.elapsed_time(a1))
        return float(np.median(ms))

    sh.set_stream(stream)
    k2_alone = alone(sh.rebuild_phi)
    w = allreduce_async()                     # the replica is global again
    if w:
        w.wait()
    sh.prepare()
    k3_alone = alone(sh.rebuild_theta)

    def k5():
        r = sh.conservation(1)
        if not r[0]:
            r = sh.conservation(2, T_local if not dist else T_all)
        k5.report = r
    k5_ms = alone(k5)
    k5_ok = k5.report[0] == 0 or (dist is not None)   # N>1: columns are rank-local here

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:      # rank 0 at N=1 only
        nd = args.cpu_sample_docs or min(CPU_SAMPLE_DOCS[args.workload], SHAPES[args.workload]["num_docs"])
        cpu = cpu_baseline(args, K, nd)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "shard-proxy" if args.shard else args.scaling,
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": make_config(args, world, T_step),
            "layout": {"docs_this_rank": corp.num_docs, "tokens_this_rank": T_local, "runs": st["runs"],
                       "slices": st["slices"], "word_contexts": st["word_contexts"],
                       "doc_blocks": st["doc_blocks"], "theta_nnz_after_last_step": st["theta_nnz"]},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic["bytes_per_launch"] if traffic else None,
                         "traffic_source": (f"{traffic['source']} (committed ncu --set full capture of the same "
                                            f"command's K1 at the iteration named; ncu cannot run inside the "
                                            f"timed region)" if traffic else None),
                         "frac_of_nominal_8tbs": achieved / 8000.0,
                         "kernel": "gf::sample_kernel (K1)", "algorithmic_bytes_per_launch": st["sample_bytes"],
                         "kernel_ms": k1_ms, "peak_source": peak_src},
            "kernels": {
                "phi_rebuild": kernel_block("gf::phi_rebuild_kernel (K2, + memset of the 32-bit columns), alone",
                                            k2_alone, st["phi_bytes"], peak),
                "theta_rebuild": kernel_block("gf::theta_rebuild_kernel (K3), alone", k3_alone,
                                              st["theta_bytes"], peak),
                "in_step_ms": {"phi_rebuild": acc[1], "theta_rebuild": acc[4]},
                "note": "alone = median of 3 launches timed by CUDA events after the timed region; inside the "
                        "step K2 and K3 run concurrently (main / side stream), in_step_ms includes that contention",
            },
            "conservation": {"ms": k5_ms, "frac_of_step": k5_ms / ms_step, "ok": bool(k5_ok),
                             "what": "K5 (gf_shard_conservation stages 1+2: theta row/column sums, phi row "
                                     "sums, n_k, T; 2 tiny D2H reads) -- the per-iteration cost of "
                                     "TrainConfig(check_conservation=True), not in the timed step"},
            "kernel_ms": {"sample": acc[0], "phi_rebuild": acc[1], "allreduce_and_prepare": acc[2],
                          "theta_rebuild_exposed": acc[3], "theta_rebuild": acc[4]},
            "loglik_per_token": ll,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "preprocess": {"value": T_local / prep_s, "unit": "tokens/s", "seconds": prep_s,
                           "path": "DeviceShard.load_tokens: H2D of doc-major tokens + K4 partition (CUB radix "
                                   "sorts, splitmix64 z0) + device layout (runs, slices, zdoc positions)",
                           "reference": "gibbsflow partition(): ~3.6 s per 10M tokens single-threaded (SURVEY 6)"},
            "clocks": clocks.summary(),
            "gpu_launches": args.steps * launches_per_step,
        }
        print(json.dumps(line), flush=True)
    sh.close()
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
