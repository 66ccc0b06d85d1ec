"""Training engine -- deferred-mode CGS on one or more B200s.

One process per GPU.  Rank r of G owns document shard r of
`greedy_boundaries(doc_lengths, G)` (corpus.py:210-237; C = G, M = 1 --
WorkSchedule1, every configured corpus fits in 180 GB of HBM), its theta rows
(never exchanged) and a phi replica.  One iteration (PAPER.md
section 6.2):

    K1 sample(it)     every token against the iteration-start theta / phi
    K2 rebuild_phi    this shard's replica + n_k into the sync buffer
    allreduce(sync)   NCCL sum over ranks on torch's NCCL stream ...
    K3 rebuild_theta  ... overlapped with the allreduce on the compute stream
    prepare           Eq. 1 denominators from the global n_k

The allreduce is an integer sum, so the result equals SPEC's pairwise
reduce_phi / broadcast_phi bit for bit.  The Philox
stream is keyed by token identity, so every G draws from the same uniforms;
the trained models agree statistically (fp32 S sums may round differently
when a shard's slice layout changes, which can flip a rare boundary draw).
"""

import time
from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

from .corpus import greedy_boundaries, make_chunk
from .errors import CapacityError, ShapeMismatchError
from .model import PhiMatrix, ThetaRows, concat_theta, conservation_report, phi_dtype


@dataclass
class TrainConfig:
    """SPEC.md:312-314."""

    num_topics: int
    iterations: int = 100
    alpha: Optional[float] = None        # default 50 / K
    beta: float = 0.01
    workers: int = 1                     # G: one process (rank) per GPU
    chunks_per_worker: int = 1           # M: only WorkSchedule1 (M = 1)
    seed: int = 42
    mode: str = "deferred"
    fanout: int = 32
    phi_width: int = 32                  # width of the exported PhiMatrix
    memory_budget: Optional[int] = None
    eval_every: int = 1
    heavy_threshold: int = 65535         # device phi: 16-bit columns below it
    check_conservation: bool = False
    phi_sync: str = "nccl"               # G > 1: "nccl" all_reduce, or "peer" (IPC peer-memory kernel)

    def __post_init__(self):
        if not 1 <= self.num_topics < 2**16:
            raise ValueError(f"topic count {self.num_topics} outside [1, 65536)")
        if self.alpha is None:
            self.alpha = 50.0 / self.num_topics
        if not (self.alpha > 0 and self.beta > 0):
            raise ValueError("alpha and beta must be > 0")
        if self.mode != "deferred":
            raise ValueError("the B200 engine runs deferred mode; exact (per-token) CGS is the CPU oracle")
        if self.fanout != 32:
            raise ValueError("the device tree is 32-ary (one warp per level)")
        if self.chunks_per_worker != 1:
            raise ValueError("only WorkSchedule1 (M = 1): every configured corpus fits in HBM")
        phi_dtype(self.phi_width)
        if not 0 <= self.heavy_threshold <= 65535:
            raise ValueError(f"heavy_threshold {self.heavy_threshold} outside [0, 65535] (16-bit phi columns)")
        if self.phi_sync not in ("nccl", "peer"):
            raise ValueError(f"phi_sync must be 'nccl' or 'peer', not {self.phi_sync!r}")


@dataclass
class IterationReport:
    """SPEC.md:316-319.  loglik_per_token describes the model the iteration
    started from (it is fused into the sampling pass)."""

    iteration: int
    elapsed_sec: float
    tokens_per_sec: float
    loglik_per_token: Optional[float]
    conservation: Optional[str] = None

    def csv_row(self):
        ll = "" if self.loglik_per_token is None else f"{self.loglik_per_token:.10f}"
        return f"{self.iteration},{self.elapsed_sec:.6f},{self.tokens_per_sec:.3f},{ll}"


CSV_HEADER = "iteration,elapsed_sec,tokens_per_sec,loglik_per_token"


def _dist():
    try:
        import torch.distributed as dist

        return dist if dist.is_available() and dist.is_initialized() else None
    except ImportError:
        return None


class Trainer:
    """Device-resident trainer for this rank's shard."""

    def __init__(self, corpus, cfg, group=None, device=None, shard_factory=None, init_assignments=None):
        """init_assignments: optional uint16 topics for this rank's chunk (word-group
        order) replacing partition()'s Stream(seed, chunk_id) draw -- e.g. to resume
        from a chunk store, or to start G ranks from the state of another G."""
        self.cfg = cfg
        self.corpus = corpus
        self.group = group
        d = _dist()
        self.dist = d
        self.rank = d.get_rank(group) if d else 0
        self.world = d.get_world_size(group) if d else 1
        if cfg.workers != self.world:
            raise ShapeMismatchError(f"cfg.workers={cfg.workers} but {self.world} rank(s) are running")
        K, V = cfg.num_topics, corpus.vocab_size
        lo, hi = greedy_boundaries(corpus.doc_lengths, self.world)[self.rank]
        a, b = int(corpus.doc_ptr[lo]), int(corpus.doc_ptr[hi])
        self.chunk = make_chunk(self.rank, lo, hi, corpus.doc_ids[a:b], corpus.word_ids[a:b], V, K, cfg.seed)
        if init_assignments is not None:
            z0 = np.ascontiguousarray(init_assignments, dtype=np.uint16)
            if z0.shape != (self.chunk.token_count,):
                raise ShapeMismatchError(f"init_assignments has {z0.size} entries, shard has {self.chunk.token_count}")
            self.chunk = replace(self.chunk, assignments=z0)
        if device is None:
            device = self._local_device()
        self.device = device
        if self.world > 1 and self._backend() == "nccl":
            import torch

            torch.cuda.set_device(device)          # before the first NCCL collective (one GPU per rank)
        if corpus.num_tokens >= 2**32:
            # n_k (sync buffer) and the theta / phi cells it bounds are 32-bit words
            raise CapacityError(f"corpus has {corpus.num_tokens} tokens; topic totals are 32-bit (at most 2^32 - 1)")
        freq = np.bincount(self.chunk.word_ids, minlength=V).astype(np.int64)
        self.global_freq = self._allreduce_np(freq)
        if shard_factory is None:
            from .shard import DeviceShard

            shard_factory = DeviceShard
        stream = None
        if self.world > 1:
            import torch

            # the shard runs on torch's current stream so the phi all_reduce
            # (NCCL, or gloo on the CUDA sync tensor) is ordered after K2 and
            # before prepare / the next K1 without host synchronisation
            if self._backend() == "nccl" or torch.cuda.is_available():
                stream = torch.cuda.current_stream(device)
        self.shard = shard_factory(K, V, cfg.alpha, cfg.beta, seed=cfg.seed, device=device,
                                   heavy_threshold=cfg.heavy_threshold, global_word_freq=self.global_freq,
                                   stream=stream)
        self.shard.load(self.chunk)
        self._peer = self.world > 1 and cfg.phi_sync == "peer"
        if self._peer:
            # map every rank's sync buffer (same node): the phi sum becomes one
            # kernel on the shard's stream (gf_shard_peer_allreduce)
            parts = [None] * self.world
            self.dist.all_gather_object(parts, self.shard.peer_handle(), group=self.group)
            self.shard.peer_open(self.rank, self.world, parts)
        self._sync_t = self.shard.sync_tensor() if self.world > 1 and not self._peer else None
        self.num_tokens = corpus.num_tokens
        self.iteration = 0
        # counts from the initial assignments
        self.shard.rebuild_phi()
        self._allreduce_sync()
        self.shard.prepare()
        self.shard.rebuild_theta()
        self.shard.check_errors()

    # ------------------------------------------------------------ plumbing --
    def _backend(self):
        return self.dist.get_backend(self.group) if self.dist else None

    def _local_device(self):
        import os

        return int(os.environ.get("LOCAL_RANK", "0")) if self.world > 1 else 0

    def _allreduce_np(self, arr):
        if self.world == 1:
            return arr
        import torch

        if self._backend() == "nccl":
            t = torch.as_tensor(arr).to(f"cuda:{self.device}")
            self.dist.all_reduce(t, group=self.group)
            return t.cpu().numpy()
        t = torch.as_tensor(arr).clone()
        self.dist.all_reduce(t, group=self.group)
        return t.numpy()

    def _allreduce_sync(self, async_op=False):
        if self.world == 1:
            return None
        if self._peer:
            self.shard.peer_allreduce()
            return None
        return self.dist.all_reduce(self._sync_t, group=self.group, async_op=async_op)

    # -------------------------------------------------------------- steps --
    def step(self):
        """One deferred iteration; returns the IterationReport."""
        it = self.iteration
        t0 = time.perf_counter()
        sh = self.shard
        if self.world == 1 or self._peer:
            sh.iterate(it)                       # K1, then K3 beside K2 (+ peer phi exchange) + prepare
        else:
            sh.sample(it)
            sh.rebuild_phi()
            work = self._allreduce_sync(async_op=True)
            sh.rebuild_theta()                   # overlaps the phi allreduce
            if work is not None:
                work.wait()
            sh.prepare()
        ll = None
        if self.cfg.eval_every and it % self.cfg.eval_every == 0:
            ll = float(self._allreduce_np(np.array([sh.loglik_sum()], np.float64))[0]) / self.num_tokens
        else:
            sh.synchronize()
        sh.check_errors()
        elapsed = time.perf_counter() - t0
        report = IterationReport(it, elapsed, self.num_tokens / elapsed if elapsed > 0 else float("inf"), ll)
        if self.cfg.check_conservation:
            report.conservation = self.conservation().detail
        self.iteration += 1
        return report

    def conservation(self):
        """check_conservation (model.py:180-225) of the resident model by K5,
        nothing exported: each rank reduces its theta rows and the (global) phi;
        the theta column sums are summed over ranks on the device and the first
        bad document is the lowest-ranked report (shards are contiguous in
        document order)."""
        sh = self.shard
        row = sh.conservation(1)
        if self.world > 1:
            rows = [None] * self.world
            self.dist.all_gather_object(rows, row, group=self.group)
            row = next((r for r in rows if r[0]), row)
            cols = sh.conservation_columns()
            self.dist.all_reduce(cols, group=self.group)
        if row[0]:
            return conservation_report(*row)
        return conservation_report(*sh.conservation(2, self.num_tokens))

    def evaluate(self):
        """loglik_per_token of the current model."""
        from . import _lib

        _lib.check(_lib.lib().gf_shard_evaluate(self.shard._h))
        return float(self._allreduce_np(np.array([self.shard.loglik_sum()], np.float64))[0]) / self.num_tokens

    # -------------------------------------------------------------- export --
    def theta(self, gather=True):
        rp, ids, cn = self.shard.get_theta()
        local = ThetaRows(rp, ids, cn, self.cfg.num_topics)
        if self.world == 1 or not gather:
            return local
        parts = [None] * self.world
        self.dist.all_gather_object(parts, (rp, ids, cn), group=self.group)
        return concat_theta([ThetaRows(p[0], p[1], p[2], self.cfg.num_topics) for p in parts])

    def phi(self):
        if self.cfg.phi_width == 16:
            self.shard.check_phi_width(16)
        counts, totals = self.shard.get_phi()
        return PhiMatrix(counts.astype(phi_dtype(self.cfg.phi_width), copy=False), totals)

    def assignments(self):
        return self.shard.get_assignments()

    # ---------------------------------------------------- checkpoint/resume --
    def save_checkpoint(self, prefix):
        """Resume point after the completed iterations: every rank writes its
        chunk with the current assignments (GFCHUNK1, `<prefix>.rank<r>.gfc`,
        the state a snapshot lacks: corpus.py:305-327); rank 0 also writes the
        model snapshot (GFSNAP1, `<prefix>.gfsnap`, model.py:228-255) whose
        metadata records the iteration to resume at."""
        from .corpus import save_chunk
        from .model import save_snapshot

        save_chunk(replace(self.chunk, assignments=self.assignments()), f"{prefix}.rank{self.rank}.gfc")
        theta, phi = self.theta(gather=True), self.phi()
        if self.rank == 0:
            meta = {"iteration": self.iteration, "seed": self.cfg.seed, "num_topics": self.cfg.num_topics,
                    "workers": self.world, "alpha": self.cfg.alpha, "beta": self.cfg.beta}
            save_snapshot(theta, phi, f"{prefix}.gfsnap", metadata=meta)
        if self.dist:
            self.dist.barrier(group=self.group)

    @classmethod
    def resume(cls, corpus, cfg, prefix, group=None, device=None, shard_factory=None):
        """A trainer continuing a checkpoint: this rank's assignments from its
        chunk store, the iteration counter from the snapshot metadata.  Draws
        are keyed by (seed, iteration, token), so the resumed run repeats the
        uninterrupted one."""
        from .corpus import load_chunk
        from .model import load_snapshot

        _, _, meta = load_snapshot(f"{prefix}.gfsnap")
        if meta.get("num_topics") != cfg.num_topics or meta.get("seed") != cfg.seed:
            raise ShapeMismatchError("checkpoint was written with another num_topics / seed")
        d = _dist()
        rank = d.get_rank(group) if d else 0
        ch = load_chunk(f"{prefix}.rank{rank}.gfc")
        tr = cls(corpus, cfg, group=group, device=device, shard_factory=shard_factory,
                 init_assignments=ch.assignments)
        if (tr.chunk.doc_lo, tr.chunk.doc_hi) != (ch.doc_lo, ch.doc_hi):
            raise ShapeMismatchError("checkpoint shard does not match this rank's documents")
        tr.iteration = int(meta["iteration"])
        return tr

    def close(self):
        self.shard.close()


def train(corpus, cfg, group=None, device=None, metrics_path=None):
    """returns (ThetaRows, PhiMatrix, [IterationReport])."""
    tr = Trainer(corpus, cfg, group=group, device=device)
    reports = []
    try:
        for _ in range(cfg.iterations):
            reports.append(tr.step())
        theta, phi = tr.theta(gather=True), tr.phi()
    finally:
        tr.close()
    if metrics_path is not None and tr.rank == 0:
        with open(metrics_path, "w") as fh:
            fh.write(CSV_HEADER + "\n")
            for r in reports:
                fh.write(r.csv_row() + "\n")
    return theta, phi, reports


fit = train  # the north star's fit/transform naming


def transform(theta):
    """Normalised doc-topic proportions of the TRAINING documents (an invented
    convenience: inference on unseen documents is a SPEC non-goal)."""
    K = theta.num_topics
    out = np.zeros((theta.num_rows, K), np.float64)
    rows = np.repeat(np.arange(theta.num_rows), np.diff(theta.row_ptr))
    out[rows, theta.topic_ids.astype(np.int64)] = theta.counts
    s = out.sum(axis=1, keepdims=True)
    return out / np.maximum(s, 1)


def reduce_phi(replicas, num_workers=None):
    """pairwise tree merge in ceil(log2 G) rounds (round r:
    replica j += replica j + 2^r for j = 0 mod 2^(r+1)).  Host-side form for
    replicas already exported; on the device the NCCL allreduce does this."""
    if not replicas:
        raise ValueError("no replicas")
    shape = replicas[0].counts.shape
    for r in replicas:
        if r.counts.shape != shape:
            raise ShapeMismatchError(f"replica shape {r.counts.shape} != {shape}")
    acc = [np.array(r.counts, dtype=np.int64) for r in replicas]
    tot = [np.array(r.topic_totals, dtype=np.int64) for r in replicas]
    G = len(acc)
    step = 1
    while step < G:
        for j in range(0, G, 2 * step):
            if j + step < G:
                acc[j] += acc[j + step]
                tot[j] += tot[j + step]
        step *= 2
    dtype = replicas[0].counts.dtype
    if acc[0].max(initial=0) > np.iinfo(dtype).max:
        from .errors import CountOverflowError

        k, v = np.unravel_index(int(acc[0].argmax()), acc[0].shape)
        raise CountOverflowError(f"phi cell (topic {k}, word {v}) count {int(acc[0][k, v])} "
                                 f"exceeds {dtype.itemsize * 8}-bit range")
    return PhiMatrix(acc[0].astype(dtype), tot[0])


def broadcast_phi(global_phi, num_workers):
    """every worker observes one immutable snapshot."""
    global_phi.counts.setflags(write=False)
    global_phi.topic_totals.setflags(write=False)
    return [global_phi] * num_workers
