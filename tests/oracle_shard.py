"""A CPU stand-in for `DeviceShard` backed by the oracle -- TEST INFRASTRUCTURE.

It implements the interface `engine.Trainer` drives (load / rebuild_phi /
prepare / rebuild_theta / sample / loglik_sum / sync_tensor / get_*), keeps the
phi sync buffer in exactly the device layout (`shard.sync_layout`: u32 heavy
columns, packed u16 light columns, n_k) as a CPU int32 tensor, and samples with
the oracle's "thin" mode (the device's draw form).  It lets the multi-rank
engine logic -- sharding, vocabulary allreduce, packed phi allreduce, loglik
reduction, theta gather -- run under torch.distributed/gloo on a CPU box.
"""

import numpy as np
import torch

import oracle
from paper_1803_04631_b200.errors import CountOverflowError
from paper_1803_04631_b200.shard import sync_layout


class OracleShard:
    def __init__(self, num_topics, vocab_size, alpha, beta, seed=0, device=0, heavy_threshold=65535,
                 global_word_freq=None, stream=None):
        self.K, self.V = int(num_topics), int(vocab_size)
        self.alpha, self.beta, self.seed = float(alpha), float(beta), int(seed)
        self.col, (self.o16, self.onk, self.total) = sync_layout(global_word_freq, self.K, heavy_threshold)
        self.Kp = self.K + (self.K & 1)
        self.sync = torch.zeros(self.total, dtype=torch.int32)
        self.ll = 0.0
        self._h = None

    # --- lifecycle
    def load(self, chunk):
        self.chunk = chunk
        self.z = chunk.assignments.copy()
        self.tok_local = (chunk.doc_ids - chunk.doc_lo).astype(np.int32)
        self.doc_len = np.diff(chunk.dw_ptr).astype(np.int64)
        return self

    def close(self):
        pass

    # --- phi sync buffer in the device layout
    def _pack(self, counts, totals):
        buf = self.sync.numpy().view(np.uint32)
        buf[:] = 0
        heavy = self.col < 0
        hv = np.flatnonzero(heavy)
        buf[: self.o16].reshape(-1, self.K)[:] = counts[:, hv].T.astype(np.uint32) if len(hv) else 0
        lv = np.flatnonzero(~heavy)
        if len(lv):
            if counts[:, lv].max() > 65535:
                raise CountOverflowError("light phi column overflow")
            l16 = np.zeros((len(lv), self.Kp), np.uint16)
            l16[:, : self.K] = counts[:, lv].T
            buf[self.o16: self.onk] = l16.reshape(-1).view(np.uint32)
        buf[self.onk:] = totals.astype(np.uint32)

    def _unpack(self):
        buf = self.sync.numpy().view(np.uint32)
        counts = np.zeros((self.K, self.V), np.uint32)
        heavy = self.col < 0
        hv = np.flatnonzero(heavy)
        if len(hv):
            counts[:, hv] = buf[: self.o16].reshape(-1, self.K).T
        lv = np.flatnonzero(~heavy)
        if len(lv):
            counts[:, lv] = buf[self.o16: self.onk].view(np.uint16).reshape(len(lv), self.Kp)[:, : self.K].T
        return counts, buf[self.onk:].astype(np.int64)

    def sync_tensor(self):
        return self.sync

    # --- kernels
    def rebuild_phi(self):
        c, t = oracle.rebuild_phi(self.z, self.chunk.word_ids, self.K, self.V)
        self._pack(c, t)

    def prepare(self):
        self.phi, self.totals = self._unpack()

    def rebuild_theta(self):
        self.theta = oracle.rebuild_theta(self.z, self.chunk.dw_ptr, self.chunk.dw_tok, 0, self.K)

    def sample(self, iteration):
        rp, ids, cn = self.theta
        self.ll = oracle.loglik_naive(self.K, self.V, self.alpha, self.beta, self.tok_local, self.chunk.word_ids,
                                      rp, ids, cn, self.doc_len, self.phi, self.totals) * len(self.z)
        self.z = oracle.sample_tokens(self.K, self.V, self.alpha, self.beta, self.seed, iteration,
                                      self.chunk.doc_ids, self.chunk.word_ids, self.z, self.chunk.doc_lo,
                                      rp, ids, cn, self.phi, self.totals, mode="thin")

    def iterate(self, iteration):
        """gf_shard_iterate's order: sample, then the counts of the new state."""
        self.sample(iteration)
        self.rebuild_phi()
        self.prepare()
        self.rebuild_theta()

    def loglik_sum(self):
        return self.ll

    def check_errors(self):
        pass

    def synchronize(self):
        pass

    # --- export
    def get_theta(self):
        return self.theta

    def get_phi(self):
        return self._unpack()

    def get_assignments(self):
        return self.z.copy()

    def check_phi_width(self, width):
        pass

    # --- K5 stand-in: the oracle's reductions in the device report layout
    def conservation(self, stage, num_tokens=0):
        rp, ids, cn = self.theta
        if stage == 1:
            D = len(rp) - 1
            sums = np.bincount(np.repeat(np.arange(D), np.diff(rp)), weights=cn, minlength=D).astype(np.int64)
            bad = np.flatnonzero(sums != self.doc_len)
            self._cols = torch.as_tensor(np.bincount(ids.astype(np.int64), weights=cn, minlength=self.K)
                                         .astype(np.int64))
            if bad.size:
                d = int(bad[0])
                return (1, self.chunk.doc_lo + d, int(sums[d]), int(self.doc_len[d]))
            return (0, 0, 0, 0)
        counts, totals = self._unpack()
        cols = self._cols.numpy()
        for code, val in ((2, cols), (3, counts.sum(axis=1, dtype=np.int64))):
            bad = np.flatnonzero(val != totals)
            if bad.size:
                k = int(bad[0])
                return (code, k, int(val[k]), int(totals[k]))
        if int(totals.sum()) != num_tokens:
            return (4, 0, int(totals.sum()), int(num_tokens))
        return (0, 0, 0, 0)

    def conservation_columns(self):
        return self._cols
