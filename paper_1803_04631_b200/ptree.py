"""Prefix-tree draw primitive (ptree.py:1-151) with the search on the B200.

`build` accumulates the prefix sums left to right in the tree dtype exactly as
the reference (host, numpy: the levels are the tree's data, not a hot path).
Every search -- `sample`, `sample_with_stats`, `sample_many`,
`sample_total_and_draw` -- runs the ballot descent of K1 on the device
(gf_ptree_sample, or gf_ptree_sample_f64 for the reference's fp64 oracle mode)
and returns the minimal index with prefix > u, identical to the reference's
scan (ptree.py:7-11).  There is no host search path: without the library or
a device the calls raise.
"""

import numpy as np

from . import _lib
from .errors import EmptyDistributionError

_DEVICE_SEARCH = {np.dtype(np.float32): "gf_ptree_sample", np.dtype(np.float64): "gf_ptree_sample_f64"}


class PrefixTree:
    """Immutable search tree over the prefix sums of non-negative weights
    (ptree.py:23-113): levels[0] is the leaf prefix array, each higher level
    the last boundary of every group of `fanout` entries, up to the root."""

    def __init__(self, levels, fanout):
        self.levels = levels
        self.fanout = fanout
        self.total = float(levels[0][-1])
        self.dtype = levels[0].dtype

    @property
    def height(self):
        return len(self.levels) - 1

    @property
    def num_leaves(self):
        return len(self.levels[0])

    def leaf_weights(self):
        """ptree.py:50-52: the individual leaf weights (prefix differences)."""
        return np.diff(self.levels[0], prepend=self.dtype.type(0))

    def level_sums(self, level):
        """ptree.py:54-56: per-node weight totals at `level`."""
        return np.diff(self.levels[level], prepend=self.dtype.type(0))

    def prefix_before(self, index):
        """ptree.py:58-62: prefix sum of the leaves strictly left of `index`."""
        if index == 0:
            return self.dtype.type(0)
        return self.levels[0][index - 1]

    # ---------------------------------------------------------- device --
    def _search(self, us, device, stats):
        if self.levels[-1][0] <= 0:
            raise EmptyDistributionError("cannot sample: total weight is zero")
        fn = _DEVICE_SEARCH.get(self.dtype)
        if fn is None:
            raise ValueError(f"device search supports float32 and float64 trees, not {self.dtype}")
        us = _lib.carr(us, self.dtype)
        top = self.levels[-1][0]
        if us.size and (np.any(us < 0) or np.any(us >= top)):
            raise ValueError("u values outside [0, total)")
        pre = _lib.carr(self.levels[0], self.dtype)
        idx = np.empty(len(us), np.int64)
        vis = np.empty(len(us), np.int32) if stats else None
        wid = np.empty(len(us), np.int32) if stats else None
        _lib.check(getattr(_lib.lib(), fn)(device, _lib.ptr(pre), len(pre), self.fanout, _lib.ptr(us), len(us),
                                           _lib.ptr(idx), _lib.ptr(vis) if stats else None,
                                           _lib.ptr(wid) if stats else None))
        return idx, vis, wid

    def _descend(self, u, device=0):
        """ptree.py:77-99: (index, levels visited, widest scan) for one u."""
        top = self.levels[-1][0]
        if top <= 0:
            raise EmptyDistributionError("cannot sample: total weight is zero")
        u = self.dtype.type(u)
        if u < 0 or u >= top:
            raise ValueError(f"u={u!r} outside [0, {top!r})")
        idx, vis, wid = self._search(np.array([u], self.dtype), device, True)
        return int(idx[0]), int(vis[0]), int(wid[0])

    def sample(self, u, device=0):
        """ptree.py:64-71: the minimal index k with prefix(k) > u."""
        return self._descend(u, device)[0]

    def sample_with_stats(self, u, device=0):
        """ptree.py:73-75: like `sample`, also (levels visited, widest scan)."""
        return self._descend(u, device)

    def sample_many(self, us, device=0):
        """ptree.py:101-113: one warp-ballot descent per u on the device."""
        return self._search(np.asarray(us), device, False)[0]


def build(weights, fanout=32, dtype=np.float32):
    """ptree.py:116-136."""
    if fanout < 2:
        raise ValueError(f"fanout must be >= 2, got {fanout}")
    w = np.asarray(weights)
    if w.ndim != 1 or w.size == 0:
        raise EmptyDistributionError("weights must be a non-empty 1-d array")
    if not np.all(w >= 0):
        raise ValueError("weights must be non-negative")
    levels = [np.cumsum(w.astype(dtype, copy=False), dtype=dtype)]
    while len(levels[-1]) > 1:
        prev = levels[-1]
        tails = np.minimum(np.arange(fanout - 1, len(prev) + fanout - 1, fanout), len(prev) - 1)
        levels.append(prev[tails])
    return PrefixTree(levels, fanout)


def sample_total_and_draw(tree, stream, device=0):
    """ptree.py:139-151: u = stream.uniform() * total in the tree dtype, the
    measure-zero round-up to total guarded to nextafter(total, 0), then the
    device descent.  Returns (index, u) so the draw can be replayed."""
    if tree.total <= 0:
        raise EmptyDistributionError("cannot sample: total weight is zero")
    u = tree.dtype.type(stream.uniform() * tree.total)
    top = tree.levels[-1][0]
    if u >= top:
        u = np.nextafter(top, tree.dtype.type(0))
    return tree.sample(u, device), float(u)
