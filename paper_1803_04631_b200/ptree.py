"""Prefix-tree draw primitive (ptree.py:116-151) with the search on the B200.

`build` accumulates the prefix sums left to right in the tree dtype exactly as
the reference (host, numpy); `PrefixTree.sample_many` runs the 32-ary (or any
fanout <= 32) ballot descent of K1 on the device (gf_ptree_sample) and returns
the minimal index with prefix > u, identical to the reference's scan.
"""

import numpy as np

from . import _lib
from .errors import EmptyDistributionError


class PrefixTree:
    def __init__(self, levels, fanout):
        self.levels = levels
        self.fanout = fanout
        self.total = float(levels[0][-1])
        self.dtype = levels[0].dtype

    @property
    def height(self):
        return len(self.levels) - 1

    def sample_many(self, us, device=0):
        if self.dtype != np.float32:
            raise ValueError("the device search runs in fp32 (the paper's precision)")
        if self.levels[-1][0] <= 0:
            raise EmptyDistributionError("cannot sample: total weight is zero")
        us = _lib.carr(us, np.float32)
        out = np.empty(len(us), np.int64)
        pre = _lib.carr(self.levels[0], np.float32)
        _lib.check(_lib.lib().gf_ptree_sample(device, _lib.ptr(pre), len(pre), self.fanout, _lib.ptr(us),
                                              len(us), _lib.ptr(out)))
        return out

    def sample(self, u, device=0):
        return int(self.sample_many(np.array([u], np.float32), device)[0])


def build(weights, fanout=32, dtype=np.float32):
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
