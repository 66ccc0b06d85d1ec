"""splitmix64 counter streams (rng.py:1-89), computed by the native library
(gf_stream_key / gf_stream_uniforms), bit-identical to the reference."""

import ctypes

import numpy as np

from . import _lib


def stream_key(*parts):
    """rng.py:45-53: fold integer parts into one uint64 key."""
    arr = np.array([p & 0xFFFFFFFFFFFFFFFF for p in parts], dtype=np.uint64)
    return np.uint64(_lib.lib().gf_stream_key(_lib.ptr(arr), len(arr)))


class Stream:
    """rng.py:56-81: stateful view over a counter-based uniform stream."""

    def __init__(self, *parts):
        self.key = stream_key(*parts)
        self.counter = 0

    def uniforms(self, n):
        out = np.empty(int(n), dtype=np.float64)
        _lib.check(_lib.lib().gf_stream_uniforms(int(self.key), self.counter, int(n), _lib.ptr(out)))
        self.counter += int(n)
        return out

    def uniform(self):
        return float(self.uniforms(1)[0])

    def integer(self, n):
        return min(int(self.uniform() * n), n - 1)
