"""ctypes binding of libgfb200.so (include/gibbsflow_b200.h).

The library is built in-tree (`paper_1803_04631_b200/_lib/libgfb200.so`, by
`__graft_entry__.build()` / `make -C paper_1803_04631_b200/csrc`).  There is no
fallback: if the library is missing the import of any device-facing function
fails loudly, and on a machine without a CUDA device the shard constructor
raises `NoDeviceError`.
"""

import ctypes
import os

import numpy as np

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
# GF_LIB: another build of the same library (A/B of kernel variants on one box)
SO_PATH = os.environ.get("GF_LIB") or os.path.join(_HERE, "_lib", "libgfb200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "gibbsflow_b200.h")

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_f64 = ctypes.c_double
_int = ctypes.c_int
_pp = ctypes.POINTER(ctypes.c_void_p)

# name -> (restype, argtypes), mirroring the header one for one
SIGNATURES = {
    "gf_last_error": (ctypes.c_char_p, []),
    "gf_abi_version": (_int, []),
    "gf_device_count": (_int, [_p]),
    "gf_stream_key": (_u64, [_p, _int]),
    "gf_stream_uniforms": (_int, [_u64, _u64, _i64, _p]),
    "gf_greedy_boundaries": (_int, [_p, _i64, _i64, _p]),
    "gf_partition_chunk": (_int, [_p, _p, _i64, _i64, _i64, _i32, _i32, _u64, _i64] + [_p] * 9),
    "gf_partition_chunk_gpu": (_int, [_int, _p, _p, _i64, _i64, _i64, _i32, _i32, _u64, _i64] + [_p] * 9),
    "gf_shard_load_tokens": (_int, [_p, _i64, _i64, _i64, _p, _p, _u64, _i64]),
    "gf_shard_create": (_int, [_pp, _int, _i32, _i32, _f64, _f64, _u64, _u32]),
    "gf_shard_destroy": (_int, [_p]),
    "gf_shard_set_stream": (_int, [_p, _p]),
    "gf_shard_set_params": (_int, [_p, _f64, _f64, _u64]),
    "gf_shard_set_vocab": (_int, [_p, _p]),
    "gf_shard_load": (_int, [_p, _i64, _i64, _i64, _p, _p, _p, _i64, _p, _p, _p, _p, _p]),
    "gf_shard_rebuild_phi": (_int, [_p]),
    "gf_shard_rebuild_theta": (_int, [_p]),
    "gf_shard_prepare": (_int, [_p]),
    "gf_shard_sample": (_int, [_p, _u32]),
    "gf_shard_iterate": (_int, [_p, _u32]),
    "gf_shard_evaluate": (_int, [_p]),
    "gf_shard_sample_export": (_int, [_p, _u32, _p]),
    "gf_shard_set_phases": (_int, [_p, _int]),
    "gf_shard_set_phase_cuts": (_int, [_p, _p, _int]),
    "gf_shard_num_phases": (_int, [_p, _p]),
    "gf_shard_phase_range": (_int, [_p, _int, _p, _p]),
    "gf_shard_sample_phase": (_int, [_p, _u32, _int]),
    "gf_shard_loglik_sum": (_int, [_p, _p]),
    "gf_shard_loglik_sum_async": (_int, [_p, _p, _p]),
    "gf_shard_check_errors": (_int, [_p]),
    "gf_shard_synchronize": (_int, [_p]),
    "gf_shard_sync_buffer": (_int, [_p, _pp, _p]),
    "gf_shard_peer_handle": (_int, [_p, _p]),
    "gf_shard_peer_open": (_int, [_p, _int, _int, _p]),
    "gf_shard_peer_allreduce": (_int, [_p]),
    "gf_shard_peer_close": (_int, [_p]),
    "gf_shard_rebuild_phi_exchange": (_int, [_p]),
    "gf_sync_layout": (_int, [_p, _i32, _i32, _u32, _p, _p]),
    "gf_host_alloc": (_int, [_i64, _pp]),
    "gf_host_free": (_int, [_p, _i64]),
    "gf_shard_get_assignments": (_int, [_p, _p]),
    "gf_shard_set_assignments": (_int, [_p, _p]),
    "gf_shard_copy_assignments_async": (_int, [_p, _p, _i64, _i64, _int, _p]),
    "gf_shard_assignments_imported": (_int, [_p]),
    "gf_shard_copy_doc_assignments_async": (_int, [_p, _p, _i64, _i64, _int, _p]),
    "gf_shard_doc_assignments_imported": (_int, [_p]),
    "gf_shard_set_block_phases": (_int, [_p, _p, _int]),
    "gf_shard_phase_doc_range": (_int, [_p, _int, _p, _p]),
    "gf_shard_theta_nnz": (_int, [_p, _p]),
    "gf_shard_get_theta": (_int, [_p, _p, _p, _p]),
    "gf_shard_set_theta": (_int, [_p, _p, _p, _p]),
    "gf_shard_get_phi": (_int, [_p, _p, _p]),
    "gf_shard_set_phi": (_int, [_p, _p, _p]),
    "gf_shard_get_phi_w": (_int, [_p, _p, _i32, _p]),
    "gf_shard_set_phi_w": (_int, [_p, _p, _i32, _p]),
    "gf_shard_phi_argmax": (_int, [_p, _p, _p, _p]),
    "gf_shard_stats": (_int, [_p, _p, _int]),
    "gf_shard_reset_stats": (_int, [_p]),
    "gf_shard_last_times": (_int, [_p, _p, _int]),
    "gf_shard_conservation": (_int, [_p, _int, _i64, _p]),
    "gf_shard_conservation_buffer": (_int, [_p, _pp, _p]),
    "gf_check_conservation": (_int, [_int, _i32, _i64, _i64] + [_p] * 5 + [_i32, _p, _i64, _p]),
    "gf_snapshot_write": (_int, [ctypes.c_char_p, _i64, _i64, _i64, _i64, _i32] + [_p] * 5
                          + [ctypes.c_char_p, _i64]),
    "gf_snapshot_header": (_int, [ctypes.c_char_p, _p]),
    "gf_snapshot_read": (_int, [ctypes.c_char_p] + [_p] * 6),
    "gf_ptree_sample": (_int, [_int, _p, _i64, _i32, _p, _i64, _p, _p, _p]),
    "gf_ptree_sample_f64": (_int, [_int, _p, _i64, _i32, _p, _i64, _p, _p, _p]),
    "gf_uci_scan": (_int, [ctypes.c_char_p, _p, _p]),
    "gf_uci_tokens": (_int, [ctypes.c_char_p, _i64, _p, _p, _p]),
    "gf_synth_lengths": (_int, [_u64, _i64, _i64, _f64, _f64, _p]),
    "gf_synth_tokens": (_int, [_u64, _i64, _i64, _p, _i32, _i32, _f64, _f64, _p, _p]),
}

_ERRORS = {
    1: errors.CountOverflowError,
    2: errors.ShapeMismatchError,
    3: errors.ConsistencyError,
    4: errors.CapacityError,
    5: errors.TrainingError,
    6: ValueError,
    7: errors.PartitionError,
    8: errors.EmptyDistributionError,
    9: errors.NoDeviceError,
    10: errors.CorpusFormatError,
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(
                f"{SO_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')"
            )
        L = ctypes.CDLL(SO_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc):
    if rc != 0:
        msg = lib().gf_last_error().decode("utf-8", "replace")
        raise _ERRORS.get(rc, errors.GibbsflowError)(msg)


def ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def carr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class _PinnedBlock:
    """A gf_host_alloc block exposed to numpy (`__array_interface__`); it goes
    back to the library's cache when the last array viewing it is collected."""

    def __init__(self, nbytes):
        import weakref

        p = ctypes.c_void_p()
        check(lib().gf_host_alloc(nbytes, ctypes.byref(p)))
        self.__array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (p.value, False), "version": 3}
        fin = weakref.finalize(self, lib().gf_host_free, ctypes.c_void_p(p.value), nbytes)
        fin.atexit = False                       # the driver releases pinned memory at exit


_PINNED_MIN = 1 << 20


def pinned_empty(shape, dtype):
    """np.empty in a cached pinned block (results of the one-call API: DMA'd
    directly, no first-touch page faults, full-speed upload when handed back);
    small arrays, or a failed pinned allocation, get ordinary memory."""
    dtype = np.dtype(dtype)
    shape = tuple(int(x) for x in np.atleast_1d(shape))
    n = int(np.prod(shape)) * dtype.itemsize
    if n < _PINNED_MIN:
        return np.empty(shape, dtype)
    try:
        blk = _PinnedBlock(n)
    except errors.GibbsflowError:
        return np.empty(shape, dtype)
    return np.asarray(blk).view(dtype).reshape(shape)


def device_count():
    n = ctypes.c_int(0)
    lib().gf_device_count(ctypes.byref(n))
    return n.value
