"""DeviceShard: one document shard resident on one B200 (the C-ABI gf_shard).

This is the runtime object behind every reference-facing call
(`rebuild_theta`, `rebuild_phi_replica`, `sample_chunk`, `train`): a Chunk
(corpus.py:160-198) uploaded once, its theta rows and a phi replica kept in
HBM, and the four hot kernels driven through the C ABI:

    sample(it)      K1  SPEC.md:359-367 (+ fused loglik)
    rebuild_phi()   K2  model.py:142-161 (replica -> sync buffer)
    prepare()           Eq. 1 denominators from the (global) n_k
    rebuild_theta() K3  model.py:109-124
"""

import ctypes

import numpy as np

from . import _lib
from .errors import CountOverflowError


class _CudaArray:
    """__cuda_array_interface__ view of a device buffer owned by a shard."""

    def __init__(self, ptr, n, typestr, owner):
        self._owner = owner
        self.__cuda_array_interface__ = {
            "shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
            "version": 3, "strides": None, "stream": None,
        }


class ResidentShards:
    """Shards kept resident for the reference-facing one-call functions
    (sampler.sample_chunk, model.rebuild_theta / rebuild_phi_replica,
    eval.loglik_per_token): a chunk handed in again -- the same token arrays,
    e.g. the same Chunk or a dataclasses.replace() of it with new assignments --
    reuses its shard instead of repeating the K4 layout.  Only what the call
    passes is uploaded: the assignments through the staged import (a device-side
    diff rewrites only changed runs), theta / phi when given.  Least recently
    used shards beyond `capacity` are closed (release() closes all)."""

    def __init__(self, capacity=4):
        from collections import OrderedDict

        self.capacity = capacity
        self._lru = OrderedDict()

    @staticmethod
    def _key(arrays, extra):
        return tuple(id(a) for a in arrays) + tuple(extra)

    def get(self, arrays, extra, build):
        """The live shard for (token arrays, extra) or a new one from build()."""
        import weakref

        key = self._key(arrays, extra)
        ent = self._lru.get(key)
        if ent is not None and all(r() is a for r, a in zip(ent[0], arrays)):
            self._lru.move_to_end(key)
            return ent[1], False
        if ent is not None:
            ent[1].close()
            del self._lru[key]
        sh = build()
        self._lru[key] = ([weakref.ref(a) for a in arrays], sh)
        while len(self._lru) > self.capacity:
            self._lru.popitem(last=False)[1][1].close()
        return sh, True

    def find(self, arrays, pred):
        """The most recently used live shard of these arrays whose extra key
        satisfies pred (or None)."""
        ids = tuple(id(a) for a in arrays)
        for key in reversed(list(self._lru)):
            refs, sh = self._lru[key]
            if key[: len(ids)] == ids and pred(key[len(ids):]) and all(r() is a for r, a in zip(refs, arrays)):
                self._lru.move_to_end(key)
                return sh
        return None

    def drop(self, arrays, extra):
        ent = self._lru.pop(self._key(arrays, extra), None)
        if ent is not None:
            ent[1].close()

    def release(self):
        while self._lru:
            self._lru.popitem()[1][1].close()


RESIDENT = ResidentShards()
API_PHASES = [0.5, 0.75, 0.875, 0.9375, 1.0]


def chunk_shard(chunk, num_topics, vocab_size, alpha=1.0, beta=1.0, seed=0, device=0, global_word_freq=None,
                layout="chunk", any_vocab=False):
    """The resident shard of `chunk` with its assignments current (staged
    import: nothing is rewritten when they did not change).  any_vocab: any
    resident shard of the chunk with this K will do (theta needs no phi
    layout).  vocab_size may be a callable, evaluated only for a new shard."""
    arrays = (chunk.word_ids, chunk.doc_ids, chunk.dw_tok, chunk.group_offsets)
    if any_vocab:
        want = (int(num_topics), int(device), int(chunk.doc_lo), int(chunk.doc_hi))
        sh = RESIDENT.find(arrays, lambda e: (e[0],) + tuple(e[2:5]) == want)
        if sh is not None:
            _import_assignments(sh, chunk)
            return sh
    if callable(vocab_size):          # only needed for a new shard (an O(T) scan for some callers)
        vocab_size = vocab_size()
    extra = (int(num_topics), int(vocab_size), int(device), int(chunk.doc_lo), int(chunk.doc_hi), layout)

    def build():
        # word phases (halving sizes): sample_chunk's result streams back while
        # the later phases sample (gf_shard_sample_export)
        sh = DeviceShard(num_topics, vocab_size, alpha, beta, seed=seed, device=device,
                         global_word_freq=global_word_freq, phases=API_PHASES)
        return sh.load(chunk)

    sh, fresh = RESIDENT.get(arrays, extra, build)
    if not fresh:
        sh.set_params(alpha, beta, seed)
        _import_assignments(sh, chunk)
    return sh


def _import_assignments(sh, chunk):
    z = chunk.assignments
    if not (isinstance(z, np.ndarray) and z.dtype == np.uint16 and z.flags.c_contiguous):
        z = np.ascontiguousarray(z, dtype=np.uint16)
    sh.copy_assignments_async(z, 0, len(z), True)
    sh.assignments_imported()


def sync_layout(global_word_freq, num_topics, heavy_threshold=65535):
    """gf_sync_layout: (word_col int32[V], (phi16 off, n_k off, total) in u32 words)."""
    freq = _lib.carr(global_word_freq, np.int64)
    col = np.empty(len(freq), np.int32)
    lay = np.empty(3, np.int64)
    _lib.check(_lib.lib().gf_sync_layout(_lib.ptr(freq), len(freq), int(num_topics), int(heavy_threshold),
                                         _lib.ptr(col), _lib.ptr(lay)))
    return col, (int(lay[0]), int(lay[1]), int(lay[2]))


class DeviceShard:
    def __init__(self, num_topics, vocab_size, alpha, beta, seed=0, device=0,
                 heavy_threshold=65535, global_word_freq=None, stream=None, phases=1):
        self.K = int(num_topics)
        self.V = int(vocab_size)
        self.alpha = float(alpha)
        self.beta = float(beta)
        self.device = int(device)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().gf_shard_create(ctypes.byref(h), self.device, self.K, self.V, self.alpha,
                                              self.beta, int(seed) & 0xFFFFFFFFFFFFFFFF, int(heavy_threshold)))
        self._h = h
        self.heavy_threshold = int(heavy_threshold)
        if stream is not None:
            self.set_stream(stream)
        if np.ndim(phases) != 0 or phases != 1:
            self.set_phases(phases)
        if global_word_freq is not None:
            f = _lib.carr(global_word_freq, np.int64)
            if len(f) != self.V:
                raise ValueError("global_word_freq must have vocab_size entries")
            _lib.check(_lib.lib().gf_shard_set_vocab(self._h, _lib.ptr(f)))
        self.chunk = None
        self._shape = (0, 0)

    # ---------------------------------------------------------------- life --
    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().gf_shard_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_stream(self, stream):
        """Run on a CUDA stream: a torch.cuda.Stream or a raw cudaStream_t int."""
        handle = getattr(stream, "cuda_stream", stream)
        _lib.check(_lib.lib().gf_shard_set_stream(self._h, ctypes.c_void_p(int(handle))))

    def load(self, chunk):
        """Upload a Chunk.  Its group directory may be in any order (e.g. the
        heavy-first order of sort_word_groups_desc, corpus.py:290-302): the
        token arrays are word-sorted, so ascending offsets are ascending words
        and the device builds its own heavy-first schedule."""
        c = chunk
        go = np.asarray(c.group_offsets, np.int64)
        order = np.argsort(go, kind="stable") if go.size > 1 and np.any(go[1:] < go[:-1]) else None
        gw, gs = c.group_words, c.group_sizes
        if order is not None:
            gw, go, gs = np.asarray(gw)[order], go[order], np.asarray(gs)[order]
        self._keep = [
            _lib.carr(c.doc_ids, np.int32), _lib.carr(c.word_ids, np.int32),
            _lib.carr(c.assignments, np.uint16), _lib.carr(gw, np.int32),
            _lib.carr(go, np.int64), _lib.carr(gs, np.int64),
            _lib.carr(c.dw_ptr, np.int64), _lib.carr(c.dw_tok, np.int64),
        ]
        d, w, z, gw, go, gs, dp, dt = self._keep
        _lib.check(_lib.lib().gf_shard_load(self._h, int(c.doc_lo), int(c.doc_hi), int(c.token_count),
                                            _lib.ptr(d), _lib.ptr(w), _lib.ptr(z), len(gw), _lib.ptr(gw),
                                            _lib.ptr(go), _lib.ptr(gs), _lib.ptr(dp), _lib.ptr(dt)))
        self._keep = None
        self.chunk = c
        self._shape = (int(c.token_count), int(c.doc_hi - c.doc_lo))
        return self

    def load_tokens(self, doc_lo, doc_hi, doc_ids, word_ids, seed, chunk_id=0):
        """K4: load documents [doc_lo, doc_hi) straight from their doc-major
        tokens (the Corpus slice, corpus.py:253-255) -- partition, dw-map,
        splitmix64 z0 and the shard layout all on the device.  Equivalent to
        load(make_chunk(chunk_id, doc_lo, doc_hi, doc_ids, word_ids, V, K, seed));
        `chunk` stays None (export with get_assignments / get_theta / get_phi)."""
        d = _lib.carr(doc_ids, np.int32)
        w = _lib.carr(word_ids, np.int32)
        _lib.check(_lib.lib().gf_shard_load_tokens(self._h, int(doc_lo), int(doc_hi), len(d), _lib.ptr(d),
                                                   _lib.ptr(w), int(seed) & 0xFFFFFFFFFFFFFFFF, int(chunk_id)))
        self.chunk = None
        self._shape = (len(d), int(doc_hi - doc_lo))
        return self

    # -------------------------------------------------------------- kernels --
    def rebuild_phi(self):
        _lib.check(_lib.lib().gf_shard_rebuild_phi(self._h))

    def rebuild_theta(self):
        _lib.check(_lib.lib().gf_shard_rebuild_theta(self._h))

    def prepare(self):
        _lib.check(_lib.lib().gf_shard_prepare(self._h))

    def sample(self, iteration):
        _lib.check(_lib.lib().gf_shard_sample(self._h, int(iteration)))

    # ------------------------------------------ streamed sampling (phases) --
    def set_phases(self, num_phases):
        """Split the slice schedule into word-group phases (applies at the next load):
        an int P gives ~T/P tokens each; a sequence gives cumulative token
        fractions (strictly increasing, ending at 1.0)."""
        if np.ndim(num_phases) == 0:
            _lib.check(_lib.lib().gf_shard_set_phases(self._h, int(num_phases)))
        else:
            cuts = np.ascontiguousarray(num_phases, dtype=np.float64)
            _lib.check(_lib.lib().gf_shard_set_phase_cuts(self._h, _lib.ptr(cuts), len(cuts)))

    def set_block_phases(self, cuts):
        """Document-block phases (applies at the next load): phase 0 = the words
        not cut at document-block boundaries, phase p >= 1 = the document blocks
        starting below cuts[p-1] of the doc-major tokens (cumulative fractions,
        strictly increasing, ending at 1.0).  No theta row is streamed twice."""
        cuts = np.ascontiguousarray(cuts, dtype=np.float64)
        _lib.check(_lib.lib().gf_shard_set_block_phases(self._h, _lib.ptr(cuts), len(cuts)))

    def phase_doc_range(self, phase):
        """(tok_begin, tok_end) in doc-major order: final once phases 0..phase ran."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.lib().gf_shard_phase_doc_range(self._h, int(phase), ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    @property
    def num_phases(self):
        n = ctypes.c_int()
        _lib.check(_lib.lib().gf_shard_num_phases(self._h, ctypes.byref(n)))
        return n.value

    def phase_range(self, phase):
        """(tok_begin, tok_end): the assignments (word-group order) phase `phase` samples."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.lib().gf_shard_phase_range(self._h, int(phase), ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def sample_phase(self, iteration, phase):
        _lib.check(_lib.lib().gf_shard_sample_phase(self._h, int(iteration), int(phase)))

    def sample_export(self, iteration):
        """K1 over every phase with each phase's new assignments copied back
        while the later phases sample (gf_shard_sample_export); returns them
        (word-group order) in a pinned block."""
        out = _lib.pinned_empty(self.num_tokens, np.uint16)
        _lib.check(_lib.lib().gf_shard_sample_export(self._h, int(iteration), _lib.ptr(out)))
        return out

    def iterate(self, iteration):
        _lib.check(_lib.lib().gf_shard_iterate(self._h, int(iteration)))

    def initialize(self):
        """Counts from the initial assignments (one GPU: replica == global)."""
        self.rebuild_phi()
        self.prepare()
        self.rebuild_theta()
        self.check_errors()

    def loglik_sum_async(self, out, stream=None):
        """Enqueue the loglik read without blocking: `out` is a pinned float64
        array of 2; after the stream reaches the copy, out[0] - out[1] is the
        value loglik_sum() returns."""
        if out.dtype != np.float64 or len(out) < 2 or not out.flags.c_contiguous:
            raise ValueError("out must be a contiguous float64 array of >= 2 entries")
        handle = getattr(stream, "cuda_stream", stream)
        _lib.check(_lib.lib().gf_shard_loglik_sum_async(self._h, _lib.ptr(out),
                                                        ctypes.c_void_p(int(handle)) if handle else None))

    def loglik_sum(self):
        v = ctypes.c_double()
        _lib.check(_lib.lib().gf_shard_loglik_sum(self._h, ctypes.byref(v)))
        return v.value

    def check_errors(self):
        _lib.check(_lib.lib().gf_shard_check_errors(self._h))

    def synchronize(self):
        _lib.check(_lib.lib().gf_shard_synchronize(self._h))

    def sync_tensor(self):
        """The phi sync buffer as a torch int32 CUDA tensor (zero-copy)."""
        import torch

        p = ctypes.c_void_p()
        n = ctypes.c_int64()
        _lib.check(_lib.lib().gf_shard_sync_buffer(self._h, ctypes.byref(p), ctypes.byref(n)))
        return torch.as_tensor(_CudaArray(p.value, n.value, "<i4", self), device=f"cuda:{self.device}")

    # ------------------------------------------- peer-memory phi exchange --
    PEER_HANDLE_BYTES = 128

    def peer_handle(self):
        """IPC handles (bytes) of this shard's sync buffer and signal slots."""
        buf = ctypes.create_string_buffer(self.PEER_HANDLE_BYTES)
        _lib.check(_lib.lib().gf_shard_peer_handle(self._h, buf))
        return buf.raw

    def peer_open(self, rank, world, handles):
        """Map the other ranks' buffers; `handles` = the ranks' peer_handle() in rank order."""
        blob = b"".join(handles)
        if len(handles) != world or len(blob) != world * self.PEER_HANDLE_BYTES:
            raise ValueError("need one peer handle per rank")
        _lib.check(_lib.lib().gf_shard_peer_open(self._h, int(rank), int(world), blob))

    def peer_allreduce(self):
        """Sum the sync buffers of the peer group in place (stream-ordered)."""
        _lib.check(_lib.lib().gf_shard_peer_allreduce(self._h))

    def rebuild_phi_exchange(self):
        """K2X: rebuild the replica and sum it over the peer group in one kernel."""
        _lib.check(_lib.lib().gf_shard_rebuild_phi_exchange(self._h))

    def peer_close(self):
        _lib.check(_lib.lib().gf_shard_peer_close(self._h))

    # --------------------------------------------------------- import/export --
    @property
    def num_tokens(self):
        return self._shape[0]

    @property
    def num_docs(self):
        return self._shape[1]

    def get_assignments(self):
        out = _lib.pinned_empty(self.num_tokens, np.uint16)
        _lib.check(_lib.lib().gf_shard_get_assignments(self._h, _lib.ptr(out)))
        return out

    def get_assignments_into(self, out):
        if out.dtype != np.uint16 or not out.flags.c_contiguous or len(out) != self.num_tokens:
            raise ValueError("out must be a contiguous uint16 array of num_tokens entries")
        _lib.check(_lib.lib().gf_shard_get_assignments(self._h, _lib.ptr(out)))
        return out

    def set_assignments(self, z):
        z = _lib.carr(z, np.uint16)
        if len(z) != self.num_tokens:
            raise ValueError("assignments length mismatch")
        _lib.check(_lib.lib().gf_shard_set_assignments(self._h, _lib.ptr(z)))

    def copy_assignments_async(self, host, offset, count, to_device, stream=None):
        """Asynchronous copy of assignments [offset, offset + count) between the
        pinned uint16 `host` array (full length) and the device, on `stream`
        (torch.cuda.Stream / raw handle; None: the shard's stream)."""
        if host.dtype != np.uint16 or not host.flags.c_contiguous or len(host) != self.num_tokens:
            raise ValueError("host must be a contiguous uint16 array of num_tokens entries")
        handle = getattr(stream, "cuda_stream", stream)
        _lib.check(_lib.lib().gf_shard_copy_assignments_async(
            self._h, _lib.ptr(host), int(offset), int(count), 1 if to_device else 0,
            ctypes.c_void_p(int(handle)) if handle else None))

    def assignments_imported(self):
        """After a complete host -> device import by copy_assignments_async
        (stream-ordered after it): refresh the doc-major copy, counts go stale."""
        _lib.check(_lib.lib().gf_shard_assignments_imported(self._h))

    def copy_doc_assignments_async(self, host, offset, count, to_device, stream=None):
        """copy_assignments_async in the shard's document-major order (per
        document its tokens by word group, heavy words first)."""
        if host.dtype != np.uint16 or not host.flags.c_contiguous or len(host) != self.num_tokens:
            raise ValueError("host must be a contiguous uint16 array of num_tokens entries")
        handle = getattr(stream, "cuda_stream", stream)
        _lib.check(_lib.lib().gf_shard_copy_doc_assignments_async(
            self._h, _lib.ptr(host), int(offset), int(count), 1 if to_device else 0,
            ctypes.c_void_p(int(handle)) if handle else None))

    def doc_assignments_imported(self):
        """After a complete doc-major host -> device import (stream-ordered)."""
        _lib.check(_lib.lib().gf_shard_doc_assignments_imported(self._h))

    def get_theta(self):
        """(row_ptr int64[D_s+1], topic_ids uint16, counts uint16) of local rows."""
        nnz = ctypes.c_int64()
        _lib.check(_lib.lib().gf_shard_theta_nnz(self._h, ctypes.byref(nnz)))
        rp = _lib.pinned_empty(self.num_docs + 1, np.int64)
        ids = _lib.pinned_empty(nnz.value, np.uint16)
        cn = _lib.pinned_empty(nnz.value, np.uint16)
        _lib.check(_lib.lib().gf_shard_get_theta(self._h, _lib.ptr(rp), _lib.ptr(ids), _lib.ptr(cn)))
        return rp, ids, cn

    def set_theta(self, row_ptr, topic_ids, counts):
        rp = _lib.carr(row_ptr, np.int64)
        ids = _lib.carr(topic_ids, np.uint16)
        cn = _lib.carr(counts, np.uint16)
        if len(rp) != self.num_docs + 1:
            raise ValueError("theta row_ptr must have num_local_docs + 1 entries")
        _lib.check(_lib.lib().gf_shard_set_theta(self._h, _lib.ptr(rp), _lib.ptr(ids), _lib.ptr(cn)))

    def get_phi(self, width=32):
        """(counts [K, V] row-major, uint32 -- or uint16 for width 16, which
        raises the reference's overflow text for a cell above 65535 --,
        topic_totals int64[K]) from the sync buffer."""
        kv = _lib.pinned_empty((self.K, self.V), np.uint16 if width == 16 else np.uint32)
        tot = np.empty(self.K, np.int64)
        _lib.check(_lib.lib().gf_shard_get_phi_w(self._h, _lib.ptr(kv), int(width), _lib.ptr(tot)))
        return kv, tot

    def set_phi(self, counts, totals):
        """Import a K x V PhiMatrix (uint16 or uint32 cells, as given)."""
        kv = np.ascontiguousarray(counts)
        if kv.dtype not in (np.uint16, np.uint32):
            kv = kv.astype(np.uint32)
        tot = _lib.carr(totals, np.int64)
        if kv.shape != (self.K, self.V):
            raise ValueError(f"phi must be {self.K} x {self.V}")
        _lib.check(_lib.lib().gf_shard_set_phi_w(self._h, _lib.ptr(kv), kv.dtype.itemsize * 8, _lib.ptr(tot)))

    def set_params(self, alpha, beta, seed):
        """gf_shard_set_params: new hyper-parameters / Philox key, same shard."""
        _lib.check(_lib.lib().gf_shard_set_params(self._h, float(alpha), float(beta),
                                                  int(seed) & 0xFFFFFFFFFFFFFFFF))
        self.alpha, self.beta = float(alpha), float(beta)

    def phi_argmax(self):
        m = ctypes.c_int64()
        k = ctypes.c_int32()
        v = ctypes.c_int32()
        _lib.check(_lib.lib().gf_shard_phi_argmax(self._h, ctypes.byref(m), ctypes.byref(k), ctypes.byref(v)))
        return m.value, k.value, v.value

    def check_phi_width(self, width):
        """model.py:152-157: raise naming the argmax cell if it exceeds `width`."""
        if width == 16:
            m, k, v = self.phi_argmax()
            if m > 65535:
                raise CountOverflowError(f"phi cell (topic {k}, word {v}) count {m} exceeds 16-bit range")

    # ---------------------------------------------------- K5 conservation --
    def conservation(self, stage, num_tokens=0):
        """gf_shard_conservation: stage 1 reduces the resident theta / phi and
        returns the row report (code, global doc, row sum, length); stage 2
        compares the (possibly rank-summed) theta column sums, the phi row sums
        and sum n_k with n_k / num_tokens.  Reports: model.conservation_report."""
        rep = np.zeros(4, np.int64)
        _lib.check(_lib.lib().gf_shard_conservation(self._h, int(stage), int(num_tokens), _lib.ptr(rep)))
        return tuple(int(x) for x in rep)

    def conservation_columns(self):
        """The K theta column sums of stage 1 as a torch int64 CUDA tensor
        (zero-copy) for a cross-rank allreduce before stage 2."""
        import torch

        p = ctypes.c_void_p()
        n = ctypes.c_int64()
        _lib.check(_lib.lib().gf_shard_conservation_buffer(self._h, ctypes.byref(p), ctypes.byref(n)))
        return torch.as_tensor(_CudaArray(p.value, n.value, "<i8", self), device=f"cuda:{self.device}")

    # ------------------------------------------------------------ counters --
    def stats(self):
        st = np.zeros(11, np.int64)
        _lib.check(_lib.lib().gf_shard_stats(self._h, _lib.ptr(st), 11))
        keys = ["sample_bytes", "phi_bytes", "theta_bytes", "runs", "slices", "tokens", "theta_nnz",
                "kernels_per_iterate", "sample_launches", "word_contexts", "doc_blocks"]
        return dict(zip(keys, st.tolist()))

    def reset_stats(self):
        _lib.check(_lib.lib().gf_shard_reset_stats(self._h))

    def last_times(self):
        ms = np.zeros(4, np.float32)
        _lib.check(_lib.lib().gf_shard_last_times(self._h, _lib.ptr(ms), 4))
        return dict(zip(["sample", "phi", "prepare", "theta_exposed"], ms.tolist()))
