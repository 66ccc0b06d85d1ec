"""CPU ORACLE for the gibbsflow hot path -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference package `gibbsflow` (/root/reference/pkg) and of
the SPEC sections for the parts the package does not implement (sampler,
engine, eval).  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import this module, and only as
the checker or the CPU baseline; the product package
(`paper_1803_04631_b200`) never imports it.

Numeric work lives in `gf_oracle.c` (plain C, OpenMP), loaded by ctypes from
`oracle/_build/libgforacle.so` (built by `make -C oracle`, which
`__graft_entry__.build()` runs).  Small bookkeeping (directory sort, pairwise
reduce, conservation report) is numpy here, each citing its reference line.

Parity pinning: tests/test_oracle_golden.py checks every function below that
has reference code against tests/golden/* (generated from the reference by
tests/golden/make_golden.py).  The sampler / loglik have no reference code and
are pinned by SPEC examples + analytic tests ("sampler parity pinned by SPEC
examples and exact distributions").
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libgforacle.so")
_lib = None

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_f64 = ctypes.c_double


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        L.gfo_stream_key.restype = _u64
        L.gfo_stream_key.argtypes = [_p, ctypes.c_int]
        L.gfo_stream_uniforms.argtypes = [_u64, _u64, _i64, _p]
        L.gfo_philox4x32_10.argtypes = [_p, _p, _p]
        L.gfo_token_uniforms.argtypes = [_u64, _u32, _u32, _u32, _u32, _p, _p]
        L.gfo_greedy_boundaries.restype = ctypes.c_int
        L.gfo_greedy_boundaries.argtypes = [_p, _i64, _i64, _p]
        L.gfo_partition_chunk.restype = _i64
        L.gfo_partition_chunk.argtypes = [_p, _p, _i64, _i64, _i64, _i32, _i32, _u64, _i64] + [_p] * 8
        L.gfo_rebuild_theta.restype = ctypes.c_int
        L.gfo_rebuild_theta.argtypes = [_p, _p, _p, _i64, _i32, _i64, _p, _p, _p, _p, _p]
        L.gfo_rebuild_phi.argtypes = [_p, _p, _i64, _i32, _i32, _p, _p]
        L.gfo_sample_tokens.restype = ctypes.c_int
        L.gfo_sample_tokens.argtypes = [_i32, _i32, _f64, _f64, _u64, _u32, _i64, _p, _p, _p,
                                        _i64, _p, _p, _p, _p, _p, ctypes.c_int, _p]
        L.gfo_sample_tokens_thin.restype = ctypes.c_int
        L.gfo_sample_tokens_thin.argtypes = L.gfo_sample_tokens.argtypes
        L.gfo_conditional.argtypes = [_i32, _i32, _f64, _f64, _p, _p, _p, _i32, ctypes.c_int, _p, _p]
        L.gfo_loglik_naive.restype = _f64
        L.gfo_loglik_naive.argtypes = [_i32, _i32, _f64, _f64, _i64, _p, _p, _p, _p, _p, _p, _p, _p,
                                       ctypes.c_int]
        L.gfo_loglik_sq.restype = _f64
        L.gfo_loglik_sq.argtypes = [_i32, _i32, _f64, _f64, _i64, _p, _p, _i64, _p, _p, _p, _p, _p, _p,
                                    ctypes.c_int]
        L.gfo_synth_lengths.restype = ctypes.c_int
        L.gfo_synth_lengths.argtypes = [_u64, _i64, _i64, _f64, _f64, _p]
        L.gfo_synth_tokens.restype = ctypes.c_int
        L.gfo_synth_tokens.argtypes = [_u64, _i64, _i64, _p, _i32, _i32, _f64, _f64, _p, _p]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------- rng.py ----
def ptree_levels(weights, fanout, dtype):
    """ptree.py:116-136: level 0 = left-to-right cumsum in `dtype`, each level
    above keeps every fanout-th boundary (clamped to the last)."""
    levels = [np.cumsum(np.asarray(weights).astype(dtype, copy=False), dtype=dtype)]
    while len(levels[-1]) > 1:
        prev = levels[-1]
        tails = np.minimum(np.arange(fanout - 1, len(prev) + fanout - 1, fanout), len(prev) - 1)
        levels.append(prev[tails])
    return levels


def ptree_descend(levels, fanout, u):
    """ptree.py:77-99 as a plain loop (small cases only): (index, levels
    visited, widest scan) -- the first child whose boundary exceeds u, else
    the last child."""
    u = levels[0].dtype.type(u)
    idx = visited = widest = 0
    for level in range(len(levels) - 2, -1, -1):
        bounds = levels[level]
        lo = idx * fanout
        hi = min(lo + fanout, len(bounds))
        idx = hi - 1
        for j in range(lo, hi):
            if bounds[j] > u:
                idx = j
                break
        visited += 1
        widest = max(widest, hi - lo)
    return idx, visited, widest


def stream_key(*parts):
    """rng.py:45-53 (mix64 over uint64-masked parts)."""
    arr = np.array([p & 0xFFFFFFFFFFFFFFFF for p in parts], dtype=np.uint64)
    return np.uint64(lib().gfo_stream_key(_ptr(arr), len(arr)))


def stream_uniforms(parts, n, counter=0):
    """Stream(*parts).uniforms(n) after `counter` draws (rng.py:56-81, 84-89)."""
    out = np.empty(n, dtype=np.float64)
    lib().gfo_stream_uniforms(int(stream_key(*parts)), counter, n, _ptr(out))
    return out


def philox4x32_10(ctr, key):
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    out = np.empty(4, dtype=np.uint32)
    lib().gfo_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def token_uniforms(seed, iteration, doc, word, occ):
    u1, u2 = _f64(), _f64()
    lib().gfo_token_uniforms(seed, iteration, doc, word, occ, ctypes.byref(u1), ctypes.byref(u2))
    return u1.value, u2.value


# ------------------------------------------------- synthetic corpora ----
def synth_lengths(seed, num_docs, mean_len, sigma=0.6, doc_begin=0):
    """Document lengths of the benchmark corpus (gf_synth_ref.c; equal to the
    product generator's gf_synth_lengths)."""
    out = np.empty(int(num_docs), np.int64)
    if lib().gfo_synth_lengths(seed & 0xFFFFFFFFFFFFFFFF, int(doc_begin), int(num_docs), float(mean_len),
                               float(sigma), _ptr(out)) != 0:
        raise ValueError("bad synthetic corpus shape")
    return out


def synth_generate(num_docs, vocab_size, mean_len, seed=20261017, k_true=100, zipf_s=1.07, doc_alpha=0.1,
                   sigma=0.6, doc_begin=0):
    """Documents [doc_begin, doc_begin + num_docs) of the benchmark corpus as a
    corpus_from_tokens dict (doc ids relative to doc_begin) -- the arrays
    paper_1803_04631_b200.synth.generate returns, without the product library."""
    lengths = synth_lengths(seed, num_docs, mean_len, sigma, doc_begin)
    ptr = np.zeros(len(lengths) + 1, np.int64)
    np.cumsum(lengths, out=ptr[1:])
    T = int(ptr[-1])
    docs = np.empty(T, np.int32)
    words = np.empty(T, np.int32)
    if lib().gfo_synth_tokens(seed & 0xFFFFFFFFFFFFFFFF, int(doc_begin), int(num_docs), _ptr(ptr), int(vocab_size),
                              int(k_true), float(zipf_s), float(doc_alpha), _ptr(docs), _ptr(words)) != 0:
        raise ValueError("bad synthetic corpus shape")
    if doc_begin:
        docs -= np.int32(doc_begin)
    return dict(doc_ids=docs, word_ids=words, doc_lengths=lengths, doc_ptr=ptr, D=int(num_docs),
                V=int(vocab_size), T=T)


# ------------------------------------------------------------- corpus.py ----
def corpus_from_tokens(doc_ids, word_ids, vocab_size):
    """corpus.py:42-76 restated: stable doc sort, drop empty docs, compact ids.
    Returns dict(doc_ids i32, word_ids i32, doc_lengths i64, doc_ptr i64, D, V, T)."""
    doc_ids = np.asarray(doc_ids, dtype=np.int64)
    word_ids = np.asarray(word_ids, dtype=np.int64)
    order = np.argsort(doc_ids, kind="stable")
    doc_ids, word_ids = doc_ids[order], word_ids[order]
    kept, inverse = np.unique(doc_ids, return_inverse=True)
    doc_ids = inverse.astype(np.int32)
    lengths = np.bincount(doc_ids, minlength=len(kept)).astype(np.int64)
    ptr = np.zeros(len(kept) + 1, dtype=np.int64)
    np.cumsum(lengths, out=ptr[1:])
    return dict(doc_ids=doc_ids, word_ids=word_ids.astype(np.int32), doc_lengths=lengths,
                doc_ptr=ptr, D=len(kept), V=int(vocab_size), T=int(doc_ids.size))


def greedy_boundaries(lengths, num_chunks):
    """corpus.py:210-237; raises ValueError (PartitionError) when C > D."""
    L = _c(lengths, np.int64)
    out = np.empty(2 * num_chunks, dtype=np.int64)
    if lib().gfo_greedy_boundaries(_ptr(L), len(L), num_chunks, _ptr(out)) != 0:
        raise ValueError(f"cannot give every chunk a document: {num_chunks} chunks > {len(L)} docs")
    return [(int(out[2 * c]), int(out[2 * c + 1])) for c in range(num_chunks)]


def partition(corpus, num_chunks, num_topics, seed):
    """corpus.py:240-287; returns a list of dicts with the Chunk fields."""
    chunks = []
    for cid, (lo, hi) in enumerate(greedy_boundaries(corpus["doc_lengths"], num_chunks)):
        a, b = int(corpus["doc_ptr"][lo]), int(corpus["doc_ptr"][hi])
        docs = _c(corpus["doc_ids"][a:b], np.int32)
        words = _c(corpus["word_ids"][a:b], np.int32)
        n = b - a
        out_doc = np.empty(n, np.int32)
        out_word = np.empty(n, np.int32)
        out_z = np.empty(n, np.uint16)
        gw = np.empty(corpus["V"], np.int32)
        go = np.empty(corpus["V"], np.int64)
        gs = np.empty(corpus["V"], np.int64)
        dw_ptr = np.empty(hi - lo + 1, np.int64)
        dw_tok = np.empty(n, np.int64)
        ng = lib().gfo_partition_chunk(_ptr(docs), _ptr(words), n, lo, hi, corpus["V"], num_topics,
                                       seed & 0xFFFFFFFFFFFFFFFF, cid, _ptr(out_doc), _ptr(out_word),
                                       _ptr(out_z), _ptr(gw), _ptr(go), _ptr(gs), _ptr(dw_ptr),
                                       _ptr(dw_tok))
        chunks.append(dict(chunk_id=cid, doc_lo=lo, doc_hi=hi, token_count=n, doc_ids=out_doc,
                           word_ids=out_word, assignments=out_z, group_words=gw[:ng].copy(),
                           group_offsets=go[:ng].copy(), group_sizes=gs[:ng].copy(),
                           dw_ptr=dw_ptr, dw_tok=dw_tok))
    return chunks


def sort_word_groups_desc(group_words, group_offsets, group_sizes):
    """corpus.py:290-302: (-size, +word) order of the directory."""
    order = np.lexsort((group_words, -np.asarray(group_sizes)))
    return group_words[order], group_offsets[order], group_sizes[order]


# -------------------------------------------------------------- model.py ----
class OracleOverflow(Exception):
    pass


def rebuild_theta(z, dw_ptr, dw_tok, doc_lo, num_topics):
    """model.py:91-124.  Raises OracleOverflow(doc, count) like CountOverflowError."""
    z = _c(z, np.uint16)
    dw_ptr = _c(dw_ptr, np.int64)
    dw_tok = _c(dw_tok, np.int64)
    nd = len(dw_ptr) - 1
    n = len(z)
    row_ptr = np.empty(nd + 1, np.int64)
    ids = np.empty(max(n, 1), np.uint16)
    cnts = np.empty(max(n, 1), np.uint16)
    ed, ec = _i64(), _i64()
    rc = lib().gfo_rebuild_theta(_ptr(z), _ptr(dw_ptr), _ptr(dw_tok), nd, num_topics, doc_lo,
                                 _ptr(row_ptr), _ptr(ids), _ptr(cnts), ctypes.byref(ed), ctypes.byref(ec))
    if rc:
        raise OracleOverflow(ed.value, ec.value)
    nnz = int(row_ptr[-1])
    return row_ptr, ids[:nnz].copy(), cnts[:nnz].copy()


def rebuild_phi(z, word_ids, num_topics, vocab_size):
    """model.py:142-161 (dense int64 K x V counts, int64 totals)."""
    z = _c(z, np.uint16)
    w = _c(word_ids, np.int32)
    counts = np.empty((num_topics, vocab_size), np.int64)
    totals = np.empty(num_topics, np.int64)
    lib().gfo_rebuild_phi(_ptr(z), _ptr(w), len(z), num_topics, vocab_size, _ptr(counts), _ptr(totals))
    return counts, totals


def concat_theta(parts):
    """model.py:127-139 over (row_ptr, ids, counts) triples."""
    row_ptr = [np.zeros(1, np.int64)]
    base = 0
    for rp, _, _ in parts:
        row_ptr.append(rp[1:] + base)
        base += int(rp[-1])
    return (np.concatenate(row_ptr), np.concatenate([p[1] for p in parts]),
            np.concatenate([p[2] for p in parts]))


def check_conservation(row_ptr, topic_ids, counts, phi_counts, phi_totals, doc_lengths, num_tokens):
    """model.py:180-225: first violated invariant, same texts."""
    nrows = len(row_ptr) - 1
    row_sums = np.zeros(nrows, np.int64)
    np.add.at(row_sums, np.repeat(np.arange(nrows), np.diff(row_ptr)), counts.astype(np.int64))
    bad = np.flatnonzero(row_sums != doc_lengths)
    if bad.size:
        d = int(bad[0])
        return False, f"theta row {d} sums to {int(row_sums[d])}, document length is {int(doc_lengths[d])}"
    K = phi_counts.shape[0]
    col = np.zeros(K, np.int64)
    np.add.at(col, topic_ids.astype(np.int64), counts.astype(np.int64))
    bad = np.flatnonzero(col != phi_totals)
    if bad.size:
        k = int(bad[0])
        return False, f"topic {k}: theta column sum {int(col[k])} != phi total {int(phi_totals[k])}"
    rs = phi_counts.sum(axis=1, dtype=np.int64)
    bad = np.flatnonzero(rs != phi_totals)
    if bad.size:
        k = int(bad[0])
        return False, f"topic {k}: phi row sum {int(rs[k])} != stored total {int(phi_totals[k])}"
    total = int(phi_totals.sum())
    if total != num_tokens:
        return False, f"totals sum to {total}, corpus has {num_tokens} tokens"
    return True, "ok"


# ------------------------------------------------------------- sampler ------
def sample_tokens(K, V, alpha, beta, seed, iteration, tok_doc, tok_word, z, doc_lo,
                  th_ptr, th_ids, th_cnt, phi_counts, phi_totals, nthreads=0, mode="direct"):
    """SPEC.md:249-284, 359-367 deferred sampler (fp64 oracle mode).  Returns z'.
    phi_counts is K x V; theta CSR rows are local (doc - doc_lo).
    mode="direct": exclusion-adjusted S/Q exactly as SPEC sample_sparse;
    mode="thin": the device's draw-by-draw form (exclusion by thinning)."""
    tok_doc = _c(tok_doc, np.int32)
    tok_word = _c(tok_word, np.int32)
    zz = _c(z, np.uint16).copy()
    th_ptr = _c(th_ptr, np.int64)
    th_ids = _c(th_ids, np.uint16)
    th_cnt = _c(th_cnt, np.uint16)
    phi = _c(phi_counts, np.uint32)
    tot = _c(phi_totals, np.int64)
    err = _i64()
    fn = lib().gfo_sample_tokens if mode == "direct" else lib().gfo_sample_tokens_thin
    rc = fn(K, V, alpha, beta, seed & 0xFFFFFFFFFFFFFFFF, iteration, len(zz),
                                 _ptr(tok_doc), _ptr(tok_word), _ptr(zz), doc_lo, _ptr(th_ptr),
                                 _ptr(th_ids), _ptr(th_cnt), _ptr(phi), _ptr(tot), nthreads,
                                 ctypes.byref(err))
    if rc:
        raise ValueError(f"consistency error at token {err.value}")
    return zz


def conditional(K, V, alpha, beta, theta_dense, phi_col, totals, z, exclusion=True):
    """Exact exclusion-adjusted Eq. 1 distribution and the
    S/Q-decomposed distribution."""
    th = _c(theta_dense, np.int64)
    ph = _c(phi_col, np.uint32)
    tot = _c(totals, np.int64)
    p = np.empty(K, np.float64)
    pd = np.empty(K, np.float64)
    lib().gfo_conditional(K, V, alpha, beta, _ptr(th), _ptr(ph), _ptr(tot), z, int(exclusion),
                          _ptr(p), _ptr(pd))
    return p, pd


def loglik_naive(K, V, alpha, beta, tok_doc, tok_word, th_ptr, th_ids, th_cnt, doc_len,
                 phi_counts, phi_totals, nthreads=0):
    """SPEC.md:402-410, O(T K), 64-bit.  theta rows indexed by the global doc id."""
    args = [_c(tok_doc, np.int32), _c(tok_word, np.int32), _c(th_ptr, np.int64),
            _c(th_ids, np.uint16), _c(th_cnt, np.uint16), _c(doc_len, np.int64),
            _c(phi_counts, np.uint32), _c(phi_totals, np.int64)]
    return lib().gfo_loglik_naive(K, V, alpha, beta, len(args[0]), *[_ptr(a) for a in args], nthreads)


def loglik_sq(K, V, alpha, beta, tok_doc, tok_word, doc_lo, th_ptr, th_ids, th_cnt, doc_len_local,
              phi_counts, phi_totals, nthreads=0):
    """SPEC.md:402-410 in the S + Q form, O(T K_d): word-grouped tokens (a
    partitioned chunk), theta rows and doc lengths over the chunk's local docs."""
    args = [_c(tok_doc, np.int32), _c(tok_word, np.int32)]
    rest = [_c(th_ptr, np.int64), _c(th_ids, np.uint16), _c(th_cnt, np.uint16), _c(doc_len_local, np.int64),
            _c(phi_counts, np.uint32), _c(phi_totals, np.int64)]
    return lib().gfo_loglik_sq(K, V, alpha, beta, len(args[0]), _ptr(args[0]), _ptr(args[1]), int(doc_lo),
                               *[_ptr(a) for a in rest], nthreads)


# -------------------------------------------------------------- engine ------
def reduce_phi_pairwise(replicas):
    """in round r, replica j += replica j + 2^r for j = 0 mod 2^(r+1).
    Returns (sum, rounds) where rounds lists the (src -> dst) pairs of each round."""
    reps = [np.array(r, dtype=np.int64, copy=True) for r in replicas]
    G = len(reps)
    rounds = []
    step = 1
    while step < G:
        pairs = []
        for j in range(0, G, 2 * step):
            if j + step < G:
                reps[j] += reps[j + step]
                pairs.append((j + step, j))
        rounds.append(pairs)
        step *= 2
    return reps[0], rounds
