"""Corpus and word-grouped chunks -- the reference's data layout (corpus.py).

`Corpus` / `Chunk` keep the reference's fields and dtypes (corpus.py:20-39,
160-198) because they are the interchange format of the drop-in API.  The
chunking itself (greedy boundaries, stable word sort, group directory,
doc-word map, splitmix64 initial topics) runs in the native library
(gf_greedy_boundaries / gf_partition_chunk) and is bit-identical to the
reference (tests/test_host_native.py against tests/golden/partition.npz).
"""

import os
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .errors import CorpusFormatError, PartitionError


@dataclass(frozen=True)
class Corpus:
    """corpus.py:20-39.  Token order is grouped by document; no empty docs."""

    num_docs: int
    vocab_size: int
    num_tokens: int
    doc_lengths: np.ndarray  # int64[num_docs]
    doc_ptr: np.ndarray  # int64[num_docs + 1]
    doc_ids: np.ndarray  # int32[num_tokens]
    word_ids: np.ndarray  # int32[num_tokens]
    vocab: list

    def doc_slice(self, d):
        return slice(int(self.doc_ptr[d]), int(self.doc_ptr[d + 1]))


def corpus_from_tokens(doc_ids, word_ids, vocab_size, vocab=None):
    """corpus.py:42-76: stable doc sort, drop empty documents, compact ids."""
    doc_ids = np.asarray(doc_ids, dtype=np.int64)
    word_ids = np.asarray(word_ids, dtype=np.int64)
    if doc_ids.size == 0:
        raise CorpusFormatError("corpus has no tokens")
    if word_ids.min() < 0 or word_ids.max() >= vocab_size:
        raise CorpusFormatError("word id outside [0, vocab_size)")
    if doc_ids.size > 1 and np.any(doc_ids[1:] < doc_ids[:-1]):
        order = np.argsort(doc_ids, kind="stable")
        doc_ids, word_ids = doc_ids[order], word_ids[order]
    kept, inverse = np.unique(doc_ids, return_inverse=True)
    doc_ids = inverse.astype(np.int32)
    lengths = np.bincount(doc_ids, minlength=len(kept)).astype(np.int64)
    ptr = np.zeros(len(kept) + 1, dtype=np.int64)
    np.cumsum(lengths, out=ptr[1:])
    return Corpus(
        num_docs=len(kept),
        vocab_size=int(vocab_size),
        num_tokens=int(doc_ids.size),
        doc_lengths=lengths,
        doc_ptr=ptr,
        doc_ids=doc_ids,
        word_ids=word_ids.astype(np.int32),
        vocab=vocab if vocab is not None else _LazyVocab(int(vocab_size)),
    )


def _read_bow_header(lines):
    """corpus.py:79-91: the three UCI header lines (D, W, NNZ)."""
    if len(lines) < 3:
        raise CorpusFormatError("docword header truncated: expected 3 lines")
    out = []
    for lineno, raw in enumerate(lines[:3], start=1):
        try:
            out.append(int(raw.strip()))
        except ValueError:
            raise CorpusFormatError(f"docword line {lineno}: malformed header value {raw.strip()!r}") from None
    return tuple(out)


def _read_vocab(vocab_path, num_words):
    """corpus.py:148-157."""
    with open(vocab_path, "r", encoding="utf-8") as fh:
        vocab = [line.rstrip("\n") for line in fh]
    while vocab and vocab[-1] == "":
        vocab.pop()
    if len(vocab) != num_words:
        raise CorpusFormatError(f"vocab file has {len(vocab)} entries, docword header says {num_words}")
    return vocab


def load_uci_bow(docword_path, vocab_path):
    """corpus.py:94-145: a UCI bag-of-words corpus (docword + vocab files).
    Native parse (gf_uci_scan / gf_uci_tokens: same checks, same error texts)
    and expansion of each "docID wordID count" triple into `count` tokens in
    document order; empty documents are dropped."""
    import ctypes

    path = os.fsencode(docword_path)
    hdr = np.zeros(3, np.int64)
    n = ctypes.c_int64()
    _lib.check(_lib.lib().gf_uci_scan(path, _lib.ptr(hdr), ctypes.byref(n)))
    num_words = int(hdr[1])
    vocab = _read_vocab(vocab_path, num_words)
    if n.value == 0:
        raise CorpusFormatError("corpus has no tokens")
    docs = np.empty(n.value, np.int32)
    words = np.empty(n.value, np.int32)
    nd = ctypes.c_int64()
    _lib.check(_lib.lib().gf_uci_tokens(path, n.value, _lib.ptr(docs), _lib.ptr(words), ctypes.byref(nd)))
    lengths = np.bincount(docs, minlength=nd.value).astype(np.int64)
    ptr = np.zeros(nd.value + 1, np.int64)
    np.cumsum(lengths, out=ptr[1:])
    return Corpus(num_docs=int(nd.value), vocab_size=num_words, num_tokens=int(n.value), doc_lengths=lengths,
                  doc_ptr=ptr, doc_ids=docs, word_ids=words, vocab=vocab)


class _LazyVocab(list):
    """["w0", "w1", ...] without materialising 1M strings up front."""

    def __init__(self, n):
        super().__init__()
        self._n = n

    def __len__(self):
        return self._n

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [f"w{v}" for v in range(*i.indices(self._n))]
        if i < 0:
            i += self._n
        if not 0 <= i < self._n:
            raise IndexError(i)
        return f"w{i}"

    def __iter__(self):
        return (f"w{v}" for v in range(self._n))


@dataclass(frozen=True)
class Chunk:
    """corpus.py:160-198: whole documents [doc_lo, doc_hi), word-grouped."""

    chunk_id: int
    doc_lo: int
    doc_hi: int
    token_count: int
    doc_ids: np.ndarray  # int32[token_count], global doc ids
    word_ids: np.ndarray  # int32[token_count]
    assignments: np.ndarray  # uint16[token_count]
    group_words: np.ndarray  # int32[num_groups]
    group_offsets: np.ndarray  # int64[num_groups]
    group_sizes: np.ndarray  # int64[num_groups]
    dw_ptr: np.ndarray  # int64[num_local_docs + 1]
    dw_tok: np.ndarray  # int64[token_count]

    @property
    def num_local_docs(self):
        return self.doc_hi - self.doc_lo

    @property
    def num_groups(self):
        return len(self.group_words)

    def word_groups(self):
        for w, off, size in zip(self.group_words, self.group_offsets, self.group_sizes):
            yield int(w), slice(int(off), int(off + size))

    def doc_token_positions(self, local_doc):
        return self.dw_tok[self.dw_ptr[local_doc] : self.dw_ptr[local_doc + 1]]


def _doc_word_map(doc_ids, doc_lo, num_local_docs):
    """corpus.py:201-207: positions of each local document's tokens, ascending."""
    local = np.asarray(doc_ids).astype(np.int64) - doc_lo
    dw_tok = np.argsort(local, kind="stable").astype(np.int64)
    counts = np.bincount(local, minlength=num_local_docs)
    dw_ptr = np.zeros(num_local_docs + 1, dtype=np.int64)
    np.cumsum(counts, out=dw_ptr[1:])
    return dw_ptr, dw_tok


def greedy_boundaries(doc_lengths, num_chunks):
    """corpus.py:210-237 (native)."""
    L = _lib.carr(doc_lengths, np.int64)
    if num_chunks > len(L):
        raise PartitionError(
            f"cannot give every chunk a document: {num_chunks} chunks > {len(L)} docs"
        )
    out = np.empty(2 * max(num_chunks, 1), dtype=np.int64)
    _lib.check(_lib.lib().gf_greedy_boundaries(_lib.ptr(L), len(L), int(num_chunks), _lib.ptr(out)))
    return [(int(out[2 * c]), int(out[2 * c + 1])) for c in range(num_chunks)]


def make_chunk(chunk_id, lo, hi, doc_ids, word_ids, vocab_size, num_topics, seed, device=None):
    """One chunk of partition() from its doc-major tokens (corpus.py:252-286):
    on the host (native counting sorts), or with `device` on that GPU (K4:
    stable radix sorts + splitmix64 z0 on the device; bit-identical)."""
    docs = _lib.carr(doc_ids, np.int32)
    words = _lib.carr(word_ids, np.int32)
    n = len(docs)
    out_doc = np.empty(n, np.int32)
    out_word = np.empty(n, np.int32)
    out_z = np.empty(n, np.uint16)
    gw = np.empty(vocab_size, np.int32)
    go = np.empty(vocab_size, np.int64)
    gs = np.empty(vocab_size, np.int64)
    ng = np.zeros(1, np.int64)
    dw_ptr = np.empty(hi - lo + 1, np.int64)
    dw_tok = np.empty(n, np.int64)
    args = (_lib.ptr(docs), _lib.ptr(words), n, lo, hi, vocab_size, num_topics,
            int(seed) & 0xFFFFFFFFFFFFFFFF, chunk_id, _lib.ptr(out_doc), _lib.ptr(out_word),
            _lib.ptr(out_z), _lib.ptr(gw), _lib.ptr(go), _lib.ptr(gs), _lib.ptr(ng),
            _lib.ptr(dw_ptr), _lib.ptr(dw_tok))
    if device is None:
        _lib.check(_lib.lib().gf_partition_chunk(*args))
    else:
        _lib.check(_lib.lib().gf_partition_chunk_gpu(int(device), *args))
    k = int(ng[0])
    return Chunk(chunk_id=chunk_id, doc_lo=lo, doc_hi=hi, token_count=n, doc_ids=out_doc,
                 word_ids=out_word, assignments=out_z, group_words=gw[:k].copy(),
                 group_offsets=go[:k].copy(), group_sizes=gs[:k].copy(), dw_ptr=dw_ptr, dw_tok=dw_tok)


def partition(corpus, num_chunks, num_topics, seed, device=None):
    """corpus.py:240-287: C chunks of whole documents, word-grouped, with
    initial topics from Stream(seed, chunk_id).  `device`: run the sorts and
    z0 on that GPU (K4, bit-identical to the host path)."""
    if num_chunks < 1:
        raise PartitionError("need at least one chunk")
    if not 1 <= num_topics < 2**16:
        raise ValueError(f"topic count {num_topics} outside [1, 65536)")
    chunks = []
    for cid, (lo, hi) in enumerate(greedy_boundaries(corpus.doc_lengths, num_chunks)):
        a, b = int(corpus.doc_ptr[lo]), int(corpus.doc_ptr[hi])
        chunks.append(make_chunk(cid, lo, hi, corpus.doc_ids[a:b], corpus.word_ids[a:b],
                                 corpus.vocab_size, num_topics, seed, device=device))
    return chunks


def sort_word_groups_desc(chunk):
    """corpus.py:290-302: directory by (-size, +word); token arrays untouched."""
    order = np.lexsort((chunk.group_words, -chunk.group_sizes))
    return replace(
        chunk,
        group_words=chunk.group_words[order],
        group_offsets=chunk.group_offsets[order],
        group_sizes=chunk.group_sizes[order],
    )


# ----------------------------------------------------------- chunk store ----
CHUNK_MAGIC = b"GFCHUNK1"
_DIR_RECORD = np.dtype([("word", "<u4"), ("offset", "<u8"), ("len", "<u8")])   # packed, 20 bytes


def save_chunk(chunk, path):
    """corpus.py:305-327 chunk store (GFCHUNK1, little-endian): magic; u64
    chunk_id, doc_lo, doc_hi, token_count; doc ids u32[T], word ids u32[T],
    topics u16[T] in word-group order; the group directory as packed (word u32,
    offset u64, len u64) records in processing order.  The assignments are the
    part a model snapshot lacks, so this is the resume checkpoint."""
    import struct

    rec = np.empty(len(chunk.group_words), dtype=_DIR_RECORD)
    rec["word"] = chunk.group_words
    rec["offset"] = chunk.group_offsets
    rec["len"] = chunk.group_sizes
    with open(path, "wb") as fh:
        fh.write(CHUNK_MAGIC)
        fh.write(struct.pack("<4Q", int(chunk.chunk_id), int(chunk.doc_lo), int(chunk.doc_hi), int(chunk.token_count)))
        for arr, dt in ((chunk.doc_ids, "<u4"), (chunk.word_ids, "<u4"), (chunk.assignments, "<u2")):
            fh.write(np.ascontiguousarray(arr).astype(dt, copy=False).tobytes())
        fh.write(rec.tobytes())


def load_chunk(path):
    """corpus.py:330-364: read a GFCHUNK1 chunk; the doc-word map is rebuilt."""
    import struct

    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[: len(CHUNK_MAGIC)] != CHUNK_MAGIC:
        raise CorpusFormatError(f"{path}: bad chunk magic")
    pos = len(CHUNK_MAGIC)
    if len(blob) < pos + 32:
        raise CorpusFormatError(f"{path}: truncated header")
    cid, lo, hi, n = struct.unpack_from("<4Q", blob, pos)
    pos += 32
    if len(blob) < pos + 10 * n:
        raise CorpusFormatError(f"{path}: truncated token arrays")
    docs = np.frombuffer(blob, dtype="<u4", count=n, offset=pos).astype(np.int32)
    pos += 4 * n
    words = np.frombuffer(blob, dtype="<u4", count=n, offset=pos).astype(np.int32)
    pos += 4 * n
    topics = np.frombuffer(blob, dtype="<u2", count=n, offset=pos).astype(np.uint16)
    pos += 2 * n
    if (len(blob) - pos) % _DIR_RECORD.itemsize:
        raise CorpusFormatError(f"{path}: truncated group directory")
    rec = np.frombuffer(blob, dtype=_DIR_RECORD, offset=pos)
    dw_ptr, dw_tok = _doc_word_map(docs, int(lo), int(hi - lo))
    return Chunk(chunk_id=int(cid), doc_lo=int(lo), doc_hi=int(hi), token_count=int(n), doc_ids=docs,
                 word_ids=words, assignments=topics, group_words=rec["word"].astype(np.int32),
                 group_offsets=rec["offset"].astype(np.int64), group_sizes=rec["len"].astype(np.int64),
                 dw_ptr=dw_ptr, dw_tok=dw_tok)
