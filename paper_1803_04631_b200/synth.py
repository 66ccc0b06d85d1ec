"""Seeded LDA-generative synthetic corpora (gf_synth_*).

Shapes used by the benchmark (BASELINE.json configs):
  tiny     D=1,000     V=1,000    mean length 100   (~100K tokens), K=32
  nytimes  D=299,752   V=101,636  mean length 332   (~99.5M tokens), K=1024
  pubmed   D=8,200,000 V=141,043  mean length 90    (~738M tokens), K=1024
  z4shard  D=5,000,000 V=1,000,000 mean length 100  (~500M tokens): one GPU's
           document shard of BASELINE configs[4] (~4B tokens, V=1M, K=1024,
           doc-sharded across 8 B200s)
"""

import numpy as np

from . import _lib
from .corpus import Corpus, _LazyVocab

SHAPES = {
    "tiny": dict(num_docs=1_000, vocab_size=1_000, mean_len=100.0),
    "nytimes": dict(num_docs=299_752, vocab_size=101_636, mean_len=332.08),
    "pubmed": dict(num_docs=8_200_000, vocab_size=141_043, mean_len=89.98),
    "z4shard": dict(num_docs=5_000_000, vocab_size=1_000_000, mean_len=100.0),
}


def doc_lengths(seed, num_docs, mean_len, sigma=0.6, doc_begin=0):
    out = np.empty(num_docs, np.int64)
    _lib.check(_lib.lib().gf_synth_lengths(seed, doc_begin, num_docs, float(mean_len), float(sigma), _lib.ptr(out)))
    return out


def generate(num_docs, vocab_size, mean_len, seed=20261017, k_true=100, zipf_s=1.07, doc_alpha=0.1,
             sigma=0.6, doc_begin=0):
    """Corpus of documents [doc_begin, doc_begin + num_docs) (global ids kept
    relative: doc ids in the returned Corpus start at 0)."""
    lengths = doc_lengths(seed, num_docs, mean_len, sigma, doc_begin)
    ptr = np.zeros(num_docs + 1, np.int64)
    np.cumsum(lengths, out=ptr[1:])
    T = int(ptr[-1])
    docs = np.empty(T, np.int32)
    words = np.empty(T, np.int32)
    _lib.check(_lib.lib().gf_synth_tokens(seed, doc_begin, num_docs, _lib.ptr(ptr), vocab_size, k_true,
                                          float(zipf_s), float(doc_alpha), _lib.ptr(docs), _lib.ptr(words)))
    if doc_begin:
        docs -= doc_begin
    return Corpus(num_docs=num_docs, vocab_size=vocab_size, num_tokens=T, doc_lengths=lengths, doc_ptr=ptr,
                  doc_ids=docs, word_ids=words, vocab=_LazyVocab(vocab_size))


def shaped(name, seed=20261017, **kw):
    args = dict(SHAPES[name])
    args.update(kw)
    return generate(seed=seed, **args)
