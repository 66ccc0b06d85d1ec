"""The sparsity-aware CGS sampler on the B200.

`sample_chunk` is SPEC.md:359-367 in deferred mode: every draw of the chunk
uses the iteration-start theta / phi snapshot, the token's own contribution
excluded, two independent uniforms.  The
draw runs in K1 (csrc/k_sample.cu); the RNG is Philox4x32-10 keyed by `seed`
with counter (global doc, word, occurrence in its (doc, word) run, iteration),
so every shard / GPU count draws from the same uniforms.
"""

from dataclasses import dataclass

import numpy as np

from .model import PhiMatrix, ThetaRows


@dataclass
class SamplerContext:
    """SPEC.md:235-238."""

    alpha: float
    beta: float
    num_topics: int
    vocab_size: int
    exclusion: bool = True

    def __post_init__(self):
        if not (self.alpha > 0 and self.beta > 0):
            raise ValueError("alpha and beta must be > 0")
        if not self.exclusion:
            raise NotImplementedError("the B200 sampler always applies exclusion (SPEC.md:292)")


def _local_theta(theta, chunk):
    if theta.num_rows == chunk.num_local_docs:
        return theta.row_ptr, theta.topic_ids, theta.counts
    if theta.num_rows >= chunk.doc_hi:
        a, b = int(theta.row_ptr[chunk.doc_lo]), int(theta.row_ptr[chunk.doc_hi])
        rp = theta.row_ptr[chunk.doc_lo: chunk.doc_hi + 1] - a
        return rp, theta.topic_ids[a:b], theta.counts[a:b]
    raise ValueError("theta rows match neither the chunk nor the corpus")


def sample_chunk(chunk, phi, theta, ctx, cfg=None, iteration=0, seed=None, device=0):
    """Resample every assignment of `chunk` once; returns the new uint16 array.
    `phi` is the global PhiMatrix, `theta` the ThetaRows of the chunk's
    documents (local rows or the whole corpus).

    The chunk's shard stays resident between calls (shard.RESIDENT): a chunk
    sampled again -- the same Chunk, or a dataclasses.replace() of it with the
    new assignments -- skips the K4 layout; its assignments go through the
    staged import and theta / phi are uploaded as given (phi at its own width)
    and validated on the device."""
    from .errors import CountOverflowError
    from .shard import RESIDENT, chunk_shard

    if seed is None:
        seed = getattr(cfg, "seed", 0) if cfg is not None else 0
    args = (ctx.num_topics, ctx.vocab_size, ctx.alpha, ctx.beta, seed, device)
    sh = chunk_shard(chunk, *args)
    try:
        sh.set_phi(phi.counts, phi.topic_totals)
    except CountOverflowError:
        # the hybrid 16/32-bit columns of the chunk's own word frequencies
        # cannot hold this phi: a chunk-light word has a GLOBAL cell above
        # 65535 (C > 1).  Lay the shard out by the global frequencies instead.
        arrays = (chunk.word_ids, chunk.doc_ids, chunk.dw_tok, chunk.group_offsets)
        RESIDENT.drop(arrays, (ctx.num_topics, ctx.vocab_size, device, chunk.doc_lo, chunk.doc_hi, "chunk"))
        freq = np.asarray(phi.counts).sum(axis=0, dtype=np.int64)
        sh = chunk_shard(chunk, *args, global_word_freq=freq, layout="global")
        sh.set_phi(phi.counts, phi.topic_totals)
    sh.set_theta(*_local_theta(theta, chunk))
    sh.prepare()
    z = sh.sample_export(iteration)       # K1, the result copied back phase by phase
    sh.check_errors()
    return z
