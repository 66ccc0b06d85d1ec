"""Quality / throughput metrics."""

import numpy as np



def loglik_per_token(theta, phi, corpus, alpha, beta, device=0):
    """(1/T) sum_t log sum_k (theta_dk + a)/(L_d + K a) *
    (phi_kv + b)/(n_k + V b), fp64, evaluated on the device as
    log((S_full + Q_v) / (L_d + K a)) per (doc, word) run (the same identity the
    sampler fuses).  theta holds one row per corpus document.  The corpus is
    laid out once by K4 on the device (load_tokens) and stays resident
    (shard.RESIDENT) for later calls on the same corpus arrays."""
    from . import _lib
    from .shard import RESIDENT, DeviceShard

    if corpus.num_tokens == 0:
        raise ValueError("empty corpus")
    K, V = phi.num_topics, phi.vocab_size

    def build():
        sh = DeviceShard(K, V, alpha, beta, device=device)
        return sh.load_tokens(0, corpus.num_docs, corpus.doc_ids, corpus.word_ids, seed=0)

    sh, fresh = RESIDENT.get((corpus.doc_ids, corpus.word_ids), (K, V, int(device), "eval"), build)
    if not fresh:
        sh.set_params(alpha, beta, 0)
    sh.set_phi(phi.counts, phi.topic_totals)
    sh.set_theta(theta.row_ptr, theta.topic_ids, theta.counts)
    sh.prepare()
    _lib.check(_lib.lib().gf_shard_evaluate(sh._h))
    return sh.loglik_sum() / corpus.num_tokens


def tokens_per_sec(num_tokens, iterations, elapsed):
    """SPEC.md:411-419, PAPER Eq. 2: T * iterations / elapsed."""
    if iterations == 0:
        return 0.0
    if elapsed <= 0:
        raise ValueError("elapsed must be > 0")
    return num_tokens * iterations / elapsed
