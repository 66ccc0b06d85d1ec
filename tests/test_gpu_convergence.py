"""Convergence evidence that does not lean on shared random numbers.

* An independent-seed band: the oracle's direct-mode sampler (SPEC
  sample_sparse, exact per-token conditional in fp64, oracle/gf_oracle.c) run
  with Philox keys different from the device's gives independent chains from
  the same initial state; the device trajectory must lie within 1% of the band
  they span at every matched iteration (BASELINE configs[0], 50 iterations).
* SPEC.md acceptance #7 on the device: planted disjoint-support topics (D=200,
  V=50, K=5, ~50 tokens/doc), 100 iterations, loglik_per_token up by >= 0.5
  nats over initialisation for >= 95% of 20 seeds.  The GPU runs deferred mode
  (section 6: every draw of an iteration reads the iteration-start
  counts); SPEC's "exact mode" is the sequential CPU schedule, not this path.
"""

import numpy as np
import pytest

import oracle
from paper_1803_04631_b200 import corpus as cp
from paper_1803_04631_b200 import engine, synth

pytestmark = pytest.mark.gpu


def oracle_direct_trajectory(corp, K, init_seed, philox_seed, iters):
    """Deferred iterations of the oracle's direct sampler (fp64 Eq. 1 with
    exclusion) keyed by `philox_seed`, from partition(init_seed)'s state."""
    a, b = 50.0 / K, 0.01
    ch = cp.partition(corp, 1, K, init_seed)[0]
    z = ch.assignments.copy()
    lls = []
    for it in range(iters):
        rp, ids, cn = oracle.rebuild_theta(z, ch.dw_ptr, ch.dw_tok, 0, K)
        phi, tot = oracle.rebuild_phi(z, ch.word_ids, K, corp.vocab_size)
        lls.append(oracle.loglik_naive(K, corp.vocab_size, a, b, ch.doc_ids, ch.word_ids, rp, ids, cn,
                                       corp.doc_lengths, phi, tot))
        z = oracle.sample_tokens(K, corp.vocab_size, a, b, philox_seed, it, ch.doc_ids, ch.word_ids, z, 0,
                                 rp, ids, cn, phi, tot, mode="direct")
    return np.array(lls)


def test_device_trajectory_inside_independent_seed_band():
    K, iters = 32, 50
    corp = synth.shaped("tiny")
    _, _, reps = engine.train(corp, engine.TrainConfig(num_topics=K, iterations=iters, seed=42))
    gpu = np.array([r.loglik_per_token for r in reps])
    band = np.array([oracle_direct_trajectory(corp, K, 42, s, iters) for s in (1001, 2002, 3003, 4004)])
    lo, hi = band.min(axis=0), band.max(axis=0)
    np.testing.assert_allclose(band[:, 0], band[0, 0], rtol=1e-12)   # same initial model for every chain
    assert gpu[0] == pytest.approx(band[0, 0], rel=1e-6)
    # distance outside the band, relative to the band edge (0 inside)
    out = np.maximum(lo - gpu, 0) + np.maximum(gpu - hi, 0)
    rel = out / np.abs(np.where(gpu < lo, lo, hi))
    assert rel.max() < 0.01, (rel.max(), int(rel.argmax()))
    # and the chains really are independent of the device's uniforms: the band
    # has width (seed-to-seed spread) after the first iterations
    assert (hi[5:] - lo[5:]).max() > 0
    assert gpu[-1] > gpu[0] + 0.05


def planted_corpus(seed, D=200, V=50, K=5, mean_len=50, alpha=0.1):
    """K topics with disjoint 10-word supports; per document theta ~ Dir(alpha)
    (sparse: documents are mostly about one topic -- SPEC #7 leaves the mixing
    open; with Dir(0.5) mixtures the attainable gain at alpha = 50/K is ~0.4
    nats, measured on both the device and the oracle), length ~ Poisson(mean_len)
    (>= 1), z ~ theta, w uniform over topic z's words."""
    r = np.random.default_rng(seed)
    per = V // K
    docs, words = [], []
    for d in range(D):
        th = r.dirichlet(np.full(K, alpha))
        n = max(1, int(r.poisson(mean_len)))
        z = r.choice(K, size=n, p=th)
        docs.append(np.full(n, d))
        words.append(z * per + r.integers(0, per, n))
    return cp.corpus_from_tokens(np.concatenate(docs), np.concatenate(words), V)


def test_planted_topic_convergence_spec7():
    gains = []
    for seed in range(20):
        corp = planted_corpus(1000 + seed)
        cfg = engine.TrainConfig(num_topics=5, iterations=100, seed=seed)
        tr = engine.Trainer(corp, cfg)
        first = tr.step().loglik_per_token                 # the initial model's loglik (iteration 0)
        last = first
        for _ in range(cfg.iterations - 1):
            last = tr.step().loglik_per_token
        last = tr.evaluate()                               # the model after the 100th iteration
        tr.close()
        gains.append(last - first)
        if seed < 3:                                       # the oracle's direct sampler gets the same gain
            ref = oracle_direct_trajectory(corp, 5, seed, 99 + seed, 101)
            assert abs((ref[-1] - ref[0]) - gains[-1]) < 0.05 * abs(ref[-1] - ref[0]), (ref[-1] - ref[0], gains[-1])
    gains = np.array(gains)
    assert np.mean(gains >= 0.5) >= 0.95, gains
