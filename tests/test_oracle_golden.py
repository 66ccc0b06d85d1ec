"""Pin the CPU oracle (oracle/) to the reference package via golden vectors.

Every fixture under tests/golden/ was produced by running the reference
`gibbsflow` itself (tests/golden/make_golden.py).  Parts of the hot path that
have no reference code (sampler, loglik, reduce) are pinned by the SPEC's hand
examples and by exact-distribution / chi-square checks.
"""

import json
import os

import numpy as np
import pytest
from scipy import stats

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=False)


# ---------------------------------------------------------------- rng ------
def test_stream_keys_and_uniforms_match_reference():
    g = load("rng.npz")
    parts = json.loads(str(g["key_parts"]))
    for i, p in enumerate(parts):
        assert oracle.stream_key(*p) == g["keys"][i]
        np.testing.assert_array_equal(oracle.stream_uniforms(p, 257), g["uniforms"][i])


def test_stream_integer_draws_match_reference():
    # Stream.integer(n) = min(int(u*n), n-1)   (rng.py:116-118)
    g = load("rng.npz")
    u = oracle.stream_uniforms([5], 300)
    got = np.minimum((u * 7).astype(np.int64), 6)
    np.testing.assert_array_equal(got, g["integers_seed5_n7"])


def test_stream_counter_offset():
    a = oracle.stream_uniforms([9, 1], 100)
    b = oracle.stream_uniforms([9, 1], 60, counter=40)
    np.testing.assert_array_equal(a[40:], b)


@pytest.mark.parametrize(
    "ctr,key,expect",
    [  # Random123 kat_vectors, philox4x32_10
        ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
        ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
        ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
         [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
    ],
)
def test_philox_known_answers(ctr, key, expect):
    np.testing.assert_array_equal(oracle.philox4x32_10(ctr, key), np.array(expect, np.uint32))


# ------------------------------------------------------------- corpus ------
def test_greedy_boundaries_match_reference():
    with open(os.path.join(GOLD, "bounds.json")) as fh:
        cases = json.load(fh)
    assert len(cases) > 100
    for c in cases:
        got = oracle.greedy_boundaries(c["lengths"], c["C"])
        assert [list(b) for b in got] == c["bounds"]


def test_greedy_rejects_more_chunks_than_docs():
    with pytest.raises(ValueError):
        oracle.greedy_boundaries([3, 3], 3)


def _golden_corpora():
    g = load("partition.npz")
    return g, json.loads(str(g["meta"]))


@pytest.mark.parametrize("name", ["small", "single", "rand25", "zipf", "zipf_k1024"])
def test_partition_matches_reference(name):
    g, meta = _golden_corpora()
    m = next(x for x in meta if x["name"] == name)
    corp = oracle.corpus_from_tokens(g[f"{name}__corpus_doc_ids"], g[f"{name}__corpus_word_ids"], m["V"])
    np.testing.assert_array_equal(corp["doc_lengths"], g[f"{name}__corpus_doc_lengths"])
    chunks = oracle.partition(corp, m["C"], m["K"], m["seed"])
    assert len(chunks) == m["C"]
    for ch in chunks:
        pre = f"{name}__c{ch['chunk_id']}__"
        assert [ch["doc_lo"], ch["doc_hi"], ch["token_count"]] == g[pre + "range"].tolist()
        for f in ("doc_ids", "word_ids", "assignments", "group_words", "group_offsets",
                  "group_sizes", "dw_ptr", "dw_tok"):
            np.testing.assert_array_equal(ch[f], g[pre + f], err_msg=f)
            assert ch[f].dtype == g[pre + f].dtype, f
        gw, go, gs = oracle.sort_word_groups_desc(ch["group_words"], ch["group_offsets"], ch["group_sizes"])
        np.testing.assert_array_equal(gw, g[pre + "desc_group_words"])
        np.testing.assert_array_equal(go, g[pre + "desc_group_offsets"])
        np.testing.assert_array_equal(gs, g[pre + "desc_group_sizes"])
        # count rebuilds on the partitioned chunk
        rp, ids, cn = oracle.rebuild_theta(ch["assignments"], ch["dw_ptr"], ch["dw_tok"], ch["doc_lo"], m["K"])
        np.testing.assert_array_equal(rp, g[pre + "theta_row_ptr"])
        np.testing.assert_array_equal(ids, g[pre + "theta_topic_ids"])
        np.testing.assert_array_equal(cn, g[pre + "theta_counts"])
        pc, pt = oracle.rebuild_phi(ch["assignments"], ch["word_ids"], m["K"], m["V"])
        np.testing.assert_array_equal(pc, g[pre + "phi_counts"])
        np.testing.assert_array_equal(pt, g[pre + "phi_totals"])
    parts = [oracle.rebuild_theta(c["assignments"], c["dw_ptr"], c["dw_tok"], c["doc_lo"], m["K"]) for c in chunks]
    rp, ids, cn = oracle.concat_theta(parts)
    np.testing.assert_array_equal(rp, g[f"{name}__concat_row_ptr"])
    np.testing.assert_array_equal(ids, g[f"{name}__concat_topic_ids"])
    np.testing.assert_array_equal(cn, g[f"{name}__concat_counts"])


# -------------------------------------------------------------- model ------
def hand_chunk(doc, word, z):
    """tests/test_model.py:9-33 pattern: word-grouped chunk from triples."""
    order = np.argsort(word, kind="stable")
    doc, word, z = np.asarray(doc)[order], np.asarray(word)[order], np.asarray(z)[order]
    lo = int(doc.min())
    local = doc.astype(np.int64) - lo
    nd = int(doc.max()) + 1 - lo
    dw_tok = np.argsort(local, kind="stable").astype(np.int64)
    dw_ptr = np.zeros(nd + 1, np.int64)
    np.cumsum(np.bincount(local, minlength=nd), out=dw_ptr[1:])
    return doc, word, z.astype(np.uint16), lo, dw_ptr, dw_tok


def test_rebuilds_match_reference_on_hand_chunks():
    g = load("counts.npz")
    meta = json.loads(str(g["meta"]))
    for m in meta:
        pre = f"h{m['i']}__"
        doc, word, z, lo, dw_ptr, dw_tok = hand_chunk(g[pre + "doc"], g[pre + "word"], g[pre + "z"])
        rp, ids, cn = oracle.rebuild_theta(z, dw_ptr, dw_tok, lo, m["K"])
        np.testing.assert_array_equal(rp, g[pre + "theta_row_ptr"])
        np.testing.assert_array_equal(ids, g[pre + "theta_topic_ids"])
        np.testing.assert_array_equal(cn, g[pre + "theta_counts"])
        pc, pt = oracle.rebuild_phi(z, word, m["K"], m["V"])
        np.testing.assert_array_equal(pc, g[pre + "phi_counts"])
        np.testing.assert_array_equal(pt, g[pre + "phi_totals"])


def test_overflow_messages_match_reference():
    with open(os.path.join(GOLD, "messages.json")) as fh:
        msgs = json.load(fh)
    n = 70000
    doc, word, z, lo, dw_ptr, dw_tok = hand_chunk(np.full(n, 3), np.zeros(n, int), np.zeros(n, int))
    with pytest.raises(oracle.OracleOverflow) as ei:
        oracle.rebuild_theta(z, dw_ptr, dw_tok, lo, 2)
    d, c = ei.value.args
    assert f"document {d}: topic count {c} exceeds 16-bit range" == msgs["theta_overflow_doc3"]


def conservation_cases():
    """The four states make_golden.py hands to the reference's
    check_conservation (model.py:180-225) for messages.json."""

    def model(lengths, V, K, seed):
        r = np.random.default_rng(seed)
        doc_ids = np.repeat(np.arange(len(lengths)), lengths)
        corp = oracle.corpus_from_tokens(doc_ids, r.integers(0, V, doc_ids.size), V)
        chunks = oracle.partition(corp, min(3, corp["D"]), K, seed)
        parts = [oracle.rebuild_theta(c["assignments"], c["dw_ptr"], c["dw_tok"], c["doc_lo"], K) for c in chunks]
        rp, ids, cn = oracle.concat_theta(parts)
        phi = np.zeros((K, V), np.int64)
        tot = np.zeros(K, np.int64)
        for c in chunks:
            pc, pt = oracle.rebuild_phi(c["assignments"], c["word_ids"], K, V)
            phi += pc
            tot += pt
        return corp, rp, ids, cn, phi, tot

    out = [("conservation_ok",) + model([5, 8, 3, 9], 7, 3, 1)]
    corp, rp, ids, cn, phi, tot = model([5, 8, 3, 9], 7, 3, 2)
    phi[1, 0] += 1
    tot[1] += 1
    out.append(("conservation_phi_fault", corp, rp, ids, cn, phi, tot))
    corp, rp, ids, cn, phi, tot = model([5, 8, 3], 7, 3, 4)
    phi[2, 1] += 1
    out.append(("conservation_stale_totals", corp, rp, ids, cn, phi, tot))
    corp, rp, ids, cn, phi, tot = model([5, 8, 3], 7, 3, 5)
    cn = cn.copy()
    cn[rp[1]] += 1
    out.append(("conservation_theta_row", corp, rp, ids, cn, phi, tot))
    return out


def test_conservation_texts_match_reference():
    with open(os.path.join(GOLD, "messages.json")) as fh:
        msgs = json.load(fh)
    for name, corp, rp, ids, cn, phi, tot in conservation_cases():
        got = oracle.check_conservation(rp, ids, cn, phi, tot, corp["doc_lengths"], corp["T"])[1]
        assert got == msgs[name], name


# -------------------------------------------------------------- ptree ------
def test_ptree_golden_is_sequential_scan():
    """ptree.py:116-151: level 0 is the sequential fp32 cumsum; draw = minimal
    index with prefix > u.  The GPU search is checked against the same arrays."""
    g = load("ptree.npz")
    meta = json.loads(str(g["meta"]))
    for m in meta:
        i = m["i"]
        w = g[f"t{i}__w"]
        np.testing.assert_array_equal(np.cumsum(w, dtype=np.float32), g[f"t{i}__prefix"])
        idx = np.searchsorted(g[f"t{i}__prefix"], g[f"t{i}__u"], side="right")
        np.testing.assert_array_equal(idx, g[f"t{i}__idx"])
        np.testing.assert_array_equal(idx, g[f"t{i}__idx_many"])


def test_ptree_api_golden():
    """ptree.py:54-151 (sample_with_stats, level_sums, prefix_before, fp64 mode,
    fanouts > 32, sample_total_and_draw) against the reference's own outputs;
    the host-side levels of the repo's build() match too."""
    from paper_1803_04631_b200 import ptree

    g = load("ptree_api.npz")
    for m in json.loads(str(g["meta"])):
        i, dt, F = m["i"], np.dtype(m["dtype"]), m["fanout"]
        levels = oracle.ptree_levels(g[f"a{i}__w"], F, dt)
        tree = ptree.build(g[f"a{i}__w"], fanout=F, dtype=dt)
        assert tree.height == m["height"] == len(levels) - 1
        for lvl in range(len(levels)):
            np.testing.assert_array_equal(tree.level_sums(lvl), g[f"a{i}__sums{lvl}"])
            np.testing.assert_array_equal(tree.levels[lvl], levels[lvl])
        np.testing.assert_array_equal([tree.prefix_before(j) for j in range(0, m["n"], 97)],
                                      g[f"a{i}__prefix_before"])
        got = [oracle.ptree_descend(levels, F, u) for u in g[f"a{i}__u"]]
        np.testing.assert_array_equal([x[0] for x in got], g[f"a{i}__idx"])
        np.testing.assert_array_equal([x[1] for x in got], g[f"a{i}__visited"])
        np.testing.assert_array_equal([x[2] for x in got], g[f"a{i}__widest"])
    # fp64 sample_total_and_draw: u = Stream.uniform() * total (ptree.py:139-151)
    w = g["draw64__w"]
    levels = oracle.ptree_levels(w, 4, np.float64)
    us = oracle.stream_uniforms((77, 3), len(g["draw64__u"])) * float(levels[0][-1])
    np.testing.assert_array_equal(us, g["draw64__u"])
    np.testing.assert_array_equal([oracle.ptree_descend(levels, 4, u)[0] for u in us], g["draw64__idx"])


# ------------------------------------------------------------ sampler ------
def test_spec_sample_dense_example():
    # K=2, theta_d=[1,0], phi_.v=[1,1], totals=[2,2], a=0.5, b=0.1, V=3 -> [0.75, 0.25]
    p, pd = oracle.conditional(2, 3, 0.5, 0.1, [1, 0], [1, 1], [2, 2], 0, exclusion=False)
    np.testing.assert_allclose(p, [0.75, 0.25], rtol=1e-12)
    np.testing.assert_allclose(pd, [0.75, 0.25], rtol=1e-12)   # SPEC.md:274 identity


def test_spec_exclusion_examples():
    # theta {3:1}, z=3 -> empty row; {1:2}, z=1 -> {1:1}
    K, V, a, b = 4, 5, 0.3, 0.1
    phi = np.array([2, 3, 1, 4], np.uint32)
    tot = np.array([10, 12, 9, 11], np.int64)
    p, _ = oracle.conditional(K, V, a, b, [0, 0, 0, 1], phi, tot, 3)
    p0, _ = oracle.conditional(K, V, a, b, [0, 0, 0, 0], phi - np.array([0, 0, 0, 1], np.uint32),
                               tot - np.array([0, 0, 0, 1]), 3, exclusion=False)
    np.testing.assert_allclose(p, p0, rtol=1e-12)
    p, _ = oracle.conditional(K, V, a, b, [0, 2, 0, 0], phi, tot, 1)
    p0, _ = oracle.conditional(K, V, a, b, [0, 1, 0, 0], phi - np.array([0, 1, 0, 0], np.uint32),
                               tot - np.array([0, 1, 0, 0]), 1, exclusion=False)
    np.testing.assert_allclose(p, p0, rtol=1e-12)


def test_decomposition_identity_1000_states():
    # SPEC acceptance #2 in 64-bit mode: p1+p2 decomposition == Eq. 1 within 1e-12
    r = np.random.default_rng(1)
    worst = 0.0
    for _ in range(1000):
        K = int(r.integers(1, 65))
        V = int(r.integers(1, 33))
        th = r.integers(0, 5, K)
        z = int(r.integers(0, K))
        th[z] += 1
        ph = r.integers(0, 9, K).astype(np.uint32)
        ph[z] += 1
        tot = ph.astype(np.int64) + r.integers(0, 50, K)
        p, pd = oracle.conditional(K, V, 50.0 / K, 0.01, th, ph, tot, z)
        worst = max(worst, float(np.max(np.abs(p - pd) / p)))
    assert worst <= 1e-12


def _single_run_state(K, V, r):
    """One document, one word, many tokens with the same topic: every token
    draws from the same exclusion-adjusted conditional (fixed counts)."""
    th = r.integers(0, 6, K)
    z = int(r.integers(0, K))
    th[z] += 1
    ids = np.flatnonzero(th).astype(np.uint16)
    cnt = th[ids].astype(np.uint16)
    phi = r.integers(0, 20, (K, V)).astype(np.uint32)
    v = int(r.integers(0, V))
    phi[z, v] += 1
    tot = phi.sum(axis=1).astype(np.int64) + r.integers(0, 30, K)
    return th, z, ids, cnt, phi, tot, v


@pytest.mark.parametrize("K", [3, 17, 64])
def test_oracle_sampler_chi_square(K):
    # SPEC acceptance #4 (1e6 draws, p > 0.001) for the oracle sampler itself
    r = np.random.default_rng(100 + K)
    V = 7
    th, z, ids, cnt, phi, tot, v = _single_run_state(K, V, r)
    n = 1_000_000
    alpha, beta = 50.0 / K, 0.01
    zp = oracle.sample_tokens(K, V, alpha, beta, 42, 3, np.zeros(n, np.int32), np.full(n, v, np.int32),
                              np.full(n, z, np.uint16), 0, np.array([0, len(ids)]), ids, cnt, phi, tot)
    hist = np.bincount(zp, minlength=K)
    p, _ = oracle.conditional(K, V, alpha, beta, th, phi[:, v], tot, z)
    keep = p * n >= 5
    _, pval = stats.chisquare(hist[keep], p[keep] / p[keep].sum() * hist[keep].sum())
    assert pval > 0.001
    assert hist[~keep].sum() <= max(50, 5 * p[~keep].sum() * n)


@pytest.mark.parametrize("K", [3, 17, 64])
def test_thinning_sampler_has_the_exclusion_distribution(K):
    """The device's draw form (exclusion by thinning, oracle mode "thin")
    samples the same exclusion-adjusted Eq. 1 as SPEC sample_sparse."""
    r = np.random.default_rng(200 + K)
    V = 5
    th, z, ids, cnt, phi, tot, v = _single_run_state(K, V, r)
    n = 1_000_000
    alpha, beta = 50.0 / K, 0.01
    p, _ = oracle.conditional(K, V, alpha, beta, th, phi[:, v], tot, z)
    pvals = []
    for seed in (1, 2, 3):
        zp = oracle.sample_tokens(K, V, alpha, beta, seed, 0, np.zeros(n, np.int32), np.full(n, v, np.int32),
                                  np.full(n, z, np.uint16), 0, np.array([0, len(ids)]), ids, cnt, phi, tot,
                                  mode="thin")
        hist = np.bincount(zp, minlength=K)
        keep = p * n >= 5
        pvals.append(stats.chisquare(hist[keep], p[keep] / p[keep].sum() * hist[keep].sum())[1])
    assert sum(pv > 0.001 for pv in pvals) >= 2, pvals


def test_thinning_singleton_topic_is_never_kept_in_s_branch():
    # theta_d = {z: 1}: after exclusion z has no S mass; thinning must reproduce
    # exactly the Q-only conditional
    K, V = 6, 3
    th = np.zeros(K, np.int64)
    th[2] = 1
    phi = np.full((K, V), 4, np.uint32)
    tot = phi.sum(axis=1).astype(np.int64)
    n = 400_000
    zp = oracle.sample_tokens(K, V, 0.3, 0.1, 9, 0, np.zeros(n, np.int32), np.zeros(n, np.int32),
                              np.full(n, 2, np.uint16), 0, np.array([0, 1]), np.array([2], np.uint16),
                              np.array([1], np.uint16), phi, tot, mode="thin")
    p, _ = oracle.conditional(K, V, 0.3, 0.1, th, phi[:, 0], tot, 2)
    _, pv = stats.chisquare(np.bincount(zp, minlength=K), p * n)
    assert pv > 0.001


def test_oracle_sampler_is_deterministic_and_thread_invariant():
    r = np.random.default_rng(5)
    K, V = 16, 9
    th, z, ids, cnt, phi, tot, v = _single_run_state(K, V, r)
    n = 5000
    args = (K, V, 50.0 / K, 0.01, 7, 1, np.zeros(n, np.int32), np.full(n, v, np.int32),
            np.full(n, z, np.uint16), 0, np.array([0, len(ids)]), ids, cnt, phi, tot)
    a = oracle.sample_tokens(*args, nthreads=1)
    b = oracle.sample_tokens(*args, nthreads=4)
    np.testing.assert_array_equal(a, b)


# --------------------------------------------------------------- eval ------
def test_spec_loglik_examples():
    # K=1 -> mean of log((phi_0v + b)/(T + bV))
    V, b = 4, 0.01
    doc = np.array([0, 0, 1], np.int32)
    word = np.array([0, 2, 2], np.int32)
    phi = np.array([[1, 0, 2, 0]], np.uint32)
    tot = np.array([3], np.int64)
    ll = oracle.loglik_naive(1, V, 50.0, b, doc, word, [0, 1, 2], np.array([0, 0], np.uint16),
                             np.array([2, 1], np.uint16), [2, 1], phi, tot)
    want = np.mean([np.log((1 + b) / (3 + b * V)), np.log((2 + b) / (3 + b * V)), np.log((2 + b) / (3 + b * V))])
    assert ll == pytest.approx(want, rel=1e-12)
    # prior only (zero counts, so DocLen = sum of theta = 0) -> log(1/V)
    K = 5
    ll = oracle.loglik_naive(K, V, 0.1, b, doc, word, [0, 0, 0], np.zeros(0, np.uint16),
                             np.zeros(0, np.uint16), [0, 0], np.zeros((K, V), np.uint32), np.zeros(K, np.int64))
    assert ll == pytest.approx(np.log(1.0 / V), rel=1e-12)


# ------------------------------------------------------------- engine ------
def test_spec_reduce_examples():
    s, rounds = oracle.reduce_phi_pairwise([[[1, 2], [3, 4]], [[5, 6], [7, 8]]])
    assert s.tolist() == [[6, 8], [10, 12]] and len(rounds) == 1
    _, rounds = oracle.reduce_phi_pairwise([np.zeros(2)] * 4)   # Fig. 6 structure
    assert rounds == [[(1, 0), (3, 2)], [(2, 0)]]
    r = np.random.default_rng(0)
    for G in (3, 5, 8):
        reps = [r.integers(0, 100, (3, 4)) for _ in range(G)]
        s, rounds = oracle.reduce_phi_pairwise(reps)
        np.testing.assert_array_equal(s, np.sum(reps, axis=0))
        assert len(rounds) == int(np.ceil(np.log2(G)))


def test_loglik_sq_form_equals_naive_formula():
    """The O(T K_d) S + Q form used for large trajectories equals SPEC.md:405."""
    from paper_1803_04631_b200 import corpus as cp
    from paper_1803_04631_b200 import synth

    K = 24
    corp = synth.generate(150, 300, 40.0, seed=4)
    ch = cp.partition(corp, 1, K, 3)[0]
    rp, ids, cn = oracle.rebuild_theta(ch.assignments, ch.dw_ptr, ch.dw_tok, 0, K)
    phi, tot = oracle.rebuild_phi(ch.assignments, ch.word_ids, K, corp.vocab_size)
    a, b = 50.0 / K, 0.01
    naive = oracle.loglik_naive(K, corp.vocab_size, a, b, ch.doc_ids, ch.word_ids, rp, ids, cn,
                                corp.doc_lengths, phi, tot)
    sq = oracle.loglik_sq(K, corp.vocab_size, a, b, ch.doc_ids, ch.word_ids, 0, rp, ids, cn, corp.doc_lengths,
                          phi, tot)
    assert sq == pytest.approx(naive, rel=1e-12)


def low_acceptance_state(K=100, V=5, seed=0):
    """A token that is the only occurrence of its word in its topic z (phi_vz = 1)
    in a document dominated by z: thinning rejects a z proposal ~97% of the time
    (the 64-try cap is reached with probability ~0.16), and under the exact
    conditional the token leaves z with probability ~0.66."""
    r = np.random.default_rng(seed)
    th = np.zeros(K, np.int64)
    z = 7
    th[z] = 100
    others = r.choice([k for k in range(K) if k != z], 30, replace=False)
    np.add.at(th, r.choice(others, 100), 1)
    phi = r.integers(0, 3, (K, V)).astype(np.uint32)
    v = 2
    phi[:, v] = 0
    phi[z, v] = 1
    tot = phi.sum(axis=1).astype(np.int64) + r.integers(1000, 5000, K)
    return th, z, phi, tot, v


def test_thinning_is_exact_at_low_acceptance():
    """the thinning loop must not keep z after its retry cap -- the
    64th rejection ends in an exact draw, so even a state where most proposals
    of z are rejected samples the exclusion-adjusted Eq. 1."""
    K, V, alpha, beta = 100, 5, 0.5, 0.01
    th, z, phi, tot, v = low_acceptance_state(K, V)
    ids = np.flatnonzero(th).astype(np.uint16)
    p, _ = oracle.conditional(K, V, alpha, beta, th, phi[:, v], tot, z)
    ps = (phi[:, v] + beta) / (tot + V * beta)
    full = (th + alpha) * ps
    rej = (full[z] - (th[z] - 1 + alpha) * (phi[z, v] - 1 + beta) / (tot[z] - 1 + V * beta)) / full.sum()
    assert rej ** 64 > 0.1                                   # the cap is really exercised
    n = 1_000_000
    zp = oracle.sample_tokens(K, V, alpha, beta, 42, 3, np.zeros(n, np.int32), np.full(n, v, np.int32),
                              np.full(n, z, np.uint16), 0, np.array([0, len(ids)]), ids,
                              th[ids].astype(np.uint16), phi, tot, mode="thin")
    hist = np.bincount(zp, minlength=K)
    keep = p * n >= 5
    assert stats.chisquare(hist[keep], p[keep] / p[keep].sum() * hist[keep].sum())[1] > 0.001
    assert abs(hist[z] / n - p[z]) < 0.003
