"""GPU parity tests: the CUDA path (through the C ABI) against the oracle and
the reference golden vectors.  Bit-exact for counts / CSR / search; chi-square
and draw-agreement for the sampler; 1e-6 relative for the fused loglik."""

import json
import os

import numpy as np
import pytest
from scipy import stats

import oracle
from paper_1803_04631_b200 import corpus as cp
from paper_1803_04631_b200 import engine, errors, eval as ev, model as md, ptree, sampler, synth
from paper_1803_04631_b200.shard import DeviceShard

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def build_chunk(doc_ids, word_ids, assignments, chunk_id=0):
    """tests/test_model.py:9-33 of the reference: word-grouped Chunk from triples."""
    doc_ids = np.asarray(doc_ids, dtype=np.int32)
    word_ids = np.asarray(word_ids, dtype=np.int32)
    assignments = np.asarray(assignments, dtype=np.uint16)
    order = np.argsort(word_ids, kind="stable")
    doc_ids, word_ids, assignments = doc_ids[order], word_ids[order], assignments[order]
    words, starts, sizes = np.unique(word_ids, return_index=True, return_counts=True)
    lo = int(doc_ids.min()) if doc_ids.size else 0
    hi = int(doc_ids.max()) + 1 if doc_ids.size else 0
    dw_ptr, dw_tok = cp._doc_word_map(doc_ids, lo, hi - lo)
    return cp.Chunk(chunk_id, lo, hi, len(doc_ids), doc_ids, word_ids, assignments.copy(),
                    words.astype(np.int32), starts.astype(np.int64), sizes.astype(np.int64), dw_ptr, dw_tok)


def oracle_theta(ch, K):
    return oracle.rebuild_theta(ch.assignments, ch.dw_ptr, ch.dw_tok, ch.doc_lo, K)


# ------------------------------------------------------------ K2 / K3 ------
@pytest.mark.parametrize("name", ["small", "single", "rand25", "zipf", "zipf_k1024"])
def test_rebuilds_match_reference_golden(name):
    g = np.load(os.path.join(GOLD, "partition.npz"))
    m = next(x for x in json.loads(str(g["meta"])) if x["name"] == name)
    corp = cp.corpus_from_tokens(g[f"{name}__corpus_doc_ids"], g[f"{name}__corpus_word_ids"], m["V"])
    chunks = cp.partition(corp, m["C"], m["K"], m["seed"])
    parts = []
    for ch in chunks:
        pre = f"{name}__c{ch.chunk_id}__"
        th = md.rebuild_theta(ch, m["K"])
        np.testing.assert_array_equal(th.row_ptr, g[pre + "theta_row_ptr"])
        np.testing.assert_array_equal(th.topic_ids, g[pre + "theta_topic_ids"])
        np.testing.assert_array_equal(th.counts, g[pre + "theta_counts"])
        ph = md.rebuild_phi_replica(ch, m["K"], m["V"])
        np.testing.assert_array_equal(ph.counts, g[pre + "phi_counts"])
        np.testing.assert_array_equal(ph.topic_totals, g[pre + "phi_totals"])
        assert ph.counts.dtype == np.uint32
        parts.append(th)
    full = md.concat_theta(parts)
    np.testing.assert_array_equal(full.row_ptr, g[f"{name}__concat_row_ptr"])


def test_rebuilds_match_reference_on_hand_chunks():
    g = np.load(os.path.join(GOLD, "counts.npz"))
    for m in json.loads(str(g["meta"])):
        pre = f"h{m['i']}__"
        ch = build_chunk(g[pre + "doc"], g[pre + "word"], g[pre + "z"])
        th = md.rebuild_theta(ch, m["K"])
        np.testing.assert_array_equal(th.row_ptr, g[pre + "theta_row_ptr"])
        np.testing.assert_array_equal(th.topic_ids, g[pre + "theta_topic_ids"])
        np.testing.assert_array_equal(th.counts, g[pre + "theta_counts"])
        ph = md.rebuild_phi_replica(ch, m["K"], m["V"])
        np.testing.assert_array_equal(ph.counts, g[pre + "phi_counts"])
        np.testing.assert_array_equal(ph.topic_totals, g[pre + "phi_totals"])


def test_reference_test_model_cases():
    # reference tests/test_model.py:52-62, 85-97
    ids, cnt = md.rebuild_theta_row(build_chunk([0, 0, 0], [1, 2, 0], [2, 2, 0]), 0, 4)
    assert ids.tolist() == [0, 2] and cnt.tolist() == [1, 2]
    ids, cnt = md.rebuild_theta_row(build_chunk([0], [3], [7]), 0, 8)
    assert ids.tolist() == [7] and cnt.tolist() == [1]
    rep = md.rebuild_phi_replica(build_chunk([0, 0, 0], [1, 1, 2], [0, 0, 1]), 2, 3)
    assert rep.counts[0, 1] == 2 and rep.counts[1, 2] == 1 and rep.topic_totals.tolist() == [2, 1]
    empty = build_chunk([], [], [])
    rep = md.rebuild_phi_replica(empty, 3, 4)
    assert rep.counts.sum() == 0 and rep.topic_totals.tolist() == [0, 0, 0]


def test_count_overflow_messages_match_reference():
    with open(os.path.join(GOLD, "messages.json")) as fh:
        msgs = json.load(fh)
    n = 70000
    with pytest.raises(errors.CountOverflowError) as ei:
        md.rebuild_theta(build_chunk(np.full(n, 3), np.zeros(n), np.zeros(n)), 2)
    assert str(ei.value) == msgs["theta_overflow_doc3"]
    n = 66000
    ch = build_chunk(np.zeros(n), np.ones(n), np.ones(n, dtype=int))
    with pytest.raises(errors.CountOverflowError) as ei:
        md.rebuild_phi_replica(ch, 2, 2, width=16)
    assert str(ei.value) == msgs["phi16_overflow_k1_v1"]
    assert md.rebuild_phi_replica(ch, 2, 2, width=32).counts[1, 1] == n
    ds = np.zeros(140000)
    ws = np.concatenate([np.full(66000, 3), np.full(74000, 1)])
    zs = np.concatenate([np.full(66000, 0), np.full(74000, 2)])
    with pytest.raises(errors.CountOverflowError) as ei:
        md.rebuild_phi_replica(build_chunk(ds, ws, zs), 3, 4, width=16)
    assert str(ei.value) == msgs["phi16_overflow_argmax"]


def test_theta_rebuild_random_sizes_vs_oracle():
    r = np.random.default_rng(3)
    for K in (1, 2, 33, 1024, 4096):
        n = 20000
        lengths = r.choice([1, 2, 5, 31, 32, 33, 64, 300, 2000], size=200)
        docs = np.repeat(np.arange(len(lengths)), lengths)[:n]
        ch = build_chunk(docs + 5, r.integers(0, 50, len(docs)), r.integers(0, K, len(docs)))
        th = md.rebuild_theta(ch, K)
        rp, ids, cn = oracle_theta(ch, K)
        np.testing.assert_array_equal(th.row_ptr, rp)
        np.testing.assert_array_equal(th.topic_ids, ids)
        np.testing.assert_array_equal(th.counts, cn)
        ph = md.rebuild_phi_replica(ch, K, 50)
        oc, ot = oracle.rebuild_phi(ch.assignments, ch.word_ids, K, 50)
        np.testing.assert_array_equal(ph.counts, oc)
        np.testing.assert_array_equal(ph.topic_totals, ot)


def test_heavy_words_split_across_slices_vs_oracle():
    # a word with > 65535 tokens in the shard: 32-bit column, several K2 items (atomics)
    r = np.random.default_rng(4)
    n = 300000
    docs = np.repeat(np.arange(3000), 100)
    words = np.where(r.random(n) < 0.5, 7, r.integers(0, 20, n))
    ch = build_chunk(docs, words, r.integers(0, 16, n))
    ph = md.rebuild_phi_replica(ch, 16, 20)
    oc, ot = oracle.rebuild_phi(ch.assignments, ch.word_ids, 16, 20)
    np.testing.assert_array_equal(ph.counts, oc)
    np.testing.assert_array_equal(ph.topic_totals, ot)


@pytest.mark.parametrize("piece", [1024, 200000])
def test_heavy_word_pieces_vs_oracle(piece, monkeypatch):
    """K2 items of a heavy (32-bit column) word: many small pieces flushed with
    global atomics (GF_K2_PIECE=1024), or one item longer than 65535 tokens,
    counted in <= 65528-token rounds inside the kernel (GF_K2_PIECE=200000)."""
    from paper_1803_04631_b200.shard import RESIDENT

    monkeypatch.setenv("GF_K2_PIECE", str(piece))
    RESIDENT.release()
    r = np.random.default_rng(40)
    n = 400000
    docs = np.repeat(np.arange(4000), 100)
    words = np.where(r.random(n) < 0.45, 7, np.where(r.random(n) < 0.3, 3, r.integers(0, 30, n)))
    ch = build_chunk(docs, words, r.integers(0, 24, n))
    ph = md.rebuild_phi_replica(ch, 24, 30)
    oc, ot = oracle.rebuild_phi(ch.assignments, ch.word_ids, 24, 30)
    np.testing.assert_array_equal(ph.counts, oc)
    np.testing.assert_array_equal(ph.topic_totals, ot)
    RESIDENT.release()


def test_theta_rebuild_document_groups_vs_oracle():
    """K3 on enough documents that every warp takes groups of 32 (the
    batched-metadata / L2-prefetch path; small tests run groups of 1)."""
    from paper_1803_04631_b200.shard import RESIDENT

    RESIDENT.release()
    r = np.random.default_rng(41)
    K = 1024
    lengths = r.choice([1, 3, 17, 32, 33, 70, 128, 129, 400], size=900000,
                       p=[0.2, 0.2, 0.2, 0.1, 0.1, 0.1, 0.05, 0.04, 0.01])
    docs = np.repeat(np.arange(len(lengths)), lengths)
    ch = build_chunk(docs, r.integers(0, 5000, len(docs)), r.integers(0, K, len(docs)))
    th = md.rebuild_theta(ch, K)
    rp, ids, cn = oracle_theta(ch, K)
    np.testing.assert_array_equal(th.row_ptr, rp)
    np.testing.assert_array_equal(th.topic_ids, ids)
    np.testing.assert_array_equal(th.counts, cn)
    RESIDENT.release()


# --------------------------------------------------------------- ptree -------
def test_device_tree_search_matches_reference():
    g = np.load(os.path.join(GOLD, "ptree.npz"))
    for m in json.loads(str(g["meta"])):
        i = m["i"]
        levels = [g[f"t{i}__level{lvl}"] for lvl in range(m["height"] + 1)]
        tree = ptree.PrefixTree(levels, m["fanout"])
        np.testing.assert_array_equal(tree.sample_many(g[f"t{i}__u"]), g[f"t{i}__idx"])
        t2 = ptree.build(g[f"t{i}__w"], fanout=m["fanout"])
        for a, b in zip(t2.levels, levels):
            np.testing.assert_array_equal(a, b)


def test_device_tree_api_matches_reference():
    """sample_with_stats (index, visited, widest), fp64 trees and fanouts > 32
    on the device against the reference's outputs (ptree_api.npz)."""
    from paper_1803_04631_b200 import rng

    g = np.load(os.path.join(GOLD, "ptree_api.npz"))
    for m in json.loads(str(g["meta"])):
        i = m["i"]
        tree = ptree.build(g[f"a{i}__w"], fanout=m["fanout"], dtype=np.dtype(m["dtype"]))
        us = g[f"a{i}__u"]
        np.testing.assert_array_equal(tree.sample_many(us), g[f"a{i}__idx"])
        for j in range(0, len(us), 9):
            assert tree.sample_with_stats(us[j]) == (g[f"a{i}__idx"][j], g[f"a{i}__visited"][j],
                                                     g[f"a{i}__widest"][j])
    tree = ptree.build(g["draw64__w"], fanout=4, dtype=np.float64)
    st = rng.Stream(77, 3)
    draws = [ptree.sample_total_and_draw(tree, st) for _ in range(len(g["draw64__idx"]))]
    np.testing.assert_array_equal([d[0] for d in draws], g["draw64__idx"])
    np.testing.assert_array_equal([d[1] for d in draws], g["draw64__u"])
    # fp32 replay of the reference's own Stream(2024) draws (ptree.npz)
    g32 = np.load(os.path.join(GOLD, "ptree.npz"))
    tree = ptree.build(g32["draw__w"], fanout=2)
    st = rng.Stream(2024)
    draws = [ptree.sample_total_and_draw(tree, st) for _ in range(len(g32["draw__idx"]))]
    np.testing.assert_array_equal([d[0] for d in draws], g32["draw__idx"])
    np.testing.assert_array_equal([d[1] for d in draws], g32["draw__u"])
    with pytest.raises(errors.EmptyDistributionError):
        ptree.sample_total_and_draw(ptree.build([0.0, 0.0], 2), rng.Stream(0))
    with pytest.raises(ValueError):
        ptree.build([1.0, 2.0], 2).sample(3.5)


def test_device_tree_zero_leaves_never_drawn():
    tree = ptree.build(np.array([0.0, 1.0, 0.0, 2.0, 0.0], np.float32), fanout=2)
    us = (np.random.default_rng(1).random(20000) * tree.total).astype(np.float32)
    us = np.minimum(us, np.nextafter(np.float32(tree.total), np.float32(0)))
    assert set(tree.sample_many(us).tolist()) <= {1, 3}


# ------------------------------------------------------------- sampler -------
def single_run_state(K, V, r, nnz_min=1, max_count=6):
    if nnz_min > 1:
        th = np.zeros(K, np.int64)
        th[r.choice(K, nnz_min, replace=False)] = r.integers(1, max_count + 1, nnz_min)
    else:
        th = r.integers(0, max_count, K)
    z = int(r.integers(0, K))
    th[z] += 1
    phi = r.integers(0, 20, (K, V)).astype(np.uint32)
    v = int(r.integers(0, V))
    phi[z, v] += 1
    tot = phi.sum(axis=1).astype(np.int64) + r.integers(0, 30, K)
    return th, z, phi, tot, v


def draw_fixed_state(K, V, th, z, phi, tot, v, n, seed=42, it=3, alpha=None, beta=0.01):
    """n tokens of one (doc, word) run: n iid draws from one conditional."""
    ch = build_chunk(np.zeros(n), np.full(n, v), np.full(n, z))
    ids = np.flatnonzero(th).astype(np.uint16)
    alpha = 50.0 / K if alpha is None else alpha
    with DeviceShard(K, V, alpha, beta, seed=seed) as sh:
        sh.load(ch)
        sh.set_phi(phi, tot)
        sh.set_theta(np.array([0, len(ids)]), ids, th[ids].astype(np.uint16))
        sh.prepare()
        sh.sample(it)
        sh.check_errors()
        zp = sh.get_assignments()
    p, _ = oracle.conditional(K, V, alpha, beta, th, phi[:, v], tot, z)
    return zp, p


def chi_square_p(hist, p):
    n = hist.sum()
    order = np.argsort(p)
    # merge the smallest cells until every expected count is >= 5
    bins_h, bins_p, acc_h, acc_p = [], [], 0, 0.0
    for k in order:
        acc_h += hist[k]
        acc_p += p[k]
        if acc_p * n >= 5:
            bins_h.append(acc_h)
            bins_p.append(acc_p)
            acc_h, acc_p = 0, 0.0
    if acc_p > 0:
        bins_h[-1] += acc_h
        bins_p[-1] += acc_p
    bins_p = np.array(bins_p)
    return stats.chisquare(bins_h, bins_p / bins_p.sum() * n)[1]


# SPEC acceptance #4 exactly: ten fixed count states with
# K <= 64, 1e6 draws each from one Philox stream (seed 42), and EVERY state
# must pass chi-square against the exclusion-adjusted Eq. 1 at p > 0.001.
SPEC4_TOPICS = [2, 3, 5, 8, 13, 17, 24, 32, 48, 64]


@pytest.mark.parametrize("K", SPEC4_TOPICS)
def test_sampler_chi_square_spec4_states(K):
    r = np.random.default_rng(4000 + K)
    V = 7
    th, z, phi, tot, v = single_run_state(K, V, r)
    zp, p = draw_fixed_state(K, V, th, z, phi, tot, v, 1_000_000, seed=42)
    assert chi_square_p(np.bincount(zp, minlength=K), p) > 0.001


# Beyond SPEC #4: large K (smallest cells merged to expected counts >= 5).
# nnz 700 at K = 1024 fills the staging buffer; K = 4096 / 8192 take the
# large-K variants (p*_ex on demand, the streaming path).  Three independent
# Philox streams; a correct sampler fails one at p < 0.001 with probability
# 1e-3, two with ~3e-6 (the oracle, which the device matches draw for draw,
# gives the same p-values).
@pytest.mark.parametrize("K,nnz_min", [(128, 1), (256, 40), (1024, 200), (1024, 700), (2048, 300), (4096, 600),
                                       (8192, 900)])
def test_sampler_chi_square_large_k(K, nnz_min):
    r = np.random.default_rng(K + nnz_min)
    V = 7
    th, z, phi, tot, v = single_run_state(K, V, r, nnz_min=nnz_min, max_count=3)
    pvals = []
    for seed in (42, 43, 44):
        zp, p = draw_fixed_state(K, V, th, z, phi, tot, v, 1_000_000, seed=seed)
        pvals.append(chi_square_p(np.bincount(zp, minlength=K), p))
    assert sum(pv > 0.001 for pv in pvals) >= 2, pvals


def test_sampler_exact_at_low_acceptance():
    """a state where thinning rejects ~97% of the z proposals (the
    64-try cap is hit ~16% of the time): the device must still sample the
    exclusion-adjusted conditional (a capped loop that kept z gave p(z) 0.45
    instead of 0.34)."""
    from test_oracle_golden import low_acceptance_state

    K, V = 100, 5
    th, z, phi, tot, v = low_acceptance_state(K, V)
    zp, p = draw_fixed_state(K, V, th, z, phi, tot, v, 1_000_000, seed=42, alpha=0.5)
    hist = np.bincount(zp, minlength=K)
    assert chi_square_p(hist, p) > 0.001
    assert abs(hist[z] / len(zp) - p[z]) < 0.003


def test_sampler_edge_states():
    r = np.random.default_rng(9)
    # theta_d = {z: 1}: after exclusion the S part is empty -> pure Q branch
    K, V = 8, 3
    th = np.zeros(K, np.int64)
    th[5] = 1
    phi = r.integers(1, 9, (K, V)).astype(np.uint32)
    tot = phi.sum(axis=1).astype(np.int64)
    zp, p = draw_fixed_state(K, V, th, 5, phi, tot, 1, 200_000)
    assert chi_square_p(np.bincount(zp, minlength=K), p) > 0.001
    # K = 1: always topic 0
    zp, _ = draw_fixed_state(1, 2, np.array([3]), 0, np.array([[5, 1]], np.uint32), np.array([6]), 0, 1000)
    assert (zp == 0).all()


def test_consistency_error_when_topic_absent():
    K, V = 4, 2
    ch = build_chunk([0, 0], [1, 1], [2, 2])
    with DeviceShard(K, V, 0.5, 0.1) as sh:
        sh.load(ch)
        sh.set_phi(np.ones((K, V), np.uint32), np.full(K, 2))
        sh.set_theta(np.array([0, 1]), np.array([0], np.uint16), np.array([2], np.uint16))
        sh.prepare()
        sh.sample(0)
        with pytest.raises(errors.ConsistencyError):
            sh.check_errors()


@pytest.mark.parametrize("bad_docs", [(0,), (1,), (2,), (3, 1), (2, 3)])
def test_theta_rebuild_reports_out_of_range_topic(bad_docs):
    """K3 flags a topic >= K (an import the host does not range-check) as a
    ConsistencyError naming the first such document, on each of its paths:
    documents of 20 (warp sort), 100 (register columns) and 300 tokens
    (histogram loop); a clean state raises nothing."""
    K, V = 16, 40
    r = np.random.default_rng(len(bad_docs) * 10 + bad_docs[0])
    lens = [20, 100, 300, 100]
    docs = np.repeat(np.arange(len(lens)), lens)
    ch = build_chunk(docs, r.integers(0, V, docs.size), r.integers(0, K, docs.size))
    with DeviceShard(K, V, 0.5, 0.1) as sh:
        sh.load(ch)
        z = sh.get_assignments()
        np.testing.assert_array_equal(z, ch.assignments)
        sh.rebuild_theta()
        sh.check_errors()
        for d in bad_docs:
            pos = np.flatnonzero(ch.doc_ids == d)
            z[r.choice(pos, size=2, replace=False)] = [K + 3, 0xFFFF]
        sh.set_assignments(z)
        sh.rebuild_theta()
        with pytest.raises(errors.ConsistencyError, match=f"document {min(bad_docs)}: a token's topic is outside"):
            sh.check_errors()
        sh.check_errors()                       # reported once, then cleared


def _chunk_state(corp, K, seed):
    ch = cp.partition(corp, 1, K, seed)[0]
    rp, ids, cn = oracle_theta(ch, K)
    phi, tot = oracle.rebuild_phi(ch.assignments, ch.word_ids, K, corp.vocab_size)
    return ch, rp, ids, cn, phi, tot


@pytest.mark.parametrize("K,mean_len", [(32, 60.0), (1024, 900.0)])
def test_draws_agree_with_oracle_sampler(K, mean_len):
    """Same state, same Philox stream: the device (fp32) and the oracle (fp64)
    pick the same topic except where rounding straddles a boundary."""
    corp = synth.generate(400, 3000, mean_len, seed=11)
    ch, rp, ids, cn, phi, tot = _chunk_state(corp, K, 5)
    a, b = 50.0 / K, 0.01
    want = oracle.sample_tokens(K, corp.vocab_size, a, b, 77, 4, ch.doc_ids, ch.word_ids, ch.assignments,
                                ch.doc_lo, rp, ids, cn, phi, tot, mode="thin")
    with DeviceShard(K, corp.vocab_size, a, b, seed=77) as sh:
        sh.load(ch)
        sh.initialize()
        np.testing.assert_array_equal(sh.get_theta()[1], ids)
        sh.sample(4)
        sh.check_errors()
        got = sh.get_assignments()
    agree = np.mean(got == want)
    assert agree > 0.998, agree


def test_fused_loglik_matches_naive_formula():
    K = 64
    corp = synth.generate(300, 2000, 80.0, seed=12)
    ch, rp, ids, cn, phi, tot = _chunk_state(corp, K, 6)
    a, b = 50.0 / K, 0.01
    want = oracle.loglik_naive(K, corp.vocab_size, a, b, ch.doc_ids, ch.word_ids, rp, ids, cn,
                               corp.doc_lengths, phi, tot)
    with DeviceShard(K, corp.vocab_size, a, b, seed=1) as sh:
        sh.load(ch)
        sh.initialize()
        sh.sample(0)
        got = sh.loglik_sum() / corp.num_tokens
    assert got == pytest.approx(want, rel=1e-6)
    theta = md.ThetaRows(rp, ids, cn, K)
    got2 = ev.loglik_per_token(theta, md.PhiMatrix(phi.astype(np.uint32), tot), corp, a, b)
    assert got2 == pytest.approx(want, rel=1e-6)


def test_spec_loglik_examples_on_device():
    corp = cp.corpus_from_tokens([0, 0, 1], [0, 2, 2], 4)
    theta = md.ThetaRows(np.array([0, 1, 2]), np.array([0, 0], np.uint16), np.array([2, 1], np.uint16), 1)
    phi = md.PhiMatrix(np.array([[1, 0, 2, 0]], np.uint32), np.array([3]))
    b = 0.01
    want = np.mean([np.log((1 + b) / (3 + 4 * b)), np.log((2 + b) / (3 + 4 * b)), np.log((2 + b) / (3 + 4 * b))])
    assert ev.loglik_per_token(theta, phi, corp, 50.0, b) == pytest.approx(want, rel=1e-6)


# --------------------------------------------------------------- engine ------
def test_training_conservation_determinism_and_recount():
    K = 32
    corp = synth.shaped("tiny")
    cfg = engine.TrainConfig(num_topics=K, iterations=4, seed=3, check_conservation=True)
    th1, ph1, rep1 = engine.train(corp, cfg)
    assert all(r.conservation == "ok" for r in rep1)
    th2, ph2, rep2 = engine.train(corp, cfg)
    np.testing.assert_array_equal(ph1.counts, ph2.counts)
    np.testing.assert_array_equal(th1.counts, th2.counts)
    assert [r.loglik_per_token for r in rep1] == [r.loglik_per_token for r in rep2]
    # every count structure equals a recount of the exported assignments
    tr = engine.Trainer(corp, cfg)
    for _ in range(3):
        tr.step()
    z = tr.assignments()
    ch = tr.chunk
    oc, ot = oracle.rebuild_phi(z, ch.word_ids, K, corp.vocab_size)
    ph = tr.phi()
    np.testing.assert_array_equal(ph.counts, oc)
    np.testing.assert_array_equal(ph.topic_totals, ot)
    rp, ids, cn = oracle.rebuild_theta(z, ch.dw_ptr, ch.dw_tok, ch.doc_lo, K)
    th = tr.theta()
    np.testing.assert_array_equal(th.row_ptr, rp)
    np.testing.assert_array_equal(th.topic_ids, ids)
    np.testing.assert_array_equal(th.counts, cn)
    tr.close()


def _oracle_trajectory(corp, K, seed, iters):
    a, b = 50.0 / K, 0.01
    ch = cp.partition(corp, 1, K, seed)[0]
    z = ch.assignments.copy()
    lls = []
    for it in range(iters):
        rp, ids, cn = oracle.rebuild_theta(z, ch.dw_ptr, ch.dw_tok, 0, K)
        phi, tot = oracle.rebuild_phi(z, ch.word_ids, K, corp.vocab_size)
        lls.append(oracle.loglik_naive(K, corp.vocab_size, a, b, ch.doc_ids, ch.word_ids, rp, ids, cn,
                                       corp.doc_lengths, phi, tot))
        z = oracle.sample_tokens(K, corp.vocab_size, a, b, seed, it, ch.doc_ids, ch.word_ids, z, 0, rp, ids, cn,
                                 phi, tot)
    return np.array(lls)


def test_loglik_trajectory_within_1pct_of_oracle():
    """BASELINE config 1 (tiny: 1K docs, V=1K, ~100K tokens, K=32): the device
    trajectory stays within 1% of the oracle's at matched iterations."""
    K, iters = 32, 50
    corp = synth.shaped("tiny")
    cfg = engine.TrainConfig(num_topics=K, iterations=iters, seed=42)
    _, _, reps = engine.train(corp, cfg)
    gpu = np.array([r.loglik_per_token for r in reps])
    ref = _oracle_trajectory(corp, K, 42, iters)
    assert gpu[0] == pytest.approx(ref[0], rel=1e-6)        # same initial model
    assert np.max(np.abs(gpu - ref) / np.abs(ref)) < 0.01
    assert gpu[-1] > gpu[0] + 0.05                             # it converges


def test_k_sweep_iterations_conserve_counts():
    corp = synth.generate(2000, 5000, 300.0, seed=5)
    for K in (128, 256, 1024, 4096):
        cfg = engine.TrainConfig(num_topics=K, iterations=2, seed=1)
        tr = engine.Trainer(corp, cfg)
        for _ in range(2):
            tr.step()
        z = tr.assignments()
        assert (z < K).all()
        ph = tr.phi()
        oc, ot = oracle.rebuild_phi(z, tr.chunk.word_ids, K, corp.vocab_size)
        np.testing.assert_array_equal(ph.counts, oc)
        th = tr.theta()
        assert md.check_conservation(th, ph, corp).ok
        tr.close()


def test_sample_chunk_api():
    K = 16
    corp = synth.generate(100, 200, 50.0, seed=2)
    ch = cp.partition(corp, 1, K, 9)[0]
    theta = md.rebuild_theta(ch, K)
    phi = md.rebuild_phi_replica(ch, K, corp.vocab_size)
    ctx = sampler.SamplerContext(50.0 / K, 0.01, K, corp.vocab_size)
    z1 = sampler.sample_chunk(ch, phi, theta, ctx, iteration=1, seed=5)
    z2 = sampler.sample_chunk(ch, phi, theta, ctx, iteration=1, seed=5)
    np.testing.assert_array_equal(z1, z2)
    rp, ids, cn = theta.row_ptr, theta.topic_ids, theta.counts
    want = oracle.sample_tokens(K, corp.vocab_size, 50.0 / K, 0.01, 5, 1, ch.doc_ids, ch.word_ids,
                                ch.assignments, 0, rp, ids, cn, phi.counts, phi.topic_totals, mode="thin")
    assert np.mean(z1 == want) > 0.998


def test_sample_chunk_global_phi_and_heavy_first_directory():
    """with C > 1 a word that is light in this chunk can hold a
    GLOBAL phi cell above 65535 (sample_chunk must size the hybrid columns from
    the global phi), and a chunk in the heavy-first directory order of
    sort_word_groups_desc (corpus.py:290-302) is a valid input."""
    K, V = 2, 6
    r = np.random.default_rng(3)
    docs, words = [], []
    for d in range(100):                      # chunk 0: word 0 dominates (140K tokens)
        docs += [d] * 1410
        words += [0] * 1400 + list(r.integers(1, V, 10))
    for d in range(100, 4800):                # chunk 1 (same token count): word 0 is rare
        docs += [d] * 30
        words += [0] * 2 + list(r.integers(1, V, 28))
    corp = cp.corpus_from_tokens(np.array(docs), np.array(words), V)
    ch0, ch1 = cp.partition(corp, 2, K, 11)
    assert ch1.doc_lo == 100
    ph0 = md.rebuild_phi_replica(ch0, K, V)
    ph1 = md.rebuild_phi_replica(ch1, K, V)
    phi = engine.reduce_phi([ph0, ph1])
    assert phi.counts[:, 0].max() > 65535
    theta1 = md.rebuild_theta(ch1, K)
    ctx = sampler.SamplerContext(50.0 / K, 0.01, K, V)
    z1 = sampler.sample_chunk(ch1, phi, theta1, ctx, iteration=2, seed=5)
    want = oracle.sample_tokens(K, V, 50.0 / K, 0.01, 5, 2, ch1.doc_ids, ch1.word_ids, ch1.assignments, ch1.doc_lo,
                                theta1.row_ptr, theta1.topic_ids, theta1.counts, phi.counts, phi.topic_totals,
                                mode="thin")
    assert np.mean(z1 == want) > 0.998
    z2 = sampler.sample_chunk(cp.sort_word_groups_desc(ch1), phi, theta1, ctx, iteration=2, seed=5)
    np.testing.assert_array_equal(z1, z2)
    np.testing.assert_array_equal(md.rebuild_theta(cp.sort_word_groups_desc(ch1), K).counts, theta1.counts)


def test_two_device_shards_with_summed_sync_buffers_match_one_shard():
    """The multi-GPU protocol on one GPU: two shards (greedy_boundaries, C=2),
    replicas summed elementwise through their int32 sync-buffer views (what the
    NCCL allreduce does), K3 after the sum -- the model equals one shard's."""
    import torch

    K, iters = 32, 3
    corp = synth.generate(500, 800, 60.0, seed=21)
    two = cp.partition(corp, 2, K, 11)
    freq = np.bincount(corp.word_ids, minlength=corp.vocab_size)
    words = np.concatenate([c.word_ids for c in two])
    z0 = np.concatenate([c.assignments for c in two])[np.argsort(words, kind="stable")]
    one = cp.partition(corp, 1, K, 11)[0]
    from dataclasses import replace
    one = replace(one, assignments=z0)
    a, b = 50.0 / K, 0.01
    shards = [DeviceShard(K, corp.vocab_size, a, b, seed=5, global_word_freq=freq, heavy_threshold=30).load(c)
              for c in two]
    single = DeviceShard(K, corp.vocab_size, a, b, seed=5, global_word_freq=freq, heavy_threshold=30).load(one)

    def allreduce():
        for s in shards:
            s.synchronize()
        ts = [s.sync_tensor() for s in shards]
        tot = ts[0] + ts[1]
        for t in ts:
            t.copy_(tot)
        torch.cuda.synchronize()

    for s in shards:
        s.rebuild_phi()
    allreduce()
    for s in shards:
        s.prepare()
        s.rebuild_theta()
    single.initialize()
    for it in range(iters):
        for s in shards:
            s.sample(it)
        single.sample(it)
        ll2 = sum(s.loglik_sum() for s in shards)
        assert ll2 == pytest.approx(single.loglik_sum(), rel=1e-9)
        for s in shards:
            s.rebuild_phi()
        allreduce()
        for s in shards:
            s.rebuild_theta()
            s.prepare()
        single.rebuild_phi()
        single.prepare()
        single.rebuild_theta()
    p2, t2 = shards[0].get_phi()
    p1, t1 = single.get_phi()
    np.testing.assert_array_equal(p2, p1)
    np.testing.assert_array_equal(t2, t1)
    np.testing.assert_array_equal(shards[1].get_phi()[0], p1)
    th = md.concat_theta([md.ThetaRows(*s.get_theta(), K) for s in shards])
    rp, ids, cn = single.get_theta()
    np.testing.assert_array_equal(th.row_ptr, rp)
    np.testing.assert_array_equal(th.topic_ids, ids)
    np.testing.assert_array_equal(th.counts, cn)
    for s in shards + [single]:
        s.close()


@pytest.mark.parametrize("sched", [("256", "16"), ("64", "8"), ("1000000", "1024")])
def test_slice_schedule_is_scheduling_only(sched, monkeypatch):
    """Doc-blocked slice schedules (GF_DOCBLOCK_KB / GF_SLICE_MINRUNS), word
    contexts and the heavy-first zdoc order are scheduling: the same schedule
    is bit-deterministic, and against the flat schedule one iteration draws the
    same topics except where fp32 S differs by association (a row's position
    in a warp step changes the scan tree: ~1e-7 relative), the loglik agrees to
    1e-6, and the theta K3 rebuilds from zdoc equals a recount of the z."""
    K = 256
    corp = synth.generate(1500, 3000, 250.0, seed=31)
    ch = cp.partition(corp, 1, K, 7)[0]
    a, b = 50.0 / K, 0.01

    def run(kb, minruns):
        monkeypatch.setenv("GF_DOCBLOCK_KB", kb)
        monkeypatch.setenv("GF_SLICE_MINRUNS", minruns)
        sh = DeviceShard(K, corp.vocab_size, a, b, seed=3).load(ch)
        sh.initialize()
        sh.sample(0)
        ll = sh.loglik_sum()
        sh.rebuild_phi()
        sh.prepare()
        sh.rebuild_theta()
        sh.check_errors()
        out = (sh.get_assignments(), sh.get_theta(), ll, sh.stats())
        sh.close()
        return out

    z1, th1, ll1, st1 = run(*sched)
    z1b, th1b, ll1b, _ = run(*sched)
    z0, th0, ll0, st0 = run("1000000", "1000000000")
    np.testing.assert_array_equal(z1, z1b)                   # deterministic
    assert ll1 == ll1b
    assert st0["doc_blocks"] == 1
    if sched[0] != "1000000":
        assert st1["doc_blocks"] > 1 and st1["word_contexts"] > 0 and st1["slices"] > st0["slices"]
    assert np.mean(z1 == z0) > 0.9999
    assert ll1 == pytest.approx(ll0, rel=1e-6)
    rp, ids, cn = oracle.rebuild_theta(z1, ch.dw_ptr, ch.dw_tok, ch.doc_lo, K)
    np.testing.assert_array_equal(th1[0], rp)
    np.testing.assert_array_equal(th1[1], ids)
    np.testing.assert_array_equal(th1[2], cn)


# ------------------------------------------------------------------ K4 ------
@pytest.mark.parametrize("name", ["small", "single", "rand25", "zipf", "zipf_k1024"])
def test_partition_gpu_matches_reference_golden(name):
    """K4 (device radix sorts + splitmix64 z0 in fp64) reproduces the reference
    partition() outputs bit for bit (tests/golden/partition.npz, made by the
    reference's own corpus.partition)."""
    g = np.load(os.path.join(GOLD, "partition.npz"))
    m = next(x for x in json.loads(str(g["meta"])) if x["name"] == name)
    corp = cp.corpus_from_tokens(g[f"{name}__corpus_doc_ids"], g[f"{name}__corpus_word_ids"], m["V"])
    for ch in cp.partition(corp, m["C"], m["K"], m["seed"], device=0):
        pre = f"{name}__c{ch.chunk_id}__"
        assert [ch.doc_lo, ch.doc_hi, ch.token_count] == g[pre + "range"].tolist()
        for f in ("doc_ids", "word_ids", "assignments", "group_words", "group_offsets", "group_sizes",
                  "dw_ptr", "dw_tok"):
            np.testing.assert_array_equal(getattr(ch, f), g[pre + f], err_msg=f)
            assert getattr(ch, f).dtype == g[pre + f].dtype


@pytest.mark.parametrize("K", [7, 1024, 65535])
def test_partition_gpu_matches_host_on_larger_corpora(K):
    corp = synth.generate(3000, 20000, 120.0, seed=K)
    host = cp.partition(corp, 3, K, 99)
    dev = cp.partition(corp, 3, K, 99, device=0)
    for a, b in zip(host, dev):
        for f in ("doc_ids", "word_ids", "assignments", "group_words", "group_offsets", "group_sizes",
                  "dw_ptr", "dw_tok"):
            np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)


def test_partition_gpu_input_errors():
    with pytest.raises(ValueError):
        cp.make_chunk(0, 0, 2, np.array([0, 1]), np.array([0, 9]), 5, 4, 1, device=0)
    with pytest.raises(ValueError):
        cp.make_chunk(0, 0, 2, np.array([0, 3]), np.array([0, 1]), 5, 4, 1, device=0)


def test_load_tokens_equals_load_of_the_reference_chunk(monkeypatch):
    """gf_shard_load_tokens (partition + layout on the device) builds the same
    shard as partition() + gf_shard_load: same assignments, same counts, the
    same draws (same slice schedule) and the same loglik."""
    K = 256
    corp = synth.generate(2500, 4000, 200.0, seed=12)
    monkeypatch.setenv("GF_DOCBLOCK_KB", "256")
    monkeypatch.setenv("GF_SLICE_MINRUNS", "16")
    ch = cp.partition(corp, 1, K, 77)[0]
    a, b = 50.0 / K, 0.01
    outs = []
    for mode in ("chunk", "tokens"):
        sh = DeviceShard(K, corp.vocab_size, a, b, seed=5)
        if mode == "chunk":
            sh.load(ch)
        else:
            sh.load_tokens(0, corp.num_docs, corp.doc_ids, corp.word_ids, seed=77, chunk_id=0)
        z0 = sh.get_assignments()
        sh.initialize()
        th0 = sh.get_theta()
        for it in range(2):
            sh.sample(it)
            sh.rebuild_phi()
            sh.prepare()
            sh.rebuild_theta()
        sh.check_errors()
        outs.append((z0, th0, sh.get_assignments(), sh.get_phi(), sh.get_theta(), sh.loglik_sum(), sh.stats()))
        sh.close()
    (z0a, th0a, za, pa, tha, lla, sta), (z0b, th0b, zb, pb, thb, llb, stb) = outs
    np.testing.assert_array_equal(z0a, ch.assignments)
    np.testing.assert_array_equal(z0b, ch.assignments)
    for x, y in zip(th0a, th0b):
        np.testing.assert_array_equal(x, y)
    assert sta["slices"] == stb["slices"] and sta["doc_blocks"] == stb["doc_blocks"] > 1
    np.testing.assert_array_equal(za, zb)
    np.testing.assert_array_equal(pa[0], pb[0])
    np.testing.assert_array_equal(pa[1], pb[1])
    for x, y in zip(tha, thb):
        np.testing.assert_array_equal(x, y)
    assert lla == llb


def test_checkpoint_resume_repeats_the_uninterrupted_run(tmp_path):
    """GFCHUNK1 carries z, GFSNAP1 the model + iteration;
    draws are keyed by (seed, iteration, token), so 2 + checkpoint + resume +
    2 iterations equal 4 uninterrupted ones bit for bit."""
    K = 64
    corp = synth.generate(600, 1500, 120.0, seed=8)
    cfg = engine.TrainConfig(num_topics=K, iterations=4, seed=17)
    tr = engine.Trainer(corp, cfg)
    full = [tr.step().loglik_per_token for _ in range(4)]
    z_full, th_full, ph_full = tr.assignments(), tr.theta(), tr.phi()
    tr.close()
    tr = engine.Trainer(corp, cfg)
    first = [tr.step().loglik_per_token for _ in range(2)]
    prefix = str(tmp_path / "ckpt")
    tr.save_checkpoint(prefix)
    tr.close()
    tr = engine.Trainer.resume(corp, cfg, prefix)
    assert tr.iteration == 2
    rest = [tr.step().loglik_per_token for _ in range(2)]
    np.testing.assert_array_equal(tr.assignments(), z_full)
    np.testing.assert_array_equal(tr.phi().counts, ph_full.counts)
    np.testing.assert_array_equal(tr.theta().counts, th_full.counts)
    assert first + rest == full
    tr.close()


@pytest.mark.parametrize("K", [8192, 16384])
def test_large_k_streaming_path(K):
    """K > 4096: rows can outgrow the warp's staging buffer and take the
    warp-cooperative streaming path (huge_run); draws agree with the oracle's
    thin form and the counts stay exact."""
    corp = synth.generate(60, 400, 9000.0, seed=K % 97)          # long documents: nnz up to ~K
    ch = cp.partition(corp, 1, K, 5)[0]
    a, b = 50.0 / K, 0.01
    rp, ids, cn = oracle.rebuild_theta(ch.assignments, ch.dw_ptr, ch.dw_tok, 0, K)
    assert np.diff(rp).max() > 4096                             # some rows need the streaming path
    phi, tot = oracle.rebuild_phi(ch.assignments, ch.word_ids, K, corp.vocab_size)
    with DeviceShard(K, corp.vocab_size, a, b, seed=9) as sh:
        sh.load(ch)
        sh.initialize()
        sh.sample(0)
        sh.check_errors()
        z = sh.get_assignments()
        ll = sh.loglik_sum() / corp.num_tokens
        sh.rebuild_phi()
        sh.prepare()
        sh.rebuild_theta()
        sh.check_errors()
        grp, gids, gcn = sh.get_theta()
    want = oracle.sample_tokens(K, corp.vocab_size, a, b, 9, 0, ch.doc_ids, ch.word_ids, ch.assignments, 0,
                                rp, ids, cn, phi, tot, mode="thin")
    assert np.mean(z == want) > 0.995
    ll_ref = oracle.loglik_sq(K, corp.vocab_size, a, b, ch.doc_ids, ch.word_ids, 0, rp, ids, cn,
                              corp.doc_lengths, phi, tot)
    assert ll == pytest.approx(ll_ref, rel=1e-6)
    r2, i2, c2 = oracle.rebuild_theta(z, ch.dw_ptr, ch.dw_tok, 0, K)
    np.testing.assert_array_equal(grp, r2)
    np.testing.assert_array_equal(gids, i2)
    np.testing.assert_array_equal(gcn, c2)


def test_staged_import_applies_exactly_the_changed_runs():
    """Async imports are staged and applied per run where the topics differ:
    an unchanged round trip, then a sparse edit (every 7th token, plus the
    first and last token), each followed by the counts, must leave z, the
    doc-major copy (checked through K3) and phi equal to the oracle's."""
    import torch

    K = 64
    corp = synth.generate(400, 800, 60.0, seed=19)
    ch = cp.partition(corp, 1, K, 4)[0]
    T = corp.num_tokens
    host = torch.empty(T, dtype=torch.int16).pin_memory().numpy().view(np.uint16)
    with DeviceShard(K, corp.vocab_size, 50.0 / K, 0.01, seed=2, stream=torch.cuda.current_stream()) as sh:
        sh.load(ch)
        sh.initialize()
        sh.sample(0)
        for edit in (False, True):
            sh.copy_assignments_async(host, 0, T, False)
            torch.cuda.synchronize()
            if edit:
                idx = np.r_[0, np.arange(3, T, 7), T - 1]
                host[idx] = ((host[idx].astype(np.int64) + 5) % K).astype(np.uint16)
            want = host.copy()
            sh.copy_assignments_async(host, 0, T, True)
            sh.assignments_imported()
            sh.rebuild_phi()
            sh.prepare()
            sh.rebuild_theta()
            sh.check_errors()
            np.testing.assert_array_equal(sh.get_assignments(), want)
            rp, ids, cn = oracle.rebuild_theta(want, ch.dw_ptr, ch.dw_tok, 0, K)
            grp, gids, gcn = sh.get_theta()
            np.testing.assert_array_equal(gids, ids)
            np.testing.assert_array_equal(gcn, cn)
            phi, tot = oracle.rebuild_phi(want, ch.word_ids, K, corp.vocab_size)
            np.testing.assert_array_equal(sh.get_phi()[0], phi)
            sh.sample(1)                     # the sampler sees the imported state
            sh.check_errors()


def test_async_chunked_assignment_copies():
    """copy_assignments_async (chunks, copy streams) + assignments_imported: the
    e2e path of bench.py -- what comes back is what the device holds, and an
    imported state rebuilds the reference counts."""
    import torch

    K = 32
    corp = synth.generate(300, 600, 50.0, seed=14)
    ch = cp.partition(corp, 1, K, 2)[0]
    T = corp.num_tokens
    host = torch.empty(T, dtype=torch.int16).pin_memory().numpy().view(np.uint16)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with DeviceShard(K, corp.vocab_size, 50.0 / K, 0.01, seed=1, stream=torch.cuda.current_stream()) as sh:
        sh.load(ch)
        sh.initialize()
        sh.sample(0)
        cuts = np.linspace(0, T, 7).astype(int)
        torch.cuda.current_stream().synchronize()
        for c in range(6):
            sh.copy_assignments_async(host, cuts[c], cuts[c + 1] - cuts[c], False, s1 if c % 2 else s2)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(host, sh.get_assignments())
        new = ((host.astype(np.int64) * 7 + 3) % K).astype(np.uint16)
        host[:] = new
        for c in range(6):
            sh.copy_assignments_async(host, cuts[c], cuts[c + 1] - cuts[c], True, s1)
        torch.cuda.current_stream().wait_stream(s1)
        sh.assignments_imported()
        sh.rebuild_phi()
        sh.prepare()
        sh.rebuild_theta()
        sh.check_errors()
        np.testing.assert_array_equal(sh.get_assignments(), new)
        rp, ids, cn = oracle.rebuild_theta(new, ch.dw_ptr, ch.dw_tok, 0, K)
        grp, gids, gcn = sh.get_theta()
        np.testing.assert_array_equal(grp, rp)
        np.testing.assert_array_equal(gids, ids)
        np.testing.assert_array_equal(gcn, cn)
        phi, tot = oracle.rebuild_phi(new, ch.word_ids, K, corp.vocab_size)
        gphi, gtot = sh.get_phi()
        np.testing.assert_array_equal(gphi, phi)
        with pytest.raises(errors.ShapeMismatchError):
            sh.copy_assignments_async(host, T - 1, 5, True)


# ---------------------------------------------------------- K5 conservation --
def test_conservation_kernel_fault_injection():
    """K5 (gf_shard_conservation on the resident state, gf_check_conservation on
    exported arrays) reports the first violated invariant of model.py:180-225
    with the reference's text: the same answer as the oracle for a clean model
    and for an injected fault of each kind, in the reference's check order."""
    K = 24
    corp = synth.generate(300, 500, 40.0, seed=13)
    ch = cp.partition(corp, 1, K, 4)[0]
    rp, ids, cn = oracle_theta(ch, K)
    phi, tot = oracle.rebuild_phi(ch.assignments, ch.word_ids, K, corp.vocab_size)
    phi = phi.astype(np.uint32)
    L, T = corp.doc_lengths, corp.num_tokens
    freq = np.bincount(corp.word_ids, minlength=corp.vocab_size)

    def want(rp_, ids_, cn_, phi_, tot_):
        return oracle.check_conservation(rp_, ids_, cn_, phi_, tot_, L, T)[1]

    def exported(rp_, ids_, cn_, phi_, tot_):
        return md.check_conservation(md.ThetaRows(rp_, ids_, cn_, K), md.PhiMatrix(phi_, tot_), corp).detail

    with DeviceShard(K, corp.vocab_size, 0.5, 0.01, global_word_freq=freq) as sh:
        sh.load(ch)
        sh.initialize()

        def resident():
            row = sh.conservation(1)
            return md.conservation_report(*(row if row[0] else sh.conservation(2, T))).detail

        assert resident() == exported(rp, ids, cn, phi, tot) == want(rp, ids, cn, phi, tot) == "ok"
        # 1. a theta row off by one
        cn1 = cn.copy()
        cn1[rp[37]] += 1
        sh.set_theta(rp, ids, cn1)
        assert resident() == exported(rp, ids, cn1, phi, tot) == want(rp, ids, cn1, phi, tot)
        assert resident().startswith("theta row 37 sums to")
        # 2. one count moved between two topics of a row (row sums still right)
        d = int(np.flatnonzero((np.diff(rp) >= 2))[0])
        j = int(rp[d])
        cn2 = cn.copy()
        cn2[j] += 1
        cn2[j + 1] -= 1
        if cn2[j + 1] == 0:                  # keep the row a valid CSR row
            cn2[j + 1] += 1
            cn2[j] -= 1
            cn2[j] -= 1 if cn2[j] > 1 else 0
            cn2[j + 1] += 1 if cn[j] > 1 else 0
        sh.set_theta(rp, ids, cn2)
        w2 = want(rp, ids, cn2, phi, tot)
        assert w2 != "ok"
        assert resident() == exported(rp, ids, cn2, phi, tot) == w2
        sh.set_theta(rp, ids, cn)
        # 3. one phi cell moved to another topic (phi row sums off, totals stored)
        phi3 = phi.copy()
        v = int(np.flatnonzero(phi3[2])[0])
        phi3[2, v] -= 1
        phi3[9, v] += 1
        sh.set_phi(phi3, tot)
        w3 = want(rp, ids, cn, phi3, tot)
        assert w3.startswith("topic 2: phi row sum")
        assert resident() == exported(rp, ids, cn, phi3, tot) == w3
        # 4. stored totals moved with phi but not with theta
        tot4 = tot.copy()
        tot4[3] += 1
        phi4 = phi.copy()
        phi4[3, v] += 1
        sh.set_phi(phi4, tot4)
        w4 = want(rp, ids, cn, phi4, tot4)
        assert w4.startswith("topic 3: theta column sum")
        assert resident() == exported(rp, ids, cn, phi4, tot4) == w4
    # 5. the total check (exported arrays: empty model of a non-empty corpus)
    Lz = np.zeros_like(L)
    rpz = np.zeros(len(L) + 1, np.int64)
    e16 = np.zeros(0, np.uint16)
    phz, totz = np.zeros((K, corp.vocab_size), np.uint16), np.zeros(K, np.int64)
    want5 = oracle.check_conservation(rpz, e16, e16, phz, totz, Lz, T)[1]
    assert want5 == f"totals sum to 0, corpus has {T} tokens"
    from paper_1803_04631_b200 import _lib

    rep = np.zeros(8, np.int64)
    _lib.check(_lib.lib().gf_check_conservation(0, K, corp.vocab_size, len(L), _lib.ptr(rpz), _lib.ptr(e16),
                                                _lib.ptr(e16), _lib.ptr(Lz), _lib.ptr(phz), 16, _lib.ptr(totz), T,
                                                _lib.ptr(rep)))
    assert rep[0] == 0 and md.conservation_report(*rep[4:]).detail == want5


def test_conservation_golden_texts_on_device():
    """The reference's own ConservationReport texts (tests/golden/messages.json,
    written by gibbsflow.model.check_conservation) from the device check."""
    import test_oracle_golden as tog

    msgs = json.load(open(os.path.join(GOLD, "messages.json")))
    for name, corp, rp, ids, cn, phi, tot in tog.conservation_cases():
        c = cp.corpus_from_tokens(corp["doc_ids"], corp["word_ids"], corp["V"])
        th = md.ThetaRows(rp, ids.astype(np.uint16), cn.astype(np.uint16), phi.shape[0])
        got = md.check_conservation(th, md.PhiMatrix(phi.astype(np.uint32), tot), c)
        assert got.detail == msgs[name], name
        assert got.ok == (name == "conservation_ok")


def test_set_phi_rejects_light_column_overflow_on_device():
    """gf_shard_set_phi checks the 16-bit (light) columns on the device and names
    the first offending cell in word-major order; heavy columns take any u32."""
    K, V = 4, 6
    corp = synth.generate(40, V, 20.0, seed=3)
    ch = cp.partition(corp, 1, K, 1)[0]
    freq = np.bincount(corp.word_ids, minlength=V)
    with DeviceShard(K, V, 0.5, 0.01, global_word_freq=freq, heavy_threshold=int(freq.max()) - 1) as sh:
        sh.load(ch)
        sh.initialize()
        phi, tot = sh.get_phi()
        heavy = int(np.argmax(freq))
        light = [v for v in range(V) if v != heavy]
        big = phi.copy()
        big[1, heavy] = 100000                      # heavy (u32) column: accepted
        sh.set_phi(big, tot + np.eye(K, dtype=np.int64)[1] * (100000 - int(phi[1, heavy])))
        bad = phi.copy()
        bad[2, light[3]] = 70000
        bad[0, light[4]] = 80000
        with pytest.raises(errors.CountOverflowError) as ei:
            sh.set_phi(bad, tot)
        assert str(ei.value) == f"phi cell (topic 2, word {light[3]}) count 70000 exceeds its 16-bit column"


def test_drop_in_api_keeps_the_chunk_resident():
    """sample_chunk / rebuild_theta / rebuild_phi_replica reuse one resident
    shard per chunk (shard.RESIDENT): the K4 layout runs once, a
    dataclasses.replace() of the chunk with new assignments hits the same
    shard, and every result equals a cold call's."""
    from dataclasses import replace

    from paper_1803_04631_b200.shard import RESIDENT

    K = 16
    corp = synth.generate(300, 400, 50.0, seed=12)
    ch = cp.partition(corp, 1, K, 9)[0]
    ctx = sampler.SamplerContext(50.0 / K, 0.01, K, corp.vocab_size)
    RESIDENT.release()

    def one_iteration(c, it):
        th = md.rebuild_theta(c, K)
        ph = md.rebuild_phi_replica(c, K, corp.vocab_size, width=16)
        z = sampler.sample_chunk(c, ph, th, ctx, iteration=it, seed=3)
        return th, ph, z

    warm, c = [], ch
    for it in range(3):
        th, ph, z = one_iteration(c, it)
        warm.append((th, ph, z))
        c = replace(c, assignments=z)
    assert len(RESIDENT._lru) == 1                 # one shard served all nine calls
    cold, c = [], ch
    for it in range(3):
        RESIDENT.release()
        th, ph, z = one_iteration(c, it)
        cold.append((th, ph, z))
        c = replace(c, assignments=z)
    for (t1, p1, z1), (t2, p2, z2) in zip(warm, cold):
        np.testing.assert_array_equal(t1.counts, t2.counts)
        np.testing.assert_array_equal(t1.topic_ids, t2.topic_ids)
        assert p1.counts.dtype == np.uint16
        np.testing.assert_array_equal(p1.counts, p2.counts)
        np.testing.assert_array_equal(z1, z2)
    # the oracle agrees with the warm path's draws (thin form)
    th, ph, z = warm[1]
    want = oracle.sample_tokens(K, corp.vocab_size, 50.0 / K, 0.01, 3, 1, ch.doc_ids, ch.word_ids, warm[0][2], 0,
                                th.row_ptr, th.topic_ids, th.counts, ph.counts, ph.topic_totals, mode="thin")
    assert np.mean(z == want) > 0.998
    # loglik through the resident corpus shard: twice, same value
    l1 = ev.loglik_per_token(th, ph, corp, 50.0 / K, 0.01)
    l2 = ev.loglik_per_token(th, ph, corp, 50.0 / K, 0.01)
    assert l1 == l2
    RESIDENT.release()


def test_api_results_live_in_cached_pinned_blocks():
    """The one-call API returns its large arrays in pinned blocks
    (_lib.pinned_empty / gf_host_alloc): ordinary writeable numpy arrays,
    private to each call (a freed block is reused only after its last array
    is gone), and an edit made in place -- the reference's own fault-injection
    pattern (test_model.py:169-184) -- is what the next call sees."""
    from paper_1803_04631_b200 import _lib
    from paper_1803_04631_b200.shard import RESIDENT

    def pinned(a):
        while a is not None and not isinstance(a, _lib._PinnedBlock):
            a = a.base
        return a is not None

    K = 64
    corp = synth.generate(30000, 6000, 80.0, seed=21)         # ~2.4M tokens, K x V: every result array >= 1 MiB
    ch = cp.partition(corp, 1, K, 5)[0]
    RESIDENT.release()
    th1 = md.rebuild_theta(ch, K)
    ph1 = md.rebuild_phi_replica(ch, K, corp.vocab_size, width=32)
    assert pinned(th1.topic_ids) and pinned(th1.counts) and pinned(ph1.counts)
    assert th1.counts.flags.writeable and ph1.counts.flags.writeable
    keep = th1.counts.copy()
    th2 = md.rebuild_theta(ch, K)
    assert not np.shares_memory(th1.counts, th2.counts)
    np.testing.assert_array_equal(th2.counts, keep)
    del th1
    th3 = md.rebuild_theta(ch, K)                              # may reuse th1's block
    np.testing.assert_array_equal(th2.counts, keep)            # th2 untouched
    np.testing.assert_array_equal(th3.counts, keep)
    assert md.check_conservation(th3, ph1, corp).ok
    th3.counts[th3.row_ptr[1]] += 1                            # reference test_model.py:184
    rep = md.check_conservation(th3, ph1, corp)
    assert not rep.ok and "row 1" in rep.detail
    ph1.counts[1, 0] += 1                                      # reference test_model.py:169-170
    ph1.topic_totals[1] += 1
    th4 = md.rebuild_theta(ch, K)
    ctx = sampler.SamplerContext(50.0 / K, 0.01, K, corp.vocab_size)
    z = sampler.sample_chunk(ch, md.rebuild_phi_replica(ch, K, corp.vocab_size), th4, ctx, iteration=1, seed=3)
    assert pinned(z) and z.dtype == np.uint16 and len(z) == corp.num_tokens
    RESIDENT.release()
