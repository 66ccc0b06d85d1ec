"""Document-block phases (gf_shard_set_block_phases / phase_doc_range) and the
document-major assignment transfers (gf_shard_copy_doc_assignments_async /
doc_assignments_imported) that the end-to-end step streams with.

Block phases reorder the slice schedule only (the slices themselves, hence
every warp step's rows, are the same), so running them in order is the
unphased gf_shard_sample bit for bit; a document range is final once its
phase has run; a doc-major round trip is exact and a doc-major import keeps
z and its doc-major copy consistent.
"""

import numpy as np
import pytest

from paper_1803_04631_b200 import corpus as cp
from paper_1803_04631_b200 import synth
from paper_1803_04631_b200.shard import DeviceShard

pytestmark = pytest.mark.gpu

K = 128
CUTS = [0.5, 0.75, 0.9, 1.0]


@pytest.fixture(scope="module")
def chunk():
    corp = synth.generate(6000, 800, 120.0, seed=43)
    return corp, cp.partition(corp, 1, K, 9)[0]


@pytest.fixture(autouse=True)
def small_blocks(monkeypatch):
    # many document blocks and block-scheduled words on a small corpus
    monkeypatch.setenv("GF_DOCBLOCK_KB", "48")
    monkeypatch.setenv("GF_SLICE_MINRUNS", "8")


def _shard(corp, ch, block_cuts=None):
    sh = DeviceShard(K, corp.vocab_size, 50.0 / K, 0.01, seed=5)
    if block_cuts is not None:
        sh.set_block_phases(block_cuts)
    sh.load(ch)
    sh.initialize()
    return sh


def _counts(sh):
    sh.rebuild_phi()
    sh.prepare()
    sh.rebuild_theta()
    sh.check_errors()


def _doc_major(sh):
    out = np.empty(sh.num_tokens, np.uint16)
    sh.copy_doc_assignments_async(out, 0, sh.num_tokens, False)
    sh.synchronize()
    return out


def test_block_phase_ranges_tile_the_doc_major_order(chunk):
    corp, ch = chunk
    sh = _shard(corp, ch, CUTS)
    assert sh.stats()["doc_blocks"] > 4
    P = sh.num_phases
    assert P == len(CUTS) + 1
    ranges = [sh.phase_doc_range(p) for p in range(P)]
    assert ranges[0] == (0, 0)                       # the unblocked words own no range
    assert ranges[1][0] == 0 and ranges[-1][1] == ch.token_count
    for (a0, b0), (a1, b1) in zip(ranges[1:], ranges[2:]):
        assert b0 == a1 and a0 <= b0
    assert sum(b > a for a, b in ranges[1:]) >= 3      # several non-empty block ranges
    sh.close()


def test_block_phases_in_order_equal_one_sample(chunk):
    corp, ch = chunk
    a, b = _shard(corp, ch), _shard(corp, ch, CUTS)
    for it in range(3):
        a.sample(it)
        for p in range(b.num_phases):
            b.sample_phase(it, p)
        assert a.loglik_sum() == b.loglik_sum()
        np.testing.assert_array_equal(a.get_assignments(), b.get_assignments())
        _counts(a)
        _counts(b)
    a.close()
    b.close()


def test_doc_range_is_final_after_its_phase(chunk):
    corp, ch = chunk
    sh = _shard(corp, ch, CUTS)
    P = sh.num_phases
    early = {}
    for p in range(P):
        sh.sample_phase(0, p)
        if p >= 1:
            lo, hi = sh.phase_doc_range(p)
            early[p] = _doc_major(sh)[lo:hi].copy()
    final = _doc_major(sh)
    for p, got in early.items():
        lo, hi = sh.phase_doc_range(p)
        np.testing.assert_array_equal(final[lo:hi], got)
    sh.close()


def test_doc_major_round_trip_and_import(chunk):
    corp, ch = chunk
    sh = _shard(corp, ch, CUTS)
    sh.sample(0)
    _counts(sh)
    zd = _doc_major(sh)
    z = sh.get_assignments()
    # an unchanged round trip changes nothing
    host = np.ascontiguousarray(zd)
    sh.copy_doc_assignments_async(host, 0, len(host), True)
    sh.doc_assignments_imported()
    _counts(sh)
    np.testing.assert_array_equal(sh.get_assignments(), z)
    np.testing.assert_array_equal(_doc_major(sh), zd)
    # a sparse edit arrives in both orders and the counts stay conserved
    r = np.random.default_rng(7)
    idx = r.choice(len(host), size=500, replace=False)
    edited = host.copy()
    edited[idx] = (edited[idx].astype(np.int64) + 1 + r.integers(0, K - 1, len(idx))) % K
    sh.copy_doc_assignments_async(edited, 0, len(edited), True)
    sh.doc_assignments_imported()
    _counts(sh)
    np.testing.assert_array_equal(_doc_major(sh), edited)
    z2 = sh.get_assignments()
    assert np.count_nonzero(z2 != z) == len(idx)
    assert np.array_equal(np.sort(z2[z2 != z]), np.sort(edited[idx]))
    code = sh.conservation(1, ch.token_count)[0]
    assert code == 0
    assert sh.conservation(2, ch.token_count)[0] == 0
    sh.close()
