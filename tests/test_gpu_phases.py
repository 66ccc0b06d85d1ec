"""Streamed sampling phases (gf_shard_set_phases / sample_phase / phase_range).

A phase-split schedule is scheduling only: running the phases in order is one
gf_shard_sample bit for bit, the phases' z ranges tile the word-group order,
and against the unsplit schedule the draws agree except where an fp32 S sum
rounds differently (same bar as test_slice_schedule_is_scheduling_only).
"""

import numpy as np
import pytest

import oracle
from paper_1803_04631_b200 import corpus as cp
from paper_1803_04631_b200 import synth
from paper_1803_04631_b200.shard import DeviceShard

pytestmark = pytest.mark.gpu

K = 256


@pytest.fixture(scope="module")
def chunk():
    corp = synth.generate(1200, 2500, 180.0, seed=41)
    return corp, cp.partition(corp, 1, K, 9)[0]


def _shard(corp, ch, phases):
    sh = DeviceShard(K, corp.vocab_size, 50.0 / K, 0.01, seed=5, phases=phases).load(ch)
    sh.initialize()
    return sh


def _counts(sh):
    sh.rebuild_phi()
    sh.prepare()
    sh.rebuild_theta()
    sh.check_errors()


@pytest.mark.parametrize("P", [1, 2, 5])
def test_phase_ranges_tile_the_assignments(chunk, P):
    corp, ch = chunk
    sh = _shard(corp, ch, P)
    assert sh.num_phases == P
    ranges = [sh.phase_range(p) for p in range(P)]
    assert ranges[0][0] == 0 and ranges[-1][1] == ch.token_count
    for (a0, b0), (a1, b1) in zip(ranges, ranges[1:]):
        assert b0 == a1 and a0 <= b0
    # boundaries fall on word-group boundaries
    starts = set(int(x) for x in ch.group_offsets) | {ch.token_count}
    assert all(a in starts for a, _ in ranges)
    if P > 1:   # roughly T/P tokens each (word granularity)
        sizes = np.array([b - a for a, b in ranges])
        assert sizes.max() < 2.5 * ch.token_count / P
    sh.close()


def test_phases_in_order_equal_one_sample(chunk):
    corp, ch = chunk
    a, b = _shard(corp, ch, 4), _shard(corp, ch, 4)
    for it in range(3):
        a.sample(it)
        for p in range(4):
            b.sample_phase(it, p)
        assert a.loglik_sum() == b.loglik_sum()
        np.testing.assert_array_equal(a.get_assignments(), b.get_assignments())
        _counts(a)
        _counts(b)
    a.close()
    b.close()


def test_phase_output_is_final_after_its_phase(chunk):
    """z[phase_range(p)] is written by phase p alone: later phases leave it."""
    corp, ch = chunk
    sh = _shard(corp, ch, 3)
    sh.sample_phase(0, 0)
    sh.synchronize()
    lo, hi = sh.phase_range(0)
    z0 = sh.get_assignments()[lo:hi].copy()
    sh.sample_phase(0, 1)
    sh.sample_phase(0, 2)
    np.testing.assert_array_equal(sh.get_assignments()[lo:hi], z0)
    sh.close()


def test_phase_split_is_scheduling_only(chunk):
    corp, ch = chunk
    one, four = _shard(corp, ch, 1), _shard(corp, ch, 4)
    one.sample(0)
    four.sample(0)
    z1, z4 = one.get_assignments(), four.get_assignments()
    assert np.mean(z1 == z4) > 0.9999
    assert four.loglik_sum() == pytest.approx(one.loglik_sum(), rel=1e-6)
    _counts(four)
    rp, ids, cn = oracle.rebuild_theta(z4, ch.dw_ptr, ch.dw_tok, ch.doc_lo, K)
    th = four.get_theta()
    np.testing.assert_array_equal(th[1], ids)
    np.testing.assert_array_equal(th[2], cn)
    one.close()
    four.close()


def test_phase_arguments_are_checked(chunk):
    corp, ch = chunk
    sh = _shard(corp, ch, 2)
    with pytest.raises(ValueError, match="phase 2 out of range"):
        sh.sample_phase(0, 2)
    with pytest.raises(ValueError, match="out of range"):
        sh.phase_range(-1)
    with pytest.raises(ValueError, match="phases must be"):
        sh.set_phases(0)
    sh.close()


def test_more_phases_than_word_groups():
    """Phases beyond the number of word groups are empty (no launch) and the
    phase sequence still equals one sample."""
    corp = synth.generate(60, 40, 30.0, seed=3)
    ch = cp.partition(corp, 1, K, 1)[0]
    a, b = _shard(corp, ch, 1), _shard(corp, ch, 100)
    assert b.num_phases == 100
    ranges = [b.phase_range(p) for p in range(100)]
    assert sum(1 for x, y in ranges if y > x) <= ch.num_groups
    assert ranges[0][0] == 0 and ranges[-1][1] == ch.token_count
    a.sample(0)
    for p in range(100):
        b.sample_phase(0, p)
    assert a.loglik_sum() == pytest.approx(b.loglik_sum(), rel=1e-6)
    assert np.mean(a.get_assignments() == b.get_assignments()) > 0.999
    a.close()
    b.close()


def test_uneven_phase_cuts():
    """set_phases(sequence): phase p holds the groups starting below cuts[p] * T."""
    corp = synth.generate(1200, 2500, 180.0, seed=41)
    ch = cp.partition(corp, 1, K, 9)[0]
    cuts = [0.5, 0.75, 0.875, 1.0]
    sh = _shard(corp, ch, cuts)
    assert sh.num_phases == 4
    T = ch.token_count
    starts = np.asarray(ch.group_offsets)
    for p, c in enumerate(cuts):
        lo, hi = sh.phase_range(p)
        inside = starts[(starts >= lo) & (starts < hi)]
        assert np.all(inside < c * T)                         # every group of phase p starts below its cut
        if p + 1 < len(cuts) and hi < T:
            assert hi >= c * T                               # and the next group starts at or above it
    one = _shard(corp, ch, 1)
    one.sample(0)
    for p in range(4):
        sh.sample_phase(0, p)
    assert np.mean(one.get_assignments() == sh.get_assignments()) > 0.9999
    for bad in ([0.5, 0.4, 1.0], [0.5, 0.9], [0.0, 1.0]):
        with pytest.raises(ValueError, match="phase cuts"):
            sh.set_phases(bad)
    one.close()
    sh.close()


@pytest.mark.parametrize("P", [1, 5])
def test_sample_export_equals_sample_then_copy(chunk, P, monkeypatch):
    """gf_shard_sample_export (sample_chunk's device half: each phase's
    assignments copied back while the later phases sample) returns exactly
    what sample + get_assignments gives, and leaves the same device state."""
    from paper_1803_04631_b200 import _lib

    monkeypatch.setattr(_lib, "_PINNED_MIN", 0)      # a pinned result: the overlapped path
    corp, ch = chunk
    a, b = _shard(corp, ch, P), _shard(corp, ch, P)
    for it in range(3):
        a.sample(it)
        za = a.get_assignments()
        zb = b.sample_export(it)
        np.testing.assert_array_equal(za, zb)
        np.testing.assert_array_equal(b.get_assignments(), zb)
        assert a.loglik_sum() == b.loglik_sum()
        _counts(a)
        _counts(b)
    a.close()
    b.close()
