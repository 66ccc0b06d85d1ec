"""Multi-rank engine logic on CPU: world_size 2 over torch.distributed/gloo with
the oracle-backed shard (tests/oracle_shard.py) in place of the device shard.

Checks the distributed protocol of engine.Trainer -- document sharding by
greedy_boundaries, global word-frequency allreduce (fixes the hybrid phi
layout), the packed phi sync-buffer allreduce (u16 pairs summed as int32
without carries), loglik reduction, theta gather -- and the G-invariance the
token-keyed Philox stream promises: 2 ranks train the identical model as 1.
"""

import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _corpus():
    from paper_1803_04631_b200 import synth

    # vocabulary with a few words above the 16-bit column threshold (scaled down
    # to threshold 40 here) so both phi column widths travel through the allreduce
    return synth.generate(300, 400, 30.0, seed=5)


CFG = dict(num_topics=16, iterations=3, seed=7, heavy_threshold=40)


def _run_rank(rank, world, port, out):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle_shard import OracleShard
    from paper_1803_04631_b200 import engine

    corp = _corpus()
    tr = engine.Trainer(corp, engine.TrainConfig(workers=world, check_conservation=True, **CFG),
                        shard_factory=OracleShard)
    reps = [tr.step() for _ in range(CFG["iterations"])]
    lls = [r.loglik_per_token for r in reps]
    theta = tr.theta(gather=True)
    phi = tr.phi()
    z = [None] * world
    dist.all_gather_object(z, (tr.chunk.doc_lo, tr.chunk.doc_hi, tr.assignments()))
    # K5 across ranks: rank 1 corrupts its first theta row -> every rank reports
    # that document by its global index; the rank-summed columns catch a
    # column fault that no single rank sees
    rp, ids, cn = tr.shard.theta
    if rank == 1:
        cn = cn.copy()
        cn[0] += 1
        tr.shard.theta = (rp, ids, cn)
    row_fault = tr.conservation().detail
    if rank == 1:
        cn = cn.copy()
        cn[0] -= 1
        k0, k1 = int(ids[0]), int(ids[1])
        ids = ids.copy()
        ids[0], ids[1] = ids[1], ids[0]                  # moves counts between topics k0 and k1
        tr.shard.theta = (rp, ids, cn)
    col_fault = tr.conservation().detail
    if rank == 0:
        np.savez(out, lls=np.array(lls), phi=phi.counts, tot=phi.topic_totals, rp=theta.row_ptr,
                 ids=theta.topic_ids, cn=theta.counts, bounds=np.array([(a, b) for a, b, _ in z]),
                 cons=np.array([r.conservation for r in reps] + [row_fault, col_fault]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def two_rank_result():
    out = os.path.join(tempfile.mkdtemp(), "r.npz")
    mp.spawn(_run_rank, args=(2, _free_port(), out), nprocs=2, join=True)
    return np.load(out)


def test_two_ranks_train_the_same_model_as_one(two_rank_result):
    from oracle_shard import OracleShard
    from paper_1803_04631_b200 import corpus as cp
    from paper_1803_04631_b200 import engine

    corp = _corpus()
    # same initial state as the 2-rank run: partition()'s z0 is keyed by
    # (seed, chunk id), so map the two chunks' draws into the single chunk's
    # word-group order (a stable word sort of the concatenated chunks)
    two = cp.partition(corp, 2, CFG["num_topics"], CFG["seed"])
    words = np.concatenate([c.word_ids for c in two])
    z0 = np.concatenate([c.assignments for c in two])[np.argsort(words, kind="stable")]
    tr = engine.Trainer(corp, engine.TrainConfig(workers=1, **CFG), shard_factory=OracleShard, init_assignments=z0)
    lls = [tr.step().loglik_per_token for _ in range(CFG["iterations"])]
    theta, phi = tr.theta(), tr.phi()
    r = two_rank_result
    np.testing.assert_array_equal(r["phi"], phi.counts)
    np.testing.assert_array_equal(r["tot"], phi.topic_totals)
    np.testing.assert_array_equal(r["rp"], theta.row_ptr)
    np.testing.assert_array_equal(r["ids"], theta.topic_ids)
    np.testing.assert_array_equal(r["cn"], theta.counts)
    np.testing.assert_allclose(r["lls"], lls, rtol=1e-12)
    # shards are greedy_boundaries(C = G) (corpus.py:210-237)
    assert [tuple(b) for b in r["bounds"]] == cp.greedy_boundaries(corp.doc_lengths, 2)


def test_two_rank_conservation_reports(two_rank_result):
    """Trainer.conservation (K5 protocol: local row check, rank-summed theta
    columns) over 2 gloo ranks: ok every iteration, and the reference's texts
    (model.py:180-225) for an injected row fault and column fault."""
    from paper_1803_04631_b200 import corpus as cp

    corp = _corpus()
    cons = [str(c) for c in two_rank_result["cons"]]
    assert cons[:-2] == ["ok"] * CFG["iterations"]
    lo1 = cp.greedy_boundaries(corp.doc_lengths, 2)[1][0]
    assert cons[-2].startswith(f"theta row {lo1} sums to ") and cons[-2].endswith(
        f"document length is {int(corp.doc_lengths[lo1])}")
    assert cons[-1].startswith("topic ") and ": theta column sum " in cons[-1] and "!= phi total" in cons[-1]


def test_packed_phi_allreduce_is_exact(two_rank_result):
    """The summed sync buffer equals a recount of all final assignments."""
    import oracle

    r = two_rank_result
    assert int(r["tot"].sum()) == _corpus().num_tokens
    assert (r["phi"].sum(axis=1) == r["tot"]).all()


def test_reduce_phi_spec_examples():
    from paper_1803_04631_b200 import engine
    from paper_1803_04631_b200.model import PhiMatrix

    a = PhiMatrix(np.array([[1, 2], [3, 4]], np.uint32), np.array([3, 7]))
    b = PhiMatrix(np.array([[5, 6], [7, 8]], np.uint32), np.array([11, 15]))
    g = engine.reduce_phi([a, b], 2)
    assert g.counts.tolist() == [[6, 8], [10, 12]] and g.topic_totals.tolist() == [14, 22]
    rng = np.random.default_rng(0)
    for G in (3, 5, 8):
        reps = [PhiMatrix(rng.integers(0, 50, (3, 4)).astype(np.uint32), np.zeros(3, np.int64)) for _ in range(G)]
        g = engine.reduce_phi(reps, G)
        np.testing.assert_array_equal(g.counts, np.sum([p.counts for p in reps], axis=0))
    handles = engine.broadcast_phi(g, 4)
    assert len(handles) == 4 and all(h is handles[0] for h in handles)


def _run_rank_resume(rank, world, port, out, prefix):
    """2 iterations, checkpoint, a NEW trainer resumes and runs the 3rd."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle_shard import OracleShard
    from paper_1803_04631_b200 import engine

    corp = _corpus()
    cfg = engine.TrainConfig(workers=world, **CFG)
    tr = engine.Trainer(corp, cfg, shard_factory=OracleShard)
    lls = [tr.step().loglik_per_token for _ in range(2)]
    tr.save_checkpoint(prefix)
    tr.close()
    from paper_1803_04631_b200.model import load_snapshot

    tr = engine.Trainer.resume(corp, cfg, prefix, shard_factory=OracleShard)
    meta = load_snapshot(f"{prefix}.gfsnap")[2]
    lls.append(tr.step().loglik_per_token)
    theta = tr.theta(gather=True)
    phi = tr.phi()
    if rank == 0:
        np.savez(out, lls=np.array(lls), phi=phi.counts, rp=theta.row_ptr, cn=theta.counts,
                 it=np.array([meta["iteration"], meta["workers"]]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_checkpoint_resume_repeats_the_run(two_rank_result, tmp_path):
    """Every rank writes its GFCHUNK1 (z) and rank 0 the GFSNAP1 snapshot; the
    resumed 2-rank run continues exactly where the uninterrupted one went."""
    out = str(tmp_path / "resume.npz")
    prefix = str(tmp_path / "ckpt")
    mp.spawn(_run_rank_resume, args=(2, _free_port(), out, prefix), nprocs=2, join=True)
    r, full = np.load(out), two_rank_result
    assert r["it"].tolist() == [2, 2]
    assert os.path.exists(prefix + ".rank0.gfc") and os.path.exists(prefix + ".rank1.gfc")
    np.testing.assert_array_equal(r["phi"], full["phi"])
    np.testing.assert_array_equal(r["rp"], full["rp"])
    np.testing.assert_array_equal(r["cn"], full["cn"])
    np.testing.assert_allclose(r["lls"], full["lls"], rtol=1e-12)
