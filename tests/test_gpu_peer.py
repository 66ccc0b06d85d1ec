"""Peer-memory phi exchange (csrc/k_peer.cu) on the GPU.

Two ranks run as two processes on cuda:0 (the GPU box has one GPU; CUDA IPC
maps another process's allocation on the same device exactly like a peer
GPU's, and the exchange kernel's cross-rank barriers only wait for blocks of
the OTHER process, which the device time-slices in).  torch.distributed/gloo
carries the IPC handles and the reference sums.

Checks: one exchange == the elementwise uint32 sum of the two replicas (the
all_reduce it replaces), bit-exact; repeated exchanges (epochs) stay exact;
the fused K2 + exchange kernel (K2X, what gf_shard_iterate runs with a peer
group) gives the same sum;
a Trainer with phi_sync="peer" keeps phi/n_k conserved against the gathered
assignments every iteration and tracks the one-rank loglik.
"""

import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _corpus():
    from paper_1803_04631_b200 import synth

    return synth.generate(600, 500, 40.0, seed=11)


CFG = dict(num_topics=64, seed=3, heavy_threshold=60)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1803_04631_b200 import engine
    from paper_1803_04631_b200.corpus import greedy_boundaries, make_chunk
    from paper_1803_04631_b200.shard import DeviceShard

    corp = _corpus()
    K, V = CFG["num_topics"], corp.vocab_size
    res = {}

    # --- 1. raw exchange vs the elementwise sum of the replicas
    lo, hi = greedy_boundaries(corp.doc_lengths, world)[rank]
    a, b = int(corp.doc_ptr[lo]), int(corp.doc_ptr[hi])
    chunk = make_chunk(rank, lo, hi, corp.doc_ids[a:b], corp.word_ids[a:b], V, K, 5)
    freq = torch.as_tensor(np.bincount(chunk.word_ids, minlength=V).astype(np.int64))
    dist.all_reduce(freq)
    sh = DeviceShard(K, V, 50.0 / K, 0.01, seed=5, device=0, heavy_threshold=CFG["heavy_threshold"],
                     global_word_freq=freq.numpy())
    sh.load(chunk)
    sh.rebuild_phi()
    sh.synchronize()
    mine = sh.sync_tensor().cpu()
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    expect = torch.stack(parts).view(torch.int32).sum(0, dtype=torch.int64).to(torch.int32)
    handles = [None] * world
    dist.all_gather_object(handles, sh.peer_handle())
    sh.peer_open(rank, world, handles)
    sh.peer_allreduce()
    sh.synchronize()
    sh.check_errors()
    got = sh.sync_tensor().cpu()
    res["exchange_exact"] = bool(torch.equal(got, expect))
    res["n_words"] = int(got.numel())
    # epochs: rebuild + exchange again, several times
    ok = True
    for _ in range(3):
        sh.rebuild_phi()
        sh.peer_allreduce()
        sh.synchronize()
        ok &= bool(torch.equal(sh.sync_tensor().cpu(), expect))
    sh.check_errors()
    res["epochs_exact"] = ok
    # K2X: the replica rebuild fused with the stripe-pipelined exchange
    ok = True
    for _ in range(3):
        sh.rebuild_phi_exchange()
        sh.synchronize()
        ok &= bool(torch.equal(sh.sync_tensor().cpu(), expect))
    sh.check_errors()
    res["fused_exact"] = ok
    sh.peer_close()
    sh.close()

    # --- 2. Trainer with phi_sync="peer": conservation every iteration
    cfg = engine.TrainConfig(workers=world, phi_sync="peer", check_conservation=True, **CFG)
    tr = engine.Trainer(corp, cfg, device=0)
    reps = [tr.step() for _ in range(4)]
    res["conservation"] = [r.conservation for r in reps]
    res["lls"] = [r.loglik_per_token for r in reps]
    if rank == 0:
        np.save(out, res, allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def _rank_exchange_only(rank, world, port, out):
    """Raw exchange at world 3: slabs of unequal length (n not divisible by 3 or 4)."""
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1803_04631_b200.corpus import greedy_boundaries, make_chunk
    from paper_1803_04631_b200.shard import DeviceShard

    corp = synth_corpus = _corpus()
    K, V = 61, synth_corpus.vocab_size                   # odd K: packed u16 columns have a pad cell
    lo, hi = greedy_boundaries(corp.doc_lengths, world)[rank]
    a, b = int(corp.doc_ptr[lo]), int(corp.doc_ptr[hi])
    chunk = make_chunk(rank, lo, hi, corp.doc_ids[a:b], corp.word_ids[a:b], V, K, 7)
    freq = torch.as_tensor(np.bincount(chunk.word_ids, minlength=V).astype(np.int64))
    dist.all_reduce(freq)
    sh = DeviceShard(K, V, 50.0 / K, 0.01, seed=5, device=0, heavy_threshold=60, global_word_freq=freq.numpy())
    sh.load(chunk)
    sh.rebuild_phi()
    sh.synchronize()
    mine = sh.sync_tensor().cpu()
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    expect = torch.stack(parts).view(torch.int32).sum(0, dtype=torch.int64).to(torch.int32)
    handles = [None] * world
    dist.all_gather_object(handles, sh.peer_handle())
    sh.peer_open(rank, world, handles)
    sh.peer_allreduce()
    sh.synchronize()
    sh.check_errors()
    ok = bool(torch.equal(sh.sync_tensor().cpu(), expect))
    flags = [None] * world
    dist.all_gather_object(flags, (ok, int(mine.numel())))
    if rank == 0:
        np.save(out, np.array([f[0] for f in flags] + [flags[0][1]], dtype=np.int64))
    sh.peer_close()
    sh.close()
    dist.barrier()
    dist.destroy_process_group()


def test_peer_exchange_three_ranks():
    import torch.multiprocessing as mp

    out = os.path.join(tempfile.mkdtemp(), "peer3.npy")
    mp.spawn(_rank_exchange_only, args=(3, _free_port(), out), nprocs=3, join=True)
    r = np.load(out)
    assert r[-1] % 3 != 0 or r[-1] % 4 != 0        # the slabs really are uneven / unaligned
    assert r[:-1].tolist() == [1, 1, 1]


@pytest.fixture(scope="module")
def peer_result():
    import torch.multiprocessing as mp

    out = os.path.join(tempfile.mkdtemp(), "peer.npy")
    mp.spawn(_rank_main, args=(2, _free_port(), out), nprocs=2, join=True)
    return np.load(out, allow_pickle=True).item()


def test_peer_exchange_equals_replica_sum(peer_result):
    assert peer_result["n_words"] > 0
    assert peer_result["exchange_exact"]


def test_peer_exchange_repeated_epochs(peer_result):
    assert peer_result["epochs_exact"]


def test_fused_k2_exchange_equals_replica_sum(peer_result):
    """K2X (gf_shard_rebuild_phi_exchange): rebuilding the replica and summing it
    over the group in one stripe-pipelined kernel gives the all_reduce result,
    bit-exact, epoch after epoch."""
    assert peer_result["fused_exact"]


def test_trainer_peer_sync_conserves_counts(peer_result):
    assert all(c == "ok" for c in peer_result["conservation"]), peer_result["conservation"]


def test_trainer_peer_sync_tracks_one_rank(peer_result):
    from paper_1803_04631_b200 import engine

    tr = engine.Trainer(_corpus(), engine.TrainConfig(**CFG), device=0)
    ref = [tr.step().loglik_per_token for _ in range(4)]
    got = peer_result["lls"]
    # iteration 0 starts from a different z0 split (chunk-keyed draws), so
    # compare levels, not draws: the trajectories stay within 1%
    assert np.all(np.abs(np.array(got) - np.array(ref)) < 0.01 * np.abs(np.array(ref))), (got, ref)
