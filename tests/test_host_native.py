"""CPU tests of the product's native host side (no GPU needed): the C ABI
loads and exports every declared symbol; host preprocessing is bit-exact with
the reference golden vectors; the product path refuses to run without a GPU."""

import json
import os
import re

import numpy as np
import pytest

from paper_1803_04631_b200 import _lib, corpus, errors, rng, shard, synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_abi_exports_every_header_symbol():
    with open(_lib.HEADER) as fh:
        text = fh.read()
    declared = set(re.findall(r"^\s*(?:int|uint64_t|const char\*)\s+(gf_\w+)\s*\(", text, re.M))
    assert len(declared) >= 30
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    assert L.gf_abi_version() == 1


def test_no_device_fails_loudly():
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(errors.NoDeviceError):
        shard.DeviceShard(8, 10, 0.1, 0.01)


def test_stream_matches_reference():
    g = np.load(os.path.join(GOLD, "rng.npz"))
    parts = json.loads(str(g["key_parts"]))
    for i, p in enumerate(parts):
        assert rng.stream_key(*p) == g["keys"][i]
        np.testing.assert_array_equal(rng.Stream(*p).uniforms(257), g["uniforms"][i])
    s = rng.Stream(5)
    np.testing.assert_array_equal([s.integer(7) for _ in range(300)], g["integers_seed5_n7"])


def test_greedy_boundaries_match_reference():
    with open(os.path.join(GOLD, "bounds.json")) as fh:
        for c in json.load(fh):
            assert [list(b) for b in corpus.greedy_boundaries(c["lengths"], c["C"])] == c["bounds"]
    with pytest.raises(errors.PartitionError):
        corpus.greedy_boundaries([3, 3], 3)


@pytest.mark.parametrize("name", ["small", "single", "rand25", "zipf", "zipf_k1024"])
def test_partition_matches_reference(name):
    g = np.load(os.path.join(GOLD, "partition.npz"))
    m = next(x for x in json.loads(str(g["meta"])) if x["name"] == name)
    corp = corpus.corpus_from_tokens(g[f"{name}__corpus_doc_ids"], g[f"{name}__corpus_word_ids"], m["V"])
    chunks = corpus.partition(corp, m["C"], m["K"], m["seed"])
    for ch in chunks:
        pre = f"{name}__c{ch.chunk_id}__"
        assert [ch.doc_lo, ch.doc_hi, ch.token_count] == g[pre + "range"].tolist()
        for f in ("doc_ids", "word_ids", "assignments", "group_words", "group_offsets", "group_sizes",
                  "dw_ptr", "dw_tok"):
            np.testing.assert_array_equal(getattr(ch, f), g[pre + f], err_msg=f)
            assert getattr(ch, f).dtype == g[pre + f].dtype
        srt = corpus.sort_word_groups_desc(ch)
        np.testing.assert_array_equal(srt.group_words, g[pre + "desc_group_words"])


def test_partition_guards():
    c = corpus.corpus_from_tokens([0, 0, 1], [0, 1, 1], 2)
    with pytest.raises(errors.PartitionError):
        corpus.partition(c, 3, 2, 0)
    with pytest.raises(ValueError):
        corpus.partition(c, 1, 70000, 0)
    with pytest.raises(errors.CorpusFormatError):
        corpus.corpus_from_tokens([0], [5], 2)


def test_sync_layout_hybrid_columns():
    col, (o16, onk, tot) = shard.sync_layout([70000, 3, 0, 65535, 65536], 5)
    assert col.tolist() == [~0, 0, 1, 2, ~1]
    assert (o16, onk, tot) == (2 * 5, 2 * 5 + 3 * 3, 2 * 5 + 3 * 3 + 5)
    col, lay = shard.sync_layout([1, 2, 3], 4, heavy_threshold=0)
    assert (col < 0).all() and lay == (12, 12, 16)


def test_synth_is_deterministic_and_shardable():
    a = synth.generate(200, 300, 40.0, seed=7)
    b = synth.generate(200, 300, 40.0, seed=7)
    np.testing.assert_array_equal(a.word_ids, b.word_ids)
    part = synth.generate(50, 300, 40.0, seed=7, doc_begin=100)
    np.testing.assert_array_equal(part.doc_lengths, a.doc_lengths[100:150])
    np.testing.assert_array_equal(part.word_ids, a.word_ids[a.doc_ptr[100]:a.doc_ptr[150]])
    assert abs(a.doc_lengths.mean() - 40.0) < 6.0
    # Zipf skew: the heaviest word carries a few percent of the tokens
    top = np.bincount(a.word_ids, minlength=300).max() / a.num_tokens
    assert 0.01 < top < 0.5
