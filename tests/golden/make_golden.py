"""Generate the golden fixtures that pin `oracle/` (and through it the CUDA path)
to the reference package `gibbsflow` (/root/reference/pkg).

Test infrastructure only.  Runs in the dev container, never on the GPU box:
the reference tree does not travel.  The reference is imported from a
throw-away copy under /tmp with numba's cache redirected, so nothing is ever
written into /root/reference.

    python tests/golden/make_golden.py          # rewrites tests/golden/*.npz|json

What is captured (each block names the reference function it exercises):
  rng.npz        stream_key / Stream.uniforms / Stream.integer      rng.py:45-81
  bounds.json    greedy_boundaries on random + test-suite cases      corpus.py:210-237
  partition.npz  partition() + sort_word_groups_desc() outputs       corpus.py:240-302
  counts.npz     rebuild_theta / concat_theta / rebuild_phi_replica  model.py:109-161
  messages.json  CountOverflowError / ConservationReport texts       model.py:91-225
  ptree.npz      ptree.build levels + sample / sample_many indices   ptree.py:116-151
  ptree_api.npz  sample_with_stats, fp64 trees, fanouts > 32,
                 sample_total_and_draw in fp64                      ptree.py:54-151
"""

import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = "/root/reference/pkg/src"


def import_reference():
    tmp = tempfile.mkdtemp(prefix="gfref_")
    shutil.copytree(REF_PKG, os.path.join(tmp, "src"))
    os.environ["NUMBA_CACHE_DIR"] = os.path.join(tmp, "numba_cache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, os.path.join(tmp, "src"))
    import gibbsflow  # noqa: F401
    from gibbsflow import corpus, model, ptree, rng, errors

    return corpus, model, ptree, rng, errors


def small_corpus(cp, doc_lengths, vocab_size, seed):
    r = np.random.default_rng(seed)
    doc_ids = np.repeat(np.arange(len(doc_lengths)), doc_lengths)
    word_ids = r.integers(0, vocab_size, doc_ids.size)
    return cp.corpus_from_tokens(doc_ids, word_ids, vocab_size)


def zipf_corpus(cp, num_docs, vocab_size, mean_len, seed):
    """Zipf-skewed words, lognormal-ish lengths: heavy groups, long and short docs."""
    r = np.random.default_rng(seed)
    lengths = np.maximum(1, r.lognormal(np.log(mean_len), 0.6, num_docs).astype(np.int64))
    doc_ids = np.repeat(np.arange(num_docs), lengths)
    ranks = np.arange(1, vocab_size + 1, dtype=np.float64)
    p = ranks ** -1.07
    p /= p.sum()
    perm = r.permutation(vocab_size)
    word_ids = perm[r.choice(vocab_size, size=doc_ids.size, p=p)]
    return cp.corpus_from_tokens(doc_ids, word_ids, vocab_size)


def main():
    cp, md, pt, rng, errors = import_reference()
    out = {}

    # ---------------- rng (rng.py:45-81) ----------------
    key_parts = [(0,), (1,), (42,), (7, 3), (42, 3, 0), (1, 2), (2, 1), (0, 1, 2),
                 (20261017, 5), (2**64 - 1, 0), (123456789, 987654321, 5, 9)]
    keys = np.array([rng.stream_key(*p) for p in key_parts], dtype=np.uint64)
    uniforms = np.stack([rng.Stream(*p).uniforms(257) for p in key_parts])
    s = rng.Stream(5)
    integers = np.array([s.integer(7) for _ in range(300)], dtype=np.int64)
    np.savez_compressed(
        os.path.join(HERE, "rng.npz"),
        key_parts=json.dumps([list(p) for p in key_parts]),
        keys=keys, uniforms=uniforms, integers_seed5_n7=integers,
    )

    # ---------------- greedy_boundaries (corpus.py:210-237) ----------------
    r = np.random.default_rng(5)
    cases = [([5, 3, 2, 6], 2), ([10, 1, 1], 2), ([50, 50, 50, 1], 3), ([4, 1, 7], 1)]
    for _ in range(200):
        lengths = r.integers(1, 40, size=int(r.integers(1, 30))).tolist()
        cases.append((lengths, int(r.integers(1, len(lengths) + 1))))
    bounds = [
        {"lengths": L, "C": C, "bounds": [list(map(int, b)) for b in cp.greedy_boundaries(np.array(L), C)]}
        for L, C in cases
    ]
    with open(os.path.join(HERE, "bounds.json"), "w") as fh:
        json.dump(bounds, fh)

    # ---------------- partition + sort (corpus.py:240-302) ----------------
    part = {}
    pcases = [
        ("small", small_corpus(cp, [5, 3, 2, 6], 8, 0), 2, 4, 1),
        ("single", small_corpus(cp, [4, 1, 7], 8, 0), 1, 3, 1),
        ("rand25", small_corpus(cp, np.random.default_rng(11).integers(1, 30, 25).tolist(), 12, 0), 5, 6, 3),
        ("zipf", zipf_corpus(cp, 300, 500, 40, 7), 3, 32, 42),
        ("zipf_k1024", zipf_corpus(cp, 120, 2000, 150, 9), 2, 1024, 20261017),
    ]
    meta = []
    for name, corp, C, K, seed in pcases:
        chunks = cp.partition(corp, C, K, seed)
        meta.append({"name": name, "C": C, "K": K, "seed": seed, "V": corp.vocab_size,
                     "D": corp.num_docs, "T": corp.num_tokens})
        part[f"{name}__corpus_doc_ids"] = corp.doc_ids
        part[f"{name}__corpus_word_ids"] = corp.word_ids
        part[f"{name}__corpus_doc_lengths"] = corp.doc_lengths
        for ch in chunks:
            pre = f"{name}__c{ch.chunk_id}__"
            part[pre + "range"] = np.array([ch.doc_lo, ch.doc_hi, ch.token_count], dtype=np.int64)
            for f in ("doc_ids", "word_ids", "assignments", "group_words", "group_offsets",
                      "group_sizes", "dw_ptr", "dw_tok"):
                part[pre + f] = getattr(ch, f)
            srt = cp.sort_word_groups_desc(ch)
            part[pre + "desc_group_words"] = srt.group_words
            part[pre + "desc_group_offsets"] = srt.group_offsets
            part[pre + "desc_group_sizes"] = srt.group_sizes
            # count rebuilds on the partitioned chunk (model.py:109-161)
            th = md.rebuild_theta(ch, K)
            part[pre + "theta_row_ptr"] = th.row_ptr
            part[pre + "theta_topic_ids"] = th.topic_ids
            part[pre + "theta_counts"] = th.counts
            ph = md.rebuild_phi_replica(ch, K, corp.vocab_size)
            part[pre + "phi_counts"] = ph.counts
            part[pre + "phi_totals"] = ph.topic_totals
        full = md.concat_theta([md.rebuild_theta(ch, K) for ch in chunks])
        part[f"{name}__concat_row_ptr"] = full.row_ptr
        part[f"{name}__concat_topic_ids"] = full.topic_ids
        part[f"{name}__concat_counts"] = full.counts
    part["meta"] = json.dumps(meta)
    np.savez_compressed(os.path.join(HERE, "partition.npz"), **part)

    # ---------------- rebuilds on hand-built chunks (model.py:91-161) ----------------
    def build_chunk(doc_ids, word_ids, assignments):
        doc_ids = np.asarray(doc_ids, dtype=np.int32)
        word_ids = np.asarray(word_ids, dtype=np.int32)
        assignments = np.asarray(assignments, dtype=np.uint16)
        order = np.argsort(word_ids, kind="stable")
        doc_ids, word_ids, assignments = doc_ids[order], word_ids[order], assignments[order]
        words, starts, sizes = np.unique(word_ids, return_index=True, return_counts=True)
        doc_lo = int(doc_ids.min()) if doc_ids.size else 0
        doc_hi = int(doc_ids.max()) + 1 if doc_ids.size else 0
        dw_ptr, dw_tok = cp._doc_word_map(doc_ids, doc_lo, doc_hi - doc_lo)
        return cp.Chunk(0, doc_lo, doc_hi, len(doc_ids), doc_ids, word_ids, assignments.copy(),
                        words.astype(np.int32), starts.astype(np.int64), sizes.astype(np.int64),
                        dw_ptr, dw_tok)

    counts = {}
    r = np.random.default_rng(23)
    cmeta = []
    for i in range(40):
        n = int(r.integers(1, 400))
        K = int(r.integers(1, 70))
        V = int(r.integers(1, 40))
        D = int(r.integers(1, 12))
        ds, ws, zs = r.integers(0, D, n), r.integers(0, V, n), r.integers(0, K, n)
        ch = build_chunk(ds, ws, zs)
        th = md.rebuild_theta(ch, K)
        ph = md.rebuild_phi_replica(ch, K, V)
        pre = f"h{i}__"
        counts[pre + "doc"] = ds.astype(np.int32)
        counts[pre + "word"] = ws.astype(np.int32)
        counts[pre + "z"] = zs.astype(np.uint16)
        counts[pre + "theta_row_ptr"] = th.row_ptr
        counts[pre + "theta_topic_ids"] = th.topic_ids
        counts[pre + "theta_counts"] = th.counts
        counts[pre + "phi_counts"] = ph.counts
        counts[pre + "phi_totals"] = ph.topic_totals
        cmeta.append({"i": i, "K": K, "V": V, "doc_lo": ch.doc_lo, "doc_hi": ch.doc_hi})
    counts["meta"] = json.dumps(cmeta)
    np.savez_compressed(os.path.join(HERE, "counts.npz"), **counts)

    # ---------------- error / report texts ----------------
    msgs = {}
    n = 70000
    ch = build_chunk(np.zeros(n), np.zeros(n), np.zeros(n))
    try:
        md.rebuild_theta_row(ch, 0, 2)
    except errors.CountOverflowError as e:
        msgs["theta_overflow_doc0"] = str(e)
    ch = build_chunk(np.full(n, 3), np.zeros(n), np.zeros(n))  # doc 3 (doc_lo=3)
    try:
        md.rebuild_theta(ch, 2)
    except errors.CountOverflowError as e:
        msgs["theta_overflow_doc3"] = str(e)
    n = 66000
    ch = build_chunk(np.zeros(n), np.ones(n), np.ones(n, dtype=int))
    try:
        md.rebuild_phi_replica(ch, 2, 2, width=16)
    except errors.CountOverflowError as e:
        msgs["phi16_overflow_k1_v1"] = str(e)
    # two overflowing cells with different counts: argmax names the larger
    ds = np.zeros(140000)
    ws = np.concatenate([np.full(66000, 3), np.full(74000, 1)])
    zs = np.concatenate([np.full(66000, 0), np.full(74000, 2)])
    ch = build_chunk(ds, ws, zs)
    try:
        md.rebuild_phi_replica(ch, 3, 4, width=16)
    except errors.CountOverflowError as e:
        msgs["phi16_overflow_argmax"] = str(e)

    def make_model(doc_lengths, vocab_size, num_topics, seed):
        corp = small_corpus(cp, doc_lengths, vocab_size, seed)
        chunks = cp.partition(corp, min(3, corp.num_docs), num_topics, seed)
        theta = md.concat_theta([md.rebuild_theta(c, num_topics) for c in chunks])
        phi = md.zero_phi(num_topics, vocab_size)
        for c in chunks:
            rep = md.rebuild_phi_replica(c, num_topics, vocab_size)
            phi.counts += rep.counts
            phi.topic_totals += rep.topic_totals
        return corp, theta, phi

    corp, theta, phi = make_model([5, 8, 3, 9], 7, 3, 1)
    msgs["conservation_ok"] = md.check_conservation(theta, phi, corp).detail
    corp, theta, phi = make_model([5, 8, 3, 9], 7, 3, 2)
    phi.counts[1, 0] += 1
    phi.topic_totals[1] += 1
    msgs["conservation_phi_fault"] = md.check_conservation(theta, phi, corp).detail
    corp, theta, phi = make_model([5, 8, 3], 7, 3, 4)
    phi.counts[2, 1] += 1
    msgs["conservation_stale_totals"] = md.check_conservation(theta, phi, corp).detail
    corp, theta, phi = make_model([5, 8, 3], 7, 3, 5)
    theta.counts[theta.row_ptr[1]] += 1
    msgs["conservation_theta_row"] = md.check_conservation(theta, phi, corp).detail
    with open(os.path.join(HERE, "messages.json"), "w") as fh:
        json.dump(msgs, fh, indent=1)

    # ---------------- ptree (ptree.py:116-151) ----------------
    pz = {}
    r = np.random.default_rng(7)
    pmeta = []
    for i in range(24):
        nleaf = int(r.integers(1, 2050))
        fanout = [2, 4, 8, 32][i % 4]
        w = r.random(nleaf).astype(np.float32)
        w[r.random(nleaf) < 0.2] = 0.0
        if w.sum() == 0:
            w[0] = 1.0
        tree = pt.build(w, fanout=fanout)
        us = (r.random(64) * tree.total).astype(np.float32)
        us = np.minimum(us, np.nextafter(np.float32(tree.levels[-1][0]), np.float32(0)))
        pz[f"t{i}__w"] = w
        pz[f"t{i}__prefix"] = tree.levels[0]
        pz[f"t{i}__u"] = us
        pz[f"t{i}__idx"] = np.array([tree.sample(u) for u in us], dtype=np.int64)
        pz[f"t{i}__idx_many"] = tree.sample_many(us).astype(np.int64)
        pmeta.append({"i": i, "fanout": fanout, "height": tree.height, "n": nleaf})
        for lvl, arr in enumerate(tree.levels):
            pz[f"t{i}__level{lvl}"] = arr
    # sample_total_and_draw replay: indices drawn from Stream(2024) on a fixed tree
    w = np.array([0.0, 1.0, 0.0, 2.0, 0.5, 0.0, 3.0], dtype=np.float32)
    tree = pt.build(w, fanout=2)
    st = rng.Stream(2024)
    draws = [pt.sample_total_and_draw(tree, st) for _ in range(100)]
    pz["draw__w"] = w
    pz["draw__idx"] = np.array([d[0] for d in draws], dtype=np.int64)
    pz["draw__u"] = np.array([d[1] for d in draws], dtype=np.float64)
    pz["meta"] = json.dumps(pmeta)
    np.savez_compressed(os.path.join(HERE, "ptree.npz"), **pz)

    ptree_api(pt, rng)
    stores(cp, md)
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))


def ptree_api(pt=None, rng=None):
    """The rest of the PrefixTree surface (ptree.py:54-151): per-u descent
    stats, the fp64 oracle mode, fanouts wider than one warp ballot."""
    if pt is None:
        _, _, pt, rng, _ = import_reference()
    r = np.random.default_rng(19)
    pz, meta = {}, []
    cases = [(np.float32, 2), (np.float32, 8), (np.float32, 32), (np.float32, 64), (np.float32, 100),
             (np.float64, 2), (np.float64, 8), (np.float64, 32), (np.float64, 50)]
    for i, (dt, fanout) in enumerate(cases):
        nleaf = int(r.integers(1, 5000))
        w = r.random(nleaf)
        w[r.random(nleaf) < 0.25] = 0.0
        if w.sum() == 0:
            w[0] = 1.0
        tree = pt.build(w, fanout=fanout, dtype=dt)
        top = tree.levels[-1][0]
        us = np.minimum((r.random(80) * tree.total).astype(dt), np.nextafter(top, dt(0)))
        stats = [tree.sample_with_stats(u) for u in us]
        pz[f"a{i}__w"] = w
        pz[f"a{i}__u"] = us
        pz[f"a{i}__idx"] = np.array([x[0] for x in stats], np.int64)
        pz[f"a{i}__visited"] = np.array([x[1] for x in stats], np.int32)
        pz[f"a{i}__widest"] = np.array([x[2] for x in stats], np.int32)
        pz[f"a{i}__prefix_before"] = np.array([tree.prefix_before(j) for j in range(0, nleaf, 97)], dt)
        for lvl in range(len(tree.levels)):
            pz[f"a{i}__sums{lvl}"] = tree.level_sums(lvl)
        meta.append({"i": i, "dtype": np.dtype(dt).name, "fanout": fanout, "height": tree.height, "n": nleaf})
    w = r.random(300)
    tree = pt.build(w, fanout=4, dtype=np.float64)
    st = rng.Stream(77, 3)
    draws = [pt.sample_total_and_draw(tree, st) for _ in range(200)]
    pz["draw64__w"] = w
    pz["draw64__idx"] = np.array([d[0] for d in draws], np.int64)
    pz["draw64__u"] = np.array([d[1] for d in draws], np.float64)
    pz["meta"] = json.dumps(meta)
    np.savez_compressed(os.path.join(HERE, "ptree_api.npz"), **pz)


def stores(cp=None, md=None):
    """GFCHUNK1 / GFSNAP1 files written by the reference's own save_chunk /
    save_snapshot (corpus.py:305-327, model.py:228-255) for byte-level parity."""
    if cp is None:
        cp, md, _, _, _ = import_reference()
    corp = zipf_corpus(cp, 40, 60, 30.0, 11)
    (ch,) = cp.partition(corp, 1, 9, 3)
    ch = cp.sort_word_groups_desc(ch)
    cp.save_chunk(ch, os.path.join(HERE, "store_chunk.gfc"))
    theta = md.rebuild_theta(ch, 9)
    phi = md.rebuild_phi_replica(ch, 9, 60, width=16)
    md.save_snapshot(theta, phi, os.path.join(HERE, "store_snapshot.gfsnap"), metadata={"iteration": 3, "note": "ref"})
    np.savez_compressed(os.path.join(HERE, "store_inputs.npz"), doc_ids=corp.doc_ids, word_ids=corp.word_ids,
                        meta=json.dumps({"V": 60, "K": 9, "seed": 3}))
    # UCI bag of words (corpus.py:94-157): unsorted triples, empty documents,
    # blank lines, padding spaces -- loaded by the reference itself
    r = np.random.default_rng(5)
    D, W = 40, 25
    trip = {(int(d), int(w)): int(c) for d, w, c in zip(r.integers(1, D + 1, 300), r.integers(1, W + 1, 300),
                                                          r.integers(1, 6, 300)) if d % 7}
    items = list(trip.items())
    r.shuffle(items)
    lines = [str(D), " %d " % W, str(len(items))]
    for i, ((d, w), c) in enumerate(items):
        lines.append(f"{d}  {w} {c}" if i % 5 else f" {d} {w}\t{c} ")
        if i % 17 == 0:
            lines.append("   ")
    with open(os.path.join(HERE, "uci_docword.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    with open(os.path.join(HERE, "uci_vocab.txt"), "w") as fh:
        fh.write("\n".join(f"w{i}" for i in range(W)) + "\n\n")
    c = cp.load_uci_bow(os.path.join(HERE, "uci_docword.txt"), os.path.join(HERE, "uci_vocab.txt"))
    np.savez_compressed(os.path.join(HERE, "uci_expected.npz"), doc_ids=c.doc_ids, word_ids=c.word_ids,
                        doc_lengths=c.doc_lengths, doc_ptr=c.doc_ptr, vocab=np.array(c.vocab),
                        meta=json.dumps({"num_docs": c.num_docs, "vocab_size": c.vocab_size,
                                         "num_tokens": c.num_tokens}))


if __name__ == "__main__":
    if sys.argv[1:] == ["--stores-only"]:
        stores()
    elif sys.argv[1:] == ["--ptree-api-only"]:
        ptree_api()
    else:
        main()
