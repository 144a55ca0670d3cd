"""Host-side file formats of the reference API (paper_2201_02791_b200.io):
round trips and the format details a reference-written directory relies on."""
import os

import numpy as np
import pytest

import paper_2201_02791_b200 as kb
from paper_2201_02791_b200.errors import ParseError, ProvenanceError, ReferenceError_, ShapeError


def test_dataset_dir_round_trip_named(tmp_path):
    d = tmp_path / "ds"
    d.mkdir()
    (d / "train.txt").write_text("a\tr1\tb\nb\tr2\tc\n# comment\n\nc\tr1\ta\n")
    (d / "valid.txt").write_text("a r2 c\n")   # space separated is accepted
    (d / "test.txt").write_text("b\tr1\tnew\n")
    g, s = kb.load_dataset_dir(str(d))
    assert g.entity_names == ["a", "b", "c", "new"] and g.relation_names == ["r1", "r2"]
    np.testing.assert_array_equal(s.train, [[0, 0, 1], [1, 1, 2], [2, 0, 0]])
    np.testing.assert_array_equal(s.test, [[1, 0, 3]])
    out = tmp_path / "out"
    kb.write_dataset_dir(g, s, str(out))
    g2, s2 = kb.load_dataset_dir(str(out))     # now through the written dictionaries
    assert g2.entity_names == g.entity_names and g2.num_relations == 2
    for a, b in ((s.train, s2.train), (s.valid, s2.valid), (s.test, s2.test)):
        np.testing.assert_array_equal(a, b)


def test_integer_mode_and_errors(tmp_path):
    f = tmp_path / "t.txt"
    f.write_text("0\t1\t2\n3\t0\t1\n")
    g, s = kb.load_triples(str(f))
    assert (g.num_entities, g.num_relations) == (4, 2) and g.entity_names is None
    bad = tmp_path / "bad.txt"
    bad.write_text("0\t1\n")
    with pytest.raises(ParseError):
        kb.load_triples(str(bad))
    named = tmp_path / "n.txt"
    named.write_text("a\tr\tb\n")
    with pytest.raises(ReferenceError_):   # fixed dictionaries: unknown token
        kb.load_triples(str(named), entity_dict={"a": 0}, relation_dict={"r": 0})


def test_features(tmp_path):
    g = kb.KnowledgeGraph(3, 1, np.array([[0, 0, 1], [1, 0, 2]]))
    f = tmp_path / "f.txt"
    f.write_text("2 0.5 1\n0 1 2\n1 3 4\n")
    kb.load_features(str(f), g)
    np.testing.assert_array_equal(g.features, [[1, 2], [3, 4], [0.5, 1]])
    f.write_text("0 1\n1 2 3\n2 4\n")
    with pytest.raises(ShapeError):
        kb.load_features(str(f), g)


@pytest.mark.parametrize("fmt", ["tsv", "npy"])
def test_partition_directory_round_trip(tmp_path, fmt):
    graph, split = kb.generate_synthetic(400, 5, 6.0, seed=1)
    pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, 3, seed=0), graph, 2)
    d = tmp_path / "parts"
    kb.write_partitions(pset, str(d), fmt=fmt)
    assert os.path.isfile(d / "p0" / ("core_edges." + fmt))
    back = kb.read_partitions(str(d), graph)
    assert (back.num_parts, back.hops, back.method, back.seed) == (3, 2, pset.method, pset.seed)
    for a, b in zip(pset.partitions, back.partitions):
        np.testing.assert_array_equal(a.core, b.core)
        np.testing.assert_array_equal(a.support, b.support)
        np.testing.assert_array_equal(a.local_vertices(), b.local_vertices())
        np.testing.assert_array_equal(a.core_edge_ids, b.core_edge_ids)
        np.testing.assert_array_equal(a.support_edge_ids, b.support_edge_ids)
        for r in ("core_vertices", "replicated_vertices", "support_vertices"):
            np.testing.assert_array_equal(getattr(a, r), getattr(b, r))
    st = kb.partition_stats(back)
    assert st.core_edges == [p.num_core_edges for p in pset.partitions]
    assert abs(st.rf - kb.replication_factor(pset)) < 1e-12 and "RF =" in st.format()
    meta = (d / "meta").read_text().replace("hops=2", "hops=3")
    (d / "meta").write_text(meta)
    with pytest.raises(ProvenanceError):
        kb.read_partitions(str(d))


def test_candidates_and_results_files(tmp_path):
    c = tmp_path / "c.txt"
    c.write_text("0\t3,1,2\n# x\n1\t5\n")
    cand = kb.read_candidates(str(c))
    np.testing.assert_array_equal(cand[0], [3, 1, 2])
    np.testing.assert_array_equal(cand[1], [5])
    res = kb.EvalResult(mrr=0.5, hits={1: 0.25, 3: 0.5, 10: 1.0},
                        records=[kb.RankRecord(0, 1, 2, "tail", 2.0, 9), kb.RankRecord(0, 1, 2, "head", 1.5, 9)])
    out = tmp_path / "r.txt"
    kb.write_results(res, str(out))
    lines = out.read_text().splitlines()
    assert lines[0] == "0\t1\t2\ttail\t2.0" and lines[2] == "# mrr=0.500000" and lines[-1] == "# hits@10=1.000000"


def _loop_resolve(graph, triples, used):
    """The reference's per-triple resolution (ref:partition.py:398-417)."""
    idx = {}
    for eid, key in enumerate(map(tuple, graph.triples.tolist())):
        idx.setdefault(key, []).append(eid)
    out = []
    for key in map(tuple, triples.tolist()):
        ids, k = idx.get(key), used.get(key, 0)
        if not ids:
            raise ProvenanceError("not found")
        if k >= len(ids):
            raise ProvenanceError("occurs more often")
        out.append(ids[k])
        used[key] = k + 1
    return np.asarray(out, dtype=np.int64)


def test_edge_id_resolution_with_duplicates_matches_loop():
    from paper_2201_02791_b200.io import _EdgeIdResolver
    rng = np.random.default_rng(3)
    base = np.stack([rng.integers(0, 30, 200), rng.integers(0, 4, 200), rng.integers(0, 30, 200)], 1)
    tri = np.concatenate([base, base[rng.integers(0, 200, 150)], base[:20]])   # duplicates, some x3
    graph = kb.KnowledgeGraph(30, 4, tri)
    res, used = _EdgeIdResolver(graph), {}
    perm = rng.permutation(len(tri))
    for chunk in np.array_split(tri[perm], 4):          # batches share the use counts
        np.testing.assert_array_equal(res(chunk), _loop_resolve(graph, chunk, used))
    with pytest.raises(ProvenanceError, match="occurs more often"):
        res(tri[:1])                                    # every occurrence is used up
    with pytest.raises(ProvenanceError, match="not found"):
        _EdgeIdResolver(graph)(np.array([[0, 0, 0], [29, 3, 99]]))   # out-of-range tail
    fresh = _EdgeIdResolver(graph)
    missing = np.array([[a, b, c] for a in range(30) for b in range(4) for c in range(30)
                        if not ((tri == [a, b, c]).all(1)).any()][:1])
    with pytest.raises(ProvenanceError, match="not found"):
        fresh(np.concatenate([tri[:5], missing]))


def test_reference_reads_our_tsv_directory_and_we_read_theirs(tmp_path):
    """Interoperability with the reference's own reader/writer (this
    container only: /root/reference is absent on the GPU box)."""
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference package not available")
    import sys
    sys.path.insert(0, src)
    try:
        import kgdist as kg
    finally:
        sys.path.remove(src)
    graph, split = kb.generate_synthetic(300, 4, 5.0, seed=2)
    pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, 2, seed=0), graph, 2)
    kb.write_partitions(pset, str(tmp_path / "ours"))
    rgraph = kg.KnowledgeGraph(graph.num_entities, graph.num_relations, graph.triples)
    theirs = kg.read_partitions(str(tmp_path / "ours"), rgraph)
    kg.write_partitions(theirs, str(tmp_path / "theirs"))
    back = kb.read_partitions(str(tmp_path / "theirs"), graph)
    for a, b, c in zip(pset.partitions, theirs.partitions, back.partitions):
        np.testing.assert_array_equal(a.core_edge_ids, b.core_edge_ids)
        np.testing.assert_array_equal(b.core_edge_ids, c.core_edge_ids)
        np.testing.assert_array_equal(b.support_edge_ids, c.support_edge_ids)
        np.testing.assert_array_equal(a.local_vertices(), c.local_vertices())
