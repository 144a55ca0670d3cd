"""Host-side drop-in surface (CPU): reference signatures of the trainer's
planning/assembly helpers, module-level names the reference exposes, graph
adjacency indices and statistics. Checked against the oracle restatement."""

import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest

import kg_oracle as ko
import paper_2201_02791_b200 as kb
from paper_2201_02791_b200 import trainer as tr


def test_plan_batches_reference_signature():
    mc = kb.ModelConfig(2, [4, 4, 4], 2, 3, negatives_per_positive=2, mode="embedding")
    for cores in ([7, 3, 5], [10], [1, 100]):
        views = [SimpleNamespace(num_core=c) for c in cores]
        for bs, fixed in ((None, None), (4, None), (None, 5), (1000, None)):
            got = tr._plan_batches(views, mc, kb.TrainConfig(batch_size=bs, fixed_num_batches=fixed))
            assert got == ko.plan(cores, 2, bs, fixed)
    with pytest.raises(kb.ValidationError):
        tr._plan_batches([SimpleNamespace(num_core=0)], mc, kb.TrainConfig())


def test_assemble_embed_list_and_dict_forms():
    graph, _ = kb.generate_synthetic(120, 4, 4.0, seed=2)
    pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, 3, seed=0), graph, 1)
    base = np.zeros((graph.num_entities, 2))
    tables = [np.full((graph.num_entities, 2), float(w + 1)) for w in range(3)]
    a = tr._assemble_embed(pset, tables, base)
    b = tr._assemble_embed(pset, dict(enumerate(tables)), base)
    np.testing.assert_array_equal(a, b)
    ends = [np.concatenate([p.core_vertices, p.replicated_vertices]) for p in pset.partitions]
    want = ko.owner_merge(ends, [p.id for p in pset.partitions], tables, base)
    np.testing.assert_array_equal(a, want)


@pytest.mark.parametrize("mod,names", [
    ("graph", ["load_dataset_dir", "load_features", "load_triples", "read_dictionary", "write_dataset_dir",
               "write_dictionary", "write_triples", "GraphStats", "graph_stats", "generate_synthetic"]),
    ("partition", ["PartitionStats", "partition_stats", "read_partitions", "write_partitions",
                   "neighborhood_expand", "replication_factor"]),
    ("sampler", ["LayerBlock", "ComputeGraph", "compute_graph_for_seeds"]),
    ("trainer", ["bench_components", "format_bench_rows", "optimizer_step", "_plan_batches", "_assemble_embed"]),
    ("evaluate", ["read_candidates", "write_results", "filtered_candidates", "rank_triplet"]),
])
def test_reference_module_names(mod, names):
    import importlib
    m = importlib.import_module(f"paper_2201_02791_b200.{mod}")
    for n in names:
        assert getattr(m, n) is not None, n
    with pytest.raises(AttributeError):
        getattr(m, "no_such_name_here")


def test_format_bench_rows():
    rows = [dict(partitioner="vertexcut", workers=2, rounds=3, epoch_time=0.25, cg_build=0.0, encode=0.0,
                 loss_step=0.01),
            dict(partitioner="random", workers=1, rounds=5, epoch_time=1.5, cg_build=0.0, encode=0.0,
                 loss_step=0.02)]
    lines = kb.trainer.format_bench_rows(rows).splitlines()
    assert len(lines) == 3 and "epoch_s" in lines[0]
    assert "vertexcut" in lines[1] and "random" in lines[2]
    assert len({len(x) for x in lines}) == 1          # fixed width


def test_graph_adjacency_and_stats():
    graph, _ = kb.generate_synthetic(60, 3, 3.0, seed=9)
    t = graph.triples
    for v in range(graph.num_entities):
        out_ids = np.flatnonzero(t[:, 0] == v)
        in_ids = np.flatnonzero(t[:, 2] == v)
        np.testing.assert_array_equal(graph.out_edge_ids(v), out_ids)
        np.testing.assert_array_equal(graph.in_edge_ids(v), in_ids)
        assert graph.out_index(v) == [(int(t[e, 1]), int(t[e, 2])) for e in out_ids]
        assert graph.in_index(v) == [(int(t[e, 1]), int(t[e, 0])) for e in in_ids]
    st = kb.graph_stats(graph)
    od = np.bincount(t[:, 0], minlength=60)
    idg = np.bincount(t[:, 2], minlength=60)
    assert (st.out_degree_min, st.out_degree_max, st.in_degree_min, st.in_degree_max) == \
        (od.min(), od.max(), idg.min(), idg.max())
    assert st.out_degree_mean == pytest.approx(od.mean()) and "out-degree" in st.format()
