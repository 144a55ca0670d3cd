"""The oracle's restatement of the reference's input producers
(oracle/kg_inputs.py, used by `bench.py --impl reference`) against the
golden fixtures made by the unmodified reference: FB15k-237-shaped graph
checksum, vertex-cut assignments and halo sizes at P = 1/2/4/8."""

import numpy as np
import pytest

import kg_inputs as ki
from conftest import load_golden


@pytest.fixture(scope="module")
def fb():
    return ki.synthetic_graph(14541, 237, 272115 / 14541, seed=0)


def test_generator_matches_golden(fb):
    g = load_golden("fb_structure")
    assert fb.checksum() == bytes(g["checksum"]).decode()
    assert len(fb.train) == int(g["num_train"]) and len(fb.valid) == int(g["num_valid"])


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_vertex_cut_and_halo_match_golden(fb, P):
    g = load_golden("fb_structure")
    parts = ki.partition_inputs(fb, P, seed=0, hops=2)
    assign = np.empty(len(fb.train), dtype=np.int8)
    for p in parts:
        assign[p.core_edge_ids] = p.pid
    np.testing.assert_array_equal(assign, g[f"assign_P{P}"])
    assert [len(p.support) for p in parts] == g[f"support_counts_P{P}"].tolist()
    assert [p.pool_size for p in parts] == g[f"pool_P{P}"].tolist()
