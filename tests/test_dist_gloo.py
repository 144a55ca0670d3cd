"""N>1 host-side logic on CPU with a world_size-2 gloo process group:
partition ownership, payload all-gather into partition order, the
reference's pairwise-tree mean (ref:trainer.py:63-86) on the gathered
payloads, and the ownership-based embedding assembly (ref:trainer.py:319-333)."""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, P, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2201_02791_b200.trainer import gather_partition_payloads
    import kg_oracle as ko
    D = 11
    rng = np.random.default_rng(0)
    payloads = rng.normal(size=(P, D)).astype(np.float32)          # payload of partition p
    mine = [p for p in range(P) if p % world == rank]                # Trainer.local_wids
    local = torch.as_tensor(payloads[mine])
    out = torch.empty((P, D), dtype=torch.float32)
    gather_partition_payloads(local, P, world, out)
    ok_order = bool(np.array_equal(out.numpy(), payloads))
    tree = ko.tree_mean([[p.astype(np.float64)] for p in out.numpy()])[0]
    q.put((rank, ok_order, tree.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("P", [2, 4, 6])
def test_gather_order_and_tree_mean_world2(P):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + P
    procs = [ctx.Process(target=_worker, args=(r, world, port, P, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(ok for _, ok, _ in res)
    # every rank computes the identical reduction (bitwise-identical replicas)
    assert res[0][2] == res[1][2]


def test_assemble_embed_ownership():
    sys.path.insert(0, ROOT)
    from paper_2201_02791_b200.graph import generate_synthetic
    from paper_2201_02791_b200.partition import neighborhood_expand, vertex_cut_partition
    from paper_2201_02791_b200.trainer import _assemble_embed
    graph, _ = generate_synthetic(200, 4, 4.0, seed=1)
    pset = neighborhood_expand(vertex_cut_partition(graph, 3, seed=0), graph, 2)
    base = np.zeros((graph.num_entities, 2))
    tables = {w: np.full((graph.num_entities, 2), float(w + 1)) for w in range(3)}
    out = _assemble_embed(pset, tables, base)
    owner = np.full(graph.num_entities, -1)
    for p in pset.partitions:
        ends = np.concatenate([p.core_vertices, p.replicated_vertices])
        free = ends[owner[ends] < 0]
        owner[free] = p.id
    for v in range(graph.num_entities):
        assert out[v, 0] == (owner[v] + 1 if owner[v] >= 0 else 0)
