"""Runtime behaviour of the training entry points on the GPU (`-m gpu`):

* `kg_preload_kernels` loads the library's kernels up front;
* `kg_epoch_end` (the trainer's epoch-end bookkeeping) against a float64
  numpy restatement: per-worker mean round loss, status words returned and
  cleared;
* successive `train()` calls are bitwise identical (process-wide streams and
  persistent graph pools are reused, not shared between live graphs) and
  add no device memory after the first call;
* the float64 public API sums in a fixed order: the same loss evaluated
  twice is bitwise equal (what central-difference gradient checks need,
  ref tests/test_model.py gradcheck).
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2201_02791_b200 as kb  # noqa: E402
from paper_2201_02791_b200 import _lib  # noqa: E402


def test_preload_kernels_loads_the_library():
    lib = _lib.require_cuda()
    n = ctypes.c_int32(0)
    _lib.check(lib.kg_preload_kernels(ctypes.byref(n)), "kg_preload_kernels")
    assert n.value >= 100      # every module's functions (250 at the time of writing)


@pytest.mark.parametrize("nloc,rounds,ld", [(1, 9, 9), (2, 5, 7), (3, 1, 1), (1, 300, 301)])
def test_epoch_end_means_and_flags(nloc, rounds, ld):
    g = torch.Generator(device="cuda").manual_seed(nloc * 100 + rounds)
    losses = torch.rand((nloc, ld), device="cuda", generator=g, dtype=torch.float32)
    flags = [torch.tensor([v], dtype=torch.int32, device="cuda") for v in (0, 4, 1 | 16, 0)[: nloc + 1]]
    while len(flags) < nloc + 1:
        flags.append(torch.tensor([2], dtype=torch.int32, device="cuda"))
    ptrs = torch.tensor([f.data_ptr() for f in flags], dtype=torch.int64, device="cuda")
    out = torch.empty(nloc + len(flags), dtype=torch.float64, device="cuda")
    want_flags = [int(f.item()) for f in flags]
    _lib.call("kg_epoch_end", losses.data_ptr(), ld, nloc, rounds, ptrs.data_ptr(), len(flags), out.data_ptr(),
              _lib.stream_handle())
    got = out.cpu().numpy()
    want = losses[:, :rounds].double().cpu().numpy().mean(axis=1)
    np.testing.assert_allclose(got[:nloc], want, rtol=1e-14, atol=0)
    assert [int(x) for x in got[nloc:]] == want_flags
    assert all(int(f.item()) == 0 for f in flags)   # cleared


def _small_job():
    graph, _ = kb.generate_synthetic(400, 5, 6.0, seed=3)
    pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, 2, seed=0), graph, 2)
    mc = kb.ModelConfig(2, [16, 16, 16], 2, graph.num_relations, 1, mode="embedding")
    return graph, pset, mc


def test_train_calls_repeat_bitwise_without_memory_growth():
    graph, pset, mc = _small_job()
    tc = kb.TrainConfig(epochs=40, batch_size=256, optimizer="adam", learning_rate=0.01, seed=0)
    p1, r1 = kb.train(pset, graph, mc, tc)          # may grow the caches (first call of this shape)
    torch.cuda.synchronize()
    reserved = torch.cuda.memory_reserved()
    p2, r2 = kb.train(pset, graph, mc, tc)
    p3, r3 = kb.train(pset, graph, mc, tc)
    torch.cuda.synchronize()
    for a, b in ((p1, p2), (p2, p3)):
        for x, y in zip(a.dense_blocks() + [a.entity_embed], b.dense_blocks() + [b.entity_embed]):
            assert np.array_equal(x, y)
    assert r1.loss_curve == r2.loss_curve == r3.loss_curve
    assert torch.cuda.memory_reserved() == reserved   # later calls reuse the pools and the cache


def test_float64_loss_is_deterministic():
    graph, pset, mc = _small_job()
    params = kb.init_params(mc, np.random.default_rng(0), num_entities=graph.num_entities)
    view = kb.full_graph_view(graph)
    rng = np.random.default_rng(1)
    neg = kb.sample_negatives(view, 1, rng)
    batch = kb.make_batches(view.core_edges[:64], neg[:64], 128, rng)[0]
    cg = kb.build_compute_graph(batch, view, mc.num_layers)
    ids = np.arange(graph.num_entities)
    runs = [kb.loss_and_grad(params, mc, batch, cg, params.entity_embed, ids) for _ in range(3)]
    assert runs[0][0] == runs[1][0] == runs[2][0]


@pytest.mark.parametrize("n,dims,seed", [(14541, [100, 100, 100], 0), (1000, [32, 16], 7), (5, [3, 4, 2], 3)])
def test_device_drawn_initial_table_is_numpys(n, dims, seed):
    from paper_2201_02791_b200.trainer import _init_params_device
    mc = kb.ModelConfig(len(dims) - 1, dims, 2, 11, 1, mode="embedding")
    want = kb.init_params(mc, np.random.default_rng(seed), num_entities=n)
    got, table, (host, ev) = _init_params_device(mc, seed, n, torch.device("cuda"))
    ev.synchronize()
    assert np.array_equal(got.entity_embed, want.entity_embed)
    assert np.array_equal(table.cpu().numpy(), want.entity_embed)
    for a, b in zip(got.dense_blocks(), want.dense_blocks()):
        assert np.array_equal(a, b)


def test_feature_mode_training_matches_oracle():
    """Feature mode (input rows from graph.features, no embedding table,
    ref:trainer.py:186-236 with features) through train() at P = 2 vs the
    oracle restatement on the same fp32-representable start."""
    import kg_oracle as ko
    graph, _ = kb.generate_synthetic(300, 4, 5.0, seed=11)
    feats = np.random.default_rng(3).normal(size=(graph.num_entities, 12)).astype(np.float32).astype(np.float64)
    graph = kb.KnowledgeGraph(graph.num_entities, graph.num_relations, graph.triples, features=feats)
    pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, 2, seed=0), graph, 2)
    mc = kb.ModelConfig(2, [12, 16, 8], 2, graph.num_relations, 1, mode="feature")
    p0 = kb.init_params(mc, np.random.default_rng(5))
    q = lambda a: a.astype(np.float32).astype(np.float64)
    p0 = kb.ModelParams([q(b) for b in p0.bases], [q(c) for c in p0.coeffs], q(p0.decoder), None)
    tc = kb.TrainConfig(epochs=3, batch_size=128, optimizer="adam", learning_rate=0.01, seed=0)
    got, rep = kb.train(pset, graph, mc, tc, initial_params=p0)
    views, ends = [], []
    for part in pset.partitions:
        views.append(ko.make_view(part.core, part.support, graph.num_entities, graph.num_relations,
                                  partition_id=part.id, pool_size=part.pool_size))
        ends.append(np.concatenate([part.core_vertices, part.replicated_vertices]))
    op = ko.OParams([b.copy() for b in p0.bases], [c.copy() for c in p0.coeffs], p0.decoder.copy(), None)
    want, curve, rounds, sizes = ko.train(views, ends, op, 1, 3, batch_size=128, seed=0, features=feats)
    assert rep.rounds_per_epoch == rounds and rep.batch_sizes == sizes
    np.testing.assert_allclose(rep.loss_curve, curve, rtol=1e-5)
    for a, b in zip(got.dense_blocks(), want.dense()):
        assert np.linalg.norm(a - b) <= 1e-4 * max(np.linalg.norm(b), 1e-30)
    assert got.entity_embed is None
