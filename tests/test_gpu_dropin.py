"""Drop-in surface of the package on the GPU (`-m gpu`), against the oracle:

* `ComputeGraph.layers` (LayerBlock, ref:sampler.py:239-307) — bit-exact
  edge lists, relation pointers, by_dst/by_src permutations and segments;
* the float64 compatibility entry points `allreduce_mean` and
  `Optimizer.step` (ref:trainer.py:63-151) — bitwise equal to the reference's
  numpy arithmetic (oracle tree_mean / OAdam), untouched rows untouched.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import kg_oracle as ko  # noqa: E402
import paper_2201_02791_b200 as kb  # noqa: E402


def _views(n=300, R=6, deg=5.0, parts=2, hops=2, seed=4):
    graph, _ = kb.generate_synthetic(n, R, deg, seed=seed)
    pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, parts, seed=0), graph, hops)
    out = []
    for p in pset.partitions:
        v = kb.build_view(p, graph.num_entities, graph.num_relations)
        ov = ko.make_view(p.core, p.support, graph.num_entities, graph.num_relations, pool_size=p.pool_size)
        out.append((v, ov))
    return out


def _segments(vals):
    if len(vals) == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    starts = np.flatnonzero(np.diff(vals, prepend=vals[0] - 1))
    return starts, vals[starts]


@pytest.mark.parametrize("hops", [0, 1, 2, 3])
def test_layers_match_oracle(hops):
    rng = np.random.default_rng(hops)
    for v, ov in _views(hops=max(hops, 1)):
        for size in (1, 5, 40):
            seeds = rng.choice(v.num_vertices, size=min(size, v.num_vertices), replace=False)
            cg = kb.compute_graph_for_seeds(seeds, v, hops)
            og = ko.closure(ov, seeds, hops)
            assert cg.num_layers == len(og.layers) == hops
            for blk, ob in zip(cg.layers, og.layers):
                assert blk.num_targets == ob.num_targets
                for f in ("dst", "src", "rel"):
                    got = getattr(blk, f)
                    assert got.dtype == np.int64
                    np.testing.assert_array_equal(got, getattr(ob, f))
                np.testing.assert_array_equal(blk.norm, ob.norm)        # exact 1/count in float64
                np.testing.assert_array_equal(blk.rel_indptr, ob.group_ptr)
                by_dst = np.argsort(ob.dst, kind="stable")
                by_src = np.argsort(ob.src, kind="stable")
                np.testing.assert_array_equal(blk.by_dst, by_dst)
                np.testing.assert_array_equal(blk.by_src, by_src)
                for (segs, uniq), (ws, wu) in (((blk.dst_segs, blk.dst_uniq), _segments(ob.dst[by_dst])),
                                               ((blk.src_segs, blk.src_uniq), _segments(ob.src[by_src]))):
                    np.testing.assert_array_equal(segs, ws)
                    np.testing.assert_array_equal(uniq, wu)
                # reference invariants (ref tests test_sampler.py:210-219)
                loops = blk.rel == v.self_loop_rel
                assert loops.sum() == blk.num_targets
                np.testing.assert_array_equal(np.sort(blk.dst[loops]), np.arange(blk.num_targets))
                assert blk.num_edges == len(blk.dst)


def _payloads(P, shapes, dtype, seed):
    rng = np.random.default_rng(seed)
    return [[rng.standard_normal(s).astype(dtype) for s in shapes] for _ in range(P)]


@pytest.mark.parametrize("P", [1, 2, 3, 5, 7, 8, 11])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_allreduce_mean_bitwise(P, dtype):
    shapes = [(2, 7, 5), (13, 2), (9,)]
    pl = _payloads(P, shapes, dtype, P)
    got = kb.allreduce_mean(pl)
    want = ko.tree_mean(pl)
    for a, b in zip(got, want):
        assert a.dtype == b.dtype and a.shape == b.shape
        np.testing.assert_array_equal(a, b)


def test_allreduce_mean_identity_and_errors():
    blocks = [np.random.default_rng(0).standard_normal((6, 3))]
    for P in (2, 4, 8):
        out = kb.allreduce_mean([blocks] * P)
        np.testing.assert_array_equal(out[0], blocks[0])      # bitwise (power-of-two P)
    with pytest.raises(kb.ProtocolError):
        kb.allreduce_mean([])
    with pytest.raises(kb.ProtocolError):
        kb.allreduce_mean([[np.zeros(3)], [np.zeros(4)]])


def _model(num_entities=30, dims=(4, 5, 3), R=3, seed=0):
    mc = kb.ModelConfig(len(dims) - 1, list(dims), 2, R, mode="embedding")
    return mc, kb.init_params(mc, np.random.default_rng(seed), num_entities=num_entities)


@pytest.mark.parametrize("opt,clip", [("adam", None), ("adam", 0.5), ("sgd", None), ("sgd", 0.3)])
def test_optimizer_step_bitwise(opt, clip):
    mc, p = _model()
    op = ko.OParams([b.copy() for b in p.bases], [c.copy() for c in p.coeffs], p.decoder.copy(),
                    p.entity_embed.copy())
    tc = kb.TrainConfig(optimizer=opt, learning_rate=0.05, grad_clip=clip)
    ours = kb.Optimizer(tc, p)
    ref = ko.OAdam(op, optimizer=opt, lr=0.05, grad_clip=clip)
    rng = np.random.default_rng(7)
    for step in range(4):
        grads = [rng.standard_normal(b.shape) for b in p.dense_blocks()]
        ids = rng.integers(0, 30, size=12)            # duplicates on purpose
        rows = rng.standard_normal((12, p.entity_embed.shape[1]))
        untouched = np.setdiff1d(np.arange(30), ids)
        before = p.entity_embed[untouched].copy()
        ours.step(p, [g.copy() for g in grads], ids, rows)
        ref.step(op, [g.copy() for g in grads], ids, rows)
        for a, b in zip(p.dense_blocks(), op.dense()):
            if clip is None:
                np.testing.assert_array_equal(a, b)
            else:   # the clip norm's summation order differs from numpy's pairwise sum
                np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-15)
        np.testing.assert_array_equal(p.entity_embed, op.embed)
        np.testing.assert_array_equal(p.entity_embed[untouched], before)


def test_optimizer_sgd_exact_and_adam_first_step():
    """ref tests test_trainer.py:75-96 restated: SGD lr 0.5, g = 1 moves by
    exactly 0.5; Adam's first step with g = 2, lr 0.1 moves by 0.1*2/(2+1e-8)."""
    mc, p = _model()
    start = [b.copy() for b in p.dense_blocks()]
    kb.Optimizer(kb.TrainConfig(optimizer="sgd", learning_rate=0.5), p).step(
        p, [np.ones_like(b) for b in p.dense_blocks()])
    for a, b in zip(p.dense_blocks(), start):
        np.testing.assert_array_equal(a, b - 0.5)
    mc, p = _model()
    start = [b.copy() for b in p.dense_blocks()]
    kb.Optimizer(kb.TrainConfig(optimizer="adam", learning_rate=0.1), p).step(
        p, [np.full_like(b, 2.0) for b in p.dense_blocks()])
    for a, b in zip(p.dense_blocks(), start):
        np.testing.assert_allclose(b - a, 0.1 * 2.0 / (2.0 + 1e-8), rtol=1e-12)


def test_optimizer_nonfinite_raises():
    mc, p = _model()
    g = [np.zeros_like(b) for b in p.dense_blocks()]
    g[0][0, 0, 0] = np.nan
    with pytest.raises(kb.NumericError):
        kb.Optimizer(kb.TrainConfig(optimizer="sgd"), p).step(p, g)
