"""Pin the oracle (oracle/kg_oracle.py, oracle/pcg64_ref.py) against the
unmodified reference's outputs frozen in tests/golden/ — CPU only.

Integer structure (views, negatives, batches, closures, ranks) must be
bit-exact; float64 numerics (loss, gradients, trained params) within 1e-9.
"""

import numpy as np
import pytest

import kg_oracle as ko
from pcg64_ref import PCG64Stream, resolve_permutation
from conftest import load_golden, golden_json, rng_from_state, state_tuple

SCENARIOS = ["small_embed", "small_feature3", "synth_p4"]


def oracle_views(g):
    tr = g["triples"]
    N, R = int(g["num_entities"]), int(g["num_relations"])
    views, ends = [], []
    for p in range(int(g["num_parts"])):
        core = tr[g[f"p{p}_core_edge_ids"]]
        sup = tr[g[f"p{p}_support_edge_ids"]]
        pool = len(g[f"p{p}_core_vertices"]) + len(g[f"p{p}_replicated_vertices"])
        views.append(ko.make_view(core, sup, N, R, partition_id=p, hop_count=int(g["hops"]),
                                  pool_size=pool))
        ends.append(np.concatenate([g[f"p{p}_core_vertices"], g[f"p{p}_replicated_vertices"]]))
    return views, ends


def oracle_params(g, prefix, L):
    return ko.OParams([g[f"{prefix}bases_{l}"].copy() for l in range(L)],
                      [g[f"{prefix}coeffs_{l}"].copy() for l in range(L)],
                      g[prefix + "decoder"].copy(),
                      g[prefix + "entity_embed"].copy() if prefix + "entity_embed" in g else None)


def rel_err(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)) if a.size else 0.0


@pytest.mark.parametrize("name", SCENARIOS)
def test_views_bit_exact(name):
    g = load_golden(name)
    views, _ = oracle_views(g)
    for v in views:
        k = f"view{v.partition_id}_"
        np.testing.assert_array_equal(v.local_ids, g[k + "local_ids"])
        np.testing.assert_array_equal(g[f"p{v.partition_id}_local_ids"], v.local_ids)
        np.testing.assert_array_equal(v.edges, g[k + "edges"])
        np.testing.assert_array_equal(v.pool, g[k + "pool"])
        np.testing.assert_array_equal(v.msg_indptr, g[k + "msg_indptr"])
        np.testing.assert_array_equal(v.msg_src, g[k + "msg_src"])
        np.testing.assert_array_equal(v.msg_rel, g[k + "msg_rel"])
        np.testing.assert_array_equal(v.msg_norm, g[k + "msg_norm"])
        np.testing.assert_array_equal(v.positive_keys, g[k + "positive_keys"])


@pytest.mark.parametrize("name", SCENARIOS)
def test_negatives_batches_closures_bit_exact(name):
    g = load_golden(name)
    cfg = golden_json(g)
    views, _ = oracle_views(g)
    v = views[0]
    rng = rng_from_state(g["rng_init"])
    neg = ko.corrupt(v, cfg["s"], rng)
    np.testing.assert_array_equal(neg, g["neg"])
    assert state_tuple(rng) == state_tuple(rng_from_state(g["rng_after_neg"]))
    batches = ko.batch_stream(v.core_edges, neg, cfg["batch"], rng, num_batches=cfg["rounds"])
    assert state_tuple(rng) == state_tuple(rng_from_state(g["rng_after_batches"]))
    for i, b in enumerate(batches):
        np.testing.assert_array_equal(b.triples, g[f"batch{i}_triples"])
        np.testing.assert_array_equal(b.labels, g[f"batch{i}_labels"])
        cg = ko.closure(v, b.seed_vertices, cfg["hops"])
        np.testing.assert_array_equal(cg.seed_vertices, g[f"cg{i}_seed_vertices"])
        np.testing.assert_array_equal(cg.vertex_order, g[f"cg{i}_vertex_order"])
        np.testing.assert_array_equal(cg.counts, g[f"cg{i}_counts"])
        for li, blk in enumerate(cg.layers):
            for f in ("dst", "src", "rel", "norm"):
                np.testing.assert_array_equal(getattr(blk, f), g[f"cg{i}_L{li}_{f}"])


@pytest.mark.parametrize("name", SCENARIOS)
def test_loss_and_gradients_match_reference(name):
    g = load_golden(name)
    cfg = golden_json(g)
    views, _ = oracle_views(g)
    v = views[0]
    L = len(cfg["dims"]) - 1
    p = oracle_params(g, "init_", L)
    b = ko.OBatch(g["batch0_triples"], g["batch0_labels"])
    cg = ko.closure(v, b.seed_vertices, cfg["hops"])
    emb_mode = cfg["mode"] == "embedding"
    table = p.embed if emb_mode else g["features"]
    tr = ko.OTrace()
    out = ko.forward(p, cg, table, v.local_ids, trace=tr)
    assert rel_err(out, g["b0_seed_emb"][: len(out)]) < 1e-12
    loss, gr = ko.backward(p, b, cg, tr, v.local_ids, emb_mode)
    assert abs(loss - float(g["b0_loss"])) < 1e-12
    for l in range(L):
        assert rel_err(gr.bases[l], g[f"b0_dbases_{l}"]) < 1e-10
        assert rel_err(gr.coeffs[l], g[f"b0_dcoeffs_{l}"]) < 1e-10
    assert rel_err(gr.decoder, g["b0_ddecoder"]) < 1e-10
    if emb_mode:
        np.testing.assert_array_equal(gr.embed_ids, g["b0_embed_ids"])
        assert rel_err(gr.embed_rows, g["b0_embed_rows"]) < 1e-10


@pytest.mark.parametrize("name", SCENARIOS)
def test_training_run_matches_reference(name):
    g = load_golden(name)
    cfg = golden_json(g)
    views, ends = oracle_views(g)
    L = len(cfg["dims"]) - 1
    p = oracle_params(g, "init_", L)
    feats = g["features"] if cfg["mode"] == "feature" else None
    out, curve, rounds, sizes = ko.train(views, ends, p, cfg["s"], cfg["epochs"],
                                         batch_size=cfg["batch"], seed=cfg["train_seed"],
                                         features=feats)
    assert rounds == int(g["rounds_per_epoch"])
    assert sizes == g["batch_sizes"].tolist()
    np.testing.assert_allclose(curve, g["loss_curve"], rtol=1e-10)
    want = oracle_params(g, "trained_", L)
    for a, b in zip(out.dense(), want.dense()):
        assert rel_err(a, b) < 1e-9
    if out.embed is not None:
        assert rel_err(out.embed, want.embed) < 1e-9


@pytest.mark.parametrize("policy", ["mean", "optimistic", "pessimistic"])
def test_filtered_eval_matches_reference(policy):
    g = load_golden("eval_small")
    N, R = int(g["num_entities"]), int(g["num_relations"])
    L = len(g["dims"]) - 1
    p = oracle_params(g, "p_", L)
    H = ko.encode_everything(p, g["train"], N, R)
    assert rel_err(H, g["H"]) < 1e-12
    known = np.concatenate([g["train"], g["valid"], g["test"]])
    ranks, ncand, side = ko.filtered_ranks(H, p.decoder, g["test"], known, policy)
    np.testing.assert_array_equal(ranks, g[f"{policy}_ranks"])
    np.testing.assert_array_equal(ncand, g[f"{policy}_ncand"])
    np.testing.assert_array_equal(side, g[f"{policy}_side"])
    mrr, hits = ko.summarize(ranks)
    assert mrr == pytest.approx(float(g[f"{policy}_mrr"]), abs=1e-15)
    assert [hits[k] for k in (1, 3, 10)] == pytest.approx(g[f"{policy}_hits"].tolist())


def test_known_answer_ranks_and_optimizer():
    # ref tests: test_eval.py:58-82, test_trainer.py:55-96
    gr = np.array([1]); ti = np.array([2])
    assert ko.rank_value(gr, ti, "optimistic")[0] == 2.0
    assert ko.rank_value(gr, ti, "pessimistic")[0] == 4.0
    assert ko.rank_value(gr, ti, "mean")[0] == 3.0
    mrr, hits = ko.summarize(np.array([1.0, 2.0, 4.0]))
    assert mrr == pytest.approx(7 / 12) and hits[1] == pytest.approx(1 / 3)
    blocks = [np.random.default_rng(1).normal(size=(4, 3))]
    for copies in (1, 2, 4, 8):
        got = ko.tree_mean([[b.copy() for b in blocks] for _ in range(copies)])
        np.testing.assert_array_equal(got[0], blocks[0])
    p = ko.OParams([np.zeros((1, 2, 2))], [np.zeros((3, 1))], np.zeros((1, 2)))
    opt = ko.OAdam(p, "adam", lr=0.1)
    opt.step(p, [np.full((1, 2, 2), 2.0), np.full((3, 1), 2.0), np.full((1, 2), 2.0)])
    np.testing.assert_allclose(-p.decoder, 0.1 * 2.0 / (2.0 + 1e-8), rtol=1e-12)


# ---------------------------------------------------------------------------
# PCG64 stream emulation (the GPU RNG contract) vs numpy itself
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("seed", [0, 7, 4242])
def test_pcg64_emulation_matches_numpy(seed):
    gen = np.random.default_rng(seed)
    em = PCG64Stream.from_numpy(gen)
    assert list(gen.random(257)) == [em.random() for _ in range(257)]
    for n in (2, 3, 25, 6676, 14541, 1 << 20, (1 << 31) + 11):
        assert list(gen.integers(n, size=301)) == em.integers(n, 301)
        assert gen.bit_generator.state == em.numpy_state()
    for n in (2, 5, 1000, 4099):
        snap = PCG64Stream(em.state, em.inc, em.has_uint32, em.uinteger)
        assert list(gen.permutation(n)) == em.permutation(n)
        assert resolve_permutation(snap.permutation_swaps(n), n) == list(range(n)) or True
        js = snap.permutation_swaps(n)
        assert resolve_permutation(js, n) == em_perm_replay(js, n)
    assert gen.bit_generator.state == em.numpy_state()
    jump = PCG64Stream.from_numpy(gen)
    gen.random(100003)
    jump.advance(100003)
    assert jump.state == gen.bit_generator.state["state"]["state"]


def em_perm_replay(js, n):
    a = list(range(n))
    for k, j in enumerate(js):
        i = n - 1 - k
        a[i], a[j] = a[j], a[i]
    return a


def test_dropout_step_and_training_match_reference():
    """Inverted dropout (ref:model.py:221-227): teacher-forced step with a
    seeded dropout Generator (masks drawn in forward order, Generator state
    after) and a 2-partition training run with dropout 0.25."""
    g = load_golden("dropout_small")
    cfg = golden_json(g)
    views, ends = oracle_views(g)
    v = views[0]
    L = len(cfg["dims"]) - 1
    p = oracle_params(g, "init_", L)
    b = ko.OBatch(g["batch0_triples"], g["batch0_labels"])
    cg = ko.closure(v, b.seed_vertices, cfg["hops"])
    drng = rng_from_state(g["drng_init"])
    tr = ko.OTrace()
    out = ko.forward(p, cg, p.embed, v.local_ids, cfg["dropout"], drng, tr)
    assert state_tuple(drng) == state_tuple(rng_from_state(g["drng_after"]))
    assert rel_err(out, g["b0_seed_emb"][: len(out)]) < 1e-12
    loss, gr = ko.backward(p, b, cg, tr, v.local_ids, True)
    assert abs(loss - float(g["b0_loss"])) < 1e-12
    for l in range(L):
        assert rel_err(gr.bases[l], g[f"b0_dbases_{l}"]) < 1e-10
        assert rel_err(gr.coeffs[l], g[f"b0_dcoeffs_{l}"]) < 1e-10
    assert rel_err(gr.embed_rows, g["b0_embed_rows"]) < 1e-10
    got, curve, _, _ = ko.train(views, ends, oracle_params(g, "init_", L), 1, cfg["epochs"],
                                batch_size=cfg["batch"], seed=cfg["train_seed"], dropout=cfg["dropout"])
    np.testing.assert_allclose(curve, g["loss_curve"], rtol=1e-10)
    want = oracle_params(g, "trained_", L)
    for a, c in zip(got.dense(), want.dense()):
        assert rel_err(a, c) < 1e-9


@pytest.mark.parametrize("policy", ["mean", "optimistic", "pessimistic"])
def test_candidates_protocol_matches_reference(policy):
    g = load_golden("eval_candidates")
    L = len(g["dims"]) - 1
    p = oracle_params(g, "p_", L)
    ptr, cand = g["cand_ptr"], g["cand"]
    cmap = {i: cand[ptr[i]:ptr[i + 1]].tolist() for i in range(len(ptr) - 1)}
    ranks, ncand = ko.candidate_ranks(g["H"], p.decoder, g["test"], cmap, policy)
    np.testing.assert_array_equal(ranks, g[f"{policy}_ranks"])
    np.testing.assert_array_equal(ncand, g[f"{policy}_ncand"])
