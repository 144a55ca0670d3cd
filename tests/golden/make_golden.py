"""Generate the golden fixtures under tests/golden/ by running the UNMODIFIED
reference (`kgdist`, /root/reference/pkg/src) in this container.

The reference is pure Python, so it cannot travel to the GPU box; this script
freezes its outputs (integer structure bit-exact, float64 numerics as-is) into
small .npz files that the oracle (oracle/kg_oracle.py) is pinned against in
the CPU suite, and that the GPU parity tests compare against on the box.

Run:  python tests/golden/make_golden.py      (needs /root/reference)
"""

from __future__ import annotations

import copy
import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = os.environ.get("KGDIST_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)

import kgdist  # noqa: E402
import importlib  # noqa: E402
kev = importlib.import_module("kgdist.evaluate")
from kgdist import model as kmodel  # noqa: E402
from kgdist import partition as kpart  # noqa: E402
from kgdist import sampler as ksamp  # noqa: E402
from kgdist import trainer as ktrain  # noqa: E402
from kgdist.graph import KnowledgeGraph, generate_synthetic  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def rng_state(rng):
    st = rng.bit_generator.state
    return np.array([st["state"]["state"] >> 64, st["state"]["state"] & (2**64 - 1),
                     st["state"]["inc"] >> 64, st["state"]["inc"] & (2**64 - 1),
                     st["has_uint32"], st["uinteger"]], dtype=np.uint64)


def multigraph(num_entities, num_relations, num_edges, seed):
    """Duplicate-allowing random multigraph without self loops (the same
    construction the reference's tests use for their small fixtures)."""
    rng = np.random.default_rng(seed)
    heads = rng.integers(0, num_entities, num_edges)
    rels = rng.integers(0, num_relations, num_edges)
    tails = rng.integers(0, num_entities, num_edges)
    bad = heads == tails
    while bad.any():
        tails[bad] = rng.integers(0, num_entities, int(bad.sum()))
        bad = heads == tails
    return KnowledgeGraph(num_entities, num_relations,
                          np.stack([heads, rels, tails], axis=1).astype(np.int64))


def dump_partitions(prefix, pset, out):
    out[f"{prefix}num_parts"] = np.int64(pset.num_parts)
    for p in pset.partitions:
        k = f"{prefix}p{p.id}_"
        out[k + "core_edge_ids"] = p.core_edge_ids
        out[k + "support_edge_ids"] = (p.support_edge_ids if p.support_edge_ids is not None
                                       else np.zeros(0, np.int64))
        out[k + "core_vertices"] = p.core_vertices
        out[k + "replicated_vertices"] = p.replicated_vertices
        out[k + "support_vertices"] = p.support_vertices
        out[k + "local_ids"] = p.local_vertices()


def dump_view(prefix, view, out):
    out[prefix + "local_ids"] = view.local_ids
    out[prefix + "edges"] = view.edges
    out[prefix + "num_core"] = np.int64(view.num_core)
    out[prefix + "pool"] = view.pool
    out[prefix + "msg_indptr"] = view.msg_indptr
    out[prefix + "msg_src"] = view.msg_src
    out[prefix + "msg_rel"] = view.msg_rel
    out[prefix + "msg_norm"] = view.msg_norm
    out[prefix + "positive_keys"] = view.positive_keys


def dump_cg(prefix, cg, out):
    out[prefix + "seed_vertices"] = cg.seed_vertices
    out[prefix + "vertex_order"] = cg.vertex_order
    out[prefix + "counts"] = np.asarray(cg.layer_vertex_counts, dtype=np.int64)
    for li, blk in enumerate(cg.layers):
        q = f"{prefix}L{li}_"
        out[q + "dst"] = blk.dst
        out[q + "src"] = blk.src
        out[q + "rel"] = blk.rel
        out[q + "norm"] = blk.norm


def dump_params(prefix, params, out):
    for l, (b, c) in enumerate(zip(params.bases, params.coeffs)):
        out[f"{prefix}bases_{l}"] = b
        out[f"{prefix}coeffs_{l}"] = c
    out[prefix + "decoder"] = params.decoder
    if params.entity_embed is not None:
        out[prefix + "entity_embed"] = params.entity_embed


def fp32_params(params):
    """Round every parameter to fp32 and back so CPU fp64 and GPU fp32 runs
    start from bit-identical values (SURVEY.md BASELINE.md §3 'same inputs')."""
    q = params.copy()
    q.bases = [b.astype(np.float32).astype(np.float64) for b in q.bases]
    q.coeffs = [c.astype(np.float32).astype(np.float64) for c in q.coeffs]
    q.decoder = q.decoder.astype(np.float32).astype(np.float64)
    if q.entity_embed is not None:
        q.entity_embed = q.entity_embed.astype(np.float32).astype(np.float64)
    return q


# ---------------------------------------------------------------------------
# Scenario A: small multigraph, 2 partitions, every hot-path stage
# ---------------------------------------------------------------------------

def scenario_small(name, graph, parts, hops, part_seed, dims, s, batch, rounds,
                   train_seed, epochs, num_bases=2, mode="embedding"):
    out = {}
    out["triples"] = graph.triples
    out["num_entities"] = np.int64(graph.num_entities)
    out["num_relations"] = np.int64(graph.num_relations)
    out["graph_checksum"] = np.frombuffer(graph.checksum().encode(), dtype=np.uint8)
    pset = kpart.neighborhood_expand(
        kpart.vertex_cut_partition(graph, parts, part_seed), graph, hops)
    dump_partitions("", pset, out)
    out["hops"] = np.int64(hops)
    views = [ksamp.build_view(p, graph.num_entities, graph.num_relations)
             for p in pset.partitions]
    for v in views:
        dump_view(f"view{v.partition_id}_", v, out)

    # negatives + batches + compute graphs for partition 0, one epoch
    view = views[0]
    rng = np.random.default_rng(4242)
    out["rng_init"] = rng_state(rng)
    neg = ksamp.sample_negatives(view, s, rng)
    out["neg"] = neg
    out["rng_after_neg"] = rng_state(rng)
    batches = ksamp.make_batches(view.core_edges, neg, batch, rng, num_batches=rounds)
    out["rng_after_batches"] = rng_state(rng)
    for i, b in enumerate(batches):
        out[f"batch{i}_triples"] = b.triples
        out[f"batch{i}_labels"] = b.labels
        cg = ksamp.build_compute_graph(b, view, hops)
        dump_cg(f"cg{i}_", cg, out)

    # model math on batch 0 from fp32-representable params
    mc = kmodel.ModelConfig(num_layers=len(dims) - 1, dims=list(dims), num_bases=num_bases,
                            num_relations=graph.num_relations, negatives_per_positive=s,
                            mode=mode)
    params = fp32_params(kmodel.init_params(mc, np.random.default_rng(train_seed),
                                            num_entities=graph.num_entities))
    dump_params("init_", params, out)
    if mode == "feature":
        feats = np.random.default_rng(train_seed + 1).normal(size=(graph.num_entities, dims[0]))
        feats = feats.astype(np.float32).astype(np.float64)
        graph.features = feats
        out["features"] = feats
    table = params.entity_embed if mode == "embedding" else graph.features
    b0 = batches[0]
    cg0 = ksamp.build_compute_graph(b0, view, hops)
    cache = kmodel.EncodeCache()
    emb = kmodel.encode(params, mc, cg0, table, view.local_ids, cache=cache)
    loss, grads = kmodel.loss_from_cache(params, mc, b0, cg0, cache, view.local_ids)
    out["b0_seed_emb"] = emb
    out["b0_loss"] = np.float64(loss)
    for l in range(mc.num_layers):
        out[f"b0_dbases_{l}"] = grads.bases[l]
        out[f"b0_dcoeffs_{l}"] = grads.coeffs[l]
    out["b0_ddecoder"] = grads.decoder
    if grads.embed_ids is not None:
        out["b0_embed_ids"] = grads.embed_ids
        out["b0_embed_rows"] = grads.embed_rows

    # full training run (P partitions) through the public train()
    tc = ktrain.TrainConfig(epochs=epochs, batch_size=batch, optimizer="adam",
                            learning_rate=0.01, seed=train_seed)
    got, report = ktrain.train(pset, graph, mc, tc, initial_params=params)
    dump_params("trained_", got, out)
    out["loss_curve"] = np.asarray(report.loss_curve)
    out["rounds_per_epoch"] = np.int64(report.rounds_per_epoch)
    out["batch_sizes"] = np.asarray(report.batch_sizes, dtype=np.int64)
    out["config_json"] = np.frombuffer(json.dumps({
        "dims": list(dims), "num_bases": num_bases, "s": s, "batch": batch,
        "rounds": rounds, "train_seed": train_seed, "epochs": epochs, "mode": mode,
        "parts": parts, "hops": hops, "part_seed": part_seed}).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(f"wrote {name}.npz ({len(out)} arrays)")


# ---------------------------------------------------------------------------
# Scenario B: filtered evaluation (all tie policies) on a synthetic split
# ---------------------------------------------------------------------------

def scenario_eval(name, n, R, deg, seed, dims):
    graph, split = generate_synthetic(n, R, deg, seed=seed)
    mc = kmodel.ModelConfig(num_layers=len(dims) - 1, dims=list(dims), num_bases=2,
                            num_relations=R, mode="embedding")
    params = fp32_params(kmodel.init_params(mc, np.random.default_rng(seed + 1),
                                            num_entities=n))
    out = {"train": split.train, "valid": split.valid, "test": split.test,
           "num_entities": np.int64(n), "num_relations": np.int64(R),
           "dims": np.asarray(dims, dtype=np.int64)}
    dump_params("p_", params, out)
    H = kev.encode_all_entities(params, mc, graph)
    out["H"] = H
    for pol in (kev.TIE_MEAN, kev.TIE_OPTIMISTIC, kev.TIE_PESSIMISTIC):
        res = kev.evaluate(params, mc, graph, split, which="test", tie_policy=pol)
        out[f"{pol}_mrr"] = np.float64(res.mrr)
        out[f"{pol}_hits"] = np.asarray([res.hits[k] for k in (1, 3, 10)])
        out[f"{pol}_ranks"] = np.asarray([r.rank for r in res.records])
        out[f"{pol}_ncand"] = np.asarray([r.num_candidates for r in res.records])
        out[f"{pol}_side"] = np.asarray([0 if r.corrupted_side == "tail" else 1
                                         for r in res.records], dtype=np.int8)
        out[f"{pol}_hrt"] = np.asarray([(r.head, r.rel, r.tail) for r in res.records])
    res = kev.evaluate(params, mc, graph, split, which="valid")
    out["valid_mrr"] = np.float64(res.mrr)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(f"wrote {name}.npz")


# ---------------------------------------------------------------------------
# Scenario C: FB15k-237-shaped generator + vertex cut (bit-exact structure)
# ---------------------------------------------------------------------------

def scenario_fb_structure(name):
    graph, split = generate_synthetic(14541, 237, 272115 / 14541, seed=0)
    out = {
        "checksum": np.frombuffer(graph.checksum(split).encode(), dtype=np.uint8),
        "num_train": np.int64(len(split.train)),
        "num_valid": np.int64(len(split.valid)),
        "num_test": np.int64(len(split.test)),
        "train_sha": np.frombuffer(hashlib.sha256(split.train.tobytes()).hexdigest().encode(),
                                   dtype=np.uint8),
    }
    for P in (1, 2, 4, 8):
        pset = kpart.vertex_cut_partition(graph, P, seed=0)
        assign = np.empty(graph.num_edges, dtype=np.int8)
        for p in pset.partitions:
            assign[p.core_edge_ids] = p.id
        out[f"assign_P{P}"] = assign
        ex = kpart.neighborhood_expand(pset, graph, 2)
        out[f"support_counts_P{P}"] = np.asarray([len(p.support) for p in ex.partitions])
        out[f"vertex_counts_P{P}"] = np.asarray([len(p.local_vertices()) for p in ex.partitions])
        out[f"pool_P{P}"] = np.asarray([len(p.core_vertices) + len(p.replicated_vertices)
                                        for p in ex.partitions])
        v0 = ksamp.build_view(ex.partitions[0], graph.num_entities, graph.num_relations)
        h = hashlib.sha256()
        for a in (v0.local_ids, v0.msg_indptr, v0.msg_src, v0.msg_rel, v0.positive_keys):
            h.update(np.ascontiguousarray(a, dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(v0.msg_norm).tobytes())
        out[f"view0_sha_P{P}"] = np.frombuffer(h.hexdigest().encode(), dtype=np.uint8)
        rng = np.random.default_rng(0 ^ 0)
        neg = ksamp.sample_negatives(v0, 1, rng)
        out[f"neg0_sha_P{P}"] = np.frombuffer(
            hashlib.sha256(neg.astype(np.int64).tobytes()).hexdigest().encode(), dtype=np.uint8)
        out[f"neg0_head_P{P}"] = neg[:64]
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(f"wrote {name}.npz")


def scenario_candidates(name):
    """Given-candidates protocol (ref:evaluate.py:168-180): per test index a
    candidate list (some without the true tail -> appended, some with
    duplicates of it), all tie policies."""
    n, R, dims = 200, 6, (8, 8, 8)
    graph, split = generate_synthetic(n, R, 5.0, seed=5)
    mc = kmodel.ModelConfig(num_layers=2, dims=list(dims), num_bases=2, num_relations=R, mode="embedding")
    params = fp32_params(kmodel.init_params(mc, np.random.default_rng(6), num_entities=n))
    rng = np.random.default_rng(17)
    cmap, flat, ptr = {}, [], [0]
    for i, (h, r, t) in enumerate(split.test.tolist()):
        c = rng.integers(0, n, int(rng.integers(5, 40)))
        if i % 3 == 0:
            c = np.concatenate([c, [t]])
        if i % 7 == 0:
            c = np.concatenate([c, [t, t]])
        cmap[i] = c.tolist()
        flat += cmap[i]
        ptr.append(len(flat))
    out = {"train": split.train, "valid": split.valid, "test": split.test,
           "num_entities": np.int64(n), "num_relations": np.int64(R), "dims": np.asarray(dims, dtype=np.int64),
           "cand": np.asarray(flat, dtype=np.int64), "cand_ptr": np.asarray(ptr, dtype=np.int64)}
    dump_params("p_", params, out)
    out["H"] = kev.encode_all_entities(params, mc, graph)
    for pol in (kev.TIE_MEAN, kev.TIE_OPTIMISTIC, kev.TIE_PESSIMISTIC):
        res = kev.evaluate(params, mc, graph, split, which="test", protocol="candidates", candidates=cmap,
                           tie_policy=pol)
        out[f"{pol}_mrr"] = np.float64(res.mrr)
        out[f"{pol}_ranks"] = np.asarray([r.rank for r in res.records])
        out[f"{pol}_ncand"] = np.asarray([r.num_candidates for r in res.records])
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(f"wrote {name}.npz")


def scenario_dropout(name):
    """Inverted dropout (ref:model.py:221-227): one teacher-forced training
    step with a seeded dropout Generator (masks, loss, gradients, Generator
    state after) and a 2-partition training run with dropout 0.25."""
    out = {}
    graph = multigraph(60, 4, 260, seed=21)
    dims, hops = (6, 8, 8, 5), 3
    out["triples"] = graph.triples
    out["num_entities"] = np.int64(graph.num_entities)
    out["num_relations"] = np.int64(graph.num_relations)
    pset = kpart.neighborhood_expand(kpart.vertex_cut_partition(graph, 2, 3), graph, hops)
    dump_partitions("", pset, out)
    out["hops"] = np.int64(hops)
    mc = kmodel.ModelConfig(num_layers=3, dims=list(dims), num_bases=2,
                            num_relations=graph.num_relations, negatives_per_positive=1,
                            dropout=0.25, mode="embedding")
    params = fp32_params(kmodel.init_params(mc, np.random.default_rng(8),
                                            num_entities=graph.num_entities))
    dump_params("init_", params, out)
    view = ksamp.build_view(pset.partitions[0], graph.num_entities, graph.num_relations)
    rng = np.random.default_rng(99)
    neg = ksamp.sample_negatives(view, 1, rng)
    b0 = ksamp.make_batches(view.core_edges, neg, 40, rng, num_batches=2)[0]
    out["batch0_triples"] = b0.triples
    out["batch0_labels"] = b0.labels
    cg0 = ksamp.build_compute_graph(b0, view, hops)
    drng = np.random.default_rng(1234)
    out["drng_init"] = rng_state(drng)
    cache = kmodel.EncodeCache()
    emb = kmodel.encode(params, mc, cg0, params.entity_embed, view.local_ids, training=True,
                        dropout_rng=drng, cache=cache)
    loss, grads = kmodel.loss_from_cache(params, mc, b0, cg0, cache, view.local_ids)
    out["drng_after"] = rng_state(drng)
    out["b0_seed_emb"] = emb
    out["b0_loss"] = np.float64(loss)
    for l in range(mc.num_layers):
        out[f"b0_dbases_{l}"] = grads.bases[l]
        out[f"b0_dcoeffs_{l}"] = grads.coeffs[l]
    out["b0_ddecoder"] = grads.decoder
    out["b0_embed_ids"] = grads.embed_ids
    out["b0_embed_rows"] = grads.embed_rows
    tc = ktrain.TrainConfig(epochs=2, batch_size=48, optimizer="adam", learning_rate=0.01, seed=3)
    got, report = ktrain.train(pset, graph, mc, tc, initial_params=params)
    dump_params("trained_", got, out)
    out["loss_curve"] = np.asarray(report.loss_curve)
    out["config_json"] = np.frombuffer(json.dumps({
        "dims": list(dims), "hops": hops, "dropout": 0.25, "parts": 2, "part_seed": 3,
        "batch": 48, "epochs": 2, "train_seed": 3}).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(f"wrote {name}.npz ({len(out)} arrays)")


if __name__ == "__main__":
    if "--dropout-only" in sys.argv:
        scenario_dropout("dropout_small")
        sys.exit(0)
    if "--candidates-only" in sys.argv:
        scenario_candidates("eval_candidates")
        sys.exit(0)
    scenario_small("small_embed", multigraph(40, 5, 160, seed=11), parts=2, hops=2,
                   part_seed=1, dims=(5, 6, 4), s=2, batch=32, rounds=4,
                   train_seed=9, epochs=2)
    scenario_small("small_feature3", multigraph(30, 3, 90, seed=3), parts=1, hops=3,
                   part_seed=2, dims=(4, 5, 5, 3), s=1, batch=24, rounds=3,
                   train_seed=5, epochs=2, num_bases=3, mode="feature")
    scenario_small("synth_p4", generate_synthetic(300, 7, 5.0, seed=2)[0], parts=4, hops=2,
                   part_seed=0, dims=(16, 16, 8), s=1, batch=128, rounds=5,
                   train_seed=1, epochs=2)
    scenario_eval("eval_small", 200, 6, 5.0, seed=5, dims=(8, 8, 8))
    scenario_dropout("dropout_small")
    scenario_candidates("eval_candidates")
    if "--fb" in sys.argv:
        scenario_fb_structure("fb_structure")
