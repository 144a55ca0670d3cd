"""Feature-mode vs embedding-mode training against the oracle on a small graph (diagnostic)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import kg_oracle as ko
import paper_2201_02791_b200 as kb

q = lambda a: None if a is None else a.astype(np.float32).astype(np.float64)
for P in (1, 2):
    for mode in ("feature", "embedding"):
        graph, _ = kb.generate_synthetic(300, 4, 5.0, seed=11)
        feats = q(np.random.default_rng(3).normal(size=(graph.num_entities, 12)))
        if mode == "feature":
            graph = kb.KnowledgeGraph(graph.num_entities, graph.num_relations, graph.triples, features=feats)
        pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, P, seed=0), graph, 2)
        mc = kb.ModelConfig(2, [12, 16, 8], 2, graph.num_relations, 1, mode=mode)
        p0 = kb.init_params(mc, np.random.default_rng(5), num_entities=graph.num_entities)
        p0 = kb.ModelParams([q(b) for b in p0.bases], [q(c) for c in p0.coeffs], q(p0.decoder), q(p0.entity_embed))
        tc = kb.TrainConfig(epochs=3, batch_size=128, optimizer="adam", learning_rate=0.01, seed=0)
        got, rep = kb.train(pset, graph, mc, tc, initial_params=p0)
        views, ends = [], []
        for part in pset.partitions:
            views.append(ko.make_view(part.core, part.support, graph.num_entities, graph.num_relations,
                                      partition_id=part.id, pool_size=part.pool_size))
            ends.append(np.concatenate([part.core_vertices, part.replicated_vertices]))
        op = ko.OParams([b.copy() for b in p0.bases], [c.copy() for c in p0.coeffs], p0.decoder.copy(),
                        None if p0.entity_embed is None else p0.entity_embed.copy())
        want, curve, rounds, sizes = ko.train(views, ends, op, 1, 3, batch_size=128, seed=0,
                                              features=feats if mode == "feature" else None)
        print(P, mode, "rounds", rep.rounds_per_epoch, rounds, "dev", [round(x, 6) for x in rep.loss_curve],
              "oracle", [round(x, 6) for x in curve], flush=True)
