import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_02791_b200 as kb
from paper_2201_02791_b200 import _lib
graph, split = kb.generate_synthetic(2000, 20, 8.0, seed=1)
pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, 1, seed=0), graph, 2)
mc = kb.ModelConfig(2, [32, 32, 32], 2, graph.num_relations, 1, mode="embedding")
tr = kb.Trainer(pset, graph, mc, kb.TrainConfig(batch_size=2048, seed=0))
for k in range(6):
    if tr.round_in_epoch == 0 or tr.round_in_epoch >= tr.rounds:
        tr.begin_epoch()
    tr.run_round()
    torch.cuda.synchronize()
    print("round", k, "ok", flush=True)
print("stale err:", _lib.last_error())
v = kb.build_view(pset.partitions[0], graph.num_entities, graph.num_relations)
print("view ok", v.n)
