"""Criterion 09 of the reference acceptance suite, split into its parts
(size / message-edge work / wall clock) to classify its result on a GPU.
Run from baseline/_ref/ref_tests with the kgdist alias on PYTHONPATH."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import test_acceptance as ta  # noqa: E402
from kgdist.partition import neighborhood_expand, random_edge_partition, vertex_cut_partition
from kgdist.trainer import TrainConfig, train

graph = ta._clustered_graph()
mc = ta.tiny_config(graph.num_relations, dims=(16, 16), mode=ta.MODE_EMBEDDING)
tc = TrainConfig(epochs=2, fixed_num_batches=8, optimizer="adam", seed=0)
rnd = neighborhood_expand(random_edge_partition(graph, 4, seed=0), graph, mc.num_layers)
vc = neighborhood_expand(vertex_cut_partition(graph, 4, seed=0), graph, mc.num_layers)
m = graph.num_edges
size_ok = all(p.num_total_edges >= 0.95 * m for p in rnd.partitions)
w_vc, w_rnd = ta._epoch_work(vc, mc, tc), ta._epoch_work(rnd, mc, tc)
times = {}
for name, ps in (("vertexcut", vc), ("random", rnd)):
    train(ps, graph, mc, tc)                      # warm (graph capture, first-epoch setup)
    _, rep = train(ps, graph, mc, TrainConfig(epochs=6, fixed_num_batches=8, optimizer="adam", seed=0))
    times[name] = float(np.mean(rep.epoch_seconds[1:]))
print(dict(size_ok=size_ok, work_vertexcut=int(w_vc), work_random=int(w_rnd), work_ok=bool(w_vc < w_rnd),
           epoch_s=times, wall_ok=bool(times["vertexcut"] < times["random"])))
