"""Configs 4 and 5 on one GPU:
  4: ogbl-wikikg2-shaped synthetic KG (2.5M entities, 535 relations, ~16M
     train triples), RGCN dims [128,128,128], 2 bases, P = 8 vertex-cut
     partitions with 2-hop halos, b = 1,048,576 per GPU;
  5: ogbl-citation2-shaped graph (2.93M nodes, 1 relation, ~30.4M edges),
     3-layer RGCN dims [32,32,32,32], 3-hop halos, P = 8, 256/P batches per
     epoch (b ~ 237k per GPU).
One GPU runs partition `--part` exactly as it would in the 8-GPU job (its
per-round work does not depend on the other ranks apart from the small dense
gradient exchange).

Prints one JSON line: triples/s of the partition, and for the message-passing
kernels the algorithmic bytes per launch / measured launch time
against the measured HBM peak. `--scale` shrinks the graph for quick checks.
python tools/bench_config4.py [--scale 1.0] [--rounds 8]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2201_02791_b200 as kb
from paper_2201_02791_b200 import _lib
from paper_2201_02791_b200.partition import PartitionSet

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4, choices=[4, 5])
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--parts", type=int, default=8)
ap.add_argument("--part", type=int, default=0)
ap.add_argument("--batch", type=int, default=1048576)
ap.add_argument("--rounds", type=int, default=8)
args = ap.parse_args()

t0 = time.perf_counter()
if args.config == 4:
    n_ent, R, deg, dims, hops = int(2_500_000 * args.scale), 535, 6.4, [128, 128, 128], 2
else:
    n_ent, R, dims, hops = int(2_927_963 * args.scale), 1, [32, 32, 32, 32], 3
    deg = 30_387_995 / 2_927_963
graph, split = kb.generate_synthetic(n_ent, R, deg, seed=0)
t_gen = time.perf_counter() - t0
t0 = time.perf_counter()
pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, args.parts, seed=0), graph, hops)
t_part = time.perf_counter() - t0
one = PartitionSet([pset.partitions[args.part]], pset.num_entities, pset.num_relations, pset.hops, pset.seed,
                   pset.method, pset.graph_checksum)
mc = kb.ModelConfig(len(dims) - 1, dims, 2, R, 1, mode="embedding")
if args.config == 4:
    tc = kb.TrainConfig(batch_size=args.batch, seed=0)
else:   # 256 / P batches per epoch
    tc = kb.TrainConfig(fixed_num_batches=max(1, 256 // args.parts), seed=0)
t0 = time.perf_counter()
tr = kb.Trainer(one, graph, mc, tc)
t_setup = time.perf_counter() - t0
w = tr.workers[0]


def step():
    if tr.round_in_epoch == 0 or tr.round_in_epoch >= tr.rounds:
        tr.begin_epoch()
    tr.run_round()


# eager per-kernel breakdown of one round on a single stream (kernel times are
# ms-scale here; forked streams would fold contention into the event times)
tr.use_graphs = False
tr.fork_streams = False
step()
torch.cuda.synchronize()
bd, _ = _lib.kernel_breakdown(step)
tr.fork_streams = True
tr.use_graphs = True
for _ in range(3):
    step()
tr.prepare()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.rounds):
    step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / args.rounds
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6530.3) if os.path.exists(
    os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6530.3
kern = {}
fused = bd.get("k_csc_dots", (0, 0.0))[0] == 0        # eager single stream: one CSC pass per layer
for name in ("k_aggregate", "k_csc_backward", "k_csc_dots"):
    n, t = bd.get(name, (0, 0.0))
    model = "csc_family" if (name == "k_csc_backward" and fused) else name
    alg = bench.algorithmic_bytes(model, tr, w)
    if n:
        per = t / n
        kern[name] = {"launches": n, "ms_per_launch": per, "alg_bytes_per_launch": alg / mc.num_layers,
                      "byte_model": model, "achieved_gbs": alg / mc.num_layers / (per * 1e-3) / 1e9,
                      "frac_hbm": alg / mc.num_layers / (per * 1e-3) / 1e9 / peak}
shapes = bench.layer_shapes(tr, w)
top = sorted(bd.items(), key=lambda x: -x[1][1])[:12]
print(json.dumps({
    "workload": f"config {args.config} synthetic KG scale {args.scale}: {graph.num_entities} entities, {R} relations, "
                f"{len(graph.triples)} train triples; dims {dims}; partition {args.part} of {args.parts} "
                f"({hops}-hop halo)",
    "n_local": w.view.n, "messages": int(w.view.e) if hasattr(w.view, "e") else None,
    "batch": w.b, "rounds_per_epoch": tr.rounds, "layer_shapes_T_S_E": shapes,
    "ms_per_round": ms, "triples_per_s": w.b / (ms * 1e-3),
    "kernels": kern, "peak_hbm_gbs": peak,
    "eager_breakdown_ms": {k: round(v[1], 3) for k, v in top},
    "host_s": {"generate": round(t_gen, 1), "partition_expand": round(t_part, 1), "trainer_setup": round(t_setup, 1)},
}))
