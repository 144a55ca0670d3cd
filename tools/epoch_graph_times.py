"""Replay time of one sampler epoch graph (negatives + shuffle + gather +
per-round closure/loss-group prep) for partition 0 of an FB15k-237-shaped
graph cut into P parts, in isolation, plus the eager per-kernel split of the
same work. python tools/epoch_graph_times.py [P ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2201_02791_b200 as kb
from paper_2201_02791_b200 import _lib
from paper_2201_02791_b200.partition import PartitionSet

Ps = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]
graph, split = kb.generate_synthetic(14541, 237, 272115 / 14541, seed=0)
mc = kb.ModelConfig(2, [100, 100, 100], 2, 237, 1, mode="embedding")
for P in Ps:
    pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, P, seed=0), graph, 2)
    tc = kb.TrainConfig(batch_size=65536, seed=0)
    tr = kb.Trainer(pset, graph, mc, tc)
    w = tr.workers[0]
    smp = w.sampler
    torch.cuda.synchronize()
    g = smp.slots[0]["graph"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(smp.side):
        for _ in range(2):
            g.replay()
        e0.record()
        reps = 5
        for _ in range(reps):
            g.replay()
        e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps

    def eager():
        with torch.cuda.stream(smp.side):
            smp._body(0)
        torch.cuda.synchronize()

    bd, _ = _lib.kernel_breakdown(eager)
    top = sorted(bd.items(), key=lambda x: -x[1][1])[:None if os.environ.get("EGT_ALL") else 8]
    print(f"P={P}: rounds/epoch {tr.rounds}, stream {smp.total}, epoch graph {ms:.3f} ms | " +
          ", ".join(f"{k} {v[1]:.3f}" + (f" (x{v[0]})" if os.environ.get("EGT_ALL") else "") for k, v in top))
    del tr
