"""Warm in-situ per-kernel breakdown of training steps (events around every
library launch; not a bench number). python tools/breakdown.py [P] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2201_02791_b200 as kb
from paper_2201_02791_b200 import _lib

steps = int(sys.argv[2]) if len(sys.argv) > 2 else 9
graph, split = kb.generate_synthetic(14541, 237, 272115 / 14541, seed=0)
pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, 1, seed=0), graph, 2)
mc = kb.ModelConfig(2, [100, 100, 100], 2, 237, 1, mode="embedding")
tc = kb.TrainConfig(batch_size=65536, seed=0)
tr = kb.Trainer(pset, graph, mc, tc)


def run(n):
    for _ in range(n):
        if tr.round_in_epoch == 0 or tr.round_in_epoch >= tr.rounds:
            tr.begin_epoch()
        tr.run_round()
    torch.cuda.synchronize()


run(12)
agg, _ = _lib.kernel_breakdown(run, steps)
tot = sum(v[1] for v in agg.values())
print(f"{steps} steps, summed kernel time {tot:.3f} ms ({tot / steps:.3f} ms/step)")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:32s} {n:6d} {ms:9.3f} ms  {1000 * ms / n:8.1f} us/launch  {100 * ms / tot:5.1f}%")
