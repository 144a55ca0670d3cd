#!/usr/bin/env python
"""Step time with some kernels knocked out (KG_KNOCKOUT="k_a,k_b"; results are
wrong, only the timing is meaningful): how much each kernel adds to the
critical path of the FB-shape round. Same loop as bench.py (graphs, L2 flush).

    for k in "" k_aggregate_combine ...; do KG_KNOCKOUT=$k python tools/knockout.py; done
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2201_02791_b200 as kb  # noqa: E402


def main(steps=40, warmup=5, reps=3):
    graph, split, pset, mc, tc = bench.build_inputs(1, bench.BATCH)
    tr = kb.Trainer(pset, graph, mc, tc)
    tr.use_graphs = True

    def step():
        if tr.round_in_epoch == 0 or tr.round_in_epoch >= tr.rounds:
            tr.begin_epoch()
        tr.run_round()

    for _ in range(warmup):
        step()
    tr.prepare()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    best = []
    for _ in range(reps):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda.synchronize()
        for k in range(steps):
            flush.zero_()
            evs[k][0].record()
            step()
            evs[k][1].record()
        torch.cuda.synchronize()
        best.append(sum(a.elapsed_time(b) for a, b in evs) / steps)
    print(f"knockout={os.environ.get('KG_KNOCKOUT', '')!r:60s} ms/step {min(best):.4f} "
          f"(reps {', '.join(f'{x:.4f}' for x in best)})", flush=True)


if __name__ == "__main__":
    main()
