#!/usr/bin/env python
"""torch.profiler view of Trainer construction (the e2e setup cost).

    python tools/setup_profile.py > gpurun_out/setup_profile.txt
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2201_02791_b200 as kb  # noqa: E402


def main():
    graph, split, pset, mc, tc = bench.build_inputs(1, bench.BATCH)
    tc = kb.TrainConfig(epochs=20, batch_size=bench.BATCH, optimizer="adam", learning_rate=0.01, seed=0)
    kb.train(pset, graph, mc, tc)            # warm process-level state
    for i in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tr = kb.Trainer(pset, graph, mc, tc)
        torch.cuda.synchronize()
        print(f"Trainer() {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
        tr.close()
        del tr
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        tr = kb.Trainer(pset, graph, mc, tc)
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=45))
    print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=30))


if __name__ == "__main__":
    main()
