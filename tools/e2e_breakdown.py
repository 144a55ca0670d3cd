#!/usr/bin/env python
"""Where the end-to-end train() wall time goes (bench.py's e2e leg, repeated).

    python tools/e2e_breakdown.py [--repeats 5] [--rounds 180] [--profile]

Prints setup / epochs / finish seconds per call and, with --profile, the top
cProfile entries of the last call.
"""
import argparse
import cProfile
import math
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2201_02791_b200 as kb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--rounds", type=int, default=180)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--gc", action="store_true", help="gc.collect() before every call")
    a = ap.parse_args()
    world, rank, local = bench.dist_setup()      # torchrun: one partition per rank
    graph, split, pset, mc, tc = bench.build_inputs(world, bench.BATCH)
    tr = kb.Trainer(pset, graph, mc, tc)
    epochs = math.ceil(a.rounds / tr.rounds)
    del tr
    for i in range(a.repeats):
        tc2 = kb.TrainConfig(epochs=epochs, batch_size=bench.BATCH, optimizer="adam", learning_rate=0.01, seed=0)
        prof = cProfile.Profile() if a.profile else None
        if a.gc:
            import gc
            gc.collect()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if prof:
            prof.enable()
        _, rep = kb.train(pset, graph, mc, tc2)
        torch.cuda.synchronize()
        if prof:
            prof.disable()
        wall = time.perf_counter() - t0
        ep = rep.epoch_seconds
        if rank != 0:
            continue
        print(f"call {i}: wall {wall*1e3:.1f} ms setup {rep.setup_seconds*1e3:.1f} epochs {sum(ep)*1e3:.1f} "
              f"(first {ep[0]*1e3:.2f}, median {sorted(ep)[len(ep)//2]*1e3:.2f}, max {max(ep)*1e3:.2f}) "
              f"finish {rep.finish_seconds*1e3:.1f} -> {epochs*tr_rounds(rep)*bench.BATCH/wall/1e6:.1f} M/s",
              flush=True)
        from paper_2201_02791_b200 import _lib as libm
        if libm.capture_times:
            print("   captures (begin, body, end, upload ms):", libm.capture_times, flush=True)
            libm.capture_times.clear()
        from paper_2201_02791_b200 import trainer as trm
        if trm.setup_marks:
            m = trm.setup_marks
            print("   setup marks:", [(b[0], round((b[1] - a[1]) * 1e3, 1)) for a, b in zip(m, m[1:])], flush=True)
        if prof and wall > 0.2:
            pstats.Stats(prof).sort_stats("tottime").print_stats(15)


def tr_rounds(rep):
    return rep.rounds_per_epoch


if __name__ == "__main__":
    main()
