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
    ap.add_argument("--nogc", action="store_true", help="cyclic GC disabled during each call")
    ap.add_argument("--sample", action="store_true", help="sample the main thread's stack during setup spikes")
    ap.add_argument("--pause", type=float, default=0.0, help="seconds of idle host time between calls")
    a = ap.parse_args()
    samples = []
    if a.sample:
        import threading
        import traceback
        main_id = threading.main_thread().ident

        def sampler():
            while True:
                fr = sys._current_frames().get(main_id)
                if fr is not None:
                    st = traceback.extract_stack(fr)[-8:]
                    samples.append((time.perf_counter(), tuple(f"{os.path.basename(x.filename)}:{x.lineno}:{x.name}"
                                                               for x in st)))
                time.sleep(0.002)
        threading.Thread(target=sampler, daemon=True).start()
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
        if a.pause:
            time.sleep(a.pause)
        ms0 = torch.cuda.memory_stats()
        t0 = time.perf_counter()
        if prof:
            prof.enable()
        if a.nogc:
            import gc
            gc.disable()
        _, rep = kb.train(pset, graph, mc, tc2)
        if a.nogc:
            gc.enable()
        torch.cuda.synchronize()
        if prof:
            prof.disable()
        wall = time.perf_counter() - t0
        ms1 = torch.cuda.memory_stats()
        seg = {k: ms1.get(k, 0) - ms0.get(k, 0) for k in ("segment.all.allocated", "segment.all.freed",
                                                          "allocated_bytes.all.allocated", "num_alloc_retries",
                                                          "num_device_alloc", "num_device_free")}
        ep = rep.epoch_seconds
        if rank != 0:
            continue
        print(f"call {i}: wall {wall*1e3:.1f} ms setup {rep.setup_seconds*1e3:.1f} epochs {sum(ep)*1e3:.1f} "
              f"(first {ep[0]*1e3:.2f}, median {sorted(ep)[len(ep)//2]*1e3:.2f}, max {max(ep)*1e3:.2f}) "
              f"finish {rep.finish_seconds*1e3:.1f} -> {epochs*tr_rounds(rep)*bench.BATCH/wall/1e6:.1f} M/s",
              flush=True)
        print(f"   cudaMalloc/cudaFree this call: {seg}; allocated {torch.cuda.memory_allocated() / 2**20:.1f} MiB, "
              f"reserved {torch.cuda.memory_reserved() / 2**20:.1f} MiB after the call", flush=True)
        if a.sample:
            import collections
            if rep.setup_seconds > 0.06:
                win = [st for t, st in samples if t0 <= t <= t0 + rep.setup_seconds]
                for st, c in collections.Counter(win).most_common(4):
                    print(f"   [{c} samples] " + " <- ".join(reversed(st)), flush=True)
            if rep.epoch_seconds[0] > 0.02:
                a0 = t0 + rep.setup_seconds
                win = [st for t, st in samples if a0 <= t <= a0 + 0.2]
                print("   first-epoch host samples:", flush=True)
                for st, c in collections.Counter(win).most_common(6):
                    print(f"   [{c} samples] " + " <- ".join(reversed(st)), flush=True)
            samples.clear()
        from paper_2201_02791_b200 import _lib as libm2
        if libm2.slow_calls:
            print("   slow library calls:", libm2.slow_calls, flush=True)
            libm2.slow_calls.clear()
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
