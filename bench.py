#!/usr/bin/env python
"""Training-throughput benchmark of the partitioned RGCN + DistMult hot path.

Metric (BASELINE.json): train triples/s, RGCN+DistMult, FB15k-237 shape,
1/2/4/8 B200. Workload (BASELINE.json configs[0..1]): the reference's own
synthetic FB15k-237-shaped graph (14,541 entities / 237 relations / 272,116
train triples, generate_synthetic(seed=0)), P = world size self-sufficient
partitions (vertex cut seed 0 + 2-hop halo), one partition per GPU, RGCN 2x100
with 2 bases + DistMult, 1 negative per positive, Adam lr 0.01, edge
mini-batch b = 65,536 labelled triples per GPU (weak scaling).

A step = one synchronized training round on every rank: closure of the batch,
RGCN forward, DistMult+BCE, RGCN backward, all-gather of the dense gradients
(NCCL) + fused tree-mean/Adam, sparse embedding Adam; epoch boundaries
(negative sampling + shuffle on the GPU) fall inside the timed steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

METRIC = "train triples/s, RGCN+DistMult FB15k-237 shape, 1/2/4/8 B200; filtered MRR"
UNIT = "triples/s"
FB = dict(num_entities=14541, num_relations=237, avg_degree=272115 / 14541, seed=0)
DIMS = [100, 100, 100]
BASES = 2
BATCH = 65536


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--roofline-kernel", default="k_aggregate")
    ap.add_argument("--parts", type=int, default=0,
                    help="diagnostic: partitions (a multiple of the rank count; default one per GPU)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-rounds", type=int, default=2, help="bounded CPU baseline sample (rounds)")
    return ap.parse_args()


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    if world > 1 and not torch.distributed.is_initialized():
        # stdout carries exactly one JSON line: keep NCCL's init banner off it
        os.environ.setdefault("NCCL_DEBUG", "WARN")
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            torch.distributed.init_process_group("nccl" if torch.cuda.is_available() else "gloo",
                                                 device_id=torch.device("cuda", local) if torch.cuda.is_available()
                                                 else None)
            torch.distributed.barrier()
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
    return world, rank, local


def build_inputs(P, batch):
    import paper_2201_02791_b200 as kb
    graph, split = kb.generate_synthetic(FB["num_entities"], FB["num_relations"], FB["avg_degree"], FB["seed"])
    pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, P, seed=0), graph, 2)
    mc = kb.ModelConfig(2, list(DIMS), BASES, graph.num_relations, 1, mode=kb.MODE_EMBEDDING)
    tc = kb.TrainConfig(epochs=1, batch_size=batch, optimizer="adam", learning_rate=0.01, seed=0)
    return graph, split, pset, mc, tc


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML polling thread)
# ---------------------------------------------------------------------------
class ClockSampler:
    def __init__(self, index):
        self.samples, self.reasons, self.stop_flag = [], set(), False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = repr(e)

    def _run(self):
        nv = self.nv
        names = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                 "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}
        while not self.stop_flag:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_flag = True
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# algorithmic bytes of the instrumented kernels
# ---------------------------------------------------------------------------
def layer_shapes(tr, w):
    """Per layer l (input first): (targets T, sources S, message edges into T)."""
    import torch
    v = w.view
    counts = [int(x) for x in w.bufs.counts.cpu().tolist()]
    order = w.bufs.order.long()
    deg = (v.d_indptr[1:] - v.d_indptr[:-1]).long()
    L = tr.mc.num_layers
    out = []
    for l in range(L):
        t = L - 1 - l
        T, S = counts[t], counts[t + 1]
        E = int(deg[order[:T]].sum().item())
        out.append((T, S, E))
    return out


def algorithmic_bytes(kernel, tr, w):
    """Bytes a launch must move at minimum (fp32 values, int32 ids, per unit
    figures of SURVEY.md §8(d) restated in DESIGN.md §4)."""
    dims, B = tr.mc.dims, tr.mc.num_bases
    total = 0
    for l, (T, S, E) in enumerate(layer_shapes(tr, w)):
        di, do = dims[l], dims[l + 1]
        if kernel == "k_aggregate":
            # per message edge: src+rel+norm (12 B) + gathered source row; per
            # target: self row read + B*d_in accumulator row written
            total += E * (12 + 4 * di) + T * (4 * di + 4 * B * di + 4)
        elif kernel == "k_csc_backward":
            # per source row: Y row read, dS row written; per CSC edge: dst+rel+
            # norm+pos (16 B) + dZ row gathered + B floats edge dots written;
            # per target: self dZ row + B self dots
            total += S * (8 * B * do + 4) + E * (16 + 4 * do + 4 * B) + T * (4 * do + 4 * B)
    return total


# ---------------------------------------------------------------------------
# our implementation
# ---------------------------------------------------------------------------
def run_ours(args, world, rank, local):
    import torch
    import paper_2201_02791_b200 as kb
    from paper_2201_02791_b200 import _lib

    lib = _lib.require_cuda()
    dev = torch.device("cuda", local)
    P = args.parts or world
    graph, split, pset, mc, tc = build_inputs(P, args.batch)
    tr = kb.Trainer(pset, graph, mc, tc)
    tr.use_graphs = os.environ.get("KG_CUDA_GRAPHS", "1") != "0"
    tr.timer_prefix = args.roofline_kernel      # events around this kernel are captured into the graphs

    def step():
        if tr.round_in_epoch == 0 or tr.round_in_epoch >= tr.rounds:
            tr.begin_epoch()
        tr.run_round()

    for _ in range(max(args.warmup, 3)):
        step()
    tr.prepare()          # remaining one-time captures (train() overlaps them with device work)
    torch.cuda.synchronize()
    tr.check()

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if tr.dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    import ctypes
    launches0 = lib.kg_launch_count()
    g0 = tr.graph_kernel_launches
    kt_ms, kt_n = ctypes.c_double(0), ctypes.c_int64(0)
    lib.kg_kernel_timer_begin(args.roofline_kernel.encode())   # eager launches (graphs off)
    with ClockSampler(local) as clk:
        # the K timed steps: no host synchronisation inside the loop (the host
        # runs ahead, as in a training loop), events on the launch stream
        for k in range(args.steps):
            flush.zero_()                      # L2 flush between timed steps (outside the events)
            evs[k][0].record()
            step()
            evs[k][1].record()
        torch.cuda.synchronize()
    launches = lib.kg_launch_count() - launches0 + tr.graph_kernel_launches - g0
    if tr.dist:
        torch.distributed.barrier()
    step_ms = sum(a.elapsed_time(b) for a, b in evs)
    # roofline kernel: its events are captured into the replayed graphs; read
    # them over a few extra steps (each read synchronises, so not in the loop above)
    for _ in range(min(args.steps, 6)):
        flush.zero_()
        step()
        if tr.use_graphs and tr.last_timer_handle is not None:
            ms, n = ctypes.c_double(0), ctypes.c_int64(0)
            lib.kg_kernel_timer_read(tr.last_timer_handle, ctypes.byref(ms), ctypes.byref(n))
            kt_ms.value += ms.value
            kt_n.value += n.value
    torch.cuda.synchronize()
    e_ms, e_n = ctypes.c_double(0), ctypes.c_int64(0)
    lib.kg_kernel_timer_end(ctypes.byref(e_ms), ctypes.byref(e_n))
    kt_ms.value += e_ms.value
    kt_n.value += e_n.value
    tr.check()
    t_max = torch.tensor([step_ms], dtype=torch.float64, device=dev)
    rank_ms = [step_ms]
    if tr.dist:
        every = [torch.zeros_like(t_max) for _ in range(world)]
        torch.distributed.all_gather(every, t_max)
        rank_ms = [float(x.item()) for x in every]
        torch.distributed.all_reduce(t_max, op=torch.distributed.ReduceOp.MAX)
    total_ms = float(t_max.item())
    triples_per_step = sum(tr.sizes)          # every partition's batch, all ranks
    value = args.steps * triples_per_step / (total_ms / 1e3)

    # live roofline of the instrumented kernel (rank 0's launches)
    w0 = tr.workers[0]
    alg = algorithmic_bytes(args.roofline_kernel, tr, w0)
    per_launch_alg = alg / max(tr.mc.num_layers, 1)
    avg_launch_ms = kt_ms.value / max(kt_n.value, 1)
    peaks = {}
    pk_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.isfile(pk_path):
        peaks = json.load(open(pk_path))
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = per_launch_alg / (avg_launch_ms / 1e3) / 1e9 if avg_launch_ms > 0 else None
    # DRAM bytes per launch of this kernel from one ncu --set full capture of
    # the same command (tools/ncu_traffic.sh -> profiles/r1_roofline_traffic.json)
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "r1_roofline_traffic.json")
    if args.roofline_kernel == "k_aggregate" and os.path.isfile(tpath):
        tj = json.load(open(tpath))
        traffic, traffic_src = tj.get("traffic_bytes_per_launch"), tj.get("source")
    roofline = {"bound": "hbm", "kernel": args.roofline_kernel, "achieved": achieved, "peak": peak,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
                "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
                "traffic": traffic, "traffic_source": traffic_src, "alg_bytes_per_launch": per_launch_alg,
                "avg_launch_ms": avg_launch_ms, "launches_timed": kt_n.value,
                # launches per step (one per layer) x average launch / average step
                "kernel_share_of_step": (avg_launch_ms * max(tr.mc.num_layers, 1) / (step_ms / args.steps))
                if step_ms > 0 else None,
                "note": "FB15k-237 working set is L2-resident (H7): effective bandwidth vs HBM peak"}

    # e2e through the public API (host inputs -> train() -> host params)
    e2e = None
    if not args.no_e2e:
        # >= 900 rounds (100 epochs at P = 1, a short FB15k-237 run) so train()
        # takes its CUDA-graph path and its one-time setup (views, epoch/round
        # graph captures, allocator growth: 20-450 ms on a fresh process,
        # tools/e2e_breakdown.py) is amortised as in a real run; one untimed
        # call first absorbs process-level one-time costs (module load, graph
        # machinery), not per-run work
        epochs = max(1, math.ceil(args.steps / tr.rounds), math.ceil(900 / tr.rounds))
        # warm-up on the same (CUDA-graph, >= 64 rounds) path as the timed call
        kb.train(pset, graph, mc, kb.TrainConfig(epochs=math.ceil(64 / tr.rounds), batch_size=args.batch,
                                                 optimizer="adam", learning_rate=0.01, seed=0))
        tc2 = kb.TrainConfig(epochs=epochs, batch_size=args.batch, optimizer="adam", learning_rate=0.01, seed=0)
        if tr.dist:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        params, report = kb.train(pset, graph, mc, tc2)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        wt = torch.tensor([wall], dtype=torch.float64, device=dev)
        if tr.dist:
            torch.distributed.all_reduce(wt, op=torch.distributed.ReduceOp.MAX)
        wall = float(wt.item())
        steps_e2e = epochs * tr.rounds
        own = [pset.partitions[wid] for wid in tr.local_wids]
        h2d = sum(12 * (p.num_core_edges + len(p.support)) for p in own)            # partition triples (int32)
        h2d += 4 * tr.D + sum(4 * mc.dims[0] * len(p.local_vertices()) for p in own)   # params + local rows
        d2h = 8 * steps_e2e + 4 * tr.D + 4 * mc.dims[0] * graph.num_entities        # losses + params
        e2e = {"value": steps_e2e * triples_per_step / wall, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d * world / steps_e2e), "d2h_bytes_per_step": int(d2h * world / steps_e2e),
               "wall_s": wall, "steps": steps_e2e, "api": "paper_2201_02791_b200.train()",
               "final_loss": report.loss_curve[-1], "setup_s": report.setup_seconds,
               "epochs_s": float(sum(report.epoch_seconds)), "finish_s": report.finish_seconds,
               "epoch_ms": [round(x * 1e3, 2) for x in report.epoch_seconds]}
        from paper_2201_02791_b200 import trainer as _trm
        if _trm.setup_marks:
            m = _trm.setup_marks
            e2e["setup_marks_ms"] = [(b[0], round((b[1] - a[1]) * 1e3, 2)) for a, b in zip(m, m[1:])]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, pset, graph, mc)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(args.warmup, 3), "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"fb15k237-shape synthetic KG, P={P} partitions (vertex cut + 2-hop "
                                       f"halo), b={args.batch}/partition",
                           "model": "RGCN 2x100 (2 bases) + DistMult, 1 neg/pos, Adam 0.01, embedding mode",
                           "global_batch": triples_per_step, "per_gpu_batch": args.batch * P // world,
                           "rounds_per_epoch": tr.rounds, "parallelism": f"dp{world} (one partition per GPU)" if P == world
                           else f"dp{world}, {P // world} partitions per GPU",
                           "l2": "flushed between timed steps (256 MiB write)",
                           "graph": {"entities": graph.num_entities, "relations": graph.num_relations,
                                     "train_triples": graph.num_edges}},
                "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline, "cpu_baseline": cpu,
                "rank_ms": [round(x, 3) for x in rank_ms],
                "step_ms": [round(a.elapsed_time(b), 4) for a, b in evs],
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)


def cpu_baseline(args, pset, graph, mc, rounds=None):
    """The fp64 numpy port of the reference (oracle/) timed on this host's
    cores on a bounded sample of the same workload: one epoch's sampling plus
    `rounds` training rounds at the same batch size."""
    import kg_oracle as ko
    rounds = rounds or args.cpu_rounds
    views, ends = [], []
    for p in pset.partitions[:1]:
        views.append(ko.make_view(p.core, p.support, graph.num_entities, graph.num_relations,
                                  partition_id=p.id, pool_size=p.pool_size))
        ends.append(np.concatenate([p.core_vertices, p.replicated_vertices]))
    op = ko.init_params(mc.dims, mc.num_bases, mc.num_relations, np.random.default_rng(0),
                        num_entities=graph.num_entities)
    t0 = time.perf_counter()
    ko.train(views, ends, op, 1, 1, batch_size=args.batch, seed=0, max_rounds=rounds)
    secs = time.perf_counter() - t0
    threads = os.cpu_count()
    try:
        import threadpoolctl
        threads = max(i.get("num_threads", 1) for i in threadpoolctl.threadpool_info()) or threads
    except Exception:
        pass
    return {"value": rounds * args.batch / secs, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"oracle/kg_oracle.py train(): P=1 partition, one epoch of sampling + {rounds} rounds of "
                      f"b={args.batch} ({secs:.1f} s, fp64 numpy/OpenBLAS)"}


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU algorithm (numpy port under
    oracle/, the reference being pure Python that cannot travel) on this
    host's cores, same metric/config; rank 0 only."""
    if rank != 0:
        return
    import kg_oracle as ko
    sys.path.insert(0, ROOT)
    import paper_2201_02791_b200 as kb
    graph, split = kb.generate_synthetic(FB["num_entities"], FB["num_relations"], FB["avg_degree"], FB["seed"])
    pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, world, seed=0), graph, 2)
    views, ends = [], []
    for p in pset.partitions:
        views.append(ko.make_view(p.core, p.support, graph.num_entities, graph.num_relations,
                                  partition_id=p.id, pool_size=p.pool_size))
        ends.append(np.concatenate([p.core_vertices, p.replicated_vertices]))
    mc_dims = list(DIMS)
    op = ko.init_params(mc_dims, BASES, graph.num_relations, np.random.default_rng(0),
                        num_entities=graph.num_entities)
    # warmup rounds then timed rounds; each round processes P * b triples
    ko.train(views, ends, op, 1, 1, batch_size=args.batch, seed=0, max_rounds=max(1, min(args.warmup, 1)))
    t0 = time.perf_counter()
    done = 0
    rounds_per_epoch = ko.plan([v.num_core for v in views], 1, args.batch)[1]
    while done < args.steps:
        k = min(args.steps - done, rounds_per_epoch)
        ko.train(views, ends, op, 1, 1, batch_size=args.batch, seed=0, max_rounds=k)
        done += k
    secs = time.perf_counter() - t0
    value = args.steps * world * args.batch / secs
    threads = os.cpu_count()
    try:
        import threadpoolctl
        threads = max(i.get("num_threads", 1) for i in threadpoolctl.threadpool_info()) or threads
    except Exception:
        pass
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"fb15k237-shape synthetic KG, P={world} partitions (vertex cut + 2-hop halo), "
                                   f"b={args.batch}/partition", "parallelism": f"{world} partitions, in-order on CPU"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{args.steps} rounds x {world} partitions of b={args.batch} (per-epoch "
                                       f"sampling included), oracle/kg_oracle.py fp64 numpy port"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, int(os.environ.get("WORLD_SIZE", str(args.gpus))), rank)
        return
    world, rank, local = dist_setup()
    try:
        run_ours(args, world, rank, local)
    finally:
        import torch
        if torch.distributed.is_initialized():
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
