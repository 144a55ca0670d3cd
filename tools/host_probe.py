"""Host time per round / epoch boundary in the bench loop (is the host ahead
of the device?). torchrun-aware: one partition per rank as bench.py."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2201_02791_b200 as kb

world, rank, local = bench.dist_setup()
graph, split, pset, mc, tc = bench.build_inputs(world, bench.BATCH)
tr = kb.Trainer(pset, graph, mc, tc)
tr.use_graphs = True

def step():
    if tr.round_in_epoch == 0 or tr.round_in_epoch >= tr.rounds:
        t0 = time.perf_counter(); tr.begin_epoch(); be.append(time.perf_counter() - t0)
    t0 = time.perf_counter(); tr.run_round(); rr.append(time.perf_counter() - t0)

be, rr = [], []
for _ in range(8):
    step()
tr.prepare(); torch.cuda.synchronize()
be.clear(); rr.clear()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if tr.dist:
    torch.distributed.barrier()
torch.cuda.synchronize()
t0 = time.perf_counter(); e0.record()
for _ in range(60):
    step()
t_host = time.perf_counter() - t0
e1.record(); torch.cuda.synchronize()
t_all = time.perf_counter() - t0
from paper_2201_02791_b200 import sampler as smp
if rank == 0:
    nt = getattr(smp, "next_times", [])[-len(be):]
    print(f"   ready-wait host {1e3*sum(nt)/max(len(nt),1):.3f} ms per epoch", flush=True)
    print(f"world {world} rounds/epoch {tr.rounds}: host enqueue {t_host*1e3/60:.3f} ms/round, device {e0.elapsed_time(e1)/60:.3f} ms/round, "
          f"begin_epoch host {1e3*sum(be)/max(len(be),1):.3f} ms (x{len(be)}), run_round host {1e3*sum(rr)/len(rr):.3f} ms", flush=True)
