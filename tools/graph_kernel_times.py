"""In-graph per-kernel durations: for each library kernel name the round's
graphs are re-captured with CUDA events around that kernel only (external
event nodes), replayed, and the event time read back. Diagnostic; the
events themselves add a little per-launch overhead.
python tools/graph_kernel_times.py [rounds]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2201_02791_b200 as kb
from paper_2201_02791_b200 import _lib

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 8
graph, split = kb.generate_synthetic(14541, 237, 272115 / 14541, seed=0)
pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, 1, seed=0), graph, 2)
mc = kb.ModelConfig(2, [100, 100, 100], 2, 237, 1, mode="embedding")
tc = kb.TrainConfig(batch_size=65536, seed=0)
tr = kb.Trainer(pset, graph, mc, tc)
tr.use_graphs = True
lib = _lib.require_cuda()

# discover the kernel names of one eager round
tr.use_graphs = False


def step():
    if tr.round_in_epoch == 0 or tr.round_in_epoch >= tr.rounds:
        tr.begin_epoch()
    tr.run_round()


step()
names, _ = _lib.kernel_breakdown(step)
tr.use_graphs = True
res = []
for name in sorted(names):
    tr._graphs = {}
    tr._timer_handles = {}
    tr._graph_pool = None
    torch.cuda.synchronize()
    tr._eager_rounds = 2
    tr.timer_prefix = name
    tot_ms, tot_n = 0.0, 0
    for r in range(rounds):
        step()
        if r >= 2 and tr.last_timer_handle is not None:
            ms, n = ctypes.c_double(), ctypes.c_int64()
            lib.kg_kernel_timer_read(tr.last_timer_handle, ctypes.byref(ms), ctypes.byref(n))
            tot_ms += ms.value
            tot_n += n.value
    per_round = tot_ms / max(rounds - 2, 1) * 1000.0
    res.append((per_round, name, tot_n / max(rounds - 2, 1)))
torch.cuda.synchronize()
res.sort(reverse=True)
total = sum(r[0] for r in res)
print(f"sum of in-graph kernel time per round: {total:.1f} us (compute graph only; side streams overlap)")
for us, name, n in res:
    print(f"{name:28s} {n:5.1f}/round {us:8.1f} us/round {us / max(n, 1e-9):7.1f} us/launch")
