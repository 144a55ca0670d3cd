"""Graph-replay time of each phase of one training round, captured separately
(closure, forward, loss groups, loss compute, backward, update) on the FB-shape
bench workload. Diagnostic only (phases replayed in isolation on warm caches).
python tools/phase_times.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2201_02791_b200 as kb
from paper_2201_02791_b200.model import device_backward, device_forward, device_loss

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
graph, split = kb.generate_synthetic(14541, 237, 272115 / 14541, seed=0)
pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, 1, seed=0), graph, 2)
mc = kb.ModelConfig(2, [100, 100, 100], 2, 237, 1, mode="embedding")
tc = kb.TrainConfig(batch_size=65536, seed=0)
os.environ["KG_CUDA_GRAPHS"] = "0"
tr = kb.Trainer(pset, graph, mc, tc)
tr.use_graphs = False
tr.begin_epoch() if hasattr(tr, "begin_epoch") else None
for _ in range(3):
    tr.run_round()
torch.cuda.synchronize()
w = tr.workers[0]
gslot = tr.grads_local[0]
sd = tr.start_dev[0:1]
side = tr._loss_stream
phases = {
    "closure": lambda: w.closure(sd),
    "forward": lambda: device_forward(tr.model, w.bufs),
    "loss_groups": lambda: device_loss(tr.model, w.bufs, w.stream, 0, w.b, gslot, tr.loss_scratch[0:1],
                                       start_dev=sd, part="groups"),
    "loss_compute": lambda: device_loss(tr.model, w.bufs, w.stream, 0, w.b, gslot, tr.loss_scratch[0:1],
                                        start_dev=sd, part="compute"),
    "backward_serial": lambda: device_backward(tr.model, w.bufs, gslot, input_grad=w.emb),
    "backward_side": lambda: device_backward(tr.model, w.bufs, gslot, input_grad=w.emb, side=side),
    "update": tr._update_body,
    "compute_body": tr._compute_body,
}
pool = torch.cuda.graph_pool_handle()
res = {}
saved = (tr.round_dev.clone(), tr.step_dev.clone())
for name, fn in phases.items():
    tr.round_dev.copy_(saved[0])
    tr.step_dev.copy_(saved[1])
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        g.capture_begin()
        fn()
        g.capture_end()
    torch.cuda.current_stream().wait_stream(cs)
    for _ in range(3):
        g.replay()
        tr.round_dev.copy_(saved[0])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
        if name == "update":
            tr.round_dev.copy_(saved[0])
    e1.record()
    torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / reps * 1000.0
    tr.round_dev.copy_(saved[0])
for k, v in res.items():
    print(f"{k:18s} {v:8.1f} us")
