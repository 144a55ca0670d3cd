"""Config 3: filtered link-prediction eval of the
FB15k-237-shaped test split (15,117 triples -> 30,234 rank records x 14,541
candidates, d = 100). Times encode_all_entities + evaluate and prints the
per-kernel breakdown. python tools/eval_bench.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2201_02791_b200 as kb
from paper_2201_02791_b200 import _lib

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
graph, split = kb.generate_synthetic(14541, 237, 272115 / 14541, seed=0)
mc = kb.ModelConfig(2, [100, 100, 100], 2, 237, 1, mode="embedding")
params = kb.init_params(mc, np.random.default_rng(0), num_entities=graph.num_entities)
kb.evaluate(params, mc, graph, split, which="test")   # warm-up (allocations, known keys)
torch.cuda.synchronize()
walls = []
for _ in range(reps):
    t0 = time.perf_counter()
    res = kb.evaluate(params, mc, graph, split, which="test")
    torch.cuda.synchronize()
    walls.append(time.perf_counter() - t0)
bd, _ = _lib.kernel_breakdown(kb.evaluate, params, mc, graph, split, which="test")
nrec = len(res.records)
flop = 2.0 * nrec * graph.num_entities * mc.dims[-1]
print(f"records {nrec}, wall min {min(walls) * 1e3:.2f} ms, MRR {res.mrr:.6f}, hits {res.hits}")
tot = sum(ms for _, ms in bd.values())
for k, (n, ms) in sorted(bd.items(), key=lambda x: -x[1][1]):
    extra = f"  {flop / (ms * 1e-3) / 1e12:7.1f} TFLOP/s (2*rec*N*d)" if k == "k_rank_tiles" else ""
    print(f"{k:22s} {n:4d} {ms:9.3f} ms{extra}")
print(f"kernel total {tot:.3f} ms")
