"""Multi-GPU consistency check (run under torchrun): P = world partitions
trained with NCCL all-gather + fused tree-mean Adam must give params bitwise
identical to the single-process run over the same P partitions (identical
tree arithmetic). Rank 0 prints one JSON line."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2201_02791_b200 as kb


def digest(params):
    h = hashlib.sha256()
    for b in params.dense_blocks():
        h.update(np.ascontiguousarray(b).tobytes())
    h.update(np.ascontiguousarray(params.entity_embed).tobytes())
    return h.hexdigest()


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    n_ent = int(os.environ.get("DC_ENTITIES", "3000"))
    graph, split = kb.generate_synthetic(n_ent, 30, 8.0, seed=1)
    P = world
    pset = kb.neighborhood_expand(kb.vertex_cut_partition(graph, P, seed=0), graph, 2)
    mc = kb.ModelConfig(2, [32, 32, 32], 2, graph.num_relations, 1, mode="embedding")
    tc = kb.TrainConfig(epochs=2, batch_size=4096, seed=3)
    p0 = kb.init_params(mc, np.random.default_rng(3), num_entities=graph.num_entities)
    out = {}
    if rank == 0:
        single, rep1 = kb.train(pset, graph, mc, tc, initial_params=p0)
        out["single"] = digest(single)
        out["single_loss"] = rep1.loss_curve
    torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    multi, rep = kb.train(pset, graph, mc, tc, initial_params=p0)
    if rank == 0:
        out["multi"] = digest(multi)
        out["multi_loss"] = rep.loss_curve
        out["bitwise_equal"] = out["single"] == out["multi"]
        out["world"] = world
        print(json.dumps(out), flush=True)
    torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
