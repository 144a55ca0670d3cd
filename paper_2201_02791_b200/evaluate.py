"""Filtered link-prediction evaluation on the GPU (drop-in for
ref:evaluate.py): full-graph encode, all-entity DistMult scoring with the
filter-and-rank fused into the scoring kernel, MRR / Hits@k."""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np

from . import _lib
from .errors import IntegrityError, KGError, ValidationError
from .model import MODE_EMBEDDING, DeviceModel, ModelConfig, ModelParams, ViewBuffers, device_forward
from .sampler import closure_device, full_graph_view

TIE_MEAN = "mean"
TIE_OPTIMISTIC = "optimistic"
TIE_PESSIMISTIC = "pessimistic"
_POLICY = {TIE_MEAN: 0, TIE_OPTIMISTIC: 1, TIE_PESSIMISTIC: 2}

SIDE_TAIL = "tail"
SIDE_HEAD = "head"
HITS_KS = (1, 3, 10)


class RankRecord(NamedTuple):
    head: int
    rel: int
    tail: int
    corrupted_side: str
    rank: float
    num_candidates: int


@dataclass
class EvalResult:
    mrr: float
    hits: dict
    records: list

    def format_summary(self) -> str:
        cols = " ".join(f"hits@{k}={self.hits[k]:.4f}" for k in sorted(self.hits))
        return f"records={len(self.records)} mrr={self.mrr:.4f} {cols}"


def _rank(num_greater: int, num_ties: int, tie_policy: str) -> float:
    if tie_policy == TIE_MEAN:
        return 1.0 + num_greater + num_ties / 2.0
    if tie_policy == TIE_OPTIMISTIC:
        return 1.0 + num_greater
    if tie_policy == TIE_PESSIMISTIC:
        return 1.0 + num_greater + num_ties
    raise ValidationError(f"unknown tie policy {tie_policy!r}")


def rank_triplet(candidate_scores: np.ndarray, true_index: int, tie_policy: str = TIE_MEAN) -> float:
    """Rank of the true entity among candidate scores (ref:evaluate.py:77-90)."""
    scores = np.asarray(candidate_scores, dtype=np.float64)
    if not 0 <= true_index < len(scores):
        raise IntegrityError("true entity missing from candidate list")
    ts = scores[true_index]
    return _rank(int((scores > ts).sum()), int((scores == ts).sum()) - 1, tie_policy)


def filtered_candidates(test_triplet, side: str, all_known_triples, num_entities: int) -> np.ndarray:
    """Entities whose substitution on `side` is not a known triple, plus the
    true entity (ref:evaluate.py:54-74); host helper for small checks."""
    h, r, t = (int(x) for x in test_triplet)
    known = all_known_triples
    if not isinstance(known, set):
        known = {tuple(row) for row in np.asarray(known).reshape(-1, 3).tolist()}
    if side not in (SIDE_TAIL, SIDE_HEAD):
        raise ValidationError(f"unknown side {side!r}")
    out = [e for e in range(num_entities)
           if (e == (t if side == SIDE_TAIL else h))
           or (((h, r, e) if side == SIDE_TAIL else (e, r, t)) not in known)]
    return np.array(out, dtype=np.int64)


def _device_encode_all(params: ModelParams, config: ModelConfig, graph):
    """Full-graph encode on the device; returns (H tensor (N, d_out), view)."""
    import torch
    view = full_graph_view(graph)
    dev = view.device
    N = graph.num_entities
    if config.mode == MODE_EMBEDDING:
        if params.entity_embed is None:
            raise ValidationError("embedding mode requires an entity table")
        table = params.entity_embed
    else:
        if graph.features is None:
            raise ValidationError("feature mode requires graph features")
        table = graph.features
    seeds = torch.arange(N, dtype=torch.int32, device=dev)
    cg = closure_device(view, config.num_layers, seed_ids=seeds)
    model = DeviceModel.from_params(config, params, dev)
    rows = torch.as_tensor(np.ascontiguousarray(table, dtype=np.float32)).to(dev)
    bufs = ViewBuffers(config, view, 1, input_rows=rows)
    bufs.order.copy_(cg.d_order)
    bufs.pos.copy_(cg.d_pos)
    bufs.counts.copy_(cg.d_counts)
    device_forward(model, bufs)
    return bufs.H[-1], model, view


def encode_all_entities(params: ModelParams, config: ModelConfig, graph) -> np.ndarray:
    """Embeddings of every entity from message passing over the whole graph
    (ref:evaluate.py:107-122); rows align with entity ids."""
    H, _, _ = _device_encode_all(params, config, graph)
    return H.double().cpu().numpy()


def _known_keys(triples: np.ndarray, col_a: int, col_c: int, N: int, R: int, dev):
    import torch
    lib = _lib.require_cuda()
    k = len(triples)
    d = torch.as_tensor(np.ascontiguousarray(triples, dtype=np.int32)).to(dev)
    keys = torch.empty(max(k, 1), dtype=torch.int64, device=dev)
    n = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(lib.kg_known_keys_workspace_bytes(max(k, 1)), dtype=torch.uint8, device=dev)
    _lib.call("kg_known_keys", d.data_ptr(), k, col_a, col_c, N, R, keys.data_ptr(), n.data_ptr(), ws.data_ptr(),
              ws.numel(), _lib.stream_handle())
    return keys, int(n.item())


def _result(records: list) -> EvalResult:
    ranks = np.array([rec.rank for rec in records], dtype=np.float64)
    return EvalResult(mrr=float((1.0 / ranks).mean()), hits={k: float((ranks <= k).mean()) for k in HITS_KS},
                      records=records)


def _known_pair_bound(tkeys, ntk: int, hkeys, nhk: int, dq, N: int, R: int) -> int:
    """Known candidates the tensor-core ranker scores separately: for every
    query and side, the distinct known triples sharing its (anchor, relation)
    (an upper bound: the true entity is included). Device searchsorted over
    the sorted unique keys."""
    import torch
    q = dq.to(torch.int64)
    total = 0
    for keys, n, a in ((tkeys, ntk, 0), (hkeys, nhk, 2)):
        if n == 0:
            continue
        base = (q[:, a] * R + q[:, 1]) * N
        k = keys[:n]
        total += int((torch.searchsorted(k, base + N) - torch.searchsorted(k, base)).sum().item())
    return max(total, 1)


def _evaluate_candidates(params, config, graph, q, candidates: dict, tie_policy: str) -> EvalResult:
    """Given-candidates protocol (ref:evaluate.py:168-180): the tail of every
    query against its candidate list (the true tail appended when absent)."""
    import torch
    nq = len(q)
    lists, tpos = [], np.empty(nq, dtype=np.int32)
    for i, t in enumerate(np.asarray(q)[:, 2].tolist()):
        cand = np.asarray(candidates.get(i, []), dtype=np.int64)
        if len(cand) == 0:
            raise ValidationError(f"no candidates for test index {i}")
        pos = np.flatnonzero(cand == t)
        if len(pos) == 0:
            cand = np.concatenate([cand, [t]])
            pos = [len(cand) - 1]
        lists.append(cand)
        tpos[i] = int(pos[0])
    ptr = np.zeros(nq + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(c) for c in lists])
    flat = np.concatenate(lists)
    if flat.min() < 0 or flat.max() >= graph.num_entities:
        raise IntegrityError("candidate entity id out of range")
    H, model, view = _device_encode_all(params, config, graph)
    dev = view.device
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt)).to(dev)
    dq, dptr, dc, dt_ = t(q, np.int32), t(ptr, np.int64), t(flat, np.int32), t(tpos, np.int32)
    ranks = torch.empty(nq, dtype=torch.float64, device=dev)
    ncand = torch.empty(nq, dtype=torch.int32, device=dev)
    _lib.call("kg_eval_candidates", H.data_ptr(), config.dims[-1], model.decoder_ptr(), dq.data_ptr(), nq,
              dptr.data_ptr(), dc.data_ptr(), dt_.data_ptr(), _POLICY[tie_policy], ranks.data_ptr(),
              ncand.data_ptr(), _lib.stream_handle())
    r, c = ranks.cpu().numpy(), ncand.cpu().numpy()
    rows = np.asarray(q, dtype=np.int64)
    records = list(map(RankRecord, rows[:, 0].tolist(), rows[:, 1].tolist(), rows[:, 2].tolist(),
                       [SIDE_TAIL] * nq, r.tolist(), c.tolist()))
    return EvalResult(mrr=float((1.0 / r).mean()), hits={k: float((r <= k).mean()) for k in HITS_KS},
                      records=records)


def evaluate(params: ModelParams, config: ModelConfig, graph, split, which: str = "test",
             protocol: str = "filtered", candidates: Optional[dict] = None, tie_policy: str = TIE_MEAN,
             chunk: int = 512, impl: int = 0) -> EvalResult:
    """Rank every triple of the split against all entities on both sides,
    filtered by train+valid+test (ref:evaluate.py:136-218). impl 0: tensor-core
    scores (d <= 128); 1: exact CUDA-core fmaf chains."""
    import torch
    if which not in ("valid", "test"):
        raise ValidationError("which must be valid or test")
    q = split.valid if which == "valid" else split.test
    if len(q) == 0:
        raise ValidationError(f"{which} split is empty")
    if protocol not in ("filtered", "candidates"):
        raise ValidationError(f"unknown protocol {protocol!r}")
    if protocol == "candidates" and candidates is None:
        raise ValidationError("candidates protocol requires a candidate map")
    if tie_policy not in _POLICY:
        raise ValidationError(f"unknown tie policy {tie_policy!r}")
    if protocol == "candidates":
        return _evaluate_candidates(params, config, graph, q, candidates, tie_policy)
    H, model, view = _device_encode_all(params, config, graph)
    dev = view.device
    N, R = graph.num_entities, graph.num_relations
    known = split.all_triples()
    tkeys, ntk = _known_keys(known, 0, 2, N, R, dev)
    hkeys, nhk = _known_keys(known, 2, 0, N, R, dev)
    nq = len(q)
    dq = torch.as_tensor(np.ascontiguousarray(q, dtype=np.int32)).to(dev)
    ranks = torch.empty(2 * nq, dtype=torch.float64, device=dev)
    ncand = torch.empty(2 * nq, dtype=torch.int32, device=dev)
    lib = _lib.require_cuda()
    pairs = _known_pair_bound(tkeys, ntk, hkeys, nhk, dq, N, R)
    ws = torch.empty(lib.kg_eval_workspace_bytes(nq, N, config.dims[-1], pairs), dtype=torch.uint8, device=dev)
    overflow = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("kg_eval_filtered", H.data_ptr(), config.dims[-1], N, model.decoder_ptr(), R, dq.data_ptr(), nq,
              tkeys.data_ptr(), ntk, hkeys.data_ptr(), nhk, _POLICY[tie_policy], chunk, impl, pairs,
              ranks.data_ptr(), ncand.data_ptr(), overflow.data_ptr(), ws.data_ptr(), ws.numel(),
              _lib.stream_handle())
    if int(overflow.item()):
        raise KGError("internal: known-candidate pair bound exceeded")
    r = ranks.cpu().numpy()
    c = ncand.cpu().numpy()
    # record order of the reference: per chunk, its tail records then its head records
    idx, sides = [], []
    for a in range(0, nq, chunk):
        blk = np.arange(a, min(a + chunk, nq))
        idx += [blk, blk]
        sides += [SIDE_TAIL] * len(blk) + [SIDE_HEAD] * len(blk)
    rows = np.asarray(q, dtype=np.int64)[np.concatenate(idx)]
    records = list(map(RankRecord, rows[:, 0].tolist(), rows[:, 1].tolist(), rows[:, 2].tolist(), sides,
                       r.tolist(), c.tolist()))
    return EvalResult(mrr=float((1.0 / r).mean()), hits={k: float((r <= k).mean()) for k in HITS_KS},
                      records=records)


# Reference module-level names that live in io.py here (ref:evaluate.py:232-253); resolved
# lazily so `from <pkg>.evaluate import X` works as with the reference.
_IO_NAMES = ('read_candidates', 'write_results')


def __getattr__(name):
    if name in _IO_NAMES:
        from . import io
        return getattr(io, name)
    raise AttributeError(name)
