"""Filtered link-prediction evaluation on the GPU (drop-in for
ref:evaluate.py): full-graph encode, all-entity DistMult scoring with the
filter-and-rank fused into the scoring kernel, MRR / Hits@k."""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np

from . import _lib
from .errors import IntegrityError, KGError, ValidationError
from .model import MODE_EMBEDDING, ModelConfig, ModelParams
from .sampler import full_graph_view

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


def _device_encode_all64(params: ModelParams, config: ModelConfig, graph):
    """Full-graph encode in float64 on the device (kg_encode_full_f64): the
    evaluation's embeddings carry the reference's precision, so ranks among
    near-tied candidates follow the reference (ref:evaluate.py:107-122).
    Returns (H float64 tensor (N, d_out), view)."""
    import ctypes
    import torch
    view = full_graph_view(graph)
    dev = view.device
    if config.mode == MODE_EMBEDDING:
        if params.entity_embed is None:
            raise ValidationError("embedding mode requires an entity table")
        table = params.entity_embed
    else:
        if graph.features is None:
            raise ValidationError("feature mode requires graph features")
        table = graph.features
    table = np.asarray(table)
    if table.ndim != 2 or table.shape[1] != config.dims[0]:
        raise ValidationError(f"input width != d_in {config.dims[0]}")
    f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
    L, B = config.num_layers, config.num_bases
    bases = [f64(b) for b in params.bases]
    coeffs = [f64(c) for c in params.coeffs]
    inp = f64(table[: graph.num_entities])
    N = graph.num_entities
    out = torch.empty((N, config.dims[-1]), dtype=torch.float64, device=dev)
    lib = _lib.require_cuda()
    csr = view.csr()
    ws = torch.empty(lib.kg_encode_full_f64_workspace_bytes(N, csr.e, csr.chunk, B, max(config.dims)),
                     dtype=torch.uint8, device=dev)
    dims = (ctypes.c_int32 * (L + 1))(*config.dims)
    pb = (ctypes.c_void_p * L)(*[b.data_ptr() for b in bases])
    pc = (ctypes.c_void_p * L)(*[c.data_ptr() for c in coeffs])
    _lib.call("kg_encode_full_f64", ctypes.byref(csr), view.d_ref_src.data_ptr(), view.d_ref_rel.data_ptr(),
              view.d_msg_cnt.data_ptr(), L, dims, B, pb, pc, inp.data_ptr(), out.data_ptr(), ws.data_ptr(),
              ws.numel(), _lib.stream_handle())
    return out, view


def encode_all_entities(params: ModelParams, config: ModelConfig, graph) -> np.ndarray:
    """Embeddings of every entity from message passing over the whole graph
    (ref:evaluate.py:107-122), computed in float64 on the device; rows align
    with entity ids."""
    H, _ = _device_encode_all64(params, config, graph)
    return H.cpu().numpy()


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
    H64, view = _device_encode_all64(params, config, graph)
    H = H64.float()
    dev = view.device
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt)).to(dev)
    dec = t(params.decoder, np.float32)
    dq, dptr, dc, dt_ = t(q, np.int32), t(ptr, np.int64), t(flat, np.int32), t(tpos, np.int32)
    ranks = torch.empty(nq, dtype=torch.float64, device=dev)
    ncand = torch.empty(nq, dtype=torch.int32, device=dev)
    _lib.call("kg_eval_candidates", H.data_ptr(), config.dims[-1], dec.data_ptr(), dq.data_ptr(), nq,
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
    filtered by train+valid+test (ref:evaluate.py:136-218), from the float64
    full-graph encode. impl 0: tensor-core scores (3xTF32, d <= 128) with
    every candidate inside the per-row error band around the true score
    decided in float64 (ranks follow the reference's float64 scores);
    impl 1: CUDA-core tiles, an exact sequential fmaf chain per fp32 score."""
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
    H64, view = _device_encode_all64(params, config, graph)
    H = H64.float()
    dev = view.device
    dec64 = torch.as_tensor(np.ascontiguousarray(params.decoder, dtype=np.float64)).to(dev)
    dec = dec64.float()
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
    _lib.call("kg_eval_filtered", H.data_ptr(), config.dims[-1], N, dec.data_ptr(), R, dq.data_ptr(), nq,
              tkeys.data_ptr(), ntk, hkeys.data_ptr(), nhk, _POLICY[tie_policy], chunk, impl, pairs,
              ranks.data_ptr(), ncand.data_ptr(), overflow.data_ptr(), H64.data_ptr() if impl == 0 else None,
              dec64.data_ptr() if impl == 0 else None, ws.data_ptr(), ws.numel(), _lib.stream_handle())
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
