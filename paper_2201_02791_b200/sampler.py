"""Partition-local sampling on the GPU: view build, constraint negatives,
edge mini-batch stream and layered closures (drop-in for ref:sampler.py).

Public functions keep the reference's names, signatures and numpy-in /
numpy-out behaviour; the state they need for training stays resident in HBM
(`PartitionView` owns the device CSR/CSC, the positive-key table and the
local-id map). numpy Generators passed in are advanced exactly as the
reference's calls would advance them, so host code that keeps drawing from
the same Generator sees the same stream.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import os

import numpy as np

from . import _lib
from .errors import IntegrityError, SamplingError, ValidationError
from .partition import Partition

MAX_RESAMPLE_ROUNDS = 100
CHUNK_EDGES = int(os.environ.get("KG_CHUNK_EDGES", "64"))   # messages per warp work chunk (hub rows are split; <= 64)


def _torch():
    import torch
    return torch


def _dev_i32(a, device):
    torch = _torch()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32)).to(device, non_blocking=False)


def _bits(x: int) -> int:
    return max(int(x), 0).bit_length()


# ---------------------------------------------------------------------------
# Partition view (ref:sampler.py:32-134)
# ---------------------------------------------------------------------------

class PartitionView:
    """Local-id view of one partition, resident on the GPU.

    Device state: d_edges (m,3) local triples (core first), the destination
    CSR and source CSR of the 2m message edges with fp32 1/c norms, the
    relation-grouped CSC positions, the sorted unique positive keys.
    The reference's numpy fields (local_ids, edges, msg_indptr, msg_src,
    msg_rel, msg_norm, positive_keys, pool) are exposed as properties that
    copy to the host on first access.
    """

    def __init__(self, partition_id, num_relations, hop_count, num_core, pool_size, device):
        self.partition_id = int(partition_id)
        self.num_relations = int(num_relations)
        self.hop_count = int(hop_count)
        self.num_core = int(num_core)
        self.pool_size = int(pool_size)
        self.device = device
        self._host = {}

    # -- shape -------------------------------------------------------------
    @property
    def num_vertices(self) -> int:
        return self.n

    @property
    def self_loop_rel(self) -> int:
        return 2 * self.num_relations

    @property
    def num_messages(self) -> int:
        return 2 * self.m

    # -- reference numpy fields (host copies) ------------------------------
    def _cached(self, key, fn):
        if key not in self._host:
            self._host[key] = fn()
        return self._host[key]

    @property
    def local_ids(self) -> np.ndarray:
        return self._cached("local_ids", lambda: self.d_local_ids.cpu().numpy().astype(np.int64))

    @property
    def edges(self) -> np.ndarray:
        return self._cached("edges", lambda: self.d_edges.cpu().numpy().astype(np.int64).reshape(-1, 3))

    @property
    def core_edges(self) -> np.ndarray:
        return self.edges[: self.num_core]

    @property
    def pool(self) -> np.ndarray:
        return np.arange(self.pool_size, dtype=np.int64)

    @property
    def msg_indptr(self) -> np.ndarray:
        return self._cached("indptr", lambda: self.d_indptr.cpu().numpy().astype(np.int64))

    @property
    def msg_src(self) -> np.ndarray:
        return self._cached("msg_src", lambda: self.d_ref_src.cpu().numpy().astype(np.int64))

    @property
    def msg_rel(self) -> np.ndarray:
        return self._cached("msg_rel", lambda: self.d_ref_rel.cpu().numpy().astype(np.int64))

    @property
    def msg_norm(self) -> np.ndarray:
        return self._cached("msg_norm", lambda: 1.0 / self.d_msg_cnt.cpu().numpy().astype(np.float64))

    @property
    def positive_keys(self) -> np.ndarray:
        return self._cached("keys", lambda: self.d_pos_keys[: self.n_keys].cpu().numpy())

    def triple_keys(self, triples: np.ndarray) -> np.ndarray:
        n = self.num_vertices
        return (triples[:, 0] * self.num_relations + triples[:, 1]) * n + triples[:, 2]

    def is_positive(self, triples: np.ndarray) -> np.ndarray:
        """Membership in the local positive set, on the GPU (ref:sampler.py:60-70)."""
        torch = _torch()
        triples = np.asarray(triples).reshape(-1, 3)
        k = len(triples)
        if k == 0:
            return np.zeros(0, dtype=bool)
        d_t = _dev_i32(triples, self.device)
        out = torch.empty(k, dtype=torch.uint8, device=self.device)
        _lib.call("kg_is_positive", d_t.data_ptr(), k, self.n, self.num_relations,
                  self.d_pos_keys.data_ptr(), self.d_n_keys.data_ptr(), out.data_ptr(),
                  _lib.stream_handle())
        return out.cpu().numpy().astype(bool)

    # -- C ABI descriptor -----------------------------------------------------
    def csr(self) -> "_lib.KgGraphCsr":
        return self._csr


def _device():
    torch = _torch()
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def build_view(partition: Partition, num_entities: int, num_relations: int) -> PartitionView:
    """GPU build of the local-id view with bidirectional message edges and
    per-(destination, relation) mean normalisation (ref:sampler.py:73-118)."""
    torch = _torch()
    dev = _device()
    st = _lib.stream_handle()
    lib = _lib.require_cuda()
    core = np.ascontiguousarray(partition.core, dtype=np.int32)
    sup = np.ascontiguousarray(partition.support, dtype=np.int32)
    m_core, m_sup = len(core), len(sup)
    m = m_core + m_sup
    N = int(num_entities)
    edges_g = torch.as_tensor(np.concatenate([core, sup]).reshape(-1, 3)).to(dev)
    ws_bytes = lib.kg_view_workspace_bytes(max(m, 1), N)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    g2l = torch.empty(N, dtype=torch.int32, device=dev)
    if partition._local is not None:
        # explicit local order (e.g. full_graph_view's identity ids)
        local = torch.as_tensor(np.ascontiguousarray(partition._local, dtype=np.int32)).to(dev)
        g2l.fill_(-1)
        g2l[local.long()] = torch.arange(len(local), dtype=torch.int32, device=dev)
        n_local = len(local)
    else:
        local = torch.empty(N, dtype=torch.int32, device=dev)
        n_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.call("kg_view_local_ids", edges_g.data_ptr(), m_core,
                  edges_g.data_ptr() + m_core * 3 * 4, m_sup, N, local.data_ptr(), g2l.data_ptr(),
                  n_dev.data_ptr(), ws.data_ptr(), ws_bytes, st)
        n_local = int(n_dev.item())
        local = local[:n_local]
    if n_local == 0:
        raise ValidationError("partition has no vertices")
    v = PartitionView(partition.id, num_relations, partition.hop_count, m_core, partition.pool_size, dev)
    v.n, v.m = n_local, m
    e = 2 * m
    i32 = dict(dtype=torch.int32, device=dev)
    v.d_local_ids = local
    v.d_edges = torch.empty((m, 3), **i32)
    v.d_ref_src = torch.empty(e, **i32)
    v.d_ref_rel = torch.empty(e, **i32)
    v.d_msg_cnt = torch.empty(e, **i32)
    v.d_indptr = torch.empty(n_local + 1, **i32)
    v.d_src = torch.empty(e, **i32)
    v.d_rel = torch.empty(e, **i32)
    v.d_norm = torch.empty(e, dtype=torch.float32, device=dev)
    v.d_c_indptr = torch.empty(n_local + 1, **i32)
    v.d_c_dst = torch.empty(e, **i32)
    v.d_c_rel = torch.empty(e, **i32)
    v.d_c_norm = torch.empty(e, dtype=torch.float32, device=dev)
    v.d_rel_perm = torch.empty(e, **i32)
    v.d_rel_ptr = torch.empty(2 * num_relations + 1, **i32)
    v.d_pos_keys = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
    v.d_n_keys = torch.zeros(1, **i32)
    C = CHUNK_EDGES
    cap_chunks, cap_split_chunks, cap_split_rows = n_local + e // C + 1, 2 * e // C + 1, e // C + 1
    for pre in ("ck", "cc"):
        setattr(v, f"d_{pre}_ptr", torch.empty(n_local + 1, **i32))
        setattr(v, f"d_{pre}_row", torch.empty(cap_chunks, **i32))
        setattr(v, f"d_{pre}_slot", torch.empty(cap_chunks, **i32))
        setattr(v, f"d_{pre}_split", torch.empty(cap_split_rows, **i32))
        setattr(v, f"d_{pre}_counts", torch.zeros(4, **i32))
        setattr(v, f"d_{pre}_desc", torch.empty(4 * cap_chunks, **i32))
    c = _lib.KgGraphCsr()
    c.n, c.R, c.e, c.chunk = n_local, num_relations, e, C
    for f in ("indptr", "src", "rel", "norm", "c_indptr", "c_dst", "c_rel", "c_norm", "rel_perm", "rel_ptr",
              "ck_ptr", "ck_row", "ck_slot", "ck_split", "ck_counts",
              "cc_ptr", "cc_row", "cc_slot", "cc_split", "cc_counts", "ck_desc", "cc_desc"):
        setattr(c, f, getattr(v, "d_" + f).data_ptr())
    v._csr = c
    ws_bytes2 = lib.kg_view_workspace_bytes(max(m, 1), n_local)
    if ws_bytes2 > ws_bytes:
        ws = torch.empty(ws_bytes2, dtype=torch.uint8, device=dev)
        ws_bytes = ws_bytes2
    import ctypes
    _lib.call("kg_view_build", edges_g.data_ptr(), m, g2l.data_ptr(), v.d_edges.data_ptr(),
              v.d_ref_src.data_ptr(), v.d_ref_rel.data_ptr(), v.d_msg_cnt.data_ptr(), ctypes.byref(c),
              v.d_pos_keys.data_ptr(), v.d_n_keys.data_ptr(), ws.data_ptr(), ws_bytes, st)
    v.n_keys = int(v.d_n_keys.item())
    if m and int(v.d_edges.min().item()) < 0:
        raise IntegrityError("partition edge references a vertex missing from its vertex list")
    return v


def full_graph_view(graph) -> PartitionView:
    """Whole graph as one partition with identity ids (ref:sampler.py:121-134)."""
    whole = Partition(id=0, core=graph.triples, support=np.zeros((0, 3), dtype=np.int64),
                      core_vertices=np.arange(graph.num_entities, dtype=np.int64),
                      replicated_vertices=np.zeros(0, dtype=np.int64),
                      support_vertices=np.zeros(0, dtype=np.int64), hop_count=0,
                      core_edge_ids=np.arange(graph.num_edges, dtype=np.int64))
    whole._local = np.arange(graph.num_entities, dtype=np.int64)
    return build_view(whole, graph.num_entities, graph.num_relations)


# ---------------------------------------------------------------------------
# Negative sampling (ref:sampler.py:144-182)
# ---------------------------------------------------------------------------

def _round_window(k: int, pool: int) -> int:
    thr = ((1 << 32) - pool) % pool
    p = thr / float(1 << 32)
    mean = k * p
    return int(k + 2 * mean + 8 * math.sqrt(mean + 1.0) + 64)


def _neg_round(view, s, neg, col, pend_in, k_in, k_max, g_dev, W, pend_out, k_out, consumed, ws):
    lib = _lib.require_cuda()
    buf = ws.get("neg_round", lib.kg_neg_round_workspace_bytes(W))
    _lib.call("kg_neg_round", neg.data_ptr(), col.data_ptr(), view.d_edges.data_ptr(), s, pend_in.data_ptr(),
              k_in.data_ptr(), k_max, view.pool_size, view.n, view.num_relations, view.d_pos_keys.data_ptr(),
              view.d_n_keys.data_ptr(), g_dev.data_ptr(), W, pend_out.data_ptr(), k_out.data_ptr(),
              consumed.data_ptr(), buf.data_ptr(), buf.numel(), _lib.stream_handle())


def _neg_buffers(view, s, dev):
    torch = _torch()
    total = view.num_core * s
    return dict(neg=torch.empty((total, 3), dtype=torch.int32, device=dev),
                col=torch.empty(total, dtype=torch.int8, device=dev),
                pend=[torch.empty(total, dtype=torch.int32, device=dev) for _ in range(2)],
                k=[torch.zeros(1, dtype=torch.int32, device=dev) for _ in range(2)],
                consumed=torch.zeros(MAX_RESAMPLE_ROUNDS, dtype=torch.int64, device=dev))


def sample_negatives_device(view: PartitionView, s: int, g_dev, ws: Optional["_lib.Workspace"] = None,
                            bufs: Optional[dict] = None, async_rounds: int = 0):
    """Constraint negatives on the device from the device-resident PCG64
    state g_dev (advanced in place). With async_rounds > 0 only that many
    resampling rounds are enqueued, without any host synchronisation; the
    caller validates with `negatives_pending()`. Otherwise rounds run until
    every row is accepted (host-checked). Returns the (s*m, 3) tensor."""
    torch = _torch()
    if s < 0:
        raise ValidationError("negatives_per_positive must be >= 0")
    m = view.num_core
    dev = view.device
    if s == 0 or m == 0:
        return torch.zeros((0, 3), dtype=torch.int32, device=dev)
    if view.pool_size < 2:
        raise SamplingError("partition has fewer than 2 core vertices")
    ws = ws or _lib.Workspace(dev)
    b = bufs or _neg_buffers(view, s, dev)
    total = m * s
    st = _lib.stream_handle()
    _lib.call("kg_neg_init", view.d_edges.data_ptr(), m, s, g_dev.data_ptr(), b["neg"].data_ptr(), b["col"].data_ptr(),
              b["pend"][0].data_ptr(), st)
    b["k"][0].fill_(total)
    b["consumed"].zero_()
    W = _round_window(total, view.pool_size)
    cur = 0
    if async_rounds:
        for r in range(async_rounds):
            _neg_round(view, s, b["neg"], b["col"], b["pend"][cur], b["k"][cur], total, g_dev, W, b["pend"][1 - cur],
                       b["k"][1 - cur], b["consumed"][r:r + 1], ws)
            cur = 1 - cur
        b["cur"] = cur
        return b["neg"]
    k = total
    for r in range(MAX_RESAMPLE_ROUNDS):
        if k == 0:
            break
        while True:
            _neg_round(view, s, b["neg"], b["col"], b["pend"][cur], b["k"][cur], total, g_dev, W, b["pend"][1 - cur],
                       b["k"][1 - cur], b["consumed"][r:r + 1], ws)
            if int(b["consumed"][r].item()) >= 0:
                break
            W *= 2                      # window too small: state untouched, retry wider
        cur = 1 - cur
        k = int(b["k"][cur].item())
    b["cur"] = cur
    if k > 0:
        row = int(b["pend"][cur][0].item())
        e = view.core_edges[row // s]
        raise SamplingError(f"could not corrupt edge {tuple(int(x) for x in e)} after "
                            f"{MAX_RESAMPLE_ROUNDS} rounds")
    return b["neg"]


def sample_negatives(view: PartitionView, negatives_per_positive: int,
                     rng: np.random.Generator) -> np.ndarray:
    """Corrupt every core edge s times inside the partition's core-vertex pool
    (ref:sampler.py:144-182); returns (s*num_core, 3) int64 local triples and
    advances `rng` exactly as the reference's draws would."""
    g_dev = _lib.pcg_to_device(_lib.pcg_from_numpy(rng), view.device)
    neg = sample_negatives_device(view, negatives_per_positive, g_dev)
    _lib.pcg_to_numpy(_lib.pcg_from_device(g_dev), rng)
    return neg.cpu().numpy().astype(np.int64).reshape(-1, 3)


# ---------------------------------------------------------------------------
# Batching (ref:sampler.py:189-232)
# ---------------------------------------------------------------------------

def permutation_device(n: int, g_dev, device, ws: Optional["_lib.Workspace"] = None, check: bool = True,
                       out=None):
    """rng.permutation(n) on the GPU, bit-exact, from the device-resident
    PCG64 state g_dev (advanced in place). Returns (perm int32 tensor,
    consumed-count tensor; -1 there means the draw buffer was too small)."""
    torch = _torch()
    lib = _lib.require_cuda()
    st = _lib.stream_handle()
    ws = ws or _lib.Workspace(device)
    perm = out if out is not None else torch.empty(n, dtype=torch.int32, device=device)
    consumed = ws.get("perm_consumed", 8)[:8].view(torch.int64)
    if n <= 1:
        perm.zero_()
        consumed.zero_()
        return perm, consumed
    js = ws.get("perm_js", 4 * n)
    W = lib.kg_perm_draws_buffer_len(n)
    while True:
        U = ws.get("perm_U", 4 * W)
        snap = g_dev.clone() if check else None
        _lib.call("kg_perm_draws_buffered", n, g_dev.data_ptr(), U.data_ptr(), W, js.data_ptr(), consumed.data_ptr(),
                  st)
        if not check or int(consumed.item()) >= 0:
            break
        g_dev.copy_(snap)
        W = ((2 * W) // 1024 + 1) * 1024
    rb = lib.kg_perm_resolve_workspace_bytes(n)
    buf = ws.get("perm_resolve", rb)
    _lib.call("kg_perm_resolve", js.data_ptr(), n, perm.data_ptr(), buf.data_ptr(), buf.numel(), st)
    return perm, consumed


@dataclass
class EdgeMiniBatch:
    """One batch of labelled triples (ref:sampler.py:189-199). Device batches
    are windows of an epoch's shuffled stream: rows (start + q) mod total."""
    triples: np.ndarray
    labels: np.ndarray

    @property
    def seed_vertices(self) -> np.ndarray:
        return np.unique(self.triples[:, [0, 2]])

    def __len__(self) -> int:
        return len(self.triples)


@dataclass
class DeviceStream:
    """An epoch's shuffled triple stream in HBM (int32 (total,3) + fp32 labels)."""
    triples: object
    labels: object
    total: int

    def batch(self, start: int, size: int) -> EdgeMiniBatch:
        rows = (np.arange(start, start + size) % self.total)
        t = self.triples.cpu().numpy().astype(np.int64)[rows]
        y = self.labels.cpu().numpy().astype(np.float64)[rows]
        return EdgeMiniBatch(t, y)


def stream_device(pos, neg, g_dev, device, ws=None, check=True, out=None):
    """concat(pos, neg)[perm] with labels, perm = rng.permutation(total)."""
    torch = _torch()
    npos, nneg = int(pos.shape[0]), int(neg.shape[0])
    total = npos + nneg
    perm_out = out["perm"] if out is not None else None
    perm, consumed = permutation_device(total, g_dev, device, ws, check=check, out=perm_out)
    if out is not None:
        tri, lab = out["tri"], out["lab"]
    else:
        tri = torch.empty((total, 3), dtype=torch.int32, device=device)
        lab = torch.empty(total, dtype=torch.float32, device=device)
    if total:
        _lib.call("kg_stream_gather", pos.data_ptr(), npos, neg.data_ptr(), nneg, perm.data_ptr(),
                  tri.data_ptr(), lab.data_ptr(), _lib.stream_handle())
    return DeviceStream(tri, lab, total), consumed


def make_batches(positives: np.ndarray, negatives: np.ndarray, batch_size: int,
                 rng: np.random.Generator, num_batches: Optional[int] = None) -> list:
    """Jointly shuffle positives and negatives on the GPU and chunk into
    batches; with num_batches the stream wraps around (ref:sampler.py:202-232)."""
    if batch_size < 1:
        raise ValidationError("batch_size must be >= 1")
    pos = np.asarray(positives, dtype=np.int64).reshape(-1, 3)
    neg = np.asarray(negatives, dtype=np.int64).reshape(-1, 3)
    total = len(pos) + len(neg)
    if total == 0:
        return []
    dev = _device()
    g_dev = _lib.pcg_to_device(_lib.pcg_from_numpy(rng), dev)
    ds, _ = stream_device(_dev_i32(pos, dev).reshape(-1, 3), _dev_i32(neg, dev).reshape(-1, 3), g_dev, dev)
    _lib.pcg_to_numpy(_lib.pcg_from_device(g_dev), rng)
    tri = ds.triples.cpu().numpy().astype(np.int64)
    lab = ds.labels.cpu().numpy().astype(np.float64)
    if num_batches is None:
        return [EdgeMiniBatch(tri[a:a + batch_size], lab[a:a + batch_size])
                for a in range(0, total, batch_size)]
    out = []
    for i in range(num_batches):
        rows = np.arange(i * batch_size, (i + 1) * batch_size) % total
        out.append(EdgeMiniBatch(tri[rows], lab[rows]))
    return out


# ---------------------------------------------------------------------------
# Compute graph (ref:sampler.py:239-376)
# ---------------------------------------------------------------------------

@dataclass
class LayerBlock:
    """Message edges feeding one convolution, sorted by (relation, dst, src)
    (ref:sampler.py:239-262). dst/src are compute-graph positions; by_dst /
    by_src are stable permutations with their segment starts and unique keys.
    The device kernels never materialise this: it is the inspection form of
    a layer, built on request by `ComputeGraph.layers`."""
    dst: np.ndarray
    src: np.ndarray
    rel: np.ndarray
    norm: np.ndarray
    rel_indptr: np.ndarray        # (2R + 2,) group boundaries by relation
    num_targets: int
    by_dst: np.ndarray
    dst_segs: np.ndarray
    dst_uniq: np.ndarray
    by_src: np.ndarray
    src_segs: np.ndarray
    src_uniq: np.ndarray

    @property
    def num_edges(self) -> int:
        return len(self.dst)


def _device_segments(sorted_vals):
    """Segment starts and keys of a sorted device vector (ref:sampler.py:265-269)."""
    torch = _torch()
    if sorted_vals.numel() == 0:
        z = torch.zeros(0, dtype=torch.int64, device=sorted_vals.device)
        return z, z
    head = torch.ones_like(sorted_vals, dtype=torch.bool)
    head[1:] = sorted_vals[1:] != sorted_vals[:-1]
    starts = torch.nonzero(head).reshape(-1)
    return starts, sorted_vals[starts]


def _device_block(cg: "ComputeGraph", k: int) -> LayerBlock:
    """Layer k's block on the device (ref:sampler.py:298-307, 359-368): every
    partition message entering A_k (dst-CSR ranges of the targets) plus one
    self-loop per target, lexsorted by (rel, dst, src) with three stable
    sorts, then the by_dst / by_src permutations and segments."""
    torch = _torch()
    v = cg.view
    counts = cg.layer_vertex_counts
    T = counts[k]
    dev = v.device
    i64 = dict(dtype=torch.int64, device=dev)
    tgt = cg.d_order[:T].long()
    pos = cg.d_pos.long()
    indptr = v.d_indptr.long()
    starts = indptr[tgt]
    lens = indptr[tgt + 1] - starts
    E = int(lens.sum().item())
    excl = torch.cumsum(lens, 0) - lens
    eidx = torch.repeat_interleave(starts - excl, lens) + torch.arange(E, **i64)
    sl = v.self_loop_rel
    loops = torch.arange(T, **i64)
    dst = torch.cat([torch.repeat_interleave(loops, lens), loops])
    src = torch.cat([pos[v.d_ref_src.long()[eidx]], loops])
    rel = torch.cat([v.d_ref_rel.long()[eidx], torch.full((T,), sl, **i64)])
    norm = torch.cat([1.0 / v.d_msg_cnt[eidx].double(), torch.ones(T, dtype=torch.float64, device=dev)])
    order = torch.arange(E + T, **i64)
    for key in (src, dst, rel):               # LSD: np.lexsort((src, dst, rel))
        order = order[torch.sort(key[order], stable=True).indices]
    dst, src, rel, norm = dst[order], src[order], rel[order], norm[order]
    rel_indptr = torch.searchsorted(rel, torch.arange(sl + 2, **i64))
    by_dst = torch.sort(dst, stable=True).indices
    dst_segs, dst_uniq = _device_segments(dst[by_dst])
    by_src = torch.sort(src, stable=True).indices
    src_segs, src_uniq = _device_segments(src[by_src])
    h = [t.cpu().numpy() for t in (dst, src, rel, norm, rel_indptr, by_dst, dst_segs, dst_uniq, by_src,
                                   src_segs, src_uniq)]
    return LayerBlock(h[0], h[1], h[2], h[3], h[4], T, *h[5:])


class ComputeGraph:
    """Layered closure of a batch, resident on the GPU.

    Device state: d_order (vertex_order, seeds ascending then each hop's new
    sources ascending), d_pos (local id -> position, -1 absent) and d_counts
    (|A_0| .. |A_hops|, device int32). The RGCN kernels walk the partition
    CSR/CSC restricted to A_k, so nothing per-layer is materialised for
    training; `layers` builds the reference's LayerBlocks (output layer
    first) on the device when asked for.
    """

    def __init__(self, view: PartitionView, hops: int, d_order, d_pos, d_counts):
        self.view = view
        self.hops = hops
        self.d_order = d_order
        self.d_pos = d_pos
        self.d_counts = d_counts
        self._host = {}

    @property
    def num_layers(self) -> int:
        return self.hops

    @property
    def layer_vertex_counts(self) -> list:
        if "counts" not in self._host:
            self._host["counts"] = [int(x) for x in self.d_counts[: self.hops + 1].cpu().tolist()]
        return self._host["counts"]

    @property
    def num_seeds(self) -> int:
        return self.layer_vertex_counts[0]

    @property
    def vertex_order(self) -> np.ndarray:
        if "order" not in self._host:
            c = self.layer_vertex_counts[-1]
            self._host["order"] = self.d_order[:c].cpu().numpy().astype(np.int64)
        return self._host["order"]

    @property
    def seed_vertices(self) -> np.ndarray:
        return self.vertex_order[: self.num_seeds]

    @property
    def pos(self) -> np.ndarray:
        if "pos" not in self._host:
            self._host["pos"] = self.d_pos.cpu().numpy().astype(np.int64)
        return self._host["pos"]

    def layer_vertex_sets(self) -> list:
        return [self.vertex_order[:c] for c in self.layer_vertex_counts]

    @property
    def layers(self) -> list:
        """LayerBlock per convolution, output layer first (ref:sampler.py:277)."""
        if "layers" not in self._host:
            self._host["layers"] = [_device_block(self, k) for k in range(self.hops)]
        return self._host["layers"]

    def seed_positions(self, local_ids: np.ndarray) -> np.ndarray:
        p = self.pos[np.asarray(local_ids)]
        if len(p) and p.min() < 0:
            raise IntegrityError("vertex not present in compute graph")
        return p


def closure_device(view: PartitionView, hops: int, *, stream: Optional[DeviceStream] = None, start: int = 0,
                   size: int = 0, seed_ids=None, out=None, ws=None, start_dev=None) -> ComputeGraph:
    """Run kg_closure for a stream window (batch offset `start`, or the
    device int64 `start_dev` for graph replay) or an explicit seed tensor."""
    torch = _torch()
    lib = _lib.require_cuda()
    dev = view.device
    n = view.n
    if out is None:
        out = (torch.empty(n, dtype=torch.int32, device=dev), torch.empty(n, dtype=torch.int32, device=dev),
               torch.zeros(hops + 1, dtype=torch.int32, device=dev))
    order, pos, counts = out
    ws = ws or _lib.Workspace(dev)
    nb = lib.kg_closure_workspace_bytes(n)
    buf = ws.get("closure", nb)
    import ctypes
    if stream is not None:
        _lib.call("kg_closure", stream.triples.data_ptr(), stream.total, start, _lib.ptr(start_dev), size, 0,
                  ctypes.byref(view.csr()), hops, order.data_ptr(), pos.data_ptr(), counts.data_ptr(),
                  buf.data_ptr(), buf.numel(), _lib.stream_handle())
    else:
        _lib.call("kg_closure", 0, 0, 0, 0, int(seed_ids.numel()), seed_ids.data_ptr(),
                  ctypes.byref(view.csr()), hops, order.data_ptr(), pos.data_ptr(), counts.data_ptr(),
                  buf.data_ptr(), buf.numel(), _lib.stream_handle())
    return ComputeGraph(view, hops, order, pos, counts)


def compute_graph_for_seeds(seeds: np.ndarray, view: PartitionView, hops: int) -> ComputeGraph:
    """ref:sampler.py:320-376 on the GPU."""
    if hops < 0:
        raise ValidationError("hops must be >= 0")
    seeds = np.asarray(seeds, dtype=np.int64).reshape(-1)
    if len(seeds) == 0:
        raise ValidationError("empty batch")
    if seeds.min() < 0 or seeds.max() >= view.num_vertices:
        raise IntegrityError("batch references a vertex outside the partition")
    d = _dev_i32(seeds, view.device)
    return closure_device(view, hops, seed_ids=d)


def build_compute_graph(batch: EdgeMiniBatch, view: PartitionView, hops: int) -> ComputeGraph:
    """Layered n-hop closure of the batch endpoints (ref:sampler.py:310-317)."""
    return compute_graph_for_seeds(batch.triples[:, [0, 2]].reshape(-1), view, hops)


# ---------------------------------------------------------------------------
# Asynchronous epoch sampling (negatives + shuffle) on a side stream
# ---------------------------------------------------------------------------

def _setup_mark(name: str) -> None:
    from .trainer import _mark   # diagnostics (KG_SETUP_TIMES=1)
    _mark(name)


class EpochSampler:
    """Per-partition epoch pipeline: the negatives and the shuffled stream of
    epoch e+1 are produced on a side CUDA stream while epoch e trains. The
    PCG64 state lives on the device, so the whole chain is enqueued without
    host synchronisation; at the epoch boundary `next()` checks the few
    device status words (all negatives accepted, draw windows large enough)
    and, in the rare case they are not, redoes that epoch synchronously from
    a snapshot of the epoch's starting RNG state. Bit-exact either way."""

    ASYNC_ROUNDS = 3
    NSLOTS = 3   # epochs e+1 and e+2 are sampled (and round-prepped) while e trains

    def __init__(self, view: PartitionView, s: int, g_dev, prep=None, pool=None, side=None):
        """prep(slot, DeviceStream), optional: enqueues per-round
        precomputation for an epoch's stream; it becomes part of the slot's
        captured epoch graph, right after the sampling."""
        torch = _torch()
        self.view, self.s, self.g = view, s, g_dev
        self.pool = pool   # graph memory pool of the epoch graphs (None: one private pool per capture)
        self.dev = view.device
        self.side = side if side is not None else torch.cuda.Stream(self.dev)
        self.ws = _lib.Workspace(self.dev)
        core = view.num_core
        total = core * (s + 1)
        self.total = total
        self.core = view.d_edges[:core]
        self.slots = []
        for _ in range(self.NSLOTS):
            self.slots.append(dict(
                neg=_neg_buffers(view, s, self.dev) if s > 0 and core > 0 else None,
                out=dict(perm=torch.empty(max(total, 1), dtype=torch.int32, device=self.dev),
                         tri=torch.empty((max(total, 1), 3), dtype=torch.int32, device=self.dev),
                         lab=torch.empty(max(total, 1), dtype=torch.float32, device=self.dev)),
                g_start=torch.empty_like(g_dev), ready=torch.cuda.Event(), released=None,
                status=torch.zeros(3, dtype=torch.int64, device=self.dev),
                host=torch.zeros(3, dtype=torch.int64, pin_memory=True), stream=None, graph=None))
        self.parity = 0   # slot of the next epoch handed out
        self.redos = 0    # epochs re-run synchronously (status words flagged a short window)
        self._prep = prep
        # one CUDA graph per slot holds the whole epoch pipeline (negatives,
        # shuffle, gather, round prep): an epoch boundary costs one replay.
        # Slot 0 is captured and started now; the others are captured and
        # started by prefetch() (called while the device runs queued rounds,
        # so their host-side capture cost overlaps device work) or, at the
        # latest, when next() needs them. Slots always start in epoch order
        # (the device RNG stream is consumed in that order).
        self.filled = [False] * self.NSLOTS
        _setup_mark("sampler_alloc")
        self._capture(0)
        _setup_mark("sampler_capture")
        self._fill(0)

    def slot_of(self, ds) -> int:
        for i, slot in enumerate(self.slots):
            if slot["out"]["tri"].data_ptr() == ds.triples.data_ptr():
                return i
        raise ValueError("stream does not belong to this sampler")

    def _body(self, parity):
        """The epoch's kernels (current stream = side stream)."""
        torch = _torch()
        slot = self.slots[parity]
        slot["g_start"].copy_(self.g)
        if slot["neg"] is not None:
            neg = sample_negatives_device(self.view, self.s, self.g, self.ws, bufs=slot["neg"],
                                          async_rounds=self.ASYNC_ROUNDS)
            b = slot["neg"]
            slot["status"][0:1].copy_(b["k"][b["cur"]])
            slot["status"][1:2].copy_(b["consumed"].min().view(1))
        else:
            neg = slot.setdefault("empty_neg", torch.zeros((0, 3), dtype=torch.int32, device=self.dev))
            slot["status"][:2].zero_()
        ds, consumed = stream_device(self.core, neg, self.g, self.dev, self.ws, check=False, out=slot["out"])
        slot["status"][2:3].copy_(consumed)
        slot["host"].copy_(slot["status"], non_blocking=True)
        if self._prep is not None:
            self._prep(parity, self.slot_stream(parity))

    def _capture(self, parity):
        torch = _torch()
        slot = self.slots[parity]
        g = torch.cuda.CUDAGraph()
        self.side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.side):
            _lib.capture(g, lambda: self._body(parity), self.pool)
        slot["graph"] = g
        slot["stream"] = self.slot_stream(parity)

    def _fill(self, k):
        if self.slots[k]["graph"] is None:
            self._capture(k)
        self._enqueue(k)
        self.filled[k] = True

    def prefetch(self) -> bool:
        """Start the earliest epoch slot that should be in flight but is not
        (at most one per call); True if one was started."""
        for i in range(self.NSLOTS - 1):
            k = (self.parity + i) % self.NSLOTS
            if not self.filled[k]:
                self._fill(k)
                return True
        return False

    def _enqueue(self, parity):
        torch = _torch()
        slot = self.slots[parity]
        with torch.cuda.stream(self.side):
            if slot["released"] is not None:
                self.side.wait_event(slot["released"])
            slot["graph"].replay()
            slot["ready"].record(self.side)

    def close(self) -> None:
        """Drop the captured epoch graphs (call after the device is idle)."""
        for slot in self.slots:
            slot["graph"] = None

    def slot_stream(self, slot: int) -> DeviceStream:
        """The (fixed-address) stream buffers of a slot, for graph capture."""
        o = self.slots[slot]["out"]
        return DeviceStream(o["tri"], o["lab"], self.total)

    def next(self) -> DeviceStream:
        """Stream of the next epoch (main stream ordered after it); enqueues
        the epoch after that."""
        torch = _torch()
        slot = self.slots[self.parity]
        if not self.filled[self.parity]:
            self._fill(self.parity)
        slot["ready"].synchronize()
        k_left, min_consumed, perm_consumed = (int(x) for x in slot["host"].tolist())
        if k_left > 0 or min_consumed < 0 or perm_consumed < 0:
            self._redo(slot)
            # epochs already started behind this one drew from the device RNG
            # state this epoch left when it stopped short: run them again, in
            # order, from the state the re-run leaves (nothing consumed them yet)
            for i in range(1, self.NSLOTS):
                k = (self.parity + i) % self.NSLOTS
                if self.filled[k]:
                    self._enqueue(k)
        torch.cuda.current_stream().wait_event(slot["ready"])
        out = slot["stream"]
        # the previous epoch's slot (all its compute is enqueued by now) is
        # refilled with epoch e + NSLOTS - 1 once that compute has run
        free = (self.parity + self.NSLOTS - 1) % self.NSLOTS
        other = self.slots[free]
        other["released"] = torch.cuda.Event()
        other["released"].record(torch.cuda.current_stream())
        self.filled[self.parity] = False
        self.parity = (self.parity + 1) % self.NSLOTS
        # start the slots ahead in epoch order; a slot not captured yet is left
        # to prefetch() (it also catches up any gap)
        for i in range(self.NSLOTS - 1):
            k = (self.parity + i) % self.NSLOTS
            if not self.filled[k]:
                if self.slots[k]["graph"] is None:
                    break
                self._enqueue(k)
                self.filled[k] = True
        return out

    def _redo(self, slot):
        """Synchronous, host-checked re-run of one epoch from its start state."""
        torch = _torch()
        self.redos += 1
        with torch.cuda.stream(self.side):
            self.g.copy_(slot["g_start"])
            if slot["neg"] is not None:
                neg = sample_negatives_device(self.view, self.s, self.g, self.ws, bufs=slot["neg"])
            else:
                neg = torch.zeros((0, 3), dtype=torch.int32, device=self.dev)
            stream_device(self.core, neg, self.g, self.dev, self.ws, check=True, out=slot["out"])
            if self._prep is not None:
                self._prep(next(i for i, x in enumerate(self.slots) if x is slot), slot["stream"])
            slot["ready"].record(self.side)
        slot["ready"].synchronize()
