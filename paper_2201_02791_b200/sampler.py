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

import numpy as np

from . import _lib
from .errors import IntegrityError, SamplingError, ValidationError
from .partition import Partition

MAX_RESAMPLE_ROUNDS = 100
CHUNK_EDGES = 64          # messages per warp work chunk (hub rows are split)


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
    c = _lib.KgGraphCsr()
    c.n, c.R, c.e, c.chunk = n_local, num_relations, e, C
    for f in ("indptr", "src", "rel", "norm", "c_indptr", "c_dst", "c_rel", "c_norm", "rel_perm", "rel_ptr",
              "ck_ptr", "ck_row", "ck_slot", "ck_split", "ck_counts",
              "cc_ptr", "cc_row", "cc_slot", "cc_split", "cc_counts"):
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


def sample_negatives_device(view: PartitionView, s: int, pcg, ws: Optional["_lib.Workspace"] = None):
    """Device-resident negatives: returns ((s*m,3) int32 tensor, advanced pcg).
    Bit-exact with the reference's draws from the same PCG64 state."""
    torch = _torch()
    if s < 0:
        raise ValidationError("negatives_per_positive must be >= 0")
    m = view.num_core
    dev = view.device
    if s == 0 or m == 0:
        return torch.zeros((0, 3), dtype=torch.int32, device=dev), pcg
    if view.pool_size < 2:
        raise SamplingError("partition has fewer than 2 core vertices")
    lib = _lib.require_cuda()
    st = _lib.stream_handle()
    ws = ws or _lib.Workspace(dev)
    total = m * s
    neg = torch.empty((total, 3), dtype=torch.int32, device=dev)
    col = torch.empty(total, dtype=torch.int8, device=dev)
    pend = [torch.empty(total, dtype=torch.int32, device=dev), torch.empty(total, dtype=torch.int32, device=dev)]
    g = _lib.pcg_copy(pcg)
    _lib.call("kg_neg_init", view.d_edges.data_ptr(), m, s, g, neg.data_ptr(), col.data_ptr(),
              pend[0].data_ptr(), st)
    _lib.pcg_advance(g, total)
    counters = torch.zeros(4, dtype=torch.int64, device=dev)   # [consumed, next_count (int32)]
    k = total
    cur = 0
    for _ in range(MAX_RESAMPLE_ROUNDS):
        if k == 0:
            break
        W = _round_window(k, view.pool_size)
        while True:
            nbytes = lib.kg_neg_round_workspace_bytes(W)
            buf = ws.get("neg_round", nbytes)
            _lib.call("kg_neg_round", neg.data_ptr(), col.data_ptr(), view.d_edges.data_ptr(), s,
                      pend[cur].data_ptr(), k, view.pool_size, view.n, view.num_relations,
                      view.d_pos_keys.data_ptr(), view.d_n_keys.data_ptr(), g, W,
                      pend[1 - cur].data_ptr(), counters.data_ptr() + 8, counters.data_ptr(),
                      buf.data_ptr(), buf.numel(), st)
            host = counters.cpu()
            consumed = int(host[0])
            if consumed > 0:
                break
            W *= 2
        next_k = int(host[1]) & 0xFFFFFFFF       # int32 next_count written at byte offset 8
        _lib.pcg_consume32(g, consumed)
        cur = 1 - cur
        k = next_k
    if k > 0:
        row = int(pend[cur][0].item())
        e = view.core_edges[row // s]
        raise SamplingError(f"could not corrupt edge {tuple(int(x) for x in e)} after "
                            f"{MAX_RESAMPLE_ROUNDS} rounds")
    return neg, g


def sample_negatives(view: PartitionView, negatives_per_positive: int,
                     rng: np.random.Generator) -> np.ndarray:
    """Corrupt every core edge s times inside the partition's core-vertex pool
    (ref:sampler.py:144-182); returns (s*num_core, 3) int64 local triples."""
    pcg = _lib.pcg_from_numpy(rng)
    neg, g = sample_negatives_device(view, negatives_per_positive, pcg)
    _lib.pcg_to_numpy(g, rng)
    return neg.cpu().numpy().astype(np.int64).reshape(-1, 3)


# ---------------------------------------------------------------------------
# Batching (ref:sampler.py:189-232)
# ---------------------------------------------------------------------------

def permutation_device(n: int, pcg, device, ws: Optional["_lib.Workspace"] = None):
    """rng.permutation(n) on the GPU, bit-exact; returns (int32 tensor, pcg)."""
    torch = _torch()
    lib = _lib.require_cuda()
    st = _lib.stream_handle()
    ws = ws or _lib.Workspace(device)
    g = _lib.pcg_copy(pcg)
    if n <= 1:
        return torch.zeros(n, dtype=torch.int32, device=device), g
    js = ws.get("perm_js", 4 * n)
    W = lib.kg_perm_draws_buffer_len(n)
    consumed_t = torch.zeros(1, dtype=torch.int64, device=device)
    while True:
        U = ws.get("perm_U", 4 * W)
        _lib.call("kg_perm_draws_buffered", n, g, U.data_ptr(), W, js.data_ptr(), consumed_t.data_ptr(), st)
        consumed = int(consumed_t.item())
        if consumed >= 0:
            break
        W = ((2 * W) // 1024 + 1) * 1024
    perm = torch.empty(n, dtype=torch.int32, device=device)
    rb = lib.kg_perm_resolve_workspace_bytes(n)
    buf = ws.get("perm_resolve", rb)
    _lib.call("kg_perm_resolve", js.data_ptr(), n, perm.data_ptr(), buf.data_ptr(), buf.numel(), st)
    _lib.pcg_consume32(g, consumed)
    return perm, g


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


def stream_device(pos, neg, pcg, device, ws=None):
    """concat(pos, neg)[perm] with labels, perm = rng.permutation(total)."""
    torch = _torch()
    npos, nneg = int(pos.shape[0]), int(neg.shape[0])
    total = npos + nneg
    perm, g = permutation_device(total, pcg, device, ws)
    tri = torch.empty((total, 3), dtype=torch.int32, device=device)
    lab = torch.empty(total, dtype=torch.float32, device=device)
    if total:
        _lib.call("kg_stream_gather", pos.data_ptr(), npos, neg.data_ptr(), nneg, perm.data_ptr(),
                  tri.data_ptr(), lab.data_ptr(), _lib.stream_handle())
    return DeviceStream(tri, lab, total), g


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
    ds, g = stream_device(_dev_i32(pos, dev).reshape(-1, 3), _dev_i32(neg, dev).reshape(-1, 3),
                          _lib.pcg_from_numpy(rng), dev)
    _lib.pcg_to_numpy(g, rng)
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

class ComputeGraph:
    """Layered closure of a batch, resident on the GPU.

    Device state: d_order (vertex_order, seeds ascending then each hop's new
    sources ascending), d_pos (local id -> position, -1 absent) and d_counts
    (|A_0| .. |A_hops|, device int32). Nothing per-layer is materialised: the
    RGCN kernels walk the partition CSR/CSC restricted to A_k.
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

    def seed_positions(self, local_ids: np.ndarray) -> np.ndarray:
        p = self.pos[np.asarray(local_ids)]
        if len(p) and p.min() < 0:
            raise IntegrityError("vertex not present in compute graph")
        return p


def closure_device(view: PartitionView, hops: int, *, stream: Optional[DeviceStream] = None, start: int = 0,
                   size: int = 0, seed_ids=None, out=None, ws=None) -> ComputeGraph:
    """Run kg_closure for a stream window or an explicit seed id tensor."""
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
        _lib.call("kg_closure", stream.triples.data_ptr(), stream.total, start, size, 0,
                  ctypes.byref(view.csr()), hops, order.data_ptr(), pos.data_ptr(), counts.data_ptr(),
                  buf.data_ptr(), buf.numel(), _lib.stream_handle())
    else:
        _lib.call("kg_closure", 0, 0, 0, int(seed_ids.numel()), seed_ids.data_ptr(),
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
