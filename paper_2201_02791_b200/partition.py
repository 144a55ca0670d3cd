"""Self-sufficient partitions: vertex-cut core edges plus the n-hop halo
(host input producers; ref:partition.py:33-346).

Membership is bit-exact with the reference: the sequential greedy vertex cut
runs natively (kg_vertex_cut_assign, float64 arithmetic identical to numpy's)
and the halo expansion is a set-valued BFS whose outputs are sorted id sets,
so any correct traversal order yields identical partitions.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

from . import _lib
from .errors import ValidationError
from .graph import KnowledgeGraph, as_triples

import os

_HOST_EXPAND = os.environ.get("KG_HOST_EXPAND", "0") == "1"   # tests: force the host BFS on a GPU box

ROLE_CORE = "core"
ROLE_REPLICATED = "replicated"
ROLE_SUPPORT = "support"


@dataclass
class Partition:
    """One partition: core edges it owns + support edges of its halo
    (ref:partition.py:33-105)."""
    id: int
    core: np.ndarray
    support: np.ndarray
    core_vertices: np.ndarray
    replicated_vertices: np.ndarray
    support_vertices: np.ndarray
    hop_count: int
    core_edge_ids: Optional[np.ndarray] = None
    support_edge_ids: Optional[np.ndarray] = None
    _local: Optional[np.ndarray] = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        self.core = as_triples(self.core)
        self.support = as_triples(self.support)

    @property
    def num_core_edges(self) -> int:
        return len(self.core)

    @property
    def num_total_edges(self) -> int:
        return len(self.core) + len(self.support)

    def all_edges(self) -> np.ndarray:
        return np.concatenate([self.core, self.support], axis=0)

    def local_vertices(self) -> np.ndarray:
        """Host restatement of the local-id order (core endpoints by first
        appearance, then support endpoints); the training path computes the
        same order on the GPU inside build_view (kg_view_local_ids)."""
        if self._local is None:
            def first(vals):
                if len(vals) == 0:
                    return np.zeros(0, np.int64)
                _, idx = np.unique(vals, return_index=True)
                return vals[np.sort(idx)]
            c = first(self.core[:, [0, 2]].reshape(-1))
            s = self.support[:, [0, 2]].reshape(-1)
            s = first(s[~np.isin(s, c)]) if len(s) else np.zeros(0, np.int64)
            self._local = np.concatenate([c, s]).astype(np.int64)
        return self._local

    def global_to_local(self, num_entities: int) -> np.ndarray:
        g2l = np.full(num_entities, -1, dtype=np.int64)
        loc = self.local_vertices()
        g2l[loc] = np.arange(len(loc))
        return g2l

    def vertex_roles(self) -> dict:
        return {ROLE_CORE: self.core_vertices, ROLE_REPLICATED: self.replicated_vertices,
                ROLE_SUPPORT: self.support_vertices}

    @property
    def pool_size(self) -> int:
        """Number of legal corruption targets: core-edge endpoints
        (ref:sampler.py:102, 111)."""
        return len(self.core_vertices) + len(self.replicated_vertices)


@dataclass
class PartitionSet:
    partitions: list
    num_entities: int
    num_relations: int
    hops: int
    seed: int
    method: str
    graph_checksum: str

    @property
    def num_parts(self) -> int:
        return len(self.partitions)

    @property
    def expanded(self) -> bool:
        return self.hops > 0 or any(len(p.support) for p in self.partitions)


def _sorted_endpoints(tri: np.ndarray, ids: np.ndarray, n: int, mark: np.ndarray) -> np.ndarray:
    """np.unique(tri[ids][:, [0, 2]]) through a reusable vertex mark array."""
    mark[tri[ids, 0]] = True
    mark[tri[ids, 2]] = True
    out = np.flatnonzero(mark)
    mark[out] = False
    return out


def _build_set(graph: KnowledgeGraph, assign: np.ndarray, P: int, seed: int, method: str) -> PartitionSet:
    """Partition records from a per-edge assignment (ref:partition.py:112-134)."""
    n = graph.num_entities
    ids = [np.flatnonzero(assign == p) for p in range(P)]
    mark = np.zeros(n, dtype=bool)
    ends = [_sorted_endpoints(graph.triples, i, n, mark) for i in ids]
    count = np.zeros(n, dtype=np.int64)
    for e in ends:
        count[e] += 1
    shared = count >= 2
    parts = []
    for p in range(P):
        parts.append(Partition(
            id=p, core=graph.triples[ids[p]], support=np.zeros((0, 3), np.int64),
            core_vertices=ends[p][~shared[ends[p]]], replicated_vertices=ends[p][shared[ends[p]]],
            support_vertices=np.zeros(0, np.int64), hop_count=0,
            core_edge_ids=ids[p].astype(np.int64)))
    return PartitionSet(parts, n, graph.num_relations, 0, seed, method, graph.checksum())


def vertex_cut_partition(graph: KnowledgeGraph, num_parts: int, seed: int, epsilon: float = 0.05,
                         balance_weight: float = 1.0) -> PartitionSet:
    """HDRF-family greedy streaming vertex cut (ref:partition.py:141-191):
    seeded edge order, replication affinity + balance score, hard cap at
    max(ceil(m/P), floor((1+eps) m / P))."""
    m = graph.num_edges
    if num_parts < 1:
        raise ValidationError("num_parts must be >= 1")
    if num_parts > m:
        raise ValidationError(f"num_parts ({num_parts}) exceeds edge count ({m})")
    order = np.ascontiguousarray(np.random.default_rng(seed).permutation(m), dtype=np.int64)
    cap = max(math.ceil(m / num_parts), math.floor((1.0 + epsilon) * m / num_parts))
    tri = np.ascontiguousarray(graph.triples, dtype=np.int64)
    assign = np.empty(m, dtype=np.int64)
    _lib.check(_lib.load().kg_vertex_cut_assign(tri.ctypes.data, m, graph.num_entities, num_parts,
                                                order.ctypes.data, float(balance_weight), int(cap),
                                                assign.ctypes.data), "vertex_cut_partition")
    return _build_set(graph, assign, num_parts, seed, "vertexcut")


def random_edge_partition(graph: KnowledgeGraph, num_parts: int, seed: int) -> PartitionSet:
    """Uniform random edge assignment (ref:partition.py:194-204)."""
    m = graph.num_edges
    if num_parts < 1:
        raise ValidationError("num_parts must be >= 1")
    if num_parts > m:
        raise ValidationError(f"num_parts ({num_parts}) exceeds edge count ({m})")
    assign = np.random.default_rng(seed).integers(num_parts, size=m)
    return _build_set(graph, assign, num_parts, seed, "random")


def _incidence(graph: KnowledgeGraph):
    """CSR: vertex -> ids of edges touching it (either endpoint)."""
    ends = graph.triples[:, [0, 2]].reshape(-1)
    eid = np.repeat(np.arange(graph.num_edges, dtype=np.int64), 2)
    order = np.argsort(ends, kind="stable")
    ptr = np.zeros(graph.num_entities + 1, dtype=np.int64)
    np.cumsum(np.bincount(ends, minlength=graph.num_entities), out=ptr[1:])
    return ptr, eid[order]


def _cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def _expand_device(pset: PartitionSet, graph: KnowledgeGraph, hops: int) -> list:
    """The halo BFS of every partition on the GPU (kg_halo_incidence /
    kg_halo_expand): flags + ascending stream compaction, so the sets are
    exactly the reference's."""
    import torch
    lib = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    st = _lib.stream_handle()
    m, n = graph.num_edges, graph.num_entities
    tri = torch.as_tensor(np.ascontiguousarray(graph.triples, dtype=np.int32)).to(dev)
    ws = torch.empty(lib.kg_halo_workspace_bytes(m, n), dtype=torch.uint8, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    ptr = torch.empty(n + 1, **i32)
    inc = torch.empty(max(2 * m, 1), **i32)
    _lib.call("kg_halo_incidence", tri.data_ptr(), m, n, ptr.data_ptr(), inc.data_ptr(), ws.data_ptr(), ws.numel(), st)
    sup = torch.empty(max(m, 1), **i32)
    sv = torch.empty(max(n, 1), **i32)
    cv = torch.empty(max(n, 1), **i32)
    cnt = torch.zeros(3, **i32)
    tri64 = None
    out = []
    for part in pset.partitions:
        if part.core_edge_ids is None:
            raise ValidationError("partition lacks edge ids; reload with the source graph")
        core = torch.as_tensor(np.ascontiguousarray(part.core_edge_ids, dtype=np.int32)).to(dev)
        _lib.call("kg_halo_expand", tri.data_ptr(), m, n, ptr.data_ptr(), inc.data_ptr(), core.data_ptr(),
                  core.numel(), hops, sup.data_ptr(), cnt[0:1].data_ptr(), sv.data_ptr(), cnt[1:2].data_ptr(),
                  cv.data_ptr(), cnt[2:3].data_ptr(), ws.data_ptr(), ws.numel(), st)
        ns, nv, _ = (int(x) for x in cnt.tolist())
        sup_ids = sup[:ns].long()
        if tri64 is None:
            tri64 = tri.long()
        out.append(replace(part, support=tri64[sup_ids].cpu().numpy(), support_vertices=sv[:nv].cpu().numpy().astype(
            np.int64), support_edge_ids=sup_ids.cpu().numpy(), hop_count=hops, _local=None))
    return out


def neighborhood_expand(pset: PartitionSet, graph: KnowledgeGraph, hops: int) -> PartitionSet:
    """Copy each partition's n-hop bidirectional closure in as support
    edges/vertices (ref:partition.py:234-282). Idempotent at equal hops.
    On a CUDA device the BFS runs on the GPU (kg_halo_expand); the host
    restatement below serves CPU-only environments (input preparation, not
    the training path). Both produce the reference's sorted sets."""
    if hops < 0:
        raise ValidationError("hops must be >= 0")
    if pset.expanded:
        if pset.hops == hops:
            return pset
        raise ValidationError(f"partition set already expanded with hops={pset.hops}, "
                              f"cannot re-expand to {hops}")
    if hops == 0:
        return pset
    if _cuda_available() and not _HOST_EXPAND:
        return PartitionSet(_expand_device(pset, graph, hops), pset.num_entities, pset.num_relations, hops,
                            pset.seed, pset.method, pset.graph_checksum)
    ptr, inc = _incidence(graph)
    tri = graph.triples
    out = []
    for part in pset.partitions:
        if part.core_edge_ids is None:
            raise ValidationError("partition lacks edge ids; reload with the source graph")
        edge_in = np.zeros(graph.num_edges, dtype=bool)
        edge_in[part.core_edge_ids] = True
        seen = np.zeros(graph.num_entities, dtype=bool)
        core_ends = np.unique(tri[part.core_edge_ids][:, [0, 2]])
        seen[core_ends] = True
        front = core_ends
        for _ in range(hops):
            lens = ptr[front + 1] - ptr[front]
            if lens.sum() == 0:
                break
            starts = np.repeat(ptr[front] - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens)
            touched = inc[starts + np.arange(lens.sum())]
            edge_in[touched] = True
            nb = np.unique(tri[touched][:, [0, 2]])
            front = nb[~seen[nb]]
            seen[front] = True
            if len(front) == 0:
                break
        sup_ids = np.flatnonzero(edge_in)
        core_mask = np.zeros(graph.num_edges, dtype=bool)
        core_mask[part.core_edge_ids] = True
        sup_ids = sup_ids[~core_mask[sup_ids]]
        verts = np.flatnonzero(seen)
        is_core = np.zeros(graph.num_entities, dtype=bool)
        is_core[core_ends] = True
        out.append(replace(part, support=tri[sup_ids], support_vertices=verts[~is_core[verts]],
                           support_edge_ids=sup_ids, hop_count=hops, _local=None))
    return PartitionSet(out, pset.num_entities, pset.num_relations, hops, pset.seed, pset.method,
                        pset.graph_checksum)


def replication_factor(pset: PartitionSet) -> float:
    """Mean covered-vertex count / |V| (ref:partition.py:289-300)."""
    if pset.num_entities == 0:
        raise ValidationError("replication factor undefined for an empty graph")
    return sum(len(np.unique(p.all_edges()[:, [0, 2]])) for p in pset.partitions) / pset.num_entities


# Reference module-level names that live in io.py here (ref:partition.py:304-482); resolved
# lazily so `from <pkg>.partition import X` works as with the reference.
_IO_NAMES = ('PartitionStats', 'partition_stats', 'read_partitions', 'write_partitions')


def __getattr__(name):
    if name in _IO_NAMES:
        from . import io
        return getattr(io, name)
    raise AttributeError(name)
