"""CPU restatement of the reference's input producers — TEST / BASELINE
INFRASTRUCTURE ONLY (never imported by the package).

The synthetic generator (ref:graph.py:336-393), the greedy streaming vertex
cut (ref:partition.py:141-191, assembly :112-138) and the n-hop halo
expansion (ref:partition.py:211-282), in plain numpy / Python with the
reference's exact draw order, so `bench.py --impl reference` builds the
benchmark's partitions without loading the package's kernel library. Pinned
against the golden fixtures by tests/test_oracle_inputs.py (graph checksum,
edge assignments and halo sizes at FB15k-237 shape, P = 1/2/4/8).

Outputs are plain containers: `SynthGraph` (triples + split) and, per
partition, `PartInput` (core/support triples, core/replicated vertex ids in
ascending order, pool size) — what oracle/kg_oracle.make_view consumes.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np


@dataclass
class SynthGraph:
    num_entities: int
    num_relations: int
    train: np.ndarray
    valid: np.ndarray
    test: np.ndarray

    def checksum(self, with_split: bool = True) -> str:
        """ref:graph.py:101-109 (the partition provenance digest)."""
        h = hashlib.sha256()
        h.update(b"kg-v1")
        h.update(np.int64([self.num_entities, self.num_relations]).tobytes())
        h.update(np.ascontiguousarray(self.train).tobytes())
        if with_split:
            h.update(np.ascontiguousarray(self.valid).tobytes())
            h.update(np.ascontiguousarray(self.test).tobytes())
        return h.hexdigest()


def synthetic_graph(num_entities: int, num_relations: int, avg_degree: float, seed: int,
                    train_fraction: float = 0.9) -> SynthGraph:
    """ref:graph.py:336-393 — heads uniform; tails by preferential attachment
    (p = 0.75 from the pool of earlier tails) else uniform; self loops and
    repeated (h, r, t) rejected (a rejected draw still consumed its numbers);
    then a seeded permutation splits off valid / test (each
    int(m * (1 - train_fraction) / 2)), every part kept in original order."""
    rng = np.random.default_rng(seed)
    target = max(1, round(num_entities * avg_degree / train_fraction))
    budget = 50 * target + 1000
    seen, rows, tails = set(), [], []
    tries = 0
    while len(rows) < target and tries < budget:
        tries += 1
        h = int(rng.integers(num_entities))
        if tails and rng.random() < 0.75:
            t = tails[int(rng.integers(len(tails)))]
        else:
            t = int(rng.integers(num_entities))
        if h == t:
            continue
        r = int(rng.integers(num_relations))
        if (h, r, t) in seen:
            continue
        seen.add((h, r, t))
        rows.append((h, r, t))
        tails.append(t)
    tri = np.array(rows, dtype=np.int64).reshape(-1, 3)
    m = len(tri)
    k = int(m * (1.0 - train_fraction) / 2.0)
    perm = rng.permutation(m)
    return SynthGraph(num_entities, num_relations, tri[np.sort(perm[2 * k:])], tri[np.sort(perm[:k])],
                      tri[np.sort(perm[k:2 * k])])


@dataclass
class PartInput:
    pid: int
    core: np.ndarray               # (m_p, 3) core triples, ascending edge id
    support: np.ndarray            # (s_p, 3) halo triples, ascending edge id
    core_vertices: np.ndarray      # endpoints owned by this partition only
    replicated_vertices: np.ndarray
    core_edge_ids: np.ndarray
    support_edge_ids: np.ndarray

    @property
    def pool_size(self) -> int:
        return len(self.core_vertices) + len(self.replicated_vertices)


def vertex_cut_assign(train: np.ndarray, num_entities: int, P: int, seed: int, epsilon: float = 0.05,
                      balance_weight: float = 1.0) -> np.ndarray:
    """ref:partition.py:141-188 — edges in a seeded random order; partition
    score = sum over endpoints of [holds it] * (2 - partial-degree share) plus
    balance * (max - size) / (1 + max - min); full partitions (>= cap) get
    -inf; lowest index wins ties (np.argmax). Returns the partition per edge."""
    m = len(train)
    rng = np.random.default_rng(seed)
    order = rng.permutation(m)
    theta = np.zeros(num_entities, dtype=np.int64)
    holds = np.zeros((P, num_entities), dtype=bool)
    size = np.zeros(P, dtype=np.int64)
    cap = max(math.ceil(m / P), math.floor((1.0 + epsilon) * m / P))
    out = np.empty(m, dtype=np.int64)
    for e in order.tolist():
        u, v = int(train[e, 0]), int(train[e, 2])
        du, dv = theta[u], theta[v]
        tot = du + dv
        su = du / tot if tot else 0.5
        sv = dv / tot if tot else 0.5
        sc = holds[:, u] * (2.0 - su) + holds[:, v] * (2.0 - sv)
        hi = size.max()
        sc = sc + balance_weight * (hi - size) / (1.0 + hi - size.min())
        sc[size >= cap] = -np.inf
        p = int(np.argmax(sc))
        out[e] = p
        holds[p, u] = holds[p, v] = True
        size[p] += 1
        theta[u] += 1
        theta[v] += 1
    return out


def partition_inputs(g: SynthGraph, P: int, seed: int, hops: int) -> list:
    """Vertex cut + n-hop halo (ref:partition.py:112-138, 234-282): per
    partition the core edges (ascending id), core / replicated endpoint sets
    (an endpoint of >= 2 partitions' core edges is replicated) and the halo
    edges reached by `hops` rounds of bidirectional expansion from the core
    endpoints."""
    tri = g.train
    n = g.num_entities
    assign = vertex_cut_assign(tri, n, P, seed)
    ids = [np.flatnonzero(assign == p) for p in range(P)]
    ends = [np.unique(tri[i][:, [0, 2]]) for i in ids]
    inc = np.zeros(n, dtype=np.int64)
    for e in ends:
        inc[e] += 1
    # incident-edge CSR (either endpoint), edge ids ascending per vertex
    flat = tri[:, [0, 2]].ravel()
    eid = np.repeat(np.arange(len(tri), dtype=np.int64), 2)
    srt = np.argsort(flat, kind="stable")
    ptr = np.concatenate([[0], np.cumsum(np.bincount(flat, minlength=n))])
    inc_e = eid[srt]
    out = []
    for p in range(P):
        rep = ends[p][inc[ends[p]] >= 2]
        own = ends[p][inc[ends[p]] < 2]
        taken = np.zeros(len(tri), dtype=bool)
        taken[ids[p]] = True
        seen_v = np.zeros(n, dtype=bool)
        front = ends[p]
        seen_v[front] = True
        for _ in range(hops):
            lo, hi = ptr[front], ptr[front + 1]
            sel = np.concatenate([inc_e[a:b] for a, b in zip(lo.tolist(), hi.tolist())]) if len(front) else \
                np.zeros(0, dtype=np.int64)
            sel = np.unique(sel)
            taken[sel] = True
            nb = np.unique(tri[sel][:, [0, 2]])
            front = nb[~seen_v[nb]]
            seen_v[front] = True
            if len(front) == 0:
                break
        sup = np.flatnonzero(taken)
        sup = sup[~np.isin(sup, ids[p])]
        out.append(PartInput(p, tri[ids[p]], tri[sup], own, rep, ids[p], sup))
    return out
