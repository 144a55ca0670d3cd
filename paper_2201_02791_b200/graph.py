"""Knowledge-graph data model and the synthetic generator (host input
producers; ref:graph.py:20-124, 336-393).

The generator's sequential edge loop runs natively (kg_generate_synthetic in
csrc/kg_host.cpp) with the PCG64 stream of `np.random.default_rng(seed)`
reproduced bit-for-bit, so graphs are identical to the reference's for the
same arguments (pinned by tests/test_host_inputs.py against the golden
fixtures).
"""

from __future__ import annotations

import ctypes
import hashlib
from dataclasses import dataclass, field
from typing import NamedTuple, Optional

import numpy as np

from . import _lib
from .errors import ShapeError, ValidationError


class Triplet(NamedTuple):
    head: int
    rel: int
    tail: int


def as_triples(x) -> np.ndarray:
    arr = np.asarray(x, dtype=np.int64)
    if arr.size == 0:
        return arr.reshape(0, 3)
    if arr.ndim != 2 or arr.shape[1] != 3:
        raise ShapeError(f"expected an (n, 3) triple array, got shape {arr.shape}")
    return arr


@dataclass
class KnowledgeGraph:
    """Directed multigraph of (head, relation, tail) over dense ids; adjacency
    is the training edges only (ref:graph.py:35-109)."""
    num_entities: int
    num_relations: int
    triples: np.ndarray
    features: Optional[np.ndarray] = None
    entity_names: Optional[list] = None
    relation_names: Optional[list] = None

    def __post_init__(self):
        self.triples = as_triples(self.triples)
        if self.num_entities < 0 or self.num_relations < 0:
            raise ValidationError("entity/relation counts must be non-negative")
        if len(self.triples):
            ends = self.triples[:, [0, 2]]
            if ends.max() >= self.num_entities or self.triples.min() < 0:
                raise ValidationError("triple ids out of range for this graph")
            if self.triples[:, 1].max() >= self.num_relations:
                raise ValidationError("relation id out of range for this graph")
        if self.features is not None:
            self.features = np.asarray(self.features, dtype=np.float64)
            if self.features.shape[0] != self.num_entities:
                raise ShapeError(f"feature rows ({self.features.shape[0]}) != num_entities "
                                 f"({self.num_entities})")

    @property
    def num_edges(self) -> int:
        return len(self.triples)

    @property
    def edges(self) -> list:
        return [Triplet(*row) for row in self.triples.tolist()]

    # -- adjacency indices over edge ids (ref:graph.py:69-99) ----------------
    def _edge_index(self, col: int) -> tuple:
        key = "_adj_out" if col == 0 else "_adj_in"
        idx = self.__dict__.get(key)
        if idx is None:
            ends = self.triples[:, col]
            order = np.argsort(ends, kind="stable")
            indptr = np.concatenate([[0], np.cumsum(np.bincount(ends, minlength=self.num_entities))])
            idx = (indptr.astype(np.int64), order)
            self.__dict__[key] = idx
        return idx

    def out_edge_ids(self, v: int) -> np.ndarray:
        """Ids of the edges leaving v, ascending."""
        indptr, order = self._edge_index(0)
        return order[indptr[v]:indptr[v + 1]]

    def in_edge_ids(self, v: int) -> np.ndarray:
        """Ids of the edges entering v, ascending."""
        indptr, order = self._edge_index(2)
        return order[indptr[v]:indptr[v + 1]]

    def out_index(self, v: int) -> list:
        """(rel, tail) of every edge leaving v."""
        t = self.triples[self.out_edge_ids(v)]
        return list(zip(t[:, 1].tolist(), t[:, 2].tolist()))

    def in_index(self, v: int) -> list:
        """(rel, head) of every edge entering v."""
        t = self.triples[self.in_edge_ids(v)]
        return list(zip(t[:, 1].tolist(), t[:, 0].tolist()))

    def checksum(self, split: Optional["DatasetSplit"] = None) -> str:
        """Same digest as ref:graph.py:101-109 (partition provenance)."""
        h = hashlib.sha256()
        h.update(b"kg-v1")
        h.update(np.int64([self.num_entities, self.num_relations]).tobytes())
        h.update(np.ascontiguousarray(self.triples).tobytes())
        if split is not None:
            h.update(np.ascontiguousarray(split.valid).tobytes())
            h.update(np.ascontiguousarray(split.test).tobytes())
        return h.hexdigest()


@dataclass
class DatasetSplit:
    train: np.ndarray
    valid: np.ndarray
    test: np.ndarray

    def __post_init__(self):
        self.train = as_triples(self.train)
        self.valid = as_triples(self.valid)
        self.test = as_triples(self.test)

    def all_triples(self) -> np.ndarray:
        return np.concatenate([self.train, self.valid, self.test], axis=0)


def generate_synthetic(num_entities: int, num_relations: int, avg_degree: float, seed: int,
                       train_fraction: float = 0.9) -> tuple:
    """Skewed random multidigraph with a 90/5/5 split (ref:graph.py:336-393):
    heads uniform, tails by preferential attachment (p = 0.75), no duplicate
    triples, no self loops."""
    if num_entities < 2:
        raise ValidationError("num_entities must be >= 2")
    if num_relations < 1:
        raise ValidationError("num_relations must be >= 1")
    if avg_degree <= 0:
        raise ValidationError("avg_degree must be > 0")
    gen = np.random.default_rng(seed)
    target = max(1, round(num_entities * avg_degree / train_fraction))
    out = np.empty((target, 3), dtype=np.int64)
    st = _lib.pcg_from_numpy(gen)
    m = _lib.load().kg_generate_synthetic(num_entities, num_relations, target, ctypes.byref(st),
                                          out.ctypes.data, 50 * target + 1000)
    _lib.pcg_to_numpy(st, gen)
    triples = out[:m]
    n_valid = int(m * (1.0 - train_fraction) / 2.0)
    perm = gen.permutation(m)
    valid = triples[np.sort(perm[:n_valid])]
    test = triples[np.sort(perm[n_valid:2 * n_valid])]
    train = triples[np.sort(perm[2 * n_valid:])]
    split = DatasetSplit(train, valid, test)
    return KnowledgeGraph(num_entities, num_relations, train), split


@dataclass
class GraphStats:
    """Degree summary (ref:graph.py:401-420)."""
    num_entities: int
    num_relations: int
    num_edges: int
    out_degree_min: int
    out_degree_mean: float
    out_degree_max: int
    in_degree_min: int
    in_degree_mean: float
    in_degree_max: int

    def format(self) -> str:
        return (f"entities={self.num_entities} relations={self.num_relations} edges={self.num_edges}\n"
                f"out-degree min/mean/max = {self.out_degree_min}/{self.out_degree_mean:.3f}/"
                f"{self.out_degree_max}\n"
                f"in-degree  min/mean/max = {self.in_degree_min}/{self.in_degree_mean:.3f}/{self.in_degree_max}")


def graph_stats(graph: KnowledgeGraph) -> GraphStats:
    n = graph.num_entities
    if n == 0:
        return GraphStats(0, graph.num_relations, graph.num_edges, 0, 0.0, 0, 0, 0.0, 0)
    deg = [np.bincount(graph.triples[:, c], minlength=n) for c in (0, 2)]
    f = [(int(x.min()), float(x.mean()), int(x.max())) for x in deg]
    return GraphStats(n, graph.num_relations, graph.num_edges, *f[0], *f[1])


# Reference module-level names that live in io.py here (ref:graph.py:131-333); resolved
# lazily so `from <pkg>.graph import X` works as with the reference.
_IO_NAMES = ('load_dataset_dir', 'load_features', 'load_triples', 'read_dictionary', 'write_dataset_dir', 'write_dictionary', 'write_triples')


def __getattr__(name):
    if name in _IO_NAMES:
        from . import io
        return getattr(io, name)
    raise AttributeError(name)
