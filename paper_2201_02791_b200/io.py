"""Host-side file formats and utilities of the reference API, so a `kgdist`
user finds every entry point here too. These are not on the GPU hot path;
the on-disk formats match the reference's (directories written by either
package load in the other):

  dataset directory  train.txt [valid.txt test.txt] (tab or space separated
                     triples) [entities.dict relations.dict] (`id<TAB>name`)
                     ref:graph.py:131-296
  feature file       `vertex_id v1 ... vd` per line            ref:graph.py:299-329
  partition dir      meta (key=value + sha256 over the keys), p<i>/
                     core_edges.tsv, support_edges.tsv, vertices.tsv
                     (global id, role, local id)               ref:partition.py:336-482
                     or (fmt="npy", memory-mapped) core_edges.npy,
                     support_edges.npy, vertices.npy, roles.npy
  candidates file    `test_index<TAB>c1,c2,...`                 ref:evaluate.py:232-242
  results file       one rank record per line + `# mrr=` / `# hits@k=` ref:evaluate.py:245-253
"""

from __future__ import annotations

import hashlib
import os
import time
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .errors import FormatError, ParseError, ProvenanceError, ReferenceError_, ShapeError
from .graph import DatasetSplit, KnowledgeGraph
from .partition import (ROLE_CORE, ROLE_REPLICATED, ROLE_SUPPORT, Partition, PartitionSet,
                        replication_factor)

# ---------------------------------------------------------------------------
# triples, dictionaries, dataset directories
# ---------------------------------------------------------------------------


def _rows(path: str) -> list:
    """Token triples of a triple file (comments and blank lines skipped)."""
    out = []
    with open(path, "r", encoding="utf-8") as fh:
        for n, raw in enumerate(fh, 1):
            text = raw.rstrip("\n")
            if not text or text.startswith("#"):
                continue
            cols = text.split("\t") if "\t" in text else text.split()
            if len(cols) != 3:
                raise ParseError(f"{path}:{n}: expected 3 columns, got {len(cols)}")
            out.append(cols)
    return out


def read_dictionary(path: str) -> dict:
    """`id<TAB>name` lines -> {name: id}."""
    out = {}
    with open(path, "r", encoding="utf-8") as fh:
        for n, raw in enumerate(fh, 1):
            text = raw.rstrip("\n")
            if not text or text.startswith("#"):
                continue
            cols = text.split("\t")
            if len(cols) != 2:
                raise ParseError(f"{path}:{n}: expected 2 columns, got {len(cols)}")
            try:
                out[cols[1]] = int(cols[0])
            except ValueError as exc:
                raise ParseError(f"{path}:{n}: non-integer id {cols[0]!r}") from exc
    return out


def _is_int(tok: str) -> bool:
    return tok.lstrip("-").isdigit()


class _Ids:
    """token -> dense id: a fixed dictionary, or first occurrence."""

    def __init__(self, fixed: Optional[dict], kind: str):
        self.table = dict(fixed) if fixed else {}
        self.fixed = fixed is not None
        self.kind = kind

    def __call__(self, tok: str, where: str) -> int:
        got = self.table.get(tok)
        if got is not None:
            return got
        if self.fixed:
            raise ReferenceError_(f"{where}: unknown {self.kind} {tok!r}")
        self.table[tok] = len(self.table)
        return self.table[tok]

    def size(self) -> int:
        if not self.table:
            return 0
        return max(self.table.values()) + 1 if self.fixed else len(self.table)

    def names(self) -> Optional[list]:
        if not self.table:
            return None
        names = [None] * self.size()
        for tok, i in self.table.items():
            names[i] = tok
        return names


def load_triples(train_path: str, valid_path: Optional[str] = None, test_path: Optional[str] = None,
                 entity_dict: Optional[dict] = None, relation_dict: Optional[dict] = None) -> tuple:
    """Triple files -> (KnowledgeGraph, DatasetSplit) (ref:graph.py:198-254).
    Without dictionaries, files made only of integers keep their ids;
    otherwise tokens get dense ids in first-occurrence order (train, valid,
    test)."""
    parts = {"train": _rows(train_path), "valid": _rows(valid_path) if valid_path else [],
             "test": _rows(test_path) if test_path else []}
    every = [r for k in ("train", "valid", "test") for r in parts[k]]
    numeric = (entity_dict is None and relation_dict is None and every
               and all(_is_int(a) and _is_int(b) and _is_int(c) for a, b, c in every))
    ent_names = rel_names = None
    if numeric:
        arr = {k: np.asarray(v, dtype=np.int64).reshape(-1, 3) for k, v in parts.items()}
        allv = np.concatenate(list(arr.values()))
        if len(allv) and allv.min() < 0:
            raise ParseError("negative ids in integer-mode triple file")
        n_ent = int(allv[:, [0, 2]].max()) + 1 if len(allv) else 0
        n_rel = int(allv[:, 1].max()) + 1 if len(allv) else 0
    else:
        ent, rel = _Ids(entity_dict, "entity"), _Ids(relation_dict, "relation")
        arr = {}
        for k in ("train", "valid", "test"):
            arr[k] = np.asarray([(ent(h, k), rel(r, k), ent(t, k)) for h, r, t in parts[k]],
                                dtype=np.int64).reshape(-1, 3)
        n_ent, n_rel = ent.size(), rel.size()
        ent_names, rel_names = ent.names(), rel.names()
    split = DatasetSplit(arr["train"], arr["valid"], arr["test"])
    graph = KnowledgeGraph(n_ent, n_rel, split.train, entity_names=ent_names, relation_names=rel_names)
    return graph, split


def load_dataset_dir(path: str) -> tuple:
    """train.txt [valid.txt test.txt entities.dict relations.dict] (ref:graph.py:257-273)."""
    if not os.path.isfile(os.path.join(path, "train.txt")):
        raise ParseError(f"no train.txt under {path}")

    def opt(name):
        f = os.path.join(path, name)
        return f if os.path.isfile(f) else None

    ed, rd = opt("entities.dict"), opt("relations.dict")
    return load_triples(os.path.join(path, "train.txt"), opt("valid.txt"), opt("test.txt"),
                        entity_dict=read_dictionary(ed) if ed else None,
                        relation_dict=read_dictionary(rd) if rd else None)


def write_triples(triples: np.ndarray, path: str, entity_names=None, relation_names=None) -> None:
    t = np.asarray(triples, dtype=np.int64).reshape(-1, 3)
    with open(path, "w", encoding="utf-8") as fh:
        for h, r, tl in t.tolist():
            fh.write("\t".join((entity_names[h] if entity_names else str(h),
                                relation_names[r] if relation_names else str(r),
                                entity_names[tl] if entity_names else str(tl))) + "\n")


def write_dictionary(names: Sequence[str], path: str) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(f"{i}\t{name}\n" for i, name in enumerate(names))


def write_dataset_dir(graph: KnowledgeGraph, split: DatasetSplit, path: str) -> None:
    """Inverse of load_dataset_dir (ref:graph.py:289-296)."""
    os.makedirs(path, exist_ok=True)
    for name, arr in (("train.txt", split.train), ("valid.txt", split.valid), ("test.txt", split.test)):
        write_triples(arr, os.path.join(path, name), graph.entity_names, graph.relation_names)
    if graph.entity_names:
        write_dictionary(graph.entity_names, os.path.join(path, "entities.dict"))
    if graph.relation_names:
        write_dictionary(graph.relation_names, os.path.join(path, "relations.dict"))


def load_features(path: str, graph: KnowledgeGraph) -> KnowledgeGraph:
    """Attach a `vertex_id v1 ... vd` file as graph.features (ref:graph.py:299-329)."""
    rows, width = {}, None
    with open(path, "r", encoding="utf-8") as fh:
        for n, raw in enumerate(fh, 1):
            text = raw.strip()
            if not text or text.startswith("#"):
                continue
            cols = text.split()
            try:
                vid, vals = int(cols[0]), [float(x) for x in cols[1:]]
            except ValueError as exc:
                raise ParseError(f"{path}:{n}: non-numeric token") from exc
            width = len(vals) if width is None else width
            if len(vals) != width:
                raise ShapeError(f"{path}:{n}: expected {width} values, got {len(vals)}")
            if not 0 <= vid < graph.num_entities:
                raise ShapeError(f"{path}:{n}: vertex id {vid} out of range")
            rows[vid] = vals
    if len(rows) != graph.num_entities:
        raise ShapeError(f"feature file has {len(rows)} rows, graph has {graph.num_entities} entities")
    feats = np.zeros((graph.num_entities, width or 0), dtype=np.float64)
    if rows:
        ids = np.fromiter(rows.keys(), dtype=np.int64, count=len(rows))
        feats[ids] = np.asarray(list(rows.values()), dtype=np.float64).reshape(len(rows), -1)
    graph.features = feats
    return graph


# ---------------------------------------------------------------------------
# partitions
# ---------------------------------------------------------------------------


@dataclass
class PartitionStats:
    """Per-partition sizes and the replication factor (ref:partition.py:303-346)."""
    num_parts: int
    hops: int
    method: str
    core_edges: list
    support_edges: list
    total_edges: list
    vertices: list
    rf: float

    @staticmethod
    def mean_std(values):
        a = np.asarray(values, dtype=np.float64)
        return float(a.mean()), float(a.std())

    def format(self) -> str:
        out = [f"partitioner={self.method} parts={self.num_parts} hops={self.hops}",
               f"{'part':>4} {'core edges':>12} {'support edges':>14} {'total edges':>12} {'vertices':>10}"]
        out += [f"{i:>4} {c:>12} {s:>14} {t:>12} {v:>10}"
                for i, (c, s, t, v) in enumerate(zip(self.core_edges, self.support_edges, self.total_edges,
                                                     self.vertices))]
        cm, cs = self.mean_std(self.core_edges)
        tm, ts = self.mean_std(self.total_edges)
        out += [f"core edges  mean±std = {cm:.1f} ± {cs:.1f}", f"total edges mean±std = {tm:.1f} ± {ts:.1f}",
                f"RF = {self.rf:.4f}"]
        return "\n".join(out)


def partition_stats(pset: PartitionSet) -> PartitionStats:
    ps = pset.partitions
    return PartitionStats(pset.num_parts, pset.hops, pset.method, [p.num_core_edges for p in ps],
                          [len(p.support) for p in ps], [p.num_total_edges for p in ps],
                          [len(p.local_vertices()) for p in ps], replication_factor(pset))


_META = ("version", "num_parts", "hops", "seed", "partitioner", "num_entities", "num_relations",
         "graph_checksum")
_ROLE_CODE = {ROLE_CORE: 0, ROLE_REPLICATED: 1, ROLE_SUPPORT: 2}
PARTITION_FORMATS = ("tsv", "npy")


def _meta_sha(fields: dict) -> str:
    return hashlib.sha256("\n".join(f"{k}={fields[k]}" for k in _META).encode()).hexdigest()


def write_partitions(pset: PartitionSet, out_dir: str, fmt: str = "tsv") -> None:
    """Partition directory (ref:partition.py:362-384).

    fmt="tsv" writes the reference's text layout (readable by either package);
    fmt="npy" writes per partition core_edges.npy /
    support_edges.npy (int64 (m,3)) and vertices.npy / roles.npy (global id
    and role code 0 core / 1 replicated / 2 support, in local-id order), which
    read_partitions memory-maps instead of parsing. The manifest is the same
    (its checksum covers the same keys)."""
    if fmt not in PARTITION_FORMATS:
        raise FormatError(f"unknown partition format {fmt!r}")
    os.makedirs(out_dir, exist_ok=True)
    fields = dict(version=1, num_parts=pset.num_parts, hops=pset.hops, seed=pset.seed, partitioner=pset.method,
                  num_entities=pset.num_entities, num_relations=pset.num_relations,
                  graph_checksum=pset.graph_checksum)
    with open(os.path.join(out_dir, "meta"), "w", encoding="utf-8") as fh:
        fh.writelines(f"{k}={fields[k]}\n" for k in _META)
        fh.write(f"meta_checksum={_meta_sha(fields)}\n")
    for p in pset.partitions:
        d = os.path.join(out_dir, f"p{p.id}")
        os.makedirs(d, exist_ok=True)
        local = p.local_vertices()
        if fmt == "npy":
            np.save(os.path.join(d, "core_edges.npy"), np.ascontiguousarray(p.core, dtype=np.int64))
            np.save(os.path.join(d, "support_edges.npy"), np.ascontiguousarray(p.support, dtype=np.int64))
            roles = np.full(len(local), -1, dtype=np.int8)
            pos = np.argsort(local, kind="stable")
            for role, verts in p.vertex_roles().items():
                roles[pos[np.searchsorted(local[pos], verts)]] = _ROLE_CODE[role]
            np.save(os.path.join(d, "vertices.npy"), np.ascontiguousarray(local, dtype=np.int64))
            np.save(os.path.join(d, "roles.npy"), roles)
            continue
        np.savetxt(os.path.join(d, "core_edges.tsv"), p.core, fmt="%d", delimiter="\t")
        np.savetxt(os.path.join(d, "support_edges.tsv"), p.support, fmt="%d", delimiter="\t")
        lid = {int(g): i for i, g in enumerate(local)}
        with open(os.path.join(d, "vertices.tsv"), "w", encoding="utf-8") as fh:
            for role, verts in p.vertex_roles().items():
                fh.writelines(f"{int(g)}\t{role}\t{lid[int(g)]}\n" for g in verts)


class _EdgeIndex:
    """Graph triples sorted by key (h*R + r)*N + t, built once per read."""

    def __init__(self, graph: KnowledgeGraph):
        tri = np.asarray(graph.triples, dtype=np.int64).reshape(-1, 3)
        self.N, self.R = int(graph.num_entities), max(int(graph.num_relations), 1)
        keys = self.keys(tri)
        self.order = np.argsort(keys, kind="stable")
        self.sorted = keys[self.order]
        # end of each sorted position's run of equal keys
        n = len(keys)
        last = np.r_[self.sorted[1:] != self.sorted[:-1], True] if n else np.zeros(0, bool)
        ends = np.where(last, np.arange(1, n + 1), 0)
        self.run_end = np.minimum.accumulate(np.where(last, ends, n)[::-1])[::-1] if n else ends

    def keys(self, t: np.ndarray) -> np.ndarray:
        return (t[:, 0] * self.R + t[:, 1]) * self.N + t[:, 2]


class _EdgeIdResolver:
    """Graph edge index of partition triples, vectorised: duplicates of a
    triple consume its graph occurrences in order, across every batch passed
    to the same resolver (ref:partition.py:398-417 keeps a dict of lists and
    a per-key use count; here the graph is key-sorted once and use counts
    live in an array). Raises at the first offending triple, as the
    reference's loop does."""

    def __init__(self, graph_or_index):
        self.ix = graph_or_index if isinstance(graph_or_index, _EdgeIndex) else _EdgeIndex(graph_or_index)
        self.used = np.zeros(len(self.ix.sorted), dtype=np.int64)   # at the first sorted position of a key

    def __call__(self, triples: np.ndarray) -> np.ndarray:
        ix = self.ix
        t = np.asarray(triples, dtype=np.int64).reshape(-1, 3)
        if len(t) == 0:
            return np.zeros(0, dtype=np.int64)
        ok = ((t[:, 0] >= 0) & (t[:, 0] < ix.N) & (t[:, 2] >= 0) & (t[:, 2] < ix.N)
              & (t[:, 1] >= 0) & (t[:, 1] < ix.R))
        keys = np.where(ok, ix.keys(np.where(ok[:, None], t, 0)), -1)
        # work in key order: sorted needles make searchsorted cache-friendly
        srt = np.argsort(keys, kind="stable")
        ks = keys[srt]
        lo_s = np.searchsorted(ix.sorted, ks, "left")
        inb = lo_s < len(ix.sorted)
        found_s = inb & (ix.sorted[np.where(inb, lo_s, 0)] == ks) & (ks >= 0)
        cnt_s = np.where(found_s, ix.run_end[np.where(inb, lo_s, 0)] - lo_s, 0)
        first = np.r_[True, ks[1:] != ks[:-1]]
        grp_start = np.maximum.accumulate(np.where(first, np.arange(len(ks)), 0))
        k_s = np.arange(len(ks)) - grp_start + np.where(found_s, self.used[np.where(found_s, lo_s, 0)], 0)
        lo, found, cnt, k = (np.empty_like(a) for a in (lo_s, found_s, cnt_s, k_s))
        lo[srt], found[srt], cnt[srt], k[srt] = lo_s, found_s, cnt_s, k_s
        bad = ~found | (k >= cnt)
        if bad.any():
            i = int(np.argmax(bad))
            key = tuple(int(x) for x in t[i])
            if not found[i]:
                raise ProvenanceError(f"partition edge {key} not found in graph")
            raise ProvenanceError(f"partition edge {key} occurs more often than in the graph")
        np.add.at(self.used, lo, 1)
        return ix.order[lo + k]


def _read_manifest(in_dir: str) -> dict:
    meta = os.path.join(in_dir, "meta")
    if not os.path.isfile(meta):
        raise FormatError(f"missing manifest {meta}")
    fields = {}
    with open(meta, "r", encoding="utf-8") as fh:
        for raw in fh:
            text = raw.strip()
            if not text:
                continue
            if "=" not in text:
                raise FormatError(f"malformed manifest line {text!r}")
            k, v = text.split("=", 1)
            fields[k] = v
    missing = [k for k in _META + ("meta_checksum",) if k not in fields]
    if missing:
        raise FormatError(f"manifest missing key {missing[0]!r}")
    if _meta_sha(fields) != fields["meta_checksum"]:
        raise ProvenanceError("manifest checksum mismatch (tampered or corrupt meta file)")
    return fields


def _need(path: str) -> str:
    if not os.path.isfile(path):
        raise FormatError(f"missing partition file {path}")
    return path


def _part_tsv(d: str) -> tuple:
    """(core, support, local ids, role per local id) of a text partition."""
    def triples(name):
        return np.loadtxt(_need(os.path.join(d, name)), dtype=np.int64, delimiter="\t", ndmin=2).reshape(-1, 3)
    core, support = triples("core_edges.tsv"), triples("support_edges.tsv")
    rows = []
    with open(_need(os.path.join(d, "vertices.tsv")), "r", encoding="utf-8") as fh:
        for raw in fh:
            g, role, li = raw.strip().split("\t")
            if role not in _ROLE_CODE:
                raise FormatError(f"unknown vertex role {role!r}")
            rows.append((int(li), int(g), _ROLE_CODE[role]))
    rows.sort()
    local = np.asarray([g for _, g, _ in rows], dtype=np.int64)
    roles = np.asarray([c for _, _, c in rows], dtype=np.int8)
    return core, support, local, roles


def _part_npy(d: str) -> tuple:
    """Memory-mapped (no parse, no copy) binary partition."""
    def arr(name, dtype, ndim):
        a = np.load(_need(os.path.join(d, name)), mmap_mode="r", allow_pickle=False)
        if a.dtype != dtype or a.ndim != ndim or (ndim == 2 and a.shape[1] != 3):
            raise FormatError(f"{os.path.join(d, name)}: expected {np.dtype(dtype).name} with {ndim} dims")
        return a
    core, support = arr("core_edges.npy", np.int64, 2), arr("support_edges.npy", np.int64, 2)
    local, roles = arr("vertices.npy", np.int64, 1), arr("roles.npy", np.int8, 1)
    if len(local) != len(roles):
        raise FormatError(f"{d}: vertices.npy and roles.npy differ in length")
    if len(roles) and (roles.min() < 0 or roles.max() > 2):
        raise FormatError(f"{d}: unknown vertex role code")
    return core, support, local, roles


def read_partitions(in_dir: str, graph: Optional[KnowledgeGraph] = None) -> PartitionSet:
    """Load a partition directory (text or binary layout, detected per
    partition); with `graph`, check provenance and map every edge back to its
    graph index (ref:partition.py:420-482)."""
    fields = _read_manifest(in_dir)
    if graph is not None and graph.checksum() != fields["graph_checksum"]:
        raise ProvenanceError("partition directory was built from a different graph")
    hops = int(fields["hops"])
    index = _EdgeIndex(graph) if graph is not None else None
    core_ids = _EdgeIdResolver(index) if graph is not None else None
    parts = []
    for pid in range(int(fields["num_parts"])):
        d = os.path.join(in_dir, f"p{pid}")
        binary = os.path.isfile(os.path.join(d, "core_edges.npy"))
        core, support, local, roles = _part_npy(d) if binary else _part_tsv(d)
        by_role = [np.sort(np.asarray(local[roles == c], dtype=np.int64)) for c in range(3)]
        part = Partition(id=pid, core=core, support=support, core_vertices=by_role[0],
                         replicated_vertices=by_role[1], support_vertices=by_role[2], hop_count=hops)
        part._local = np.asarray(local, dtype=np.int64)
        if graph is not None:
            part.core_edge_ids = core_ids(core)
            part.support_edge_ids = _EdgeIdResolver(index)(support)
        parts.append(part)
    return PartitionSet(parts, int(fields["num_entities"]), int(fields["num_relations"]), hops,
                        int(fields["seed"]), fields["partitioner"], fields["graph_checksum"])


# ---------------------------------------------------------------------------
# evaluation files, component benchmark
# ---------------------------------------------------------------------------


def read_candidates(path: str) -> dict:
    """`test_index<TAB>c1,c2,...` -> {index: int64 array} (ref:evaluate.py:232-242)."""
    out = {}
    with open(path, "r", encoding="utf-8") as fh:
        for raw in fh:
            text = raw.strip()
            if not text or text.startswith("#"):
                continue
            idx, ids = text.split("\t")
            out[int(idx)] = np.asarray([int(x) for x in ids.split(",") if x], dtype=np.int64)
    return out


def write_results(result, path: str) -> None:
    """Rank records + summary lines (ref:evaluate.py:245-253)."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(f"{r.head}\t{r.rel}\t{r.tail}\t{r.corrupted_side}\t{r.rank}\n" for r in result.records)
        fh.write(f"# mrr={result.mrr:.6f}\n")
        fh.writelines(f"# hits@{k}={result.hits[k]:.6f}\n" for k in sorted(result.hits))


def bench_components(graph: KnowledgeGraph, model_config, train_config, worker_counts: list,
                     partitioners: list = ("vertexcut",), partition_seed: int = 0) -> list:
    """Per (partitioner, worker count): rounds per epoch and the mean epoch /
    per-batch phase times of a training run (ref:trainer.py:487-520). On the
    device the phases overlap inside one CUDA-graph round, so the per-batch
    fields report the round time (cg_build/encode 0, loss_step = round)."""
    from .partition import neighborhood_expand, random_edge_partition, vertex_cut_partition
    from .trainer import train
    rows = []
    for method in partitioners:
        for count in worker_counts:
            fn = vertex_cut_partition if method == "vertexcut" else random_edge_partition
            pset = neighborhood_expand(fn(graph, count, partition_seed), graph, model_config.num_layers)
            t0 = time.perf_counter()
            _, report = train(pset, graph, model_config, train_config)
            wall = time.perf_counter() - t0
            timing = report.mean_timings()
            if not timing["epoch_time"]:
                timing["epoch_time"] = wall / max(train_config.epochs, 1)
            rows.append({"partitioner": method, "workers": count, "rounds": report.rounds_per_epoch, **timing})
    return rows


def format_bench_rows(rows: list) -> str:
    """Fixed-width table of bench_components rows (ref:trainer.py:519-528)."""
    cols = (("partitioner", 12, "s"), ("workers", 7, "d"), ("rounds", 6, "d"), ("epoch_time", 10, ".4f"),
            ("cg_build", 11, ".6f"), ("encode", 10, ".6f"), ("loss_step", 12, ".6f"))
    names = {"epoch_time": "epoch_s", "cg_build": "cg_build_s", "encode": "encode_s", "loss_step": "loss_step_s"}
    out = [" ".join(f"{names.get(k, k):>{w}}" for k, w, _ in cols)]
    out += [" ".join(format(r[k], f">{w}{f}") for k, w, f in cols) for r in rows]
    return "\n".join(out)
