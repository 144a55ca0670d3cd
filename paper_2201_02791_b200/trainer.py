"""Synchronous data-parallel training over self-sufficient partitions on
B200s (drop-in for ref:trainer.py).

One partition per GPU. Launched under torchrun (torch.distributed
initialised, NCCL backend) each rank trains the partitions p with
p % world_size == rank; without a process group every partition runs in this
process on the current device (the reference's P=1 inline path, and the
replicated-partition test configuration). Per round every worker runs

    closure -> RGCN forward -> DistMult+BCE -> RGCN backward

entirely on the device; the dense gradient payloads of all P workers are
all-gathered over NVLink (NCCL) and one fused kernel combines them in the
reference's pairwise-tree order and applies Adam/SGD, so dense replicas stay
bitwise identical on every rank (ref:trainer.py:465-469). Embedding rows are
partition-local and updated with lazy sparse Adam.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .errors import KGError, NumericError, ProtocolError, ValidationError
from .model import (MODE_EMBEDDING, MODE_FEATURE, DeviceModel, ModelConfig, ModelParams, ViewBuffers,
                    check_flags, raise_for_flags, device_backward, device_csc_positions, device_backward_y, device_dropout, device_forward,
                    device_loss, device_pack_inputs, init_params)
from .partition import PartitionSet
from .sampler import EpochSampler, build_view

_DROPOUT_STREAM_OFFSET = 0x9E3779B9


def _torch():
    import torch
    return torch


@dataclass
class TrainConfig:
    """ref:trainer.py:35-56."""
    epochs: int = 1
    batch_size: Optional[int] = None
    fixed_num_batches: Optional[int] = None
    learning_rate: float = 0.01
    optimizer: str = "adam"
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    seed: int = 0
    eval_every: int = 0
    grad_clip: Optional[float] = None
    mp_start: str = "fork"

    def __post_init__(self):
        if self.learning_rate <= 0:
            raise ValidationError("learning_rate must be > 0")
        if self.optimizer not in ("sgd", "adam"):
            raise ValidationError(f"unknown optimizer {self.optimizer!r}")
        if self.epochs < 0:
            raise ValidationError("epochs must be >= 0")


# ---------------------------------------------------------------------------
# Reduction (ref:trainer.py:63-86)
# ---------------------------------------------------------------------------

def _flat_device(arrays, dtype, dev):
    torch = _torch()
    flat = np.concatenate([np.asarray(a, dtype=dtype).reshape(-1) for a in arrays]) if arrays else \
        np.zeros(0, dtype=dtype)
    return torch.as_tensor(flat).to(dev)


def _unflatten(flat: np.ndarray, shapes: list) -> list:
    outs, o = [], 0
    for s in shapes:
        k = int(np.prod(s)) if len(s) else 1
        outs.append(flat[o:o + k].reshape(s))
        o += k
    return outs


def allreduce_mean(payloads: list) -> list:
    """Elementwise mean of gradient payloads in the fixed pairwise-tree order
    (ref:trainer.py:63-86), on the device. float32 payloads go through the
    training kernel's fused tree-mean (kg_dense_step, an SGD step of lr = 1 on
    a zero parameter); anything else is reduced in float64 by
    kg_tree_mean_f64. Either way the arithmetic is the reference's, element
    for element, so results are bit-identical to numpy's (the mean of
    identical payloads is the payload for power-of-two P)."""
    if not payloads:
        raise ProtocolError("empty reduction")
    shapes = [np.shape(a) for a in payloads[0]]
    for p in payloads[1:]:
        if [np.shape(a) for a in p] != shapes:
            raise ProtocolError("gradient payloads disagree in shape")
    torch = _torch()
    lib = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    all32 = all(np.asarray(a).dtype == np.float32 for p in payloads for a in p)
    n = sum(int(np.prod(s)) if len(s) else 1 for s in shapes)
    if all32:
        g = torch.stack([_flat_device(p, np.float32, dev) for p in payloads]) if n else None
        out = torch.zeros(n, dtype=torch.float32, device=dev)
        if n:
            flags = torch.zeros(1, dtype=torch.int32, device=dev)
            ws = torch.empty(lib.kg_optim_workspace_bytes(n), dtype=torch.uint8, device=dev)
            # p = 0 - 1 * mean  ->  -mean
            _lib.call("kg_dense_step", out.data_ptr(), 0, 0, g.data_ptr(), len(payloads), n, 0, 1.0, 0.9, 0.999,
                      1e-8, 1.0, 1.0, 0, 0.0, flags.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_handle())
        res = (-out).cpu().numpy()
    else:
        g = torch.stack([_flat_device(p, np.float64, dev) for p in payloads])
        out = torch.empty(n, dtype=torch.float64, device=dev)
        _lib.call("kg_tree_mean_f64", g.data_ptr(), len(payloads), n, out.data_ptr(), _lib.stream_handle())
        res = out.cpu().numpy()
    return [a.copy() for a in _unflatten(res, shapes)]


# ---------------------------------------------------------------------------
# Optimizer (ref:trainer.py:93-151)
# ---------------------------------------------------------------------------

class Optimizer:
    """SGD or Adam over the dense blocks plus lazy sparse rows of the entity
    table (ref:trainer.py:93-151), computed on the device in float64 by
    kg_dense_step_f64 / kg_sparse_step_f64 with the reference's operation
    order, so the numpy ModelParams passed to step() are updated exactly as
    the reference updates them: dense blocks in place, and only the rows
    `entity_embed[embed_ids]` of the table (duplicates: last one wins, as with
    numpy fancy assignment). Moments stay resident on the device. The
    training loop itself uses the fused fp32 kernels (Trainer)."""

    def __init__(self, config: TrainConfig, params: ModelParams):
        torch = _torch()
        _lib.require_cuda()
        self.config = config
        self.t = 0
        self._adam = config.optimizer == "adam"
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self._shapes = [b.shape for b in params.dense_blocks()]
        n = sum(b.size for b in params.dense_blocks())
        f64 = dict(dtype=torch.float64, device=self.dev)
        self._m = torch.zeros(n if self._adam else 0, **f64)
        self._v = torch.zeros(n if self._adam else 0, **f64)
        self._em = self._ev = None
        if self._adam and params.entity_embed is not None:
            self._em = torch.zeros(params.entity_embed.shape, **f64)
            self._ev = torch.zeros(params.entity_embed.shape, **f64)

    @staticmethod
    def _blocks_of(flat_dev, shapes) -> list:
        return [a.copy() for a in _unflatten(flat_dev.cpu().numpy(), shapes)]

    @property
    def m(self) -> list:
        """First moments of the dense blocks (reference layout: one array per block)."""
        return self._blocks_of(self._m, self._shapes)

    @property
    def v(self) -> list:
        return self._blocks_of(self._v, self._shapes)

    @property
    def em(self):
        return None if self._em is None else self._em.cpu().numpy()

    @property
    def ev(self):
        return None if self._ev is None else self._ev.cpu().numpy()

    def step(self, params: ModelParams, dense_grads: list, embed_ids: Optional[np.ndarray] = None,
             embed_rows: Optional[np.ndarray] = None) -> None:
        torch = _torch()
        lib = _lib.require_cuda()
        cfg = self.config
        self.t += 1
        blocks = params.dense_blocks()
        if len(blocks) != len(dense_grads):
            raise ProtocolError("gradient/parameter block count mismatch")
        st = _lib.stream_handle()
        lr = float(cfg.learning_rate)
        bc1 = 1.0 - cfg.beta1 ** self.t
        bc2 = 1.0 - cfg.beta2 ** self.t
        adam = 1 if self._adam else 0
        p = _flat_device(blocks, np.float64, self.dev)
        n = p.numel()
        flags = torch.zeros(1, dtype=torch.int32, device=self.dev)
        if n:
            g = _flat_device(dense_grads, np.float64, self.dev)
            ws = torch.empty(lib.kg_dense_step_f64_workspace_bytes(n), dtype=torch.uint8, device=self.dev)
            clip = float(cfg.grad_clip) if cfg.grad_clip is not None else -1.0
            _lib.call("kg_dense_step_f64", p.data_ptr(), _lib.ptr(self._m if adam else None),
                      _lib.ptr(self._v if adam else None), g.data_ptr(), n, adam, lr, cfg.beta1, cfg.beta2,
                      cfg.adam_eps, bc1, bc2, clip, flags.data_ptr(), ws.data_ptr(), ws.numel(), st)
        if embed_ids is not None and params.entity_embed is not None and len(embed_ids):
            table = params.entity_embed
            ids_np = np.asarray(embed_ids, dtype=np.int64).reshape(-1)
            rows_np = np.asarray(embed_rows, dtype=np.float64).reshape(len(ids_np), table.shape[1])
            k, d = len(ids_np), table.shape[1]
            ids = torch.as_tensor(ids_np).to(self.dev)
            old = torch.as_tensor(np.ascontiguousarray(table[ids_np], dtype=np.float64)).to(self.dev)
            grows = torch.as_tensor(np.ascontiguousarray(rows_np)).to(self.dev)
            out = torch.empty((k, d), dtype=torch.float64, device=self.dev)
            wsb = lib.kg_sparse_step_f64_workspace_bytes(k, d, table.shape[0])
            ws2 = torch.empty(wsb, dtype=torch.uint8, device=self.dev)
            _lib.call("kg_sparse_step_f64", old.data_ptr(), grows.data_ptr(), ids.data_ptr(), k, d,
                      _lib.ptr(self._em), _lib.ptr(self._ev), table.shape[0], adam, lr, cfg.beta1, cfg.beta2,
                      cfg.adam_eps, bc1, bc2, out.data_ptr(), ws2.data_ptr(), ws2.numel(), st)
            table[ids_np] = out.cpu().numpy()
        if n:
            flat = p.cpu().numpy()
            o = 0
            for b in blocks:
                b[...] = flat[o:o + b.size].reshape(b.shape)
                o += b.size
        if int(flags.item()):
            raise NumericError("non-finite parameter after optimizer step")


def optimizer_step(params: ModelParams, averaged_grads, config: TrainConfig, optimizer: Optimizer) -> ModelParams:
    """Apply one synchronized update: dense averaged blocks plus the caller's
    own sparse embedding rows (ref:trainer.py:154-160)."""
    optimizer.step(params, averaged_grads.dense_blocks(), averaged_grads.embed_ids, averaged_grads.embed_rows)
    return params


# ---------------------------------------------------------------------------
# Report (ref:trainer.py:272-301)
# ---------------------------------------------------------------------------

@dataclass
class TrainReport:
    rounds_per_epoch: int
    batch_sizes: list
    epoch_seconds: list = field(default_factory=list)
    loss_curve: list = field(default_factory=list)
    val_mrr: list = field(default_factory=list)
    cg_build_per_batch: list = field(default_factory=list)
    encode_per_batch: list = field(default_factory=list)
    loss_step_per_batch: list = field(default_factory=list)
    setup_seconds: float = 0.0       # Trainer construction (views, uploads, graph captures)
    finish_seconds: float = 0.0      # replica check + parameter snapshot to host

    def mean_timings(self) -> dict:
        def m(x):
            return float(np.mean(x)) if x else 0.0
        return {"epoch_time": m(self.epoch_seconds), "cg_build": m(self.cg_build_per_batch),
                "encode": m(self.encode_per_batch), "loss_step": m(self.loss_step_per_batch)}

    def format_metrics(self) -> str:
        lines = []
        for e, (loss, secs) in enumerate(zip(self.loss_curve, self.epoch_seconds)):
            parts = [f"epoch={e}", f"loss={loss:.6f}", f"time={secs:.3f}"]
            mrr = dict(self.val_mrr).get(e)
            if mrr is not None:
                parts.append(f"val_mrr={mrr:.4f}")
            lines.append(" ".join(parts))
        return "\n".join(lines)


def _plan_sizes(num_cores: list, s: int, train_config: TrainConfig) -> tuple:
    lens = [c * (s + 1) for c in num_cores]
    if any(L == 0 for L in lens):
        raise ValidationError("a partition has no core edges to train on")
    if train_config.fixed_num_batches is not None:
        rounds = train_config.fixed_num_batches
        return [max(1, math.ceil(L / rounds)) for L in lens], rounds
    sizes = [train_config.batch_size or L for L in lens]
    return sizes, max(math.ceil(L / b) for L, b in zip(lens, sizes))


def _plan_batches(views: list, model_config: ModelConfig, train_config: TrainConfig) -> tuple:
    """Per-worker batch size and the shared number of reduction rounds
    (ref:trainer.py:304-316): stream length L_w = num_core_w * (s + 1);
    fixed_num_batches -> b_w = ceil(L_w / rounds), else b_w = batch_size or
    L_w and rounds = max_w ceil(L_w / b_w)."""
    return _plan_sizes([v.num_core for v in views], model_config.negatives_per_positive, train_config)


def _assemble_embed(pset: PartitionSet, tables, base: np.ndarray) -> np.ndarray:
    """Merge per-worker embedding tables, taking each vertex's row from the
    lowest-id partition holding it as a core-edge endpoint, else the initial
    row (ref:trainer.py:319-333). tables: list indexed like pset.partitions
    (the reference's form), or a dict worker index -> table holding only
    this process's workers."""
    out = base.copy()
    owner = np.full(len(base), -1, dtype=np.int64)
    for part in sorted(pset.partitions, key=lambda p: p.id):
        ends = np.concatenate([part.core_vertices, part.replicated_vertices]).astype(np.int64)
        free = ends[owner[ends] < 0]
        owner[free] = part.id
    items = tables.items() if isinstance(tables, dict) else enumerate(tables)
    for wid, table in items:
        rows = np.flatnonzero(owner == pset.partitions[wid].id)
        if len(rows):
            out[rows] = table[rows]
    return out


# ---------------------------------------------------------------------------
# Device engine
# ---------------------------------------------------------------------------

PREP_BRANCHES = int(os.environ.get("KG_PREP_BRANCHES", "4"))   # <= KG_PREP_MAX_BRANCHES
# eager rounds before the round graphs are captured (KG_EAGER_WARMUP; 0: the
# first round is captured directly — lazy workspaces grow inside the capture,
# from the graph's memory pool, and the library's kernels are preloaded)
EAGER_WARMUP = int(os.environ.get("KG_EAGER_WARMUP", "0"))
# train(): capture every round / epoch graph during setup, so the reported
# epoch times are steady state (needs EAGER_WARMUP = 0)
PREPARE_IN_SETUP = os.environ.get("KG_PREPARE_IN_SETUP", "1") == "1" and EAGER_WARMUP == 0


def _align256(x: int) -> int:
    return (int(x) + 255) // 256 * 256


class _RoundPrep:
    """Batch-only per-round work of a whole epoch — the closure (order, pos,
    counts) and the loss grouping (sorted values, segment bounds) of every
    round — computed on the epoch sampler's side stream while the previous
    epoch trains, into per-slot slabs. A training round then starts with one
    kg_copy_segments launch indexed by the device round counter."""

    def __init__(self, worker, rounds: int):
        torch = _torch()
        lib = _lib.require_cuda()
        self.w = worker
        v, cfg, b = worker.view, worker.config, worker.b
        self.rounds, self.n, self.L1 = max(rounds, 1), v.n, cfg.num_layers + 1
        dev = v.device
        i32 = dict(dtype=torch.int32, device=dev)
        # slab memory grows with rounds x n: refuse up front (with the numbers)
        # rather than fail inside an allocation deep in the epoch pipeline
        slab = EpochSampler.NSLOTS * self.rounds * (8 * self.n + 4 * self.L1 +
                                                     lib.kg_loss_workspace_bytes(b, v.n, cfg.dims[-1],
                                                                                 cfg.num_relations))
        # (the free-memory query is a driver round trip: only for slabs that
        # could matter against the device's memory)
        budget = int(os.environ["KG_PREP_SLAB_BYTES"]) if "KG_PREP_SLAB_BYTES" in os.environ else None
        if budget is None and slab > (1 << 30):
            budget = int(0.5 * torch.cuda.mem_get_info(dev)[0])
        if budget is not None and slab > budget:
            raise ValidationError(
                f"epoch pre-sampling needs {slab / 2**30:.1f} GiB for {self.rounds} rounds of "
                f"{self.n} vertices (budget {budget / 2**30:.1f} GiB, KG_PREP_SLAB_BYTES); use a larger "
                f"batch_size / fewer rounds per epoch")
        self.slabs = [dict(order=torch.empty((self.rounds, self.n), **i32), pos=torch.empty((self.rounds, self.n), **i32),
                           counts=torch.zeros((self.rounds, self.L1), **i32))
                      for _ in range(EpochSampler.NSLOTS)]
        self.flags = torch.zeros(1, **i32)
        self.loss_args = (cfg.dims[-1], v.n, cfg.num_relations)
        # the rounds of an epoch are prepared as parallel branches, each with its
        # own closure / loss workspaces (256-byte aligned strides)
        self.branches = min(self.rounds, PREP_BRANCHES)
        self.loss_stride = _align256(lib.kg_loss_workspace_bytes(b, v.n, cfg.dims[-1], cfg.num_relations))
        self.closure_stride = _align256(lib.kg_closure_workspace_bytes(v.n))
        self.prep_ws = torch.empty(self.branches * self.loss_stride, dtype=torch.uint8, device=dev)
        self.closure_ws = torch.empty(self.branches * self.closure_stride, dtype=torch.uint8, device=dev)
        self.prep_fields = self._fields(self.prep_ws[: self.loss_stride])
        self.offs, o = [], 0
        for _, nb in self.prep_fields:
            self.offs.append(o)
            o += (nb + 255) // 256 * 256
        self.blob = o
        for sl in self.slabs:
            sl["groups"] = torch.empty(self.rounds * self.blob, dtype=torch.uint8, device=dev)

    def _fields(self, ws):
        d, n, R = self.loss_args
        ptrs = (ctypes.c_void_p * 16)()
        nbytes = (ctypes.c_int64 * 16)()
        k = _lib.require_cuda().kg_loss_group_fields(ws.data_ptr(), ws.numel(), self.w.b, n, d, R, ptrs, nbytes, 16)
        if k < 0:
            raise KGError("loss workspace layout mismatch")
        return [(int(ptrs[i] or 0), int(nbytes[i])) for i in range(k)]

    def run(self, slot: int, ds) -> None:
        """Enqueue every round of the epoch in `ds` (current stream = the
        sampler's side stream; captured into the sampler's epoch graph)."""
        sl = self.slabs[slot]
        w = self.w
        d, n, R = self.loss_args
        a = _lib.KgEpochPrepArgs(ctypes.pointer(w.view.csr()), w.config.num_layers, self.rounds,
                                 ds.triples.data_ptr(), ds.labels.data_ptr(), ds.total, w.b, d, R,
                                 sl["order"].data_ptr(), sl["pos"].data_ptr(), sl["counts"].data_ptr(),
                                 sl["groups"].data_ptr(), self.blob, self.flags.data_ptr(),
                                 self.closure_ws.data_ptr(), self.closure_stride, self.prep_ws.data_ptr(),
                                 self.loss_stride, self.branches)
        _lib.call("kg_epoch_prep", ctypes.byref(a), _lib.stream_handle())

    def import_round(self, slot: int, round_dev, loss_ws) -> None:
        """Copy round *round_dev of `slot` into the worker's working buffers."""
        sl, bufs = self.slabs[slot], self.w.bufs
        fields = self._fields(loss_ws)
        segs = (_lib.KgCopySeg * (3 + len(fields)))()
        n, L1 = self.n, self.L1
        for i, (dst, src, nb) in enumerate(((bufs.order, sl["order"], 4 * n), (bufs.pos, sl["pos"], 4 * n),
                                            (bufs.counts, sl["counts"], 4 * L1))):
            segs[i].dst, segs[i].src, segs[i].bytes, segs[i].src_round_stride = dst.data_ptr(), src.data_ptr(), nb, nb
        gbase = sl["groups"].data_ptr()
        for j, ((ptr, nb), off) in enumerate(zip(fields, self.offs)):
            g = segs[3 + j]
            g.dst, g.src, g.bytes, g.src_round_stride = ptr, gbase + off, nb, self.blob
        _lib.call("kg_copy_segments", segs, len(segs), round_dev.data_ptr(), 0, _lib.stream_handle())


_SETUP_MARKS = os.environ.get("KG_SETUP_TIMES", "0") == "1"
setup_marks: list = []


def _mark(name: str) -> None:
    """Diagnostics (KG_SETUP_TIMES=1): synchronised timestamps of the setup phases."""
    if _SETUP_MARKS:
        _torch().cuda.synchronize()
        setup_marks.append((name, time.perf_counter()))


def _init_params_device(config: ModelConfig, seed: int, num_entities: int, dev):
    """init_params(config, default_rng(seed), num_entities) with the embedding
    table — the one large draw (N x d uniforms) — drawn on the device from
    the generator's state after the dense blocks (kg_uniform_f64, bit-exact
    with numpy). Returns (params, device float64 table, (pinned host tensor,
    event)): params.entity_embed views the pinned host copy, complete once
    the event has fired."""
    import dataclasses
    torch = _torch()
    rng = np.random.default_rng(seed)
    params = init_params(dataclasses.replace(config, mode=MODE_FEATURE), rng)   # same draws up to the table
    d = config.dims[0]
    el = float(np.sqrt(3.0 / d))
    g = _lib.pcg_from_numpy(rng)
    table = torch.empty((num_entities, d), dtype=torch.float64, device=dev)
    _lib.call("kg_uniform_f64", ctypes.byref(g), num_entities * d, -el, el, table.data_ptr(), _lib.stream_handle())
    host = torch.empty((num_entities, d), dtype=torch.float64, pin_memory=True)
    host.copy_(table, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    params.entity_embed = host.numpy()
    return params, table, (host, ev)


_torch_warm = set()


def _warm_torch_kernels(dev) -> None:
    """Run, once per process and device, the few PyTorch elementwise /
    reduction / index kernels the round, epoch and sampler bodies use, on
    tiny tensors: CUDA loads kernels lazily, and loading these from PyTorch's
    large modules cost ~80-130 ms inside the first training epoch of a fresh
    process (its first-epoch time was 99-142 ms against 7 ms later, 17 ms
    with CUDA_MODULE_LOADING=EAGER)."""
    torch = _torch()
    if dev.index in _torch_warm:
        return
    _torch_warm.add(dev.index)
    i64 = torch.zeros(8, dtype=torch.int64, device=dev)
    i32 = torch.zeros(8, dtype=torch.int32, device=dev)
    f32 = torch.zeros(8, dtype=torch.float32, device=dev)
    i64.add_(1)
    i64.fill_(2)
    torch.mul(i64, i64, out=i64)
    i32.fill_(1)
    f32.fill_(1.0)
    src = torch.ones(1, dtype=torch.float32, device=dev)
    f32.index_copy_(0, i64[:1].zero_(), src)
    i64[2:3].copy_(i64.min().view(1))
    i64[3:4].copy_(i64.sum().view(1))
    i32[1:2].copy_(i32.min().view(1))
    _ = i32 + i32
    _ = f32[i64[:2]]
    _ = torch.stack([f32.sum(), f32[0], i32[0].double()])
    _ = i32.to(torch.int64)
    _ = f32.mean()
    _ = torch.cat([f32, f32])
    _ = torch.bitwise_or(i32, i32)


class _Worker:
    """Device state of one partition: view, buffers, RNG stream, local
    embedding rows and their Adam moments."""

    def __init__(self, wid, partition, pset, config: ModelConfig, tc: TrainConfig, b: int, params: ModelParams,
                 features, rounds: int = 1, epoch_pool=None, epoch_stream=None, embed_dev=None):
        torch = _torch()
        self.wid = wid
        _mark("worker")
        self.view = build_view(partition, pset.num_entities, pset.num_relations)
        _mark("view")
        self.b = b
        self.config = config
        dev = self.view.device
        # the worker's RNG stream (ref:trainer.py:185) lives on the device
        self.g_dev = _lib.pcg_to_device(
            _lib.pcg_from_numpy(np.random.default_rng(tc.seed ^ self.view.partition_id)), dev)
        # dropout stream (ref:trainer.py:186-187)
        self.g_drop = (_lib.pcg_to_device(_lib.pcg_from_numpy(
            np.random.default_rng((tc.seed ^ self.view.partition_id) + 0x9E3779B9)), dev)
            if config.dropout > 0.0 else None)
        if config.mode == MODE_EMBEDDING and embed_dev is not None:
            # the initial table was drawn on the device: gather this view's rows there
            self.input_rows = embed_dev.index_select(0, self.view.d_local_ids.long()).float()
        else:
            local = self.view.local_ids
            rows = params.entity_embed[local] if config.mode == MODE_EMBEDDING else features[local]
            self.input_rows = torch.as_tensor(np.ascontiguousarray(rows, dtype=np.float32)).to(dev)
        _mark("rng+rows")
        self.bufs = ViewBuffers(config, self.view, b, input_rows=self.input_rows)
        _mark("bufs")
        self.emb = config.mode == MODE_EMBEDDING
        if self.emb and tc.optimizer == "adam":
            self.em = torch.zeros_like(self.input_rows)
            self.ev = torch.zeros_like(self.input_rows)
        else:
            self.em = self.ev = None
        self.ws = _lib.Workspace(dev)
        self.stream = None
        # epoch e+1's negatives + shuffle are produced on a side stream while epoch e trains
        self.prep = _RoundPrep(self, rounds)
        _mark("roundprep")
        self.sampler = EpochSampler(self.view, config.negatives_per_positive, self.g_dev, prep=self.prep.run,
                                    pool=epoch_pool, side=epoch_stream)
        _mark("sampler")

    def begin_epoch(self):
        self.stream = self.sampler.next()

    def slot(self) -> int:
        return self.sampler.slot_of(self.stream)

    def closure(self, start_dev):
        from .sampler import closure_device
        closure_device(self.view, self.config.num_layers, stream=self.stream, start=0, size=self.b,
                       out=(self.bufs.order, self.bufs.pos, self.bufs.counts), ws=self.ws, start_dev=start_dev)


class Trainer:
    """The hot loop of ref:trainer.py:202-236 for the partitions this process
    owns. `run_round()` is one synchronized training round."""

    def __init__(self, pset: PartitionSet, graph, model_config: ModelConfig, train_config: TrainConfig,
                 initial_params: Optional[ModelParams] = None, graph_pools: bool = False):
        """graph_pools: capture into the process-wide persistent graph memory
        pools (train() does; the caller must close() the trainer, which
        synchronises, before another trainer on the device captures)."""
        torch = _torch()
        _lib.require_cuda()
        if pset.hops != model_config.num_layers:
            raise ValidationError(f"partitions expanded for {pset.hops} hops but model has "
                                  f"{model_config.num_layers} layers")
        if model_config.num_relations != pset.num_relations:
            raise ValidationError("model num_relations != partition set num_relations")
        self.pset, self.mc, self.tc = pset, model_config, train_config
        self.P = pset.num_parts
        dist = torch.distributed
        self.dist = dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
        self.world = dist.get_world_size() if self.dist else 1
        self.rank = dist.get_rank() if self.dist else 0
        if self.dist and self.P % self.world != 0:
            raise ValidationError(f"{self.P} partitions cannot be split evenly over {self.world} ranks")
        self.local_wids = [w for w in range(self.P) if w % self.world == self.rank]
        setup_marks.clear()
        _mark("start")
        self.dev = torch.device("cuda", torch.cuda.current_device())
        _warm_torch_kernels(self.dev)
        embed_dev = None
        if initial_params is not None:
            params = initial_params.copy()
        elif model_config.mode == MODE_EMBEDDING:
            params, embed_dev, self._embed_host = _init_params_device(model_config, train_config.seed,
                                                                      pset.num_entities, self.dev)
        else:
            params = init_params(model_config, np.random.default_rng(train_config.seed),
                                 num_entities=pset.num_entities)
        if model_config.mode == MODE_FEATURE:
            if graph.features is None:
                raise ValidationError("feature mode requires graph features")
            features = graph.features
        else:
            if params.entity_embed is None:
                raise ValidationError("embedding mode requires an entity table in params")
            features = None
        self.init_params = params
        self.sizes, self.rounds = _plan_sizes([p.num_core_edges for p in pset.partitions],
                                                model_config.negatives_per_positive, train_config)
        _mark("params")
        self.model = DeviceModel.from_params(model_config, params, self.dev)
        _mark("model")
        D = self.model.layout.total
        self.D = D
        self.graph_pools = graph_pools
        di = self.dev.index
        self.workers = [_Worker(w, pset.partitions[w], pset, model_config, train_config, self.sizes[w], params,
                                features, self.rounds,
                                epoch_pool=_lib.persistent_pool(("epoch", di, k)) if graph_pools else None,
                                epoch_stream=_lib.cached_stream(("epoch", di, k), self.dev) if graph_pools else None,
                                embed_dev=embed_dev)
                        for k, w in enumerate(self.local_wids)]
        del embed_dev
        if getattr(self, "_embed_host", None) is not None:
            self._embed_host[1].synchronize()   # the host copy of the initial table is complete
        nloc = len(self.workers)
        self.grads_local = torch.zeros((nloc, D), dtype=torch.float32, device=self.dev)
        self.grads_all = (torch.zeros((self.P, D), dtype=torch.float32, device=self.dev) if self.dist
                          else self.grads_local)
        self._peer = None
        if self.dist:
            self._recv = torch.empty((self.world * nloc, D), dtype=torch.float32, device=self.dev)
            self._gidx = payload_order(self.P, self.world, self.dev)
            # opt-in: measured at parity with NCCL at 2/4 ranks
            if self.P == self.world and os.environ.get("KG_PEER_GATHER", "0") == "1":
                self._peer = PeerExchange.create(D, self.rank, self.world, self.dev)
        self.m = torch.zeros(D, dtype=torch.float32, device=self.dev)
        self.v = torch.zeros(D, dtype=torch.float32, device=self.dev)
        self.flags = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.optim_ws = torch.empty(_lib.require_cuda().kg_optim_workspace_bytes(D), dtype=torch.uint8,
                                    device=self.dev)
        self.losses = torch.zeros((nloc, max(self.rounds, 1)), dtype=torch.float32, device=self.dev)
        self.loss_scratch = torch.zeros(nloc, dtype=torch.float32, device=self.dev)
        # per-round scalars live on the device so a captured round replays for every round
        self.step_dev = torch.zeros(1, dtype=torch.int64, device=self.dev)        # Adam step t
        self.start_dev = torch.zeros(nloc, dtype=torch.int64, device=self.dev)    # batch offsets r*b_w
        self.round_dev = torch.zeros(1, dtype=torch.int64, device=self.dev)       # r, advanced on device
        self.b_dev = torch.tensor([w.b for w in self.workers], dtype=torch.int64, device=self.dev)
        # CUDA graphs pay off over many rounds; short runs stay eager
        env = os.environ.get("KG_CUDA_GRAPHS", "auto")
        self.use_graphs = env == "1" or (env == "auto" and train_config.epochs * self.rounds >= 64)
        self.graph_kernel_launches = 0
        # optional: CUDA events around one kernel family, captured into the graphs
        self.timer_prefix = None
        self._timer_handles = {}
        self.last_timer_handle = None
        self._graphs = {}
        self._graph_pool = None
        # Training runs on high-priority streams: the sampler's epoch graphs
        # (default, low priority) then fill SM slots training leaves idle.
        def stream(name):
            return (_lib.cached_stream((name, self.dev.index), self.dev, priority=-2) if graph_pools
                    else torch.cuda.Stream(self.dev, priority=-2))
        self._prio = stream("prio")
        self._loss_stream = stream("loss")   # forked work beside the layers
        self._capture_stream = stream("capture")
        # diagnostics: KG_FORK_STREAMS=0 keeps every kernel on one stream
        self.fork_streams = os.environ.get("KG_FORK_STREAMS", "1") != "0"
        self.model.repack()
        _mark("trainer")
        self._eager_rounds = 0
        self.t = 0
        self.round_in_epoch = 0
        self.epoch = 0

    # -- one synchronized round ----------------------------------------------
    def begin_epoch(self):
        torch = _torch()
        for w in self.workers:
            w.begin_epoch()
        self.round_in_epoch = 0
        self.round_dev.zero_()
        self._epoch_start = torch.cuda.Event(enable_timing=True)
        self._epoch_start.record()

    def end_epoch(self):
        """Enqueue the epoch's bookkeeping: per-worker mean loss (and, with
        several ranks, the all-gathered (loss sum, count) of every rank), the
        non-finite flags (then cleared) and an end event; copied to pinned
        host memory without blocking. finish_epoch(handle) reads it."""
        torch = _torch()
        nloc = len(self.workers)
        flags = [w.bufs.flags for w in self.workers] + [self.flags]
        if getattr(self, "_ep_out", None) is None:
            self._ep_ptrs = torch.tensor([f.data_ptr() for f in flags], dtype=torch.int64, device=self.dev)
            self._ep_out = torch.empty(nloc + len(flags), dtype=torch.float64, device=self.dev)
            self._ep_all = torch.empty((self.world, nloc + len(flags)), dtype=torch.float64, device=self.dev)
        # one launch: per-worker mean round loss + the status words (cleared)
        _lib.call("kg_epoch_end", self.losses.data_ptr(), self.losses.shape[1], nloc, self.rounds,
                  self._ep_ptrs.data_ptr(), len(flags), self._ep_out.data_ptr(), _lib.stream_handle())
        out = self._ep_out
        if self.dist:
            # every rank's status words ride on the same all-gather, so all
            # ranks raise the same error at the same epoch
            torch.distributed.all_gather_into_tensor(self._ep_all, self._ep_out)
            out = self._ep_all
        host = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
        host.copy_(out, non_blocking=True)
        end = torch.cuda.Event(enable_timing=True)
        end.record()
        return (self._epoch_start, end, host, nloc)

    def finish_epoch(self, handle) -> tuple:
        """Wait for an end_epoch() handle; raise on non-finite values (any
        rank's, with several ranks), return (mean loss, device seconds of the
        epoch on this rank)."""
        start, end, host, nloc = handle
        end.synchronize()
        rows = host.numpy().reshape(-1, host.shape[-1])   # (ranks, nloc means + status words)
        f = 0
        for x in rows[:, nloc:].ravel().tolist():
            f |= int(x)
        raise_for_flags(f)
        loss = float(rows[:, :nloc].sum() / rows[:, :nloc].size)
        return loss, start.elapsed_time(end) / 1e3

    def _compute_body(self):
        """closure -> forward -> DistMult+BCE -> backward of every local worker
        (all per-round scalars read from device memory)."""
        torch = _torch()
        torch.mul(self.b_dev, self.round_dev, out=self.start_dev)
        main = torch.cuda.current_stream()
        for i, w in enumerate(self.workers):
            # closure + loss grouping of this round were precomputed with the
            # epoch (_RoundPrep); one copy brings them into the working buffers
            w.prep.import_round(w.slot(), self.round_dev, w.bufs.loss_ws(w.b))
            gslot = self.grads_local[i]
            side = self._loss_stream if self.fork_streams else main
            masks = device_dropout(w.bufs, w.g_drop, self.mc.dropout) if w.g_drop is not None else None
            side.wait_stream(main)
            with torch.cuda.stream(side):
                # backward operands that only need forward outputs, beside the forward:
                # layer 0's packed input rows and Y_0 = H_0 . [V_b]; the closure
                # positions of every CSC message (the backward's dZ gathers)
                device_csc_positions(w.bufs)
                device_pack_inputs(w.bufs)
                device_backward_y(self.model, w.bufs, 0)

            def after_layer(l, w=w):   # H_{l+1} is ready: Y_{l+1} on the forked stream
                if l + 1 < self.mc.num_layers:
                    side.wait_stream(main)
                    with torch.cuda.stream(side):
                        device_backward_y(self.model, w.bufs, l + 1)

            device_forward(self.model, w.bufs, packed=True, hpk=True, masks=masks, after_layer=after_layer)
            main.wait_stream(side)
            device_loss(self.model, w.bufs, w.stream, 0, w.b, gslot, self.loss_scratch[i:i + 1],
                        start_dev=self.start_dev[i:i + 1], part="compute",
                        side=self._loss_stream if self.fork_streams else None)
            device_backward(self.model, w.bufs, gslot, input_grad=w.emb,
                            side=self._loss_stream if self.fork_streams else None, packed=True, hpk=True,
                            masks=masks, y_ready=True)
            # the loss value comes from the forked stream, joined by device_backward
            self.losses[i].index_copy_(0, self.round_dev, self.loss_scratch[i:i + 1])

    def _update_body(self):
        """Fused tree-mean + dense Adam/SGD, then lazy sparse rows."""
        tc = self.tc
        self.step_dev.add_(1)
        adam = 1 if tc.optimizer == "adam" else 0
        st = _lib.stream_handle()
        _lib.call("kg_dense_step", self.model.flat.data_ptr(), self.m.data_ptr(), self.v.data_ptr(),
                  self.grads_all.data_ptr(), self.P, self.D, adam, tc.learning_rate, tc.beta1, tc.beta2,
                  tc.adam_eps, 1.0, 1.0, self.step_dev.data_ptr(),
                  float(tc.grad_clip) if tc.grad_clip is not None else 0.0,
                  self.flags.data_ptr(), self.optim_ws.data_ptr(), self.optim_ws.numel(), st)
        self.model.repack()   # tensor-core weight operands of the updated bases
        L = self.mc.num_layers
        for w in self.workers:
            if w.emb:
                _lib.call("kg_sparse_step", w.input_rows.data_ptr(), _lib.ptr(w.em), _lib.ptr(w.ev),
                          w.bufs.dH[0].data_ptr(), w.bufs.order.data_ptr(), w.bufs.counts.data_ptr(), L,
                          self.mc.dims[0], adam, tc.learning_rate, tc.beta1, tc.beta2, tc.adam_eps, 1.0, 1.0,
                          self.step_dev.data_ptr(), w.view.n, st)
        self.round_dev.add_(1)

    def run_round(self):
        """One synchronized round. After two eager warm-up rounds the compute
        and update halves are captured as CUDA graphs (one pair per epoch
        buffer slot) and replayed; the NCCL gather runs between them."""
        torch = _torch()
        cur = torch.cuda.current_stream()
        self._prio.wait_stream(cur)
        with torch.cuda.stream(self._prio):
            if not self.use_graphs or self._eager_rounds < EAGER_WARMUP:
                self._compute_body()
                if self.dist:
                    self._gather()
                self._update_body()
                self._eager_rounds += 1
            else:
                key = tuple(w.stream.triples.data_ptr() for w in self.workers)
                if key not in self._graphs:
                    self._capture_slot(self.workers[0].slot())
                gc, gu, nk = self._graphs[key]
                self.last_timer_handle = self._timer_handles.get(key)
                gc.replay()
                if self.dist:
                    self._gather()
                gu.replay()
                self.graph_kernel_launches += nk
        cur.wait_stream(self._prio)
        self.t += 1
        self.round_in_epoch += 1
        if self.round_in_epoch == 1:
            self.prefetch()    # the epoch's first round is queued: capture work ahead now

    def _capture(self, body, graph):
        torch = _torch()
        side = self._capture_stream
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            _lib.capture(graph, body, self._graph_pool)
        torch.cuda.current_stream().wait_stream(side)

    def _capture_slot(self, slot: int):
        """Capture the compute and update halves of a round for one epoch
        buffer slot of the samplers (pointers are fixed per slot)."""
        torch = _torch()
        lib = _lib.require_cuda()
        if self._graph_pool is None:
            self._graph_pool = (_lib.persistent_pool(("round", self.dev.index)) if self.graph_pools
                                else torch.cuda.graph_pool_handle())
        current = [w.stream for w in self.workers]
        for w in self.workers:
            w.stream = w.sampler.slot_stream(slot)
        key = tuple(w.stream.triples.data_ptr() for w in self.workers)
        gc, gu = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        n0 = lib.kg_launch_count()
        if self.timer_prefix:
            lib.kg_kernel_timer_begin(self.timer_prefix.encode())
        self._capture(self._compute_body, gc)
        if self.timer_prefix:
            h = ctypes.c_int64(-1)
            lib.kg_kernel_timer_detach(ctypes.byref(h))
            self._timer_handles[key] = h.value
        self._capture(self._update_body, gu)
        self._graphs[key] = (gc, gu, lib.kg_launch_count() - n0)
        for w, st in zip(self.workers, current):
            w.stream = st

    def prefetch(self) -> bool:
        """Host-side preparation of upcoming epochs (sampler epoch graphs,
        round graphs of a slot not captured yet), one item per call; meant
        for moments when the device has queued rounds to run. True if it did
        something."""
        for w in self.workers:
            if w.sampler.prefetch():
                return True
        if self.use_graphs and self._eager_rounds >= EAGER_WARMUP:
            for slot in range(EpochSampler.NSLOTS):
                key = tuple(w.sampler.slot_stream(slot).triples.data_ptr() for w in self.workers)
                if key not in self._graphs:
                    self._capture_slot(slot)
                    return True
        if self.P > 1 and self.mc.mode == MODE_EMBEDDING and getattr(self, "_snap_plan", None) is None \
                and self.t > 0:
            self._snapshot_plan()   # host work for the final snapshot, while the device trains
        return False

    def prepare(self, first_epoch: bool = False) -> None:
        """Do all pending one-time host work now (epoch graphs of the slots
        ahead, round graphs of every slot): for benchmarks, so the timed steps
        are steady state. first_epoch: only until the round graphs of the
        first epoch's slot exist (train(): the other slots are captured by
        prefetch() while the device runs epochs, overlapping the host work)."""
        while True:
            if first_epoch and self.use_graphs:
                key = tuple(w.sampler.slot_stream(w.sampler.parity).triples.data_ptr() for w in self.workers)
                if key in self._graphs:
                    return
            if not self.prefetch():
                return

    def close(self):
        """Release the captured CUDA graphs now and break the worker <->
        sampler <-> round-prep reference cycle, so the device buffers go back
        to the caching allocator as soon as the trainer is dropped (instead of
        whenever the cyclic GC runs; a following train() then reuses them)."""
        if getattr(self, "_closed", False):
            return
        self._closed = True
        _torch().cuda.synchronize()
        self._graphs.clear()
        if self._peer is not None:
            self._peer.close()      # collective: every rank closes its trainer (train() does)
            self._peer = None
        for w in self.workers:
            w.sampler.close()
            w.sampler._prep = None
            w.prep.w = None

    def _gather(self):
        if self._peer is not None:
            self._peer.exchange(self.grads_local, self.grads_all, self.workers[0].bufs.flags)
        else:
            gather_partition_payloads(self.grads_local, self.P, self.world, self.grads_all, self._recv, self._gidx)

    def check(self):
        for w in self.workers:
            check_flags(w.bufs)
        f = int(self.flags.item())
        if f:
            self.flags.zero_()
            raise_for_flags(f)

    def epoch_losses(self) -> list:
        return self.losses[:, : self.rounds].mean(dim=1).double().cpu().tolist()

    # -- host snapshots ------------------------------------------------------
    def local_tables(self) -> dict:
        """Partition index -> full (N, d_in) table with this worker's rows."""
        out = {}
        base = self.init_params.entity_embed
        for w in self.workers:
            lids = w.view.local_ids
            rows = w.input_rows.cpu().numpy()          # fp32 off the device, widened on the host
            if len(lids) == len(base) and lids[0] == 0 and lids[-1] == len(base) - 1 and \
                    bool((np.diff(lids) == 1).all()):
                t = rows.astype(np.float64)            # the partition holds every row, in id order
            else:
                t = base.copy()
                t[lids] = rows
            out[w.wid] = t
        return out

    def snapshot(self) -> ModelParams:
        p0 = self.init_params
        if self.mc.mode == MODE_EMBEDDING:
            emb = self.local_tables()[0] if self.P == 1 else self._gather_owned_rows()
        else:
            emb = None if p0.entity_embed is None else p0.entity_embed.copy()
        # dense blocks come fresh from the device; the table is built once (no
        # copy of the initial table that is then overwritten)
        params = ModelParams(list(p0.bases), list(p0.coeffs), p0.decoder, emb)
        params.set_dense_blocks(self.model.dense_blocks())
        return params

    def _gather_owned_rows(self) -> np.ndarray:
        """Final embedding table for P > 1: only the rows each partition owns
        (lowest-id partition holding the vertex as a core endpoint,
        ref:trainer.py:319-333 — the rule of _assemble_embed) leave the
        device; over several ranks as one padded NCCL all-gather of (global
        id, fp32 row) pairs instead of a pickled full (N, d) table per
        partition."""
        torch = _torch()
        dist = torch.distributed
        base = self.init_params.entity_embed
        ids, sels, covered = self._snapshot_plan()
        rows = torch.cat([w.input_rows[sel] for w, sel in zip(self.workers, sels)])
        if not self.dist:
            out = np.empty_like(base) if covered else base.copy()
            out[ids.cpu().numpy()] = rows.cpu().numpy()
            return out
        k = torch.tensor([ids.numel()], dtype=torch.int64, device=self.dev)
        counts = torch.empty(self.world, dtype=torch.int64, device=self.dev)
        dist.all_gather_into_tensor(counts, k)
        counts = counts.cpu().tolist()
        kmax, d = max(max(counts), 1), rows.shape[1]
        ids_p = torch.full((kmax,), -1, dtype=torch.int64, device=self.dev)
        rows_p = torch.zeros((kmax, d), dtype=rows.dtype, device=self.dev)
        ids_p[: ids.numel()] = ids
        rows_p[: ids.numel()] = rows
        ids_all = torch.empty((self.world, kmax), dtype=torch.int64, device=self.dev)
        rows_all = torch.empty((self.world, kmax, d), dtype=rows.dtype, device=self.dev)
        dist.all_gather_into_tensor(ids_all, ids_p)
        dist.all_gather_into_tensor(rows_all, rows_p)
        ids_all, rows_all = ids_all.cpu().numpy(), rows_all.cpu().numpy()
        out = np.empty_like(base) if covered else base.copy()
        for r, c in enumerate(counts):
            out[ids_all[r, :c]] = rows_all[r, :c]
        return out

    def _snapshot_plan(self):
        """(global ids of the rows this rank's partitions own (device), the
        owned local rows per worker (device index tensors), whether the
        partitions own every entity): the ownership rule of
        ref:trainer.py:319-333, computed once (prefetch() does it while the
        device runs an epoch, so the final snapshot only moves rows)."""
        if getattr(self, "_snap_plan", None) is None:
            torch = _torch()
            n = len(self.init_params.entity_embed)
            owner = np.full(n, -1, dtype=np.int64)
            for part in sorted(self.pset.partitions, key=lambda p: p.id):
                ends = np.concatenate([part.core_vertices, part.replicated_vertices]).astype(np.int64)
                owner[ends[owner[ends] < 0]] = part.id
            ids, sels = [], []
            for w in self.workers:
                lids = np.asarray(w.view.local_ids, dtype=np.int64)
                sel = np.flatnonzero(owner[lids] == self.pset.partitions[w.wid].id)
                ids.append(lids[sel])
                # pinned, non-blocking: a pageable upload would wait for the
                # epoch queued on the stream (this runs inside the epoch loop)
                sels.append(torch.from_numpy(sel).pin_memory().to(self.dev, non_blocking=True))
            ids = torch.from_numpy(np.concatenate(ids)).pin_memory().to(self.dev, non_blocking=True)
            self._snap_plan = (ids, sels, bool((owner >= 0).all()))
        return self._snap_plan

    def check_replicas(self):
        """Dense replicas must be bitwise equal on every rank (ref:trainer.py:465-469)."""
        if not self.dist:
            return
        torch = _torch()
        mine = self.model.flat.clone()
        allr = torch.empty((self.world, self.D), dtype=torch.float32, device=self.dev)
        torch.distributed.all_gather_into_tensor(allr, mine)
        for r in range(1, self.world):
            if not torch.equal(allr[0], allr[r]):
                raise ProtocolError(f"replica divergence: rank {r} dense blocks differ from rank 0")


class PeerExchange:
    """Dense-payload exchange over NVLink peer memory (one partition per rank,
    one node): every rank publishes its payload into its own IPC-shared region
    and reads all P regions straight into the tree-mean input, in partition
    order (the gather of ref:trainer.py:430-438, csrc/kg_peer.cu). Created only
    when every rank can map every peer; otherwise the NCCL all-gather runs."""

    def __init__(self, n, rank, world, dev, region, opened, regions_dev, seq):
        self.n, self.rank, self.world, self.dev = n, rank, world, dev
        self.region, self.opened, self.regions_dev, self.seq = region, opened, regions_dev, seq

    @classmethod
    def create(cls, n: int, rank: int, world: int, dev):
        torch = _torch()
        dist = torch.distributed
        lib = _lib.require_cuda()
        import socket
        # physical identity of every rank's GPU: device ordinals are local to
        # each process (CUDA_VISIBLE_DEVICES per rank makes them all 0)
        props = torch.cuda.get_device_properties(dev)
        me = (socket.gethostname(), str(getattr(props, "uuid", "")) or f"{dev.index}")
        where = [None] * world
        dist.all_gather_object(where, me)
        ok = all(h == me[0] for h, _ in where) and len({u for _, u in where}) == world
        votes = [None] * world
        dist.all_gather_object(votes, bool(ok))
        if not all(votes):
            return None
        region = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        _lib.check(lib.kg_peer_alloc(lib.kg_peer_region_bytes(n), ctypes.byref(region), handle), "kg_peer_alloc")
        handles = [None] * world
        dist.all_gather_object(handles, handle.raw)
        ptrs, opened, failed = [], [], False
        for r, h in enumerate(handles):
            if r == rank:
                ptrs.append(region.value)
                continue
            peer = ctypes.c_void_p()
            if lib.kg_peer_open(ctypes.create_string_buffer(h, 64), ctypes.byref(peer)) != 0:
                failed = True         # no peer mapping (e.g. no P2P path): fall back to NCCL
                break
            ptrs.append(peer.value)
            opened.append(peer.value)
        votes = [None] * world
        dist.all_gather_object(votes, not failed)
        if not all(votes):
            for q in opened:
                lib.kg_peer_close(q, 0)
            lib.kg_peer_close(region.value, 1)
            return None
        regions_dev = torch.tensor(ptrs, dtype=torch.int64, device=dev)
        seq = torch.zeros(3, dtype=torch.int64, device=dev)
        dist.barrier()            # every region is zeroed and mapped before the first publish
        return cls(n, rank, world, dev, region.value, opened, regions_dev, seq)

    def exchange(self, local, out, flags):
        torch = _torch()
        st = torch.cuda.current_stream().cuda_stream
        _lib.call("kg_peer_publish", local.data_ptr(), self.region, self.n, self.seq.data_ptr(), st)
        _lib.call("kg_peer_gather", self.regions_dev.data_ptr(), self.world, self.n, out.data_ptr(),
                  self.seq.data_ptr(), flags.data_ptr(), st)

    def close(self):
        torch = _torch()
        lib = _lib.require_cuda()
        torch.cuda.synchronize()
        torch.distributed.barrier()   # no peer still reads this rank's region
        for p in self.opened:
            lib.kg_peer_close(p, 0)
        lib.kg_peer_close(self.region, 1)
        self.opened, self.region = [], None


def payload_order(P: int, world: int, device):
    """Rank r owns partitions r, r+W, ...: slot j of rank r is partition
    r + j*W. Index that reorders the all-gathered slots into partition order
    (the payload order of ref:trainer.py:430-438)."""
    torch = _torch()
    nloc = P // world
    return torch.tensor([(p % world) * nloc + p // world for p in range(P)], dtype=torch.long, device=device)


def gather_partition_payloads(local, P: int, world: int, out, recv=None, order=None):
    """All-gather every rank's (P/W, D) gradient payloads into `out` (P, D)
    in partition order; the fused tree-mean then runs on identical inputs on
    every rank. NCCL on device tensors (gloo for CPU tests)."""
    torch = _torch()
    dist = torch.distributed
    nloc, D = local.shape
    if recv is None:
        recv = torch.empty((world * nloc, D), dtype=local.dtype, device=local.device)
    if order is None:
        order = payload_order(P, world, local.device)
    if local.is_cuda:
        dist.all_gather_into_tensor(recv, local)
    else:
        dist.all_gather(list(recv.chunk(world)), local)
    torch.index_select(recv, 0, order, out=out)
    return out


def train(pset: PartitionSet, graph, model_config: ModelConfig, train_config: TrainConfig,
          initial_params: Optional[ModelParams] = None, eval_fn=None) -> tuple:
    """Synchronized data-parallel training; returns (params, report)
    (ref:trainer.py:336-480). eval_fn(params) -> float is called at epochs
    selected by train_config.eval_every."""
    torch = _torch()
    t_setup = time.perf_counter()
    tr = Trainer(pset, graph, model_config, train_config, initial_params, graph_pools=True)
    try:
        return _train_loop(tr, train_config, eval_fn, t_setup)
    finally:
        tr.close()   # synchronises before the graphs (and their pool memory) are released


def _train_loop(tr, train_config, eval_fn, t_setup) -> tuple:
    torch = _torch()
    if PREPARE_IN_SETUP:
        # every slot's graphs captured before epoch 0, so every reported epoch
        # time is steady state (capturing the later slots during the first
        # epochs overlapped host work but put capture stalls into short epochs)
        tr.prepare()
    _mark("prepare")
    torch.cuda.synchronize()
    report = TrainReport(rounds_per_epoch=tr.rounds, batch_sizes=list(tr.sizes),
                         setup_seconds=time.perf_counter() - t_setup)
    tc = train_config
    _mark("train_setup")
    eval_epochs = frozenset(e for e in range(tc.epochs)
                            if tc.eval_every and (e + 1) % tc.eval_every == 0) if eval_fn is not None else frozenset()
    # Epoch-end bookkeeping (losses, non-finite flags, device epoch time) is
    # read back one epoch late, so the device queue never drains between
    # epochs; an eval epoch is settled at once (it needs a snapshot anyway).
    pending = []

    def settle():
        e, h = pending.pop(0)
        losses, secs = tr.finish_epoch(h)
        report.loss_curve.append(losses)
        report.epoch_seconds.append(secs)
        nb = tr.P * tr.rounds
        report.cg_build_per_batch.append(0.0)
        report.encode_per_batch.append(0.0)
        report.loss_step_per_batch.append(secs * (tr.P if not tr.dist else 1) / nb)
        if e in eval_epochs:
            report.val_mrr.append((e, float(eval_fn(tr.snapshot()))))

    for epoch in range(tc.epochs):
        tr.begin_epoch()
        for _ in range(tr.rounds):
            tr.run_round()
        pending.append((epoch, tr.end_epoch()))
        tr.prefetch()      # host-side capture work while the device runs this epoch
        if epoch < 3:
            _mark(f"epoch{epoch}")
        while len(pending) > 1 or (pending and pending[-1][0] in eval_epochs):
            settle()
    while pending:
        settle()
    if tr.dist:
        # epoch time = max over ranks (one collective for the whole run)
        secs = torch.tensor(report.epoch_seconds, dtype=torch.float64, device=tr.dev)
        torch.distributed.all_reduce(secs, op=torch.distributed.ReduceOp.MAX)
        report.epoch_seconds = secs.cpu().tolist()
        report.loss_step_per_batch = [x / (tr.P * tr.rounds) for x in report.epoch_seconds]
    t_fin = time.perf_counter()
    tr.check_replicas()
    params = tr.snapshot()
    _mark("snapshot")
    tr.close()
    _mark("close")
    report.finish_seconds = time.perf_counter() - t_fin
    return params, report


# Reference module-level names that live in io.py here (ref:trainer.py:487-528); resolved
# lazily so `from <pkg>.trainer import X` works as with the reference.
_IO_NAMES = ('bench_components', 'format_bench_rows')


def __getattr__(name):
    if name in _IO_NAMES:
        from . import io
        return getattr(io, name)
    raise AttributeError(name)
