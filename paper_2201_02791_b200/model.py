"""RGCN encoder (basis-decomposed) + DistMult decoder with BCE loss and exact
gradients, executed by the sm_100a kernels (drop-in for ref:model.py).

Host API objects (ModelConfig, ModelParams, Gradients) keep the reference's
fields and float64 numpy arrays; the device engine keeps every dense block in
one flat fp32 buffer in `dense_blocks()` order
[bases_0..bases_{L-1}, coeffs_0..coeffs_{L-1}, decoder], which is also the
all-reduce payload layout, and every activation in (n_local, d) buffers
indexed by partition-local vertex id.
"""

from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .errors import FormatError, IntegrityError, NumericError, ProtocolError, ShapeError, ValidationError

MODE_FEATURE = "feature"
MODE_EMBEDDING = "embedding"


@dataclass
class ModelConfig:
    """ref:model.py:26-57."""
    num_layers: int
    dims: list
    num_bases: int
    num_relations: int
    negatives_per_positive: int = 1
    dropout: float = 0.0
    mode: str = MODE_FEATURE

    def __post_init__(self):
        if self.num_layers < 1:
            raise ValidationError("num_layers must be >= 1")
        if self.num_bases < 1:
            raise ValidationError("num_bases must be >= 1")
        if len(self.dims) != self.num_layers + 1:
            raise ValidationError("dims must have num_layers + 1 entries")
        if self.mode not in (MODE_FEATURE, MODE_EMBEDDING):
            raise ValidationError(f"unknown mode {self.mode!r}")
        if not 0.0 <= self.dropout < 1.0:
            raise ValidationError("dropout must be in [0, 1)")

    @property
    def num_rel_groups(self) -> int:
        return 2 * self.num_relations + 1

    def to_json(self) -> str:
        return json.dumps({"num_layers": self.num_layers, "dims": list(self.dims),
                           "num_bases": self.num_bases, "num_relations": self.num_relations,
                           "negatives_per_positive": self.negatives_per_positive,
                           "dropout": self.dropout, "mode": self.mode})

    @classmethod
    def from_json(cls, blob: str) -> "ModelConfig":
        return cls(**json.loads(blob))


@dataclass
class ModelParams:
    """ref:model.py:64-98 (float64 host arrays)."""
    bases: list
    coeffs: list
    decoder: np.ndarray
    entity_embed: Optional[np.ndarray] = None

    def dense_blocks(self) -> list:
        return [*self.bases, *self.coeffs, self.decoder]

    def set_dense_blocks(self, blocks: list) -> None:
        n = len(self.bases)
        self.bases = list(blocks[:n])
        self.coeffs = list(blocks[n:2 * n])
        self.decoder = blocks[2 * n]

    def copy(self) -> "ModelParams":
        return ModelParams([b.copy() for b in self.bases], [c.copy() for c in self.coeffs],
                           self.decoder.copy(),
                           None if self.entity_embed is None else self.entity_embed.copy())

    def num_parameters(self) -> int:
        total = sum(b.size for b in self.dense_blocks())
        return total + (0 if self.entity_embed is None else self.entity_embed.size)


@dataclass
class Gradients:
    bases: list
    coeffs: list
    decoder: np.ndarray
    embed_ids: Optional[np.ndarray] = None
    embed_rows: Optional[np.ndarray] = None

    def dense_blocks(self) -> list:
        return [*self.bases, *self.coeffs, self.decoder]


def init_params(config: ModelConfig, rng: np.random.Generator,
                num_entities: Optional[int] = None) -> ModelParams:
    """Fan-scaled uniform init (ref:model.py:108-128); draw order per layer
    bases then coeffs, then the decoder, then the embedding table."""
    bases, coeffs = [], []
    B, G = config.num_bases, config.num_rel_groups
    for din, dout in zip(config.dims[:-1], config.dims[1:]):
        a = np.sqrt(6.0 / (din + dout))
        bases.append(rng.uniform(-a, a, size=(B, din, dout)))
        c = 1.0 / np.sqrt(B)
        coeffs.append(rng.uniform(-c, c, size=(G, B)))
    d_out = config.dims[-1]
    dl = np.sqrt(3.0 / d_out)
    decoder = rng.uniform(-dl, dl, size=(config.num_relations, d_out))
    embed = None
    if config.mode == MODE_EMBEDDING:
        if num_entities is None:
            raise ValidationError("embedding mode needs num_entities at init")
        el = np.sqrt(3.0 / config.dims[0])
        embed = rng.uniform(-el, el, size=(num_entities, config.dims[0]))
    return ModelParams(bases, coeffs, decoder, embed)


def layer_weights(params: ModelParams, layer: int) -> np.ndarray:
    """All 2R+1 relation matrices of a layer (host helper; the device path
    never materialises them)."""
    return np.tensordot(params.coeffs[layer], params.bases[layer], axes=(1, 0))


# ---------------------------------------------------------------------------
# Flat dense layout
# ---------------------------------------------------------------------------

class DenseLayout:
    """Offsets of every dense block inside the flat fp32 buffer."""

    def __init__(self, config: ModelConfig):
        self.config = config
        L, B, G = config.num_layers, config.num_bases, config.num_rel_groups
        self.shapes = [(B, config.dims[l], config.dims[l + 1]) for l in range(L)]
        self.shapes += [(G, B)] * L
        self.shapes.append((config.num_relations, config.dims[-1]))
        self.sizes = [int(np.prod(s)) for s in self.shapes]
        self.offsets = [int(x) for x in np.concatenate([[0], np.cumsum(self.sizes)[:-1]])]
        self.total = int(sum(self.sizes))

    def bases_off(self, l):
        return self.offsets[l]

    def coeffs_off(self, l):
        return self.offsets[self.config.num_layers + l]

    def decoder_off(self):
        return self.offsets[-1]

    def pack(self, blocks: list) -> np.ndarray:
        for b, s in zip(blocks, self.shapes):
            if tuple(np.shape(b)) != s:
                raise ShapeError(f"dense block shape {np.shape(b)} != {s}")
        return np.concatenate([np.asarray(b, dtype=np.float32).reshape(-1) for b in blocks])

    def unpack(self, flat: np.ndarray) -> list:
        flat = np.asarray(flat, dtype=np.float64)
        return [flat[o:o + n].reshape(s).copy() for o, n, s in zip(self.offsets, self.sizes, self.shapes)]


def _torch():
    import torch
    return torch


class DeviceModel:
    """Dense parameters on the device (one flat fp32 buffer)."""

    def __init__(self, config: ModelConfig, device, flat=None):
        torch = _torch()
        self.config = config
        self.layout = DenseLayout(config)
        self.device = device
        self.flat = flat if flat is not None else torch.zeros(self.layout.total, dtype=torch.float32,
                                                              device=device)
        self._lp = []
        for l in range(config.num_layers):
            lp = _lib.KgLayerParams()
            lp.d_in, lp.d_out = config.dims[l], config.dims[l + 1]
            lp.B, lp.G = config.num_bases, config.num_rel_groups
            lp.bases = self.flat.data_ptr() + 4 * self.layout.bases_off(l)
            lp.coeffs = self.flat.data_ptr() + 4 * self.layout.coeffs_off(l)
            lp.packed = None
            self._lp.append(lp)
        self._lp_packed = None   # copies pointing at pre-packed weights (see repack)
        self.wpack = None

    def repack(self) -> None:
        """Re-pack every layer's tensor-core weight operands from the current
        bases (enqueued on the current stream). Callers that use
        layer(l, packed=True) must repack after every parameter update."""
        torch = _torch()
        lib = _lib.require_cuda()
        if self._lp_packed is None:
            sizes = [lib.kg_rgcn_weights_bytes(lp.d_in, lp.d_out, lp.B) for lp in self._lp]
            offs = [sum(sizes[:l]) for l in range(len(sizes))]
            self.wpack = torch.empty(max(sum(sizes), 4) // 4, dtype=torch.float32, device=self.device)
            self._lp_packed = []
            for lp, off in zip(self._lp, offs):
                q = _lib.KgLayerParams()
                ctypes.memmove(ctypes.byref(q), ctypes.byref(lp), ctypes.sizeof(lp))
                q.packed = self.wpack.data_ptr() + off
                self._lp_packed.append(q)
        st = _lib.stream_handle()
        for q in self._lp_packed:
            _lib.call("kg_rgcn_pack_weights", ctypes.byref(q), q.packed, st)

    @classmethod
    def from_params(cls, config: ModelConfig, params: ModelParams, device) -> "DeviceModel":
        torch = _torch()
        flat = torch.as_tensor(DenseLayout(config).pack(params.dense_blocks())).to(device)
        return cls(config, device, flat)

    def layer(self, l, packed: bool = False) -> "_lib.KgLayerParams":
        if packed:
            if self._lp_packed is None:
                raise RuntimeError("repack() must run before packed layers are used")
            return self._lp_packed[l]
        return self._lp[l]

    def decoder_ptr(self) -> int:
        return self.flat.data_ptr() + 4 * self.layout.decoder_off()

    def dense_blocks(self) -> list:
        return self.layout.unpack(self.flat.cpu().numpy())


class ViewBuffers:
    """Activation / gradient / closure buffers of one partition view."""

    def __init__(self, config: ModelConfig, view, b_max: int, input_rows=None):
        torch = _torch()
        dev = view.device
        n = view.n
        self.config = config
        self.view = view
        self.n = n
        L = config.num_layers
        f32 = dict(dtype=torch.float32, device=dev)
        self.H = [input_rows if input_rows is not None else torch.zeros((n, config.dims[0]), **f32)]
        self.H += [torch.zeros((n, config.dims[l]), **f32) for l in range(1, L + 1)]
        self.dH = [torch.zeros((n, config.dims[l]), **f32) for l in range(L + 1)]
        self.order = torch.empty(n, dtype=torch.int32, device=dev)
        self.pos = torch.empty(n, dtype=torch.int32, device=dev)
        self.counts = torch.zeros(L + 1, dtype=torch.int32, device=dev)
        self.flags = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ws = _lib.Workspace(dev)
        lib = _lib.require_cuda()
        self.layer_ws_bytes = max(lib.kg_layer_workspace_bytes(ctypes.byref(view.csr()), config.dims[l],
                                                               config.dims[l + 1], config.num_bases)
                                  for l in range(L))
        self.loss_ws_bytes = lib.kg_loss_workspace_bytes(max(b_max, 1), n, config.dims[-1],
                                                         config.num_relations)
        self.b_max = b_max

    def drop_masks(self) -> list:
        """Inverted-dropout masks of the non-last layers' outputs, (n, d_{l+1})
        by closure position (allocated on first use)."""
        if getattr(self, "_masks", None) is None:
            torch = _torch()
            L = self.config.num_layers
            self._masks = [torch.empty((self.n, self.config.dims[l + 1]), dtype=torch.float32,
                                       device=self.view.device) for l in range(L - 1)]
        return self._masks

    def hpk(self, l: int):
        """Layer l's input rows (by closure position) as tensor-core operand
        records for the backward Y GEMM (written by layer l-1's forward, or by
        device_pack_inputs for l = 0)."""
        key = f"hpk{l}"
        nbytes = _lib.require_cuda().kg_pack_rows_bytes(self.n, self.config.dims[l])
        return self.ws.get(key, nbytes)

    def layer_ws(self, l: int = 0):
        """Per-layer scratch: a layer's side-stream gradient work may still read
        its workspace while the next (lower) layer runs."""
        return self.ws.get(f"layer{l}", self.layer_ws_bytes)

    def loss_ws(self, b):
        if b > self.b_max:
            self.b_max = b
            self.loss_ws_bytes = _lib.require_cuda().kg_loss_workspace_bytes(
                b, self.n, self.config.dims[-1], self.config.num_relations)
        return self.ws.get("loss", self.loss_ws_bytes)


def device_pack_inputs(bufs: ViewBuffers) -> None:
    """Layer 0's input rows H_0[order[p]], p < counts[L], as operand records
    (bufs.hpk(0)); only needs the closure, so it can run on a side stream."""
    L = bufs.config.num_layers
    out = bufs.hpk(0)
    _lib.call("kg_pack_rows", bufs.H[0].data_ptr(), bufs.config.dims[0], bufs.order.data_ptr(),
              bufs.counts.data_ptr(), L, bufs.n, bufs.config.dims[0], out.data_ptr(), _lib.stream_handle())


def device_dropout(bufs: ViewBuffers, g_dev, p: float) -> list:
    """Masks of every non-last layer, in forward order (the reference's draw
    order, ref:model.py:221-227), from the device PCG64 state g_dev (advanced
    in place)."""
    L = bufs.config.num_layers
    masks = bufs.drop_masks()
    st = _lib.stream_handle()
    for l in range(L - 1):
        _lib.call("kg_dropout_mask", g_dev.data_ptr(), bufs.counts.data_ptr(), L - 1 - l, bufs.config.dims[l + 1],
                  float(p), bufs.n, masks[l].data_ptr(), st)
    return masks


def device_backward_y(model: DeviceModel, bufs: ViewBuffers, l: int) -> None:
    """Layer l's backward operand Y = H_l[A_{t+1}] . [V_0 | .. | V_{B-1}]
    ahead of time (needs packed weights and bufs.hpk(l)); kg_rgcn_backward
    then runs with y_ready."""
    L = model.config.num_layers
    ws = bufs.layer_ws(l)
    _lib.call("kg_rgcn_backward_y", ctypes.byref(bufs.view.csr()), ctypes.byref(model.layer(l, True)),
              bufs.H[l].data_ptr(), bufs.hpk(l).data_ptr(), bufs.order.data_ptr(), bufs.counts.data_ptr(),
              L - 1 - l, ws.data_ptr(), ws.numel(), _lib.stream_handle())


def device_forward(model: DeviceModel, bufs: ViewBuffers, packed: bool = False, hpk: bool = False,
                   masks: Optional[list] = None, after_layer=None) -> None:
    """All layers over the closure in bufs.order/counts (ref:model.py:196-235).
    packed: use the model's pre-packed weight operands (DeviceModel.repack);
    hpk: also emit each hidden layer's output as the next layer's packed
    backward operand (bufs.hpk)."""
    L = model.config.num_layers
    csr = ctypes.byref(bufs.view.csr())
    st = _lib.stream_handle()
    for l in range(L):
        ws = bufs.layer_ws(l)
        _lib.call("kg_rgcn_forward", csr, ctypes.byref(model.layer(l, packed)), bufs.H[l].data_ptr(),
                  bufs.H[l + 1].data_ptr(), bufs.order.data_ptr(), bufs.pos.data_ptr(), bufs.counts.data_ptr(),
                  L - 1 - l, 1 if l < L - 1 else 0, masks[l].data_ptr() if (masks and l < L - 1) else None,
                  bufs.hpk(l + 1).data_ptr() if (hpk and l < L - 1) else None, ws.data_ptr(), ws.numel(), st)
        if after_layer is not None:
            after_layer(l)


def device_loss(model: DeviceModel, bufs: ViewBuffers, stream, start: int, b: int, grad_flat, loss_out,
                scores_out=None, start_dev=None, part: str = "all", side=None) -> None:
    """DistMult + BCE (ref:model.py:254-281): loss -> loss_out (device scalar),
    d_decoder -> grad_flat's decoder block, dH_L -> bufs.dH[L] seed rows.
    part "groups" / "compute" run the two halves separately (the batch-only
    grouping can overlap the layers on another stream); "all" runs both."""
    cfg = model.config
    L = cfg.num_layers
    ws = bufs.loss_ws(b)
    fn = {"all": "kg_distmult_loss", "groups": "kg_loss_groups", "compute": "kg_loss_compute"}[part]
    args = [bufs.H[L].data_ptr(), cfg.dims[-1], bufs.n, model.decoder_ptr(),
            cfg.num_relations, stream.triples.data_ptr(), stream.labels.data_ptr(), stream.total, start,
            _lib.ptr(start_dev), b,
            bufs.order.data_ptr(), bufs.counts.data_ptr(), bufs.dH[L].data_ptr(),
            grad_flat.data_ptr() + 4 * model.layout.decoder_off(), loss_out.data_ptr(),
            0 if scores_out is None else scores_out.data_ptr(), bufs.flags.data_ptr(), ws.data_ptr(),
            ws.numel(), _lib.stream_handle()]
    if part == "compute":
        args.append(None if side is None else side.cuda_stream)
    _lib.call(fn, *args)


def device_csc_positions(bufs: ViewBuffers) -> None:
    """pos[c_dst] of every CSC message for the closure in bufs (the backward's
    dZ gathers then take one dependent load per message); after this call
    device_backward uses it until bufs.pos changes (the caller re-runs it)."""
    torch = _torch()
    if getattr(bufs, "c_pos", None) is None:
        bufs.c_pos = torch.empty(max(int(bufs.view.csr().e), 1), dtype=torch.int32, device=bufs.view.device)
    _lib.call("kg_csc_positions", ctypes.byref(bufs.view.csr()), bufs.pos.data_ptr(), bufs.c_pos.data_ptr(),
              _lib.stream_handle())
    bufs.c_pos_ready = bufs.c_pos


def device_backward(model: DeviceModel, bufs: ViewBuffers, grad_flat, input_grad: bool, side=None,
                    packed: bool = False, hpk: bool = False, masks: Optional[list] = None,
                    y_ready: bool = False) -> None:
    """Layer gradients in reverse (ref:model.py:283-296): d bases / d coeffs
    into grad_flat, dL/dH_0 rows into bufs.dH[0] when input_grad. With a side
    stream (torch.cuda.Stream) the parameter-gradient branch of every layer
    runs on it; it is joined back into the current stream before returning."""
    torch = _torch()
    L = model.config.num_layers
    csr = ctypes.byref(bufs.view.csr())
    st = _lib.stream_handle()
    lay = model.layout
    for l in range(L - 1, -1, -1):
        ws = bufs.layer_ws(l)
        dh_in = bufs.dH[l].data_ptr() if (l > 0 or input_grad) else 0
        _lib.call("kg_rgcn_backward", csr, ctypes.byref(model.layer(l, packed)), bufs.H[l].data_ptr(),
                  bufs.H[l + 1].data_ptr() if l < L - 1 else 0, bufs.dH[l + 1].data_ptr(), dh_in,
                  bufs.order.data_ptr(), bufs.pos.data_ptr(), _lib.ptr(getattr(bufs, "c_pos_ready", None)),
                  bufs.counts.data_ptr(), L - 1 - l,
                  grad_flat.data_ptr() + 4 * lay.bases_off(l), grad_flat.data_ptr() + 4 * lay.coeffs_off(l),
                  bufs.hpk(l).data_ptr() if hpk else None, masks[l].data_ptr() if (masks and l < L - 1) else None,
                  1 if y_ready else 0, ws.data_ptr(), ws.numel(), st, None if side is None else side.cuda_stream)
    if side is not None:
        torch.cuda.current_stream().wait_stream(side)


FLAG_NONFINITE_SCORE, FLAG_NONFINITE_LOSS, FLAG_NONFINITE_PARAM = 1, 2, 4   # include/kgdist_b200.h
FLAG_BAD_VERTEX, FLAG_PEER_TIMEOUT = 8, 16


def raise_for_flags(f: int, what: str = "") -> None:
    """Map a device status word (KG_FLAG_* bits) to the reference's error."""
    if not f:
        return
    if f & FLAG_PEER_TIMEOUT:
        raise ProtocolError("peer payload exchange timed out (a rank stopped publishing)")
    if f & FLAG_NONFINITE_SCORE:
        raise NumericError(f"non-finite score {what}".strip())
    if f & FLAG_NONFINITE_LOSS:
        raise NumericError("non-finite loss")
    if f & FLAG_NONFINITE_PARAM:
        raise NumericError("non-finite parameter after optimizer step")
    if f & FLAG_BAD_VERTEX:
        raise IntegrityError("vertex not present in compute graph")
    raise NumericError(f"device status {f:#x}")


def check_flags(bufs: ViewBuffers, what: str = "") -> None:
    f = int(bufs.flags.item())
    if f:
        bufs.flags.zero_()
        raise_for_flags(f, what)


# ---------------------------------------------------------------------------
# Public numpy-facing API (ref:model.py:188-312)
# ---------------------------------------------------------------------------

@dataclass
class EncodeCache:
    """Holds the device state of one encode() for loss_from_cache()."""
    model: Optional[DeviceModel] = None
    bufs: Optional[ViewBuffers] = None
    seed_embeddings: Optional[np.ndarray] = None
    f64: Optional[dict] = None   # float64 path: H / acc / Z per layer, masks


def _input_rows(config, cg, input_table, input_ids, device):
    torch = _torch()
    input_table = np.asarray(input_table)
    if input_table.ndim != 2 or input_table.shape[1] != config.dims[0]:
        raise ShapeError(f"input width {input_table.shape[1] if input_table.ndim == 2 else '?'} "
                         f"!= d_in {config.dims[0]}")
    ids = np.asarray(input_ids)[: cg.view.n]
    if len(ids) != cg.view.n:
        raise IntegrityError("input_ids must cover every local vertex of the view")
    return torch.as_tensor(np.ascontiguousarray(input_table[ids], dtype=np.float32)).to(device)


# Precision of the public numpy API (encode / loss_from_cache /
# loss_and_grad): "f64" runs the float64 device kernels (kg_model64.cu), the
# reference's own precision; "f32" runs the training hot path's fp32 /
# tensor-core kernels (what Trainer uses; parity tests of those kernels
# select it with `api_precision("f32")`). KG_API_PRECISION sets the default.
API_PRECISION = os.environ.get("KG_API_PRECISION", "f64")


class api_precision:
    """Context manager: `with api_precision("f32"): ...`."""

    def __init__(self, prec: str):
        if prec not in ("f32", "f64"):
            raise ValidationError(f"unknown precision {prec!r}")
        self.prec = prec

    def __enter__(self):
        global API_PRECISION
        self.saved, API_PRECISION = API_PRECISION, self.prec
        return self

    def __exit__(self, *exc):
        global API_PRECISION
        API_PRECISION = self.saved


def _draw_masks(config, cg, bufs, dropout_rng, dev):
    """Dropout masks of the non-last layers from the caller's Generator (device
    PCG64 stream at numpy's positions); the Generator advances as numpy's."""
    g_dev = _lib.pcg_to_device(_lib.pcg_from_numpy(dropout_rng), dev)
    masks = device_dropout(bufs, g_dev, config.dropout)
    counts = cg.d_counts.cpu().tolist()
    L = config.num_layers
    dropout_rng.bit_generator.advance(sum(int(counts[L - 1 - l]) * config.dims[l + 1] for l in range(L - 1)))
    return masks


def _encode64(params: ModelParams, config: ModelConfig, cg, input_table, input_ids, drop, dropout_rng,
              cache) -> np.ndarray:
    """Float64 forward over the closure (kg_forward_layer_f64 per layer)."""
    torch = _torch()
    view = cg.view
    dev = view.device
    n = view.n
    L = config.num_layers
    f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
    input_table = np.asarray(input_table)
    if input_table.ndim != 2 or input_table.shape[1] != config.dims[0]:
        raise ShapeError(f"input width {input_table.shape[1] if input_table.ndim == 2 else '?'} "
                         f"!= d_in {config.dims[0]}")
    ids = np.asarray(input_ids)[:n]
    if len(ids) != n:
        raise IntegrityError("input_ids must cover every local vertex of the view")
    counts = cg.layer_vertex_counts
    bases = [f64(b) for b in params.bases]
    coeffs = [f64(c) for c in params.coeffs]
    H = [f64(input_table[ids])] + [torch.zeros((n, config.dims[l]), dtype=torch.float64, device=dev)
                                   for l in range(1, L + 1)]
    masks = None
    if drop:
        bufs = ViewBuffers(config, view, 1)
        bufs.order.copy_(cg.d_order)
        bufs.counts.copy_(cg.d_counts)
        masks = _draw_masks(config, cg, bufs, dropout_rng, dev)
    scale = 1.0 / (1.0 - config.dropout) if drop else 1.0
    csr = view.csr()
    st = _lib.stream_handle()
    accs, Zs = [], []
    for l in range(L):
        t = L - 1 - l
        T = counts[t]
        din, dout = config.dims[l], config.dims[l + 1]
        acc = torch.empty((max(T, 1), config.num_bases * din), dtype=torch.float64, device=dev)
        Z = torch.empty((max(T, 1), dout), dtype=torch.float64, device=dev)
        mask = masks[l] if (masks is not None and l < L - 1) else None
        _lib.call("kg_forward_layer_f64", ctypes.byref(csr), view.d_ref_src.data_ptr(), view.d_ref_rel.data_ptr(),
                  view.d_msg_cnt.data_ptr(), cg.d_order.data_ptr(), cg.d_pos.data_ptr(), T, din, dout,
                  config.num_bases, bases[l].data_ptr(), coeffs[l].data_ptr(), H[l].data_ptr(), acc.data_ptr(),
                  Z.data_ptr(), H[l + 1].data_ptr(), 1 if l < L - 1 else 0, _lib.ptr(mask), scale, st)
        accs.append(acc)
        Zs.append(Z)
    seeds = cg.seed_vertices
    out = H[L][torch.as_tensor(seeds, device=dev)].cpu().numpy()
    if cache is not None:
        cache.model = None
        cache.bufs = None
        cache.f64 = dict(H=H, acc=accs, Z=Zs, masks=masks, scale=scale, bases=bases, coeffs=coeffs)
        cache.seed_embeddings = out
    return out


def _loss_from_cache64(params, config, batch, cg, cache, input_ids) -> tuple:
    torch = _torch()
    view = cg.view
    dev = view.device
    n = view.n
    L = config.num_layers
    c = cache.f64
    H, bases, coeffs = c["H"], c["bases"], c["coeffs"]
    tri = torch.as_tensor(np.ascontiguousarray(batch.triples, dtype=np.int32)).to(dev)
    lab = torch.as_tensor(np.asarray(batch.labels, dtype=np.float64)).to(dev)
    dec = torch.as_tensor(np.ascontiguousarray(params.decoder, dtype=np.float64)).to(dev)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    d_dec = torch.zeros_like(dec)
    dH = [torch.zeros((n, config.dims[l]), dtype=torch.float64, device=dev) for l in range(L + 1)]
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    st = _lib.stream_handle()
    _lib.call("kg_loss_f64", tri.data_ptr(), lab.data_ptr(), len(batch.triples), H[L].data_ptr(), dec.data_ptr(),
              config.dims[-1], loss.data_ptr(), d_dec.data_ptr(), dH[L].data_ptr(), flags.data_ptr(), st)
    f = int(flags.item())
    if f:
        raise_for_flags(f)
    lv = float(loss.item())
    if not np.isfinite(lv):
        raise NumericError("non-finite loss")
    csr = view.csr()
    lib = _lib.require_cuda()
    counts = cg.layer_vertex_counts
    B, G = config.num_bases, config.num_rel_groups
    db, dc = [None] * L, [None] * L
    for l in range(L - 1, -1, -1):
        t = L - 1 - l
        T = counts[t]
        din, dout = config.dims[l], config.dims[l + 1]
        ws = torch.empty(lib.kg_layer64_workspace_bytes(n, din, dout, B), dtype=torch.uint8, device=dev)
        dZ = torch.empty((max(T, 1), dout), dtype=torch.float64, device=dev)
        d_b = torch.empty((B, din, dout), dtype=torch.float64, device=dev)
        d_c = torch.empty((G, B), dtype=torch.float64, device=dev)
        mask = c["masks"][l] if (c["masks"] is not None and l < L - 1) else None
        want_in = l > 0 or config.mode == MODE_EMBEDDING
        _lib.call("kg_backward_layer_f64", ctypes.byref(csr), view.d_ref_src.data_ptr(), view.d_ref_rel.data_ptr(),
                  view.d_msg_cnt.data_ptr(), cg.d_order.data_ptr(), cg.d_pos.data_ptr(), T, din, dout, B,
                  bases[l].data_ptr(), coeffs[l].data_ptr(), H[l].data_ptr(), c["acc"][l].data_ptr(),
                  c["Z"][l].data_ptr(), dH[l + 1].data_ptr(), 1 if l < L - 1 else 0, _lib.ptr(mask), c["scale"],
                  dZ.data_ptr(), d_b.data_ptr(), d_c.data_ptr(), dH[l].data_ptr() if want_in else None,
                  ws.data_ptr(), ws.numel(), st)
        db[l], dc[l] = d_b.cpu().numpy(), d_c.cpu().numpy()
    g = Gradients(db, dc, d_dec.cpu().numpy())
    if config.mode == MODE_EMBEDDING:
        order = cg.vertex_order
        g.embed_ids = np.asarray(input_ids)[order]
        g.embed_rows = dH[0][torch.as_tensor(order, device=dev)].cpu().numpy()
    return lv, g


def encode(params: ModelParams, config: ModelConfig, cg, input_table: np.ndarray, input_ids: np.ndarray,
           training: bool = False, dropout_rng: Optional[np.random.Generator] = None,
           cache: Optional[EncodeCache] = None) -> np.ndarray:
    """Graph convolutions over a (device) compute graph; returns the seed
    embeddings in cg.seed_vertices order (ref:model.py:196-235). Float64 on
    the device by default (API_PRECISION)."""
    if cg.num_layers != config.num_layers:
        raise ShapeError(f"compute graph has {cg.num_layers} layers, model has {config.num_layers}")
    drop = training and config.dropout > 0.0
    if drop and dropout_rng is None:
        raise ValidationError("training with dropout needs a dropout rng")
    if API_PRECISION == "f64":
        return _encode64(params, config, cg, input_table, input_ids, drop, dropout_rng, cache)
    view = cg.view
    dev = view.device
    model = DeviceModel.from_params(config, params, dev)
    rows = _input_rows(config, cg, input_table, input_ids, dev)
    bufs = ViewBuffers(config, view, 1, input_rows=rows)
    bufs.order.copy_(cg.d_order)
    bufs.pos.copy_(cg.d_pos)
    bufs.counts.copy_(cg.d_counts)
    masks = _draw_masks(config, cg, bufs, dropout_rng, dev) if drop else None
    bufs.masks = masks
    device_forward(model, bufs, masks=masks)
    seeds = cg.seed_vertices
    import torch
    out = bufs.H[-1][torch.as_tensor(seeds, device=dev)].double().cpu().numpy()
    if cache is not None:
        cache.model, cache.bufs, cache.seed_embeddings = model, bufs, out
    return out


def score(head_embedding: np.ndarray, relation_diag: np.ndarray, tail_embedding: np.ndarray) -> float:
    """Bilinear diagonal score sum_k h_k m_k t_k (ref:model.py:238-243)."""
    if not (np.shape(head_embedding) == np.shape(relation_diag) == np.shape(tail_embedding)):
        raise IntegrityError("score operands must share one embedding width")
    return float(np.sum(np.asarray(head_embedding) * relation_diag * tail_embedding))


def score_batch(seed_embeddings: np.ndarray, params: ModelParams, cg, triples: np.ndarray) -> np.ndarray:
    """ref:model.py:246-251 (host helper over already-encoded seeds)."""
    hs = seed_embeddings[cg.seed_positions(triples[:, 0])]
    ht = seed_embeddings[cg.seed_positions(triples[:, 2])]
    return np.einsum("ij,ij,ij->i", hs, params.decoder[triples[:, 1]], ht)


def loss_from_cache(params: ModelParams, config: ModelConfig, batch, cg, cache: EncodeCache,
                    input_ids: np.ndarray) -> tuple:
    """BCE over the batch and exact gradients from the cached device
    activations (ref:model.py:254-301); returns (loss, Gradients)."""
    torch = _torch()
    if getattr(cache, "f64", None) is not None:
        if len(batch.triples) == 0:
            raise ValidationError("empty batch")
        if not np.isin(batch.triples[:, [0, 2]], cg.seed_vertices).all():
            raise IntegrityError("vertex not present in compute graph")
        return _loss_from_cache64(params, config, batch, cg, cache, input_ids)
    from .sampler import DeviceStream
    model, bufs = cache.model, cache.bufs
    dev = bufs.view.device
    tri = torch.as_tensor(np.ascontiguousarray(batch.triples, dtype=np.int32)).to(dev)
    lab = torch.as_tensor(np.asarray(batch.labels, dtype=np.float32)).to(dev)
    stream = DeviceStream(tri, lab, len(batch.triples))
    if len(batch.triples) == 0:
        raise ValidationError("empty batch")
    seeds_ok = np.isin(batch.triples[:, [0, 2]], cg.seed_vertices).all()
    if not seeds_ok:
        raise IntegrityError("vertex not present in compute graph")
    grad = torch.zeros(model.layout.total, dtype=torch.float32, device=dev)
    loss_t = torch.zeros(1, dtype=torch.float32, device=dev)
    device_loss(model, bufs, stream, 0, len(batch.triples), grad, loss_t)
    check_flags(bufs)
    emb = config.mode == MODE_EMBEDDING
    device_csc_positions(bufs)
    device_backward(model, bufs, grad, input_grad=emb, masks=getattr(bufs, "masks", None))
    blocks = model.layout.unpack(grad.cpu().numpy())
    L = config.num_layers
    g = Gradients(blocks[:L], blocks[L:2 * L], blocks[2 * L])
    if emb:
        order = cg.vertex_order
        g.embed_ids = np.asarray(input_ids)[order]
        g.embed_rows = bufs.dH[0][torch.as_tensor(order, device=dev)].double().cpu().numpy()
    return float(loss_t.item()), g


def loss_and_grad(params: ModelParams, config: ModelConfig, batch, cg, input_table: np.ndarray,
                  input_ids: np.ndarray, training: bool = False,
                  dropout_rng: Optional[np.random.Generator] = None) -> tuple:
    cache = EncodeCache()
    encode(params, config, cg, input_table, input_ids, training=training, dropout_rng=dropout_rng,
           cache=cache)
    return loss_from_cache(params, config, batch, cg, cache, input_ids)


CHECKPOINT_VERSION = 1


def save_checkpoint(params: ModelParams, config: ModelConfig, path: str) -> None:
    """npz checkpoint in the reference's format (ref:model.py:319-331)."""
    arrays = {"decoder": params.decoder}
    for l, (b, c) in enumerate(zip(params.bases, params.coeffs)):
        arrays[f"bases_{l}"] = b
        arrays[f"coeffs_{l}"] = c
    if params.entity_embed is not None:
        arrays["entity_embed"] = params.entity_embed
    meta = json.dumps({"version": CHECKPOINT_VERSION, "config": config.to_json()})
    np.savez_compressed(path, _meta=np.frombuffer(meta.encode(), dtype=np.uint8), **arrays)


def load_checkpoint(path: str) -> tuple:
    with np.load(path) as data:
        if "_meta" not in data:
            raise FormatError(f"{path} is not a model checkpoint")
        meta = json.loads(bytes(data["_meta"]).decode())
        if meta.get("version") != CHECKPOINT_VERSION:
            raise FormatError(f"unsupported checkpoint version {meta.get('version')}")
        config = ModelConfig.from_json(meta["config"])
        L = config.num_layers
        params = ModelParams([data[f"bases_{l}"] for l in range(L)], [data[f"coeffs_{l}"] for l in range(L)],
                             data["decoder"], data["entity_embed"] if "entity_embed" in data else None)
    return params, config
