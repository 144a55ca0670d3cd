"""ctypes binding of the sm_100a kernel library (include/kgdist_b200.h).

The library is built in-tree by `make` (or __graft_entry__.build()) into
paper_2201_02791_b200/lib/libkgdist_b200.so. There is no CPU fallback: every
compute entry point needs a CUDA device, and `require_cuda()` fails loudly
when the device or the library is missing.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int, c_int8, c_int32, c_int64, c_uint32, c_uint64, c_void_p

import numpy as np

from .errors import STATUS_ERRORS, DeviceError, KGError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libkgdist_b200.so")
ABI_VERSION = 1


class KgPcg64(ctypes.Structure):
    _fields_ = [("state_hi", c_uint64), ("state_lo", c_uint64), ("inc_hi", c_uint64),
                ("inc_lo", c_uint64), ("has_uint32", c_uint32), ("uinteger", c_uint32)]


class KgGraphCsr(ctypes.Structure):
    _fields_ = [("n", c_int32), ("R", c_int32), ("e", c_int64),
                ("indptr", c_void_p), ("src", c_void_p), ("rel", c_void_p), ("norm", c_void_p),
                ("c_indptr", c_void_p), ("c_dst", c_void_p), ("c_rel", c_void_p), ("c_norm", c_void_p),
                ("rel_perm", c_void_p), ("rel_ptr", c_void_p), ("chunk", c_int32),
                ("ck_ptr", c_void_p), ("ck_row", c_void_p), ("ck_slot", c_void_p), ("ck_split", c_void_p),
                ("ck_counts", c_void_p), ("cc_ptr", c_void_p), ("cc_row", c_void_p), ("cc_slot", c_void_p),
                ("cc_split", c_void_p), ("cc_counts", c_void_p), ("ck_desc", c_void_p), ("cc_desc", c_void_p)]


class KgLayerParams(ctypes.Structure):
    _fields_ = [("d_in", c_int32), ("d_out", c_int32), ("B", c_int32), ("G", c_int32),
                ("bases", c_void_p), ("coeffs", c_void_p), ("packed", c_void_p)]


class KgCopySeg(ctypes.Structure):
    _fields_ = [("dst", c_void_p), ("src", c_void_p), ("bytes", c_int64), ("dst_round_stride", c_int64),
                ("src_round_stride", c_int64)]


class KgEpochPrepArgs(ctypes.Structure):
    _fields_ = [("g", POINTER(KgGraphCsr)), ("hops", c_int32), ("rounds", c_int32), ("stream_triples", c_void_p),
                ("labels", c_void_p), ("total", c_int64), ("b", c_int64), ("d", c_int32), ("R", c_int32),
                ("order", c_void_p), ("pos", c_void_p), ("counts", c_void_p), ("groups", c_void_p),
                ("groups_stride", c_int64), ("flags", c_void_p), ("closure_ws", c_void_p),
                ("closure_ws_bytes", c_int64), ("loss_ws", c_void_p), ("loss_ws_bytes", c_int64),
                ("branches", c_int32)]


P = c_void_p
ST = c_int  # kg_status

# name -> (restype, argtypes)
_PROTOS = {
    "kg_abi_version": (c_int, []),
    "kg_graph_upload": (ST, [P, P]),
    "kg_last_error": (c_int, [ctypes.c_char_p, c_int64]),
    "kg_launch_count": (c_int64, []),
    "kg_kernel_timer_begin": (ST, [ctypes.c_char_p]),
    "kg_kernel_timer_end": (ST, [POINTER(c_double), POINTER(c_int64)]),
    "kg_kernel_timer_dump": (ST, [ctypes.c_char_p, c_int64]),
    "kg_kernel_timer_detach": (ST, [POINTER(c_int64)]),
    "kg_kernel_timer_read": (ST, [c_int64, POINTER(c_double), POINTER(c_int64)]),
    "kg_kernel_timer_read_named": (ST, [c_int64, ctypes.c_char_p, POINTER(c_double), POINTER(c_int64)]),
    "kg_kernel_timer_span": (ST, [c_int64, ctypes.c_char_p, ctypes.c_char_p, POINTER(c_double), POINTER(c_int64)]),
    "kg_preload_kernels": (ST, [POINTER(c_int32)]),
    "kg_epoch_end": (ST, [P, c_int64, c_int32, c_int32, P, c_int32, P, P]),
    "kg_copy_segments": (ST, [POINTER(KgCopySeg), c_int32, P, c_int64, P]),
    "kg_loss_group_fields": (c_int32, [P, c_int64, c_int64, c_int32, c_int32, c_int32, POINTER(c_void_p),
                                       POINTER(c_int64), c_int32]),
    "kg_sort_workspace_bytes": (c_int64, [c_int64]),
    "kg_sort_pairs_u64": (ST, [P, P, c_int64, c_int, P, c_int64, P]),
    "kg_scan_workspace_bytes": (c_int64, [c_int64]),
    "kg_exclusive_scan_u32": (ST, [P, P, c_int64, P, P, c_int64, P]),
    "kg_pcg64_advance": (None, [POINTER(KgPcg64), c_uint64]),
    "kg_pcg64_consume32": (None, [POINTER(KgPcg64), c_uint64]),
    "kg_pcg64_peek64": (None, [POINTER(KgPcg64), P, c_int64]),
    "kg_view_workspace_bytes": (c_int64, [c_int64, c_int64]),
    "kg_view_local_ids": (ST, [P, c_int64, P, c_int64, c_int64, P, P, P, P, c_int64, P]),
    "kg_view_build": (ST, [P, c_int64, P, P, P, P, P, POINTER(KgGraphCsr), P, P, P, c_int64, P]),
    "kg_neg_init": (ST, [P, c_int64, c_int32, P, P, P, P, P]),
    "kg_neg_round_workspace_bytes": (c_int64, [c_int64]),
    "kg_neg_round": (ST, [P, P, P, c_int32, P, P, c_int64, c_int64, c_int32, c_int32, P, P, P,
                          c_int64, P, P, P, P, c_int64, P]),
    "kg_is_positive": (ST, [P, c_int64, c_int32, c_int32, P, P, P, P]),
    "kg_perm_draws_buffer_len": (c_int64, [c_int64]),
    "kg_perm_draws_buffered": (ST, [c_int64, P, P, c_int64, P, P, P]),
    "kg_perm_resolve_workspace_bytes": (c_int64, [c_int64]),
    "kg_perm_resolve": (ST, [P, c_int64, P, P, c_int64, P]),
    "kg_stream_gather": (ST, [P, c_int64, P, c_int64, P, P, P, P]),
    "kg_closure_workspace_bytes": (c_int64, [c_int32]),
    "kg_closure": (ST, [P, c_int64, c_int64, P, c_int64, P, POINTER(KgGraphCsr), c_int32, P, P, P, P,
                        c_int64, P]),
    "kg_layer_workspace_bytes": (c_int64, [POINTER(KgGraphCsr), c_int32, c_int32, c_int32]),
    "kg_rgcn_forward": (ST, [POINTER(KgGraphCsr), POINTER(KgLayerParams), P, P, P, P, P, c_int32, c_int32,
                             P, P, P, c_int64, P]),
    "kg_rgcn_backward": (ST, [POINTER(KgGraphCsr), POINTER(KgLayerParams), P, P, P, P, P, P, P, P, c_int32,
                              P, P, P, P, c_int32, P, c_int64, P, P]),
    "kg_csc_positions": (ST, [POINTER(KgGraphCsr), P, P, P]),
    "kg_rgcn_backward_y": (ST, [POINTER(KgGraphCsr), POINTER(KgLayerParams), P, P, P, P, c_int32, P, c_int64, P]),
    "kg_dropout_mask": (ST, [P, P, c_int32, c_int32, c_double, c_int64, P, P]),
    "kg_uniform_f64": (ST, [P, c_int64, c_double, c_double, P, P]),
    "kg_eval_candidates": (ST, [P, c_int32, P, P, c_int64, P, P, P, c_int32, P, P, P]),
    "kg_pack_rows_bytes": (c_int64, [c_int64, c_int64]),
    "kg_pack_rows": (ST, [P, c_int64, P, P, c_int32, c_int64, c_int64, P, P]),
    "kg_rgcn_weights_bytes": (c_int64, [c_int32, c_int32, c_int32]),
    "kg_rgcn_pack_weights": (ST, [POINTER(KgLayerParams), P, P]),
    "kg_gemm_workspace_bytes": (c_int64, [c_int64, c_int64, c_int64]),
    "kg_gemm_f32": (ST, [P, c_int64, P, P, c_int64, P, c_int64, P, c_int64, c_int64, c_int64, c_int32, c_int32,
                         c_int32, P, c_int64, P]),
    "kg_loss_workspace_bytes": (c_int64, [c_int64, c_int32, c_int32, c_int32]),
    "kg_distmult_loss": (ST, [P, c_int32, c_int32, P, c_int32, P, P, c_int64, c_int64, P, c_int64, P, P, P,
                              P, P, P, P, P, c_int64, P]),
    "kg_loss_groups": (ST, [P, c_int32, c_int32, P, c_int32, P, P, c_int64, c_int64, P, c_int64, P, P, P,
                            P, P, P, P, P, c_int64, P]),
    "kg_loss_compute": (ST, [P, c_int32, c_int32, P, c_int32, P, P, c_int64, c_int64, P, c_int64, P, P, P,
                             P, P, P, P, P, c_int64, P, P]),
    "kg_epoch_prep": (ST, [POINTER(KgEpochPrepArgs), P]),
    "kg_optim_workspace_bytes": (c_int64, [c_int64]),
    "kg_dense_step": (ST, [P, P, P, P, c_int32, c_int64, c_int32, c_float, c_float, c_float, c_float,
                           c_double, c_double, P, c_float, P, P, c_int64, P]),
    "kg_tree_mean_f64": (ST, [P, c_int64, c_int64, P, P]),
    "kg_dense_step_f64_workspace_bytes": (c_int64, [c_int64]),
    "kg_dense_step_f64": (ST, [P, P, P, P, c_int64, c_int32, c_double, c_double, c_double, c_double, c_double,
                               c_double, c_double, P, P, c_int64, P]),
    "kg_sparse_step_f64_workspace_bytes": (c_int64, [c_int64, c_int32, c_int64]),
    "kg_sparse_step_f64": (ST, [P, P, P, c_int64, c_int32, P, P, c_int64, c_int32, c_double, c_double, c_double,
                                c_double, c_double, c_double, P, P, c_int64, P]),
    "kg_peer_region_bytes": (c_int64, [c_int64]),
    "kg_peer_alloc": (ST, [c_int64, POINTER(c_void_p), P]),
    "kg_peer_open": (ST, [P, POINTER(c_void_p)]),
    "kg_peer_close": (ST, [P, c_int32]),
    "kg_peer_publish": (ST, [P, P, c_int64, P, P]),
    "kg_peer_gather": (ST, [P, c_int32, c_int64, P, P, P, P]),
    "kg_sparse_step": (ST, [P, P, P, P, P, P, c_int32, c_int32, c_int32, c_float, c_float, c_float,
                            c_float, c_double, c_double, P, c_int32, P]),
    "kg_eval_workspace_bytes": (c_int64, [c_int64, c_int32, c_int32, c_int64]),
    "kg_eval_filtered": (ST, [P, c_int32, c_int32, P, c_int32, P, c_int64, P, c_int64, P, c_int64,
                              c_int32, c_int32, c_int32, c_int64, P, P, P, P, P, P, c_int64, P]),
    "kg_encode_full_f64_workspace_bytes": (c_int64, [c_int32, c_int64, c_int32, c_int32, c_int32]),
    "kg_encode_full_f64": (ST, [POINTER(KgGraphCsr), P, P, P, c_int32, P, c_int32, P, P, P, P, P, c_int64, P]),
    "kg_known_keys_workspace_bytes": (c_int64, [c_int64]),
    "kg_known_keys": (ST, [P, c_int64, c_int32, c_int32, c_int32, c_int32, P, P, P, c_int64, P]),
    "kg_forward_layer_f64": (ST, [POINTER(KgGraphCsr), P, P, P, P, P, c_int32, c_int32, c_int32, c_int32, P, P, P, P,
                                  P, P, c_int32, P, c_double, P]),
    "kg_loss_f64": (ST, [P, P, c_int64, P, P, c_int32, P, P, P, P, P]),
    "kg_layer64_workspace_bytes": (c_int64, [c_int64, c_int32, c_int32, c_int32]),
    "kg_backward_layer_f64": (ST, [POINTER(KgGraphCsr), P, P, P, P, P, c_int32, c_int32, c_int32, c_int32, P, P, P,
                                   P, P, P, c_int32, P, c_double, P, P, P, P, P, c_int64, P]),
    "kg_halo_workspace_bytes": (c_int64, [c_int64, c_int64]),
    "kg_halo_incidence": (ST, [P, c_int64, c_int64, P, P, P, c_int64, P]),
    "kg_halo_expand": (ST, [P, c_int64, c_int64, P, P, P, c_int64, c_int32, P, P, P, P, P, P, P, c_int64, P]),
    "kg_generate_synthetic": (c_int64, [c_int64, c_int32, c_int64, POINTER(KgPcg64), P, c_int64]),
    "kg_vertex_cut_assign": (ST, [P, c_int64, c_int64, c_int32, P, c_double, c_int64, P]),
}

_lib = None


def exported_symbols() -> list:
    return sorted(_PROTOS)


def load():
    """Load the shared library (no device needed) and bind every prototype."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("KG_LIB") or LIB_PATH     # KG_LIB: diagnostics (an A/B build variant)
    if not os.path.isfile(path):
        raise DeviceError(f"kernel library not built: {path} (run `make` or "
                          f"__graft_entry__.build())")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.kg_abi_version() != ABI_VERSION:
        raise DeviceError("kernel library ABI version mismatch; rebuild")
    _lib = lib
    return lib


_preloaded = False


def require_cuda():
    """The compute path has no CPU fallback: fail loudly without a device.
    The first call per process also loads every kernel of the library
    (kg_preload_kernels): lazy loading would otherwise land in the first
    training epoch."""
    global _preloaded
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("paper_2201_02791_b200 needs a CUDA device (B200, sm_100a); "
                          "no CPU fallback exists")
    lib = load()
    if not _preloaded and os.environ.get("KG_PRELOAD", "1") != "0":
        _preloaded = True
        n = c_int32(0)
        check(lib.kg_preload_kernels(ctypes.byref(n)), "kg_preload_kernels")
        global preloaded_kernels
        preloaded_kernels = n.value
    return lib


preloaded_kernels = 0


def last_error() -> str:
    buf = ctypes.create_string_buffer(512)
    load().kg_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def check(status: int, what: str = "") -> None:
    if status != 0:
        cls = STATUS_ERRORS.get(int(status), KGError)
        raise cls(f"{what}: {last_error()}" if what else last_error())


SLOW_CALLS = os.environ.get("KG_SLOW_CALLS", "0") == "1"   # diagnostics: library calls > 5 ms of host time
slow_calls: list = []


def call(name: str, *args):
    """Invoke a kg_status-returning entry point and raise on failure."""
    fn = getattr(require_cuda(), name)
    if SLOW_CALLS:
        import time
        t0 = time.perf_counter()
        st = fn(*args)
        dt = (time.perf_counter() - t0) * 1e3
        if dt > 5:
            slow_calls.append((name, round(dt, 1)))
        check(st, name)
        return
    check(fn(*args), name)


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


_persistent_pools: dict = {}


def persistent_pool(key):
    """A CUDA-graph memory pool that outlives the graphs captured into it: a
    one-node anchor graph keeps it referenced, so when a trainer's graphs are
    destroyed their memory returns to this pool and the next trainer's
    captures reuse it (no new device segments per train() call, no growth).
    Only for graphs that never run concurrently with each other (one pool per
    device for the round graphs, one per device and worker for the sampler's
    epoch graphs, all on one stream) and whose owner synchronises before
    destroying them (Trainer.close())."""
    torch = _torch_mod()
    hit = _persistent_pools.get(key)
    if hit is None:
        handle = torch.cuda.graph_pool_handle()
        anchor = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            anchor.capture_begin(pool=handle)
            torch.zeros(1, device="cuda")
            anchor.capture_end()
        torch.cuda.current_stream().wait_stream(side)
        hit = _persistent_pools[key] = (handle, anchor)
    return hit[0]


_cached_streams: dict = {}


def cached_stream(key, device, priority: int = 0):
    """A process-wide CUDA stream per key (stream creation is a driver call;
    successive trainers reuse theirs, and work of an earlier trainer on the
    same key stays ordered before the new one's)."""
    torch = _torch_mod()
    st = _cached_streams.get(key)
    if st is None:
        st = _cached_streams[key] = torch.cuda.Stream(device, priority=priority)
    return st


def _torch_mod():
    import torch
    return torch


CAPTURE_TIMES = os.environ.get("KG_CAPTURE_TIMES", "0") == "1"   # diagnostics
capture_times: list = []   # (begin, body, end+instantiate, upload) ms per capture


def capture(graph, body, pool=None) -> None:
    """Capture body() into `graph` on the current stream and upload it.
    The cyclic garbage collector is held off while capturing: it could
    otherwise destroy an unreachable earlier trainer's CUDA graphs or events
    mid-capture, which invalidates the capture."""
    import gc
    import time
    t0 = time.perf_counter()
    enabled = gc.isenabled()
    gc.disable()
    try:
        if pool is None:
            graph.capture_begin()
        else:
            graph.capture_begin(pool=pool)
        t1 = time.perf_counter()
        try:
            body()
        finally:
            t2 = time.perf_counter()
            graph.capture_end()
    finally:
        if enabled:
            gc.enable()
    t3 = time.perf_counter()
    graph_upload(graph)
    if CAPTURE_TIMES:
        capture_times.append((round((t1 - t0) * 1e3, 2), round((t2 - t1) * 1e3, 2), round((t3 - t2) * 1e3, 2),
                              round((time.perf_counter() - t3) * 1e3, 2)))


def graph_upload(graph) -> None:
    """Upload a just-instantiated torch CUDAGraph to the device now (the
    first replay would otherwise pay for it inside the timed loop)."""
    call("kg_graph_upload", graph.raw_cuda_graph_exec(), stream_handle())


def stream_handle() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream


class Workspace:
    """Grow-only scratch buffers keyed by purpose (one device allocation each)."""

    def __init__(self, device):
        self.device = device
        self._bufs = {}

    def get(self, key: str, nbytes: int):
        import torch
        nbytes = max(int(nbytes), 256)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(nbytes + (nbytes >> 3), dtype=torch.uint8, device=self.device)
            self._bufs[key] = buf
        return buf


# ---------------------------------------------------------------------------
# numpy Generator <-> kg_pcg64
# ---------------------------------------------------------------------------
M64 = (1 << 64) - 1


def pcg_from_numpy(gen: np.random.Generator) -> KgPcg64:
    st = gen.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise KGError("sampler streams require a numpy PCG64 Generator (np.random.default_rng)")
    s, inc = st["state"]["state"], st["state"]["inc"]
    return KgPcg64(s >> 64, s & M64, inc >> 64, inc & M64, st["has_uint32"], st["uinteger"])


def pcg_to_numpy(g: KgPcg64, gen: np.random.Generator) -> None:
    gen.bit_generator.state = {
        "bit_generator": "PCG64",
        "state": {"state": (g.state_hi << 64) | g.state_lo, "inc": (g.inc_hi << 64) | g.inc_lo},
        "has_uint32": int(g.has_uint32), "uinteger": int(g.uinteger)}


def pcg_copy(g: KgPcg64) -> KgPcg64:
    return KgPcg64(g.state_hi, g.state_lo, g.inc_hi, g.inc_lo, g.has_uint32, g.uinteger)


def pcg_advance(g: KgPcg64, delta: int) -> None:
    load().kg_pcg64_advance(ctypes.byref(g), c_uint64(delta))


def pcg_consume32(g: KgPcg64, count: int) -> None:
    load().kg_pcg64_consume32(ctypes.byref(g), c_uint64(count))


def kernel_breakdown(fn, *args, **kw):
    """Run fn with every library launch bracketed by CUDA events (warm, in
    situ); returns ({kernel: (launches, total_ms)}, fn's result)."""
    lib = require_cuda()
    lib.kg_kernel_timer_begin(b"")
    try:
        res = fn(*args, **kw)
    finally:
        buf = ctypes.create_string_buffer(1 << 16)
        lib.kg_kernel_timer_dump(buf, 1 << 16)
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.rsplit(",", 2)
        out[name] = (int(cnt), float(ms))
    return out, res


# ---------------------------------------------------------------------------
# device-resident PCG64 state (40-byte kg_pcg64 in HBM)
# ---------------------------------------------------------------------------
def pcg_to_device(g: KgPcg64, device):
    import torch
    raw = np.frombuffer(bytes(g), dtype=np.uint8).copy()
    return torch.as_tensor(raw).to(device)


def pcg_from_device(t) -> KgPcg64:
    raw = t.cpu().numpy().tobytes()
    return KgPcg64.from_buffer_copy(raw[: ctypes.sizeof(KgPcg64)])
