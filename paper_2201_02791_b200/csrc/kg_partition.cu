// N1: n-hop halo expansion on the GPU (ref:partition.py:211-282).
//
// The reference expands each partition with a set-valued BFS over the
// incident-edge CSR: the frontier starts as the core-edge endpoints; each hop
// marks every edge incident to a frontier vertex as included and makes the
// endpoints of those edges not seen before the next frontier. Its outputs are
// sorted sets (support edge ids, support vertices), so any traversal order
// gives the same partition: here a warp per frontier vertex marks flags in
// parallel and stream compaction emits the sets in ascending order —
// bit-identical to the reference by construction. wikikg2 / citation2 shapes
// (16M / 30M edges, P = 8): numpy took 46 / 85 s for all partitions.
#include "kg_common.cuh"

namespace kg {

__global__ void k_inc_count(const int32_t* __restrict__ tri, int64_t m, uint32_t* __restrict__ deg) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    atomicAdd(deg + tri[e * 3], 1u);
    atomicAdd(deg + tri[e * 3 + 2], 1u);
  }
}

__global__ void k_inc_fill(const int32_t* __restrict__ tri, int64_t m, const uint32_t* __restrict__ ptr,
                           uint32_t* __restrict__ cursor, int32_t* __restrict__ inc) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = tri[e * 3], w = tri[e * 3 + 2];
    inc[ptr[u] + atomicAdd(cursor + u, 1u)] = (int32_t)e;
    inc[ptr[w] + atomicAdd(cursor + w, 1u)] = (int32_t)e;
  }
}

__global__ void k_halo_init(const int32_t* __restrict__ tri, const int32_t* __restrict__ core_ids, int64_t n_core,
                            uint32_t* __restrict__ edge_in, uint32_t* __restrict__ core_e,
                            uint32_t* __restrict__ seen, uint32_t* __restrict__ is_core) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_core; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = core_ids[i];
    edge_in[e] = 1u;
    core_e[e] = 1u;
    const int32_t u = tri[(int64_t)e * 3], w = tri[(int64_t)e * 3 + 2];
    seen[u] = seen[w] = 1u;
    is_core[u] = is_core[w] = 1u;
  }
}

// one warp per frontier vertex: include its incident edges, flag the
// endpoints not seen before this hop
__global__ void __launch_bounds__(256) k_halo_hop(const int32_t* __restrict__ tri,
                                                  const uint32_t* __restrict__ ptr, const int32_t* __restrict__ inc,
                                                  const int32_t* __restrict__ front, const int32_t* __restrict__ nfront,
                                                  uint32_t* __restrict__ edge_in, const uint32_t* __restrict__ seen,
                                                  uint32_t* __restrict__ next) {
  const int lane = (int)lane_id(), nw = (gridDim.x * blockDim.x) >> 5;
  const int64_t nf = *nfront;
  for (int64_t i = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); i < nf; i += nw) {
    const int32_t v = front[i];
    for (uint32_t k = ptr[v] + lane; k < ptr[v + 1]; k += 32) {
      const int32_t e = inc[k];
      edge_in[e] = 1u;
      const int32_t a = tri[(int64_t)e * 3], b = tri[(int64_t)e * 3 + 2];
      if (!seen[a]) next[a] = 1u;
      if (!seen[b]) next[b] = 1u;
    }
  }
}

__global__ void k_halo_merge(int64_t n, uint32_t* __restrict__ next, uint32_t* __restrict__ seen) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    if (next[v]) seen[v] = 1u;
  }
}

// flags for the outputs: support edges = included and not core; support
// vertices = seen and not a core endpoint
__global__ void k_halo_outputs(int64_t m, int64_t n, const uint32_t* __restrict__ core_e,
                               uint32_t* __restrict__ edge_in, const uint32_t* __restrict__ is_core,
                               uint32_t* __restrict__ seen) {
  const int64_t tot = m > n ? m : n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < m && core_e[i]) edge_in[i] = 0u;
    if (i < n && is_core[i]) seen[i] = 0u;
  }
}

struct HaloWs {
  uint32_t *deg, *ptr, *cursor, *edge_in, *core_e, *seen, *is_core, *next;
  int32_t *front, *nfront;
  char* cws;
};

static size_t halo_ws(int64_t m, int64_t n, HaloWs* w, void* base, size_t cap) {
  Arena a(base, cap);
  HaloWs r;
  r.deg = a.take<uint32_t>(n + 1);
  r.ptr = a.take<uint32_t>(n + 1);
  r.cursor = a.take<uint32_t>(n + 1);
  r.edge_in = a.take<uint32_t>(m);
  r.core_e = a.take<uint32_t>(m);
  r.seen = a.take<uint32_t>(n);
  r.is_core = a.take<uint32_t>(n);
  r.next = a.take<uint32_t>(n);
  r.front = a.take<int32_t>(n);
  r.nfront = a.take<int32_t>(4);
  const int64_t big = m > n + 1 ? m : n + 1;
  r.cws = a.take<char>(compact_workspace(big) > scan_workspace(big) ? compact_workspace(big) : scan_workspace(big));
  if (w) *w = r;
  return a.used + 1024;
}

}  // namespace kg

using namespace kg;

extern "C" {

int64_t kg_halo_workspace_bytes(int64_t m, int64_t n) { return (int64_t)halo_ws(m, n, nullptr, nullptr, 0); }

kg_status kg_halo_incidence(const int32_t* tri, int64_t m, int64_t n, uint32_t* ptr_out, int32_t* inc, void* ws,
                            int64_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  HaloWs w;
  KG_REQUIRE((size_t)ws_bytes >= halo_ws(m, n, &w, ws, (size_t)ws_bytes), KG_ERR_VALIDATION,
             "halo workspace too small");
  KG_REQUIRE(2 * m < ((int64_t)1 << 32), KG_ERR_VALIDATION, "too many edges for a 32-bit incidence CSR");
  KG_CUDA(cudaMemsetAsync(w.deg, 0, (size_t)(n + 1) * 4, st));
  KG_CUDA(cudaMemsetAsync(w.cursor, 0, (size_t)(n + 1) * 4, st));
  KG_LAUNCH("k_inc_count", k_inc_count, persistent_blocks(m, 256, 8), 256, 0, st, tri, m, w.deg);
  kg_status s = exclusive_scan_u32(w.deg, ptr_out, n + 1, nullptr, w.cws, scan_workspace(n + 1), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_inc_fill", k_inc_fill, persistent_blocks(m, 256, 8), 256, 0, st, tri, m, ptr_out, w.cursor, inc);
  return KG_OK;
}

kg_status kg_halo_expand(const int32_t* tri, int64_t m, int64_t n, const uint32_t* ptr, const int32_t* inc,
                         const int32_t* core_ids, int64_t n_core, int32_t hops, int32_t* support_ids,
                         int32_t* n_support, int32_t* support_vertices, int32_t* n_support_vertices,
                         int32_t* core_vertices, int32_t* n_core_vertices, void* ws, int64_t ws_bytes,
                         void* stream) {
  cudaStream_t st = as_stream(stream);
  HaloWs w;
  KG_REQUIRE((size_t)ws_bytes >= halo_ws(m, n, &w, ws, (size_t)ws_bytes), KG_ERR_VALIDATION,
             "halo workspace too small");
  KG_REQUIRE(hops >= 0, KG_ERR_VALIDATION, "hops must be >= 0");
  KG_CUDA(cudaMemsetAsync(w.edge_in, 0, (size_t)m * 4, st));
  KG_CUDA(cudaMemsetAsync(w.core_e, 0, (size_t)m * 4, st));
  KG_CUDA(cudaMemsetAsync(w.seen, 0, (size_t)n * 4, st));
  KG_CUDA(cudaMemsetAsync(w.is_core, 0, (size_t)n * 4, st));
  KG_CUDA(cudaMemsetAsync(w.next, 0, (size_t)n * 4, st));
  if (n_core > 0)
    KG_LAUNCH("k_halo_init", k_halo_init, persistent_blocks(n_core, 256, 8), 256, 0, st, tri, core_ids, n_core,
              w.edge_in, w.core_e, w.seen, w.is_core);
  const size_t cw = compact_workspace(m > n ? m : n);
  // frontier 0 = the core endpoints (ascending)
  kg_status s = compact_flags(w.is_core, n, w.front, w.nfront, 0, nullptr, w.cws, cw, st);
  if (s != KG_OK) return s;
  for (int h = 0; h < hops; ++h) {
    KG_LAUNCH("k_halo_hop", k_halo_hop, persistent_blocks(n * 32, 256, 8), 256, 0, st, tri, ptr, inc, w.front,
              w.nfront, w.edge_in, w.seen, w.next);
    KG_LAUNCH("k_halo_merge", k_halo_merge, persistent_blocks(n, 256, 8), 256, 0, st, n, w.next, w.seen);
    // the next frontier: vertices first seen in this hop (flags cleared by compact_flags_ex)
    s = compact_flags_ex(w.next, n, w.front, nullptr, w.nfront, nullptr, w.cws, cw, st);
    if (s != KG_OK) return s;
  }
  s = compact_flags(w.is_core, n, core_vertices, n_core_vertices, 0, nullptr, w.cws, cw, st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_halo_outputs", k_halo_outputs, persistent_blocks(m > n ? m : n, 256, 8), 256, 0, st, m, n, w.core_e,
            w.edge_in, w.is_core, w.seen);
  s = compact_flags(w.edge_in, m, support_ids, n_support, 0, nullptr, w.cws, cw, st);
  if (s != KG_OK) return s;
  return compact_flags(w.seen, n, support_vertices, n_support_vertices, 0, nullptr, w.cws, cw, st);
}

}  // extern "C"

// this module's anchor for kg_preload_kernels (kg_primitives.cu)
extern "C" const void* kg_anchor_partition() { return reinterpret_cast<const void*>(&kg::k_inc_count); }
