// Static work chunks over a CSR (hub rows).
//
// FB15k-237's preferential-attachment hubs receive ~8.4k messages while the
// mean row has ~37; a warp per row serialises the hub. Every row v is cut
// into max(1, ceil(deg(v)/C)) chunks of <= C messages; one warp processes one
// chunk, rows with a single chunk write their result directly and rows with
// several chunks write per-chunk partials that a second pass adds in chunk
// order (deterministic). The table depends only on the partition, so it is
// built once per view.
#include "kg_common.cuh"

namespace kg {

__global__ void k_chunk_counts(const int32_t* __restrict__ indptr, int32_t n, int C, uint32_t* __restrict__ nch,
                               uint32_t* __restrict__ split_flag) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    int32_t deg = indptr[v + 1] - indptr[v];
    uint32_t k = deg > 0 ? (uint32_t)((deg + C - 1) / C) : 1u;
    nch[v] = k;
    split_flag[v] = k > 1 ? k : 0u;   // number of partial slots this row needs
  }
}

__global__ void k_chunk_fill(const uint32_t* __restrict__ nch, const uint32_t* __restrict__ ptr_u,
                             const uint32_t* __restrict__ slot_base, int32_t n, int32_t* __restrict__ ptr,
                             int32_t* __restrict__ row, int32_t* __restrict__ slot, const uint32_t* __restrict__ total) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    uint32_t a = ptr_u[v], k = nch[v];
    ptr[v] = (int32_t)a;
    for (uint32_t j = 0; j < k; ++j) {
      row[a + j] = (int32_t)v;
      slot[a + j] = k > 1 ? (int32_t)(slot_base[v] + j) : -1;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ptr[n] = (int32_t)*total;
}

__global__ void k_split_flags(const uint32_t* __restrict__ nch, int32_t n, uint32_t* __restrict__ f) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    f[v] = nch[v] > 1 ? 1u : 0u;
}

__global__ void k_chunk_desc(const int32_t* __restrict__ indptr, int32_t n, int C, const int32_t* __restrict__ ptr,
                             const int32_t* __restrict__ slot, const uint32_t* __restrict__ total,
                             int4* __restrict__ desc) {
  const int64_t nc = *total;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c0 = ptr[v], k = ptr[v + 1] - c0, lo = indptr[v], hi = indptr[v + 1];
    for (int32_t j = 0; j < k && c0 + j < nc; ++j) {
      const int32_t beg = lo + j * C, cnt = min(beg + C, hi) - beg;
      desc[c0 + j] = make_int4(v, beg, cnt | (k == 1 ? 1 << 16 : 0) | (j == 0 ? 1 << 17 : 0), slot[c0 + j]);
    }
  }
}

__global__ void k_chunk_totals(const uint32_t* __restrict__ tot_chunks, const uint32_t* __restrict__ tot_slots,
                               int32_t* __restrict__ counts) {
  counts[0] = (int32_t)*tot_chunks;
  counts[1] = (int32_t)*tot_slots;
}

size_t chunk_workspace(int64_t n) {
  return align_up(n * 4) * 5 + scan_workspace(n) * 2 + compact_workspace(n) + 4096;
}

kg_status build_chunk_table(const int32_t* indptr, int32_t n, int C, int32_t* ptr, int32_t* row, int32_t* slot,
                            int32_t* split, int32_t* counts, int32_t* desc, void* ws, size_t ws_bytes,
                            cudaStream_t st) {
  KG_REQUIRE(ws_bytes >= chunk_workspace(n), KG_ERR_VALIDATION, "chunk workspace too small");
  Arena a(ws, ws_bytes);
  uint32_t* nch = a.take<uint32_t>(n);
  uint32_t* ptr_u = a.take<uint32_t>(n);
  uint32_t* slots = a.take<uint32_t>(n);
  uint32_t* slot_base = a.take<uint32_t>(n);
  uint32_t* tots = a.take<uint32_t>(4);
  char* sws = a.take<char>(scan_workspace(n));
  char* cws = a.take<char>(compact_workspace(n));
  int g = persistent_blocks(n, 256, 8);
  KG_LAUNCH("k_chunk_counts", k_chunk_counts, g, 256, 0, st, indptr, n, C, nch, slots);
  kg_status s = exclusive_scan_u32(nch, ptr_u, n, tots + 0, sws, scan_workspace(n), st);
  if (s != KG_OK) return s;
  s = exclusive_scan_u32(slots, slot_base, n, tots + 1, sws, scan_workspace(n), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_chunk_fill", k_chunk_fill, g, 256, 0, st, nch, ptr_u, slot_base, n, ptr, row, slot, tots + 0);
  KG_LAUNCH("k_split_flags", k_split_flags, g, 256, 0, st, nch, n, slots);
  s = compact_flags(slots, n, split, counts + 2, 0, nullptr, cws, compact_workspace(n), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_chunk_totals", k_chunk_totals, 1, 1, 0, st, tots + 0, tots + 1, counts);
  if (desc)
    KG_LAUNCH("k_chunk_desc", k_chunk_desc, g, 256, 0, st, indptr, n, C, ptr, slot, tots + 0,
              reinterpret_cast<int4*>(desc));
  return KG_OK;
}

}  // namespace kg

// this module's anchor for kg_preload_kernels (kg_primitives.cu)
extern "C" const void* kg_anchor_chunks() { return reinterpret_cast<const void*>(&kg::k_chunk_counts); }
