// R1/R2: partition view build on the GPU.
//
// Replaces ref:partition.py:61-74 (local ids by first appearance) and
// ref:sampler.py:73-118 (bidirectional messages, stable dst sort, 1/c norms,
// positive keys). Every order is reproduced exactly by stable radix sorts:
//   S1 key dst                -> reference message order (np.argsort stable)
//   S2 key dst*2R + rel       -> working CSR, relation-sorted rows, norm runs
//   S3 key src*2R + rel       -> CSC (messages by source) for the backward
//   S4 key csc rel            -> relation groups for d coeff reductions
//   S5 key (h*R+r)*n+t        -> sorted unique positive keys
#include "kg_common.cuh"

namespace kg {

static int bits_for(uint64_t maxval) {
  int b = 0;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

constexpr uint32_t NONE32 = 0xFFFFFFFFu;

__global__ void k_fill_u32(uint32_t* a, int64_t n, uint32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

__global__ void k_fill_i32(int32_t* a, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

// first[v] = min position of v in (h0,t0,h1,t1,...) of triples (m,3)
__global__ void k_first_seen(const int32_t* __restrict__ tri, int64_t m, uint32_t* __restrict__ first,
                             const uint32_t* __restrict__ exclude) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * m;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = i >> 1;
    int32_t v = tri[e * 3 + ((i & 1) ? 2 : 0)];
    if (exclude && exclude[v] != NONE32) continue;
    atomicMin(&first[v], (uint32_t)i);
  }
}

__global__ void k_first_keys(const uint32_t* __restrict__ first, int64_t N, uint32_t sentinel,
                             uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, int32_t* __restrict__ count) {
  int local = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N; v += (int64_t)gridDim.x * blockDim.x) {
    uint32_t f = first[v];
    keys[v] = (f == NONE32) ? sentinel : f;
    vals[v] = (uint32_t)v;
    local += (f != NONE32);
  }
  local = __reduce_add_sync(0xffffffffu, local);
  if (lane_id() == 0 && local) atomicAdd(count, local);
}

__global__ void k_assemble_local(const uint32_t* __restrict__ core_v, const uint32_t* __restrict__ sup_v,
                                 const int32_t* __restrict__ counts, int64_t N, int32_t* __restrict__ local_ids,
                                 int32_t* __restrict__ g2l, int32_t* __restrict__ n_local) {
  int32_t nc = counts[0], ns = counts[1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nc) {
      int32_t v = (int32_t)core_v[i];
      local_ids[i] = v;
      g2l[v] = (int32_t)i;
    }
    if (i < ns) {
      int32_t v = (int32_t)sup_v[i];
      local_ids[nc + i] = v;
      g2l[v] = (int32_t)(nc + i);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_local = nc + ns;
}

// ---------------------------------------------------------------------------
// message graph
// ---------------------------------------------------------------------------
__global__ void k_localize(const int32_t* __restrict__ eg, int64_t m, const int32_t* __restrict__ g2l,
                           int32_t* __restrict__ el) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    el[e * 3 + 0] = g2l[eg[e * 3 + 0]];
    el[e * 3 + 1] = eg[e * 3 + 1];
    el[e * 3 + 2] = g2l[eg[e * 3 + 2]];
  }
}

struct Msg {
  int32_t src, dst, rel;
};

__device__ __forceinline__ Msg msg_of(const int32_t* __restrict__ el, int64_t m, int32_t R, int64_t i) {
  Msg x;
  if (i < m) {
    x.src = el[i * 3 + 0];
    x.dst = el[i * 3 + 2];
    x.rel = el[i * 3 + 1];
  } else {
    int64_t e = i - m;
    x.src = el[e * 3 + 2];
    x.dst = el[e * 3 + 0];
    x.rel = el[e * 3 + 1] + R;
  }
  return x;
}

// which: 0 dst, 1 dst*2R+rel, 2 src*2R+rel
__global__ void k_msg_keys(const int32_t* __restrict__ el, int64_t m, int32_t R, int which,
                           uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * m; i += (int64_t)gridDim.x * blockDim.x) {
    Msg x = msg_of(el, m, R, i);
    uint64_t k;
    if (which == 0) k = (uint64_t)x.dst;
    else if (which == 1) k = (uint64_t)x.dst * (uint64_t)(2 * R) + (uint64_t)x.rel;
    else k = (uint64_t)x.src * (uint64_t)(2 * R) + (uint64_t)x.rel;
    keys[i] = k;
    vals[i] = (uint32_t)i;
  }
}

__global__ void k_count_rows(const int32_t* __restrict__ el, int64_t m, int use_src, uint32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * m; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = i < m ? i : i - m;
    bool fwd = i < m;
    // message src = fwd ? h : t ; dst = fwd ? t : h
    int32_t v = use_src ? el[e * 3 + (fwd ? 0 : 2)] : el[e * 3 + (fwd ? 2 : 0)];
    atomicAdd(&cnt[v], 1u);
  }
}

__global__ void k_u32_to_i32_ptr(const uint32_t* __restrict__ a, int32_t* __restrict__ b, int64_t n, int32_t last) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (i < n) ? (int32_t)a[i] : last;
}

// run boundaries of sorted keys -> flags
__global__ void k_boundaries(const uint64_t* __restrict__ keys, int64_t n, uint32_t* __restrict__ flags) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    flags[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1u : 0u;
}

// run length for each sorted position -> count per message id
__global__ void k_run_lengths(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ run_id_excl,
                              const int32_t* __restrict__ run_start, int32_t nruns_host_unused,
                              const uint32_t* __restrict__ nruns, const uint32_t* __restrict__ perm, int64_t n,
                              int32_t* __restrict__ cnt_by_msg) {
  uint32_t R = *nruns;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    uint32_t id = run_id_excl[k] + flags[k] - 1;   // inclusive id - 1
    int64_t s = run_start[id];
    int64_t e = (id + 1 < R) ? run_start[id + 1] : n;
    cnt_by_msg[perm[k]] = (int32_t)(e - s);
  }
}

__global__ void k_scatter_run_starts(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ run_id_excl,
                                     int64_t n, int32_t* __restrict__ run_start) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    if (flags[k]) run_start[run_id_excl[k]] = (int32_t)k;
}

// gather layout arrays from a message permutation
__global__ void k_gather_ref(const int32_t* __restrict__ el, int64_t m, int32_t R, const uint32_t* __restrict__ perm,
                             const int32_t* __restrict__ cnt_by_msg, int32_t* __restrict__ src,
                             int32_t* __restrict__ rel, int32_t* __restrict__ cnt) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 2 * m; k += (int64_t)gridDim.x * blockDim.x) {
    uint32_t i = perm[k];
    Msg x = msg_of(el, m, R, i);
    src[k] = x.src;
    rel[k] = x.rel;
    cnt[k] = cnt_by_msg[i];
  }
}

__global__ void k_gather_csr(const int32_t* __restrict__ el, int64_t m, int32_t R, const uint32_t* __restrict__ perm,
                             const int32_t* __restrict__ cnt_by_msg, int use_dst, int32_t* __restrict__ other,
                             int32_t* __restrict__ rel, float* __restrict__ norm) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 2 * m; k += (int64_t)gridDim.x * blockDim.x) {
    uint32_t i = perm[k];
    Msg x = msg_of(el, m, R, i);
    other[k] = use_dst ? x.dst : x.src;
    rel[k] = x.rel;
    norm[k] = 1.0f / (float)cnt_by_msg[i];
  }
}

__global__ void k_rel_keys(const int32_t* __restrict__ c_rel, int64_t e, uint64_t* __restrict__ keys,
                           uint32_t* __restrict__ vals, uint32_t* __restrict__ gcount) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < e; k += (int64_t)gridDim.x * blockDim.x) {
    keys[k] = (uint64_t)c_rel[k];
    vals[k] = (uint32_t)k;
    atomicAdd(&gcount[c_rel[k]], 1u);
  }
}

__global__ void k_u32_copy_i32(const uint32_t* __restrict__ a, int32_t* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (int32_t)a[i];
}

__global__ void k_pos_keys(const int32_t* __restrict__ el, int64_t m, int32_t n, int32_t R,
                           uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (uint64_t)el[e * 3 + 0], r = (uint64_t)el[e * 3 + 1], t = (uint64_t)el[e * 3 + 2];
    keys[e] = (h * (uint64_t)R + r) * (uint64_t)n + t;
    vals[e] = (uint32_t)e;
  }
}

__global__ void k_gather_keys(const uint64_t* __restrict__ keys, const int32_t* __restrict__ idx,
                              const int32_t* __restrict__ count, int64_t cap, int64_t* __restrict__ out) {
  int32_t c = *count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap && i < c; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)keys[idx[i]];
}

static int grid_for(int64_t n) { return persistent_blocks(n, 256, 8); }

}  // namespace kg

using namespace kg;

extern "C" {

int64_t kg_view_workspace_bytes(int64_t m, int64_t num_entities) {
  int64_t e = 2 * m;
  int64_t big = e > num_entities ? e : num_entities;
  size_t b = 0;
  b += align_up(big * sizeof(uint64_t));          // keys
  b += align_up(big * sizeof(uint32_t));          // vals / perm
  b += align_up(big * sizeof(uint32_t)) * 3;      // flags / scan / misc
  b += align_up(big * sizeof(int32_t)) * 2;       // cnt_by_msg, run_start
  b += align_up((num_entities + 1) * sizeof(uint32_t)) * 2;
  b += sort_workspace(big);
  b += compact_workspace(big);
  b += scan_workspace(big);
  return (int64_t)(b + 8192);
}

kg_status kg_view_local_ids(const int32_t* core, int64_t m_core, const int32_t* support, int64_t m_sup,
                            int64_t N, int32_t* local_ids, int32_t* g2l, int32_t* n_local, void* ws,
                            int64_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(N > 0 && N < (int64_t(1) << 31), KG_ERR_VALIDATION, "num_entities out of range");
  KG_REQUIRE((size_t)ws_bytes >= (size_t)kg_view_workspace_bytes(m_core + m_sup, N), KG_ERR_VALIDATION,
             "view workspace too small");
  Arena a(ws, (size_t)ws_bytes);
  uint32_t* first_c = a.take<uint32_t>(N);
  uint32_t* first_s = a.take<uint32_t>(N);
  uint32_t* keys = a.take<uint32_t>(N);
  uint32_t* vals = a.take<uint32_t>(N);
  uint32_t* keys2 = a.take<uint32_t>(N);
  uint32_t* vals2 = a.take<uint32_t>(N);
  int32_t* counts = a.take<int32_t>(2);
  char* sws = a.take<char>(sort32_workspace(N));
  int g = grid_for(N);
  KG_LAUNCH("k_fill_u32", k_fill_u32, g, 256, 0, st, first_c, N, NONE32);
  KG_LAUNCH("k_fill_u32", k_fill_u32, g, 256, 0, st, first_s, N, NONE32);
  KG_LAUNCH("k_fill_i32", k_fill_i32, g, 256, 0, st, g2l, N, -1);
  KG_CUDA(cudaMemsetAsync(counts, 0, 2 * sizeof(int32_t), st));
  if (m_core) KG_LAUNCH("k_first_seen", k_first_seen, grid_for(2 * m_core), 256, 0, st, core, m_core, first_c, nullptr);
  if (m_sup) KG_LAUNCH("k_first_seen", k_first_seen, grid_for(2 * m_sup), 256, 0, st, support, m_sup, first_s, first_c);
  KG_CHECK_LAUNCH("k_first_seen");
  uint32_t sent_c = (uint32_t)(2 * m_core), sent_s = (uint32_t)(2 * m_sup);
  KG_LAUNCH("k_first_keys", k_first_keys, g, 256, 0, st, first_c, N, sent_c, keys, vals, counts + 0);
  KG_LAUNCH("k_first_keys", k_first_keys, g, 256, 0, st, first_s, N, sent_s, keys2, vals2, counts + 1);
  KG_CHECK_LAUNCH("k_first_keys");
  kg_status s = sort_pairs_u32(keys, vals, N, bits_for(sent_c), sws, sort32_workspace(N), st);
  if (s != KG_OK) return s;
  s = sort_pairs_u32(keys2, vals2, N, bits_for(sent_s), sws, sort32_workspace(N), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_assemble_local", k_assemble_local, g, 256, 0, st, vals, vals2, counts, N, local_ids, g2l, n_local);
  KG_CHECK_LAUNCH("k_assemble_local");
  return KG_OK;
}

kg_status kg_view_build(const int32_t* edges_global, int64_t m, const int32_t* g2l, int32_t* el,
                        int32_t* ref_src, int32_t* ref_rel, int32_t* msg_cnt, const kg_graph_csr* G,
                        int64_t* pos_keys, int32_t* n_keys, void* ws, int64_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  const int32_t n = G->n, R = G->R;
  const int64_t e = 2 * m;
  KG_REQUIRE(n > 0, KG_ERR_VALIDATION, "empty partition");
  KG_REQUIRE(e < (int64_t(1) << 31), KG_ERR_VALIDATION, "too many messages for int32 ids");
  KG_REQUIRE((size_t)ws_bytes >= (size_t)kg_view_workspace_bytes(m, n), KG_ERR_VALIDATION,
             "view workspace too small");
  Arena a(ws, (size_t)ws_bytes);
  int64_t big = e > n ? e : n;
  uint64_t* keys = a.take<uint64_t>(big);
  uint32_t* perm = a.take<uint32_t>(big);
  uint32_t* flags = a.take<uint32_t>(big);
  uint32_t* scan = a.take<uint32_t>(big);
  uint32_t* misc = a.take<uint32_t>(big);
  int32_t* cnt_by_msg = a.take<int32_t>(big);
  int32_t* run_start = a.take<int32_t>(big);
  uint32_t* rowcnt = a.take<uint32_t>(n + 1);
  uint32_t* nruns = a.take<uint32_t>(4);
  char* sws = a.take<char>(sort_workspace(big));
  char* cws = a.take<char>(compact_workspace(big));
  char* scws = a.take<char>(scan_workspace(big));
  int g = grid_for(e);
  kg_status s;

  if (m == 0) {
    KG_CUDA(cudaMemsetAsync(G->indptr, 0, (n + 1) * sizeof(int32_t), st));
    KG_CUDA(cudaMemsetAsync(G->c_indptr, 0, (n + 1) * sizeof(int32_t), st));
    KG_CUDA(cudaMemsetAsync(G->rel_ptr, 0, (2 * R + 1) * sizeof(int32_t), st));
    KG_CUDA(cudaMemsetAsync(n_keys, 0, sizeof(int32_t), st));
    kg_status s0 = build_chunk_table(G->indptr, n, G->chunk, G->ck_ptr, G->ck_row, G->ck_slot, G->ck_split,
                                     G->ck_counts, G->ck_desc, ws, (size_t)ws_bytes, st);
    if (s0 != KG_OK) return s0;
    return build_chunk_table(G->c_indptr, n, G->chunk, G->cc_ptr, G->cc_row, G->cc_slot, G->cc_split, G->cc_counts,
                             G->cc_desc, ws, (size_t)ws_bytes, st);
  }
  KG_LAUNCH("k_localize", k_localize, grid_for(m), 256, 0, st, edges_global, m, g2l, el);
  KG_CHECK_LAUNCH("k_localize");

  // destination CSR indptr (shared by reference order and working CSR)
  KG_CUDA(cudaMemsetAsync(rowcnt, 0, (n + 1) * sizeof(uint32_t), st));
  KG_LAUNCH("k_count_rows", k_count_rows, g, 256, 0, st, el, m, 0, rowcnt);
  s = exclusive_scan_u32(rowcnt, rowcnt, n, nullptr, scws, scan_workspace(big), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_u32_to_i32_ptr", k_u32_to_i32_ptr, grid_for(n + 1), 256, 0, st, rowcnt, G->indptr, n, (int32_t)e);

  // S2: (dst, rel) runs -> counts c_{dst,rel} per message, working CSR
  KG_LAUNCH("k_msg_keys", k_msg_keys, g, 256, 0, st, el, m, R, 1, keys, perm);
  s = sort_pairs_u64(keys, perm, e, bits_for((uint64_t)n * 2 * R), sws, sort_workspace(big), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_boundaries", k_boundaries, g, 256, 0, st, keys, e, flags);
  s = exclusive_scan_u32(flags, scan, e, nruns, scws, scan_workspace(big), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_scatter_run_starts", k_scatter_run_starts, g, 256, 0, st, flags, scan, e, run_start);
  KG_LAUNCH("k_run_lengths", k_run_lengths, g, 256, 0, st, flags, scan, run_start, 0, nruns, perm, e, cnt_by_msg);
  KG_LAUNCH("k_gather_csr", k_gather_csr, g, 256, 0, st, el, m, R, perm, cnt_by_msg, 0, G->src, G->rel, G->norm);
  KG_CHECK_LAUNCH("working csr");

  // S1: reference order (stable by destination)
  KG_LAUNCH("k_msg_keys", k_msg_keys, g, 256, 0, st, el, m, R, 0, keys, perm);
  s = sort_pairs_u64(keys, perm, e, bits_for((uint64_t)n), sws, sort_workspace(big), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_gather_ref", k_gather_ref, g, 256, 0, st, el, m, R, perm, cnt_by_msg, ref_src, ref_rel, msg_cnt);
  KG_CHECK_LAUNCH("reference order");

  // S3: CSC by (src, rel)
  KG_CUDA(cudaMemsetAsync(rowcnt, 0, (n + 1) * sizeof(uint32_t), st));
  KG_LAUNCH("k_count_rows", k_count_rows, g, 256, 0, st, el, m, 1, rowcnt);
  s = exclusive_scan_u32(rowcnt, rowcnt, n, nullptr, scws, scan_workspace(big), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_u32_to_i32_ptr", k_u32_to_i32_ptr, grid_for(n + 1), 256, 0, st, rowcnt, G->c_indptr, n, (int32_t)e);
  KG_LAUNCH("k_msg_keys", k_msg_keys, g, 256, 0, st, el, m, R, 2, keys, perm);
  s = sort_pairs_u64(keys, perm, e, bits_for((uint64_t)n * 2 * R), sws, sort_workspace(big), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_gather_csr", k_gather_csr, g, 256, 0, st, el, m, R, perm, cnt_by_msg, 1, G->c_dst, G->c_rel, G->c_norm);
  KG_CHECK_LAUNCH("csc");

  // S4: CSC positions grouped by relation
  KG_CUDA(cudaMemsetAsync(misc, 0, (2 * R + 1) * sizeof(uint32_t), st));
  KG_LAUNCH("k_rel_keys", k_rel_keys, g, 256, 0, st, G->c_rel, e, keys, perm, misc);
  s = sort_pairs_u64(keys, perm, e, bits_for((uint64_t)2 * R), sws, sort_workspace(big), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_u32_copy_i32", k_u32_copy_i32, g, 256, 0, st, perm, G->rel_perm, e);
  s = exclusive_scan_u32(misc, misc, 2 * R, nullptr, scws, scan_workspace(big), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_u32_to_i32_ptr", k_u32_to_i32_ptr, 1, 256, 0, st, misc, G->rel_ptr, 2 * R, (int32_t)e);
  KG_CHECK_LAUNCH("relation groups");

  // S5: sorted unique positive keys
  KG_LAUNCH("k_pos_keys", k_pos_keys, grid_for(m), 256, 0, st, el, m, n, R, keys, perm);
  uint64_t maxkey = ((uint64_t)(n - 1) * (uint64_t)R + (uint64_t)(R - 1)) * (uint64_t)n + (uint64_t)(n - 1);
  s = sort_pairs_u64(keys, perm, m, bits_for(maxkey), sws, sort_workspace(big), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_boundaries", k_boundaries, grid_for(m), 256, 0, st, keys, m, flags);
  s = compact_flags(flags, m, reinterpret_cast<int32_t*>(misc), n_keys, 0, nullptr, cws, compact_workspace(big), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_gather_keys", k_gather_keys, grid_for(m), 256, 0, st, keys, reinterpret_cast<int32_t*>(misc), n_keys, m, pos_keys);
  KG_CHECK_LAUNCH("positive keys");

  // static work chunks for hub rows (destination CSR and source CSC)
  KG_REQUIRE(G->chunk >= 1, KG_ERR_VALIDATION, "chunk size must be >= 1");
  KG_REQUIRE((size_t)ws_bytes >= chunk_workspace(n), KG_ERR_VALIDATION, "view workspace too small for chunks");
  s = build_chunk_table(G->indptr, n, G->chunk, G->ck_ptr, G->ck_row, G->ck_slot, G->ck_split, G->ck_counts,
                        G->ck_desc, ws,
                        (size_t)ws_bytes, st);
  if (s != KG_OK) return s;
  s = build_chunk_table(G->c_indptr, n, G->chunk, G->cc_ptr, G->cc_row, G->cc_slot, G->cc_split, G->cc_counts,
                        G->cc_desc, ws,
                        (size_t)ws_bytes, st);
  if (s != KG_OK) return s;
  return KG_OK;
}

}  // extern "C"

// this module's anchor for kg_preload_kernels (kg_primitives.cu)
extern "C" const void* kg_anchor_view() { return reinterpret_cast<const void*>(&kg::k_fill_u32); }
