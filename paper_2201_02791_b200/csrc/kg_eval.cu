// R25/R26: filtered link-prediction ranking (ref:evaluate.py:136-225).
//
// For every query triple and both corrupted sides the reference forms
// q = H[anchor] * decoder[r], scores = q @ H.T over all N entities, counts
// candidates scoring strictly greater / equal to the true entity, and then
// removes known (train+valid+test) collisions. Here the all-entity scoring is
// a tiled GEMM whose epilogue compares each score against the true score and
// only keeps two integer counts per query (the N-wide score row never
// reaches HBM). Known collisions come from sorted unique keys
// (a*R + r)*N + c, so the filter list of a query is one contiguous key range.
//
// Every score -- bulk tile, true score, filtered candidate -- is the same
// sequential fmaf chain over k = 0..d-1 starting from 0, so the comparisons
// are exact (the reference compares entries of one matrix, evaluate.py:200).
#include "kg_gemm.cuh"

namespace kg {

constexpr int QB = 64, CB = 64, KT = 32, ET = 256;

struct EvalArgs {
  const float* H;
  int d, N, R;
  const float* dec;
  const int32_t* qry;   // (nq, 3)
  int64_t nq;
  const float* true_score;   // (2*nq) [side*nq + q]
  unsigned long long* greater;
  unsigned long long* equal;
};

__device__ __forceinline__ float score_chain(const float* __restrict__ Ha, const float* __restrict__ M,
                                             const float* __restrict__ Hc, int d) {
  float s = 0.f;
  for (int k = 0; k < d; ++k) s = fmaf(Ha[k] * M[k], Hc[k], s);
  return s;
}

__global__ void k_true_scores(EvalArgs a, float* __restrict__ ts) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < 2 * a.nq; x += (int64_t)gridDim.x * blockDim.x) {
    int side = (int)(x / a.nq);
    int64_t q = x - side * a.nq;
    int32_t h = a.qry[q * 3], r = a.qry[q * 3 + 1], t = a.qry[q * 3 + 2];
    int32_t anc = side == 0 ? h : t, tru = side == 0 ? t : h;
    ts[x] = score_chain(a.H + (int64_t)anc * a.d, a.dec + (int64_t)r * a.d, a.H + (int64_t)tru * a.d, a.d);
  }
}

// block: QB (query,side) rows x all candidates in CB tiles; thread 4x4 outputs
__global__ void __launch_bounds__(ET) k_rank_tiles(EvalArgs a) {
  __shared__ float Qs[KT][QB + 4];
  __shared__ float Cs[KT][CB + 4];
  __shared__ unsigned gcnt[QB], ecnt[QB];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int64_t x0 = (int64_t)blockIdx.x * QB;   // row index over 2*nq
  if (tid < QB) { gcnt[tid] = 0; ecnt[tid] = 0; }
  float tsc[4];
  int64_t xi[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    xi[i] = x0 + ty * 4 + i;
    tsc[i] = xi[i] < 2 * a.nq ? a.true_score[xi[i]] : 0.f;
  }
  unsigned gl[4] = {0, 0, 0, 0}, el[4] = {0, 0, 0, 0};
  for (int64_t c0 = 0; c0 < a.N; c0 += CB) {
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    for (int k0 = 0; k0 < a.d; k0 += KT) {
      __syncthreads();
      for (int idx = tid; idx < QB * KT; idx += ET) {
        int qq = idx / KT, kk = idx % KT;
        int64_t x = x0 + qq;
        int k = k0 + kk;
        float v = 0.f;
        if (x < 2 * a.nq && k < a.d) {
          int side = (int)(x / a.nq);
          int64_t q = x - side * a.nq;
          int32_t anc = a.qry[q * 3 + (side == 0 ? 0 : 2)], r = a.qry[q * 3 + 1];
          v = a.H[(int64_t)anc * a.d + k] * a.dec[(int64_t)r * a.d + k];
        }
        Qs[kk][qq] = v;
      }
      for (int idx = tid; idx < CB * KT; idx += ET) {
        int cc = idx / KT, kk = idx % KT;
        int64_t c = c0 + cc;
        int k = k0 + kk;
        Cs[kk][cc] = (c < a.N && k < a.d) ? a.H[c * a.d + k] : 0.f;
      }
      __syncthreads();
      const int kmax = min(KT, a.d - k0);
      for (int kk = 0; kk < kmax; ++kk) {
        float qv[4], cv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) qv[i] = Qs[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) cv[j] = Cs[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(qv[i], cv[j], acc[i][j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t c = c0 + tx * 4 + j;
      if (c >= a.N) continue;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        gl[i] += acc[i][j] > tsc[i];
        el[i] += acc[i][j] == tsc[i];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    atomicAdd(&gcnt[ty * 4 + i], gl[i]);
    atomicAdd(&ecnt[ty * 4 + i], el[i]);
  }
  __syncthreads();
  if (tid < QB) {
    int64_t x = x0 + tid;
    if (x < 2 * a.nq) {
      a.greater[x] = gcnt[tid];
      a.equal[x] = ecnt[tid];
    }
  }
}

__device__ __forceinline__ int64_t lb64(const int64_t* __restrict__ k, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (k[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_rank_finish(EvalArgs a, const int64_t* __restrict__ tkeys, int64_t ntk,
                              const int64_t* __restrict__ hkeys, int64_t nhk, int policy, int chunk,
                              double* __restrict__ ranks, int32_t* __restrict__ ncand) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < 2 * a.nq; x += (int64_t)gridDim.x * blockDim.x) {
    int side = (int)(x / a.nq);
    int64_t q = x - side * a.nq;
    int32_t h = a.qry[q * 3], r = a.qry[q * 3 + 1], t = a.qry[q * 3 + 2];
    int32_t anc = side == 0 ? h : t, tru = side == 0 ? t : h;
    const int64_t* keys = side == 0 ? tkeys : hkeys;
    int64_t nk = side == 0 ? ntk : nhk;
    int64_t base = ((int64_t)anc * a.R + r) * (int64_t)a.N;
    int64_t lo = lb64(keys, nk, base), hi = lb64(keys, nk, base + a.N);
    float ts = a.true_score[x];
    long long g = (long long)a.greater[x];
    long long e = (long long)a.equal[x] - 1;   // the true entity itself
    int32_t nknown = 0;
    const float* Ha = a.H + (int64_t)anc * a.d;
    const float* M = a.dec + (int64_t)r * a.d;
    for (int64_t j = lo; j < hi; ++j) {
      int32_t c = (int32_t)(keys[j] - base);
      if (c == tru) continue;
      ++nknown;
      float s = score_chain(Ha, M, a.H + (int64_t)c * a.d, a.d);
      g -= s > ts;
      e -= s == ts;
    }
    double rank;
    if (policy == 0) rank = 1.0 + (double)g + (double)e / 2.0;
    else if (policy == 1) rank = 1.0 + (double)g;
    else rank = 1.0 + (double)g + (double)e;
    int64_t cb = q / chunk, qi = q - cb * chunk;
    int64_t cs = (a.nq - cb * chunk) < chunk ? (a.nq - cb * chunk) : chunk;
    int64_t rec = 2 * cb * chunk + side * cs + qi;
    ranks[rec] = rank;
    ncand[rec] = a.N - 1 - nknown;
  }
}

// --- given-candidates protocol (ref:evaluate.py:168-180) ----------------------
// One warp per query: q = H[h] * dec[r] held in the lanes (feature f = lane +
// 32 j), every score — the true candidate's included — is the same per-lane
// fmaf chain plus the same xor-tree warp sum, so the comparisons are exact.
constexpr int CQ_J = 8;   // d <= 256

__device__ __forceinline__ float cand_dot(const float (&q)[CQ_J], const float* __restrict__ Hc, int d) {
  const int lane = (int)lane_id();
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < CQ_J; ++j) {
    const int f = lane + 32 * j;
    if (f < d) s = fmaf(q[j], __ldg(Hc + f), s);
  }
  return warp_sum(s);
}

__global__ void __launch_bounds__(256) k_rank_candidates(const float* __restrict__ H, int d,
                                                         const float* __restrict__ dec,
                                                         const int32_t* __restrict__ qry, int64_t nq,
                                                         const int64_t* __restrict__ cptr,
                                                         const int32_t* __restrict__ cand,
                                                         const int32_t* __restrict__ tpos, int policy,
                                                         double* __restrict__ ranks, int32_t* __restrict__ ncand) {
  const int lane = (int)lane_id(), nw = (gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); i < nq; i += nw) {
    const int32_t h = qry[i * 3], r = qry[i * 3 + 1];
    float q[CQ_J];
#pragma unroll
    for (int j = 0; j < CQ_J; ++j) {
      const int f = lane + 32 * j;
      q[j] = f < d ? H[(int64_t)h * d + f] * dec[(int64_t)r * d + f] : 0.f;
    }
    const int64_t lo = cptr[i], hi = cptr[i + 1];
    const float ts = cand_dot(q, H + (int64_t)cand[lo + tpos[i]] * d, d);
    long long g = 0, e = 0;
    for (int64_t c = lo; c < hi; ++c) {
      const float sc = cand_dot(q, H + (int64_t)cand[c] * d, d);
      g += sc > ts;
      e += sc == ts;
    }
    e -= 1;   // the true candidate itself
    if (lane == 0) {
      double rank;
      if (policy == 0) rank = 1.0 + (double)g + (double)e / 2.0;
      else if (policy == 1) rank = 1.0 + (double)g;
      else rank = 1.0 + (double)g + (double)e;
      ranks[i] = rank;
      ncand[i] = (int32_t)(hi - lo - 1);
    }
  }
}

// --- known keys --------------------------------------------------------------
__global__ void k_known_keys(const int32_t* __restrict__ tri, int64_t k, int ca, int cc, int32_t N, int32_t R,
                             uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = ((uint64_t)tri[i * 3 + ca] * (uint64_t)R + (uint64_t)tri[i * 3 + 1]) * (uint64_t)N + (uint64_t)tri[i * 3 + cc];
    vals[i] = (uint32_t)i;
  }
}

__global__ void k_key_bounds(const uint64_t* __restrict__ keys, int64_t n, uint32_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

__global__ void k_key_gather(const uint64_t* __restrict__ keys, const int32_t* __restrict__ idx,
                             const int32_t* __restrict__ cnt, int64_t* __restrict__ out) {
  int32_t c = *cnt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)keys[idx[i]];
}

static int bits_for(uint64_t maxval) {
  int b = 0;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

}  // namespace kg

using namespace kg;

extern "C" {

int64_t kg_known_keys_workspace_bytes(int64_t k) {
  return (int64_t)(align_up(k * 8) + align_up(k * 4) * 3 + sort_workspace(k) + compact_workspace(k) + 4096);
}

kg_status kg_known_keys(const int32_t* tri, int64_t k, int32_t ca, int32_t cc, int32_t N, int32_t R,
                        int64_t* keys_out, int32_t* n_out, void* ws, int64_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(ws_bytes >= kg_known_keys_workspace_bytes(k), KG_ERR_VALIDATION, "keys workspace too small");
  if (k == 0) {
    KG_CUDA(cudaMemsetAsync(n_out, 0, 4, st));
    return KG_OK;
  }
  Arena a(ws, (size_t)ws_bytes);
  uint64_t* keys = a.take<uint64_t>(k);
  uint32_t* vals = a.take<uint32_t>(k);
  uint32_t* flags = a.take<uint32_t>(k);
  int32_t* idx = a.take<int32_t>(k);
  char* sws = a.take<char>(sort_workspace(k));
  char* cws = a.take<char>(compact_workspace(k));
  int g = persistent_blocks(k, 256, 8);
  KG_LAUNCH("k_known_keys", k_known_keys, g, 256, 0, st, tri, k, ca, cc, N, R, keys, vals);
  uint64_t maxkey = ((uint64_t)(N - 1) * R + (R - 1)) * (uint64_t)N + (N - 1);
  kg_status s = sort_pairs_u64(keys, vals, k, bits_for(maxkey), sws, sort_workspace(k), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_key_bounds", k_key_bounds, g, 256, 0, st, keys, k, flags);
  s = compact_flags(flags, k, idx, n_out, 0, nullptr, cws, compact_workspace(k), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_key_gather", k_key_gather, g, 256, 0, st, keys, idx, n_out, keys_out);
  KG_CHECK_LAUNCH("known keys");
  return KG_OK;
}

int64_t kg_eval_workspace_bytes(int64_t nq, int32_t N, int32_t d, int64_t known_pairs) {
  const size_t simt = align_up(2 * nq * 4) + align_up(2 * nq * 8) * 2 + 1024;
  const size_t tc = d <= 128 ? umma_rank_workspace(nq, N, d, known_pairs) + 1024 : 0;
  return (int64_t)(simt > tc ? simt : tc);
}

kg_status kg_eval_filtered(const float* H, int32_t d, int32_t N, const float* dec, int32_t R, const int32_t* qry,
                           int64_t nq, const int64_t* tkeys, int64_t ntk, const int64_t* hkeys, int64_t nhk,
                           int32_t policy, int32_t chunk, int32_t impl, int64_t known_pairs, double* ranks,
                           int32_t* ncand, uint32_t* overflow, const double* H64, const double* dec64, void* ws,
                           int64_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(policy >= 0 && policy <= 2, KG_ERR_VALIDATION, "unknown tie policy");
  KG_REQUIRE(chunk >= 1 && nq >= 1, KG_ERR_VALIDATION, "bad chunk / empty split");
  KG_REQUIRE(ws_bytes >= kg_eval_workspace_bytes(nq, N, d, known_pairs), KG_ERR_VALIDATION,
             "eval workspace too small");
  if (impl == 0 && d <= 128)
    return umma_rank_filtered(H, d, N, dec, R, qry, nq, tkeys, ntk, hkeys, nhk, policy, chunk, known_pairs, ranks,
                              ncand, overflow, ws, (size_t)ws_bytes, st, H64, dec64);
  if (overflow) KG_CUDA(cudaMemsetAsync(overflow, 0, 4, st));
  Arena a(ws, (size_t)ws_bytes);
  float* ts = a.take<float>(2 * nq);
  unsigned long long* gr = a.take<unsigned long long>(2 * nq);
  unsigned long long* eq = a.take<unsigned long long>(2 * nq);
  EvalArgs e{H, d, N, R, dec, qry, nq, ts, gr, eq};
  KG_LAUNCH("k_true_scores", k_true_scores, persistent_blocks(2 * nq, 256, 8), 256, 0, st, e, ts);
  KG_LAUNCH("k_rank_tiles", k_rank_tiles, (unsigned)ceil_div(2 * nq, QB), ET, 0, st, e);
  KG_CHECK_LAUNCH("k_rank_tiles");
  KG_LAUNCH("k_rank_finish", k_rank_finish, persistent_blocks(2 * nq, 128, 8), 128, 0, st, e, tkeys, ntk, hkeys, nhk, policy, chunk, ranks,
                                                                   ncand);
  KG_CHECK_LAUNCH("k_rank_finish");
  return KG_OK;
}

kg_status kg_eval_candidates(const float* H, int32_t d, const float* dec, const int32_t* qry, int64_t nq,
                             const int64_t* cand_ptr, const int32_t* cand, const int32_t* true_pos, int32_t policy,
                             double* ranks, int32_t* ncand, void* stream) {
  KG_REQUIRE(policy >= 0 && policy <= 2, KG_ERR_VALIDATION, "unknown tie policy");
  KG_REQUIRE(d >= 1 && d <= 32 * CQ_J, KG_ERR_SHAPE, "candidates protocol supports d <= %d", 32 * CQ_J);
  if (nq <= 0) return KG_OK;
  KG_LAUNCH("k_rank_candidates", k_rank_candidates, persistent_blocks(nq * 32, 256, 8), 256, 0, as_stream(stream), H,
            d, dec, qry, nq, cand_ptr, cand, true_pos, policy, ranks, ncand);
  return KG_OK;
}

}  // extern "C"

// this module's anchor for kg_preload_kernels (kg_primitives.cu)
extern "C" const void* kg_anchor_eval() { return reinterpret_cast<const void*>(&kg::k_true_scores); }
