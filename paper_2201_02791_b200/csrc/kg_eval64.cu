// R24 full-graph encode for evaluation in float64 (ref:evaluate.py:107-122,
// model.py:151-164, 196-235).
//
// `encode_all_entities` feeds the filtered ranking, where the reference's
// float64 scores decide ranks among 14,541 candidates: an fp32 forward leaves
// H within ~3e-6 (rel-L2) of the reference, enough to reorder near-tied
// candidates in ~0.7 % of the records. The evaluation encode therefore runs
// in float64 (one full-graph forward, not the training hot path): per layer
//   acc_b[v] = sum_{e into v} (1/c_e) a[r_e, b] H[src_e] + a[2R, b] H[v]
//   Z = [acc_0 | .. | acc_{B-1}] . [V_0; ..; V_{B-1}],  H' = ReLU(Z) (not last)
// with 1/c_e recomputed exactly from the per-(dst, relation) counts. The
// reference transforms before it aggregates; the sums agree to ~1e-15.
#include "kg_common.cuh"

namespace kg {

// Hub rows (8.4k messages at FB shape) use the view's static chunk table
// (kg_chunks.cu): one warp per <= C-message chunk of a row; rows with one
// chunk write acc directly, split rows write per-chunk partials that a second
// pass adds in chunk order. Within a chunk, lanes load 32 messages' metadata
// at once (the per-message weight 1/c * a[r, b] is formed by its own lane)
// and broadcast it, then lanes sweep the columns.
constexpr int A64_MAXB = 8;

__device__ __forceinline__ void a64_chunk_sums(int32_t lo, int32_t hi, const int32_t* __restrict__ src,
                                               const int32_t* __restrict__ rel, const int32_t* __restrict__ cnt,
                                               const double* __restrict__ coeffs, int B,
                                               const double* __restrict__ H, int d, int c,
                                               double (&s)[A64_MAXB]) {
  const int lane = (int)lane_id();
#pragma unroll
  for (int b = 0; b < A64_MAXB; ++b) s[b] = 0.0;
  for (int32_t e0 = lo; e0 < hi; e0 += 32) {
    const int32_t e = e0 + lane;
    int32_t my_src = 0;
    double my_w[A64_MAXB];
#pragma unroll
    for (int b = 0; b < A64_MAXB; ++b) my_w[b] = 0.0;
    if (e < hi) {
      my_src = src[e];
      const double inv = 1.0 / (double)cnt[e];
      const double* a = coeffs + (int64_t)rel[e] * B;
#pragma unroll
      for (int b = 0; b < A64_MAXB; ++b)
        if (b < B) my_w[b] = inv * a[b];
    }
    const int m = hi - e0 < 32 ? hi - e0 : 32;
#pragma unroll 4
    for (int j = 0; j < m; ++j) {
      const int32_t u = __shfl_sync(0xffffffffu, my_src, j);
      const double x = c < d ? H[(int64_t)u * d + c] : 0.0;
#pragma unroll
      for (int b = 0; b < A64_MAXB; ++b) {
        const double w = __shfl_sync(0xffffffffu, my_w[b], j);
        if (b < B) s[b] = fma(w, x, s[b]);
      }
    }
  }
}

__global__ void __launch_bounds__(256) k64_aggregate(const int32_t* __restrict__ indptr,
                                                     const int32_t* __restrict__ src, const int32_t* __restrict__ rel,
                                                     const int32_t* __restrict__ cnt, int self_rel,
                                                     const double* __restrict__ coeffs, int B,
                                                     const double* __restrict__ H, int d, int C,
                                                     const int32_t* __restrict__ ck_ptr,
                                                     const int32_t* __restrict__ ck_row,
                                                     const int32_t* __restrict__ ck_slot,
                                                     const int32_t* __restrict__ ck_counts,
                                                     double* __restrict__ acc, double* __restrict__ part) {
  const int lane = (int)lane_id(), nw = (gridDim.x * blockDim.x) >> 5;
  const int64_t nchunks = ck_counts[0];
  for (int64_t k = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); k < nchunks; k += nw) {
    const int32_t v = ck_row[k], j = (int32_t)(k - ck_ptr[v]), slot = ck_slot[k];
    const int32_t lo = indptr[v] + j * C, end = indptr[v + 1], hi = lo + C < end ? lo + C : end;
    const double* as = coeffs + (int64_t)self_rel * B;
    for (int c0 = 0; c0 < d; c0 += 32) {
      const int c = c0 + lane;
      double s[A64_MAXB];
      a64_chunk_sums(lo, hi, src, rel, cnt, coeffs, B, H, d, c, s);
      if (c >= d) continue;
      if (slot < 0) {
        const double x = H[(int64_t)v * d + c];
#pragma unroll
        for (int b = 0; b < A64_MAXB; ++b)
          if (b < B) acc[((int64_t)v * B + b) * d + c] = fma(as[b], x, s[b]);
      } else {
#pragma unroll
        for (int b = 0; b < A64_MAXB; ++b)
          if (b < B) part[((int64_t)slot * B + b) * d + c] = s[b];
      }
    }
  }
}

// split rows: partials added in chunk order, then the self-loop
__global__ void __launch_bounds__(256) k64_combine(const int32_t* __restrict__ ck_ptr,
                                                   const int32_t* __restrict__ ck_slot,
                                                   const int32_t* __restrict__ ck_split,
                                                   const int32_t* __restrict__ ck_counts, int self_rel,
                                                   const double* __restrict__ coeffs, int B,
                                                   const double* __restrict__ H, int d,
                                                   const double* __restrict__ part, double* __restrict__ acc) {
  const int64_t nrows = ck_counts[2];
  const int64_t items = nrows * B * d;
  const double* as = coeffs + (int64_t)self_rel * B;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < items; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ((int64_t)B * d), bc = i - r * B * d;
    const int b = (int)(bc / d), c = (int)(bc - (int64_t)b * d);
    const int32_t v = ck_split[r];
    double s = 0.0;
    for (int32_t k = ck_ptr[v]; k < ck_ptr[v + 1]; ++k) s += part[((int64_t)ck_slot[k] * B + b) * d + c];
    acc[((int64_t)v * B + b) * d + c] = fma(as[b], H[(int64_t)v * d + c], s);
  }
}

// C[M,N] = A[M,K] . W[K,N] (row-major, float64), optional ReLU; 64x64 tiles,
// 256 threads with 4x4 outputs each, K staged 16 at a time in shared memory.
constexpr int G64_T = 64, G64_K = 16;
__global__ void __launch_bounds__(256) k64_gemm(const double* __restrict__ A, const double* __restrict__ W,
                                                double* __restrict__ C, int64_t M, int K, int N, int relu) {
  __shared__ double As[G64_K][G64_T + 1];
  __shared__ double Ws[G64_K][G64_T + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * G64_T;
  const int n0 = blockIdx.x * G64_T;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += G64_K) {
    for (int i = threadIdx.x; i < G64_K * G64_T; i += 256) {
      const int kk = i % G64_K, mm = i / G64_K;          // A tile: row mm, col kk
      const int64_t gm = m0 + mm;
      As[kk][mm] = (gm < M && k0 + kk < K) ? A[gm * K + k0 + kk] : 0.0;
      const int nn = i % G64_T, kw = i / G64_T;          // W tile: row kw, col nn
      Ws[kw][nn] = (k0 + kw < K && n0 + nn < N) ? W[(int64_t)(k0 + kw) * N + n0 + nn] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < G64_K; ++kk) {
      double a[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = Ws[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], w[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn < N) C[gm * N + gn] = relu ? fmax(acc[i][j], 0.0) : acc[i][j];
    }
  }
}

}  // namespace kg

using namespace kg;

extern "C" {

int64_t kg_encode_full_f64_workspace_bytes(int32_t n, int64_t e, int32_t C, int32_t B, int32_t d_max) {
  const int64_t split_chunks = 2 * e / (C > 0 ? C : 1) + 1;
  return (int64_t)(align_up((size_t)n * B * d_max * 8) + 2 * align_up((size_t)n * d_max * 8) +
                   align_up((size_t)split_chunks * B * d_max * 8) + 1024);
}

kg_status kg_encode_full_f64(const kg_graph_csr* g, const int32_t* src, const int32_t* rel, const int32_t* cnt,
                             int32_t L, const int32_t* dims, int32_t B, const double* const* bases,
                             const double* const* coeffs, const double* input, double* out, void* ws,
                             int64_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(L >= 1 && B >= 1 && B <= A64_MAXB, KG_ERR_VALIDATION, "encode_f64: 1 <= B <= 8 and L >= 1");
  const int32_t n = g->n;
  int d_max = 0;
  for (int l = 0; l <= L; ++l) d_max = dims[l] > d_max ? dims[l] : d_max;
  KG_REQUIRE(ws_bytes >= kg_encode_full_f64_workspace_bytes(n, g->e, g->chunk, B, d_max), KG_ERR_VALIDATION,
             "encode_f64 workspace too small");
  if (n == 0) return KG_OK;
  Arena a(ws, (size_t)ws_bytes);
  double* acc = a.take<double>((size_t)n * B * d_max);
  double* buf[2] = {a.take<double>((size_t)n * d_max), a.take<double>((size_t)n * d_max)};
  double* part = a.take<double>((size_t)(2 * g->e / g->chunk + 1) * B * d_max);
  const int64_t cap_chunks = n + g->e / g->chunk + 1;
  const double* h = input;
  for (int l = 0; l < L; ++l) {
    const int din = dims[l], dout = dims[l + 1];
    KG_LAUNCH("k64_aggregate", k64_aggregate, persistent_blocks(cap_chunks * 32, 256, 8), 256, 0, st, g->indptr, src,
              rel, cnt, 2 * g->R, coeffs[l], B, h, din, g->chunk, g->ck_ptr, g->ck_row, g->ck_slot, g->ck_counts,
              acc, part);
    KG_LAUNCH("k64_combine", k64_combine, persistent_blocks((g->e / g->chunk + 1) * B * din, 256, 8), 256, 0, st,
              g->ck_ptr, g->ck_slot, g->ck_split, g->ck_counts, 2 * g->R, coeffs[l], B, h, din, part, acc);
    double* dst = l == L - 1 ? out : buf[l & 1];
    const dim3 grid((unsigned)ceil_div(dout, G64_T), (unsigned)ceil_div(n, G64_T));
    // bases[l] is (B, din, dout) row-major = the stacked [V_0; ..; V_{B-1}] (B*din, dout)
    KG_LAUNCH("k64_gemm", k64_gemm, grid, 256, 0, st, acc, bases[l], dst, (int64_t)n, B * din, dout,
              l < L - 1 ? 1 : 0);
    h = dst;
  }
  return KG_OK;
}

}  // extern "C"

// this module's anchor for kg_preload_kernels (kg_primitives.cu)
extern "C" const void* kg_anchor_eval64() { return reinterpret_cast<const void*>(&kg::k64_aggregate); }
