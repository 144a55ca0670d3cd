// Float64 device path of the public numpy API `encode` / `loss_from_cache` /
// `loss_and_grad` (ref:model.py:151-301): the reference's own precision, so
// gradient checks by central differences and 1e-12 comparisons hold. The
// training loop keeps the fp32 tensor-core kernels (kg_rgcn.cu, kg_loss.cu).
//
// Layer l over the closure (targets p < T at position p, local id order[p];
// rows of H by local id):
//   acc_b[p] = sum_{e into order[p]} (1/c_e) a[r_e, b] H_in[src_e] + a[2R, b] H_in[order[p]]
//   Z[p]     = [acc_0 | .. | acc_{B-1}][p] . [V_0; ..; V_{B-1}]
//   H_out[order[p]] = ReLU(Z[p]) (not last) * dropout mask
// Backward (dZ[p] = dH_out[order[p]] * mask * [Z > 0]):
//   d V_b    = acc_b^T dZ
//   d a[g,b] = sum_{e in g} (1/c_e) <H_in[src_e] V_b, dZ[dst_e]>  (+ self loops)
//   dH_in[u] = sum_b dS_b[u] V_b^T,  dS_b[u] = sum_{e: src_e = u} (1/c_e) a[r_e, b] dZ[dst_e] (+ self)
// The forward aggregate and the loss are deterministic (fixed summation order:
// one warp per destination row over its messages in order; one warp over the
// batch in order), so a loss evaluated twice is bitwise the same — central
// differences of it (ref tests: step 1e-5, tolerance 1e-5) see no atomic-order
// noise. Gradient sums over messages use float64 atomics (order noise ~1e-16
// relative).
#include "kg_common.cuh"

namespace kg {

constexpr int M64_MAXB = 8;

// closure aggregate: one warp per target row (its first chunk's warp) over
// all of the row's messages in order — deterministic, no atomics
__global__ void __launch_bounds__(256) k64c_aggregate(const int32_t* __restrict__ src, const int32_t* __restrict__ rel,
                                                      const int32_t* __restrict__ cnt, const int4* __restrict__ desc,
                                                      const int32_t* __restrict__ ck_counts,
                                                      const int32_t* __restrict__ indptr,
                                                      const int32_t* __restrict__ pos, int32_t T, int self_rel,
                                                      const double* __restrict__ coeffs, int B,
                                                      const double* __restrict__ H, int d, double* __restrict__ acc) {
  const int lane = (int)lane_id(), nw = (gridDim.x * blockDim.x) >> 5;
  const int64_t nchunks = ck_counts[0];
  for (int64_t k = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); k < nchunks; k += nw) {
    const int4 dsc = desc[k];
    if (!(dsc.z & (1 << 17))) continue;   // the row's first chunk takes the whole row
    const int32_t v = dsc.x, lo = indptr[v], hi = indptr[v + 1];
    const int32_t p = pos[v];
    if (p < 0 || p >= T) continue;
    const bool first = true;
    for (int c = lane; c < d; c += 32) {
      double s[M64_MAXB];
#pragma unroll
      for (int b = 0; b < M64_MAXB; ++b) s[b] = 0.0;
      for (int32_t e = lo; e < hi; ++e) {
        const double w = 1.0 / (double)cnt[e];
        const double x = H[(int64_t)src[e] * d + c];
        const double* a = coeffs + (int64_t)rel[e] * B;
#pragma unroll
        for (int b = 0; b < M64_MAXB; ++b)
          if (b < B) s[b] = fma(w * a[b], x, s[b]);
      }
      if (first) {   // the row's self loop, once
        const double x = H[(int64_t)v * d + c];
        const double* a = coeffs + (int64_t)self_rel * B;
#pragma unroll
        for (int b = 0; b < M64_MAXB; ++b)
          if (b < B) s[b] = fma(a[b], x, s[b]);
      }
#pragma unroll
      for (int b = 0; b < M64_MAXB; ++b)
        if (b < B) acc[((int64_t)p * B + b) * d + c] = s[b];
    }
  }
}

// C[M,N] (+)= op(A) . W, row-major float64: A is (M,K) (ta = 0) or its
// transpose stored (K,M) (ta = 1); 64x64 tiles, 4x4 per thread.
constexpr int T64 = 64, K64 = 16;
__global__ void __launch_bounds__(256) k64c_gemm(const double* __restrict__ A, const double* __restrict__ W,
                                                 double* __restrict__ C, int64_t M, int K, int N, int ta,
                                                 int64_t lda, int64_t ldw, int64_t ldc) {
  __shared__ double As[K64][T64 + 1];
  __shared__ double Ws[K64][T64 + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * T64;
  const int n0 = blockIdx.x * T64;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += K64) {
    for (int i = threadIdx.x; i < K64 * T64; i += 256) {
      const int kk = i % K64, mm = i / K64;
      const int64_t gm = m0 + mm;
      double av = 0.0;
      if (gm < M && k0 + kk < K) av = ta ? A[(int64_t)(k0 + kk) * lda + gm] : A[gm * lda + k0 + kk];
      As[kk][mm] = av;
      const int nn = i % T64, kw = i / T64;
      Ws[kw][nn] = (k0 + kw < K && n0 + nn < N) ? W[(int64_t)(k0 + kw) * ldw + n0 + nn] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < K64; ++kk) {
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
      if (gn < N) C[gm * ldc + gn] = acc[i][j];
    }
  }
}

// H_out[order[p]] = act(Z[p]) * mask[p]; Z keeps the pre-activation
__global__ void k64c_activate(const double* __restrict__ Z, const int32_t* __restrict__ order, int32_t T, int d,
                              int relu, const float* __restrict__ mask, double mask_scale, double* __restrict__ H) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)T * d;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / d, c = i - p * d;
    double z = Z[i];
    if (relu) z = z > 0.0 ? z : 0.0;
    if (mask) z = mask[i] != 0.f ? z * mask_scale : 0.0;
    H[(int64_t)order[p] * d + c] = z;
  }
}

// dZ[p] = dH[order[p]] * mask * [Z > 0] (relu layers)
__global__ void k64c_dz(const double* __restrict__ dH, const double* __restrict__ Z, const int32_t* __restrict__ order,
                        int32_t T, int d, int relu, const float* __restrict__ mask, double mask_scale,
                        double* __restrict__ dZ) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)T * d;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / d, c = i - p * d;
    double g = dH[(int64_t)order[p] * d + c];
    if (mask) g = mask[i] != 0.f ? g * mask_scale : 0.0;
    if (relu && !(Z[i] > 0.0)) g = 0.0;
    dZ[i] = g;
  }
}

// per message into a target: the edge dots (d a) and the source scatter (dS);
// warp per chunk, one message at a time, lanes over columns
__global__ void __launch_bounds__(256) k64c_backward_msgs(
    const int32_t* __restrict__ src, const int32_t* __restrict__ rel, const int32_t* __restrict__ cnt,
    const int4* __restrict__ desc, const int32_t* __restrict__ ck_counts, const int32_t* __restrict__ pos, int32_t T,
    int self_rel, const double* __restrict__ coeffs, int B, const double* __restrict__ Y, int64_t n, int dout,
    const double* __restrict__ dZ, double* __restrict__ d_coeffs, double* __restrict__ dS) {
  const int lane = (int)lane_id(), nw = (gridDim.x * blockDim.x) >> 5;
  const int64_t nchunks = ck_counts[0];
  for (int64_t k = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); k < nchunks; k += nw) {
    const int4 dsc = desc[k];
    const int32_t v = dsc.x, lo = dsc.y, hi = dsc.y + (dsc.z & 0xffff);
    const int32_t p = pos[v];
    if (p < 0 || p >= T) continue;
    const bool first = dsc.z & (1 << 17);
    const double* dz = dZ + (int64_t)p * dout;
    for (int32_t e = lo - (first ? 1 : 0); e < hi; ++e) {
      const bool self = e < lo;                  // the row's self loop (first chunk only)
      const int32_t u = self ? v : src[e], r = self ? self_rel : rel[e];
      const double w = self ? 1.0 : 1.0 / (double)cnt[e];
      for (int b = 0; b < B; ++b) {
        const double* y = Y + ((int64_t)b * n + u) * dout;
        double dp = 0.0;
        for (int c = lane; c < dout; c += 32) dp = fma(y[c], dz[c], dp);
        dp = warp_sum_d(dp);
        if (lane == 0) atomicAdd(d_coeffs + (int64_t)r * B + b, w * dp);
        const double wa = w * coeffs[(int64_t)r * B + b];
        for (int c = lane; c < dout; c += 32) atomicAdd(dS + ((int64_t)u * B + b) * dout + c, wa * dz[c]);
      }
    }
  }
}

// Wt[(b*dout + j), k] = V_b[k, j]: the stacked transposed bases for dH_in = dS . Wt
__global__ void k64c_transpose_bases(const double* __restrict__ V, int B, int din, int dout, double* __restrict__ Wt) {
  const int64_t total = (int64_t)B * din * dout;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / ((int64_t)din * dout), r = i - b * din * dout, k = r / dout, j = r - k * dout;
    Wt[(b * dout + j) * din + k] = V[i];
  }
}

// DistMult + BCE over the batch (ref:model.py:254-281): loss = mean(softplus(g) - y g),
// dg = (sigmoid(g) - y) / b; d decoder and dH at the seed rows. One warp walks
// the batch in order (lanes over d): the loss and both gradients are summed in
// a fixed order (the public float64 API path; not the training kernels).
__global__ void __launch_bounds__(32) k64c_loss(const int32_t* __restrict__ tri, const double* __restrict__ y, int64_t b,
                          const double* __restrict__ H, const double* __restrict__ dec, int d, double* __restrict__ loss,
                          double* __restrict__ d_dec, double* __restrict__ dH, uint32_t* __restrict__ flags) {
  const int lane = (int)lane_id();
  double total = 0.0;
  for (int64_t i = 0; i < b; ++i) {
    const int32_t h = tri[i * 3], r = tri[i * 3 + 1], t = tri[i * 3 + 2];
    const double* hs = H + (int64_t)h * d;
    const double* ht = H + (int64_t)t * d;
    const double* m = dec + (int64_t)r * d;
    double g = 0.0;
    for (int c = lane; c < d; c += 32) g = fma(hs[c] * m[c], ht[c], g);
    g = warp_sum_d(g);
    if (!isfinite(g)) {
      if (lane == 0) atomicOr(flags, KG_FLAG_NONFINITE_SCORE);
      continue;
    }
    const double yi = y[i];
    // logaddexp(0, g) as numpy evaluates it; sigmoid as scipy's expit
    const double sp = g > 0.0 ? g + log1p(exp(-g)) : (g < 0.0 ? log1p(exp(g)) : 0.6931471805599453);
    const double sg = g >= 0.0 ? 1.0 / (1.0 + exp(-g)) : exp(g) / (1.0 + exp(g));
    const double dg = (sg - yi) / (double)b;
    total += (sp - yi * g) / (double)b;
    for (int c = lane; c < d; c += 32) {
      const double xh = hs[c], xt = ht[c], mc = m[c];
      d_dec[(int64_t)r * d + c] += dg * xh * xt;
      dH[(int64_t)h * d + c] += dg * (mc * xt);
      dH[(int64_t)t * d + c] += dg * (mc * xh);
    }
    __syncwarp();
  }
  if (lane == 0) *loss += total;
}

static dim3 gemm_grid(int64_t M, int N) {
  return dim3((unsigned)ceil_div(N, T64), (unsigned)ceil_div(M > 0 ? M : 1, T64));
}

}  // namespace kg

using namespace kg;

extern "C" {

int64_t kg_layer64_workspace_bytes(int64_t n, int32_t din, int32_t dout, int32_t B) {
  return (int64_t)(align_up((size_t)B * n * dout * 8) + align_up((size_t)n * B * dout * 8) +
                   align_up((size_t)B * din * dout * 8) + 1024);
}

kg_status kg_forward_layer_f64(const kg_graph_csr* g, const int32_t* src, const int32_t* rel, const int32_t* cnt,
                               const int32_t* order, const int32_t* pos, int32_t T, int32_t din, int32_t dout,
                               int32_t B, const double* bases, const double* coeffs, const double* H_in, double* acc,
                               double* Z, double* H_out, int32_t relu, const float* mask, double mask_scale,
                               void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(B >= 1 && B <= M64_MAXB, KG_ERR_VALIDATION, "float64 path: 1 <= B <= %d", M64_MAXB);
  if (T <= 0) return KG_OK;
  const int64_t cap_chunks = g->n + g->e / g->chunk + 1;
  KG_CUDA(cudaMemsetAsync(acc, 0, (size_t)T * B * din * 8, st));
  KG_LAUNCH("k64c_aggregate", k64c_aggregate, persistent_blocks(cap_chunks * 32, 256, 8), 256, 0, st, src, rel, cnt,
            reinterpret_cast<const int4*>(g->ck_desc), g->ck_counts, g->indptr, pos, T, 2 * g->R, coeffs, B, H_in, din,
            acc);
  KG_LAUNCH("k64c_gemm", k64c_gemm, gemm_grid(T, dout), 256, 0, st, acc, bases, Z, (int64_t)T, B * din, dout, 0,
            (int64_t)B * din, (int64_t)dout, (int64_t)dout);
  KG_LAUNCH("k64c_activate", k64c_activate, persistent_blocks((int64_t)T * dout, 256, 8), 256, 0, st, Z, order, T,
            dout, relu, mask, mask_scale, H_out);
  return KG_OK;
}

kg_status kg_loss_f64(const int32_t* triples, const double* labels, int64_t b, const double* H, const double* decoder,
                      int32_t d, double* loss, double* d_decoder, double* dH, uint32_t* flags, void* stream) {
  if (b <= 0) return KG_OK;
  KG_LAUNCH("k64c_loss", k64c_loss, 1, 32, 0, as_stream(stream), triples, labels, b, H, decoder, d, loss, d_decoder,
            dH, flags);
  return KG_OK;
}

kg_status kg_backward_layer_f64(const kg_graph_csr* g, const int32_t* src, const int32_t* rel, const int32_t* cnt,
                                const int32_t* order, const int32_t* pos, int32_t T, int32_t din, int32_t dout,
                                int32_t B, const double* bases, const double* coeffs, const double* H_in,
                                const double* acc, const double* Z, const double* dH_out, int32_t relu,
                                const float* mask, double mask_scale, double* dZ, double* d_bases, double* d_coeffs,
                                double* dH_in, void* ws, int64_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(B >= 1 && B <= M64_MAXB, KG_ERR_VALIDATION, "float64 path: 1 <= B <= %d", M64_MAXB);
  const int64_t n = g->n;
  KG_REQUIRE(ws_bytes >= kg_layer64_workspace_bytes(n, din, dout, B), KG_ERR_VALIDATION, "workspace too small");
  Arena a(ws, (size_t)ws_bytes);
  double* Y = a.take<double>((size_t)B * n * dout);
  double* dS = a.take<double>((size_t)n * B * dout);
  double* Wt = a.take<double>((size_t)B * din * dout);
  const int G = 2 * g->R + 1;
  KG_CUDA(cudaMemsetAsync(d_coeffs, 0, (size_t)G * B * 8, st));
  if (T <= 0) {
    KG_CUDA(cudaMemsetAsync(d_bases, 0, (size_t)B * din * dout * 8, st));
    return KG_OK;
  }
  KG_LAUNCH("k64c_dz", k64c_dz, persistent_blocks((int64_t)T * dout, 256, 8), 256, 0, st, dH_out, Z, order, T, dout,
            relu, mask, mask_scale, dZ);
  // d V = acc^T dZ  ((B*din) x dout, reduction over the T targets)
  KG_LAUNCH("k64c_gemm", k64c_gemm, gemm_grid((int64_t)B * din, dout), 256, 0, st, acc, dZ, d_bases,
            (int64_t)B * din, T, dout, 1, (int64_t)B * din, (int64_t)dout, (int64_t)dout);
  // Y_b = H_in . V_b over all local rows (rows outside the closure are unused)
  for (int b = 0; b < B; ++b)
    KG_LAUNCH("k64c_gemm", k64c_gemm, gemm_grid(n, dout), 256, 0, st, H_in, bases + (int64_t)b * din * dout,
              Y + (int64_t)b * n * dout, n, din, dout, 0, (int64_t)din, (int64_t)dout, (int64_t)dout);
  KG_CUDA(cudaMemsetAsync(dS, 0, (size_t)n * B * dout * 8, st));
  const int64_t cap_chunks = g->n + g->e / g->chunk + 1;
  KG_LAUNCH("k64c_backward_msgs", k64c_backward_msgs, persistent_blocks(cap_chunks * 32, 256, 8), 256, 0, st, src, rel,
            cnt, reinterpret_cast<const int4*>(g->ck_desc), g->ck_counts, pos, T, 2 * g->R, coeffs, B, Y, n, dout, dZ,
            d_coeffs, dS);
  if (dH_in) {
    KG_LAUNCH("k64c_transpose_bases", k64c_transpose_bases, persistent_blocks((int64_t)B * din * dout, 256, 4), 256, 0,
              st, bases, B, din, dout, Wt);
    KG_LAUNCH("k64c_gemm", k64c_gemm, gemm_grid(n, din), 256, 0, st, dS, Wt, dH_in, n, B * dout, din, 0,
              (int64_t)B * dout, (int64_t)din, (int64_t)din);
  }
  return KG_OK;
}

}  // extern "C"

// this module's anchor for kg_preload_kernels (kg_primitives.cu)
extern "C" const void* kg_anchor_model64() { return reinterpret_cast<const void*>(&kg::k64c_aggregate); }
