// R13/R14: RGCN layer forward and backward in basis-factored form.
//
// The reference materialises W_g = sum_b a_gb V_b for all 2R+1 groups and runs
// one dgemm per group (ref:model.py:131-185). Here nothing per-relation is
// ever formed:
//   forward   acc_b[v] = sum_{e->v} norm_e a[r_e,b] X[src_e] + a[2R,b] X[v]
//             Z[v]     = sum_b acc_b[v] V_b                 (one GEMM, K = B*d_in)
//   backward  dS_b[u]  = sum_{e: src=u} norm_e a[r_e,b] dZ[dst_e] + a[2R,b] dZ[u]
//             dX       = sum_b dS_b V_b^T                   (GEMM)
//             dV_b     = X^T dS_b                            (split-K GEMM)
//             d a[r,b] = sum_{e in r} norm_e <(X V_b)[src_e], dZ[dst_e]>
// The gather/scatter passes are warp-per-row over the relation-sorted CSR
// (forward) and CSC (backward): no atomics, fixed summation order.
// Within a (row, relation) run the destination norm is constant, so the
// forward pass sums the run's source rows first and applies norm*a[r,b] once.
#include "kg_gemm.cuh"

namespace kg {

constexpr int MAXB = 4;

template <int VEC>
struct VecIO;
template <>
struct VecIO<4> {
  __device__ __forceinline__ static void load(const float* p, float* x) {
    float4 v = __ldg(reinterpret_cast<const float4*>(p));
    x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
  }
  __device__ __forceinline__ static void store(float* p, const float* x) {
    *reinterpret_cast<float4*>(p) = make_float4(x[0], x[1], x[2], x[3]);
  }
};
template <>
struct VecIO<1> {
  __device__ __forceinline__ static void load(const float* p, float* x) { x[0] = __ldg(p); }
  __device__ __forceinline__ static void store(float* p, const float* x) { *p = x[0]; }
};

struct AggArgs {
  const int32_t* indptr;
  const int32_t* src;
  const int32_t* rel;
  const float* norm;
  const float* coeffs;   // (G, B)
  int32_t G, B, d;
  const float* H;        // (n, d) by local id
  const int32_t* order;
  const int32_t* counts;
  int t;
  float* acc;            // (count, B*d) compact
};

// Slot s of lane l covers features [(s*32 + l)*VEC, +VEC).
template <int VEC, int S>
__global__ void __launch_bounds__(256) k_aggregate(AggArgs a) {
  extern __shared__ float coef[];
  for (int i = threadIdx.x; i < a.G * a.B; i += blockDim.x) coef[i] = a.coeffs[i];
  __syncthreads();
  const int lane = lane_id();
  const int32_t T = a.counts[a.t];
  const int d = a.d, B = a.B;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  bool slot_ok[S];
#pragma unroll
  for (int s = 0; s < S; ++s) slot_ok[s] = (s * 32 + lane) * VEC < d;
  for (int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; p < T; p += warps) {
    const int32_t v = a.order[p];
    float acc[MAXB][S][VEC];
    float run[S][VEC];
#pragma unroll
    for (int b = 0; b < MAXB; ++b)
#pragma unroll
      for (int s = 0; s < S; ++s)
#pragma unroll
        for (int c = 0; c < VEC; ++c) acc[b][s][c] = 0.f;
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
      for (int c = 0; c < VEC; ++c) run[s][c] = 0.f;
    const int32_t e0 = a.indptr[v], e1 = a.indptr[v + 1];
    for (int32_t base = e0; base < e1; base += 32) {
      const int cnt = min(32, e1 - base);
      int32_t my_src = 0, my_rel = -1;
      float my_norm = 0.f;
      if (lane < cnt) {
        my_src = a.src[base + lane];
        my_rel = a.rel[base + lane];
        my_norm = a.norm[base + lane];
      }
      const int32_t rel_after = (base + 32 < e1) ? a.rel[base + 32] : -1;
      for (int j = 0; j < cnt; j += 4) {
        float xs[4][S][VEC];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          int32_t u = __shfl_sync(0xffffffffu, my_src, (j + q) & 31);
          if (j + q < cnt) {
#pragma unroll
            for (int s = 0; s < S; ++s)
              if (slot_ok[s]) VecIO<VEC>::load(a.H + (int64_t)u * d + (s * 32 + lane) * VEC, xs[q][s]);
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          int32_t r = __shfl_sync(0xffffffffu, my_rel, (j + q) & 31);
          int32_t rn = __shfl_sync(0xffffffffu, my_rel, (j + q + 1) & 31);
          float w = __shfl_sync(0xffffffffu, my_norm, (j + q) & 31);
          if (j + q < cnt) {
            if (j + q + 1 >= cnt) rn = rel_after;
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
              for (int c = 0; c < VEC; ++c) run[s][c] += xs[q][s][c];
            if (rn != r) {
#pragma unroll
              for (int b = 0; b < MAXB; ++b) {
                if (b < B) {
                  float cf = w * coef[r * B + b];
#pragma unroll
                  for (int s = 0; s < S; ++s)
#pragma unroll
                    for (int c = 0; c < VEC; ++c) acc[b][s][c] = fmaf(cf, run[s][c], acc[b][s][c]);
                }
              }
#pragma unroll
              for (int s = 0; s < S; ++s)
#pragma unroll
                for (int c = 0; c < VEC; ++c) run[s][c] = 0.f;
            }
          }
        }
      }
    }
    // self-loop group 2R (norm 1)
    float xv[S][VEC];
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (slot_ok[s]) VecIO<VEC>::load(a.H + (int64_t)v * d + (s * 32 + lane) * VEC, xv[s]);
    float* out = a.acc + p * (int64_t)B * d;
#pragma unroll
    for (int b = 0; b < MAXB; ++b) {
      if (b < B) {
        float cf = coef[(a.G - 1) * B + b];
#pragma unroll
        for (int s = 0; s < S; ++s) {
          if (slot_ok[s]) {
            float o[VEC];
#pragma unroll
            for (int c = 0; c < VEC; ++c) o[c] = fmaf(cf, xv[s][c], acc[b][s][c]);
            VecIO<VEC>::store(out + (int64_t)b * d + (s * 32 + lane) * VEC, o);
          }
        }
      }
    }
  }
}

struct CscArgs {
  const int32_t* c_indptr;
  const int32_t* c_dst;
  const int32_t* c_rel;
  const float* c_norm;
  const float* coeffs;   // (G, B)
  int32_t G, B, d;       // d = d_out
  const float* Y;        // (count_S, B*d) compact: X V_b per source
  const float* dZ;       // (count_T, d) compact
  const int32_t* order;
  const int32_t* pos;
  const int32_t* counts;
  int t;                 // targets A_t, sources A_{t+1}
  float* dS;             // (count_S, B*d)
  float* ed;             // (e, B) per CSC position
  float* ed_self;        // (count_T, B)
};

template <int VEC, int S>
__global__ void __launch_bounds__(256) k_csc_backward(CscArgs a) {
  extern __shared__ float coef[];
  for (int i = threadIdx.x; i < a.G * a.B; i += blockDim.x) coef[i] = a.coeffs[i];
  __syncthreads();
  const int lane = lane_id();
  const int32_t T = a.counts[a.t];
  const int32_t Sn = a.counts[a.t + 1];
  const int d = a.d, B = a.B;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  bool slot_ok[S];
#pragma unroll
  for (int s = 0; s < S; ++s) slot_ok[s] = (s * 32 + lane) * VEC < d;
  for (int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q < Sn; q += warps) {
    const int32_t u = a.order[q];
    float y[MAXB][S][VEC];
    float acc[MAXB][S][VEC];
    float run[S][VEC];
#pragma unroll
    for (int b = 0; b < MAXB; ++b)
#pragma unroll
      for (int s = 0; s < S; ++s)
#pragma unroll
        for (int c = 0; c < VEC; ++c) { acc[b][s][c] = 0.f; y[b][s][c] = 0.f; }
#pragma unroll
    for (int b = 0; b < MAXB; ++b)
      if (b < B)
#pragma unroll
        for (int s = 0; s < S; ++s)
          if (slot_ok[s]) VecIO<VEC>::load(a.Y + (q * B + b) * (int64_t)d + (s * 32 + lane) * VEC, y[b][s]);
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
      for (int c = 0; c < VEC; ++c) run[s][c] = 0.f;
    const int32_t e0 = a.c_indptr[u], e1 = a.c_indptr[u + 1];
    for (int32_t base = e0; base < e1; base += 32) {
      const int cnt = min(32, e1 - base);
      int32_t my_dst = 0, my_rel = -1, my_pw = -1;
      float my_norm = 0.f;
      if (lane < cnt) {
        my_dst = a.c_dst[base + lane];
        my_rel = a.c_rel[base + lane];
        my_norm = a.c_norm[base + lane];
        int32_t pw = a.pos[my_dst];
        my_pw = (pw >= 0 && pw < T) ? pw : -1;
      }
      const int32_t rel_after = (base + 32 < e1) ? a.c_rel[base + 32] : -1;
      float my_dot[MAXB];
#pragma unroll
      for (int b = 0; b < MAXB; ++b) my_dot[b] = 0.f;
      for (int j = 0; j < cnt; ++j) {
        int32_t pw = __shfl_sync(0xffffffffu, my_pw, j);
        int32_t r = __shfl_sync(0xffffffffu, my_rel, j);
        int32_t rn = __shfl_sync(0xffffffffu, my_rel, (j + 1) & 31);
        if (j + 1 >= cnt) rn = rel_after;
        float w = __shfl_sync(0xffffffffu, my_norm, j);
        if (pw >= 0) {
          float z[S][VEC];
#pragma unroll
          for (int s = 0; s < S; ++s) {
            if (slot_ok[s]) VecIO<VEC>::load(a.dZ + (int64_t)pw * d + (s * 32 + lane) * VEC, z[s]);
            else
#pragma unroll
              for (int c = 0; c < VEC; ++c) z[s][c] = 0.f;
          }
#pragma unroll
          for (int s = 0; s < S; ++s)
#pragma unroll
            for (int c = 0; c < VEC; ++c) run[s][c] = fmaf(w, z[s][c], run[s][c]);
#pragma unroll
          for (int b = 0; b < MAXB; ++b) {
            if (b < B) {
              float dp = 0.f;
#pragma unroll
              for (int s = 0; s < S; ++s)
#pragma unroll
                for (int c = 0; c < VEC; ++c) dp = fmaf(y[b][s][c], z[s][c], dp);
              dp = warp_sum(dp);
              if (lane == j) my_dot[b] = w * dp;
            }
          }
        }
        if (rn != r) {
#pragma unroll
          for (int b = 0; b < MAXB; ++b) {
            if (b < B && r >= 0) {
              float cf = coef[r * B + b];
#pragma unroll
              for (int s = 0; s < S; ++s)
#pragma unroll
                for (int c = 0; c < VEC; ++c) acc[b][s][c] = fmaf(cf, run[s][c], acc[b][s][c]);
            }
          }
#pragma unroll
          for (int s = 0; s < S; ++s)
#pragma unroll
            for (int c = 0; c < VEC; ++c) run[s][c] = 0.f;
        }
      }
      if (lane < cnt && my_pw >= 0) {
#pragma unroll
        for (int b = 0; b < MAXB; ++b)
          if (b < B) a.ed[(int64_t)(base + lane) * B + b] = my_dot[b];
      }
    }
    // self-loop (u is a target iff q < T)
    if (q < T) {
      float z[S][VEC];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (slot_ok[s]) VecIO<VEC>::load(a.dZ + q * (int64_t)d + (s * 32 + lane) * VEC, z[s]);
        else
#pragma unroll
          for (int c = 0; c < VEC; ++c) z[s][c] = 0.f;
      }
#pragma unroll
      for (int b = 0; b < MAXB; ++b) {
        if (b < B) {
          float cf = coef[(a.G - 1) * B + b];
          float dp = 0.f;
#pragma unroll
          for (int s = 0; s < S; ++s)
#pragma unroll
            for (int c = 0; c < VEC; ++c) {
              acc[b][s][c] = fmaf(cf, z[s][c], acc[b][s][c]);
              dp = fmaf(y[b][s][c], z[s][c], dp);
            }
          dp = warp_sum(dp);
          if (lane == 0) a.ed_self[q * B + b] = dp;
        }
      }
    }
    float* out = a.dS + q * (int64_t)B * d;
#pragma unroll
    for (int b = 0; b < MAXB; ++b)
      if (b < B)
#pragma unroll
        for (int s = 0; s < S; ++s)
          if (slot_ok[s]) VecIO<VEC>::store(out + (int64_t)b * d + (s * 32 + lane) * VEC, acc[b][s]);
  }
}

// d coeffs: block per relation group (2R message groups + 1 self-loop group)
__global__ void __launch_bounds__(256) k_dcoeff_reduce(const int32_t* __restrict__ rel_ptr,
                                                       const int32_t* __restrict__ rel_perm,
                                                       const int32_t* __restrict__ c_dst,
                                                       const int32_t* __restrict__ pos,
                                                       const int32_t* __restrict__ counts, int t,
                                                       const float* __restrict__ ed, const float* __restrict__ ed_self,
                                                       int32_t G, int32_t B, float* __restrict__ d_coeffs) {
  __shared__ float red[MAXB][256];
  const int g = blockIdx.x;
  const int32_t T = counts[t];
  float s[MAXB] = {0.f, 0.f, 0.f, 0.f};
  if (g < G - 1) {
    for (int32_t j = rel_ptr[g] + threadIdx.x; j < rel_ptr[g + 1]; j += blockDim.x) {
      int32_t cj = rel_perm[j];
      int32_t pw = pos[c_dst[cj]];
      if (pw >= 0 && pw < T) {
#pragma unroll
        for (int b = 0; b < MAXB; ++b)
          if (b < B) s[b] += ed[(int64_t)cj * B + b];
      }
    }
  } else {
    for (int32_t q = threadIdx.x; q < T; q += blockDim.x) {
#pragma unroll
      for (int b = 0; b < MAXB; ++b)
        if (b < B) s[b] += ed_self[(int64_t)q * B + b];
    }
  }
#pragma unroll
  for (int b = 0; b < MAXB; ++b) red[b][threadIdx.x] = s[b];
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
#pragma unroll
      for (int b = 0; b < MAXB; ++b) red[b][threadIdx.x] += red[b][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < B) d_coeffs[g * B + threadIdx.x] = red[threadIdx.x][0];
}

// dZ[p] = dH[v_p] * (H_out[v_p] > 0) (mask skipped when H_out == nullptr)
__global__ void k_dz(const float* __restrict__ dH, const float* __restrict__ Hout, const int32_t* __restrict__ order,
                     const int32_t* __restrict__ counts, int t, int d, float* __restrict__ dZ) {
  const int32_t T = counts[t];
  const int64_t total = (int64_t)T * d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = i / d;
    int k = (int)(i - p * d);
    int64_t src = (int64_t)order[p] * d + k;
    float g = dH[src];
    if (Hout && !(Hout[src] > 0.f)) g = 0.f;
    dZ[i] = g;
  }
}

// Wy[i][b*do+o] = V_b[i][o];  Wb[b*do+o][i] = V_b[i][o]
__global__ void k_weight_views(const float* __restrict__ V, int B, int di, int dO, float* __restrict__ Wy,
                               float* __restrict__ Wb) {
  const int64_t total = (int64_t)B * di * dO;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    int b = (int)(x / ((int64_t)di * dO));
    int rem = (int)(x - (int64_t)b * di * dO);
    int i = rem / dO, o = rem % dO;
    float val = V[x];
    Wy[(int64_t)i * (B * dO) + b * dO + o] = val;
    Wb[(int64_t)(b * dO + o) * di + i] = val;
  }
}

// d_bases[b][i][o] = Rm[i][b*do+o]
__global__ void k_dbases_layout(const float* __restrict__ Rm, int B, int di, int dO, float* __restrict__ dV) {
  const int64_t total = (int64_t)B * di * dO;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    int b = (int)(x / ((int64_t)di * dO));
    int rem = (int)(x - (int64_t)b * di * dO);
    int i = rem / dO, o = rem % dO;
    dV[x] = Rm[(int64_t)i * (B * dO) + b * dO + o];
  }
}

static bool vec4_ok(int d) { return d % 4 == 0 && d <= 128; }

template <int VEC, int S>
static kg_status launch_agg(const AggArgs& a, int blocks, size_t smem, cudaStream_t st) {
  KG_LAUNCH("k_aggregate", (k_aggregate<VEC, S>), blocks, 256, smem, st, a);
  return KG_OK;
}
template <int VEC, int S>
static kg_status launch_csc(const CscArgs& a, int blocks, size_t smem, cudaStream_t st) {
  KG_LAUNCH("k_csc_backward", (k_csc_backward<VEC, S>), blocks, 256, smem, st, a);
  return KG_OK;
}

static kg_status run_aggregate(const AggArgs& a, int64_t rows_max, cudaStream_t st) {
  int blocks = persistent_blocks(rows_max * 32, 256, 8);
  size_t smem = (size_t)a.G * a.B * sizeof(float);
  int d = a.d;
  if (vec4_ok(d)) launch_agg<4, 1>(a, blocks, smem, st);
  else if (d <= 32) launch_agg<1, 1>(a, blocks, smem, st);
  else if (d <= 64) launch_agg<1, 2>(a, blocks, smem, st);
  else if (d <= 128) launch_agg<1, 4>(a, blocks, smem, st);
  else if (d <= 256) launch_agg<1, 8>(a, blocks, smem, st);
  else KG_REQUIRE(false, KG_ERR_SHAPE, "feature width %d > 256 unsupported", d);
  KG_CHECK_LAUNCH("k_aggregate");
  return KG_OK;
}

static kg_status run_csc(const CscArgs& a, int64_t rows_max, cudaStream_t st) {
  int blocks = persistent_blocks(rows_max * 32, 256, 8);
  size_t smem = (size_t)a.G * a.B * sizeof(float);
  int d = a.d;
  if (vec4_ok(d)) launch_csc<4, 1>(a, blocks, smem, st);
  else if (d <= 32) launch_csc<1, 1>(a, blocks, smem, st);
  else if (d <= 64) launch_csc<1, 2>(a, blocks, smem, st);
  else if (d <= 128) launch_csc<1, 4>(a, blocks, smem, st);
  else if (d <= 256) launch_csc<1, 8>(a, blocks, smem, st);
  else KG_REQUIRE(false, KG_ERR_SHAPE, "feature width %d > 256 unsupported", d);
  KG_CHECK_LAUNCH("k_csc_backward");
  return KG_OK;
}

struct LayerWs {
  float* acc;     // forward (n, B*d_in)
  float* Wy;      // (d_in, B*d_out)
  float* Wb;      // (B*d_out, d_in)
  float* dZ;      // (n, d_out)
  float* Y;       // (n, B*d_out)
  float* dS;      // (n, B*d_out)
  float* ed;      // (e, B)
  float* ed_self; // (n, B)
  float* Rm;      // (d_in, B*d_out)
  char* tn;       // split-K partials
};

static size_t layer_ws(int64_t n, int64_t e, int di, int dO, int B, LayerWs* w, void* base, size_t cap) {
  Arena a(base, cap);
  LayerWs l;
  l.acc = a.take<float>((size_t)n * B * di);
  l.Wy = a.take<float>((size_t)B * di * dO);
  l.Wb = a.take<float>((size_t)B * di * dO);
  l.dZ = a.take<float>((size_t)n * dO);
  l.Y = a.take<float>((size_t)n * B * dO);
  l.dS = a.take<float>((size_t)n * B * dO);
  l.ed = a.take<float>((size_t)e * B);
  l.ed_self = a.take<float>((size_t)n * B);
  l.Rm = a.take<float>((size_t)di * B * dO);
  l.tn = a.take<char>(gemm_tn_workspace(n, di, (int64_t)B * dO));
  if (w) *w = l;
  return a.used + 256;
}

}  // namespace kg

using namespace kg;

extern "C" {

int64_t kg_layer_workspace_bytes(int32_t n, int64_t e, int32_t d_in, int32_t d_out, int32_t B) {
  return (int64_t)layer_ws(n, e, d_in, d_out, B, nullptr, nullptr, 0);
}

kg_status kg_rgcn_forward(const kg_graph_csr* G, const kg_layer_params* lp, const float* H_in, float* H_out,
                          const int32_t* order, const int32_t* counts, int32_t t, int32_t relu, void* ws,
                          int64_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(lp->B >= 1 && lp->B <= MAXB, KG_ERR_VALIDATION, "num_bases must be in [1, %d]", MAXB);
  KG_REQUIRE(lp->G == 2 * G->R + 1, KG_ERR_SHAPE, "coeff groups %d != 2R+1", lp->G);
  LayerWs w;
  size_t need = layer_ws(G->n, G->e, lp->d_in, lp->d_out, lp->B, &w, ws, (size_t)ws_bytes);
  KG_REQUIRE((size_t)ws_bytes >= need, KG_ERR_VALIDATION, "layer workspace too small");
  AggArgs a{G->indptr, G->src, G->rel, G->norm, lp->coeffs, lp->G, lp->B, lp->d_in, H_in, order, counts, t, w.acc};
  kg_status s = run_aggregate(a, G->n, st);
  if (s != KG_OK) return s;
  GemmArgs g{};
  g.A = w.acc;
  g.lda = (int64_t)lp->B * lp->d_in;
  g.B = lp->bases;   // (B*d_in, d_out)
  g.ldb = lp->d_out;
  g.C = H_out;
  g.ldc = lp->d_out;
  g.c_rows = order;
  g.M_dev = counts;
  g.M_dev_index = t;
  g.M_max = G->n;
  g.K = (int64_t)lp->B * lp->d_in;
  g.N = lp->d_out;
  g.relu = relu;
  return gemm_nn(g, st);
}

kg_status kg_rgcn_backward(const kg_graph_csr* G, const kg_layer_params* lp, const float* H_in, const float* H_out,
                           const float* dH_out, float* dH_in, const int32_t* order, const int32_t* pos,
                           const int32_t* counts, int32_t t, float* d_bases, float* d_coeffs, void* ws,
                           int64_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  const int B = lp->B, di = lp->d_in, dO = lp->d_out;
  KG_REQUIRE(B >= 1 && B <= MAXB, KG_ERR_VALIDATION, "num_bases must be in [1, %d]", MAXB);
  LayerWs w;
  size_t need = layer_ws(G->n, G->e, di, dO, B, &w, ws, (size_t)ws_bytes);
  KG_REQUIRE((size_t)ws_bytes >= need, KG_ERR_VALIDATION, "layer workspace too small");
  const int64_t wn = (int64_t)B * di * dO;
  KG_LAUNCH("k_weight_views", k_weight_views, persistent_blocks(wn, 256, 2), 256, 0, st, lp->bases, B, di, dO, w.Wy, w.Wb);
  KG_LAUNCH("k_dz", k_dz, persistent_blocks((int64_t)G->n * dO, 256, 8), 256, 0, st, dH_out, H_out, order, counts, t, dO, w.dZ);
  KG_CHECK_LAUNCH("backward prep");
  // Y = X[A_{t+1}] . [V_0 | .. | V_{B-1}]
  GemmArgs gy{};
  gy.A = H_in; gy.lda = di; gy.a_rows = order;
  gy.B = w.Wy; gy.ldb = (int64_t)B * dO;
  gy.C = w.Y; gy.ldc = (int64_t)B * dO;
  gy.M_dev = counts; gy.M_dev_index = t + 1; gy.M_max = G->n;
  gy.K = di; gy.N = (int64_t)B * dO;
  kg_status s = gemm_nn(gy, st);
  if (s != KG_OK) return s;
  CscArgs c{G->c_indptr, G->c_dst, G->c_rel, G->c_norm, lp->coeffs, lp->G, B, dO, w.Y, w.dZ, order, pos, counts,
            t, w.dS, w.ed, w.ed_self};
  s = run_csc(c, G->n, st);
  if (s != KG_OK) return s;
  // dV = X^T dS  (reduction over the source rows)
  GemmArgs gv{};
  gv.A = H_in; gv.lda = di; gv.a_rows = order;
  gv.B = w.dS; gv.ldb = (int64_t)B * dO;
  gv.M_dev = counts; gv.M_dev_index = t + 1; gv.M_max = G->n;
  gv.K = di; gv.N = (int64_t)B * dO;
  s = gemm_tn(gv, w.Rm, w.tn, st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_dbases_layout", k_dbases_layout, persistent_blocks(wn, 256, 2), 256, 0, st, w.Rm, B, di, dO, d_bases);
  if (dH_in) {
    GemmArgs gx{};
    gx.A = w.dS; gx.lda = (int64_t)B * dO;
    gx.B = w.Wb; gx.ldb = di;
    gx.C = dH_in; gx.ldc = di; gx.c_rows = order;
    gx.M_dev = counts; gx.M_dev_index = t + 1; gx.M_max = G->n;
    gx.K = (int64_t)B * dO; gx.N = di;
    s = gemm_nn(gx, st);
    if (s != KG_OK) return s;
  }
  KG_LAUNCH("k_dcoeff_reduce", k_dcoeff_reduce, lp->G, 256, 0, st, G->rel_ptr, G->rel_perm, G->c_dst, pos, counts, t, w.ed, w.ed_self, lp->G,
                                         B, d_coeffs);
  KG_CHECK_LAUNCH("k_dcoeff_reduce");
  return KG_OK;
}

}  // extern "C"
