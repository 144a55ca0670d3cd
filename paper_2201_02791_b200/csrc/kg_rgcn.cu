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
//
// Gather/scatter passes run one warp per static work chunk (<= 64 messages of
// one row, kg_chunks.cu) so preferential-attachment hubs are spread over many
// warps; rows cut into several chunks are finished by a combine pass (one
// block per row) that adds the chunk partials in a fixed order (no atomics,
// deterministic). Lanes cover the feature dimension (float4 per lane for
// d % 4 == 0, d <= 128). A chunk's metadata (2 messages per lane) is fetched
// in one shot and each message carries its own coefficients norm_e*a[r_e,b],
// so gathered rows stream with UNR loads in flight per lane and no serial
// dependency between messages.
#include "kg_gemm.cuh"

#include <stdlib.h>

namespace kg {

constexpr int MAXB = 4;
constexpr int UNR = 8;     // gathered rows in flight per lane
constexpr int MAXC = 64;   // messages per chunk handled by one warp (2 per lane)
#ifndef KG_GATHER_BPS
#define KG_GATHER_BPS 4    // resident 256-thread blocks per SM of the gather kernels (4: +7 % HBM at wikikg2 shape, no spills; 5 spills)
#endif

// Sum x[0..7] over the 32 lanes of a warp, 9 shuffles: on return lane l holds
// the total of entry ((l>>4)&1)*4 + ((l>>3)&1)*2 + ((l>>2)&1).
__device__ __forceinline__ float warp_sum8(const float* x) {
  const unsigned l = lane_id();
  const bool b4 = l & 16, b3 = l & 8, b2 = l & 4;
  float y[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float send = b4 ? x[i] : x[i + 4];
    float keep = b4 ? x[i + 4] : x[i];
    y[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  float z[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    float send = b3 ? y[i] : y[i + 2];
    float keep = b3 ? y[i + 2] : y[i];
    z[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  float send = b2 ? z[0] : z[1];
  float keep = b2 ? z[1] : z[0];
  float w = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  w += __shfl_xor_sync(0xffffffffu, w, 2);
  w += __shfl_xor_sync(0xffffffffu, w, 1);
  return w;
}

__device__ __forceinline__ int sum8_entry(unsigned l) { return ((l >> 4) & 1) * 4 + ((l >> 3) & 1) * 2 + ((l >> 2) & 1); }

// Sum x[0..3] over the 32 lanes, 7 shuffles: lane l holds the total of entry
// ((l>>4)&1)*2 + ((l>>3)&1).
__device__ __forceinline__ float warp_sum4(const float* x) {
  const unsigned l = lane_id();
  const bool b4 = l & 16, b3 = l & 8;
  float y[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    float send = b4 ? x[i] : x[i + 2];
    float keep = b4 ? x[i + 2] : x[i];
    y[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  float send = b3 ? y[0] : y[1];
  float keep = b3 ? y[1] : y[0];
  float w = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  w += __shfl_xor_sync(0xffffffffu, w, 4);
  w += __shfl_xor_sync(0xffffffffu, w, 2);
  w += __shfl_xor_sync(0xffffffffu, w, 1);
  return w;
}

__device__ __forceinline__ int sum4_entry(unsigned l) { return ((l >> 4) & 1) * 2 + ((l >> 3) & 1); }

#ifndef KG_WIDE_UNR
#define KG_WIDE_UNR 4   // rows in flight per lane in the fused wide-row (EPI = 1) CSC pass: 8 or 4
#endif

// Sum x[0..7] over the LPR (>= 8) lanes of a lane group (xor offsets < LPR),
// transposed: 7 shuffles + log2(LPR / 8) for eight totals instead of
// 8 * log2(LPR). On return the lane holds the total of entry
// entry8<LPR>(lane); lanes differing only in the bits below LPR / 8 agree.
template <int LPR>
__device__ __forceinline__ float group_sum8(const float* x, unsigned l) {
  constexpr unsigned O1 = LPR / 2, O2 = LPR / 4, O3 = LPR / 8;
  const bool b1 = l & O1, b2 = l & O2, b3 = l & O3;
  float y[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = b1 ? x[i] : x[i + 4], keep = b1 ? x[i + 4] : x[i];
    y[i] = keep + __shfl_xor_sync(0xffffffffu, send, O1);
  }
  float z[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = b2 ? y[i] : y[i + 2], keep = b2 ? y[i + 2] : y[i];
    z[i] = keep + __shfl_xor_sync(0xffffffffu, send, O2);
  }
  const float send = b3 ? z[0] : z[1], keep = b3 ? z[1] : z[0];
  float w = keep + __shfl_xor_sync(0xffffffffu, send, O3);
#pragma unroll
  for (unsigned o = O3 / 2; o >= 1; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
  return w;
}

template <int LPR>
__device__ __forceinline__ int entry8(unsigned l) {
  return ((l & (LPR / 2)) ? 4 : 0) + ((l & (LPR / 4)) ? 2 : 0) + ((l & (LPR / 8)) ? 1 : 0);
}

// Sum x[0..3] over the LPR (>= 4) lanes of a lane group, transposed (3
// shuffles + log2(LPR / 4)); the lane holds the total of entry entry4<LPR>.
template <int LPR>
__device__ __forceinline__ float group_sum4(const float* x, unsigned l) {
  constexpr unsigned O1 = LPR / 2, O2 = LPR / 4;
  const bool b1 = l & O1, b2 = l & O2;
  float y[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = b1 ? x[i] : x[i + 2], keep = b1 ? x[i + 2] : x[i];
    y[i] = keep + __shfl_xor_sync(0xffffffffu, send, O1);
  }
  const float send = b2 ? y[0] : y[1], keep = b2 ? y[1] : y[0];
  float w = keep + __shfl_xor_sync(0xffffffffu, send, O2);
#pragma unroll
  for (unsigned o = O2 / 2; o >= 1; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
  return w;
}

template <int LPR>
__device__ __forceinline__ int entry4(unsigned l) {
  return ((l & (LPR / 2)) ? 2 : 0) + ((l & (LPR / 4)) ? 1 : 0);
}

#ifndef KG_NARROW_UNR
#define KG_NARROW_UNR 4   // rows in flight per lane in the fused narrow-row (EPI = 4) CSC pass: 8 or 4
#endif
#ifndef KG_CSC_WIDE_BPS
#define KG_CSC_WIDE_BPS 4     // resident blocks per SM of the fused wide-row CSC pass
#endif
#ifndef KG_CSC_NARROW_BPS
#define KG_CSC_NARROW_BPS 4   // resident blocks per SM of the fused narrow-row CSC pass
#endif
#ifndef KG_WIDE_NOPRED
#define KG_WIDE_NOPRED 0     // 1: the fused wide-row pass gathers unpredicated
#endif
#ifndef KG_NARROW_NOPRED
#define KG_NARROW_NOPRED 0   // 1: that pass gathers unpredicated (dummy slots read a live row, weight 0)
#endif

struct Chunks {
  const int32_t* ptr;
  const int32_t* row;
  const int32_t* slot;
  const int32_t* split;
  const int32_t* counts;
  int C;
  const int4* desc;      // {row, first message, count | single<<16 | first<<17, slot} per chunk
};

constexpr int CH_SINGLE = 1 << 16, CH_FIRST = 1 << 17;

struct AggArgs {
  const int32_t* indptr;
  const int32_t* src;
  const int32_t* rel;
  const float* norm;
  Chunks ck;
  const float* coeffs;   // (G, B)
  int32_t G, B, d;
  const float* H;        // (n, d) by local id
  const int32_t* pos;
  const int32_t* counts;
  int t;
  float* acc;            // packed GEMM records of the (count, B*d) rows, by position
  int64_t acc_nk;        // signed records per 128-row block (packed_nk(n, B*d)), 0: row-major acc
  float* partial;        // (split chunks, B*d)
};

template <int NB, int VEC, int S>
__device__ __forceinline__ void zero3(float (&a)[NB][S][VEC]) {
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
      for (int c = 0; c < VEC; ++c) a[b][s][c] = 0.f;
}

// metadata of message `lane + 32*h` of the chunk, coefficient c_b = norm * a[rel, b]
template <int NB>
struct EdgeMeta {
  uint32_t off[2];         // element offset of the gathered row: src * d (forward) / dst position * d (backward)
  float cf[2][NB];
};

// Lane base pointers of a gather: column (s * LPR + cl) * VEC of row 0. Lanes
// past the row width point at column 0, so every lane loads real data and the
// message loop needs no per-lane predicate (their sums are never stored, and
// the dots multiply them by zero Y entries).
template <int S, int VEC, int LPR>
__device__ __forceinline__ void lane_bases(const float* base, int cl, const bool (&ok)[S], const float* (&p)[S]) {
#pragma unroll
  for (int s = 0; s < S; ++s) p[s] = base + (ok[s] ? (s * LPR + cl) * VEC : 0);
}

// EPI > 1 (narrow rows, d <= 128 / EPI): lanes split into EPI groups of
// LPR = 32 / EPI lanes; each group gathers a different message, so a warp
// load moves EPI rows and EPI x UNR rows are in flight per warp. The groups'
// sums are folded with xor shuffles before the row is finished.
#ifndef KG_AGG_UNR
#define KG_AGG_UNR 8   // gathered rows in flight per lane in the forward aggregate
#endif
#ifndef KG_AGG_BPS
#define KG_AGG_BPS KG_GATHER_BPS
#endif
// narrow rows (4 messages per warp load): 4 rows in flight per lane and 5
// resident blocks per SM (48 registers) gather faster past L2 than 8 rows at
// 4 blocks (config 5: 0.64 -> 0.70 of HBM); wide rows keep 8 rows at 4 blocks
constexpr int AGG_NARROW_BPS = 5;
template <int EPI>
constexpr int agg_unr() { return EPI >= 4 ? 4 : KG_AGG_UNR; }
template <int NB, int VEC, int S, int EPI>
__global__ void __launch_bounds__(256, EPI >= 4 ? AGG_NARROW_BPS : KG_AGG_BPS) k_aggregate(AggArgs a) {
  extern __shared__ float coef[];
  for (int i = threadIdx.x; i < a.G * a.B; i += blockDim.x) coef[i] = a.coeffs[i];
  __syncthreads();
  const int lane = lane_id();
  constexpr int LPR = 32 / EPI;
  const int grp = lane / LPR, cl = lane % LPR;
  const int32_t T = a.counts[a.t];
  const int32_t NC = a.ck.counts[0];
  const int d = a.d;
  constexpr int B = NB;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  bool slot_ok[S];
#pragma unroll
  for (int s = 0; s < S; ++s) slot_ok[s] = (s * LPR + cl) * VEC < d;
  const float* hb[S];
  lane_bases<S, VEC, LPR>(a.H, cl, slot_ok, hb);
  for (int64_t c = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); c < NC; c += warps) {
    const int4 dsc = a.ck.desc[c];
    const int32_t v = dsc.x, beg = dsc.y, cnt = dsc.z & 0xffff;
    const bool single = dsc.z & CH_SINGLE;
    const int32_t p = a.pos[v];
    if (p < 0 || p >= T) continue;
    // message slots past cnt (the loop runs in groups of UNR * EPI) gather the
    // chunk's first row with weight zero: no per-message predicate or zeroing
    EdgeMeta<NB> m;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = lane + 32 * h;
      m.off[h] = 0;
#pragma unroll
      for (int b = 0; b < NB; ++b) m.cf[h][b] = 0.f;
      if (e < cnt) {
        m.off[h] = (uint32_t)a.src[beg + e] * (uint32_t)d;
        const int32_t r = a.rel[beg + e];
        const float w = a.norm[beg + e];
#pragma unroll
        for (int b = 0; b < NB; ++b)
          if (b < B) m.cf[h][b] = w * coef[r * B + b];
      }
    }
    {
      const uint32_t off0 = __shfl_sync(0xffffffffu, m.off[0], 0);
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (lane + 32 * h >= cnt) m.off[h] = off0;
    }
    float acc[NB][S][VEC];
    zero3<NB, VEC, S>(acc);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int nh = min(32, cnt - 32 * h);
      for (int j = 0; j < nh; j += agg_unr<EPI>() * EPI) {
        float xs[agg_unr<EPI>()][S][VEC];
#pragma unroll
        for (int q = 0; q < agg_unr<EPI>(); ++q) {
          const uint32_t off = __shfl_sync(0xffffffffu, m.off[h], (j + q * EPI + grp) & 31);
#pragma unroll
          for (int s = 0; s < S; ++s) VecIO<VEC>::load(hb[s] + off, xs[q][s]);
        }
#pragma unroll
        for (int q = 0; q < agg_unr<EPI>(); ++q) {
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            if (b < B) {
              const float cf = __shfl_sync(0xffffffffu, m.cf[h][b], (j + q * EPI + grp) & 31);
#pragma unroll
              for (int s = 0; s < S; ++s)
#pragma unroll
                for (int cc = 0; cc < VEC; ++cc) acc[b][s][cc] = fmaf(cf, xs[q][s][cc], acc[b][s][cc]);
            }
          }
        }
      }
    }
    if (EPI > 1) {
      // fold the message groups (lanes cl, cl + LPR, ...): every lane holds the total
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int s2 = 0; s2 < S; ++s2)
#pragma unroll
            for (int cc = 0; cc < VEC; ++cc) acc[b][s2][cc] += __shfl_xor_sync(0xffffffffu, acc[b][s2][cc], o);
    }
    // the first lane group owns the row's columns from here on
    bool own[S];
#pragma unroll
    for (int s2 = 0; s2 < S; ++s2) own[s2] = slot_ok[s2] && grp == 0;
    float* out;
    if (single) {
      // self-loop group 2R (norm 1), then the finished row
      float xv[S][VEC];
#pragma unroll
      for (int s = 0; s < S; ++s)
        if (own[s]) VecIO<VEC>::load(a.H + (int64_t)v * d + (s * LPR + cl) * VEC, xv[s]);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (b < B) {
          float cf = coef[(a.G - 1) * B + b];
#pragma unroll
          for (int s = 0; s < S; ++s)
            if (own[s])
#pragma unroll
              for (int cc = 0; cc < VEC; ++cc) acc[b][s][cc] = fmaf(cf, xv[s][cc], acc[b][s][cc]);
        }
      }
      if (a.acc_nk) {
        // finished row: straight into the GEMM's packed A records
#pragma unroll
        for (int b = 0; b < NB; ++b)
          if (b < B)
#pragma unroll
            for (int s = 0; s < S; ++s)
              if (own[s]) packed_store<VEC>(a.acc, a.acc_nk, p, b * d + (s * LPR + cl) * VEC, acc[b][s]);
        packed_zero_pad(a.acc, a.acc_nk, p, B * d, lane, 32);
        continue;
      }
      out = a.acc + (int64_t)p * B * d;   // row-major (the GEMM packs it)
    } else {
      out = a.partial + (int64_t)dsc.w * B * d;
    }
#pragma unroll
    for (int b = 0; b < NB; ++b)
      if (b < B)
#pragma unroll
        for (int s = 0; s < S; ++s)
          if (own[s]) VecIO<VEC>::store(out + (int64_t)b * d + (s * LPR + cl) * VEC, acc[b][s]);
  }
}

// Rows cut into several chunks (hubs): one 256-thread block per row. Thread
// (g, c) sums the partials of chunks g, g + G, ... of V-wide column c (in chunk
// order); the G group sums are then added in group order — a fixed summation
// order (deterministic, no atomics) with G-fold parallelism over the chunks.
constexpr int CB_THREADS = 256;

template <int V>
struct BlockPartialSum {
  float red[V][CB_THREADS];
  // returns, for threads with g == 0 and c < ncols, the column total of
  // V-wide column c0 + c; `valid` tells the caller whether it holds one
  __device__ __forceinline__ void run(const float* __restrict__ part, int width, int np, int c0, int ncols,
                                      float* tot, bool& valid) {
    const int groups = CB_THREADS / ncols;
    const int g = threadIdx.x / ncols, c = threadIdx.x - g * ncols;
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.f;
    if (g < groups) {
      const float* src = part + (int64_t)(c0 + c) * V;
      int k = g;
      for (; k + 3 * groups < np; k += 4 * groups) {
        float y[4][V];
#pragma unroll
        for (int u = 0; u < 4; ++u) VecIO<V>::load(src + (int64_t)(k + u * groups) * width, y[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] += y[u][i];
      }
      for (; k < np; k += groups) {
        float y[V];
        VecIO<V>::load(src + (int64_t)k * width, y);
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] += y[i];
      }
    }
#pragma unroll
    for (int i = 0; i < V; ++i) red[i][threadIdx.x] = acc[i];
    __syncthreads();
    valid = g == 0 && c < ncols;
    if (valid) {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        float t = red[i][c];
        for (int q = 1; q < groups; ++q) t += red[i][q * ncols + c];
        tot[i] = t;
      }
    }
    __syncthreads();
  }
};

template <bool V4>
__global__ void __launch_bounds__(CB_THREADS) k_aggregate_combine(AggArgs a) {
  constexpr int V = V4 ? 4 : 1;
  __shared__ BlockPartialSum<V> bs;
  const int32_t T = a.counts[a.t];
  const int32_t NS = a.ck.counts[2];
  const int width = a.B * a.d, cols = width / V;
  for (int64_t r = blockIdx.x; r < NS; r += gridDim.x) {
    const int32_t v = a.ck.split[r];
    const int32_t p = a.pos[v];
    if (p < 0 || p >= T) continue;
    const int32_t c0 = a.ck.ptr[v], np = a.ck.ptr[v + 1] - c0;
    const float* part = a.partial + (int64_t)a.ck.slot[c0] * width;
    for (int cb = 0; cb < cols; cb += CB_THREADS) {
      const int ncols = min(CB_THREADS, cols - cb);
      float tot[V];
      bool valid;
      bs.run(part, width, np, cb, ncols, tot, valid);
      if (valid) {
        const int col = (cb + (int)threadIdx.x) * V;
        const int b = col / a.d, kk = col - b * a.d;
        const float cf = a.coeffs[(a.G - 1) * a.B + b];
        float h[V], x[V];
        VecIO<V>::load(a.H + (int64_t)v * a.d + kk, h);
#pragma unroll
        for (int i = 0; i < V; ++i) {
          const float self = cf * h[i];
          x[i] = tot[i] + self;
        }
        if (a.acc_nk) packed_store<V>(a.acc, a.acc_nk, p, col, x);
        else VecIO<V>::store(a.acc + (int64_t)p * width + col, x);
      }
    }
    if (a.acc_nk && threadIdx.x < 32) packed_zero_pad(a.acc, a.acc_nk, p, width, threadIdx.x, 32);
  }
}

struct CscArgs {
  const int32_t* c_indptr;
  const int32_t* c_dst;
  const int32_t* c_rel;
  const float* c_norm;
  Chunks ck;
  const float* coeffs;   // (G, B)
  int32_t G, B, d;       // d = d_out
  const float* Y;        // (count_S, B*d) compact: X V_b per source position
  const float* dZ;       // (count_T, d) compact
  const int32_t* pos;
  const int32_t* c_pos;  // optional: pos[c_dst[e]] per CSC message for this round (kg_csc_positions)
  const int32_t* counts;
  int t;                 // targets A_t, sources A_{t+1}
  float* dS;             // (count_S, B*d)
  float* ed;             // (e, B) per CSC position
  float* ed_self;        // (count_T, B)
  float* partial;        // (split chunks, B*d)
  float* dS_pk;          // optional: dS also as packed GEMM A records (dX = dS . Wb)
  int64_t dS_nk;
  int self_dots;         // k_csc_combine: also the split rows' self dots (MODE 0 runs)
};

// MODE 0: dS and edge dots in one pass. MODE 1: dS only (the critical path:
// dX = dS . Wb feeds the next layer). MODE 2: edge dots + self dots only (they
// feed only d coeffs, so this pass runs on the forked stream).
// EPI > 1 (narrow rows): message groups as in k_aggregate; the edge dots
// then reduce within a lane group (log2(LPR) shuffles per message).
template <int NB, int VEC, int S, int MODE, int EPI>
__global__ void __launch_bounds__(256, (MODE == 0 && EPI >= 4) ? KG_CSC_NARROW_BPS
                                      : (MODE == 0 && EPI == 1) ? KG_CSC_WIDE_BPS : KG_GATHER_BPS)
    k_csc_backward(CscArgs a) {
  extern __shared__ float coef[];
  for (int i = threadIdx.x; i < a.G * a.B; i += blockDim.x) coef[i] = a.coeffs[i];
  __syncthreads();
  const unsigned lane = lane_id();
  constexpr int LPR = 32 / EPI;
  constexpr int U = (MODE == 0 && EPI == 4) ? KG_NARROW_UNR : (MODE == 0 && EPI == 1) ? KG_WIDE_UNR : UNR;
  // predicated gathers (skip marker ~0 in the offset) where registers are short
  constexpr bool PRED = MODE == 0 && !(EPI == 4 && KG_NARROW_NOPRED) && !(EPI == 1 && KG_WIDE_NOPRED);
  const int grp = (int)lane / LPR, cl = (int)lane % LPR;
  const int32_t T = a.counts[a.t];
  const int32_t Sn = a.counts[a.t + 1];
  const int32_t NC = a.ck.counts[0];
  const int d = a.d;
  constexpr int B = NB;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  bool slot_ok[S];
#pragma unroll
  for (int s = 0; s < S; ++s) slot_ok[s] = (s * LPR + cl) * VEC < d;
  const float* zb[S];
  lane_bases<S, VEC, LPR>(a.dZ, cl, slot_ok, zb);
  for (int64_t c = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); c < NC; c += warps) {
    const int4 dsc = a.ck.desc[c];
    const int32_t u = dsc.x, beg = dsc.y, cnt = dsc.z & 0xffff;
    const bool single = dsc.z & CH_SINGLE, first = dsc.z & CH_FIRST;
    const int32_t q = a.pos[u];
    if (q < 0 || q >= Sn) {
      // not a source of this layer: its edge dots are zero (k_dcoeff_partial
      // sums every edge of a relation without a membership test)
      if (MODE != 1)
        for (int x = (int)lane; x < cnt * B; x += 32) a.ed[(int64_t)beg * B + x] = 0.f;
      continue;
    }
    // metadata: destination position (-1 if not a target) and coefficients
    // messages to non-targets and the slots past cnt gather the chunk's first
    // target row with weight zero (no per-message predicate); a chunk without
    // targets gathers nothing
    EdgeMeta<NB> m;
    float nrm[2];
    bool live[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = (int)lane + 32 * h;
      m.off[h] = PRED ? ~0u : 0u;   // predicated pass: ~0 marks a message to skip
      nrm[h] = 0.f;
      live[h] = false;
#pragma unroll
      for (int b = 0; b < NB; ++b) m.cf[h][b] = 0.f;
      if (e < cnt) {
        const int32_t r = a.c_rel[beg + e];
        const float nw = a.c_norm[beg + e];
        const int32_t pw = a.c_pos ? a.c_pos[beg + e] : a.pos[a.c_dst[beg + e]];
        if (pw >= 0 && pw < T) {
          m.off[h] = (uint32_t)pw * (uint32_t)d;
          nrm[h] = nw;
          live[h] = true;
          if (MODE != 2)
#pragma unroll
            for (int b = 0; b < NB; ++b)
              if (b < B) m.cf[h][b] = nw * coef[r * B + b];
        }
      }
    }
    int ngather = cnt;
    if (!PRED) {
      const unsigned v0 = __ballot_sync(0xffffffffu, live[0]), v1 = __ballot_sync(0xffffffffu, live[1]);
      if ((v0 | v1) == 0) {
        ngather = 0;
        if (MODE != 1)
          for (int x = (int)lane; x < cnt * B; x += 32) a.ed[(int64_t)beg * B + x] = 0.f;
      } else {
        const uint32_t o0 = __shfl_sync(0xffffffffu, v0 ? m.off[0] : m.off[1], v0 ? __ffs(v0) - 1 : __ffs(v1) - 1);
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (!live[h]) m.off[h] = o0;
      }
    }
    float y[NB][S][VEC];
    float acc[NB][S][VEC];
    zero3<NB, VEC, S>(acc);
    zero3<NB, VEC, S>(y);
    if (MODE != 1)
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (b < B)
#pragma unroll
          for (int s = 0; s < S; ++s)
            if (slot_ok[s]) VecIO<VEC>::load(a.Y + ((int64_t)q * B + b) * d + (s * LPR + cl) * VEC, y[b][s]);
    // wide rows: the two message halves share one copy of the loop body (a
    // rolled loop with the half's metadata selected: the unrolled pair made
    // the fused pass 3,160 instructions and instruction-cache misses a top
    // stall; rolled 936). Narrow rows keep the unrolled pair (rolling them
    // spills).
#pragma unroll(EPI == 1 ? 1 : 2)
    for (int h = 0; h < 2; ++h) {
      const int nh = min(32, ngather - 32 * h);
      const uint32_t offh = h ? m.off[1] : m.off[0];
      const float nrmh = h ? nrm[1] : nrm[0];
      float cfh[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) cfh[b] = h ? m.cf[1][b] : m.cf[0][b];
      for (int j = 0; j < nh; j += U * EPI) {
        float zs[U][S][VEC];
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const uint32_t off = __shfl_sync(0xffffffffu, offh, (j + k * EPI + grp) & 31);
          if (!PRED) {
#pragma unroll
            for (int s = 0; s < S; ++s) VecIO<VEC>::load(zb[s] + off, zs[k][s]);
          } else {
            const bool ld = j + k * EPI + grp < nh && off != ~0u;
#pragma unroll
            for (int s = 0; s < S; ++s) {
              if (ld && slot_ok[s])
                VecIO<VEC>::load(a.dZ + off + (s * LPR + cl) * VEC, zs[k][s]);
              else
#pragma unroll
                for (int cc = 0; cc < VEC; ++cc) zs[k][s][cc] = 0.f;
            }
          }
        }
        // dS_b += c_eb * dZ[dst]
        if (MODE != 2)
#pragma unroll
        for (int k = 0; k < U; ++k) {
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            if (b < B) {
              const float cf = __shfl_sync(0xffffffffu, cfh[b], (j + k * EPI + grp) & 31);
#pragma unroll
              for (int s = 0; s < S; ++s)
#pragma unroll
                for (int cc = 0; cc < VEC; ++cc) acc[b][s][cc] = fmaf(cf, zs[k][s][cc], acc[b][s][cc]);
            }
          }
        }
        // per-edge dots <Y_b[u], dZ[dst]>, message groups: one transposed
        // reduction of the UNR (= 8) messages inside each lane group
        if (MODE != 1 && EPI > 1)
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          if (b < B) {
            float part[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
              float dp = 0.f;
#pragma unroll
              for (int s = 0; s < S; ++s)
#pragma unroll
                for (int cc = 0; cc < VEC; ++cc) dp = fmaf(y[b][s][cc], zs[k][s][cc], dp);
              part[k] = dp;
            }
            float tot;
            int k;
            if constexpr (U == 8) {
              tot = group_sum8<LPR>(part, (unsigned)cl);
              k = entry8<LPR>((unsigned)cl);
            } else {
              tot = group_sum4<LPR>(part, (unsigned)cl);
              k = entry4<LPR>((unsigned)cl);
            }
            const int e = j + k * EPI + grp;
            const float wk = __shfl_sync(0xffffffffu, nrmh, e & 31);
            if ((cl & (LPR / U - 1)) == 0 && e < nh) a.ed[(int64_t)(beg + 32 * h + e) * B + b] = wk * tot;
          }
        }
        // per-edge dots, one message per warp load: one transposed warp reduction per b
        if (MODE != 1 && EPI == 1)
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          if (b < B) {
            float part[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
              float dp = 0.f;
#pragma unroll
              for (int s = 0; s < S; ++s)
#pragma unroll
                for (int cc = 0; cc < VEC; ++cc) dp = fmaf(y[b][s][cc], zs[k][s][cc], dp);
              part[k] = dp;
            }
            float tot;
            int k;
            if constexpr (U == 8) {
              tot = warp_sum8(part);
              k = sum8_entry(lane);
            } else {
              tot = warp_sum4(part);
              k = sum4_entry(lane);
            }
            const float wk = __shfl_sync(0xffffffffu, nrmh, (j + k) & 31);
            if ((lane & (32 / U - 1)) == 0 && j + k < nh) a.ed[(int64_t)(beg + 32 * h + j + k) * B + b] = wk * tot;
          }
        }
      }
    }
    if (MODE == 2) {
      // self dot for d a[2R,b], by the row's first chunk (split rows too)
      if (first && q < T) {
        float z[S][VEC];
#pragma unroll
        for (int s = 0; s < S; ++s) {
          if (slot_ok[s] && grp == 0) VecIO<VEC>::load(a.dZ + (int64_t)q * d + (s * LPR + cl) * VEC, z[s]);
          else
#pragma unroll
            for (int cc = 0; cc < VEC; ++cc) z[s][cc] = 0.f;
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          if (b < B) {
            float dp = 0.f;
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
              for (int cc = 0; cc < VEC; ++cc) dp = fmaf(y[b][s][cc], z[s][cc], dp);
            dp = warp_sum(dp);
            if (lane == 0) a.ed_self[(int64_t)q * B + b] = dp;
          }
        }
      }
      continue;
    }
    if (EPI > 1) {
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int s2 = 0; s2 < S; ++s2)
#pragma unroll
            for (int cc = 0; cc < VEC; ++cc) acc[b][s2][cc] += __shfl_xor_sync(0xffffffffu, acc[b][s2][cc], o);
    }
    bool own[S];   // the first lane group owns the row's columns from here on
#pragma unroll
    for (int s2 = 0; s2 < S; ++s2) own[s2] = slot_ok[s2] && grp == 0;
    float* out;
    if (single) {
      if (q < T) {
        // self-loop (norm 1): dS += a[2R,b] dZ[u]; self dot for d a[2R,b]
        float z[S][VEC];
#pragma unroll
        for (int s = 0; s < S; ++s) {
          if (own[s]) VecIO<VEC>::load(a.dZ + (int64_t)q * d + (s * LPR + cl) * VEC, z[s]);
          else
#pragma unroll
            for (int cc = 0; cc < VEC; ++cc) z[s][cc] = 0.f;
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          if (b < B) {
            float cf = coef[(a.G - 1) * B + b];
            float dp = 0.f;
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
              for (int cc = 0; cc < VEC; ++cc) {
                acc[b][s][cc] = fmaf(cf, z[s][cc], acc[b][s][cc]);
                dp = fmaf(y[b][s][cc], z[s][cc], dp);
              }
            if (MODE == 0) {
              dp = warp_sum(dp);
              if (lane == 0) a.ed_self[(int64_t)q * B + b] = dp;
            }
          }
        }
      }
      out = a.dS ? a.dS + (int64_t)q * B * d : nullptr;   // row-major dS only for a consumer that reads it
      if (a.dS_pk) {
#pragma unroll
        for (int b = 0; b < NB; ++b)
          if (b < B)
#pragma unroll
            for (int s = 0; s < S; ++s)
              if (own[s]) packed_store<VEC>(a.dS_pk, a.dS_nk, q, b * d + (s * LPR + cl) * VEC, acc[b][s]);
        packed_zero_pad(a.dS_pk, a.dS_nk, q, B * d, lane, 32);
      }
    } else {
      out = a.partial + (int64_t)dsc.w * B * d;
    }
    if (out)
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (b < B)
#pragma unroll
          for (int s = 0; s < S; ++s)
            if (own[s]) VecIO<VEC>::store(out + (int64_t)b * d + (s * LPR + cl) * VEC, acc[b][s]);
  }
}

// c_pos[e] = pos[c_dst[e]]: the closure position of every CSC message's
// destination for this round, so the CSC passes gather dZ rows with one
// dependent load per message instead of two (c_dst, then pos).
__global__ void k_csc_positions(const int32_t* __restrict__ c_dst, int64_t e, const int32_t* __restrict__ pos,
                                int32_t* __restrict__ c_pos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x)
    c_pos[i] = pos[c_dst[i]];
}

// Split source rows: one block per row (chunk-order partial sums as in
// k_aggregate_combine, plus the self-loop term into dS), then the self dots
// <Y_b[u], dZ[u]> for d a[2R, b] by warp 0.
template <bool V4>
__global__ void __launch_bounds__(CB_THREADS) k_csc_combine(CscArgs a) {
  constexpr int V = V4 ? 4 : 1;
  __shared__ BlockPartialSum<V> bs;
  const int32_t T = a.counts[a.t];
  const int32_t Sn = a.counts[a.t + 1];
  const int32_t NS = a.ck.counts[2];
  const int width = a.B * a.d, cols = width / V;
  for (int64_t r = blockIdx.x; r < NS; r += gridDim.x) {
    const int32_t u = a.ck.split[r];
    const int32_t q = a.pos[u];
    if (q < 0 || q >= Sn) continue;
    const int32_t c0 = a.ck.ptr[u], np = a.ck.ptr[u + 1] - c0;
    const float* part = a.partial + (int64_t)a.ck.slot[c0] * width;
    const bool self = q < T;
    for (int cb = 0; cb < cols; cb += CB_THREADS) {
      const int ncols = min(CB_THREADS, cols - cb);
      float tot[V];
      bool valid;
      bs.run(part, width, np, cb, ncols, tot, valid);
      if (valid) {
        const int col = (cb + (int)threadIdx.x) * V;
        const int b = col / a.d, kk = col - b * a.d;
        float z[V], x[V];
        if (self) VecIO<V>::load(a.dZ + (int64_t)q * a.d + kk, z);
        else
#pragma unroll
          for (int i = 0; i < V; ++i) z[i] = 0.f;
        const float cf = a.coeffs[(a.G - 1) * a.B + b];
#pragma unroll
        for (int i = 0; i < V; ++i) x[i] = tot[i] + cf * z[i];
        if (a.dS) VecIO<V>::store(a.dS + (int64_t)q * width + col, x);
        if (a.dS_pk) packed_store<V>(a.dS_pk, a.dS_nk, q, col, x);
      }
    }
    if (a.dS_pk && threadIdx.x < 32) packed_zero_pad(a.dS_pk, a.dS_nk, q, width, threadIdx.x, 32);
    if (a.self_dots && self && threadIdx.x < 32) {
      const int lane = threadIdx.x;
      for (int b = 0; b < a.B; ++b) {
        float dp = 0.f;
        for (int k = lane * V; k < a.d; k += 32 * V) {
          float y[V], z[V];
          VecIO<V>::load(a.Y + ((int64_t)q * a.B + b) * a.d + k, y);
          VecIO<V>::load(a.dZ + (int64_t)q * a.d + k, z);
#pragma unroll
          for (int i = 0; i < V; ++i) dp = fmaf(y[i], z[i], dp);
        }
        dp = warp_sum(dp);
        if (lane == 0) a.ed_self[(int64_t)q * a.B + b] = dp;
      }
    }
  }
}

// d coeffs (ref:model.py:294): d a[g,b] = sum over the edges of relation
// group g of the edge dots (ed is zero for edges outside the layer), plus the
// self-loop group over ed_self. Block (g, s) sums the s-th of `split`
// contiguous slices of the group (fixed order: thread-strided then a fixed
// tree), k_dcoeff_final adds the slices in order -> deterministic, and heavy
// relations are spread over several blocks (split grows with the average
// group size, up to DC_SPLIT).
constexpr int DC_SPLIT = 1024;   // few relation groups (citation2: 3) still fill the GPU

static int dcoeff_split(int64_t e, int64_t groups) {
  int64_t s = (e / (groups > 0 ? groups : 1) + 4095) / 4096;
  return (int)(s < 1 ? 1 : (s > DC_SPLIT ? DC_SPLIT : s));
}

__global__ void __launch_bounds__(256) k_dcoeff_partial(const int32_t* __restrict__ rel_ptr,
                                                        const int32_t* __restrict__ rel_perm,
                                                        const int32_t* __restrict__ counts, int t,
                                                        const float* __restrict__ ed,
                                                        const float* __restrict__ ed_self, int32_t G, int32_t B,
                                                        float* __restrict__ part) {
  __shared__ float red[MAXB][256];
  const int g = blockIdx.x, sl = blockIdx.y, split = gridDim.y;
  int64_t lo, hi;
  if (g < G - 1) {
    lo = rel_ptr[g];
    hi = rel_ptr[g + 1];
  } else {
    lo = 0;
    hi = counts[t];
  }
  const int64_t len = hi - lo, a0 = lo + len * sl / split, a1 = lo + len * (sl + 1) / split;
  float s[MAXB] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t j = a0 + threadIdx.x; j < a1; j += blockDim.x) {
    const float* src = g < G - 1 ? ed + (int64_t)__ldg(rel_perm + j) * B : ed_self + j * B;
#pragma unroll
    for (int b = 0; b < MAXB; ++b)
      if (b < B) s[b] += src[b];
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
  if (threadIdx.x < B) part[((int64_t)g * split + sl) * B + threadIdx.x] = red[threadIdx.x][0];
}

__global__ void k_dcoeff_final(const float* __restrict__ part, int32_t G, int32_t B, int split,
                               float* __restrict__ d_coeffs) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < (int64_t)G * B;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = x / B, b = x - g * B;
    float s = 0.f;
    for (int sl = 0; sl < split; ++sl) s += part[(g * split + sl) * B + b];
    d_coeffs[x] = s;
  }
}

// dZ[p] = dH[v_p] * (H_out[v_p] > 0) (mask skipped when H_out == nullptr); warp per row
template <bool V4>
__global__ void __launch_bounds__(256) k_dz(const float* __restrict__ dH, const float* __restrict__ Hout,
                                            const int32_t* __restrict__ order, const int32_t* __restrict__ counts,
                                            int t, int d, const float* __restrict__ mask, float* __restrict__ dZ) {
  const int32_t T = counts[t];
  const int lane = lane_id(), nw = (gridDim.x * blockDim.x) >> 5;
  constexpr int V = V4 ? 4 : 1;
  for (int64_t p = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); p < T; p += nw) {
    const int64_t src = (int64_t)order[p] * d;
    for (int k = lane * V; k < d; k += 32 * V) {
      float g[V], h[V];
      VecIO<V>::load(dH + src + k, g);
      if (Hout) {
        VecIO<V>::load(Hout + src + k, h);
#pragma unroll
        for (int i = 0; i < V; ++i)
          if (!(h[i] > 0.f)) g[i] = 0.f;
      }
      if (mask) {   // dropout on this output: dA/dZ' = mask (then the ReLU test above)
        float mk[V];
        VecIO<V>::load(mask + p * d + k, mk);
#pragma unroll
        for (int i = 0; i < V; ++i) g[i] *= mk[i];
      }
      VecIO<V>::store(dZ + p * d + k, g);
    }
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

// Tensor-core B operands of one layer, packed once per optimizer step:
//   fwd  (B*d_in x d_out)  Z = acc . [V_b]      element (o, b*d_in+i)
//   y    (d_in x B*d_out)  Y = X . [V_0|..]     element (b*d_out+o, i)
//   dx   (B*d_out x d_in)  dX = dS . [V_b]^T    element (i, b*d_out+o)
// each as records of R = pad16(N) rows x 16 K values (pads zero), tf32 hi | lo
// halves (split once here, not per GEMM tile).
struct WeightsLayout {
  int64_t off[3], rows[3], nk[3], total;
};

static WeightsLayout weights_layout(int di, int dO, int B) {
  WeightsLayout w;
  const int64_t N[3] = {dO, (int64_t)B * dO, di}, K[3] = {(int64_t)B * di, di, (int64_t)B * dO};
  int64_t o = 0;
  for (int j = 0; j < 3; ++j) {
    w.rows[j] = (N[j] + 15) / 16 * 16;
    w.nk[j] = packed_records(K[j]);
    w.off[j] = o;
    o += (w.rows[j] * w.nk[j] * 2 * PK_K + 63) / 64 * 64;   // 256-byte aligned sections
  }
  w.total = o;
  return w;
}

__global__ void k_pack_weights(const float* __restrict__ V, int B, int di, int dO, WeightsLayout L,
                               float* __restrict__ out) {
  const int j = blockIdx.y;
  const int64_t R = L.rows[j], nk = L.nk[j], count = R * nk * PK_K;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < count; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kc = x / (R * PK_K);
    const int rem = (int)(x - kc * R * PK_K);
    const int n = rem / PK_K, kk = rem - n * PK_K;
    const int64_t k = kc * PK_K + kk;
    float val = 0.f;
    if (j == 0) {          // (o = n, b*di + i = k)
      if (n < dO && k < (int64_t)B * di) val = V[k * dO + n];
    } else if (j == 1) {   // (b*dO + o = n, i = k)
      if (n < B * dO && k < di) {
        const int b = n / dO, o = n - b * dO;
        val = V[((int64_t)b * di + k) * dO + o];
      }
    } else {               // (i = n, b*dO + o = k)
      if (n < di && k < (int64_t)B * dO) {
        const int b = (int)(k / dO), o = (int)(k - (int64_t)b * dO);
        val = V[((int64_t)b * di + n) * dO + o];
      }
    }
    float hi, lo;   // B operands stay split (hi | lo halves): reused by every tile
    split_tf32(val, hi, lo);
    float* rec = out + L.off[j] + kc * 2 * R * PK_K;
    rec[pk_off(n, kk)] = hi;
    rec[R * PK_K + pk_off(n, kk)] = lo;
  }
}

// float4 lanes only when they fill most of the warp (d > 64); narrower rows use
// one float per lane so all 32 lanes gather
static bool vec4_ok(int d) { return d % 4 == 0 && d > 64 && d <= 128; }

// chunk capacities of kg_graph_csr (see the header)
static int64_t cap_chunks(const kg_graph_csr* G) { return (int64_t)G->n + G->e / G->chunk + 1; }
static int64_t cap_split_chunks(const kg_graph_csr* G) { return 2 * G->e / G->chunk + 1; }
static int64_t cap_split_rows(const kg_graph_csr* G) { return G->e / G->chunk + 1; }

template <int VEC, int S, int EPI = 1>
static kg_status launch_agg(const AggArgs& a, int blocks, int cblocks, size_t smem, cudaStream_t st) {
  switch (a.B) {
    case 1: KG_LAUNCH("k_aggregate", (k_aggregate<1, VEC, S, EPI>), blocks, 256, smem, st, a); break;
    case 2: KG_LAUNCH("k_aggregate", (k_aggregate<2, VEC, S, EPI>), blocks, 256, smem, st, a); break;
    case 3: KG_LAUNCH("k_aggregate", (k_aggregate<3, VEC, S, EPI>), blocks, 256, smem, st, a); break;
    default: KG_LAUNCH("k_aggregate", (k_aggregate<4, VEC, S, EPI>), blocks, 256, smem, st, a); break;
  }
  if (a.d % 4 == 0) KG_LAUNCH("k_aggregate_combine", k_aggregate_combine<true>, cblocks, CB_THREADS, 0, st, a);
  else KG_LAUNCH("k_aggregate_combine", k_aggregate_combine<false>, cblocks, CB_THREADS, 0, st, a);
  return KG_OK;
}
template <int VEC, int S, int MODE, int EPI = 1>
static kg_status launch_csc_mode(const CscArgs& a, int blocks, size_t smem, cudaStream_t st) {
  const char* name = MODE == 2 ? "k_csc_dots" : "k_csc_backward";
  switch (a.B) {
    case 1: KG_LAUNCH(name, (k_csc_backward<1, VEC, S, MODE, EPI>), blocks, 256, smem, st, a); break;
    case 2: KG_LAUNCH(name, (k_csc_backward<2, VEC, S, MODE, EPI>), blocks, 256, smem, st, a); break;
    case 3: KG_LAUNCH(name, (k_csc_backward<3, VEC, S, MODE, EPI>), blocks, 256, smem, st, a); break;
    default: KG_LAUNCH(name, (k_csc_backward<4, VEC, S, MODE, EPI>), blocks, 256, smem, st, a); break;
  }
  return KG_OK;
}

// mode 0: dS + dots (+ combine); 1: dS (+ combine without self dots); 2: dots only
template <int VEC, int S, int EPI = 1>
static kg_status launch_csc(const CscArgs& a0, int blocks, int cblocks, size_t smem, cudaStream_t st, int mode) {
  CscArgs a = a0;
  a.self_dots = mode == 0;
  kg_status s = mode == 0 ? launch_csc_mode<VEC, S, 0, EPI>(a, blocks, smem, st)
              : mode == 1 ? launch_csc_mode<VEC, S, 1, EPI>(a, blocks, smem, st)
                          : launch_csc_mode<VEC, S, 2, EPI>(a, blocks, smem, st);
  if (s != KG_OK || mode == 2) return s;
  if (a.d % 4 == 0) KG_LAUNCH("k_csc_combine", k_csc_combine<true>, cblocks, CB_THREADS, 0, st, a);
  else KG_LAUNCH("k_csc_combine", k_csc_combine<false>, cblocks, CB_THREADS, 0, st, a);
  return KG_OK;
}

template <typename F4, typename F1a, typename F1b, typename F1c, typename F1d>
static kg_status dispatch_width(int d, F4 f4, F1a f1, F1b f2, F1c f4s, F1d f8) {
  if (vec4_ok(d)) return f4();
  if (d <= 32) return f1();
  if (d <= 64) return f2();
  if (d <= 128) return f4s();
  if (d <= 256) return f8();
  KG_REQUIRE(false, KG_ERR_SHAPE, "feature width %d > 256 unsupported", d);
  return KG_ERR_SHAPE;
}

static kg_status run_aggregate(const AggArgs& a, const kg_graph_csr* G, cudaStream_t st) {
  KG_REQUIRE(G->chunk <= MAXC, KG_ERR_VALIDATION, "chunk size %d > %d", G->chunk, MAXC);
  KG_REQUIRE((int64_t)G->n * a.d < (1LL << 32), KG_ERR_SHAPE, "feature table of %lld x %d exceeds 32-bit offsets",
             (long long)G->n, a.d);
  int blocks = persistent_blocks(cap_chunks(G) * 32, 256, KG_AGG_BPS);
  int cblocks = persistent_blocks(cap_split_rows(G) * CB_THREADS, CB_THREADS, 8);   // one block per split row
  size_t smem = (size_t)a.G * a.B * sizeof(float);
  // narrow rows: several messages per warp load (float4 lanes, EPI groups)
  const bool al16 = ((uintptr_t)a.H & 15) == 0;
  if (a.d % 4 == 0 && a.d <= 32 && al16)
    return launch_agg<4, 1, 4>(a, persistent_blocks(cap_chunks(G) * 32, 256, AGG_NARROW_BPS), cblocks, smem, st);
  if (a.d % 4 == 0 && a.d <= 64 && al16) return launch_agg<4, 1, 2>(a, blocks, cblocks, smem, st);
  return dispatch_width(
      a.d, [&] { return launch_agg<4, 1>(a, blocks, cblocks, smem, st); },
      [&] { return launch_agg<1, 1>(a, blocks, cblocks, smem, st); },
      [&] { return launch_agg<1, 2>(a, blocks, cblocks, smem, st); },
      [&] { return launch_agg<1, 4>(a, blocks, cblocks, smem, st); },
      [&] { return launch_agg<1, 8>(a, blocks, cblocks, smem, st); });
}

static kg_status run_csc(const CscArgs& a, const kg_graph_csr* G, cudaStream_t st, int mode = 0) {
  KG_REQUIRE(G->chunk <= MAXC, KG_ERR_VALIDATION, "chunk size %d > %d", G->chunk, MAXC);
  KG_REQUIRE((int64_t)G->n * a.d < (1LL << 32), KG_ERR_SHAPE, "feature table of %lld x %d exceeds 32-bit offsets",
             (long long)G->n, a.d);
  int blocks = persistent_blocks(cap_chunks(G) * 32, 256, KG_GATHER_BPS);
  int cblocks = persistent_blocks(cap_split_rows(G) * CB_THREADS, CB_THREADS, 8);   // one block per split row
  size_t smem = (size_t)a.G * a.B * sizeof(float);
  // narrow rows: the dS-only pass gathers several messages per warp load
  const bool al16 = ((uintptr_t)a.dZ & 15) == 0 && ((uintptr_t)a.Y & 15) == 0;
  if (a.d % 4 == 0 && a.d <= 32 && al16)
    return launch_csc<4, 1, 4>(a, mode == 0 ? persistent_blocks(cap_chunks(G) * 32, 256, KG_CSC_NARROW_BPS) : blocks,
                               cblocks, smem, st, mode);
  if (a.d % 4 == 0 && a.d <= 64 && al16) return launch_csc<4, 1, 2>(a, blocks, cblocks, smem, st, mode);
  return dispatch_width(
      a.d, [&] {
        return launch_csc<4, 1>(a, mode == 0 ? persistent_blocks(cap_chunks(G) * 32, 256, KG_CSC_WIDE_BPS) : blocks,
                                cblocks, smem, st, mode);
      },
      [&] { return launch_csc<1, 1>(a, blocks, cblocks, smem, st, mode); },
      [&] { return launch_csc<1, 2>(a, blocks, cblocks, smem, st, mode); },
      [&] { return launch_csc<1, 4>(a, blocks, cblocks, smem, st, mode); },
      [&] { return launch_csc<1, 8>(a, blocks, cblocks, smem, st, mode); });
}

struct LayerWs {
  float* acc;     // forward (n, B*d_in) as packed GEMM records
  float* partial; // (split chunks, B*max(d_in, d_out))
  float* Wy;      // (d_in, B*d_out)
  float* Wb;      // (B*d_out, d_in)
  float* dZ;      // (n, d_out)
  float* Y;       // (n, B*d_out)
  float* dS;      // (n, B*d_out)
  float* dS_pk;   // dS as packed GEMM A records
  float* ed;      // (e, B)
  float* ed_self; // (n, B)
  float* Rm;      // (d_in, B*d_out)
  float* dc_part; // (G, DC_SPLIT, B) d-coeff slice partials
  char* gemm;     // packed GEMM operands (main-stream GEMMs run back to back)
  char* gemm_tn;  // packed operands + split-K partials of dV (may run on the side stream)
};

static size_t layer_ws(int64_t n, int64_t e, int64_t split_chunks, int di, int dO, int B, int R, LayerWs* w,
                       void* base, size_t cap) {
  const int64_t G = 2 * (int64_t)R + 1;
  Arena a(base, cap);
  LayerWs l;
  l.acc = a.take<float>(packed_bytes(n, (int64_t)B * di) / sizeof(float));
  l.partial = a.take<float>((size_t)split_chunks * B * (di > dO ? di : dO));
  l.Wy = a.take<float>((size_t)B * di * dO);
  l.Wb = a.take<float>((size_t)B * di * dO);
  l.dZ = a.take<float>((size_t)n * dO);
  l.Y = a.take<float>((size_t)n * B * dO);
  l.dS = a.take<float>((size_t)n * B * dO);
  l.dS_pk = a.take<float>(packed_bytes(n, (int64_t)B * dO) / sizeof(float));
  l.ed = a.take<float>((size_t)e * B);
  l.ed_self = a.take<float>((size_t)n * B);
  l.Rm = a.take<float>((size_t)di * B * dO);
  l.dc_part = a.take<float>((size_t)G * DC_SPLIT * B);
  size_t gw = 0;
  const size_t nn[3] = {gemm_nn_workspace(n, (int64_t)B * di, dO), gemm_nn_workspace(n, di, (int64_t)B * dO),
                        gemm_nn_workspace(n, (int64_t)B * dO, di)};
  for (size_t x : nn) gw = x > gw ? x : gw;
  l.gemm = a.take<char>(gw);
  l.gemm_tn = a.take<char>(gemm_tn_workspace(n, di, (int64_t)B * dO));
  if (w) *w = l;
  return a.used + 256;
}

// fork point main -> side stream (record + wait are capture-safe; one event is
// enough since each wait binds to the most recent record)
static cudaEvent_t fork_event() {
  static cudaEvent_t ev = nullptr;
  if (!ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  return ev;
}

// Producers write packed GEMM records directly. A record carries fp32 in the
// 64-byte-swizzle layout, so a producer's row piece is whole sectors and costs
// the same bytes as a row-major row: k_aggregate (whose only output is the GEMM
// operand) and the dS pass (which also keeps dS row-major for the dV GEMM)
// save the pack pass (wikikg2 scale: 42.2 -> 40.7 ms/round). Setting
// KG_DIRECT_PACK_MAX_MB restores the size limit (row-major output + a pack
// pass past it; tests exercise both paths).
static bool direct_pack(int64_t rows, int64_t K) {
  const char* env = getenv("KG_DIRECT_PACK_MAX_MB");
  if (!env) return true;
  return packed_bytes(rows, K) <= ((size_t)atoll(env) << 20);
}

// dZ footprint (bytes) up to which the CSC backward runs as two concurrent
// passes (dS on the critical stream, edge dots on the side stream). Default 0:
// always one fused pass. The split once won at FB shape (L2-resident dZ), but
// the round is throughput-bound across streams (the kernels' summed in-graph
// time is ~1.9x the round), so gathering dZ twice costs more than the
// critical pass saves: fused 0.477 vs split 0.483 ms per round (alternating
// A/B, gpurun_out r3zg). KG_CSC_SPLIT_MAX_MB=48 restores the split.
static int64_t csc_split_max_bytes() {
  const char* env = getenv("KG_CSC_SPLIT_MAX_MB");
  return (int64_t)(env ? atoll(env) : 0) << 20;
}

static Chunks csr_chunks(const kg_graph_csr* G) {
  return Chunks{G->ck_ptr, G->ck_row, G->ck_slot, G->ck_split, G->ck_counts, G->chunk,
                reinterpret_cast<const int4*>(G->ck_desc)};
}
static Chunks csc_chunks(const kg_graph_csr* G) {
  return Chunks{G->cc_ptr, G->cc_row, G->cc_slot, G->cc_split, G->cc_counts, G->chunk,
                reinterpret_cast<const int4*>(G->cc_desc)};
}

}  // namespace kg

namespace kg {
// Y = X[A_{t+1}] . [V_0 | .. | V_{B-1}], rows by closure position
static kg_status y_gemm(const kg_graph_csr* G, const kg_layer_params* lp, const float* H_in,
                        const float* H_in_packed, const float* Wy, const int32_t* order, const int32_t* counts,
                        int32_t t, float* Y, void* gemm_ws, cudaStream_t st) {
  const int B = lp->B, di = lp->d_in, dO = lp->d_out;
  GemmArgs gy{};
  gy.A = H_in; gy.lda = di; gy.a_rows = order;
  gy.a_packed = H_in_packed;
  gy.B = Wy; gy.ldb = (int64_t)B * dO;
  gy.C = Y; gy.ldc = (int64_t)B * dO;
  gy.M_dev = counts; gy.M_dev_index = t + 1; gy.M_max = G->n;
  gy.K = di; gy.N = (int64_t)B * dO;
  if (lp->packed) gy.b_packed = lp->packed + weights_layout(di, dO, B).off[1];
  return gemm_nn(gy, gemm_ws, st);
}
}  // namespace kg

using namespace kg;

extern "C" {

kg_status kg_rgcn_backward_y(const kg_graph_csr* G, const kg_layer_params* lp, const float* H_in,
                             const float* H_in_packed, const int32_t* order, const int32_t* counts, int32_t t,
                             void* ws, int64_t ws_bytes, void* stream) {
  KG_REQUIRE(lp->packed != nullptr, KG_ERR_VALIDATION, "kg_rgcn_backward_y needs packed weights");
  LayerWs w;
  size_t need = layer_ws(G->n, G->e, cap_split_chunks(G), lp->d_in, lp->d_out, lp->B, G->R, &w, ws,
                         (size_t)ws_bytes);
  KG_REQUIRE((size_t)ws_bytes >= need, KG_ERR_VALIDATION, "layer workspace too small");
  // gemm_tn is the side-stream region (the forward of the same layer may be
  // using w.gemm concurrently)
  return y_gemm(G, lp, H_in, H_in_packed, nullptr, order, counts, t, w.Y, w.gemm_tn, as_stream(stream));
}

int64_t kg_layer_workspace_bytes(const kg_graph_csr* G, int32_t d_in, int32_t d_out, int32_t B) {
  return (int64_t)layer_ws(G->n, G->e, cap_split_chunks(G), d_in, d_out, B, G->R, nullptr, nullptr, 0);
}

kg_status kg_rgcn_forward(const kg_graph_csr* G, const kg_layer_params* lp, const float* H_in, float* H_out,
                          const int32_t* order, const int32_t* pos, const int32_t* counts, int32_t t, int32_t relu,
                          const float* dropout_mask, float* H_out_packed, void* ws, int64_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(lp->B >= 1 && lp->B <= MAXB, KG_ERR_VALIDATION, "num_bases must be in [1, %d]", MAXB);
  KG_REQUIRE(lp->G == 2 * G->R + 1, KG_ERR_SHAPE, "coeff groups %d != 2R+1", lp->G);
  LayerWs w;
  size_t need = layer_ws(G->n, G->e, cap_split_chunks(G), lp->d_in, lp->d_out, lp->B, G->R, &w, ws,
                         (size_t)ws_bytes);
  KG_REQUIRE((size_t)ws_bytes >= need, KG_ERR_VALIDATION, "layer workspace too small");
  AggArgs a{G->indptr, G->src, G->rel, G->norm, csr_chunks(G), lp->coeffs, lp->G, lp->B, lp->d_in, H_in, pos,
            counts, t, w.acc, direct_pack(G->n, (int64_t)lp->B * lp->d_in) ? packed_nk(G->n, (int64_t)lp->B * lp->d_in) : 0,
            w.partial};
  kg_status s = run_aggregate(a, G, st);
  if (s != KG_OK) return s;
  GemmArgs g{};
  if (a.acc_nk) g.a_packed = w.acc;
  else g.A = w.acc;
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
  if (lp->packed) g.b_packed = lp->packed + weights_layout(lp->d_in, lp->d_out, lp->B).off[0];
  g.c_packed = H_out_packed;   // next layer's backward Y = H . [V_b] operand, by position
  g.mul = dropout_mask;        // by position, (counts[t], d_out)
  return gemm_nn(g, w.gemm, st);
}

kg_status kg_csc_positions(const kg_graph_csr* G, const int32_t* pos, int32_t* c_pos, void* stream) {
  if (G->e == 0) return KG_OK;
  KG_LAUNCH("k_csc_positions", k_csc_positions, persistent_blocks(G->e, 256, 8), 256, 0, as_stream(stream), G->c_dst,
            G->e, pos, c_pos);
  return KG_OK;
}

kg_status kg_rgcn_backward(const kg_graph_csr* G, const kg_layer_params* lp, const float* H_in, const float* H_out,
                           const float* dH_out, float* dH_in, const int32_t* order, const int32_t* pos,
                           const int32_t* c_pos, const int32_t* counts, int32_t t, float* d_bases, float* d_coeffs,
                           const float* H_in_packed, const float* dropout_mask, int32_t y_ready, void* ws,
                           int64_t ws_bytes, void* stream, void* side_stream) {
  cudaStream_t st = as_stream(stream);
  const int B = lp->B, di = lp->d_in, dO = lp->d_out;
  KG_REQUIRE(B >= 1 && B <= MAXB, KG_ERR_VALIDATION, "num_bases must be in [1, %d]", MAXB);
  LayerWs w;
  size_t need = layer_ws(G->n, G->e, cap_split_chunks(G), di, dO, B, G->R, &w, ws, (size_t)ws_bytes);
  KG_REQUIRE((size_t)ws_bytes >= need, KG_ERR_VALIDATION, "layer workspace too small");
  const int64_t wn = (int64_t)B * di * dO;
  const WeightsLayout wl = weights_layout(di, dO, B);
  if (!lp->packed)
    KG_LAUNCH("k_weight_views", k_weight_views, persistent_blocks(wn, 256, 2), 256, 0, st, lp->bases, B, di, dO, w.Wy,
              w.Wb);
  if (dO % 4 == 0)
    KG_LAUNCH("k_dz", k_dz<true>, persistent_blocks((int64_t)G->n * 32, 256, 8), 256, 0, st, dH_out, H_out, order,
              counts, t, dO, dropout_mask, w.dZ);
  else
    KG_LAUNCH("k_dz", k_dz<false>, persistent_blocks((int64_t)G->n * 32, 256, 8), 256, 0, st, dH_out, H_out, order,
              counts, t, dO, dropout_mask, w.dZ);
  // Y = X[A_{t+1}] . [V_0 | .. | V_{B-1}]  (unless kg_rgcn_backward_y made it)
  kg_status s = KG_OK;
  if (!y_ready) {
    s = y_gemm(G, lp, H_in, H_in_packed, w.Wy, order, counts, t, w.Y, w.gemm, st);
    if (s != KG_OK) return s;
  }
  CscArgs c{G->c_indptr, G->c_dst, G->c_rel, G->c_norm, csc_chunks(G), lp->coeffs, lp->G, B, dO, w.Y, w.dZ, pos,
            c_pos, counts, t, w.dS, w.ed, w.ed_self, w.partial,
            direct_pack(G->n, (int64_t)B * dO) ? w.dS_pk : nullptr, packed_nk(G->n, (int64_t)B * dO), 1};
  // (past L2, where the transposing pack pass and the row-major dS cost HBM
  // traffic; L2-resident operands keep the split-record pack + TN path, whose
  // wider grid finishes sooner on the side stream)
  const bool records_tn = H_in_packed != nullptr && c.dS_pk != nullptr && di <= 128 && B * dO <= 256 &&
                          (!records_split(G->n) || getenv("KG_TN_RECORDS")) && !getenv("KG_TN_ROWMAJOR");
  if (records_tn) c.dS = nullptr;   // nothing reads row-major dS then
  // The parameter gradients (dV, d coeffs) feed only the optimizer: with a side
  // stream they leave the critical path (the caller joins it before the update).
  // There the CSC pass splits: dS on `st`, the edge/self dots (d coeffs) on the
  // side stream concurrently; dV follows dS on the side stream.
  cudaStream_t sd = st;
  const int split = dcoeff_split(G->e, lp->G);
  // Split passes only while dZ stays L2-resident: past that, the second pass
  // would re-read every gathered dZ row from HBM, so one fused pass (MODE 0)
  // runs on `st` and only the reductions move to the side stream.
  const bool fuse = (int64_t)G->n * dO * 4 > csc_split_max_bytes();
  if (side_stream && fuse) {
    sd = as_stream(side_stream);
    s = run_csc(c, G, st, 0);
    if (s != KG_OK) return s;
    KG_CUDA(cudaEventRecord(fork_event(), st));
    KG_CUDA(cudaStreamWaitEvent(sd, fork_event(), 0));
    KG_LAUNCH("k_dcoeff_reduce", k_dcoeff_partial, dim3((unsigned)lp->G, (unsigned)split, 1), 256, 0, sd,
              G->rel_ptr, G->rel_perm, counts, t, w.ed, w.ed_self, lp->G, B, w.dc_part);
    KG_LAUNCH("k_dcoeff_final", k_dcoeff_final, persistent_blocks((int64_t)lp->G * B, 256, 2), 256, 0, sd,
              w.dc_part, lp->G, B, split, d_coeffs);
  } else if (side_stream) {
    sd = as_stream(side_stream);
    KG_CUDA(cudaEventRecord(fork_event(), st));
    KG_CUDA(cudaStreamWaitEvent(sd, fork_event(), 0));
    s = run_csc(c, G, sd, 2);
    if (s != KG_OK) return s;
    KG_LAUNCH("k_dcoeff_reduce", k_dcoeff_partial, dim3((unsigned)lp->G, (unsigned)split, 1), 256, 0, sd,
              G->rel_ptr, G->rel_perm, counts, t, w.ed, w.ed_self, lp->G, B, w.dc_part);
    KG_LAUNCH("k_dcoeff_final", k_dcoeff_final, persistent_blocks((int64_t)lp->G * B, 256, 2), 256, 0, sd,
              w.dc_part, lp->G, B, split, d_coeffs);
    s = run_csc(c, G, st, 1);
    if (s != KG_OK) return s;
    KG_CUDA(cudaEventRecord(fork_event(), st));
    KG_CUDA(cudaStreamWaitEvent(sd, fork_event(), 0));
  } else {
    s = run_csc(c, G, st, 0);
    if (s != KG_OK) return s;
  }
  // dV = X^T dS  (reduction over the source rows): straight from the X and
  // dS operand records when both exist (MN-major operands, no transposing
  // pack, no row-major dS), else from row-major X / dS
  if (records_tn) {
    s = umma_gemm_tn_records(H_in_packed, di, c.dS_pk, (int64_t)B * dO, counts, t + 1, G->n, w.Rm, w.gemm_tn, sd);
  } else {
    GemmArgs gv{};
    gv.A = H_in; gv.lda = di; gv.a_rows = order;
    gv.B = w.dS; gv.ldb = (int64_t)B * dO;
    gv.M_dev = counts; gv.M_dev_index = t + 1; gv.M_max = G->n;
    gv.K = di; gv.N = (int64_t)B * dO;
    s = gemm_tn(gv, w.Rm, w.gemm_tn, sd);
  }
  if (s != KG_OK) return s;
  KG_LAUNCH("k_dbases_layout", k_dbases_layout, persistent_blocks(wn, 256, 2), 256, 0, sd, w.Rm, B, di, dO, d_bases);
  if (!side_stream) {
    KG_LAUNCH("k_dcoeff_reduce", k_dcoeff_partial, dim3((unsigned)lp->G, (unsigned)split, 1), 256, 0, sd,
              G->rel_ptr, G->rel_perm, counts, t, w.ed, w.ed_self, lp->G, B, w.dc_part);
    KG_LAUNCH("k_dcoeff_final", k_dcoeff_final, persistent_blocks((int64_t)lp->G * B, 256, 2), 256, 0, sd,
              w.dc_part, lp->G, B, split, d_coeffs);
  }
  if (dH_in) {
    GemmArgs gx{};
    gx.A = w.dS; gx.lda = (int64_t)B * dO;
    gx.a_packed = c.dS_pk;   // nullptr: the GEMM packs dS itself
    gx.B = w.Wb; gx.ldb = di;
    gx.C = dH_in; gx.ldc = di; gx.c_rows = order;
    gx.M_dev = counts; gx.M_dev_index = t + 1; gx.M_max = G->n;
    gx.K = (int64_t)B * dO; gx.N = di;
    if (lp->packed) gx.b_packed = lp->packed + wl.off[2];
    s = gemm_nn(gx, w.gemm, st);
    if (s != KG_OK) return s;
  }
  return KG_OK;
}

int64_t kg_rgcn_weights_bytes(int32_t d_in, int32_t d_out, int32_t B) {
  return weights_layout(d_in, d_out, B).total * (int64_t)sizeof(float);
}

kg_status kg_rgcn_pack_weights(const kg_layer_params* lp, float* out, void* stream) {
  KG_REQUIRE(lp->B >= 1 && lp->B <= MAXB, KG_ERR_VALIDATION, "num_bases must be in [1, %d]", MAXB);
  KG_REQUIRE(lp->d_out <= 256 && (int64_t)lp->B * lp->d_out <= 256 && lp->d_in <= 256, KG_ERR_SHAPE,
             "packed weights need d_in, d_out, B*d_out <= 256");
  const WeightsLayout L = weights_layout(lp->d_in, lp->d_out, lp->B);
  int64_t most = 0;
  for (int j = 0; j < 3; ++j) most = L.rows[j] * L.nk[j] * PK_K > most ? L.rows[j] * L.nk[j] * PK_K : most;
  dim3 grid((unsigned)persistent_blocks(most, 256, 2), 3, 1);
  KG_LAUNCH("k_pack_weights", k_pack_weights, grid, 256, 0, as_stream(stream), lp->bases, lp->B, lp->d_in, lp->d_out,
            L, out);
  return KG_OK;
}

}  // extern "C"

// this module's anchor for kg_preload_kernels (kg_primitives.cu)
extern "C" const void* kg_anchor_rgcn() { return reinterpret_cast<const void*>(&kg::k_csc_positions); }
