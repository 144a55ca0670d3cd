// R16-R18: DistMult scoring fused with the BCE loss and its gradient
// (ref:model.py:238-281).
//
//   g_i   = sum_k H[h_i,k] m[r_i,k] H[t_i,k]
//   loss  = mean(softplus(g) - y g)          (deterministic two-level sum)
//   dg_i  = (sigmoid(g_i) - y_i) / b
//   d m_r = sum_{i: r_i = r} dg_i H[h_i] * H[t_i]
//   dH_v  = sum_{i: h_i = v} dg_i m_{r_i} * H[t_i] + sum_{i: t_i = v} dg_i m_{r_i} * H[h_i]
//
// The two scatters are done without atomics: the batch's relation ids and
// endpoint ids are stable-radix-sorted once, every group is cut into
// sub-chunks of CH_REL / CH_ENT rows summed by one warp each, and a second pass adds the
// sub-chunk partials of a group in order (hub rows get many warps, fixed
// summation order -> bitwise reproducible).
#include "kg_common.cuh"

namespace kg {

// rows per sub-chunk: relation groups (the d_decoder scatter: few, large
// groups) use short sub-chunks for parallelism, endpoint groups (dH) longer ones
#ifndef KG_CH_REL
#define KG_CH_REL 16
#endif
constexpr int CH_REL = KG_CH_REL, CH_ENT = 64;

struct LossArgs {
  const float* H;
  int d;
  const float* dec;
  const int32_t* tri;
  const float* labels;
  int64_t total, start, b;
  const int64_t* start_dev;   // when set, the batch offset is read on the device (graph replay)
  float* dg;
  float* per;
  float* scores;
  uint32_t* flags;
};

__device__ __forceinline__ int64_t row_of(const LossArgs& a, int64_t i) {
  // the batch offset is < total, so only wrapped rows pay for the 64-bit modulo
  int64_t r = (a.start_dev ? __ldg(a.start_dev) : a.start) + i;
  if (r >= a.total) r %= a.total;
  return r;
}

// SU triples per warp iteration: their row loads are all in flight together,
// and lane u finishes triple u (softplus, sigmoid) so the epilogues overlap.
constexpr int SU = 4;

template <bool V4>
__global__ void __launch_bounds__(256) k_score(LossArgs a) {
  const int lane = lane_id();
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int64_t i0 = warp_uniform(((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * SU); i0 < a.b;
       i0 += (int64_t)warps * SU) {
    float s[SU];
    int64_t rows[SU];
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      s[u] = 0.f;
      rows[u] = i0 + u < a.b ? row_of(a, i0 + u) : -1;
    }
    if (V4) {
      for (int k = 4 * lane; k < a.d; k += 128) {
        float x[SU][4], m[SU][4], y[SU][4];
#pragma unroll
        for (int u = 0; u < SU; ++u) {
          if (rows[u] >= 0) {
            const int32_t* tr = a.tri + rows[u] * 3;
            VecIO<4>::load(a.H + (int64_t)__ldg(tr) * a.d + k, x[u]);
            VecIO<4>::load(a.dec + (int64_t)__ldg(tr + 1) * a.d + k, m[u]);
            VecIO<4>::load(a.H + (int64_t)__ldg(tr + 2) * a.d + k, y[u]);
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) x[u][c] = m[u][c] = y[u][c] = 0.f;
          }
        }
#pragma unroll
        for (int u = 0; u < SU; ++u)
#pragma unroll
          for (int c = 0; c < 4; ++c) s[u] = fmaf(x[u][c] * m[u][c], y[u][c], s[u]);
      }
    } else {
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        if (rows[u] < 0) continue;
        const int32_t* tr = a.tri + rows[u] * 3;
        const float* Hh = a.H + (int64_t)__ldg(tr) * a.d;
        const float* M = a.dec + (int64_t)__ldg(tr + 1) * a.d;
        const float* Ht = a.H + (int64_t)__ldg(tr + 2) * a.d;
        for (int k = lane; k < a.d; k += 32) s[u] = fmaf(Hh[k] * M[k], Ht[k], s[u]);
      }
    }
    float mine = 0.f;
    int64_t row = -1;
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      const float t = warp_sum(s[u]);
      if (lane == u) {
        mine = t;
        row = rows[u];
      }
    }
    if (lane < SU && row >= 0) {
      const int64_t i = i0 + lane;
      const float sc = mine;
      const float y = a.labels[row];
      if (!isfinite(sc)) atomicOr(a.flags, KG_FLAG_NONFINITE_SCORE);
      const float sp = fmaxf(sc, 0.f) + log1pf(expf(-fabsf(sc)));   // softplus = logaddexp(0, g)
      a.per[i] = sp - y * sc;
      const float sig = 1.f / (1.f + expf(-sc));
      a.dg[i] = (sig - y) / (float)a.b;
      if (a.scores) a.scores[i] = sc;
    }
  }
}

// deterministic mean: per-block partial (fixed order), then single-block final
__global__ void k_block_sums(const float* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) s += x[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_final_mean(const double* __restrict__ part, int nb, int64_t n, float* __restrict__ out,
                             uint32_t* __restrict__ flags) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double m = red[0] / (double)n;
    *out = (float)m;
    if (!isfinite(m)) atomicOr(flags, KG_FLAG_NONFINITE_LOSS);
  }
}

// sort keys: relation ids (b) and endpoint ids (2b, occurrence o<b head, o>=b tail)
__global__ void k_loss_keys(LossArgs a, uint32_t* __restrict__ rk, uint32_t* __restrict__ rv,
                            uint32_t* __restrict__ vk, uint32_t* __restrict__ vv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.b; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = row_of(a, i);
    rk[i] = (uint32_t)a.tri[row * 3 + 1];
    rv[i] = (uint32_t)i;
    vk[i] = (uint32_t)a.tri[row * 3];
    vv[i] = (uint32_t)i;
    vk[a.b + i] = (uint32_t)a.tri[row * 3 + 2];
    vv[a.b + i] = (uint32_t)(a.b + i);
  }
}

__device__ __forceinline__ int64_t lower_bound_u32(const uint32_t* __restrict__ k, int64_t n, uint32_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (k[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// group g has key gkey(g) = ids ? ids[g] : g ; bounds into the sorted keys
__global__ void k_group_bounds(const uint32_t* __restrict__ keys, int64_t n, const int32_t* __restrict__ ids,
                               const int32_t* __restrict__ ng_dev, int32_t ng_host, int32_t* __restrict__ lo,
                               uint32_t* __restrict__ nsub, int ch) {
  const int32_t ng = ng_dev ? *ng_dev : ng_host;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x) {
    uint32_t key = ids ? (uint32_t)ids[g] : (uint32_t)g;
    int64_t a = lower_bound_u32(keys, n, key);
    int64_t e = lower_bound_u32(keys, n, key + 1);
    lo[g] = (int32_t)a;
    nsub[g] = (uint32_t)((e - a + ch - 1) / ch);
  }
}

__global__ void k_group_len(const uint32_t* __restrict__ keys, int64_t n, const int32_t* __restrict__ ids,
                            const int32_t* __restrict__ ng_dev, int32_t ng_host, int32_t* __restrict__ hi) {
  const int32_t ng = ng_dev ? *ng_dev : ng_host;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x) {
    uint32_t key = ids ? (uint32_t)ids[g] : (uint32_t)g;
    hi[g] = (int32_t)lower_bound_u32(keys, n, key + 1);
  }
}

// kind 0: d_dec rows (value = triple index); kind 1: dH rows (value = occurrence)
template <int KIND, int SL>
__global__ void __launch_bounds__(256) k_sub_partials(LossArgs a, const uint32_t* __restrict__ vals,
                                                      const int32_t* __restrict__ lo, const int32_t* __restrict__ hi,
                                                      const uint32_t* __restrict__ sub_start,
                                                      const uint32_t* __restrict__ total_sub,
                                                      const uint32_t* __restrict__ sgroup,
                                                      float* __restrict__ partial, int ch) {
  const uint32_t S = *total_sub;
  const int lane = lane_id();
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); s < S; s += warps) {
    const int32_t g = (int32_t)__ldg(sgroup + s);   // owning group (precomputed with the bounds)
    const int64_t r0 = lo[g] + (int64_t)(s - sub_start[g]) * ch;
    const int64_t r1 = r0 + ch < hi[g] ? r0 + ch : hi[g];
    float acc[SL];
#pragma unroll
    for (int q = 0; q < SL; ++q) acc[q] = 0.f;
    for (int64_t base = r0; base < r1; base += 32) {
      const int cnt = (int)min((int64_t)32, r1 - base);
      // lane i fetches the metadata of row base+i: (row A, row B, dg)
      int32_t ra = 0, rb = 0;
      float my_dg = 0.f;
      if (lane < cnt) {
        uint32_t v = vals[base + lane];
        int64_t ti = (KIND == 1 && v >= a.b) ? v - a.b : v;
        int64_t row = row_of(a, ti);
        int32_t hh = a.tri[row * 3], rr = a.tri[row * 3 + 1], tt = a.tri[row * 3 + 2];
        my_dg = a.dg[ti];
        if (KIND == 0) {            // d m_r += dg * H[h] * H[t]
          ra = hh;
          rb = tt;
        } else {                    // dH_v += dg * m_r * H[other]
          ra = -1 - rr;             // decoder row, tagged negative
          rb = (v >= a.b) ? hh : tt;
        }
      }
      for (int j = 0; j < cnt; j += 4) {
        float xa[4][SL], xb[4][SL], w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          int32_t A = __shfl_sync(0xffffffffu, ra, (j + u) & 31);
          int32_t Bv = __shfl_sync(0xffffffffu, rb, (j + u) & 31);
          w[u] = __shfl_sync(0xffffffffu, my_dg, (j + u) & 31);
          const float* pa = (KIND == 0) ? a.H + (int64_t)A * a.d : a.dec + (int64_t)(-1 - A) * a.d;
          const float* pb = a.H + (int64_t)Bv * a.d;
#pragma unroll
          for (int q = 0; q < SL; ++q) {
            int k = q * 32 + lane;
            bool ok = (j + u < cnt) && k < a.d;
            xa[u][q] = ok ? __ldg(pa + k) : 0.f;
            xb[u][q] = ok ? __ldg(pb + k) : 0.f;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int q = 0; q < SL; ++q) acc[q] = fmaf(w[u], xa[u][q] * xb[u][q], acc[q]);
      }
    }
    float* out = partial + s * (int64_t)a.d;
#pragma unroll
    for (int q = 0; q < SL; ++q) {
      int k = q * 32 + lane;
      if (k < a.d) out[k] = acc[q];
    }
  }
}

// float4 lanes (d % 4 == 0, d <= 128): lane l owns features 4l..4l+3; 8 rows
// of each operand in flight per lane.
template <int KIND>
__global__ void __launch_bounds__(256) k_sub_partials_v4(LossArgs a, const uint32_t* __restrict__ vals,
                                                         const int32_t* __restrict__ lo,
                                                         const int32_t* __restrict__ hi,
                                                         const uint32_t* __restrict__ sub_start,
                                                         const uint32_t* __restrict__ total_sub,
                                                         const uint32_t* __restrict__ sgroup,
                                                         float* __restrict__ partial, int ch) {
  const uint32_t S = *total_sub;
  const int lane = lane_id();
  const bool on = 4 * lane < a.d;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); s < S; s += warps) {
    const int32_t g = (int32_t)__ldg(sgroup + s);   // owning group (precomputed with the bounds)
    const int64_t r0 = lo[g] + (int64_t)(s - sub_start[g]) * ch;
    const int64_t r1 = r0 + ch < hi[g] ? r0 + ch : hi[g];
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int64_t base = r0; base < r1; base += 32) {
      const int cnt = (int)min((int64_t)32, r1 - base);
      int32_t ra = 0, rb = 0;
      float my_dg = 0.f;
      if (lane < cnt) {
        uint32_t v = vals[base + lane];
        int64_t ti = (KIND == 1 && v >= a.b) ? v - a.b : v;
        int64_t row = row_of(a, ti);
        int32_t hh = a.tri[row * 3], rr = a.tri[row * 3 + 1], tt = a.tri[row * 3 + 2];
        my_dg = a.dg[ti];
        if (KIND == 0) {
          ra = hh;
          rb = tt;
        } else {
          ra = -1 - rr;
          rb = (v >= a.b) ? hh : tt;
        }
      }
      for (int j = 0; j < cnt; j += 8) {
        float xa[8][4], xb[8][4], w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int32_t A = __shfl_sync(0xffffffffu, ra, (j + u) & 31);
          const int32_t Bv = __shfl_sync(0xffffffffu, rb, (j + u) & 31);
          w[u] = __shfl_sync(0xffffffffu, my_dg, (j + u) & 31);
          const float* pa = (KIND == 0) ? a.H + (int64_t)A * a.d : a.dec + (int64_t)(-1 - A) * a.d;
          const float* pb = a.H + (int64_t)Bv * a.d;
          if (on && j + u < cnt) {
            VecIO<4>::load(pa + 4 * lane, xa[u]);
            VecIO<4>::load(pb + 4 * lane, xb[u]);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) xa[u][i] = xb[u][i] = 0.f;
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[i] = fmaf(w[u], xa[u][i] * xb[u][i], acc[i]);
      }
    }
    if (on) VecIO<4>::store(partial + s * (int64_t)a.d + 4 * lane, acc);
  }
}

__global__ void k_group_finish(const float* __restrict__ partial, const uint32_t* __restrict__ sub_start,
                               const uint32_t* __restrict__ nsub, const int32_t* __restrict__ ids,
                               const int32_t* __restrict__ ng_dev, int32_t ng_host, int d, float* __restrict__ out) {
  const int32_t ng = ng_dev ? *ng_dev : ng_host;
  const int64_t total = (int64_t)ng * d;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    int64_t g = x / d;
    int k = (int)(x - g * d);
    float s = 0.f;
    uint32_t a0 = sub_start[g], n0 = nsub[g];
    for (uint32_t j = 0; j < n0; ++j) s += partial[(int64_t)(a0 + j) * d + k];
    int64_t row = ids ? ids[g] : g;
    out[row * d + k] = s;
  }
}

__global__ void k_sub_groups(const uint32_t* __restrict__ nsub, const uint32_t* __restrict__ sub_start,
                             const int32_t* __restrict__ ng_dev, int32_t ng_host, uint32_t* __restrict__ sgroup) {
  const int32_t ng = ng_dev ? *ng_dev : ng_host;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t a0 = sub_start[g], n0 = nsub[g];
    for (uint32_t j = 0; j < n0; ++j) sgroup[a0 + j] = (uint32_t)g;
  }
}

struct SegWs {
  int32_t* lo;
  int32_t* hi;
  uint32_t* nsub;
  uint32_t* sub_start;
  uint32_t* total;
  uint32_t* sgroup;   // group of every sub-chunk
  float* partial;
  char* scan;
  int ch;             // rows per sub-chunk
};

static size_t seg_ws(int64_t nelem, int64_t ngroups, int d, int ch, SegWs* w, Arena& a) {
  SegWs s;
  s.ch = ch;
  s.lo = a.take<int32_t>(ngroups + 1);
  s.hi = a.take<int32_t>(ngroups + 1);
  s.nsub = a.take<uint32_t>(ngroups + 1);
  s.sub_start = a.take<uint32_t>(ngroups + 1);
  s.total = a.take<uint32_t>(4);
  s.sgroup = a.take<uint32_t>((size_t)(nelem / ch + ngroups + 1));
  s.partial = a.take<float>((size_t)(nelem / ch + ngroups + 1) * d);
  s.scan = a.take<char>(scan_workspace(ngroups + 1));
  if (w) *w = s;
  return a.used;
}

static kg_status seg_bounds(const uint32_t* keys, int64_t nelem, const int32_t* ids, const int32_t* ng_dev,
                            int32_t ng_max, SegWs& w, cudaStream_t st) {
  int gb = persistent_blocks(ng_max, 256, 8);
  KG_LAUNCH("k_group_bounds", k_group_bounds, gb, 256, 0, st, keys, nelem, ids, ng_dev, ng_max, w.lo, w.nsub, w.ch);
  KG_LAUNCH("k_group_len", k_group_len, gb, 256, 0, st, keys, nelem, ids, ng_dev, ng_max, w.hi);
  // with a device-resident group count the caller zeroed nsub[0:ng_max] so the
  // scan sees 0 beyond *ng_dev
  kg_status s = exclusive_scan_u32(w.nsub, w.sub_start, ng_max, w.total, w.scan, scan_workspace(ng_max + 1), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_sub_groups", k_sub_groups, gb, 256, 0, st, w.nsub, w.sub_start, ng_dev, ng_max, w.sgroup);
  return KG_OK;
}

template <int KIND>
static kg_status seg_sums(const LossArgs& la, const uint32_t* vals, int64_t nelem, const int32_t* ids,
                          const int32_t* ng_dev, int32_t ng_max, float* out, SegWs& w, cudaStream_t st) {
  int64_t max_sub = nelem / w.ch + ng_max + 1;
  int pb = persistent_blocks(max_sub * 32, 256, 8);
  const bool v4 = la.d % 4 == 0 && la.d <= 128 && (((uintptr_t)la.H | (uintptr_t)la.dec) & 15) == 0;
  if (v4) KG_LAUNCH("k_sub_partials", (k_sub_partials_v4<KIND>), pb, 256, 0, st, la, vals, w.lo, w.hi, w.sub_start, w.total, w.sgroup, w.partial, w.ch);
  else if (la.d <= 32) KG_LAUNCH("k_sub_partials", (k_sub_partials<KIND, 1>), pb, 256, 0, st, la, vals, w.lo, w.hi, w.sub_start, w.total, w.sgroup, w.partial, w.ch);
  else if (la.d <= 64) KG_LAUNCH("k_sub_partials", (k_sub_partials<KIND, 2>), pb, 256, 0, st, la, vals, w.lo, w.hi, w.sub_start, w.total, w.sgroup, w.partial, w.ch);
  else if (la.d <= 128) KG_LAUNCH("k_sub_partials", (k_sub_partials<KIND, 4>), pb, 256, 0, st, la, vals, w.lo, w.hi, w.sub_start, w.total, w.sgroup, w.partial, w.ch);
  else if (la.d <= 256) KG_LAUNCH("k_sub_partials", (k_sub_partials<KIND, 8>), pb, 256, 0, st, la, vals, w.lo, w.hi, w.sub_start, w.total, w.sgroup, w.partial, w.ch);
  else KG_REQUIRE(false, KG_ERR_SHAPE, "embedding width %d > 256 unsupported", la.d);
  KG_LAUNCH("k_group_finish", k_group_finish, persistent_blocks((int64_t)ng_max * la.d, 256, 8), 256, 0, st, w.partial, w.sub_start, w.nsub,
                                                                                   ids, ng_dev, ng_max, la.d, out);
  return KG_OK;
}

static int bits_for(uint64_t maxval) {
  int b = 0;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

}  // namespace kg

using namespace kg;

extern "C" {

// One arena layout shared by the grouping and the compute halves (they may run
// on different streams: the grouping touches keys/sort/segment-bound regions,
// the compute half dg/per/partials).
struct LossWs {
  float* dg;
  float* per;
  double* part;
  uint32_t *rk, *rv, *vk, *vv;
  char* sws;
  SegWs wr, wv;
  int64_t ngmax;
};

static size_t loss_arena(void* ws, size_t bytes, int64_t b, int32_t n_local, int32_t d, int32_t R, LossWs* L) {
  Arena a(ws, bytes);
  LossWs w;
  w.ngmax = 2 * b < (int64_t)n_local ? 2 * b : (int64_t)n_local;
  w.dg = a.take<float>(b);
  w.per = a.take<float>(b);
  w.part = a.take<double>(1024);
  w.rk = a.take<uint32_t>(b);
  w.rv = a.take<uint32_t>(b);
  w.vk = a.take<uint32_t>(2 * b);
  w.vv = a.take<uint32_t>(2 * b);
  w.sws = a.take<char>(sort32_workspace(2 * b));
  seg_ws(b, R, d, CH_REL, &w.wr, a);
  seg_ws(2 * b, w.ngmax, d, CH_ENT, &w.wv, a);
  if (L) *L = w;
  return a.used + 4096;
}

static kg_status loss_groups(const LossArgs& la, int32_t n_local, int32_t R, const int32_t* order,
                             const int32_t* counts, LossWs& w, cudaStream_t st) {
  const int64_t b = la.b;
  KG_LAUNCH("k_loss_keys", k_loss_keys, persistent_blocks(b, 256, 8), 256, 0, st, la, w.rk, w.rv, w.vk, w.vv);
  kg_status s = sort_pairs_u32(w.rk, w.rv, b, bits_for((uint64_t)R), w.sws, sort32_workspace(2 * b), st);
  if (s != KG_OK) return s;
  s = sort_pairs_u32(w.vk, w.vv, 2 * b, bits_for((uint64_t)n_local), w.sws, sort32_workspace(2 * b), st);
  if (s != KG_OK) return s;
  KG_CUDA(cudaMemsetAsync(w.wr.nsub, 0, (R + 1) * sizeof(uint32_t), st));
  KG_CUDA(cudaMemsetAsync(w.wv.nsub, 0, (w.ngmax + 1) * sizeof(uint32_t), st));
  s = seg_bounds(w.rk, b, nullptr, nullptr, R, w.wr, st);
  if (s != KG_OK) return s;
  // seed groups: A_0 = order[0:counts[0]] (ascending, exactly the distinct endpoints)
  return seg_bounds(w.vk, 2 * b, order, counts, (int32_t)w.ngmax, w.wv, st);
}

static cudaEvent_t loss_fork_event() {
  static cudaEvent_t ev = nullptr;
  if (!ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  return ev;
}

// With a side stream only the dH reduction (which the backward needs) stays on
// `st`; the loss mean and d_decoder (optimizer inputs) run on `side`.
static kg_status loss_compute(const LossArgs& la, int32_t R, const int32_t* order, const int32_t* counts,
                              float* dH, float* d_decoder, float* loss_out, uint32_t* flags, LossWs& w,
                              cudaStream_t st, cudaStream_t side = nullptr) {
  const int64_t b = la.b;
  const bool v4 = la.d % 4 == 0 && (((uintptr_t)la.H | (uintptr_t)la.dec) & 15) == 0;
  KG_LAUNCH("k_score", v4 ? k_score<true> : k_score<false>, persistent_blocks(ceil_div(b, SU) * 32, 256, 8), 256, 0,
            st, la);
  cudaStream_t sd = st;
  if (side) {
    sd = side;
    KG_CUDA(cudaEventRecord(loss_fork_event(), st));
    KG_CUDA(cudaStreamWaitEvent(sd, loss_fork_event(), 0));
  }
  int nb = persistent_blocks(b, 256, 4);
  if (nb > 1024) nb = 1024;
  KG_LAUNCH("k_block_sums", k_block_sums, nb, 256, 0, sd, w.per, b, w.part);
  KG_LAUNCH("k_final_mean", k_final_mean, 1, 256, 0, sd, w.part, nb, b, loss_out, flags);
  kg_status s = seg_sums<0>(la, w.rv, b, nullptr, nullptr, R, d_decoder, w.wr, sd);
  if (s != KG_OK) return s;
  return seg_sums<1>(la, w.vv, 2 * b, order, counts, (int32_t)w.ngmax, dH, w.wv, st);
}

int32_t kg_loss_group_fields(void* ws, int64_t ws_bytes, int64_t b, int32_t n_local, int32_t d, int32_t R,
                             void** ptrs, int64_t* bytes, int32_t max) {
  LossWs w;
  if (loss_arena(ws, (size_t)ws_bytes, b, n_local, d, R, &w) > (size_t)ws_bytes) return -1;
  const int64_t nr = (int64_t)R + 1, nv = w.ngmax + 1;
  const int64_t sr = b / CH_REL + R + 1, sv = 2 * b / CH_ENT + w.ngmax + 1;   // sub-chunk capacities (seg_ws)
  void* p[] = {w.rv, w.vv, w.wr.lo, w.wr.hi, w.wr.nsub, w.wr.sub_start, w.wr.total, w.wr.sgroup,
               w.wv.lo, w.wv.hi, w.wv.nsub, w.wv.sub_start, w.wv.total, w.wv.sgroup};
  const int64_t sz[] = {4 * b, 8 * b, 4 * nr, 4 * nr, 4 * nr, 4 * nr, 16, 4 * sr,
                        4 * nv, 4 * nv, 4 * nv, 4 * nv, 16, 4 * sv};
  const int32_t n = (int32_t)(sizeof(sz) / sizeof(sz[0]));
  if (n > max) return -1;
  for (int32_t i = 0; i < n; ++i) {
    ptrs[i] = p[i];
    bytes[i] = sz[i];
  }
  return n;
}

int64_t kg_loss_workspace_bytes(int64_t b, int32_t n, int32_t d, int32_t R) {
  return (int64_t)loss_arena(nullptr, 0, b, n, d, R, nullptr);
}

#define KG_LOSS_SETUP()                                                                                     \
  cudaStream_t st = as_stream(stream);                                                                      \
  KG_REQUIRE(b >= 1 && total >= 1, KG_ERR_VALIDATION, "empty batch");                                       \
  LossWs w;                                                                                                 \
  KG_REQUIRE(loss_arena(ws, (size_t)ws_bytes, b, n_local, d, R, &w) <= (size_t)ws_bytes, KG_ERR_VALIDATION, \
             "loss workspace too small");                                                                   \
  LossArgs la{H, d, decoder, tri, labels, total, start, b, start_dev, w.dg, w.per, scores_out, flags}

kg_status kg_distmult_loss(const float* H, int32_t d, int32_t n_local, const float* decoder, int32_t R,
                           const int32_t* tri,
                           const float* labels, int64_t total, int64_t start, const int64_t* start_dev, int64_t b,
                           const int32_t* order,
                           const int32_t* counts, float* dH, float* d_decoder, float* loss_out, float* scores_out,
                           uint32_t* flags, void* ws, int64_t ws_bytes, void* stream) {
  KG_LOSS_SETUP();
  kg_status s = loss_groups(la, n_local, R, order, counts, w, st);
  if (s != KG_OK) return s;
  return loss_compute(la, R, order, counts, dH, d_decoder, loss_out, flags, w, st);
}

// The batch-only half of kg_distmult_loss (sort keys, group bounds). It needs
// the closure's seed order but not H, so it can run on a second stream while
// the layers run; kg_loss_compute must follow it (same ws) on any stream.
kg_status kg_loss_groups(const float* H, int32_t d, int32_t n_local, const float* decoder, int32_t R,
                         const int32_t* tri, const float* labels, int64_t total, int64_t start,
                         const int64_t* start_dev, int64_t b, const int32_t* order, const int32_t* counts,
                         float* dH, float* d_decoder, float* loss_out, float* scores_out, uint32_t* flags, void* ws,
                         int64_t ws_bytes, void* stream) {
  KG_LOSS_SETUP();
  return loss_groups(la, n_local, R, order, counts, w, st);
}

kg_status kg_loss_compute(const float* H, int32_t d, int32_t n_local, const float* decoder, int32_t R,
                          const int32_t* tri, const float* labels, int64_t total, int64_t start,
                          const int64_t* start_dev, int64_t b, const int32_t* order, const int32_t* counts,
                          float* dH, float* d_decoder, float* loss_out, float* scores_out, uint32_t* flags,
                          void* ws, int64_t ws_bytes, void* stream, void* side_stream) {
  KG_LOSS_SETUP();
  return loss_compute(la, R, order, counts, dH, d_decoder, loss_out, flags, w, st,
                      side_stream ? as_stream(side_stream) : nullptr);
}


// The batch-only work of a whole epoch (SURVEY.md §8 R7/R8 + the loss
// grouping of R16), one host call: for every round r the closure of rows
// [r*b, (r+1)*b) into order/pos/counts row r, the loss grouping into loss_ws,
// and an export of kg_loss_group_fields into groups + r*groups_stride (fields
// at 256-byte aligned offsets, in kg_loss_group_fields order). Issued as ~25
// launches per round from C, so capturing it into an epoch graph costs
// microseconds per launch instead of a Python round trip each.
kg_status kg_epoch_prep(const kg_epoch_prep_args* a, void* stream) {
  KG_REQUIRE(a != nullptr && a->g != nullptr, KG_ERR_VALIDATION, "kg_epoch_prep: null arguments");
  KG_REQUIRE(a->rounds >= 1 && a->b >= 1 && a->hops >= 0, KG_ERR_VALIDATION, "kg_epoch_prep: bad sizes");
  const int32_t n = a->g->n, L1 = a->hops + 1;
  int K = a->branches < 1 ? 1 : a->branches;
  K = K > a->rounds ? a->rounds : K;
  K = K > KG_PREP_MAX_BRANCHES ? KG_PREP_MAX_BRANCHES : K;
  // per-branch export lists (the branch's loss workspace -> the round's slab row)
  kg_copy_seg segs[KG_PREP_MAX_BRANCHES][16];
  int32_t nf = 0;
  for (int k = 0; k < K; ++k) {
    void* ptrs[16];
    int64_t sz[16];
    char* lws = static_cast<char*>(a->loss_ws) + (int64_t)k * a->loss_ws_bytes;
    nf = kg_loss_group_fields(lws, a->loss_ws_bytes, a->b, n, a->d, a->R, ptrs, sz, 16);
    KG_REQUIRE(nf > 0, KG_ERR_VALIDATION, "kg_epoch_prep: loss workspace too small");
    int64_t off = 0;
    for (int32_t i = 0; i < nf; ++i) {
      segs[k][i].dst = a->groups + off;
      segs[k][i].src = ptrs[i];
      segs[k][i].bytes = sz[i];
      segs[k][i].dst_round_stride = a->groups_stride;
      segs[k][i].src_round_stride = 0;
      off += (int64_t)align_up((size_t)sz[i]);
    }
    KG_REQUIRE(off <= a->groups_stride, KG_ERR_VALIDATION, "kg_epoch_prep: groups stride %lld < %lld",
               (long long)a->groups_stride, (long long)off);
  }
  // rounds are independent: with K > 1 they run as K parallel branches (forked
  // from and joined back into `stream`; capture-safe), round r on branch r % K
  cudaStream_t st = as_stream(stream), br[KG_PREP_MAX_BRANCHES];
  static cudaStream_t aux[KG_PREP_MAX_BRANCHES] = {};
  static cudaEvent_t ev = nullptr;
  if (K > 1) {
    if (!ev) {
      int lo = 0, hi = 0;
      KG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      for (int k = 0; k < KG_PREP_MAX_BRANCHES; ++k)
        KG_CUDA(cudaStreamCreateWithPriority(&aux[k], cudaStreamNonBlocking, lo));   // lowest priority
      KG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    KG_CUDA(cudaEventRecord(ev, st));
    for (int k = 0; k < K; ++k) {
      KG_CUDA(cudaStreamWaitEvent(aux[k], ev, 0));
      br[k] = aux[k];
    }
  } else {
    br[0] = st;
  }
  for (int32_t r = 0; r < a->rounds; ++r) {
    const int k = r % K;
    void* bs = br[k];
    const int64_t start = (int64_t)r * a->b;
    int32_t* order = a->order + (int64_t)r * n;
    int32_t* counts = a->counts + (int64_t)r * L1;
    char* cws = static_cast<char*>(a->closure_ws) + (int64_t)k * a->closure_ws_bytes;
    char* lws = static_cast<char*>(a->loss_ws) + (int64_t)k * a->loss_ws_bytes;
    kg_status s = kg_closure(a->stream_triples, a->total, start, nullptr, a->b, nullptr, a->g, a->hops, order,
                             a->pos + (int64_t)r * n, counts, cws, a->closure_ws_bytes, bs);
    if (s != KG_OK) return s;
    s = kg_loss_groups(nullptr, a->d, n, nullptr, a->R, a->stream_triples, a->labels, a->total, start, nullptr,
                       a->b, order, counts, nullptr, nullptr, nullptr, nullptr, a->flags, lws, a->loss_ws_bytes, bs);
    if (s != KG_OK) return s;
    s = kg_copy_segments(segs[k], nf, nullptr, r, bs);
    if (s != KG_OK) return s;
  }
  if (K > 1) {
    for (int k = 0; k < K; ++k) {
      KG_CUDA(cudaEventRecord(ev, aux[k]));
      KG_CUDA(cudaStreamWaitEvent(st, ev, 0));
    }
  }
  return KG_OK;
}

}  // extern "C"

// this module's anchor for kg_preload_kernels (kg_primitives.cu)
extern "C" const void* kg_anchor_loss() { return reinterpret_cast<const void*>(&kg::k_block_sums); }
