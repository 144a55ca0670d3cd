// R19/R20: gradient reduction + optimizer (ref:trainer.py:63-151).
//
// kg_dense_step fuses the reference's pairwise-tree allreduce_mean
// (ref:trainer.py:77-86: ((g0+g1)+(g2+g3))..., odd tail carried, then / P)
// with the SGD/Adam update of the flat dense block buffer. The P payloads
// arrive already gathered on every rank (NCCL all-gather over NVLink), so
// every rank computes the identical tree in the identical order and the
// dense replicas stay bitwise equal (ref:trainer.py:465-469).
#include "kg_common.cuh"

namespace kg {

constexpr int MAXP = 64;

__device__ __forceinline__ float tree_mean_at(const float* __restrict__ g, int P, int64_t n, int64_t i) {
  float v[MAXP];
  for (int w = 0; w < P; ++w) v[w] = g[(int64_t)w * n + i];
  int cnt = P;
  while (cnt > 1) {
    int half = cnt / 2;
    for (int j = 0; j < half; ++j) v[j] = v[2 * j] + v[2 * j + 1];
    if (cnt & 1) v[half] = v[cnt - 1];
    cnt = half + (cnt & 1);
  }
  return v[0] / (float)P;
}

__global__ void k_tree_mean(const float* __restrict__ g, int P, int64_t n, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = tree_mean_at(g, P, n, i);
}

__global__ void k_sumsq_blocks(const float* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += (double)x[i] * (double)x[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_clip_scale(const double* __restrict__ part, int nb, float clip, float* __restrict__ scale) {
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
    double nrm = sqrt(red[0]);
    *scale = nrm > (double)clip ? (float)((double)clip / nrm) : 1.0f;
  }
}

struct StepArgs {
  float* p;
  float* m;
  float* v;
  const float* g;        // P payloads (P*n) or a single reduced gradient (P = 1)
  int P;
  int64_t n;
  int adam;
  float lr, b1, b2, eps;
  float inv_bc1, inv_bc2;
  const int64_t* step_dev;  // when set: Adam step t read on the device (graph replay)
  const float* scale;    // optional clip scale (device)
  uint32_t* flags;
};

// Adam bias corrections for the device step counter: computed once per block
// (two fp64 pow per thread would cost more than the update itself); every
// thread of the block must call it.
__device__ __forceinline__ void bias_corrections(const int64_t* step_dev, float b1, float b2, float& i1, float& i2) {
  if (!step_dev) return;
  __shared__ float bc[2];
  if (threadIdx.x == 0) {
    const double t = (double)*step_dev;
    bc[0] = (float)(1.0 / (1.0 - pow((double)b1, t)));
    bc[1] = (float)(1.0 / (1.0 - pow((double)b2, t)));
  }
  __syncthreads();
  i1 = bc[0];
  i2 = bc[1];
}

__global__ void k_dense_step(StepArgs a) {
  const float sc = a.scale ? *a.scale : 1.f;
  bias_corrections(a.step_dev, a.b1, a.b2, a.inv_bc1, a.inv_bc2);
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    float g = (a.P == 1) ? a.g[i] : tree_mean_at(a.g, a.P, a.n, i);
    g *= sc;
    float p = a.p[i];
    if (!a.adam) {
      p -= a.lr * g;
    } else {
      float m = a.m[i] * a.b1 + (1.f - a.b1) * g;
      float v = a.v[i] * a.b2 + (1.f - a.b2) * g * g;
      a.m[i] = m;
      a.v[i] = v;
      p -= a.lr * (m * a.inv_bc1) / (sqrtf(v * a.inv_bc2) + a.eps);
    }
    a.p[i] = p;
    bad |= !isfinite(p);
  }
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) atomicOr(a.flags, KG_FLAG_NONFINITE_PARAM);
}

// Lazy (row-wise) step on the rows of A_k: one warp per row, float4 lanes
// when the row width allows it.
template <bool V4>
__global__ void __launch_bounds__(256) k_sparse_step(float* __restrict__ table, float* __restrict__ m,
                                                     float* __restrict__ v, const float* __restrict__ grad,
                                                     const int32_t* __restrict__ rows,
                                                     const int32_t* __restrict__ counts, int k, int d, int adam,
                                                     float lr, float b1, float b2, float eps, float inv_bc1,
                                                     float inv_bc2, const int64_t* __restrict__ step_dev) {
  bias_corrections(step_dev, b1, b2, inv_bc1, inv_bc2);
  const int32_t nrows = counts[k];
  const int lane = lane_id(), nw = (gridDim.x * blockDim.x) >> 5;
  constexpr int V = V4 ? 4 : 1;
  for (int64_t p = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); p < nrows; p += nw) {
    const int64_t base = (int64_t)rows[p] * d;
    for (int j = lane * V; j < d; j += 32 * V) {
      const int64_t idx = base + j;
      float g[V], t[V];
      VecIO<V>::load(grad + idx, g);
      VecIO<V>::load(table + idx, t);
      if (!adam) {
#pragma unroll
        for (int i = 0; i < V; ++i) t[i] -= lr * g[i];
      } else {
        float mm[V], vv[V];
        VecIO<V>::load(m + idx, mm);
        VecIO<V>::load(v + idx, vv);
#pragma unroll
        for (int i = 0; i < V; ++i) {
          mm[i] = mm[i] * b1 + (1.f - b1) * g[i];
          vv[i] = vv[i] * b2 + (1.f - b2) * g[i] * g[i];
          t[i] -= lr * (mm[i] * inv_bc1) / (sqrtf(vv[i] * inv_bc2) + eps);
        }
        VecIO<V>::store(m + idx, mm);
        VecIO<V>::store(v + idx, vv);
      }
      VecIO<V>::store(table + idx, t);
    }
  }
}

}  // namespace kg

using namespace kg;

extern "C" {

int64_t kg_optim_workspace_bytes(int64_t n) {
  return (int64_t)(align_up(n * sizeof(float)) + align_up(1024 * sizeof(double)) + 1024);
}

kg_status kg_dense_step(float* params, float* m, float* v, const float* grads_all, int32_t P, int64_t n,
                        int32_t optimizer, float lr, float beta1, float beta2, float eps, double bc1, double bc2,
                        const int64_t* step_dev, float grad_clip, uint32_t* flags, void* ws, int64_t ws_bytes,
                        void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(P >= 1 && P <= MAXP, KG_ERR_PROTOCOL, "payload count %d out of range", P);
  KG_REQUIRE(ws_bytes >= kg_optim_workspace_bytes(n), KG_ERR_VALIDATION, "optim workspace too small");
  Arena a(ws, (size_t)ws_bytes);
  float* gmean = a.take<float>(n);
  double* part = a.take<double>(1024);
  float* scale = a.take<float>(1);
  StepArgs s{params, m, v, grads_all, P, n, optimizer == 1, lr, beta1, beta2, eps,
             (float)(1.0 / bc1), (float)(1.0 / bc2), step_dev, nullptr, flags};
  int blocks = persistent_blocks(n, 256, 4);
  if (grad_clip > 0.f) {
    const float* g = grads_all;
    if (P > 1) {
      KG_LAUNCH("k_tree_mean", k_tree_mean, blocks, 256, 0, st, grads_all, P, n, gmean);
      g = gmean;
    }
    int nb = persistent_blocks(n, 256, 2);
    if (nb > 1024) nb = 1024;
    KG_LAUNCH("k_sumsq_blocks", k_sumsq_blocks, nb, 256, 0, st, g, n, part);
    KG_LAUNCH("k_clip_scale", k_clip_scale, 1, 256, 0, st, part, nb, grad_clip, scale);
    s.g = g;
    s.P = 1;
    s.scale = scale;
  }
  KG_LAUNCH("k_dense_step", k_dense_step, blocks, 256, 0, st, s);
  KG_CHECK_LAUNCH("k_dense_step");
  return KG_OK;
}

kg_status kg_sparse_step(float* table, float* m, float* v, const float* grad, const int32_t* rows,
                         const int32_t* counts, int32_t k, int32_t d, int32_t optimizer, float lr, float beta1,
                         float beta2, float eps, double bc1, double bc2, const int64_t* step_dev, int32_t n_max,
                         void* stream) {
  const bool v4 = d % 4 == 0 && (((uintptr_t)table | (uintptr_t)grad | (uintptr_t)m | (uintptr_t)v) & 15) == 0;
  auto kern = v4 ? k_sparse_step<true> : k_sparse_step<false>;
  KG_LAUNCH("k_sparse_step", kern, persistent_blocks((int64_t)n_max * 32, 256, 8), 256, 0, as_stream(stream), table,
            m, v, grad, rows, counts, k, d, optimizer == 1, lr, beta1, beta2, eps, (float)(1.0 / bc1),
            (float)(1.0 / bc2), step_dev);
  KG_CHECK_LAUNCH("k_sparse_step");
  return KG_OK;
}

}  // extern "C"

// Epoch-end bookkeeping in one launch (one block): out[w] = mean over the
// epoch's rounds of worker w's round losses (float64, rounds summed in a
// fixed order), out[nloc + j] = status word j (then cleared). Replaces the
// handful of small tensor ops (mean, cast, cat, or, zero) that sat on the
// stream at every epoch boundary.
namespace kg {
__global__ void __launch_bounds__(256) k_epoch_end(const float* __restrict__ losses, int64_t ld, int32_t nloc,
                                                   int32_t rounds, const unsigned long long* __restrict__ flag_ptrs,
                                                   int32_t nflags, double* __restrict__ out) {
  __shared__ double part[256];
  for (int w = 0; w < nloc; ++w) {
    double s = 0.0;
    for (int r = threadIdx.x; r < rounds; r += blockDim.x) s += (double)losses[(int64_t)w * ld + r];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o) part[threadIdx.x] += part[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[w] = rounds > 0 ? part[0] / (double)rounds : 0.0;
    __syncthreads();
  }
  for (int j = threadIdx.x; j < nflags; j += blockDim.x) {
    uint32_t* f = reinterpret_cast<uint32_t*>(flag_ptrs[j]);
    out[nloc + j] = (double)*f;
    *f = 0u;
  }
}
}  // namespace kg

extern "C" kg_status kg_epoch_end(const float* losses, int64_t ld, int32_t nloc, int32_t rounds,
                                  const uint64_t* flag_ptrs, int32_t nflags, double* out, void* stream) {
  KG_LAUNCH("k_epoch_end", kg::k_epoch_end, 1, 256, 0, as_stream(stream), losses, ld, nloc, rounds,
            reinterpret_cast<const unsigned long long*>(flag_ptrs), nflags, out);
  return KG_OK;
}

// this module's anchor for kg_preload_kernels (kg_primitives.cu)
extern "C" const void* kg_anchor_optim() { return reinterpret_cast<const void*>(&kg::k_tree_mean); }
