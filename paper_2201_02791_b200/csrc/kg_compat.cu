// R19/R20 compatibility entry points in float64 (ref:trainer.py:63-151).
//
// The training loop uses the fp32 fused tree-mean + Adam of kg_optim.cu. The
// public host API (`allreduce_mean(payloads)`, `Optimizer.step(params, ...)`)
// takes float64 numpy arrays and the reference pins it exactly: the mean of
// identical payloads is bitwise the payload (ref tests test_trainer.py:44-61),
// SGD is exact (:75-83), untouched rows stay untouched. These kernels
// therefore compute in float64 with the reference's elementwise operation
// order and explicit round-to-nearest intrinsics (no FMA contraction), so the
// device results are bit-identical to numpy's.
#include "kg_common.cuh"

namespace kg {

// ((g0+g1)+(g2+g3))..., odd tail carried, then / P  (ref:trainer.py:77-86).
// Node j of tree level L covers payloads [j*2^L, min((j+1)*2^L, P)), so the
// level-by-level tree equals a binary-counter stack over the leaves (merge
// equal-sized neighbours as they complete) finished by merging the stack
// from the top: any P with O(log P) registers, bit-identical sums.
__global__ void k_tree_mean_f64(const double* __restrict__ g, int64_t P, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double val[64];
    int64_t size[64];
    int top = 0;
    for (int64_t w = 0; w < P; ++w) {
      val[top] = g[w * n + i];
      size[top] = 1;
      ++top;
      while (top >= 2 && size[top - 1] == size[top - 2]) {
        val[top - 2] = __dadd_rn(val[top - 2], val[top - 1]);
        size[top - 2] *= 2;
        --top;
      }
    }
    while (top >= 2) {
      val[top - 2] = __dadd_rn(val[top - 2], val[top - 1]);
      --top;
    }
    out[i] = __ddiv_rn(val[0], (double)P);
  }
}

__global__ void k_sumsq_f64(const double* __restrict__ g, int64_t n, double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = __dadd_rn(s, __dmul_rn(g[i], g[i]));
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// scale = clip / ||g|| when ||g|| > clip, else 1 (ref:trainer.py:113-117)
__global__ void k_clip_scale_f64(const double* __restrict__ part, int nb, double clip, double* __restrict__ scale) {
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int i = 0; i < nb; ++i) s = __dadd_rn(s, part[i]);
  const double nrm = __dsqrt_rn(s);
  scale[0] = nrm > clip ? __ddiv_rn(clip, nrm) : 1.0;
  scale[1] = nrm > clip ? 1.0 : 0.0;   // whether the gradient is rescaled
}

struct Step64 {
  double lr, b1, b2, omb1, omb2, eps, bc1, bc2;
  int adam;
};

// Dense blocks (ref:trainer.py:124-134):
//   m *= b1; m += (1-b1)*g; v *= b2; v += ((1-b2)*g)*g;
//   p -= (lr*(m/bc1)) / (sqrt(v/bc2) + eps)          (SGD: p -= lr*g)
__global__ void k_dense_step_f64(double* __restrict__ p, double* __restrict__ m, double* __restrict__ v,
                                 const double* __restrict__ g, int64_t n, Step64 s,
                                 const double* __restrict__ scale, uint32_t* __restrict__ flags) {
  const bool rescale = scale != nullptr && scale[1] != 0.0;
  const double sc = rescale ? scale[0] : 1.0;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = rescale ? __dmul_rn(g[i], sc) : g[i];
    double pi = p[i];
    if (!s.adam) {
      pi = __dsub_rn(pi, __dmul_rn(s.lr, gi));
    } else {
      const double mi = __dadd_rn(__dmul_rn(m[i], s.b1), __dmul_rn(s.omb1, gi));
      const double vi = __dadd_rn(__dmul_rn(v[i], s.b2), __dmul_rn(__dmul_rn(s.omb2, gi), gi));
      m[i] = mi;
      v[i] = vi;
      const double num = __dmul_rn(s.lr, __ddiv_rn(mi, s.bc1));
      const double den = __dadd_rn(__dsqrt_rn(__ddiv_rn(vi, s.bc2)), s.eps);
      pi = __dsub_rn(pi, __ddiv_rn(num, den));
    }
    p[i] = pi;
    bad |= !isfinite(pi);
  }
  if (__any_sync(__activemask(), bad) && flags) atomicOr(flags, KG_FLAG_NONFINITE_PARAM);
}

// Last occurrence of every id in the update list (numpy fancy assignment
// `a[ids] = x` keeps the last duplicate).
__global__ void k_last_occurrence(const int64_t* __restrict__ ids, int64_t k, int32_t* __restrict__ lastpos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
    atomicMax(lastpos + ids[i], (int32_t)i);
}

// Lazy sparse rows (ref:trainer.py:136-147). Every occurrence i computes its
// output row from the OLD moments (the reference gathers em[ids] once), the
// row results go to out_rows (the caller assigns table[ids] = out_rows);
// moments are written back by the last occurrence only (phase 2).
__global__ void k_sparse_rows_f64(const double* __restrict__ old_rows, const double* __restrict__ grad_rows,
                                  const int64_t* __restrict__ ids, int64_t k, int d, const double* __restrict__ em,
                                  const double* __restrict__ ev, Step64 s, double* __restrict__ out_rows,
                                  double* __restrict__ m_new, double* __restrict__ v_new) {
  const int64_t total = k * (int64_t)d;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / d, c = q - i * d;
    const double gi = grad_rows[q];
    const double t = old_rows[q];
    if (!s.adam) {
      out_rows[q] = __dsub_rn(t, __dmul_rn(s.lr, gi));
    } else {
      const int64_t src = ids[i] * d + c;
      // em[ids]*b1 + (1-b1)*rows ; ev[ids]*b2 + (1-b2)*rows**2
      const double mi = __dadd_rn(__dmul_rn(em[src], s.b1), __dmul_rn(s.omb1, gi));
      const double vi = __dadd_rn(__dmul_rn(ev[src], s.b2), __dmul_rn(s.omb2, __dmul_rn(gi, gi)));
      m_new[q] = mi;
      v_new[q] = vi;
      const double num = __dmul_rn(s.lr, __ddiv_rn(mi, s.bc1));
      const double den = __dadd_rn(__dsqrt_rn(__ddiv_rn(vi, s.bc2)), s.eps);
      out_rows[q] = __dsub_rn(t, __ddiv_rn(num, den));
    }
  }
}

__global__ void k_sparse_moments_f64(const int64_t* __restrict__ ids, int64_t k, int d,
                                     const int32_t* __restrict__ lastpos, const double* __restrict__ m_new,
                                     const double* __restrict__ v_new, double* __restrict__ em,
                                     double* __restrict__ ev) {
  const int64_t total = k * (int64_t)d;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / d, c = q - i * d;
    const int64_t id = ids[i];
    if (lastpos[id] != (int32_t)i) continue;
    em[id * d + c] = m_new[q];
    ev[id * d + c] = v_new[q];
  }
}

}  // namespace kg

using namespace kg;

extern "C" {

kg_status kg_tree_mean_f64(const double* payloads, int64_t P, int64_t n, double* out, void* stream) {
  KG_REQUIRE(P >= 1, KG_ERR_PROTOCOL, "empty reduction");
  if (n == 0) return KG_OK;
  KG_LAUNCH("k_tree_mean_f64", k_tree_mean_f64, persistent_blocks(n, 256, 4), 256, 0, as_stream(stream), payloads,
            P, n, out);
  return KG_OK;
}

int64_t kg_dense_step_f64_workspace_bytes(int64_t n) {
  (void)n;
  return (int64_t)(align_up(1024 * sizeof(double)) + align_up(2 * sizeof(double)));
}

kg_status kg_dense_step_f64(double* params, double* m, double* v, const double* grads, int64_t n, int32_t optimizer,
                            double lr, double beta1, double beta2, double eps, double bc1, double bc2,
                            double grad_clip, uint32_t* flags, void* ws, int64_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(ws_bytes >= kg_dense_step_f64_workspace_bytes(n), KG_ERR_VALIDATION, "workspace too small");
  if (n == 0) return KG_OK;
  Arena a(ws, (size_t)ws_bytes);
  double* part = a.take<double>(1024);
  double* scale = a.take<double>(2);
  Step64 s{lr, beta1, beta2, 1.0 - beta1, 1.0 - beta2, eps, bc1, bc2, optimizer == 1};
  const double* sc = nullptr;
  if (grad_clip >= 0.0) {   // None is passed as a negative value
    int nb = persistent_blocks(n, 256, 2);
    if (nb > 1024) nb = 1024;
    KG_LAUNCH("k_sumsq_f64", k_sumsq_f64, nb, 256, 0, st, grads, n, part);
    KG_LAUNCH("k_clip_scale_f64", k_clip_scale_f64, 1, 32, 0, st, part, nb, grad_clip, scale);
    sc = scale;
  }
  KG_LAUNCH("k_dense_step_f64", k_dense_step_f64, persistent_blocks(n, 256, 4), 256, 0, st, params, m, v, grads, n,
            s, sc, flags);
  return KG_OK;
}

int64_t kg_sparse_step_f64_workspace_bytes(int64_t k, int32_t d, int64_t num_rows) {
  return (int64_t)(2 * align_up((size_t)k * d * sizeof(double)) + align_up((size_t)num_rows * sizeof(int32_t)));
}

kg_status kg_sparse_step_f64(const double* old_rows, const double* grad_rows, const int64_t* ids, int64_t k,
                             int32_t d, double* em, double* ev, int64_t num_rows, int32_t optimizer, double lr,
                             double beta1, double beta2, double eps, double bc1, double bc2, double* out_rows,
                             void* ws, int64_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(ws_bytes >= kg_sparse_step_f64_workspace_bytes(k, d, num_rows), KG_ERR_VALIDATION,
             "workspace too small");
  if (k == 0 || d == 0) return KG_OK;
  Arena a(ws, (size_t)ws_bytes);
  double* m_new = a.take<double>((size_t)k * d);
  double* v_new = a.take<double>((size_t)k * d);
  int32_t* lastpos = a.take<int32_t>((size_t)num_rows);
  Step64 s{lr, beta1, beta2, 1.0 - beta1, 1.0 - beta2, eps, bc1, bc2, optimizer == 1};
  const int64_t total = k * (int64_t)d;
  KG_LAUNCH("k_sparse_rows_f64", k_sparse_rows_f64, persistent_blocks(total, 256, 4), 256, 0, st, old_rows,
            grad_rows, ids, k, d, em, ev, s, out_rows, m_new, v_new);
  if (optimizer == 1) {
    KG_CUDA(cudaMemsetAsync(lastpos, 0xff, (size_t)num_rows * sizeof(int32_t), st));
    KG_LAUNCH("k_last_occurrence", k_last_occurrence, persistent_blocks(k, 256, 4), 256, 0, st, ids, k, lastpos);
    KG_LAUNCH("k_sparse_moments_f64", k_sparse_moments_f64, persistent_blocks(total, 256, 4), 256, 0, st, ids, k, d,
              lastpos, m_new, v_new, em, ev);
  }
  return KG_OK;
}

}  // extern "C"

// this module's anchor for kg_preload_kernels (kg_primitives.cu)
extern "C" const void* kg_anchor_compat() { return reinterpret_cast<const void*>(&kg::k_tree_mean_f64); }
