#pragma once
#include "kg_common.cuh"

namespace kg {

struct GemmArgs {
  const float* A;          // NN: (rows, lda) gathered by a_rows; TN: same, rows = data rows
  int64_t lda;
  const int32_t* a_rows;   // optional row ids for A
  const float* B;          // (K or data rows, ldb)
  int64_t ldb;
  float* C;                // NN output (row ids c_rows), ldc
  int64_t ldc;
  const int32_t* c_rows;
  int64_t M;               // rows (host) if M_dev == nullptr
  const int32_t* M_dev;    // device row count (counts[] array)
  int M_dev_index;
  int64_t M_max;           // upper bound for grid sizing
  int64_t K;               // NN: reduction length; TN: output rows
  int64_t N;
  int relu;
  const float* a_packed;   // NN only: A already in hi/lo records (see packed_store), a_rows ignored
  const float* b_packed;   // NN only: B already in records (N_pad rows, one block; kg_rgcn_pack_weights)
  float* c_packed;         // NN only, optional: the output also as A records by MMA row (K = N)
  const float* mul;        // NN only, optional: output row m scaled by mul[m*N + n] after ReLU (dropout)
};

// --- packed tensor-core operand records (kg_umma.cu) -----------------------
// An operand with 128-row blocks is stored as records (block, kc) of 128 x 16
// values in the K-major 64-byte-swizzle canonical UMMA layout: 8-row groups of
// 512 B, each row's 16
// K values in 64 contiguous bytes whose 16-byte chunks are XOR-permuted by
// (row >> 1) & 3. A row's piece of a record is two whole 32-byte sectors, so a
// row-at-a-time producer (k_aggregate, the dS pass) writes complete sectors
// even when the operand spills past L2 (the no-swizzle layout interleaves 8
// rows at 16 B and cost DRAM read-modify-writes there). Producers that emit
// this layout directly save the separate pack pass.
// Two record formats, chosen by the operand's row capacity (records_split):
//   fp32   one 128x16 fp32 half; the GEMM's split warps make the tf32 hi/lo
//          halves in shared memory (large operands: HBM carries 4 B/value);
//   split  [hi | lo] tf32 halves written by the producer (L2-resident
//          operands, where the in-GEMM split would only add latency).
// Device helpers take the record count per block as a signed `nk`: negative
// means split records of -nk per block.
constexpr int PK_ROWS = 128;
constexpr int PK_K = 16;
constexpr int64_t PK_REC = PK_ROWS * PK_K;   // floats per record half

// float offset of element (r, k), k < PK_K, inside a record half (any row count)
__host__ __device__ __forceinline__ int pk_off(int r, int k) {
  return (r >> 3) * 128 + (r & 7) * 16 + ((((k >> 2) ^ (r >> 1)) & 3) << 2) + (k & 3);
}

inline int64_t packed_records(int64_t K) { return (K + PK_K - 1) / PK_K; }
// split records for operands of up to KG_SPLIT_ROWS_MAX rows (default 65,536:
// FB15k-237 shape and smaller stay L2-resident)
bool records_split(int64_t rows);
// signed record count (see above)
inline int64_t packed_nk(int64_t rows, int64_t K) { return records_split(rows) ? -packed_records(K) : packed_records(K); }
inline size_t packed_bytes(int64_t rows, int64_t K) {
  return (size_t)((rows + PK_ROWS - 1) / PK_ROWS) * (size_t)packed_records(K) * PK_REC * sizeof(float) *
         (records_split(rows) ? 2 : 1);
}

#ifdef __CUDACC__
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));   // nearest tf32: |lo| <= 2^-12 |x|
  hi = __uint_as_float(h);
  lo = x - hi;
}

// float pointer of element (row, k) (the hi half for split records)
__device__ __forceinline__ float* packed_at(float* P, int64_t nk, int64_t row, int k) {
  const int r = (int)(row & (PK_ROWS - 1)), kk = k & (PK_K - 1);
  const bool sp = nk < 0;
  const int64_t rec = (row / PK_ROWS) * (sp ? -nk : nk) + (k / PK_K);
  return P + rec * (sp ? 2 * PK_REC : PK_REC) + pk_off(r, kk);
}

// V consecutive values starting at k (k % V == 0, V in {1, 2, 4})
template <int V>
__device__ __forceinline__ void packed_store4(float* p, const float* v) {
  if constexpr (V == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else if constexpr (V == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
    *p = v[0];
  }
}

template <int V>
__device__ __forceinline__ void packed_store(float* P, int64_t nk, int64_t row, int k, const float* v) {
  float* ph = packed_at(P, nk, row, k);
  if (nk > 0) {
    packed_store4<V>(ph, v);
    return;
  }
  float h[V], l[V];
#pragma unroll
  for (int i = 0; i < V; ++i) split_tf32(v[i], h[i], l[i]);
  packed_store4<V>(ph, h);
  packed_store4<V>(ph + PK_REC, l);
}

// zero the K padding [K, 16*nk) of one row (lanes of a warp share the work)
__device__ __forceinline__ void packed_zero_pad(float* P, int64_t nk, int64_t row, int K, int lane, int nlanes) {
  const int64_t n = nk < 0 ? -nk : nk;
  for (int k = K + lane; k < n * PK_K; k += nlanes) {
    float* p = packed_at(P, nk, row, k);
    p[0] = 0.f;
    if (nk < 0) p[PK_REC] = 0.f;
  }
}
#endif

// CUDA-core reference implementations (kg_gemm.cu): used by tests as a
// cross-check of the tensor-core kernels.
kg_status simt_gemm_nn(const GemmArgs& g, cudaStream_t st);
size_t simt_gemm_tn_workspace(int64_t rows_max, int64_t K, int64_t N);
kg_status simt_gemm_tn(const GemmArgs& g, float* out, void* ws, cudaStream_t st);
kg_status reduce_splits(const float* part, int splits, int64_t count, float* out, cudaStream_t st);

// tcgen05 3xTF32 kernels (kg_umma.cu): the product path. Both need a
// workspace for the packed (canonical-layout) operands.
size_t umma_nn_workspace(int64_t M_max, int64_t K, int64_t N);
kg_status umma_gemm_nn(const GemmArgs& g, void* ws, cudaStream_t st);
size_t umma_tn_workspace(int64_t rows_max, int64_t K, int64_t N);
kg_status umma_gemm_tn(const GemmArgs& g, float* out, void* ws, cudaStream_t st);

// dV = X^T dS from the producers' operand records read as MN-major operands
// (kg_umma.cu): X records (x_cols <= 128 columns) and dS records (N <= 256)
// of the same rows (device count M_dev[M_dev_index]); out (x_cols, N).
// ws: at least umma_tn_workspace(rows_max, x_cols, N) bytes.
kg_status umma_gemm_tn_records(const float* Xp, int64_t x_cols, const float* Dp, int64_t N, const int32_t* M_dev,
                               int M_dev_index, int64_t rows_max, float* out, void* ws, cudaStream_t st);

size_t umma_tn_records_test_workspace(int64_t M, int64_t K, int64_t N);
kg_status umma_gemm_tn_via_records(const GemmArgs& g, float* out, void* ws, cudaStream_t st);

// Filtered ranking on the tensor cores (kg_umma.cu), d <= 128.
size_t umma_rank_workspace(int64_t nq, int32_t N, int d, int64_t max_pairs);
kg_status umma_rank_filtered(const float* H, int d, int32_t N, const float* dec, int32_t R, const int32_t* qry,
                             int64_t nq, const int64_t* tkeys, int64_t ntk, const int64_t* hkeys, int64_t nhk,
                             int policy, int chunk, int64_t max_pairs, double* ranks, int32_t* ncand,
                             uint32_t* overflow, void* ws, size_t ws_bytes, cudaStream_t st, const double* H64,
                             const double* dec64);

inline size_t gemm_nn_workspace(int64_t M_max, int64_t K, int64_t N) { return umma_nn_workspace(M_max, K, N); }
inline kg_status gemm_nn(const GemmArgs& g, void* ws, cudaStream_t st) { return umma_gemm_nn(g, ws, st); }
inline size_t gemm_tn_workspace(int64_t rows_max, int64_t K, int64_t N) {
  size_t a = umma_tn_workspace(rows_max, K, N), b = simt_gemm_tn_workspace(rows_max, K, N);
  return a > b ? a : b;
}
inline kg_status gemm_tn(const GemmArgs& g, float* out, void* ws, cudaStream_t st) {
  return umma_gemm_tn(g, out, ws, st);
}

}  // namespace kg
