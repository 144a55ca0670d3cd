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
};

// CUDA-core reference implementations (kg_gemm.cu): used by tests as a
// cross-check of the tensor-core kernels.
kg_status simt_gemm_nn(const GemmArgs& g, cudaStream_t st);
size_t simt_gemm_tn_workspace(int64_t rows_max, int64_t K, int64_t N);
kg_status simt_gemm_tn(const GemmArgs& g, float* out, void* ws, cudaStream_t st);
kg_status reduce_splits(const float* part, int splits, int64_t count, float* out, cudaStream_t st);

// tcgen05 3xTF32 kernels (kg_umma.cu): the product path. Both need a
// workspace for the packed (hi/lo, canonical-layout) operands.
size_t umma_nn_workspace(int64_t M_max, int64_t K, int64_t N);
kg_status umma_gemm_nn(const GemmArgs& g, void* ws, cudaStream_t st);
size_t umma_tn_workspace(int64_t rows_max, int64_t K, int64_t N);
kg_status umma_gemm_tn(const GemmArgs& g, float* out, void* ws, cudaStream_t st);

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
