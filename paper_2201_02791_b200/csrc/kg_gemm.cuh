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

kg_status gemm_nn(const GemmArgs& g, cudaStream_t st);
size_t gemm_tn_workspace(int64_t rows_max, int64_t K, int64_t N);
kg_status gemm_tn(const GemmArgs& g, float* out, void* ws, cudaStream_t st);

}  // namespace kg
