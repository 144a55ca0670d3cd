// Shared helpers for the kgdist-b200 sm_100a kernel library.
//
// Everything here is plain CUDA C++ compiled with
//   -gencode arch=compute_100a,code=sm_100a
// The C ABI (include/kgdist_b200.h) takes raw device pointers, element
// counts and a cudaStream_t passed as void*; memory is owned by the caller
// (PyTorch tensors on the Python side), scratch comes from caller workspaces.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/kgdist_b200.h"

namespace kg {

// --- error plumbing ------------------------------------------------------
void set_error(const char* fmt, ...);
kg_status from_cuda(cudaError_t e, const char* where);

#define KG_CHECK_LAUNCH(where)                                      \
  do {                                                              \
    cudaError_t _e = cudaGetLastError();                            \
    if (_e != cudaSuccess) return ::kg::from_cuda(_e, where);       \
  } while (0)

#define KG_CUDA(call)                                               \
  do {                                                              \
    cudaError_t _e = (call);                                        \
    if (_e != cudaSuccess) return ::kg::from_cuda(_e, #call);       \
  } while (0)

// Every kernel launch goes through KG_LAUNCH: it counts launches
// (kg_launch_count) and, while kg_kernel_timer_begin(prefix) is active,
// brackets matching kernels with CUDA events on their own stream.
// Clears (and remembers) a runtime error left by an earlier call whose
// status was not consumed, so it is not misattributed to the next launch.
void check_stale(const char* before);

struct LaunchScope {
  cudaStream_t st;
  int slot;
  LaunchScope(const char* name, cudaStream_t s);
  void done();
};

// Diagnostics only: KG_KNOCKOUT="name1,name2" skips those launches (results
// are then wrong) to measure how much a kernel adds to the step time.
bool knocked_out(const char* name);

#define KG_LAUNCH(name, kern, grid, block, smem, st_, ...)          \
  do {                                                              \
    auto _kp = kern;                                                \
    if (::kg::knocked_out(name)) break;                             \
    ::kg::check_stale(name);                                        \
    ::kg::LaunchScope _ls(name, st_);                               \
    _kp<<<(grid), (block), (smem), (st_)>>>(__VA_ARGS__);           \
    _ls.done();                                                     \
    cudaError_t _le = cudaGetLastError();                           \
    if (_le != cudaSuccess) return ::kg::from_cuda(_le, name);      \
  } while (0)

#define KG_REQUIRE(cond, status, ...)                               \
  do {                                                              \
    if (!(cond)) { ::kg::set_error(__VA_ARGS__); return status; }   \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Number of SMs of the current device (148 on B200), cached per process.
int num_sms();

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Bump allocator over a caller workspace.
struct Arena {
  char* base;
  size_t cap;
  size_t used;
  Arena(void* p, size_t n) : base(static_cast<char*>(p)), cap(n), used(0) {}
  template <typename T>
  T* take(size_t count) {
    size_t off = align_up(used);
    used = off + count * sizeof(T);
    if (base == nullptr) return nullptr;           // sizing pass
    if (used > cap) return nullptr;
    return reinterpret_cast<T*>(base + off);
  }
};

// --- device helpers ------------------------------------------------------
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// V consecutive floats (V = 4: 16-byte aligned float4; V = 1: scalar)
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

// Broadcast from lane 0: tells the compiler the value is warp-uniform, so loops
// and loads derived from it stay convergent (no collective fallback around the
// __shfl_sync calls inside per-warp work loops).
__device__ __forceinline__ int64_t warp_uniform(int64_t v) {
  const int lo = __shfl_sync(0xffffffffu, (int)(v & 0xffffffff), 0);
  const int hi = __shfl_sync(0xffffffffu, (int)(v >> 32), 0);
  return ((int64_t)hi << 32) | (uint32_t)lo;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Grid-stride persistent launch size: a multiple of the SM count.
inline int persistent_blocks(int64_t work_items, int items_per_block, int blocks_per_sm = 4) {
  int64_t want = ceil_div(work_items > 0 ? work_items : 1, items_per_block);
  int64_t cap = (int64_t)num_sms() * blocks_per_sm;
  return (int)(want < cap ? want : cap);
}

// --- primitives (kg_primitives.cu) ---------------------------------------
// Exclusive prefix sum of n uint32 values; out may alias in. total (device,
// optional) receives the grand total.
size_t scan_workspace(int64_t n);
kg_status exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* total,
                             void* ws, size_t ws_bytes, cudaStream_t st);

// Stable LSD radix sort of (key, value) pairs on the low `key_bits` bits.
// keys/vals are sorted in place (ping-pong buffers come from the workspace).
size_t sort_workspace(int64_t n);
kg_status sort_pairs_u64(uint64_t* keys, uint32_t* vals, int64_t n, int key_bits, void* ws,
                         size_t ws_bytes, cudaStream_t st);
size_t sort32_workspace(int64_t n);
kg_status sort_pairs_u32(uint32_t* keys, uint32_t* vals, int64_t n, int key_bits, void* ws,
                         size_t ws_bytes, cudaStream_t st);

// Stream compaction of indices i in [0, n) with flag[i] != 0 into out (ascending),
// count written to *count_out (device).  Flags are uint32 0/1.
size_t compact_workspace(int64_t n);
kg_status compact_flags(const uint32_t* flags, int64_t n, int32_t* out, int32_t* count_out,
                        int32_t out_offset_const, const int32_t* out_offset_dev, void* ws,
                        size_t ws_bytes, cudaStream_t st);
// Closure-style compaction: out[off + rank(i)] = i for flagged i with off =
// *off_d (0 if null), pos_out[i] = off + rank(i), *count_abs = off + total,
// and the flags are cleared for the next use.
kg_status compact_flags_ex(uint32_t* flags, int64_t n, int32_t* out, const int32_t* off_d, int32_t* count_abs,
                           int32_t* pos_out, void* ws, size_t ws_bytes, cudaStream_t st);

// Static work-chunk table of a CSR (kg_chunks.cu).
size_t chunk_workspace(int64_t n);
kg_status build_chunk_table(const int32_t* indptr, int32_t n, int C, int32_t* ptr, int32_t* row, int32_t* slot,
                            int32_t* split, int32_t* counts, int32_t* desc, void* ws, size_t ws_bytes,
                            cudaStream_t st);

}  // namespace kg
