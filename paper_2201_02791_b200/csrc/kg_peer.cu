// Peer-memory exchange of the dense gradient payloads (one partition per
// rank on one NVLink/NVSwitch node). Replaces the NCCL all-gather between the
// compute and update halves of a round (ref:trainer.py:430-438 gathers every
// worker's payload before the pairwise-tree mean, ref:trainer.py:77-86):
//
//   kg_peer_publish  copies this rank's payload into its own IPC-shared region
//                    (slot = round parity) and releases the region's flag;
//   kg_peer_gather   acquires every peer's flag and reads the P payloads over
//                    NVLink straight into the (P, n) tree-mean input, in
//                    partition order.
//
// Region layout: [u64 flag | pad to 256 B][slot 0: n floats][slot 1: n floats].
// A rank re-uses slot s&1 at round s+2 only after its gather of round s+1,
// which needed every peer's round-s+1 flag, i.e. every peer finished reading
// round s: two slots are enough. Every wait is bounded (5 s) and reports
// through the worker flags (bit 8) instead of hanging the device.
#include <algorithm>
#include <cstring>

#include "kg_common.cuh"

namespace kg {
namespace {

constexpr size_t kPeerHeader = 256;
constexpr uint32_t kPeerTimeoutFlag = KG_FLAG_PEER_TIMEOUT;
// A few CTAs only: the gather's wait for the slowest rank must not hold the
// SMs the sampler's epoch graph and the forked streams run on (a full-grid
// spin cost 70 us/round at 2 ranks); 32 CTAs still read ~1 MB over NVLink in
// about a microsecond.
constexpr int kPeerBlocks = 32;
constexpr unsigned long long kPeerTimeoutNs = 5ull * 1000 * 1000 * 1000;

__host__ __device__ inline size_t peer_slot_bytes(int64_t n) { return ((size_t)n * sizeof(float) + 255) / 256 * 256; }

__device__ inline unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ inline unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ inline void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// seq[0] = rounds exchanged so far, seq[1] / seq[2] = block-arrival counters
__global__ void k_peer_publish(const float* __restrict__ src, char* region, int64_t n,
                               unsigned long long* seq) {
  const unsigned long long s = seq[0];
  float* dst = reinterpret_cast<float*>(region + kPeerHeader + (s & 1) * peer_slot_bytes(n));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long prev = atomicAdd(&seq[1], 1ull);
    if (prev == gridDim.x - 1) {           // last block: every slice is written and fenced
      seq[1] = 0;
      __threadfence_system();
      st_release_sys(reinterpret_cast<unsigned long long*>(region), s + 1);
    }
  }
}

__global__ void k_peer_gather(char* const* __restrict__ regions, int P, int64_t n, float* __restrict__ out,
                              unsigned long long* seq, uint32_t* flags) {
  __shared__ int timed_out;
  const unsigned long long s = seq[0];
  if (threadIdx.x == 0) timed_out = 0;
  __syncthreads();
  if ((int)threadIdx.x < P) {
    const unsigned long long* f = reinterpret_cast<const unsigned long long*>(regions[threadIdx.x]);
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(f) < s + 1) {
      if (globaltimer() - t0 > kPeerTimeoutNs) {
        atomicOr(flags, kPeerTimeoutFlag);
        timed_out = 1;
        break;
      }
      __nanosleep(100);
    }
  }
  __syncthreads();
  if (!timed_out) {
    // Remote loads take ~1-2 us over NVLink: keep UNR 16-byte loads in flight
    // per thread (the flag acquire above orders them; .cg skips L1).
    const size_t off = kPeerHeader + (s & 1) * peer_slot_bytes(n);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    constexpr int UNR = 8;
    if ((n & 3) == 0) {
      const int64_t n4 = n >> 2, total4 = (int64_t)P * n4;
      float4* o4 = reinterpret_cast<float4*>(out);
      for (int64_t base = tid; base < total4; base += stride * UNR) {
        float4 v[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int64_t i = base + u * stride;
          if (i < total4) {
            const int p = (int)(i / n4);
            v[u] = __ldcg(reinterpret_cast<const float4*>(regions[p] + off) + (i - (int64_t)p * n4));
          }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          if (base + u * stride < total4) o4[base + u * stride] = v[u];
      }
    } else {
      const int64_t total = (int64_t)P * n;
      for (int64_t base = tid; base < total; base += stride * UNR) {
        float v[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int64_t i = base + u * stride;
          if (i < total) {
            const int p = (int)(i / n);
            v[u] = __ldcg(reinterpret_cast<const float*>(regions[p] + off) + (i - (int64_t)p * n));
          }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          if (base + u * stride < total) out[base + u * stride] = v[u];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long prev = atomicAdd(&seq[2], 1ull);
    if (prev == gridDim.x - 1) {           // every block has read seq[0] and its slice
      seq[2] = 0;
      seq[0] = s + 1;
    }
  }
}

}  // namespace
}  // namespace kg

using namespace kg;

extern "C" {

int64_t kg_peer_region_bytes(int64_t n) { return (int64_t)(kPeerHeader + 2 * peer_slot_bytes(n)); }

kg_status kg_peer_alloc(int64_t bytes, void** region, void* ipc_handle) {
  KG_REQUIRE(bytes > 0 && region && ipc_handle, KG_ERR_VALIDATION, "kg_peer_alloc: bad arguments");
  KG_CUDA(cudaMalloc(region, (size_t)bytes));
  KG_CUDA(cudaMemset(*region, 0, (size_t)bytes));
  KG_CUDA(cudaDeviceSynchronize());
  cudaIpcMemHandle_t h;
  KG_CUDA(cudaIpcGetMemHandle(&h, *region));
  memcpy(ipc_handle, &h, sizeof(h));
  return KG_OK;
}

kg_status kg_peer_open(const void* ipc_handle, void** region) {
  KG_REQUIRE(ipc_handle && region, KG_ERR_VALIDATION, "kg_peer_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  KG_CUDA(cudaIpcOpenMemHandle(region, h, cudaIpcMemLazyEnablePeerAccess));
  return KG_OK;
}

kg_status kg_peer_close(void* region, int32_t owned) {
  if (!region) return KG_OK;
  KG_CUDA(owned ? cudaFree(region) : cudaIpcCloseMemHandle(region));
  return KG_OK;
}

kg_status kg_peer_publish(const float* local, void* region, int64_t n, int64_t* seq, void* stream) {
  KG_REQUIRE(n > 0 && local && region && seq, KG_ERR_VALIDATION, "kg_peer_publish: bad arguments");
  const int blocks = (int)std::min<int64_t>(ceil_div(n, 256), kPeerBlocks);
  KG_LAUNCH("k_peer_publish", k_peer_publish, blocks, 256, 0, as_stream(stream), local,
            static_cast<char*>(region), n, reinterpret_cast<unsigned long long*>(seq));
  return KG_OK;
}

kg_status kg_peer_gather(void* const* regions_dev, int32_t P, int64_t n, float* out, int64_t* seq,
                         uint32_t* flags, void* stream) {
  KG_REQUIRE(P >= 1 && P <= 256 && n > 0 && regions_dev && out && seq && flags, KG_ERR_VALIDATION,
             "kg_peer_gather: bad arguments");
  const int blocks = (int)std::min<int64_t>(ceil_div((int64_t)P * n, 256), kPeerBlocks);
  KG_LAUNCH("k_peer_gather", k_peer_gather, blocks, 256, 0, as_stream(stream),
            reinterpret_cast<char* const*>(regions_dev), P, n, out, reinterpret_cast<unsigned long long*>(seq),
            flags);
  return KG_OK;
}

}  // extern "C"

// this module's anchor for kg_preload_kernels (kg_primitives.cu)
extern "C" const void* kg_anchor_peer() { return reinterpret_cast<const void*>(&kg::k_peer_publish); }
