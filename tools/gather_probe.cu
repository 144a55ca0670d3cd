// Row-gather throughput probe (diagnostic, not part of the library): how fast
// can one B200 gather E random 400-byte rows of an L2-resident table and sum
// them per 32-message unit, with
//   reg<UNR>   plain float4 loads, UNR rows in flight per lane, then FMAs
//   bulk<NS>   per-warp ring of NS 16-message stages filled by
//              cp.async.bulk (one 1-D bulk copy per row, mbarrier tx count)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_probe tools/gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

template <int UNR>
__global__ void __launch_bounds__(256, 4) k_reg(const float* __restrict__ H, const int* __restrict__ idx, const float* __restrict__ w,
                                               int E, int d, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * 8;
  const int units = E / 32;
  const bool ok = lane * 4 < d;
  const float* hb = H + (ok ? lane * 4 : 0);
  for (int u = blockIdx.x * 8 + (threadIdx.x >> 5); u < units; u += warps) {
    const uint32_t off = (uint32_t)__ldg(idx + u * 32 + lane) * (uint32_t)d;
    const float cf = __ldg(w + u * 32 + lane);
    float a0 = 0, a1 = 0, a2 = 0, a3 = 0, b0 = 0, b1 = 0, b2 = 0, b3 = 0;
    for (int j = 0; j < 32; j += UNR) {
      float4 x[UNR];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const uint32_t o = __shfl_sync(0xffffffffu, off, j + q);
        x[q] = __ldg(reinterpret_cast<const float4*>(hb + o));
      }
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const float c = __shfl_sync(0xffffffffu, cf, j + q);
        const float c2 = c * 0.5f;
        a0 = fmaf(c, x[q].x, a0); a1 = fmaf(c, x[q].y, a1); a2 = fmaf(c, x[q].z, a2); a3 = fmaf(c, x[q].w, a3);
        b0 = fmaf(c2, x[q].x, b0); b1 = fmaf(c2, x[q].y, b1); b2 = fmaf(c2, x[q].z, b2); b3 = fmaf(c2, x[q].w, b3);
      }
    }
    if (ok) {
      *reinterpret_cast<float4*>(out + (int64_t)u * 2 * d + lane * 4) = make_float4(a0, a1, a2, a3);
      *reinterpret_cast<float4*>(out + (int64_t)u * 2 * d + d + lane * 4) = make_float4(b0, b1, b2, b3);
    }
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// per-warp ring of NS stages x 16 rows; WPB warps per block
template <int NS, int WPB>
__global__ void __launch_bounds__(WPB * 32, 1) k_bulk(const float* __restrict__ H, const int* __restrict__ idx,
                                                     const float* __restrict__ w, int E, int d, float* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[WPB][NS];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t rb = (uint32_t)d * 4;
  uint8_t* ring = sm + (size_t)wid * NS * 16 * rb;
  if (lane == 0)
    for (int s = 0; s < NS; ++s) mbar_init(smem_u32(&bars[wid][s]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int warps = gridDim.x * WPB;
  const int units = E / 16;   // 16-row stages; a 32-message output unit = 2 stages
  const int u0 = (blockIdx.x * WPB + wid) * 2;
  // this warp's stage sequence: units u0, u0+1, u0+2W, u0+2W+1, ...
  auto unit_of = [&](int i) { return u0 + (i >> 1) * 2 * warps + (i & 1); };
  int nst = 0;
  while (unit_of(nst) < units) ++nst;   // stages of this warp (small loop, fine for a probe)
  auto issue = [&](int i) {
    const int s = i % NS, u = unit_of(i);
    const uint32_t bar = smem_u32(&bars[wid][s]);
    if (lane == 0) mbar_expect_tx(bar, 16 * rb);
    __syncwarp();
    if (lane < 16) {
      const int r = __ldg(idx + u * 16 + lane);
      bulk_g2s(smem_u32(ring + (size_t)(s * 16 + lane) * rb), H + (int64_t)r * d, rb, bar);
    }
  };
  for (int i = 0; i < NS - 1 && i < nst; ++i) issue(i);
  const bool ok = lane * 4 < d;
  float a0 = 0, a1 = 0, a2 = 0, a3 = 0, b0 = 0, b1 = 0, b2 = 0, b3 = 0;
  for (int i = 0; i < nst; ++i) {
    if (i + NS - 1 < nst) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + NS - 1);
    }
    const int s = i % NS, u = unit_of(i);
    const float cf = lane < 16 ? __ldg(w + u * 16 + lane) : 0.f;
    mbar_wait(smem_u32(&bars[wid][s]), (uint32_t)((i / NS) & 1));
    const float* st = reinterpret_cast<const float*>(ring + (size_t)s * 16 * rb) + (ok ? lane * 4 : 0);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const float4 x = *reinterpret_cast<const float4*>(st + q * d);
      const float c = __shfl_sync(0xffffffffu, cf, q);
      const float c2 = c * 0.5f;
      a0 = fmaf(c, x.x, a0); a1 = fmaf(c, x.y, a1); a2 = fmaf(c, x.z, a2); a3 = fmaf(c, x.w, a3);
      b0 = fmaf(c2, x.x, b0); b1 = fmaf(c2, x.y, b1); b2 = fmaf(c2, x.z, b2); b3 = fmaf(c2, x.w, b3);
    }
    __syncwarp();
    if (i & 1) {
      const int uo = u >> 1;
      if (ok) {
        *reinterpret_cast<float4*>(out + (int64_t)uo * 2 * d + lane * 4) = make_float4(a0, a1, a2, a3);
        *reinterpret_cast<float4*>(out + (int64_t)uo * 2 * d + d + lane * 4) = make_float4(b0, b1, b2, b3);
      }
      a0 = a1 = a2 = a3 = b0 = b1 = b2 = b3 = 0;
    }
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 14541, d = argc > 2 ? atoi(argv[2]) : 100;
  const int E = (argc > 3 ? atoi(argv[3]) : 600000) / 32 * 32;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<int> hidx(E);
  std::vector<float> hw(E);
  uint64_t x = 88172645463325252ull;
  for (int i = 0; i < E; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    hidx[i] = (int)(x % (uint64_t)n);
    hw[i] = 1.0f / (1 + (i & 7));
  }
  float *H, *w, *out;
  int* idx;
  CK(cudaMalloc(&H, (size_t)n * d * 4));
  CK(cudaMalloc(&w, (size_t)E * 4));
  CK(cudaMalloc(&idx, (size_t)E * 4));
  CK(cudaMalloc(&out, (size_t)E / 32 * 2 * d * 4 + 1024));
  CK(cudaMemset(H, 0, (size_t)n * d * 4));
  CK(cudaMemcpy(idx, hidx.data(), (size_t)E * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(w, hw.data(), (size_t)E * 4, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double bytes = (double)E * d * 4;
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    const int reps = 20;
    CK(cudaEventRecord(e0));
    for (int i = 0; i < reps; ++i) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double us = ms * 1e3 / reps;
    printf("%-14s %8.2f us  %6.2f TB/s gathered  (%d rows of %d B)\n", name, us, bytes / us * 1e-6, E, d * 4);
  };
  run("reg<4>", [&] { k_reg<4><<<sms * 4, 256>>>(H, idx, w, E, d, out); });
  run("reg<8>", [&] { k_reg<8><<<sms * 4, 256>>>(H, idx, w, E, d, out); });
  run("reg<16>", [&] { k_reg<16><<<sms * 4, 256>>>(H, idx, w, E, d, out); });
  auto bulk = [&](auto ns_tag, auto wpb_tag, const char* name) {
    constexpr int NS = decltype(ns_tag)::value, WPB = decltype(wpb_tag)::value;
    const size_t smem = (size_t)WPB * NS * 16 * d * 4;
    if (smem > 227 * 1024) { printf("%-14s skip (smem %zu)\n", name, smem); return; }
    CK(cudaFuncSetAttribute(k_bulk<NS, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    run(name, [&] { k_bulk<NS, WPB><<<sms, WPB * 32, smem>>>(H, idx, w, E, d, out); });
  };
  bulk(std::integral_constant<int, 2>{}, std::integral_constant<int, 16>{}, "bulk<2,16w>");
  bulk(std::integral_constant<int, 4>{}, std::integral_constant<int, 8>{}, "bulk<4,8w>");
  bulk(std::integral_constant<int, 3>{}, std::integral_constant<int, 12>{}, "bulk<3,12w>");
  bulk(std::integral_constant<int, 8>{}, std::integral_constant<int, 4>{}, "bulk<8,4w>");
  bulk(std::integral_constant<int, 6>{}, std::integral_constant<int, 6>{}, "bulk<6,6w>");
  bulk(std::integral_constant<int, 4>{}, std::integral_constant<int, 16>{}, "bulk<4,16w>");
  CK(cudaGetLastError());
  return 0;
}
