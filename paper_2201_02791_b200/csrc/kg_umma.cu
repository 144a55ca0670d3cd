// Basis-transform GEMMs of the RGCN layer on the 5th-gen tensor cores.
//
//   NN  C[row(p), :] (+relu) = A[arow(p), 0:K] . B[0:K, 0:N]
//   TN  P_z[0:Mf, 0:N]       = sum_{p in split z} A[arow(p), 0:Mf]^T . Bm[p, 0:N]
//
// tcgen05.mma kind::tf32 with 3xTF32 split (x = hi + lo, D += Ahi Bhi +
// Ahi Blo + Alo Bhi, ~fp32 accuracy: plain TF32 would break the 1e-4
// gradient tolerance). One CTA per SM (persistent), 128
// threads; the accumulator (128 lanes x N_pad fp32 columns) lives in TMEM.
// Operand chunks of 32 K-values are staged by all threads into shared memory
// in the K-major no-swizzle canonical UMMA layout (core matrices of 8 rows x
// 16 B), split into hi/lo on the way, double-buffered; one elected thread
// issues the MMAs and commits them to per-stage mbarriers, so staging of
// chunk k+1 overlaps the tensor-core work of chunk k. The epilogue reads
// TMEM with tcgen05.ld (32x32b.x16) and applies ReLU / the row scatter.
#include "kg_gemm.cuh"

namespace kg {

constexpr int UM = 128;        // MMA M (rows per tile)
constexpr int UKC = 32;        // K values staged per chunk
constexpr int UKG = UKC / 4;   // 16-byte k-groups per chunk
constexpr int UTHREADS = 128;

__host__ __device__ inline int pad16(int n) { return (n + 15) / 16 * 16; }

// byte offset of element (r, k) inside an R-row chunk tile (k < UKC)
__device__ __forceinline__ uint32_t tile_off(int r, int k, int R) {
  return (uint32_t)(((k >> 2) * (R >> 3) + (r >> 3)) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: LBO = k-group stride, SBO = 8-row-group stride (bytes)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                       // version 1 (sm_100)
  return d;                                     // base offset 0, layout SWIZZLE_NONE
}

__device__ __forceinline__ uint32_t make_idesc(int n_pad) {
  return (1u << 4)                              // D format f32
         | (2u << 7) | (2u << 10)               // A, B format tf32
         | ((uint32_t)(n_pad >> 3) << 17)       // N
         | ((uint32_t)(UM >> 4) << 24);         // M
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));   // nearest tf32: |lo| <= 2^-12 |x|
  hi = __uint_as_float(h);
  lo = x - hi;
}

// no "memory" clobber: ordering against the MMA is established by
// fence.proxy.async + __syncthreads, and global loads must stay free to be
// hoisted above earlier stores
__device__ __forceinline__ void sts128(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d));
}

__device__ __forceinline__ void store_split(uint32_t hi_base, uint32_t lo_base, uint32_t off, const float* v) {
  float h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) split_tf32(v[i], h[i], l[i]);
  sts128(hi_base + off, h[0], h[1], h[2], h[3]);
  sts128(lo_base + off, l[0], l[1], l[2], l[3]);
}

// Stage rows-by-K operand: element (r, k) = X[rowid(r0 + r)][kb + k], k contiguous.
// Warp instruction covers 8 rows x 4 k-groups (16 B each); all of a thread's
// loads are issued before any split/store (8 x 16 B in flight per thread).
__device__ __forceinline__ void stage_rowsK(uint32_t hi_base, uint32_t lo_base, const float* __restrict__ X, int64_t ldx,
                                            const int32_t* __restrict__ rowid, int64_t r0, int64_t rows, int64_t kb,
                                            int64_t K, int R) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int rr = lane & 7, gg = lane >> 3;
  const bool vec = ((ldx & 3) == 0) && ((kb & 3) == 0);
  constexpr int IT = (UM / 8) * (UKG / 4) / (UTHREADS / 32);   // 8 items per thread for R = 128
  float v[IT][4];
#pragma unroll
  for (int q = 0; q < IT; ++q) {
    const int it = warp + q * (UTHREADS / 32);
    const int rg = it % (R / 8);
    const int g = (it / (R / 8)) * 4 + gg;
    const int r = rg * 8 + rr;
    v[q][0] = v[q][1] = v[q][2] = v[q][3] = 0.f;
    const int64_t row = r0 + r;
    if (row < rows) {
      const int64_t grow = rowid ? (int64_t)__ldg(rowid + row) : row;
      const float* p = X + grow * ldx + kb + g * 4;
      const int64_t k0 = kb + g * 4;
      if (vec && k0 + 4 <= K) {
        float4 t = __ldg(reinterpret_cast<const float4*>(p));
        v[q][0] = t.x; v[q][1] = t.y; v[q][2] = t.z; v[q][3] = t.w;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (k0 + i < K) v[q][i] = __ldg(p + i);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < IT; ++q) {
    const int it = warp + q * (UTHREADS / 32);
    const int rg = it % (R / 8);
    const int g = (it / (R / 8)) * 4 + gg;
    store_split(hi_base, lo_base, tile_off(rg * 8 + rr, g * 4, R), v[q]);
  }
}

// Stage cols-by-K operand: element (r, k) = X[rowid(kb + k)][r], r contiguous;
// batches of 8 items (32 loads) in flight per thread.
__device__ __forceinline__ void stage_colsK(uint32_t hi_base, uint32_t lo_base, const float* __restrict__ X, int64_t ldx,
                                            const int32_t* __restrict__ rowid, int64_t kb, int64_t kend, int ncols, int R) {
  constexpr int BATCH = 8;
  const int total = R * UKG;
  for (int base = threadIdx.x; base < total; base += BATCH * UTHREADS) {
    float v[BATCH][4];
#pragma unroll
    for (int q = 0; q < BATCH; ++q) {
      const int idx = base + q * UTHREADS;
      const int r = idx % R, g = idx / R;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t kk = kb + g * 4 + i;
        float x = 0.f;
        if (idx < total && r < ncols && kk < kend) {
          const int64_t grow = rowid ? (int64_t)__ldg(rowid + kk) : kk;
          x = __ldg(X + grow * ldx + r);
        }
        v[q][i] = x;
      }
    }
#pragma unroll
    for (int q = 0; q < BATCH; ++q) {
      const int idx = base + q * UTHREADS;
      if (idx < total) store_split(hi_base, lo_base, tile_off(idx % R, (idx / R) * 4, R), v[q]);
    }
  }
}

struct UmmaSmem {
  // per stage: A hi, A lo (UM x UKC), B hi, B lo (NP x UKC)
  __host__ __device__ static size_t a_bytes() { return (size_t)UM * UKC * 4; }
  __host__ __device__ static size_t b_bytes(int np) { return (size_t)np * UKC * 4; }
  __host__ __device__ static size_t stage_bytes(int np) { return 2 * a_bytes() + 2 * b_bytes(np); }
  __host__ __device__ static size_t total(int np) { return 2 * stage_bytes(np) + 128; }
};

template <bool TN>
__global__ void __launch_bounds__(UTHREADS, 1) k_umma_gemm(GemmArgs g, int np, uint32_t tmem_cols) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_stage[2];
  __shared__ uint64_t bar_done;
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t sbase = smem_u32(smem);
  const size_t SB = UmmaSmem::stage_bytes(np);
  auto a_hi = [&](int s) { return sbase + (uint32_t)(s * SB); };
  auto a_lo = [&](int s) { return sbase + (uint32_t)(s * SB + UmmaSmem::a_bytes()); };
  auto b_hi = [&](int s) { return sbase + (uint32_t)(s * SB + 2 * UmmaSmem::a_bytes()); };
  auto b_lo = [&](int s) { return sbase + (uint32_t)(s * SB + 2 * UmmaSmem::a_bytes() + UmmaSmem::b_bytes(np)); };

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar_stage[0], 1);
    mbar_init(&bar_stage[1], 1);
    mbar_init(&bar_done, 1);
    fence_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  const uint32_t idesc = make_idesc(np);

  const int64_t M = g.M_dev ? (int64_t)g.M_dev[g.M_dev_index] : g.M;
  // NN: tiles over data rows, reduce over g.K. TN: one tile of features (blockIdx.y), reduce over this CTA's rows.
  int64_t ntiles, k_lo = 0, k_hi;
  if (!TN) {
    ntiles = (M + UM - 1) / UM;
    k_hi = g.K;
  } else {
    ntiles = 1;
    int64_t per = (M + gridDim.x - 1) / gridDim.x;
    per = (per + UKC - 1) / UKC * UKC;
    k_lo = (int64_t)blockIdx.x * per;
    k_hi = k_lo + per < M ? k_lo + per : M;
  }
  uint32_t ph_stage[2] = {0, 0}, ph_done = 0;
  int64_t gc = 0;   // global chunk counter (stage = gc & 1)
  for (int64_t tile = TN ? 0 : blockIdx.x; tile < ntiles; tile += TN ? 1 : gridDim.x) {
    const int64_t m0 = TN ? (int64_t)blockIdx.y * UM : tile * UM;
    int kc = 0;
    for (int64_t kb = k_lo; kb < k_hi; kb += UKC, ++kc, ++gc) {
      const int s = (int)(gc & 1);
      if (gc >= 2) {
        mbar_wait(&bar_stage[s], ph_stage[s]);
        ph_stage[s] ^= 1;
      }
      if (!TN) {
        stage_rowsK(a_hi(s), a_lo(s), g.A, g.lda, g.a_rows, m0, M, kb, g.K, UM);
        stage_colsK(b_hi(s), b_lo(s), g.B, g.ldb, nullptr, kb, g.K, (int)g.N, np);
      } else {
        // A^T: element (feature m, data row k) = A[arow(k)][m0 + m]
        stage_colsK(a_hi(s), a_lo(s), g.A + m0, g.lda, g.a_rows, kb, k_hi, (int)(g.K - m0 < UM ? g.K - m0 : UM), UM);
        stage_colsK(b_hi(s), b_lo(s), g.B, g.ldb, nullptr, kb, k_hi, (int)g.N, np);
      }
      fence_async_smem();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
#pragma unroll
        for (int j = 0; j < UKC / 8; ++j) {
          const uint32_t lbo_a = (UM / 8) * 128, lbo_b = (uint32_t)(np / 8) * 128;
          const uint32_t koff_a = (uint32_t)(2 * j) * lbo_a, koff_b = (uint32_t)(2 * j) * lbo_b;
          uint64_t dah = make_desc(a_hi(s) + koff_a, lbo_a, 128), dal = make_desc(a_lo(s) + koff_a, lbo_a, 128);
          uint64_t dbh = make_desc(b_hi(s) + koff_b, lbo_b, 128), dbl = make_desc(b_lo(s) + koff_b, lbo_b, 128);
          const uint32_t acc = (kc > 0 || j > 0) ? 1u : 0u;
          mma_tf32(tmem, dah, dbh, idesc, acc);
          mma_tf32(tmem, dah, dbl, idesc, 1u);
          mma_tf32(tmem, dal, dbh, idesc, 1u);
        }
        mma_commit(&bar_stage[s]);
      }
    }
    if (kc == 0) continue;   // empty reduction range (TN split with no rows)
    if (tid == 0) mma_commit(&bar_done);
    mbar_wait(&bar_done, ph_done);
    ph_done ^= 1;
    tc_fence_after();
    // epilogue: warp w owns TMEM lanes / tile rows [32w, 32w+32)
    const int r = warp * 32 + (tid & 31);
    const int64_t m = m0 + r;
    const int64_t out_rows = TN ? g.K : M;
    float* crow = nullptr;
    if (m < out_rows) {
      if (!TN) crow = g.C + (g.c_rows ? (int64_t)g.c_rows[m] : m) * g.ldc;
      else crow = g.C + ((int64_t)blockIdx.x * g.K + m) * g.ldc;
    }
    for (int c0 = 0; c0 < np; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
      if (crow) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int64_t n = c0 + i;
          if (n < g.N) crow[n] = g.relu ? fmaxf(v[i], 0.f) : v[i];
        }
      }
    }
    tc_fence_before();
    __syncthreads();
  }
  // TN CTAs with an empty range still own a partial slot: zero it
  if (TN && k_lo >= k_hi) {
    for (int idx = tid; idx < UM * g.N; idx += UTHREADS) {
      int64_t m = (int64_t)blockIdx.y * UM + idx / g.N;
      if (m < g.K) g.C[((int64_t)blockIdx.x * g.K + m) * g.ldc + idx % g.N] = 0.f;
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
}

static uint32_t tmem_cols_for(int np) {
  uint32_t c = 32;
  while ((int)c < np) c <<= 1;
  return c;
}

template <bool TN>
static kg_status launch_umma(const GemmArgs& g, int np, dim3 grid, cudaStream_t st) {
  size_t smem = UmmaSmem::total(np);
  static bool attr_set[2] = {false, false};
  if (!attr_set[TN]) {
    KG_CUDA(cudaFuncSetAttribute(k_umma_gemm<TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_set[TN] = true;
  }
  KG_REQUIRE(smem <= 200 * 1024, KG_ERR_SHAPE, "umma tile too large (N_pad %d)", np);
  KG_LAUNCH(TN ? "k_umma_gemm_tn" : "k_umma_gemm_nn", k_umma_gemm<TN>, grid, UTHREADS, smem, st, g, np,
            tmem_cols_for(np));
  return KG_OK;
}

kg_status umma_gemm_nn(const GemmArgs& g, cudaStream_t st) {
  if (g.M_max <= 0 || g.N <= 0) return KG_OK;
  KG_REQUIRE(g.N <= 256, KG_ERR_SHAPE, "umma NN supports N <= 256 (got %lld)", (long long)g.N);
  int np = pad16((int)g.N);
  int64_t tiles = ceil_div(g.M_max, UM);
  int ctas = (int)(tiles < num_sms() ? tiles : num_sms());
  return launch_umma<false>(g, np, dim3(ctas, 1, 1), st);
}

int umma_tn_splits(int64_t rows_max) {
  // >= 64 data rows (2 chunks) per split, at most one CTA per SM
  int64_t s = ceil_div(rows_max, 64);
  if (s > num_sms()) s = num_sms();
  return (int)(s < 1 ? 1 : s);
}

kg_status umma_gemm_tn(const GemmArgs& g, float* out, void* ws, cudaStream_t st) {
  KG_REQUIRE(g.N <= 256, KG_ERR_SHAPE, "umma TN supports N <= 256");
  int np = pad16((int)g.N);
  int splits = umma_tn_splits(g.M_max);
  GemmArgs h = g;
  h.C = static_cast<float*>(ws);
  h.ldc = g.N;
  dim3 grid((unsigned)splits, (unsigned)ceil_div(g.K, UM), 1);
  kg_status s = launch_umma<true>(h, np, grid, st);
  if (s != KG_OK) return s;
  return reduce_splits(h.C, splits, g.K * g.N, out, st);
}

size_t umma_tn_workspace(int64_t rows_max, int64_t K, int64_t N) {
  return align_up((size_t)umma_tn_splits(rows_max) * K * N * sizeof(float));
}

}  // namespace kg
