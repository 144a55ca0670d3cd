// Basis-transform GEMMs of the RGCN layer on the 5th-gen tensor cores.
//
//   NN  C[row(p), :] (+relu) = A[arow(p), 0:K] . B[0:K, 0:N]
//   TN  P_z[0:Mf, 0:N]       = sum_{p in split z} A[arow(p), 0:Mf]^T . Bm[p, 0:N]
//
// tcgen05.mma kind::tf32 with a 3xTF32 split (x = hi + lo, D += Ahi Bhi +
// Ahi Blo + Alo Bhi, ~fp32 accuracy; plain TF32 would break the 1e-4
// gradient tolerance). One persistent CTA per SM, 256
// threads; the fp32 accumulator (128 lanes x N_pad columns) lives in TMEM.
//
// Pipeline per K-chunk of 16 values:
//   cp.async   raw fp32 rows (gathered by a_rows, zero-filled at the edges)
//              into a 4-deep shared-memory ring, issued 3 chunks ahead
//   convert    all threads split the arrived chunk into hi/lo tf32 operands
//              in the K-major no-swizzle canonical UMMA layout (core matrices
//              of 8 rows x 16 B), double-buffered
//   mma        one elected thread issues 2 K-steps x 3 MMAs and commits them
//              to the operand buffer's mbarrier (reuse guard)
// so global-memory latency overlaps conversion and tensor-core work. The
// epilogue reads TMEM with tcgen05.ld (32x32b.x16; warps w and w+4 share
// lanes 32(w%4).. and split the columns) and applies ReLU / the row scatter.
#include "kg_gemm.cuh"

namespace kg {

constexpr int UM = 128;        // MMA M (rows per tile)
constexpr int UKC = 16;        // K values per chunk
constexpr int UKG = UKC / 4;   // 16-byte k-groups per chunk
constexpr int UNS = 4;         // raw ring depth
constexpr int UTHREADS = 256;

__host__ __device__ inline int pad16(int n) { return (n + 15) / 16 * 16; }

// byte offset of element (r, k) inside an R-row operand chunk (k < UKC)
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

__device__ __forceinline__ void sts128(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d));
}

// cp.async with zero fill: copies `bytes` (0 => all zeros) of a 16 B / 4 B slot
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp4(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Raw copy of a rows x cols fp32 block: row i = X + rowid(r0 + i) * ld + c0 (cols contiguous).
// Rows >= nrows / cols >= ncols are zero-filled. dst row stride = dcols floats.
__device__ __forceinline__ void copy_block(uint32_t dst, int dcols, const float* __restrict__ X, int64_t ld,
                                           const int32_t* __restrict__ rowid, int64_t r0, int64_t nrows, int rows,
                                           int64_t c0, int64_t ncols, int cols, bool vec) {
  if (vec) {
    const int per_row = cols / 4;
    for (int idx = threadIdx.x; idx < rows * per_row; idx += UTHREADS) {
      const int i = idx / per_row, q = idx % per_row;
      const int64_t row = r0 + i, col = c0 + 4 * q;
      int bytes = 0;
      const float* src = X;
      if (row < nrows && col < ncols) {
        const int64_t g = rowid ? (int64_t)__ldg(rowid + row) : row;
        src = X + g * ld + col;
        bytes = (int)((ncols - col) >= 4 ? 16 : (ncols - col) * 4);
      }
      cp16(dst + (uint32_t)((i * dcols + 4 * q) * 4), src, bytes);
    }
  } else {
    for (int idx = threadIdx.x; idx < rows * cols; idx += UTHREADS) {
      const int i = idx / cols, q = idx % cols;
      const int64_t row = r0 + i, col = c0 + q;
      int bytes = 0;
      const float* src = X;
      if (row < nrows && col < ncols) {
        const int64_t g = rowid ? (int64_t)__ldg(rowid + row) : row;
        src = X + g * ld + col;
        bytes = 4;
      }
      cp4(dst + (uint32_t)((i * dcols + q) * 4), src, bytes);
    }
  }
}

struct UmmaSmem {
  __host__ __device__ static size_t rawA() { return (size_t)UM * UKC * 4; }        // one raw A chunk
  __host__ __device__ static size_t rawB(int np) { return (size_t)np * UKC * 4; }  // one raw B chunk
  __host__ __device__ static size_t opA() { return (size_t)UM * UKC * 4; }
  __host__ __device__ static size_t opB(int np) { return (size_t)np * UKC * 4; }
  __host__ __device__ static size_t raw_stage(int np) { return rawA() + rawB(np); }
  __host__ __device__ static size_t op_buf(int np) { return 2 * opA() + 2 * opB(np); }
  __host__ __device__ static size_t total(int np) { return UNS * raw_stage(np) + 2 * op_buf(np) + 128; }
};

template <bool TN>
__global__ void __launch_bounds__(UTHREADS, 1) k_umma_gemm(GemmArgs g, int np, uint32_t tmem_cols) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_op[2];
  __shared__ uint64_t bar_done;
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t sbase = smem_u32(smem);
  auto raw_a = [&](int s) { return sbase + (uint32_t)(s * UmmaSmem::raw_stage(np)); };
  auto raw_b = [&](int s) { return sbase + (uint32_t)(s * UmmaSmem::raw_stage(np) + UmmaSmem::rawA()); };
  const uint32_t opbase = sbase + (uint32_t)(UNS * UmmaSmem::raw_stage(np));
  auto a_hi = [&](int b) { return opbase + (uint32_t)(b * UmmaSmem::op_buf(np)); };
  auto a_lo = [&](int b) { return a_hi(b) + (uint32_t)UmmaSmem::opA(); };
  auto b_hi = [&](int b) { return a_hi(b) + (uint32_t)(2 * UmmaSmem::opA()); };
  auto b_lo = [&](int b) { return b_hi(b) + (uint32_t)UmmaSmem::opB(np); };
  const float* rawf = reinterpret_cast<const float*>(smem);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar_op[0], 1);
    mbar_init(&bar_op[1], 1);
    mbar_init(&bar_done, 1);
    fence_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  const uint32_t idesc = make_idesc(np);

  const int64_t M = g.M_dev ? (int64_t)g.M_dev[g.M_dev_index] : g.M;
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
  const int64_t mf0 = TN ? (int64_t)blockIdx.y * UM : 0;            // TN feature tile
  const int64_t mf_n = TN ? (g.K - mf0 < UM ? g.K - mf0 : UM) : 0;
  // 16-byte cp.async needs 16-byte aligned rows; otherwise 4-byte copies
  const bool a16 = ((uintptr_t)g.A & 15) == 0, b16 = ((uintptr_t)g.B & 15) == 0;
  const bool vecA = a16 && (g.lda & 3) == 0 && (!TN || (mf0 & 3) == 0);
  const bool vecB = b16 && (g.ldb & 3) == 0;
  uint32_t ph_op[2] = {0, 0}, ph_done = 0;
  int64_t gop = 0;   // operand-buffer uses (buffer = gop & 1)

  for (int64_t tile = TN ? 0 : blockIdx.x; tile < ntiles; tile += TN ? 1 : gridDim.x) {
    const int64_t m0 = TN ? mf0 : tile * UM;
    const int nk = (int)((k_hi - k_lo + UKC - 1) / UKC);
    if (nk == 0) continue;
    // issue raw chunk kc into ring slot kc % UNS (one commit group per chunk)
    auto issue = [&](int kc) {
      if (kc < nk) {
        const int s = kc % UNS;
        const int64_t kb = k_lo + (int64_t)kc * UKC;
        if (!TN) {
          // A rows m0.. (gathered), K columns kb..kb+UKC; raw[r][k]
          copy_block(raw_a(s), UKC, g.A, g.lda, g.a_rows, m0, M, UM, kb, g.K, UKC, vecA && (kb & 3) == 0);
          // B rows kb.. (K x N row-major); raw[k][n]
          copy_block(raw_b(s), np, g.B, g.ldb, nullptr, kb, g.K, UKC, 0, g.N, np, vecB);
        } else {
          // A^T: data rows kb.. (gathered), feature columns mf0..; raw[k][m]
          copy_block(raw_a(s), UM, g.A, g.lda, g.a_rows, kb, k_hi, UKC, mf0, g.K, UM, vecA);
          copy_block(raw_b(s), np, g.B, g.ldb, nullptr, kb, k_hi, UKC, 0, g.N, np, vecB);
        }
      }
      cp_commit();   // uniform group accounting (empty groups past the end)
    };
#pragma unroll
    for (int j = 0; j < UNS - 1; ++j) issue(j);
    for (int kc = 0; kc < nk; ++kc) {
      issue(kc + UNS - 1);
      cp_wait<UNS - 1>();   // this thread's copies of chunk kc have landed
      const int ob = (int)(gop & 1);
      if (gop >= 2) {
        mbar_wait(&bar_op[ob], ph_op[ob]);   // MMAs that read this operand buffer are done
        ph_op[ob] ^= 1;
      }
      __syncthreads();                       // every thread's copies of chunk kc are visible
      const int s = kc % UNS;
      const float* ra = rawf + (size_t)s * UmmaSmem::raw_stage(np) / 4;
      const float* rb = ra + UmmaSmem::rawA() / 4;
      // convert: A (UM x UKC) and B (np x UKC) into hi/lo operands
      for (int idx = tid; idx < (UM + np) * UKG; idx += UTHREADS) {
        float v[4];
        uint32_t hib, lob, off;
        if (idx < UM * UKG) {
          const int r = idx % UM, gq = idx / UM;
#pragma unroll
          for (int i = 0; i < 4; ++i) v[i] = TN ? ra[(gq * 4 + i) * UM + r] : ra[r * UKC + gq * 4 + i];
          hib = a_hi(ob);
          lob = a_lo(ob);
          off = tile_off(r, gq * 4, UM);
        } else {
          const int j = idx - UM * UKG;
          const int n = j % np, gq = j / np;
#pragma unroll
          for (int i = 0; i < 4; ++i) v[i] = rb[(gq * 4 + i) * np + n];
          hib = b_hi(ob);
          lob = b_lo(ob);
          off = tile_off(n, gq * 4, np);
        }
        float h[4], l[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) split_tf32(v[i], h[i], l[i]);
        sts128(hib + off, h[0], h[1], h[2], h[3]);
        sts128(lob + off, l[0], l[1], l[2], l[3]);
      }
      fence_async_smem();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const uint32_t lbo_a = (UM / 8) * 128, lbo_b = (uint32_t)(np / 8) * 128;
#pragma unroll
        for (int j = 0; j < UKC / 8; ++j) {
          const uint32_t ka = (uint32_t)(2 * j) * lbo_a, kbb = (uint32_t)(2 * j) * lbo_b;
          uint64_t dah = make_desc(a_hi(ob) + ka, lbo_a, 128), dal = make_desc(a_lo(ob) + ka, lbo_a, 128);
          uint64_t dbh = make_desc(b_hi(ob) + kbb, lbo_b, 128), dbl = make_desc(b_lo(ob) + kbb, lbo_b, 128);
          const uint32_t acc = (kc > 0 || j > 0) ? 1u : 0u;
          mma_tf32(tmem, dah, dbh, idesc, acc);
          mma_tf32(tmem, dah, dbl, idesc, 1u);
          mma_tf32(tmem, dal, dbh, idesc, 1u);
        }
        mma_commit(&bar_op[ob]);
      }
      ++gop;
    }
    cp_wait<0>();
    if (tid == 0) mma_commit(&bar_done);
    mbar_wait(&bar_done, ph_done);
    ph_done ^= 1;
    tc_fence_after();
    // epilogue: warps w and w+4 read TMEM lanes [32(w%4), +32) and split the columns
    const int lanegrp = warp & 3;
    const int r = lanegrp * 32 + (tid & 31);
    const int64_t m = m0 + r;
    const int64_t out_rows = TN ? g.K : M;
    float* crow = nullptr;
    if (m < out_rows) {
      if (!TN) crow = g.C + (g.c_rows ? (int64_t)g.c_rows[m] : m) * g.ldc;
      else crow = g.C + ((int64_t)blockIdx.x * g.K + m) * g.ldc;
    }
    const int nchunks = np / 16;
    for (int cidx = (warp >> 2); cidx < nchunks; cidx += 2) {
      const int c0 = cidx * 16;
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(lanegrp * 32) << 16) + (uint32_t)c0, v);
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
  // TN CTAs with an empty row range still own a partial slot: zero it
  if (TN && k_lo >= k_hi) {
    for (int idx = tid; idx < UM * g.N; idx += UTHREADS) {
      int64_t m = mf0 + idx / g.N;
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
    KG_CUDA(cudaFuncSetAttribute(k_umma_gemm<TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr_set[TN] = true;
  }
  KG_REQUIRE(smem <= 220 * 1024, KG_ERR_SHAPE, "umma tile too large (N_pad %d)", np);
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
  // >= 64 data rows (4 chunks) per split, at most one CTA per SM
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
