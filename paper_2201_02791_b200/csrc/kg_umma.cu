// Basis-transform GEMMs of the RGCN layer on the 5th-gen tensor cores.
//
//   NN  C[row(p), :] (+relu) = A[arow(p), 0:K] . B[0:K, 0:N]
//   TN  P_z[0:Mf, 0:N]       = sum_{p in split z} A[arow(p), 0:Mf]^T . Bm[p, 0:N]
//
// tcgen05.mma kind::tf32 with a 3xTF32 split (x = hi + lo, D += Ahi Bhi +
// Ahi Blo + Alo Bhi, ~fp32 accuracy; plain TF32 would break the 1e-4
// gradient tolerance).
//
// Two kernels per GEMM:
//   k_umma_pack    high-occupancy elementwise pass: gathers the operand rows
//                  and writes them (fp32) in the K-major 64-byte-swizzle
//                  canonical UMMA layout, one contiguous "record" per (row
//                  block, 16-wide K chunk). Both operands of a GEMM are
//                  packed by one launch; producers that can (k_aggregate,
//                  the GEMM epilogue, the dS pass) write records directly.
//   k_umma_packed  warp-specialised tensor-core loop: warp 0 lane 0 streams
//                  fp32 records into a shared-memory ring with cp.async.bulk
//                  (mbarrier transaction counting); warps 6..9 split each
//                  staged record in place into tf32 hi + lo halves (so HBM
//                  and L2 carry 4 bytes per operand value, not 8); warp 1
//                  lane 0 issues the 2 K-steps x 3 MMAs per record and
//                  commits them to the slot's "empty" barrier; warps 2..5
//                  drain the fp32 accumulator from TMEM (tcgen05.ld 32x32b)
//                  and apply ReLU / the row scatter. Two TMEM accumulators let
//                  the epilogue of tile i overlap the MMAs of tile i+1.
// The earliest variant converted row-major operands inside the GEMM with its
// own address math and was issue-latency bound at one CTA per SM
// (profiles/r1_v11_umma_stalls.txt); the split here is a flat elementwise
// pass over a staged record.
#include "kg_gemm.cuh"

namespace kg {

constexpr int UM = PK_ROWS;    // MMA M (rows per tile)
constexpr int UKC = PK_K;      // K values per record
constexpr int UMAXS = 8;       // max ring stages
constexpr int UTHREADS = 320;  // producer warp, MMA warp, 4 epilogue warps, 4 split warps
constexpr int USPLIT0 = 6;     // first split warp
constexpr size_t USMEM_CAP = 200 * 1024;

__host__ __device__ inline int pad16(int n) { return (n + 15) / 16 * 16; }

// byte offset of element (r, k) inside a record half (k < UKC)
__host__ __device__ __forceinline__ uint32_t tile_off(int r, int k, int R) {
  (void)R;
  return (uint32_t)pk_off(r, k) * 4u;
}
// floats per GEMM operand record in global memory (fp32)
__host__ __device__ inline int64_t rec_floats(int R) { return (int64_t)R * UKC; }
// floats per ranking record (tf32 hi + lo halves, split at pack time)
__host__ __device__ inline int64_t rec_floats_split(int R) { return (int64_t)2 * R * UKC; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, 64-byte swizzle (pk_off): SBO = 512 B between 8-row groups, LBO
// unused (16 B). Records sit at 512-byte aligned shared addresses (base offset
// 0); the second tf32 K-step of a record starts 32 B into the swizzle atom.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                       // LBO 16 B (ignored for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;              // SBO
  d |= (uint64_t)1 << 46;                       // version 1 (sm_100)
  d |= (uint64_t)4 << 61;                       // layout SWIZZLE_64B
  return d;
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

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

// 1-D bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
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

// ---------------------------------------------------------------------------
// Operand packing.
//   rows mode (cols_mode = 0): MMA row = source row (gathered by rowid, count
//     nrows, possibly on the device), k = source column (static, ncols).
//   cols mode (cols_mode = 1): MMA row = source column (static), k = source
//     row (gathered, count possibly on the device).
// Record (blk, kc) lives at out + (blk * nk_alloc + kc) * rec_floats(R);
// entries past the valid rows / columns are written as zeros.
struct PackJob {
  const float* src;
  int64_t ld;
  const int32_t* rowid;
  const int32_t* nrows_dev;
  int nrows_idx;
  int64_t nrows;      // if nrows_dev == nullptr
  int64_t ncols;
  int R;              // record rows (128 for A, N_pad for B)
  int cols_mode;
  int64_t nk_alloc;   // records per block in the layout
  float* out;
  int split;          // 1: ranking records (hi | lo halves), 0: fp32 GEMM records
};

__device__ __forceinline__ void pack_store(float* rec, int R, int r, int q, const float* v, int split) {
  const uint32_t off = tile_off(r, 4 * q, R) >> 2;
  if (!split) {
    *reinterpret_cast<float4*>(rec + off) = make_float4(v[0], v[1], v[2], v[3]);
    return;
  }
  float h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) split_tf32(v[i], h[i], l[i]);
  *reinterpret_cast<float4*>(rec + off) = make_float4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<float4*>(rec + (int64_t)R * UKC + off) = make_float4(l[0], l[1], l[2], l[3]);
}

// One block per record (grid-stride over records): the per-element index
// decode is shifts and compares only (the first version's 64-bit div/mod per
// element made the transposed packs compute-bound at wikikg2 scale).
__global__ void __launch_bounds__(256) k_umma_pack(PackJob j0, PackJob j1) {
  const PackJob& j = blockIdx.y == 0 ? j0 : j1;
  if (!j.src) return;
  const int64_t nrows = j.nrows_dev ? (int64_t)j.nrows_dev[j.nrows_idx] : j.nrows;
  const int R = j.R;
  if (!j.cols_mode) {
    // record (blk, kc): items (r, q), q fastest -> 4 lanes read 64 B of one row
    const int64_t nk = j.nk_alloc, nrec = (nrows + R - 1) / R * nk;
    const bool vec = ((uintptr_t)j.src & 15) == 0 && (j.ld & 3) == 0;
    for (int64_t rec = blockIdx.x; rec < nrec; rec += gridDim.x) {
      const int64_t blk = rec / nk, kc = rec - blk * nk;
      float* out = j.out + rec * (j.split ? rec_floats_split(R) : rec_floats(R));
      for (int i = threadIdx.x; i < R * 4; i += blockDim.x) {
        const int q = i & 3, r = i >> 2;
        const int64_t row = blk * R + r, c0 = kc * UKC + 4 * q;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (row < nrows) {
          const float* src = j.src + (j.rowid ? (int64_t)__ldg(j.rowid + row) : row) * j.ld;
          if (vec && c0 + 3 < j.ncols) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(src + c0));
            v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
          } else {
#pragma unroll
            for (int t = 0; t < 4; ++t)
              if (c0 + t < j.ncols) v[t] = __ldg(src + c0 + t);
          }
        }
        pack_store(out, R, r, q, v, j.split);
      }
    }
  } else {
    // record (blk, kc) with kc over 16-row groups of the source: a warp owns
    // 8 MMA rows x 4 K chunks, so each store fills one 512-byte swizzle atom
    // and each load reads 8 consecutive source columns (one sector) of a row
    const int64_t nkd = (nrows + UKC - 1) / UKC, nblk = (j.ncols + R - 1) / R;
    // the record's 16 source rows: offsets staged once per record (the
    // gathered row ids were re-read by every item: the pass was issue-bound)
    __shared__ int64_t roff[UKC];
    for (int64_t rec = blockIdx.x; rec < nblk * nkd; rec += gridDim.x) {
      const int64_t blk = rec / nkd, kc = rec - blk * nkd;
      float* out = j.out + (blk * j.nk_alloc + kc) * (j.split ? rec_floats_split(R) : rec_floats(R));
      __syncthreads();   // the previous record's readers are done
      if (threadIdx.x < UKC) {
        const int64_t k = kc * UKC + threadIdx.x;
        roff[threadIdx.x] = k < nrows ? (j.rowid ? (int64_t)__ldg(j.rowid + k) : k) * j.ld : -1;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < R * 4; i += blockDim.x) {
        const int q = (i >> 3) & 3, m = ((i >> 5) << 3) + (i & 7);
        const int64_t col = blk * R + m;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (col < j.ncols) {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int64_t o = roff[4 * q + t];
            if (o >= 0) v[t] = __ldg(j.src + o + col);
          }
        }
        pack_store(out, R, m, q, v, j.split);
      }
    }
  }
}

// ---------------------------------------------------------------------------
struct PackedArgs {
  const float* Ap;        // A records, R = UM
  const float* Bp;        // B records, R = np (single block)
  int64_t a_nk_alloc;     // records per A block
  int np;
  // NN: tiles = ceil(M / UM), every tile uses records kc in [0, nk)
  // TN: CTA (x, y) uses A block y and records [x*per, ...) of nk_dyn
  int tn;
  int64_t M;              // NN rows / TN data rows (if M_dev == nullptr)
  const int32_t* M_dev;
  int M_dev_index;
  int64_t nk;             // NN: static record count
  float* C;
  int64_t ldc;
  const int32_t* c_rows;
  int64_t N;
  int64_t out_rows;       // TN: feature rows (g.K)
  int relu;
  float* c_packed;        // NN: optional packed copy of the output (records by MMA row, K = np)
  int64_t c_nk;
  const float* mul;       // NN: optional per-element output scale by MMA row (ld N)
  int a_split;            // A records already hold hi | lo halves (records_split of the row capacity)
  int b_split;            // B records already hold hi | lo halves (NN: weights, split once per step)
  int exp;                // diagnostics (KG_GEMM_EXP, NN): 1 no epilogue stores, 2 no MMAs
};

__device__ __forceinline__ uint32_t stage_bytes(int np) { return (uint32_t)((UM + np) * UKC * 2 * 4); }

// NN epilogue staging: per epilogue warp a 32-row x 32-column slab (row
// stride EP_LD floats: conflict-free float4 writes by row and reads by column)
constexpr int EP_LD = 36;
constexpr size_t EP_SLAB_BYTES = (size_t)4 * 32 * EP_LD * sizeof(float);

// NN epilogue of one warp's 32 accumulator rows, 32 columns at a time: the
// TMEM rows (one per lane) go through a shared-memory slab so that global
// stores are row-contiguous (8 lanes x float4 per row segment) instead of one
// row per lane (a warp store touching 32 rows), and the packed copy of the
// output is written as whole 512-byte swizzle atoms (one coalesced float4 per
// lane). ReLU, then the per-element scale (dropout), as before.
__device__ __forceinline__ void nn_epilogue(const PackedArgs& g, uint32_t taddr, int64_t tile, int lanegrp, int lane,
                                            int64_t M, int np, bool vec, float* slab) {
  const int64_t m0 = tile * UM + lanegrp * 32;   // first output row (MMA row) of this warp
  const int64_t ml = m0 + lane;
  const int64_t crow_l = ml < M ? (g.c_rows ? (int64_t)__ldg(g.c_rows + ml) : ml) : -1;
  const bool mul_vec = g.mul && (g.N & 3) == 0 && ((uintptr_t)g.mul & 15) == 0;
  const int64_t pnk = g.c_nk < 0 ? -g.c_nk : g.c_nk;
  for (int c0 = 0; c0 < np; c0 += 32) {
    float v[32];
    tmem_ld16(taddr + (uint32_t)c0, v);
    tmem_ld16(taddr + (uint32_t)c0 + 16u, v + 16);
    if (g.relu) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      *reinterpret_cast<float4*>(slab + lane * EP_LD + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    __syncwarp();
    // row segments: lane -> (row it * 4 + lane / 8, column quad lane % 8)
    const int q = lane & 7;
    const int col = c0 + 4 * q;
#pragma unroll 2
    for (int it = 0; it < 8; ++it) {
      const int rr = it * 4 + (lane >> 3);
      const int64_t crow = __shfl_sync(0xffffffffu, crow_l, rr);
      float4* sp = reinterpret_cast<float4*>(slab + rr * EP_LD + 4 * q);
      float4 x = *sp;
      if (crow >= 0 && col < g.N) {
        const int64_t m = m0 + rr;
        if (g.mul) {
          if (mul_vec) {
            const float4 s = __ldg(reinterpret_cast<const float4*>(g.mul + m * g.N + col));
            x.x *= s.x; x.y *= s.y; x.z *= s.z; x.w *= s.w;
          } else {
            float* xv = reinterpret_cast<float*>(&x);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (col + i < g.N) xv[i] *= __ldg(g.mul + m * g.N + col + i);
          }
          if (g.c_packed) *sp = x;
        }
        float* dst = g.C + crow * g.ldc + col;
        if (vec && col + 3 < g.N) {
          *reinterpret_cast<float4*>(dst) = x;
        } else {
          const float* xv = reinterpret_cast<const float*>(&x);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (col + i < g.N) dst[i] = xv[i];
        }
      }
    }
    if (g.c_packed) {
      __syncwarp();
      // records kc = c0/16 + j: this warp's rows are 4 swizzle atoms of 8 rows;
      // lane i writes 16-byte chunk i of an atom = row i/4, K quad (i%4) ^ ((i/8)%4)
      const int ri = lane >> 2, kq = (lane & 3) ^ ((lane >> 3) & 3);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t kc = c0 / 16 + j;
        if (kc >= pnk) break;
        float* rec = g.c_packed + (tile * pnk + kc) * (g.c_nk < 0 ? 2 * PK_REC : PK_REC);
#pragma unroll
        for (int at = 0; at < 4; ++at) {
          const int rl = at * 8 + ri;
          float4 x = *reinterpret_cast<const float4*>(slab + rl * EP_LD + j * 16 + kq * 4);
          if (m0 + rl >= M) x = make_float4(0.f, 0.f, 0.f, 0.f);
          float* dst = rec + (lanegrp * 4 + at) * 128 + lane * 4;
          if (g.c_nk < 0) {
            float4 hi, lo;
            split_tf32(x.x, hi.x, lo.x);
            split_tf32(x.y, hi.y, lo.y);
            split_tf32(x.z, hi.z, lo.z);
            split_tf32(x.w, hi.w, lo.w);
            *reinterpret_cast<float4*>(dst) = hi;
            *reinterpret_cast<float4*>(dst + PK_REC) = lo;
          } else {
            *reinterpret_cast<float4*>(dst) = x;
          }
        }
      }
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(UTHREADS, 1) k_umma_packed(PackedArgs g, int nstages, uint32_t acc_cols) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_full[UMAXS], bar_empty[UMAXS], bar_split[UMAXS], bar_tfull[2], bar_tempty[2];
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int np = g.np;

  // work assignment
  const int64_t M = g.M_dev ? (int64_t)g.M_dev[g.M_dev_index] : g.M;
  int64_t ntiles, c_lo = 0, c_hi;
  if (!g.tn) {
    ntiles = (M + UM - 1) / UM;
    c_hi = g.nk;
  } else {
    ntiles = 1;
    const int64_t nkd = (M + UKC - 1) / UKC;
    const int64_t per = (nkd + gridDim.x - 1) / gridDim.x;
    c_lo = (int64_t)blockIdx.x * per;
    c_hi = c_lo + per < nkd ? c_lo + per : nkd;
    if (c_lo >= c_hi) {   // empty split: its partial slot is zero
      const int64_t mf0 = (int64_t)blockIdx.y * UM;
      for (int idx = tid; idx < UM * g.N; idx += UTHREADS) {
        const int64_t m = mf0 + idx / g.N;
        if (m < g.out_rows) g.C[((int64_t)blockIdx.x * g.out_rows + m) * g.ldc + idx % g.N] = 0.f;
      }
      return;
    }
  }
  const int64_t tile0 = g.tn ? 0 : blockIdx.x, tstep = g.tn ? 1 : gridDim.x;
  const int nk = (int)(c_hi - c_lo);
  if (tile0 >= ntiles) return;

  const uint32_t sbase = smem_u32(smem);
  const uint32_t sb = stage_bytes(np), a_half = (uint32_t)(UM * UKC * 4), b_half = (uint32_t)(np * UKC * 4);
  const uint32_t a_bytes = 2 * a_half;
  const bool presplit = g.a_split && g.b_split;   // nothing to split: the MMA waits on the loads
  auto full = [&](int s) { return smem_u32(&bar_full[s]); };
  auto empty = [&](int s) { return smem_u32(&bar_empty[s]); };

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(2 * acc_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
      mbar_init(smem_u32(&bar_split[s]), 4);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&bar_tfull[a]), 1);
      mbar_init(smem_u32(&bar_tempty[a]), 4);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    if (lane == 0) {
      // producer: stream (A record, B record) pairs through the ring
      int64_t it = 0;
      for (int64_t tile = tile0; tile < ntiles; tile += tstep) {
        const int64_t ablk = g.tn ? blockIdx.y : tile;
        const int64_t arf = g.a_split ? rec_floats_split(UM) : rec_floats(UM);
        const float* arec = g.Ap + (ablk * g.a_nk_alloc + c_lo) * arf;
        const uint32_t acopy = g.a_split ? 2 * a_half : a_half;
        const int64_t brf = g.b_split ? rec_floats_split(np) : rec_floats(np);
        const float* brec = g.Bp + c_lo * brf;
        const uint32_t bcopy = g.b_split ? 2 * b_half : b_half;
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = (int)(it % nstages);
          if (it >= nstages) mbar_wait(empty(s), (uint32_t)((it / nstages - 1) & 1));
          const uint32_t dst = sbase + (uint32_t)s * sb;
          mbar_expect_tx(full(s), acopy + bcopy);
          bulk_g2s(dst, arec + (int64_t)kc * arf, acopy, full(s));
          bulk_g2s(dst + a_bytes, brec + (int64_t)kc * brf, bcopy, full(s));
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // MMA issuer
      const uint32_t idesc = make_idesc(np);
      int64_t it = 0, tcount = 0;
      for (int64_t tile = tile0; tile < ntiles; tile += tstep, ++tcount) {
        const int acc = (int)(tcount & 1);
        if (tcount >= 2) mbar_wait(smem_u32(&bar_tempty[acc]), (uint32_t)((tcount / 2 - 1) & 1));
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)acc * acc_cols;
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = (int)(it % nstages);
          mbar_wait(presplit ? full(s) : smem_u32(&bar_split[s]), (uint32_t)((it / nstages) & 1));
          tc_fence_after();
          const uint32_t a_hi = sbase + (uint32_t)s * sb, a_lo = a_hi + a_half;
          const uint32_t b_hi = a_hi + a_bytes, b_lo = b_hi + b_half;
#pragma unroll
          for (int j = 0; j < UKC / 8; ++j) {
            if (g.exp & 2) break;
            const uint32_t ko = (uint32_t)j * 32u;
            const uint64_t dah = make_desc(a_hi + ko), dal = make_desc(a_lo + ko);
            const uint64_t dbh = make_desc(b_hi + ko), dbl = make_desc(b_lo + ko);
            mma_tf32(d, dah, dbh, idesc, (kc > 0 || j > 0) ? 1u : 0u);
            mma_tf32(d, dah, dbl, idesc, 1u);
            mma_tf32(d, dal, dbh, idesc, 1u);
          }
          mma_commit(empty(s));   // slot reusable once these MMAs have read it
        }
        mma_commit(smem_u32(&bar_tfull[acc]));
      }
    }
  } else if (warp >= USPLIT0) {
    if (presplit) ntiles = tile0;   // nothing to split: skip to the teardown barrier
    // split warps 6..9: each staged fp32 record becomes tf32 hi (in place) +
    // lo (the slot's second half), x = hi + lo exactly
    const int st = tid - USPLIT0 * 32;
    const int na = g.a_split ? 0 : UM * UKC / 4, nb = g.b_split ? 0 : np * UKC / 4;
    int64_t it = 0;
    for (int64_t tile = tile0; tile < ntiles; tile += tstep) {
      for (int kc = 0; kc < nk; ++kc, ++it) {
        const int s = (int)(it % nstages);
        mbar_wait(full(s), (uint32_t)((it / nstages) & 1));
        float* base = reinterpret_cast<float*>(smem + (size_t)s * sb);
        float4* ah = reinterpret_cast<float4*>(base);
        float4* al = reinterpret_cast<float4*>(base + UM * UKC);
        float4* bh = reinterpret_cast<float4*>(base + 2 * UM * UKC);
        float4* bl = reinterpret_cast<float4*>(base + 2 * UM * UKC + np * UKC);
        for (int i = st; i < na + nb; i += 128) {
          float4* h = i < na ? ah + i : bh + (i - na);
          float4* l = i < na ? al + i : bl + (i - na);
          const float4 x = *h;
          float4 hi, lo;
          split_tf32(x.x, hi.x, lo.x);
          split_tf32(x.y, hi.y, lo.y);
          split_tf32(x.z, hi.z, lo.z);
          split_tf32(x.w, hi.w, lo.w);
          *h = hi;
          *l = lo;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tcgen05 reads
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bar_split[s]));
      }
    }
  } else {
    // epilogue warps 2..5: TMEM lanes 32 * (warp % 4) ..
    const int lanegrp = warp & 3;
    const int r = lanegrp * 32 + lane;
    const bool vec = ((uintptr_t)g.C & 15) == 0 && (g.ldc & 3) == 0;
    float* slab = reinterpret_cast<float*>(smem + (size_t)nstages * sb) + lanegrp * 32 * EP_LD;
    int64_t tcount = 0;
    for (int64_t tile = tile0; tile < ntiles; tile += tstep, ++tcount) {
      const int acc = (int)(tcount & 1);
      mbar_wait(smem_u32(&bar_tfull[acc]), (uint32_t)((tcount / 2) & 1));
      tc_fence_after();
      if (!g.tn) {
        if (!(g.exp & 1))
          nn_epilogue(g, tmem + (uint32_t)acc * acc_cols + ((uint32_t)(lanegrp * 32) << 16), tile, lanegrp, lane, M, np,
                    vec, slab);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bar_tempty[acc]));
        continue;
      }
      float* crow = nullptr;
      if (!g.tn) {
        const int64_t m = tile * UM + r;
        if (m < M) crow = g.C + (g.c_rows ? (int64_t)__ldg(g.c_rows + m) : m) * g.ldc;
      } else {
        const int64_t m = (int64_t)blockIdx.y * UM + r;
        if (m < g.out_rows) crow = g.C + ((int64_t)blockIdx.x * g.out_rows + m) * g.ldc;
      }
      const uint32_t taddr = tmem + (uint32_t)acc * acc_cols + ((uint32_t)(lanegrp * 32) << 16);
      for (int c0 = 0; c0 < np; c0 += 16) {
        float v[16];
        tmem_ld16(taddr + (uint32_t)c0, v);
        if (crow) {
          if (g.relu) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
          }
          if (g.mul) {   // inverted-dropout mask of this output row
            const float* mr = g.mul + (tile * UM + r) * g.N;
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (c0 + i < g.N) v[i] *= __ldg(mr + c0 + i);
          }
          if (g.c_packed) {   // pad columns hold exact zeros (zero B rows)
            const int64_t m = tile * UM + r;
#pragma unroll
            for (int i = 0; i < 16; i += 4) packed_store<4>(g.c_packed, g.c_nk, m, c0 + i, v + i);
          }
          if (vec && c0 + 16 <= g.N) {
#pragma unroll
            for (int i = 0; i < 16; i += 4)
              *reinterpret_cast<float4*>(crow + c0 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (c0 + i < g.N) crow[c0 + i] = v[i];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bar_tempty[acc]));
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * acc_cols));
}

bool records_split(int64_t rows) {
  const char* env = getenv("KG_SPLIT_ROWS_MAX");
  return rows <= (env ? atoll(env) : 65536LL);
}

static uint32_t acc_cols_for(int np) {
  uint32_t c = 32;
  while ((int)c < np) c <<= 1;
  return c;
}

static int stages_for(int np) {
  int s = (int)(USMEM_CAP / ((size_t)(UM + np) * UKC * 8));
  return s > UMAXS ? UMAXS : s;
}

static kg_status launch_pack(const PackJob& a, const PackJob& b, int64_t items_max, cudaStream_t st) {
  // items_max / 512 approximates the record count (R*4 items per record)
  dim3 grid((unsigned)persistent_blocks(items_max, 512, 8), 2, 1);
  KG_LAUNCH("k_umma_pack", k_umma_pack, grid, 256, 0, st, a, b);
  return KG_OK;
}

static kg_status launch_packed(const PackedArgs& p, dim3 grid, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    KG_CUDA(cudaFuncSetAttribute(k_umma_packed, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(USMEM_CAP + EP_SLAB_BYTES)));
    attr_set = true;
  }
  const int ns = stages_for(p.np);
  const size_t smem = (size_t)ns * (UM + p.np) * UKC * 8 + (p.tn ? 0 : EP_SLAB_BYTES);
  KG_LAUNCH(p.tn ? "k_umma_gemm_tn" : "k_umma_gemm_nn", k_umma_packed, grid, UTHREADS, smem, st, p, ns,
            acc_cols_for(p.np));
  return KG_OK;
}

// NN workspace: A records (tiles x nk) + B records (nk)
static size_t nn_pack_sizes(int64_t M_max, int64_t K, int64_t N, size_t* a_bytes) {
  const int np = pad16((int)N);
  const int64_t nk = ceil_div(K, UKC), tiles = ceil_div(M_max > 0 ? M_max : 1, UM);
  size_t a = align_up((size_t)(tiles * nk * (records_split(M_max) ? rec_floats_split(UM) : rec_floats(UM))) * 4);
  size_t b = align_up((size_t)(nk * rec_floats_split(np)) * 4);
  if (a_bytes) *a_bytes = a;
  return a + b;
}

size_t umma_nn_workspace(int64_t M_max, int64_t K, int64_t N) { return nn_pack_sizes(M_max, K, N, nullptr); }

kg_status umma_gemm_nn(const GemmArgs& g, void* ws, cudaStream_t st) {
  if (g.M_max <= 0 || g.N <= 0) return KG_OK;
  KG_REQUIRE(g.N <= 256, KG_ERR_SHAPE, "umma NN supports N <= 256 (got %lld)", (long long)g.N);
  const int np = pad16((int)g.N);
  const int64_t nk = ceil_div(g.K, UKC), tiles = ceil_div(g.M_max, UM);
  size_t a_bytes = 0;
  nn_pack_sizes(g.M_max, g.K, g.N, &a_bytes);
  float* Ap = static_cast<float*>(ws);
  float* Bp = reinterpret_cast<float*>(static_cast<char*>(ws) + a_bytes);
  const int a_split = records_split(g.M_max) ? 1 : 0;
  PackJob ja{g.A, g.lda, g.a_rows, g.M_dev, g.M_dev_index, g.M, g.K, UM, 0, nk, Ap, a_split};
  if (g.a_packed) {   // producer already wrote the A records
    ja.src = nullptr;
    Ap = const_cast<float*>(g.a_packed);
  }
  PackJob jb{g.B, g.ldb, nullptr, nullptr, 0, g.K, g.N, np, 1, nk, Bp, 1};
  if (g.b_packed) {   // weights packed once per optimizer step
    jb.src = nullptr;
    Bp = const_cast<float*>(g.b_packed);
  }
  if (ja.src || jb.src) {
    const int64_t items = ja.src ? tiles * nk * UM * 4 : nk * np * 4;
    kg_status s = launch_pack(ja, jb, items, st);
    if (s != KG_OK) return s;
  }
  PackedArgs p{};
  p.Ap = Ap; p.Bp = Bp; p.a_nk_alloc = nk; p.np = np; p.tn = 0; p.a_split = a_split; p.b_split = 1;
  p.M = g.M; p.M_dev = g.M_dev; p.M_dev_index = g.M_dev_index; p.nk = nk;
  p.C = g.C; p.ldc = g.ldc; p.c_rows = g.c_rows; p.N = g.N; p.out_rows = 0; p.relu = g.relu;
  p.c_packed = g.c_packed; p.c_nk = packed_nk(g.M_max, g.N); p.mul = g.mul;
  static const int gemm_exp = getenv("KG_GEMM_EXP") ? atoi(getenv("KG_GEMM_EXP")) : 0;
  p.exp = gemm_exp;
  const int ctas = (int)(tiles < num_sms() ? tiles : num_sms());
  return launch_packed(p, dim3((unsigned)ctas, 1, 1), st);
}

int umma_tn_splits(int64_t rows_max, int64_t K) {
  // >= 12 records (192 data rows) per split, one CTA per SM over all feature blocks
  const int64_t blocks = ceil_div(K, UM);
  int64_t s = ceil_div(ceil_div(rows_max, UKC), 12);
  const int64_t cap = num_sms() / blocks > 0 ? num_sms() / blocks : 1;
  if (s > cap) s = cap;
  return (int)(s < 1 ? 1 : s);
}

// TN workspace: A^T records (feature blocks x nk_alloc) + B^T records + split partials
static size_t tn_sizes(int64_t rows_max, int64_t K, int64_t N, size_t* a_bytes, size_t* b_bytes) {
  const int np = pad16((int)N);
  const int64_t nk = ceil_div(rows_max > 0 ? rows_max : 1, UKC), blocks = ceil_div(K, UM);
  size_t a = align_up((size_t)(blocks * nk * rec_floats(UM)) * 4);
  size_t b = align_up((size_t)(nk * rec_floats(np)) * 4);
  if (a_bytes) *a_bytes = a;
  if (b_bytes) *b_bytes = b;
  return a + b + align_up((size_t)umma_tn_splits(rows_max, K) * K * N * sizeof(float));
}

size_t umma_tn_workspace(int64_t rows_max, int64_t K, int64_t N) { return tn_sizes(rows_max, K, N, nullptr, nullptr); }

kg_status umma_gemm_tn(const GemmArgs& g, float* out, void* ws, cudaStream_t st) {
  KG_REQUIRE(g.N <= 256, KG_ERR_SHAPE, "umma TN supports N <= 256");
  if (g.K <= 0 || g.N <= 0) return KG_OK;
  const int np = pad16((int)g.N);
  const int64_t rows_max = g.M_max > 0 ? g.M_max : 1;
  const int64_t nk_alloc = ceil_div(rows_max, UKC), blocks = ceil_div(g.K, UM);
  size_t a_bytes = 0, b_bytes = 0;
  tn_sizes(rows_max, g.K, g.N, &a_bytes, &b_bytes);
  float* Ap = static_cast<float*>(ws);
  float* Bp = reinterpret_cast<float*>(static_cast<char*>(ws) + a_bytes);
  float* part = reinterpret_cast<float*>(static_cast<char*>(ws) + a_bytes + b_bytes);
  // A^T: MMA rows = feature columns of A, k = data rows (gathered)
  PackJob ja{g.A, g.lda, g.a_rows, g.M_dev, g.M_dev_index, g.M, g.K, UM, 1, nk_alloc, Ap, 0};
  // Bm^T: MMA rows = output columns, k = data rows
  PackJob jb{g.B, g.ldb, nullptr, g.M_dev, g.M_dev_index, g.M, g.N, np, 1, nk_alloc, Bp, 0};
  const int64_t items = (blocks * UM > np ? blocks * UM : np) * nk_alloc * 4;
  kg_status s = launch_pack(ja, jb, items, st);
  if (s != KG_OK) return s;
  const int splits = umma_tn_splits(rows_max, g.K);
  PackedArgs p{};
  p.Ap = Ap; p.Bp = Bp; p.a_nk_alloc = nk_alloc; p.np = np; p.tn = 1;
  p.M = g.M; p.M_dev = g.M_dev; p.M_dev_index = g.M_dev_index; p.nk = 0;
  p.C = part; p.ldc = g.N; p.c_rows = nullptr; p.N = g.N; p.out_rows = g.K; p.relu = 0;
  s = launch_packed(p, dim3((unsigned)splits, (unsigned)blocks, 1), st);
  if (s != KG_OK) return s;
  return reduce_splits(part, splits, g.K * g.N, out, st);
}

// ---------------------------------------------------------------------------
// TN straight from the producers' records: dV = X^T dS.
//
// The records of X (written by the forward epilogue / the input pack) and of
// dS (written by the CSC pass) hold, per 128-row block and 16-column chunk,
// 8-row x 64-byte swizzle atoms (pk_off). For dV the data rows are the
// reduction (K) dimension, so the operands are needed K-major along the data
// rows — the transpose of the records. (tcgen05's MN-major operand mode is
// not usable with kind::tf32: with a transpose bit set the MMA yields zeros
// on this part.) Instead of a global transposing pack, the producer copies
// each chunk's 16-row slice (1 KB) of a stage into shared memory and the four
// split warps transpose it there into K-major records (MMA row = column of X
// or dS, K = the stage's 16 data rows), splitting fp32 into tf32 hi + lo on
// the way; rows past the device row count are written as zeros. The X and dS
// records are read once, nothing else touches HBM: no transposing pack pass
// and no row-major dS. Split-K over CTAs (contiguous 16-row groups) + the
// fixed-order reduce.
struct TnMnArgs {
  const float* Xp;     // X records: 128-row blocks x xk chunks (hi|lo if split)
  const float* Dp;     // dS records: 128-row blocks x dk chunks
  int xk, dk;          // 16-column chunks per block (M = 16*xk <= 128, N = 16*dk <= 256)
  int split;           // records hold hi | lo halves
  const int32_t* M_dev;
  int M_dev_index;
  int64_t rows;        // data rows if M_dev == nullptr
  float* part;         // (splits, out_rows, N) partials
  int64_t out_rows;    // X columns (<= 128)
  int64_t N;
};

constexpr int TM_SLICE = 16 * UKC * 4;   // bytes of a 16-row slice of one chunk (two atoms)

struct TnStage {   // byte offsets inside one ring stage
  uint32_t sa, sb, ka, kb, size;
};

__host__ __device__ inline TnStage tn_stage(int xk, int dk, int split) {
  TnStage t;
  const uint32_t m = split ? 2u : 1u;
  t.sa = 0;
  t.sb = t.sa + (uint32_t)xk * TM_SLICE * m;
  t.ka = (t.sb + (uint32_t)dk * TM_SLICE * m + 1023u) & ~1023u;
  t.kb = t.ka + 2u * UM * UKC * 4u;                 // A K-major tile: hi + lo (128 rows)
  t.size = t.kb + 2u * (uint32_t)(16 * dk) * UKC * 4u;
  t.size = (t.size + 1023u) & ~1023u;
  return t;
}

__global__ void __launch_bounds__(UTHREADS, 1) k_umma_tn_rec(TnMnArgs g, int nstages, uint32_t acc_cols) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_full[UMAXS], bar_empty[UMAXS], bar_split[UMAXS], bar_tfull;
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t rows = g.M_dev ? (int64_t)g.M_dev[g.M_dev_index] : g.rows;
  const int64_t ngrp = (rows + 15) / 16;
  const int64_t per = (ngrp + gridDim.x - 1) / gridDim.x;
  const int64_t c_lo = (int64_t)blockIdx.x * per, c_hi = c_lo + per < ngrp ? c_lo + per : ngrp;
  const int np = 16 * g.dk;
  if (c_lo >= c_hi) {   // empty split: its partial slot is zero
    for (int idx = tid; idx < g.out_rows * g.N; idx += UTHREADS)
      g.part[(int64_t)blockIdx.x * g.out_rows * g.N + idx] = 0.f;
    return;
  }
  const int nk = (int)(c_hi - c_lo);
  const TnStage L = tn_stage(g.xk, g.dk, g.split);
  const uint32_t sbase = smem_u32(smem);
  auto full = [&](int s) { return smem_u32(&bar_full[s]); };
  auto empty = [&](int s) { return smem_u32(&bar_empty[s]); };
  // K-major A rows past 16*xk (M padding to 128) stay zero in every stage
  for (int s = 0; s < nstages; ++s) {
    float* ka = reinterpret_cast<float*>(smem + (size_t)s * L.size + L.ka);
    for (int i = tid; i < (UM - 16 * g.xk) * UKC; i += UTHREADS) {
      const int m = 16 * g.xk + i / UKC, k = i % UKC;
      ka[pk_off(m, k)] = 0.f;
      ka[UM * UKC + pk_off(m, k)] = 0.f;
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(acc_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
      mbar_init(smem_u32(&bar_split[s]), 4);
    }
    mbar_init(smem_u32(&bar_tfull), 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // zero padding visible to the MMAs
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  const int64_t xrec = g.split ? rec_floats_split(UM) : rec_floats(UM);   // floats per record
  const int64_t lo_off = (int64_t)UM * UKC;                                 // lo half inside a split record
  const uint32_t mult = g.split ? 2u : 1u;

  if (warp == 0) {
    if (lane == 0) {   // producer: per 16-row group, each chunk's 1 KB slice (hi, and lo when split)
      const uint32_t bytes = (uint32_t)(g.xk + g.dk) * TM_SLICE * mult;
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % nstages;
        if (kc >= nstages) mbar_wait(empty(s), (uint32_t)((kc / nstages - 1) & 1));
        const int64_t grp = c_lo + kc, blk = grp / 8, r16 = (grp & 7) * 16;
        const uint32_t dst = sbase + (uint32_t)s * L.size;
        mbar_expect_tx(full(s), bytes);
        for (int c = 0; c < g.xk; ++c) {
          const float* rec = g.Xp + (blk * g.xk + c) * xrec + r16 * UKC;
          bulk_g2s(dst + L.sa + (uint32_t)c * TM_SLICE * mult, rec, TM_SLICE, full(s));
          if (g.split) bulk_g2s(dst + L.sa + (uint32_t)c * TM_SLICE * 2 + TM_SLICE, rec + lo_off, TM_SLICE, full(s));
        }
        for (int c = 0; c < g.dk; ++c) {
          const float* rec = g.Dp + (blk * g.dk + c) * xrec + r16 * UKC;
          bulk_g2s(dst + L.sb + (uint32_t)c * TM_SLICE * mult, rec, TM_SLICE, full(s));
          if (g.split) bulk_g2s(dst + L.sb + (uint32_t)c * TM_SLICE * 2 + TM_SLICE, rec + lo_off, TM_SLICE, full(s));
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // MMA issuer: D(128 x np) += X^T . dS over the CTA's row groups
      const uint32_t idesc = make_idesc(np);
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % nstages;
        mbar_wait(smem_u32(&bar_split[s]), (uint32_t)((kc / nstages) & 1));
        tc_fence_after();
        const uint32_t a_hi = sbase + (uint32_t)s * L.size + L.ka, a_lo = a_hi + UM * UKC * 4;
        const uint32_t b_hi = sbase + (uint32_t)s * L.size + L.kb, b_lo = b_hi + (uint32_t)np * UKC * 4;
#pragma unroll
        for (int j = 0; j < UKC / 8; ++j) {
          const uint32_t ko = (uint32_t)j * 32u;
          const uint64_t dah = make_desc(a_hi + ko), dal = make_desc(a_lo + ko);
          const uint64_t dbh = make_desc(b_hi + ko), dbl = make_desc(b_lo + ko);
          mma_tf32(tmem, dah, dbh, idesc, (kc > 0 || j > 0) ? 1u : 0u);
          mma_tf32(tmem, dah, dbl, idesc, 1u);
          mma_tf32(tmem, dal, dbh, idesc, 1u);
        }
        mma_commit(empty(s));
      }
      mma_commit(smem_u32(&bar_tfull));
    }
  } else if (warp >= USPLIT0) {
    // split warps: staged slices (data row r, column f of chunk c) -> K-major
    // records (MMA row 16c + f, k = r), fp32 split into tf32 hi + lo; rows
    // past the row count -> zeros
    const int st = tid - USPLIT0 * 32;
    for (int kc = 0; kc < nk; ++kc) {
      const int s = kc % nstages;
      mbar_wait(full(s), (uint32_t)((kc / nstages) & 1));
      uint8_t* base = smem + (size_t)s * L.size;
      const int64_t row0 = (c_lo + kc) * 16;
      const int valid = rows - row0 < 16 ? (int)(rows - row0) : 16;
      const int na = g.xk * 64, nb = g.dk * 64;   // float4 quads (16 rows x 4 per chunk)
      for (int i = st; i < na + nb; i += 128) {
        const bool isa = i < na;
        const int ii = isa ? i : i - na;
        const int c = ii >> 6, r = (ii >> 2) & 15, q = ii & 3;
        const float* slice = reinterpret_cast<const float*>(base + (isa ? L.sa : L.sb) + (uint32_t)c * TM_SLICE * mult);
        const int off = pk_off(r, 4 * q);
        float hv[4], lv[4];
        const float4 x = *reinterpret_cast<const float4*>(slice + off);
        if (g.split) {
          const float4 y = *reinterpret_cast<const float4*>(slice + TM_SLICE / 4 + off);
          hv[0] = x.x; hv[1] = x.y; hv[2] = x.z; hv[3] = x.w;
          lv[0] = y.x; lv[1] = y.y; lv[2] = y.z; lv[3] = y.w;
        } else {
          split_tf32(x.x, hv[0], lv[0]);
          split_tf32(x.y, hv[1], lv[1]);
          split_tf32(x.z, hv[2], lv[2]);
          split_tf32(x.w, hv[3], lv[3]);
        }
        if (r >= valid) {
#pragma unroll
          for (int t = 0; t < 4; ++t) hv[t] = lv[t] = 0.f;
        }
        float* kt = reinterpret_cast<float*>(base + (isa ? L.ka : L.kb));
        const int half = (isa ? UM : np) * UKC;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int o = pk_off(16 * c + 4 * q + t, r);
          kt[o] = hv[t];
          kt[half + o] = lv[t];
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tcgen05 reads
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bar_split[s]));
    }
  } else {
    // epilogue warps 2..5: feature row m = TMEM lane, columns n < N
    const int lanegrp = warp & 3, m = lanegrp * 32 + lane;
    mbar_wait(smem_u32(&bar_tfull), 0u);
    tc_fence_after();
    const uint32_t taddr = tmem + ((uint32_t)(lanegrp * 32) << 16);
    float* crow = m < g.out_rows ? g.part + ((int64_t)blockIdx.x * g.out_rows + m) * g.N : nullptr;
    for (int c0 = 0; c0 < np; c0 += 16) {
      float v[16];
      tmem_ld16(taddr + (uint32_t)c0, v);
      if (crow) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (c0 + i < g.N) crow[c0 + i] = v[i];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(acc_cols));
}

kg_status umma_gemm_tn_records(const float* Xp, int64_t x_cols, const float* Dp, int64_t N, const int32_t* M_dev,
                               int M_dev_index, int64_t rows_max, float* out, void* ws, cudaStream_t st) {
  KG_REQUIRE(x_cols <= 128 && N <= 256, KG_ERR_SHAPE, "record TN supports d_in <= 128, N <= 256");
  if (x_cols <= 0 || N <= 0) return KG_OK;
  TnMnArgs a{};
  a.Xp = Xp; a.Dp = Dp;
  a.xk = (int)ceil_div(x_cols, UKC); a.dk = (int)ceil_div(N, UKC);
  a.split = records_split(rows_max) ? 1 : 0;
  a.M_dev = M_dev; a.M_dev_index = M_dev_index; a.rows = rows_max;
  a.out_rows = x_cols; a.N = N;
  const int splits = umma_tn_splits(rows_max, x_cols);
  a.part = static_cast<float*>(ws);
  const TnStage L = tn_stage(a.xk, a.dk, a.split);
  int ns = (int)(USMEM_CAP / L.size);
  if (ns > UMAXS) ns = UMAXS;
  KG_REQUIRE(ns >= 2, KG_ERR_SHAPE, "record TN stage does not fit shared memory");
  static bool attr = false;
  if (!attr) {
    KG_CUDA(cudaFuncSetAttribute(k_umma_tn_rec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)USMEM_CAP));
    attr = true;
  }
  KG_LAUNCH("k_umma_gemm_tn", k_umma_tn_rec, dim3((unsigned)splits, 1, 1), UTHREADS, (size_t)ns * L.size, st, a, ns,
            acc_cols_for(16 * a.dk));
  return reduce_splits(a.part, splits, x_cols * N, out, st);
}

// Test entry: pack row-major A (gathered) and B rows into records, then the
// record TN (the product path gets the records from their producers).
size_t umma_tn_records_test_workspace(int64_t M, int64_t K, int64_t N) {
  return packed_bytes(M, K) + packed_bytes(M, N) + align_up((size_t)umma_tn_splits(M, K) * K * N * 4) + 1024;
}

kg_status umma_gemm_tn_via_records(const GemmArgs& g, float* out, void* ws, cudaStream_t st) {
  const int64_t M = g.M_max;
  float* Xp = static_cast<float*>(ws);
  float* Dp = reinterpret_cast<float*>(static_cast<char*>(ws) + align_up(packed_bytes(M, g.K)));
  void* rest = static_cast<char*>(ws) + align_up(packed_bytes(M, g.K)) + align_up(packed_bytes(M, g.N));
  const int sp = records_split(M) ? 1 : 0;
  const int64_t xk = ceil_div(g.K, UKC), dk = ceil_div(g.N, UKC), tiles = ceil_div(M, UM);
  PackJob ja{g.A, g.lda, g.a_rows, g.M_dev, g.M_dev_index, g.M, g.K, UM, 0, xk, Xp, sp};
  PackJob jb{g.B, g.ldb, nullptr, g.M_dev, g.M_dev_index, g.M, g.N, UM, 0, dk, Dp, sp};
  kg_status s = launch_pack(ja, jb, tiles * (xk > dk ? xk : dk) * UM * 4, st);
  if (s != KG_OK) return s;
  return umma_gemm_tn_records(Xp, g.K, Dp, g.N, g.M_dev, g.M_dev_index, M, out, rest, st);
}

// ---------------------------------------------------------------------------
// Filtered ranking on the tensor cores (R25/R26, ref:evaluate.py:192-217).
//
// Rows x = side*nq + q are the (query, side) pairs; q_x = H[anchor] * dec[r]
// (fp32 product). k_rank_umma keeps a 128-row query tile resident in shared
// memory and streams record tiles through a ring: first the tile's "diagonal"
// B rows (the true entity of each row), then every candidate block; D = Q.C^T
// on tcgen05 (3xTF32, 128 x 128 per virtual tile, TMEM double buffer). The
// epilogue never writes a score: virtual tile 0 yields the true score as the
// diagonal D[x][x] (a tcgen05 element depends only on its A and B rows, so it
// is bit-identical to the bulk element of the true column —
// tools/check_mma_position.py), then 8 epilogue warps count candidates
// scoring greater / equal, branch-free. Known (train+valid+test) candidates
// are a short pair list per query: their scores come from the same kernel in
// diagonal-only mode (A rows = the pair's query, B rows = the candidate) and
// are subtracted from the counts before the tie policy of
// ref:evaluate.py:93-100 is applied.
struct RankArgs {
  const float* Qp;    // A records, 128-row blocks over rows
  const float* Tp;    // diagonal B records, same blocking
  const float* Cp;    // candidate records (ncols columns), may be null
  int nk;
  int64_t rows;
  int32_t ncols;      // 0: diagonal only
  float* ts;          // out: diagonal per row
  uint32_t* greater;  // out (accumulated): candidates scoring > ts
  uint32_t* equal;    // out (accumulated): candidates scoring == ts
  // Banded mode (float64 refinement, kq != null): a candidate c counts as
  // greater only when its score exceeds ts + w(x, c); scores within
  // [ts - w, ts + w] are recorded (candidate id, RK_NEAR slots per row,
  // nearc[x] counts them all) and decided in float64 afterwards.
  const float* kq;     // per row: error-bound factor of the query
  const float* kt;     // per row: kq * ||H[true]||
  const float* hn;     // per candidate: ||H[c]||
  uint32_t* nearc;
  int32_t* near_c;
};

// Band half-width for (row, candidate): kq ||H[c]|| + kq ||H[true]|| — the
// tensor-core scores of both are within kq/2 ||H|| of float64 (see
// k_row_exact). Evaluated with explicit rounding so every site agrees.
__device__ __forceinline__ float rk_band(float kq, float hn_c, float kt) { return __fmaf_rn(kq, hn_c, kt); }

constexpr int RK_NEAR = 32;   // near-tie slots per row; rows with more are rescanned in float64

constexpr int RK_EPI_WARPS = 8;
constexpr int RK_THREADS = 64 + 32 * RK_EPI_WARPS;
constexpr int RK_MAXS = 8;
constexpr uint32_t RK_REC = 128 * UKC * 8;   // bytes per 128-row record (hi + lo)
constexpr size_t RK_SMEM_CAP = 220 * 1024;

__device__ __forceinline__ int64_t rk_lower_bound(const int64_t* __restrict__ k, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (k[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void rk_query(const int32_t* __restrict__ qry, int64_t nq, int64_t x, int& side,
                                         int64_t& q, int32_t& anc, int32_t& rel, int32_t& tru) {
  side = (int)(x / nq);
  q = x - side * nq;
  const int32_t h = qry[q * 3], tl = qry[q * 3 + 2];
  rel = qry[q * 3 + 1];
  anc = side == 0 ? h : tl;
  tru = side == 0 ? tl : h;
}

// A rows: q_x (or, for the known-pair pass, q of the pair's row); diagonal B
// rows: H[tru(x)] (or H[c] of the pair).
__global__ void __launch_bounds__(256) k_eval_pack(const float* __restrict__ H, const float* __restrict__ dec,
                                                   const int32_t* __restrict__ qry, int64_t nq,
                                                   const int32_t* __restrict__ pair_x,
                                                   const int32_t* __restrict__ pair_c,
                                                   const int32_t* __restrict__ rows_dev, int64_t rows_host, int d,
                                                   int nk, float* __restrict__ Qp, float* __restrict__ Tp) {
  const int64_t rows = rows_dev ? (int64_t)*rows_dev : rows_host, tiles = (rows + 127) / 128;
  const int64_t items = tiles * nk * 128 * 4;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < items;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int q4 = (int)(idx & 3);
    const int64_t t = idx >> 2;
    const int r = (int)(t & 127);
    const int64_t u = t >> 7;
    const int64_t kc = u % nk, blk = u / nk;
    const int64_t i = blk * 128 + r;
    const int k0 = (int)kc * UKC + 4 * q4;
    float vq[4] = {0.f, 0.f, 0.f, 0.f}, vt[4] = {0.f, 0.f, 0.f, 0.f};
    if (i < rows) {
      const int64_t x = pair_x ? pair_x[i] : i;
      int side;
      int64_t q;
      int32_t anc, rel, tru;
      rk_query(qry, nq, x, side, q, anc, rel, tru);
      const int32_t c = pair_c ? pair_c[i] : tru;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = k0 + j;
        if (k < d) {
          vq[j] = H[(int64_t)anc * d + k] * dec[(int64_t)rel * d + k];
          vt[j] = H[(int64_t)c * d + k];
        }
      }
    }
    pack_store(Qp + (blk * nk + kc) * rec_floats_split(128), 128, r, q4, vq, 1);
    pack_store(Tp + (blk * nk + kc) * rec_floats_split(128), 128, r, q4, vt, 1);
  }
}

__global__ void __launch_bounds__(RK_THREADS, 1) k_rank_umma(RankArgs a, const int32_t* __restrict__ rows_dev,
                                                             int nstages) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_full[RK_MAXS], bar_empty[RK_MAXS], bar_tfull[2], bar_tempty[2];
  __shared__ __align__(8) uint64_t bar_afull, bar_aempty;
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t rows = rows_dev ? (int64_t)*rows_dev : a.rows, qtiles = (rows + 127) / 128;
  const int nblk = (a.ncols + 127) / 128, nj = nblk + 1, nk = a.nk;
  if ((int64_t)blockIdx.x >= qtiles) return;
  const uint32_t sbase = smem_u32(smem), ring = sbase + (uint32_t)nk * RK_REC;
  auto full = [&](int s) { return smem_u32(&bar_full[s]); };
  auto empty = [&](int s) { return smem_u32(&bar_empty[s]); };
  const int64_t RF = rec_floats_split(128);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&bar_tfull[i]), 1);
      mbar_init(smem_u32(&bar_tempty[i]), RK_EPI_WARPS);
    }
    mbar_init(smem_u32(&bar_afull), 1);
    mbar_init(smem_u32(&bar_aempty), 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    if (lane == 0) {   // producer
      int64_t it = 0, tc = 0;
      for (int64_t tile = blockIdx.x; tile < qtiles; tile += gridDim.x, ++tc) {
        if (tc > 0) mbar_wait(smem_u32(&bar_aempty), (uint32_t)((tc - 1) & 1));
        mbar_expect_tx(smem_u32(&bar_afull), (uint32_t)nk * RK_REC);
        for (int kc = 0; kc < nk; ++kc)
          bulk_g2s(sbase + (uint32_t)kc * RK_REC, a.Qp + (tile * nk + kc) * RF, RK_REC, smem_u32(&bar_afull));
        for (int j = 0; j < nj; ++j)
          for (int kc = 0; kc < nk; ++kc, ++it) {
            const int s = (int)(it % nstages);
            if (it >= nstages) mbar_wait(empty(s), (uint32_t)((it / nstages - 1) & 1));
            mbar_expect_tx(full(s), RK_REC);
            const float* src = j == 0 ? a.Tp + (tile * nk + kc) * RF : a.Cp + ((int64_t)(j - 1) * nk + kc) * RF;
            bulk_g2s(ring + (uint32_t)s * RK_REC, src, RK_REC, full(s));
          }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // MMA issuer
      const uint32_t idesc = make_idesc(128);
      const uint32_t half = 128 * UKC * 4;
      int64_t it = 0, jc = 0, tc = 0;
      for (int64_t tile = blockIdx.x; tile < qtiles; tile += gridDim.x, ++tc) {
        mbar_wait(smem_u32(&bar_afull), (uint32_t)(tc & 1));
        tc_fence_after();
        for (int j = 0; j < nj; ++j, ++jc) {
          const int acc = (int)(jc & 1);
          if (jc >= 2) mbar_wait(smem_u32(&bar_tempty[acc]), (uint32_t)((jc / 2 - 1) & 1));
          tc_fence_after();
          const uint32_t dt = tmem + (uint32_t)acc * 128;
          for (int kc = 0; kc < nk; ++kc, ++it) {
            const int s = (int)(it % nstages);
            mbar_wait(full(s), (uint32_t)((it / nstages) & 1));
            tc_fence_after();
            const uint32_t a_hi = sbase + (uint32_t)kc * RK_REC, a_lo = a_hi + half;
            const uint32_t b_hi = ring + (uint32_t)s * RK_REC, b_lo = b_hi + half;
#pragma unroll
            for (int jj = 0; jj < UKC / 8; ++jj) {
              const uint32_t ko = (uint32_t)jj * 32u;
              const uint64_t dah = make_desc(a_hi + ko), dal = make_desc(a_lo + ko);
              const uint64_t dbh = make_desc(b_hi + ko), dbl = make_desc(b_lo + ko);
              mma_tf32(dt, dah, dbh, idesc, (kc > 0 || jj > 0) ? 1u : 0u);
              mma_tf32(dt, dah, dbl, idesc, 1u);
              mma_tf32(dt, dal, dbh, idesc, 1u);
            }
            mma_commit(empty(s));
          }
          mma_commit(smem_u32(&bar_tfull[acc]));
        }
        mma_commit(smem_u32(&bar_aempty));
      }
    }
  } else {   // epilogue warps: TMEM lanes 32*(warp%4).., column half (warp-2)/4
    const int lanegrp = warp & 3, r = lanegrp * 32 + lane, colh = (warp - 2) >> 2;
    int64_t jc = 0;
    const bool banded = a.kq != nullptr;
    for (int64_t tile = blockIdx.x; tile < qtiles; tile += gridDim.x) {
      const int64_t x = tile * 128 + r;
      float ts = 0.f;
      const float kq = (banded && x < rows) ? a.kq[x] : 0.f, kt = (banded && x < rows) ? a.kt[x] : 0.f;
      uint32_t g = 0, e = 0;
      for (int j = 0; j < nj; ++j, ++jc) {
        const int acc = (int)(jc & 1);
        mbar_wait(smem_u32(&bar_tfull[acc]), (uint32_t)((jc / 2) & 1));
        tc_fence_after();
        const uint32_t taddr = tmem + (uint32_t)acc * 128 + ((uint32_t)(lanegrp * 32) << 16);
        if (j == 0) {
          float v[32];
          tmem_ld16(taddr + (uint32_t)(lanegrp * 32), v);
          tmem_ld16(taddr + (uint32_t)(lanegrp * 32 + 16), v + 16);
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i == lane) ts = v[i];
        } else if (banded) {
          const int32_t c0 = (j - 1) * 128 + colh * 64;
          const int nvalid = a.ncols - c0;
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            float v[16];
            tmem_ld16(taddr + (uint32_t)(colh * 64 + ch * 16), v);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const bool ok = ch * 16 + i < nvalid && x < rows;
              const float w = ok ? rk_band(kq, __ldg(a.hn + c0 + ch * 16 + i), kt) : 0.f;
              const float band_hi = __fadd_rn(ts, w), band_lo = __fsub_rn(ts, w);
              g += (ok && v[i] > band_hi) ? 1u : 0u;
              if (ok && v[i] >= band_lo && v[i] <= band_hi) {   // rare: near-tie, decided in float64
                const uint32_t k = atomicAdd(a.nearc + x, 1u);
                if (k < (uint32_t)RK_NEAR) a.near_c[x * RK_NEAR + k] = c0 + ch * 16 + i;
              }
            }
          }
        } else {
          const int32_t c0 = (j - 1) * 128 + colh * 64;
          const int nvalid = a.ncols - c0;   // columns of this half that exist
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            float v[16];
            tmem_ld16(taddr + (uint32_t)(colh * 64 + ch * 16), v);
            if (nvalid >= (ch + 1) * 16) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                g += v[i] > ts ? 1u : 0u;
                e += v[i] == ts ? 1u : 0u;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const bool ok = ch * 16 + i < nvalid;
                g += (ok && v[i] > ts) ? 1u : 0u;
                e += (ok && v[i] == ts) ? 1u : 0u;
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bar_tempty[acc]));
      }
      if (x < rows) {
        if (colh == 0) a.ts[x] = ts;
        if (a.greater && nj > 1) {
          atomicAdd(a.greater + x, g);
          atomicAdd(a.equal + x, e);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// --- float64 near-tie refinement (banded mode) ------------------------------
// s64(x, c) = sum_k (H[anc,k] * dec[rel,k]) * H[c,k] in float64 — the
// reference's q = H[anchor] * decoder[r] product is exact in float64, its
// dgemm differs from this warp sum only in summation order (~1e-16). Every
// use (true score, near pairs, dense rows, known pairs) goes through this one
// function, so a candidate compares identically wherever it is decided.
__device__ __forceinline__ double rk_dot64(const double* __restrict__ H, const double* __restrict__ dec, int d,
                                           int32_t anc, int32_t rel, int32_t c, int lane) {
  double s = 0.0;
  for (int k = lane; k < d; k += 32)
    s = fma(H[(int64_t)anc * d + k] * dec[(int64_t)rel * d + k], H[(int64_t)c * d + k], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// ||H[c]|| per candidate (float)
__global__ void k_hnorm(const double* __restrict__ H, int32_t N, int d, float* __restrict__ hn) {
  const int lane = (int)lane_id(), nw = (gridDim.x * blockDim.x) >> 5;
  for (int64_t c = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); c < N; c += nw) {
    double s = 0.0;
    for (int k = lane; k < d; k += 32) s = fma(H[c * d + k], H[c * d + k], s);
    s = warp_sum_d(s);
    if (lane == 0) hn[c] = (float)sqrt(s);
  }
}

// per row: the float64 true score and the error-bound factors. The fp32
// rounding of H and q, the 3xTF32 split and the fp32 accumulation of d
// products keep a tensor-core score within (d + 16) 2^-24 sum_k |q_k H[c,k]|
// <= (d + 16) 2^-24 ||q|| ||H[c]|| of float64; kq = 2 (d + 16) 2^-23 ||q||
// gives the band a 4x margin over the sum of both scores' bounds.
__global__ void k_row_exact(const double* __restrict__ H, const double* __restrict__ dec, int d,
                            const int32_t* __restrict__ qry, int64_t nq, const float* __restrict__ hn,
                            double* __restrict__ ts64, float* __restrict__ kq, float* __restrict__ kt) {
  const int lane = (int)lane_id(), nw = (gridDim.x * blockDim.x) >> 5;
  for (int64_t x = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); x < 2 * nq; x += nw) {
    int side;
    int64_t q;
    int32_t anc, rel, tru;
    rk_query(qry, nq, x, side, q, anc, rel, tru);
    const double t = rk_dot64(H, dec, d, anc, rel, tru, lane);
    double qq = 0.0;
    for (int k = lane; k < d; k += 32) {
      const double v = H[(int64_t)anc * d + k] * dec[(int64_t)rel * d + k];
      qq = fma(v, v, qq);
    }
    qq = warp_sum_d(qq);
    if (lane == 0) {
      ts64[x] = t;
      const float f = (float)(2.0 * (d + 16) * 0x1p-23 * sqrt(qq));
      kq[x] = f;
      kt[x] = __fmul_rn(f, hn[tru]);
    }
  }
}

// near pairs of every row in float64; rows with more than RK_NEAR near
// candidates are rescanned over all N candidates (their counts replaced)
__global__ void k_near_refine(const double* __restrict__ H, const double* __restrict__ dec, int d, int32_t N,
                              const int32_t* __restrict__ qry, int64_t nq, const double* __restrict__ ts64,
                              const uint32_t* __restrict__ nearc, const int32_t* __restrict__ near_c,
                              uint32_t* __restrict__ greater, uint32_t* __restrict__ equal) {
  const int lane = (int)lane_id(), nw = (gridDim.x * blockDim.x) >> 5;
  for (int64_t x = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); x < 2 * nq; x += nw) {
    const uint32_t n = nearc[x];
    if (n == 0) continue;
    int side;
    int64_t q;
    int32_t anc, rel, tru;
    rk_query(qry, nq, x, side, q, anc, rel, tru);
    const double t = ts64[x];
    uint32_t g = 0, e = 0;
    const bool dense = n > (uint32_t)RK_NEAR;
    const int64_t cnt = dense ? N : n;
    for (int64_t i = 0; i < cnt; ++i) {
      const int32_t c = dense ? (int32_t)i : near_c[x * RK_NEAR + i];
      const double s = rk_dot64(H, dec, d, anc, rel, c, lane);
      g += s > t;
      e += s == t;
    }
    if (lane == 0) {
      if (dense) {
        greater[x] = g;
        equal[x] = e;
      } else {
        greater[x] += g;
        equal[x] += e;
      }
    }
  }
}

// known candidates (banded mode): decided by the same rule as in the main
// pass — float64 when the row was rescanned or the pair's score is in band
__global__ void k_known_fix64(const int32_t* __restrict__ px, const int32_t* __restrict__ pc,
                              const float* __restrict__ ps, const uint32_t* __restrict__ npairs,
                              const float* __restrict__ ts, const float* __restrict__ kq,
                              const float* __restrict__ kt, const float* __restrict__ hn,
                              const double* __restrict__ ts64, const uint32_t* __restrict__ nearc,
                              const double* __restrict__ H, const double* __restrict__ dec, int d,
                              const int32_t* __restrict__ qry, int64_t nq, uint32_t* __restrict__ greater,
                              uint32_t* __restrict__ equal) {
  const int lane = (int)lane_id(), nw = (gridDim.x * blockDim.x) >> 5;
  const int64_t n = *npairs;
  for (int64_t i = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); i < n; i += nw) {
    const int32_t x = px[i];
    const float s = ps[i], t = ts[x], w = rk_band(kq[x], hn[pc[i]], kt[x]);
    const float lo = __fsub_rn(t, w), hi = __fadd_rn(t, w);
    const bool dense = nearc[x] > (uint32_t)RK_NEAR;
    if (dense || (s >= lo && s <= hi)) {
      int side;
      int64_t q;
      int32_t anc, rel, tru;
      rk_query(qry, nq, x, side, q, anc, rel, tru);
      const double s64 = rk_dot64(H, dec, d, anc, rel, pc[i], lane);
      if (lane == 0) {
        if (s64 > ts64[x]) atomicSub(greater + x, 1u);
        if (s64 == ts64[x]) atomicSub(equal + x, 1u);
      }
    } else if (s > hi && lane == 0) {
      atomicSub(greater + x, 1u);
    }
  }
}

// known (train+valid+test) candidates other than the true one, per row x
__global__ void k_known_count(const int32_t* __restrict__ qry, int64_t nq, int32_t N, int32_t R,
                              const int64_t* __restrict__ tkeys, int64_t ntk, const int64_t* __restrict__ hkeys,
                              int64_t nhk, uint32_t* __restrict__ cnt, int64_t* __restrict__ lo_out) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < 2 * nq; x += (int64_t)gridDim.x * blockDim.x) {
    int side;
    int64_t q;
    int32_t anc, rel, tru;
    rk_query(qry, nq, x, side, q, anc, rel, tru);
    const int64_t* keys = side == 0 ? tkeys : hkeys;
    const int64_t nkeys = side == 0 ? ntk : nhk;
    const int64_t base = ((int64_t)anc * R + rel) * (int64_t)N;
    const int64_t lo = rk_lower_bound(keys, nkeys, base), hi = rk_lower_bound(keys, nkeys, base + N);
    const int64_t t = rk_lower_bound(keys, nkeys, base + tru);
    const bool has_true = t < hi && keys[t] == base + tru;
    cnt[x] = (uint32_t)(hi - lo - (has_true ? 1 : 0));
    lo_out[x] = lo;
  }
}

__global__ void k_known_pairs(const int32_t* __restrict__ qry, int64_t nq, int32_t N, int32_t R,
                              const int64_t* __restrict__ tkeys, const int64_t* __restrict__ hkeys,
                              const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ off,
                              const int64_t* __restrict__ lo, int64_t max_pairs, uint32_t* npairs,
                              int32_t* __restrict__ px, int32_t* __restrict__ pc) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < 2 * nq; x += (int64_t)gridDim.x * blockDim.x) {
    int side;
    int64_t q;
    int32_t anc, rel, tru;
    rk_query(qry, nq, x, side, q, anc, rel, tru);
    const int64_t* keys = side == 0 ? tkeys : hkeys;
    const int64_t base = ((int64_t)anc * R + rel) * (int64_t)N;
    uint32_t o = off[x];
    const uint32_t n = cnt[x];
    for (int64_t j = lo[x]; o < off[x] + n && (int64_t)o < max_pairs; ++j) {
      const int32_t c = (int32_t)(keys[j] - base);
      if (c == tru) continue;
      px[o] = (int32_t)x;
      pc[o] = c;
      ++o;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {   // clamped pair count for the diagonal pass
    const uint32_t t = npairs[0];
    npairs[1] = (int64_t)t < max_pairs ? t : (uint32_t)max_pairs;
    npairs[2] = (int64_t)t > max_pairs ? 1u : 0u;   // overflow: caller's bound too small
  }
}

// subtract known candidates that were counted as greater / equal
__global__ void k_known_fix(const int32_t* __restrict__ px, const float* __restrict__ ps,
                            const uint32_t* __restrict__ npairs, const float* __restrict__ ts,
                            uint32_t* __restrict__ greater, uint32_t* __restrict__ equal) {
  const uint32_t n = *npairs;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t x = px[i];
    const float s = ps[i], t = ts[x];
    if (s > t) atomicSub(greater + x, 1u);
    if (s == t) atomicSub(equal + x, 1u);
  }
}

__global__ void k_rank_policy(int64_t nq, int32_t N, int policy, int chunk, const uint32_t* __restrict__ greater,
                              const uint32_t* __restrict__ equal, const uint32_t* __restrict__ known,
                              double* __restrict__ ranks, int32_t* __restrict__ ncand) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < 2 * nq; x += (int64_t)gridDim.x * blockDim.x) {
    const int side = (int)(x / nq);
    const int64_t q = x - side * nq;
    const double g = (double)greater[x], e = (double)equal[x] - 1.0;   // minus the true entity itself
    double rank;
    if (policy == 0) rank = 1.0 + g + e / 2.0;
    else if (policy == 1) rank = 1.0 + g;
    else rank = 1.0 + g + e;
    const int64_t cb = q / chunk, qi = q - cb * chunk;
    const int64_t cs = (nq - cb * chunk) < chunk ? (nq - cb * chunk) : chunk;
    const int64_t rec = 2 * cb * chunk + side * cs + qi;
    ranks[rec] = rank;
    ncand[rec] = N - 1 - (int32_t)known[x];
  }
}

struct RankWs {
  float *Qp, *Tp, *Cp, *Pq, *Pc, *ts, *ps;
  uint32_t *greater, *equal, *cnt, *off, *npairs;
  int64_t* lo;
  int32_t *px, *pc;
  char* scan;
  double* ts64;
  float *kq, *kt, *hn;
  uint32_t* nearc;
  int32_t* near_c;
};

static size_t rank_ws(int64_t nq, int32_t N, int d, int64_t max_pairs, RankWs* w, void* base, size_t cap) {
  Arena a(base, cap);
  const int64_t nk = ceil_div(d, UKC), qt = ceil_div(2 * nq, 128), cb = ceil_div(N, 128), pt = ceil_div(max_pairs, 128);
  RankWs r;
  r.Qp = a.take<float>((size_t)(qt * nk * rec_floats_split(128)));
  r.Tp = a.take<float>((size_t)(qt * nk * rec_floats_split(128)));
  r.Cp = a.take<float>((size_t)(cb * nk * rec_floats_split(128)));
  r.Pq = a.take<float>((size_t)((pt > 0 ? pt : 1) * nk * rec_floats_split(128)));
  r.Pc = a.take<float>((size_t)((pt > 0 ? pt : 1) * nk * rec_floats_split(128)));
  r.ts = a.take<float>(2 * nq);
  r.ps = a.take<float>(max_pairs > 0 ? max_pairs : 1);
  r.greater = a.take<uint32_t>(2 * nq);
  r.equal = a.take<uint32_t>(2 * nq);
  r.cnt = a.take<uint32_t>(2 * nq);
  r.off = a.take<uint32_t>(2 * nq);
  r.npairs = a.take<uint32_t>(4);
  r.lo = a.take<int64_t>(2 * nq);
  r.px = a.take<int32_t>(max_pairs > 0 ? max_pairs : 1);
  r.pc = a.take<int32_t>(max_pairs > 0 ? max_pairs : 1);
  r.scan = a.take<char>(scan_workspace(2 * nq));
  r.ts64 = a.take<double>(2 * nq);
  r.kq = a.take<float>(2 * nq);
  r.kt = a.take<float>(2 * nq);
  r.hn = a.take<float>(N);
  r.nearc = a.take<uint32_t>(2 * nq);
  r.near_c = a.take<int32_t>((size_t)2 * nq * RK_NEAR);
  if (w) *w = r;
  return a.used + 1024;
}

size_t umma_rank_workspace(int64_t nq, int32_t N, int d, int64_t max_pairs) {
  return rank_ws(nq, N, d, max_pairs, nullptr, nullptr, 0);
}

static kg_status launch_rank(const RankArgs& ra, const int32_t* rows_dev, int64_t rows_max, cudaStream_t st) {
  int ns = (int)((RK_SMEM_CAP - (size_t)ra.nk * RK_REC) / RK_REC);
  if (ns > RK_MAXS) ns = RK_MAXS;
  KG_REQUIRE(ns >= 2, KG_ERR_SHAPE, "ranking tile does not fit shared memory");
  const size_t smem = (size_t)(ra.nk + ns) * RK_REC;
  static bool attr = false;
  if (!attr) {
    KG_CUDA(cudaFuncSetAttribute(k_rank_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RK_SMEM_CAP));
    attr = true;
  }
  const int64_t qt = ceil_div(rows_max > 0 ? rows_max : 1, 128);
  const int ctas = (int)(qt < num_sms() ? qt : num_sms());
  KG_LAUNCH("k_rank_umma", k_rank_umma, ctas, RK_THREADS, smem, st, ra, rows_dev, ns);
  return KG_OK;
}

kg_status umma_rank_filtered(const float* H, int d, int32_t N, const float* dec, int32_t R, const int32_t* qry,
                             int64_t nq, const int64_t* tkeys, int64_t ntk, const int64_t* hkeys, int64_t nhk,
                             int policy, int chunk, int64_t max_pairs, double* ranks, int32_t* ncand,
                             uint32_t* overflow, void* ws, size_t ws_bytes, cudaStream_t st, const double* H64,
                             const double* dec64) {
  KG_REQUIRE(d >= 1 && d <= 128, KG_ERR_SHAPE, "tensor-core ranking supports d <= 128");
  RankWs w;
  KG_REQUIRE(rank_ws(nq, N, d, max_pairs, &w, ws, ws_bytes) <= ws_bytes, KG_ERR_VALIDATION,
             "eval workspace too small");
  const int nk = (int)ceil_div(d, UKC);
  const int64_t rows = 2 * nq, qt = ceil_div(rows, 128), cb = ceil_div(N, 128);
  // operands: query rows + their true entities, all candidates
  KG_LAUNCH("k_eval_pack", k_eval_pack, persistent_blocks(qt * nk * 128 * 4, 256, 8), 256, 0, st, H, dec, qry, nq,
            (const int32_t*)nullptr, (const int32_t*)nullptr, (const int32_t*)nullptr, rows, d, nk, w.Qp, w.Tp);
  PackJob jc{H, d, nullptr, nullptr, 0, N, d, 128, 0, nk, w.Cp, 1};
  PackJob none{};
  kg_status s = launch_pack(jc, none, cb * nk * 128 * 4, st);
  if (s != KG_OK) return s;
  KG_CUDA(cudaMemsetAsync(w.greater, 0, (size_t)rows * 4, st));
  KG_CUDA(cudaMemsetAsync(w.equal, 0, (size_t)rows * 4, st));
  const bool banded = H64 != nullptr && dec64 != nullptr;
  const int g1 = persistent_blocks(rows, 256, 8);
  if (banded) {
    KG_CUDA(cudaMemsetAsync(w.nearc, 0, (size_t)rows * 4, st));
    KG_LAUNCH("k_hnorm", k_hnorm, persistent_blocks((int64_t)N * 32, 256, 8), 256, 0, st, H64, N, d, w.hn);
    KG_LAUNCH("k_row_exact", k_row_exact, persistent_blocks(rows * 32, 256, 8), 256, 0, st, H64, dec64, d, qry, nq,
              w.hn, w.ts64, w.kq, w.kt);
  }
  s = launch_rank(RankArgs{w.Qp, w.Tp, w.Cp, nk, rows, N, w.ts, w.greater, w.equal, banded ? w.kq : nullptr, w.kt,
                           w.hn, w.nearc, w.near_c},
                  nullptr, rows, st);
  if (s != KG_OK) return s;
  if (banded)
    KG_LAUNCH("k_near_refine", k_near_refine, persistent_blocks(rows * 32, 256, 8), 256, 0, st, H64, dec64, d, N, qry,
              nq, w.ts64, w.nearc, w.near_c, w.greater, w.equal);
  // known candidates: pair list (row, candidate), diagonal scores, fix-up
  KG_LAUNCH("k_known_count", k_known_count, g1, 256, 0, st, qry, nq, N, R, tkeys, ntk, hkeys, nhk, w.cnt, w.lo);
  s = exclusive_scan_u32(w.cnt, w.off, rows, w.npairs, w.scan, scan_workspace(rows), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("k_known_pairs", k_known_pairs, g1, 256, 0, st, qry, nq, N, R, tkeys, hkeys, w.cnt, w.off, w.lo,
            max_pairs, w.npairs, w.px, w.pc);
  const int64_t pt = ceil_div(max_pairs > 0 ? max_pairs : 1, 128);
  KG_LAUNCH("k_eval_pack", k_eval_pack, persistent_blocks(pt * nk * 128 * 4, 256, 8), 256, 0, st, H, dec, qry, nq,
            (const int32_t*)w.px, (const int32_t*)w.pc, (const int32_t*)(w.npairs + 1), (int64_t)0, d, nk, w.Pq,
            w.Pc);
  s = launch_rank(RankArgs{w.Pq, w.Pc, nullptr, nk, 0, 0, w.ps, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                           nullptr},
                  reinterpret_cast<const int32_t*>(w.npairs + 1), max_pairs, st);
  if (s != KG_OK) return s;
  if (banded)
    KG_LAUNCH("k_known_fix64", k_known_fix64, persistent_blocks((max_pairs > 0 ? max_pairs : 1) * 32, 256, 8), 256, 0,
              st, w.px, w.pc, w.ps, w.npairs + 1, w.ts, w.kq, w.kt, w.hn, w.ts64, w.nearc, H64, dec64, d, qry, nq,
              w.greater, w.equal);
  else
    KG_LAUNCH("k_known_fix", k_known_fix, persistent_blocks(max_pairs > 0 ? max_pairs : 1, 256, 8), 256, 0, st, w.px,
              w.ps, w.npairs + 1, w.ts, w.greater, w.equal);
  if (overflow) KG_CUDA(cudaMemcpyAsync(overflow, w.npairs + 2, 4, cudaMemcpyDeviceToDevice, st));
  KG_LAUNCH("k_rank_policy", k_rank_policy, g1, 256, 0, st, nq, N, policy, chunk, w.greater, w.equal, w.cnt, ranks,
            ncand);
  return KG_OK;
}

}  // namespace kg

using namespace kg;

extern "C" {

int64_t kg_pack_rows_bytes(int64_t rows, int64_t cols) { return (int64_t)packed_bytes(rows, cols); }

kg_status kg_pack_rows(const float* src, int64_t ld, const int32_t* rowid, const int32_t* counts,
                       int32_t count_index, int64_t n_max, int64_t cols, float* out, void* stream) {
  KG_REQUIRE(n_max >= 0 && cols >= 1, KG_ERR_VALIDATION, "bad pack shape");
  if (n_max == 0) return KG_OK;
  const int64_t nk = ceil_div(cols, UKC), tiles = ceil_div(n_max, UM);
  PackJob ja{src, ld, rowid, counts, count_index, n_max, cols, UM, 0, nk, out, records_split(n_max) ? 1 : 0};
  PackJob none{};
  return launch_pack(ja, none, tiles * nk * UM * 4, as_stream(stream));
}

}  // extern "C"

// this module's anchor for kg_preload_kernels (kg_primitives.cu)
extern "C" const void* kg_anchor_umma() { return reinterpret_cast<const void*>(&kg::k_umma_pack); }
