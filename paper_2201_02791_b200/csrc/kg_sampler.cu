// R3-R8: constraint-based negatives, the edge mini-batch stream and the
// layered closure, all reproducing the reference's numpy index streams
// bit-for-bit (ref:sampler.py:144-182, 202-232, 320-376).
#include "kg_common.cuh"
#include "kg_pcg64.cuh"

namespace kg {

static int grid_for(int64_t n) { return persistent_blocks(n, 256, 8); }

// ---------------------------------------------------------------------------
// uint32 stream generation (positional): U[p] for p in [0, W) from state g
// ---------------------------------------------------------------------------
constexpr int GEN_WORDS = 16;   // next64 words per thread

__global__ void k_gen_u32(const kg_pcg64* __restrict__ gp, int64_t W, uint32_t* __restrict__ U) {
  const kg_pcg64 g = *gp;
  const u128 s0 = state_of(g), inc = inc_of(g);
  const int64_t off = g.has_uint32 ? 1 : 0;
  const int64_t nwords = (W - off + 1) / 2 + 1;
  for (int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * GEN_WORDS; w0 < nwords;
       w0 += (int64_t)gridDim.x * blockDim.x * GEN_WORDS) {
    u128 s = apply_jump(pcg_jump((uint64_t)w0, inc), s0);
    for (int j = 0; j < GEN_WORDS; ++j) {
      int64_t w = w0 + j;
      if (w >= nwords) break;
      s = pcg_step(s, inc);
      uint64_t x = pcg_output(s);
      int64_t p = off + 2 * w;
      if (p < W) U[p] = (uint32_t)x;
      if (p + 1 < W) U[p + 1] = (uint32_t)(x >> 32);
    }
  }
  if (g.has_uint32 && blockIdx.x == 0 && threadIdx.x == 0 && W > 0) U[0] = g.uinteger;
}

// ---------------------------------------------------------------------------
// negatives
// ---------------------------------------------------------------------------
constexpr int COIN_PER_THREAD = 16;

__global__ void k_neg_init(const int32_t* __restrict__ core, int64_t m, int32_t s, const kg_pcg64* __restrict__ gp,
                           int32_t* __restrict__ neg, int8_t* __restrict__ col, int32_t* __restrict__ pending) {
  const kg_pcg64 g = *gp;
  const u128 s0 = state_of(g), inc = inc_of(g);
  const int64_t total = m * s;
  for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * COIN_PER_THREAD; i0 < total;
       i0 += (int64_t)gridDim.x * blockDim.x * COIN_PER_THREAD) {
    u128 st = apply_jump(pcg_jump((uint64_t)i0, inc), s0);
    for (int j = 0; j < COIN_PER_THREAD; ++j) {
      int64_t i = i0 + j;
      if (i >= total) break;
      st = pcg_step(st, inc);
      uint64_t x = pcg_output(st);
      // random() < 0.5  <=>  (x >> 11) * 2^-53 < 0.5  <=>  top bit clear
      col[i] = (x >> 63) ? 2 : 0;
      int64_t e = i / s;
      neg[i * 3 + 0] = core[e * 3 + 0];
      neg[i * 3 + 1] = core[e * 3 + 1];
      neg[i * 3 + 2] = core[e * 3 + 2];
      pending[i] = (int32_t)i;
    }
  }
}

__device__ __forceinline__ bool key_present(const int64_t* __restrict__ keys, int32_t nk, int64_t key) {
  int32_t lo = 0, hi = nk;
  while (lo < hi) {
    int32_t mid = (lo + hi) >> 1;
    if (keys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo < nk && keys[lo] == key;
}

__device__ __forceinline__ int64_t triple_key(int32_t h, int32_t r, int32_t t, int32_t n, int32_t R) {
  return ((int64_t)h * R + r) * (int64_t)n + t;
}

__global__ void k_lemire_flags(const uint32_t* __restrict__ U, int64_t W, uint32_t n, uint32_t thr,
                               uint32_t* __restrict__ flags) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < W; p += (int64_t)gridDim.x * blockDim.x) {
    uint64_t mm = (uint64_t)U[p] * n;
    flags[p] = ((uint32_t)mm >= thr) ? 1u : 0u;
  }
}

__global__ void k_neg_assign(const uint32_t* __restrict__ U, const uint32_t* __restrict__ flags,
                             const uint32_t* __restrict__ rank, int64_t W, uint32_t n_pool,
                             const int32_t* __restrict__ pending, const int32_t* __restrict__ kp,
                             int32_t* __restrict__ neg,
                             const int8_t* __restrict__ col, const int32_t* __restrict__ core, int32_t s,
                             int32_t n_local, int32_t R, const int64_t* __restrict__ keys,
                             const int32_t* __restrict__ n_keys, uint32_t* __restrict__ bad,
                             int64_t* __restrict__ consumed) {
  const int32_t nk = *n_keys;
  const int64_t k = *kp;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < W; p += (int64_t)gridDim.x * blockDim.x) {
    if (!flags[p]) continue;
    uint32_t q = rank[p];
    if (q >= k) continue;
    uint32_t draw = (uint32_t)(((uint64_t)U[p] * n_pool) >> 32);
    int32_t row = pending[q];
    int c = col[row];
    neg[(int64_t)row * 3 + c] = (int32_t)draw;
    int32_t orig = core[(int64_t)(row / s) * 3 + c];
    int32_t h = neg[(int64_t)row * 3 + 0], r = neg[(int64_t)row * 3 + 1], t = neg[(int64_t)row * 3 + 2];
    bool b = ((int32_t)draw == orig) || key_present(keys, nk, triple_key(h, r, t, n_local, R));
    bad[q] = b ? 1u : 0u;
    if (q == k - 1) *consumed = p + 1;
  }
}

__global__ void k_scatter_pending(const uint32_t* __restrict__ bad, const uint32_t* __restrict__ rank,
                                  const int32_t* __restrict__ kp, const int32_t* __restrict__ pending,
                                  int32_t* __restrict__ next, const uint32_t* __restrict__ total,
                                  int32_t* __restrict__ next_count) {
  const int64_t k = *kp;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < k; q += (int64_t)gridDim.x * blockDim.x)
    if (bad[q]) next[rank[q]] = pending[q];
  if (blockIdx.x == 0 && threadIdx.x == 0) *next_count = (int32_t)*total;
}

// Device-resident PCG64 bookkeeping (one thread): the sampler's RNG state
// lives in HBM so an epoch's sampling is a sync-free chain of kernels.
__global__ void k_pcg_advance(kg_pcg64* __restrict__ g, uint64_t delta) {
  u128 s = apply_jump(pcg_jump(delta, inc_of(*g)), state_of(*g));
  g->state_hi = s.hi;
  g->state_lo = s.lo;
}

// numpy Generator.uniform(low, high, size=count) from the stream position
// `g` (host state, passed by value): out[j] = low + (high - low) * random_j,
// random_j = (next64_j >> 11) * 2^-53, multiply and add rounded separately as
// numpy's C code does (ref:model.py:108-128, the embedding-table draw).
constexpr int UNIF_PER_THREAD = 16;
__global__ void k_uniform_f64(kg_pcg64 g, int64_t count, double low, double range, double* __restrict__ out) {
  const u128 s0 = state_of(g), inc = inc_of(g);
  for (int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * UNIF_PER_THREAD; j0 < count;
       j0 += (int64_t)gridDim.x * blockDim.x * UNIF_PER_THREAD) {
    u128 st = apply_jump(pcg_jump((uint64_t)j0, inc), s0);
    for (int k = 0; k < UNIF_PER_THREAD && j0 + k < count; ++k) {
      st = pcg_step(st, inc);
      const double u = (double)(pcg_output(st) >> 11) * (1.0 / 9007199254740992.0);
      out[j0 + k] = __dadd_rn(low, __dmul_rn(range, u));
    }
  }
}

// Inverted dropout (ref:model.py:221-227): keep = rng.random((T, d)) >= p,
// mask = keep / (1 - p). random() is (next64 >> 11) * 2^-53, one next64 per
// value in row-major order, so value j sits at stream position j: each thread
// jumps to its first position and steps. T = counts[t] lives on the device.
constexpr int DROP_PER_THREAD = 32;

__global__ void k_dropout_mask(const kg_pcg64* __restrict__ gp, const int32_t* __restrict__ counts, int t, int d,
                               double p, float scale, float* __restrict__ mask) {
  const kg_pcg64 g = *gp;
  const u128 s0 = state_of(g), inc = inc_of(g);
  const int64_t total = (int64_t)counts[t] * d;
  for (int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * DROP_PER_THREAD; j0 < total;
       j0 += (int64_t)gridDim.x * blockDim.x * DROP_PER_THREAD) {
    u128 st = apply_jump(pcg_jump((uint64_t)j0, inc), s0);
    for (int k = 0; k < DROP_PER_THREAD && j0 + k < total; ++k) {
      st = pcg_step(st, inc);
      const double u = (double)(pcg_output(st) >> 11) * (1.0 / 9007199254740992.0);
      mask[j0 + k] = u >= p ? scale : 0.f;
    }
  }
}

// advance by counts[t] * d next64 draws (after k_dropout_mask)
__global__ void k_pcg_advance_count(kg_pcg64* __restrict__ g, const int32_t* __restrict__ counts, int t, int d) {
  const uint64_t delta = (uint64_t)counts[t] * (uint64_t)d;
  u128 s = apply_jump(pcg_jump(delta, inc_of(*g)), state_of(*g));
  g->state_hi = s.hi;
  g->state_lo = s.lo;
}

// consume `*count` next_uint32 draws; *count < 0 (failed draw) leaves g as is.
// With `need` set, a zero count while need[0] > 0 means the window was too
// small: it is flagged as -1 so the host retries with a larger window.
__global__ void k_pcg_consume32(kg_pcg64* __restrict__ g, int64_t* __restrict__ count,
                                const int32_t* __restrict__ need) {
  int64_t c = *count;
  if (need && *need > 0 && c == 0) {
    *count = -1;
    return;
  }
  if (c <= 0) return;
  uint64_t cnt = (uint64_t)c;
  if (g->has_uint32) {
    g->has_uint32 = 0;
    cnt -= 1;
  }
  if (cnt == 0) return;
  uint64_t words = (cnt + 1) / 2;
  u128 s = apply_jump(pcg_jump(words, inc_of(*g)), state_of(*g));
  uint64_t x = pcg_output(s);
  g->state_hi = s.hi;
  g->state_lo = s.lo;
  g->has_uint32 = (cnt & 1) ? 1u : 0u;
  g->uinteger = (uint32_t)(x >> 32);
}

__global__ void k_is_positive(const int32_t* __restrict__ tri, int64_t k, int32_t n, int32_t R,
                              const int64_t* __restrict__ keys, const int32_t* __restrict__ n_keys,
                              uint8_t* __restrict__ out) {
  const int32_t nk = *n_keys;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = key_present(keys, nk, triple_key(tri[i * 3], tri[i * 3 + 1], tri[i * 3 + 2], n, R)) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// permutation: speculative single-warp Fisher-Yates draw
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smear(uint32_t x) {
  x |= x >> 1; x |= x >> 2; x |= x >> 4; x |= x >> 8; x |= x >> 16;
  return x;
}

constexpr int RING_Q = 1024;           // uint32 per quarter
constexpr int RING = 4 * RING_Q;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// One warp walks i = n-1 .. 1 over a speculative window of 128 uint32 stream
// positions (4 per lane, position p + 32r + lane). With a uniform mask over
// the window, offset o is certainly accepted when (U & mask) <= i - o and
// certainly rejected when (U & mask) > i; the first ambiguous offset is
// resolved exactly and the window restarts after it. Positions stream through
// a 4-quarter shared-memory ring filled by cp.async two quarters ahead.
constexpr int PR = 8;            // positions per lane per window
constexpr int PW = 32 * PR;      // window

__global__ void __launch_bounds__(32) k_perm_draws(const uint32_t* __restrict__ U, int64_t W, int64_t n,
                                                   int32_t* __restrict__ js, int64_t* __restrict__ consumed) {
  __shared__ __align__(16) uint32_t ring[RING];
  const unsigned lane = lane_id();
  int64_t issued = 0;
  auto issue = [&](int64_t q) {
    int64_t base = q * RING_Q;
    uint32_t* dst = ring + (q & 3) * RING_Q;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int64_t e = base + (int64_t)(j * 32 + lane) * 4;
      if (e + 4 <= W) cp_async16(dst + (j * 32 + lane) * 4, U + e);
    }
    cp_async_commit();
  };
  int64_t i = n - 1, p = 0;
  int64_t waited_q = -1;
  bool ok = true;
  while (i >= 1) {
    const int64_t need_q = (p + PW - 1) / RING_Q;
    if (need_q > waited_q) {
      while (issued <= need_q + 2) {
        if (issued * RING_Q < W) issue(issued);
        else cp_async_commit();
        ++issued;
      }
      cp_async_wait<2>();
      __syncwarp();
      waited_q = need_q;
    }
    if (p + PW > W) { ok = false; break; }
    const uint32_t ii = (uint32_t)i;
    const uint32_t mask = smear(ii);
    if (ii < 32) {
      // one exact draw for this i (lane 0), broadcast
      int64_t pp = p;
      uint32_t v = 0;
      if (lane == 0) {
        while (true) {
          if (pp >= W) { pp = -1; break; }
          uint32_t u = (pp < (waited_q + 1) * RING_Q) ? ring[pp & (RING - 1)] : U[pp];
          ++pp;
          v = u & mask;
          if (v <= ii) break;
        }
      }
      pp = __shfl_sync(0xffffffffu, pp, 0);
      v = __shfl_sync(0xffffffffu, v, 0);
      if (pp < 0) { ok = false; break; }
      if (lane == 0) js[i] = (int32_t)v;
      p = pp;
      i -= 1;
      continue;
    }
    // draws at offsets < Wl all have indices in [2^k, ii] (one mask): the
    // window shrinks near a power of two instead of drawing one at a time
    const int Wl = (int)min((uint32_t)PW, ii - (mask >> 1));
    uint32_t v[PR];
    unsigned acc_b[PR], amb_b[PR];
#pragma unroll
    for (int r = 0; r < PR; ++r) {
      v[r] = ring[(p + r * 32 + lane) & (RING - 1)] & mask;
      const uint32_t o = r * 32 + lane;
      const bool in = (int)o < Wl;
      const bool acc_sure = in && v[r] + o <= ii;
      const bool rej_sure = v[r] > ii;
      acc_b[r] = __ballot_sync(0xffffffffu, acc_sure);
      amb_b[r] = __ballot_sync(0xffffffffu, in && !acc_sure && !rej_sure);
    }
    int f = PW;
#pragma unroll
    for (int r = PR - 1; r >= 0; --r)
      if (amb_b[r]) f = r * 32 + __ffs(amb_b[r]) - 1;
    const int stop = f < Wl ? f : Wl;   // first position not decided by this window
    int before = 0;   // accepts at offsets < 32r (running over r)
#pragma unroll
    for (int r = 0; r < PR; ++r) {
      unsigned lim = (stop >= (r + 1) * 32) ? 0xffffffffu : (stop <= r * 32 ? 0u : ((1u << (stop - r * 32)) - 1u));
      unsigned am = acc_b[r] & lim;
      if ((am >> lane) & 1u) {
        uint32_t il = ii - before - __popc(am & lanemask_lt());
        js[il] = (int32_t)v[r];
      }
      before += __popc(am);
    }
    int taken = Wl;
    if (f < Wl) {
      uint32_t il_f = ii - before;
      uint32_t vf = 0;
#pragma unroll
      for (int r = 0; r < PR; ++r) {
        uint32_t x = __shfl_sync(0xffffffffu, v[r], f & 31);
        if ((f >> 5) == r) vf = x;
      }
      if (vf <= il_f) {
        if (lane == 0) js[il_f] = (int32_t)vf;
        before += 1;
      }
      taken = f + 1;
    }
    p += taken;
    i -= before;
  }
  cp_async_wait<0>();
  if (lane == 0) *consumed = ok ? p : -1;
}

// Block-parallel variant (8 warps, window of 2048 stream positions). Every
// position is classified against the window's bounds as above (certain
// accept: v <= i - o; certain reject: v > i; else ambiguous), but an
// ambiguous position no longer ends the window: one thread walks the (few)
// ambiguous positions in stream order, each decided with its exact index
// i - (accepts before it), and the window runs to its end (or to the first
// position whose index could leave the mask's power-of-two range). The
// accepts' indices then follow from a prefix count over the window. Same
// draws, same stream positions as the one-warp walk, ~8x the positions per
// step (ambiguity stays rare: ~o / 2^k per position at offset o).
constexpr int PB_WARPS = 8, PB_T = 32 * PB_WARPS, PB_R = 8, PB_W = PB_T * PB_R;   // 2048 positions
constexpr int PB_Q = 1024, PB_NQ = 16, PB_RING = PB_NQ * PB_Q, PB_AHEAD = 8;    // 64 KB ring, 8 quarters ahead

__global__ void __launch_bounds__(PB_T) k_perm_draws_block(const uint32_t* __restrict__ U, int64_t W, int64_t n,
                                                           int32_t* __restrict__ js, int64_t* __restrict__ consumed) {
  extern __shared__ __align__(16) uint32_t pring[];
  __shared__ unsigned accw[PB_W / 32], ambw[PB_W / 32], cpre[PB_W / 32 + 1];
  __shared__ int64_t sh_p, sh_i;
  __shared__ int sh_taken, sh_ok;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int64_t issued = 0, waited = -1;
  auto issue = [&](int64_t q) {
    const int64_t base = q * PB_Q;
    uint32_t* dst = pring + (q & (PB_NQ - 1)) * PB_Q;
    for (int j = t; j < PB_Q / 4; j += PB_T) {
      const int64_t e = base + (int64_t)j * 4;
      if (e + 4 <= W) cp_async16(dst + j * 4, U + e);
    }
    cp_async_commit();
  };
  if (t == 0) { sh_p = 0; sh_i = n - 1; sh_ok = 1; }
  __syncthreads();
  while (true) {
    const int64_t p = sh_p, i = sh_i;
    if (i < 32 || !sh_ok) break;
    // the window's positions in the ring (quarters up to need_q landed)
    const int64_t need_q = (p + PB_W - 1) / PB_Q;
    if (need_q > waited) {
      while (issued <= need_q + PB_AHEAD) {
        if (issued * PB_Q < W) issue(issued);
        else cp_async_commit();
        ++issued;
      }
      cp_async_wait<PB_AHEAD>();
      __syncthreads();
      waited = need_q;
    }
    if (p >= W) {   // draw buffer exhausted: the caller retries with a larger one
      if (t == 0) sh_ok = 0;
      __syncthreads();
      break;
    }
    const uint32_t ii = (uint32_t)i, mask = smear(ii);
    const int64_t avail = W - p;   // only positions < W were loaded
    const int Wl = (int)min((int64_t)min((uint32_t)PB_W, ii - (mask >> 1)), avail);
    uint32_t v[PB_R];
#pragma unroll
    for (int r = 0; r < PB_R; ++r) {
      const int o = r * PB_T + t;
      v[r] = pring[(p + o) & (PB_RING - 1)] & mask;
      const bool in = o < Wl;
      const bool acc = in && v[r] + (uint32_t)o <= ii;
      const bool amb = in && !acc && v[r] <= ii;
      const unsigned ab = __ballot_sync(0xffffffffu, acc), mb = __ballot_sync(0xffffffffu, amb);
      if (lane == 0) { accw[r * PB_WARPS + warp] = ab; ambw[r * PB_WARPS + warp] = mb; }
    }
    __syncthreads();
    if (warp == 0) {
      // word w covers positions 32w .. 32w + 31 (o = r*256 + warp*32 + lane,
      // w = o / 32). Lane l owns words 2l, 2l + 1: certain-accept prefix by a
      // warp scan; then the ambiguous positions in stream order, each decided
      // with its exact index (certain accepts before it + the ambiguous ones
      // accepted so far); then the prefix again over all accepts.
      auto scan_words = [&]() {
        const unsigned c0 = __popc(accw[2 * lane]), c1 = __popc(accw[2 * lane + 1]);
        unsigned x = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        cpre[2 * lane] = x - c0 - c1;
        cpre[2 * lane + 1] = x - c1;
        if (lane == 31) cpre[PB_W / 32] = x;
        __syncwarp();
      };
      scan_words();
      const unsigned has = __ballot_sync(0xffffffffu, (ambw[2 * lane] | ambw[2 * lane + 1]) != 0u);
      if (has) {
        unsigned res[2] = {0u, 0u};   // lane-owned resolved accepts
        unsigned extra = 0;           // ambiguous accepts so far (warp-uniform)
        unsigned hm = has;
        while (hm) {
          const int l = __ffs(hm) - 1;
          hm &= hm - 1;
          for (int h = 0; h < 2; ++h) {
            const int w = 2 * l + h;
            unsigned m = ambw[w];
            while (m) {
              const int b = __ffs(m) - 1;
              m &= m - 1;
              const int o = w * 32 + b;
              const unsigned before = cpre[w] + __popc(accw[w] & ((1u << b) - 1u)) + extra;
              const uint32_t vo = pring[(p + o) & (PB_RING - 1)] & mask;
              if (vo <= ii - before) {
                ++extra;
                if (lane == l) res[h] |= 1u << b;
              }
            }
          }
        }
        __syncwarp();
        accw[2 * lane] |= res[0];
        accw[2 * lane + 1] |= res[1];
        __syncwarp();
        scan_words();
      }
      if (lane == 0) sh_taken = Wl;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < PB_R; ++r) {
      const int w = r * PB_WARPS + warp;
      const unsigned m = accw[w];
      if ((m >> lane) & 1u) {
        const uint32_t il = ii - cpre[w] - __popc(m & lanemask_lt());
        js[il] = (int32_t)v[r];
      }
    }
    __syncthreads();
    if (t == 0) {
      sh_p = p + sh_taken;
      sh_i = i - cpre[PB_W / 32];
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  // the last indices (i < 32): one exact draw at a time
  if (t == 0) {
    int64_t pp = sh_p, i = sh_i;
    bool ok = sh_ok;
    while (ok && i >= 1) {
      const uint32_t ii = (uint32_t)i, mask = smear(ii);
      while (true) {
        if (pp >= W) { ok = false; break; }
        const uint32_t x = U[pp++] & mask;
        if (x <= ii) { js[i] = (int32_t)x; break; }
      }
      --i;
    }
    *consumed = ok ? pp : -1;
  }
}

// group swap targets: members of group j are the i with js[i] == j (ascending)
__global__ void k_group_count(const int32_t* __restrict__ js, int64_t n, uint32_t* __restrict__ cnt) {
  for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[js[i]], 1u);
}

__global__ void k_group_fill(const int32_t* __restrict__ js, int64_t n, const uint32_t* __restrict__ start,
                             uint32_t* __restrict__ fill, int32_t* __restrict__ members) {
  for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t j = js[i];
    uint32_t slot = atomicAdd(&fill[j], 1u);
    members[start[j] + slot] = (int32_t)i;
  }
}

// sort each (small) group ascending; T(p) = first member > p; ptr = T or self
__global__ void k_group_sort_T(int32_t* __restrict__ members, const uint32_t* __restrict__ start,
                               const uint32_t* __restrict__ cnt, int64_t n, int32_t* __restrict__ ptr) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    uint32_t a = start[p], c = cnt[p];
    int32_t* g = members + a;
    for (uint32_t x = 1; x < c; ++x) {
      int32_t key = g[x];
      int32_t y = (int32_t)x - 1;
      while (y >= 0 && g[y] > key) { g[y + 1] = g[y]; --y; }
      g[y + 1] = key;
    }
    int32_t t = (int32_t)p;
    for (uint32_t x = 0; x < c; ++x)
      if (g[x] > (int32_t)p) { t = g[x]; break; }
    ptr[p] = t;
  }
}

// One pointer-jumping round. The rounds are a fixed chain of launches (a
// captured graph cannot branch), so each round records whether it moved any
// pointer and a round after a round that moved none returns at once: the
// chain costs its launch latencies past convergence, not full passes.
__global__ void k_pointer_jump(int32_t* __restrict__ ptr, int64_t n, const uint32_t* __restrict__ prev_moved,
                               uint32_t* __restrict__ moved) {
  if (prev_moved && *prev_moved == 0u) return;
  bool any = false;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int32_t q = ptr[p];
    int32_t r = ptr[q];
    if (r != q) {
      ptr[p] = r;
      any = true;
    }
  }
  if (__syncthreads_or(any) && threadIdx.x == 0) *moved = 1u;
}

__global__ void k_perm_final(const int32_t* __restrict__ js, int64_t n, const int32_t* __restrict__ members,
                             const uint32_t* __restrict__ start, const uint32_t* __restrict__ cnt,
                             const int32_t* __restrict__ root, int32_t* __restrict__ perm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == 0) { perm[0] = root[0]; continue; }
    int32_t j = js[i];
    const int32_t* g = members + start[j];
    uint32_t c = cnt[j];
    int32_t succ = -1;
    for (uint32_t x = 0; x < c; ++x)
      if (g[x] == (int32_t)i) { if (x + 1 < c) succ = g[x + 1]; break; }
    perm[i] = succ >= 0 ? root[succ] : j;
  }
}

__global__ void k_stream_gather(const int32_t* __restrict__ pos, int64_t npos, const int32_t* __restrict__ neg,
                                int64_t nneg, const int32_t* __restrict__ perm, int32_t* __restrict__ out,
                                float* __restrict__ labels) {
  int64_t total = npos + nneg;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = perm[k];
    const int32_t* src = i < npos ? pos + i * 3 : neg + (i - npos) * 3;
    out[k * 3 + 0] = src[0];
    out[k * 3 + 1] = src[1];
    out[k * 3 + 2] = src[2];
    labels[k] = i < npos ? 1.0f : 0.0f;
  }
}

// ---------------------------------------------------------------------------
// closure
// ---------------------------------------------------------------------------
__global__ void k_closure_clear(int32_t* __restrict__ pos, uint32_t* __restrict__ flags, int64_t n,
                                int32_t* __restrict__ bad) {
  if (blockIdx.x == 0 && threadIdx.x < 4) bad[threadIdx.x] = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    pos[i] = -1;
    flags[i] = 0;
  }
}

__global__ void k_mark_batch(const int32_t* __restrict__ tri, int64_t total, int64_t start,
                             const int64_t* __restrict__ start_dev, int64_t b, const int32_t* __restrict__ ids,
                             int32_t n, uint32_t* __restrict__ flags, int32_t* __restrict__ bad) {
  if (start_dev) start = *start_dev;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < b; q += (int64_t)gridDim.x * blockDim.x) {
    if (tri) {
      int64_t row = (start + q) % total;
      int32_t h = tri[row * 3], t = tri[row * 3 + 2];
      if (h < 0 || h >= n || t < 0 || t >= n) { *bad = 1; continue; }
      flags[h] = 1u;
      flags[t] = 1u;
    } else {
      int32_t v = ids[q];
      if (v < 0 || v >= n) { *bad = 1; continue; }
      flags[v] = 1u;
    }
  }
}

// warp per active vertex: flag unplaced sources of its messages
// warp per static CSR chunk of an active vertex: flag unplaced sources
__global__ void k_mark_sources(const int32_t* __restrict__ ck_ptr, const int32_t* __restrict__ ck_row,
                               const int32_t* __restrict__ ck_counts, int C, const int32_t* __restrict__ counts,
                               int hop, const int32_t* __restrict__ indptr, const int32_t* __restrict__ src,
                               const int32_t* __restrict__ pos, uint32_t* __restrict__ flags) {
  const int32_t active = counts[hop];
  const int32_t NC = ck_counts[0];
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int64_t c = warp_uniform((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); c < NC; c += warps) {
    int32_t v = ck_row[c];
    int32_t p = pos[v];
    if (p < 0 || p >= active) continue;
    int32_t beg = indptr[v] + (int32_t)(c - ck_ptr[v]) * C;
    int32_t end = min(beg + C, indptr[v + 1]);
    for (int32_t e = beg + (int32_t)lane_id(); e < end; e += 32) {
      int32_t u = src[e];
      if (pos[u] < 0) flags[u] = 1u;
    }
  }
}

}  // namespace kg

using namespace kg;

extern "C" {

// --- host PCG64 bookkeeping ----------------------------------------------
void kg_pcg64_advance(kg_pcg64* g, uint64_t delta) {
  u128 s = apply_jump(pcg_jump(delta, inc_of(*g)), state_of(*g));
  g->state_hi = s.hi;
  g->state_lo = s.lo;
}

void kg_pcg64_consume32(kg_pcg64* g, uint64_t count) {
  if (count == 0) return;
  if (g->has_uint32) {
    g->has_uint32 = 0;   // numpy keeps the stale uinteger value
    count -= 1;
  }
  if (count == 0) return;
  // ceil(count/2) fresh words; numpy leaves uinteger = high half of the last
  // word whether or not that half was consumed (has_uint32 = count odd)
  uint64_t words = (count + 1) / 2;
  u128 s = apply_jump(pcg_jump(words, inc_of(*g)), state_of(*g));
  uint64_t x = pcg_output(s);
  g->state_hi = s.hi;
  g->state_lo = s.lo;
  g->has_uint32 = (count & 1) ? 1 : 0;
  g->uinteger = (uint32_t)(x >> 32);
}

void kg_pcg64_peek64(const kg_pcg64* g, uint64_t* out, int64_t count) {
  u128 s = state_of(*g), inc = inc_of(*g);
  for (int64_t i = 0; i < count; ++i) {
    s = pcg_step(s, inc);
    out[i] = pcg_output(s);
  }
}

// --- negatives -------------------------------------------------------------
kg_status kg_neg_init(const int32_t* core, int64_t m, int32_t s, kg_pcg64* g, int32_t* neg, int8_t* col,
                      int32_t* pending, void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(s >= 1 && m >= 1, KG_ERR_VALIDATION, "neg_init needs s >= 1 and m >= 1");
  KG_REQUIRE(m * (int64_t)s < (int64_t(1) << 31), KG_ERR_VALIDATION, "too many negatives");
  int64_t total = m * s;
  int blocks = persistent_blocks(ceil_div(total, COIN_PER_THREAD), 256, 8);
  KG_LAUNCH("k_neg_init", k_neg_init, blocks, 256, 0, st, core, m, s, g, neg, col, pending);
  KG_LAUNCH("k_pcg_advance", k_pcg_advance, 1, 1, 0, st, g, (uint64_t)total);   // one next64 per coin
  return KG_OK;
}

int64_t kg_neg_round_workspace_bytes(int64_t W) {
  return (int64_t)(align_up(W * 4) * 5 + scan_workspace(W) + 8192);
}

kg_status kg_neg_round(int32_t* neg, const int8_t* col, const int32_t* core, int32_t s, const int32_t* pending,
                       const int32_t* k_dev, int64_t k_max, int64_t pool_size, int32_t n_local, int32_t R,
                       const int64_t* pos_keys, const int32_t* n_keys, kg_pcg64* g, int64_t W,
                       int32_t* next_pending, int32_t* next_count, int64_t* consumed, void* ws, int64_t ws_bytes,
                       void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(pool_size >= 2 && pool_size <= 0xFFFFFFFFLL, KG_ERR_SAMPLING, "pool size out of range");
  KG_REQUIRE(W >= k_max && k_max >= 1, KG_ERR_VALIDATION, "bad resampling window");
  KG_REQUIRE(ws_bytes >= kg_neg_round_workspace_bytes(W), KG_ERR_VALIDATION, "neg workspace too small");
  Arena a(ws, (size_t)ws_bytes);
  uint32_t* U = a.take<uint32_t>(W);
  uint32_t* flags = a.take<uint32_t>(W);
  uint32_t* rank = a.take<uint32_t>(W);
  uint32_t* bad = a.take<uint32_t>(W);
  uint32_t* bad_rank = a.take<uint32_t>(W);
  uint32_t* totals = a.take<uint32_t>(4);
  char* sws = a.take<char>(scan_workspace(W));
  uint32_t n = (uint32_t)pool_size;
  KG_CUDA(cudaMemsetAsync(consumed, 0, sizeof(int64_t), st));
  KG_CUDA(cudaMemsetAsync(bad, 0, k_max * sizeof(uint32_t), st));
  KG_LAUNCH("k_gen_u32", k_gen_u32, persistent_blocks(ceil_div(W / 2 + 2, GEN_WORDS), 256, 8), 256, 0, st, g, W, U);
  KG_LAUNCH("k_lemire_flags", k_lemire_flags, grid_for(W), 256, 0, st, U, W, n, lemire_threshold(n), flags);
  kg_status r = exclusive_scan_u32(flags, rank, W, totals, sws, scan_workspace(W), st);
  if (r != KG_OK) return r;
  KG_LAUNCH("k_neg_assign", k_neg_assign, grid_for(W), 256, 0, st, U, flags, rank, W, n, pending, k_dev, neg, col,
            core, s, n_local, R, pos_keys, n_keys, bad, consumed);
  r = exclusive_scan_u32(bad, bad_rank, k_max, totals + 1, sws, scan_workspace(W), st);
  if (r != KG_OK) return r;
  KG_LAUNCH("k_scatter_pending", k_scatter_pending, grid_for(k_max), 256, 0, st, bad, bad_rank, k_dev, pending,
            next_pending, totals + 1, next_count);
  // advance the device state by the draws used (-1 flags a too-small window)
  KG_LAUNCH("k_pcg_consume32", k_pcg_consume32, 1, 1, 0, st, g, consumed, k_dev);
  return KG_OK;
}

kg_status kg_is_positive(const int32_t* triples, int64_t k, int32_t n_local, int32_t R, const int64_t* pos_keys,
                         const int32_t* n_keys, uint8_t* out, void* stream) {
  if (k <= 0) return KG_OK;
  KG_LAUNCH("k_is_positive", k_is_positive, grid_for(k), 256, 0, as_stream(stream), triples, k, n_local, R, pos_keys, n_keys, out);
  KG_CHECK_LAUNCH("k_is_positive");
  return KG_OK;
}

// --- permutation -----------------------------------------------------------
int64_t kg_perm_draws_buffer_len(int64_t n) {
  // expected draws < 2n (acceptance >= 1/2 per attempt); generous slack
  return ((2 * n + 8192 + 4 * 1024) / 1024 + 4) * 1024;
}

kg_status kg_perm_draws_buffered(int64_t n, kg_pcg64* g, uint32_t* U, int64_t W, int32_t* js, int64_t* consumed32,
                                 void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(n >= 1 && n < (int64_t(1) << 31), KG_ERR_VALIDATION, "permutation size out of range");
  if (n == 1) {
    KG_CUDA(cudaMemsetAsync(consumed32, 0, sizeof(int64_t), st));
    return KG_OK;
  }
  KG_REQUIRE(W % 4 == 0 && W >= 4096, KG_ERR_VALIDATION, "draw buffer must be a multiple of 4 >= 4096");
  KG_LAUNCH("k_gen_u32", k_gen_u32, persistent_blocks(ceil_div(W / 2 + 2, GEN_WORDS), 256, 8), 256, 0, st, g, W, U);
  // the block walk pays a block barrier per window: it wins on long streams
  // (P = 1 at FB shape: 1.68 -> 1.22 ms), the one-warp walk on short ones
  const char* pe = getenv("KG_PERM_BLOCK_MIN");
  if (n >= (pe ? atoll(pe) : 262144LL)) {
    static bool attr = false;
    if (!attr) {
      KG_CUDA(cudaFuncSetAttribute(k_perm_draws_block, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   PB_RING * (int)sizeof(uint32_t)));
      attr = true;
    }
    KG_LAUNCH("k_perm_draws", k_perm_draws_block, 1, PB_T, PB_RING * sizeof(uint32_t), st, U, W, n, js, consumed32);
  } else {
    KG_LAUNCH("k_perm_draws", k_perm_draws, 1, 32, 0, st, U, W, n, js, consumed32);
  }
  KG_LAUNCH("k_pcg_consume32", k_pcg_consume32, 1, 1, 0, st, g, consumed32, (const int32_t*)nullptr);
  return KG_OK;
}

int64_t kg_perm_resolve_workspace_bytes(int64_t n) {
  return (int64_t)(align_up(n * 4) * 5 + scan_workspace(n) + 4096 + align_up(64 * 4));
}

kg_status kg_perm_resolve(const int32_t* js, int64_t n, int32_t* perm, void* ws, int64_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  KG_REQUIRE(ws_bytes >= kg_perm_resolve_workspace_bytes(n), KG_ERR_VALIDATION, "perm workspace too small");
  if (n == 1) {
    KG_CUDA(cudaMemsetAsync(perm, 0, sizeof(int32_t), st));
    return KG_OK;
  }
  Arena a(ws, (size_t)ws_bytes);
  uint32_t* cnt = a.take<uint32_t>(n);
  uint32_t* start = a.take<uint32_t>(n);
  uint32_t* fill = a.take<uint32_t>(n);
  int32_t* members = a.take<int32_t>(n);
  int32_t* root = a.take<int32_t>(n);
  char* sws = a.take<char>(scan_workspace(n));
  KG_CUDA(cudaMemsetAsync(cnt, 0, n * 4, st));
  KG_CUDA(cudaMemsetAsync(fill, 0, n * 4, st));
  int gb = grid_for(n);
  KG_LAUNCH("k_group_count", k_group_count, gb, 256, 0, st, js, n, cnt);
  kg_status r = exclusive_scan_u32(cnt, start, n, nullptr, sws, scan_workspace(n), st);
  if (r != KG_OK) return r;
  KG_LAUNCH("k_group_fill", k_group_fill, gb, 256, 0, st, js, n, start, fill, members);
  KG_LAUNCH("k_group_sort_T", k_group_sort_T, gb, 256, 0, st, members, start, cnt, n, root);
  int rounds = 1;
  while ((int64_t(1) << rounds) < n) ++rounds;
  uint32_t* moved = a.take<uint32_t>(rounds + 1);
  KG_CUDA(cudaMemsetAsync(moved, 0, (size_t)(rounds + 1) * 4, st));
  for (int it = 0; it < rounds + 1; ++it)
    KG_LAUNCH("k_pointer_jump", k_pointer_jump, gb, 256, 0, st, root, n, it ? moved + it - 1 : nullptr, moved + it);
  KG_LAUNCH("k_perm_final", k_perm_final, gb, 256, 0, st, js, n, members, start, cnt, root, perm);
  KG_CHECK_LAUNCH("perm resolve");
  return KG_OK;
}

kg_status kg_stream_gather(const int32_t* pos, int64_t npos, const int32_t* neg, int64_t nneg, const int32_t* perm,
                           int32_t* stream_triples, float* labels, void* stream) {
  if (npos + nneg == 0) return KG_OK;
  KG_LAUNCH("k_stream_gather", k_stream_gather, grid_for(npos + nneg), 256, 0, as_stream(stream), pos, npos, neg, nneg, perm,
                                                                        stream_triples, labels);
  KG_CHECK_LAUNCH("k_stream_gather");
  return KG_OK;
}

// --- uniform draws ---------------------------------------------------------------
kg_status kg_uniform_f64(const kg_pcg64* g, int64_t count, double low, double high, double* out, void* stream) {
  if (count <= 0) return KG_OK;
  KG_LAUNCH("k_uniform_f64", k_uniform_f64, persistent_blocks(ceil_div(count, UNIF_PER_THREAD), 256, 8), 256, 0,
            as_stream(stream), *g, count, low, high - low, out);
  return KG_OK;
}

// --- dropout -------------------------------------------------------------------
kg_status kg_dropout_mask(kg_pcg64* g, const int32_t* counts, int32_t t, int32_t d, double p, int64_t n_max,
                          float* mask, void* stream) {
  KG_REQUIRE(p > 0.0 && p < 1.0, KG_ERR_VALIDATION, "dropout must be in (0, 1)");
  cudaStream_t st = as_stream(stream);
  KG_LAUNCH("k_dropout_mask", k_dropout_mask, persistent_blocks(ceil_div(n_max * d, DROP_PER_THREAD), 256, 8), 256, 0,
            st, g, counts, t, d, p, (float)(1.0 / (1.0 - p)), mask);
  KG_LAUNCH("k_pcg_advance", k_pcg_advance_count, 1, 1, 0, st, g, counts, t, d);
  return KG_OK;
}

// --- closure -------------------------------------------------------------------
int64_t kg_closure_workspace_bytes(int32_t n) {
  return (int64_t)(align_up((int64_t)n * 4) + compact_workspace(n) + 4096);
}

kg_status kg_closure(const int32_t* tri, int64_t total, int64_t start, const int64_t* start_dev, int64_t b,
                     const int32_t* seed_ids, const kg_graph_csr* G, int32_t hops, int32_t* order, int32_t* pos,
                     int32_t* counts, void* ws, int64_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  const int32_t n = G->n;
  KG_REQUIRE(hops >= 0, KG_ERR_VALIDATION, "hops must be >= 0");
  KG_REQUIRE(b >= 1, KG_ERR_VALIDATION, "empty batch");
  KG_REQUIRE(ws_bytes >= kg_closure_workspace_bytes(n), KG_ERR_VALIDATION, "closure workspace too small");
  Arena a(ws, (size_t)ws_bytes);
  uint32_t* flags = a.take<uint32_t>(n);
  int32_t* bad = a.take<int32_t>(4);
  char* cws = a.take<char>(compact_workspace(n));
  // pos = -1, flags = 0, bad = 0; every compaction below clears the flags it read
  KG_LAUNCH("k_closure_clear", k_closure_clear, grid_for(n), 256, 0, st, pos, flags, n, bad);
  KG_LAUNCH("k_mark_batch", k_mark_batch, grid_for(b), 256, 0, st, tri, total, start, start_dev, b, seed_ids, n,
            flags, bad);
  // A_0 in ascending id order; pos and counts[0] written by the same pass
  kg_status r = compact_flags_ex(flags, n, order, nullptr, counts, pos, cws, compact_workspace(n), st);
  if (r != KG_OK) return r;
  for (int h = 0; h < hops; ++h) {
    KG_LAUNCH("k_mark_sources", k_mark_sources, persistent_blocks(((int64_t)n + G->e / G->chunk + 1) * 32, 256, 8), 256,
              0, st, G->ck_ptr, G->ck_row, G->ck_counts, G->chunk, counts, h, G->indptr, G->src, pos, flags);
    // append newly reached vertices (ascending) after counts[h]; counts[h+1] = counts[h] + new
    r = compact_flags_ex(flags, n, order, counts + h, counts + h + 1, pos, cws, compact_workspace(n), st);
    if (r != KG_OK) return r;
  }
  return KG_OK;
}

}  // extern "C"

// this module's anchor for kg_preload_kernels (kg_primitives.cu)
extern "C" const void* kg_anchor_sampler() { return reinterpret_cast<const void*>(&kg::k_gen_u32); }
