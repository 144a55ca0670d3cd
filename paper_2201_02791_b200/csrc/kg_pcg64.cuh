// PCG64 (numpy's default BitGenerator) in 128-bit integer arithmetic for
// host and device, plus the positional helpers the sampler kernels use to
// reproduce numpy Generator streams bit-for-bit:
//   random()          -> (next64 >> 11) * 2^-53          (sampler.py:164, model.py:225)
//   integers(n)       -> Lemire on buffered next_uint32  (sampler.py:173)
//   permutation(n)    -> masked rejection on next_uint32 (sampler.py:220)
// numpy is an un-vendored dependency of the reference (pyproject.toml:10-13);
// the stream contract is restated in oracle/pcg64_ref.py and pinned there.
#pragma once
#include <stdint.h>

#ifndef __CUDACC__
#define __host__
#define __device__
#define __forceinline__ inline
#endif

#include "../../include/kgdist_b200.h"

namespace kg {

struct u128 {
  uint64_t lo, hi;
};

__host__ __device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) { return u128{lo, hi}; }

__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

__host__ __device__ __forceinline__ u128 mul128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo * b.lo;
  r.hi = mulhi64(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}

__host__ __device__ __forceinline__ u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}

// numpy PCG64 multiplier 0x2360ED051FC65DA44385DF649FCCF645
__host__ __device__ __forceinline__ u128 pcg_mult() {
  return mk128(0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL);
}

// LCG step, then XSL-RR output of the new state (numpy pcg64_next64)
__host__ __device__ __forceinline__ uint64_t pcg_output(u128 s) {
  uint64_t x = s.hi ^ s.lo;
  unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__host__ __device__ __forceinline__ u128 pcg_step(u128 s, u128 inc) { return add128(mul128(s, pcg_mult()), inc); }

// Affine map s -> A*s + C equal to `delta` LCG steps (Brown's jump-ahead).
struct Jump {
  u128 A, C;
};

__host__ __device__ inline Jump pcg_jump(uint64_t delta, u128 inc) {
  u128 acc_a = mk128(0, 1), acc_c = mk128(0, 0);
  u128 cur_a = pcg_mult(), cur_c = inc;
  while (delta) {
    if (delta & 1) {
      acc_a = mul128(acc_a, cur_a);
      acc_c = add128(mul128(acc_c, cur_a), cur_c);
    }
    cur_c = mul128(add128(cur_a, mk128(0, 1)), cur_c);
    cur_a = mul128(cur_a, cur_a);
    delta >>= 1;
  }
  return Jump{acc_a, acc_c};
}

__host__ __device__ __forceinline__ u128 apply_jump(const Jump& j, u128 s) { return add128(mul128(j.A, s), j.C); }

// next64 number k (0-based) drawn from state s (i.e. the output after k+1 steps)
__host__ __device__ inline uint64_t pcg_nth64(u128 s, u128 inc, uint64_t k) {
  Jump j = pcg_jump(k + 1, inc);
  return pcg_output(apply_jump(j, s));
}

__host__ __device__ __forceinline__ u128 state_of(const kg_pcg64& g) { return mk128(g.state_hi, g.state_lo); }
__host__ __device__ __forceinline__ u128 inc_of(const kg_pcg64& g) { return mk128(g.inc_hi, g.inc_lo); }

// uint32 stream position p -> (next64 index, half) given the buffered word.
// With has_uint32 set, position 0 is the buffered `uinteger`.
struct Pos32 {
  int64_t word;   // -1 => buffered uinteger
  int half;       // 0 = low 32 bits, 1 = high 32 bits
};

__host__ __device__ __forceinline__ Pos32 pos32(uint64_t p, uint32_t has_uint32) {
  Pos32 r;
  if (has_uint32) {
    if (p == 0) {
      r.word = -1;
      r.half = 0;
      return r;
    }
    p -= 1;
  }
  r.word = (int64_t)(p >> 1);
  r.half = (int)(p & 1);
  return r;
}

__host__ __device__ __forceinline__ uint32_t lemire_threshold(uint32_t n) {
  return (uint32_t)((0x100000000ULL - n) % n);
}

}  // namespace kg
