// Host-side native input producers: the synthetic
// KG generator (ref:graph.py:336-393) and the streaming vertex-cut greedy
// (ref:partition.py:141-191), both bit-exact with the reference's numpy
// arithmetic. All pointers here are HOST pointers.
//
// Compiled with -ffp-contract=off: the vertex-cut score must round exactly
// like numpy's float64 expression (no fused multiply-add).
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <vector>

#include "../../include/kgdist_b200.h"
#include "kg_pcg64.cuh"

namespace {

using kg::u128;

struct HostRng {
  u128 s, inc;
  uint32_t has32, uint32v;

  explicit HostRng(const kg_pcg64& g)
      : s(kg::state_of(g)), inc(kg::inc_of(g)), has32(g.has_uint32), uint32v(g.uinteger) {}

  void store(kg_pcg64* g) const {
    g->state_hi = s.hi;
    g->state_lo = s.lo;
    g->has_uint32 = has32;
    g->uinteger = uint32v;
  }

  uint64_t next64() {
    s = kg::pcg_step(s, inc);
    return kg::pcg_output(s);
  }

  uint32_t next32() {
    if (has32) {
      has32 = 0;
      return uint32v;
    }
    uint64_t x = next64();
    has32 = 1;
    uint32v = (uint32_t)(x >> 32);
    return (uint32_t)x;
  }

  double random() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }

  // Generator.integers(n), 1 <= n <= 2^32 - 1 (n == 1 draws nothing)
  uint32_t integers(uint32_t n) {
    if (n == 1) return 0;
    uint64_t m = (uint64_t)next32() * n;
    uint32_t left = (uint32_t)m;
    if (left < n) {
      uint32_t thr = kg::lemire_threshold(n);
      while (left < thr) {
        m = (uint64_t)next32() * n;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

// open-addressing set of 64-bit keys
struct KeySet {
  std::vector<uint64_t> slots;
  uint64_t mask;
  explicit KeySet(int64_t expect) {
    uint64_t cap = 64;
    while (cap < (uint64_t)(expect * 2 + 16)) cap <<= 1;
    slots.assign(cap, ~0ULL);
    mask = cap - 1;
  }
  static uint64_t mix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
  }
  // true if inserted (was absent)
  bool insert(uint64_t key) {
    uint64_t i = mix(key) & mask;
    while (true) {
      if (slots[i] == ~0ULL) {
        slots[i] = key;
        return true;
      }
      if (slots[i] == key) return false;
      i = (i + 1) & mask;
    }
  }
};

}  // namespace

extern "C" {

// Edge loop of generate_synthetic: writes up to `target` (h, r, t) rows into
// out (host int64, row-major) and returns the count; *g is advanced exactly
// as numpy's Generator would be (the caller continues with permutation()).
int64_t kg_generate_synthetic(int64_t num_entities, int32_t num_relations, int64_t target, kg_pcg64* g,
                              int64_t* out, int64_t max_attempts) {
  HostRng rng(*g);
  KeySet seen(target);
  std::vector<int32_t> tail_pool;
  tail_pool.reserve((size_t)target);
  const double pref_prob = 0.75;
  int64_t m = 0, attempts = 0;
  const uint32_t N = (uint32_t)num_entities, R = (uint32_t)num_relations;
  while (m < target && attempts < max_attempts) {
    ++attempts;
    int64_t h = rng.integers(N);
    int64_t t;
    if (!tail_pool.empty() && rng.random() < pref_prob) {
      t = tail_pool[rng.integers((uint32_t)tail_pool.size())];
    } else {
      t = rng.integers(N);
    }
    if (h == t) continue;
    int64_t r = rng.integers(R);
    uint64_t key = ((uint64_t)h * R + (uint64_t)r) * (uint64_t)N + (uint64_t)t;
    if (!seen.insert(key)) continue;
    out[m * 3 + 0] = h;
    out[m * 3 + 1] = r;
    out[m * 3 + 2] = t;
    ++m;
    tail_pool.push_back((int32_t)t);
  }
  rng.store(g);
  return m;
}

// Greedy streaming vertex cut over edges visited in `order` (host int64):
// score_p = [p holds u](2 - share_u) + [p holds v](2 - share_v)
//         + bw * (max_s - size_p) / (1 + max_s - min_s), -inf at the cap,
// argmax with lowest-index ties (ref:partition.py:173-188).
kg_status kg_vertex_cut_assign(const int64_t* triples, int64_t m, int64_t num_entities, int32_t P,
                               const int64_t* order, double balance_weight, int64_t cap, int64_t* assign) {
  if (P < 1 || P > 4096) return KG_ERR_VALIDATION;
  std::vector<int64_t> theta((size_t)num_entities, 0);
  std::vector<uint8_t> member((size_t)num_entities * (size_t)P, 0);
  std::vector<int64_t> sizes((size_t)P, 0);
  std::vector<double> score((size_t)P);
  // endpoints in visit order (one gather pass), so the sequential loop reads
  // them linearly and can prefetch the vertex state of edges a few ahead
  std::vector<int64_t> eu((size_t)m), ev((size_t)m);
  for (int64_t k = 0; k < m; ++k) {
    eu[(size_t)k] = triples[order[k] * 3 + 0];
    ev[(size_t)k] = triples[order[k] * 3 + 2];
  }
  constexpr int64_t AHEAD = 16;
  for (int64_t k = 0; k < m; ++k) {
    if (k + AHEAD < m) {
      const int64_t pu = eu[(size_t)(k + AHEAD)], pv = ev[(size_t)(k + AHEAD)];
      __builtin_prefetch(&theta[(size_t)pu], 1);
      __builtin_prefetch(&theta[(size_t)pv], 1);
      __builtin_prefetch(&member[(size_t)pu * P], 1);
      __builtin_prefetch(&member[(size_t)pv * P], 1);
    }
    int64_t e = order[k];
    int64_t u = eu[(size_t)k], v = ev[(size_t)k];
    int64_t du = theta[u], dv = theta[v];
    int64_t tot = du + dv;
    double su = tot ? (double)du / (double)tot : 0.5;
    double sv = tot ? (double)dv / (double)tot : 0.5;
    int64_t max_s = sizes[0], min_s = sizes[0];
    for (int p = 1; p < P; ++p) {
      if (sizes[p] > max_s) max_s = sizes[p];
      if (sizes[p] < min_s) min_s = sizes[p];
    }
    const double denom = (1.0 + (double)max_s) - (double)min_s;
    const uint8_t* mu = &member[(size_t)u * P];
    const uint8_t* mv = &member[(size_t)v * P];
    int best = 0;
    for (int p = 0; p < P; ++p) {
      double a = mu[p] ? (2.0 - su) : 0.0;
      double b = mv[p] ? (2.0 - sv) : 0.0;
      double s = a + b;
      double bal = balance_weight * (double)(max_s - sizes[p]);
      s = s + bal / denom;
      if (sizes[p] >= cap) s = -INFINITY;
      score[p] = s;
      if (p > 0 && s > score[best]) best = p;
    }
    assign[e] = best;
    member[(size_t)u * P + best] = 1;
    member[(size_t)v * P + best] = 1;
    sizes[best] += 1;
    theta[u] += 1;
    theta[v] += 1;
  }
  return KG_OK;
}

}  // extern "C"
