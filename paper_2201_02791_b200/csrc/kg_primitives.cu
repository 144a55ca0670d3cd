// Device-wide primitives used by the view builder, the sampler and the
// per-batch grouping: exclusive scan, stable LSD radix sort, flag compaction.
//
// Radix sort: 8-bit digits, tiles of 4096 keys (256 threads x 16 rounds).
// Per pass: (1) per-tile digit histogram, (2) one exclusive scan over the
// digit-major [256 x tiles] histogram, (3) stable scatter — inside a tile the
// rank of a key among equal digits is built round by round from warp
// match_any groups plus an ordered per-warp prefix, so the sort is stable
// (the reference's np.argsort(kind="stable") order, sampler.py:91).
#include "kg_common.cuh"

#include <stdarg.h>
#include <string.h>

namespace kg {

static thread_local char g_last_error[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

static thread_local char g_stale[256] = "";

void check_stale(const char* before) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    snprintf(g_stale, sizeof(g_stale), "stale %s cleared before %s", cudaGetErrorString(e), before);
}

kg_status from_cuda(cudaError_t e, const char* where) {
  set_error("CUDA error %s at %s%s%s", cudaGetErrorString(e), where, g_stale[0] ? " | " : "", g_stale);
  return KG_ERR_CUDA;
}

int num_sms() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

// ---------------------------------------------------------------------------
// Exclusive scan (uint32)
// ---------------------------------------------------------------------------
constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

// Block-wide exclusive scan of SCAN_TILE values held in smem `s` (in place);
// returns the tile total to every thread.
__device__ uint32_t block_scan_tile(uint32_t* s) {
  __shared__ uint32_t warp_tot[SCAN_THREADS / 32];
  const int t = threadIdx.x;
  uint32_t v[SCAN_ITEMS];
  uint32_t run = 0;
#pragma unroll
  for (int j = 0; j < SCAN_ITEMS; ++j) {
    v[j] = run;
    run += s[t * SCAN_ITEMS + j];
  }
  // warp inclusive scan of per-thread totals
  uint32_t inc = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if ((t & 31) >= o) inc += y;
  }
  if ((t & 31) == 31) warp_tot[t >> 5] = inc;
  __syncthreads();
  if (t < 32) {
    uint32_t w = (t < SCAN_THREADS / 32) ? warp_tot[t] : 0;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (t >= o) wi += y;
    }
    if (t < SCAN_THREADS / 32) warp_tot[t] = wi - w;   // exclusive warp offsets
    if (t == SCAN_THREADS / 32 - 1) warp_tot[SCAN_THREADS / 32 - 1 + 0] = wi - w;
    __syncwarp();
  }
  __syncthreads();
  uint32_t base = warp_tot[t >> 5] + (inc - run);
#pragma unroll
  for (int j = 0; j < SCAN_ITEMS; ++j) s[t * SCAN_ITEMS + j] = base + v[j];
  __syncthreads();
  // total = last element exclusive + its value is not kept; recompute from last thread
  __shared__ uint32_t total;
  if (t == SCAN_THREADS - 1) total = base + run;
  __syncthreads();
  return total;
}

__global__ void scan_tile_sums(const uint32_t* __restrict__ in, int64_t n, uint32_t* __restrict__ sums) {
  __shared__ uint32_t s[SCAN_TILE];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  for (int j = threadIdx.x; j < SCAN_TILE; j += SCAN_THREADS) {
    int64_t i = base + j;
    s[j] = i < n ? in[i] : 0u;
  }
  __syncthreads();
  uint32_t tot = block_scan_tile(s);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void scan_tiles_apply(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int64_t n,
                                 const uint32_t* __restrict__ tile_off, uint32_t* total) {
  __shared__ uint32_t s[SCAN_TILE];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  for (int j = threadIdx.x; j < SCAN_TILE; j += SCAN_THREADS) {
    int64_t i = base + j;
    s[j] = i < n ? in[i] : 0u;
  }
  __syncthreads();
  uint32_t tot = block_scan_tile(s);
  uint32_t off = tile_off ? tile_off[blockIdx.x] : 0u;
  for (int j = threadIdx.x; j < SCAN_TILE; j += SCAN_THREADS) {
    int64_t i = base + j;
    if (i < n) out[i] = s[j] + off;
  }
  if (total && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *total = off + tot;
}

// Small inputs: one 1024-thread CTA walks tiles of 8192 values with a running
// carry (1 launch instead of tile sums + recursive scan + apply). Values are
// staged through padded shared memory so each thread scans 8 consecutive
// values in registers. With `c.out` set it also performs the flag compaction
// c.out[off + rank(i)] = i (flags = in), optionally writing pos_out[i] =
// off + rank(i), the absolute count off + total, and clearing the flags.
struct CompactSpec {
  int32_t* out;              // compaction target (nullptr: plain scan)
  int32_t off_c;
  const int32_t* off_d;      // device offset added to off_c (optional)
  int32_t* count_out;        // total (or off + total when count_abs)
  int count_abs;
  int32_t* pos_out;          // inverse map (optional)
  int clear_flags;           // zero in[] after reading it
};

constexpr int SS_THREADS = 1024;
constexpr int SS_ITEMS = 8;
constexpr int SS_TILE = SS_THREADS * SS_ITEMS;
constexpr int64_t SCAN_SINGLE_MAX = 4 * SS_TILE;

__device__ __forceinline__ int ss_pad(int i) { return i + (i >> 5); }

__global__ void __launch_bounds__(SS_THREADS) scan_single(uint32_t* in, uint32_t* out, int64_t n, uint32_t* total,
                                                          CompactSpec c) {
  __shared__ uint32_t s[SS_TILE + SS_TILE / 32 + 1];
  __shared__ uint32_t wsum[SS_THREADS / 32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int32_t off = c.out ? c.off_c + (c.off_d ? *c.off_d : 0) : 0;
  uint32_t carry = 0;
  for (int64_t base = 0; base < n; base += SS_TILE) {
    uint32_t f[SS_ITEMS];
#pragma unroll
    for (int j = 0; j < SS_ITEMS; ++j) {
      const int64_t i = base + j * SS_THREADS + t;
      f[j] = i < n ? in[i] : 0u;
      if (c.clear_flags && i < n) in[i] = 0u;
      s[ss_pad(j * SS_THREADS + t)] = f[j];
    }
    __syncthreads();
    uint32_t x[SS_ITEMS], run = 0;
#pragma unroll
    for (int j = 0; j < SS_ITEMS; ++j) {
      x[j] = run;
      run += s[ss_pad(t * SS_ITEMS + j)];
    }
    uint32_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
      const uint32_t v = wsum[lane];
      uint32_t vi = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, vi, o);
        if (lane >= o) vi += y;
      }
      wsum[lane] = vi - v;   // exclusive warp offsets; vi of lane 31 = tile total
      if (lane == 31) s[ss_pad(SS_TILE - 1) + 1] = vi;   // spare slot past the padded tile
    }
    __syncthreads();
    const uint32_t tbase = carry + wsum[w] + inc - run;
    const uint32_t tile_total = s[ss_pad(SS_TILE - 1) + 1];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < SS_ITEMS; ++j) s[ss_pad(t * SS_ITEMS + j)] = tbase + x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < SS_ITEMS; ++j) {
      const int64_t i = base + j * SS_THREADS + t;
      if (i < n) {
        const uint32_t v = s[ss_pad(j * SS_THREADS + t)];
        if (out) out[i] = v;
        if (c.out && f[j]) {
          c.out[off + (int64_t)v] = (int32_t)i;
          if (c.pos_out) c.pos_out[i] = off + (int32_t)v;
        }
      }
    }
    carry += tile_total;
    __syncthreads();
  }
  if (t == 0) {
    if (total) *total = carry;
    if (c.count_out) *c.count_out = (c.count_abs ? off : 0) + (int32_t)carry;
  }
}

size_t scan_workspace(int64_t n) {
  size_t bytes = 0;
  int64_t m = n;
  while (m > SCAN_TILE) {
    int64_t tiles = ceil_div(m, SCAN_TILE);
    bytes += align_up(tiles * sizeof(uint32_t));
    m = tiles;
  }
  return bytes + 256;
}

kg_status exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* total, void* ws,
                             size_t ws_bytes, cudaStream_t st) {
  if (n <= 0) {
    if (total) KG_CUDA(cudaMemsetAsync(total, 0, sizeof(uint32_t), st));
    return KG_OK;
  }
  if (n <= SCAN_SINGLE_MAX) {
    KG_LAUNCH("scan_single", scan_single, 1, SS_THREADS, 0, st, const_cast<uint32_t*>(in), out, n, total,
              CompactSpec{});
    return KG_OK;
  }
  KG_REQUIRE(ws_bytes >= scan_workspace(n), KG_ERR_VALIDATION, "scan workspace too small");
  int64_t tiles = ceil_div(n, SCAN_TILE);
  uint32_t* sums = static_cast<uint32_t*>(ws);
  char* rest = static_cast<char*>(ws) + align_up(tiles * sizeof(uint32_t));
  KG_LAUNCH("scan_tile_sums", scan_tile_sums, (unsigned)tiles, SCAN_THREADS, 0, st, in, n, sums);
  KG_CHECK_LAUNCH("scan_tile_sums");
  kg_status s = exclusive_scan_u32(sums, sums, tiles, nullptr, rest,
                                   ws_bytes - align_up(tiles * sizeof(uint32_t)), st);
  if (s != KG_OK) return s;
  KG_LAUNCH("scan_tiles_apply", scan_tiles_apply, (unsigned)tiles, SCAN_THREADS, 0, st, in, out, n, sums, total);
  KG_CHECK_LAUNCH("scan_tiles_apply");
  return KG_OK;
}

// ---------------------------------------------------------------------------
// Stable LSD radix sort
// ---------------------------------------------------------------------------
constexpr int RS_THREADS = 256;
constexpr int RS_ROUNDS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ROUNDS;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int64_t RS_SELF_OFFSET_TILES = 64;   // up to 256 K keys: offsets computed in the scatter

// tile_major = 0: hist[d * tiles + tile] (scanned as one array);
// tile_major = 1: hist[tile * 256 + d] (read back by radix_scatter's own offsets)
template <typename K>
__global__ void __launch_bounds__(RS_THREADS) radix_hist(const K* __restrict__ keys, int64_t n, int shift,
                                                          uint32_t* __restrict__ hist, int64_t tiles, int tile_major) {
  __shared__ uint32_t cnt[256];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll 4
  for (int j = 0; j < RS_ROUNDS; ++j) {
    int64_t i = base + j * RS_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&cnt[(unsigned)(keys[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  if (tile_major) hist[(int64_t)blockIdx.x * 256 + threadIdx.x] = cnt[threadIdx.x];
  else hist[(int64_t)threadIdx.x * tiles + blockIdx.x] = cnt[threadIdx.x];
}

// Exclusive scan of one value per thread over a 256-thread block.
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t x, uint32_t* wsum /* smem [8] */) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  uint32_t before = 0;
#pragma unroll
  for (int q = 0; q < RS_WARPS; ++q)
    if (q < w) before += wsum[q];
  return before + inc - x;
}

// offs == nullptr: the digit offsets of this tile are derived here from the
// tile-major histogram (sum over all tiles per digit, exclusive scan over
// digits, plus the same digit's counts in earlier tiles) — no scan launches.
template <typename K>
__global__ void __launch_bounds__(RS_THREADS) radix_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                             K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                             int64_t n, int shift,
                                                             const uint32_t* __restrict__ offs, int64_t tiles,
                                                             const uint32_t* __restrict__ hist_tm) {
  __shared__ uint32_t base[256];
  __shared__ uint32_t wcnt[RS_WARPS][256];
  __shared__ uint32_t woff[RS_WARPS][256];
  const int t = threadIdx.x, w = t >> 5;
  if (offs) {
    base[t] = offs[(int64_t)t * tiles + blockIdx.x];
  } else {
    uint32_t tot = 0, pre = 0;
    for (int64_t q = 0; q < tiles; ++q) {
      const uint32_t h = __ldg(hist_tm + q * 256 + t);
      tot += h;
      if (q < (int64_t)blockIdx.x) pre += h;
    }
    base[t] = block_excl_scan256(tot, &woff[0][0]) + pre;
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < RS_WARPS; ++q) wcnt[q][t] = 0;
  __syncthreads();
  int64_t tile0 = (int64_t)blockIdx.x * RS_TILE;
  for (int j = 0; j < RS_ROUNDS; ++j) {
    int64_t i = tile0 + j * RS_THREADS + t;
    bool valid = i < n;
    K key = valid ? kin[i] : K(0);
    uint32_t val = valid ? vin[i] : 0u;
    unsigned d = valid ? ((unsigned)(key >> shift) & 255u) : 256u;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    unsigned rank = __popc(peers & lanemask_lt());
    bool leader = (__ffs(peers) - 1) == (int)lane_id();
    if (leader && valid) wcnt[w][d] = __popc(peers);
    __syncthreads();
    {
      uint32_t run = base[t];
#pragma unroll
      for (int q = 0; q < RS_WARPS; ++q) {
        uint32_t c = wcnt[q][t];
        woff[q][t] = run;
        run += c;
        wcnt[q][t] = 0;
      }
      base[t] = run;
    }
    __syncthreads();
    if (valid) {
      uint32_t dst = woff[w][d] + rank;
      kout[dst] = key;
      vout[dst] = val;
    }
  }
}

template <typename K>
static size_t sort_ws_bytes(int64_t n) {
  int64_t tiles = ceil_div(n > 0 ? n : 1, RS_TILE);
  int64_t hist = tiles * 256;
  return align_up(n * sizeof(K)) + align_up(n * sizeof(uint32_t)) + align_up(hist * sizeof(uint32_t)) +
         scan_workspace(hist) + 1024;
}

size_t sort_workspace(int64_t n) { return sort_ws_bytes<uint64_t>(n); }
size_t sort32_workspace(int64_t n) { return sort_ws_bytes<uint32_t>(n); }

template <typename K>
static kg_status sort_pairs(K* keys, uint32_t* vals, int64_t n, int key_bits, void* ws, size_t ws_bytes,
                            cudaStream_t st) {
  if (n <= 1 || key_bits <= 0) return KG_OK;
  KG_REQUIRE(ws_bytes >= sort_ws_bytes<K>(n), KG_ERR_VALIDATION, "sort workspace too small");
  KG_REQUIRE(n < (int64_t(1) << 32), KG_ERR_VALIDATION, "sort supports < 2^32 items");
  int64_t tiles = ceil_div(n, RS_TILE);
  int64_t hist_n = tiles * 256;
  Arena a(ws, ws_bytes);
  K* k2 = a.take<K>(n);
  uint32_t* v2 = a.take<uint32_t>(n);
  uint32_t* hist = a.take<uint32_t>(hist_n);
  char* scan_ws = a.take<char>(scan_workspace(hist_n));
  int passes = (key_bits + 7) / 8;
  K* ka = keys;
  uint32_t* va = vals;
  K* kb = k2;
  uint32_t* vb = v2;
  const bool self_offsets = tiles <= RS_SELF_OFFSET_TILES;
  for (int p = 0; p < passes; ++p) {
    int shift = 8 * p;
    KG_LAUNCH("radix_hist", (radix_hist<K>), (unsigned)tiles, RS_THREADS, 0, st, ka, n, shift, hist, tiles,
              self_offsets ? 1 : 0);
    if (self_offsets) {
      KG_LAUNCH("radix_scatter", (radix_scatter<K>), (unsigned)tiles, RS_THREADS, 0, st, ka, va, kb, vb, n, shift,
                (const uint32_t*)nullptr, tiles, (const uint32_t*)hist);
    } else {
      kg_status s = exclusive_scan_u32(hist, hist, hist_n, nullptr, scan_ws, scan_workspace(hist_n), st);
      if (s != KG_OK) return s;
      KG_LAUNCH("radix_scatter", (radix_scatter<K>), (unsigned)tiles, RS_THREADS, 0, st, ka, va, kb, vb, n, shift,
                (const uint32_t*)hist, tiles, (const uint32_t*)nullptr);
    }
    K* tk = ka; ka = kb; kb = tk;
    uint32_t* tv = va; va = vb; vb = tv;
  }
  if (ka != keys) {
    KG_CUDA(cudaMemcpyAsync(keys, ka, n * sizeof(K), cudaMemcpyDeviceToDevice, st));
    KG_CUDA(cudaMemcpyAsync(vals, va, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  }
  return KG_OK;
}

kg_status sort_pairs_u64(uint64_t* keys, uint32_t* vals, int64_t n, int key_bits, void* ws, size_t ws_bytes,
                         cudaStream_t st) {
  return sort_pairs<uint64_t>(keys, vals, n, key_bits, ws, ws_bytes, st);
}

kg_status sort_pairs_u32(uint32_t* keys, uint32_t* vals, int64_t n, int key_bits, void* ws, size_t ws_bytes,
                         cudaStream_t st) {
  return sort_pairs<uint32_t>(keys, vals, n, key_bits > 32 ? 32 : key_bits, ws, ws_bytes, st);
}

// ---------------------------------------------------------------------------
// Flag compaction: out[off + rank(i)] = i for flagged i, ascending.
// ---------------------------------------------------------------------------
__global__ void compact_scatter(uint32_t* flags, const uint32_t* __restrict__ pos, int64_t n,
                                const uint32_t* __restrict__ total, CompactSpec c) {
  const int32_t off = c.off_c + (c.off_d ? *c.off_d : 0);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (flags[i]) {
      c.out[off + pos[i]] = (int32_t)i;
      if (c.pos_out) c.pos_out[i] = off + (int32_t)pos[i];
      if (c.clear_flags) flags[i] = 0u;
    }
  }
  if (c.count_out && blockIdx.x == 0 && threadIdx.x == 0) *c.count_out = (c.count_abs ? off : 0) + (int32_t)*total;
}

size_t compact_workspace(int64_t n) { return align_up(n * sizeof(uint32_t)) + 256 + scan_workspace(n) + 256; }

static kg_status compact_run(uint32_t* flags, int64_t n, const CompactSpec& c, void* ws, size_t ws_bytes,
                             cudaStream_t st) {
  KG_REQUIRE(ws_bytes >= compact_workspace(n), KG_ERR_VALIDATION, "compact workspace too small");
  if (n > 0 && n <= SCAN_SINGLE_MAX) {
    KG_LAUNCH("scan_single", scan_single, 1, SS_THREADS, 0, st, flags, (uint32_t*)nullptr, n, (uint32_t*)nullptr, c);
    return KG_OK;
  }
  Arena a(ws, ws_bytes);
  uint32_t* pos = a.take<uint32_t>(n);
  uint32_t* total = a.take<uint32_t>(1);
  char* sws = a.take<char>(scan_workspace(n));
  kg_status s = exclusive_scan_u32(flags, pos, n, total, sws, scan_workspace(n), st);
  if (s != KG_OK) return s;
  int blocks = persistent_blocks(n, 256, 8);
  KG_LAUNCH("compact_scatter", compact_scatter, blocks, 256, 0, st, flags, pos, n, total, c);
  return KG_OK;
}

kg_status compact_flags(const uint32_t* flags, int64_t n, int32_t* out, int32_t* count_out, int32_t off_c,
                        const int32_t* off_d, void* ws, size_t ws_bytes, cudaStream_t st) {
  CompactSpec c{out, off_c, off_d, count_out, 0, nullptr, 0};
  return compact_run(const_cast<uint32_t*>(flags), n, c, ws, ws_bytes, st);
}

kg_status compact_flags_ex(uint32_t* flags, int64_t n, int32_t* out, const int32_t* off_d, int32_t* count_abs,
                           int32_t* pos_out, void* ws, size_t ws_bytes, cudaStream_t st) {
  CompactSpec c{out, 0, off_d, count_abs, 1, pos_out, 1};
  return compact_run(flags, n, c, ws, ws_bytes, st);
}

// Round-indexed segment copy: seg i copies bytes from src + r*src_stride to
// dst + r*dst_stride, r = *round_dev (device) or round_host. One launch moves
// a round's precomputed closure / grouping into the fixed working buffers.
constexpr int KG_MAX_SEGS = 24;
struct SegList {
  kg_copy_seg seg[KG_MAX_SEGS];
  int n;
};

// blockIdx.y = segment: the segments copy in parallel (a serial loop over
// segments would chain one memory latency per segment).
__global__ void __launch_bounds__(256) k_copy_segments(SegList L, const int64_t* __restrict__ round_dev,
                                                       int64_t round_host) {
  const int64_t r = round_dev ? *round_dev : round_host;
  const kg_copy_seg& g = L.seg[blockIdx.y];
  const char* src = static_cast<const char*>(g.src) + r * g.src_round_stride;
  char* dst = static_cast<char*>(g.dst) + r * g.dst_round_stride;
  const bool v16 = (((uintptr_t)src | (uintptr_t)dst | (uintptr_t)g.bytes) & 15) == 0;
  if (v16) {
    const int64_t n = g.bytes / 16;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
      reinterpret_cast<int4*>(dst)[x] = __ldg(reinterpret_cast<const int4*>(src) + x);
  } else {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < g.bytes;
         x += (int64_t)gridDim.x * blockDim.x)
      dst[x] = src[x];
  }
}

}  // namespace kg

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

int kg_abi_version(void) { return KG_ABI_VERSION; }

kg_status kg_graph_upload(void* graph_exec, void* stream) {
  KG_CUDA(cudaGraphUpload(reinterpret_cast<cudaGraphExec_t>(graph_exec), kg::as_stream(stream)));
  return KG_OK;
}

kg_status kg_copy_segments(const kg_copy_seg* segs, int32_t n, const int64_t* round_dev, int64_t round_host,
                           void* stream) {
  KG_REQUIRE(n >= 0 && n <= kg::KG_MAX_SEGS, KG_ERR_VALIDATION, "at most %d segments", kg::KG_MAX_SEGS);
  if (n == 0) return KG_OK;
  kg::SegList L{};
  int64_t most = 0;
  for (int i = 0; i < n; ++i) {
    L.seg[i] = segs[i];
    most = segs[i].bytes > most ? segs[i].bytes : most;
  }
  L.n = n;
  // enough blocks per segment for the largest; the grid totals ~2 waves
  const int64_t per = kg::ceil_div(most / 16 + 1, 256);
  const int64_t cap = kg::ceil_div((int64_t)kg::num_sms() * 16, n);
  const dim3 grid((unsigned)(per < cap ? per : cap), (unsigned)n, 1);
  KG_LAUNCH("k_copy_segments", kg::k_copy_segments, grid, 256, 0, kg::as_stream(stream), L, round_dev, round_host);
  return KG_OK;
}

int kg_last_error(char* buf, int64_t n) {
  if (buf && n > 0) {
    strncpy(buf, kg::g_last_error, (size_t)n - 1);
    buf[n - 1] = 0;
  }
  return (int)strlen(kg::g_last_error);
}

int64_t kg_sort_workspace_bytes(int64_t n) { return (int64_t)kg::sort_workspace(n); }

kg_status kg_sort_pairs_u64(uint64_t* keys, uint32_t* vals, int64_t n, int key_bits, void* ws, int64_t ws_bytes,
                            void* stream) {
  return kg::sort_pairs_u64(keys, vals, n, key_bits, ws, (size_t)ws_bytes, kg::as_stream(stream));
}

int64_t kg_scan_workspace_bytes(int64_t n) { return (int64_t)kg::scan_workspace(n); }

kg_status kg_exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* total, void* ws,
                                int64_t ws_bytes, void* stream) {
  return kg::exclusive_scan_u32(in, out, n, total, ws, (size_t)ws_bytes, kg::as_stream(stream));
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Launch accounting and the live per-kernel event timer (bench.py roofline)
// ---------------------------------------------------------------------------
#include <vector>

namespace kg {

static int64_t g_launches = 0;
static bool g_timer_on = false;
static char g_timer_prefix[512] = "";
static std::vector<cudaEvent_t> g_ev_start, g_ev_end;
static std::vector<const char*> g_ev_name;
static size_t g_ev_used = 0;

// inside stream capture the records must become external event nodes of the graph
static unsigned record_flags(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
}

// `name` is one of the comma-separated exact names in `list`
static bool in_list(const char* list, const char* name) {
  const size_t n = strlen(name);
  for (const char* p = list; (p = strstr(p, name)) != nullptr; p += n) {
    const bool start = p == list || p[-1] == ',';
    const bool end = p[n] == 0 || p[n] == ',';
    if (start && end) return true;
  }
  return false;
}

bool knocked_out(const char* name) {
  static const char* list = getenv("KG_KNOCKOUT");
  if (list == nullptr || !*list) return false;
  return in_list(list, name);
}

LaunchScope::LaunchScope(const char* name, cudaStream_t s) : st(s), slot(-1) {
  ++g_launches;
  // timed kernels: a comma-separated list of exact names, "" = all
  if (!g_timer_on || (g_timer_prefix[0] && !in_list(g_timer_prefix, name))) return;
  if (g_ev_used == g_ev_start.size()) {
    cudaEvent_t a, b;
    if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return;
    g_ev_start.push_back(a);
    g_ev_end.push_back(b);
    g_ev_name.push_back(name);
  }
  slot = (int)g_ev_used++;
  g_ev_name[slot] = name;
  cudaEventRecordWithFlags(g_ev_start[slot], st, record_flags(st));
}

void LaunchScope::done() {
  if (slot >= 0) cudaEventRecordWithFlags(g_ev_end[slot], st, record_flags(st));
}

}  // namespace kg

extern "C" {

int64_t kg_launch_count(void) { return kg::g_launches; }

kg_status kg_kernel_timer_begin(const char* prefix) {
  strncpy(kg::g_timer_prefix, prefix ? prefix : "", sizeof(kg::g_timer_prefix) - 1);
  kg::g_ev_used = 0;
  kg::g_timer_on = true;
  return KG_OK;
}

// Per-kernel breakdown of the launches recorded since kg_kernel_timer_begin:
// writes "name,count,total_ms" lines into buf (host) and ends the timer.
kg_status kg_kernel_timer_dump(char* buf, int64_t n) {
  kg::g_timer_on = false;
  std::vector<std::pair<const char*, std::pair<int64_t, double>>> agg;
  for (size_t i = 0; i < kg::g_ev_used; ++i) {
    float ms = 0.f;
    KG_CUDA(cudaEventSynchronize(kg::g_ev_end[i]));
    KG_CUDA(cudaEventElapsedTime(&ms, kg::g_ev_start[i], kg::g_ev_end[i]));
    size_t j = 0;
    for (; j < agg.size(); ++j)
      if (strcmp(agg[j].first, kg::g_ev_name[i]) == 0) break;
    if (j == agg.size()) agg.push_back({kg::g_ev_name[i], {0, 0.0}});
    agg[j].second.first += 1;
    agg[j].second.second += ms;
  }
  int64_t off = 0;
  if (buf && n > 0) buf[0] = 0;
  for (auto& a : agg) {
    if (!buf || off >= n - 1) break;
    off += snprintf(buf + off, (size_t)(n - off), "%s,%lld,%.6f\n", a.first, (long long)a.second.first,
                    a.second.second);
  }
  kg::g_ev_used = 0;
  return KG_OK;
}

// Graph capture support: the event pairs recorded while a stream was being
// captured became event-record nodes of that graph; detaching keeps them out
// of the reuse pool so every replay re-records them.
struct TimedLaunch {
  cudaEvent_t start, end;
  const char* name;
};
static std::vector<std::vector<TimedLaunch>> g_detached;

kg_status kg_kernel_timer_detach(int64_t* handle) {
  kg::g_timer_on = false;
  std::vector<TimedLaunch> grp;
  for (size_t i = 0; i < kg::g_ev_used; ++i) grp.push_back({kg::g_ev_start[i], kg::g_ev_end[i], kg::g_ev_name[i]});
  // hand the events over: the pool forgets them
  kg::g_ev_start.erase(kg::g_ev_start.begin(), kg::g_ev_start.begin() + kg::g_ev_used);
  kg::g_ev_end.erase(kg::g_ev_end.begin(), kg::g_ev_end.begin() + kg::g_ev_used);
  kg::g_ev_name.erase(kg::g_ev_name.begin(), kg::g_ev_name.begin() + kg::g_ev_used);
  kg::g_ev_used = 0;
  g_detached.push_back(grp);
  *handle = (int64_t)g_detached.size() - 1;
  return KG_OK;
}

kg_status kg_kernel_timer_read_named(int64_t handle, const char* name, double* total_ms, int64_t* launches) {
  KG_REQUIRE(handle >= 0 && handle < (int64_t)g_detached.size(), KG_ERR_VALIDATION, "bad timer handle");
  double tot = 0.0;
  int64_t cnt = 0;
  for (auto& tl : g_detached[handle]) {
    if (name && *name && strcmp(name, tl.name) != 0) continue;
    float ms = 0.f;
    KG_CUDA(cudaEventSynchronize(tl.end));
    KG_CUDA(cudaEventElapsedTime(&ms, tl.start, tl.end));
    tot += ms;
    ++cnt;
  }
  *total_ms = tot;
  *launches = cnt;
  return KG_OK;
}

kg_status kg_kernel_timer_read(int64_t handle, double* total_ms, int64_t* launches) {
  return kg_kernel_timer_read_named(handle, nullptr, total_ms, launches);
}

// Makespan of concurrent launch pairs: the i-th launch of `a` and the i-th of
// `b` (e.g. the two CSC passes of one layer on two streams) cover
// [min start, max end]; returns the summed spans and the pair count.
kg_status kg_kernel_timer_span(int64_t handle, const char* a, const char* b, double* total_ms, int64_t* pairs) {
  KG_REQUIRE(handle >= 0 && handle < (int64_t)g_detached.size(), KG_ERR_VALIDATION, "bad timer handle");
  std::vector<const TimedLaunch*> la, lb;
  for (auto& tl : g_detached[handle]) {
    if (strcmp(tl.name, a) == 0) la.push_back(&tl);
    else if (strcmp(tl.name, b) == 0) lb.push_back(&tl);
  }
  const size_t n = la.size() < lb.size() ? la.size() : lb.size();
  double tot = 0.0;
  for (size_t i = 0; i < n; ++i) {
    KG_CUDA(cudaEventSynchronize(la[i]->end));
    KG_CUDA(cudaEventSynchronize(lb[i]->end));
    float ea = 0.f, sb = 0.f, eb = 0.f;   // relative to a's start
    KG_CUDA(cudaEventElapsedTime(&ea, la[i]->start, la[i]->end));
    KG_CUDA(cudaEventElapsedTime(&sb, la[i]->start, lb[i]->start));
    KG_CUDA(cudaEventElapsedTime(&eb, la[i]->start, lb[i]->end));
    const float lo = sb < 0.f ? sb : 0.f, hi = eb > ea ? eb : ea;
    tot += hi - lo;
  }
  *total_ms = tot;
  *pairs = (int64_t)n;
  return KG_OK;
}

kg_status kg_kernel_timer_end(double* total_ms, int64_t* launches) {
  kg::g_timer_on = false;
  double tot = 0.0;
  for (size_t i = 0; i < kg::g_ev_used; ++i) {
    float ms = 0.f;
    KG_CUDA(cudaEventSynchronize(kg::g_ev_end[i]));
    KG_CUDA(cudaEventElapsedTime(&ms, kg::g_ev_start[i], kg::g_ev_end[i]));
    tot += ms;
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = (int64_t)kg::g_ev_used;
  kg::g_ev_used = 0;
  return KG_OK;
}

}  // extern "C"

// this module's anchor for kg_preload_kernels (kg_primitives.cu)
extern "C" const void* kg_anchor_primitives() { return reinterpret_cast<const void*>(&kg::scan_tile_sums); }

// ---------------------------------------------------------------------------
// Eager loading of the library's kernels. Under CUDA's lazy module loading
// every kernel is loaded at its first launch; in a fresh process that put
// ~80 ms of loading into the first training epoch (measured: first-epoch
// 99 ms lazy vs 17 ms with CUDA_MODULE_LOADING=EAGER). The host side calls
// this once per process (_lib.require_cuda): every function of every module
// of this library is loaded up front (cuModuleEnumerateFunctions + cuFuncLoad,
// through the driver entry points; one anchor kernel per translation unit
// names its module). Process-wide eager loading would also load all of
// PyTorch's kernels.
#include <cuda.h>
extern "C" {
const void* kg_anchor_chunks();
const void* kg_anchor_compat();
const void* kg_anchor_eval();
const void* kg_anchor_eval64();
const void* kg_anchor_gemm();
const void* kg_anchor_loss();
const void* kg_anchor_model64();
const void* kg_anchor_optim();
const void* kg_anchor_partition();
const void* kg_anchor_peer();
const void* kg_anchor_primitives();
const void* kg_anchor_rgcn();
const void* kg_anchor_sampler();
const void* kg_anchor_umma();
const void* kg_anchor_view();

kg_status kg_preload_kernels(int32_t* loaded) {
  typedef CUresult (*PFuncGetModule)(CUmodule*, CUfunction);
  typedef CUresult (*PModuleGetFunctionCount)(unsigned int*, CUmodule);
  typedef CUresult (*PModuleEnumerateFunctions)(CUfunction*, unsigned int, CUmodule);
  typedef CUresult (*PFuncLoad)(CUfunction);
  void *p1 = nullptr, *p2 = nullptr, *p3 = nullptr, *p4 = nullptr;
  cudaDriverEntryPointQueryResult q;
  KG_CUDA(cudaGetDriverEntryPoint("cuFuncGetModule", &p1, cudaEnableDefault, &q));
  KG_CUDA(cudaGetDriverEntryPoint("cuModuleGetFunctionCount", &p2, cudaEnableDefault, &q));
  KG_CUDA(cudaGetDriverEntryPoint("cuModuleEnumerateFunctions", &p3, cudaEnableDefault, &q));
  KG_CUDA(cudaGetDriverEntryPoint("cuFuncLoad", &p4, cudaEnableDefault, &q));
  if (loaded) *loaded = 0;
  if (!p1 || !p2 || !p3 || !p4) return KG_OK;   // older driver: stay lazy
  const void* (*anchors[])() = {kg_anchor_chunks, kg_anchor_compat, kg_anchor_eval, kg_anchor_eval64, kg_anchor_gemm, kg_anchor_loss, kg_anchor_model64, kg_anchor_optim, kg_anchor_partition, kg_anchor_peer, kg_anchor_primitives, kg_anchor_rgcn, kg_anchor_sampler, kg_anchor_umma, kg_anchor_view};
  int32_t n_loaded = 0;
  for (auto a : anchors) {
    cudaFunction_t f;
    KG_CUDA(cudaGetFuncBySymbol(&f, a()));
    CUmodule mod;
    if (((PFuncGetModule)p1)(&mod, (CUfunction)f) != CUDA_SUCCESS) continue;
    unsigned int count = 0;
    if (((PModuleGetFunctionCount)p2)(&count, mod) != CUDA_SUCCESS || count == 0) continue;
    std::vector<CUfunction> fs(count);
    if (((PModuleEnumerateFunctions)p3)(fs.data(), count, mod) != CUDA_SUCCESS) continue;
    for (CUfunction fn : fs)
      if (((PFuncLoad)p4)(fn) == CUDA_SUCCESS) ++n_loaded;
  }
  if (loaded) *loaded = n_loaded;
  return KG_OK;
}
}  // extern "C"
