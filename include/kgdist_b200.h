/*
 * kgdist_b200 — C ABI of the B200-native (sm_100a) training hot path of the
 * partitioned RGCN + DistMult KG-embedding scheme (arXiv 2201.02791,
 * reference package `kgdist`).
 *
 * The reference has no FFI: its boundary is the Python API re-exported by
 * kgdist/__init__.py:8-41. Each entry point below replaces the numpy body of
 * one reference function (cited as ref:<file>:<line>, ref = pkg/src/kgdist);
 * the package `paper_2201_02791_b200` keeps the reference's Python names and
 * calls these through ctypes.
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless noted; the caller owns every
 *    buffer (PyTorch tensors on the Python side). Scratch space comes from a
 *    caller workspace sized by the matching *_workspace_bytes() call.
 *  - `stream` is a cudaStream_t passed as void*. Every call is asynchronous
 *    on that stream; device-side failures (non-finite values, exhausted
 *    resampling) are written to a device status word the caller checks at
 *    its sync points.
 *  - Ids are int32 local vertex ids, relation ids int32, values fp32.
 *  - Return value kg_status maps 1:1 onto the reference's KGError classes
 *    (ref:errors.py:8-49); kg_last_error() returns the message.
 */
#ifndef KGDIST_B200_H
#define KGDIST_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KG_ABI_VERSION 1

typedef enum kg_status {
  KG_OK = 0,
  KG_ERR_VALIDATION = 1, /* ValidationError   */
  KG_ERR_SHAPE = 2,      /* ShapeError        */
  KG_ERR_INTEGRITY = 3,  /* IntegrityError    */
  KG_ERR_SAMPLING = 4,   /* SamplingError     */
  KG_ERR_NUMERIC = 5,    /* NumericError      */
  KG_ERR_PROTOCOL = 6,   /* ProtocolError     */
  KG_ERR_CUDA = 7        /* CUDA runtime failure (no reference analogue) */
} kg_status;

/* Device status-word bits (written by kernels, read by the host at syncs). */
#define KG_FLAG_NONFINITE_SCORE 1u
#define KG_FLAG_NONFINITE_LOSS 2u
#define KG_FLAG_NONFINITE_PARAM 4u
#define KG_FLAG_BAD_VERTEX 8u
#define KG_FLAG_PEER_TIMEOUT 16u  /* kg_peer_gather: a peer payload did not arrive within 5 s */

/* numpy PCG64 BitGenerator state (Generator.bit_generator.state). */
typedef struct kg_pcg64 {
  uint64_t state_hi, state_lo;
  uint64_t inc_hi, inc_lo;
  uint32_t has_uint32;
  uint32_t uinteger;
} kg_pcg64;

/* Partition message graph resident in HBM (built by kg_view_build).
 * Row v of the destination CSR lists messages entering v sorted by
 * (relation, original order); the source CSR (CSC) lists messages leaving v
 * sorted by (relation, original order). Self-loops are implicit (group 2R). */
typedef struct kg_graph_csr {
  int32_t n;          /* local vertices                                   */
  int32_t R;          /* relations before inverse doubling                */
  int64_t e;          /* message edges = 2 * edges                        */
  int32_t* indptr;    /* [n+1]                                            */
  int32_t* src;       /* [e]                                              */
  int32_t* rel;       /* [e]                                              */
  float* norm;        /* [e]   1 / c_{dst,rel}                            */
  int32_t* c_indptr;  /* [n+1]                                            */
  int32_t* c_dst;     /* [e]                                              */
  int32_t* c_rel;     /* [e]                                              */
  float* c_norm;      /* [e]                                              */
  int32_t* rel_perm;  /* [e]   CSC positions grouped by relation          */
  int32_t* rel_ptr;   /* [2R+1] group starts into rel_perm (+ end)        */
  /* Static work chunks (<= `chunk` messages each) so hub rows are spread
   * over many warps. For the CSR (ck_*) and the CSC (cc_*):
   * ptr[n+1] chunk range of row v; row[] owning row of each chunk; slot[]
   * partial-sum slot of a chunk whose row has > 1 chunk (-1 otherwise);
   * split[] rows with > 1 chunk; counts[4] = {chunks, split chunks, split
   * rows, -} (device). Capacities: chunks <= n + e/chunk + 1, split chunks
   * <= 2e/chunk + 1, split rows <= e/chunk + 1. */
  int32_t chunk;
  int32_t* ck_ptr;
  int32_t* ck_row;
  int32_t* ck_slot;
  int32_t* ck_split;
  int32_t* ck_counts;
  int32_t* cc_ptr;
  int32_t* cc_row;
  int32_t* cc_slot;
  int32_t* cc_split;
  int32_t* cc_counts;
  /* Per-chunk descriptors (4 x int32 per chunk, same capacity as ck_row /
   * cc_row): {row, first message, message count | 1<<16 if the row has a
   * single chunk | 1<<17 if it is the row's first chunk, partial slot}, so a
   * gather warp resolves its chunk with one 16-byte load. */
  int32_t* ck_desc;
  int32_t* cc_desc;
} kg_graph_csr;

/* One RGCN layer's parameters (ref:model.py:64-79). */
typedef struct kg_layer_params {
  int32_t d_in, d_out, B, G; /* G = 2R + 1 relation groups                 */
  const float* bases;        /* (B, d_in, d_out)                           */
  const float* coeffs;       /* (G, B)                                     */
  /* Optional: the bases as tensor-core operand records written by
   * kg_rgcn_pack_weights from the CURRENT bases (repack after every update);
   * NULL = forward/backward pack them on the fly. */
  const float* packed;
} kg_layer_params;

/* ---------------------------------------------------------------------- */
/* Library                                                                 */
/* ---------------------------------------------------------------------- */
int kg_abi_version(void);
/* cudaGraphUpload of an instantiated graph (e.g. torch CUDAGraph
 * .raw_cuda_graph_exec()), so its first replay does not pay the upload. */
kg_status kg_graph_upload(void* graph_exec, void* stream);
int kg_last_error(char* buf, int64_t n); /* host buffer */
/* Number of kernels this library has launched in the process. */
int64_t kg_launch_count(void);
/* Bracket every launch of the kernels named in `prefix` (comma-separated
 * exact kernel names, "" = all kernels; host string) with CUDA events on the
 * launching stream; _end synchronises and returns the summed device time and
 * the launch count. */
kg_status kg_kernel_timer_begin(const char* prefix);
kg_status kg_kernel_timer_end(double* total_ms, int64_t* launches);
/* Ends the timer and writes "name,launches,total_ms" lines (host buffer). */
kg_status kg_kernel_timer_dump(char* buf, int64_t n);
/* While a stream is being captured into a CUDA graph the timer's event
 * records become graph nodes: _detach ends the timer and keeps those events
 * as a group (handle) that every replay re-records; _read sums the group's
 * elapsed time after a replay (synchronises on its events). */
kg_status kg_kernel_timer_detach(int64_t* handle);
kg_status kg_kernel_timer_read(int64_t handle, double* total_ms, int64_t* launches);
/* As _read, restricted to the launches of kernel `name` (host string). */
kg_status kg_kernel_timer_read_named(int64_t handle, const char* name, double* total_ms, int64_t* launches);
/* Makespan of concurrent launch pairs (i-th launch of kernel a with the i-th
 * of kernel b): summed [min start, max end] spans and the pair count. */
kg_status kg_kernel_timer_span(int64_t handle, const char* a, const char* b, double* total_ms, int64_t* pairs);
/* Load every kernel of the library now instead of at its first launch (CUDA
 * lazy module loading); *loaded = functions loaded (0 on drivers without the
 * enumeration entry points). Called once per process by the host package. */
kg_status kg_preload_kernels(int32_t* loaded);
/* Epoch-end bookkeeping (ref:trainer.py:446-462, the epoch loss and the
 * non-finite checks): out[w] = mean of losses[w*ld + r] over r < rounds
 * (float64), out[nloc + j] = *flag_ptrs[j] (status words, then cleared). */
kg_status kg_epoch_end(const float* losses, int64_t ld, int32_t nloc, int32_t rounds, const uint64_t* flag_ptrs,
                       int32_t nflags, double* out, void* stream);

/* ---------------------------------------------------------------------- */
/* Primitives (stable radix sort / scan) used by every stage below          */
/* ---------------------------------------------------------------------- */
int64_t kg_sort_workspace_bytes(int64_t n);
kg_status kg_sort_pairs_u64(uint64_t* keys, uint32_t* vals, int64_t n, int key_bits, void* ws,
                            int64_t ws_bytes, void* stream);
/* Round-indexed copies (<= 16 segments, one launch): segment i copies
 * `bytes` from src + r*src_round_stride to dst + r*dst_round_stride with
 * r = *round_dev (device int64, e.g. inside a CUDA graph) or round_host. */
typedef struct kg_copy_seg {
  void* dst;
  const void* src;
  int64_t bytes;
  int64_t dst_round_stride;
  int64_t src_round_stride;
} kg_copy_seg;
kg_status kg_copy_segments(const kg_copy_seg* segs, int32_t n, const int64_t* round_dev, int64_t round_host,
                           void* stream);
int64_t kg_scan_workspace_bytes(int64_t n);
kg_status kg_exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* total, void* ws,
                                int64_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------- */
/* PCG64 host bookkeeping (host pointers)                                  */
/* ---------------------------------------------------------------------- */
/* Jump ahead `delta` next64 draws (numpy bit_generator.advance). */
void kg_pcg64_advance(kg_pcg64* g, uint64_t delta);
/* Account for `count` next_uint32 draws (buffered half-words included). */
void kg_pcg64_consume32(kg_pcg64* g, uint64_t count);
/* First `count` next64 outputs (host buffer), for self-checks. */
void kg_pcg64_peek64(const kg_pcg64* g, uint64_t* out, int64_t count);

/* ---------------------------------------------------------------------- */
/* R1/R2  Partition view (replaces ref:partition.py:61-74 local ids and    */
/*        ref:sampler.py:73-118 build_view)                                */
/* ---------------------------------------------------------------------- */
int64_t kg_view_workspace_bytes(int64_t m, int64_t num_entities);
/* Local ids: core endpoints in first-appearance order over (h0,t0,h1,..),
 * then support-only endpoints likewise. Inputs are global (m,3) triples.
 * Writes local_ids[0..n_local), g2l[num_entities] (-1 if absent) and the
 * count *n_local (device int32). */
kg_status kg_view_local_ids(const int32_t* core, int64_t m_core, const int32_t* support, int64_t m_sup,
                            int64_t num_entities, int32_t* local_ids, int32_t* g2l, int32_t* n_local,
                            void* ws, int64_t ws_bytes, void* stream);
/* Message graph: edges_global (m,3) core-then-support global triples.
 * Outputs: edges_local (m,3); reference-order message arrays ref_src,
 * ref_rel, msg_cnt [2m] (stable-by-destination, ref:sampler.py:91; norm =
 * 1/msg_cnt); the working CSR/CSC in *g (arrays preallocated by caller,
 * g->n and g->R set); sorted unique positive keys pos_keys[*n_keys]. */
kg_status kg_view_build(const int32_t* edges_global, int64_t m, const int32_t* g2l, int32_t* edges_local,
                        int32_t* ref_src, int32_t* ref_rel, int32_t* msg_cnt, const kg_graph_csr* g,
                        int64_t* pos_keys, int32_t* n_keys, void* ws, int64_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------- */
/* R3/R4  Constraint-based negatives (ref:sampler.py:60-70, 144-182)        */
/* ---------------------------------------------------------------------- */
/* The sampler's PCG64 state lives in device memory (`g`, a kg_pcg64 in
 * HBM): every entry below reads it and advances it on the device, so an
 * epoch of sampling is one asynchronous kernel chain (no host syncs).
 *
 * neg = repeat(core, s); col[i] = 0 (head) if random() < 0.5 else 2;
 * pending = 0..s*m-1; advances g by s*m next64 draws. */
kg_status kg_neg_init(const int32_t* core, int64_t m, int32_t s, kg_pcg64* g, int32_t* neg, int8_t* col,
                      int32_t* pending, void* stream);
int64_t kg_neg_round_workspace_bytes(int64_t window);
/* One resampling round over the *k_dev pending rows (ascending, <= k_max):
 * draws integers(pool_size, size=k) from `window` uint32 stream positions,
 * writes the corrupted entity, rejects originals and local positives,
 * advances g. Outputs next_pending[*next_count] and *consumed32 (uint32
 * draws used; -1 => window too small, g untouched: retry larger). */
kg_status kg_neg_round(int32_t* neg, const int8_t* col, const int32_t* core, int32_t s,
                       const int32_t* pending, const int32_t* k_dev, int64_t k_max, int64_t pool_size,
                       int32_t n_local, int32_t R, const int64_t* pos_keys, const int32_t* n_keys, kg_pcg64* g,
                       int64_t window, int32_t* next_pending, int32_t* next_count, int64_t* consumed32, void* ws,
                       int64_t ws_bytes, void* stream);
/* is_positive over (k,3) local triples -> out[k] (0/1). */
kg_status kg_is_positive(const int32_t* triples, int64_t k, int32_t n_local, int32_t R, const int64_t* pos_keys,
                         const int32_t* n_keys, uint8_t* out, void* stream);

/* ---------------------------------------------------------------------- */
/* R5  Edge mini-batch stream (ref:sampler.py:202-232)                      */
/* ---------------------------------------------------------------------- */
/* Fisher-Yates swap targets js[i] for i = n-1..1 of rng.permutation(n)
 * (bit-exact, masked rejection). U is a device buffer of W uint32 stream
 * positions (W = kg_perm_draws_buffer_len(n)); *consumed32 = uint32 draws
 * used, or -1 if W was too small (retry with a larger buffer). */
int64_t kg_perm_draws_buffer_len(int64_t n);
kg_status kg_perm_draws_buffered(int64_t n, kg_pcg64* g, uint32_t* U, int64_t W, int32_t* js, int64_t* consumed32,
                                 void* stream);
int64_t kg_perm_resolve_workspace_bytes(int64_t n);
/* Final permutation from the swap targets without replaying the swaps. */
kg_status kg_perm_resolve(const int32_t* js, int64_t n, int32_t* perm, void* ws, int64_t ws_bytes,
                          void* stream);
/* stream[k] = concat(pos, neg)[perm[k]], labels 1/0. */
kg_status kg_stream_gather(const int32_t* pos, int64_t npos, const int32_t* neg, int64_t nneg,
                           const int32_t* perm, int32_t* stream_triples, float* labels, void* stream);

/* ---------------------------------------------------------------------- */
/* R7/R8  Layered closure (ref:sampler.py:310-376)                          */
/* ---------------------------------------------------------------------- */
int64_t kg_closure_workspace_bytes(int32_t n);
/* start_dev (optional, device int64) overrides `start` so a captured CUDA
 * graph can be replayed for every round. Seeds = endpoints of batch rows
 * (start+q) mod total, q < b, of the
 * (total,3) stream; or, when stream_triples == NULL, the ids seed_ids[b].
 * Writes vertex_order (seeds ascending, then each hop's new sources
 * ascending), pos[n] (-1 if absent) and counts[hops+1] (device). */
kg_status kg_closure(const int32_t* stream_triples, int64_t total, int64_t start, const int64_t* start_dev,
                     int64_t b, const int32_t* seed_ids, const kg_graph_csr* g, int32_t hops,
                     int32_t* vertex_order, int32_t* pos, int32_t* counts, void* ws, int64_t ws_bytes,
                     void* stream);

/* ---------------------------------------------------------------------- */
/* R13-R17  RGCN layer forward / backward, DistMult + BCE                  */
/* ---------------------------------------------------------------------- */
int64_t kg_layer_workspace_bytes(const kg_graph_csr* g, int32_t d_in, int32_t d_out, int32_t B);
/* ref:model.py:151-164, 216-220: Z[v] = sum_b (sum_{e->v} norm a[r,b] H[src]
 * + a[2R,b] H[v]) V_b for v in A_t = vertex_order[0:counts[t]];
 * H_out[v] = relu(Z) (relu != 0) or Z. H_in/H_out rows indexed by local id. */
kg_status kg_rgcn_forward(const kg_graph_csr* g, const kg_layer_params* lp, const float* H_in, float* H_out,
                          const int32_t* vertex_order, const int32_t* pos, const int32_t* counts, int32_t t,
                          int32_t relu, const float* dropout_mask, float* H_out_packed, void* ws,
                          int64_t ws_bytes, void* stream);
/* dropout_mask (optional, kg_dropout_mask, (counts[t], d_out) by position):
 * H_out = relu(Z) * mask. H_out_packed (optional, kg_pack_rows_bytes(n,
 * d_out)): the output rows by position p < counts[t] also as tensor-core
 * operand records — exactly what the next layer's kg_rgcn_backward takes as
 * H_in_packed. */
/* ref:model.py:167-185, 286-296: gradients of one layer. dH_out holds
 * dL/dA of the layer output for v in A_t (by local id); H_out (NULL for the
 * last layer) supplies the ReLU mask. Writes d_bases (B,d_in,d_out),
 * d_coeffs (G,B) and, if dH_in != NULL, dL/dH_in for v in A_{t+1}.
 * side_stream (optional): d_bases / d_coeffs are then produced on it, off the
 * dH_in critical path; the caller must order side_stream before reading them
 * and before reusing ws (one ws per layer). */
kg_status kg_rgcn_backward(const kg_graph_csr* g, const kg_layer_params* lp, const float* H_in,
                           const float* H_out, const float* dH_out, float* dH_in, const int32_t* vertex_order,
                           const int32_t* pos, const int32_t* c_pos, const int32_t* counts, int32_t t,
                           float* d_bases, float* d_coeffs, const float* H_in_packed, const float* dropout_mask,
                           int32_t y_ready, void* ws, int64_t ws_bytes, void* stream, void* side_stream);
/* c_pos (optional, g->e int32) = pos[c_dst[e]] for the round's closure,
 * written by kg_csc_positions; the CSC passes then skip one dependent load
 * per message. NULL: looked up per message. */
kg_status kg_csc_positions(const kg_graph_csr* g, const int32_t* pos, int32_t* c_pos, void* stream);
/* The backward's first GEMM, Y = H_in[vertex_order[p]] . [V_0 | .. | V_{B-1}]
 * for p < counts[t+1], ahead of time (it needs only forward outputs): call it
 * on any stream ordered before kg_rgcn_backward(..., y_ready = 1, ...) with
 * the same ws. Needs lp->packed. */
kg_status kg_rgcn_backward_y(const kg_graph_csr* g, const kg_layer_params* lp, const float* H_in,
                             const float* H_in_packed, const int32_t* vertex_order, const int32_t* counts, int32_t t,
                             void* ws, int64_t ws_bytes, void* stream);
/* H_in_packed (optional): H_in[vertex_order[p]], p < counts[t+1], as operand
 * records (the previous layer's H_out_packed, or kg_pack_rows).
 * dropout_mask (optional): the mask this layer's forward applied to H_out. */
int64_t kg_pack_rows_bytes(int64_t rows, int64_t cols);
kg_status kg_pack_rows(const float* src, int64_t ld, const int32_t* rowid, const int32_t* counts,
                       int32_t count_index, int64_t n_max, int64_t cols, float* out, void* stream);
/* Pre-pack the three tensor-core weight operands of one layer (forward
 * Z = acc.V, backward Y = X.[V_b] and dX = dS.[V_b]^T) into `out`
 * (kg_rgcn_weights_bytes); set lp->packed = out for the calls that follow. */
int64_t kg_rgcn_weights_bytes(int32_t d_in, int32_t d_out, int32_t B);
kg_status kg_rgcn_pack_weights(const kg_layer_params* lp, float* out, void* stream);
/* Dense GEMM of the factored layer (standalone entry for checks):
 * trans 0: C[c_rows(p)] = A[a_rows(p), :K] . B[K, N] (+relu), p < M;
 * trans 1: C[K, N] = sum_{p<M} A[a_rows(p), :K]^T . B[p, :N].
 * impl 0: tcgen05 3xTF32 tensor cores (product path); 1: CUDA-core fp32. */
int64_t kg_gemm_workspace_bytes(int64_t M, int64_t K, int64_t N);
kg_status kg_gemm_f32(const float* A, int64_t lda, const int32_t* a_rows, const float* B, int64_t ldb, float* C,
                      int64_t ldc, const int32_t* c_rows, int64_t M, int64_t K, int64_t N, int32_t relu,
                      int32_t trans, int32_t impl, void* ws, int64_t ws_bytes, void* stream);
int64_t kg_loss_workspace_bytes(int64_t b, int32_t n, int32_t d, int32_t R);
/* ref:model.py:254-281: DistMult scores of batch rows (start+q) mod total,
 * BCE loss (mean, device scalar), d_decoder (R,d) and dH (rows of the
 * seeds, by local id). Non-finite score/loss sets bits in *flags. */
kg_status kg_distmult_loss(const float* H, int32_t d, int32_t n_local, const float* decoder, int32_t R,
                           const int32_t* stream_triples, const float* labels, int64_t total, int64_t start,
                           const int64_t* start_dev, int64_t b, const int32_t* vertex_order, const int32_t* counts,
                           float* dH,
                           float* d_decoder, float* loss_out, float* scores_out, uint32_t* flags, void* ws,
                           int64_t ws_bytes, void* stream);
/* The batch-derived fields kg_loss_groups leaves in ws (sorted values and
 * segment bounds), as (pointer, bytes) pairs; returns their count (<= max).
 * A trainer may precompute them for every round and copy them back in. */
int32_t kg_loss_group_fields(void* ws, int64_t ws_bytes, int64_t b, int32_t n_local, int32_t d, int32_t R,
                             void** ptrs, int64_t* bytes, int32_t max);
/* kg_distmult_loss in two halves with identical arguments and workspace:
 * kg_loss_groups only sorts the batch keys and builds the segment bounds
 * (needs the closure's seed order, not H), so a trainer can run it on a
 * second stream concurrently with the layers; kg_loss_compute (ordered after
 * it) scores, reduces the loss and scatters d_decoder / dH. */
kg_status kg_loss_groups(const float* H, int32_t d, int32_t n_local, const float* decoder, int32_t R,
                         const int32_t* stream_triples, const float* labels, int64_t total, int64_t start,
                         const int64_t* start_dev, int64_t b, const int32_t* vertex_order, const int32_t* counts,
                         float* dH, float* d_decoder, float* loss_out, float* scores_out, uint32_t* flags, void* ws,
                         int64_t ws_bytes, void* stream);
/* side_stream (optional): the loss mean and d_decoder are produced on it
 * (only dH stays on `stream`); order it before reading them. */
kg_status kg_loss_compute(const float* H, int32_t d, int32_t n_local, const float* decoder, int32_t R,
                          const int32_t* stream_triples, const float* labels, int64_t total, int64_t start,
                          const int64_t* start_dev, int64_t b, const int32_t* vertex_order, const int32_t* counts,
                          float* dH, float* d_decoder, float* loss_out, float* scores_out, uint32_t* flags,
                          void* ws, int64_t ws_bytes, void* stream, void* side_stream);

/* R7/R8 + R16 batch-only half, for a whole epoch in one call: for every
 * round r < rounds, kg_closure of stream rows [r*b, (r+1)*b) into
 * order/pos (rounds, n) and counts (rounds, hops+1) row r, kg_loss_groups
 * into loss_ws, and the kg_loss_group_fields exported to
 * groups + r*groups_stride at 256-byte aligned offsets. Replaces the
 * build_compute_graph call of every round of ref:trainer.py:212-214 (plus
 * the batch grouping of the loss) for a trainer that prepares an epoch ahead. */
typedef struct kg_epoch_prep_args {
  const kg_graph_csr* g;
  int32_t hops;
  int32_t rounds;
  const int32_t* stream_triples; /* (total, 3) */
  const float* labels;           /* (total)    */
  int64_t total;
  int64_t b;
  int32_t d;
  int32_t R;
  int32_t* order;
  int32_t* pos;
  int32_t* counts;
  uint8_t* groups;
  int64_t groups_stride;
  uint32_t* flags;
  void* closure_ws;
  int64_t closure_ws_bytes;
  void* loss_ws;
  int64_t loss_ws_bytes;
  /* >= 1: rounds run as this many concurrent branches (at most
   * KG_PREP_MAX_BRANCHES), branch k using the workspaces at
   * closure_ws + k*closure_ws_bytes and loss_ws + k*loss_ws_bytes. */
  int32_t branches;
} kg_epoch_prep_args;
#define KG_PREP_MAX_BRANCHES 4
kg_status kg_epoch_prep(const kg_epoch_prep_args* a, void* stream);

/* ---------------------------------------------------------------------- */
/* R19/R20  Reduction + optimizer (ref:trainer.py:63-151)                  */
/* ---------------------------------------------------------------------- */
int64_t kg_optim_workspace_bytes(int64_t n);
/* step_dev (optional, device int64 Adam step t) overrides bc1/bc2 for
 * graph replay. Dense step on the flat block buffer. grads_all holds P payloads
 * back to back (P*n); they are combined in the reference's pairwise-tree
 * order and divided by P (ref:trainer.py:77-86) inside the same kernel.
 * optimizer: 0 = sgd, 1 = adam. grad_clip <= 0 disables clipping. */
kg_status kg_dense_step(float* params, float* m, float* v, const float* grads_all, int32_t P, int64_t n,
                        int32_t optimizer, float lr, float beta1, float beta2, float eps, double bc1,
                        double bc2, const int64_t* step_dev, float grad_clip, uint32_t* flags, void* ws,
                        int64_t ws_bytes, void* stream);
/* Peer-memory exchange of the dense gradient payloads, one partition per rank
 * on one NVLink node: replaces the all-gather of ref:trainer.py:430-438 ahead
 * of the tree mean (ref:trainer.py:77-86). kg_peer_alloc returns a zeroed
 * region of kg_peer_region_bytes(n) and its 64-byte cudaIpcMemHandle;
 * kg_peer_open maps a peer's handle. Per round, kg_peer_publish copies this
 * rank's n floats into its region (slot = round parity) and releases the
 * region's flag; kg_peer_gather waits (bounded, 5 s; timeout sets KG_FLAG_PEER_TIMEOUT in
 * flags) for every peer's flag and writes the (P, n) payloads in partition
 * order to out. seq: 3 zeroed int64 device words private to this rank.
 * regions_dev: device array of the P region pointers (own + opened). */
int64_t kg_peer_region_bytes(int64_t n);
kg_status kg_peer_alloc(int64_t bytes, void** region, void* ipc_handle);
kg_status kg_peer_open(const void* ipc_handle, void** region);
kg_status kg_peer_close(void* region, int32_t owned);
kg_status kg_peer_publish(const float* local, void* region, int64_t n, int64_t* seq, void* stream);
kg_status kg_peer_gather(void* const* regions_dev, int32_t P, int64_t n, float* out, int64_t* seq,
                         uint32_t* flags, void* stream);
/* float64 compatibility entry points of the public host API
 * (`allreduce_mean`, `Optimizer.step`; ref:trainer.py:63-151): reference
 * operation order with round-to-nearest intrinsics, bit-identical to numpy.
 * kg_tree_mean_f64: payloads (P, n) back to back -> pairwise-tree mean.
 * kg_dense_step_f64: flat dense blocks; grad_clip < 0 disables clipping.
 * kg_sparse_step_f64: k (possibly repeated) row ids of a num_rows x d table,
 * old_rows = table[ids], grad_rows; out_rows = the rows the reference assigns
 * to table[ids]; em/ev (num_rows x d) updated from the last occurrence of each
 * id (numpy fancy-assignment semantics). */
kg_status kg_tree_mean_f64(const double* payloads, int64_t P, int64_t n, double* out, void* stream);
int64_t kg_dense_step_f64_workspace_bytes(int64_t n);
kg_status kg_dense_step_f64(double* params, double* m, double* v, const double* grads, int64_t n, int32_t optimizer,
                            double lr, double beta1, double beta2, double eps, double bc1, double bc2,
                            double grad_clip, uint32_t* flags, void* ws, int64_t ws_bytes, void* stream);
int64_t kg_sparse_step_f64_workspace_bytes(int64_t k, int32_t d, int64_t num_rows);
kg_status kg_sparse_step_f64(const double* old_rows, const double* grad_rows, const int64_t* ids, int64_t k,
                             int32_t d, double* em, double* ev, int64_t num_rows, int32_t optimizer, double lr,
                             double beta1, double beta2, double eps, double bc1, double bc2, double* out_rows,
                             void* ws, int64_t ws_bytes, void* stream);
/* Lazy sparse rows (ref:trainer.py:136-147): rows = vertex_order[0:counts[k]]
 * of the (n,d) table; grad rows by local id. */
kg_status kg_sparse_step(float* table, float* m, float* v, const float* grad, const int32_t* rows,
                         const int32_t* counts, int32_t k, int32_t d, int32_t optimizer, float lr,
                         float beta1, float beta2, float eps, double bc1, double bc2, const int64_t* step_dev,
                         int32_t n_max, void* stream);

/* Full-graph float64 encode for evaluation (ref:evaluate.py:107-122): every
 * vertex of the whole-graph view g is a target at every layer; src / rel /
 * cnt are the view's messages in reference order (same destination rows as
 * g->indptr) with the per-(dst, relation) message counts (norm = 1 / cnt
 * exactly); g's chunk table spreads hub rows over warps. dims[L+1];
 * bases[l] (B, d_l, d_{l+1}), coeffs[l] (2R+1, B): HOST arrays of DEVICE
 * float64 pointers. input (n, d_0), out (n, d_L) float64. B <= 8. */
int64_t kg_encode_full_f64_workspace_bytes(int32_t n, int64_t e, int32_t chunk, int32_t B, int32_t d_max);
kg_status kg_encode_full_f64(const kg_graph_csr* g, const int32_t* src, const int32_t* rel, const int32_t* cnt,
                             int32_t L, const int32_t* dims, int32_t B, const double* const* bases,
                             const double* const* coeffs, const double* input, double* out, void* ws,
                             int64_t ws_bytes, void* stream);

/* Given-candidates protocol (ref:evaluate.py:168-180), tail side only:
 * query i ranks candidate cand[cand_ptr[i] + true_pos[i]] (its true tail;
 * the caller appends it when absent) against cand[cand_ptr[i]..cand_ptr[i+1]).
 * ranks / ncand (= list length - 1) per query. d <= 256. */
kg_status kg_eval_candidates(const float* H, int32_t d, const float* decoder, const int32_t* queries, int64_t nq,
                             const int64_t* cand_ptr, const int32_t* cand, const int32_t* true_pos, int32_t policy,
                             double* ranks, int32_t* ncand, void* stream);

/* ---------------------------------------------------------------------- */
/* Float64 public-API path (encode / loss_from_cache, ref:model.py:151-301) */
/* ---------------------------------------------------------------------- */
/* One layer over the closure: targets p < T (local id order[p]); H_in /
 * H_out (n, d) float64 by local id; acc (T, B*din) and Z (T, dout) by
 * position are kept for the backward. src / rel / cnt: the view's messages in
 * reference order (norm = 1/cnt exactly). mask (optional, fp32 (T, dout) by
 * position, nonzero = keep) scales kept values by mask_scale. */
kg_status kg_forward_layer_f64(const kg_graph_csr* g, const int32_t* src, const int32_t* rel, const int32_t* cnt,
                               const int32_t* order, const int32_t* pos, int32_t T, int32_t din, int32_t dout,
                               int32_t B, const double* bases, const double* coeffs, const double* H_in, double* acc,
                               double* Z, double* H_out, int32_t relu, const float* mask, double mask_scale,
                               void* stream);
/* DistMult + BCE: loss (device scalar, accumulated), d_decoder (R, d) and
 * dH (n, d) by local id (accumulated; caller zeroes). */
kg_status kg_loss_f64(const int32_t* triples, const double* labels, int64_t b, const double* H, const double* decoder,
                      int32_t d, double* loss, double* d_decoder, double* dH, uint32_t* flags, void* stream);
int64_t kg_layer64_workspace_bytes(int64_t n, int32_t din, int32_t dout, int32_t B);
/* Layer gradients: dZ (T, dout) scratch, d_bases (B, din, dout), d_coeffs
 * (2R+1, B), dH_in (n, din) by local id (optional). */
kg_status kg_backward_layer_f64(const kg_graph_csr* g, const int32_t* src, const int32_t* rel, const int32_t* cnt,
                                const int32_t* order, const int32_t* pos, int32_t T, int32_t din, int32_t dout,
                                int32_t B, const double* bases, const double* coeffs, const double* H_in,
                                const double* acc, const double* Z, const double* dH_out, int32_t relu,
                                const float* mask, double mask_scale, double* dZ, double* d_bases, double* d_coeffs,
                                double* dH_in, void* ws, int64_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------- */
/* N1  n-hop halo expansion (ref:partition.py:211-282)                     */
/* ---------------------------------------------------------------------- */
/* tri: the graph's (m,3) int32 triples on the device. kg_halo_incidence
 * builds the incident-edge CSR (ptr[n+1], inc[2m]: edge ids touching each
 * vertex, any order). kg_halo_expand grows one partition from its core edge
 * ids by `hops` rounds of bidirectional BFS and writes, ascending, the
 * support edge ids (included, not core), the support vertices (reached, not
 * core endpoints) and the core endpoints, with their counts (device int32).
 * Output capacities: m, n, n. */
int64_t kg_halo_workspace_bytes(int64_t m, int64_t n);
kg_status kg_halo_incidence(const int32_t* tri, int64_t m, int64_t n, uint32_t* ptr, int32_t* inc, void* ws,
                            int64_t ws_bytes, void* stream);
kg_status kg_halo_expand(const int32_t* tri, int64_t m, int64_t n, const uint32_t* ptr, const int32_t* inc,
                         const int32_t* core_ids, int64_t n_core, int32_t hops, int32_t* support_ids,
                         int32_t* n_support, int32_t* support_vertices, int32_t* n_support_vertices,
                         int32_t* core_vertices, int32_t* n_core_vertices, void* ws, int64_t ws_bytes,
                         void* stream);

/* ---------------------------------------------------------------------- */
/* Dropout (ref:model.py:221-227)                                          */
/* ---------------------------------------------------------------------- */
/* mask[j] = (rng.random() >= p) / (1 - p) for j < counts[t] * d (row-major
 * (T, d) as numpy draws it), then advances g by counts[t] * d next64 draws.
 * n_max bounds counts[t] for the launch size. */
kg_status kg_dropout_mask(kg_pcg64* g, const int32_t* counts, int32_t t, int32_t d, double p, int64_t n_max,
                          float* mask, void* stream);
/* numpy Generator.uniform(low, high, size=count) from the host stream state
 * *g (not advanced: the caller moves its own generator on by count next64
 * draws): out[j] = low + (high - low) * random_j, bit-exact with numpy. The
 * trainer draws the initial embedding table this way (ref:model.py:108-128). */
kg_status kg_uniform_f64(const kg_pcg64* g, int64_t count, double low, double high, double* out, void* stream);

/* ---------------------------------------------------------------------- */
/* R24-R26  Filtered evaluation (ref:evaluate.py:93-225)                   */
/* ---------------------------------------------------------------------- */
/* Ranks of every query triple against all N entities, tail side and head
 * side, minus known collisions: tail_keys = sorted unique (h*R+r)*N+t of
 * train+valid+test, head_keys = sorted unique (t*R+r)*N+h. Records are
 * written in the reference order (per chunk: tail records, head records).
 * policy: 0 mean, 1 optimistic, 2 pessimistic. */
/* impl 0: all-entity scores on the tcgen05 tensor cores (3xTF32, d <= 128;
 * true score and candidate scores come from the same MMA arithmetic), known
 * candidates skipped in the fused compare/count epilogue; impl 1 (or d > 128):
 * CUDA-core tiles with an exact sequential fmaf chain per score. */
/* known_pairs: an upper bound on sum over (query, side) of the known
 * candidates other than the true entity (impl 0 scores them in a separate
 * pass); *overflow (device uint32, optional) is set when it was too small.
 * H64 / decoder64 (optional, impl 0): the same embeddings and decoder in
 * float64 (H = their fp32 rounding). The tensor-core pass then counts a
 * candidate as greater only outside a per-row error band around the true
 * score and decides every candidate inside the band (and the known ones in
 * it) from float64 scores (H64[a] * dec64[r]) . H64[c] — the reference's
 * arithmetic — so ranks follow the float64 scores exactly. */
int64_t kg_eval_workspace_bytes(int64_t nq, int32_t N, int32_t d, int64_t known_pairs);
kg_status kg_eval_filtered(const float* H, int32_t d, int32_t N, const float* decoder, int32_t R,
                           const int32_t* queries, int64_t nq, const int64_t* tail_keys, int64_t n_tail,
                           const int64_t* head_keys, int64_t n_head, int32_t policy, int32_t chunk,
                           int32_t impl, int64_t known_pairs, double* ranks, int32_t* ncand, uint32_t* overflow,
                           const double* H64, const double* decoder64, void* ws, int64_t ws_bytes, void* stream);
/* Sorted unique keys (a*R + r)*N + c of (k,3) triples with (a,c) = (col_a, col_c). */
int64_t kg_known_keys_workspace_bytes(int64_t k);
kg_status kg_known_keys(const int32_t* triples, int64_t k, int32_t col_a, int32_t col_c, int32_t N, int32_t R,
                        int64_t* keys_out, int32_t* n_out, void* ws, int64_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------- */
/* Host-side input producers (HOST pointers)        */
/* ---------------------------------------------------------------------- */
/* Edge loop of ref:graph.py:336-381 generate_synthetic: writes up to target
 * (h,r,t) rows to out (int64) and returns the count; advances *g exactly as
 * numpy's Generator (the caller continues with permutation()). */
int64_t kg_generate_synthetic(int64_t num_entities, int32_t num_relations, int64_t target, kg_pcg64* g,
                              int64_t* out, int64_t max_attempts);
/* Greedy streaming vertex cut of ref:partition.py:141-191 over edges in
 * `order` (int64); assign[e] = partition (int64). */
kg_status kg_vertex_cut_assign(const int64_t* triples, int64_t m, int64_t num_entities, int32_t P,
                               const int64_t* order, double balance_weight, int64_t cap, int64_t* assign);

#ifdef __cplusplus
}
#endif
#endif /* KGDIST_B200_H */
