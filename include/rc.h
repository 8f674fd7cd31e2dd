/* librc -- RcLLM beyond-prefix selective-attention prefill on B200 (sm_100a).
 *
 * C-ABI boundary of the hot path named by BASELINE.json north_star / SURVEY.md §8(b).
 * Paper: "RcLLM: Accelerating Generative Recommendation via Beyond-Prefix KV Caching"
 * (arxiv 2605.07443), PAPER.md line numbers cited per call.
 *
 * Conventions
 *   - Every function returns rc_status (0 = RC_OK, < 0 = error) and never throws; the message
 *     of the last error on the calling thread is rc_last_error(). On error there are no
 *     partial effects (pools, sequences and outputs are left as they were).
 *   - Device pointers are plain CUDA device addresses on the context's device; host pointers
 *     are read synchronously before the call returns. rc_stream is a cudaStream_t (NULL =
 *     legacy default stream). All GPU work is enqueued asynchronously on that stream; device
 *     outputs are valid once the stream reaches that point.
 *   - One rc_ctx per (process, device); a context is not thread-safe.
 *   - bf16 values are raw IEEE bfloat16 bit patterns (uint16), row-major.
 *   - Token classes: PREFIX = shared system prompt (exact prefix KV, never recomputed),
 *     FORCED = always recomputed (instruction tail, item misses, window), HIST = history token
 *     mapped to a prototype, ITEM = candidate-item token.
 */
#ifndef RC_H
#define RC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef int32_t rc_status;
#define RC_OK 0
#define RC_E_INVALID (-1)     /* bad argument, shape or state                               */
#define RC_E_NOMEM (-2)       /* device or pinned-host allocation failed                    */
#define RC_E_CAPACITY (-3)    /* pool / arena / workspace capacity exceeded                 */
#define RC_E_NOTFOUND (-4)    /* block id not resident (RC_MISS_ERROR), unknown sequence    */
#define RC_E_EXISTS (-5)      /* duplicate block id on registration                         */
#define RC_E_CUDA (-6)        /* CUDA runtime error (message has the CUDA error string)     */
#define RC_E_PEER (-7)        /* peer pool not attached / not accessible                    */
#define RC_E_UNSUPPORTED (-8) /* parameter combination not built (lambda < 1 with head_dim != 128) */

typedef struct rc_ctx rc_ctx;
typedef uint64_t rc_seq;     /* handle of an assembled request (its stitched KV) */
typedef void* rc_stream;     /* cudaStream_t */

enum { RC_POOL_ITEM_BF16 = 0, RC_POOL_HIST_INT8 = 1, RC_POOL_PREFIX_BF16 = 2, RC_POOL_ITEM_HOST_BF16 = 3 };
enum { RC_TOK_PREFIX = 0, RC_TOK_FORCED = 1, RC_TOK_HIST = 2, RC_TOK_ITEM = 3 };
enum { RC_MISS_ERROR = 0, RC_MISS_RECOMPUTE = 1 };

/* Decoder shape (Llama / Qwen2 family). head_dim in {16, 64, 128}; d_model <= 8192;
 * 2*n_kv_heads*head_dim <= 2048 (the R4 deviation of a token sums that many fixed-point terms and
 * must stay below 2^51 for the R6 selection key), else rc_create fails with INVALID. */
typedef struct rc_model_desc {
  int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ff, vocab;
  double rope_theta; /* RoPE base (rotate-half pairs) */
  float rms_eps;
  int32_t qkv_bias; /* 1: q/k/v projections carry a bias (Qwen2) */
} rc_model_desc;

/* Model weights: device bf16 pointers in HF layout (nn.Linear weight = [out][in]). The
 * per-layer members point to host arrays of n_layers device pointers. The library copies
 * q|k|v into one packed [(H+2H_kv)*d_h][d] matrix and gate|up into [2F][d] (interleaved in
 * 128-row chunks) at rc_create; the other tensors are used in place and must outlive the ctx. */
typedef struct rc_weights {
  const void* embed;      /* [vocab][d]   */
  const void* final_norm; /* [d]          */
  const void* lm_head;    /* [vocab][d]   */
  const void* const* ln1; /* [d]          */
  const void* const* wq;  /* [H*d_h][d]   */
  const void* const* wk;  /* [H_kv*d_h][d] */
  const void* const* wv;  /* [H_kv*d_h][d] */
  const void* const* bq;  /* [H*d_h] or NULL array when !qkv_bias */
  const void* const* bk;
  const void* const* bv;
  const void* const* wo;  /* [d][H*d_h]   */
  const void* const* ln2; /* [d]          */
  const void* const* wg;  /* [F][d]       */
  const void* const* wu;  /* [F][d]       */
  const void* const* wd;  /* [d][F]       */
} rc_weights;

/* Capacities (library-owned HBM, allocated at rc_create). Rows are tokens. */
typedef struct rc_pool_desc {
  int64_t item_rows;        /* item pool tokens (bf16), incl. the remote-fetch region      */
  int64_t remote_rows;      /* of item_rows: tokens reserved for rc_fetch_remote (LRU)      */
  int64_t hist_rows;        /* prototype rows (int8 + fp32 scales)                          */
  int64_t prefix_rows;      /* prefix pool tokens (bf16)                                    */
  int64_t arena_rows;       /* stitched-KV arena tokens (sum of live padded requests)       */
  int32_t max_seq_len;      /* longest prompt; <= 8192 (R6 key packing)                      */
  int32_t max_batch_tokens; /* largest sum of n in one rc_selective_prefill call            */
  int64_t host_item_rows;   /* host-tier item pool tokens (pinned host DRAM, same layout;
                               NEXT-2); 0 = none. Blocks there become resident in HBM only
                               through rc_fetch_host                                          */
} rc_pool_desc;

/* One request in decomposed form (output of rc_decompose_prompt; host memory). */
typedef struct rc_request {
  int32_t n;                 /* prompt length                                               */
  const int32_t* token_ids;  /* [n]                                                         */
  const uint8_t* cls;        /* [n] RC_TOK_*; PREFIX positions must be exactly 0..P-1       */
  const int64_t* src_id;     /* [n] prototype id (HIST), item id (ITEM), else ignored       */
  const int32_t* src_off;    /* [n] token offset inside the item block (ITEM), else 0       */
  uint64_t prefix_id;        /* registered PREFIX block (ignored when P == 0)               */
  int32_t n_cand;            /* candidates, slot order                                      */
  const int32_t* cand_idtok; /* [n_cand] ID token of each candidate (its first token, R19)  */
  const int32_t* hist_proto_dev; /* optional DEVICE int32 [number of HIST positions]: their prototype
                                 ids in position order, e.g. straight from rc_semlib_match (NEXT-3,
                                 PAPER.md:549) -- resolved to pool rows on the device, src_id of HIST
                                 positions ignored; NULL = the host src_id. An id that is not a
                                 registered prototype (< 2^31) leaves that position's stitched K/V
                                 unwritten and counts in rc_device_error_count (check it) */
} rc_request;

/* A prompt as segments: system prompt, history tokens,
 * candidate item blocks in request order, instruction tail. */
typedef struct rc_prompt {
  int32_t prefix_len;
  const int32_t* prefix_tokens;
  int32_t n_hist;
  const int64_t* hist_proto;  /* [n_hist] prototype id of every history token (LSH match)   */
  const int32_t* hist_tokens; /* [n_hist]                                                    */
  int32_t n_cand;
  const int64_t* cand_item;   /* [n_cand]                                                    */
  const int32_t* cand_len;    /* [n_cand]                                                    */
  const int32_t* cand_tokens; /* concatenated tokens of all candidates                       */
  int32_t n_tail;
  const int32_t* tail_tokens;
} rc_prompt;

typedef struct rc_prefill_params {
  int32_t r_rev_bp;           /* recompute ratio of history tokens, basis points (R5)        */
  int32_t r_item_bp;          /* recompute ratio of item tokens, basis points; 10000 = all   */
  float lambda;               /* Eq. 3 lambda in [0, 1]: 1 = deviation only (R3, default);
                                 < 1 adds the attention-mass term (NEXT-1, R2 / R2-FX):
                                 S = rint((1 - lambda) A + lambda D) in fp64 from this fp32 */
  int32_t check_layer;        /* c: layers < c full over U, deviation at c (R1), 0 <= c < L   */
  int32_t window;             /* last `window` positions always recomputed (R7)              */
  const int32_t* forced_sel;  /* optional host list: Sel positions per request, concatenated,
                                 ascending, must contain every FORCED position (test mode)   */
  const int32_t* forced_sel_off; /* [n_req+1] offsets into forced_sel (with forced_sel)      */
  int32_t attn_kernel;        /* attention launch shape (d_h = 128): RC_ATTN_AUTO chooses by grid
                                 size; the others force one (tests). Results agree within the
                                 rounding of the online softmax, not bit for bit */
  uint64_t* score_out;        /* optional device [sum of |U| over the batch], U rows request-major:
                                 the selection score of every U row (Eq. 3 fixed point, DESIGN.md
                                 R4 / R2-FX; only HIST/ITEM rows are meaningful); NULL = none */
  int32_t deterministic;      /* the layers < c (which decide Sel) always sum split-K / stream-K
                                 partial tiles in K order, so Sel is reproducible run to run;
                                 1 = the layers >= c as well (logits and hidden states bitwise
                                 reproducible, at the cost of a workspace round trip per split
                                 tile); 0 = those partials meet in fp32 reduce-adds in arrival order */
  /* Gradual filtering (NEXT-1 variant, reading R-GF; the CacheBlend scheme PAPER.md:557
     cites for "token importance persists across layers"). gradual_layers = g in [0, RC_MAX_GRADUAL]
     (0 = the one-shot selection above; zero-initialised fields keep it off): Sel_0 is taken at the
     check layer with the ratios r_start_*_bp (r_*_bp <= r_start_*_bp <= 10000); each layer
     l = c + i, i = 1..g, computes q/k/v for the rows of Sel_{i-1}, scores their HIST/ITEM rows by
     the Eq. 3 divergence (R4 fixed point) of that layer's fresh K/V against the stitched K/V, stores
     the fresh K/V of all of Sel_{i-1}, and keeps Sel_i = FORCED u window u per-class top-k_i among
     Sel_{i-1} at ratio r_i = r_start - floor((r_start - r) i / g); its attention and MLP run on
     Sel_i. Needs c + g <= L - 1; not with forced_sel or RC_ZERO_COPY_V (UNSUPPORTED). rc_sel_count
     and sel_pos_out / hidden refer to the final Sel_g. */
  int32_t gradual_layers;
  int32_t r_start_rev_bp, r_start_item_bp;
  int32_t* sel_trace;         /* optional device [sum_i |Sel_i|]: the positions of Sel_0 .. Sel_g,
                                 step-major, request-major within a step, ascending (each step's
                                 sizes: rc_sel_count at r_i); NULL = none */
} rc_prefill_params;
enum { RC_MAX_GRADUAL = 16 };
enum { RC_ATTN_AUTO = 0, RC_ATTN_SINGLE = 1, RC_ATTN_PAIRED = 2, RC_ATTN_SPLIT2 = 3, RC_ATTN_ADAPTIVE = 4,
       RC_ATTN_CHUNKED = 5 };
/* RC_ATTN_CHUNKED: the persistent paired kernel with every pair's causal KV range cut into chunks
   sized on the device so that all (pair, KV head, chunk) items fill the SMs about twice; partials
   merged by the last-arriving chunk (small grids, e.g. one request's selected rows at batch 1) */
/* RC_ATTN_SPLIT2: every query tile's KV range in two CTAs + merge; RC_ATTN_ADAPTIVE: the same launch,
   but tiles shorter than half the longest prompt's KV run unsplit (decided on the device from the
   selected positions; measured slower than unsplit at cfg3 batch 1, so AUTO does not choose it) */

/* ---------------------------------------------------------------- lifecycle */
rc_status rc_create(const rc_model_desc* m, const rc_weights* w, const rc_pool_desc* p, int32_t device,
                    rc_ctx** out);
void rc_destroy(rc_ctx* ctx);
const char* rc_last_error(void);
int32_t rc_abi_version(void); /* 1 */

/* Split a prompt into per-position arrays (SPEC.md:62-70 worked example:
 * 207 + 50 + 87 -> segment offsets 0, 207, 257, total 344). Host only. Capacity `cap`
 * positions; seg_start gets 2 + n_cand + 1 offsets (prefix, history, items..., tail).
 * Errors: INVALID (negative length), CAPACITY (n > cap). */
rc_status rc_decompose_prompt(const rc_prompt* pr, int32_t cap, int32_t* n_out, int32_t* token_ids, uint8_t* cls,
                              int64_t* src_id, int32_t* src_off, int32_t* seg_start);

/* ---------------------------------------------------------------- offline pools */
/* Register precomputed KV blocks (the offline artifacts of PAPER.md:384-386, 458) into
 * library-owned pool pages. kv: DEVICE, layout [n_tok_total][L][2][H_kv][d_h] (bf16 for
 * ITEM/PREFIX, int8 for HIST), K stored post-RoPE at the block's canonical positions
 * canon_pos[i] .. canon_pos[i]+n_tokens[i]-1 (R14). scales: DEVICE f32 [n_tok_total][L][2][H_kv]
 * for HIST (per token/layer/K-V/kv-head, R15), else NULL. HIST blocks are single tokens
 * (prototypes, n_tokens = 1). PREFIX blocks must have canon_pos = 0. Copies on `stream`;
 * the caller may free kv/scales after the stream passes this point. All-or-nothing.
 * Canonical positions must lie inside one prompt: 0 <= canon_pos[i] and canon_pos[i] + n_tokens[i]
 * <= max_seq_len (the alignment offset indexes the RoPE table over [-max_seq_len, max_seq_len]).
 * Errors: EXISTS (duplicate id), CAPACITY (pool full), INVALID (kind / shape / positions). */
rc_status rc_pool_register_blocks(rc_ctx* ctx, int32_t kind, int32_t n_blocks, const uint64_t* block_ids,
                                  const int32_t* n_tokens, const int32_t* canon_pos, const void* kv,
                                  const float* scales, rc_stream stream);
/* Resident blocks of a kind (host query). */
rc_status rc_pool_contains(rc_ctx* ctx, int32_t kind, int32_t n, const uint64_t* block_ids, uint8_t* out);

/* ---------------------------------------------------------------- online path */
/* Retrieval + alignment (PAPER.md:548-551, 566 steps (i)-(ii)): allocate each request's
 * stitched KV in the arena, resolve HIST tokens to prototype rows and ITEM tokens to item pool
 * rows, and enqueue the gather kernel that writes bf16(rot(Delta, deq(pool))) for layers
 * gather_from..L-1 and the exact PREFIX KV for all layers. Delta = position -
 * canonical position (may be negative). Item misses: RC_MISS_RECOMPUTE turns their tokens
 * FORCED; RC_MISS_ERROR fails with NOTFOUND and lists up to *n_missing (in:
 * capacity, out: count) distinct ids in out_missing. Unknown prototype / prefix -> NOTFOUND.
 * Errors: INVALID (n > max_seq_len, bad classes), CAPACITY (arena full). */
rc_status rc_assemble(rc_ctx* ctx, int32_t n_req, const rc_request* reqs, int32_t miss_policy, int32_t gather_from,
                      rc_seq* out_seqs, uint64_t* out_missing, int32_t* n_missing, rc_stream stream);

/* Device-side input errors since creation (unresolvable device-fed prototype ids); synchronises. */
int64_t rc_device_error_count(rc_ctx* ctx);

/* |Sel| per request for the given parameters (host; fixed by the layout, R5). */
rc_status rc_sel_count(rc_ctx* ctx, int32_t n_req, const rc_seq* seqs, const rc_prefill_params* prm,
                       int32_t* counts);

/* Selective recomputation over a ragged batch:
 * layers < c over all non-prefix tokens U; Eq. 3 at layer c: the deviation D in the R4 fixed
 * point and, for lambda < 1, the attention mass A of the layer-c softmax of U over the fresh
 * keys (two extra passes: row log-sum-exp, then column sums, R2-FX);
 * per-class top-k heavy hitters (R5/R6) + FORCED + window; layers c..L-1 for the
 * selected tokens only over the whole stitched KV (causal by position, R11), updating the
 * stitched KV at Sel; LM head on the last position. r_bp = 10000 with no PREFIX is full
 * prefill. Outputs (DEVICE, caller-allocated, each may be NULL):
 *   logits      f32 [n_req][vocab]          last-position logits
 *   cand_scores f32 [sum n_cand]            logits[cand_idtok] (R19), request-major
 *   sel_pos     i32 [sum |Sel|]             selected positions, ascending per request
 *   hidden      f32 [sum |Sel|][d]          x_L at Sel (before the final norm, R20)
 * Position n-1 must be recomputed (its logits are the output): FORCED, or inside the window.
 * Errors: INVALID (params, c < gather_from of a sequence, forced_sel malformed, last position
 * neither FORCED nor in the window),
 * UNSUPPORTED (lambda < 1 with head_dim != 128), CAPACITY (sum n > max_batch_tokens),
 * NOMEM (attention-mass workspace on first lambda < 1 call), NOTFOUND (seq). */
rc_status rc_selective_prefill(rc_ctx* ctx, int32_t n_req, const rc_seq* seqs, const rc_prefill_params* prm,
                               float* logits, float* cand_scores, int32_t* sel_pos, float* hidden,
                               rc_stream stream);

/* Free the stitched KV of sequences (unknown handles are ignored). */
void rc_release(rc_ctx* ctx, int32_t n, const rc_seq* seqs);

/* ---------------------------------------------------------------- multi-GPU (§8(e)) */
/* Alg. 1 similarity-aware item placement with global replicas, host only.
 * Phase 1 heat h_i = occurrences of item i in the historical requests (CSR hist_off [n_hist+1] /
 * hist_items); Phase 2 the top ceil(hot_bp/10000 * n_items) items by heat (ties -> smaller id)
 * are replicated on all k instances (part_out = -1); Phases 3-5 the cold items form a graph with
 * edge weight = number of historical requests in which both occur, partitioned k ways
 * minimising the edge cut with every part's token weight (item_tokens) <= (1+eps) * total/k
 * (multilevel heavy-edge coarsening + greedy + boundary refinement, `passes` per level; a
 * self-contained stand-in for METIS). Outputs: part_out [n_items] in -1..k-1, edge cut,
 * heat_out [n_items] (may be NULL). Deterministic. Errors: INVALID. */
rc_status rc_place_items(int32_t n_items, const int32_t* item_tokens, int32_t n_hist, const int64_t* hist_off,
                         const int32_t* hist_items, int32_t k, int32_t hot_bp, double balance_eps, int32_t passes,
                         int32_t* part_out, int64_t* cut_out, int64_t* heat_out);
/* Eq. 2 affinity routing, host only, requests in arrival order:
 * Affinity(R,p) = alpha * |I(R) n C(p)|/|I(R)| + beta * (1 - Load(p)), Load(p) = backlog[p] /
 * max(1, max_q backlog[q]) (queue tokens); route = argmax, ties -> smaller p;
 * the chosen backlog grows by req_tokens[r]. C(p) = resident[p * n_items + i] != 0.
 * backlog [k] is read and updated in place. Errors: INVALID (empty request, id out of range). */
rc_status rc_route(int32_t n_req, const int64_t* req_off, const int32_t* req_items, const int64_t* req_tokens,
                   int32_t k, int32_t n_items, const uint8_t* resident, double alpha, double beta, int64_t* backlog,
                   int32_t* route_out);
/* Export the item pool allocation as a CUDA IPC handle (64 bytes) for peers. */
rc_status rc_pool_export(rc_ctx* ctx, void* ipc_handle_out, int64_t* pool_rows_out);
/* Map peers' item pools (one-sided NVLink reads). rank = the peer's index used in
 * rc_fetch_remote; a handle equal to this context's own export maps loopback. */
rc_status rc_peer_attach(rc_ctx* ctx, int32_t n_peers, const int32_t* peer_rank, const int32_t* peer_device,
                         const void* const* ipc_handles, const int64_t* pool_rows);
/* This pool's own item blocks (not remote-cache copies) for publishing to peers: up to `cap`
 * entries of (id, first pool row, n_tokens, canonical start); *n_out = the total count.
 * Pass cap = 0 to query the size. Errors: CAPACITY (cap < count; n_out still set). */
rc_status rc_pool_list(rc_ctx* ctx, int32_t cap, uint64_t* item_ids, int64_t* pool_rows, int32_t* n_tokens,
                       int32_t* canon_pos, int32_t* n_out);
/* Load an attached peer's item directory (its rc_pool_list, exchanged by the caller through
 * torch.distributed), replacing any earlier one for that rank. Host arrays, copied. Every entry
 * must lie inside the peer's pool rows and the position range. All-or-nothing.
 * Errors: PEER (rank not attached), INVALID (entry out of range). */
rc_status rc_peer_directory(rc_ctx* ctx, int32_t peer_rank, int32_t n, const uint64_t* item_ids,
                            const int64_t* pool_rows, const int32_t* n_tokens, const int32_t* canon_pos);
/* Pull item blocks from their owners' pools over NVLink into this context's remote-cache
 * region and make them resident here (the beyond-paper replacement of "cache misses are
 * computed on-the-fly"). owner_rank[i] = the attached peer holding
 * item_ids[i]; rows, lengths and canonical positions come from that peer's directory
 * (rc_peer_directory). Already-resident and repeated ids are skipped. The region is an LRU
 * cache: blocks not used by this call may be evicted (least recently used first; rc_assemble
 * and fetches mark use), planned on the host before any state changes; then ONE batched copy
 * kernel (one-sided peer reads, 16-byte vectors) moves every block on `stream`. Ordering: the
 * caller orders a fetch after the rc_assemble calls that read blocks it may evict.
 * Errors: PEER (rank not attached), NOTFOUND (id not in the owner's directory), CAPACITY (the
 * blocks of one call exceed the region) -- with no partial effects. */
rc_status rc_fetch_remote(rc_ctx* ctx, int32_t n_items, const uint64_t* item_ids, const int32_t* owner_rank,
                          rc_stream stream);
/* Host tier (the paper's CPU-resident item cache with its PCIe transfer,
 * PAPER.md:551, 566): copy item blocks registered with RC_POOL_ITEM_HOST_BF16 into this
 * context's remote-cache region (LRU, shared with rc_fetch_remote) with the copy engines (one
 * 2-D H2D copy per block: L*2*H_kv runs of n_tokens*d_h*2 bytes), so the transfer uses no SMs and
 * overlaps kernels when issued on a side stream -- e.g. the next batch's host-tier items while
 * the current batch computes. Already-resident ids are skipped. Ordering: a fetch may evict
 * remote blocks that are not part of this call; the caller orders it after the rc_assemble that
 * read them (stream or event). Errors: NOTFOUND (id in no tier), CAPACITY (remote region too
 * small for one call), INVALID (no host tier). */
rc_status rc_fetch_host(rc_ctx* ctx, int32_t n_items, const uint64_t* item_ids, rc_stream stream);
/* First pool row of resident item blocks (-1 if absent), for building fetch requests. */
rc_status rc_pool_locate(rc_ctx* ctx, int32_t n, const uint64_t* item_ids, int64_t* rows_out);

/* ---------------------------------------------------------------- semantic library (NEXT-3) */
/* Online LSH matching of history tokens to prototypes (SPEC.md:237-263
 * embed_token / match_token) under DESIGN.md reading R-LSH: position-aware unit embeddings of
 * D = 64 (48 seeded feature-hash lexical dims + 16 sinusoidal dims of the log2 bucket of the
 * history offset), 8 tables x 16-bit random-hyperplane signatures, fixed fp32 reduction order.
 * Build (host arrays, copied): prototype pi = (proto_token[pi], proto_offset[pi]) with centroid
 * embed(token, offset); hyperplanes fp32 [128][64] (table-major); replaces any earlier library.
 * Errors: INVALID (n_proto <= 0, n_buckets not in [1, 32], negative offset), NOMEM. */
rc_status rc_semlib_build(rc_ctx* ctx, int32_t n_proto, const int32_t* proto_token, const int32_t* proto_offset,
                          int32_t n_buckets, const float* hyperplanes, uint64_t seed);
/* Match n history tokens (DEVICE int32 token ids and history offsets) -> DEVICE proto_out int32
 * [n] (max-cosine prototype over the union of the 8 LSH buckets, ties -> smaller id; no candidate
 * -> best of the query's log bucket, else of all prototypes) and cos_out f32 [n]. Async on
 * `stream`. Errors: INVALID (no library, null pointers). */
rc_status rc_semlib_match(rc_ctx* ctx, int32_t n, const int32_t* token, const int32_t* offset, int32_t* proto_out,
                          float* cos_out, rc_stream stream);

/* ---------------------------------------------------------------- profiling */
/* Kernel classes for per-kind timing. */
enum { RC_K_GEMM = 0, RC_K_ATTN = 1, RC_K_GATHER = 2, RC_K_SELECT = 3, RC_K_SMALL = 4, RC_K_LMHEAD = 5,
       RC_K_FETCH = 6, RC_K_COUNT = 7 };
/* Start recording a CUDA event pair around every subsequent librc kernel launch of this ctx. */
rc_status rc_profile_begin(rc_ctx* ctx);
/* Synchronize the device, stop recording and report per kind (arrays of n_kinds): summed kernel
 * time in ms, launch count, algorithmic FLOPs (GEMM: 2MNK; attention: 4 H d_h sum_q (pos_q+1))
 * and algorithmic bytes (gather: pool reads + stitched writes). */
rc_status rc_profile_end(rc_ctx* ctx, int32_t n_kinds, double* ms, int64_t* count, double* flops, double* bytes);

/* ---------------------------------------------------------------- diagnostics (tests) */
/* Stitched KV of one layer of a sequence -> DEVICE bf16 k_out/v_out [n][H_kv][d_h]. */
rc_status rc_seq_read_kv(rc_ctx* ctx, rc_seq seq, int32_t layer, void* k_out, void* v_out, rc_stream stream);
/* Pool materialisation ("precomputes their KV blocks
 * offline"): the stitched KV of positions pos0 .. pos0+n_tok-1 of a sequence (typically after a
 * full prefill, r = 100%) -> DEVICE kv_out in the registration layout [n_tok][L][2][H_kv][d_h]:
 * bf16 (int8 = 0), or int8 codes with DEVICE scales_out f32 [n_tok][L][2][H_kv] quantised by R15
 * (scale = absmax/127 per token, layer, K/V and kv-head; q = clamp(rint_even(x/scale), -127, 127)).
 * Async on `stream`. Errors: NOTFOUND (seq), INVALID (range). */
rc_status rc_seq_export_kv(rc_ctx* ctx, rc_seq seq, int32_t pos0, int32_t n_tok, int32_t int8, void* kv_out,
                           float* scales_out, rc_stream stream);
/* K5+K6 unit path on given bf16 operands (DEVICE): D[i] = sum |a - b| in the R4 fixed point
 * over `width` elements of K and V, then the selection of rc_selective_prefill for one request
 * whose U rows are these n_u tokens (classes cls, positions P..P+n_u-1). Outputs: dev_out
 * u64 [n_u], sel_out i32 [count]. */
rc_status rc_diag_deviation_select(int32_t n_u, int32_t width, const void* k_new, const void* k_st,
                                   const void* v_new, const void* v_st, const uint8_t* cls_host, int32_t prefix_len,
                                   int32_t r_rev_bp, int32_t r_item_bp, int32_t window, uint64_t* dev_out,
                                   int32_t* sel_out, int32_t* n_sel_out, rc_stream stream);
/* The tcgen05 GEMM on its own: C f32 [M][N] = A bf16 [M][K] * B bf16 [N][K]^T (DEVICE). */
rc_status rc_diag_gemm(int32_t M, int32_t N, int32_t K, const void* A, const void* B, float* C, int32_t bn,
                       rc_stream stream);
/* The residual GEMM on its own: X f32 [M][N] += A bf16 [M][K] * B bf16 [N][K]^T (DEVICE), through
 * the same kernel choice as the hot path (transposed = 1 offers the small-M transposed pair kernel;
 * split-K / stream-K partial tiles are summed in K order). Synchronises `stream`. N % 32 == 0. */
rc_status rc_diag_gemm_add(int32_t M, int32_t N, int32_t K, const void* A, const void* B, float* X,
                           int32_t transposed, rc_stream stream);
/* Kernel launches issued by this context since creation (every librc kernel counts). */
int64_t rc_launch_count(rc_ctx* ctx);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* RC_H */
