// Internal launcher declarations of librc (not part of the C-ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rc {

// sets the thread-local message returned by rc_last_error(); returns code
int32_t set_error(int32_t code, const char* msg);

// Every hot-path kernel is launched with programmatic dependent launch (PDL): it may start while
// the previous kernel in the stream drains, runs its prologue (barrier init, TMEM allocation,
// descriptor prefetch), and blocks in griddepcontrol.wait before touching memory the previous
// kernel produced. Kernels call griddepcontrol.launch_dependents once all their CTAs are running.
// Opt a kernel in to > 48 KB of dynamic shared memory on the CURRENT device. The attribute is
// per device, so it is set once per (kernel, device) -- a process may hold contexts on several GPUs.
cudaError_t smem_opt_in(const void* kern, int bytes);

bool pdl_enabled();  // RC_PDL=0 in the environment turns the attribute off (A/B diagnostics)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// NEXT-4 zero-copy V ("maps logical prompt sequences to scattered physical
// memory pages"): for the layers >= c, the V row a stitched-arena row resolves to. One int32 per arena
// row: bits 30-31 = source (VSRC_ARENA / VSRC_ITEM / VSRC_PREFIX), bits 0-29 = the row in that source.
enum : uint32_t { VSRC_ARENA = 0u, VSRC_ITEM = 1u, VSRC_PREFIX = 2u };
constexpr uint32_t VMAP_ROW_MASK = (1u << 30) - 1u;
struct VSrc {                    // where each source's V planes live (one layer)
  const int32_t* vmap = nullptr; // [arena rows]; nullptr: every V row is in the arena (no zero-copy)
  const uint16_t* item = nullptr;    // item pool V plane of head 0 of the layer
  int64_t item_head_stride = 0;      // item_rows * dh
  const uint16_t* prefix = nullptr;  // prefix pool V plane of head 0 of the layer
  int64_t prefix_head_stride = 0;
};
__device__ __forceinline__ const uint16_t* vsrc_row(const VSrc& v, const uint16_t* arena_head0, int64_t arena_head_stride,
                                                    int kvh, int64_t arena_row, int dh) {
  const uint32_t code = v.vmap ? static_cast<uint32_t>(__ldg(v.vmap + arena_row)) : static_cast<uint32_t>(arena_row);
  const int64_t row = code & VMAP_ROW_MASK;
  switch (code >> 30) {
    case VSRC_ITEM: return v.item + kvh * v.item_head_stride + row * dh;
    case VSRC_PREFIX: return v.prefix + kvh * v.prefix_head_stride + row * dh;
    default: return arena_head0 + kvh * arena_head_stride + row * dh;
  }
}
// ---------------------------------------------------------------- dense GEMM (tcgen05, k_gemm.cu)
// C[M][N] = A[M][K] * B[N][K]^T, A and B bf16 K-major, fp32 accumulation in TMEM; the epilogue
// decides what happens to each fp32 accumulator row.
enum EpiKind : int {
  EPI_BF16 = 0,     // out bf16 [M][ldo] (= acc + bias)
  EPI_F32 = 1,      // out f32  [M][ldo]
  EPI_ADD_F32 = 2,  // out f32  [M][ldo] += acc (residual stream)
  EPI_SWIGLU = 3,   // B rows [g0 u0 g1 u1 ...] -> out bf16 [M][ldo] = silu(g) * u
  EPI_QKV = 4,      // packed [q | k | v] heads (dims [0, dh/2, 1, dh/2+1, ..]): RoPE at pos[row] on q,k; q -> q_out, k,v -> arena
  EPI_DEV = 5,      // packed [k | v] heads: RoPE on k, bf16 round, fixed-point |new - stitched| -> dev[row]
  EPI_QKV_DEV = 6,  // EPI_QKV that first scores k, v against the stitched arena rows it overwrites:
                    // |new - stitched| -> dev[dev_row[row]] where row_reuse[dev_row[row]] (gradual steps)
};

struct EpiArgs {
  void* out = nullptr;
  int64_t ldo = 0;
  const uint16_t* bias = nullptr;  // bf16 [N]
  const int32_t* pos = nullptr;    // [M] token positions (QKV/DEV)
  const int32_t* dst_row = nullptr;  // [M] stitched-arena rows (QKV/DEV)
  uint16_t* q_out = nullptr;
  int64_t q_ld = 0;
  uint16_t* arena_k = nullptr;  // layer base of K heads: [Hk][T_cap][dh]
  uint16_t* arena_v = nullptr;
  int64_t head_stride = 0;      // T_cap * dh
  const float* rope_cos = nullptr;  // [(2*rope_zero+1)][dh/2]
  const float* rope_sin = nullptr;
  int32_t rope_zero = 0;
  int32_t n_heads = 0, n_kv_heads = 0, head_dim = 0;
  unsigned long long* dev_out = nullptr;  // [M]
  const uint8_t* row_reuse = nullptr;     // [M] (EPI_QKV_DEV: indexed through dev_row)
  const int32_t* dev_row = nullptr;       // EPI_QKV_DEV: [M] GEMM row -> index into dev_out / row_reuse
  VSrc vsrc;                              // DEV: where the stitched V rows live (zero-copy V)
  // residual epilogues: workspace for partial tiles (split-K / stream-K) summed in K order by the
  // last-arriving CTA of a tile (bitwise-reproducible x); counters zero between launches
  float* ws = nullptr;      // gemm_ws_floats()
  int* ws_cnt = nullptr;    // 2 * gemm_ws_slots()
  int32_t ws_slots = 0;
  int32_t det = 1;          // 0: partial tiles reduce-add straight into x in arrival order
  // transposed residual GEMM only (early O-projection): ready[tt] counts the attention CTAs done with
  // 256-row token tile tt; a unit waits for ready[tt] >= ready_tgt[tt] (acquire) before loading its
  // tokens instead of waiting for the whole attention grid (griddepcontrol.wait is skipped). ready[4]
  // counts finished GEMM CTAs; the last one zeroes ready[0..4] for the next layer
  int32_t* ready = nullptr;
  int32_t ready_tgt[4] = {0, 0, 0, 0};
  int32_t t_pack = 0;       // transposed kernel: two stripes' 128-token tails share a slot (RC_GEMM_T_PACK)
  int32_t no_epi = 0;       // diagnostics: transposed kernel skips its epilogue (RC_GEMM_NOEPI)
};

bool make_tmap_bf16_2d(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld_elems,
                       uint32_t box_rows);
// c: output tensor map (fp32 [rows][cols], 32x32 SW128 boxes) for EPI_ADD_F32 (TMA reduce-add), else NULL
// a64: optional map over the same A operand with gemm_t_box_rows()-row boxes; with it, small-M GEMMs
// (QKV with head_dim 128, SwiGLU, residual; N % 256 == 0) run on the transposed CTA-pair kernel
cudaError_t gemm_launch(const CUtensorMap* a, const CUtensorMap* b, const CUtensorMap* c, int M, int N, int K, int bn,
                        int epi, const EpiArgs& ep, int num_sms, cudaStream_t s, const CUtensorMap* a64 = nullptr);
int gemm_t_box_rows();
int gemm_ws_slots();
size_t gemm_ws_floats();
bool gemm_use_transposed(int M, int N, int epi, int head_dim, int num_sms);
bool make_tmap_f32_2d(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld_elems);
int gemm_box_rows_b(int bn);

// ---------------------------------------------------------------- assemble gather (k_gather.cu)
struct GatherArgs {
  const int4* meta;      // per token {dst_row, src_row, delta, kind}
  int32_t n_tok;
  int32_t layer_begin, layer_end;
  int32_t n_kv_heads, head_dim;
  const uint16_t* item_pool; int64_t item_rows;     // [L][2][Hk][item_rows][dh]
  const int8_t* hist_q; const float* hist_s; int64_t hist_rows;  // [L][2][Hk][rows][dh], [L][2][Hk][rows]
  const uint16_t* prefix_pool; int64_t prefix_rows;
  uint16_t* arena; int64_t arena_rows;
  const float* rope_cos; const float* rope_sin; int32_t rope_zero;
  int32_t skip_pool_v = 0;  // NEXT-4 zero-copy V: ITEM / PREFIX V rows stay in their pools (not copied)
};
cudaError_t gather_launch(const GatherArgs& g, int num_sms, cudaStream_t s);
// NEXT-3 device-fed prototypes: meta entries of kind RC_TOK_HIST_DEV {dst, (request << 16) | j, pos, 4}
// -> {dst, pool row, pos - canon, RC_TOK_HIST} from proto ids req_ptr[request][j] and the dense table
enum { RC_TOK_HIST_DEV = 4 };
cudaError_t resolve_hist_launch(int4* meta, int32_t n, const uint64_t* req_ptr, const int2* proto_tab, int64_t tab_cap,
                                unsigned long long* err, cudaStream_t s);

#ifdef RC_COMMON_CUH  // device helpers of the kernel files (common.cuh included first)
// Zero-copy V (NEXT-4): the 128 rows of one V tile (d_h = 128), each from the arena or a pool (vmap),
// into the two [128 rows][64 bf16] SWIZZLE_128B halves (16 KB apart) the PV MMA reads. A warp
// resolves 4 rows per lane, then every cp.async instruction moves two whole 256-byte rows (lanes
// 0-15 / 16-31, 16 bytes each: coalesced); chunk c of a row lands at ((c ^ (row & 7)) << 4) of its
// 128-byte half row, the TMA SW128 pattern; rows past the arena capacity are zero-filled like TMA
// out-of-bounds boxes. Completion is signalled per lane by cp_async_mbar_arrive.
__device__ __forceinline__ void v_rows_cp_async(uint8_t* tile, const VSrc& vs, const uint16_t* arena_v,
                                                int64_t arena_head_stride, int64_t arena_row0, int kvh, int64_t t_cap) {
  constexpr int DHV = 128;
  constexpr uint32_t HALFB = 128 * 64 * 2;
  const int lane = threadIdx.x & 31;
  uint64_t src[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t ar = arena_row0 + lane + 32 * i;
    src[i] = ar < t_cap ? reinterpret_cast<uint64_t>(vsrc_row(vs, arena_v, arena_head_stride, kvh, ar, DHV)) : 0ull;
  }
  const int c = lane & 15;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int row = 32 * i + 2 * k + (lane >> 4);
      const uint64_t p = __shfl_sync(0xffffffffu, src[i], row & 31);
      const uint16_t* s = p ? reinterpret_cast<const uint16_t*>(p) + c * 8 : arena_v;
      cp_async16(tile + (c >> 3) * HALFB + row * 128 + (((c & 7) ^ (row & 7)) << 4), s, p != 0ull);
    }
  }
}
#endif
cudaError_t vmap_identity_launch(int32_t* vmap, const int32_t* rows, int32_t n, cudaStream_t s);
cudaError_t scatter_i32_launch(int32_t* dst, const int2* idx_val, int32_t n, cudaStream_t s);  // dst[x] = y

// ---------------------------------------------------------------- attention (k_attn.cu)
struct AttnArgs {
  const uint16_t* q;    // [R][H*dh]
  uint16_t* o;          // [R][H*dh]
  const int32_t* qpos;  // [R]
  const int4* tiles;    // {row_start, n_rows, kv_base_row, 0}
  int32_t n_tiles;
  const uint16_t* k;    // layer base [Hk][T_cap][dh]
  const uint16_t* v;
  int64_t head_stride;  // T_cap*dh
  int32_t n_heads, n_kv_heads, head_dim;
  float scale_log2;     // log2(e)/sqrt(dh)
  int32_t debug_mode = 0;  // 0 = normal; 1 = skip the softmax (pipeline timing diagnostics only)
  // KV split (tcgen05 kernel): tiles[] holds n_splits consecutive entries per query tile, .w = split
  // index; each covers a contiguous share of the KV tiles and writes a partial (normalised O, m, l)
  // that a merge kernel combines (small grids only; n_splits = 1 writes o directly)
  int32_t n_splits = 1;
  float* part_o = nullptr;   // [n_tiles][Hk][128][128]
  float* part_ml = nullptr;  // [n_tiles][Hk][128][2]
  float* lse_out = nullptr;  // optional [R][H]: m + log2(l) per query row (k_attn_tc, n_splits = 1; NEXT-1)
  int32_t split_min = 0;     // > 0 with n_splits = 2: adaptive split (tiles under split_min KV tiles unsplit)
  int32_t* split_flag = nullptr;  // [n_tiles / n_splits][Hk]: split CTAs' arrival counters (zero between launches)
  int32_t* work_ctr = nullptr;    // paired kernel: {next work item, finished CTAs}, zero between launches
  // paired kernel, KV chunks (small grids): > 0 cuts every pair's KV range into chunks of about
  // (all pair-steps) / (chunk_per_cta * grid) KV tiles; partials per chunk in part_o / part_ml at slot
  // ((tile * Hk + kvh) * ATTN_MAX_CHUNKS + chunk), merged by the last-arriving chunk (split_flag)
  float chunk_per_cta = 0.f;
  unsigned long long* prof = nullptr;  // paired kernel phase timing (-DRC_ATTN_PROF builds, RC_ATTN_PROF=1)
  int32_t s_prefetch = 0;  // single-tile kernel: load S_{j+1} from TMEM before signalling P_j (RC_ATTN_SPREFETCH)
  VSrc vsrc;                      // zero-copy V: V rows through vmap (cp.async loads) instead of TMA boxes
  // single-tile kernel, unsplit: per 256-row token tile, +1 per (tile, kv head) CTA whose output rows
  // touch it, after they are written (early O-projection; EpiArgs::ready)
  int32_t* ready = nullptr;
};
int attn_tokens_per_tile(int group);
cudaError_t attn_launch(const AttnArgs& a, cudaStream_t s);
// tcgen05 version (head_dim == 128): 128-row tiles, Q via a 3-D tensor map over q [R][H][dh],
// K/V via 2-D maps over the layer's arena [Hk*T_cap][dh] (k_attn_tc.cu)
int attn_tc_tokens_per_tile(int group);
int attn_tc_choose_splits(int n_tiles, int n_kv_heads, int est_kv_tiles, int num_sms, int* split_min);
cudaError_t attn_tc_launch(const CUtensorMap* tmQ, const CUtensorMap* tmK, const CUtensorMap* tmV, const AttnArgs& a,
                           int64_t t_cap, cudaStream_t s);
// paired-tile version for large grids (k_attn_pair.cu): a.tiles holds 2 entries per CTA, both of one
// request (odd counts padded with an empty tile); n_splits must be 1
cudaError_t attn_pair_launch(const CUtensorMap* tmQ, const CUtensorMap* tmK, const CUtensorMap* tmV,
                             const AttnArgs& a, int64_t t_cap, cudaStream_t s);
bool attn_use_pairs(int n_tiles, int n_kv_heads, int num_sms);
// KV-chunked paired launch (a.chunk_per_cta > 0): at most this many pairs, chunks per pair
constexpr int ATTN_CHUNK_MAX_PAIRS = 128, ATTN_MAX_CHUNKS = 8;
bool attn_chunk_auto();        // AUTO picks the chunked launch for small grids (RC_ATTN_CHUNK_AUTO)
float attn_chunk_per_cta();    // items per CTA the chunk length aims at (RC_ATTN_CHUNK_F)
// NEXT-1 attention mass (k_attn_mass.cu): column sums of the check-layer softmax per key
struct MassArgs {
  const int4* key_tiles;  // {request, first key position, keys in tile (<= 128), 0}
  int32_t n_key_tiles;
  const int4* req;        // per request {u_off, u_cnt, P (first U position), arena_row}
  const float* lse;       // [U][H] from pass 1
  unsigned long long* mass;  // [U] accumulated (zeroed by the caller)
  int32_t n_heads, n_kv_heads;
  float scale_log2;
};
cudaError_t attn_mass_launch(const CUtensorMap* tmQ, const CUtensorMap* tmK, const MassArgs& a, int64_t t_cap,
                             cudaStream_t s);
cudaError_t mass_combine_launch(unsigned long long* dev, const unsigned long long* mass, int32_t n, double lam,
                                cudaStream_t s);
// NEXT-3 LSH prototype matching (k_semlib.cu)
struct SemlibArgs {
  unsigned long long seed = 0;
  int32_t n_buckets = 0, n_proto = 0;
  const float* pos_table = nullptr;  // [n_buckets][16] fp32
  const float* H = nullptr;          // [8 * 16][64] hyperplanes
  const float* C = nullptr;          // [n_proto][64] unit centroids
  const uint32_t* tab_sig = nullptr; // [8][n_proto] ascending signatures per table
  const int32_t* tab_id = nullptr;   // [8][n_proto] prototype ids in that order
  const int32_t* bucket_ids = nullptr;    // prototype ids grouped by log bucket
  const int32_t* bucket_start = nullptr;  // [n_buckets + 1]
};
cudaError_t semlib_embed_launch(const SemlibArgs& s, int n, const int32_t* tok, const int32_t* off, float* C,
                                uint32_t* sig, cudaStream_t st);
cudaError_t semlib_match_launch(const SemlibArgs& s, int n, const int32_t* tok, const int32_t* off, int32_t* proto_out,
                                float* cos_out, cudaStream_t st);
bool make_tmap_bf16_3d(CUtensorMap* map, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1_bytes,
                       uint64_t s2_bytes, uint32_t b0, uint32_t b1, uint32_t b2);

// ---------------------------------------------------------------- small kernels (k_small.cu)
cudaError_t embed_launch(const uint16_t* emb, const int32_t* tok, int32_t rows, int32_t d, float* x, cudaStream_t s);
cudaError_t rmsnorm_launch(const float* x, const int32_t* row_idx, int32_t rows, int32_t d, const uint16_t* g,
                           float eps, uint16_t* out, cudaStream_t s);
cudaError_t gather_rows_f32_launch(const float* src, const int32_t* idx, int32_t rows, int32_t d, float* dst,
                                   cudaStream_t s);
struct SelectArgs {
  const unsigned long long* dev;  // [U rows]
  const uint8_t* ucls;            // [U rows] class of every U row
  const int4* req;                // per request {u_off, u_cnt, sel_off, n}  (prefix length = n - u_cnt)
  const int4* req2;               // per request {k_hist, k_item, arena_base, window}
  int32_t n_req;
  int32_t* sel_pos; int32_t* sel_dst; int32_t* sel_urow;
  // gradual steps (reading R-GF): u2s[U row] = the row's index in the previous Sel, -1 outside it
  // (those rows are no candidates); map[new Sel row] = its index in the previous Sel. NULL = one shot
  const int32_t* u2s = nullptr;
  int32_t* map = nullptr;
};
// dst[idx[j]] = j for j < n
cudaError_t scatter_index_launch(int32_t* dst, const int32_t* idx, int32_t n, cudaStream_t s);
cudaError_t dev_diag_launch(const uint16_t* kn, const uint16_t* ks, const uint16_t* vn, const uint16_t* vs, int32_t n,
                            int32_t width, unsigned long long* out, cudaStream_t s);
cudaError_t select_launch(const SelectArgs& a, cudaStream_t s);
cudaError_t cand_scores_launch(const float* logits, int64_t vocab, const int32_t* cand_req, const int32_t* idtok,
                               int32_t n, float* out, cudaStream_t s);
cudaError_t pool_transpose_launch(const void* src, int elem_bytes, int32_t n_tok, int32_t L, int32_t Hk,
                                  int32_t dh, void* dst, int64_t dst_rows, int64_t dst_row0, cudaStream_t s);
cudaError_t scale_transpose_launch(const float* src, int32_t n_tok, int32_t L, int32_t Hk, float* dst,
                                   int64_t dst_rows, int64_t dst_row0, cudaStream_t s);
cudaError_t copy_rows_launch(const void* src_base, int64_t src_rows, int64_t src_row0, void* dst_base,
                             int64_t dst_rows, int64_t dst_row0, int32_t n_rows, int32_t n_planes,
                             int32_t row_bytes, cudaStream_t s);
// batched peer pull (rc_fetch_remote): segment i copies n_rows rows of every plane from a source
// pool [planes][src_rows][row_bytes] at src_row0 to dst [planes][dst_rows][row_bytes] at dst_row0
struct CopySeg {
  const void* src;
  int64_t src_rows, src_row0, dst_row0;
  int32_t n_rows, pad;
};
cudaError_t copy_segments_launch(const CopySeg* segs, int32_t n_segs, int64_t total_rows, void* dst_base,
                                 int64_t dst_rows, int32_t n_planes, int32_t row_bytes, cudaStream_t s);
cudaError_t export_kv_launch(const uint16_t* arena, int64_t arena_rows, int32_t planes, int32_t dh, int32_t row0,
                             int32_t n, int32_t int8, void* out, float* scales, cudaStream_t s);
cudaError_t read_kv_launch(const uint16_t* arena, int64_t arena_rows, int32_t layer, int32_t Hk, int32_t dh,
                           int32_t row0, int32_t n, uint16_t* k_out, uint16_t* v_out, const VSrc& vs, cudaStream_t s);

}  // namespace rc
