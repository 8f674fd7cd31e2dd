// K4/K7 on tcgen05 (d_h = 128): causal attention of query tokens over their request's stitched
// KV, S and O accumulated in TMEM (Eq. 1; R11).
//
// CTA = (query tile, kv head). Tile = TQ tokens x G grouped query heads = 128 rows (G = 4: 32
// tokens; G = 7: 18 tokens = 126 rows); row r <-> TMEM lane r. KV streamed in 128-key tiles.
//   warp 0 lane 0   TMA: Q once (3-D box [TQ][G][64] x 2 halves), K tiles (2-stage ring)
//   warp 3 lane 0   TMA: V tiles (2-stage ring)
//   warp 1 lane 0   MMA: S_j = Q K_j^T (M=128, N=128, K=128; A, B K-major SW128) into TMEM S[j%2];
//                        O_h += P_{j,h} V_{j,h} for the two 64-key halves h of the tile (A = P from
//                        TMEM, TS mode; B = V rows of that half, MN-major SW128) into TMEM O_h
//   warps 4..11     softmax: two independent groups (key half h = 0, 1) of 4 warps; thread = (row,
//                   64 keys of every tile). Each group keeps its own running max / sum and its own
//                   accumulator O_h, so the groups never synchronise inside the KV loop and the MMA
//                   warp can start PV on one half while the other is still in exp; the two partial
//                   softmaxes are merged once at the end (flash-decoding style combine).
//                   Per tile: tcgen05.ld of its S slice, causal mask by true position (skipped on
//                   full tiles), lazy O_h rescale (only when the max grows by > 2^8),
//                   P = 2^(s*scale - m) -> bf16 pairs -> TMEM over its own S columns.
// TMEM: S[2] (2 x 128 columns) + O_0, O_1 (2 x 128) = 512 columns.
#include "common.cuh"
#include "rc_internal.h"

namespace rc {
namespace {

constexpr int DH = 128, BKV = 128, ROWS = 128;
constexpr uint32_t HALF = ROWS * 64 * 2;  // one [128 rows][64 bf16] SW128 sub-tile = 16 KB
constexpr uint32_t TILE = 2 * HALF;       // 32 KB
constexpr int SCOLS = 64;                  // keys per softmax thread per tile (two key halves)
constexpr int NTHREADS = 128 + 256;        // 4 control warps + 2 x 4 softmax warps
// 2-deep K and V rings whose "empty" events are the MMA commits that already exist: K_j's slot is
// free once S_j is complete (s_full[j & 1]) and V_j's once both PV halves of step j are
// (pv_done[j & 1]), so the single MMA thread commits twice per KV step instead of five times
// (its serial barrier work bounds a one-request grid)
constexpr int KST = 2, VST = 2;
constexpr uint32_t OFF_Q = 0, OFF_K = TILE, OFF_V = OFF_K + KST * TILE, OFF_BAR = OFF_V + VST * TILE;
constexpr uint32_t OFF_RED = OFF_BAR + 256;  // [2 halves][2 (m, l)][128 rows] f32 for the final merge
constexpr uint32_t OFF_FLAG = OFF_RED + 2 * 2 * 128 * 4;  // KV split: "this CTA merges" flag
constexpr uint32_t SMEM_BYTES = OFF_FLAG + 16;
constexpr uint32_t O_COL = 256;            // O_h at 256 + 128 h
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 domain
// every 2^x of P on the SFU: measured at cfg3 batch 1, 1.49 ms per step vs 1.62 with 3/8 on the FMA pipe
#ifndef RC_TC_POLY  // diagnostics builds only (RC_BUILD_DEFS=-DRC_TC_POLY=...): 8-key chunks on the FMA pipe
#define RC_TC_POLY 0x00
#endif
constexpr unsigned POLY_CHUNKS = RC_TC_POLY;
constexpr float SPEC_SUM_MAX = 18446744073709551616.0f;  // 2^64: bound of the speculative exps' row sum

__global__ void __launch_bounds__(NTHREADS, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, const AttnArgs a, int64_t t_cap) {
  // SWIZZLE_128B atoms need a 1024-aligned dynamic window; checked below.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  uint8_t* sQ = smem + OFF_Q;
  uint8_t* sK = smem + OFF_K;
  uint8_t* sV = smem + OFF_V;
  float* red = reinterpret_cast<float*>(smem + OFF_RED);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* q_full = bars;                 // [1]
  uint64_t* k_full = bars + 1;             // [KST]
  uint64_t* v_full = k_full + KST;         // [VST]
  uint64_t* s_full = v_full + VST;         // [2]  S_j complete (also: K slot j & 1 free)
  uint64_t* p_full = s_full + 2;           // [2 S buffers][2 halves]
  uint64_t* pv_done = p_full + 4;          // [2]  both PV halves of step j complete (also: V slot free)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < KST; ++i) mbar_init(&k_full[i], 1);
    for (int i = 0; i < VST; ++i) mbar_init(&v_full[i], a.vsrc.vmap ? 32 : 1);  // zero-copy V: one per lane
    for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&pv_done[i], 1); }
    for (int i = 0; i < 4; ++i) mbar_init(&p_full[i], 4);  // p_full: 1 per warp
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // PDL: prologue above overlapped the previous kernel's tail
  griddep_launch();
  // tiles of a request are in position order and the causal KV grows with position: launch them
  // last-first, every KV head of a tile next to each other, so the longest tiles of all heads start
  // in the first wave and short ones fill the tail (longest-processing-time order over the machine)
  const int tix = a.n_tiles - 1 - static_cast<int>(blockIdx.x) / a.n_kv_heads;
  const int kvh = static_cast<int>(blockIdx.x) % a.n_kv_heads;
  const int4 tile = a.tiles[tix];
  const int row_start = tile.x, n_rows = tile.y, kv_base = tile.z;
  const int G = a.n_heads / a.n_kv_heads;
  const int TQ = ROWS / G;
  const int H = a.n_heads;
  const int max_pos = n_rows > 0 ? a.qpos[row_start + n_rows - 1] : -1;
  const int nkv_all = n_rows > 0 ? max_pos / BKV + 1 : 0;  // padded (empty) tiles do nothing
  // adaptive 2-way split (split_min > 0): a tile shorter than split_min KV tiles runs unsplit in its
  // first CTA, which writes O directly; its second CTA has nothing to do
  const bool short_tile = a.split_min > 0 && nkv_all < a.split_min;
  const int nsp = short_tile ? 1 : a.n_splits;
  const bool idle = short_tile && tile.w != 0;
  const int j0 = idle ? 0 : tile.w * nkv_all / nsp;     // this split's KV tiles [j0, j0 + nkv)
  const int nkv = idle ? 0 : (tile.w + 1) * nkv_all / nsp - j0;

  if (warp == 0) {
    if (lane == 0) {  // ---- Q + K producer
      tma_prefetch_desc(&tmQ); tma_prefetch_desc(&tmK);
      mbar_expect_tx(q_full, 2u * 128u * G * TQ);
      tma_load_3d(sQ, &tmQ, q_full, 0, kvh * G, row_start);
      tma_load_3d(sQ + HALF, &tmQ, q_full, 64, kvh * G, row_start);
      const int krow0 = static_cast<int>(kvh * t_cap + kv_base) + j0 * BKV;
      for (int j = 0; j < nkv; ++j) {
        const int s = j % KST;
        mbar_wait(&s_full[s], ((j / KST) & 1) ^ 1);  // S_{j-2} complete: slot s is free
        mbar_expect_tx(&k_full[s], TILE);
        tma_load_2d(sK + s * TILE, &tmK, &k_full[s], 0, krow0 + j * BKV);
        tma_load_2d(sK + s * TILE + HALF, &tmK, &k_full[s], 64, krow0 + j * BKV);
      }
    }
  } else if (warp == 3) {
    if (a.vsrc.vmap != nullptr) {  // ---- V producer, zero-copy (NEXT-4): rows through vmap, 4 per lane
      const int64_t row0 = static_cast<int64_t>(kv_base) + static_cast<int64_t>(j0) * BKV;
      for (int j = 0; j < nkv; ++j) {
        const int s = j % VST;
        mbar_wait(&pv_done[s], ((j / VST) & 1) ^ 1);  // PV_{j-2} complete: slot s is free
        v_rows_cp_async(sV + s * TILE, a.vsrc, a.v, a.head_stride, row0 + static_cast<int64_t>(j) * BKV, kvh, t_cap);
        cp_async_mbar_arrive(&v_full[s]);  // arrives when this lane's copies land (no wait here)
      }
    } else if (lane == 0) {  // ---- V producer
      tma_prefetch_desc(&tmV);
      const int vrow0 = static_cast<int>(kvh * t_cap + kv_base) + j0 * BKV;
      for (int j = 0; j < nkv; ++j) {
        const int s = j % VST;
        mbar_wait(&pv_done[s], ((j / VST) & 1) ^ 1);  // PV_{j-2} complete: slot s is free
        mbar_expect_tx(&v_full[s], TILE);
        tma_load_2d(sV + s * TILE, &tmV, &v_full[s], 0, vrow0 + j * BKV);
        tma_load_2d(sV + s * TILE + HALF, &tmV, &v_full[s], 64, vrow0 + j * BKV);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idS = idesc_bf16_f32(128, 128);
      constexpr uint32_t idPV = idesc_bf16_f32_bmn(128, 128);
      mbar_wait(q_full, 0);
      tc_fence_after();
      const bool no_mma = (a.debug_mode & 2) != 0;  // diagnostics: barriers only
      auto issue_s = [&](int j) {  // S_j into buffer j % 2
        const int s = j % KST;
        mbar_wait(&k_full[s], (j / KST) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < (no_mma ? 0 : DH / 16); ++k) {
          const uint64_t ad = sdesc_sw128(smem_u32(sQ + (k >> 2) * HALF)) + 2 * (k & 3);
          const uint64_t bd = sdesc_sw128(smem_u32(sK + s * TILE + (k >> 2) * HALF)) + 2 * (k & 3);
          umma_bf16(tmem + (j & 1) * 128, ad, bd, idS, k > 0);
        }
        umma_commit(&s_full[j & 1]);
      };
      if (nkv > 0) issue_s(0);
      if (nkv > 1) issue_s(1);
      for (int j = 0; j < nkv; ++j) {
        const int b = j & 1, v = j % VST;
        mbar_wait(&v_full[v], (j / VST) & 1);
        if (a.vsrc.vmap) fence_proxy_async();  // zero-copy V: cp.async (generic proxy) writes -> MMA reads
        for (int h = 0; h < 2; ++h) {
          mbar_wait(&p_full[b * 2 + h], (j >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < (no_mma ? 0 : 4); ++k) {  // 64 keys: A = P_{j,h} (8 TMEM columns per 16 keys), B = V rows
            const uint64_t bd = sdesc_sw128_mn(smem_u32(sV + v * TILE + (4 * h + k) * 2048), HALF, 1024);
            umma_bf16_ts(tmem + O_COL + h * 128, tmem + b * 128 + h * 64 + k * 8, bd, idPV,
                         (j > 0 || k > 0) ? 1u : 0u);
          }
        }
        umma_commit(&pv_done[j & 1]);
        if (j + 2 < nkv) issue_s(j + 2);  // buffer b: both halves' P_j consumed by the PVs just issued
      }
    }
  } else if (warp >= 4) {  // ---- softmax: group h = key half, thread <-> (row, 64 keys of each tile)
    const int q = warp & 3;              // TMEM lane quarter of this warp
    const int h = (warp - 4) >> 2;       // key half
    const int col0 = h * SCOLS;
    const int r = q * 32 + lane;
    const int t = r / G, g = r % G;
    const bool valid = (r < TQ * G) && (t < n_rows);
    const int p = valid ? a.qpos[row_start + t] : -1;
    const int p_first = a.qpos[row_start];  // smallest position of the tile (rows sorted by position)
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t o_col = O_COL + h * 128;
    // padding rows see no key: base 0 keeps them off the max-first path (their P is 0, l stays 0)
    float m_run = valid ? -INFINITY : 0.f, l_run = 0.f;
    uint32_t sr[SCOLS];
    // S of the next step already requested (its TMEM load issued before this step's P store was
    // fenced and signalled, when the probe found S_{j+1} complete): the load latency overlaps that hand-off
    bool have_next = false;
    for (int j = 0; j < nkv; ++j) {
      const int b = j & 1;
      if (a.debug_mode & 1) {  // diagnostics: no softmax work
        mbar_wait(&s_full[b], (j >> 1) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b * 2 + h]);
        continue;
      }
      if (!have_next) {
        mbar_wait(&s_full[b], (j >> 1) & 1);
        tc_fence_after();
        tmem_ld32(tmem + lane_base + b * 128 + col0, sr);
        tmem_ld32(tmem + lane_base + b * 128 + col0 + 32, sr + 32);
      }
      have_next = false;
      tmem_wait_ld();
      const int key0 = (j0 + j) * BKV + col0;
      const bool full = key0 + SCOLS - 1 <= p_first;  // every row sees every key of the half: no mask
      uint32_t pk[SCOLS / 2];
      // common case: exps against the running max, no row-max pass at all. Kept unless some row's sum
      // exceeds 2^64 (then some P > 2^64, or inf/NaN): the step is redone below with the max first.
      // Any P <= 2^64 keeps O and l finite over 8192 keys, and bf16/fp32 precision is relative.
      if ((a.debug_mode & 4) == 0 && !__any_sync(0xffffffffu, m_run == -INFINITY)) {
        const float ls = full ? sm_exp_pack64<false, POLY_CHUNKS>(sr, pk, key0, p, a.scale_log2, m_run)
                              : sm_exp_pack64<true, POLY_CHUNKS>(sr, pk, key0, p, a.scale_log2, m_run);
        if (!__any_sync(0xffffffffu, !(ls <= SPEC_SUM_MAX))) {
          l_run += ls;
          tmem_st32(tmem + lane_base + b * 128 + col0, pk);
          if (a.s_prefetch && j + 1 < nkv &&
              __any_sync(0xffffffffu, mbar_test(&s_full[b ^ 1], ((j + 1) >> 1) & 1))) {
            mbar_wait(&s_full[b ^ 1], ((j + 1) >> 1) & 1);  // complete for every lane: returns at once
            tc_fence_after();
            tmem_ld32(tmem + lane_base + (b ^ 1) * 128 + col0, sr);
            tmem_ld32(tmem + lane_base + (b ^ 1) * 128 + col0 + 32, sr + 32);
            have_next = true;
          }
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[b * 2 + h]);
          continue;
        }
      }
      // scores stay raw; the softmax scale (> 0) is folded into the max and into one FFMA per exp2
      const float mx = (full ? sm_rowmax64<false>(sr, key0, p) : sm_rowmax64<true>(sr, key0, p)) * a.scale_log2;
      float alpha = 1.f;
      bool need = false;
      if (mx > m_run + RESCALE_THRESHOLD || (m_run == -INFINITY && mx != -INFINITY)) {
        const float m_new = fmaxf(m_run, mx);
        if (m_run != -INFINITY) { alpha = fast_exp2(m_run - m_new); need = true; }
        m_run = m_new;
      }
      if (j > 0 && __any_sync(0xffffffffu, need)) {  // rescale this group's accumulator rows (rare)
        mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
        uint32_t o[32];
#pragma unroll
        for (int c = 0; c < DH; c += 32) {
          tmem_ld32(tmem + lane_base + o_col + c, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(tmem + lane_base + o_col + c, o);
        }
        tmem_wait_st();
      }
      l_run *= alpha;
      const float base = (m_run == -INFINITY) ? 0.f : m_run;
      // P (bf16 pairs) overwrites the first 32 of this group's own 64 S columns (already in registers)
      l_run += full ? sm_exp_pack64<false, POLY_CHUNKS>(sr, pk, key0, p, a.scale_log2, base)
                    : sm_exp_pack64<true, POLY_CHUNKS>(sr, pk, key0, p, a.scale_log2, base);
      tmem_st32(tmem + lane_base + b * 128 + col0, pk);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b * 2 + h]);
    }
    // merge the two halves: O = (O_0 2^(m_0-m) + O_1 2^(m_1-m)) / (l_0 2^(m_0-m) + l_1 2^(m_1-m))
    red[(h * 2 + 0) * 128 + r] = m_run;
    red[(h * 2 + 1) * 128 + r] = l_run;
    asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
    const float m0 = red[0 * 128 + r], l0 = red[1 * 128 + r], m1 = red[2 * 128 + r], l1 = red[3 * 128 + r];
    const float m = fmaxf(m0, m1);
    const float mb = (m == -INFINITY) ? 0.f : m;
    const float f0 = (m0 == -INFINITY) ? 0.f : fast_exp2(m0 - mb);
    const float f1 = (m1 == -INFINITY) ? 0.f : fast_exp2(m1 - mb);
    const float l_tot = l0 * f0 + l1 * f1;
    const float inv = l_tot > 0.f ? 1.f / l_tot : 0.f;
    const float w0 = f0 * inv, w1 = f1 * inv;
    if (nkv > 0) {
      mbar_wait(&pv_done[(nkv - 1) & 1], ((nkv - 1) >> 1) & 1);
    }
    tc_fence_after();
    const bool split = nsp > 1;
    // this thread writes output columns [h*64, h*64 + 64) of its row: bf16 into o, or (KV split) the
    // fp32 partial normalised by its own l plus (m, l); the split CTA of a tile that finishes last
    // merges them (no merge kernel)
    uint16_t* dst = a.o + static_cast<int64_t>(row_start + t) * H * DH + (kvh * G + g) * DH + h * 64;
    const int64_t prow = (static_cast<int64_t>(tix) * a.n_kv_heads + kvh) * ROWS + r;
    float* pdst = split ? a.part_o + prow * DH + h * 64 : nullptr;
    if (split && h == 0 && !idle) {
      a.part_ml[prow * 2] = m;
      a.part_ml[prow * 2 + 1] = nkv > 0 ? l_tot : 0.f;
    }
    if (a.lse_out && h == 0 && valid)  // NEXT-1 pass 1: log2-sum-exp of the scaled scores of this row
      a.lse_out[static_cast<int64_t>(row_start + t) * H + kvh * G + g] = l_tot > 0.f ? m + __log2f(l_tot) : -INFINITY;
#pragma unroll
    for (int c = 0; c < 64; c += 32) {
      uint32_t o0[32], o1[32];
      if (nkv > 0) {
        tmem_ld32(tmem + lane_base + O_COL + h * 64 + c, o0);
        tmem_ld32(tmem + lane_base + O_COL + 128 + h * 64 + c, o1);
        tmem_wait_ld();
      }
      if (valid && !idle) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          float y[8];
#pragma unroll
          for (int k = 0; k < 8; ++k)
            y[k] = nkv > 0 ? __uint_as_float(o0[i + k]) * w0 + __uint_as_float(o1[i + k]) * w1 : 0.f;
          if (split) {
            reinterpret_cast<float4*>(pdst + c + i)[0] = make_float4(y[0], y[1], y[2], y[3]);
            reinterpret_cast<float4*>(pdst + c + i)[1] = make_float4(y[4], y[5], y[6], y[7]);
          } else {
            uint4 u;
            u.x = pack_bf2(y[0], y[1]); u.y = pack_bf2(y[2], y[3]); u.z = pack_bf2(y[4], y[5]); u.w = pack_bf2(y[6], y[7]);
            *reinterpret_cast<uint4*>(dst + c + i) = u;
          }
        }
      }
    }
    if (split) {  // arrival count per (logical tile, KV head); the last split CTA merges and resets it
      int* flag = reinterpret_cast<int*>(smem + OFF_FLAG);
      __threadfence();
      asm volatile("bar.sync 9, 256;" ::: "memory");
      if (warp == 4 && lane == 0) {
        int* ctr = a.split_flag + (tix / a.n_splits) * a.n_kv_heads + kvh;
        const int last = atomicAdd(ctr, 1) == nsp - 1;
        if (last) *ctr = 0;
        *flag = last;
      }
      asm volatile("bar.sync 9, 256;" ::: "memory");
      if (*flag && valid) {
        __threadfence();
        const int64_t prow0 = (static_cast<int64_t>(tix / a.n_splits * a.n_splits) * a.n_kv_heads + kvh) * ROWS + r;
        const int64_t pstride = static_cast<int64_t>(a.n_kv_heads) * ROWS;  // next split of the same tile
        float mm = -INFINITY;
        for (int s2 = 0; s2 < nsp; ++s2) {
          const float2 v = __ldcg(reinterpret_cast<const float2*>(a.part_ml + (prow0 + s2 * pstride) * 2));
          if (v.y > 0.f) mm = fmaxf(mm, v.x);
        }
        float wts[8], wsum = 0.f;
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) {
          wts[s2] = 0.f;
          if (s2 >= nsp) continue;
          const float2 v = __ldcg(reinterpret_cast<const float2*>(a.part_ml + (prow0 + s2 * pstride) * 2));
          if (v.y > 0.f) wts[s2] = v.y * fast_exp2(v.x - mm);
          wsum += wts[s2];
        }
        const float inv2 = wsum > 0.f ? 1.f / wsum : 0.f;
#pragma unroll 1
        for (int c = 0; c < 64; c += 8) {
          float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          for (int s2 = 0; s2 < nsp; ++s2) {
            if (wts[s2] == 0.f) continue;
            const float4* src = reinterpret_cast<const float4*>(a.part_o + (prow0 + s2 * pstride) * DH + h * 64 + c);
            const float4 x0 = __ldcg(src), x1 = __ldcg(src + 1);
            acc[0] += wts[s2] * x0.x; acc[1] += wts[s2] * x0.y; acc[2] += wts[s2] * x0.z; acc[3] += wts[s2] * x0.w;
            acc[4] += wts[s2] * x1.x; acc[5] += wts[s2] * x1.y; acc[6] += wts[s2] * x1.z; acc[7] += wts[s2] * x1.w;
          }
          uint4 u;
          u.x = pack_bf2(acc[0] * inv2, acc[1] * inv2); u.y = pack_bf2(acc[2] * inv2, acc[3] * inv2);
          u.z = pack_bf2(acc[4] * inv2, acc[5] * inv2); u.w = pack_bf2(acc[6] * inv2, acc[7] * inv2);
          *reinterpret_cast<uint4*>(dst + c) = u;
        }
      }
    }
  }
  // early O-projection (a.ready): this CTA's output rows are written; count it on every 256-row token
  // tile its rows touch, so the next kernel (the transposed O-proj, launched early by PDL) can start the
  // token tiles whose attention is complete while the longest tiles still run
  if (a.ready) __threadfence();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (a.ready && threadIdx.x == 0 && n_rows > 0 && nsp == 1)
    for (int tt = row_start / 256; tt <= (row_start + n_rows - 1) / 256; ++tt) atomicAdd(a.ready + tt, 1);
  if (warp == 2) tmem_dealloc(tmem, 512);
}

}  // namespace

int attn_tc_tokens_per_tile(int group) { return ROWS / group; }

cudaError_t attn_tc_launch(const CUtensorMap* tmQ, const CUtensorMap* tmK, const CUtensorMap* tmV, const AttnArgs& a,
                           int64_t t_cap, cudaStream_t s) {
  if (a.n_tiles <= 0) return cudaSuccess;
  if (cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(k_attn_tc), SMEM_BYTES); e != cudaSuccess) return e;
  if (a.n_splits > 8) return cudaErrorInvalidValue;
  return launch_pdl(k_attn_tc, dim3(a.n_tiles * a.n_kv_heads), dim3(NTHREADS), SMEM_BYTES, s, *tmQ, *tmK, *tmV, a,
                    t_cap);
}

int attn_tc_choose_splits(int n_tiles, int n_kv_heads, int est_kv_tiles, int num_sms, int* split_min) {
  *split_min = 0;
  // Split only grids that leave more than half the machine idle. Measured at cfg3 batch 1 (176
  // CTAs, ~1.2 waves): a uniform 2-way split costs +0.35 ms over 32 launches, because the split
  // shares are uniform while the causal KV lengths are not and the extra partial write + merge
  // outweigh the shorter critical path.
  static const int forced = [] {
    const char* e = getenv("RC_ATTN_SPLITS");  // diagnostics: force a split count (1 = off)
    return e ? atoi(e) : 0;
  }();
  if (forced >= 1 && forced <= 8) return forced;
  const int64_t units = static_cast<int64_t>(n_tiles) * n_kv_heads;
  int best = 1;
  while (best < 8 && units * (best * 2) <= num_sms && est_kv_tiles / (best * 2) >= 4) best *= 2;
  // (an adaptive split of only the long tiles -- RC_ATTN_ADAPTIVE -- was measured at cfg3 batch 1:
  // 2.16 vs 2.03 ms per step, because the doubled grid runs in two full waves; not chosen here)
  return best;
}

}  // namespace rc
