// K4/K7 on tcgen05, paired query tiles (d_h = 128): causal attention of query tokens over their
// request's stitched KV (Eq. 1; R11). Used for large grids
// (batch 32: thousands of tiles), where the single-tile kernel (k_attn_tc.cu) is bound by the L2->SM
// stream of K/V tiles: every K/V tile is fetched once per 128 query rows.
//
// Work item = (two query tiles of ONE request, kv head): Q_0, Q_1 stay in shared memory and every
// K/V tile is loaded once for both, halving the K/V bytes per FLOP. Persistent CTAs (one per SM)
// take items from a global counter. Tile t <-> TMEM S_t (columns 128 t) and O_t (columns 256 + 128 t);
// row r of a tile <-> TMEM lane r.
//   warp 0 lane 0   scheduler (publishes each item to the other roles) + TMA: Q_0, Q_1 per item (3-D
//                   boxes [TQ][G][64] x 2 halves), K tiles (2-stage ring running across items)
//   warp 3 lane 0   TMA: V tiles (2-stage ring)
//   warp 1 lane 0   MMA, ping-pong over the two tiles: after softmax t has turned S_t(j) into P_t(j)
//                   it issues O_t += P_t(j) V_j (TS mode, A = P from TMEM) and immediately
//                   S_t(j+1) = Q_t K_{j+1}^T, so the tensor pipe works on one tile while the other
//                   tile's softmax runs. In-order execution of one thread's MMAs makes the reuse of
//                   S_t's columns safe, and the commit of S_t(j+1) also covers PV_t(j).
//   warps 4-7 / 8-11  softmax of tile 0 / tile 1: thread <-> query row; each 128-key tile in two
//                   64-key halves (tcgen05.ld of the half, causal mask by true position unless the
//                   whole tile is visible, lazy rescale when the running max grows by > 2^8, P in
//                   bf16 pairs written back over the S columns already consumed). If the second
//                   half raises the running max, the first half's stored P is rescaled in TMEM (rare).
// Tiles: a.tiles holds 2 consecutive entries per work item, both of the same request (the host pads a
// request's odd tile count with an empty tile {row, 0, kv_base, 0}).
#include "common.cuh"
#include "rc_internal.h"

namespace rc {
namespace {

constexpr int DH = 128, BKV = 128, ROWS = 128;
constexpr uint32_t HALF = ROWS * 64 * 2;  // one [128 rows][64 bf16] SW128 sub-tile = 16 KB
constexpr uint32_t TILE = 2 * HALF;       // 32 KB
constexpr int NTHREADS = 128 + 256;       // 4 control warps + 2 x 4 softmax warps
constexpr int KST = 2, VST = 2;
constexpr uint32_t OFF_Q = 0, OFF_K = 2 * TILE, OFF_V = OFF_K + KST * TILE, OFF_BAR = OFF_V + VST * TILE;
constexpr uint32_t OFF_ITEM = OFF_BAR + 256;  // [2] work-item slots (scheduler -> roles)
// KV-chunked launches: per-CTA schedule table (pairs ranked by chunk length, first item of each rank,
// KV tiles per pair, chunks per pair, chunk length) and the two tiles' "this CTA merges" flags
constexpr int MAXP = ATTN_CHUNK_MAX_PAIRS;
constexpr uint32_t OFF_SCHED = OFF_ITEM + 16;
constexpr uint32_t SCHED_INTS = MAXP + (MAXP + 1) + MAXP + MAXP + 1 + 2;
constexpr uint32_t SMEM_BYTES = OFF_SCHED + ((SCHED_INTS * 4 + 15) & ~15u);
constexpr uint32_t O_COL = 256;            // O_t at 256 + 128 t
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 domain
// 2 of 8 key chunks take 2^x on the FMA pipe: measured at cfg3 batch 32, 39.4 ms per step vs 40.3
// (3 of 8), 42.8 (4 of 8), 40.5 (none)
constexpr unsigned POLY_CHUNKS = 0x44;
constexpr float SPEC_SUM_MAX = 18446744073709551616.0f;  // 2^64: bound of the speculative exps' row sum
constexpr int N_ITEM_CONSUMERS = 2 + 8;    // MMA thread, V producer, 8 softmax warps
// Phase timing (diagnostics build only: -DRC_ATTN_PROF, env RC_ATTN_PROF=1 at run time): clock64 sums
// per role and phase, added to a.prof at the end -- [0] softmax waits for S, [1] TMEM load of S,
// [2] exp/pack, [3] P store + fence + arrival, [4] item epilogue, [5] MMA waits for P, [6] MMA waits for
// K/V, [7] MMA thread total, [8] softmax total
#ifdef RC_ATTN_PROF
#define PROF_NOW(v) const long long v = clock64()
#define PROF_ADD(i, d) (prof_acc[i] += static_cast<unsigned long long>(d))
#else
#define PROF_NOW(v)
#define PROF_ADD(i, d)
#endif

// Persistent: grid <= #SMs, each CTA takes work items (tile pair, kv head) from a global counter,
// longest pairs first, so the next item's Q/K/V loads and first S MMAs overlap the previous item's
// last softmax steps and output epilogue (a fresh CTA per item re-paid the barrier/TMEM setup and the
// Q load latency with the tensor pipe idle). Warp 0 lane 0 fetches the item and publishes it in a
// 2-slot ring (it_full / it_empty); all role loops then follow the same item sequence, and every
// barrier phase is tracked by counters that run across items. O_t is reused across items: the
// first PV of tile t in an item waits until the previous item's epilogue has read O_t (o_free).
__global__ void __launch_bounds__(NTHREADS, 1)
    k_attn_pair(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnArgs a, int64_t t_cap) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  uint8_t* sQ = smem + OFF_Q;
  uint8_t* sK = smem + OFF_K;
  uint8_t* sV = smem + OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* q_full = bars;           // [1]
  uint64_t* q_empty = q_full + 1;    // [1] every MMA of the item reading Q complete
  uint64_t* k_full = q_empty + 1;    // [KST]
  uint64_t* k_empty = k_full + KST;  // [KST]
  uint64_t* v_full = k_empty + KST;  // [VST]
  uint64_t* v_empty = v_full + VST;  // [VST]
  uint64_t* s_full = v_empty + VST;  // [2 tiles]
  uint64_t* p_full = s_full + 2;     // [2 tiles]
  uint64_t* o_done = p_full + 2;     // [2 tiles] last PV of the tile complete
  uint64_t* o_free = o_done + 2;     // [2 tiles] epilogue has read O_t
  uint64_t* it_full = o_free + 2;    // [2] item slot written
  uint64_t* it_empty = it_full + 2;  // [2] item slot read by every role
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(it_empty + 2);
  volatile int32_t* item_slot = reinterpret_cast<volatile int32_t*>(smem + OFF_ITEM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < KST; ++i) { mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1); }
    for (int i = 0; i < VST; ++i) { mbar_init(&v_full[i], a.vsrc.vmap ? 32 : 1); mbar_init(&v_empty[i], 1); }
    // p_full / o_free: one arrival per softmax warp of the tile (lane 0 after __syncwarp)
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1); mbar_init(&p_full[t], 4); mbar_init(&o_done[t], 1); mbar_init(&o_free[t], 4);
    }
    for (int i = 0; i < 2; ++i) { mbar_init(&it_full[i], 1); mbar_init(&it_empty[i], N_ITEM_CONSUMERS); }
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // PDL: the prologue above overlapped the previous kernel's tail
  griddep_launch();

  const int G = a.n_heads / a.n_kv_heads;
  const int TQ = ROWS / G;
  const int H = a.n_heads;
  const int n_pairs = a.n_tiles / 2;
  const int n_items = n_pairs * a.n_kv_heads;
  // item w: kv head w % Hk of pair n_pairs - 1 - w / Hk (a request's pairs are in position order, so
  // the longest causal pairs come first)
  // an item covers the KV tiles [c0, c0 + nkv) of its pair; nk[t] of them (from c0) are tile t's,
  // whose causal range ends at its last row's position. nch[t] > 1: tile t's range is cut into nch[t]
  // chunks and this item's output is the partial of chunk ch
  struct Item { int4 tl[2]; int nk[2]; int nch[2]; int nkv, kv_base, kvh, c0, pr, ch; };
  const bool chunked = a.chunk_per_cta > 0.f;
  int* s_order = reinterpret_cast<int*>(smem + OFF_SCHED);  // [MAXP] pair of rank r
  int* s_start = s_order + MAXP;                           // [MAXP + 1] first item of rank r
  int* s_nkv = s_start + MAXP + 1;                         // [MAXP] KV tiles of pair p
  int* s_nch = s_nkv + MAXP;                               // [MAXP] chunks of pair p
  int* s_len = s_nch + MAXP;                               // [1] chunk length
  volatile int* s_merge = s_len + 1;                       // [2] tile t: this CTA merges the partials
  auto tile_nk = [&](const int4& tl) { return tl.y > 0 ? a.qpos[tl.x + tl.y - 1] / BKV + 1 : 0; };  // rows sorted by position
  auto decode = [&](int w) {
    Item it;
    int pr;
    if (chunked) {
      int lo = 0, hi = n_pairs - 1;  // largest rank whose first item is <= w
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_start[mid] <= w) lo = mid; else hi = mid - 1;
      }
      pr = s_order[lo];
      const int local = w - s_start[lo];
      it.ch = local / a.n_kv_heads;
      it.kvh = local % a.n_kv_heads;
    } else {
      pr = n_pairs - 1 - w / a.n_kv_heads;
      it.kvh = w % a.n_kv_heads;
      it.ch = 0;
    }
    it.pr = pr;
    int nkt[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      it.tl[t] = a.tiles[2 * pr + t];
      nkt[t] = tile_nk(it.tl[t]);
    }
    const int nkvp = max(nkt[0], nkt[1]);
    const int nch = chunked ? s_nch[pr] : 1;
    it.c0 = it.ch * nkvp / nch;
    const int c1 = (it.ch + 1) * nkvp / nch;
    it.nkv = c1 - it.c0;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      it.nk[t] = max(0, min(c1, nkt[t]) - it.c0);
      int n = 0;  // chunks that reach into tile t's range
      for (int c = 0; c < nch; ++c) n += (c * nkvp / nch < nkt[t]) ? 1 : 0;
      it.nch[t] = n;
    }
    it.kv_base = it.tl[0].z;
    return it;
  };
  auto tile_bar = [](int t) {  // the 4 softmax warps of tile t
    if (t == 0) asm volatile("bar.sync 2, 128;" ::: "memory");
    else asm volatile("bar.sync 3, 128;" ::: "memory");
  };
  if (chunked) {  // per-CTA schedule (identical in every CTA): pairs ranked by chunk length, longest first
    if (warp == 0) {
      int tot = 0;
      for (int p = lane; p < n_pairs; p += 32) {
        const int v = max(tile_nk(a.tiles[2 * p]), tile_nk(a.tiles[2 * p + 1]));
        s_nkv[p] = v;
        tot += v;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      const float target = static_cast<float>(tot) * a.n_kv_heads / (a.chunk_per_cta * gridDim.x);
      const int len = max(2, static_cast<int>(ceilf(target)));
      __syncwarp();
      for (int p = lane; p < n_pairs; p += 32) {
        const int v = s_nkv[p];
        s_nch[p] = v == 0 ? 0 : min(ATTN_MAX_CHUNKS, (v + len - 1) / len);
      }
      __syncwarp();
      for (int p = lane; p < n_pairs; p += 32) {  // rank: longer chunks first (v / nch), then higher pair
        const int v = s_nkv[p], n = s_nch[p];
        int rank = 0;
        for (int q2 = 0; q2 < n_pairs; ++q2) {
          const int vq = s_nkv[q2], nq = s_nch[q2];
          // compare vq / nq with v / n (empty pairs: length -1, last)
          const long long lq = nq ? static_cast<long long>(vq) * (n ? n : 1) : -1;
          const long long lp = n ? static_cast<long long>(v) * (nq ? nq : 1) : -1;
          rank += (lq > lp || (lq == lp && q2 > p)) ? 1 : 0;
        }
        s_order[rank] = p;
      }
      __syncwarp();
      if (lane == 0) {
        int acc = 0;
        for (int r = 0; r < n_pairs; ++r) { s_start[r] = acc; acc += s_nch[s_order[r]] * a.n_kv_heads; }
        s_start[n_pairs] = acc;
        *s_len = len;
      }
    }
    __syncthreads();
  }
  const int n_items_all = chunked ? s_start[n_pairs] : n_items;
  // consumers: item i of this CTA (-1 = no more work); the slot is released right after the read
  auto next_item = [&](int i, bool warp_wide) {
    mbar_wait(&it_full[i & 1], (i >> 1) & 1);
    const int w = item_slot[i & 1];
    if (warp_wide) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&it_empty[i & 1]);
    } else {
      mbar_arrive(&it_empty[i & 1]);
    }
    return w;
  };

  if (warp == 0) {
    if (lane == 0) {  // ---- scheduler + Q/K producer
      tma_prefetch_desc(&tmQ); tma_prefetch_desc(&tmK);
      int kc = 0;  // K tiles loaded so far (ring position / phase)
      for (int i = 0;; ++i) {
        if (i >= 2) mbar_wait(&it_empty[i & 1], ((i - 2) >> 1) & 1);
        int w = atomicAdd(a.work_ctr, 1);
        if (w >= n_items_all) w = -1;
        item_slot[i & 1] = w;
        mbar_arrive(&it_full[i & 1]);  // release: the slot write is visible to the waiters
        if (w < 0) break;
        const Item it = decode(w);
        if (i >= 1) mbar_wait(q_empty, (i - 1) & 1);  // the previous item's S MMAs have read Q
        mbar_expect_tx(q_full, ((it.nk[0] > 0 ? 1u : 0u) + (it.nk[1] > 0 ? 1u : 0u)) * 2u * 128u * G * TQ);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (it.nk[t] == 0) continue;
          tma_load_3d(sQ + t * TILE, &tmQ, q_full, 0, it.kvh * G, it.tl[t].x);
          tma_load_3d(sQ + t * TILE + HALF, &tmQ, q_full, 64, it.kvh * G, it.tl[t].x);
        }
        const int krow0 = static_cast<int>(it.kvh * t_cap + it.kv_base) + it.c0 * BKV;
        for (int j = 0; j < it.nkv; ++j, ++kc) {
          const int s = kc % KST;
          mbar_wait(&k_empty[s], ((kc / KST) & 1) ^ 1);
          mbar_expect_tx(&k_full[s], TILE);
          tma_load_2d(sK + s * TILE, &tmK, &k_full[s], 0, krow0 + j * BKV);
          tma_load_2d(sK + s * TILE + HALF, &tmK, &k_full[s], 64, krow0 + j * BKV);
        }
      }
    }
  } else if (warp == 3) {
    if (a.vsrc.vmap != nullptr) {  // ---- V producer, zero-copy (NEXT-4): rows through vmap, 4 per lane
      int vc = 0;
      for (int i = 0;; ++i) {
        const int w = next_item(i, true);
        if (w < 0) break;
        const Item it = decode(w);
        for (int j = 0; j < it.nkv; ++j, ++vc) {
          const int s = vc % VST;
          mbar_wait(&v_empty[s], ((vc / VST) & 1) ^ 1);
          v_rows_cp_async(sV + s * TILE, a.vsrc, a.v, a.head_stride,
                          static_cast<int64_t>(it.kv_base) + static_cast<int64_t>(it.c0 + j) * BKV, it.kvh, t_cap);
          cp_async_mbar_arrive(&v_full[s]);  // arrives when this lane's copies land (no wait here)
        }
      }
    } else if (lane == 0) {  // ---- V producer
      tma_prefetch_desc(&tmV);
      int vc = 0;
      for (int i = 0;; ++i) {
        const int w = next_item(i, false);
        if (w < 0) break;
        const Item it = decode(w);
        const int vrow0 = static_cast<int>(it.kvh * t_cap + it.kv_base) + it.c0 * BKV;
        for (int j = 0; j < it.nkv; ++j, ++vc) {
          const int s = vc % VST;
          mbar_wait(&v_empty[s], ((vc / VST) & 1) ^ 1);
          mbar_expect_tx(&v_full[s], TILE);
          tma_load_2d(sV + s * TILE, &tmV, &v_full[s], 0, vrow0 + j * BKV);
          tma_load_2d(sV + s * TILE + HALF, &tmV, &v_full[s], 64, vrow0 + j * BKV);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
#ifdef RC_ATTN_PROF
      unsigned long long prof_acc[9] = {};
      const long long t_start = clock64();
#endif
      constexpr uint32_t idS = idesc_bf16_f32(128, 128);
      constexpr uint32_t idPV = idesc_bf16_f32_bmn(128, 128);
      const bool no_mma = (a.debug_mode & 2) != 0;  // diagnostics: barriers only
      int kc = 0, vc = 0, pc[2] = {0, 0}, n_done[2] = {0, 0};
      auto wait_k = [&](int g) {
        mbar_wait(&k_full[g % KST], (g / KST) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int t, int g) {  // S_t = Q_t K_g^T (g = global K tile index)
        const int s = g % KST;
#pragma unroll
        for (int k = 0; k < (no_mma ? 0 : DH / 16); ++k) {
          const uint64_t ad = sdesc_sw128(smem_u32(sQ + t * TILE + (k >> 2) * HALF)) + 2 * (k & 3);
          const uint64_t bd = sdesc_sw128(smem_u32(sK + s * TILE + (k >> 2) * HALF)) + 2 * (k & 3);
          umma_bf16(tmem + t * 128, ad, bd, idS, k > 0);
        }
        umma_commit(&s_full[t]);
      };
      for (int i = 0;; ++i) {
        const int w = next_item(i, false);
        if (w < 0) break;
        const Item it = decode(w);
        mbar_wait(q_full, i & 1);
        tc_fence_after();
        wait_k(kc);
#pragma unroll
        for (int t = 0; t < 2; ++t)
          if (it.nk[t] > 0) issue_s(t, kc);
        umma_commit(&k_empty[kc % KST]);
        for (int j = 0; j < it.nkv; ++j) {
          const int v = (vc + j) % VST;
          PROF_NOW(tv0);
          mbar_wait(&v_full[v], ((vc + j) / VST) & 1);
          PROF_NOW(tv1);
          PROF_ADD(6, tv1 - tv0);
          if (a.vsrc.vmap) fence_proxy_async();  // zero-copy V: cp.async (generic proxy) writes -> MMA reads
          tc_fence_after();
          bool k_ready = false;
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (j >= it.nk[t]) continue;
            if (j == 0 && n_done[t] > 0) mbar_wait(&o_free[t], (n_done[t] - 1) & 1);  // O_t read out
            PROF_NOW(tp0);
            mbar_wait(&p_full[t], pc[t] & 1);
            PROF_NOW(tp1);
            PROF_ADD(5, tp1 - tp0);
            ++pc[t];
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < (no_mma ? 0 : BKV / 16); ++k) {  // 16 keys per MMA: A = P_t (8 TMEM columns), B = V rows
              const uint64_t bd = sdesc_sw128_mn(smem_u32(sV + v * TILE + k * 2048), HALF, 1024);
              umma_bf16_ts(tmem + O_COL + t * 128, tmem + t * 128 + k * 8, bd, idPV, (j > 0 || k > 0) ? 1u : 0u);
            }
            if (j + 1 == it.nk[t]) umma_commit(&o_done[t]);
            if (j + 1 < it.nk[t]) {
              if (!k_ready) { wait_k(kc + j + 1); k_ready = true; }
              issue_s(t, kc + j + 1);
            }
          }
          umma_commit(&v_empty[v]);
          if (j + 1 < it.nkv) {
            if (!k_ready) wait_k(kc + j + 1);  // a K tile only the other (finished) tile would have used
            umma_commit(&k_empty[(kc + j + 1) % KST]);
          }
        }
        umma_commit(q_empty);
        kc += it.nkv;
#ifdef RC_ATTN_PROF
        prof_acc[7] = clock64() - t_start;
#endif
        vc += it.nkv;
#pragma unroll
        for (int t = 0; t < 2; ++t) n_done[t] += it.nk[t] > 0 ? 1 : 0;
      }
#ifdef RC_ATTN_PROF
      if (a.prof) for (int i = 5; i < 8; ++i) atomicAdd(a.prof + i, prof_acc[i]);
#endif
    }
  } else if (warp >= 4) {  // ---- softmax: tile t, thread <-> row
#ifdef RC_ATTN_PROF
    unsigned long long prof_acc[9] = {};
    const long long t_start = clock64();
#endif
    const int t = (warp - 4) >> 2;
    const int q = warp & 3;  // TMEM lane quarter of this warp
    const int r = q * 32 + lane;
    const int tt = r / G, g = r % G;
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t s_col = tmem + lane_base + t * 128;
    int sc = 0, od = 0;  // S_t commits consumed, items with tile t non-empty
    for (int i = 0;; ++i) {
      const int w = next_item(i, true);
      if (w < 0) break;
      const Item it = decode(w);
      const int n_t = it.nk[t];
      if (n_t == 0) continue;
      const int row_start = it.tl[t].x;
      const int n_rows = it.tl[t].y;
      const bool valid = (r < TQ * G) && (tt < n_rows);
      const int p = valid ? a.qpos[row_start + tt] : -1;
      const int p_first = a.qpos[row_start];  // smallest position of the tile
      // padding rows see no key: base 0 keeps them off the max-first path (their P is 0, l stays 0)
      float m_run = valid ? -INFINITY : 0.f, l_run = 0.f;
      for (int j = 0; j < n_t; ++j, ++sc) {
        PROF_NOW(tw0);
        mbar_wait(&s_full[t], sc & 1);
        tc_fence_after();
        PROF_NOW(tw1);
        PROF_ADD(0, tw1 - tw0);
        if (a.debug_mode & 1) {  // diagnostics: no softmax work
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[t]);
          continue;
        }
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t sr[64];
          PROF_NOW(th0);
          tmem_ld32(s_col + hh * 64, sr);
          tmem_ld32(s_col + hh * 64 + 32, sr + 32);
          tmem_wait_ld();
          PROF_NOW(th1);
          PROF_ADD(1, th1 - th0);
          const int key0 = (it.c0 + j) * BKV + hh * 64;
          const bool full = key0 + 63 <= p_first;  // every row sees every key of the half: no causal mask
          uint32_t pk[32];
          // common case: exps against the running max, no row-max pass at all. Kept unless some row's sum
          // exceeds 2^64 (then some P > 2^64, or inf/NaN): the half is redone below with the max first.
          // Any P <= 2^64 keeps O and l finite over 8192 keys, and bf16/fp32 precision is relative.
          if ((a.debug_mode & 4) == 0 && !__any_sync(0xffffffffu, m_run == -INFINITY)) {
            const float ls = full ? sm_exp_pack64<false, POLY_CHUNKS>(sr, pk, key0, p, a.scale_log2, m_run)
                                  : sm_exp_pack64<true, POLY_CHUNKS>(sr, pk, key0, p, a.scale_log2, m_run);
            if (!__any_sync(0xffffffffu, !(ls <= SPEC_SUM_MAX))) {
              l_run += ls;
              tmem_st32(s_col + hh * 32, pk);
              PROF_NOW(th2);
              PROF_ADD(2, th2 - th1);
              continue;
            }
          }
          const float rmax = full ? sm_rowmax64<false>(sr, key0, p) : sm_rowmax64<true>(sr, key0, p);
          // raw scores; the softmax scale (> 0) is folded into the max and into one FFMA per exp2
          const float mx = rmax * a.scale_log2;
          float alpha = 1.f;
          bool need = false;
          if (mx > m_run + RESCALE_THRESHOLD || (m_run == -INFINITY && mx != -INFINITY)) {
            const float m_new = fmaxf(m_run, mx);
            if (m_run != -INFINITY) { alpha = fast_exp2(m_run - m_new); need = true; }
            m_run = m_new;
          }
          if (__any_sync(0xffffffffu, need)) {  // rare: rebase O_t (PVs up to j-1) and this tile's first-half P
            if (j > 0) {  // the commit of S_t(j) covered PV_t(j-1): O_t is complete up to j-1
              uint32_t o[32];
#pragma unroll 1
              for (int c = 0; c < DH; c += 32) {
                tmem_ld32(tmem + lane_base + O_COL + t * 128 + c, o);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                tmem_st32(tmem + lane_base + O_COL + t * 128 + c, o);
              }
            }
            if (hh == 1) {
              uint32_t pp[32];
              tmem_wait_st();
              tmem_ld32(s_col, pp);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i)
                pp[i] = pack_bf2(__uint_as_float(pp[i] << 16) * alpha, __uint_as_float(pp[i] & 0xFFFF0000u) * alpha);
              tmem_st32(s_col, pp);
            }
            tmem_wait_st();
          }
          l_run *= alpha;
          const float base = (m_run == -INFINITY) ? 0.f : m_run;
          l_run += full ? sm_exp_pack64<false, POLY_CHUNKS>(sr, pk, key0, p, a.scale_log2, base)
                        : sm_exp_pack64<true, POLY_CHUNKS>(sr, pk, key0, p, a.scale_log2, base);
          tmem_st32(s_col + hh * 32, pk);  // P of keys [64 hh, 64 hh + 64) -> columns [32 hh, 32 hh + 32)
        }
        PROF_NOW(ts0);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
        PROF_NOW(ts1);
        PROF_ADD(3, ts1 - ts0);
      }
      PROF_NOW(te0);
      mbar_wait(&o_done[t], od & 1);
      ++od;
      tc_fence_after();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      uint16_t* dst = a.o + static_cast<int64_t>(row_start + tt) * H * DH + (it.kvh * G + g) * DH;
      const bool part = it.nch[t] > 1;  // KV-chunked tile: fp32 partial (O / l, m, l) of chunk it.ch
      const int64_t slot0 = (static_cast<int64_t>(2 * it.pr + t) * a.n_kv_heads + it.kvh) * ATTN_MAX_CHUNKS;
      float* pdst = part ? a.part_o + ((slot0 + it.ch) * ROWS + r) * DH : nullptr;
      if (part) {
        a.part_ml[((slot0 + it.ch) * ROWS + r) * 2] = m_run;
        a.part_ml[((slot0 + it.ch) * ROWS + r) * 2 + 1] = l_run;
      }
#pragma unroll 1
      for (int c = 0; c < DH; c += 32) {
        uint32_t o[32];
        tmem_ld32(tmem + lane_base + O_COL + t * 128 + c, o);
        tmem_wait_ld();
        if (c + 32 == DH) {  // O_t fully read: the next item's first PV may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&o_free[t]);
        }
        if (part) {
#pragma unroll
          for (int i2 = 0; i2 < 32; i2 += 4)
            *reinterpret_cast<float4*>(pdst + c + i2) =
                make_float4(__uint_as_float(o[i2]) * inv, __uint_as_float(o[i2 + 1]) * inv,
                            __uint_as_float(o[i2 + 2]) * inv, __uint_as_float(o[i2 + 3]) * inv);
        } else if (valid) {
#pragma unroll
          for (int i2 = 0; i2 < 32; i2 += 8) {
            uint4 u;
            u.x = pack_bf2(__uint_as_float(o[i2 + 0]) * inv, __uint_as_float(o[i2 + 1]) * inv);
            u.y = pack_bf2(__uint_as_float(o[i2 + 2]) * inv, __uint_as_float(o[i2 + 3]) * inv);
            u.z = pack_bf2(__uint_as_float(o[i2 + 4]) * inv, __uint_as_float(o[i2 + 5]) * inv);
            u.w = pack_bf2(__uint_as_float(o[i2 + 6]) * inv, __uint_as_float(o[i2 + 7]) * inv);
            *reinterpret_cast<uint4*>(dst + c + i2) = u;
          }
        }
      }
      if (part) {  // arrival count per (tile, kv head); the chunk that arrives last merges and resets it
        __threadfence();
        tile_bar(t);
        if (q == 0 && lane == 0) {
          int* ctr = a.split_flag + (2 * it.pr + t) * a.n_kv_heads + it.kvh;
          const bool last = atomicAdd(ctr, 1) == it.nch[t] - 1;
          if (last) *ctr = 0;
          s_merge[t] = last ? 1 : 0;
        }
        tile_bar(t);
        if (s_merge[t] && valid) {
          __threadfence();
          float mm = -INFINITY;
          for (int c2 = 0; c2 < it.nch[t]; ++c2) {
            const float2 v = __ldcg(reinterpret_cast<const float2*>(a.part_ml + ((slot0 + c2) * ROWS + r) * 2));
            if (v.y > 0.f) mm = fmaxf(mm, v.x);
          }
          float wts[ATTN_MAX_CHUNKS], wsum = 0.f;
#pragma unroll
          for (int c2 = 0; c2 < ATTN_MAX_CHUNKS; ++c2) {
            wts[c2] = 0.f;
            if (c2 >= it.nch[t]) continue;
            const float2 v = __ldcg(reinterpret_cast<const float2*>(a.part_ml + ((slot0 + c2) * ROWS + r) * 2));
            if (v.y > 0.f) wts[c2] = v.y * fast_exp2(v.x - mm);
            wsum += wts[c2];
          }
          const float inv2 = wsum > 0.f ? 1.f / wsum : 0.f;
#pragma unroll 1
          for (int c = 0; c < DH; c += 8) {
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int c2 = 0; c2 < ATTN_MAX_CHUNKS; ++c2) {
              if (wts[c2] == 0.f) continue;
              const float4* src = reinterpret_cast<const float4*>(a.part_o + ((slot0 + c2) * ROWS + r) * DH + c);
              const float4 x0 = __ldcg(src), x1 = __ldcg(src + 1);
              acc[0] += wts[c2] * x0.x; acc[1] += wts[c2] * x0.y; acc[2] += wts[c2] * x0.z; acc[3] += wts[c2] * x0.w;
              acc[4] += wts[c2] * x1.x; acc[5] += wts[c2] * x1.y; acc[6] += wts[c2] * x1.z; acc[7] += wts[c2] * x1.w;
            }
            uint4 u;
            u.x = pack_bf2(acc[0] * inv2, acc[1] * inv2); u.y = pack_bf2(acc[2] * inv2, acc[3] * inv2);
            u.z = pack_bf2(acc[4] * inv2, acc[5] * inv2); u.w = pack_bf2(acc[6] * inv2, acc[7] * inv2);
            *reinterpret_cast<uint4*>(dst + c) = u;
          }
        }
      }
      PROF_NOW(te1);
      PROF_ADD(4, te1 - te0);
    }
#ifdef RC_ATTN_PROF
    prof_acc[8] = clock64() - t_start;
    if (lane == 0 && a.prof)
      for (int i = 0; i < 9; ++i) if (i != 5 && i != 6 && i != 7) atomicAdd(a.prof + i, prof_acc[i]);
#endif
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
  if (threadIdx.x == 0) {  // the last CTA to finish resets the work counter for the next launch
    __threadfence();
    if (atomicAdd(a.work_ctr + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      a.work_ctr[0] = 0;
      a.work_ctr[1] = 0;
      __threadfence();
    }
  }
}
}  // namespace

cudaError_t attn_pair_launch(const CUtensorMap* tmQ, const CUtensorMap* tmK, const CUtensorMap* tmV,
                             const AttnArgs& a, int64_t t_cap, cudaStream_t s) {
  if (a.n_tiles <= 0) return cudaSuccess;
  if (a.n_tiles % 2 != 0 || a.head_dim != DH || a.n_splits != 1) return cudaErrorInvalidValue;
  const bool chunked = a.chunk_per_cta > 0.f;
  if (chunked && (a.n_tiles / 2 > ATTN_CHUNK_MAX_PAIRS || !a.part_o || !a.part_ml || !a.split_flag))
    return cudaErrorInvalidValue;
  if (cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(k_attn_pair), SMEM_BYTES); e != cudaSuccess) return e;
  if (a.work_ctr == nullptr) return cudaErrorInvalidValue;
  static const int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  static const bool persist = [] {
    const char* e = getenv("RC_ATTN_PERSIST");  // diagnostics: 0 = one CTA per work item
    return !(e && atoi(e) == 0);
  }();
  const int items = a.n_tiles / 2 * a.n_kv_heads;
  // chunked: the item count is known on the device only (it follows the tiles' causal lengths)
  const int grid = chunked ? sms : persist ? (items < sms ? items : sms) : items;
  return launch_pdl(k_attn_pair, dim3(grid), dim3(NTHREADS), SMEM_BYTES, s, *tmQ, *tmK, *tmV, a, t_cap);
}

bool attn_chunk_auto() {
  static const bool on = [] {
    const char* e = getenv("RC_ATTN_CHUNK_AUTO");  // 1 = AUTO takes the chunked launch for small grids
    return e && atoi(e) == 1;
  }();
  return on;
}

float attn_chunk_per_cta() {
  static const float f = [] {
    const char* e = getenv("RC_ATTN_CHUNK_F");  // diagnostics: items per CTA the chunk length aims at
    const float v = e ? static_cast<float>(atof(e)) : 2.0f;
    return v > 0.f ? v : 2.0f;
  }();
  return f;
}

bool attn_use_pairs(int n_tiles, int n_kv_heads, int num_sms) {
  static const int forced = [] {
    const char* e = getenv("RC_ATTN_PAIRS");  // diagnostics: 0 = never, 1 = always
    return e ? atoi(e) : -1;
  }();
  if (forced == 0 || forced == 1) return forced == 1;
  // pairs halve the CTA count: only when at least 4 waves of paired CTAs remain
  return static_cast<int64_t>(n_tiles) * n_kv_heads >= static_cast<int64_t>(8) * num_sms;
}

}  // namespace rc
