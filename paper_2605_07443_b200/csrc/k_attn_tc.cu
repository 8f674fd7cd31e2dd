// K4/K7 on tcgen05 (d_h = 128): causal attention of query tokens over their request's stitched
// KV, S and O accumulated in TMEM (Eq. 1; R11).
//
// CTA = (query tile, kv head). Tile = TQ tokens x G grouped query heads = 128 rows (G = 4: 32
// tokens; G = 7: 18 tokens = 126 rows); row r <-> TMEM lane r. KV streamed in 128-key tiles.
//   warp 0 lane 0   TMA: Q once (3-D box [TQ][G][64] x 2 halves), K tiles (2-stage ring)
//   warp 3 lane 0   TMA: V tiles (2-stage ring)
//   warp 1 lane 0   MMA: S_j = Q K_j^T (M=128, N=128, K=128; A, B K-major SW128) into TMEM S[j%2];
//                        O += P_j V_j (A = P from smem, K-major; B = V MN-major SW128) into TMEM O
//   warps 4..7      softmax: thread = row; tcgen05.ld S row, causal mask by true position,
//                   online max with lazy O rescale (only when the max grows by > 2^8, done on the
//                   TMEM accumulator with tcgen05.ld/st), P = exp2(s - m) -> bf16 -> swizzled smem
// Issue order S_0, S_1, PV_0, S_2, PV_1, ... so softmax of tile j+1 overlaps PV_j.
#include "common.cuh"
#include "rc_internal.h"

namespace rc {
namespace {

constexpr int DH = 128, BKV = 128, ROWS = 128;
constexpr uint32_t HALF = ROWS * 64 * 2;  // one [128 rows][64 bf16] SW128 sub-tile = 16 KB
constexpr uint32_t TILE = 2 * HALF;       // 32 KB
constexpr uint32_t OFF_Q = 0, OFF_K = TILE, OFF_V = 3 * TILE, OFF_P = 5 * TILE, OFF_BAR = 7 * TILE;
constexpr uint32_t OFF_RED = OFF_BAR + 256;            // [2 tile slots][2 column halves][128 rows] f32
constexpr uint32_t SMEM_BYTES = OFF_RED + 2 * 2 * 128 * 4;
constexpr int SCOLS = BKV / 2;                          // S columns per softmax thread (two warps per row)
constexpr int NTHREADS = 384;                           // 4 control warps + 8 softmax warps
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 domain

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(NTHREADS, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, const AttnArgs a, int64_t t_cap) {
  // 224 KB of tiles + barriers + exchange: no room for a manual 1 KB alignment pad, so the
  // dynamic window must itself be 1024-aligned (SWIZZLE_128B atoms); checked below.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  uint8_t* sQ = smem + OFF_Q;
  float* red = reinterpret_cast<float*>(smem + OFF_RED);
  uint8_t* sK = smem + OFF_K;
  uint8_t* sV = smem + OFF_V;
  uint8_t* sP = smem + OFF_P;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;
  uint64_t* v_empty = bars + 7;
  uint64_t* s_full = bars + 9;
  uint64_t* p_full = bars + 11;
  uint64_t* pv_done = bars + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int4 tile = a.tiles[blockIdx.x];
  const int row_start = tile.x, n_rows = tile.y, kv_base = tile.z;
  const int kvh = blockIdx.y;
  const int G = a.n_heads / a.n_kv_heads;
  const int TQ = ROWS / G;
  const int H = a.n_heads;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int max_pos = a.qpos[row_start + n_rows - 1];
  const int nkv = max_pos / BKV + 1;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1); mbar_init(&p_full[i], 256); mbar_init(&pv_done[i], 1);
    }
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S0 at +0, S1 at +128, O at +256

  if (warp == 0) {
    if (lane == 0) {  // ---- Q + K producer
      tma_prefetch_desc(&tmQ); tma_prefetch_desc(&tmK);
      mbar_expect_tx(q_full, 2u * 128u * G * TQ);
      tma_load_3d(sQ, &tmQ, q_full, 0, kvh * G, row_start);
      tma_load_3d(sQ + HALF, &tmQ, q_full, 64, kvh * G, row_start);
      const int krow0 = static_cast<int>(kvh * t_cap + kv_base);
      for (int j = 0; j < nkv; ++j) {
        const int b = j & 1;
        mbar_wait(&k_empty[b], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&k_full[b], TILE);
        tma_load_2d(sK + b * TILE, &tmK, &k_full[b], 0, krow0 + j * BKV);
        tma_load_2d(sK + b * TILE + HALF, &tmK, &k_full[b], 64, krow0 + j * BKV);
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {  // ---- V producer
      tma_prefetch_desc(&tmV);
      const int vrow0 = static_cast<int>(kvh * t_cap + kv_base);
      for (int j = 0; j < nkv; ++j) {
        const int b = j & 1;
        mbar_wait(&v_empty[b], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&v_full[b], TILE);
        tma_load_2d(sV + b * TILE, &tmV, &v_full[b], 0, vrow0 + j * BKV);
        tma_load_2d(sV + b * TILE + HALF, &tmV, &v_full[b], 64, vrow0 + j * BKV);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idS = idesc_bf16_f32(128, 128);
      constexpr uint32_t idPV = idesc_bf16_f32_bmn(128, 128);
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto issue_s = [&](int j) {
        const int b = j & 1;
        mbar_wait(&k_full[b], (j >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          const uint64_t ad = sdesc_sw128(smem_u32(sQ + (k >> 2) * HALF)) + 2 * (k & 3);
          const uint64_t bd = sdesc_sw128(smem_u32(sK + b * TILE + (k >> 2) * HALF)) + 2 * (k & 3);
          umma_bf16(tmem + b * 128, ad, bd, idS, k > 0);
        }
        umma_commit(&k_empty[b]);
        umma_commit(&s_full[b]);
      };
      issue_s(0);
      if (nkv > 1) issue_s(1);
      for (int j = 0; j < nkv; ++j) {
        const int b = j & 1;
        mbar_wait(&p_full[b], (j >> 1) & 1);
        mbar_wait(&v_full[b], (j >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k) {
          const uint64_t ad = sdesc_sw128(smem_u32(sP + b * TILE + (k >> 2) * HALF)) + 2 * (k & 3);
          const uint64_t bd = sdesc_sw128_mn(smem_u32(sV + b * TILE + k * 2048), HALF, 1024);
          umma_bf16(tmem + 256, ad, bd, idPV, (j > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&v_empty[b]);
        umma_commit(&pv_done[b]);
        if (j + 2 < nkv) issue_s(j + 2);
      }
    }
  } else if (warp >= 4) {  // ---- softmax: thread <-> (row, half of the key columns)
    const int q = warp & 3;              // TMEM lane quarter of this warp
    const int hf = (warp - 4) >> 2;      // warps 4..7: keys 0..63 of a tile, warps 8..11: keys 64..127
    const int col0 = hf * SCOLS;
    const int r = q * 32 + lane;
    const int t = r / G, g = r % G;
    const bool valid = (r < TQ * G) && (t < n_rows);
    const int p = valid ? a.qpos[row_start + t] : -1;
    const int p_first = a.qpos[row_start];  // smallest position of the tile (rows sorted by position)
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    float m_run = -INFINITY, l_run = 0.f;
    uint32_t sr[SCOLS];
    for (int j = 0; j < nkv; ++j) {
      const int b = j & 1;
      mbar_wait(&s_full[b], (j >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < SCOLS; c += 32) tmem_ld32(tmem + lane_base + b * 128 + col0 + c, sr + c);
      tmem_wait_ld();
      const int key0 = j * BKV + col0;
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};  // 4 independent chains
      if (j * BKV + BKV - 1 <= p_first) {  // every row of the tile sees every key: no causal mask
#pragma unroll
        for (int c = 0; c < SCOLS; ++c) mx4[c & 3] = fmaxf(mx4[c & 3], __uint_as_float(sr[c]));
      } else {
#pragma unroll
        for (int c = 0; c < SCOLS; ++c) {
          const float v = (key0 + c <= p) ? __uint_as_float(sr[c]) : -INFINITY;
          sr[c] = __float_as_uint(v);
          mx4[c & 3] = fmaxf(mx4[c & 3], v);
        }
      }
      // scores stay raw; the softmax scale (> 0) is folded into the max and into one FFMA per exp2
      float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * a.scale_log2;
      // combine the two column halves of this row (warp pair q+4 / q+8, named barrier 1+q)
      red[(j & 1) * 256 + hf * 128 + r] = mx;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
      mx = fmaxf(mx, red[(j & 1) * 256 + (hf ^ 1) * 128 + r]);
      float alpha = 1.f;
      bool need = false;
      if (mx > m_run + RESCALE_THRESHOLD || (m_run == -INFINITY && mx != -INFINITY)) {
        const float m_new = fmaxf(m_run, mx);
        if (m_run != -INFINITY) { alpha = fast_exp2(m_run - m_new); need = true; }
        m_run = m_new;
      }
      if (j > 0 && __any_sync(0xffffffffu, need)) {  // rescale this warp's half of the TMEM accumulator rows
        mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
        uint32_t o[32];
#pragma unroll
        for (int c = 0; c < SCOLS; c += 32) {
          tmem_ld32(tmem + lane_base + 256 + col0 + c, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(tmem + lane_base + 256 + col0 + c, o);
        }
        tmem_wait_st();
      }
      l_run *= alpha;
      const float base = (m_run == -INFINITY) ? 0.f : m_run;
      if (j >= 2) mbar_wait(&pv_done[b], ((j - 2) >> 1) & 1);  // P buffer b free (PV_{j-2} done)
      uint8_t* prow = sP + b * TILE + hf * HALF + r * 128;     // this half = one 64-key K-block of P
      float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < SCOLS; c += 8) {
        float e[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          e[i] = fast_exp2(fmaf(__uint_as_float(sr[c + i]), a.scale_log2, -base));
          ls[i & 3] += e[i];
        }
        uint4 u;
        u.x = pack_bf2(e[0], e[1]); u.y = pack_bf2(e[2], e[3]); u.z = pack_bf2(e[4], e[5]); u.w = pack_bf2(e[6], e[7]);
        const int chunk = c >> 3;
        *reinterpret_cast<uint4*>(prow + ((chunk ^ (r & 7)) << 4)) = u;
      }
      l_run += (ls[0] + ls[1]) + (ls[2] + ls[3]);
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(&p_full[b]);
    }
    // epilogue: O / l -> bf16 (l = sum of the two halves' partial sums)
    // slot (nkv & 1) was last read before the final tile's barrier by both warps of the pair
    red[(nkv & 1) * 256 + hf * 128 + r] = l_run;
    asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
    const float l_tot = l_run + red[(nkv & 1) * 256 + (hf ^ 1) * 128 + r];
    mbar_wait(&pv_done[(nkv - 1) & 1], ((nkv - 1) >> 1) & 1);
    tc_fence_after();
    const float inv = l_tot > 0.f ? 1.f / l_tot : 0.f;
    uint16_t* dst = a.o + static_cast<int64_t>(row_start + t) * H * DH + (kvh * G + g) * DH + col0;
#pragma unroll
    for (int c = 0; c < SCOLS; c += 32) {
      uint32_t o[32];
      tmem_ld32(tmem + lane_base + 256 + col0 + c, o);
      tmem_wait_ld();
      if (valid) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 u;
          u.x = pack_bf2(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv);
          u.y = pack_bf2(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv);
          u.z = pack_bf2(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv);
          u.w = pack_bf2(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv);
          *reinterpret_cast<uint4*>(dst + c + i) = u;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}
}  // namespace

int attn_tc_tokens_per_tile(int group) { return ROWS / group; }

cudaError_t attn_tc_launch(const CUtensorMap* tmQ, const CUtensorMap* tmK, const CUtensorMap* tmV, const AttnArgs& a,
                           int64_t t_cap, cudaStream_t s) {
  if (a.n_tiles <= 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_attn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(a.n_tiles, a.n_kv_heads);
  k_attn_tc<<<grid, NTHREADS, SMEM_BYTES, s>>>(*tmQ, *tmK, *tmV, a, t_cap);
  return cudaGetLastError();
}

}  // namespace rc
