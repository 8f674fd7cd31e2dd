// NEXT-1: the attention-mass term ||A_i||_1 of Eq. 3, read as
// the column mass of the check-layer softmax over fresh keys (R2) in the floor(P * 2^24) fixed
// point (R2-FX), and its combination with the deviation D into the selection score.
//
// Two passes. Pass 1 is the check-layer attention of every U query over the fresh keys (prefix
// cache + K_new of U), run by k_attn_tc with lse_out set: each query row's log2-sum-exp. Pass 2
// (here) turns the problem around: a CTA owns one 128-key tile of one request and one kv head,
// streams that request's query tiles whose positions reach the key tile, and recomputes on
// tcgen05 S^T = K Q^T (M = 128 keys, N = 128 query rows = TQ tokens x G heads, TMEM accumulator,
// double-buffered). A thread owns one key row, so the column sum is a private sum:
//   acc += floor(2^(s * scale_log2 - lse_q + 24))   for every visible query q (pos_q >= pos_key),
// per tile in 32 bits (<= 128 * 2^24), then 64 bits; one 64-bit atomic per key and kv head.
//   warp 0 lane 0  TMA: the K tile once, query tiles through a 2-stage ring (3-D boxes [TQ][G][64])
//   warp 1 lane 0  MMA issuer;  warp 2: TMEM allocator;  warps 4-7: key rows (TMEM lanes 0..127)
// U rows are the non-prefix positions in order (U row u_off + i <-> position P + i), so query
// positions follow from the row index.
#include "common.cuh"
#include "rc_internal.h"

namespace rc {
namespace {

constexpr int DH = 128, ROWS = 128;
constexpr uint32_t HALF = ROWS * 64 * 2;  // [128 rows][64 bf16] SW128 sub-tile
constexpr uint32_t TILE = 2 * HALF;
constexpr int QST = 2;
constexpr uint32_t OFF_K = 0, OFF_Q = TILE, OFF_LSE = OFF_Q + QST * TILE;  // lse/pos: [2][128] f32 + [2][128] i32
constexpr uint32_t OFF_BAR = OFF_LSE + 2 * 128 * 8;
constexpr uint32_t SMEM_BYTES = OFF_BAR + 128;

__global__ void __launch_bounds__(256, 1)
    k_attn_mass(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK, const MassArgs a,
                int64_t t_cap) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  uint8_t* sK = smem + OFF_K;
  uint8_t* sQ = smem + OFF_Q;
  float* s_lse = reinterpret_cast<float*>(smem + OFF_LSE);            // [2][128]
  int32_t* s_pos = reinterpret_cast<int32_t*>(smem + OFF_LSE + 1024);  // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* k_full = bars;              // [1]
  uint64_t* q_full = bars + 1;          // [QST]
  uint64_t* q_empty = q_full + QST;     // [QST]
  uint64_t* s_full = q_empty + QST;     // [2]
  uint64_t* s_empty = s_full + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(k_full, 1);
    for (int i = 0; i < QST; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 4); }
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();
  griddep_launch();

  const int4 kt = a.key_tiles[blockIdx.x];  // {request, first key position, keys in tile, 0}
  const int4 rq = a.req[kt.x];              // {u_off, u_cnt, P, arena_row}
  const int kvh = blockIdx.y;
  const int G = a.n_heads / a.n_kv_heads, TQ = ROWS / G, H = a.n_heads;
  const int k0 = kt.y;
  // query tiles of this request that reach the key tile: tile i holds positions P + i TQ ..
  const int n_qt = (rq.y + TQ - 1) / TQ;
  const int i0 = max(0, (k0 - rq.z) / TQ);
  const int nt = max(0, n_qt - i0);

  if (warp == 0) {
    if (lane == 0 && nt > 0) {
      tma_prefetch_desc(&tmQ); tma_prefetch_desc(&tmK);
      mbar_expect_tx(k_full, TILE);
      const int krow = static_cast<int>(kvh * t_cap + rq.w + k0);
      tma_load_2d(sK, &tmK, k_full, 0, krow);
      tma_load_2d(sK + HALF, &tmK, k_full, 64, krow);
      for (int j = 0; j < nt; ++j) {
        const int s = j % QST;
        mbar_wait(&q_empty[s], ((j / QST) & 1) ^ 1);
        mbar_expect_tx(&q_full[s], 2u * 128u * G * TQ);
        const int r0 = rq.x + (i0 + j) * TQ;
        tma_load_3d(sQ + s * TILE, &tmQ, &q_full[s], 0, kvh * G, r0);
        tma_load_3d(sQ + s * TILE + HALF, &tmQ, &q_full[s], 64, kvh * G, r0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nt > 0) {
      constexpr uint32_t idS = idesc_bf16_f32(128, 128);
      mbar_wait(k_full, 0);
      tc_fence_after();
      for (int j = 0; j < nt; ++j) {
        const int s = j % QST, b = j & 1;
        mbar_wait(&q_full[s], (j / QST) & 1);
        mbar_wait(&s_empty[b], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          const uint64_t ad = sdesc_sw128(smem_u32(sK + (k >> 2) * HALF)) + 2 * (k & 3);
          const uint64_t bd = sdesc_sw128(smem_u32(sQ + s * TILE + (k >> 2) * HALF)) + 2 * (k & 3);
          umma_bf16(tmem + b * 128, ad, bd, idS, k > 0);
        }
        umma_commit(&q_empty[s]);
        umma_commit(&s_full[b]);
      }
    }
  } else if (warp >= 4) {
    const int kr = (warp - 4) * 32 + lane;  // key row <-> TMEM lane
    const int key_pos = k0 + kr;
    const bool key_ok = kr < kt.z && key_pos >= rq.z;  // U keys only
    const uint32_t lane_base = static_cast<uint32_t>((warp - 4) * 32) << 16;
    unsigned long long acc = 0;
    for (int j = 0; j < nt; ++j) {
      const int b = j & 1;
      const int i = i0 + j;
      {  // this tile's query rows: row r = t G + g (token t, head g)
        const int t = kr / G, g = kr % G;
        const int u = i * TQ + t;  // U index within the request
        const bool ok = kr < TQ * G && u < rq.y;
        s_pos[b * 128 + kr] = ok ? rq.z + u : -1;
        s_lse[b * 128 + kr] = ok ? 24.f - a.lse[static_cast<int64_t>(rq.x + u) * H + kvh * G + g] : -INFINITY;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      mbar_wait(&s_full[b], (j >> 1) & 1);
      tc_fence_after();
      uint32_t part = 0;
#pragma unroll 1
      for (int c0 = 0; c0 < ROWS; c0 += 32) {
        uint32_t sv[32];
        tmem_ld32(tmem + lane_base + b * 128 + c0, sv);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float x = fmaf(__uint_as_float(sv[c]), a.scale_log2, s_lse[b * 128 + c0 + c]);
          const uint32_t e = __float2uint_rz(fast_exp2(x));
          part += s_pos[b * 128 + c0 + c] >= key_pos ? e : 0u;  // causal; padded rows carry pos -1
        }
      }
      acc += part;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[b]);
    }
    if (key_ok && acc) atomicAdd(a.mass + rq.x + (key_pos - rq.z), acc);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 256);
}

// S = rint((1 - lambda) A + lambda D) in IEEE fp64 (no contraction), written over D (R2-FX)
__global__ void k_mass_combine(unsigned long long* __restrict__ dev, const unsigned long long* __restrict__ mass,
                               int32_t n, double lam) {
  griddep_wait();
  griddep_launch();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double wa = __dsub_rn(1.0, lam);
  const double s = __dadd_rn(__dmul_rn(wa, static_cast<double>(mass[i])), __dmul_rn(lam, static_cast<double>(dev[i])));
  dev[i] = static_cast<unsigned long long>(rint(s));
}
}  // namespace

cudaError_t attn_mass_launch(const CUtensorMap* tmQ, const CUtensorMap* tmK, const MassArgs& a, int64_t t_cap,
                             cudaStream_t s) {
  if (a.n_key_tiles <= 0) return cudaSuccess;
  if (cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(k_attn_mass), SMEM_BYTES); e != cudaSuccess) return e;
  return launch_pdl(k_attn_mass, dim3(a.n_key_tiles, a.n_kv_heads), dim3(256), SMEM_BYTES, s, *tmQ, *tmK, a, t_cap);
}

cudaError_t mass_combine_launch(unsigned long long* dev, const unsigned long long* mass, int32_t n, double lam,
                                cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(k_mass_combine, dim3((n + 255) / 256), dim3(256), 0, s, dev, mass, n, lam);
}

}  // namespace rc
