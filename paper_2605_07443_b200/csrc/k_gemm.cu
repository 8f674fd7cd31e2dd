// K3: persistent warp-specialised tcgen05 GEMM for every dense projection of the hot path,
// with the per-row work fused into its epilogue.
//
//   C[M][N] = A[M][K] * B[N][K]^T    (A = activations, B = weight rows; both bf16, K-major)
//
// Roles (256 threads, 1 CTA/SM, grid = min(tiles, #SM), static round-robin tile order):
//   warp 0      TMA producer: A 128x64 and B BNx64 boxes, SWIZZLE_128B, STAGES-deep mbarrier ring
//   warp 1      MMA issuer (one thread): tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16
//   warp 2      TMEM allocator (2 x BN fp32 columns = double-buffered accumulator)
//   warps 4..7  epilogue: tcgen05.ld 32x32b (thread <-> accumulator row), fused epilogue op
// The epilogue of tile i overlaps the MMAs of tile i+1 (two TMEM accumulator stages).
#include <mutex>

#include "common.cuh"
#include "rc_internal.h"

namespace rc {

namespace {
constexpr int BM = 128, BK = 64;
// raster: group_m m-tiles share a sweep over n; the host sizes the group by the bytes of its A rows
// (they must stay in L2 while the sweep streams B; B is re-read ceil(num_m / group_m) times).
constexpr size_t GROUP_A_BYTES = size_t(32) << 20;  // measured: gate/up at cfg3 b32 3.14 -> 3.07 ms, DRAM 3.1 -> 1.9 GB vs 16 MB

template <int BN>
struct GemmCfg {
  static constexpr int STAGES = (BN == 256) ? 4 : 6;
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  // residual epilogue staging: per epilogue warp 2 x [32 rows][32 fp32] SW128 boxes (TMA reduce-add)
  static constexpr uint32_t STAGE_OUT = 4 * 2 * 32 * 32 * 4;
  static constexpr uint32_t SMEM = STAGES * (A_BYTES + B_BYTES) + STAGE_OUT + 1024 + 256;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
};

__device__ __forceinline__ void tma_reduce_add_2d(const void* map, const void* smem_src, int c0, int c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Residual epilogue: x[rows][cols] += acc through TMA reduce-add (fp32, atomic per element, so split-K
// partial tiles simply add up). Each epilogue warp owns its 32 accumulator rows: tcgen05.ld 32 columns,
// write them as one swizzled [32][32] box to its staging buffer, and let one lane issue the bulk
// reduction; two buffers per warp keep a store in flight while the next chunk is loaded.
template <int BN>
__device__ __forceinline__ void epilogue_add_tma(uint32_t taddr, int m0, int n0, int N, int q, const void* tmC,
                                                 uint8_t* stage, int& chunk_ctr) {
  const int lane = threadIdx.x & 31;
  uint8_t* mybuf = stage + q * 2 * 4096;
  for (int c = 0; c < BN; c += 32) {
    if (n0 + c >= N) break;
    const int buf = chunk_ctr & 1;
    if (chunk_ctr >= 2) {
      if (lane == 0) bulk_wait_read<1>();  // the reduction that last read this buffer has drained it
      __syncwarp();
    }
    uint32_t v[32];
    tmem_ld32(taddr + c, v);
    tmem_wait_ld();
    uint8_t* row = mybuf + buf * 4096 + lane * 128;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      *reinterpret_cast<uint4*>(row + ((k ^ (lane & 7)) << 4)) = make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_reduce_add_2d(tmC, mybuf + buf * 4096, n0 + c, m0 + q * 32);
      bulk_commit();
    }
    ++chunk_ctr;
  }
}

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int group_m, int& mb, int& nb) {
  const int per_group = group_m * num_n;
  const int g = t / per_group;
  const int first_m = g * group_m;
  const int gm = min(group_m, num_m - first_m);
  const int r = t - g * per_group;
  mb = first_m + r % gm;
  nb = r / gm;
}

__device__ __forceinline__ void st_bf16x16(uint16_t* dst, const float* v) {
  uint4 a, b;
  a.x = pack_bf2(v[0], v[1]); a.y = pack_bf2(v[2], v[3]); a.z = pack_bf2(v[4], v[5]); a.w = pack_bf2(v[6], v[7]);
  b.x = pack_bf2(v[8], v[9]); b.y = pack_bf2(v[10], v[11]); b.z = pack_bf2(v[12], v[13]); b.w = pack_bf2(v[14], v[15]);
  reinterpret_cast<uint4*>(dst)[0] = a;
  reinterpret_cast<uint4*>(dst)[1] = b;
}
template <int CW>
__device__ __forceinline__ void st_bf16xCW(uint16_t* dst, const float* v) {
  if constexpr (CW == 16) {
    st_bf16x16(dst, v);
  } else {
    uint4 a;
    a.x = pack_bf2(v[0], v[1]); a.y = pack_bf2(v[2], v[3]); a.z = pack_bf2(v[4], v[5]); a.w = pack_bf2(v[6], v[7]);
    reinterpret_cast<uint4*>(dst)[0] = a;
  }
}
template <int CW>
__device__ __forceinline__ void tmem_ldCW(uint32_t taddr, float* v) {
  if constexpr (CW == 16) tmem_ld16(taddr, v); else tmem_ld8(taddr, v);
}
__device__ __forceinline__ void add_bias(float* v, const uint16_t* b, int n) {
  if (b)
#pragma unroll
    for (int j = 0; j < n; ++j) v[j] += bf2f(b[j]);
}
// Per-row RoPE state of the fused QKV / deviation epilogue: position, stitched-arena row and the
// fp32 cos/sin of the row's position, loaded BEFORE the epilogue waits for the accumulator so
// the table reads overlap the tile's main loop instead of stalling every 16-column chunk.
template <int DH>
struct RopeRow {
  int pos = 0, drow = 0;
  float cs[DH / 2], sn[DH / 2];
};
template <int DH>
__device__ __forceinline__ void rope_row_load(RopeRow<DH>& rr, int row, bool row_ok, const EpiArgs& ep) {
  if (!row_ok) return;
  rr.pos = __ldg(ep.pos + row);
  rr.drow = __ldg(ep.dst_row + row);
  const float4* c4 = reinterpret_cast<const float4*>(ep.rope_cos + static_cast<int64_t>(rr.pos + ep.rope_zero) * (DH / 2));
  const float4* s4 = reinterpret_cast<const float4*>(ep.rope_sin + static_cast<int64_t>(rr.pos + ep.rope_zero) * (DH / 2));
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) {
    const float4 c = __ldg(c4 + i), sv = __ldg(s4 + i);
    rr.cs[4 * i] = c.x; rr.cs[4 * i + 1] = c.y; rr.cs[4 * i + 2] = c.z; rr.cs[4 * i + 3] = c.w;
    rr.sn[4 * i] = sv.x; rr.sn[4 * i + 1] = sv.y; rr.sn[4 * i + 2] = sv.z; rr.sn[4 * i + 3] = sv.w;
  }
}

// Fused QKV / deviation epilogue over the heads of one tile (DH compile-time: every chunk index
// is a constant, so the RoPE row stays in registers).
template <int BN, int DH, bool DEV>
__device__ __forceinline__ void epi_heads(uint32_t taddr, int n0, int N, bool row_ok, int row, const EpiArgs& ep,
                                          const RopeRow<DH>& rr, unsigned long long& dev_acc) {
  constexpr int CW = DH >= 32 ? 16 : 8;
  const int H = DEV ? 0 : ep.n_heads;
  const int Hk = ep.n_kv_heads;
  const int drow = rr.drow;
  constexpr int heads_in_tile = BN / DH;
#pragma unroll 1
  for (int hi = 0; hi < heads_in_tile; ++hi) {
    const int hh = n0 / DH + hi;  // head index in the packed output
    if (hh * DH >= N) break;
    const int col0 = hi * DH;
    const bool is_q = hh < H;
    const bool is_k = !is_q && hh < H + Hk;
    const uint16_t* bias = ep.bias ? ep.bias + hh * DH : nullptr;
    if (is_q || is_k) {
      uint16_t* dst;
      const uint16_t* st = nullptr;
      if (is_q) dst = ep.q_out + static_cast<int64_t>(row) * ep.q_ld + hh * DH;
      else {
        const int64_t off = static_cast<int64_t>(hh - H) * ep.head_stride + static_cast<int64_t>(drow) * DH;
        dst = ep.arena_k + off;
        st = ep.arena_k + off;
      }
#pragma unroll
      for (int c = 0; c < DH / 2; c += CW) {
        float lo[CW], hv[CW];
        tmem_ldCW<CW>(taddr + col0 + c, lo);
        tmem_ldCW<CW>(taddr + col0 + DH / 2 + c, hv);
        if (!row_ok) continue;
        if (bias) { add_bias(lo, bias + c, CW); add_bias(hv, bias + DH / 2 + c, CW); }
        float y0[CW], y1[CW];
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          const float cc = rr.cs[c + j], ss = rr.sn[c + j];
          y0[j] = __fsub_rn(__fmul_rn(lo[j], cc), __fmul_rn(hv[j], ss));
          y1[j] = __fadd_rn(__fmul_rn(hv[j], cc), __fmul_rn(lo[j], ss));
        }
        if constexpr (DEV) {
#pragma unroll
          for (int j = 0; j < CW; ++j) {
            dev_acc += dev_term(y0[j], st[c + j]);
            dev_acc += dev_term(y1[j], st[DH / 2 + c + j]);
          }
        } else {
          st_bf16xCW<CW>(dst + c, y0);
          st_bf16xCW<CW>(dst + DH / 2 + c, y1);
        }
      }
    } else {  // V head: no rotation
      const int64_t off = static_cast<int64_t>(hh - H - Hk) * ep.head_stride + static_cast<int64_t>(drow) * DH;
      uint16_t* dst = ep.arena_v + off;
#pragma unroll
      for (int c = 0; c < DH; c += CW) {
        float v[CW];
        tmem_ldCW<CW>(taddr + col0 + c, v);
        if (!row_ok) continue;
        if (bias) add_bias(v, bias + c, CW);
        if constexpr (DEV) {
#pragma unroll
          for (int j = 0; j < CW; ++j) dev_acc += dev_term(v[j], dst[c + j]);
        } else {
          st_bf16xCW<CW>(dst + c, v);
        }
      }
    }
  }
}

template <int BN, int EPI>
__device__ __forceinline__ void epilogue_tile(uint32_t taddr, int m0, int n0, int M, int N, int lane_base,
                                              const EpiArgs& ep, bool atomic) {
  const int row = m0 + lane_base + (threadIdx.x & 31);
  const bool row_ok = row < M;
  if constexpr (EPI == EPI_BF16 || EPI == EPI_F32 || EPI == EPI_ADD_F32) {
    for (int c = 0; c < BN; c += 16) {
      if (n0 + c >= N) break;  // uniform
      float v[16];
      tmem_ld16(taddr + c, v);
      if (!row_ok) continue;
      if (n0 + c + 16 > N) {  // ragged N tail (N % 16 != 0): element stores
        const int nv = N - n0 - c;
        for (int j = 0; j < nv; ++j) {
          float val = v[j] + ((EPI == EPI_BF16 && ep.bias) ? bf2f(ep.bias[n0 + c + j]) : 0.f);
          const int64_t idx = static_cast<int64_t>(row) * ep.ldo + n0 + c + j;
          if constexpr (EPI == EPI_BF16) static_cast<uint16_t*>(ep.out)[idx] = f2bf(val);
          else if constexpr (EPI == EPI_F32) static_cast<float*>(ep.out)[idx] = val;
          else if (atomic) atomicAdd(static_cast<float*>(ep.out) + idx, val);
          else static_cast<float*>(ep.out)[idx] += val;
        }
        continue;
      }
      if constexpr (EPI == EPI_BF16) {
        if (ep.bias) add_bias(v, ep.bias + n0 + c, 16);
        st_bf16x16(static_cast<uint16_t*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + n0 + c, v);
      } else {
        float4* o = reinterpret_cast<float4*>(static_cast<float*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + n0 + c);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float4 w = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          if constexpr (EPI == EPI_ADD_F32) {
            if (atomic) {  // split-K partial sums meet in the fp32 residual stream
              atomicAdd(o + j, w);
              continue;
            }
            const float4 x = o[j];
            w.x += x.x; w.y += x.y; w.z += x.z; w.w += x.w;
          }
          o[j] = w;
        }
      }
    }
  } else if constexpr (EPI == EPI_SWIGLU) {
    static_assert(BN == 256, "SwiGLU epilogue needs [128 gate | 128 up] tiles");
    for (int c = 0; c < 128; c += 16) {
      float g[16], u[16];
      tmem_ld16(taddr + c, g);
      tmem_ld16(taddr + 128 + c, u);
      if (!row_ok) continue;
#pragma unroll
      for (int j = 0; j < 16; ++j) g[j] = g[j] / (1.0f + __expf(-g[j])) * u[j];
      st_bf16x16(static_cast<uint16_t*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + n0 / 2 + c, g);
    }
  }
}

// Persistent schedule of one CTA: work units u0, u0 + ustep, ... (tile = unit / splits); a tile is
// tile_m rows (128, or 256 for a CTA pair whose rank-1 CTA owns rows row_off = 128 .. 255)
struct Sched {
  int u0, ustep, units, splits, num_m, num_n, group_m, tile_m, row_off;
  // stream-K tail (residual epilogue on CTA pairs): tiles [units / splits, +sk_tiles) are cut into
  // equal k-block ranges, one per cluster, after the whole-tile round-robin part
  int nk = 0, sk_tiles = 0;
};

// The it-th work unit of a CTA (cluster): whole tiles / split-K shares round-robin (u0, u0 + ustep,
// ... < units), then this cluster's k-block range [lo, hi) of the stream-K tail, one unit per tile it
// crosses. Returns false when the CTA has no more units.
__device__ __forceinline__ bool unit_at(const Sched& sc, int it, int& tile, int& kb0, int& kb1) {
  const int n_dp = sc.u0 < sc.units ? (sc.units - sc.u0 + sc.ustep - 1) / sc.ustep : 0;
  if (it < n_dp) {
    const int u = sc.u0 + it * sc.ustep;
    tile = u / sc.splits;
    const int sp = u % sc.splits;
    kb0 = sp * sc.nk / sc.splits;
    kb1 = (sp + 1) * sc.nk / sc.splits;
    return true;
  }
  if (sc.sk_tiles == 0) return false;
  const int j = it - n_dp;
  const long long w = static_cast<long long>(sc.sk_tiles) * sc.nk;
  const long long lo = w * sc.u0 / sc.ustep, hi = w * (sc.u0 + 1) / sc.ustep;
  const long long st = j == 0 ? lo : (lo / sc.nk + j) * static_cast<long long>(sc.nk);
  if (st >= hi) return false;
  const long long t = st / sc.nk;
  tile = sc.units / sc.splits + static_cast<int>(t);
  kb0 = static_cast<int>(st - t * sc.nk);
  kb1 = static_cast<int>(min(static_cast<long long>(sc.nk), hi - t * sc.nk));
  return true;
}

// hand an accumulator buffer back to the MMA issuer: every epilogue thread of a single CTA, or one
// lane per epilogue warp of both CTAs of a pair onto the leader's barrier
template <bool PAIR>
__device__ __forceinline__ void release_acc(uint64_t* tempty, int acc, uint32_t leader_tempty) {
  if constexpr (PAIR) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive_cluster(leader_tempty + acc * 8);
  } else {
    mbar_arrive(&tempty[acc]);
  }
}

// QKV / deviation tiles: the RoPE row of the next tile is loaded before waiting for its accumulator
template <int BN, int DH, int EPI, bool PAIR>
__device__ __forceinline__ void epilogue_heads_loop(uint32_t tmem_base, int q, int M, int N, const Sched& sc,
                                                    uint64_t* tfull, uint64_t* tempty, uint32_t leader_tempty,
                                                    const EpiArgs& ep) {
  constexpr bool DEV = (EPI == EPI_DEV);
  int it = 0;
  for (int u = sc.u0; u < sc.units; u += sc.ustep, ++it) {
    int mb, nb; tile_coords(u / sc.splits, sc.num_m, sc.num_n, sc.group_m, mb, nb);
    const int row = mb * sc.tile_m + sc.row_off + q * 32 + (threadIdx.x & 31);
    const bool row_ok = row < M;
    RopeRow<DH> rr;
    rope_row_load<DH>(rr, row, row_ok, ep);
    const int acc = it & 1;
    mbar_wait(&tfull[acc], (it >> 1) & 1);
    tc_fence_after();
    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
    unsigned long long dacc = 0;
    epi_heads<BN, DH, DEV>(taddr, nb * BN, N, row_ok, row, ep, rr, dacc);
    if constexpr (DEV) {
      if (row_ok && ep.row_reuse[row]) atomicAdd(ep.dev_out + row, dacc);
    }
    tc_fence_before();
    release_acc<PAIR>(tempty, acc, leader_tempty);
  }
}

// the epilogue warps (4..7) of one CTA over its whole schedule
template <int BN, int EPI, bool PAIR>
__device__ __forceinline__ void epilogue_loop(uint32_t tmem_base, int warp, int M, int N, const Sched& sc,
                                              uint64_t* tfull, uint64_t* tempty, uint32_t leader_tempty,
                                              const EpiArgs& ep, const CUtensorMap* tmC, uint8_t* sOut) {
  const int q = warp & 3;  // TMEM lane quarter accessible to this warp
  if constexpr (EPI == EPI_QKV || EPI == EPI_DEV) {
    if (ep.head_dim == 128)
      epilogue_heads_loop<BN, 128, EPI, PAIR>(tmem_base, q, M, N, sc, tfull, tempty, leader_tempty, ep);
    else if (ep.head_dim == 64)
      epilogue_heads_loop<BN, 64, EPI, PAIR>(tmem_base, q, M, N, sc, tfull, tempty, leader_tempty, ep);
    else
      epilogue_heads_loop<BN, 16, EPI, PAIR>(tmem_base, q, M, N, sc, tfull, tempty, leader_tempty, ep);
  } else {
    int chunk_ctr = 0, tile = 0, kb0 = 0, kb1 = 0;
    if (EPI == EPI_ADD_F32 && (threadIdx.x & 31) == 0) tma_prefetch_desc(tmC);
    for (int it = 0; unit_at(sc, it, tile, kb0, kb1); ++it) {
      int mb, nb; tile_coords(tile, sc.num_m, sc.num_n, sc.group_m, mb, nb);
      const int m0 = mb * sc.tile_m + sc.row_off;
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      if constexpr (EPI == EPI_ADD_F32) epilogue_add_tma<BN>(taddr, m0, nb * BN, N, q, tmC, sOut, chunk_ctr);
      else epilogue_tile<BN, EPI>(taddr, m0, nb * BN, M, N, q * 32, ep, sc.splits > 1);
      tc_fence_before();
      release_acc<PAIR>(tempty, acc, leader_tempty);
    }
    if constexpr (EPI == EPI_ADD_F32) {
      if ((threadIdx.x & 31) == 0) bulk_wait<0>();  // reductions complete before the CTA retires
      __syncwarp();
    }
  }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(256, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
           const __grid_constant__ CUtensorMap tmC, int M, int N, int K, int splits, int group_m, const EpiArgs ep) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sOut = sB + C::STAGES * C::B_BYTES;  // 1024-aligned: A/B stage sizes are multiples of 16 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(sOut + C::STAGE_OUT);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 128); }
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == 0 && lane == 0) { tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // PDL: prologue above overlapped the previous kernel's tail
  griddep_launch();

  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN, tiles = num_m * num_n;
  const int nk = (K + BK - 1) / BK;
  // work unit u = (tile u / splits, K-split u % splits); splits > 1 only for additive epilogues
  const int units = tiles * splits;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0; uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int mb, nb; tile_coords(u / splits, num_m, num_n, group_m, mb, nb);
        const int sp = u % splits;
        for (int kb = sp * nk / splits; kb < (sp + 1) * nk / splits; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::A_BYTES + C::B_BYTES);
          tma_load_2d(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, mb * BM);
#pragma unroll
          for (int h = 0; h < BN / 128; ++h)  // B boxes are 128 rows (shared with the CTA-pair kernel)
            tma_load_2d(sB + stage * C::B_BYTES + h * 128 * BK * 2, &tmB, &full[stage], kb * BK, nb * BN + h * 128);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
      int stage = 0; uint32_t phase = 0; int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int sp = u % splits, kb0 = sp * nk / splits;
        for (int kb = kb0; kb < (sp + 1) * nk / splits; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = sdesc_sw128(smem_u32(sA + stage * C::A_BYTES));
          const uint64_t bd = sdesc_sw128(smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(d_tmem, ad + 2 * k, bd + 2 * k, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          umma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue warps
    const Sched sc{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), units, splits, num_m, num_n, group_m, BM, 0};
    epilogue_loop<BN, EPI, false>(tmem_base, warp, M, N, sc, tfull, tempty, 0u, ep, &tmC, sOut);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, C::TMEM_COLS);
}

// ------------------------------------------------------------------ CTA-pair GEMM (cta_group::2)
// Tile = 256 x 256 over a cluster of 2 CTAs on one TPC: each CTA stages its own 128 rows of A and
// 128 of the 256 rows of B (so 32 KB of operands per k-block per SM instead of 48 KB: the per-SM
// L2->SMEM feed, ~120 GB/s, is what bounds the single-CTA GEMM at high clocks); the leader issues
// one M=256, N=256 MMA per 16-deep k-step that writes rows 0..127 into its TMEM and 128..255 into
// the peer's. Barriers: full[s] lives in the leader (both producers' TMA bytes are counted there,
// the leader's expect_tx is its only arrival; the peer's bytes may land before it: tx goes
// negative while the arrival is still pending, so the phase cannot complete early),
// empty[s] / tfull[a] in both (the leader's commits multicast), tempty[a] in the leader (one
// arrival per epilogue warp of both CTAs). Epilogues are the single-CTA ones on 128-row halves.
struct PairCfg {
  static constexpr int STAGES = 6;
  static constexpr uint32_t A_BYTES = BM * BK * 2;     // 16 KB: this CTA's 128 rows of A
  static constexpr uint32_t B_BYTES = 128 * BK * 2;    // 16 KB: this CTA's half of the 256 rows of B
  static constexpr uint32_t STAGE_OUT = 4 * 2 * 32 * 32 * 4;
  static constexpr uint32_t SMEM = STAGES * (A_BYTES + B_BYTES) + STAGE_OUT + 1024 + 256;
  static constexpr uint32_t TMEM_COLS = 512;
};

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    k_gemm_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, int M, int N, int K, int splits, int group_m,
                int sk_tiles, const EpiArgs ep) {
  using C = PairCfg;
  constexpr int BN = 256;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sOut = sB + C::STAGES * C::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOut + C::STAGE_OUT);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    // full[s]: one arrival (the leader's expect_tx for both CTAs' bytes); the peer's TMA only
    // completes transactions on it (a release.cluster arrive per k-block costs a fence each time)
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 8); }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); }
  if (warp == 2) tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  cluster_sync();  // barrier inits and both TMEM allocations visible pair-wide
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();
  griddep_launch();

  const int num_m = (M + 2 * BM - 1) / (2 * BM), num_n = (N + BN - 1) / BN, tiles = num_m * num_n;
  const int nk = (K + BK - 1) / BK;
  const int units = (tiles - sk_tiles) * splits;  // round-robin part; the last sk_tiles tiles are stream-K
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const uint32_t leader_full = mapa_shared(full, 0);
  const uint32_t leader_tempty = mapa_shared(tempty, 0);
  Sched sc{cid, ncl, units, splits, num_m, num_n, group_m, 2 * BM, static_cast<int>(rank) * BM};
  sc.nk = nk;
  sc.sk_tiles = sk_tiles;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      int stage = 0; uint32_t phase = 0;
      int kb0 = 0, kb1 = 0, tl = 0;
      for (int it = 0; unit_at(sc, it, tl, kb0, kb1); ++it) {
        int mb, nb; tile_coords(tl, num_m, num_n, group_m, mb, nb);
        const int arow = mb * 2 * BM + rank * BM, brow = nb * BN + rank * 128;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fb = leader_full + stage * 8;
          if (leader) mbar_expect_tx(&full[stage], 2 * (C::A_BYTES + C::B_BYTES));
          tma_load_2d_pair(sA + stage * C::A_BYTES, &tmA, fb, kb * BK, arow);
          tma_load_2d_pair(sB + stage * C::B_BYTES, &tmB, fb, kb * BK, brow);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---------------- MMA issuer (leader only)
      constexpr uint32_t idesc = idesc_bf16_f32(2 * BM, BN);
      int stage = 0; uint32_t phase = 0;
      int tl = 0, kb0 = 0, kb1 = 0;
      for (int it = 0; unit_at(sc, it, tl, kb0, kb1); ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = sdesc_sw128(smem_u32(sA + stage * C::A_BYTES));
          const uint64_t bd = sdesc_sw128(smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16_pair(d_tmem, ad + 2 * k, bd + 2 * k, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          umma_commit_pair(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit_pair(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue warps (both CTAs, own 128 rows)
    epilogue_loop<BN, EPI, true>(tmem_base, warp, M, N, sc, tfull, tempty, leader_tempty, ep, &tmC, sOut);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the leader's last MMAs into this CTA's TMEM are complete (tfull waited) on both sides
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
}

template <int EPI>
cudaError_t launch_pair(const CUtensorMap* a, const CUtensorMap* b, const CUtensorMap* c, int M, int N, int K,
                        const EpiArgs& ep, int num_sms, cudaStream_t s) {
  if (EPI == EPI_ADD_F32 && c == nullptr) return cudaErrorInvalidValue;
  using C = PairCfg;
  if (cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(k_gemm_pair<EPI>), C::SMEM); e != cudaSuccess) return e;
  const int pairs = num_sms / 2;
  const int num_m = (M + 2 * BM - 1) / (2 * BM);
  const int tiles = num_m * ((N + 255) / 256);
  const int nk = (K + BK - 1) / BK;
  int splits = 1, sk_tiles = 0;
  if (EPI == EPI_ADD_F32) {
    static const bool sk_on = [] { const char* e = std::getenv("RC_GEMM_STREAMK"); return !(e && std::atoi(e) == 0); }();
    if (sk_on && tiles > pairs && tiles % pairs != 0) {
      // whole tiles round-robin, the partial last wave cut into equal k-block ranges (the reduce-add
      // epilogue makes partial tiles free to combine): e.g. cfg3 batch 32, 1264 tiles on 74 pairs =
      // 17 full waves + 6 tiles spread over all 74 pairs instead of an 18th wave on 6 of them
      sk_tiles = tiles % pairs;
    } else {
      auto cost = [&](int sp) {
        const int64_t units = static_cast<int64_t>(tiles) * sp;
        return ((units + pairs - 1) / pairs) * ((nk + sp - 1) / sp + 6);
      };
      int64_t best = cost(1);
      for (int sp = 2; sp <= 16 && nk / sp >= 8; ++sp)
        if (cost(sp) * 100 < best * 95) { best = cost(sp); splits = sp; }
    }
  }
  const int units = tiles * splits;
  const int grid = 2 * (units < pairs ? units : pairs);
  static const size_t group_a_bytes = [] {
    const char* e = std::getenv("RC_GROUP_A_MB");
    return e ? static_cast<size_t>(std::atoi(e)) << 20 : GROUP_A_BYTES;
  }();
  const int group_m = static_cast<int>(std::max<size_t>(
      2, std::min<size_t>(num_m, group_a_bytes / (static_cast<size_t>(2 * BM) * K * 2))));
  return launch_pdl(k_gemm_pair<EPI>, dim3(grid), dim3(256), C::SMEM, s, *a, *b, c ? *c : *a, M, N, K, splits,
                    group_m, sk_tiles, ep);
}

template <int BN, int EPI>
cudaError_t launch_one(const CUtensorMap* a, const CUtensorMap* b, const CUtensorMap* c, int M, int N, int K,
                       const EpiArgs& ep, int num_sms, cudaStream_t s) {
  if (EPI == EPI_ADD_F32 && c == nullptr) return cudaErrorInvalidValue;
  using C = GemmCfg<BN>;
  if (cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(k_gemm<BN, EPI>), C::SMEM); e != cudaSuccess) return e;
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int nk = (K + BK - 1) / BK;
  // split-K for additive epilogues when the tile count fills the SMs badly: pick the split that
  // minimises waves * (k-blocks per unit + fixed per-unit overhead of ~6 k-blocks)
  int splits = 1;
  if (EPI == EPI_ADD_F32) {
    auto cost = [&](int sp) {
      const int64_t units = static_cast<int64_t>(tiles) * sp;
      return ((units + num_sms - 1) / num_sms) * ((nk + sp - 1) / sp + 6);
    };
    int64_t best = cost(1);
    for (int sp = 2; sp <= 16 && nk / sp >= 8; ++sp)
      if (cost(sp) * 100 < best * 95) { best = cost(sp); splits = sp; }
  }
  const int units = tiles * splits;
  const int grid = units < num_sms ? units : num_sms;
  const int num_m = (M + BM - 1) / BM;
  static const size_t group_a_bytes = [] {
    const char* e = std::getenv("RC_GROUP_A_MB");  // diagnostics: L2 budget of the A group
    return e ? static_cast<size_t>(std::atoi(e)) << 20 : GROUP_A_BYTES;
  }();
  const int group_m = static_cast<int>(std::max<size_t>(
      4, std::min<size_t>(num_m, group_a_bytes / (static_cast<size_t>(BM) * K * 2))));
  return launch_pdl(k_gemm<BN, EPI>, dim3(grid), dim3(256), C::SMEM, s, *a, *b, c ? *c : *a, M, N, K, splits, group_m,
                    ep);
}

using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}
}  // namespace

int gemm_box_rows_b(int bn) { return bn < 128 ? bn : 128; }

bool make_tmap_bf16_2d(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld_elems,
                       uint32_t box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_bf16_3d(CUtensorMap* map, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1_bytes,
                       uint64_t s2_bytes, uint32_t b0, uint32_t b1, uint32_t b2) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1_bytes, s2_bytes};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_f32_2d(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld_elems) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_elems * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

cudaError_t gemm_launch(const CUtensorMap* a, const CUtensorMap* b, const CUtensorMap* c, int M, int N, int K, int bn,
                        int epi, const EpiArgs& ep, int num_sms, cudaStream_t s) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  // CTA pairs for 256-wide GEMMs with M >= 1024: at cfg3 batch 32 they lift the GEMMs from 0.92 to
  // 0.99 of the measured sustained peak; at M = 625 (one request's Sel) the 256-row quantisation
  // (768 rows computed) costs more than the halved operand feed saves. RC_GEMM_PAIR=0/1 forces.
  static const int pair_mode = [] { const char* e = std::getenv("RC_GEMM_PAIR"); return e ? std::atoi(e) : -1; }();
  // (the residual GEMMs split K over pairs; measured at M = 625 they gain 7% even with the padding)
  const bool pair = pair_mode == 1 || (pair_mode == -1 && (M >= 1024 || (epi == EPI_ADD_F32 && M > 2 * BM)));
  if (pair && bn == 256 && M > BM && num_sms >= 2) {
    switch (epi) {
      case EPI_BF16: return launch_pair<EPI_BF16>(a, b, c, M, N, K, ep, num_sms, s);
      case EPI_F32: return launch_pair<EPI_F32>(a, b, c, M, N, K, ep, num_sms, s);
      case EPI_ADD_F32: return launch_pair<EPI_ADD_F32>(a, b, c, M, N, K, ep, num_sms, s);
      case EPI_SWIGLU: return launch_pair<EPI_SWIGLU>(a, b, c, M, N, K, ep, num_sms, s);
      case EPI_QKV: return launch_pair<EPI_QKV>(a, b, c, M, N, K, ep, num_sms, s);
      case EPI_DEV: return launch_pair<EPI_DEV>(a, b, c, M, N, K, ep, num_sms, s);
      default: return cudaErrorInvalidValue;
    }
  }
#define RC_GEMM_CASE(BN_, E_) \
  if (bn == BN_ && epi == E_) return launch_one<BN_, E_>(a, b, c, M, N, K, ep, num_sms, s);
  RC_GEMM_CASE(256, EPI_BF16) RC_GEMM_CASE(256, EPI_F32) RC_GEMM_CASE(256, EPI_ADD_F32)
  RC_GEMM_CASE(256, EPI_SWIGLU) RC_GEMM_CASE(256, EPI_QKV) RC_GEMM_CASE(256, EPI_DEV)
  RC_GEMM_CASE(128, EPI_BF16) RC_GEMM_CASE(128, EPI_F32) RC_GEMM_CASE(128, EPI_ADD_F32)
  RC_GEMM_CASE(128, EPI_QKV) RC_GEMM_CASE(128, EPI_DEV)
#undef RC_GEMM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace rc
