// K3: persistent warp-specialised tcgen05 GEMMs for every dense projection of the hot path,
// with the per-row work fused into the epilogue.
//
//   C[M][N] = A[M][K] * B[N][K]^T    (A = activations, B = weight rows; both bf16, K-major)
//
// Three kernels share the epilogue building blocks:
//   k_gemm       one CTA, 128 x BN tiles (small shapes, BN = 128)
//   k_gemm_pair  a CTA pair (cta_group::2) on one TPC, 256 x 256 tiles: large M (the U pass of
//                layers < c, large batches). Each SM stages 128 rows of A and 128 of the 256 rows
//                of B per k-block (32 KB instead of the 48 KB of a 128 x 256 single-CTA tile): the
//                shared-memory operand feed (TMA writes + MMA reads) is what bounds a single CTA
//   k_gemm_t     a CTA pair, transposed: C^T = B A^T. The weight rows take the pair's 256-row MMA
//                side and the M tokens its N side (N' <= 256 per tile, any multiple of 32), so one
//                request's |Sel| = 625 rows cost 256 + 256 + 128 columns instead of 768 padded pair
//                rows or 128 x 256 single-CTA tiles at 2/3 of the feed rate (batch-1 TTFT)
// Roles (256 threads per CTA, one CTA per SM): warp 0 TMA producer, warp 1 MMA issuer (one thread;
// the pair's leader), warp 2 TMEM allocator (2 x 256 fp32 columns: the epilogue of one unit
// overlaps the next unit's MMAs), warps 4..7 epilogue (tcgen05.ld 32x32b: thread <-> TMEM lane).
//
// Packed weight layouts (rc_create): q|k|v heads with the dims of every head in the order
// [0, dh/2, 1, dh/2 + 1, ...] (RoPE rotate-half partners adjacent: columns 2i, 2i+1 of a normal
// tile, lanes 2i, 2i+1 of a transposed one), gate|up interleaved by row [g0, u0, g1, u1, ...].
//
// Residual epilogues (x += acc) are bitwise reproducible: a unit that covers a whole tile adds it
// with one TMA reduce-add per element; a unit covering part of a tile's K range (split-K, the
// stream-K tail) writes its accumulator to a workspace slot, and the CTA whose arrival completes
// the tile sums the slots in K order and adds that sum once.
#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "rc_internal.h"

namespace rc {

namespace {
constexpr int BM = 128, BK = 64;
constexpr int WS_TILE = 128 * 256;  // floats of one workspace slot: [256 columns][128 lanes]
// raster: group_m m-tiles share a sweep over n; the host sizes the group by the bytes of its A rows
// (they must stay in L2 while the sweep streams B; B is re-read ceil(num_m / group_m) times).
constexpr size_t GROUP_B_BYTES = size_t(56) << 20;  // n-grouped raster: weight bands kept in L2 per group
constexpr size_t GROUP_A_BYTES = size_t(32) << 20;  // measured: gate/up at cfg3 b32 3.14 -> 3.07 ms, DRAM 3.1 -> 1.9 GB vs 16 MB

template <int BN>
struct GemmCfg {
  static constexpr int STAGES = (BN == 256) ? 4 : 6;
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  // epilogue staging: per epilogue warp 2 x 4 KB (fp32 [32][32] reduce-add boxes)
  static constexpr uint32_t STAGE_OUT = 4 * 2 * 4096;
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
// the 128 epilogue threads (warps 4..7) only
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

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
  } else if constexpr (CW == 8) {
    uint4 a;
    a.x = pack_bf2(v[0], v[1]); a.y = pack_bf2(v[2], v[3]); a.z = pack_bf2(v[4], v[5]); a.w = pack_bf2(v[6], v[7]);
    reinterpret_cast<uint4*>(dst)[0] = a;
  } else {
    uint2 a;
    a.x = pack_bf2(v[0], v[1]); a.y = pack_bf2(v[2], v[3]);
    reinterpret_cast<uint2*>(dst)[0] = a;
  }
}
template <int CW>
__device__ __forceinline__ void tmem_ldCW(uint32_t taddr, float* v) {
  if constexpr (CW == 16) tmem_ld16(taddr, v); else tmem_ld8(taddr, v);
}

// ------------------------------------------------------------------ work units
// A unit is a tile, or a K range of a tile. seg / nseg: its place among the units of that tile in K
// order (nseg = 1: the whole tile); slot: the tile's index in the workspace.
struct Unit {
  int tile, kb0, kb1, seg, nseg, slot, seg_stride;  // workspace slot of a partial: (slot*2 + rank)*seg_stride + seg
};

// Persistent schedule of one CTA (pair): whole tiles / split-K shares round-robin (u0, u0 + ustep,
// ... < units), then this pair's k-block range of the stream-K tail (the last sk_tiles tiles, cut into
// equal ranges over min(ustep, sk_tiles * nk) pairs so that every range is non-empty).
struct Sched {
  int u0, ustep, units, splits, num_m, num_n, group_m, tile_m, row_off;
  int nk = 0, sk_tiles = 0;
};

__device__ __forceinline__ long long ceil_div_ll(long long a, long long b) { return (a + b - 1) / b; }

__device__ __forceinline__ bool unit_at(const Sched& sc, int it, Unit& un) {
  const int n_dp = sc.u0 < sc.units ? (sc.units - sc.u0 + sc.ustep - 1) / sc.ustep : 0;
  if (it < n_dp) {
    const int u = sc.u0 + it * sc.ustep;
    un.tile = u / sc.splits;
    const int sp = u % sc.splits;
    un.kb0 = sp * sc.nk / sc.splits;
    un.kb1 = (sp + 1) * sc.nk / sc.splits;
    un.seg = sp;
    un.nseg = sc.splits;
    un.slot = un.tile;
    un.seg_stride = sc.splits;
    return true;
  }
  if (sc.sk_tiles == 0) return false;
  const long long w = static_cast<long long>(sc.sk_tiles) * sc.nk;
  const int P = static_cast<int>(min(static_cast<long long>(sc.ustep), w));  // participating pairs
  if (sc.u0 >= P) return false;
  const int j = it - n_dp;
  const long long lo = w * sc.u0 / P, hi = w * (sc.u0 + 1) / P;
  const long long st = j == 0 ? lo : (lo / sc.nk + j) * static_cast<long long>(sc.nk);
  if (st >= hi) return false;
  const long long t = st / sc.nk;
  un.tile = sc.units / sc.splits + static_cast<int>(t);
  un.kb0 = static_cast<int>(st - t * sc.nk);
  un.kb1 = static_cast<int>(min(static_cast<long long>(sc.nk), hi - t * sc.nk));
  // pairs whose ranges meet tile t: the one holding its first k-block .. the one holding its last
  const long long c_first = ceil_div_ll((t * sc.nk + 1) * P, w) - 1;
  const long long c_last = ceil_div_ll((t + 1) * sc.nk * P, w) - 1;
  un.nseg = static_cast<int>(c_last - c_first + 1);
  un.seg = static_cast<int>(sc.u0 - c_first);
  un.slot = static_cast<int>(t);
  un.seg_stride = (P + sc.sk_tiles - 1) / sc.sk_tiles + 1;  // >= nseg of every tail tile
  return true;
}

// group_m < 0: the transposed raster, -group_m n-tiles share a sweep over m (B stays in L2, A is
// re-read ceil(num_n / -group_m) times); the host picks the raster with the lower estimated traffic
__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int group_m, int& mb, int& nb) {
  if (group_m < 0) {
    const int gn_max = -group_m;
    const int per_group = gn_max * num_m;
    const int g = t / per_group;
    const int first_n = g * gn_max;
    const int gn = min(gn_max, num_n - first_n);
    const int r = t - g * per_group;
    nb = first_n + r % gn;
    mb = r / gn;
    return;
  }
  const int per_group = group_m * num_n;
  const int g = t / per_group;
  const int first_m = g * group_m;
  const int gm = min(group_m, num_m - first_m);
  const int r = t - g * per_group;
  mb = first_m + r % gm;
  nb = r / gm;
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

// ------------------------------------------------------------------ residual (reduce-add) epilogue
// One 32-column chunk of a warp's 32 accumulator lanes -> a swizzled fp32 [32][32] box in this warp's
// staging buffer -> one TMA reduce-add into x. Normal tiles: box row = lane (token), column = chunk
// column (feature). Transposed tiles: box row = chunk column (token), column = lane (feature).
template <bool TRANS>
__device__ __forceinline__ void add_chunk(const uint32_t* v, uint8_t* mybuf, int& chunk_ctr, const void* tmC, int c0,
                                          int c1) {
  const int lane = threadIdx.x & 31;
  const int buf = chunk_ctr & 1;
  if (chunk_ctr >= 2) {
    if (lane == 0) bulk_wait_read<1>();  // the reduction that last read this buffer has drained it
    __syncwarp();
  }
  uint8_t* box = mybuf + buf * 4096;
  if constexpr (!TRANS) {
    uint8_t* row = box + lane * 128;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      *reinterpret_cast<uint4*>(row + ((k ^ (lane & 7)) << 4)) = make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < 32; ++k)
      *reinterpret_cast<uint32_t*>(box + k * 128 + (((lane >> 2) ^ (k & 7)) << 4) + (lane & 3) * 4) = v[k];
  }
  fence_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_reduce_add_2d(tmC, box, c0, c1);
    bulk_commit();
  }
  ++chunk_ctr;
}

// x += acc for one unit (`ncols` accumulator columns, a multiple of 32; taddr already offset to this
// warp's lanes). Box coordinates of chunk c: normal (base0 + c, base1), transposed (base0, base1 + c).
template <bool TRANS>
__device__ __forceinline__ void epilogue_add(uint32_t taddr, int ncols, int base0, int base1, int q, const void* tmC,
                                             uint8_t* sOut, int& chunk_ctr, const Unit& un, int rank,
                                             const EpiArgs& ep, int* s_flag) {
  const int lane = threadIdx.x & 31;
  uint8_t* mybuf = sOut + q * 2 * 4096;
  if (un.nseg == 1 || !ep.det) {  // a whole tile, or order-free partials: straight into x
    for (int c = 0; c < ncols; c += 32) {
      uint32_t v[32];
      tmem_ld32(taddr + c, v);
      tmem_wait_ld();
      add_chunk<TRANS>(v, mybuf, chunk_ctr, tmC, TRANS ? base0 : base0 + c, TRANS ? base1 + c : base1);
    }
    return;
  }
  // partial unit: accumulator -> workspace slot, layout [col / 4][lane][4] (a thread's 4 consecutive
  // columns are one 16-byte vector; a warp's vectors are 512 contiguous bytes)
  float* slot0 = ep.ws + static_cast<int64_t>((un.slot * 2 + rank) * un.seg_stride) * WS_TILE;
  float4* mine = reinterpret_cast<float4*>(slot0 + static_cast<int64_t>(un.seg) * WS_TILE);
  const int row = q * 32 + lane;
  for (int c = 0; c < ncols; c += 32) {
    uint32_t v[32];
    tmem_ld32(taddr + c, v);
    tmem_wait_ld();
#pragma unroll
    for (int k = 0; k < 8; ++k)
      __stcg(mine + ((c >> 2) + k) * 128 + row, make_float4(__uint_as_float(v[4 * k]), __uint_as_float(v[4 * k + 1]),
                                                          __uint_as_float(v[4 * k + 2]), __uint_as_float(v[4 * k + 3])));
  }
  __threadfence();
  epi_bar();
  if (threadIdx.x == 128) {
    int* cnt = ep.ws_cnt + un.slot * 2 + rank;
    const int old = atomicAdd(cnt, 1);
    const int last = old == un.nseg - 1;
    if (last) atomicExch(cnt, 0);  // ready for the next launch
    *s_flag = last;
  }
  epi_bar();
  const int last = *s_flag;
  epi_bar();  // s_flag may be rewritten by the next partial unit
  if (!last) return;
  __threadfence();
  const float4* base = reinterpret_cast<const float4*>(slot0);
  for (int c = 0; c < ncols; c += 32) {
    float a[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) a[k] = 0.f;
    // K order (segment 0, 1, ...): bitwise reproducible; four segments' loads in flight at a time
    for (int s0 = 0; s0 < un.nseg; s0 += 4) {
      float4 w[4][8];
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          w[g][k] = s0 + g < un.nseg ? __ldcg(base + static_cast<int64_t>(s0 + g) * (WS_TILE / 4) + ((c >> 2) + k) * 128 + row)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        if (s0 + g >= un.nseg) break;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          a[4 * k] = __fadd_rn(a[4 * k], w[g][k].x);
          a[4 * k + 1] = __fadd_rn(a[4 * k + 1], w[g][k].y);
          a[4 * k + 2] = __fadd_rn(a[4 * k + 2], w[g][k].z);
          a[4 * k + 3] = __fadd_rn(a[4 * k + 3], w[g][k].w);
        }
      }
    }
    uint32_t v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = __float_as_uint(a[k]);
    add_chunk<TRANS>(v, mybuf, chunk_ctr, tmC, TRANS ? base0 : base0 + c, TRANS ? base1 + c : base1);
  }
}

// ------------------------------------------------------------------ normal-orientation epilogues
// Per-row RoPE state of the fused QKV / deviation epilogue: position, stitched-arena row and the
// fp32 cos/sin of the row's position, loaded BEFORE the epilogue waits for the accumulator so
// the table reads overlap the tile's main loop instead of stalling every chunk.
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

// Fused QKV / deviation epilogue over the heads of one tile. Columns of a head come in rotate-half
// pairs: column 2i = dim i, 2i + 1 = dim i + DH/2 (packed layout). MODE 0: QKV (store q, k, v);
// 1: DEV (k, v only, score against the stitched rows, no store); 2: QKV_DEV (score k, v against the
// stitched rows, then overwrite them; `score` = this row's k/v are scored).
template <int BN, int DH, int MODE>
__device__ __forceinline__ void epi_heads(uint32_t taddr, int n0, int N, bool row_ok, int row, const EpiArgs& ep,
                                          const RopeRow<DH>& rr, unsigned long long& dev_acc, bool score) {
  constexpr bool DEV = MODE == 1;
  constexpr int CW = DH >= 32 ? 16 : 8;  // dims per chunk and half: 2 CW accumulator columns
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
    uint16_t* dst;
    if (is_q) dst = ep.q_out + static_cast<int64_t>(row) * ep.q_ld + hh * DH;
    else if (is_k) dst = ep.arena_k + static_cast<int64_t>(hh - H) * ep.head_stride + static_cast<int64_t>(drow) * DH;
    else if (DEV && ep.vsrc.vmap)  // zero-copy V: the stitched V row may live in a pool
      dst = const_cast<uint16_t*>(vsrc_row(ep.vsrc, ep.arena_v, ep.head_stride, hh - H - Hk, drow, DH));
    else dst = ep.arena_v + static_cast<int64_t>(hh - H - Hk) * ep.head_stride + static_cast<int64_t>(drow) * DH;
#pragma unroll
    for (int c = 0; c < DH; c += 2 * CW) {
      float v[2 * CW];
      tmem_ldCW<CW>(taddr + col0 + c, v);
      tmem_ldCW<CW>(taddr + col0 + c + CW, v + CW);
      if (!row_ok) continue;
      if (bias)
#pragma unroll
        for (int j = 0; j < 2 * CW; ++j) v[j] += bf2f(bias[c + j]);
      const int i0 = c / 2;
      float y0[CW], y1[CW];
      if (is_q || is_k) {
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          const float lo = v[2 * j], hv = v[2 * j + 1];
          const float cc = rr.cs[i0 + j], ss = rr.sn[i0 + j];
          y0[j] = __fsub_rn(__fmul_rn(lo, cc), __fmul_rn(hv, ss));
          y1[j] = __fadd_rn(__fmul_rn(hv, cc), __fmul_rn(lo, ss));
        }
      } else {
#pragma unroll
        for (int j = 0; j < CW; ++j) { y0[j] = v[2 * j]; y1[j] = v[2 * j + 1]; }
      }
      if constexpr (DEV) {
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          dev_acc += dev_term(y0[j], dst[i0 + j]);
          dev_acc += dev_term(y1[j], dst[DH / 2 + i0 + j]);
        }
      } else {
        if constexpr (MODE == 2) {
          if (!is_q && score)  // the stitched value is read before this thread overwrites it
#pragma unroll
            for (int j = 0; j < CW; ++j) {
              dev_acc += dev_term(y0[j], dst[i0 + j]);
              dev_acc += dev_term(y1[j], dst[DH / 2 + i0 + j]);
            }
        }
        st_bf16xCW<CW>(dst + i0, y0);
        st_bf16xCW<CW>(dst + DH / 2 + i0, y1);
      }
    }
  }
}

template <int BN, int EPI>
__device__ __forceinline__ void epilogue_tile(uint32_t taddr, int m0, int n0, int M, int N, int lane_base,
                                              const EpiArgs& ep) {
  const int row = m0 + lane_base + (threadIdx.x & 31);
  const bool row_ok = row < M;
  if constexpr (EPI == EPI_BF16 || EPI == EPI_F32) {
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
          else static_cast<float*>(ep.out)[idx] = val;
        }
        continue;
      }
      if constexpr (EPI == EPI_BF16) {
        if (ep.bias)
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] += bf2f(ep.bias[n0 + c + j]);
        st_bf16x16(static_cast<uint16_t*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + n0 + c, v);
      } else {
        float4* o = reinterpret_cast<float4*>(static_cast<float*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + n0 + c);
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
    }
  } else if constexpr (EPI == EPI_SWIGLU) {
    // columns (2i, 2i + 1) = (gate, up) of feature n0/2 + i
    static_assert(BN == 256, "SwiGLU epilogue needs 256-wide [g u g u ...] tiles");
    for (int c = 0; c < BN; c += 32) {
      float a[16], b[16];
      tmem_ld16(taddr + c, a);
      tmem_ld16(taddr + c + 16, b);
      if (!row_ok) continue;
      float o[16];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        o[j] = a[2 * j] / (1.0f + __expf(-a[2 * j])) * a[2 * j + 1];
        o[8 + j] = b[2 * j] / (1.0f + __expf(-b[2 * j])) * b[2 * j + 1];
      }
      st_bf16x16(static_cast<uint16_t*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + (n0 + c) / 2, o);
    }
  }
}

// QKV / deviation tiles: the RoPE row of the next tile is loaded before waiting for its accumulator
template <int BN, int DH, int EPI, bool PAIR>
__device__ __forceinline__ void epilogue_heads_loop(uint32_t tmem_base, int q, int M, int N, const Sched& sc,
                                                    uint64_t* tfull, uint64_t* tempty, uint32_t leader_tempty,
                                                    const EpiArgs& ep) {
  constexpr int MODE = EPI == EPI_DEV ? 1 : EPI == EPI_QKV_DEV ? 2 : 0;
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
    const int drow = (MODE == 2 && row_ok) ? ep.dev_row[row] : row;
    const bool score = MODE != 0 && row_ok && ep.row_reuse[drow];
    epi_heads<BN, DH, MODE>(taddr, nb * BN, N, row_ok, row, ep, rr, dacc, score);
    if constexpr (MODE != 0) {
      if (score) atomicAdd(ep.dev_out + drow, dacc);  // integer: order-independent
    }
    tc_fence_before();
    release_acc<PAIR>(tempty, acc, leader_tempty);
  }
}

// the epilogue warps (4..7) of one CTA over its whole schedule
template <int BN, int EPI, bool PAIR>
__device__ __forceinline__ void epilogue_loop(uint32_t tmem_base, int warp, int M, int N, const Sched& sc,
                                              uint64_t* tfull, uint64_t* tempty, uint32_t leader_tempty,
                                              const EpiArgs& ep, const CUtensorMap* tmC, uint8_t* sOut, int rank,
                                              int* s_flag) {
  const int q = warp & 3;  // TMEM lane quarter accessible to this warp
  if constexpr (EPI == EPI_QKV || EPI == EPI_DEV || EPI == EPI_QKV_DEV) {
    if (ep.head_dim == 128)
      epilogue_heads_loop<BN, 128, EPI, PAIR>(tmem_base, q, M, N, sc, tfull, tempty, leader_tempty, ep);
    else if (ep.head_dim == 64)
      epilogue_heads_loop<BN, 64, EPI, PAIR>(tmem_base, q, M, N, sc, tfull, tempty, leader_tempty, ep);
    else
      epilogue_heads_loop<BN, 16, EPI, PAIR>(tmem_base, q, M, N, sc, tfull, tempty, leader_tempty, ep);
  } else {
    int chunk_ctr = 0;
    Unit un;
    if (EPI == EPI_ADD_F32 && (threadIdx.x & 31) == 0) tma_prefetch_desc(tmC);
    for (int it = 0; unit_at(sc, it, un); ++it) {
      int mb, nb; tile_coords(un.tile, sc.num_m, sc.num_n, sc.group_m, mb, nb);
      const int m0 = mb * sc.tile_m + sc.row_off;
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      if constexpr (EPI == EPI_ADD_F32) {
        const int ncols = min(BN, (N - nb * BN + 31) / 32 * 32);
        epilogue_add<false>(taddr, ncols, nb * BN, m0 + q * 32, q, tmC, sOut, chunk_ctr, un, rank, ep, s_flag);
      } else {
        epilogue_tile<BN, EPI>(taddr, m0, nb * BN, M, N, q * 32, ep);
      }
      tc_fence_before();
      release_acc<PAIR>(tempty, acc, leader_tempty);
    }
    if constexpr (EPI == EPI_ADD_F32) {
      if ((threadIdx.x & 31) == 0) bulk_wait<0>();  // reductions complete before the CTA retires
      __syncwarp();
    }
  }
}

// ------------------------------------------------------------------ single-CTA GEMM
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
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);

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
  // work unit u = (tile u / splits, K-split u % splits); splits > 1 only for the residual epilogue
  const int units = tiles * splits;
  Sched sc{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), units, splits, num_m, num_n, group_m, BM, 0};
  sc.nk = nk;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0; uint32_t phase = 0;
      Unit un;
      for (int it = 0; unit_at(sc, it, un); ++it) {
        int mb, nb; tile_coords(un.tile, num_m, num_n, group_m, mb, nb);
        for (int kb = un.kb0; kb < un.kb1; ++kb) {
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
      int stage = 0; uint32_t phase = 0;
      Unit un;
      for (int it = 0; unit_at(sc, it, un); ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = un.kb0; kb < un.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = sdesc_sw128(smem_u32(sA + stage * C::A_BYTES));
          const uint64_t bd = sdesc_sw128(smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(d_tmem, ad + 2 * k, bd + 2 * k, idesc, (kb != un.kb0 || k != 0) ? 1u : 0u);
          umma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue warps
    epilogue_loop<BN, EPI, false>(tmem_base, warp, M, N, sc, tfull, tempty, 0u, ep, &tmC, sOut, 0, s_flag);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, C::TMEM_COLS);
}

// ------------------------------------------------------------------ CTA-pair GEMM (cta_group::2)
// Tile = 256 x 256 over a cluster of 2 CTAs on one TPC: each CTA stages its own 128 rows of A and
// 128 of the 256 rows of B; the leader issues one M=256, N=256 MMA per 16-deep k-step that writes
// rows 0..127 into its TMEM and 128..255 into the peer's. Barriers: full[s] lives in the leader
// (both producers' TMA bytes are counted there, the leader's expect_tx is its only arrival; the
// peer's bytes may land before it: tx goes negative while the arrival is still pending, so the phase
// cannot complete early), empty[s] / tfull[a] in both (the leader's commits multicast), tempty[a] in
// the leader (one arrival per epilogue warp of both CTAs). Epilogues are the single-CTA ones on
// 128-row halves.
struct PairCfg {
  static constexpr int STAGES = 6;
  static constexpr uint32_t A_BYTES = BM * BK * 2;     // 16 KB: this CTA's 128 rows of A
  static constexpr uint32_t B_BYTES = 128 * BK * 2;    // 16 KB: this CTA's half of the 256 rows of B
  static constexpr uint32_t STAGE_OUT = 4 * 2 * 4096;
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
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
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
      Unit un;
      for (int it = 0; unit_at(sc, it, un); ++it) {
        int mb, nb; tile_coords(un.tile, num_m, num_n, group_m, mb, nb);
        const int arow = mb * 2 * BM + rank * BM, brow = nb * BN + rank * 128;
        for (int kb = un.kb0; kb < un.kb1; ++kb) {
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
      Unit un;
      for (int it = 0; unit_at(sc, it, un); ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = un.kb0; kb < un.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = sdesc_sw128(smem_u32(sA + stage * C::A_BYTES));
          const uint64_t bd = sdesc_sw128(smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16_pair(d_tmem, ad + 2 * k, bd + 2 * k, idesc, (kb != un.kb0 || k != 0) ? 1u : 0u);
          umma_commit_pair(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit_pair(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue warps (both CTAs, own 128 rows)
    epilogue_loop<BN, EPI, true>(tmem_base, warp, M, N, sc, tfull, tempty, leader_tempty, ep, &tmC, sOut,
                                 static_cast<int>(rank), s_flag);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the leader's last MMAs into this CTA's TMEM are complete (tfull waited) on both sides
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
}

// ------------------------------------------------------------------ transposed CTA-pair GEMM
// C^T[N][M] = B[N][K] A[M][K]^T for small M. Tile = 256 weight rows (stripe s; 128 per CTA, the
// MMA's M) x N' tokens (the MMA's N: 256, or 128 for a short last tile). Each CTA stages its 128
// weight rows and N'/2 token rows (one TMA box) per k-block.
struct TCfg {
  static constexpr int STAGES = 6;
  static constexpr uint32_t A_BYTES = 128 * BK * 2;    // this CTA's 128 weight rows
  static constexpr uint32_t B_BYTES = 128 * BK * 2;    // up to 128 token rows
  // epilogue staging: ADD 4 warps x 2 fp32 boxes; QKV 2 x [32][128] bf16 + 4 x 4 KB cos/sin; SwiGLU 4 x 1 KB
  static constexpr uint32_t STAGE_OUT = 4 * 2 * 4096;
  static constexpr uint32_t SMEM = STAGES * (A_BYTES + B_BYTES) + STAGE_OUT + 1024 + 256;
  static constexpr uint32_t TMEM_COLS = 512;
};

// early O-projection: wait until `target` attention CTAs have signalled the token tile (acquire), then
// order this thread's later TMA (async-proxy) reads after the generic-proxy writes it synchronised with.
// Bounded: a signal that never comes traps (a launch error) instead of hanging the GPU.
__device__ __forceinline__ void wait_ready(const int32_t* ctr, int target) {
  const long long t_start = clock64();
  while (true) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= target) break;
    __nanosleep(128);
    if (clock64() - t_start > (1ll << 33)) __trap();
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

struct TSched {
  int cid, ncl, nstripes, nfull, tail_n, splits, nk;
  int pack = 0;  // 1: the 128-token tail tiles of two stripes share one slot (see at_packed)
  int ttmajor = 0;  // 1 (early O-projection): token tile major, so every pair's first units are the
                    // token tiles whose attention finishes first (short causal ranges) and the last
                    // token tile's units come last
  // the it-th unit of this pair: weight stripe s, first token t0, N' (ncols) and the K range. Tiles of
  // 256 tokens (the last one 128 when the remainder fits), round-robin over units in stripe-major
  // order: a stripe's token tiles are adjacent, so its 256 weight rows stream from HBM once. (Cutting
  // the stripes x tokens into equal contiguous ranges per pair balanced the waves but streamed every
  // stripe's weights 3x through L2: SwiGLU 3.9 -> 4.9 ms per cfg3 batch-1 step, not kept.)
  // Packed schedule (no split-K, 128-token tail): the slots of stripes (2j, 2j + 1) are their 2 nfull
  // full tiles and ONE slot holding both 128-token tails back to back, dealt round-robin; every slot is
  // 256 token columns, so |Sel| = 625 costs 2.5 slots per stripe: SwiGLU at cfg3 batch 1 = 280 slots on
  // 74 pairs = 4 rounds of 256 columns instead of up to 4.5 (the tails of 336 tiles dealt round-robin
  // left every third pair with 1152 columns against a 969 average). A stripe's tiles stay in one round.
  __device__ __forceinline__ bool at_packed(int it, int& s, int& t0, int& ncols, Unit& un) const {
    const int per2 = 2 * nfull + 1;
    const int nslots = (nstripes / 2) * per2 + ((nstripes & 1) ? nfull + 1 : 0);
    int left = it, tt = 0;
    for (int k = 0;; ++k) {
      const int q = cid + k * ncl;
      if (q >= nslots) return false;
      const int j = q / per2, r = q % per2;
      const bool last_odd = 2 * j + 1 >= nstripes;  // the odd stripe out: its tail has a slot alone
      const int cnt = (r == 2 * nfull && !last_odd) ? 2 : 1;
      if (left < cnt) {
        if (last_odd) { s = 2 * j; tt = r; }
        else if (r < 2 * nfull) { s = 2 * j + r / nfull; tt = r % nfull; }
        else { s = 2 * j + left; tt = nfull; }
        break;
      }
      left -= cnt;
    }
    const int ntt = nfull + 1;
    t0 = tt * 256;
    ncols = tt < nfull ? 256 : tail_n;
    un.tile = s * ntt + tt;
    un.kb0 = 0; un.kb1 = nk;
    un.seg = 0; un.nseg = 1; un.slot = un.tile; un.seg_stride = 1;
    return true;
  }
  __device__ __forceinline__ bool at(int it, int& s, int& t0, int& ncols, Unit& un) const {
    if (pack) return at_packed(it, s, t0, ncols, un);
    const int ntt = nfull + (tail_n > 0 ? 1 : 0);
    const int u = cid + it * ncl;
    if (u >= nstripes * ntt * splits) return false;
    const int tile = u / splits, sp = u % splits;
    s = ttmajor ? tile % nstripes : tile / ntt;
    const int tt = ttmajor ? tile / nstripes : tile % ntt;
    t0 = tt * 256;
    ncols = tt < nfull ? 256 : tail_n;
    un.tile = tile;
    un.kb0 = sp * nk / splits;
    un.kb1 = (sp + 1) * nk / splits;
    un.seg = sp;
    un.nseg = splits;
    un.slot = tile;
    un.seg_stride = splits;
    return true;
  }
};

// SwiGLU on a transposed tile: lanes (2i, 2i + 1) hold (gate, up) of one feature for 32 tokens; the
// even lane finishes tokens 0..15 and the odd lane 16..31 of the chunk, through a per-warp
// [32 tokens][16 features] bf16 staging tile written out as 32-byte token rows.
__device__ __forceinline__ void epi_t_swiglu(uint32_t taddr, int ncols, int t0, int M, int fo0, uint8_t* wbuf,
                                             const EpiArgs& ep) {
  const int lane = threadIdx.x & 31;
  const bool odd = lane & 1;
  uint16_t* st = reinterpret_cast<uint16_t*>(wbuf);  // [32][16]
  for (int c = 0; c < ncols; c += 32) {
    uint32_t r[32];
    tmem_ld32(taddr + c, r);
    tmem_wait_ld();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float send = __uint_as_float(odd ? r[k] : r[k + 16]);
      const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
      const float g = odd ? recv : __uint_as_float(r[k]);
      const float u = odd ? __uint_as_float(r[k + 16]) : recv;
      st[((odd ? 16 : 0) + k) * 16 + (lane >> 1)] = f2bf(g / (1.0f + __expf(-g)) * u);
    }
    __syncwarp();
    const int t = t0 + c + lane;
    if (t < M) {
      const uint4* src = reinterpret_cast<const uint4*>(st + lane * 16);
      uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(ep.out) + static_cast<int64_t>(t) * ep.ldo + fo0);
      dst[0] = src[0];
      dst[1] = src[1];
    }
    __syncwarp();
  }
}

// QKV on a transposed tile: this CTA's 128 lanes are one head (hh); lanes (2i, 2i + 1) of warp q are
// dims (16q + i, 64 + 16q + i). Everything position-dependent is fetched ahead: the tile's token
// positions and arena rows (lane l <-> tokens 32j + l) and the first chunk's cos/sin before the
// accumulator wait, each next chunk's cos/sin while the current one is rotated. Per chunk every lane
// puts its own token's 16 cos/sin values into a per-warp table; RoPE partners meet through one
// shuffle per token; the rotated chunk goes through a CTA-wide [32 tokens][128 dims] bf16 tile
// (double-buffered, one named barrier per chunk) and out as 256-byte rows to q_out or the arena.
struct QkvPre {
  int pos[8], dst[8];
  float4 cs[4], sn[4];
};
__device__ __forceinline__ void qkv_rope_fetch(QkvPre& p, int pos, int q, const EpiArgs& ep) {
  const float4* cp = reinterpret_cast<const float4*>(ep.rope_cos + static_cast<int64_t>(pos + ep.rope_zero) * 64 + 16 * q);
  const float4* sp = reinterpret_cast<const float4*>(ep.rope_sin + static_cast<int64_t>(pos + ep.rope_zero) * 64 + 16 * q);
#pragma unroll
  for (int j = 0; j < 4; ++j) { p.cs[j] = __ldg(cp + j); p.sn[j] = __ldg(sp + j); }
}
__device__ __forceinline__ void qkv_prefetch(QkvPre& p, int t0, int M, int q, bool rot, const EpiArgs& ep) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int t = t0 + 32 * j + lane;
    p.pos[j] = t < M ? __ldg(ep.pos + t) : 0;
    p.dst[j] = t < M ? __ldg(ep.dst_row + t) : 0;
  }
  if (rot) qkv_rope_fetch(p, p.pos[0], q, ep);
}
__device__ __forceinline__ void epi_t_qkv(uint32_t taddr, int ncols, int t0, int M, int hh, int q, uint8_t* sbuf,
                                          int& chunk_ctr, QkvPre& pre, const EpiArgs& ep) {
  const int lane = threadIdx.x & 31;
  const bool odd = lane & 1;
  const int H = ep.n_heads, Hk = ep.n_kv_heads;
  const bool rot = hh < H + Hk;
  const int dim = 16 * q + (lane >> 1) + (odd ? 64 : 0);
  const float bias = ep.bias ? bf2f(ep.bias[hh * 128 + q * 32 + lane]) : 0.f;
  float* tcs = reinterpret_cast<float*>(sbuf + 16384 + q * 4096);  // per warp [32 tokens][16] cos, then sin
  float* tsn = tcs + 512;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = 32 * j;
    if (c >= ncols) break;
    if (rot) {
      __syncwarp();  // the previous chunk's table reads are done
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        reinterpret_cast<float4*>(tcs + lane * 16)[v] = pre.cs[v];
        reinterpret_cast<float4*>(tsn + lane * 16)[v] = pre.sn[v];
      }
      if (j + 1 < 8 && c + 32 < ncols) qkv_rope_fetch(pre, pre.pos[j + 1], q, ep);  // next chunk, in flight
    }
    uint32_t r[32];
    tmem_ld32(taddr + c, r);
    tmem_wait_ld();
    __syncwarp();
    uint16_t* st = reinterpret_cast<uint16_t*>(sbuf + (chunk_ctr & 1) * 8192);  // [32][128]
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const float x = __uint_as_float(r[k]) + bias;
      float y = x;
      if (rot) {
        const float partner = __shfl_xor_sync(0xffffffffu, x, 1);
        const float cs = tcs[k * 16 + (lane >> 1)], sn = tsn[k * 16 + (lane >> 1)];
        // even lane: y0 = x0 c - x1 s; odd lane: y1 = x1 c + x0 s (R13, products rounded first)
        y = odd ? __fadd_rn(__fmul_rn(x, cs), __fmul_rn(partner, sn))
                : __fsub_rn(__fmul_rn(x, cs), __fmul_rn(partner, sn));
      }
      st[k * 128 + dim] = f2bf(y);
    }
    epi_bar();
    // warp q writes tokens 8q .. 8q + 7 of the chunk: half a warp per 256-byte row
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = 8 * q + (lane >> 4) + 2 * i;
      const int drow = __shfl_sync(0xffffffffu, pre.dst[j], k);
      const int t = t0 + c + k;
      if (t >= M) continue;
      uint16_t* dst;
      if (hh < H) dst = ep.q_out + static_cast<int64_t>(t) * ep.q_ld + hh * 128;
      else if (rot) dst = ep.arena_k + static_cast<int64_t>(hh - H) * ep.head_stride + static_cast<int64_t>(drow) * 128;
      else dst = ep.arena_v + static_cast<int64_t>(hh - H - Hk) * ep.head_stride + static_cast<int64_t>(drow) * 128;
      reinterpret_cast<uint4*>(dst)[lane & 15] = reinterpret_cast<const uint4*>(st + k * 128)[lane & 15];
    }
    ++chunk_ctr;
  }
}

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    k_gemm_t(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX128,
             const __grid_constant__ CUtensorMap tmX64, const __grid_constant__ CUtensorMap tmC, int M, int N, int K,
             int splits, const EpiArgs ep) {
  using C = TCfg;
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
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 8); }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch_desc(&tmW); tma_prefetch_desc(&tmX128); tma_prefetch_desc(&tmX64); }
  if (warp == 2) tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // early O-projection: the only input the previous kernel (attention) produces is the token operand,
  // gated per token tile by ep.ready below; everything older completed before any attention CTA
  // passed its own griddepcontrol.wait
  if (ep.ready == nullptr) griddep_wait();
  griddep_launch();

  const int nfull = M / 256, rem = M - nfull * 256;
  TSched sc{static_cast<int>(blockIdx.x >> 1), static_cast<int>(gridDim.x >> 1), N / 256, nfull,
            rem > 0 ? (rem <= 128 ? 128 : 256) : 0, splits, (K + BK - 1) / BK};
  sc.pack = ep.t_pack && splits == 1 && sc.tail_n == 128 && nfull >= 1 && ep.ready == nullptr;
  sc.ttmajor = ep.ready != nullptr;
  const uint32_t leader_full = mapa_shared(full, 0);
  const uint32_t leader_tempty = mapa_shared(tempty, 0);

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      int stage = 0; uint32_t phase = 0;
      int s, t0, ncols;
      Unit un;
      for (int it = 0; sc.at(it, s, t0, ncols, un); ++it) {
        const int wrow = s * 256 + rank * 128;
        const int half = ncols / 2;
        const int trow = t0 + rank * half;
        if (ep.ready) wait_ready(ep.ready + t0 / 256, ep.ready_tgt[t0 / 256]);
        for (int kb = un.kb0; kb < un.kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fb = leader_full + stage * 8;
          if (leader) mbar_expect_tx(&full[stage], 2 * (C::A_BYTES + static_cast<uint32_t>(half) * BK * 2));
          tma_load_2d_pair(sA + stage * C::A_BYTES, &tmW, fb, kb * BK, wrow);
          // one box per CTA: 128 token rows (full tile) or 64 (tail); the TMA issue count matters (four
          // 32-row boxes per full tile measured 12 % slower than two 64-row boxes at cfg3 batch 1)
          tma_load_2d_pair(sB + stage * C::B_BYTES, half == 128 ? &tmX128 : &tmX64, fb, kb * BK, trow);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---------------- MMA issuer (leader only)
      int stage = 0; uint32_t phase = 0;
      int s, t0, ncols;
      Unit un;
      for (int it = 0; sc.at(it, s, t0, ncols, un); ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t idesc = idesc_bf16_f32(256, ncols);
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = un.kb0; kb < un.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = sdesc_sw128(smem_u32(sA + stage * C::A_BYTES));
          const uint64_t bd = sdesc_sw128(smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16_pair(d_tmem, ad + 2 * k, bd + 2 * k, idesc, (kb != un.kb0 || k != 0) ? 1u : 0u);
          umma_commit_pair(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit_pair(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue warps (both CTAs, own 128 weight rows)
    const int q = warp & 3;
    int chunk_ctr = 0;
    int s, t0, ncols;
    Unit un;
    if (EPI == EPI_ADD_F32 && lane == 0) tma_prefetch_desc(&tmC);
    for (int it = 0; sc.at(it, s, t0, ncols, un); ++it) {
      const int acc = it & 1;
      const int f0 = s * 256 + static_cast<int>(rank) * 128;
      QkvPre pre;
      if constexpr (EPI == EPI_QKV) qkv_prefetch(pre, t0, M, q, f0 / 128 < ep.n_heads + ep.n_kv_heads, ep);
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * 256;
      if (ep.no_epi) {  // diagnostics (RC_GEMM_NOEPI=1): main loop only, the output is not written
      } else if constexpr (EPI == EPI_ADD_F32) {
        epilogue_add<true>(taddr, ncols, f0 + q * 32, t0, q, &tmC, sOut, chunk_ctr, un, static_cast<int>(rank), ep,
                           s_flag);
      } else if constexpr (EPI == EPI_SWIGLU) {
        epi_t_swiglu(taddr, ncols, t0, M, (f0 + q * 32) / 2, sOut + q * 1024, ep);
      } else if constexpr (EPI == EPI_QKV) {
        epi_t_qkv(taddr, ncols, t0, M, f0 / 128, q, sOut, chunk_ctr, pre, ep);
      }
      tc_fence_before();
      release_acc<true>(tempty, acc, leader_tempty);
    }
    if constexpr (EPI == EPI_ADD_F32) {
      if (lane == 0) bulk_wait<0>();
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
  if (ep.ready && threadIdx.x == 0) {  // the last CTA to finish zeroes the token-tile counters
    __threadfence();
    if (atomicAdd(ep.ready + 4, 1) == static_cast<int>(gridDim.x) - 1) {
#pragma unroll
      for (int i = 0; i < 5; ++i) atomicExch(ep.ready + i, 0);
      __threadfence();
    }
  }
}

// split-K: minimise waves * (k-blocks per unit + ~6 k-blocks of fixed per-unit cost) + the ordered
// sum of the partial tiles (deterministic mode: ~16 k-blocks of workspace round trips at the end),
// within the workspace (tiles * 2 halves * splits slots)
int choose_splits(int64_t tiles, int nk, int workers, const EpiArgs& ep) {
  if (ep.ws == nullptr && ep.det) return 1;
  auto cost = [&](int sp) {
    const int64_t units = tiles * sp;
    return ((units + workers - 1) / workers) * ((nk + sp - 1) / sp + 6) + (sp > 1 && ep.det ? 16 : 0);
  };
  int splits = 1;
  int64_t best = cost(1);
  for (int sp = 2; sp <= 16 && nk / sp >= 8; ++sp) {
    if (ep.det && tiles * 2 * sp > ep.ws_slots) break;
    if (cost(sp) * 100 < best * 95) { best = cost(sp); splits = sp; }
  }
  return splits;
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
  if (EPI == EPI_ADD_F32 && (ep.ws != nullptr || !ep.det)) {
    static const bool sk_on = [] { const char* e = std::getenv("RC_GEMM_STREAMK"); return !(e && std::atoi(e) == 0); }();
    const int rem = tiles % pairs;
    const int64_t w = static_cast<int64_t>(rem) * nk;
    const int P = static_cast<int>(std::min<int64_t>(pairs, w));
    const int maxseg = P > 0 ? (P + rem - 1) / rem + 1 : 0;
    if (sk_on && tiles > pairs && rem != 0 && (!ep.det || rem * 2 * maxseg <= ep.ws_slots)) {
      // whole tiles round-robin, the partial last wave cut into equal k-block ranges: e.g. cfg3
      // batch 32, 1264 tiles on 74 pairs = 17 full waves + 6 tiles spread over all 74 pairs instead
      // of an 18th wave on 6 of them
      sk_tiles = rem;
    } else {
      splits = choose_splits(tiles, nk, pairs, ep);
    }
  }
  const int units = tiles * splits;
  const int grid = 2 * (units < pairs ? units : pairs);
  static const size_t group_a_bytes = [] {
    const char* e = std::getenv("RC_GROUP_A_MB");
    return e ? static_cast<size_t>(std::atoi(e)) << 20 : GROUP_A_BYTES;
  }();
  int group_m = static_cast<int>(std::max<size_t>(
      2, std::min<size_t>(num_m, group_a_bytes / (static_cast<size_t>(2 * BM) * K * 2))));
  {  // raster by estimated DRAM traffic: m-groups re-read B once per group, n-groups re-read A
    // RC_GEMM_RASTER: 0 = m-groups, 1 = n-groups, -1 (default) = n-groups for the residual projections
    // when the estimate favours them. Measured at cfg3 batch 32 (ncu): O-proj + down 3.05 -> 2.31 GB DRAM
    // per launch and 110.2 -> 106.6 ms over 1.5 steps, while gate/up got worse (2.95 -> 4.64 GB, 159.9 ->
    // 165.9 ms); L2 eviction-priority hints on top (evict_last weights, evict_first activations; removed)
    // made every class worse: the activation lines left L2 before the group's other n-tiles read them
    static const int raster = [] { const char* e = std::getenv("RC_GEMM_RASTER"); return e ? std::atoi(e) : -1; }();
    static const size_t group_b_bytes = [] {
      const char* e = std::getenv("RC_GROUP_B_MB");
      return e ? static_cast<size_t>(std::atoi(e)) << 20 : GROUP_B_BYTES;
    }();
    const int num_n = (N + 255) / 256;
    const double band = 256.0 * K * 2;  // bytes of one 256-row band of A or B
    const int gn = static_cast<int>(std::max<size_t>(1, std::min<size_t>(num_n, group_b_bytes / static_cast<size_t>(band))));
    const double tm = band * (num_m + num_n * double((num_m + group_m - 1) / group_m));
    const double tn = band * (num_n + num_m * double((num_n + gn - 1) / gn));
    if (raster == 1 || (raster == -1 && EPI == EPI_ADD_F32 && tn < 0.8 * tm)) group_m = -gn;
  }
  return launch_pdl(k_gemm_pair<EPI>, dim3(grid), dim3(256), C::SMEM, s, *a, *b, c ? *c : *a, M, N, K, splits,
                    group_m, sk_tiles, ep);
}

template <int EPI>
cudaError_t launch_t(const CUtensorMap* w, const CUtensorMap* x128, const CUtensorMap* x64, const CUtensorMap* c, int M,
                     int N, int K, const EpiArgs& ep, int num_sms, cudaStream_t s) {
  using C = TCfg;
  if (EPI == EPI_ADD_F32 && c == nullptr) return cudaErrorInvalidValue;
  if (cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(k_gemm_t<EPI>), C::SMEM); e != cudaSuccess) return e;
  const int pairs = num_sms / 2;
  const int ntt = (M + 255) / 256;
  const int tiles = (N / 256) * ntt;
  const int nk = (K + BK - 1) / BK;
  static const int max_splits = [] { const char* e = std::getenv("RC_GEMM_T_SPLITS"); return e ? std::atoi(e) : 16; }();
  const int splits = EPI == EPI_ADD_F32 ? std::min(max_splits, choose_splits(tiles, nk, pairs, ep)) : 1;
  const int units = tiles * splits;
  const int grid = 2 * (units < pairs ? units : pairs);
  return launch_pdl(k_gemm_t<EPI>, dim3(grid), dim3(256), C::SMEM, s, *w, *x128, *x64, c ? *c : *w, M, N, K, splits,
                    ep);
}

template <int BN, int EPI>
cudaError_t launch_one(const CUtensorMap* a, const CUtensorMap* b, const CUtensorMap* c, int M, int N, int K,
                       const EpiArgs& ep, int num_sms, cudaStream_t s) {
  if (EPI == EPI_ADD_F32 && c == nullptr) return cudaErrorInvalidValue;
  using C = GemmCfg<BN>;
  if (cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(k_gemm<BN, EPI>), C::SMEM); e != cudaSuccess) return e;
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int nk = (K + BK - 1) / BK;
  // split-K for the residual epilogue when the tile count fills the SMs badly (workspace slots are
  // counted as for the pair kernels: one CTA uses the rank-0 half)
  const int splits = EPI == EPI_ADD_F32 ? choose_splits(tiles, nk, num_sms, ep) : 1;
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

int gemm_ws_slots() { return 512; }
int gemm_t_box_rows() { return 64; }
size_t gemm_ws_floats() { return static_cast<size_t>(gemm_ws_slots()) * WS_TILE; }

// RC_GEMM_T: 0 never, 1 every eligible GEMM at any M, 2 every eligible GEMM at M <= 1024, 3 residual and
// SwiGLU at M <= 1024, 4 residual only; default: the residual GEMMs at M <= 1024 (where it measured faster than split-K
// CTA pairs at cfg3 batch 1) and the SwiGLU at M <= 512. SwiGLU, cfg3 batch-1 GEMM ms per step, default
// single-CTA vs transposed, two passes on one box (profiles/r02_ab_dispatch.sh): r = 5 % (M ~ 205)
// 6.40 / 6.27 vs 6.13 / 6.14, r = 10 % 8.38 / 8.41 vs 8.20 / 8.12, r = 15 % (M 625) 9.37 / 9.41 vs
// 9.50 / 9.48, r = 20 % 13.80 / 13.79 vs 13.92 / 13.88
bool gemm_use_transposed(int M, int N, int epi, int head_dim, int num_sms) {
  static const int mode = [] { const char* e = std::getenv("RC_GEMM_T"); return e ? std::atoi(e) : -1; }();
  if (mode == 0 || M <= 0 || N % 256 || num_sms < 2) return false;
  if (!(epi == EPI_ADD_F32 || epi == EPI_SWIGLU || (epi == EPI_QKV && head_dim == 128))) return false;
  if (mode == 1) return true;
  if (mode == 2) return M <= 1024;
  if (mode == 3) return (epi == EPI_ADD_F32 || epi == EPI_SWIGLU) && M <= 1024;
  if (mode == 4) return epi == EPI_ADD_F32 && M <= 1024;  // the round-2 default before the SwiGLU rule (A/B)
  return (epi == EPI_ADD_F32 && M <= 1024) || (epi == EPI_SWIGLU && M <= 512);
}

cudaError_t gemm_launch(const CUtensorMap* a, const CUtensorMap* b, const CUtensorMap* c, int M, int N, int K, int bn,
                        int epi, const EpiArgs& ep_in, int num_sms, cudaStream_t s, const CUtensorMap* a64) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  EpiArgs ep = ep_in;
  static const int t_pack = [] { const char* e = std::getenv("RC_GEMM_T_PACK"); return e ? std::atoi(e) : 1; }();
  static const int no_epi = [] { const char* e = std::getenv("RC_GEMM_NOEPI"); return e ? std::atoi(e) : 0; }();
  ep.t_pack = t_pack;
  ep.no_epi = no_epi;
  // small M (one request's selected rows): the transposed pair kernel keeps every 256-row MMA full
  if (a64 != nullptr && bn == 256 && gemm_use_transposed(M, N, epi, ep.head_dim, num_sms)) {
    switch (epi) {
      case EPI_ADD_F32: return launch_t<EPI_ADD_F32>(b, a, a64, c, M, N, K, ep, num_sms, s);
      case EPI_SWIGLU: return launch_t<EPI_SWIGLU>(b, a, a64, c, M, N, K, ep, num_sms, s);
      case EPI_QKV: return launch_t<EPI_QKV>(b, a, a64, c, M, N, K, ep, num_sms, s);
      default: break;
    }
  }
  if (ep.ready != nullptr) return cudaErrorInvalidValue;  // early O-projection needs the transposed kernel
  // CTA pairs for 256-wide GEMMs with M >= 1024: at cfg3 batch 32 they lift the GEMMs from 0.92 to
  // 0.99 of the measured sustained peak. RC_GEMM_PAIR=0/1 forces.
  static const int pair_mode = [] { const char* e = std::getenv("RC_GEMM_PAIR"); return e ? std::atoi(e) : -1; }();
  // RC_GEMM_PAIR_MIN_M: the M from which the non-residual epilogues take CTA pairs (diagnostics)
  static const int pair_min_m = [] { const char* e = std::getenv("RC_GEMM_PAIR_MIN_M"); return e ? std::atoi(e) : 1024; }();
  const bool pair = pair_mode == 1 || (pair_mode == -1 && (M >= pair_min_m || (epi == EPI_ADD_F32 && M > 2 * BM)));
  if (pair && bn == 256 && M > BM && num_sms >= 2) {
    switch (epi) {
      case EPI_BF16: return launch_pair<EPI_BF16>(a, b, c, M, N, K, ep, num_sms, s);
      case EPI_F32: return launch_pair<EPI_F32>(a, b, c, M, N, K, ep, num_sms, s);
      case EPI_ADD_F32: return launch_pair<EPI_ADD_F32>(a, b, c, M, N, K, ep, num_sms, s);
      case EPI_SWIGLU: return launch_pair<EPI_SWIGLU>(a, b, c, M, N, K, ep, num_sms, s);
      case EPI_QKV: return launch_pair<EPI_QKV>(a, b, c, M, N, K, ep, num_sms, s);
      case EPI_DEV: return launch_pair<EPI_DEV>(a, b, c, M, N, K, ep, num_sms, s);
      case EPI_QKV_DEV: return launch_pair<EPI_QKV_DEV>(a, b, c, M, N, K, ep, num_sms, s);
      default: return cudaErrorInvalidValue;
    }
  }
#define RC_GEMM_CASE(BN_, E_) \
  if (bn == BN_ && epi == E_) return launch_one<BN_, E_>(a, b, c, M, N, K, ep, num_sms, s);
  RC_GEMM_CASE(256, EPI_BF16) RC_GEMM_CASE(256, EPI_F32) RC_GEMM_CASE(256, EPI_ADD_F32)
  RC_GEMM_CASE(256, EPI_SWIGLU) RC_GEMM_CASE(256, EPI_QKV) RC_GEMM_CASE(256, EPI_DEV)
  RC_GEMM_CASE(128, EPI_BF16) RC_GEMM_CASE(128, EPI_F32) RC_GEMM_CASE(128, EPI_ADD_F32)
  RC_GEMM_CASE(128, EPI_QKV) RC_GEMM_CASE(128, EPI_DEV)
  RC_GEMM_CASE(256, EPI_QKV_DEV) RC_GEMM_CASE(128, EPI_QKV_DEV)
#undef RC_GEMM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace rc
