// K4/K7: causal attention of a set of query tokens over the stitched KV of their request
// (Eq. 1; reading R11: every selected query
// attends to ALL stitched keys at positions <= its own).
//
// One kernel serves both the dense layers l < c (queries = all of U) and the selective layers
// (queries = Sel): queries are rows with explicit positions, keys are the request's contiguous
// stitched rows [0, max_pos]. A CTA owns one (query tile, kv head): TQ tokens x G grouped query
// heads = 64 rows (GQA packing, G = H/H_kv; G = 7 gives 9 tokens = 63 rows). Flash-style
// online softmax in fp32 registers; S = Q K^T and O = P V on bf16 mma.sync m16n8k16 (v1 of
// this kernel; the tcgen05/TMEM version is the planned replacement).
#include "common.cuh"
#include "rc_internal.h"

namespace rc {
namespace {

constexpr int ROWS = 64, BKV = 64;

template <int DH>
struct AttnCfg {
  static constexpr int CPR = DH / 8;  // 16-byte chunks per row
  static constexpr int SWM = (CPR >= 8 ? 8 : CPR) - 1;
  static constexpr int SWS = (CPR >= 8) ? 0 : (CPR == 4 ? 1 : 2);
  static constexpr int TILE_BYTES = BKV * DH * 2;
  static constexpr int SMEM = ROWS * DH * 2 + 4 * TILE_BYTES;
};

template <int DH>
__device__ __forceinline__ uint32_t swz_off(int row, int chunk) {
  using C = AttnCfg<DH>;
  return static_cast<uint32_t>(row * DH * 2 + ((chunk ^ ((row >> C::SWS) & C::SWM)) << 4));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int DH>
__global__ void __launch_bounds__(128) k_attn(const AttnArgs a) {
  griddep_wait();  // PDL: inputs of the previous kernel are complete and visible
  griddep_launch();
  using C = AttnCfg<DH>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sK = smem + ROWS * DH * 2;          // [2][BKV][DH]
  uint8_t* sV = sK + 2 * C::TILE_BYTES;        // [2][BKV][DH]

  const int4 tile = a.tiles[blockIdx.x];
  const int row_start = tile.x, n_rows = tile.y, kv_base = tile.z;
  const int kvh = blockIdx.y;
  const int G = a.n_heads / a.n_kv_heads;
  const int TQ = ROWS / G;
  const int H = a.n_heads;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int max_pos = a.qpos[row_start + n_rows - 1];  // query rows are sorted by position
  const int n_kb = max_pos / BKV + 1;
  const uint16_t* kbase = a.k + static_cast<int64_t>(kvh) * a.head_stride + static_cast<int64_t>(kv_base) * DH;
  const uint16_t* vbase = a.v + static_cast<int64_t>(kvh) * a.head_stride + static_cast<int64_t>(kv_base) * DH;

  // ---- Q tile -> smem (rows r = token * G + head-in-group)
  for (int i = tid; i < ROWS * C::CPR; i += 128) {
    const int r = i / C::CPR, ch = i % C::CPR;
    const int t = r / G;
    const bool ok = (r < TQ * G) && (t < n_rows);
    const uint16_t* src = a.q;
    if (ok) src = a.q + static_cast<int64_t>(row_start + t) * H * DH + (kvh * G + r % G) * DH + ch * 8;
    cp_async16(sQ + swz_off<DH>(r, ch), src, ok);
  }
  auto load_kv = [&](int kb, int buf) {
    for (int i = tid; i < BKV * C::CPR; i += 128) {
      const int r = i / C::CPR, ch = i % C::CPR;
      const int key = kb * BKV + r;
      const bool ok = key <= max_pos;
      const int64_t off = static_cast<int64_t>(ok ? key : 0) * DH + ch * 8;
      cp_async16(sK + buf * C::TILE_BYTES + swz_off<DH>(r, ch), kbase + off, ok);
      cp_async16(sV + buf * C::TILE_BYTES + swz_off<DH>(r, ch), vbase + off, ok);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  // per-thread rows and their positions
  const int r0 = warp * 16 + (lane >> 2), r1 = r0 + 8;
  int p0 = -1, p1 = -1;
  if (r0 < TQ * G && r0 / G < n_rows) p0 = a.qpos[row_start + r0 / G];
  if (r1 < TQ * G && r1 / G < n_rows) p1 = a.qpos[row_start + r1 / G];

  float o[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  uint32_t qf[DH / 16][4];

  for (int kb = 0; kb < n_kb; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < n_kb) load_kv(kb + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk) {
        const int row = warp * 16 + (lane & 15);
        const int ch = kk * 2 + (lane >> 4);
        ldsm_x4(smem_u32(sQ + swz_off<DH>(row, ch)), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    const uint32_t kS = smem_u32(sK + buf * C::TILE_BYTES);
    const uint32_t vS = smem_u32(sV + buf * C::TILE_BYTES);
    float s[BKV / 8][4];
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
      for (int nt = 0; nt < BKV / 16; ++nt) {
        const int key = nt * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int ch = kk * 2 + ((lane >> 3) & 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kS + swz_off<DH>(key, ch), b0, b1, b2, b3);
        mma16816(s[2 * nt], qf[kk], b0, b1);
        mma16816(s[2 * nt + 1], qf[kk], b2, b3);
      }
    }
    // scale, causal mask by true position, online softmax (base 2)
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j) {
      const int key = kb * BKV + j * 8 + 2 * (lane & 3);
      s[j][0] = (key <= p0) ? s[j][0] * a.scale_log2 : -INFINITY;
      s[j][1] = (key + 1 <= p0) ? s[j][1] * a.scale_log2 : -INFINITY;
      s[j][2] = (key <= p1) ? s[j][2] * a.scale_log2 : -INFINITY;
      s[j][3] = (key + 1 <= p1) ? s[j][3] * a.scale_log2 : -INFINITY;
      mx0 = fmaxf(mx0, fmaxf(s[j][0], s[j][1]));
      mx1 = fmaxf(mx1, fmaxf(s[j][2], s[j][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float base0 = (mn0 == -INFINITY) ? 0.f : mn0;
    const float base1 = (mn1 == -INFINITY) ? 0.f : mn1;
    const float al0 = exp2f(m0 - base0), al1 = exp2f(m1 - base1);
    m0 = mn0; m1 = mn1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j) {
      s[j][0] = exp2f(s[j][0] - base0); s[j][1] = exp2f(s[j][1] - base0);
      s[j][2] = exp2f(s[j][2] - base1); s[j][3] = exp2f(s[j][3] - base1);
      rs0 += s[j][0] + s[j][1];
      rs1 += s[j][2] + s[j][3];
    }
    l0 = l0 * al0 + rs0;
    l1 = l1 * al1 + rs1;
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) { o[i][0] *= al0; o[i][1] *= al0; o[i][2] *= al1; o[i][3] *= al1; }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < BKV / 16; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_bf2(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack_bf2(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack_bf2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack_bf2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int dt = 0; dt < DH / 16; ++dt) {
        const int key = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int ch = dt * 2 + (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vS + swz_off<DH>(key, ch), b0, b1, b2, b3);
        mma16816(o[2 * dt], pa, b0, b1);
        mma16816(o[2 * dt + 1], pa, b2, b3);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  l0 += __shfl_xor_sync(0xffffffff, l0, 1);
  l0 += __shfl_xor_sync(0xffffffff, l0, 2);
  l1 += __shfl_xor_sync(0xffffffff, l1, 1);
  l1 += __shfl_xor_sync(0xffffffff, l1, 2);
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
  if (p0 >= 0) {
    uint16_t* dst = a.o + static_cast<int64_t>(row_start + r0 / G) * H * DH + (kvh * G + r0 % G) * DH;
#pragma unroll
    for (int i = 0; i < DH / 8; ++i)
      *reinterpret_cast<uint32_t*>(dst + i * 8 + 2 * (lane & 3)) = pack_bf2(o[i][0] * inv0, o[i][1] * inv0);
  }
  if (p1 >= 0) {
    uint16_t* dst = a.o + static_cast<int64_t>(row_start + r1 / G) * H * DH + (kvh * G + r1 % G) * DH;
#pragma unroll
    for (int i = 0; i < DH / 8; ++i)
      *reinterpret_cast<uint32_t*>(dst + i * 8 + 2 * (lane & 3)) = pack_bf2(o[i][2] * inv1, o[i][3] * inv1);
  }
}

template <int DH>
cudaError_t launch(const AttnArgs& a, cudaStream_t s) {
  using C = AttnCfg<DH>;
  if (cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(k_attn<DH>), C::SMEM); e != cudaSuccess) return e;
  dim3 grid(a.n_tiles, a.n_kv_heads);
  return launch_pdl(k_attn<DH>, dim3(grid), dim3(128), C::SMEM, s, a);
}
}  // namespace

int attn_tokens_per_tile(int group) { return ROWS / group; }

cudaError_t attn_launch(const AttnArgs& a, cudaStream_t s) {
  if (a.n_tiles <= 0) return cudaSuccess;
  if (a.n_heads % a.n_kv_heads != 0 || a.n_heads / a.n_kv_heads > ROWS) return cudaErrorInvalidValue;
  switch (a.head_dim) {
    case 16: return launch<16>(a, s);
    case 64: return launch<64>(a, s);
    case 128: return launch<128>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rc
