// K2: assemble gather -- pool blocks -> request-owned stitched KV, with int8 dequantisation and
// Delta-RoPE fused into the copy.
//
// Pools and the stitched arena share one HBM layout: for every (layer l, K/V, kv-head h) a
// dense [rows][d_h] matrix, so an item's tokens are contiguous 2*d_h-byte rows and a request's
// stitched KV for one (l, K/V, h) is one contiguous run of rows. Work unit = (layer, K/V, head,
// token, pair-chunk): 8 elements of the low half and the matching 8 of the high half of a
// rotate-half pair, i.e. two 16-byte loads (bf16) or two 8-byte loads (int8) and two 16-byte
// stores. Consecutive threads walk consecutive chunks, then tokens: fully coalesced rows.
//
// Arithmetic (bit-exact against oracle/assemble.py):
//   deq(q) = __fmul_rn(float(q), scale)
//   y0 = __fsub_rn(__fmul_rn(x0, c), __fmul_rn(x1, s)),  y1 = __fadd_rn(__fmul_rn(x1, c), __fmul_rn(x0, s))
//   stored = bf16 RNE; V of items and all PREFIX rows are copied byte for byte.
#include "common.cuh"
#include "rc_internal.h"

namespace rc {
namespace {

enum { KIND_PREFIX = 0, KIND_FORCED = 1, KIND_HIST = 2, KIND_ITEM = 3 };

__device__ __forceinline__ void unpack8_bf16(const uint4 u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ uint4 pack8_bf16(const float* f) {
  uint4 u;
  u.x = pack_bf2(f[0], f[1]); u.y = pack_bf2(f[2], f[3]); u.z = pack_bf2(f[4], f[5]); u.w = pack_bf2(f[6], f[7]);
  return u;
}

__global__ void __launch_bounds__(256) k_gather(const GatherArgs g) {
  const int dh = g.head_dim, half = dh / 2;
  const int cpr = dh / 16;  // pair-chunks per row
  const int Hk = g.n_kv_heads;
  const int nl = g.layer_end - g.layer_begin;
  const int64_t units = static_cast<int64_t>(nl) * 2 * Hk * g.n_tok * cpr;
  for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < units;
       u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(u % cpr);
    int64_t r = u / cpr;
    const int t = static_cast<int>(r % g.n_tok);
    r /= g.n_tok;
    const int h = static_cast<int>(r % Hk);
    r /= Hk;
    const int kv = static_cast<int>(r & 1);
    const int l = g.layer_begin + static_cast<int>(r >> 1);
    const int4 m = __ldg(&g.meta[t]);  // {dst_row, src_row, delta, kind}
    const int64_t plane = (static_cast<int64_t>(l) * 2 + kv) * Hk + h;
    const int j = c * 8;
    uint16_t* dst = g.arena + (plane * g.arena_rows + m.x) * dh;
    if (m.w == KIND_PREFIX || (m.w == KIND_ITEM && kv == 1)) {
      const uint16_t* src = (m.w == KIND_PREFIX ? g.prefix_pool + (plane * g.prefix_rows + m.y) * dh
                                                : g.item_pool + (plane * g.item_rows + m.y) * dh);
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(src + j));
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(src + half + j));
      *reinterpret_cast<uint4*>(dst + j) = a;
      *reinterpret_cast<uint4*>(dst + half + j) = b;
      continue;
    }
    float x0[8], x1[8];
    if (m.w == KIND_ITEM) {
      const uint16_t* src = g.item_pool + (plane * g.item_rows + m.y) * dh;
      unpack8_bf16(__ldg(reinterpret_cast<const uint4*>(src + j)), x0);
      unpack8_bf16(__ldg(reinterpret_cast<const uint4*>(src + half + j)), x1);
    } else if (m.w == KIND_HIST) {
      const int8_t* src = g.hist_q + (plane * g.hist_rows + m.y) * dh;
      const float sc = __ldg(&g.hist_s[plane * g.hist_rows + m.y]);
      const uint2 qa = __ldg(reinterpret_cast<const uint2*>(src + j));
      const uint2 qb = __ldg(reinterpret_cast<const uint2*>(src + half + j));
      const int8_t* pa = reinterpret_cast<const int8_t*>(&qa);
      const int8_t* pb = reinterpret_cast<const int8_t*>(&qb);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        x0[i] = __fmul_rn(static_cast<float>(pa[i]), sc);
        x1[i] = __fmul_rn(static_cast<float>(pb[i]), sc);
      }
    } else {
      continue;  // FORCED: recomputed later
    }
    if (kv == 0) {
      const float* cs = g.rope_cos + static_cast<int64_t>(m.z + g.rope_zero) * half + j;
      const float* sn = g.rope_sin + static_cast<int64_t>(m.z + g.rope_zero) * half + j;
      const float4 c0 = __ldg(reinterpret_cast<const float4*>(cs)), c1 = __ldg(reinterpret_cast<const float4*>(cs + 4));
      const float4 s0 = __ldg(reinterpret_cast<const float4*>(sn)), s1 = __ldg(reinterpret_cast<const float4*>(sn + 4));
      const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      const float ss[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
      float y0[8], y1[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        y0[i] = __fsub_rn(__fmul_rn(x0[i], cc[i]), __fmul_rn(x1[i], ss[i]));
        y1[i] = __fadd_rn(__fmul_rn(x1[i], cc[i]), __fmul_rn(x0[i], ss[i]));
      }
      *reinterpret_cast<uint4*>(dst + j) = pack8_bf16(y0);
      *reinterpret_cast<uint4*>(dst + half + j) = pack8_bf16(y1);
    } else {
      *reinterpret_cast<uint4*>(dst + j) = pack8_bf16(x0);
      *reinterpret_cast<uint4*>(dst + half + j) = pack8_bf16(x1);
    }
  }
}
}  // namespace

cudaError_t gather_launch(const GatherArgs& g, int num_sms, cudaStream_t s) {
  if (g.n_tok <= 0 || g.layer_end <= g.layer_begin) return cudaSuccess;
  if (g.head_dim % 16 != 0) return cudaErrorInvalidValue;
  const int64_t units = static_cast<int64_t>(g.layer_end - g.layer_begin) * 2 * g.n_kv_heads * g.n_tok * (g.head_dim / 16);
  int64_t blocks = (units + 255) / 256;
  const int64_t cap = static_cast<int64_t>(num_sms) * 8;
  if (blocks > cap) blocks = cap;
  k_gather<<<static_cast<int>(blocks), 256, 0, s>>>(g);
  return cudaGetLastError();
}

}  // namespace rc
