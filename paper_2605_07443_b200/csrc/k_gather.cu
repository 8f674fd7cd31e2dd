// K2: assemble gather -- pool blocks -> request-owned stitched KV, with int8 dequantisation and
// Delta-RoPE fused into the copy.
//
// Pools and the stitched arena share one HBM layout: for every plane (layer l, K/V, kv-head h) a
// dense [rows][d_h] matrix, so an item's tokens are contiguous 2*d_h-byte rows and a request's
// stitched KV for one plane is one contiguous run of rows. Grid = (token blocks, planes): a CTA
// owns one plane and a strided set of tokens, so all index math is 32-bit and per-plane bases are
// computed once. Work unit = (token, pair-chunk): 8 elements of the low half of a rotate-half pair
// and the matching 8 of the high half -- two 16-byte loads (bf16) or two 8-byte loads (int8) and
// two 16-byte stores; consecutive threads walk chunks then tokens (coalesced 256 B rows). Each
// thread keeps UNROLL units in flight.
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
constexpr int UNROLL = 4;

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

struct Unit {
  uint4 a, b;      // raw loads (bf16: 8 elems each; int8: low 8 bytes used)
  float sc;
  int4 m;
  int j;
  bool live;
};

template <int DH>
__global__ void __launch_bounds__(256) k_gather(const GatherArgs g) {
  griddep_wait();  // PDL: inputs of the previous kernel are complete and visible
  griddep_launch();
  constexpr int HALF = DH / 2, CPR = DH / 16;
  const int nl = g.layer_end - g.layer_begin;
  const int Hk = g.n_kv_heads;
  const int plane_rel = blockIdx.y;                    // (l - layer_begin, kv, h)
  const int h = plane_rel % Hk;
  const int kv = (plane_rel / Hk) & 1;
  const int l = g.layer_begin + plane_rel / (2 * Hk);
  if (l >= g.layer_end) return;
  (void)nl;
  const int64_t plane = (static_cast<int64_t>(l) * 2 + kv) * Hk + h;
  const uint16_t* item_base = g.item_pool + plane * g.item_rows * DH;
  const uint16_t* pre_base = g.prefix_pool + plane * g.prefix_rows * DH;
  const int8_t* hq_base = g.hist_q + plane * g.hist_rows * DH;
  const float* hs_base = g.hist_s + plane * g.hist_rows;
  uint16_t* dst_base = g.arena + plane * g.arena_rows * DH;
  const int units = g.n_tok * CPR;
  const int stride = gridDim.x * blockDim.x;
  for (int u0 = blockIdx.x * blockDim.x + threadIdx.x; u0 < units; u0 += stride * UNROLL) {
    Unit w[UNROLL];
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {  // issue all loads first
      const int u = u0 + k * stride;
      w[k].live = u < units;
      if (!w[k].live) continue;
      const int t = u / CPR;
      w[k].j = (u % CPR) * 8;
      w[k].m = __ldg(&g.meta[t]);
      const int4 m = w[k].m;
      const int j = w[k].j;
      if (m.w == KIND_PREFIX || m.w == KIND_ITEM) {
        const uint16_t* src = (m.w == KIND_PREFIX ? pre_base : item_base) + static_cast<int64_t>(m.y) * DH;
        w[k].a = __ldg(reinterpret_cast<const uint4*>(src + j));
        w[k].b = __ldg(reinterpret_cast<const uint4*>(src + HALF + j));
      } else if (m.w == KIND_HIST) {
        const int8_t* src = hq_base + static_cast<int64_t>(m.y) * DH;
        const uint2 qa = __ldg(reinterpret_cast<const uint2*>(src + j));
        const uint2 qb = __ldg(reinterpret_cast<const uint2*>(src + HALF + j));
        w[k].a = make_uint4(qa.x, qa.y, 0, 0);
        w[k].b = make_uint4(qb.x, qb.y, 0, 0);
        w[k].sc = __ldg(&hs_base[m.y]);
      } else {
        w[k].live = false;  // FORCED: recomputed later
      }
    }
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      if (!w[k].live) continue;
      const int4 m = w[k].m;
      const int j = w[k].j;
      uint16_t* dst = dst_base + static_cast<int64_t>(m.x) * DH;
      if (m.w == KIND_PREFIX || (m.w == KIND_ITEM && kv == 1)) {
        *reinterpret_cast<uint4*>(dst + j) = w[k].a;
        *reinterpret_cast<uint4*>(dst + HALF + j) = w[k].b;
        continue;
      }
      float x0[8], x1[8];
      if (m.w == KIND_ITEM) {
        unpack8_bf16(w[k].a, x0);
        unpack8_bf16(w[k].b, x1);
      } else {
        const int8_t* pa = reinterpret_cast<const int8_t*>(&w[k].a);
        const int8_t* pb = reinterpret_cast<const int8_t*>(&w[k].b);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          x0[i] = __fmul_rn(static_cast<float>(pa[i]), w[k].sc);
          x1[i] = __fmul_rn(static_cast<float>(pb[i]), w[k].sc);
        }
      }
      if (kv == 0) {
        const float* cs = g.rope_cos + static_cast<int64_t>(m.z + g.rope_zero) * HALF + j;
        const float* sn = g.rope_sin + static_cast<int64_t>(m.z + g.rope_zero) * HALF + j;
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
        *reinterpret_cast<uint4*>(dst + HALF + j) = pack8_bf16(y1);
      } else {
        *reinterpret_cast<uint4*>(dst + j) = pack8_bf16(x0);
        *reinterpret_cast<uint4*>(dst + HALF + j) = pack8_bf16(x1);
      }
    }
  }
}

template <int DH>
cudaError_t launch(const GatherArgs& g, int num_sms, cudaStream_t s) {
  const int planes = (g.layer_end - g.layer_begin) * 2 * g.n_kv_heads;
  const int64_t units = static_cast<int64_t>(g.n_tok) * (DH / 16);
  // one full wave of resident CTAs over all planes, each thread holding UNROLL units in flight
  static int per_sm = 0;
  if (per_sm == 0 && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather<DH>, 256, 0) != cudaSuccess)
    per_sm = 2;
  int64_t bx = (units + 256 * UNROLL - 1) / (256 * UNROLL);
  // >= 8 waves of resident CTAs in total so the per-plane tail is small
  const int64_t want = (static_cast<int64_t>(num_sms) * per_sm * 8 + planes - 1) / planes;
  if (bx > want) bx = want;
  if (bx < 1) bx = 1;
  return launch_pdl(k_gather<DH>, dim3(static_cast<unsigned>(bx), planes), dim3(256), 0, s, g);
}
}  // namespace

cudaError_t gather_launch(const GatherArgs& g, int num_sms, cudaStream_t s) {
  if (g.n_tok <= 0 || g.layer_end <= g.layer_begin) return cudaSuccess;
  switch (g.head_dim) {
    case 16: return launch<16>(g, num_sms, s);
    case 64: return launch<64>(g, num_sms, s);
    case 128: return launch<128>(g, num_sms, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rc
