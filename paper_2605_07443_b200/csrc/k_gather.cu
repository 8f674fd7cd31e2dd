// K2: assemble gather -- pool blocks -> request-owned stitched KV, with int8 dequantisation and
// Delta-RoPE fused into the copy.
//
// Pools and the stitched arena share one HBM layout: for every plane (layer l, K/V, kv-head h) a
// dense [rows][d_h] matrix, so an item's tokens are contiguous 2*d_h-byte rows and a request's
// stitched KV for one plane is one contiguous run of rows. Grid = (token blocks, layer x K/V): a
// thread unit is (token, pair-chunk) -- 8 elements of the low half of a rotate-half pair and the
// matching 8 of the high half -- applied to every KV head of that (layer, K/V), so the token's
// metadata and its fp32 cos/sin are loaded once for H_kv planes; per head two 16-byte loads
// (bf16) or two 8-byte loads (int8) and two 16-byte stores, 4 heads' loads in flight at a time;
// consecutive threads walk chunks then tokens (coalesced 256 B rows).
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

// One thread unit = (token, pair-chunk) of one (layer, K/V): the token's metadata and, for K, the
// fp32 cos/sin of its Delta are loaded once and applied to the same chunk of every KV head (the
// planes of one (layer, K/V) share the rotation), so table and metadata traffic drop by H_kv.
// Heads are processed HB at a time with all their loads issued first.
template <int DH>
__global__ void __launch_bounds__(256) k_gather(const GatherArgs g) {
  griddep_wait();  // PDL: inputs of the previous kernel are complete and visible
  griddep_launch();
  constexpr int HALF = DH / 2, CPR = DH / 16, HB = 4;
  const int Hk = g.n_kv_heads;
  const int lk = blockIdx.y;                 // (l - layer_begin, kv)
  const int kv = lk & 1;
  const int l = g.layer_begin + (lk >> 1);
  if (l >= g.layer_end) return;
  const int64_t plane0 = (static_cast<int64_t>(l) * 2 + kv) * Hk;  // plane of head 0
  const int units = g.n_tok * CPR;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < units; u += gridDim.x * blockDim.x) {
    const int t = u / CPR;
    const int j = (u % CPR) * 8;
    const int4 m = __ldg(&g.meta[t]);
    if (m.w == KIND_FORCED) continue;  // recomputed later
    if (g.skip_pool_v && kv == 1 && (m.w == KIND_ITEM || m.w == KIND_PREFIX)) continue;  // read in place (vmap)
    const bool rot = kv == 0 && (m.w == KIND_ITEM || m.w == KIND_HIST);
    float cc[8], ss[8];
    if (rot) {
      const float* cs = g.rope_cos + static_cast<int64_t>(m.z + g.rope_zero) * HALF + j;
      const float* sn = g.rope_sin + static_cast<int64_t>(m.z + g.rope_zero) * HALF + j;
      const float4 c0 = __ldg(reinterpret_cast<const float4*>(cs)), c1 = __ldg(reinterpret_cast<const float4*>(cs + 4));
      const float4 s0 = __ldg(reinterpret_cast<const float4*>(sn)), s1 = __ldg(reinterpret_cast<const float4*>(sn + 4));
      cc[0] = c0.x; cc[1] = c0.y; cc[2] = c0.z; cc[3] = c0.w; cc[4] = c1.x; cc[5] = c1.y; cc[6] = c1.z; cc[7] = c1.w;
      ss[0] = s0.x; ss[1] = s0.y; ss[2] = s0.z; ss[3] = s0.w; ss[4] = s1.x; ss[5] = s1.y; ss[6] = s1.z; ss[7] = s1.w;
    }
    for (int h0 = 0; h0 < Hk; h0 += HB) {
      uint4 ra[HB], rb[HB];
      float sc[HB];
#pragma unroll
      for (int k = 0; k < HB; ++k) {  // issue every load of this head block first
        const int h = h0 + k;
        if (h >= Hk) break;
        const int64_t plane = plane0 + h;
        if (m.w == KIND_PREFIX || m.w == KIND_ITEM) {
          const uint16_t* src = (m.w == KIND_PREFIX ? g.prefix_pool + plane * g.prefix_rows * DH
                                                    : g.item_pool + plane * g.item_rows * DH) +
                                static_cast<int64_t>(m.y) * DH;
          ra[k] = __ldg(reinterpret_cast<const uint4*>(src + j));
          rb[k] = __ldg(reinterpret_cast<const uint4*>(src + HALF + j));
        } else {  // KIND_HIST: int8 codes + fp32 scale
          const int8_t* src = g.hist_q + (plane * g.hist_rows + m.y) * DH;
          const uint2 qa = __ldg(reinterpret_cast<const uint2*>(src + j));
          const uint2 qb = __ldg(reinterpret_cast<const uint2*>(src + HALF + j));
          ra[k] = make_uint4(qa.x, qa.y, 0, 0);
          rb[k] = make_uint4(qb.x, qb.y, 0, 0);
          sc[k] = __ldg(&g.hist_s[plane * g.hist_rows + m.y]);
        }
      }
#pragma unroll
      for (int k = 0; k < HB; ++k) {
        const int h = h0 + k;
        if (h >= Hk) break;
        uint16_t* dst = g.arena + ((plane0 + h) * g.arena_rows + m.x) * DH;
        if (m.w == KIND_PREFIX || (m.w == KIND_ITEM && kv == 1)) {  // byte copy
          *reinterpret_cast<uint4*>(dst + j) = ra[k];
          *reinterpret_cast<uint4*>(dst + HALF + j) = rb[k];
          continue;
        }
        float x0[8], x1[8];
        if (m.w == KIND_ITEM) {
          unpack8_bf16(ra[k], x0);
          unpack8_bf16(rb[k], x1);
        } else {
          const int8_t* pa = reinterpret_cast<const int8_t*>(&ra[k]);
          const int8_t* pb = reinterpret_cast<const int8_t*>(&rb[k]);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            x0[i] = __fmul_rn(static_cast<float>(pa[i]), sc[k]);
            x1[i] = __fmul_rn(static_cast<float>(pb[i]), sc[k]);
          }
        }
        if (rot) {
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
}

template <int DH>
cudaError_t launch(const GatherArgs& g, int num_sms, cudaStream_t s) {
  const int lk = (g.layer_end - g.layer_begin) * 2;
  const int64_t units = static_cast<int64_t>(g.n_tok) * (DH / 16);
  static int per_sm = 0;
  if (per_sm == 0 && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather<DH>, 256, 0) != cudaSuccess)
    per_sm = 2;
  int64_t bx = (units + 255) / 256;
  // >= 8 waves of resident CTAs in total so the per-(layer, K/V) tail is small
  const int64_t want = (static_cast<int64_t>(num_sms) * per_sm * 8 + lk - 1) / lk;
  if (bx > want) bx = want;
  if (bx < 1) bx = 1;
  return launch_pdl(k_gather<DH>, dim3(static_cast<unsigned>(bx), lk), dim3(256), 0, s, g);
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
