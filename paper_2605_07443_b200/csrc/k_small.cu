// Small bandwidth / latency-bound kernels of the hot path:
//   embed       a2: x[U] = E[t]  (fp32 residual stream, R22)
//   rmsnorm     a2/a5/a7/a8: bf16(x / sqrt(mean(x^2) + eps) * g)
//   select      a4 (K6): per-request, per-class top-k by the R6 key via 8-bit radix select,
//               union FORCED and window, compaction in position order
//   gather_rows a4: x_sel = x[Sel]
//   cand_scores a8: score_c = logits[idtok_c] (R19)
// plus pool registration transposes, the NVLink / loopback fetch copy and a diagnostic reader.
#include "common.cuh"
#include "rc_internal.h"

namespace rc {
namespace {

enum { CLS_PREFIX = 0, CLS_FORCED = 1, CLS_HIST = 2, CLS_ITEM = 3 };

__global__ void k_embed(const uint16_t* __restrict__ emb, const int32_t* __restrict__ tok, int32_t rows, int32_t d,
                        float* __restrict__ x) {
  griddep_wait();  // PDL: inputs of the previous kernel are complete and visible
  griddep_launch();
  const int64_t n8 = static_cast<int64_t>(rows) * (d / 8);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / (d / 8);
    const int c = static_cast<int>(i % (d / 8)) * 8;
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(emb + static_cast<int64_t>(tok[r]) * d + c));
    float4 a = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                           __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
    float4 b = make_float4(__uint_as_float(u.z << 16), __uint_as_float(u.z & 0xFFFF0000u),
                           __uint_as_float(u.w << 16), __uint_as_float(u.w & 0xFFFF0000u));
    float4* dst = reinterpret_cast<float4*>(x + r * d + c);
    dst[0] = a;
    dst[1] = b;
  }
}

// One CTA per row; the row stays in registers between the sum of squares and the scaled write
// (V float4 per thread, one load round trip). Same summation order as a strided loop.
template <int V>
__global__ void __launch_bounds__(256) k_rmsnorm(const float* __restrict__ x, const int32_t* __restrict__ row_idx,
                                                 int32_t d, const uint16_t* __restrict__ g, float eps,
                                                 uint16_t* __restrict__ out) {
  __shared__ float red[8];
  const int r = blockIdx.x;
  const uint2* grow = reinterpret_cast<const uint2*>(g);
  const int n4 = d / 4;
  float4 v[V];
  uint2 gg[V];
  // the gains are weights (not produced by the previous kernel): fetched while it drains (PDL)
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    gg[k] = i < n4 ? __ldg(&grow[i]) : make_uint2(0u, 0u);
  }
  griddep_wait();  // PDL: inputs of the previous kernel are complete and visible
  griddep_launch();
  const int64_t src = row_idx ? row_idx[r] : r;
  const float4* xr = reinterpret_cast<const float4*>(x + src * d);
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    v[k] = i < n4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < V; ++k) ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
#pragma unroll
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffff, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / d + eps);
  uint2* orow = reinterpret_cast<uint2*>(out + static_cast<int64_t>(r) * d);
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i >= n4) break;
    uint2 o;
    o.x = pack_bf2(v[k].x * inv * __uint_as_float(gg[k].x << 16), v[k].y * inv * __uint_as_float(gg[k].x & 0xFFFF0000u));
    o.y = pack_bf2(v[k].z * inv * __uint_as_float(gg[k].y << 16), v[k].w * inv * __uint_as_float(gg[k].y & 0xFFFF0000u));
    orow[i] = o;
  }
}

__global__ void k_gather_rows(const float* __restrict__ src, const int32_t* __restrict__ idx, int32_t rows, int32_t d,
                              float* __restrict__ dst) {
  griddep_wait();  // PDL: inputs of the previous kernel are complete and visible
  griddep_launch();
  const int64_t n4 = static_cast<int64_t>(rows) * (d / 4);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / (d / 4);
    const int c = static_cast<int>(i % (d / 4));
    reinterpret_cast<float4*>(dst + r * d)[c] = reinterpret_cast<const float4*>(src + static_cast<int64_t>(idx[r]) * d)[c];
  }
}

// ----------------------------------------------------------------------------- K6 selection
constexpr int SEL_THREADS = 1024;
constexpr int SEL_MAX_U = 8192;

__device__ __forceinline__ unsigned long long sel_key(unsigned long long dev, int pos) {
  return (dev << 13) | static_cast<unsigned long long>(8191 - pos);  // R6: D desc, then pos asc
}

// Per request (one CTA): both classes' top-k by the unique R6 key in one 8-bit radix select (8
// passes over the key bytes, high to low; a histogram of each class's still-matching keys per pass,
// the digit that holds the k-th largest found with warp shuffles -- warp c scans class c's 256 bins
// as 8 per lane, a suffix sum across lanes); then the selected / FORCED flags are compacted in
// position order with a two-level warp-shuffle scan.
__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

__global__ void __launch_bounds__(SEL_THREADS) k_select(const SelectArgs a) {
  griddep_wait();  // PDL: inputs of the previous kernel are complete and visible
  griddep_launch();
  __shared__ uint8_t flag[SEL_MAX_U];
  __shared__ uint8_t cls[SEL_MAX_U];
  __shared__ int hist[2][256];
  __shared__ int sh_digit[2], sh_krem[2], sh_members[2];
  __shared__ int wsum[SEL_THREADS / 32];
  const int4 rq = a.req[blockIdx.x];
  const int4 rq2 = a.req2[blockIdx.x];
  const int u_off = rq.x, u_cnt = rq.y, sel_off = rq.z, n = rq.w;
  const int P = n - u_cnt;
  const int window = rq2.w;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 2) sh_members[tid] = 0;
  __syncthreads();
  int mh = 0, mi = 0;
  for (int i = tid; i < u_cnt; i += SEL_THREADS) {
    const int pos = P + i;
    int c = a.ucls[u_off + i];
    const bool in_win = window > 0 && pos >= n - window;
    if (in_win) c = CLS_FORCED;
    if (a.u2s && a.u2s[u_off + i] < 0) c = CLS_PREFIX;  // gradual step: outside the previous Sel
    cls[i] = static_cast<uint8_t>(c);
    flag[i] = (c == CLS_FORCED) ? 1 : 0;
    mh += c == CLS_HIST;
    mi += c == CLS_ITEM;
  }
  if (mh) atomicAdd(&sh_members[0], mh);
  if (mi) atomicAdd(&sh_members[1], mi);
  __syncthreads();
  const int kk[2] = {rq2.x, rq2.y};
  // a class needs the radix select only when its budget is positive and below its size
  const bool act0 = kk[0] > 0 && kk[0] < sh_members[0], act1 = kk[1] > 0 && kk[1] < sh_members[1];
  unsigned long long prefix[2] = {0ull, 0ull}, mask = 0ull;
  if (tid < 2) sh_krem[tid] = kk[tid];
  if (act0 || act1) {
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = tid; i < 512; i += SEL_THREADS) (&hist[0][0])[i] = 0;
      __syncthreads();
      for (int i = tid; i < u_cnt; i += SEL_THREADS) {
        const int c = cls[i] == CLS_HIST ? 0 : cls[i] == CLS_ITEM ? 1 : -1;
        if (c < 0 || !(c == 0 ? act0 : act1)) continue;
        const unsigned long long key = sel_key(a.dev[u_off + i], P + i);
        if ((key & mask) == prefix[c]) atomicAdd(&hist[c][(key >> shift) & 255], 1);
      }
      __syncthreads();
      if (warp < 2 && (warp == 0 ? act0 : act1)) {  // warp c: digit of class c's k-th largest key
        // lane l owns bins 255 - 8l .. 248 - 8l (high digits on low lanes: a prefix scan = from the top)
        int b[8], tot = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) { b[j] = hist[warp][255 - 8 * lane - j]; tot += b[j]; }
        const int incl = warp_incl_scan(tot);
        const int krem = sh_krem[warp];
        const int excl = incl - tot;
        const bool mine = excl < krem && incl >= krem;
        if (mine) {
          int cacc = excl, dgt = 0, kr = krem;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (cacc + b[j] >= krem) { dgt = 255 - 8 * lane - j; kr = krem - cacc; break; }
            cacc += b[j];
          }
          sh_digit[warp] = dgt;
          sh_krem[warp] = kr;
        }
      }
      __syncthreads();
      prefix[0] |= static_cast<unsigned long long>(sh_digit[0]) << shift;
      prefix[1] |= static_cast<unsigned long long>(sh_digit[1]) << shift;
      mask |= 255ull << shift;
    }
  }
  // keys are unique: exactly k member keys are >= the k-th largest (prefix); a class whose budget
  // covers it entirely takes every member, a zero budget none
  for (int i = tid; i < u_cnt; i += SEL_THREADS) {
    const int c = cls[i] == CLS_HIST ? 0 : cls[i] == CLS_ITEM ? 1 : -1;
    if (c < 0 || kk[c] <= 0) continue;
    const bool act = c == 0 ? act0 : act1;
    if (!act || sel_key(a.dev[u_off + i], P + i) >= prefix[c]) flag[i] = 1;
  }
  __syncthreads();
  // compaction in position order: contiguous runs per thread, two-level warp-shuffle scan
  const int per = (u_cnt + SEL_THREADS - 1) / SEL_THREADS;
  const int b = tid * per, e = min(u_cnt, b + per);
  int cnt = 0;
  for (int i = b; i < e; ++i) cnt += flag[i];
  const int winc = warp_incl_scan(cnt);
  if (lane == 31) wsum[warp] = winc;
  __syncthreads();
  if (warp == 0) {
    const int v = lane < SEL_THREADS / 32 ? wsum[lane] : 0;
    const int inc = warp_incl_scan(v);
    if (lane < SEL_THREADS / 32) wsum[lane] = inc - v;  // exclusive warp offsets
  }
  __syncthreads();
  int w = sel_off + wsum[warp] + winc - cnt;
  for (int i = b; i < e; ++i) {
    if (!flag[i]) continue;
    a.sel_pos[w] = P + i;
    a.sel_dst[w] = rq2.z + P + i;
    a.sel_urow[w] = u_off + i;
    if (a.map) a.map[w] = a.u2s[u_off + i];
    ++w;
  }
}

__global__ void k_cand_scores(const float* logits, int64_t vocab, const int32_t* cand_req, const int32_t* idtok, int32_t n,
                              float* out) {
  griddep_wait();  // PDL: inputs of the previous kernel are complete and visible
  griddep_launch();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = logits[static_cast<int64_t>(cand_req[i]) * vocab + idtok[i]];
}

// [n_tok][L][2][Hk][dh] -> [L][2][Hk][dst_rows][dh] at rows dst_row0 + t (16-byte chunks)
__global__ void k_pool_transpose(const uint8_t* __restrict__ src, int eb, int32_t n_tok, int32_t L, int32_t Hk,
                                 int32_t dh, uint8_t* __restrict__ dst, int64_t dst_rows, int64_t dst_row0) {
  griddep_wait();  // PDL: inputs of the previous kernel are complete and visible
  griddep_launch();
  const int row_bytes = dh * eb;
  const int cpr = row_bytes / 16;
  const int64_t units = static_cast<int64_t>(n_tok) * L * 2 * Hk * cpr;
  for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < units;
       u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(u % cpr);
    const int64_t p = u / cpr;  // ((t*L + l)*2 + kv)*Hk + h
    const int64_t t = p / (static_cast<int64_t>(L) * 2 * Hk);
    const int64_t plane = p % (static_cast<int64_t>(L) * 2 * Hk);
    const uint4 v = *reinterpret_cast<const uint4*>(src + p * row_bytes + c * 16);
    *reinterpret_cast<uint4*>(dst + (plane * dst_rows + dst_row0 + t) * row_bytes + c * 16) = v;
  }
}

__global__ void k_scale_transpose(const float* __restrict__ src, int32_t n_tok, int32_t planes, float* __restrict__ dst,
                                  int64_t dst_rows, int64_t dst_row0) {
  griddep_wait();  // PDL: inputs of the previous kernel are complete and visible
  griddep_launch();
  const int64_t units = static_cast<int64_t>(n_tok) * planes;
  for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < units;
       u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = u / planes, plane = u % planes;
    dst[plane * dst_rows + dst_row0 + t] = src[u];
  }
}

// rows [src_row0, +n_rows) of every plane of a [planes][src_rows][row_bytes] pool (local or a
// mapped peer pool: one-sided NVLink reads) -> [planes][dst_rows] at dst_row0
__global__ void k_copy_rows(const uint8_t* __restrict__ src, int64_t src_rows, int64_t src_row0, uint8_t* __restrict__ dst,
                            int64_t dst_rows, int64_t dst_row0, int32_t n_rows, int32_t planes, int32_t row_bytes) {
  griddep_wait();  // PDL: inputs of the previous kernel are complete and visible
  griddep_launch();
  const int cpr = row_bytes / 16;
  const int64_t units = static_cast<int64_t>(planes) * n_rows * cpr;
  for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < units;
       u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(u % cpr);
    const int64_t r = (u / cpr) % n_rows;
    const int64_t plane = u / (static_cast<int64_t>(cpr) * n_rows);
    const uint4 v = *reinterpret_cast<const uint4*>(src + (plane * src_rows + src_row0 + r) * row_bytes + c * 16);
    *reinterpret_cast<uint4*>(dst + (plane * dst_rows + dst_row0 + r) * row_bytes + c * 16) = v;
  }
}

// one grid row per segment (blockIdx.y), 16-byte units grid-strided over its planes x rows
__global__ void k_copy_segments(const CopySeg* __restrict__ segs, uint8_t* __restrict__ dst, int64_t dst_rows,
                                int32_t planes, int32_t row_bytes) {
  griddep_wait();  // PDL: the segment table (H2D) and earlier kernels are complete and visible
  griddep_launch();
  const CopySeg sg = segs[blockIdx.y];
  const uint8_t* src = static_cast<const uint8_t*>(sg.src);
  const int cpr = row_bytes / 16;
  const int64_t per_plane = static_cast<int64_t>(sg.n_rows) * cpr;
  const int64_t units = per_plane * planes;
  for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < units;
       u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t plane = u / per_plane;
    const int64_t rc = u - plane * per_plane;
    const int64_t r = rc / cpr;
    const int c = static_cast<int>(rc - r * cpr);
    const uint4 v = *reinterpret_cast<const uint4*>(src + (plane * sg.src_rows + sg.src_row0 + r) * row_bytes + c * 16);
    *reinterpret_cast<uint4*>(dst + (plane * dst_rows + sg.dst_row0 + r) * row_bytes + c * 16) = v;
  }
}

// Pool materialisation (R16/R17): stitched rows [row0, row0+n) of every plane -> the registration
// layout [n][L][2][Hk][dh] (bf16 copy), or int8 codes + fp32 scales per (token, layer, K/V, head) with
// the R15 rule: scale = absmax/127 (fp32), q = clamp(rint_even(x / scale), -127, 127), scale 0 -> q 0.
// One warp per (token, plane) row.
__global__ void k_export_kv(const uint16_t* __restrict__ arena, int64_t arena_rows, int32_t planes, int32_t dh,
                            int32_t row0, int32_t n, int32_t int8, void* __restrict__ out, float* __restrict__ scales) {
  griddep_wait();
  griddep_launch();
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  if (w >= static_cast<int64_t>(n) * planes) return;
  const int64_t t = w / planes;
  const int plane = static_cast<int>(w - t * planes);
  const uint16_t* src = arena + (static_cast<int64_t>(plane) * arena_rows + row0 + t) * dh;
  const int64_t o = (t * planes + plane) * dh;  // [t][l][kv][h][dh] == [t][plane][dh]
  if (!int8) {
    for (int j = lane; j < dh; j += 32) static_cast<uint16_t*>(out)[o + j] = src[j];
    return;
  }
  float amax = 0.f;
  for (int j = lane; j < dh; j += 32) amax = fmaxf(amax, fabsf(bf2f(src[j])));
#pragma unroll
  for (int off = 16; off; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  const float scale = __fdiv_rn(amax, 127.0f);
  for (int j = lane; j < dh; j += 32) {
    float q = 0.f;
    if (scale > 0.f) q = fminf(fmaxf(rintf(__fdiv_rn(bf2f(src[j]), scale)), -127.f), 127.f);
    static_cast<int8_t*>(out)[o + j] = static_cast<int8_t>(q);
  }
  if (lane == 0) scales[t * planes + plane] = scale;
}

__global__ void k_resolve_hist(int4* __restrict__ meta, int32_t n, const uint64_t* __restrict__ req_ptr,
                               const int2* __restrict__ tab, int64_t cap, unsigned long long* err) {
  griddep_wait();
  griddep_launch();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int4 m = meta[i];
    if (m.w != RC_TOK_HIST_DEV) continue;
    const int32_t* ids = reinterpret_cast<const int32_t*>(req_ptr[m.y >> 16]);
    const int id = ids[m.y & 0xFFFF];
    const int2 t = (id >= 0 && id < cap) ? tab[id] : make_int2(-1, 0);
    if (t.x < 0) {  // not a registered prototype: counted, and the gather leaves the row unwritten
      atomicAdd(err, 1ull);
      m.w = CLS_FORCED;
    } else {
      m.y = t.x;
      m.z = m.z - t.y;  // Delta = position - canonical position
      m.w = CLS_HIST;
    }
    meta[i] = m;
  }
}

__global__ void k_scatter_index(int32_t* __restrict__ dst, const int32_t* __restrict__ idx, int32_t n) {
  griddep_wait();
  griddep_launch();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[idx[i]] = i;
}

__global__ void k_scatter_i32(int32_t* __restrict__ dst, const int2* __restrict__ idx_val, int32_t n) {
  griddep_wait();
  griddep_launch();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int2 e = idx_val[i];
    dst[e.x] = e.y;
  }
}

__global__ void k_vmap_identity(int32_t* __restrict__ vmap, const int32_t* __restrict__ rows, int32_t n) {
  griddep_wait();
  griddep_launch();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) vmap[rows[i]] = rows[i];
}

__global__ void k_read_kv(const uint16_t* __restrict__ arena, int64_t arena_rows, int32_t layer, int32_t Hk, int32_t dh,
                          int32_t row0, int32_t n, uint16_t* __restrict__ k_out, uint16_t* __restrict__ v_out,
                          const VSrc vs) {
  griddep_wait();  // PDL: inputs of the previous kernel are complete and visible
  griddep_launch();
  const int64_t units = static_cast<int64_t>(2) * n * Hk * dh;
  for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < units;
       u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(u % dh);
    int64_t r = u / dh;
    const int h = static_cast<int>(r % Hk);
    r /= Hk;
    const int t = static_cast<int>(r % n);
    const int kv = static_cast<int>(r / n);
    const uint16_t v = kv == 1 && vs.vmap
        ? vsrc_row(vs, arena + (static_cast<int64_t>(layer) * 2 + 1) * Hk * arena_rows * dh, arena_rows * dh, h, row0 + t, dh)[j]
        : arena[(((static_cast<int64_t>(layer) * 2 + kv) * Hk + h) * arena_rows + row0 + t) * dh + j];
    (kv == 0 ? k_out : v_out)[(static_cast<int64_t>(t) * Hk + h) * dh + j] = v;
  }
}

// diagnostic K5: D[i] = sum_j term(k_new, k_st) + term(v_new, v_st) over `width` elements, one warp per row
__global__ void k_dev_diag(const uint16_t* kn, const uint16_t* ks, const uint16_t* vn, const uint16_t* vs, int32_t n,
                           int32_t width, unsigned long long* out) {
  griddep_wait();  // PDL: inputs of the previous kernel are complete and visible
  griddep_launch();
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  unsigned long long acc = 0;
  const int64_t b = static_cast<int64_t>(row) * width;
  for (int j = lane; j < width; j += 32) {
    acc += dev_term(bf2f(kn[b + j]), ks[b + j]);
    acc += dev_term(bf2f(vn[b + j]), vs[b + j]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffff, acc, o);
  if (lane == 0) out[row] = acc;
}

inline int blocks_for(int64_t units, int per = 256, int cap = 148 * 16) {
  int64_t b = (units + per - 1) / per;
  if (b < 1) b = 1;
  return static_cast<int>(b > cap ? cap : b);
}
}  // namespace

cudaError_t embed_launch(const uint16_t* emb, const int32_t* tok, int32_t rows, int32_t d, float* x, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  return launch_pdl(k_embed, dim3(blocks_for(static_cast<int64_t>(rows) * d / 8)), dim3(256), 0, s, emb, tok, rows, d, x);
}
cudaError_t rmsnorm_launch(const float* x, const int32_t* row_idx, int32_t rows, int32_t d, const uint16_t* g, float eps,
                           uint16_t* out, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  const int th = d >= 1024 ? 256 : 64;
  const int per = (d / 4 + th - 1) / th;  // float4 per thread
  if (per <= 1) return launch_pdl(k_rmsnorm<1>, dim3(rows), dim3(th), 0, s, x, row_idx, d, g, eps, out);
  if (per <= 2) return launch_pdl(k_rmsnorm<2>, dim3(rows), dim3(th), 0, s, x, row_idx, d, g, eps, out);
  if (per <= 4) return launch_pdl(k_rmsnorm<4>, dim3(rows), dim3(th), 0, s, x, row_idx, d, g, eps, out);
  if (per <= 8) return launch_pdl(k_rmsnorm<8>, dim3(rows), dim3(th), 0, s, x, row_idx, d, g, eps, out);
  return cudaErrorInvalidValue;  // d > 8192: not a supported model width
}
cudaError_t gather_rows_f32_launch(const float* src, const int32_t* idx, int32_t rows, int32_t d, float* dst,
                                   cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  return launch_pdl(k_gather_rows, dim3(blocks_for(static_cast<int64_t>(rows) * d / 4)), dim3(256), 0, s, src, idx, rows, d, dst);
}
cudaError_t select_launch(const SelectArgs& a, cudaStream_t s) {
  if (a.n_req <= 0) return cudaSuccess;
  return launch_pdl(k_select, dim3(a.n_req), dim3(SEL_THREADS), 0, s, a);
}
cudaError_t dev_diag_launch(const uint16_t* kn, const uint16_t* ks, const uint16_t* vn, const uint16_t* vs, int32_t n,
                            int32_t width, unsigned long long* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(k_dev_diag, dim3((n + 7) / 8), dim3(256), 0, s, kn, ks, vn, vs, n, width, out);
}
cudaError_t cand_scores_launch(const float* logits, int64_t vocab, const int32_t* cand_req, const int32_t* idtok,
                               int32_t n, float* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(k_cand_scores, dim3((n + 255) / 256), dim3(256), 0, s, logits, vocab, cand_req, idtok, n, out);
}
cudaError_t pool_transpose_launch(const void* src, int eb, int32_t n_tok, int32_t L, int32_t Hk, int32_t dh, void* dst,
                                  int64_t dst_rows, int64_t dst_row0, cudaStream_t s) {
  if (n_tok <= 0) return cudaSuccess;
  if ((dh * eb) % 16) return cudaErrorInvalidValue;
  const int64_t units = static_cast<int64_t>(n_tok) * L * 2 * Hk * (dh * eb / 16);
  return launch_pdl(k_pool_transpose, dim3(blocks_for(units)), dim3(256), 0, s, static_cast<const uint8_t*>(src), eb, n_tok, L, Hk, dh,
                                                     static_cast<uint8_t*>(dst), dst_rows, dst_row0);
}
cudaError_t scale_transpose_launch(const float* src, int32_t n_tok, int32_t L, int32_t Hk, float* dst, int64_t dst_rows,
                                   int64_t dst_row0, cudaStream_t s) {
  if (n_tok <= 0) return cudaSuccess;
  return launch_pdl(k_scale_transpose, dim3(blocks_for(static_cast<int64_t>(n_tok) * L * 2 * Hk)), dim3(256), 0, s, src, n_tok, L * 2 * Hk, dst,
                                                                                         dst_rows, dst_row0);
}
cudaError_t copy_rows_launch(const void* src_base, int64_t src_rows, int64_t src_row0, void* dst_base, int64_t dst_rows,
                             int64_t dst_row0, int32_t n_rows, int32_t n_planes, int32_t row_bytes, cudaStream_t s) {
  if (n_rows <= 0) return cudaSuccess;
  if (row_bytes % 16) return cudaErrorInvalidValue;
  const int64_t units = static_cast<int64_t>(n_planes) * n_rows * (row_bytes / 16);
  return launch_pdl(k_copy_rows, dim3(blocks_for(units)), dim3(256), 0, s, static_cast<const uint8_t*>(src_base), src_rows, src_row0,
                                                static_cast<uint8_t*>(dst_base), dst_rows, dst_row0, n_rows, n_planes,
                                                row_bytes);
}
cudaError_t copy_segments_launch(const CopySeg* segs, int32_t n_segs, int64_t total_rows, void* dst_base,
                                 int64_t dst_rows, int32_t n_planes, int32_t row_bytes, cudaStream_t s) {
  if (n_segs <= 0 || total_rows <= 0) return cudaSuccess;
  if (row_bytes % 16 || n_segs > 65535) return cudaErrorInvalidValue;
  // ~8 blocks of 256 threads per SM in total, at least one per segment, 8 units per thread max
  const int64_t units_per_seg = static_cast<int64_t>(n_planes) * (total_rows / n_segs + 1) * (row_bytes / 16);
  int64_t gx = std::max<int64_t>(1, 148 * 8 / n_segs);
  gx = std::min<int64_t>(gx, (units_per_seg + 255) / 256);
  return launch_pdl(k_copy_segments, dim3(static_cast<unsigned>(std::max<int64_t>(gx, 1)), n_segs), dim3(256), 0, s,
                    segs, static_cast<uint8_t*>(dst_base), dst_rows, n_planes, row_bytes);
}
cudaError_t export_kv_launch(const uint16_t* arena, int64_t arena_rows, int32_t planes, int32_t dh, int32_t row0,
                             int32_t n, int32_t int8, void* out, float* scales, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t warps = static_cast<int64_t>(n) * planes;
  return launch_pdl(k_export_kv, dim3(static_cast<unsigned>((warps + 7) / 8)), dim3(256), 0, s, arena, arena_rows, planes,
                    dh, row0, n, int8, out, scales);
}
cudaError_t read_kv_launch(const uint16_t* arena, int64_t arena_rows, int32_t layer, int32_t Hk, int32_t dh, int32_t row0,
                           int32_t n, uint16_t* k_out, uint16_t* v_out, const VSrc& vs, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(k_read_kv, dim3(blocks_for(static_cast<int64_t>(2) * n * Hk * dh)), dim3(256), 0, s, arena, arena_rows, layer, Hk, dh, row0, n,
                                                                             k_out, v_out, vs);
}
cudaError_t resolve_hist_launch(int4* meta, int32_t n, const uint64_t* req_ptr, const int2* proto_tab, int64_t tab_cap,
                                unsigned long long* err, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(k_resolve_hist, dim3(static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 1024))), dim3(256), 0,
                    s, meta, n, req_ptr, proto_tab, tab_cap, err);
}
cudaError_t scatter_i32_launch(int32_t* dst, const int2* idx_val, int32_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(k_scatter_i32, dim3(static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 1024))), dim3(256), 0,
                    s, dst, idx_val, n);
}
cudaError_t scatter_index_launch(int32_t* dst, const int32_t* idx, int32_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(k_scatter_index, dim3(static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 1024))), dim3(256), 0,
                    s, dst, idx, n);
}
cudaError_t vmap_identity_launch(int32_t* vmap, const int32_t* rows, int32_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(k_vmap_identity, dim3(static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 1024))), dim3(256), 0,
                    s, vmap, rows, n);
}

}  // namespace rc
