// NEXT-3: online LSH matching of history tokens to semantic prototypes
// ("mapped to the nearest pre-computed semantic prototype using LSH-based matching";
// SPEC.md:237-263 embed_token / match_token), under the DESIGN.md R-LSH reading that fixes the
// fp32 operation order of every integer decision (signature bits, argmax).
//
// One warp per token: lane l holds embedding components l and l + 32 (D = 64 = 48 lexical + 16
// positional). dot(a, b) = (a_l b_l + a_{l+32} b_{l+32}) per lane, then an xor butterfly over
// 16, 8, 4, 2, 1 -- every product and sum rounded to fp32 (__fmul_rn / __fadd_rn, no FMA), so all
// lanes hold the same bits and the host oracle reproduces them exactly.
//   k_semlib_embed: centroids + signatures of the prototypes (library build)
//   k_semlib_match: embed, 128 hyperplane signs -> 8 16-bit signatures, binary search of each
//                   table's sorted (signature, id) array, max cosine over the union (ties ->
//                   smaller id), fallback scan of the query's log bucket (or of all prototypes)
#include "common.cuh"
#include "rc_internal.h"

namespace rc {
namespace {

constexpr int D = 64, D_LEX = 48, T = 8, B = 16;

__device__ __forceinline__ unsigned long long splitmix64_d(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  unsigned long long z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float warp_dot(float a0, float a1, float b0, float b1) {
  float s = __fadd_rn(__fmul_rn(a0, b0), __fmul_rn(a1, b1));
#pragma unroll
  for (int o = 16; o; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  return s;
}

__device__ __forceinline__ int log_bucket(int offset, int n_buckets) {
  const int b = 31 - __clz(offset + 1);
  return b < n_buckets - 1 ? b : n_buckets - 1;
}

// unit embedding of (token, history offset): lane holds components (lane, lane + 32)
__device__ __forceinline__ void embed_warp(int token, int offset, const SemlibArgs& s, float& v0, float& v1) {
  const int lane = threadIdx.x & 31;
  const unsigned long long base = (s.seed & 0xFFFFFFFFull) << 32;
  auto lex = [&](int j) {
    const unsigned long long h = splitmix64_d(base ^ (64ull * static_cast<unsigned long long>(token) + j));
    return (h >> 63) == 0 ? 1.f : -1.f;
  };
  const int b = log_bucket(offset, s.n_buckets);
  v0 = lex(lane);                                                   // components 0..31: lexical
  v1 = lane < D_LEX - 32 ? lex(lane + 32) : s.pos_table[b * 16 + (lane - (D_LEX - 32))];  // 32..47 lex, 48..63 pos
  const float n = __fsqrt_rn(warp_dot(v0, v1, v0, v1));
  v0 = __fdiv_rn(v0, n);
  v1 = __fdiv_rn(v1, n);
}

__device__ __forceinline__ void signatures_warp(float v0, float v1, const float* __restrict__ H, uint32_t* sig) {
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int t = 0; t < T; ++t) {
    uint32_t s = 0;
#pragma unroll 4
    for (int b = 0; b < B; ++b) {
      const float* h = H + (t * B + b) * D;
      if (warp_dot(v0, v1, h[lane], h[lane + 32]) > 0.f) s |= 1u << b;
    }
    sig[t] = s;
  }
}

__global__ void k_semlib_embed(const SemlibArgs s, int n, const int32_t* __restrict__ tok,
                               const int32_t* __restrict__ off, float* __restrict__ C, uint32_t* __restrict__ sig) {
  griddep_wait();
  griddep_launch();
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= n) return;
  float v0, v1;
  embed_warp(tok[i], off[i], s, v0, v1);
  C[static_cast<int64_t>(i) * D + lane] = v0;
  C[static_cast<int64_t>(i) * D + lane + 32] = v1;
  uint32_t sg[T];
  signatures_warp(v0, v1, s.H, sg);
  if (lane == 0)
    for (int t = 0; t < T; ++t) sig[static_cast<int64_t>(t) * n + i] = sg[t];
}

// best (cosine, id) over prototypes ids[lo, hi) (by index through `ids`, or lo..hi-1 directly)
__device__ __forceinline__ void scan(const SemlibArgs& s, const int32_t* ids, int lo, int hi, float v0, float v1,
                                     float& best, int& best_id) {
  const int lane = threadIdx.x & 31;
  for (int k = lo; k < hi; ++k) {
    const int p = ids ? ids[k] : k;
    const float* c = s.C + static_cast<int64_t>(p) * D;
    const float cs = warp_dot(v0, v1, c[lane], c[lane + 32]);
    if (cs > best || (cs == best && p < best_id)) { best = cs; best_id = p; }
  }
}

__global__ void k_semlib_match(const SemlibArgs s, int n, const int32_t* __restrict__ tok,
                               const int32_t* __restrict__ off, int32_t* __restrict__ proto_out,
                               float* __restrict__ cos_out) {
  griddep_wait();
  griddep_launch();
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= n) return;
  float v0, v1;
  embed_warp(tok[i], off[i], s, v0, v1);
  uint32_t sg[T];
  signatures_warp(v0, v1, s.H, sg);
  float best = -INFINITY;
  int best_id = 0x7fffffff;
  int found = 0;
  for (int t = 0; t < T; ++t) {  // lower_bound / upper_bound of sg[t] in table t (sorted by signature, then id)
    const uint32_t* ts = s.tab_sig + static_cast<int64_t>(t) * s.n_proto;
    int lo = 0, hi = s.n_proto;
    while (lo < hi) { const int m = (lo + hi) >> 1; if (ts[m] < sg[t]) lo = m + 1; else hi = m; }
    int up = lo, h2 = s.n_proto;
    while (up < h2) { const int m = (up + h2) >> 1; if (ts[m] <= sg[t]) up = m + 1; else h2 = m; }
    found += up - lo;
    scan(s, s.tab_id + static_cast<int64_t>(t) * s.n_proto, lo, up, v0, v1, best, best_id);
  }
  if (found == 0) {  // SPEC fallback: the best prototype of the query's bucket (all prototypes if none)
    const int b = log_bucket(off[i], s.n_buckets);
    int lo = s.bucket_start[b], hi = s.bucket_start[b + 1];
    if (lo == hi) scan(s, nullptr, 0, s.n_proto, v0, v1, best, best_id);
    else scan(s, s.bucket_ids, lo, hi, v0, v1, best, best_id);
  }
  if (lane == 0) { proto_out[i] = best_id; cos_out[i] = best; }
}
}  // namespace

cudaError_t semlib_embed_launch(const SemlibArgs& s, int n, const int32_t* tok, const int32_t* off, float* C,
                                uint32_t* sig, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(k_semlib_embed, dim3((n + 7) / 8), dim3(256), 0, st, s, n, tok, off, C, sig);
}

cudaError_t semlib_match_launch(const SemlibArgs& s, int n, const int32_t* tok, const int32_t* off, int32_t* proto_out,
                                float* cos_out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(k_semlib_match, dim3((n + 7) / 8), dim3(256), 0, st, s, n, tok, off, proto_out, cos_out);
}

}  // namespace rc
