// librc host side: the C-ABI of include/rc.h -- context, pools, request assembly (a0/a1) and
// the selective-prefill layer loop (a2-a8). All arithmetic of the path runs in the kernels of
// k_gather.cu, k_gemm.cu, k_attn.cu and k_small.cu; this file does allocation, metadata and
// launch order only.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/rc.h"
#include "rc_internal.h"

using namespace rc;

namespace {
thread_local std::string g_err;
}  // namespace

int32_t rc::set_error(int32_t code, const char* msg) {
  g_err = msg;
  return code;
}

cudaError_t rc::smem_opt_in(const void* kern, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;  // (kernel, device)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({kern, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({kern, dev});
  return e;
}

bool rc::pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("RC_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

namespace {

rc_status fail(rc_status code, const std::string& msg) {
  g_err = msg;
  return code;
}
#define RC_CUDA(expr)                                                                        \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) return fail(RC_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// First-fit range allocator over [0, cap) with coalescing free list.
struct RangeAlloc {
  int64_t cap = 0;
  std::map<int64_t, int64_t> free_;  // start -> len
  void init(int64_t c) {
    cap = c;
    free_.clear();
    if (c > 0) free_[0] = c;
  }
  int64_t alloc(int64_t len) {
    if (len <= 0) return 0;
    for (auto it = free_.begin(); it != free_.end(); ++it) {
      if (it->second >= len) {
        const int64_t s = it->first, l = it->second;
        free_.erase(it);
        if (l > len) free_[s + len] = l - len;
        return s;
      }
    }
    return -1;
  }
  void release(int64_t s, int64_t len) {
    if (len <= 0) return;
    auto it = free_.emplace(s, len).first;
    auto nx = std::next(it);
    if (nx != free_.end() && it->first + it->second == nx->first) {
      it->second += nx->second;
      free_.erase(nx);
    }
    if (it != free_.begin()) {
      auto pv = std::prev(it);
      if (pv->first + pv->second == it->first) {
        pv->second += it->second;
        free_.erase(it);
      }
    }
  }
};

struct Block {
  int64_t row;
  int32_t n;
  int32_t canon;
  bool remote;
  uint64_t last_use;
};

struct Seq {
  int32_t n = 0, P = 0, gather_from = 0;
  int64_t arena_row = 0;
  std::vector<int32_t> tokens;
  std::vector<uint8_t> cls;  // after miss handling
  std::vector<int32_t> cand_idtok;
};

// Pinned host staging with per-slot events so the host never overwrites an in-flight copy.
struct Staging {
  static constexpr int SLOTS = 4;
  void* host[SLOTS] = {};
  void* dev[SLOTS] = {};
  size_t cap[SLOTS] = {};
  cudaEvent_t ev[SLOTS] = {};
  int next = 0;
  ~Staging() {
    for (int i = 0; i < SLOTS; ++i) {
      if (host[i]) cudaFreeHost(host[i]);
      if (dev[i]) cudaFree(dev[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
    }
  }
  // returns slot index; host[slot] has >= bytes
  int acquire(size_t bytes, cudaError_t* err) {
    const int s = next;
    next = (next + 1) % SLOTS;
    *err = cudaSuccess;
    if (ev[s]) {
      *err = cudaEventSynchronize(ev[s]);
      if (*err != cudaSuccess) return -1;
    } else {
      *err = cudaEventCreateWithFlags(&ev[s], cudaEventDisableTiming);
      if (*err != cudaSuccess) return -1;
    }
    if (cap[s] < bytes) {
      if (host[s]) cudaFreeHost(host[s]);
      if (dev[s]) cudaFree(dev[s]);
      host[s] = dev[s] = nullptr;
      const size_t c = std::max(bytes, static_cast<size_t>(1) << 20);
      *err = cudaMallocHost(&host[s], c);
      if (*err == cudaSuccess) *err = cudaMalloc(&dev[s], c);
      if (*err != cudaSuccess) { cap[s] = 0; return -1; }
      cap[s] = c;
    }
    return s;
  }
};

// Bump layout of several arrays inside one staging slot (16-byte aligned pieces).
struct Layout {
  size_t off = 0;
  size_t add(size_t bytes) {
    const size_t o = off;
    off += (bytes + 15) & ~size_t(15);
    return o;
  }
};

template <typename T>
T* dev_alloc(size_t n, cudaError_t* e) {
  void* p = nullptr;
  *e = cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T));
  return static_cast<T*>(p);
}

}  // namespace

struct rc_ctx {
  int device = 0;
  int num_sms = 148;
  rc_model_desc m{};
  rc_pool_desc pd{};
  // weights
  const uint16_t* embed = nullptr;
  const uint16_t* fnorm = nullptr;
  const uint16_t* lm_head = nullptr;
  std::vector<const uint16_t*> ln1, ln2, wo, wd;
  uint16_t* wqkv = nullptr;  // [L][Nqkv][d]
  uint16_t* bqkv = nullptr;  // [L][Nqkv]
  uint16_t* wgu = nullptr;   // [L][2F][d]
  int Nqkv = 0;
  // pools ([L][2][Hk][rows][dh])
  uint16_t* item_pool = nullptr;
  int8_t* hist_q = nullptr;
  float* hist_s = nullptr;
  uint16_t* prefix_pool = nullptr;
  RangeAlloc item_alloc, remote_alloc;
  int64_t hist_used = 0, prefix_used = 0;
  std::unordered_map<uint64_t, Block> items, protos, prefixes;
  // NEXT-3 device-fed prototypes: dense id -> {pool row, canonical position} (row -1 = unregistered)
  std::vector<int2> proto_tab_host;
  int2* proto_tab = nullptr;
  int64_t proto_tab_cap = 0;
  unsigned long long* dev_err = nullptr;  // device-side input errors (rc_device_error_count)
  // NEXT-2 host tier: pinned, mapped host DRAM in the pool layout [L][2][Hk][host_rows][dh]
  uint16_t* host_pool = nullptr;      // host pointer
  uint16_t* host_pool_dev = nullptr;  // its device mapping (registration writes)
  int64_t host_used = 0;
  std::unordered_map<uint64_t, Block> host_items;
  uint64_t use_clock = 1;
  // LRU index of the remote-cache region (blocks pulled from peers or the host tier): (last_use, id)
  std::set<std::pair<uint64_t, uint64_t>> lru;
  // peers
  std::unordered_map<int, std::pair<const uint16_t*, int64_t>> peers;  // rank -> (pool base, rows)
  std::unordered_map<int, std::unordered_map<uint64_t, Block>> peer_dir;  // rank -> its item directory
  std::vector<void*> ipc_opened;
  // arena
  uint16_t* arena = nullptr;
  RangeAlloc arena_alloc;
  // NEXT-4 zero-copy V (RC_ZERO_COPY_V=1): item / prefix V rows stay in their pools at the layers >= c;
  // vmap[arena row] says where each stitched V row lives (rc_internal.h VSRC_*)
  bool zc_v = false;
  int32_t* vmap = nullptr;
  std::unordered_map<uint64_t, Seq> seqs;
  uint64_t next_seq = 1;
  // rope tables
  float* rope_cos = nullptr;
  float* rope_sin = nullptr;
  int32_t rope_zero = 0;
  // workspace
  int64_t Mx = 0;
  float* x = nullptr;
  float* xs = nullptr;
  uint16_t* a = nullptr;
  uint16_t* q = nullptr;
  uint16_t* o = nullptr;
  uint16_t* h = nullptr;
  unsigned long long* dev = nullptr;
  float* logits = nullptr;
  int64_t logits_rows = 0;
  float* part_o = nullptr;   // KV-split attention partials
  float* part_ml = nullptr;
  int32_t* part_flag = nullptr;  // KV split: arrival counter per (logical tile, KV head)
  int32_t* attn_ctr = nullptr;   // paired attention work counter
  // early O-projection at small M (one request's Sel): per 256-row token tile, the attention CTAs done
  // with it ([0..3]) and the O-proj CTAs finished ([4]); zeroed by the O-proj's last CTA
  int32_t* oproj_ready = nullptr;
  bool early_on = false;         // set around the selective layers when their tile list allows it
  int32_t early_cnt[4] = {};     // attention CTAs per token tile of that list
  unsigned long long* attn_prof = nullptr;  // diagnostics: paired-attention phase cycle sums (RC_ATTN_PROF)
  size_t part_rows = 0;
  int32_t* sel_pos = nullptr;
  int32_t* sel_dst = nullptr;
  int32_t* sel_urow = nullptr;
  // gradual filtering (R-GF): second Sel arrays, U row -> previous Sel row, new -> previous Sel row
  // (5 x Mx int32, allocated on first use)
  int32_t* grad_buf = nullptr;
  // tensor maps
  CUtensorMap mA_a{}, mA_o{}, mA_h{};
  CUtensorMap mA_a64{}, mA_o64{}, mA_h64{};  // same operands, gemm_t_box_rows()-row boxes (transposed small-M GEMM)
  // residual-GEMM workspace: partial tiles summed in K order (bitwise-reproducible residual stream)
  float* gemm_ws = nullptr;
  int* gemm_cnt = nullptr;
  CUtensorMap mC_x{}, mC_xs{};  // fp32 residual streams as TMA reduce-add targets
  std::vector<CUtensorMap> mB_qkv, mB_kv, mB_o, mB_gu, mB_d;
  CUtensorMap mB_lm{};
  bool attn_tc = false;                 // tcgen05 attention (head_dim 128)
  CUtensorMap mQ3{};                    // q workspace as [R][H][dh]
  std::vector<CUtensorMap> mK_att, mV_att;  // arena K / V per layer as [Hk*T_cap][dh]
  // NEXT-1 (lambda < 1): fresh K/V of the check layer (same layout as one arena layer), per-row
  // log-sum-exp, attention mass; allocated on first use
  uint16_t* mass_k = nullptr;
  uint16_t* mass_v = nullptr;
  float* mass_lse = nullptr;
  unsigned long long* mass_a = nullptr;
  CUtensorMap mK_mass{}, mV_mass{};
  // NEXT-3 semantic library (device arrays, owned)
  SemlibArgs semlib{};
  std::vector<void*> semlib_bufs;
  int attn_tq() const { return attn_tc ? attn_tc_tokens_per_tile(m.n_heads / m.n_kv_heads)
                                       : attn_tokens_per_tile(m.n_heads / m.n_kv_heads); }
  int bn_qkv = 256, bn_kv = 256, bn_o = 256, bn_d = 256, bn_lm = 256;
  Staging stage;
  int64_t launches = 0;
  // profiling (rc_profile_begin / rc_profile_end): CUDA events around every librc launch
  struct Rec { int kind; cudaEvent_t a, b; double flops, bytes; int pending; };
  struct Pending { int32_t* host; int32_t S; std::vector<std::pair<int, int>> ranges; int layers; };
  bool prof = false;
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> evpool;
  size_t ev_used = 0;
  std::vector<Pending> pend;

  ~rc_ctx() {
    cudaSetDevice(device);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    for (cudaEvent_t e : evpool) cudaEventDestroy(e);
    for (auto& p : pend) cudaFreeHost(p.host);
    void* bufs[] = {wqkv, bqkv, wgu, item_pool, hist_q, hist_s, prefix_pool, arena, rope_cos, rope_sin, x, xs,
                    a, q, o, h, dev, logits, sel_pos, sel_dst, sel_urow, part_o, part_ml, part_flag, mass_k, mass_v,
                    mass_lse, mass_a, attn_ctr, oproj_ready, gemm_ws, gemm_cnt, vmap, proto_tab, dev_err, grad_buf};
    for (void* p : bufs)
      if (p) cudaFree(p);
    if (host_pool) cudaFreeHost(host_pool);
    for (void* p : semlib_bufs) cudaFree(p);
  }
};

namespace {
int pick_bn(int N) { return N > 128 ? 256 : 128; }

cudaEvent_t next_ev(rc_ctx* c) {
  if (c->ev_used == c->evpool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->evpool.push_back(e);
  }
  return c->evpool[c->ev_used++];
}
// Every librc kernel launch goes through RC_LAUNCH: counted, and timed per kind when profiling.
#define RC_LAUNCH(kind, flops, bytes, pending, expr)                                                     \
  do {                                                                                                  \
    c->launches++;                                                                                      \
    cudaEvent_t a_ = nullptr, b_ = nullptr;                                                             \
    if (c->prof) { a_ = next_ev(c); b_ = next_ev(c); cudaEventRecord(a_, s); }                          \
    cudaError_t e_ = (expr);                                                                            \
    if (e_ != cudaSuccess) return fail(RC_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    if (c->prof) {                                                                                      \
      cudaEventRecord(b_, s);                                                                           \
      c->recs.push_back({kind, a_, b_, static_cast<double>(flops), static_cast<double>(bytes), pending}); \
    }                                                                                                   \
  } while (0)
// every GEMM epilogue starts from the context's workspace (used by the residual epilogues)
EpiArgs epi_base(const rc_ctx* c) {
  EpiArgs e{};
  e.ws = c->gemm_ws;
  e.ws_cnt = c->gemm_cnt;
  e.ws_slots = gemm_ws_slots();
  e.head_dim = c->m.head_dim;
  return e;
}
double gemm_flops(double M, double N, double K) { return 2.0 * M * N * K; }
double gemm_bytes(double M, double N, double K, double out_b) { return (M * K + N * K) * 2.0 + M * N * out_b; }

rc_status build_rope(rc_ctx* c) {
  const int dh = c->m.head_dim, half = dh / 2;
  const int zero = c->pd.max_seq_len;
  const int64_t rows = 2 * static_cast<int64_t>(zero) + 1;
  std::vector<double> inv(half);
  for (int i = 0; i < half; ++i) inv[i] = std::pow(c->m.rope_theta, (-2.0 * i) / dh);
  std::vector<float> cs(rows * half), sn(rows * half);
  for (int64_t r = 0; r < rows; ++r) {
    const double d = static_cast<double>(r - zero);
    for (int i = 0; i < half; ++i) {
      const double ang = d * inv[i];
      cs[r * half + i] = static_cast<float>(std::cos(ang));
      sn[r * half + i] = static_cast<float>(std::sin(ang));
    }
  }
  cudaError_t e;
  c->rope_cos = dev_alloc<float>(rows * half, &e);
  if (e != cudaSuccess) return fail(RC_E_NOMEM, "rope table alloc");
  c->rope_sin = dev_alloc<float>(rows * half, &e);
  if (e != cudaSuccess) return fail(RC_E_NOMEM, "rope table alloc");
  RC_CUDA(cudaMemcpy(c->rope_cos, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice));
  RC_CUDA(cudaMemcpy(c->rope_sin, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice));
  c->rope_zero = zero;
  return RC_OK;
}

int64_t plane_count(const rc_ctx* c) { return static_cast<int64_t>(c->m.n_layers) * 2 * c->m.n_kv_heads; }

// the V sources of layer l under zero-copy V (empty VSrc: every V row in the arena)
VSrc layer_vsrc(const rc_ctx* c, int l) {
  VSrc v;
  if (!c->zc_v) return v;
  const int64_t hk = c->m.n_kv_heads, dh = c->m.head_dim;
  v.vmap = c->vmap;
  v.item = c->item_pool ? c->item_pool + ((static_cast<int64_t>(l) * 2 + 1) * hk) * c->pd.item_rows * dh : nullptr;
  v.item_head_stride = c->pd.item_rows * dh;
  v.prefix = c->prefix_pool ? c->prefix_pool + ((static_cast<int64_t>(l) * 2 + 1) * hk) * c->pd.prefix_rows * dh : nullptr;
  v.prefix_head_stride = c->pd.prefix_rows * dh;
  return v;
}

// mark a resident item block used at the current clock (keeps the remote-region LRU index in sync)
void touch(rc_ctx* c, uint64_t id, Block& b) {
  if (b.last_use == c->use_clock) return;
  if (b.remote) {
    c->lru.erase({b.last_use, id});
    c->lru.insert({c->use_clock, id});
  }
  b.last_use = c->use_clock;
}

// One block to bring into the remote-cache region.
struct FetchItem {
  uint64_t id;
  const uint16_t* src;  // source pool base (peer mapping) or nullptr (host tier)
  int64_t src_rows, src_row;
  int32_t n, canon;
};

// Plan the region rows of `todo` (all non-resident, distinct) with LRU eviction of remote blocks
// not used at the current clock, on copies of the allocator: nothing is modified unless every
// block fits (no partial effects). On success the evictions and allocations are committed and
// dst[i] holds block i's first item-pool row.
rc_status plan_remote_rows(rc_ctx* c, const std::vector<FetchItem>& todo, std::vector<int64_t>& dst) {
  RangeAlloc alloc = c->remote_alloc;
  std::vector<uint64_t> victims;
  auto next = c->lru.begin();
  const int64_t base = c->pd.item_rows - c->pd.remote_rows;
  dst.resize(todo.size());
  for (size_t i = 0; i < todo.size(); ++i) {
    int64_t row = alloc.alloc(todo[i].n);
    while (row < 0) {
      if (next == c->lru.end() || next->first == c->use_clock)
        return fail(RC_E_CAPACITY, "remote region exhausted (every block is used by this call)");
      const Block& b = c->items.at(next->second);
      alloc.release(b.row - base, b.n);
      victims.push_back(next->second);
      ++next;
      row = alloc.alloc(todo[i].n);
    }
    dst[i] = base + row;
  }
  c->remote_alloc = alloc;
  for (uint64_t v : victims) {
    c->lru.erase({c->items.at(v).last_use, v});
    c->items.erase(v);
  }
  for (size_t i = 0; i < todo.size(); ++i) {
    c->items[todo[i].id] = Block{dst[i], todo[i].n, todo[i].canon, true, c->use_clock};
    c->lru.insert({c->use_clock, todo[i].id});
  }
  return RC_OK;
}

uint16_t* arena_layer(rc_ctx* c, int l, int kv) {
  return c->arena + (static_cast<int64_t>(l) * 2 + kv) * c->m.n_kv_heads * c->pd.arena_rows * c->m.head_dim;
}
}  // namespace

extern "C" {

const char* rc_last_error(void) { return g_err.c_str(); }
int32_t rc_abi_version(void) { return 1; }
int64_t rc_launch_count(rc_ctx* ctx) { return ctx ? ctx->launches : 0; }
int64_t rc_device_error_count(rc_ctx* ctx) {
  if (!ctx || !ctx->dev_err) return 0;
  unsigned long long v = 0;
  if (cudaSetDevice(ctx->device) != cudaSuccess ||
      cudaMemcpy(&v, ctx->dev_err, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return static_cast<int64_t>(v);
}

rc_status rc_create(const rc_model_desc* md, const rc_weights* w, const rc_pool_desc* pd, int32_t device, rc_ctx** out) {
  if (!md || !w || !pd || !out) return fail(RC_E_INVALID, "null argument");
  const rc_model_desc& m = *md;
  if (m.n_layers <= 0 || m.d_model <= 0 || m.n_heads <= 0 || m.n_kv_heads <= 0 || m.n_heads % m.n_kv_heads ||
      !(m.head_dim == 16 || m.head_dim == 64 || m.head_dim == 128) || m.d_ff % 128 || m.d_model % 64 != 0 &&
      m.d_model % 16 != 0 || m.d_model > 8192)
    return fail(RC_E_INVALID, "unsupported model shape");
  if (pd->max_seq_len <= 0 || pd->max_seq_len > 8192) return fail(RC_E_INVALID, "max_seq_len must be in 1..8192 (R6)");
  // R4/R6: D sums 2*H_kv*d_h fixed-point terms below 2^40 each, and the selection key packs D << 13;
  // D < 2^51 (so the key fits 64 bits) needs at most 2^11 terms
  if (2 * static_cast<int64_t>(m.n_kv_heads) * m.head_dim > 2048)
    return fail(RC_E_INVALID, "2*n_kv_heads*head_dim must be <= 2048 (R6 selection key width)");
  if (pd->max_batch_tokens <= 0 || pd->remote_rows > pd->item_rows) return fail(RC_E_INVALID, "bad pool desc");
  if (!w->embed || !w->final_norm || !w->lm_head || !w->ln1 || !w->wq || !w->wk || !w->wv || !w->wo || !w->ln2 ||
      !w->wg || !w->wu || !w->wd || (m.qkv_bias && (!w->bq || !w->bk || !w->bv)))
    return fail(RC_E_INVALID, "missing weight pointer");
  std::unique_ptr<rc_ctx> c(new rc_ctx());
  c->device = device;
  c->m = m;
  c->pd = *pd;
  RC_CUDA(cudaSetDevice(device));
  RC_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  const int L = m.n_layers, d = m.d_model, dh = m.head_dim, H = m.n_heads, Hk = m.n_kv_heads, F = m.d_ff;
  c->Nqkv = (H + 2 * Hk) * dh;
  c->embed = static_cast<const uint16_t*>(w->embed);
  c->fnorm = static_cast<const uint16_t*>(w->final_norm);
  c->lm_head = static_cast<const uint16_t*>(w->lm_head);
  cudaError_t e;
  c->wqkv = dev_alloc<uint16_t>(static_cast<size_t>(L) * c->Nqkv * d, &e);
  if (e != cudaSuccess) return fail(RC_E_NOMEM, "packed qkv weights");
  c->wgu = dev_alloc<uint16_t>(static_cast<size_t>(L) * 2 * F * d, &e);
  if (e != cudaSuccess) return fail(RC_E_NOMEM, "packed gate/up weights");
  if (m.qkv_bias) {
    c->bqkv = dev_alloc<uint16_t>(static_cast<size_t>(L) * c->Nqkv, &e);
    if (e != cudaSuccess) return fail(RC_E_NOMEM, "packed qkv bias");
  }
  for (int l = 0; l < L; ++l) {
    c->ln1.push_back(static_cast<const uint16_t*>(w->ln1[l]));
    c->ln2.push_back(static_cast<const uint16_t*>(w->ln2[l]));
    c->wo.push_back(static_cast<const uint16_t*>(w->wo[l]));
    c->wd.push_back(static_cast<const uint16_t*>(w->wd[l]));
    // q | k | v heads; inside every head the rows in rotate-half pair order [0, dh/2, 1, dh/2+1, ...]
    // (RoPE partners adjacent in every GEMM orientation, k_gemm.cu)
    uint16_t* dq = c->wqkv + static_cast<size_t>(l) * c->Nqkv * d;
    const size_t row_b = static_cast<size_t>(d) * 2, half_b = static_cast<size_t>(dh / 2) * row_b;
    auto pack_heads = [&](uint16_t* dst, const void* src, int nheads) -> cudaError_t {
      for (int hh = 0; hh < nheads; ++hh) {
        uint8_t* dh8 = reinterpret_cast<uint8_t*>(dst) + static_cast<size_t>(hh) * 2 * half_b;
        const uint8_t* sh8 = static_cast<const uint8_t*>(src) + static_cast<size_t>(hh) * 2 * half_b;
        cudaError_t e2 = cudaMemcpy2D(dh8, 2 * row_b, sh8, row_b, row_b, dh / 2, cudaMemcpyDeviceToDevice);
        if (e2 == cudaSuccess) e2 = cudaMemcpy2D(dh8 + row_b, 2 * row_b, sh8 + half_b, row_b, row_b, dh / 2,
                                                 cudaMemcpyDeviceToDevice);
        if (e2 != cudaSuccess) return e2;
      }
      return cudaSuccess;
    };
    RC_CUDA(pack_heads(dq, w->wq[l], H));
    RC_CUDA(pack_heads(dq + static_cast<size_t>(H) * dh * d, w->wk[l], Hk));
    RC_CUDA(pack_heads(dq + static_cast<size_t>(H + Hk) * dh * d, w->wv[l], Hk));
    if (m.qkv_bias) {
      uint16_t* db = c->bqkv + static_cast<size_t>(l) * c->Nqkv;
      auto pack_bias = [&](uint16_t* dst, const void* src, int nheads) -> cudaError_t {
        for (int hh = 0; hh < nheads; ++hh) {  // element pitch 2 bytes: even slots <- first half, odd <- second
          uint16_t* dh16 = dst + static_cast<size_t>(hh) * dh;
          const uint16_t* sh16 = static_cast<const uint16_t*>(src) + static_cast<size_t>(hh) * dh;
          cudaError_t e2 = cudaMemcpy2D(dh16, 4, sh16, 2, 2, dh / 2, cudaMemcpyDeviceToDevice);
          if (e2 == cudaSuccess) e2 = cudaMemcpy2D(dh16 + 1, 4, sh16 + dh / 2, 2, 2, dh / 2, cudaMemcpyDeviceToDevice);
          if (e2 != cudaSuccess) return e2;
        }
        return cudaSuccess;
      };
      RC_CUDA(pack_bias(db, w->bq[l], H));
      RC_CUDA(pack_bias(db + H * dh, w->bk[l], Hk));
      RC_CUDA(pack_bias(db + (H + Hk) * dh, w->bv[l], Hk));
    }
    // gate/up interleaved by row: [g0, u0, g1, u1, ...]
    uint16_t* dg = c->wgu + static_cast<size_t>(l) * 2 * F * d;
    RC_CUDA(cudaMemcpy2D(dg, 2 * row_b, w->wg[l], row_b, row_b, F, cudaMemcpyDeviceToDevice));
    RC_CUDA(cudaMemcpy2D(reinterpret_cast<uint8_t*>(dg) + row_b, 2 * row_b, w->wu[l], row_b, row_b, F,
                         cudaMemcpyDeviceToDevice));
  }
  // pools + arena
  const int64_t planes = static_cast<int64_t>(L) * 2 * Hk;
  if (pd->item_rows > 0) {
    c->item_pool = dev_alloc<uint16_t>(static_cast<size_t>(planes) * pd->item_rows * dh, &e);
    if (e != cudaSuccess) return fail(RC_E_NOMEM, "item pool");
  }
  c->item_alloc.init(pd->item_rows - pd->remote_rows);
  c->remote_alloc.init(pd->remote_rows);
  if (pd->hist_rows > 0) {
    c->hist_q = dev_alloc<int8_t>(static_cast<size_t>(planes) * pd->hist_rows * dh, &e);
    if (e != cudaSuccess) return fail(RC_E_NOMEM, "history pool");
    c->hist_s = dev_alloc<float>(static_cast<size_t>(planes) * pd->hist_rows, &e);
    if (e != cudaSuccess) return fail(RC_E_NOMEM, "history scales");
  }
  if (pd->prefix_rows > 0) {
    c->prefix_pool = dev_alloc<uint16_t>(static_cast<size_t>(planes) * pd->prefix_rows * dh, &e);
    if (e != cudaSuccess) return fail(RC_E_NOMEM, "prefix pool");
  }
  if (pd->host_item_rows < 0) return fail(RC_E_INVALID, "negative host_item_rows");
  if (pd->host_item_rows > 0) {  // NEXT-2: pinned + mapped host tier
    const size_t bytes = static_cast<size_t>(planes) * pd->host_item_rows * dh * 2;
    void* hp = nullptr;
    if (cudaHostAlloc(&hp, bytes, cudaHostAllocMapped) != cudaSuccess)
      return fail(RC_E_NOMEM, "host-tier item pool (pinned)");
    c->host_pool = static_cast<uint16_t*>(hp);
    void* dp = nullptr;
    RC_CUDA(cudaHostGetDevicePointer(&dp, hp, 0));
    c->host_pool_dev = static_cast<uint16_t*>(dp);
  }
  c->arena = dev_alloc<uint16_t>(static_cast<size_t>(planes) * std::max<int64_t>(pd->arena_rows, 1) * dh, &e);
  if (e != cudaSuccess) return fail(RC_E_NOMEM, "stitched-KV arena");
  // every arena byte stays a finite bf16 (attention tiles may read rows past a request's end; they are
  // masked, and 0 * finite = 0 inside P V)
  RC_CUDA(cudaMemset(c->arena, 0, static_cast<size_t>(planes) * std::max<int64_t>(pd->arena_rows, 1) * dh * 2));
  c->arena_alloc.init(pd->arena_rows);
  {
    const char* zc = std::getenv("RC_ZERO_COPY_V");
    c->zc_v = zc && zc[0] == '1';
    std::vector<int32_t> ident(std::max<int64_t>(pd->arena_rows, 1));
    for (size_t i = 0; i < ident.size(); ++i) ident[i] = static_cast<int32_t>(i);
    c->vmap = dev_alloc<int32_t>(ident.size(), &e);
    if (e != cudaSuccess) return fail(RC_E_NOMEM, "vmap");
    RC_CUDA(cudaMemcpy(c->vmap, ident.data(), ident.size() * 4, cudaMemcpyHostToDevice));
  }
  c->dev_err = dev_alloc<unsigned long long>(1, &e);
  if (e != cudaSuccess) return fail(RC_E_NOMEM, "device error counter");
  RC_CUDA(cudaMemset(c->dev_err, 0, sizeof(unsigned long long)));
  rc_status st = build_rope(c.get());
  if (st != RC_OK) return st;
  // workspace
  const int64_t Mx = pd->max_batch_tokens;
  c->Mx = Mx;
  c->x = dev_alloc<float>(Mx * d, &e); if (e) return fail(RC_E_NOMEM, "workspace x");
  c->xs = dev_alloc<float>(Mx * d, &e); if (e) return fail(RC_E_NOMEM, "workspace xs");
  c->a = dev_alloc<uint16_t>(Mx * d, &e); if (e) return fail(RC_E_NOMEM, "workspace a");
  c->q = dev_alloc<uint16_t>(Mx * H * dh, &e); if (e) return fail(RC_E_NOMEM, "workspace q");
  c->o = dev_alloc<uint16_t>(Mx * H * dh, &e); if (e) return fail(RC_E_NOMEM, "workspace o");
  c->h = dev_alloc<uint16_t>(Mx * F, &e); if (e) return fail(RC_E_NOMEM, "workspace h");
  c->dev = dev_alloc<unsigned long long>(Mx, &e); if (e) return fail(RC_E_NOMEM, "workspace dev");
  c->sel_pos = dev_alloc<int32_t>(Mx, &e); if (e) return fail(RC_E_NOMEM, "workspace sel");
  c->sel_dst = dev_alloc<int32_t>(Mx, &e); if (e) return fail(RC_E_NOMEM, "workspace sel");
  c->sel_urow = dev_alloc<int32_t>(Mx, &e); if (e) return fail(RC_E_NOMEM, "workspace sel");
  // finite contents everywhere: GEMM tiles read stale rows past M (never stored, but reduce-added
  // into unused residual rows), which must not hold NaN bit patterns
  RC_CUDA(cudaMemset(c->x, 0, Mx * d * 4));
  RC_CUDA(cudaMemset(c->xs, 0, Mx * d * 4));
  RC_CUDA(cudaMemset(c->a, 0, Mx * d * 2));
  RC_CUDA(cudaMemset(c->o, 0, Mx * H * dh * 2));
  RC_CUDA(cudaMemset(c->h, 0, Mx * F * 2));
  // tensor maps: A operands (rows = Mx; tiles never read beyond the call's M-tile), B = weights
  c->gemm_ws = dev_alloc<float>(gemm_ws_floats(), &e); if (e) return fail(RC_E_NOMEM, "gemm workspace");
  c->gemm_cnt = dev_alloc<int>(2 * gemm_ws_slots(), &e); if (e) return fail(RC_E_NOMEM, "gemm workspace");
  c->oproj_ready = dev_alloc<int32_t>(8, &e); if (e) return fail(RC_E_NOMEM, "early O-projection counters");
  RC_CUDA(cudaMemset(c->oproj_ready, 0, 8 * sizeof(int32_t)));
  RC_CUDA(cudaMemset(c->gemm_cnt, 0, 2 * gemm_ws_slots() * sizeof(int)));
  bool ok = make_tmap_bf16_2d(&c->mA_a, c->a, Mx, d, d, 128) &&
            make_tmap_bf16_2d(&c->mA_o, c->o, Mx, H * dh, H * dh, 128) &&
            make_tmap_bf16_2d(&c->mA_h, c->h, Mx, F, F, 128) && make_tmap_f32_2d(&c->mC_x, c->x, Mx, d, d) &&
            make_tmap_f32_2d(&c->mC_xs, c->xs, Mx, d, d) && make_tmap_bf16_2d(&c->mA_a64, c->a, Mx, d, d, gemm_t_box_rows()) &&
            make_tmap_bf16_2d(&c->mA_o64, c->o, Mx, H * dh, H * dh, gemm_t_box_rows()) &&
            make_tmap_bf16_2d(&c->mA_h64, c->h, Mx, F, F, gemm_t_box_rows());
  c->bn_qkv = pick_bn(c->Nqkv);
  c->bn_kv = pick_bn(2 * Hk * dh);
  c->bn_o = pick_bn(d);
  c->bn_d = pick_bn(d);
  c->bn_lm = 256;
  c->mB_qkv.resize(L); c->mB_kv.resize(L); c->mB_o.resize(L); c->mB_gu.resize(L); c->mB_d.resize(L);
  for (int l = 0; l < L && ok; ++l) {
    const uint16_t* wq = c->wqkv + static_cast<size_t>(l) * c->Nqkv * d;
    ok = ok && make_tmap_bf16_2d(&c->mB_qkv[l], wq, c->Nqkv, d, d, gemm_box_rows_b(c->bn_qkv));
    ok = ok && make_tmap_bf16_2d(&c->mB_kv[l], wq + static_cast<size_t>(H) * dh * d, 2 * Hk * dh, d, d, gemm_box_rows_b(c->bn_kv));
    ok = ok && make_tmap_bf16_2d(&c->mB_o[l], c->wo[l], d, H * dh, H * dh, gemm_box_rows_b(c->bn_o));
    ok = ok && make_tmap_bf16_2d(&c->mB_gu[l], c->wgu + static_cast<size_t>(l) * 2 * F * d, 2 * F, d, d, gemm_box_rows_b(256));
    ok = ok && make_tmap_bf16_2d(&c->mB_d[l], c->wd[l], d, F, F, gemm_box_rows_b(c->bn_d));
  }
  ok = ok && make_tmap_bf16_2d(&c->mB_lm, c->lm_head, m.vocab, d, d, gemm_box_rows_b(c->bn_lm));
  c->attn_tc = (dh == 128) && std::getenv("RC_ATTN_LEGACY") == nullptr;
  if (c->attn_tc && ok) {
    const int G = H / Hk;
    const int TQ = attn_tc_tokens_per_tile(G);
    ok = make_tmap_bf16_3d(&c->mQ3, c->q, dh, H, Mx, static_cast<uint64_t>(dh) * 2, static_cast<uint64_t>(H) * dh * 2,
                           64, G, TQ);
    c->mK_att.resize(L); c->mV_att.resize(L);
    for (int l = 0; l < L && ok; ++l) {
      ok = make_tmap_bf16_2d(&c->mK_att[l], arena_layer(c.get(), l, 0), static_cast<uint64_t>(Hk) * pd->arena_rows, dh,
                             dh, 128) &&
           make_tmap_bf16_2d(&c->mV_att[l], arena_layer(c.get(), l, 1), static_cast<uint64_t>(Hk) * pd->arena_rows, dh,
                             dh, 128);
    }
  }
  if (!ok) return fail(RC_E_CUDA, "cuTensorMapEncodeTiled failed (driver entry point or alignment)");
  RC_CUDA(cudaDeviceSynchronize());
  *out = c.release();
  return RC_OK;
}

void rc_destroy(rc_ctx* ctx) {
  if (ctx && ctx->attn_prof) {  // diagnostics: paired-attention phase timing (RC_ATTN_PROF=1)
    unsigned long long h[16] = {};
    cudaSetDevice(ctx->device);
    if (cudaMemcpy(h, ctx->attn_prof, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess) {
      const char* nm[9] = {"softmax: wait S", "softmax: TMEM load S", "softmax: exp/pack", "softmax: P store+fence+arrive",
                           "softmax: item epilogue", "mma: wait P", "mma: wait K/V", "mma: total", "softmax: total"};
      for (int i = 0; i < 9; ++i)
        fprintf(stderr, "RC_ATTN_PROF %-30s %14llu cycles  %6.3f of its role total\n", nm[i], h[i],
                static_cast<double>(h[i]) / static_cast<double>(i >= 5 && i <= 7 ? (h[7] ? h[7] : 1) : (h[8] ? h[8] : 1)));
    }
    cudaFree(ctx->attn_prof);
  }
  delete ctx;
}

rc_status rc_decompose_prompt(const rc_prompt* pr, int32_t cap, int32_t* n_out, int32_t* token_ids, uint8_t* cls,
                              int64_t* src_id, int32_t* src_off, int32_t* seg_start) {
  if (!pr || !n_out) return fail(RC_E_INVALID, "null argument");
  if (pr->prefix_len < 0 || pr->n_hist < 0 || pr->n_cand < 0 || pr->n_tail < 0)
    return fail(RC_E_INVALID, "negative segment length");
  int64_t n = static_cast<int64_t>(pr->prefix_len) + pr->n_hist + pr->n_tail;
  for (int i = 0; i < pr->n_cand; ++i) {
    if (pr->cand_len[i] <= 0) return fail(RC_E_INVALID, "empty candidate block");
    n += pr->cand_len[i];
  }
  if (n > cap) return fail(RC_E_CAPACITY, "prompt longer than output capacity");
  int32_t p = 0, seg = 0;
  auto put = [&](int32_t t, uint8_t c, int64_t id, int32_t off) {
    token_ids[p] = t; cls[p] = c; src_id[p] = id; src_off[p] = off; ++p;
  };
  if (seg_start) seg_start[seg++] = p;
  for (int i = 0; i < pr->prefix_len; ++i) put(pr->prefix_tokens[i], RC_TOK_PREFIX, -1, 0);
  if (seg_start) seg_start[seg++] = p;
  for (int i = 0; i < pr->n_hist; ++i) put(pr->hist_tokens[i], RC_TOK_HIST, pr->hist_proto[i], 0);
  int64_t ct = 0;
  for (int c = 0; c < pr->n_cand; ++c) {
    if (seg_start) seg_start[seg++] = p;
    for (int j = 0; j < pr->cand_len[c]; ++j) put(pr->cand_tokens[ct + j], RC_TOK_ITEM, pr->cand_item[c], j);
    ct += pr->cand_len[c];
  }
  if (seg_start) seg_start[seg++] = p;
  for (int i = 0; i < pr->n_tail; ++i) put(pr->tail_tokens[i], RC_TOK_FORCED, -1, 0);
  *n_out = p;
  return RC_OK;
}

rc_status rc_pool_register_blocks(rc_ctx* c, int32_t kind, int32_t n_blocks, const uint64_t* ids, const int32_t* n_tokens,
                                  const int32_t* canon_pos, const void* kv, const float* scales, rc_stream stream) {
  if (!c || n_blocks < 0 || (n_blocks > 0 && (!ids || !n_tokens || !canon_pos || !kv)))
    return fail(RC_E_INVALID, "null argument");
  if (n_blocks == 0) return RC_OK;
  RC_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto* dir = kind == RC_POOL_ITEM_BF16 ? &c->items : kind == RC_POOL_HIST_INT8 ? &c->protos
              : kind == RC_POOL_PREFIX_BF16 ? &c->prefixes : kind == RC_POOL_ITEM_HOST_BF16 ? &c->host_items
              : nullptr;
  if (!dir) return fail(RC_E_INVALID, "unknown pool kind");
  if (kind == RC_POOL_HIST_INT8 && !scales) return fail(RC_E_INVALID, "history blocks need scales");
  int64_t total = 0;
  for (int i = 0; i < n_blocks; ++i) {
    if (n_tokens[i] <= 0) return fail(RC_E_INVALID, "empty block");
    if (kind == RC_POOL_HIST_INT8 && n_tokens[i] != 1) return fail(RC_E_INVALID, "prototype blocks are single tokens");
    if (kind == RC_POOL_PREFIX_BF16 && canon_pos[i] != 0) return fail(RC_E_INVALID, "prefix blocks start at 0");
    // the alignment offset Delta = position - canonical position indexes the RoPE table over
    // [-max_seq_len, max_seq_len]: canonical positions must lie inside one prompt
    if (canon_pos[i] < 0 || static_cast<int64_t>(canon_pos[i]) + n_tokens[i] > c->pd.max_seq_len)
      return fail(RC_E_INVALID, "canonical positions outside [0, max_seq_len)");
    if (dir->count(ids[i])) return fail(RC_E_EXISTS, "duplicate block id " + std::to_string(ids[i]));
    for (int j = 0; j < i; ++j)
      if (ids[j] == ids[i]) return fail(RC_E_EXISTS, "duplicate block id in call");
    total += n_tokens[i];
  }
  int64_t row0;
  int64_t rows_cap;
  if (kind == RC_POOL_ITEM_BF16) {
    row0 = c->item_alloc.alloc(total);
    if (row0 < 0) return fail(RC_E_CAPACITY, "item pool full");
    rows_cap = c->pd.item_rows;
  } else if (kind == RC_POOL_ITEM_HOST_BF16) {
    if (!c->host_pool) return fail(RC_E_INVALID, "no host tier (host_item_rows = 0)");
    if (c->host_used + total > c->pd.host_item_rows) return fail(RC_E_CAPACITY, "host-tier item pool full");
    row0 = c->host_used;
    rows_cap = c->pd.host_item_rows;
  } else if (kind == RC_POOL_HIST_INT8) {
    if (c->hist_used + total > c->pd.hist_rows) return fail(RC_E_CAPACITY, "history pool full");
    row0 = c->hist_used;
    rows_cap = c->pd.hist_rows;
  } else {
    if (c->prefix_used + total > c->pd.prefix_rows) return fail(RC_E_CAPACITY, "prefix pool full");
    row0 = c->prefix_used;
    rows_cap = c->pd.prefix_rows;
  }
  const int L = c->m.n_layers, Hk = c->m.n_kv_heads, dh = c->m.head_dim;
  cudaError_t e;
  if (kind == RC_POOL_HIST_INT8) {
    e = pool_transpose_launch(kv, 1, static_cast<int32_t>(total), L, Hk, dh, c->hist_q, rows_cap, row0, s);
    if (e == cudaSuccess) e = scale_transpose_launch(scales, static_cast<int32_t>(total), L, Hk, c->hist_s, rows_cap, row0, s);
    c->launches += 2;  // offline registration: counted, never profiled
  } else {
    e = pool_transpose_launch(kv, 2, static_cast<int32_t>(total), L, Hk, dh,
                              kind == RC_POOL_ITEM_BF16 ? c->item_pool
                              : kind == RC_POOL_ITEM_HOST_BF16 ? c->host_pool_dev : c->prefix_pool,
                              rows_cap, row0, s);
    c->launches += 1;
  }
  if (e != cudaSuccess) {
    if (kind == RC_POOL_ITEM_BF16) c->item_alloc.release(row0, total);
    return fail(RC_E_CUDA, std::string("register copy: ") + cudaGetErrorString(e));
  }
  int64_t r = row0;
  for (int i = 0; i < n_blocks; ++i) {
    (*dir)[ids[i]] = Block{r, n_tokens[i], canon_pos[i], false, 0};
    r += n_tokens[i];
  }
  if (kind == RC_POOL_HIST_INT8) {
    c->hist_used += total;
    // the dense device table of prototype ids < 2^31 (device-fed rc_assemble, NEXT-3)
    int64_t need = c->proto_tab_cap;
    for (int i = 0; i < n_blocks; ++i)
      if (ids[i] < (1ull << 31)) need = std::max<int64_t>(need, static_cast<int64_t>(ids[i]) + 1);
    if (static_cast<int64_t>(c->proto_tab_host.size()) < need) c->proto_tab_host.resize(need, make_int2(-1, 0));
    for (int i = 0; i < n_blocks; ++i)
      if (ids[i] < (1ull << 31)) {
        const Block& b = c->protos[ids[i]];
        c->proto_tab_host[ids[i]] = make_int2(static_cast<int>(b.row), b.canon);
      }
    if (need > c->proto_tab_cap) {
      if (c->proto_tab) cudaFree(c->proto_tab);
      cudaError_t e2;
      c->proto_tab = dev_alloc<int2>(need, &e2);
      if (e2 != cudaSuccess) { c->proto_tab = nullptr; c->proto_tab_cap = 0; return fail(RC_E_NOMEM, "prototype table"); }
      c->proto_tab_cap = need;
    }
    if (need > 0)
      RC_CUDA(cudaMemcpyAsync(c->proto_tab, c->proto_tab_host.data(), need * sizeof(int2), cudaMemcpyHostToDevice, s));
  }
  if (kind == RC_POOL_PREFIX_BF16) c->prefix_used += total;
  if (kind == RC_POOL_ITEM_HOST_BF16) c->host_used += total;
  return RC_OK;
}

rc_status rc_pool_contains(rc_ctx* c, int32_t kind, int32_t n, const uint64_t* ids, uint8_t* out) {
  if (!c || (n > 0 && (!ids || !out))) return fail(RC_E_INVALID, "null argument");
  auto* dir = kind == RC_POOL_ITEM_BF16 ? &c->items : kind == RC_POOL_HIST_INT8 ? &c->protos
              : kind == RC_POOL_PREFIX_BF16 ? &c->prefixes : kind == RC_POOL_ITEM_HOST_BF16 ? &c->host_items
              : nullptr;
  if (!dir) return fail(RC_E_INVALID, "unknown pool kind");
  for (int i = 0; i < n; ++i) out[i] = dir->count(ids[i]) ? 1 : 0;
  return RC_OK;
}

rc_status rc_pool_locate(rc_ctx* c, int32_t n, const uint64_t* ids, int64_t* rows_out) {
  if (!c || (n > 0 && (!ids || !rows_out))) return fail(RC_E_INVALID, "null argument");
  for (int i = 0; i < n; ++i) {
    auto it = c->items.find(ids[i]);
    rows_out[i] = it == c->items.end() ? -1 : it->second.row;
  }
  return RC_OK;
}

rc_status rc_assemble(rc_ctx* c, int32_t n_req, const rc_request* reqs, int32_t miss_policy, int32_t gather_from,
                      rc_seq* out_seqs, uint64_t* out_missing, int32_t* n_missing, rc_stream stream) {
  if (!c || n_req < 0 || (n_req > 0 && (!reqs || !out_seqs))) return fail(RC_E_INVALID, "null argument");
  if (gather_from < 0 || gather_from > c->m.n_layers) return fail(RC_E_INVALID, "gather_from out of range");
  if (miss_policy != RC_MISS_ERROR && miss_policy != RC_MISS_RECOMPUTE) return fail(RC_E_INVALID, "miss policy");
  RC_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // ---- validate + resolve everything before touching state (all-or-nothing)
  std::vector<Seq> built(n_req);
  std::vector<uint64_t> missing;
  std::vector<int4> meta_all, meta_pre;  // {dst_row(rel), src_row, delta, kind}; dst fixed up after alloc
  std::vector<int> meta_all_req, meta_pre_req;
  std::vector<int> n_hist_dev(n_req, 0);  // device-fed HIST tokens per request
  bool any_dev = false;
  for (int r = 0; r < n_req; ++r) any_dev |= reqs[r].hist_proto_dev != nullptr;
  if (any_dev && !c->proto_tab) return fail(RC_E_NOTFOUND, "device-fed prototypes but no prototype registered");
  for (int r = 0; r < n_req; ++r) {
    const rc_request& q = reqs[r];
    if (q.n <= 0 || q.n > c->pd.max_seq_len) return fail(RC_E_INVALID, "request length out of range");
    if (!q.token_ids || !q.cls || !q.src_id || !q.src_off || (q.n_cand > 0 && !q.cand_idtok))
      return fail(RC_E_INVALID, "null request array");
    Seq& sq = built[r];
    sq.n = q.n;
    sq.gather_from = gather_from;
    sq.tokens.assign(q.token_ids, q.token_ids + q.n);
    sq.cls.assign(q.cls, q.cls + q.n);
    sq.cand_idtok.assign(q.cand_idtok, q.cand_idtok + q.n_cand);
    int P = 0;
    while (P < q.n && q.cls[P] == RC_TOK_PREFIX) ++P;
    sq.P = P;
    const Block* pre = nullptr;
    if (P > 0) {
      auto it = c->prefixes.find(q.prefix_id);
      if (it == c->prefixes.end()) return fail(RC_E_NOTFOUND, "prefix block not registered");
      if (it->second.n < P) return fail(RC_E_INVALID, "prefix block shorter than the request's prefix");
      pre = &it->second;
    }
    for (int p = 0; p < q.n; ++p) {
      const int k = q.cls[p];
      if (q.token_ids[p] < 0 || q.token_ids[p] >= c->m.vocab) return fail(RC_E_INVALID, "token id out of range");
      if (k > RC_TOK_ITEM) return fail(RC_E_INVALID, "bad token class");
      if (k == RC_TOK_PREFIX) {
        if (p >= P) return fail(RC_E_INVALID, "PREFIX tokens must be the leading positions");
        meta_all.push_back(make_int4(p, static_cast<int>(pre->row + p), 0, RC_TOK_PREFIX));
        meta_all_req.push_back(r);
        if (gather_from > 0) { meta_pre.push_back(meta_all.back()); meta_pre_req.push_back(r); }
      } else if (k == RC_TOK_HIST) {
        if (q.hist_proto_dev) {  // resolved on the device (k_resolve_hist): y = (request, HIST index), z = position
          if (r >= (1 << 15) || n_hist_dev[r] >= (1 << 16)) return fail(RC_E_INVALID, "device-fed history too large");
          meta_all.push_back(make_int4(p, (r << 16) | n_hist_dev[r]++, p, RC_TOK_HIST_DEV));
          meta_all_req.push_back(r);
          continue;
        }
        auto it = c->protos.find(static_cast<uint64_t>(q.src_id[p]));
        if (it == c->protos.end()) return fail(RC_E_NOTFOUND, "prototype not registered: " + std::to_string(q.src_id[p]));
        meta_all.push_back(make_int4(p, static_cast<int>(it->second.row), p - it->second.canon, RC_TOK_HIST));
        meta_all_req.push_back(r);
      } else if (k == RC_TOK_ITEM) {
        auto it = c->items.find(static_cast<uint64_t>(q.src_id[p]));
        if (it == c->items.end() || q.src_off[p] < 0 || q.src_off[p] >= it->second.n) {
          if (it == c->items.end()) {
            if (std::find(missing.begin(), missing.end(), static_cast<uint64_t>(q.src_id[p])) == missing.end())
              missing.push_back(static_cast<uint64_t>(q.src_id[p]));
            sq.cls[p] = RC_TOK_FORCED;
            continue;
          }
          return fail(RC_E_INVALID, "item offset outside its block");
        }
        touch(c, it->first, it->second);
        const int delta = p - (it->second.canon + q.src_off[p]);
        meta_all.push_back(make_int4(p, static_cast<int>(it->second.row + q.src_off[p]), delta, RC_TOK_ITEM));
        meta_all_req.push_back(r);
      }
    }
  }
  ++c->use_clock;
  if (!missing.empty() && miss_policy == RC_MISS_ERROR) {
    if (n_missing) {
      const int cap = *n_missing;
      for (int i = 0; i < static_cast<int>(missing.size()) && i < cap && out_missing; ++i) out_missing[i] = missing[i];
      *n_missing = static_cast<int32_t>(missing.size());
    }
    return fail(RC_E_NOTFOUND, "candidate item blocks not resident");
  }
  if (n_missing) {
    const int cap = *n_missing;
    for (int i = 0; i < static_cast<int>(missing.size()) && i < cap && out_missing; ++i) out_missing[i] = missing[i];
    *n_missing = static_cast<int32_t>(missing.size());
  }
  // ---- allocate stitched ranges
  std::vector<int64_t> rows(n_req);
  for (int r = 0; r < n_req; ++r) {
    rows[r] = c->arena_alloc.alloc(built[r].n);
    if (rows[r] < 0) {
      for (int j = 0; j < r; ++j) c->arena_alloc.release(rows[j], built[j].n);
      return fail(RC_E_CAPACITY, "stitched-KV arena full");
    }
    built[r].arena_row = rows[r];
  }
  for (size_t i = 0; i < meta_all.size(); ++i) meta_all[i].x += static_cast<int>(rows[meta_all_req[i]]);
  for (size_t i = 0; i < meta_pre.size(); ++i) meta_pre[i].x += static_cast<int>(rows[meta_pre_req[i]]);
  // ---- zero-copy V: where each arena row's V lives at the layers >= c (identity unless ITEM / PREFIX)
  std::vector<int2> vcodes;
  if (c->zc_v) {
    for (int r = 0; r < n_req; ++r)
      for (int p = 0; p < built[r].n; ++p) vcodes.push_back(make_int2(static_cast<int>(rows[r] + p), static_cast<int>(rows[r] + p)));
    std::vector<int64_t> base(n_req + 1, 0);
    for (int r = 0; r < n_req; ++r) base[r + 1] = base[r] + built[r].n;
    for (size_t i = 0; i < meta_all.size(); ++i) {
      const int4& t = meta_all[i];
      const int r = meta_all_req[i];
      const int64_t pos = t.x - rows[r];
      if (t.w == RC_TOK_ITEM) vcodes[base[r] + pos].y = static_cast<int>((VSRC_ITEM << 30) | static_cast<uint32_t>(t.y));
      if (t.w == RC_TOK_PREFIX) vcodes[base[r] + pos].y = static_cast<int>((VSRC_PREFIX << 30) | static_cast<uint32_t>(t.y));
    }
  }
  // ---- metadata H2D + gather
  const size_t bytes = (meta_all.size() + meta_pre.size()) * sizeof(int4) + vcodes.size() * sizeof(int2) +
                       (any_dev ? n_req * sizeof(uint64_t) : 0);
  if (bytes > 0) {
    cudaError_t e;
    const int slot = c->stage.acquire(bytes, &e);
    if (slot < 0) {
      for (int r = 0; r < n_req; ++r) c->arena_alloc.release(rows[r], built[r].n);
      return fail(RC_E_NOMEM, std::string("staging: ") + cudaGetErrorString(e));
    }
    int4* hm = static_cast<int4*>(c->stage.host[slot]);
    std::copy(meta_all.begin(), meta_all.end(), hm);
    std::copy(meta_pre.begin(), meta_pre.end(), hm + meta_all.size());
    int2* hv = reinterpret_cast<int2*>(hm + meta_all.size() + meta_pre.size());
    std::copy(vcodes.begin(), vcodes.end(), hv);
    uint64_t* hp = reinterpret_cast<uint64_t*>(hv + vcodes.size());
    if (any_dev)
      for (int r = 0; r < n_req; ++r) hp[r] = reinterpret_cast<uint64_t>(reqs[r].hist_proto_dev);
    int4* dm = static_cast<int4*>(c->stage.dev[slot]);
    RC_CUDA(cudaMemcpyAsync(dm, hm, bytes, cudaMemcpyHostToDevice, s));
    if (any_dev)  // NEXT-3: prototype ids produced on the device -> pool rows and Delta, before the gather
      RC_LAUNCH(RC_K_SMALL, 0, meta_all.size() * 16.0, -1,
                resolve_hist_launch(dm, static_cast<int32_t>(meta_all.size()),
                                    reinterpret_cast<const uint64_t*>(reinterpret_cast<int2*>(dm + meta_all.size() + meta_pre.size()) + vcodes.size()),
                                    c->proto_tab, c->proto_tab_cap, c->dev_err, s));
    if (!vcodes.empty())
      RC_LAUNCH(RC_K_SMALL, 0, vcodes.size() * 12.0, -1,
                scatter_i32_launch(c->vmap, reinterpret_cast<const int2*>(dm + meta_all.size() + meta_pre.size()),
                                   static_cast<int32_t>(vcodes.size()), s));
    GatherArgs g{};
    g.n_kv_heads = c->m.n_kv_heads;
    g.head_dim = c->m.head_dim;
    g.item_pool = c->item_pool; g.item_rows = c->pd.item_rows;
    g.hist_q = c->hist_q; g.hist_s = c->hist_s; g.hist_rows = c->pd.hist_rows;
    g.prefix_pool = c->prefix_pool; g.prefix_rows = c->pd.prefix_rows;
    g.arena = c->arena; g.arena_rows = c->pd.arena_rows;
    g.rope_cos = c->rope_cos; g.rope_sin = c->rope_sin; g.rope_zero = c->rope_zero;
    // algorithmic bytes of the gather: every stitched element read once from its pool and
    // written once (bf16 rows 2*dh bytes; int8 rows dh bytes + one fp32 scale)
    const double row_b = 2.0 * c->m.head_dim, rows_per_tok = 2.0 * c->m.n_kv_heads;
    double b_all = 0, b_pre = 0;
    for (auto& t : meta_all)
      b_all += rows_per_tok * (t.w == RC_TOK_HIST || t.w == RC_TOK_HIST_DEV ? (c->m.head_dim + 4.0 + row_b) : 2 * row_b);
    b_pre = meta_pre.size() * rows_per_tok * 2 * row_b;
    g.meta = dm; g.n_tok = static_cast<int32_t>(meta_all.size());
    g.layer_begin = gather_from; g.layer_end = c->m.n_layers;
    g.skip_pool_v = c->zc_v ? 1 : 0;  // zero-copy V: item / prefix V read in place at the layers >= c
    if (g.n_tok > 0 && g.layer_end > g.layer_begin)
      RC_LAUNCH(RC_K_GATHER, 0, b_all * (g.layer_end - g.layer_begin), -1, gather_launch(g, c->num_sms, s));
    g.meta = dm + meta_all.size(); g.n_tok = static_cast<int32_t>(meta_pre.size());
    g.layer_begin = 0; g.layer_end = gather_from;
    g.skip_pool_v = 0;  // layers < c attend over the arena (their U rows are recomputed there)
    if (g.n_tok > 0 && g.layer_end > g.layer_begin)
      RC_LAUNCH(RC_K_GATHER, 0, b_pre * (g.layer_end - g.layer_begin), -1, gather_launch(g, c->num_sms, s));
    // the slot's device half is read by the gathers: reusable once they are done (any stream)
    RC_CUDA(cudaEventRecord(c->stage.ev[slot], s));
  }
  for (int r = 0; r < n_req; ++r) {
    const uint64_t id = c->next_seq++;
    c->seqs.emplace(id, std::move(built[r]));
    out_seqs[r] = id;
  }
  return RC_OK;
}

void rc_release(rc_ctx* c, int32_t n, const rc_seq* seqs) {
  if (!c || !seqs) return;
  for (int i = 0; i < n; ++i) {
    auto it = c->seqs.find(seqs[i]);
    if (it == c->seqs.end()) continue;
    c->arena_alloc.release(it->second.arena_row, it->second.n);
    c->seqs.erase(it);
  }
}

namespace {
struct ReqPlan {
  const Seq* sq;
  int32_t u_off, u_cnt, sel_off, sel_cnt, k_h, k_i, forced, window;  // the final Sel
  // gradual steps i = 0..g (R-GF); with g = 0 step 0 is the final Sel
  int32_t g_cnt[RC_MAX_GRADUAL + 1], g_off[RC_MAX_GRADUAL + 1], g_kh[RC_MAX_GRADUAL + 1], g_ki[RC_MAX_GRADUAL + 1];
};

int32_t budget(int32_t r_bp, int32_t count) { return static_cast<int32_t>((static_cast<int64_t>(r_bp) * count + 9999) / 10000); }

rc_status plan_requests(rc_ctx* c, int32_t n_req, const rc_seq* seqs, const rc_prefill_params* prm,
                        std::vector<ReqPlan>& plan) {
  if (!prm) return fail(RC_E_INVALID, "null params");
  if (!(prm->lambda >= 0.0f && prm->lambda <= 1.0f)) return fail(RC_E_INVALID, "lambda out of [0, 1]");
  if (prm->lambda < 1.0f && !c->attn_tc)
    return fail(RC_E_UNSUPPORTED, "lambda < 1 (attention-mass term) needs the tcgen05 attention (head_dim 128)");
  if (prm->r_rev_bp < 0 || prm->r_rev_bp > 10000 || prm->r_item_bp < 0 || prm->r_item_bp > 10000)
    return fail(RC_E_INVALID, "recompute ratio out of [0, 10000] bp");
  if (prm->check_layer < 0 || prm->check_layer >= c->m.n_layers) return fail(RC_E_INVALID, "check_layer out of range");
  if (prm->window < 0) return fail(RC_E_INVALID, "negative window");
  const int G = prm->gradual_layers;
  if (G < 0 || G > RC_MAX_GRADUAL) return fail(RC_E_INVALID, "gradual_layers out of [0, RC_MAX_GRADUAL]");
  if (G > 0) {
    if (prm->check_layer + G > c->m.n_layers - 1) return fail(RC_E_INVALID, "check_layer + gradual_layers beyond the last layer");
    if (prm->r_start_rev_bp < prm->r_rev_bp || prm->r_start_rev_bp > 10000 || prm->r_start_item_bp < prm->r_item_bp ||
        prm->r_start_item_bp > 10000)
      return fail(RC_E_INVALID, "gradual start ratios must lie in [r, 10000] bp");
  }
  // R-GF: r_i = r_start - floor((r_start - r) i / g)
  auto ratio = [&](int32_t r0, int32_t r, int i) {
    return G == 0 ? r : r0 - static_cast<int32_t>((static_cast<int64_t>(r0) - r) * i / G);
  };
  plan.resize(n_req);
  int32_t uo = 0, so = 0;
  int32_t go[RC_MAX_GRADUAL + 1] = {};
  for (int r = 0; r < n_req; ++r) {
    auto it = c->seqs.find(seqs[r]);
    if (it == c->seqs.end()) return fail(RC_E_NOTFOUND, "unknown sequence handle");
    const Seq& sq = it->second;
    if (prm->check_layer < sq.gather_from)
      return fail(RC_E_INVALID, "check_layer below the sequence's gather_from (layers not assembled)");
    ReqPlan& p = plan[r];
    p.sq = &sq;
    p.u_off = uo;
    p.u_cnt = sq.n - sq.P;
    p.window = prm->window;
    int nh = 0, ni = 0, nf = 0, nw = 0;
    for (int pos = sq.P; pos < sq.n; ++pos) {
      const bool in_win = prm->window > 0 && pos >= sq.n - prm->window;
      if (in_win) { ++nw; continue; }
      const int k = sq.cls[pos];
      nh += k == RC_TOK_HIST; ni += k == RC_TOK_ITEM; nf += k == RC_TOK_FORCED;
    }
    // the logits are read from the last selected row, so position n-1 must be recomputed:
    // FORCED (the instruction tail, R8) or inside the window
    if (prm->window == 0 && sq.cls[sq.n - 1] != RC_TOK_FORCED)
      return fail(RC_E_INVALID, "the last prompt position must be FORCED (instruction tail) or inside the window");
    p.k_h = budget(prm->r_rev_bp, nh);
    p.k_i = budget(prm->r_item_bp, ni);
    p.forced = nf + nw;
    p.sel_cnt = p.forced + p.k_h + p.k_i;
    if (p.sel_cnt == 0 || sq.n - 1 < sq.P) return fail(RC_E_INVALID, "request has no recomputed position");
    p.sel_off = so;
    for (int i = 0; i <= G; ++i) {
      p.g_kh[i] = budget(ratio(prm->r_start_rev_bp, prm->r_rev_bp, i), nh);
      p.g_ki[i] = budget(ratio(prm->r_start_item_bp, prm->r_item_bp, i), ni);
      p.g_cnt[i] = p.forced + p.g_kh[i] + p.g_ki[i];
      p.g_off[i] = go[i];
      go[i] += p.g_cnt[i];
    }
    uo += p.u_cnt;
    so += p.sel_cnt;
  }
  if (uo > c->Mx) return fail(RC_E_CAPACITY, "batch exceeds max_batch_tokens");
  return RC_OK;
}
}  // namespace

rc_status rc_sel_count(rc_ctx* c, int32_t n_req, const rc_seq* seqs, const rc_prefill_params* prm, int32_t* counts) {
  if (!c || !counts) return fail(RC_E_INVALID, "null argument");
  std::vector<ReqPlan> plan;
  rc_status st = plan_requests(c, n_req, seqs, prm, plan);
  if (st != RC_OK) return st;
  for (int r = 0; r < n_req; ++r) counts[r] = plan[r].sel_cnt;
  return RC_OK;
}

namespace {
// first half of a decoder layer over `rows` rows: RMSNorm + QKV projection with fused RoPE,
// q -> c->q, k/v -> arena rows d_dst. `dev` (gradual steps, R-GF): also score the k/v of the rows
// with dev->row_reuse[dev->dev_row[row]] against the stitched arena values they overwrite.
rc_status run_qkv(rc_ctx* c, int l, float* x, int32_t rows, const int32_t* d_pos, const int32_t* d_dst,
                  const EpiArgs* dev, cudaStream_t s) {
  const rc_model_desc& m = c->m;
  const int d = m.d_model, dh = m.head_dim, H = m.n_heads, Hk = m.n_kv_heads;
  const double R = rows, norm_b = R * d * 6.0;
  RC_LAUNCH(RC_K_SMALL, 0, norm_b, -1, rmsnorm_launch(x, nullptr, rows, d, c->ln1[l], m.rms_eps, c->a, s));
  EpiArgs ep = epi_base(c);
  ep.bias = c->bqkv ? c->bqkv + static_cast<size_t>(l) * c->Nqkv : nullptr;
  ep.pos = d_pos; ep.dst_row = d_dst;
  ep.q_out = c->q; ep.q_ld = H * dh;
  ep.arena_k = arena_layer(c, l, 0); ep.arena_v = arena_layer(c, l, 1);
  ep.head_stride = c->pd.arena_rows * dh;
  ep.rope_cos = c->rope_cos; ep.rope_sin = c->rope_sin; ep.rope_zero = c->rope_zero;
  ep.n_heads = H; ep.n_kv_heads = Hk; ep.head_dim = dh;
  if (dev) { ep.dev_out = dev->dev_out; ep.dev_row = dev->dev_row; ep.row_reuse = dev->row_reuse; }
  RC_LAUNCH(RC_K_GEMM, gemm_flops(R, c->Nqkv, d), gemm_bytes(R, c->Nqkv, d, 2), -1,
            gemm_launch(&c->mA_a, &c->mB_qkv[l], nullptr, rows, c->Nqkv, d, c->bn_qkv, dev ? EPI_QKV_DEV : EPI_QKV, ep,
                        c->num_sms, s, &c->mA_a64));
  return RC_OK;
}

// second half: attention of the `rows` query rows (q in c->q, positions d_pos) over the arena,
// O-projection + residual, RMSNorm, SwiGLU MLP + residual
rc_status run_rest(rc_ctx* c, int l, float* x, const CUtensorMap* mx, int32_t rows, const int32_t* d_pos,
                   const int4* d_tiles, int32_t n_tiles, int32_t n_splits, int32_t split_min, int paired,
                   double attn_flops, int attn_pending, int det, bool zc_layer, cudaStream_t s) {
  const rc_model_desc& m = c->m;
  const int d = m.d_model, dh = m.head_dim, H = m.n_heads, Hk = m.n_kv_heads, F = m.d_ff;
  const double R = rows, norm_b = R * d * 6.0;
  AttnArgs at{};
  at.q = c->q; at.o = c->o; at.qpos = d_pos; at.tiles = d_tiles; at.n_tiles = n_tiles;
  at.k = arena_layer(c, l, 0); at.v = arena_layer(c, l, 1); at.head_stride = c->pd.arena_rows * dh;
  at.n_heads = H; at.n_kv_heads = Hk; at.head_dim = dh;
  at.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(dh)));
  if (zc_layer && c->attn_tc) at.vsrc = layer_vsrc(c, l);  // NEXT-4: item / prefix V read in place
  static const int attn_debug = std::getenv("RC_ATTN_DEBUG") ? std::atoi(std::getenv("RC_ATTN_DEBUG")) : 0;
  at.debug_mode = attn_debug;
  static const bool attn_prof = std::getenv("RC_ATTN_PROF") && std::atoi(std::getenv("RC_ATTN_PROF")) == 1;
  if (attn_prof && !c->attn_prof) {
    cudaError_t e = cudaSuccess;
    c->attn_prof = dev_alloc<unsigned long long>(16, &e);
    if (e == cudaSuccess) cudaMemset(c->attn_prof, 0, 16 * sizeof(unsigned long long));
  }
  at.prof = c->attn_prof;
  // S_{j+1} TMEM load before the P_j hand-off: parity-green, measured slower at cfg3 batch 1 (attention
  // 1.59-1.60 -> 1.65 ms per step, 42.5 -> 44.0 us per selective-layer launch in ncu): off by default
  static const int s_prefetch = std::getenv("RC_ATTN_SPREFETCH") ? std::atoi(std::getenv("RC_ATTN_SPREFETCH")) : 0;
  at.s_prefetch = s_prefetch;
  at.n_splits = n_splits;
  at.split_min = split_min;
  if (paired == 2) at.chunk_per_cta = attn_chunk_per_cta();
  if (n_splits > 1 || paired == 2) {  // partial-output workspace, grown on first use
    const size_t need = static_cast<size_t>(n_tiles) * Hk * 128 * (paired == 2 ? ATTN_MAX_CHUNKS : 1);
    if (c->part_rows < need) {
      if (c->part_o) cudaFree(c->part_o);
      if (c->part_ml) cudaFree(c->part_ml);
      if (c->part_flag) cudaFree(c->part_flag);
      cudaError_t e;
      c->part_o = dev_alloc<float>(need * 128, &e);
      if (e == cudaSuccess) c->part_ml = dev_alloc<float>(need * 2, &e);
      // arrival counters per (tile, kv head): need / 128 >= n_tiles * Hk for every later launch that fits
      if (e == cudaSuccess) c->part_flag = dev_alloc<int32_t>(need / 128, &e);
      if (e == cudaSuccess) e = cudaMemset(c->part_flag, 0, need / 128 * sizeof(int32_t));
      if (e != cudaSuccess) { c->part_rows = 0; return fail(RC_E_NOMEM, "attention split workspace"); }
      c->part_rows = need;
    }
    at.part_o = c->part_o;
    at.part_ml = c->part_ml;
    at.split_flag = c->part_flag;  // per (logical tile, KV head) arrival counters, zero between launches
  }
  if (paired && !c->attn_ctr) {  // persistent paired kernel's work counter (reset by its last CTA)
    cudaError_t e = cudaSuccess;
    c->attn_ctr = dev_alloc<int32_t>(2, &e);
    if (e == cudaSuccess) e = cudaMemset(c->attn_ctr, 0, 2 * sizeof(int32_t));
    if (e != cudaSuccess) return fail(RC_E_NOMEM, "attention work counter");
  }
  at.work_ctr = c->attn_ctr;
  // early O-projection (RC_OPROJ_EARLY=1, opt-in): with the single-tile attention unsplit and the O-proj
  // on the transposed kernel, the O-proj's units wait per 256-row token tile for the attention CTAs
  // that write it instead of for the whole attention grid (its longest causal tiles). Bitwise the same
  // outputs in deterministic mode; measured within noise at cfg3 batch 1 r = 15 % and 1-1.5 % faster at
  // r = 10 / 20 % (profiles/r02_ab_oproj_early.txt): the board is at its power cap, so the overlapped
  // O-proj mostly trades clock for concurrency. Off by default.
  static const bool early_env = [] { const char* e = std::getenv("RC_OPROJ_EARLY"); return e && std::atoi(e) == 1; }();
  const bool early = early_env && c->early_on && !paired && c->attn_tc && n_splits == 1 && rows <= 1024 &&
                     !at.lse_out && gemm_use_transposed(rows, d, EPI_ADD_F32, dh, c->num_sms);
  if (early) at.ready = c->oproj_ready;
  if (paired)
    RC_LAUNCH(RC_K_ATTN, attn_flops, 0, attn_pending,
              attn_pair_launch(&c->mQ3, &c->mK_att[l], &c->mV_att[l], at, c->pd.arena_rows, s));
  else if (c->attn_tc)
    RC_LAUNCH(RC_K_ATTN, attn_flops, 0, attn_pending,
              attn_tc_launch(&c->mQ3, &c->mK_att[l], &c->mV_att[l], at, c->pd.arena_rows, s));
  else
    RC_LAUNCH(RC_K_ATTN, attn_flops, 0, attn_pending, attn_launch(at, s));
  EpiArgs eo = epi_base(c);
  eo.out = x; eo.ldo = d; eo.det = det;
  if (early) {
    eo.ready = c->oproj_ready;
    for (int i = 0; i < 4; ++i) eo.ready_tgt[i] = c->early_cnt[i] * Hk;
  }
  RC_LAUNCH(RC_K_GEMM, gemm_flops(R, d, H * dh), gemm_bytes(R, d, H * dh, 8), -1,
            gemm_launch(&c->mA_o, &c->mB_o[l], mx, rows, d, H * dh, c->bn_o, EPI_ADD_F32, eo, c->num_sms, s,
                        &c->mA_o64));
  RC_LAUNCH(RC_K_SMALL, 0, norm_b, -1, rmsnorm_launch(x, nullptr, rows, d, c->ln2[l], m.rms_eps, c->a, s));
  EpiArgs eg = epi_base(c);
  eg.out = c->h; eg.ldo = F;
  RC_LAUNCH(RC_K_GEMM, gemm_flops(R, 2.0 * F, d), gemm_bytes(R, 2.0 * F, d, 1), -1,
            gemm_launch(&c->mA_a, &c->mB_gu[l], nullptr, rows, 2 * F, d, 256, EPI_SWIGLU, eg, c->num_sms, s,
                        &c->mA_a64));
  EpiArgs ed = epi_base(c);
  ed.out = x; ed.ldo = d; ed.det = det;
  RC_LAUNCH(RC_K_GEMM, gemm_flops(R, d, F), gemm_bytes(R, d, F, 8), -1,
            gemm_launch(&c->mA_h, &c->mB_d[l], mx, rows, d, F, c->bn_d, EPI_ADD_F32, ed, c->num_sms, s,
                        &c->mA_h64));
  return RC_OK;
}

// one decoder layer over `rows` query rows (U or Sel) -- a2 / a5-a7
rc_status run_layer(rc_ctx* c, int l, float* x, const CUtensorMap* mx, int32_t rows, const int32_t* d_pos,
                    const int32_t* d_dst, const int4* d_tiles, int32_t n_tiles, int32_t n_splits, int32_t split_min,
                    int paired, double attn_flops, int attn_pending, int det, bool zc_layer, cudaStream_t s) {
  rc_status st = run_qkv(c, l, x, rows, d_pos, d_dst, nullptr, s);
  if (st != RC_OK) return st;
  return run_rest(c, l, x, mx, rows, d_pos, d_tiles, n_tiles, n_splits, split_min, paired, attn_flops, attn_pending,
                  det, zc_layer, s);
}
}  // namespace

namespace {
// NEXT-1 at the check layer c (a = RMSNorm(x_c[U]) already in c->a, D in c->dev): fresh Q/K/V of
// U into q and the scratch layer, the prefix keys (exact cache) copied next to them, pass 1 (row
// log-sum-exp over the fresh keys, k_attn_tc), pass 2 (column mass, k_attn_mass), combine into dev.
rc_status mass_scores(rc_ctx* c, int cL, int32_t U, const int32_t* d_pos, const int32_t* d_dst, const int4* d_ut,
                      int32_t n_ut, const int4* d_kt, int32_t n_kt, const int4* d_mreq, const std::vector<ReqPlan>& plan,
                      float lam, cudaStream_t s) {
  const rc_model_desc& m = c->m;
  const int d = m.d_model, dh = m.head_dim, H = m.n_heads, Hk = m.n_kv_heads;
  const int64_t rows = c->pd.arena_rows;
  cudaError_t e = cudaSuccess;
  if (!c->mass_k) {
    const size_t plane = static_cast<size_t>(Hk) * rows * dh;
    c->mass_k = dev_alloc<uint16_t>(plane, &e);
    if (e == cudaSuccess) c->mass_v = dev_alloc<uint16_t>(plane, &e);
    if (e == cudaSuccess) c->mass_lse = dev_alloc<float>(static_cast<size_t>(c->Mx) * H, &e);
    if (e == cudaSuccess) c->mass_a = dev_alloc<unsigned long long>(c->Mx, &e);
    if (e != cudaSuccess) return fail(RC_E_NOMEM, "attention-mass workspace");
    if (!make_tmap_bf16_2d(&c->mK_mass, c->mass_k, static_cast<uint64_t>(Hk) * rows, dh, dh, 128) ||
        !make_tmap_bf16_2d(&c->mV_mass, c->mass_v, static_cast<uint64_t>(Hk) * rows, dh, dh, 128))
      return fail(RC_E_CUDA, "attention-mass tensor maps");
  }
  EpiArgs ep = epi_base(c);
  ep.bias = c->bqkv ? c->bqkv + static_cast<size_t>(cL) * c->Nqkv : nullptr;
  ep.pos = d_pos; ep.dst_row = d_dst;
  ep.q_out = c->q; ep.q_ld = H * dh;
  ep.arena_k = c->mass_k; ep.arena_v = c->mass_v;
  ep.head_stride = rows * dh;
  ep.rope_cos = c->rope_cos; ep.rope_sin = c->rope_sin; ep.rope_zero = c->rope_zero;
  ep.n_heads = H; ep.n_kv_heads = Hk; ep.head_dim = dh;
  RC_LAUNCH(RC_K_GEMM, gemm_flops(U, c->Nqkv, d), gemm_bytes(U, c->Nqkv, d, 2), -1,
            gemm_launch(&c->mA_a, &c->mB_qkv[cL], nullptr, U, c->Nqkv, d, c->bn_qkv, EPI_QKV, ep, c->num_sms, s,
                        &c->mA_a64));
  for (auto& p : plan)  // the prefix keys are the exact cache: copy them next to the fresh U keys
    if (p.sq->P > 0)
      RC_LAUNCH(RC_K_SMALL, 0, 2.0 * p.sq->P * Hk * dh * 2, -1,
                copy_rows_launch(arena_layer(c, cL, 0), rows, p.sq->arena_row, c->mass_k, rows, p.sq->arena_row,
                                 p.sq->P, Hk, dh * 2, s));
  AttnArgs at{};
  at.q = c->q; at.o = c->o; at.qpos = d_pos; at.tiles = d_ut; at.n_tiles = n_ut;
  at.k = c->mass_k; at.v = c->mass_v; at.head_stride = rows * dh;
  at.n_heads = H; at.n_kv_heads = Hk; at.head_dim = dh;
  at.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(dh)));
  at.lse_out = c->mass_lse;
  RC_LAUNCH(RC_K_ATTN, 0, 0, -1, attn_tc_launch(&c->mQ3, &c->mK_mass, &c->mV_mass, at, rows, s));
  RC_CUDA(cudaMemsetAsync(c->mass_a, 0, static_cast<size_t>(U) * 8, s));
  MassArgs ma{};
  ma.key_tiles = d_kt; ma.n_key_tiles = n_kt; ma.req = d_mreq; ma.lse = c->mass_lse; ma.mass = c->mass_a;
  ma.n_heads = H; ma.n_kv_heads = Hk; ma.scale_log2 = at.scale_log2;
  RC_LAUNCH(RC_K_ATTN, 0, 0, -1, attn_mass_launch(&c->mQ3, &c->mK_mass, ma, rows, s));
  RC_LAUNCH(RC_K_SMALL, 0, U * 16.0, -1, mass_combine_launch(c->dev, c->mass_a, U, static_cast<double>(lam), s));
  return RC_OK;
}
}  // namespace

rc_status rc_selective_prefill(rc_ctx* c, int32_t n_req, const rc_seq* seqs, const rc_prefill_params* prm, float* logits,
                               float* cand_scores, int32_t* sel_pos_out, float* hidden, rc_stream stream) {
  if (!c || n_req <= 0 || !seqs) return fail(RC_E_INVALID, "null argument / empty batch");
  RC_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<ReqPlan> plan;
  rc_status st = plan_requests(c, n_req, seqs, prm, plan);
  if (st != RC_OK) return st;
  const rc_model_desc& m = c->m;
  const int L = m.n_layers, d = m.d_model, cL = prm->check_layer;
  const int TQ = c->attn_tq();
  const int32_t U = plan.back().u_off + plan.back().u_cnt;
  const int32_t S = plan.back().sel_off + plan.back().sel_cnt;
  int32_t n_cand = 0;
  for (auto& p : plan) n_cand += static_cast<int32_t>(p.sq->cand_idtok.size());
  // forced selection (test mode): validate
  const bool forced = prm->forced_sel != nullptr;
  const bool mass = !forced && prm->lambda < 1.0f;  // NEXT-1: Eq. 3 with the attention-mass term
  const int G = prm->gradual_layers;                // R-GF gradual filtering steps
  if (G > 0 && forced) return fail(RC_E_UNSUPPORTED, "gradual filtering with forced_sel");
  if (G > 0 && c->zc_v) return fail(RC_E_UNSUPPORTED, "gradual filtering with zero-copy V (RC_ZERO_COPY_V)");
  int32_t S_step[RC_MAX_GRADUAL + 1], trace_off[RC_MAX_GRADUAL + 2];
  trace_off[0] = 0;
  for (int i = 0; i <= G; ++i) {
    S_step[i] = plan.back().g_off[i] + plan.back().g_cnt[i];
    trace_off[i + 1] = trace_off[i] + S_step[i];
  }
  const int32_t S0 = S_step[0];
  if (forced) {
    if (!prm->forced_sel_off) return fail(RC_E_INVALID, "forced_sel needs forced_sel_off");
    for (int r = 0; r < n_req; ++r) {
      const int b = prm->forced_sel_off[r], e = prm->forced_sel_off[r + 1];
      if (e - b != plan[r].sel_cnt) return fail(RC_E_INVALID, "forced_sel count differs from the budget");
      const Seq& sq = *plan[r].sq;
      for (int i = b; i < e; ++i) {
        const int p = prm->forced_sel[i];
        if (p < sq.P || p >= sq.n || (i > b && p <= prm->forced_sel[i - 1]))
          return fail(RC_E_INVALID, "forced_sel positions must be ascending non-prefix positions");
      }
      if (prm->forced_sel[e - 1] != sq.n - 1) return fail(RC_E_INVALID, "forced_sel must contain the last position");
    }
  }
  // ---- host tables -> one staging slot
  Layout lay;
  const size_t o_tok = lay.add(U * 4), o_pos = lay.add(U * 4), o_dst = lay.add(U * 4), o_cls = lay.add(U),
               o_reuse = lay.add(U), o_req = lay.add(n_req * 16), o_req2 = lay.add(n_req * 16);
  int32_t n_ut = 0, n_st = 0;
  auto ntiles = [&](int cnt) { return (cnt + TQ - 1) / TQ; };
  for (auto& p : plan) { n_ut += ntiles(p.u_cnt); n_st += ntiles(p.sel_cnt); }
  // small grids (e.g. one request's selected rows) fill the SMs badly: split the KV range of every
  // query tile over several CTAs and merge (tcgen05 kernel only); every entry repeats per split
  if (prm->attn_kernel < RC_ATTN_AUTO || prm->attn_kernel > RC_ATTN_CHUNKED)
    return fail(RC_E_INVALID, "attn_kernel must be one of RC_ATTN_*");
  const int ak = c->attn_tc ? prm->attn_kernel : RC_ATTN_SINGLE;
  int split_u = 1, split_s = 1, smin_u = 0, smin_s = 0;
  if (ak == RC_ATTN_SPLIT2 || ak == RC_ATTN_ADAPTIVE) {
    split_u = mass ? 1 : 2;
    split_s = 2;
    if (ak == RC_ATTN_ADAPTIVE) {  // split only tiles reaching half the longest prompt's KV tiles
      int nmax = 0;
      for (auto& p : plan) nmax = std::max(nmax, p.sq->n);
      smin_s = std::max(2, (nmax + 127) / 128 / 2);
      smin_u = mass ? 0 : smin_s;
    }
  } else if (ak == RC_ATTN_AUTO && c->attn_tc) {
    int64_t ntok = 0;
    for (auto& p : plan) ntok += p.sq->n;
    const int est_kv = static_cast<int>(ntok / n_req / 128) + 1;
    split_u = mass ? 1 : attn_tc_choose_splits(n_ut, m.n_kv_heads, est_kv, c->num_sms, &smin_u);  // mass: U tiles feed pass 1
    if (mass) smin_u = 0;
    split_s = attn_tc_choose_splits(n_st, m.n_kv_heads, est_kv, c->num_sms, &smin_s);
  }
  // large grids: two query tiles of one request per CTA share every K/V tile load (k_attn_pair.cu);
  // a request's odd tile count is padded with one empty tile
  // (2 = the same kernel with device-sized KV chunks, for grids too small for plain pairs)
  int pair_u = 0, pair_s = 0;
  if (c->attn_tc && m.head_dim == 128 && (ak == RC_ATTN_AUTO || ak == RC_ATTN_PAIRED || ak == RC_ATTN_CHUNKED)) {
    auto mode = [&](int n_tiles, int split) {
      if (split != 1) return 0;
      if (ak == RC_ATTN_PAIRED || (ak == RC_ATTN_AUTO && attn_use_pairs(n_tiles, m.n_kv_heads, c->num_sms))) return 1;
      const int pairs_bound = n_tiles / 2 + n_req;  // padded pair count
      if (pairs_bound > ATTN_CHUNK_MAX_PAIRS) return ak == RC_ATTN_CHUNKED ? 1 : 0;
      return (ak == RC_ATTN_CHUNKED || (ak == RC_ATTN_AUTO && attn_chunk_auto())) ? 2 : 0;
    };
    pair_u = mode(n_ut, split_u);
    pair_s = mode(n_st, split_s);
    auto padded = [&](bool u) {
      int32_t n = 0;
      for (auto& p : plan) n += (ntiles(u ? p.u_cnt : p.sel_cnt) + 1) / 2 * 2;
      return n;
    };
    if (pair_u) n_ut = padded(true);
    if (pair_s) n_st = padded(false);
  }
  n_ut *= split_u;
  n_st *= split_s;
  // gradual steps 0..g-1: their own tile lists over Sel_i (launch shape of the final list)
  int32_t n_gt[RC_MAX_GRADUAL + 1] = {};
  size_t o_gt[RC_MAX_GRADUAL + 1] = {};
  for (int i = 0; i < G; ++i) {
    for (auto& p : plan) n_gt[i] += pair_s ? (ntiles(p.g_cnt[i]) + 1) / 2 * 2 : ntiles(p.g_cnt[i]);
    n_gt[i] *= split_s;
    o_gt[i] = lay.add(static_cast<size_t>(n_gt[i]) * 16);
  }
  const size_t o_rqg = lay.add(static_cast<size_t>(G) * n_req * 32);  // per step i >= 1: req, req2
  const size_t o_ut = lay.add(static_cast<size_t>(n_ut) * 16), o_st = lay.add(static_cast<size_t>(n_st) * 16),
               o_last = lay.add(n_req * 4), o_creq = lay.add(n_cand * 4), o_cid = lay.add(n_cand * 4),
               o_fsel = lay.add(forced ? static_cast<size_t>(S) * 12 : 0);
  // NEXT-1 key tiles: every 128-key tile of a request that holds U keys; per request {u_off, u_cnt, P, arena_row}
  int32_t n_kt = 0;
  if (mass)
    for (auto& p : plan) n_kt += (p.sq->n + 127) / 128 - p.sq->P / 128;
  const size_t o_kt = lay.add(static_cast<size_t>(n_kt) * 16), o_mreq = lay.add(mass ? n_req * 16 : 0);
  cudaError_t e;
  const int slot = c->stage.acquire(lay.off, &e);
  if (slot < 0) return fail(RC_E_NOMEM, std::string("staging: ") + cudaGetErrorString(e));
  uint8_t* hb = static_cast<uint8_t*>(c->stage.host[slot]);
  uint8_t* db = static_cast<uint8_t*>(c->stage.dev[slot]);
  auto H32 = [&](size_t o) { return reinterpret_cast<int32_t*>(hb + o); };
  int4* hreq = reinterpret_cast<int4*>(hb + o_req);
  int4* hreq2 = reinterpret_cast<int4*>(hb + o_req2);
  int4* hut = reinterpret_cast<int4*>(hb + o_ut);
  int4* hst = reinterpret_cast<int4*>(hb + o_st);
  int iu = 0, is = 0, ic = 0, ikt = 0;
  int kg[RC_MAX_GRADUAL + 1] = {};
  for (int r = 0; r < n_req; ++r) {
    const ReqPlan& p = plan[r];
    const Seq& sq = *p.sq;
    for (int i = 0; i < p.u_cnt; ++i) {
      const int pos = sq.P + i;
      H32(o_tok)[p.u_off + i] = sq.tokens[pos];
      H32(o_pos)[p.u_off + i] = pos;
      H32(o_dst)[p.u_off + i] = static_cast<int32_t>(sq.arena_row + pos);
      const bool in_win = p.window > 0 && pos >= sq.n - p.window;
      hb[o_cls + p.u_off + i] = sq.cls[pos];
      hb[o_reuse + p.u_off + i] = (!in_win && (sq.cls[pos] == RC_TOK_HIST || sq.cls[pos] == RC_TOK_ITEM)) ? 1 : 0;
    }
    hreq[r] = make_int4(p.u_off, p.u_cnt, p.g_off[0], sq.n);  // step 0 (= the final Sel without gradual steps)
    hreq2[r] = make_int4(p.g_kh[0], p.g_ki[0], static_cast<int>(sq.arena_row), p.window);
    const int arow = static_cast<int>(sq.arena_row);
    for (int i = 1; i <= G; ++i) {
      int4* rg = reinterpret_cast<int4*>(hb + o_rqg) + static_cast<size_t>(i - 1) * 2 * n_req;
      rg[r] = make_int4(p.u_off, p.u_cnt, p.g_off[i], sq.n);
      rg[n_req + r] = make_int4(p.g_kh[i], p.g_ki[i], arow, p.window);
    }
    for (int i = 0; i < G; ++i) {
      int4* ht = reinterpret_cast<int4*>(hb + o_gt[i]);
      int& k = kg[i];
      for (int j = 0; j < p.g_cnt[i]; j += TQ)
        for (int sp = 0; sp < split_s; ++sp) ht[k++] = make_int4(p.g_off[i] + j, std::min(TQ, p.g_cnt[i] - j), arow, sp);
      if (pair_s && ntiles(p.g_cnt[i]) % 2) ht[k++] = make_int4(p.g_off[i] + p.g_cnt[i], 0, arow, 0);
    }
    for (int i = 0; i < p.u_cnt; i += TQ)
      for (int sp = 0; sp < split_u; ++sp) hut[iu++] = make_int4(p.u_off + i, std::min(TQ, p.u_cnt - i), arow, sp);
    if (pair_u && ntiles(p.u_cnt) % 2) hut[iu++] = make_int4(p.u_off + p.u_cnt, 0, arow, 0);
    for (int i = 0; i < p.sel_cnt; i += TQ)
      for (int sp = 0; sp < split_s; ++sp) hst[is++] = make_int4(p.sel_off + i, std::min(TQ, p.sel_cnt - i), arow, sp);
    if (pair_s && ntiles(p.sel_cnt) % 2) hst[is++] = make_int4(p.sel_off + p.sel_cnt, 0, arow, 0);
    H32(o_last)[r] = p.sel_off + p.sel_cnt - 1;
    if (mass) {
      reinterpret_cast<int4*>(hb + o_mreq)[r] = make_int4(p.u_off, p.u_cnt, sq.P, arow);
      for (int k0 = sq.P / 128 * 128; k0 < sq.n; k0 += 128)
        reinterpret_cast<int4*>(hb + o_kt)[ikt++] = make_int4(r, k0, std::min(128, sq.n - k0), 0);
    }
    for (size_t j = 0; j < sq.cand_idtok.size(); ++j) { H32(o_creq)[ic] = r; H32(o_cid)[ic] = sq.cand_idtok[j]; ++ic; }
    if (forced) {
      int32_t* fs = H32(o_fsel);
      for (int i = 0; i < p.sel_cnt; ++i) {
        const int pos = prm->forced_sel[prm->forced_sel_off[r] + i];
        fs[p.sel_off + i] = pos;
        fs[S + p.sel_off + i] = static_cast<int32_t>(sq.arena_row + pos);
        fs[2 * S + p.sel_off + i] = p.u_off + (pos - sq.P);
      }
    }
  }
  RC_CUDA(cudaMemcpyAsync(db, hb, lay.off, cudaMemcpyHostToDevice, s));
  auto D32 = [&](size_t o) { return reinterpret_cast<int32_t*>(db + o); };
  const int4* d_ut = reinterpret_cast<const int4*>(db + o_ut);
  const int4* d_st = reinterpret_cast<const int4*>(db + o_st);

  // ---- a2: embedding + full layers l < c over U
  RC_LAUNCH(RC_K_SMALL, 0, static_cast<double>(U) * d * 6.0, -1, embed_launch(c->embed, D32(o_tok), U, d, c->x, s));
  double attn_u = 0;  // algorithmic attention flops over U: 4 H dh sum_{q in U} (pos_q + 1)
  for (auto& p : plan)
    for (int pos = p.sq->P; pos < p.sq->n; ++pos) attn_u += pos + 1.0;
  attn_u *= 4.0 * m.n_heads * m.head_dim;
  const int pend_idx = c->prof ? static_cast<int>(c->pend.size()) : -1;
  for (int l = 0; l < cL; ++l) {
    // the layers < c decide Sel: their residual sums are always order-fixed (reproducible selection)
    st = run_layer(c, l, c->x, &c->mC_x, U, D32(o_pos), D32(o_dst), d_ut, n_ut, split_u, smin_u, pair_u, attn_u, -1, 1,
                   false, s);
    if (st != RC_OK) return st;
  }
  // ---- a3: check-layer KV projection with fused RoPE + deviation epilogue
  if (!forced) {
    RC_CUDA(cudaMemsetAsync(c->dev, 0, static_cast<size_t>(U) * 8, s));
    RC_LAUNCH(RC_K_SMALL, 0, static_cast<double>(U) * d * 6.0, -1,
              rmsnorm_launch(c->x, nullptr, U, d, c->ln1[cL], m.rms_eps, c->a, s));
    EpiArgs ev = epi_base(c);
    ev.bias = c->bqkv ? c->bqkv + static_cast<size_t>(cL) * c->Nqkv + m.n_heads * m.head_dim : nullptr;
    ev.pos = D32(o_pos); ev.dst_row = D32(o_dst);
    ev.arena_k = arena_layer(c, cL, 0); ev.arena_v = arena_layer(c, cL, 1);
    ev.head_stride = c->pd.arena_rows * m.head_dim;
    ev.rope_cos = c->rope_cos; ev.rope_sin = c->rope_sin; ev.rope_zero = c->rope_zero;
    ev.n_heads = m.n_heads; ev.n_kv_heads = m.n_kv_heads; ev.head_dim = m.head_dim;
    ev.dev_out = c->dev; ev.row_reuse = reinterpret_cast<const uint8_t*>(db + o_reuse);
    ev.vsrc = layer_vsrc(c, cL);  // zero-copy V: the stitched V of items / prefix lives in the pools
    const double Nkv = 2.0 * m.n_kv_heads * m.head_dim;
    RC_LAUNCH(RC_K_GEMM, gemm_flops(U, Nkv, d), gemm_bytes(U, Nkv, d, 2), -1,
              gemm_launch(&c->mA_a, &c->mB_kv[cL], nullptr, U, 2 * m.n_kv_heads * m.head_dim, d, c->bn_kv, EPI_DEV, ev,
                          c->num_sms, s));
    if (mass) {  // NEXT-1: S = rint((1 - lambda) A + lambda D) over dev
      st = mass_scores(c, cL, U, D32(o_pos), D32(o_dst), d_ut, n_ut, reinterpret_cast<const int4*>(db + o_kt), n_kt,
                       reinterpret_cast<const int4*>(db + o_mreq), plan, prm->lambda, s);
      if (st != RC_OK) return st;
    }
    if (prm->score_out)
      RC_CUDA(cudaMemcpyAsync(prm->score_out, c->dev, static_cast<size_t>(U) * 8, cudaMemcpyDeviceToDevice, s));
    // ---- a4: selection
    SelectArgs sa{};
    sa.dev = c->dev; sa.ucls = reinterpret_cast<const uint8_t*>(db + o_cls);
    sa.req = reinterpret_cast<const int4*>(db + o_req); sa.req2 = reinterpret_cast<const int4*>(db + o_req2);
    sa.n_req = n_req; sa.sel_pos = c->sel_pos; sa.sel_dst = c->sel_dst; sa.sel_urow = c->sel_urow;
    RC_LAUNCH(RC_K_SELECT, 0, static_cast<double>(U) * 9.0, -1, select_launch(sa, s));
  } else {
    const int32_t* fs = D32(o_fsel);
    RC_CUDA(cudaMemcpyAsync(c->sel_pos, fs, S * 4, cudaMemcpyDeviceToDevice, s));
    RC_CUDA(cudaMemcpyAsync(c->sel_dst, fs + S, S * 4, cudaMemcpyDeviceToDevice, s));
    RC_CUDA(cudaMemcpyAsync(c->sel_urow, fs + 2 * S, S * 4, cudaMemcpyDeviceToDevice, s));
  }
  if (c->zc_v)  // Sel rows get fresh K/V in the arena at the layers >= c
    RC_LAUNCH(RC_K_SMALL, 0, S * 8.0, -1, vmap_identity_launch(c->vmap, c->sel_dst, S, s));
  if (prm->sel_trace)
    RC_CUDA(cudaMemcpyAsync(prm->sel_trace, c->sel_pos, static_cast<size_t>(S0) * 4, cudaMemcpyDeviceToDevice, s));
  RC_LAUNCH(RC_K_SMALL, 0, static_cast<double>(S0) * d * 8.0, -1,
            gather_rows_f32_launch(c->x, c->sel_urow, S0, d, c->xs, s));
  // ---- a5-a7: selective layers c..L-1 on Sel (gradual steps: layers c+1..c+g shrink it, R-GF)
  int32_t *sp = c->sel_pos, *sd = c->sel_dst, *su = c->sel_urow;
  int32_t *sp2 = nullptr, *sd2 = nullptr, *su2 = nullptr, *u2s = nullptr, *gmap = nullptr;
  if (G > 0) {
    if (!c->grad_buf) {
      c->grad_buf = dev_alloc<int32_t>(static_cast<size_t>(c->Mx) * 5, &e);
      if (e != cudaSuccess) { c->grad_buf = nullptr; return fail(RC_E_NOMEM, "gradual-filtering workspace"); }
    }
    sp2 = c->grad_buf; sd2 = sp2 + c->Mx; su2 = sd2 + c->Mx; u2s = su2 + c->Mx; gmap = u2s + c->Mx;
  }
  const int Hq = m.n_heads * m.head_dim;  // q row width (bf16), moved as Hq / 2 four-byte words
  int32_t cur = S0;
  // early O-projection over the final Sel list (one tile list for every selective layer, unsplit, not
  // paired, <= 4 token tiles of 256 rows): attention CTAs per token tile
  struct EarlyGuard { rc_ctx* c; ~EarlyGuard() { c->early_on = false; } } early_guard{c};
  c->early_on = false;
  if (G == 0 && split_s == 1 && !pair_s && S0 <= 1024) {
    bool ok = true;
    for (int i = 0; i < 4; ++i) c->early_cnt[i] = 0;
    for (int i = 0; i < n_st; ++i) {
      const int4 t = hst[i];
      if (t.y <= 0) continue;
      for (int tt = t.x / 256; tt <= (t.x + t.y - 1) / 256; ++tt) {
        if (tt >= 4) ok = false;
        else ++c->early_cnt[tt];
      }
    }
    c->early_on = ok;
  }
  for (int l = cL; l < L; ++l) {
    const int i = l - cL;
    const int det = prm->deterministic ? 1 : 0;
    const bool last_list = i >= G;  // the final Sel's tile list
    const int4* tl = last_list ? d_st : reinterpret_cast<const int4*>(db + o_gt[i]);
    const int32_t ntl = last_list ? n_st : n_gt[i];
    if (i == 0 || i > G) {
      st = run_layer(c, l, c->xs, &c->mC_xs, cur, sp, sd, tl, ntl, split_s, smin_s, pair_s, 0.0, pend_idx, det, c->zc_v, s);
      if (st != RC_OK) return st;
      continue;
    }
    // gradual step i: q/k/v of Sel_{i-1}, scored against the stitched k/v they overwrite
    RC_CUDA(cudaMemsetAsync(c->dev, 0, static_cast<size_t>(U) * 8, s));
    RC_CUDA(cudaMemsetAsync(u2s, 0xFF, static_cast<size_t>(U) * 4, s));
    RC_LAUNCH(RC_K_SMALL, 0, cur * 8.0, -1, scatter_index_launch(u2s, su, cur, s));
    EpiArgs dv{};
    dv.dev_out = c->dev; dv.dev_row = su; dv.row_reuse = reinterpret_cast<const uint8_t*>(db + o_reuse);
    st = run_qkv(c, l, c->xs, cur, sp, sd, &dv, s);
    if (st != RC_OK) return st;
    const int4* rg = reinterpret_cast<const int4*>(db + o_rqg) + static_cast<size_t>(i - 1) * 2 * n_req;
    SelectArgs sa{};
    sa.dev = c->dev; sa.ucls = reinterpret_cast<const uint8_t*>(db + o_cls);
    sa.req = rg; sa.req2 = rg + n_req;
    sa.n_req = n_req; sa.sel_pos = sp2; sa.sel_dst = sd2; sa.sel_urow = su2;
    sa.u2s = u2s; sa.map = gmap;
    RC_LAUNCH(RC_K_SELECT, 0, static_cast<double>(U) * 13.0, -1, select_launch(sa, s));
    const int32_t nxt = S_step[i];
    // compact the residual rows and the query rows of Sel_i (through scratch: x of U, o)
    RC_LAUNCH(RC_K_SMALL, 0, static_cast<double>(nxt) * d * 8.0, -1, gather_rows_f32_launch(c->xs, gmap, nxt, d, c->x, s));
    RC_CUDA(cudaMemcpyAsync(c->xs, c->x, static_cast<size_t>(nxt) * d * 4, cudaMemcpyDeviceToDevice, s));
    RC_LAUNCH(RC_K_SMALL, 0, static_cast<double>(nxt) * Hq * 4.0, -1,
              gather_rows_f32_launch(reinterpret_cast<const float*>(c->q), gmap, nxt, Hq / 2, reinterpret_cast<float*>(c->o), s));
    RC_CUDA(cudaMemcpyAsync(c->q, c->o, static_cast<size_t>(nxt) * Hq * 2, cudaMemcpyDeviceToDevice, s));
    std::swap(sp, sp2); std::swap(sd, sd2); std::swap(su, su2);
    cur = nxt;
    if (prm->sel_trace)
      RC_CUDA(cudaMemcpyAsync(prm->sel_trace + trace_off[i], sp, static_cast<size_t>(nxt) * 4, cudaMemcpyDeviceToDevice, s));
    st = run_rest(c, l, c->xs, &c->mC_xs, cur, sp, tl, ntl, split_s, smin_s, pair_s, 0.0, pend_idx, det, false, s);
    if (st != RC_OK) return st;
  }
  // ---- a8: final norm on each request's last position, LM head, candidate readout
  RC_LAUNCH(RC_K_SMALL, 0, static_cast<double>(n_req) * d * 6.0, -1,
            rmsnorm_launch(c->xs, D32(o_last), n_req, d, c->fnorm, m.rms_eps, c->a, s));
  float* lg = logits;
  if (!lg) {
    if (c->logits_rows < n_req) {
      if (c->logits) cudaFree(c->logits);
      c->logits = dev_alloc<float>(static_cast<size_t>(n_req) * m.vocab, &e);
      if (e != cudaSuccess) { c->logits = nullptr; c->logits_rows = 0; return fail(RC_E_NOMEM, "logits buffer"); }
      c->logits_rows = n_req;
    }
    lg = c->logits;
  }
  EpiArgs el = epi_base(c);
  el.out = lg; el.ldo = m.vocab;
  RC_LAUNCH(RC_K_LMHEAD, gemm_flops(n_req, m.vocab, d), gemm_bytes(n_req, m.vocab, d, 4), -1,
            gemm_launch(&c->mA_a, &c->mB_lm, nullptr, n_req, m.vocab, d, c->bn_lm, EPI_F32, el, c->num_sms, s));
  if (cand_scores && n_cand > 0)
    RC_LAUNCH(RC_K_SMALL, 0, n_cand * 12.0, -1,
              cand_scores_launch(lg, m.vocab, D32(o_creq), D32(o_cid), n_cand, cand_scores, s));
  if (c->prof) {  // Sel positions are chosen on the device: fetch them to count attention flops
    rc_ctx::Pending pd;
    pd.S = S;
    pd.layers = L - cL;
    if (cudaMallocHost(&pd.host, static_cast<size_t>(S) * 4) != cudaSuccess) return fail(RC_E_NOMEM, "profile buffer");
    RC_CUDA(cudaMemcpyAsync(pd.host, sp, static_cast<size_t>(S) * 4, cudaMemcpyDeviceToHost, s));
    c->pend.push_back(std::move(pd));
  }
  if (sel_pos_out) RC_CUDA(cudaMemcpyAsync(sel_pos_out, sp, static_cast<size_t>(S) * 4, cudaMemcpyDeviceToDevice, s));
  if (hidden) RC_CUDA(cudaMemcpyAsync(hidden, c->xs, static_cast<size_t>(S) * d * 4, cudaMemcpyDeviceToDevice, s));
  // every kernel of the layer loop reads the slot's device tables (tiles, positions, rows):
  // the slot is reusable once the last of them has run (the event is waited on by the host)
  RC_CUDA(cudaEventRecord(c->stage.ev[slot], s));
  return RC_OK;
}

rc_status rc_seq_read_kv(rc_ctx* c, rc_seq seq, int32_t layer, void* k_out, void* v_out, rc_stream stream) {
  if (!c || !k_out || !v_out) return fail(RC_E_INVALID, "null argument");
  auto it = c->seqs.find(seq);
  if (it == c->seqs.end()) return fail(RC_E_NOTFOUND, "unknown sequence");
  if (layer < 0 || layer >= c->m.n_layers) return fail(RC_E_INVALID, "layer out of range");
  RC_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  RC_LAUNCH(RC_K_SMALL, 0, 0, -1,
            read_kv_launch(c->arena, c->pd.arena_rows, layer, c->m.n_kv_heads, c->m.head_dim,
                           static_cast<int32_t>(it->second.arena_row), it->second.n, static_cast<uint16_t*>(k_out),
                           static_cast<uint16_t*>(v_out),
                           layer >= it->second.gather_from ? layer_vsrc(c, layer) : VSrc{}, s));
  return RC_OK;
}

rc_status rc_seq_export_kv(rc_ctx* c, rc_seq seq, int32_t pos0, int32_t n_tok, int32_t int8, void* kv_out,
                           float* scales_out, rc_stream stream) {
  if (!c || !kv_out || (int8 && !scales_out)) return fail(RC_E_INVALID, "null argument");
  auto it = c->seqs.find(seq);
  if (it == c->seqs.end()) return fail(RC_E_NOTFOUND, "unknown sequence");
  if (pos0 < 0 || n_tok < 0 || pos0 + n_tok > it->second.n) return fail(RC_E_INVALID, "position range outside the sequence");
  RC_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t planes = plane_count(c);
  RC_LAUNCH(RC_K_SMALL, 0, static_cast<double>(n_tok) * planes * c->m.head_dim * (int8 ? 3.0 : 4.0), -1,
            export_kv_launch(c->arena, c->pd.arena_rows, static_cast<int32_t>(planes), c->m.head_dim,
                             static_cast<int32_t>(it->second.arena_row + pos0), n_tok, int8, kv_out, scales_out, s));
  return RC_OK;
}

// ------------------------------------------------------------------ multi-GPU
rc_status rc_pool_export(rc_ctx* c, void* handle_out, int64_t* rows_out) {
  if (!c || !handle_out) return fail(RC_E_INVALID, "null argument");
  if (!c->item_pool) return fail(RC_E_INVALID, "no item pool");
  RC_CUDA(cudaSetDevice(c->device));
  cudaIpcMemHandle_t h;
  RC_CUDA(cudaIpcGetMemHandle(&h, c->item_pool));
  std::memcpy(handle_out, &h, sizeof(h));
  if (rows_out) *rows_out = c->pd.item_rows;
  return RC_OK;
}

rc_status rc_peer_attach(rc_ctx* c, int32_t n, const int32_t* rank, const int32_t* peer_dev, const void* const* handles,
                         const int64_t* rows) {
  if (!c || n < 0 || (n > 0 && (!rank || !handles || !rows))) return fail(RC_E_INVALID, "null argument");
  RC_CUDA(cudaSetDevice(c->device));
  cudaIpcMemHandle_t own{};
  const bool have_own = c->item_pool && cudaIpcGetMemHandle(&own, c->item_pool) == cudaSuccess;
  for (int i = 0; i < n; ++i) {
    if (have_own && std::memcmp(handles[i], &own, sizeof(own)) == 0) {
      c->peers[rank[i]] = {c->item_pool, c->pd.item_rows};  // loopback
      continue;
    }
    if (peer_dev && peer_dev[i] != c->device) {  // another process on this same device needs no P2P path
      int can = 0;
      cudaDeviceCanAccessPeer(&can, c->device, peer_dev[i]);
      if (!can) return fail(RC_E_PEER, "no P2P path to peer device " + std::to_string(peer_dev[i]));
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles[i], sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(RC_E_PEER, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    c->ipc_opened.push_back(p);
    c->peers[rank[i]] = {static_cast<const uint16_t*>(p), rows[i]};
  }
  return RC_OK;
}

rc_status rc_pool_list(rc_ctx* c, int32_t cap, uint64_t* ids, int64_t* rows, int32_t* n_tokens, int32_t* canon_pos,
                       int32_t* n_out) {
  if (!c || !n_out || cap < 0 || (cap > 0 && (!ids || !rows || !n_tokens || !canon_pos)))
    return fail(RC_E_INVALID, "null argument");
  int32_t n = 0;
  for (auto& kv : c->items) {
    if (kv.second.remote) continue;  // only blocks owned by this pool (not cached copies)
    if (n < cap) {
      ids[n] = kv.first; rows[n] = kv.second.row; n_tokens[n] = kv.second.n; canon_pos[n] = kv.second.canon;
    }
    ++n;
  }
  *n_out = n;
  return n > cap ? fail(RC_E_CAPACITY, "directory larger than cap (n_out holds the size)") : RC_OK;
}

rc_status rc_peer_directory(rc_ctx* c, int32_t peer_rank, int32_t n, const uint64_t* ids, const int64_t* rows,
                            const int32_t* n_tokens, const int32_t* canon_pos) {
  if (!c || n < 0 || (n > 0 && (!ids || !rows || !n_tokens || !canon_pos))) return fail(RC_E_INVALID, "null argument");
  auto pit = c->peers.find(peer_rank);
  if (pit == c->peers.end()) return fail(RC_E_PEER, "peer rank not attached");
  for (int i = 0; i < n; ++i)  // validate everything first (all-or-nothing)
    if (n_tokens[i] <= 0 || rows[i] < 0 || rows[i] + n_tokens[i] > pit->second.second || canon_pos[i] < 0 ||
        static_cast<int64_t>(canon_pos[i]) + n_tokens[i] > c->pd.max_seq_len)
      return fail(RC_E_INVALID, "directory entry outside the peer's pool or the position range");
  auto& dir = c->peer_dir[peer_rank];
  dir.clear();
  for (int i = 0; i < n; ++i) dir[ids[i]] = Block{rows[i], n_tokens[i], canon_pos[i], false, 0};
  return RC_OK;
}

rc_status rc_fetch_remote(rc_ctx* c, int32_t n_items, const uint64_t* ids, const int32_t* owner, rc_stream stream) {
  if (!c || n_items < 0 || (n_items > 0 && (!ids || !owner))) return fail(RC_E_INVALID, "null argument");
  if (n_items == 0) return RC_OK;
  if (!c->item_pool) return fail(RC_E_INVALID, "no item pool");
  RC_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // ---- validate and resolve before touching state
  std::vector<FetchItem> todo;
  std::set<uint64_t> seen;
  int64_t need = 0;
  for (int i = 0; i < n_items; ++i) {
    auto pit = c->peers.find(owner[i]);
    if (pit == c->peers.end()) return fail(RC_E_PEER, "owner rank not attached");
    if (c->items.count(ids[i]) || !seen.insert(ids[i]).second) continue;
    auto dit = c->peer_dir.find(owner[i]);
    const Block* b = nullptr;
    if (dit != c->peer_dir.end()) {
      auto bit = dit->second.find(ids[i]);
      if (bit != dit->second.end()) b = &bit->second;
    }
    if (!b) return fail(RC_E_NOTFOUND, "item " + std::to_string(ids[i]) + " not in owner's directory");
    todo.push_back(FetchItem{ids[i], pit->second.first, pit->second.second, b->row, b->n, b->canon});
    need += b->n;
  }
  if (need > c->pd.remote_rows) return fail(RC_E_CAPACITY, "remote region smaller than one fetch");
  // ---- protect the blocks of this call, plan rows (LRU evictions), then one batched copy
  ++c->use_clock;
  for (int i = 0; i < n_items; ++i) {
    auto it = c->items.find(ids[i]);
    if (it != c->items.end()) touch(c, it->first, it->second);
  }
  if (todo.empty()) return RC_OK;
  std::vector<int64_t> dst;
  rc_status st = plan_remote_rows(c, todo, dst);
  if (st != RC_OK) return st;
  std::vector<CopySeg> segs(todo.size());
  for (size_t i = 0; i < todo.size(); ++i)
    segs[i] = CopySeg{todo[i].src, todo[i].src_rows, todo[i].src_row, dst[i], todo[i].n, 0};
  cudaError_t e;
  const size_t bytes = segs.size() * sizeof(CopySeg);
  const int slot = c->stage.acquire(bytes, &e);
  if (slot < 0) return fail(RC_E_NOMEM, std::string("staging: ") + cudaGetErrorString(e));
  std::memcpy(c->stage.host[slot], segs.data(), bytes);
  RC_CUDA(cudaMemcpyAsync(c->stage.dev[slot], c->stage.host[slot], bytes, cudaMemcpyHostToDevice, s));
  const int64_t planes = plane_count(c);
  const int row_bytes = c->m.head_dim * 2;
  RC_LAUNCH(RC_K_FETCH, 0, 2.0 * planes * need * row_bytes, -1,
            copy_segments_launch(static_cast<const CopySeg*>(c->stage.dev[slot]), static_cast<int32_t>(segs.size()),
                                 need, c->item_pool, c->pd.item_rows, static_cast<int32_t>(planes), row_bytes, s));
  RC_CUDA(cudaEventRecord(c->stage.ev[slot], s));
  return RC_OK;
}

rc_status rc_fetch_host(rc_ctx* c, int32_t n_items, const uint64_t* ids, rc_stream stream) {
  if (!c || n_items < 0 || (n_items > 0 && !ids)) return fail(RC_E_INVALID, "null argument");
  if (!c->host_pool) return fail(RC_E_INVALID, "no host tier (host_item_rows = 0)");
  RC_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<FetchItem> todo;
  std::set<uint64_t> seen;
  int64_t need = 0;
  for (int i = 0; i < n_items; ++i) {
    if (c->items.count(ids[i]) || !seen.insert(ids[i]).second) continue;
    auto it = c->host_items.find(ids[i]);
    if (it == c->host_items.end()) return fail(RC_E_NOTFOUND, "item " + std::to_string(ids[i]) + " in no tier");
    todo.push_back(FetchItem{ids[i], nullptr, c->pd.host_item_rows, it->second.row, it->second.n, it->second.canon});
    need += it->second.n;
  }
  if (need > c->pd.remote_rows) return fail(RC_E_CAPACITY, "remote region smaller than one host fetch");
  ++c->use_clock;  // blocks of this call are protected from eviction by it
  for (int i = 0; i < n_items; ++i) {
    auto it = c->items.find(ids[i]);
    if (it != c->items.end()) touch(c, it->first, it->second);
  }
  if (todo.empty()) return RC_OK;
  std::vector<int64_t> dst;
  rc_status st = plan_remote_rows(c, todo, dst);
  if (st != RC_OK) return st;
  const int64_t planes = plane_count(c);
  const size_t row_bytes = static_cast<size_t>(c->m.head_dim) * 2;
  for (size_t i = 0; i < todo.size(); ++i)  // one 2-D copy per block on the copy engines (no SMs)
    RC_CUDA(cudaMemcpy2DAsync(c->item_pool + dst[i] * c->m.head_dim, c->pd.item_rows * row_bytes,
                              c->host_pool + todo[i].src_row * c->m.head_dim, c->pd.host_item_rows * row_bytes,
                              todo[i].n * row_bytes, planes, cudaMemcpyHostToDevice, s));
  return RC_OK;
}

// ------------------------------------------------------------------ NEXT-3 semantic library
rc_status rc_semlib_build(rc_ctx* c, int32_t n, const int32_t* tok, const int32_t* off, int32_t n_buckets,
                          const float* H, uint64_t seed) {
  if (!c || n <= 0 || !tok || !off || !H) return fail(RC_E_INVALID, "null argument / empty library");
  if (n_buckets < 1 || n_buckets > 32) return fail(RC_E_INVALID, "n_buckets must be in [1, 32]");
  for (int i = 0; i < n; ++i)
    if (off[i] < 0) return fail(RC_E_INVALID, "negative history offset");
  RC_CUDA(cudaSetDevice(c->device));
  for (void* p : c->semlib_bufs) cudaFree(p);
  c->semlib_bufs.clear();
  c->semlib = SemlibArgs{};
  constexpr int T = 8, D = 64;
  cudaError_t e = cudaSuccess;
  auto dalloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (e == cudaSuccess) e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) c->semlib_bufs.push_back(p);
    return p;
  };
  // positional codes: sin/cos(b 10000^(-k/8)) in fp64 by the C library, rounded once to fp32 (R-LSH)
  std::vector<float> pos(static_cast<size_t>(n_buckets) * 16);
  for (int b = 0; b < n_buckets; ++b)
    for (int k = 0; k < 8; ++k) {
      const double w = std::pow(10000.0, -static_cast<double>(k) / 8.0);
      pos[b * 16 + 2 * k] = static_cast<float>(std::sin(b * w));
      pos[b * 16 + 2 * k + 1] = static_cast<float>(std::cos(b * w));
    }
  auto* d_pos = static_cast<float*>(dalloc(pos.size() * 4));
  auto* d_H = static_cast<float*>(dalloc(static_cast<size_t>(T) * 16 * D * 4));
  auto* d_C = static_cast<float*>(dalloc(static_cast<size_t>(n) * D * 4));
  auto* d_tok = static_cast<int32_t*>(dalloc(static_cast<size_t>(n) * 4));
  auto* d_off = static_cast<int32_t*>(dalloc(static_cast<size_t>(n) * 4));
  auto* d_sig = static_cast<uint32_t*>(dalloc(static_cast<size_t>(T) * n * 4));
  auto* d_tsig = static_cast<uint32_t*>(dalloc(static_cast<size_t>(T) * n * 4));
  auto* d_tid = static_cast<int32_t*>(dalloc(static_cast<size_t>(T) * n * 4));
  auto* d_bid = static_cast<int32_t*>(dalloc(static_cast<size_t>(n) * 4));
  auto* d_bst = static_cast<int32_t*>(dalloc(static_cast<size_t>(n_buckets + 1) * 4));
  if (e != cudaSuccess) return fail(RC_E_NOMEM, "semantic library");
  RC_CUDA(cudaMemcpy(d_pos, pos.data(), pos.size() * 4, cudaMemcpyHostToDevice));
  RC_CUDA(cudaMemcpy(d_H, H, static_cast<size_t>(T) * 16 * D * 4, cudaMemcpyHostToDevice));
  RC_CUDA(cudaMemcpy(d_tok, tok, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice));
  RC_CUDA(cudaMemcpy(d_off, off, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice));
  SemlibArgs& sa = c->semlib;
  sa.seed = seed; sa.n_buckets = n_buckets; sa.n_proto = n; sa.pos_table = d_pos; sa.H = d_H; sa.C = d_C;
  cudaStream_t s = nullptr;  // offline build on the legacy stream (synchronised by the copy below)
  RC_LAUNCH(RC_K_SMALL, 0, 0, -1, semlib_embed_launch(sa, n, d_tok, d_off, d_C, d_sig, s));
  std::vector<uint32_t> sig(static_cast<size_t>(T) * n);
  RC_CUDA(cudaMemcpy(sig.data(), d_sig, sig.size() * 4, cudaMemcpyDeviceToHost));  // synchronises
  // per table: (signature, id) ascending -> the bucket map as two sorted arrays
  std::vector<uint32_t> tsig(sig.size());
  std::vector<int32_t> tid(sig.size());
  std::vector<int32_t> order(n);
  for (int t = 0; t < T; ++t) {
    for (int i = 0; i < n; ++i) order[i] = i;
    const uint32_t* st = sig.data() + static_cast<size_t>(t) * n;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return st[a] != st[b] ? st[a] < st[b] : a < b; });
    for (int i = 0; i < n; ++i) { tsig[static_cast<size_t>(t) * n + i] = st[order[i]]; tid[static_cast<size_t>(t) * n + i] = order[i]; }
  }
  // prototypes grouped by log bucket of their offset
  std::vector<int32_t> bst(n_buckets + 1, 0), bid(n);
  auto lb = [&](int o) { int b = 31 - __builtin_clz(static_cast<unsigned>(o) + 1u); return b < n_buckets - 1 ? b : n_buckets - 1; };
  for (int i = 0; i < n; ++i) ++bst[lb(off[i]) + 1];
  for (int b = 0; b < n_buckets; ++b) bst[b + 1] += bst[b];
  std::vector<int32_t> fill(bst.begin(), bst.end() - 1);
  for (int i = 0; i < n; ++i) bid[fill[lb(off[i])]++] = i;
  RC_CUDA(cudaMemcpy(d_tsig, tsig.data(), tsig.size() * 4, cudaMemcpyHostToDevice));
  RC_CUDA(cudaMemcpy(d_tid, tid.data(), tid.size() * 4, cudaMemcpyHostToDevice));
  RC_CUDA(cudaMemcpy(d_bid, bid.data(), bid.size() * 4, cudaMemcpyHostToDevice));
  RC_CUDA(cudaMemcpy(d_bst, bst.data(), bst.size() * 4, cudaMemcpyHostToDevice));
  sa.tab_sig = d_tsig; sa.tab_id = d_tid; sa.bucket_ids = d_bid; sa.bucket_start = d_bst;
  return RC_OK;
}

rc_status rc_semlib_match(rc_ctx* c, int32_t n, const int32_t* tok, const int32_t* off, int32_t* proto_out,
                          float* cos_out, rc_stream stream) {
  if (!c || n < 0 || (n > 0 && (!tok || !off || !proto_out || !cos_out))) return fail(RC_E_INVALID, "null argument");
  if (c->semlib.n_proto <= 0) return fail(RC_E_INVALID, "no semantic library (rc_semlib_build)");
  RC_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  RC_LAUNCH(RC_K_SMALL, 0, n * 16.0, -1, semlib_match_launch(c->semlib, n, tok, off, proto_out, cos_out, s));
  return RC_OK;
}

// ------------------------------------------------------------------ profiling
rc_status rc_profile_begin(rc_ctx* c) {
  if (!c) return fail(RC_E_INVALID, "null ctx");
  c->prof = true;
  c->recs.clear();
  c->ev_used = 0;
  for (auto& p : c->pend) cudaFreeHost(p.host);
  c->pend.clear();
  return RC_OK;
}

rc_status rc_profile_end(rc_ctx* c, int32_t n_kinds, double* ms, int64_t* count, double* flops, double* bytes) {
  if (!c || n_kinds <= 0 || !ms || !count || !flops || !bytes) return fail(RC_E_INVALID, "null argument");
  RC_CUDA(cudaSetDevice(c->device));
  RC_CUDA(cudaDeviceSynchronize());
  std::vector<double> pend_flops(c->pend.size(), 0.0);
  for (size_t i = 0; i < c->pend.size(); ++i) {
    double sum = 0;
    for (int j = 0; j < c->pend[i].S; ++j) sum += c->pend[i].host[j] + 1.0;
    pend_flops[i] = 4.0 * c->m.n_heads * c->m.head_dim * sum;
  }
  for (int k = 0; k < n_kinds; ++k) { ms[k] = 0; count[k] = 0; flops[k] = 0; bytes[k] = 0; }
  for (auto& r : c->recs) {
    if (r.kind >= n_kinds) continue;
    float t = 0;
    RC_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.kind] += t;
    count[r.kind] += 1;
    flops[r.kind] += r.pending >= 0 && r.pending < static_cast<int>(pend_flops.size()) ? pend_flops[r.pending] : r.flops;
    bytes[r.kind] += r.bytes;
  }
  c->prof = false;
  c->recs.clear();
  c->ev_used = 0;
  for (auto& p : c->pend) cudaFreeHost(p.host);
  c->pend.clear();
  return RC_OK;
}

// ------------------------------------------------------------------ diagnostics
rc_status rc_diag_gemm(int32_t M, int32_t N, int32_t K, const void* A, const void* B, float* C, int32_t bn,
                       rc_stream stream) {
  if (M <= 0 || N <= 0 || K <= 0 || !A || !B || !C || (bn != 128 && bn != 256)) return fail(RC_E_INVALID, "bad gemm args");
  CUtensorMap ma, mb;
  if (!make_tmap_bf16_2d(&ma, A, M, K, K, 128) || !make_tmap_bf16_2d(&mb, B, N, K, K, gemm_box_rows_b(bn)))
    return fail(RC_E_CUDA, "tensor map encode failed");
  int dev = 0, sms = 148;
  RC_CUDA(cudaGetDevice(&dev));
  RC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  EpiArgs ep{};
  ep.out = C; ep.ldo = N;
  RC_CUDA(gemm_launch(&ma, &mb, nullptr, M, N, K, bn, EPI_F32, ep, sms, static_cast<cudaStream_t>(stream)));
  return RC_OK;
}

rc_status rc_diag_gemm_add(int32_t M, int32_t N, int32_t K, const void* A, const void* B, float* X, int32_t transposed,
                           rc_stream stream) {
  if (M <= 0 || N <= 0 || K <= 0 || !A || !B || !X || N % 32) return fail(RC_E_INVALID, "bad gemm args");
  CUtensorMap ma, ma64, mb, mx;
  if (!make_tmap_bf16_2d(&ma, A, M, K, K, 128) || !make_tmap_bf16_2d(&ma64, A, M, K, K, gemm_t_box_rows()) ||
      !make_tmap_bf16_2d(&mb, B, N, K, K, gemm_box_rows_b(256)) || !make_tmap_f32_2d(&mx, X, M, N, N))
    return fail(RC_E_CUDA, "tensor map encode failed");
  int dev = 0, sms = 148;
  RC_CUDA(cudaGetDevice(&dev));
  RC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  float* ws = nullptr;
  int* cnt = nullptr;
  RC_CUDA(cudaMalloc(&ws, gemm_ws_floats() * sizeof(float)));
  RC_CUDA(cudaMalloc(&cnt, 2 * gemm_ws_slots() * sizeof(int)));
  RC_CUDA(cudaMemsetAsync(cnt, 0, 2 * gemm_ws_slots() * sizeof(int), s));
  EpiArgs ep{};
  ep.out = X; ep.ldo = N;
  ep.ws = ws; ep.ws_cnt = cnt; ep.ws_slots = gemm_ws_slots();
  cudaError_t e = gemm_launch(&ma, &mb, &mx, M, N, K, 256, EPI_ADD_F32, ep, sms, s, transposed ? &ma64 : nullptr);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(ws);
  cudaFree(cnt);
  if (e != cudaSuccess) return fail(RC_E_CUDA, std::string("diag gemm add: ") + cudaGetErrorString(e));
  return RC_OK;
}

rc_status rc_diag_deviation_select(int32_t n_u, int32_t width, const void* k_new, const void* k_st, const void* v_new,
                                   const void* v_st, const uint8_t* cls_host, int32_t prefix_len, int32_t r_rev_bp,
                                   int32_t r_item_bp, int32_t window, uint64_t* dev_out, int32_t* sel_out,
                                   int32_t* n_sel_out, rc_stream stream) {
  if (n_u <= 0 || n_u > 8192 || width <= 0 || !k_new || !k_st || !v_new || !v_st || !cls_host || !dev_out || !sel_out ||
      !n_sel_out || prefix_len < 0 || prefix_len + n_u > 8192)
    return fail(RC_E_INVALID, "bad diag args");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n = prefix_len + n_u;
  int nh = 0, ni = 0, nf = 0;
  for (int i = 0; i < n_u; ++i) {
    const int pos = prefix_len + i;
    if (window > 0 && pos >= n - window) { ++nf; continue; }
    nh += cls_host[i] == RC_TOK_HIST; ni += cls_host[i] == RC_TOK_ITEM; nf += cls_host[i] == RC_TOK_FORCED;
  }
  const int kh = budget(r_rev_bp, nh), ki = budget(r_item_bp, ni);
  const int cnt = nf + kh + ki;
  uint8_t* dcls = nullptr;
  int4* dreq = nullptr;
  int32_t *dp = nullptr, *dd = nullptr, *du = nullptr;
  RC_CUDA(cudaMalloc(&dcls, n_u));
  RC_CUDA(cudaMalloc(&dreq, 32));
  RC_CUDA(cudaMalloc(&dp, std::max(cnt, 1) * 4));
  RC_CUDA(cudaMalloc(&dd, std::max(cnt, 1) * 4));
  RC_CUDA(cudaMalloc(&du, std::max(cnt, 1) * 4));
  int4 hreq[2] = {make_int4(0, n_u, 0, n), make_int4(kh, ki, 0, window)};
  RC_CUDA(cudaMemcpyAsync(dcls, cls_host, n_u, cudaMemcpyHostToDevice, s));
  RC_CUDA(cudaMemcpyAsync(dreq, hreq, 32, cudaMemcpyHostToDevice, s));
  RC_CUDA(dev_diag_launch(static_cast<const uint16_t*>(k_new), static_cast<const uint16_t*>(k_st),
                          static_cast<const uint16_t*>(v_new), static_cast<const uint16_t*>(v_st), n_u, width,
                          reinterpret_cast<unsigned long long*>(dev_out), s));
  SelectArgs sa{};
  sa.dev = reinterpret_cast<const unsigned long long*>(dev_out);
  sa.ucls = dcls; sa.req = dreq; sa.req2 = dreq + 1; sa.n_req = 1;
  sa.sel_pos = dp; sa.sel_dst = dd; sa.sel_urow = du;
  RC_CUDA(select_launch(sa, s));
  RC_CUDA(cudaMemcpyAsync(sel_out, dp, cnt * 4, cudaMemcpyDeviceToDevice, s));
  RC_CUDA(cudaStreamSynchronize(s));
  cudaFree(dcls); cudaFree(dreq); cudaFree(dp); cudaFree(dd); cudaFree(du);
  *n_sel_out = cnt;
  return RC_OK;
}

}  // extern "C"
