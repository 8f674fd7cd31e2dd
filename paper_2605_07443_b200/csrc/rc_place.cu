// Host-side multi-GPU orchestration of librc: Alg. 1 similarity-aware item
// placement with global replicas and the Eq. 2 affinity router.
//
// Placement: heat from a historical trace, top hot_bp/10000 of the items replicated on every
// instance, co-occurrence graph of the cold items, k-way partition minimising the edge cut under a
// token-weight balance constraint -- a self-contained multilevel scheme in place of METIS:
// heavy-edge matching coarsening, greedy connectivity-driven initial assignment, and boundary
// refinement (positive-gain moves that keep balance) at every uncoarsening level. Deterministic.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <tuple>
#include <string>
#include <vector>

#include "../../include/rc.h"
#include "rc_internal.h"

namespace {
rc_status perr(rc_status c, const char* m) { return rc::set_error(c, m); }

struct Graph {
  int n = 0;
  std::vector<int64_t> w;                      // node token weight
  std::vector<int64_t> off;                    // CSR
  std::vector<int32_t> adj;
  std::vector<int64_t> ew;
};

// CSR from an edge map given as sorted (u, v, w) triples with u < v
Graph build_csr(int n, const std::vector<int64_t>& w, std::vector<std::tuple<int, int, int64_t>>& edges) {
  Graph g;
  g.n = n;
  g.w = w;
  std::vector<int64_t> deg(n + 1, 0);
  for (auto& e : edges) { deg[std::get<0>(e) + 1]++; deg[std::get<1>(e) + 1]++; }
  g.off.assign(n + 1, 0);
  for (int i = 0; i < n; ++i) g.off[i + 1] = g.off[i] + deg[i + 1];
  g.adj.resize(g.off[n]);
  g.ew.resize(g.off[n]);
  std::vector<int64_t> pos(g.off.begin(), g.off.end() - 1);
  for (auto& e : edges) {
    const int a = std::get<0>(e), b = std::get<1>(e);
    const int64_t x = std::get<2>(e);
    g.adj[pos[a]] = b; g.ew[pos[a]++] = x;
    g.adj[pos[b]] = a; g.ew[pos[b]++] = x;
  }
  return g;
}

// heavy-edge matching -> coarse graph; cmap[v] = coarse node of v
Graph coarsen(const Graph& g, std::vector<int>& cmap) {
  std::vector<int> match(g.n, -1);
  // visit nodes in ascending weight (light nodes first) for balanced coarse weights; ties by id
  std::vector<int> order(g.n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return g.w[a] < g.w[b]; });
  for (int v : order) {
    if (match[v] >= 0) continue;
    int best = -1;
    int64_t bw = 0;
    for (int64_t e = g.off[v]; e < g.off[v + 1]; ++e) {
      const int u = g.adj[e];
      if (u == v || match[u] >= 0) continue;
      if (g.ew[e] > bw || (g.ew[e] == bw && best >= 0 && u < best)) { bw = g.ew[e]; best = u; }
    }
    match[v] = best >= 0 ? best : v;
    if (best >= 0) match[best] = v;
  }
  cmap.assign(g.n, -1);
  int nc = 0;
  for (int v = 0; v < g.n; ++v) {
    if (cmap[v] >= 0) continue;
    cmap[v] = nc;
    if (match[v] != v && match[v] >= 0) cmap[match[v]] = nc;
    ++nc;
  }
  std::vector<int64_t> cw(nc, 0);
  for (int v = 0; v < g.n; ++v) cw[cmap[v]] += g.w[v];
  std::vector<std::tuple<int, int, int64_t>> ce;
  ce.reserve(g.adj.size() / 2);
  for (int v = 0; v < g.n; ++v)
    for (int64_t e = g.off[v]; e < g.off[v + 1]; ++e) {
      const int a = cmap[v], b = cmap[g.adj[e]];
      if (a < b) ce.emplace_back(a, b, g.ew[e]);
    }
  std::sort(ce.begin(), ce.end());
  std::vector<std::tuple<int, int, int64_t>> merged;
  for (auto& e : ce) {
    if (!merged.empty() && std::get<0>(merged.back()) == std::get<0>(e) && std::get<1>(merged.back()) == std::get<1>(e))
      std::get<2>(merged.back()) += std::get<2>(e);
    else
      merged.push_back(e);
  }
  return build_csr(nc, cw, merged);
}

// positive-gain boundary moves under the balance cap, fixed scan order
void refine(const Graph& g, std::vector<int>& part, int k, int64_t cap, int passes) {
  std::vector<int64_t> load(k, 0);
  for (int v = 0; v < g.n; ++v) load[part[v]] += g.w[v];
  std::vector<int64_t> conn(k);
  for (int it = 0; it < passes; ++it) {
    bool moved = false;
    for (int v = 0; v < g.n; ++v) {
      std::fill(conn.begin(), conn.end(), 0);
      for (int64_t e = g.off[v]; e < g.off[v + 1]; ++e) conn[part[g.adj[e]]] += g.ew[e];
      const int p = part[v];
      int best = p;
      int64_t gain = 0;
      for (int q = 0; q < k; ++q) {
        if (q == p || load[q] + g.w[v] > cap) continue;
        const int64_t gq = conn[q] - conn[p];
        if (gq > gain || (gq == gain && gq > 0 && q < best)) { gain = gq; best = q; }
      }
      if (best != p) {
        load[p] -= g.w[v];
        load[best] += g.w[v];
        part[v] = best;
        moved = true;
      }
    }
    if (!moved) break;
  }
}

// greedy initial assignment: heaviest first, to the part with most connectivity that fits
std::vector<int> initial(const Graph& g, int k, int64_t cap) {
  std::vector<int> order(g.n), part(g.n, -1);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return g.w[a] > g.w[b]; });
  std::vector<int64_t> load(k, 0), conn(k);
  for (int v : order) {
    std::fill(conn.begin(), conn.end(), 0);
    for (int64_t e = g.off[v]; e < g.off[v + 1]; ++e)
      if (part[g.adj[e]] >= 0) conn[part[g.adj[e]]] += g.ew[e];
    int best = -1;
    for (int q = 0; q < k; ++q) {
      if (load[q] + g.w[v] > cap) continue;
      if (best < 0 || conn[q] > conn[best] || (conn[q] == conn[best] && load[q] < load[best])) best = q;
    }
    if (best < 0) best = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
    part[v] = best;
    load[best] += g.w[v];
  }
  return part;
}

std::vector<int> partition(const Graph& g0, int k, double eps, int passes) {
  int64_t total = std::accumulate(g0.w.begin(), g0.w.end(), int64_t(0));
  const int64_t cap = static_cast<int64_t>(std::floor((1.0 + eps) * static_cast<double>(total) / k));
  std::vector<Graph> levels{g0};
  std::vector<std::vector<int>> maps;
  while (levels.back().n > std::max(40 * k, 200)) {
    std::vector<int> cmap;
    Graph c = coarsen(levels.back(), cmap);
    if (c.n > levels.back().n * 0.95) break;  // no progress (sparse graph)
    maps.push_back(std::move(cmap));
    levels.push_back(std::move(c));
  }
  std::vector<int> part = initial(levels.back(), k, cap);
  refine(levels.back(), part, k, cap, passes);
  for (int lv = static_cast<int>(maps.size()) - 1; lv >= 0; --lv) {
    const Graph& fine = levels[lv];
    std::vector<int> fp(fine.n);
    for (int v = 0; v < fine.n; ++v) fp[v] = part[maps[lv][v]];
    part.swap(fp);
    refine(fine, part, k, cap, passes);
  }
  return part;
}
}  // namespace

extern "C" {

rc_status rc_place_items(int32_t n_items, const int32_t* item_tokens, int32_t n_hist, const int64_t* hist_off,
                         const int32_t* hist_items, int32_t k, int32_t hot_bp, double balance_eps, int32_t passes,
                         int32_t* part_out, int64_t* cut_out, int64_t* heat_out) {
  if (n_items <= 0 || !item_tokens || k <= 0 || !part_out || hot_bp < 0 || hot_bp >= 10000 || balance_eps <= 0 ||
      (n_hist > 0 && (!hist_off || !hist_items)))
    return perr(RC_E_INVALID, "bad placement arguments");
  // Phase 1: heat
  std::vector<int64_t> h(n_items, 0);
  for (int r = 0; r < n_hist; ++r)
    for (int64_t e = hist_off[r]; e < hist_off[r + 1]; ++e) {
      const int i = hist_items[e];
      if (i < 0 || i >= n_items) return perr(RC_E_INVALID, "historical item id out of range");
      h[i]++;
    }
  // Phase 2: hot = ceil(hot_bp/1e4 * n) by heat desc, ties -> smaller id; replicated (-1)
  const int n_hot = static_cast<int>((static_cast<int64_t>(hot_bp) * n_items + 9999) / 10000);
  std::vector<int> order(n_items);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return h[a] > h[b]; });
  std::vector<int> cold_id(n_items, -1), cold;
  std::vector<char> hot(n_items, 0);
  for (int j = 0; j < n_hot; ++j) hot[order[j]] = 1;
  for (int i = 0; i < n_items; ++i)
    if (!hot[i]) { cold_id[i] = static_cast<int>(cold.size()); cold.push_back(i); }
  // Phase 3-4: co-occurrence graph over cold items (same historical request): every co-occurring
  // pair as one 64-bit key (u << 32 | v, u < v), sorted, runs counted = edge weights (8 bytes per
  // pair occurrence: a 1M-item catalog with a 50K-request trace is ~60M pairs)
  std::vector<uint64_t> keys;
  std::vector<int> tmp;
  for (int r = 0; r < n_hist; ++r) {
    tmp.clear();
    for (int64_t e = hist_off[r]; e < hist_off[r + 1]; ++e)
      if (!hot[hist_items[e]]) tmp.push_back(cold_id[hist_items[e]]);
    std::sort(tmp.begin(), tmp.end());
    tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
    for (size_t a = 0; a < tmp.size(); ++a)
      for (size_t b = a + 1; b < tmp.size(); ++b)
        keys.push_back(static_cast<uint64_t>(tmp[a]) << 32 | static_cast<uint32_t>(tmp[b]));
  }
  std::sort(keys.begin(), keys.end());
  std::vector<std::tuple<int, int, int64_t>> merged;
  for (size_t i = 0; i < keys.size();) {
    size_t j = i;
    while (j < keys.size() && keys[j] == keys[i]) ++j;
    merged.emplace_back(static_cast<int>(keys[i] >> 32), static_cast<int>(keys[i] & 0xffffffffu),
                        static_cast<int64_t>(j - i));
    i = j;
  }
  std::vector<uint64_t>().swap(keys);
  std::vector<int64_t> w(cold.size());
  for (size_t c = 0; c < cold.size(); ++c) w[c] = item_tokens[cold[c]];
  Graph g = build_csr(static_cast<int>(cold.size()), w, merged);
  // Phase 5
  std::vector<int> part = k == 1 ? std::vector<int>(cold.size(), 0) : partition(g, k, balance_eps, passes);
  int64_t cut = 0;
  for (auto& e : merged)
    if (part[std::get<0>(e)] != part[std::get<1>(e)]) cut += std::get<2>(e);
  for (int i = 0; i < n_items; ++i) part_out[i] = hot[i] ? -1 : part[cold_id[i]];
  if (cut_out) *cut_out = cut;
  if (heat_out)
    for (int i = 0; i < n_items; ++i) heat_out[i] = h[i];
  return RC_OK;
}

rc_status rc_route(int32_t n_req, const int64_t* req_off, const int32_t* req_items, const int64_t* req_tokens,
                   int32_t k, int32_t n_items, const uint8_t* resident, double alpha, double beta, int64_t* backlog,
                   int32_t* route_out) {
  if (n_req < 0 || k <= 0 || n_items <= 0 || !resident || !backlog || (n_req > 0 && (!req_off || !req_items ||
                                                                                      !req_tokens || !route_out)))
    return perr(RC_E_INVALID, "bad routing arguments");
  for (int r = 0; r < n_req; ++r) {
    const int64_t b = req_off[r], e = req_off[r + 1];
    if (e <= b) return perr(RC_E_INVALID, "request without candidates");
    int64_t mx = 1;
    for (int p = 0; p < k; ++p) mx = std::max(mx, backlog[p]);
    int best = 0;
    double best_s = -1e300;
    for (int p = 0; p < k; ++p) {
      int64_t hits = 0;
      for (int64_t j = b; j < e; ++j) {
        const int it = req_items[j];
        if (it < 0 || it >= n_items) return perr(RC_E_INVALID, "candidate id out of range");
        hits += resident[static_cast<int64_t>(p) * n_items + it] ? 1 : 0;
      }
      const double hit = static_cast<double>(hits) / static_cast<double>(e - b);  // Hit(R, p)
      const double load = static_cast<double>(backlog[p]) / static_cast<double>(mx);
      const double t1 = alpha * hit;
      const double t2 = beta * (1.0 - load);
      const double s = t1 + t2;  // Eq. 2
      if (s > best_s) { best_s = s; best = p; }  // strict: ties keep the smaller p
    }
    route_out[r] = best;
    backlog[best] += req_tokens[r];
  }
  return RC_OK;
}

}  // extern "C"
