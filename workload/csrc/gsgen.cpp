// gsgen.cpp -- seeded host-side workload generator (SUPPORT).
//
// Produces the synthetic stand-ins for the paper's datasets (Table 1):
//   1. a Chung-Lu expected-degree power-law parent graph (SURVEY §8(d) "Parent graph"),
//   2. a frontier-sampled node set V_s (Alg. 2, read as SURVEY R9),
//   3. node clipping to a multiple of `clip` (§7.2),
//   4. the induced subgraph G_s with ascending local IDs (Alg. 2 line 9).
//
// This module holds NONE of the GCN layer's arithmetic (no normalization, no products):
// it only emits integer CSR structure. Both the fp64 oracle (oracle/) and the CUDA path
// (paper_2010_03166_b200/) consume its output as *inputs*; neither links the other.
//
// RNG: splitmix64-seeded xoshiro256** (pure integer, reproducible across hosts).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

namespace {

struct Rng {
  uint64_t s[4];
  static uint64_t splitmix(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  explicit Rng(uint64_t seed) {
    uint64_t x = seed;
    for (auto& v : s) v = splitmix(x);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    uint64_t r = rotl(s[1] * 5, 7) * 9;
    uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
    s[2] ^= t; s[3] = rotl(s[3], 45);
    return r;
  }
  // uniform double in [0,1)
  double uniform() { return (next() >> 11) * (1.0 / 9007199254740992.0); }
  // uniform integer in [0, n) (Lemire's nearly-divisionless, exact)
  uint64_t below(uint64_t n) {
    uint64_t x = next();
    __uint128_t m = (__uint128_t)x * n;
    uint64_t l = (uint64_t)m;
    if (l < n) {
      uint64_t t = (0 - n) % n;
      while (l < t) { x = next(); m = (__uint128_t)x * n; l = (uint64_t)m; }
    }
    return (uint64_t)(m >> 64);
  }
};

// Mean of a continuous Pareto density  c * w^-gamma  on [a, b].
double pareto_mean(double a, double b, double gamma) {
  double al = gamma - 1.0;
  double c = al / (std::pow(a, -al) - std::pow(b, -al));
  if (std::fabs(gamma - 2.0) < 1e-12) return c * (std::log(b) - std::log(a));
  return c * (std::pow(b, 2.0 - gamma) - std::pow(a, 2.0 - gamma)) / (2.0 - gamma);
}

// Vose alias table for sampling node ids proportional to weights.
struct Alias {
  std::vector<double> prob;
  std::vector<uint32_t> alias;
  explicit Alias(const std::vector<double>& w) {
    size_t n = w.size();
    prob.resize(n);
    alias.resize(n);
    double sum = 0;
    for (double x : w) sum += x;
    std::vector<double> p(n);
    std::vector<uint32_t> small, large;
    for (size_t i = 0; i < n; i++) {
      p[i] = w[i] * n / sum;
      (p[i] < 1.0 ? small : large).push_back((uint32_t)i);
    }
    while (!small.empty() && !large.empty()) {
      uint32_t s = small.back(); small.pop_back();
      uint32_t l = large.back(); large.pop_back();
      prob[s] = p[s];
      alias[s] = l;
      p[l] = (p[l] + p[s]) - 1.0;
      (p[l] < 1.0 ? small : large).push_back(l);
    }
    for (uint32_t i : large) { prob[i] = 1.0; alias[i] = i; }
    for (uint32_t i : small) { prob[i] = 1.0; alias[i] = i; }
  }
  uint32_t sample(Rng& r) const {
    uint64_t i = r.below(prob.size());
    return r.uniform() < prob[i] ? (uint32_t)i : alias[i];
  }
};

// Fenwick tree over m slot weights (frontier degrees), for degree-proportional pops.
struct Fenwick {
  std::vector<int64_t> t;
  int n;
  explicit Fenwick(int n_) : t(n_ + 1, 0), n(n_) {}
  void add(int i, int64_t d) { for (++i; i <= n; i += i & -i) t[i] += d; }
  int64_t total() const { int64_t s = 0; for (int i = n; i > 0; i -= i & -i) s += t[i]; return s; }
  // smallest slot i with prefix(i) > x  (x in [0, total))
  int find(int64_t x) const {
    int pos = 0;
    int step = 1;
    while (step * 2 <= n) step *= 2;
    for (; step > 0; step >>= 1) {
      if (pos + step <= n && t[pos + step] <= x) { pos += step; x -= t[pos]; }
    }
    return pos;  // 0-based slot
  }
};

}  // namespace

extern "C" {

// ---------------------------------------------------------------------------------------
// Parent graph: Chung-Lu with i.i.d. Pareto(gamma) weights on [w_min, w_max], w_min solved
// so that mean(w) = mean_deg; endpoint pairs drawn proportional to w; self loops and
// duplicates dropped; topped up until nnz/n >= 0.98*mean_deg.
// Two-call protocol: gsgen_parent_build returns an opaque handle; query sizes, then copy.
// ---------------------------------------------------------------------------------------
struct gsgen_graph {
  int64_t n;
  std::vector<int64_t> indptr;
  std::vector<int32_t> indices;
};

void* gsgen_parent_build(int64_t n, double mean_deg, double gamma, double w_max, uint64_t seed) {
  if (n <= 1 || mean_deg <= 0 || gamma <= 1.0) return nullptr;
  Rng rng(seed);
  if (w_max <= 0) w_max = std::sqrt((double)n * mean_deg);
  // solve w_min by bisection: pareto_mean increasing in w_min
  double lo = 1e-6, hi = std::min(w_max, mean_deg) * (1 - 1e-12);
  for (int it = 0; it < 200; it++) {
    double mid = 0.5 * (lo + hi);
    if (pareto_mean(mid, w_max, gamma) < mean_deg) lo = mid; else hi = mid;
  }
  double w_min = 0.5 * (lo + hi);
  double al = gamma - 1.0;
  double A = std::pow(w_min, -al), B = std::pow(w_max, -al);
  std::vector<double> w(n);
  for (int64_t i = 0; i < n; i++) {
    double u = rng.uniform();
    w[i] = std::pow(A - u * (A - B), -1.0 / al);
  }
  Alias alias(w);

  // undirected pair keys (u<v) -> u*n+v, deduplicated
  std::vector<uint64_t> keys;
  const double target = 0.98 * mean_deg;
  int64_t want = (int64_t)std::ceil(n * mean_deg / 2.0);
  keys.reserve((size_t)(want * 1.1));
  for (int round = 0; round < 64; round++) {
    for (int64_t e = 0; e < want; e++) {
      uint32_t a = alias.sample(rng), b = alias.sample(rng);
      if (a == b) continue;
      if (a > b) std::swap(a, b);
      keys.push_back((uint64_t)a * (uint64_t)n + b);
    }
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    double realized = 2.0 * keys.size() / (double)n;
    if (realized >= target) break;
    want = (int64_t)std::ceil((target - realized) * n / 2.0 * 1.25) + 16;
  }
  auto* g = new gsgen_graph;
  g->n = n;
  g->indptr.assign(n + 1, 0);
  for (uint64_t k : keys) {
    g->indptr[k / n + 1]++;
    g->indptr[k % n + 1]++;
  }
  for (int64_t i = 0; i < n; i++) g->indptr[i + 1] += g->indptr[i];
  g->indices.resize(g->indptr[n]);
  std::vector<int64_t> cur(g->indptr.begin(), g->indptr.end() - 1);
  // keys ascending by (u,v): row x first receives all w<x (ascending), then v>x (ascending)
  for (uint64_t k : keys) {
    int64_t u = k / n, v = k % n;
    g->indices[cur[u]++] = (int32_t)v;
    g->indices[cur[v]++] = (int32_t)u;
  }
  return g;
}

void gsgen_graph_free(void* h) { delete static_cast<gsgen_graph*>(h); }
int64_t gsgen_graph_n(void* h) { return static_cast<gsgen_graph*>(h)->n; }
int64_t gsgen_graph_nnz(void* h) { return static_cast<gsgen_graph*>(h)->indptr.back(); }
void gsgen_graph_copy(void* h, int64_t* indptr, int32_t* indices) {
  auto* g = static_cast<gsgen_graph*>(h);
  std::memcpy(indptr, g->indptr.data(), g->indptr.size() * sizeof(int64_t));
  std::memcpy(indices, g->indices.data(), g->indices.size() * sizeof(int32_t));
}

// Wrap caller-provided CSR arrays (copied) as a graph handle, e.g. a hand-built test graph.
void* gsgen_graph_from_csr(int64_t n, const int64_t* indptr, const int32_t* indices) {
  auto* g = new gsgen_graph;
  g->n = n;
  g->indptr.assign(indptr, indptr + n + 1);
  g->indices.assign(indices, indices + indptr[n]);
  return g;
}

// ---------------------------------------------------------------------------------------
// Frontier sampling (Alg. 2) under SURVEY reading R9:
//   FS_0: m distinct nodes drawn uniformly from the non-isolated nodes; V_s <- FS_0.
//   repeat until |V_s| = n_target: pop slot u with prob deg(u)/sum_FS deg (Alg. 2 line 4),
//   pick u' uniformly among N(u) (line 5), FS[slot] <- u' (line 6), V_s <- V_s U {u'}
//   (Alg. 3 line 500 adds the new frontier node).
// Then clip |V_s| down to a multiple of `clip` by dropping uniformly random nodes (§7.2,
// PAPER.md:947-950), and induce (ascending local ids). Returns a subgraph handle whose
// `nodes` (parent ids, ascending) are available via gsgen_subgraph_nodes.
// ---------------------------------------------------------------------------------------
struct gsgen_subgraph {
  gsgen_graph g;
  std::vector<int64_t> nodes;
};

void* gsgen_frontier_sample(void* parent, int64_t n_target, int64_t m, int64_t clip, uint64_t seed) {
  auto* P = static_cast<gsgen_graph*>(parent);
  const int64_t N = P->n;
  Rng rng(seed);
  std::vector<int64_t> nonisolated;
  nonisolated.reserve(N);
  for (int64_t i = 0; i < N; i++)
    if (P->indptr[i + 1] > P->indptr[i]) nonisolated.push_back(i);
  if ((int64_t)nonisolated.size() < m || m <= 0 || n_target < m) return nullptr;
  if (n_target > (int64_t)nonisolated.size()) return nullptr;
  // partial Fisher-Yates for m distinct
  for (int64_t i = 0; i < m; i++) {
    int64_t j = i + (int64_t)rng.below(nonisolated.size() - i);
    std::swap(nonisolated[i], nonisolated[j]);
  }
  std::vector<uint8_t> in_vs(N, 0);
  std::vector<int64_t> vs;
  vs.reserve(n_target);
  std::vector<int64_t> fs(m);
  Fenwick fw((int)m);
  for (int64_t i = 0; i < m; i++) {
    int64_t v = nonisolated[i];
    fs[i] = v;
    in_vs[v] = 1;
    vs.push_back(v);
    fw.add((int)i, P->indptr[v + 1] - P->indptr[v]);
  }
  int64_t max_iter = 1000 * n_target + 1000000;
  for (int64_t it = 0; (int64_t)vs.size() < n_target && it < max_iter; it++) {
    int64_t tot = fw.total();
    int slot = fw.find((int64_t)rng.below((uint64_t)tot));
    int64_t u = fs[slot];
    int64_t du = P->indptr[u + 1] - P->indptr[u];
    int64_t up = P->indices[P->indptr[u] + (int64_t)rng.below((uint64_t)du)];
    int64_t dup = P->indptr[up + 1] - P->indptr[up];
    fs[slot] = up;
    fw.add(slot, dup - du);
    if (!in_vs[up]) { in_vs[up] = 1; vs.push_back(up); }
  }
  if ((int64_t)vs.size() < n_target) return nullptr;
  // clipping to a multiple of `clip` by random drops
  if (clip > 1) {
    int64_t keep = (int64_t)vs.size() / clip * clip;
    while ((int64_t)vs.size() > keep) {
      int64_t j = (int64_t)rng.below(vs.size());
      in_vs[vs[j]] = 0;
      vs[j] = vs.back();
      vs.pop_back();
    }
  }
  std::sort(vs.begin(), vs.end());
  std::vector<int32_t> local(N, -1);
  for (size_t i = 0; i < vs.size(); i++) local[vs[i]] = (int32_t)i;
  auto* s = new gsgen_subgraph;
  s->nodes = vs;
  const int64_t n = vs.size();
  s->g.n = n;
  s->g.indptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; i++) {
    int64_t v = vs[i], c = 0;
    for (int64_t k = P->indptr[v]; k < P->indptr[v + 1]; k++) c += local[P->indices[k]] >= 0;
    s->g.indptr[i + 1] = s->g.indptr[i] + c;
  }
  s->g.indices.resize(s->g.indptr[n]);
  for (int64_t i = 0; i < n; i++) {
    int64_t v = vs[i], o = s->g.indptr[i];
    for (int64_t k = P->indptr[v]; k < P->indptr[v + 1]; k++) {
      int32_t l = local[P->indices[k]];
      if (l >= 0) s->g.indices[o++] = l;  // parent lists ascending + monotone map => ascending
    }
  }
  return s;
}

void gsgen_subgraph_free(void* h) { delete static_cast<gsgen_subgraph*>(h); }
int64_t gsgen_subgraph_n(void* h) { return static_cast<gsgen_subgraph*>(h)->g.n; }
int64_t gsgen_subgraph_nnz(void* h) { return static_cast<gsgen_subgraph*>(h)->g.indptr.back(); }
void gsgen_subgraph_copy(void* h, int64_t* indptr, int32_t* indices, int64_t* nodes) {
  auto* s = static_cast<gsgen_subgraph*>(h);
  std::memcpy(indptr, s->g.indptr.data(), s->g.indptr.size() * sizeof(int64_t));
  std::memcpy(indices, s->g.indices.data(), s->g.indices.size() * sizeof(int32_t));
  if (nodes) std::memcpy(nodes, s->nodes.data(), s->nodes.size() * sizeof(int64_t));
}

// Induce the subgraph of `parent` on an explicit ascending node list (used by tests to
// check induction against a brute-force double loop).
void* gsgen_induce(void* parent, int64_t n, const int64_t* nodes) {
  auto* P = static_cast<gsgen_graph*>(parent);
  std::vector<int32_t> local(P->n, -1);
  for (int64_t i = 0; i < n; i++) local[nodes[i]] = (int32_t)i;
  auto* s = new gsgen_subgraph;
  s->nodes.assign(nodes, nodes + n);
  s->g.n = n;
  s->g.indptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; i++) {
    int64_t v = nodes[i], c = 0;
    for (int64_t k = P->indptr[v]; k < P->indptr[v + 1]; k++) c += local[P->indices[k]] >= 0;
    s->g.indptr[i + 1] = s->g.indptr[i] + c;
  }
  s->g.indices.resize(s->g.indptr[n]);
  for (int64_t i = 0; i < n; i++) {
    int64_t v = nodes[i], o = s->g.indptr[i];
    for (int64_t k = P->indptr[v]; k < P->indptr[v + 1]; k++) {
      int32_t l = local[P->indices[k]];
      if (l >= 0) s->g.indices[o++] = l;
    }
  }
  return s;
}

}  // extern "C"
