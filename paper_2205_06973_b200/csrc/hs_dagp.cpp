// dagP merge phase on the host (partition_dagp's greedy pair contraction,
// reference partition.py:396-478; Python restatement
// paper_2205_06973_b200/partition.py:_merge_groups).
//
// Same algorithm, same output: candidate pairs (u < v) are popped in the
// order of the key (-shared qubits, -union size, u, v); a popped key is
// recomputed and requeued if stale; a valid pair merges v into u when the
// contraction keeps the part graph acyclic (no path u -> .. -> v or v -> .. -> u
// other than a direct edge), after which every pairing of u is pushed again.
// A min-heap pops equal keys interchangeably, so the merge sequence does not
// depend on the heap's internals. Qubit sets are 64-bit masks (circuits of at
// most 64 qubits; the Python path handles wider ones).
#include <algorithm>
#include <cstdint>
#include <functional>
#include <queue>
#include <vector>

#include "hs_common.h"

namespace {

struct PartGraph {
  std::vector<std::vector<int>> out, inn;
  std::vector<int> pot;   // topological potential: pot[a] < pot[b] on every edge a -> b
  std::vector<int> mark;  // visit stamps for searches
  int stamp = 0;
  // transitive closure (graphs up to kClosureMax groups): bit y of row x =
  // y reachable from x by a path of >= 1 edge; queries become bit tests
  static constexpr int kClosureMax = 16384;
  int W = 0;
  std::vector<uint64_t> R;
  bool has(int x, int y) const { return R[size_t(x) * W + (y >> 6)] >> (y & 63) & 1; }

  void build_closure(int G) {
    W = (G + 63) / 64;
    R.assign(size_t(G) * W, 0);
    std::vector<int> order(G);
    for (int i = 0; i < G; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return pot[a] > pot[b]; });  // sinks first
    for (int x : order) {
      uint64_t* rx = &R[size_t(x) * W];
      for (int y : out[x]) {
        rx[y >> 6] |= 1ull << (y & 63);
        const uint64_t* ry = &R[size_t(y) * W];
        for (int w = 0; w < W; ++w) rx[w] |= ry[w];
      }
    }
  }
  // after contracting v into u: u reaches what either reached; whoever
  // reached u or v reaches u and all of it; v is gone
  void merge_closure(int u, int v, const std::vector<char>& alive) {
    uint64_t* ru = &R[size_t(u) * W];
    const uint64_t* rv = &R[size_t(v) * W];
    for (int w = 0; w < W; ++w) ru[w] |= rv[w];
    ru[u >> 6] &= ~(1ull << (u & 63));
    ru[v >> 6] &= ~(1ull << (v & 63));
    const int G = (int)alive.size();
    for (int x = 0; x < G; ++x) {
      if (!alive[x] || x == u) continue;
      uint64_t* rx = &R[size_t(x) * W];
      const bool bu = rx[u >> 6] >> (u & 63) & 1, bv = rx[v >> 6] >> (v & 63) & 1;
      if (!bu && !bv) continue;
      for (int w = 0; w < W; ++w) rx[w] |= ru[w];
      rx[u >> 6] |= 1ull << (u & 63);
      rx[v >> 6] &= ~(1ull << (v & 63));
    }
  }
  bool reaches_indirectly_closure(int src, int dst) const {
    for (int m : out[src])
      if (m != dst && has(m, dst)) return true;
    return false;
  }

  static void add_unique(std::vector<int>& v, int x) {
    if (std::find(v.begin(), v.end(), x) == v.end()) v.push_back(x);
  }
  static void erase_value(std::vector<int>& v, int x) {
    auto it = std::find(v.begin(), v.end(), x);
    if (it != v.end()) { *it = v.back(); v.pop_back(); }
  }

  // is there a path src -> ... -> dst other than the edge src -> dst?
  bool reaches_indirectly(int src, int dst) {
    const int limit = pot[dst];
    ++stamp;
    std::vector<int> stack;
    for (int m : out[src])
      if (m != dst && pot[m] < limit && mark[m] != stamp) { mark[m] = stamp; stack.push_back(m); }
    while (!stack.empty()) {
      const int x = stack.back();
      stack.pop_back();
      for (int y : out[x]) {
        if (y == dst) return true;
        if (mark[y] != stamp && pot[y] < limit) { mark[y] = stamp; stack.push_back(y); }
      }
    }
    return false;
  }

  void contract(int u, int v) {  // merge v into u (acyclic by the caller's check)
    for (int b : out[v]) {
      erase_value(inn[b], v);
      if (b != u) { add_unique(out[u], b); add_unique(inn[b], u); }
    }
    for (int a : inn[v]) {
      erase_value(out[a], v);
      if (a != u) { add_unique(inn[u], a); add_unique(out[a], u); }
    }
    out[v].clear();
    inn[v].clear();
    erase_value(out[u], u);
    erase_value(inn[u], u);
    int p = std::max(pot[v], pot[u]);
    for (int a : inn[u]) p = std::max(p, pot[a] + 1);
    pot[u] = p;
    std::vector<int> stack{u};
    while (!stack.empty()) {
      const int x = stack.back();
      stack.pop_back();
      for (int b : out[x])
        if (pot[b] <= pot[x]) { pot[b] = pot[x] + 1; stack.push_back(b); }
    }
  }
};

}  // namespace

extern "C" int hs_dagp_merge(int num_groups, const uint64_t* qmask, int num_edges, const int32_t* edge_src,
                             const int32_t* edge_dst, int limit, int32_t* merged_into) {
  if (num_groups < 0 || (num_groups && (!qmask || !merged_into)) || num_edges < 0 ||
      (num_edges && (!edge_src || !edge_dst)) || num_groups >= (1 << 20))
    return HS_ERR_INVALID;
  const int G = num_groups;
  PartGraph g;
  g.out.assign(G, {});
  g.inn.assign(G, {});
  g.mark.assign(G, 0);
  for (int e = 0; e < num_edges; ++e) {
    const int a = edge_src[e], b = edge_dst[e];
    if (a < 0 || a >= G || b < 0 || b >= G) return HS_ERR_INVALID;
    if (a == b) continue;
    PartGraph::add_unique(g.out[a], b);
    PartGraph::add_unique(g.inn[b], a);
  }
  {  // longest-path levels as the initial potential
    std::vector<int> indeg(G), ready;
    g.pot.assign(G, 0);
    for (int i = 0; i < G; ++i) indeg[i] = (int)g.inn[i].size();
    for (int i = 0; i < G; ++i)
      if (!indeg[i]) ready.push_back(i);
    while (!ready.empty()) {
      const int p = ready.back();
      ready.pop_back();
      for (int b : g.out[p]) {
        g.pot[b] = std::max(g.pot[b], g.pot[p] + 1);
        if (--indeg[b] == 0) ready.push_back(b);
      }
    }
  }
  const bool closure = G <= PartGraph::kClosureMax;
  if (closure) g.build_closure(G);
  std::vector<uint64_t> q(qmask, qmask + G);
  std::vector<char> alive(G, 1);
  for (int i = 0; i < G; ++i) merged_into[i] = i;
  // key (-shared, -union, u, v) ascending, packed: 64 - shared, 64 - union, u, v
  auto key = [&](int u, int v, uint64_t& k) -> bool {
    const int cu = __builtin_popcountll(q[u]), cv = __builtin_popcountll(q[v]);
    const int uni = __builtin_popcountll(q[u] | q[v]);
    if (uni > limit) return false;
    const int shared = cu + cv - uni;
    k = (uint64_t(64 - shared) << 54) | (uint64_t(64 - uni) << 47) | (uint64_t(u) << 20) | uint64_t(v);
    return true;
  };
  // Pairs sharing no qubit have keys after every sharing pair, so they are
  // only needed once the heap's minimum gets there: insert them then (for the
  // groups still alive, with current keys). Until that moment the reference
  // could only pop sharing pairs, so the pop sequence is the same, and the
  // heap starts with the sharing pairs only (found per qubit).
  const uint64_t kShared0 = uint64_t(64) << 54;  // keys >= this share no qubit
  std::vector<uint64_t> init;
  {
    std::vector<std::vector<int>> by_qubit(64);
    for (int u = 0; u < G; ++u)
      for (int b = 0; b < 64; ++b)
        if (q[u] >> b & 1) by_qubit[b].push_back(u);
    for (auto& lst : by_qubit)
      for (size_t i = 0; i < lst.size(); ++i)
        for (size_t j = i + 1; j < lst.size(); ++j) {
          uint64_t k;
          if (key(lst[i], lst[j], k)) init.push_back(k);
        }
    std::sort(init.begin(), init.end());
    init.erase(std::unique(init.begin(), init.end()), init.end());
  }
  std::priority_queue<uint64_t, std::vector<uint64_t>, std::greater<uint64_t>> heap(std::greater<uint64_t>(),
                                                                                    std::move(init));
  bool disjoint_in = false;
  for (;;) {
    if (!disjoint_in && (heap.empty() || heap.top() >= kShared0)) {
      disjoint_in = true;
      std::vector<int> live;
      for (int i = 0; i < G; ++i)
        if (alive[i]) live.push_back(i);
      for (size_t i = 0; i < live.size(); ++i)
        for (size_t j = i + 1; j < live.size(); ++j) {
          if (q[live[i]] & q[live[j]]) continue;
          uint64_t k;
          if (key(live[i], live[j], k)) heap.push(k);
        }
    }
    if (heap.empty()) break;
    const uint64_t entry = heap.top();
    heap.pop();
    const int u = int((entry >> 20) & 0xFFFFF), v = int(entry & 0xFFFFF);
    if (!alive[u] || !alive[v]) continue;
    uint64_t k;
    if (!key(u, v, k)) continue;
    if (k != entry) { heap.push(k); continue; }
    if (closure ? (g.reaches_indirectly_closure(u, v) || g.reaches_indirectly_closure(v, u))
                : (g.reaches_indirectly(u, v) || g.reaches_indirectly(v, u)))
      continue;
    alive[v] = 0;
    q[u] |= q[v];
    g.contract(u, v);
    if (closure) g.merge_closure(u, v, alive);
    for (int i = 0; i < G; ++i) {
      if (!alive[i] || i == u) continue;
      if (key(std::min(u, i), std::max(u, i), k)) heap.push(k);
    }
    if (merged_into) merged_into[v] = u;
  }
  // resolve chains: a group merged into a group that merged later
  std::vector<int32_t> into(G);
  for (int i = 0; i < G; ++i) into[i] = alive[i] ? i : merged_into[i];
  for (int i = 0; i < G; ++i) {
    int r = i;
    while (!alive[r]) r = into[r];
    merged_into[i] = r;
  }
  return HS_OK;
}
