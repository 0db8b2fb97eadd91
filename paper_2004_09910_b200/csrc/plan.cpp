// Pure host planning: partition balancer, micro-batch split, clock-cycle schedule emitter.
// No CUDA here; these entry points work on a machine without a GPU.
#include "plan.h"

#include <algorithm>
#include <limits>

namespace tgp {

// Min-max contiguous block partition by DP over prefix sums (reading Z8).
// best[p][e] = min over splits of layers [e, L) into p blocks of the largest block sum.
// Reconstruction takes, block by block, the shortest block that still attains the optimum,
// i.e. the lexicographically smallest boundary vector.
bool balance_minmax(const double* cost, int L, int n, int* out) {
  if (n < 1 || n > L) return false;
  std::vector<double> pre(L + 1, 0.0);
  for (int i = 0; i < L; ++i) pre[i + 1] = pre[i] + cost[i];
  const double INF = std::numeric_limits<double>::infinity();
  std::vector<std::vector<double>> best(n + 1, std::vector<double>(L + 1, INF));
  best[0][L] = 0.0;
  for (int p = 1; p <= n; ++p) {
    for (int e = L - p; e >= 0; --e) {
      double v = INF;
      for (int end = e + 1; end <= L - p + 1; ++end) v = std::min(v, std::max(pre[end] - pre[e], best[p - 1][end]));
      best[p][e] = v;
    }
  }
  const double opt = best[n][0];
  int e = 0, q = 0;
  for (int p = n; p >= 1; --p) {
    for (int end = e + 1; end <= L - p + 1; ++end) {
      if (std::max(pre[end] - pre[e], best[p - 1][end]) <= opt) {
        out[q++] = end - e;
        e = end;
        break;
      }
    }
  }
  return q == n && e == L;
}

bool split_sizes(int B, int m, int* sizes) {
  if (m < 1 || m > B) return false;
  const int q = B / m, r = B % m;
  for (int i = 0; i < m; ++i) sizes[i] = q + (i < r ? 1 : 0);
  return true;
}

bool checkpointed(int i, int m, int mode) {
  // i is 1-based.  ALWAYS: every micro-batch; EXCEPT_LAST: i < m; NEVER: none.
  if (mode == 0) return true;
  if (mode == 1) return i < m;
  return false;
}

// Alg. 1: forward clock k = 1..m+n-1 holds {(i,j): i+j-1 = k}; its copies are issued
// first, then its computes.  The backward mirrors it (readings Z2, Z3, Z5, Z6).
// relay (Table 1 "no portals" ablation): a skip tensor is tuple-threaded
// through every partition between its stash and its pop -- one hop (j-1 -> j) per partition it
// enters, travelling with the activation -- instead of one direct portal copy.
std::vector<Rec> emit_schedule(int m, int n, int mode, const std::vector<std::pair<int, int>>& routes, bool relay) {
  std::vector<Rec> out;
  auto clock = [&](int k) {
    std::vector<std::pair<int, int>> t;
    for (int j = std::max(1, k - m + 1); j <= std::min(k, n); ++j) t.emplace_back(k - j + 1, j);
    return t;
  };
  const int T = m + n - 1;
  for (int k = 1; k <= T; ++k) {
    auto t = clock(k);
    for (auto [i, j] : t)
      if (j > 1) out.push_back({0, k, K_COPY_F, i, j, j - 1, j, -1});
    for (auto [i, d] : t) skip_fwd_records(out, 0, k, i, d, routes, relay);
    for (auto [i, j] : t) out.push_back({0, k, K_F, i, j, j, j, -1});
  }
  for (int kp = 1; kp <= T; ++kp) {
    auto t = clock(m + n - kp);
    std::reverse(t.begin(), t.end());
    for (auto [i, j] : t)
      if (j < n) out.push_back({1, kp, K_COPY_B, i, j, j + 1, j, -1});
    for (auto [i, s] : t) skip_bwd_records(out, 1, kp, i, s, routes, relay);
    for (auto [i, j] : t) {
      if (checkpointed(i, m, mode)) out.push_back({1, kp, K_RECOMPUTE, i, j, j, j, -1});
      out.push_back({1, kp, K_B, i, j, j, j, -1});
    }
  }
  for (int j = 1; j <= n; ++j) out.push_back({2, 0, K_W, 0, j, j, j, -1});
  return out;
}

// the skip messages partition d receives before F_{i,d}
void skip_fwd_records(std::vector<Rec>& out, int phase, int k, int i, int d, const std::vector<std::pair<int, int>>& routes,
                      bool relay) {
  for (int r = 0; r < (int)routes.size(); ++r) {
    const int src = routes[r].first, dst = routes[r].second;
    if (src == dst) continue;
    if (!relay && dst == d) out.push_back({phase, k, K_SKIP_F, i, d, src, d, r});
    if (relay && src < d && d <= dst) out.push_back({phase, k, K_SKIP_F, i, d, d - 1, d, r});
  }
}

// the skip-gradient messages partition s receives before B_{i,s}
void skip_bwd_records(std::vector<Rec>& out, int phase, int k, int i, int s, const std::vector<std::pair<int, int>>& routes,
                      bool relay) {
  for (int r = 0; r < (int)routes.size(); ++r) {
    const int src = routes[r].first, dst = routes[r].second;
    if (src == dst) continue;
    if (!relay && src == s) out.push_back({phase, k, K_SKIP_B, i, s, dst, s, r});
    if (relay && src <= s && s < dst) out.push_back({phase, k, K_SKIP_B, i, s, s + 1, s, r});
  }
}

// Table 1 row 1 ("no Fork/Join dependency", P:268 and Fig. 7(a)): without the explicit edge
// B_{i+1,j} -> B_{i,j} the autograd engine issues the backward tasks in an order of its own.  We
// emulate it by a seeded random topological order of the backward task graph: at every step one
// ready task (i, j) is drawn uniformly -- B_{i,n} is ready at once, B_{i,j} once B_{i,j+1} was
// issued -- and issued with its incoming messages, its recompute and itself.  Every wait then
// refers to earlier-issued work, so the order cannot deadlock even with copies on the compute
// streams.  The clock field holds the issue step (1-based).
std::vector<Rec> unordered_backward(int m, int n, int mode, const std::vector<std::pair<int, int>>& routes, bool relay,
                                    uint64_t seed) {
  std::vector<Rec> out;
  std::vector<int> next_j(m + 1, n);  // per micro-batch: the partition of its next backward task
  std::vector<int> ready;             // micro-batches with a task left
  for (int i = 1; i <= m; ++i) ready.push_back(i);
  uint64_t x = seed * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
  auto rnd = [&]() {  // splitmix64
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  int step = 0;
  while (!ready.empty()) {
    const int q = (int)(rnd() % ready.size());
    const int i = ready[q], j = next_j[i];
    ++step;
    if (j < n) out.push_back({1, step, K_COPY_B, i, j, j + 1, j, -1});
    skip_bwd_records(out, 1, step, i, j, routes, relay);
    if (checkpointed(i, m, mode)) out.push_back({1, step, K_RECOMPUTE, i, j, j, j, -1});
    out.push_back({1, step, K_B, i, j, j, j, -1});
    if (--next_j[i] < 1) {
      ready[q] = ready.back();
      ready.pop_back();
    }
  }
  return out;
}

}  // namespace tgp
