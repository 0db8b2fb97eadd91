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
std::vector<Rec> emit_schedule(int m, int n, int mode, const std::vector<std::pair<int, int>>& routes) {
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
    for (auto [i, d] : t)
      for (int r = 0; r < (int)routes.size(); ++r)
        if (routes[r].second == d && routes[r].first != d) out.push_back({0, k, K_SKIP_F, i, d, routes[r].first, d, r});
    for (auto [i, j] : t) out.push_back({0, k, K_F, i, j, j, j, -1});
  }
  for (int kp = 1; kp <= T; ++kp) {
    auto t = clock(m + n - kp);
    std::reverse(t.begin(), t.end());
    for (auto [i, j] : t)
      if (j < n) out.push_back({1, kp, K_COPY_B, i, j, j + 1, j, -1});
    for (auto [i, s] : t)
      for (int r = 0; r < (int)routes.size(); ++r)
        if (routes[r].first == s && routes[r].second != s) out.push_back({1, kp, K_SKIP_B, i, s, routes[r].second, s, r});
    for (auto [i, j] : t) {
      if (checkpointed(i, m, mode)) out.push_back({1, kp, K_RECOMPUTE, i, j, j, j, -1});
      out.push_back({1, kp, K_B, i, j, j, j, -1});
    }
  }
  for (int j = 1; j <= n; ++j) out.push_back({2, 0, K_W, 0, j, j, j, -1});
  return out;
}

}  // namespace tgp
