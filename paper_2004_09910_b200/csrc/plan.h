// Pure host planning (no CUDA): balancer, split, schedule emitter.
#pragma once
#include <cstdint>
#include <utility>
#include <vector>

namespace tgp {

enum TaskKind : int32_t { K_F = 0, K_RECOMPUTE = 1, K_B = 2, K_COPY_F = 3, K_COPY_B = 4, K_SKIP_F = 5, K_SKIP_B = 6, K_W = 7 };

struct Rec {
  int32_t phase, clock, kind, i, j, src, dst, route;  // i, j, src, dst 1-based
};

bool balance_minmax(const double* cost, int L, int n, int* out);
bool split_sizes(int B, int m, int* sizes);
bool checkpointed(int i, int m, int mode);  // i 1-based; mode = tgp_checkpoint
std::vector<Rec> emit_schedule(int m, int n, int mode, const std::vector<std::pair<int, int>>& routes, bool relay = false);
void skip_fwd_records(std::vector<Rec>& out, int phase, int k, int i, int d, const std::vector<std::pair<int, int>>& routes,
                      bool relay);
void skip_bwd_records(std::vector<Rec>& out, int phase, int k, int i, int s, const std::vector<std::pair<int, int>>& routes,
                      bool relay);
// Table 1 ablation: backward records in a seeded random topological order (no Fork/Join edges)
std::vector<Rec> unordered_backward(int m, int n, int mode, const std::vector<std::pair<int, int>>& routes, bool relay,
                                    uint64_t seed);

}  // namespace tgp
