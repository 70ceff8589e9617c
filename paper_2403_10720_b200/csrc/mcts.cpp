// mcts.cpp -- SURVEY.md §8(a) row a7 / §8(b) dvc_mcts_search: the host side of
// the paper's MCTS (root-parallel mini-trees PAPER:179-186):
// UCB1 selection over the root's children, one GPU rollout batch per
// iteration (dvc_rollout_batch_ex -> the sm_100a kernels), backpropagation of
// the integer counts, and the move choice.  Every playout runs in
// the kernels; this file only keeps the tree.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "dvc_internal.h"

extern "C" int dvc_mcts_search(const dvc_state *s, const dvc_search_params *p, dvc_action_stat *table,
                               int32_t cap, int32_t *n_out, uint32_t *best_code);

extern "C" int dvc_mcts_search(const dvc_state *s, const dvc_search_params *p, dvc_action_stat *table,
                               int32_t cap, int32_t *n_out, uint32_t *best_code) {
  using namespace dvc;
  if (!s || !p || !n_out) return set_error(DVC_E_CONFIG, "null argument");
  const State *st = reinterpret_cast<const State *>(s);
  if (st->magic != kMagic) return set_error(DVC_E_CONFIG, "state was not produced by dvc_state_encode");
  if (!p->flat) return set_error(DVC_E_CONFIG, "flat = 0 (depth-capped tree) is not built yet");
  if (p->expansions < 1 || p->sims_per_child < 1 || !(p->c >= 0.0))
    return set_error(DVC_E_CONFIG, "need expansions >= 1, sims_per_child >= 1, c >= 0");
  int32_t A = 0;
  legal_actions(*st, nullptr, 0, &A);
  *n_out = A;
  if (!table || cap < A) return set_error(DVC_E_CAPACITY, "table capacity below the number of root actions");
  std::vector<uint32_t> codes((size_t)A);
  legal_actions(*st, codes.data(), A, &A);
  std::vector<uint64_t> visits((size_t)A, 0), wins((size_t)A, 0);
  std::vector<uint64_t> hist((size_t)st->P);
  uint64_t N = 0;
  const uint64_t n = p->sims_per_child;
  int it = 0;
  {
    // Expansion of the root: while children are unvisited, UCB1 selects them
    // one per iteration in ascending code order (+inf ties -> smallest code),
    // each with sims [0, n).  Those iterations are independent, so they run
    // as ONE leaf-parallel GPU batch -- the same playouts, the same counts.
    const int k = p->expansions < A ? p->expansions : A;
    std::vector<int> order((size_t)A);
    for (int a = 0; a < A; ++a) order[a] = a;
    std::sort(order.begin(), order.end(), [&](int x, int y) { return codes[x] < codes[y]; });
    std::vector<uint32_t> first((size_t)k);
    for (int i = 0; i < k; ++i) first[i] = codes[order[i]];
    std::vector<uint64_t> h((size_t)k * st->P);
    int rc = dvc_rollout_batch_ex(s, first.data(), k, p->seed, 0u, 0, n, h.data(), nullptr, p->device);
    if (rc) return rc;
    for (int i = 0; i < k; ++i) {
      visits[order[i]] = n;
      wins[order[i]] = h[(size_t)i * st->P + st->viewer];
      N += n;
    }
    it = k;
  }
  for (; it < p->expansions; ++it) {
    // selection: UCB1, unvisited children first, ties -> smallest code
    int best = -1;
    double best_v = 0.0;
    for (int a = 0; a < A; ++a) {
      double v;
      if (visits[a] == 0) {
        v = INFINITY;
      } else {
        v = (double)wins[a] / (double)visits[a] + p->c * std::sqrt(std::log((double)N) / (double)visits[a]);
      }
      if (best < 0 || v > best_v || (v == best_v && codes[a] < codes[best])) { best = a; best_v = v; }
    }
    if (visits[best] + n > (1ull << 32))
      return set_error(DVC_E_CONFIG, "a child's sim index range would pass 2^32");
    // simulation on the GPU: sims [visits, visits + n) of the chosen child
    int rc = dvc_rollout_batch_ex(s, &codes[best], 1, p->seed, 0u, visits[best], visits[best] + n, hist.data(),
                                  nullptr, p->device);
    if (rc) return rc;
    // backpropagation
    visits[best] += n;
    wins[best] += hist[st->viewer];
    N += n;
  }
  int bi = 0;
  for (int a = 1; a < A; ++a) {
    if (visits[a] > visits[bi] || (visits[a] == visits[bi] &&
        (wins[a] > wins[bi] || (wins[a] == wins[bi] && codes[a] < codes[bi])))) bi = a;
  }
  for (int a = 0; a < A; ++a) {
    table[a].code = codes[a]; table[a]._pad = 0; table[a].visits = visits[a]; table[a].wins = wins[a];
  }
  if (best_code) *best_code = codes[bi];
  return DVC_OK;
}
