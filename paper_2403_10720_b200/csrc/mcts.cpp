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

namespace {

using namespace dvc;

// ---------------------------------------------------------------------------
// Depth-capped tree over the viewer's own guesses (PAPER:143-170:
// nodes keyed by a guess (position, number), depth = the sequence of guesses,
// no expansion beyond a fixed depth).  Opponents' decisions are chance events
// drawn by the playout policy.  Each expansion evaluates all children of the
// selected leaf in ONE GPU batch (leaf parallelism); playouts whose forced
// path is impossible in their determinization are void and not counted.
struct Node {
  uint32_t code;
  int32_t depth, parent;
  uint64_t visits = 0, wins = 0, tried = 0;
  bool expanded = false;
  std::vector<int32_t> children;
};

// Where a search's rollout batches run: this process's GPU (the default), or
// a caller callback that shards the sim range over ranks and sums the counts
// (dvc_mcts_search_cb; dist.mcts_search).  The UCT arithmetic stays here.
struct Batcher {
  dvc_batch_fn fn = nullptr;
  void *ctx = nullptr;
  int flat(const dvc_state *s, const uint32_t *codes, int32_t n, uint64_t seed, uint32_t node, uint64_t s0,
           uint64_t s1, uint32_t flags, uint64_t *hist, int32_t device) const {
    if (!fn) return dvc_rollout_batch_flags_ex(s, codes, n, seed, node, s0, s1, flags, hist, device);
    std::fill(hist, hist + (size_t)n * reinterpret_cast<const dvc::State *>(s)->P, 0ull);
    const int rc = fn(ctx, nullptr, 0, codes, n, seed, node, s0, s1, flags, hist, nullptr);
    return rc ? dvc::set_error(rc < 0 ? rc : DVC_E_CONFIG, "batch callback failed") : DVC_OK;
  }
  int path(const dvc_state *s, const uint32_t *path, int32_t path_len, const uint32_t *codes, int32_t n,
           uint64_t seed, uint32_t node, uint64_t s0, uint64_t s1, uint64_t *hist, uint64_t *voids,
           int32_t device) const {
    if (!fn) return dvc_rollout_path_ex(s, path, path_len, codes, n, seed, node, s0, s1, hist, voids, device);
    std::fill(hist, hist + (size_t)n * reinterpret_cast<const dvc::State *>(s)->P, 0ull);
    std::fill(voids, voids + n, 0ull);
    const int rc = fn(ctx, path, path_len, codes, n, seed, node, s0, s1, 0u, hist, voids);
    return rc ? dvc::set_error(rc < 0 ? rc : DVC_E_CONFIG, "batch callback failed") : DVC_OK;
  }
};

}  // namespace

namespace dvc {
// ln N by the fixed recipe of DESIGN.md §R8 reading #28 (the oracle's
// ln_series, the device's ln_series_dev): the host, the oracle and the search
// kernels evaluate the same IEEE operations in the same order (this file is
// compiled with -ffp-contract=off), so their UCB1 choices agree bit for bit.
double ln_series(uint64_t N) {
  int e = 0;
  double m = std::frexp((double)N, &e);
  if (m < 0.7071067811865476) {
    m *= 2.0;
    e -= 1;
  }
  const double z = (m - 1.0) / (m + 1.0);
  const double z2 = z * z;
  double p = 1.0 / 27.0;
  for (int k = 12; k >= 0; --k) p = p * z2 + 1.0 / (double)(2 * k + 1);
  return 2.0 * (z * p) + (double)e * 0.6931471805599453;
}
}  // namespace dvc

namespace {

double ucb1(uint64_t w, uint64_t v, uint64_t parent, double c) {
  return (double)w / (double)v + c * std::sqrt(dvc::ln_series(parent) / (double)v);
}

int deep_search(const dvc_state *s, const State *st, const dvc_search_params *p, std::vector<uint32_t> &root_codes,
                std::vector<uint64_t> &rv, std::vector<uint64_t> &rw, const Batcher &B) {
  if (p->max_depth < 1 || p->max_depth > kMaxPath)
    return set_error(DVC_E_CONFIG, "max_depth must be 1..8 for the deep tree");
  const uint64_t n = p->sims_per_child;
  const int P = st->P;
  // children of deeper nodes: the root's guesses, plus STOP under consecutive rules
  std::vector<uint32_t> deep_codes;
  for (uint32_t c : root_codes) if (c != DVC_STOP) deep_codes.push_back(c);
  if (st->consecutive) deep_codes.push_back(DVC_STOP);
  if (!B.fn && search_on_device()) {
    // the same tree, iterations and batches in one cooperative GPU kernel
    rv.assign(root_codes.size(), 0);
    rw.assign(root_codes.size(), 0);
    return deep_search_gpu(s, p, root_codes.data(), (int32_t)root_codes.size(), deep_codes.data(),
                           (int32_t)deep_codes.size(), rv.data(), rw.data());
  }
  std::vector<Node> T;
  T.push_back(Node{0u, 0, -1});
  std::vector<uint64_t> hist, voids;
  for (int it = 0; it < p->expansions; ++it) {
    // ---- selection
    int32_t x = 0;
    while (T[x].expanded) {
      int32_t best = -1;
      double bv = 0.0;
      for (int32_t c : T[x].children) {
        const Node &ch = T[c];
        if (ch.tried > 0 && ch.visits == 0) continue;          // void so far: impossible path
        const double v = ch.tried == 0 ? INFINITY : ucb1(ch.wins, ch.visits, T[x].visits, p->c);
        if (best < 0 || v > bv || (v == bv && ch.code < T[best].code)) { best = c; bv = v; }
      }
      if (best < 0) break;
      x = best;
    }
    // path of codes root -> x
    std::vector<uint32_t> path;
    for (int32_t y = x; y > 0; y = T[y].parent) path.push_back(T[y].code);
    std::reverse(path.begin(), path.end());
    std::vector<int32_t> evaluated;   // nodes whose counts this batch updates
    const bool expand = !T[x].expanded && T[x].depth < p->max_depth && (x == 0 || T[x].visits > 0);
    std::vector<uint32_t> batch;
    std::vector<uint32_t> prefix = path;
    uint32_t node_word;
    if (expand) {
      const std::vector<uint32_t> &cand = (x == 0) ? root_codes : deep_codes;
      for (uint32_t c : cand) {
        T[x].children.push_back((int32_t)T.size());
        T.push_back(Node{c, T[x].depth + 1, x});
        evaluated.push_back((int32_t)T.size() - 1);
        batch.push_back(c);
      }
      T[x].expanded = true;
      node_word = (uint32_t)x;
    } else {
      if (x == 0) break;                                         // nothing left to do
      prefix.pop_back();
      evaluated.push_back(x);
      batch.push_back(T[x].code);
      node_word = (uint32_t)T[x].parent;
    }
    const uint64_t s0 = T[evaluated[0]].tried;
    if (s0 + n > (1ull << 32)) return set_error(DVC_E_CONFIG, "a node's sim index range would pass 2^32");
    hist.assign(batch.size() * (size_t)P, 0);
    voids.assign(batch.size(), 0);
    int rc = B.path(s, prefix.data(), (int32_t)prefix.size(), batch.data(), (int32_t)batch.size(), p->seed,
                    node_word, s0, s0 + n, hist.data(), voids.data(), p->device);
    if (rc) return rc;
    // ---- backpropagation
    uint64_t dv = 0, dw = 0;
    for (size_t i = 0; i < evaluated.size(); ++i) {
      Node &e = T[evaluated[i]];
      e.tried += n;
      e.visits += n - voids[i];
      e.wins += hist[i * P + st->viewer];
      dv += n - voids[i];
      dw += hist[i * P + st->viewer];
    }
    for (int32_t y = T[evaluated[0]].parent; y >= 0; y = T[y].parent) {
      T[y].visits += dv;
      T[y].wins += dw;
    }
  }
  rv.assign(root_codes.size(), 0);
  rw.assign(root_codes.size(), 0);
  for (int32_t c : T[0].children) {
    for (size_t a = 0; a < root_codes.size(); ++a)
      if (root_codes[a] == T[c].code) { rv[a] = T[c].visits; rw[a] = T[c].wins; }
  }
  return DVC_OK;
}

// Move choice (most visits, then most wins, then smallest code) and
// the per-child table.
int finish(const std::vector<uint32_t> &codes, const std::vector<uint64_t> &visits,
           const std::vector<uint64_t> &wins, dvc_action_stat *table, uint32_t *best_code) {
  const int A = (int)codes.size();
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

}  // namespace

namespace {
int mcts_search(const dvc_state *s, const dvc_search_params *p, dvc_action_stat *table, int32_t cap,
                int32_t *n_out, uint32_t *best_code, const Batcher &B) {
  using namespace dvc;
  if (!s || !p || !n_out) return set_error(DVC_E_CONFIG, "null argument");
  const State *st = reinterpret_cast<const State *>(s);
  if (st->magic != kMagic) return set_error(DVC_E_CONFIG, "state was not produced by dvc_state_encode");
  if (p->expansions < 1 || p->sims_per_child < 1 || !(p->c >= 0.0))
    return set_error(DVC_E_CONFIG, "need expansions >= 1, sims_per_child >= 1, c >= 0");
  if (p->flags & ~(uint32_t)(DVC_FLAG_CRN | DVC_FLAG_INFORMED))
    return set_error(DVC_E_CONFIG, "unknown search flag");
  if (p->flags && !p->flat) return set_error(DVC_E_CONFIG, "batch flags need flat = 1 (no path batches)");
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
  if (!p->flat) {
    int rc = deep_search(s, st, p, codes, visits, wins, B);
    if (rc) return rc;
    it = p->expansions;
  } else {
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
    const int iters = p->expansions - k;
    if (iters > 0 && !B.fn && search_on_device() && n * (uint64_t)(iters + 1) <= (1ull << 32)) {
      // The whole search on the GPU (api.cu flat_search_gpu): the same
      // selections and playouts as the host loop below, without a host round
      // trip per iteration.  ln(N) = ln_series((k + it) n), N known in advance.
      std::vector<int32_t> batch_pos((size_t)A, -1);
      for (int i = 0; i < k; ++i) batch_pos[order[i]] = i;
      std::vector<double> lnN((size_t)iters);
      for (int i = 0; i < iters; ++i) lnN[i] = ln_series((uint64_t)(k + i) * n);
      int rc = flat_search_gpu(s, codes.data(), A, first.data(), k, batch_pos.data(), lnN.data(), iters, p,
                               visits.data(), wins.data());
      if (rc) return rc;
      return finish(codes, visits, wins, table, best_code);
    }
    std::vector<uint64_t> h((size_t)k * st->P);
    int rc = B.flat(s, first.data(), k, p->seed, 0u, 0, n, p->flags, h.data(), p->device);
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
        v = ucb1(wins[a], visits[a], N, p->c);
      }
      if (best < 0 || v > best_v || (v == best_v && codes[a] < codes[best])) { best = a; best_v = v; }
    }
    if (visits[best] + n > (1ull << 32))
      return set_error(DVC_E_CONFIG, "a child's sim index range would pass 2^32");
    // simulation on the GPU: sims [visits, visits + n) of the chosen child
    int rc = B.flat(s, &codes[best], 1, p->seed, 0u, visits[best], visits[best] + n, p->flags, hist.data(),
                    p->device);
    if (rc) return rc;
    // backpropagation
    visits[best] += n;
    wins[best] += hist[st->viewer];
    N += n;
  }
  return finish(codes, visits, wins, table, best_code);
}
}  // namespace

extern "C" int dvc_mcts_search(const dvc_state *s, const dvc_search_params *p, dvc_action_stat *table,
                               int32_t cap, int32_t *n_out, uint32_t *best_code) {
  return mcts_search(s, p, table, cap, n_out, best_code, Batcher{});
}

extern "C" int dvc_mcts_search_cb(const dvc_state *s, const dvc_search_params *p, dvc_batch_fn fn, void *ctx,
                                  dvc_action_stat *table, int32_t cap, int32_t *n_out, uint32_t *best_code) {
  if (!fn) return dvc::set_error(DVC_E_CONFIG, "null batch callback");
  Batcher B;
  B.fn = fn;
  B.ctx = ctx;
  return mcts_search(s, p, table, cap, n_out, best_code, B);
}

// ---------------------------------------------------------------------------
// The "md" ablation: the paper's vanilla tree keys a node by
// the guess AND the chosen set of plausible numbers -- fan-out up
// to 11,880 at the root, which is why the paper discards it.  Flat
// (root-only) UCT over children (rho_i, a); every playout of a child plays its
// fixed determinization (dvc_rollout_batch_fixed_ex).  Same UCB1 (ln_series),
// same tie rules and move choice as the flat search above.
extern "C" int dvc_md_search(const dvc_state *s, const dvc_md_params *p, dvc_action_stat *table, int32_t cap,
                             int32_t *n_out, uint32_t *best_code, int32_t *n_det_out) {
  using namespace dvc;
  if (!s || !p || !n_out) return set_error(DVC_E_CONFIG, "null argument");
  const State *st = reinterpret_cast<const State *>(s);
  if (st->magic != kMagic) return set_error(DVC_E_CONFIG, "state was not produced by dvc_state_encode");
  if (p->expansions < 1 || p->sims_per_child < 1 || p->n_det < 1 || p->n_det > 4096 || !(p->c >= 0.0))
    return set_error(DVC_E_CONFIG, "need expansions >= 1, sims_per_child >= 1, 1 <= n_det <= 4096, c >= 0");
  int32_t A = 0;
  legal_actions(*st, nullptr, 0, &A);
  *n_out = A;
  if (!table || cap < A) return set_error(DVC_E_CAPACITY, "table capacity below the number of root actions");
  std::vector<uint32_t> codes((size_t)A);
  legal_actions(*st, codes.data(), A, &A);
  // candidate determinizations
  std::vector<uint64_t> rhos;
  if (st->N <= (uint64_t)p->n_det) {
    for (uint64_t r = 0; r < st->N; ++r) rhos.push_back(r);
  } else {
    const int32_t draws = 64 * p->n_det;
    std::vector<uint64_t> smp((size_t)draws);
    int rc = dvc_sample_determinizations(s, p->seed, 0u, 0u, draws, smp.data());
    if (rc) return rc;
    for (int32_t i = 0; i < draws && (int32_t)rhos.size() < p->n_det; ++i)
      if (std::find(rhos.begin(), rhos.end(), smp[i]) == rhos.end()) rhos.push_back(smp[i]);
  }
  const int K = (int)rhos.size();
  if (n_det_out) *n_det_out = K;
  const size_t C = (size_t)K * A;
  std::vector<uint64_t> visits(C, 0), wins(C, 0);
  const uint64_t n = p->sims_per_child;
  const int P = st->P;
  uint64_t N = 0;
  // expansion: the first min(expansions, C) iterations visit children 0, 1, ...
  // in index order (all unvisited: +inf, ties -> smallest index), independent
  // of each other -> one batch per rho_i
  const size_t k = (size_t)p->expansions < C ? (size_t)p->expansions : C;
  std::vector<uint64_t> h((size_t)A * P), rr((size_t)A);
  for (int i = 0; (size_t)i * A < k; ++i) {
    const int m = (int)std::min<size_t>((size_t)A, k - (size_t)i * A);
    for (int a = 0; a < m; ++a) rr[a] = rhos[i];
    int rc = dvc_rollout_batch_fixed_ex(s, codes.data(), rr.data(), m, p->seed, 1u + (uint32_t)i, 0, n, h.data(),
                                        p->device);
    if (rc) return rc;
    for (int a = 0; a < m; ++a) {
      visits[(size_t)i * A + a] = n;
      wins[(size_t)i * A + a] = h[(size_t)a * P + st->viewer];
      N += n;
    }
  }
  std::vector<uint64_t> hist((size_t)P);
  for (int it = (int)k; it < p->expansions; ++it) {
    size_t best = 0;
    double best_v = 0.0;
    for (size_t j = 0; j < C; ++j) {
      const double v = visits[j] == 0 ? INFINITY : ucb1(wins[j], visits[j], N, p->c);
      if (j == 0 || v > best_v) { best = j; best_v = v; }       // ties -> smallest index
    }
    if (visits[best] + n > (1ull << 32)) return set_error(DVC_E_CONFIG, "a child's sim index range would pass 2^32");
    const int i = (int)(best / A), a = (int)(best % A);
    int rc = dvc_rollout_batch_fixed_ex(s, &codes[a], &rhos[i], 1, p->seed, 1u + (uint32_t)i, visits[best],
                                        visits[best] + n, hist.data(), p->device);
    if (rc) return rc;
    visits[best] += n;
    wins[best] += hist[st->viewer];
    N += n;
  }
  std::vector<uint64_t> va((size_t)A, 0), wa((size_t)A, 0);
  for (size_t j = 0; j < C; ++j) {
    va[j % A] += visits[j];
    wa[j % A] += wins[j];
  }
  return finish(codes, va, wa, table, best_code);
}
