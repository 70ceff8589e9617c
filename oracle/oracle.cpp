// ORACLE (test infrastructure only) -- plain, scalar, single-threaded C++17
// implementation of the batched Da Vinci Code rollout (DESIGN.md §R1-§R6 =
// SURVEY.md §8(c.1)-(c.6)).  Built by __graft_entry__.build() into
// oracle/liboracle.so; only tests/, __graft_entry__.smoke() and bench.py's
// CPU-baseline leg load it.  It shares no code or headers with the CUDA path
// (paper_2403_10720_b200/csrc), which uses bitmask state; this file uses
// std::vector lines of (key, revealed) exactly as the rules read.
//
// Passages followed: rules PAPER:102-106 (§II-A, Fig. 1); random playout
// PAPER:114; per-simulation determinization PAPER:143; binary outcome and
// merge-by-sum PAPER:180, 183, 186; stop-after-correct variant PAPER:153.
//
// Flat observation format (int32): P, R, jokers, consecutive, viewer,
// pool_size, pending, correct_this_turn, then for each seat p: len_p followed by
// len_p triples (colour, key or -1 if hidden, revealed).
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#include <stdexcept>
#include <string>

namespace {

typedef uint32_t u32;
typedef uint64_t u64;

const int NONE = -1;

// ------------------------------------------------------------------ Philox (§R3)
// Philox2x32-10 (Salmon et al. SC'11; Random123 philox2x32).
struct Block { u32 v[2]; };

Block philox2(u32 c0, u32 c1, u32 k) {
  for (int r = 0; r < 10; ++r) {
    if (r > 0) k += 0x9E3779B9u;
    u64 p = (u64)0xD256D193u * c0;
    u32 hi = (u32)(p >> 32), lo = (u32)p;
    u32 n0 = hi ^ k ^ c1, n1 = lo;
    c0 = n0; c1 = n1;
  }
  Block b; b.v[0] = c0; b.v[1] = c1;
  return b;
}

const u32 STOP = 0xFFFFFFFFu;
const u32 CRN_WORD = 0xFFFFFFFEu;

// stream key K(seed, node) = word 0 of Philox2x32-10((lo32(seed), hi32(seed)), node)
u32 stream_key(u64 seed, u32 node) { return philox2((u32)seed, (u32)(seed >> 32), node).v[0]; }

// 12-bit image of an action code: target<<10 | position<<5 | value; STOP 0xFFF; CRN 0xFFE
u32 code12(u32 code) {
  if (code == STOP) return 0xFFFu;
  if (code == CRN_WORD) return 0xFFEu;
  return ((code >> 24) << 10) | (((code >> 16) & 0xFFu) << 5) | (code & 0xFFFFu);
}

// counter word c1 = t | code12 << 6 | (node mod 2^14) << 18; t = 63 for D
u32 ctr1(u32 t, u32 code, u32 node) { return t | (code12(code) << 6) | ((node & 0x3FFFu) << 18); }

u32 choose(u32 n, u32 w) { return (u32)(((u64)w * n) >> 32); }
u32 remainder(u32 n, u32 w) { return (u32)((u64)w * n); }   // the word left over by choose

u64 rank64(u64 N, u32 w0, u32 w1) {
  unsigned __int128 x = (((unsigned __int128)w1) << 32) | w0;
  return (u64)((x * N) >> 64);
}

// ------------------------------------------------------------------ rules (§R1, §R2)
struct Rules { int P, R, jokers, consecutive; };

int colour(int k) { return k & 1; }
bool is_joker(const Rules &r, int k) { return k >= 2 * r.R; }
int n_tiles(const Rules &r) { return 2 * r.R + (r.jokers ? 2 : 0); }

struct ObsTile { int c, key; bool rev; };
struct Obs {
  Rules rules;
  int viewer, pool_size, pending, corr;
  std::vector<std::vector<ObsTile>> lines;
};

Obs parse(const int32_t *f) {
  Obs o;
  o.rules.P = f[0]; o.rules.R = f[1]; o.rules.jokers = f[2]; o.rules.consecutive = f[3];
  o.viewer = f[4]; o.pool_size = f[5]; o.pending = f[6]; o.corr = f[7];
  int at = 8;
  o.lines.resize(o.rules.P);
  for (int p = 0; p < o.rules.P; ++p) {
    int len = f[at++];
    for (int i = 0; i < len; ++i) {
      ObsTile t; t.c = f[at]; t.key = f[at + 1]; t.rev = f[at + 2] != 0; at += 3;
      o.lines[p].push_back(t);
    }
  }
  return o;
}

struct Tile { int key; bool rev; };

struct Game {
  Rules rules;
  std::vector<std::vector<Tile>> lines;
  std::vector<int> pool;  // ascending keys
  int g, pend, corr;

  bool alive(int p) const {
    for (const Tile &t : lines[p]) if (!t.rev) return true;
    return false;
  }
  int n_alive() const { int n = 0; for (int p = 0; p < rules.P; ++p) n += alive(p); return n; }
  bool over() const { return n_alive() <= 1; }
  int winner() const {
    for (int p = 0; p < rules.P; ++p) if (alive(p)) return p;
    throw std::runtime_error("no winner");
  }
  // A numbered key goes immediately before the first numbered tile with a
  // larger key (right of any joker in its gap).
  void insert_numbered(int p, int k) {
    auto &ln = lines[p];
    size_t i = ln.size();
    for (size_t x = 0; x < ln.size(); ++x)
      if (!is_joker(rules, ln[x].key) && ln[x].key > k) { i = x; break; }
    ln.insert(ln.begin() + i, Tile{k, false});
  }
  int leftmost_hidden(int p) const {
    for (size_t x = 0; x < lines[p].size(); ++x) if (!lines[p][x].rev) return (int)x;
    throw std::runtime_error("no hidden tile");
  }
  // LEGAL(g): opponents in seat order after g, hidden positions left to right,
  // values of the slot's colour in ascending key order (joker last), excluding
  // the mover's own tiles and every revealed tile.
  // informed: keep a numbered value only if it lies strictly
  // between the nearest revealed numbered tiles left and right of the slot.
  void legal(std::vector<u32> &out, bool informed = false) const {
    out.clear();
    int P = rules.P, T = n_tiles(rules);
    // excluded[v]: v is in the mover's line or revealed in any line
    std::vector<bool> excluded(T, false);
    for (const Tile &t : lines[g]) if (t.key < T) excluded[t.key] = true;
    for (const auto &ln : lines) for (const Tile &t : ln) if (t.rev && t.key < T) excluded[t.key] = true;
    for (int d = 1; d < P; ++d) {
      int j = (g + d) % P;
      if (!alive(j)) continue;
      for (size_t pos = 0; pos < lines[j].size(); ++pos) {
        const Tile &t = lines[j][pos];
        if (t.rev) continue;
        int c = colour(t.key);
        int lo = -1, hi = 1 << 30;
        if (informed) {
          for (size_t x = 0; x < lines[j].size(); ++x) {
            const Tile &u = lines[j][x];
            if (!u.rev || is_joker(rules, u.key)) continue;
            if (x < pos) lo = u.key;
            else if (x > pos && hi == (1 << 30)) hi = u.key;
          }
        }
        for (int v = 0; v < T; ++v) {
          if (colour(v) != c) continue;
          if (excluded[v]) continue;
          if (informed && !is_joker(rules, v) && !(lo < v && v < hi)) continue;
          out.push_back(((u32)j << 24) | ((u32)pos << 16) | (u32)v);
        }
      }
    }
  }
  enum Step { FINISH, DECIDE, END_TURN };
  Step apply(u32 code) {
    if (code == STOP) return END_TURN;
    int j = code >> 24, pos = (code >> 16) & 0xFF, v = code & 0xFFFF;
    Tile &t = lines[j][pos];
    if (t.key == v) {            // correct: reveal the target
      t.rev = true;
      corr += 1;
      if (over()) return FINISH;
      return rules.consecutive ? DECIDE : END_TURN;   // PAPER:106 vs PAPER:153
    }
    // wrong: reveal the guesser's newly drawn tile; with no draw
    // this turn, its leftmost hidden tile
    int idx = -1;
    if (pend != NONE)
      for (size_t x = 0; x < lines[g].size(); ++x)
        if (lines[g][x].key == pend && !lines[g][x].rev) idx = (int)x;
    if (idx < 0) idx = leftmost_hidden(g);
    lines[g][idx].rev = true;
    return over() ? FINISH : END_TURN;
  }
  // draw word w = b0: pool index choose(|Q|, w); a drawn joker's gap from
  // the remainder (w * |Q|) mod 2^32 (§R3)
  void start_turn(u32 w) {
    int P = rules.P, nxt = -1;
    for (int d = 1; d <= P; ++d) { int p = (g + d) % P; if (alive(p)) { nxt = p; break; } }
    g = nxt; pend = NONE; corr = 0;
    if (!pool.empty()) {
      const u32 q = (u32)pool.size();
      u32 i = choose(q, w);
      int t = pool[i];
      pool.erase(pool.begin() + i);
      if (is_joker(rules, t)) {
        u32 gap = choose((u32)lines[g].size() + 1, remainder(q, w));
        lines[g].insert(lines[g].begin() + gap, Tile{t, false});
      } else {
        insert_numbered(g, t);
      }
      pend = t;
    }
  }
};

// ------------------------------------------------------------------ determinization (§R4)
struct Slot { int c, lo, hi; };

struct OptionTable {
  std::vector<int> joker_hs;                  // per joker dim: HS index or -1 (pool)
  std::vector<std::vector<Slot>> chains;      // per opponent offset
  std::vector<std::vector<int>> chain_hs;     // chain position -> HS index
  std::vector<int> radix;                     // len+1 per chain
  int n_states = 1;
  std::vector<u64> memo;                      // (m+1) * n_states, ~0 = unknown
  u64 count = 0;
};

struct DetSpace {
  Obs obs;
  int P, g0, m;
  std::vector<int> U, numbered_U;
  struct HS { int d, idx, c; };
  std::vector<HS> hs;
  std::vector<std::pair<int, std::vector<int>>> joker_dims;  // (joker key, options)
  std::vector<OptionTable> opts;
  u64 N = 0;

  explicit DetSpace(const Obs &o) : obs(o) {
    const Rules &R = obs.rules;
    P = R.P; g0 = obs.viewer;
    std::vector<bool> known(n_tiles(R), false);
    for (auto &t : obs.lines[g0]) known[t.key] = true;
    for (int p = 0; p < P; ++p) if (p != g0)
      for (auto &t : obs.lines[p]) if (t.rev) known[t.key] = true;
    for (int k = 0; k < n_tiles(R); ++k) if (!known[k]) {
      U.push_back(k);
      if (!is_joker(R, k)) numbered_U.push_back(k);
    }
    m = (int)numbered_U.size();
    for (int d = 1; d < P; ++d) {
      int j = (g0 + d) % P;
      for (size_t i = 0; i < obs.lines[j].size(); ++i)
        if (!obs.lines[j][i].rev) hs.push_back(HS{d, (int)i, obs.lines[j][i].c});
    }
    if (R.jokers) {
      for (int J : {2 * R.R, 2 * R.R + 1}) {
        if (std::find(U.begin(), U.end(), J) == U.end()) continue;
        std::vector<int> choices{-1};
        for (size_t h = 0; h < hs.size(); ++h) if (hs[h].c == colour(J)) choices.push_back((int)h);
        joker_dims.push_back({J, choices});
      }
    }
    // joint options, o_JB major, o_JW minor
    std::vector<std::vector<int>> joint{{}};
    for (auto &jd : joker_dims) {
      std::vector<std::vector<int>> nx;
      for (auto &o2 : joint) for (int h : jd.second) { auto v = o2; v.push_back(h); nx.push_back(v); }
      joint = nx;
    }
    for (auto &jo : joint) {
      OptionTable t;
      t.joker_hs = jo;
      build_chains(t);
      t.memo.assign((size_t)(m + 1) * t.n_states, ~(u64)0);
      std::vector<int> q(t.chains.size(), 0);
      t.count = count(t, 0, q);
      N += t.count;
      opts.push_back(std::move(t));
    }
  }

  void build_chains(OptionTable &t) {
    const Rules &R = obs.rules;
    for (int d = 1; d < P; ++d) {
      int j = (g0 + d) % P;
      const auto &line = obs.lines[j];
      std::vector<Slot> ch; std::vector<int> chh;
      for (size_t h = 0; h < hs.size(); ++h) {
        if (hs[h].d != d) continue;
        if (std::find(t.joker_hs.begin(), t.joker_hs.end(), (int)h) != t.joker_hs.end()) continue;
        int idx = hs[h].idx, lo = -1, hi = 2 * R.R;
        for (int x = idx - 1; x >= 0; --x)
          if (line[x].rev && !is_joker(R, line[x].key)) { lo = line[x].key; break; }
        for (int x = idx + 1; x < (int)line.size(); ++x)
          if (line[x].rev && !is_joker(R, line[x].key)) { hi = line[x].key; break; }
        ch.push_back(Slot{hs[h].c, lo, hi});
        chh.push_back((int)h);
      }
      t.chains.push_back(ch); t.chain_hs.push_back(chh);
      t.radix.push_back((int)ch.size() + 1);
      t.n_states *= (int)ch.size() + 1;
    }
  }

  static bool fits(const Slot &s, int u) { return colour(u) == s.c && s.lo < u && u < s.hi; }

  size_t sidx(const OptionTable &t, int i, const std::vector<int> &q) const {
    size_t x = 0;
    for (size_t j = 0; j < q.size(); ++j) x = x * t.radix[j] + q[j];
    return (size_t)i * t.n_states + x;
  }

  // N(i, q) = N(i+1, q) + sum_{j fits} N(i+1, q + e_j); N(m, q) = [all chains full]
  u64 count(OptionTable &t, int i, std::vector<int> &q) {
    size_t id = sidx(t, i, q);
    if (t.memo[id] != ~(u64)0) return t.memo[id];
    u64 v;
    if (i == m) {
      v = 1;
      for (size_t j = 0; j < q.size(); ++j) if (q[j] != (int)t.chains[j].size()) v = 0;
    } else {
      int u = numbered_U[i];
      v = count(t, i + 1, q);
      for (size_t j = 0; j < q.size(); ++j) {
        if (q[j] < (int)t.chains[j].size() && fits(t.chains[j][q[j]], u)) {
          q[j]++; v += count(t, i + 1, q); q[j]--;
        }
      }
    }
    t.memo[id] = v;
    return v;
  }

  // rho-th element in canonical order: key per HS index
  std::vector<int> unrank(u64 rho) {
    for (auto &t : opts) {
      if (rho >= t.count) { rho -= t.count; continue; }
      std::vector<int> assign(hs.size(), -1);
      for (size_t x = 0; x < joker_dims.size(); ++x)
        if (t.joker_hs[x] >= 0) assign[t.joker_hs[x]] = joker_dims[x].first;
      std::vector<int> q(t.chains.size(), 0);
      for (int i = 0; i < m; ++i) {
        int u = numbered_U[i];
        u64 w = count(t, i + 1, q);           // option: pool
        if (rho < w) continue;
        rho -= w;
        bool placed = false;
        for (size_t j = 0; j < q.size(); ++j) {  // options d = 1..P-1
          if (q[j] < (int)t.chains[j].size() && fits(t.chains[j][q[j]], u)) {
            q[j]++; w = count(t, i + 1, q);
            if (rho < w) { assign[t.chain_hs[j][q[j] - 1]] = u; placed = true; break; }
            q[j]--; rho -= w;
          }
        }
        if (!placed) throw std::runtime_error("unrank walk failed");
      }
      if (rho != 0) throw std::runtime_error("unrank: rho did not reach 0");
      return assign;
    }
    throw std::runtime_error("rho out of range");
  }

  Game game(const std::vector<int> &assign) const {
    Game G;
    G.rules = obs.rules;
    G.lines.resize(P);
    for (int p = 0; p < P; ++p)
      for (auto &t : obs.lines[p]) G.lines[p].push_back(Tile{t.key, t.rev});
    std::vector<bool> used(n_tiles(obs.rules), false);
    for (size_t h = 0; h < hs.size(); ++h) {
      int j = (g0 + hs[h].d) % P;
      G.lines[j][hs[h].idx].key = assign[h];
      used[assign[h]] = true;
    }
    for (int k : U) if (!used[k]) G.pool.push_back(k);
    G.g = g0;
    G.pend = obs.pending >= 0 ? obs.lines[g0][obs.pending].key : NONE;
    G.corr = obs.corr;
    return G;
  }
};

Game public_game(const Obs &o) {
  Game G; G.rules = o.rules; G.lines.resize(o.rules.P);
  for (int p = 0; p < o.rules.P; ++p)
    for (auto &t : o.lines[p]) G.lines[p].push_back(Tile{t.key >= 0 ? t.key : 1000 + t.c, t.rev});
  G.g = o.viewer; G.pend = NONE; G.corr = o.corr;
  return G;
}

void root_legal(const Obs &o, std::vector<u32> &out) {
  Game G = public_game(o);
  G.legal(out);
  if (o.rules.consecutive && o.corr >= 1) out.push_back(STOP);
}

// One playout (§R5): determinize with block D, apply the root action, then one
// Philox block per decision step.  Returns the winner; *steps = #decisions.
// crn: D keyed by CRN_WORD instead of the code (common determinizations
// across actions).

// fixed_rho: the \md ablation -- the playout's
// determinization is element *fixed_rho of Det(O) instead of rank64(N, D).
int playout(DetSpace &sp, u32 code, u64 seed, u32 node, u32 s, int *steps,
            std::vector<u32> &L, bool crn = false, bool informed = false, const u64 *fixed_rho = nullptr) {
  const u32 K = stream_key(seed, node);
  u64 rho;
  if (fixed_rho) {
    rho = *fixed_rho;
  } else {
    Block D = philox2(s, ctr1(63, crn ? CRN_WORD : code, node), K);
    rho = rank64(sp.N, D.v[0], D.v[1]);
  }
  Game G = sp.game(sp.unrank(rho));
  Game::Step st = G.apply(code);
  u32 k = 0;
  while (st != Game::FINISH) {
    if (k > 62) throw std::runtime_error("more than 63 decisions in one playout");
    Block B = philox2(s, ctr1(k, code, node), K);
    if (st == Game::END_TURN) G.start_turn(B.v[0]);
    G.legal(L, informed);
    u32 n = (u32)L.size() + ((G.rules.consecutive && G.corr >= 1) ? 1u : 0u);
    u32 i = choose(n, B.v[1]);
    k += 1;
    st = G.apply(i == L.size() ? STOP : L[i]);
  }
  if (steps) *steps = (int)k;
  return G.winner();
}

// Deep-tree playout: forced viewer actions F (F[0] at the
// root, F[i] at the viewer's i-th later decision), Philox keyed by F.back().
// Returns the winner, or -1 (VOID) when a forced action is not legal
// (LEGAL + STOP-when-allowed) or the game ends before all of F is applied.
int playout_path(DetSpace &sp, const std::vector<u32> &F, u64 seed, u32 node, u32 s, std::vector<u32> &L) {
  const u32 code = F.back();
  const u32 K = stream_key(seed, node);
  Block D = philox2(s, ctr1(63, code, node), K);
  u64 rho = rank64(sp.N, D.v[0], D.v[1]);
  Game G = sp.game(sp.unrank(rho));
  Game::Step st = G.apply(F[0]);
  size_t fi = 1;
  u32 k = 0;
  while (true) {
    if (st == Game::FINISH) return fi < F.size() ? -1 : G.winner();
    if (k > 62) throw std::runtime_error("more than 63 decisions in one playout");
    Block B = philox2(s, ctr1(k, code, node), K);
    if (st == Game::END_TURN) G.start_turn(B.v[0]);
    G.legal(L);
    const bool stop_ok = G.rules.consecutive && G.corr >= 1;
    u32 n = (u32)L.size() + (stop_ok ? 1u : 0u);
    u32 a;
    if (fi < F.size() && G.g == sp.g0) {
      a = F[fi++];
      bool ok = (a == STOP) ? stop_ok : (std::find(L.begin(), L.end(), a) != L.end());
      if (!ok) return -1;
    } else {
      u32 i = choose(n, B.v[1]);
      a = (i == L.size()) ? STOP : L[i];
    }
    k += 1;
    st = G.apply(a);
  }
}

thread_local std::string g_err;

}  // namespace

extern "C" {

const char *oracle_last_error() { return g_err.c_str(); }

void oracle_philox2(const uint32_t *ctr, uint32_t key, uint32_t *out) {
  Block b = philox2(ctr[0], ctr[1], key);
  std::memcpy(out, b.v, 8);
}

uint32_t oracle_stream_key(uint64_t seed, uint32_t node) { return stream_key(seed, node); }

void oracle_step_block(uint64_t seed, uint32_t node, uint32_t code, uint32_t s, uint32_t t, uint32_t *out) {
  Block b = philox2(s, ctr1(t, code, node), stream_key(seed, node));
  std::memcpy(out, b.v, 8);
}

int oracle_count(const int32_t *obs, uint64_t *N) {
  try { DetSpace sp(parse(obs)); *N = sp.N; return 0; }
  catch (std::exception &e) { g_err = e.what(); return -1; }
}

// keys_out[h] = key assigned to the h-th hidden slot (HS order)
int oracle_unrank(const int32_t *obs, uint64_t rho, int32_t *keys_out, int32_t cap, int32_t *n_out) {
  try {
    DetSpace sp(parse(obs));
    if (rho >= sp.N) { g_err = "rho out of range"; return -1; }
    auto a = sp.unrank(rho);
    if ((int)a.size() > cap) { g_err = "capacity"; return -5; }
    for (size_t i = 0; i < a.size(); ++i) keys_out[i] = a[i];
    *n_out = (int32_t)a.size();
    return 0;
  } catch (std::exception &e) { g_err = e.what(); return -1; }
}

int oracle_legal(const int32_t *obs, uint32_t *codes, int32_t cap, int32_t *n_out) {
  std::vector<u32> L;
  root_legal(parse(obs), L);
  *n_out = (int32_t)L.size();
  if ((int)L.size() > cap) return -5;
  for (size_t i = 0; i < L.size(); ++i) codes[i] = L[i];
  return 0;
}

// hist[a*P + w] += #playouts s in [s0, s1) of action a won by seat w
// flags: bit 0 = common random numbers (§R3), bit 1 = informed policy (§R10)
int oracle_rollout_flags(const int32_t *obs, const uint32_t *codes, int32_t n_codes, uint64_t seed,
                         uint32_t node, uint64_t s0, uint64_t s1, uint64_t *hist, int32_t flags) {
  try {
    Obs o = parse(obs);
    DetSpace sp(o);
    if (sp.N == 0) { g_err = "inconsistent"; return -4; }
    std::vector<u32> L;
    root_legal(o, L);
    for (int a = 0; a < n_codes; ++a)
      if (std::find(L.begin(), L.end(), codes[a]) == L.end()) { g_err = "illegal action"; return -3; }
    int P = o.rules.P;
    for (int a = 0; a < n_codes; ++a)
      for (u64 s = s0; s < s1; ++s)
        hist[(size_t)a * P + playout(sp, codes[a], seed, node, (u32)s, nullptr, L, (flags & 1) != 0,
                                     (flags & 2) != 0)] += 1;
    return 0;
  } catch (std::exception &e) { g_err = e.what(); return -1; }
}

// \md ablation batch: child a = (determinization rhos[a], action codes[a])
int oracle_rollout_fixed(const int32_t *obs, const uint32_t *codes, const uint64_t *rhos, int32_t n_codes,
                         uint64_t seed, uint32_t node, uint64_t s0, uint64_t s1, uint64_t *hist) {
  try {
    Obs o = parse(obs);
    DetSpace sp(o);
    if (sp.N == 0) { g_err = "inconsistent"; return -4; }
    std::vector<u32> L;
    root_legal(o, L);
    for (int a = 0; a < n_codes; ++a) {
      if (std::find(L.begin(), L.end(), codes[a]) == L.end()) { g_err = "illegal action"; return -3; }
      if (rhos[a] >= sp.N) { g_err = "rho out of range"; return -1; }
    }
    int P = o.rules.P;
    for (int a = 0; a < n_codes; ++a)
      for (u64 s = s0; s < s1; ++s)
        hist[(size_t)a * P + playout(sp, codes[a], seed, node, (u32)s, nullptr, L, false, false, rhos + a)] += 1;
    return 0;
  } catch (std::exception &e) { g_err = e.what(); return -1; }
}

int oracle_rollout(const int32_t *obs, const uint32_t *codes, int32_t n_codes, uint64_t seed,
                   uint32_t node, uint64_t s0, uint64_t s1, uint64_t *hist) {
  return oracle_rollout_flags(obs, codes, n_codes, seed, node, s0, s1, hist, 0);
}

// deep-tree batch: hist[a*P + w], voids[a] for forced path + codes[a]
int oracle_rollout_path(const int32_t *obs, const uint32_t *path, int32_t path_len, const uint32_t *codes,
                        int32_t n_codes, uint64_t seed, uint32_t node, uint64_t s0, uint64_t s1, uint64_t *hist,
                        uint64_t *voids) {
  try {
    Obs o = parse(obs);
    DetSpace sp(o);
    if (sp.N == 0) { g_err = "inconsistent"; return -4; }
    std::vector<u32> L;
    root_legal(o, L);
    if (path_len < 1 || std::find(L.begin(), L.end(), path[0]) == L.end()) { g_err = "illegal path[0]"; return -3; }
    int P = o.rules.P;
    for (int a = 0; a < n_codes; ++a) {
      std::vector<u32> F(path, path + path_len);
      F.push_back(codes[a]);
      for (u64 s = s0; s < s1; ++s) {
        int w = playout_path(sp, F, seed, node, (u32)s, L);
        if (w < 0) voids[a] += 1; else hist[(size_t)a * P + w] += 1;
      }
    }
    return 0;
  } catch (std::exception &e) { g_err = e.what(); return -1; }
}

// one playout: returns winner (>= 0) or a negative error; *steps = #decisions
int oracle_playout(const int32_t *obs, uint32_t code, uint64_t seed, uint32_t node, uint32_t s,
                   int32_t *steps) {
  try {
    DetSpace sp(parse(obs));
    std::vector<u32> L;
    int st = 0;
    int w = playout(sp, code, seed, node, s, &st, L);
    *steps = st;
    return w;
  } catch (std::exception &e) { g_err = e.what(); return -1; }
}

}  // extern "C"
