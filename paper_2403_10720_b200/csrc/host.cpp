// host.cpp -- SURVEY.md §8(a) row a0, host side, once per batch: validate the
// observation (dvc.h conventions), encode it into the pointer-free State, list
// the root's legal actions, and build the determinization plan (DESIGN.md §R4,
// §K2): joint joker options, per-opponent hidden-slot chains and the u64 count
// tables N(i, q) that the GPU unranks against.
//
// Bitmask implementation, independent of oracle/ (which uses lists).
#include <algorithm>
#include <cstring>
#include <vector>

#include "dvc_internal.h"

namespace dvc {
namespace {

inline int popc(uint32_t x) { return __builtin_popcount(x); }
inline uint32_t bit(int k) { return 1u << k; }

void fail(const char **err, const char *msg) { if (err) *err = msg; }

}  // namespace

// ---------------------------------------------------------------------------
// encode: validation in the order dvc.h documents (CONFIG, INCONSISTENT,
// PROTOCOL).
int encode(const dvc_observation *o, State *out, const char **err) {
  State s;
  std::memset(&s, 0, sizeof(s));
  const int P = o->rules.players, R = o->rules.ranks;
  if (P < 2 || P > 4 || R < 1 || R > 12 || (o->rules.jokers & ~1) || (o->rules.consecutive & ~1)) {
    fail(err, "rules out of range (players 2..4, ranks 1..12, flags 0/1)");
    return DVC_E_CONFIG;
  }
  if (o->viewer < 0 || o->viewer >= P || o->pool_size < 0 || o->correct_this_turn < 0) {
    fail(err, "viewer / pool_size / correct_this_turn out of range");
    return DVC_E_CONFIG;
  }
  for (int p = 0; p < P; ++p)
    if (o->line_len[p] < 0 || o->line_len[p] > 26) { fail(err, "line_len out of range"); return DVC_E_CONFIG; }

  s.magic = kMagic;
  s.P = P; s.R = R; s.jokers = o->rules.jokers; s.consecutive = o->rules.consecutive;
  s.viewer = o->viewer; s.pool_size = o->pool_size; s.corr = o->correct_this_turn;
  const int nT = 2 * R + (s.jokers ? 2 : 0);
  s.T = (nT == 32) ? 0xFFFFFFFFu : (bit(nT) - 1);

  // ---- tiles: valid, at most once, visibility consistent with the viewer
  uint32_t seen = 0;
  int hidden_opp = 0;
  for (int p = 0; p < P; ++p) {
    s.line_len[p] = o->line_len[p];
    for (int i = 0; i < o->line_len[p]; ++i) {
      const dvc_tile_obs &t = o->line[p][i];
      if (t.color > 1 || t.revealed > 1) { fail(err, "bad tile colour/revealed flag"); return DVC_E_INCONSISTENT; }
      if (t.value == DVC_HIDDEN) {
        if (p == s.viewer || t.revealed) { fail(err, "hidden value on a visible tile"); return DVC_E_INCONSISTENT; }
        s.line[p][i] = (uint8_t)(kHiddenSlot | t.color);
        ++hidden_opp;
        continue;
      }
      int key;
      if (t.value == DVC_JOKER) {
        if (!s.jokers) { fail(err, "joker without jokers rule"); return DVC_E_INCONSISTENT; }
        key = 2 * R + t.color;
      } else if (t.value < R) {
        key = 2 * t.value + t.color;
      } else {
        fail(err, "tile value out of range"); return DVC_E_INCONSISTENT;
      }
      if (p != s.viewer && !t.revealed) { fail(err, "opponent tile valued but not revealed"); return DVC_E_INCONSISTENT; }
      if (seen & bit(key)) { fail(err, "tile appears twice"); return DVC_E_INCONSISTENT; }
      seen |= bit(key);
      s.line[p][i] = (uint8_t)key;
      if (t.revealed) s.V |= bit(key);
      if (p == s.viewer || t.revealed) s.known[p] |= bit(key);
    }
  }
  if (popc(seen) + hidden_opp + s.pool_size != nT) {
    fail(err, "tile conservation: own + revealed + hidden + pool != |T|");
    return DVC_E_INCONSISTENT;
  }
  // ---- numbered order: viewer's line fully, opponents' revealed tiles
  const uint32_t numm = bit(2 * R) - 1;
  for (int p = 0; p < P; ++p) {
    int last = -1;
    for (int i = 0; i < s.line_len[p]; ++i) {
      uint8_t e = s.line[p][i];
      if (e & kHiddenSlot) continue;
      if (!(numm & bit(e))) continue;  // jokers are free
      if ((int)e <= last) { fail(err, "numbered tiles not ascending in a line"); return DVC_E_INCONSISTENT; }
      last = e;
    }
  }
  s.U = s.T & ~s.known[s.viewer] & ~s.V;
  // ---- determinization count
  {
    std::vector<uint8_t> img;
    s.N = build_plan(s, &img);
    if (s.N == 0) { fail(err, "no consistent determinization (N = 0)"); return DVC_E_INCONSISTENT; }
  }
  // ---- protocol
  s.pend_key = -1;
  if (s.pool_size > 0 && o->pending < 0) { fail(err, "pool non-empty but no pending draw"); return DVC_E_PROTOCOL; }
  if (o->pending >= 0) {
    if (o->pending >= s.line_len[s.viewer]) { fail(err, "pending index out of range"); return DVC_E_PROTOCOL; }
    if (o->line[s.viewer][o->pending].revealed) { fail(err, "pending tile is revealed"); return DVC_E_PROTOCOL; }
    s.pend_key = s.line[s.viewer][o->pending];
  }
  if (s.corr >= 1 && !s.consecutive) { fail(err, "correct_this_turn >= 1 needs consecutive rules"); return DVC_E_PROTOCOL; }
  if (!(s.known[s.viewer] & ~s.V)) { fail(err, "viewer has no hidden tile (terminal)"); return DVC_E_PROTOCOL; }
  {
    bool opp_alive = false;
    for (int p = 0; p < P; ++p) {
      if (p == s.viewer) continue;
      for (int i = 0; i < s.line_len[p]; ++i) if (s.line[p][i] & kHiddenSlot) opp_alive = true;
    }
    if (!opp_alive) { fail(err, "no opponent alive (terminal)"); return DVC_E_PROTOCOL; }
  }
  int32_t nl = 0;
  legal_actions(s, nullptr, 0, &nl);
  s.n_legal = nl;
  // plan-cache key
  uint64_t h = 1469598103934665603ull;
  const uint8_t *b = reinterpret_cast<const uint8_t *>(&s);
  for (size_t i = 0; i < offsetof(State, hash_lo); ++i) { h ^= b[i]; h *= 1099511628211ull; }
  s.hash_lo = (uint32_t)h; s.hash_hi = (uint32_t)(h >> 32);
  *out = s;
  return DVC_OK;
}

// ---------------------------------------------------------------------------
// LEGAL(viewer) + STOP.  codes may be null (count only).
int legal_actions(const State &s, uint32_t *codes, int32_t cap, int32_t *n_out) {
  const int P = s.P;
  const uint32_t avail = s.T & ~s.known[s.viewer] & ~s.V;
  int n = 0;
  for (int d = 1; d < P; ++d) {
    int j = (s.viewer + d) % P;
    bool alive = false;
    for (int i = 0; i < s.line_len[j]; ++i) if (s.line[j][i] & kHiddenSlot) alive = true;
    if (!alive) continue;
    for (int pos = 0; pos < s.line_len[j]; ++pos) {
      uint8_t e = s.line[j][pos];
      if (!(e & kHiddenSlot)) continue;
      uint32_t cand = avail & ((e & 1) ? kOdd : kEven);
      while (cand) {
        int v = __builtin_ctz(cand);
        cand &= cand - 1;
        if (codes && n < cap) codes[n] = ((uint32_t)j << 24) | ((uint32_t)pos << 16) | (uint32_t)v;
        ++n;
      }
    }
  }
  if (s.consecutive && s.corr >= 1) {
    if (codes && n < cap) codes[n] = DVC_STOP;
    ++n;
  }
  *n_out = n;
  return (codes && n > cap) ? DVC_E_CAPACITY : DVC_OK;
}

int decode_actions(const State &s, const uint32_t *codes, int32_t n, uint32_t *meta, const char **err) {
  const uint32_t avail = s.T & ~s.known[s.viewer] & ~s.V;
  for (int a = 0; a < n; ++a) {
    uint32_t c = codes[a];
    if (c == DVC_STOP) {
      if (!(s.consecutive && s.corr >= 1)) { fail(err, "STOP is not legal at this root"); return DVC_E_ILLEGAL; }
      meta[a] = 0;
      continue;
    }
    int j = (int)(c >> 24), pos = (int)((c >> 16) & 0xFF), v = (int)(c & 0xFFFF);
    if (j >= s.P || j == s.viewer || pos >= s.line_len[j] || v >= 32) { fail(err, "illegal action code"); return DVC_E_ILLEGAL; }
    uint8_t e = s.line[j][pos];
    if (!(e & kHiddenSlot) || (uint32_t)(v & 1) != (uint32_t)(e & 1) || !(avail & bit(v))) {
      fail(err, "illegal action code"); return DVC_E_ILLEGAL;
    }
    meta[a] = act_meta((uint32_t)((j - s.viewer + s.P) % s.P), (uint32_t)pos, (uint32_t)v);
  }
  return DVC_OK;
}

// Codes applied at the viewer's later decisions of a deep-tree batch
// (DESIGN.md §R9): only structurally valid here; legality is decided per
// playout (an illegal one voids the playout).
int decode_deep(const State &s, const uint32_t *codes, int32_t n, uint32_t *meta, const char **err) {
  for (int a = 0; a < n; ++a) {
    uint32_t c = codes[a];
    if (c == DVC_STOP) {
      if (!s.consecutive) { fail(err, "STOP can never be legal without consecutive rules"); return DVC_E_ILLEGAL; }
      meta[a] = 0;
      continue;
    }
    int j = (int)(c >> 24), pos = (int)((c >> 16) & 0xFF), v = (int)(c & 0xFFFF);
    if (j >= s.P || j == s.viewer || pos >= 26 || v >= 32 || !(s.T & bit(v))) {
      fail(err, "malformed action code in a deep-tree path");
      return DVC_E_ILLEGAL;
    }
    meta[a] = act_meta((uint32_t)((j - s.viewer + s.P) % s.P), (uint32_t)pos, (uint32_t)v);
  }
  return DVC_OK;
}

// ---------------------------------------------------------------------------
// Determinization plan (DESIGN.md §R4 reference algorithm, bitmask form).
namespace {
struct HS { int d, j, idx, c; };
}

uint64_t build_plan(const State &s, std::vector<uint8_t> *img) {
  const int P = s.P, R = s.R, JB = 2 * R, JW = 2 * R + 1;
  const uint32_t numm = bit(2 * R) - 1;
  std::vector<HS> hs;
  for (int d = 1; d < P; ++d) {
    int j = (s.viewer + d) % P;
    for (int i = 0; i < s.line_len[j]; ++i)
      if (s.line[j][i] & kHiddenSlot) hs.push_back(HS{d, j, i, s.line[j][i] & 1});
  }
  // joker dimensions (JB then JW, only if unaccounted)
  std::vector<std::vector<int>> dims;
  std::vector<int> dim_key;
  if (s.jokers) {
    for (int J : {JB, JW}) {
      if (!(s.U & bit(J))) continue;
      std::vector<int> ch{-1};
      for (size_t h = 0; h < hs.size(); ++h) if (hs[h].c == (J & 1)) ch.push_back((int)h);
      dims.push_back(ch);
      dim_key.push_back(J);
    }
  }
  std::vector<std::vector<int>> joint{{}};
  for (auto &ch : dims) {
    std::vector<std::vector<int>> nx;
    for (auto &o : joint) for (int h : ch) { auto v = o; v.push_back(h); nx.push_back(v); }
    joint.swap(nx);
  }
  DetPlanHdr hdr;
  std::memset(&hdr, 0, sizeof(hdr));
  hdr.n_opp = (uint32_t)(P - 1);
  hdr.viewer_hand = s.known[s.viewer];
  hdr.jb = s.jokers ? (uint32_t)JB : 0u;
  for (uint32_t u = s.U & numm; u; u &= u - 1) hdr.ukeys[hdr.m++] = (uint32_t)__builtin_ctz(u);
  for (int d = 1; d < P; ++d) hdr.opp_known[d - 1] = s.known[(s.viewer + d) % P];
  const int m = (int)hdr.m;

  std::vector<DetOpt> opts;
  std::vector<uint32_t> slots;
  std::vector<uint64_t> tab;
  uint64_t N = 0;
  for (auto &jo : joint) {
    DetOpt op;
    std::memset(&op, 0, sizeof(op));
    // seat-indexed view of which line slots hold which joker under this option
    int jk_at[4][26];
    for (int p = 0; p < 4; ++p) for (int i = 0; i < 26; ++i) jk_at[p][i] = -1;
    for (size_t x = 0; x < jo.size(); ++x) if (jo[x] >= 0) {
      const HS &h = hs[jo[x]];
      jk_at[h.j][h.idx] = dim_key[x];
      op.jmask[h.d - 1] |= bit(dim_key[x]);
    }
    // jinfo: jslot of every joker in any line (known or assigned here)
    uint32_t ji = 0;
    for (int p = 0; p < P; ++p) {
      int nnum = 0, posB = -1, posW = -1;
      for (int i = 0; i < s.line_len[p]; ++i) {
        int k = (s.line[p][i] & kHiddenSlot) ? jk_at[p][i] : s.line[p][i];
        if (k == JB) { ji |= (uint32_t)nnum; posB = i; }
        else if (k == JW) { ji |= (uint32_t)nnum << 5; posW = i; }
        else ++nnum;
      }
      if (posB >= 0 && posW >= 0 && posW < posB) ji |= 1u << 10;
    }
    op.jinfo = ji;
    // chains
    uint32_t stride = 1;
    for (int d = 1; d < P; ++d) {
      int j = (s.viewer + d) % P;
      op.slot_off[d - 1] = (uint32_t)slots.size();
      for (int i = 0; i < s.line_len[j]; ++i) {
        if (!(s.line[j][i] & kHiddenSlot) || jk_at[j][i] >= 0) continue;
        int lo = -1, hi = 2 * R;
        for (int x = i - 1; x >= 0; --x) {
          uint8_t e = s.line[j][x];
          if (!(e & kHiddenSlot) && (numm & bit(e))) { lo = e; break; }
        }
        for (int x = i + 1; x < s.line_len[j]; ++x) {
          uint8_t e = s.line[j][x];
          if (!(e & kHiddenSlot) && (numm & bit(e))) { hi = e; break; }
        }
        slots.push_back((uint32_t)(s.line[j][i] & 1) | ((uint32_t)(lo + 1) << 8) | ((uint32_t)hi << 16));
        op.len[d - 1]++;
      }
      op.stride[d - 1] = stride;
      stride *= op.len[d - 1] + 1;
    }
    op.n_states = stride;
    op.tab_off = (uint32_t)tab.size();
    tab.resize(tab.size() + (size_t)(m + 1) * stride, 0);
    uint64_t *T = tab.data() + op.tab_off;
    const int nopp = P - 1;
    // N(m, q) = [every chain full]
    {
      uint32_t full = 0;
      for (int d = 0; d < nopp; ++d) full += op.len[d] * op.stride[d];
      T[(size_t)m * stride + full] = 1;
    }
    for (int i = m - 1; i >= 0; --i) {
      const int u = (int)hdr.ukeys[i];
      for (uint32_t lin = 0; lin < stride; ++lin) {
        uint64_t v = T[(size_t)(i + 1) * stride + lin];
        for (int d = 0; d < nopp; ++d) {
          uint32_t q = (lin / op.stride[d]) % (op.len[d] + 1);
          if (q >= op.len[d]) continue;
          uint32_t sl = slots[op.slot_off[d] + q];
          int c = sl & 1, lo = (int)((sl >> 8) & 0xFF) - 1, hi = (int)((sl >> 16) & 0xFF);
          if ((u & 1) == c && lo < u && u < hi) v += T[(size_t)(i + 1) * stride + lin + op.stride[d]];
        }
        T[(size_t)i * stride + lin] = v;
      }
    }
    op.count = T[0];
    N += op.count;
    opts.push_back(op);
  }
  hdr.n_opts = (uint32_t)opts.size();
  hdr.N = N;
  if (img) {
    size_t off_opts = (sizeof(DetPlanHdr) + 15) & ~(size_t)15;
    size_t off_slots = off_opts + opts.size() * sizeof(DetOpt);
    size_t off_tab = (off_slots + slots.size() * 4 + 15) & ~(size_t)15;
    size_t total = off_tab + tab.size() * 8;
    hdr.opts_off = (uint32_t)off_opts; hdr.slots_off = (uint32_t)off_slots;
    hdr.tab_off = (uint32_t)off_tab; hdr.bytes = (uint32_t)total;
    img->assign(total, 0);
    std::memcpy(img->data(), &hdr, sizeof(hdr));
    if (!opts.empty()) std::memcpy(img->data() + off_opts, opts.data(), opts.size() * sizeof(DetOpt));
    if (!slots.empty()) std::memcpy(img->data() + off_slots, slots.data(), slots.size() * 4);
    if (!tab.empty()) std::memcpy(img->data() + off_tab, tab.data(), tab.size() * 8);
  }
  return N;
}

}  // namespace dvc
