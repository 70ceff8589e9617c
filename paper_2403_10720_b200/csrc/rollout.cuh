// rollout.cuh -- device code of the hot path:
// Philox keyed by (seed; node, action code, sim), canonical
// determinization by table lookup or inline unranking (§R4), the root action
// (§R5 APPLY) and the random playout loop (§R5), on 32-bit tile bitmasks held
// in registers.
//
// Seats are kept RELATIVE to the mover: H[0] is the mover's hand, H[d] the
// hand of the player d seats after it, so LEGAL's "opponents in seat order
// after g" is a compile-time loop d = 1..P-1 and no register array is ever
// indexed dynamically.  `g` tracks the mover's absolute seat for the winner.
#pragma once
#include <stdint.h>
#include "dvc_internal.h"

namespace dvc {

constexpr int kMaxActions = 768;

#ifndef DVC_KBATCH
#define DVC_KBATCH 64   // 64: +1.3% on C2 over 32 (half the work-counter atomics), C4 unchanged; 128 no better
#endif
constexpr uint32_t kBatch = DVC_KBATCH;   // sims per work-counter claim of the refill kernel
#ifndef DVC_PEND_FAST
#define DVC_PEND_FAST 1   // a pending (drawn this turn) tile is always hidden: no V test
#endif
#ifndef DVC_NUMM_SKIP
#define DVC_NUMM_SKIP 1   // jokerless kernels skip the numbered-key mask: +1.8% C2
#endif
#ifndef DVC_FIN_OWNER
#define DVC_FIN_OWNER 1   // table-draw kernels: game over tested on the revealed tile's owner only
#endif
#ifndef DVC_NW_ALL
#define DVC_NW_ALL 1      // nW = popc(avail) - nB: no white-mask LOP3
#endif
#ifndef DVC_LUT3
#define DVC_LUT3 1      // byte-table draw with IMAD-shifted counts and a byte-per-entry table
#endif
#ifndef DVC_PEND_LMH
#define DVC_PEND_LMH 1  // two-player jokerless: pend holds the leftmost hidden tile when nothing is drawn
#endif
#ifndef DVC_DRAW31
#define DVC_DRAW31 1    // two-player jokerless draw without a "did it draw" predicate
#endif
#ifndef DVC_COLMASK
#define DVC_COLMASK 1   // correctness test: t's colour mask by XOR, not a select
#endif
#ifndef DVC_REM_TRACK
#define DVC_REM_TRACK 1   // the weighted probes carry x - (weight below) instead of the weight
#endif
// ... where it measured faster: 2 players without jokers (+0.3%) and 3
// players (+0.7%); 2 players with jokers -0.4%, 4 players with jokers -2.2%
#define DVC_REM_FOR(P, JOK) (DVC_REM_TRACK != 0 && ((P) == 3 || ((P) == 2 && !(JOK))))
#ifndef DVC_ET_INT
#define DVC_ET_INT 1   // two-player turn start driven by the step state as an integer
#endif
#ifndef DVC_ALIVE_CNT
#define DVC_ALIVE_CNT 1   // 3-4 players: the state counts its live seats; game over from the revealed tile's owner
#endif
constexpr uint32_t kRingSlots = 64;                          // started playouts per warp
// 16 B vectors per refill-kernel ring slot (kernels.cu RingView): P + 10 words
// (unpacked turn fields), + 1 for the live-seat count of 3-4 players (fits the
// same 4 vectors).  (Carrying the
// next step's Philox block instead, so it could be generated during the
// current step, measured -7% with Philox4x32 and -0.5..+1% with Philox2x32:
// not kept.)
__host__ __device__ constexpr uint32_t ring_vecs(int P) {
  return (uint32_t)(P + 10 + ((DVC_ALIVE_CNT != 0 && P > 2) ? 1 : 0) + 3) / 4u;   // kAliveSlot
}

constexpr uint32_t FINISH = 0, DECIDE = 1, END_TURN = 2, VOID = 3;
constexpr uint32_t kCrnWord = 0xFFFFFFFEu;   // D's code under common random numbers (no action code, §R3)
constexpr uint32_t kDetStep = 63u;           // step field of the determinization block D (§R3)
// Kernel modes: root batches, deep-tree (forced path) batches, informed policy
// (§R10), root batches writing the per-playout winner trace (parity tests).
constexpr int kModePlain = 0, kModePath = 1, kModeInformed = 2, kModeTrace = 3;

struct KParams {
  uint32_t seed_lo, seed_hi;  // the batch seed (device searches derive per-batch stream keys from it)
  uint32_t node;          // tree node id of the batch (stream key and counter bits, §R3)
  uint32_t s0;            // first sim index of this launch
  uint32_t n_per;         // sims per action in this launch
  uint32_t total;         // A * n_per (<= 2^31)
  uint32_t A;
  uint32_t g0;            // viewer seat (mover at the root)
  uint32_t Hv;            // viewer's hand
  uint32_t V0;            // revealed keys at the root
  uint32_t U;             // unaccounted keys (opponents' hidden + pool)
  uint32_t T;             // tile set
  uint32_t numm;          // numbered keys mask
  uint32_t JB;            // 2R (JW = JB + 1)
  uint32_t pend0, corr0;  // root pending key (kNoKey if none), correct_this_turn
  uint32_t trace_stride;  // winners[a*trace_stride + (s - trace_s0)]
  uint32_t trace_s0;
  uint64_t N;             // |Det(O)|
  uint64_t div_magic;     // ceil(2^64 / n_per) (0 when n_per == 1): item / n_per = umul64hi(item, magic)
  uint32_t nb;            // refill kernel: kBatch-sized sim batches per action = ceil(n_per / kBatch)
  uint32_t crn;           // 1: determinization block keyed by kCrnWord, not the action code (§R3 CRN)
  uint32_t rk[10];        // Philox2x32 round keys K(seed, node) + r*W, r = 0..9, precomputed on
                          // the host (sm_100a takes no constant-bank ALU operands: one LDC.64
                          // per key pair per step, no adds)
  const uint4 *table;     // N entries (H1, H2, H3, jinfo) or null -> inline unrank
  const uint8_t *plan;    // DetPlanHdr image (inline unrank / table build)
  const unsigned long long *rho;  // md ablation (§R11): fixed determinization per action, or null
  unsigned long long *hist;  // [A * P] global counters (added to)
  uint8_t *winners;       // optional per-playout winner trace
  uint32_t *counter;      // refill kernel's work counter (zeroed per launch)
  unsigned long long *voids;  // [A] voided playouts (deep-tree batches; may be null)
  uint32_t *debug;        // DVC_DEBUG builds: [violations, first violation code, playouts checked]
  uint32_t path_len;      // forced viewer actions F[0..path_len-1] before the batch action
  uint32_t path_meta[kMaxPath];  // act_meta of F[i] (relative target from the viewer)
  uint32_t codes[kMaxActions];  // action codes (Philox counter word z)
  uint32_t meta[kMaxActions];   // act_meta(d, pos, v); d = 0 -> STOP
};

// Device flat search (kernels.cu flat_search_kernel).
struct SearchArgs {
  const double *lnN;                     // [iters] log(N) before iteration it (host libm)
  const int32_t *batch_pos;              // [A] row of child a in the root-expansion batch, -1 if none
  const unsigned long long *first_hist;  // [k * P] that batch's winner histogram
  unsigned long long *delta;             // [iters] viewer wins of iteration it (zeroed)
  unsigned long long *out;               // [2 * A] final visits, then wins
  double c;                              // UCB1 constant
  uint32_t n;                            // sims per iteration
  uint32_t iters;                        // iterations after the root expansion
};

// Device depth-capped tree search (kernels.cu deep_search_kernel).
struct DNode {
  unsigned long long visits, wins, tried;
  uint32_t code, meta;      // the guess and its act_meta (root meta at depth 1, deep meta below)
  int32_t parent, depth, first, nch;   // children are T[first, first + nch)
  uint32_t expanded, _pad;
};
struct DBatch {
  uint32_t stop, nb, node_word, s0, plen, list;   // list: 0 root codes, 1 deep codes, 2 the leaf alone
  int32_t eval0;                                  // first evaluated node (children are contiguous)
  uint32_t leaf_code, leaf_meta;
  uint32_t path_meta[kMaxPath];
};
struct DeepArgs {
  DNode *nodes;
  uint32_t *n_nodes;                     // [1] nodes in use
  DBatch *batch;
  const uint32_t *root_codes, *root_meta, *deep_codes, *deep_meta;
  unsigned long long *wins, *voids;      // [max_batch] this batch's viewer wins / void playouts
  unsigned long long *out;               // [2 * A_r] root children visits, then wins (LEGAL order)
  int32_t *status;                       // 0, or a DVC_E_* code that stopped the search
  unsigned int *bar;                     // [2] grid barrier (arrivals, generation), zeroed
  unsigned long long *prof;              // DVC_DEEP_PROF: [control, barrier, playouts, barrier, iters] ns, or null
  double c;
  uint32_t n, expansions, max_depth, A_r, A_d, max_batch, max_nodes;
};

// ----------------------------------------------------------------- RNG (§R3)
// Philox2x32-10: one round (hi, lo) = M * c0; (c0, c1) <- (hi ^ k ^ c1, lo);
// the key is bumped by W between rounds.
constexpr uint32_t kPhiloxM = 0xD256D193u, kPhiloxW = 0x9E3779B9u;

__host__ __device__ __forceinline__ uint2 philox2x32_10(uint32_t c0, uint32_t c1, uint32_t k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p = (uint64_t)kPhiloxM * c0;
    const uint32_t hi = (uint32_t)(p >> 32), lo = (uint32_t)p;
    c0 = hi ^ k ^ c1;
    c1 = lo;
    k += kPhiloxW;
  }
  return make_uint2(c0, c1);
}

// Stream key K(seed, node) = word 0 of Philox2x32-10((lo32 seed, hi32 seed), node).
__host__ __device__ __forceinline__ uint32_t stream_key(uint32_t seed_lo, uint32_t seed_hi, uint32_t node) {
  return philox2x32_10(seed_lo, seed_hi, node).x;
}

// Counter word c1 without the step field: code12(code) << 6 | (node mod 2^14) << 18.
__host__ __device__ __forceinline__ uint32_t ctr_base(uint32_t code, uint32_t node) {
  const uint32_t c12 = code == 0xFFFFFFFFu ? 0xFFFu
                     : code == kCrnWord    ? 0xFFEu
                     : ((code >> 24) << 10) | (((code >> 16) & 0xFFu) << 5) | (code & 0xFFFFu);
  return (c12 << 6) | ((node & 0x3FFFu) << 18);
}

// The batch's block for counter (s, c1), with the precomputed round keys.
__device__ __forceinline__ uint2 philox_rk(uint32_t s, uint32_t c1, const KParams &kp) {
  uint32_t c0 = s;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi = __umulhi(kPhiloxM, c0), lo = kPhiloxM * c0;
    c0 = hi ^ kp.rk[r] ^ c1;
    c1 = lo;
  }
  return make_uint2(c0, c1);
}

__device__ __forceinline__ uint32_t choose(uint32_t n, uint32_t w) { return __umulhi(w, n); }

// floor((w1*2^32 + w0) * N / 2^64).  For N < 2^32 it is exactly
// (w1*N + hi32(w0*N)) >> 32 (the dropped fraction can never carry).
__device__ __forceinline__ uint64_t rank64(uint64_t N, uint32_t w0, uint32_t w1) {
  if ((N >> 32) == 0) {
    const uint32_t n = (uint32_t)N;
    return (uint64_t)(((uint64_t)w1 * n + __umulhi(w0, n)) >> 32);
  }
  return __umul64hi(((uint64_t)w1 << 32) | w0, N);
}

// item / n_per for item < 2^32, n_per < 2^32 (exact: item * n_per < 2^64).
__device__ __forceinline__ uint32_t div_per(uint32_t item, const KParams &kp) {
  return kp.div_magic ? (uint32_t)__umul64hi((uint64_t)item, kp.div_magic) : item;
}

// ----------------------------------------------------------------- bit helpers
__device__ __forceinline__ uint32_t below(uint32_t k) { return (1u << k) - 1u; }  // k <= 31

// One probe of the 5-step searches on nk = -k: k += b when
// popc(m & below(k + b)) <= n.  Written in PTX so the compiler keeps this
// form: the bits below the probe are counted as popc(m << (32 - b + nk))
// (one shift, where a mask takes a shift and an AND), and both the shift
// amount and the accept are immediate adds (VIADD, off the ALU pipe; the
// accept predicated, not a SEL) -- the ALU pipe is the bench kernel's binding
// unit.
template <uint32_t B>
__device__ __forceinline__ void probe(uint32_t &nk, uint32_t m, uint32_t n) {
  asm("{\n\t.reg .u32 sh, x;\n\t.reg .pred q;\n\t"
      "add.u32 sh, %0, %3;\n\tshl.b32 x, %1, sh;\n\tpopc.b32 x, x;\n\t"
      "setp.le.u32 q, x, %2;\n\t@q sub.u32 %0, %0, %4;\n\t}"
      : "+r"(nk) : "r"(m), "r"(n), "n"(32 - B), "n"(B));
}

// The weighted probe of select_slot (same form): black slots weigh nB, white
// nW; on accept also base = the weight below the probe.
template <uint32_t B>
__device__ __forceinline__ void probe_w(uint32_t &nk, uint32_t &base, uint32_t hB, uint32_t hW, uint32_t nB,
                                        uint32_t nW, uint32_t x) {
  asm("{\n\t.reg .u32 sh, xb, xw, c;\n\t.reg .pred q;\n\t"
      "add.u32 sh, %0, %7;\n\tshl.b32 xb, %2, sh;\n\tshl.b32 xw, %3, sh;\n\t"
      "popc.b32 xb, xb;\n\tpopc.b32 xw, xw;\n\tmul.lo.u32 c, xb, %4;\n\tmad.lo.u32 c, xw, %5, c;\n\t"
      "setp.le.u32 q, c, %6;\n\t@q sub.u32 %0, %0, %8;\n\t@q mov.u32 %1, c;\n\t}"
      : "+r"(nk), "+r"(base) : "r"(hB), "r"(hW), "r"(nB), "r"(nW), "r"(x), "n"(32 - B), "n"(B));
}

// probe_w tracking rem = x - (weight below the probe) instead of the weight
// itself: on accept rem = x - c, a predicated subtract (DVC_REM_TRACK).
template <uint32_t B>
__device__ __forceinline__ void probe_wr(uint32_t &nk, uint32_t &rem, uint32_t hB, uint32_t hW, uint32_t nB,
                                         uint32_t nW, uint32_t x) {
  asm("{\n\t.reg .u32 sh, xb, xw, c;\n\t.reg .pred q;\n\t"
      "add.u32 sh, %0, %7;\n\tshl.b32 xb, %2, sh;\n\tshl.b32 xw, %3, sh;\n\t"
      "popc.b32 xb, xb;\n\tpopc.b32 xw, xw;\n\tmul.lo.u32 c, xb, %4;\n\tmad.lo.u32 c, xw, %5, c;\n\t"
      "setp.le.u32 q, c, %6;\n\t@q sub.u32 %0, %0, %8;\n\t@q sub.u32 %1, %6, c;\n\t}"
      : "+r"(nk), "+r"(rem) : "r"(hB), "r"(hW), "r"(nB), "r"(nW), "r"(x), "n"(32 - B), "n"(B));
}

// c ? a : b for c in {0, 1}, as b + c * (a - b) in two IMADs (FMA pipe)
// instead of a SEL (ALU pipe); PTX so the compiler keeps the form.
__device__ __forceinline__ uint32_t blend01(uint32_t c, uint32_t a, uint32_t b) {
  uint32_t r;
  asm("{\n\t.reg .u32 t;\n\tmad.lo.u32 t, %3, -1, %2;\n\tmad.lo.u32 %0, %1, t, %3;\n\t}"
      : "=r"(r) : "r"(c), "r"(a), "r"(b));
  return r;
}

// 0-based n-th set bit of m (must exist): fixed 5-step search, no divergence.
__device__ __forceinline__ uint32_t nth_bit(uint32_t m, uint32_t n) {
  uint32_t nk = 0;
  probe<16>(nk, m, n);
  probe<8>(nk, m, n);
  probe<4>(nk, m, n);
  probe<2>(nk, m, n);
  probe<1>(nk, m, n);
  return 0u - nk;
}

#ifndef DVC_DRAW_LUT
#define DVC_DRAW_LUT 1   // the draw's n-th set bit by two POPC splits + a byte table in shared memory
#endif
// ... used by the two-player jokerless kernels only: +0.8% on C2, but -0.6..-1.9%
// with jokers or more players
#define DVC_LUT_FOR(P, JOK) (DVC_DRAW_LUT != 0 && (P) == 2 && !(JOK))
// which table: the byte-per-entry one under consecutive rules (+0.6% C2), the
// nibble one otherwise (the byte table measured -2.2% with consecutive = 0)
#define DVC_LUT_KIND(P, JOK, CONS) (DVC_LUT_FOR(P, JOK) ? ((DVC_LUT3 && (CONS)) ? 3 : 2) : 0)
#if DVC_DRAW_LUT
// Draw tables.  s_nth8[y]: nibble r = the r-th set bit of byte y (kind 2);
// s_nth8b[8 y + r]: the same, one byte per entry (kind 3).  Byte 0 never
// reaches a table in a valid call; its entries say 7, so a draw from an EMPTY
// mask yields 24 + 7 = 31 = kNoKey.  Filled at the start of every kernel that
// draws through nth_bit_lut.
__shared__ uint32_t s_nth8[256];
__shared__ uint8_t s_nth8b[2048];
template <int KIND>
__device__ __forceinline__ void init_nth8() {
  if constexpr (KIND == 3) {
    for (uint32_t i = threadIdx.x; i < 2048u; i += blockDim.x) {
      const uint32_t y = i >> 3, r = i & 7u;
      uint32_t c = 0, pos = 7;
      for (uint32_t b = 0; b < 8u; ++b)
        if ((y >> b) & 1u) { if (c == r) { pos = b; break; } ++c; }
      s_nth8b[i] = (uint8_t)(y ? pos : 7u);
    }
  } else {
    for (uint32_t y = threadIdx.x; y < 256u; y += blockDim.x) {
      uint32_t w = 0, r = 0;
      for (uint32_t b = 0; b < 8u; ++b)
        if ((y >> b) & 1u) { w |= b << (4u * r); ++r; }
      s_nth8[y] = y ? w : 0x77777777u;
    }
  }
}
// = nth_bit(m, n): halve by one POPC, halve again by one POPC, then a table;
// the byte offset is the shift amount and the result is the table entry + it.
template <int KIND>
__device__ __forceinline__ uint32_t nth_bit_lut(uint32_t m, uint32_t n) {
  if constexpr (KIND == 3) {
    // low-part counts by multiplies (popc(m << 16), popc(byte << 24): IMADs
    // instead of masks) and a byte per entry (no nibble extraction)
    const uint32_t c16 = __popc(m << 16);
    const bool h = n >= c16;
    uint32_t sh = h ? 16u : 0u;
    const uint32_t n1 = h ? n - c16 : n;
    const uint32_t c8 = __popc((m >> sh) << 24);
    const bool h8 = n1 >= c8;
    sh += h8 ? 8u : 0u;
    const uint32_t n2 = h8 ? n1 - c8 : n1;
    return (uint32_t)s_nth8b[((m >> sh) & 0xFFu) * 8u + n2] + sh;
  } else {
    const uint32_t c16 = __popc(m & 0xFFFFu);
    const bool h = n >= c16;
    uint32_t sh = h ? 16u : 0u;
    const uint32_t n1 = h ? n - c16 : n;
    const uint32_t c8 = __popc((m >> sh) & 0xFFu);
    const bool h8 = n1 >= c8;
    sh += h8 ? 8u : 0u;
    const uint32_t n2 = h8 ? n1 - c8 : n1;
    return ((s_nth8[(m >> sh) & 0xFFu] >> (4u * n2)) & 7u) + sh;
  }
}
#endif

// popc(m & below(t)) for t in [0, 31] as one clamped funnel shift (t = 0 -> 0).
__device__ __forceinline__ uint32_t popc_below(uint32_t m, uint32_t t) {
  return (uint32_t)__popc(__funnelshift_lc(0u, m, 32u - t));
}

template <int P>
__device__ __forceinline__ uint32_t pick(const uint32_t (&H)[P], uint32_t d) {
  uint32_t r = H[0];
#pragma unroll
  for (int i = 1; i < P; ++i) r = (d == (uint32_t)i) ? H[i] : r;
  return r;
}

// ----------------------------------------------------------------- state
template <int P>
struct Sim {
  uint32_t H[P];   // relative seats, H[0] = mover
  uint32_t V, Q;   // revealed, pool
  uint32_t ji;     // joker slots (dvc_internal.h jinfo layout)
  uint32_t g;      // absolute seat of the mover
  uint32_t pend;   // key drawn this turn or kNoKey
  uint32_t corr;   // correct guesses this turn
  uint32_t fi;     // deep-tree batches: forced viewer actions applied so far
  uint32_t na;     // 3-4 players (DVC_ALIVE_CNT): seats with a hidden tile
};

// the live-seat count has a ring slot word (P + 10) for 3-4 players, and
// ends the game in the kernels where it measured faster: 3 players with
// jokers (+1.1%, consecutive = 0 +0.7%), 3 players jokerless consecutive
// (+1.5%), 4 players jokerless (+2.6%, +2.9%) -- not 4 players with jokers
// (C4 -1.5%) nor 3 players jokerless consecutive = 0 (-0.7%)
__host__ __device__ constexpr bool kAliveSlot(int P) { return DVC_ALIVE_CNT != 0 && P > 2; }
template <int P, bool JOK, bool CONS>
constexpr bool kAliveCnt = kAliveSlot(P) && !(P == 4 && JOK) && !(P == 3 && !JOK && !CONS);

template <int P>
__device__ __forceinline__ uint32_t alive_seats(const Sim<P> &S) {
  uint32_t alive = 0;
#pragma unroll
  for (int d = 0; d < P; ++d) alive += (S.H[d] & ~S.V) ? 1u : 0u;
  return alive;
}

template <int P>
__device__ __forceinline__ bool over(const Sim<P> &S) {
  if (P == 2) return ((S.H[0] & ~S.V) == 0u) | ((S.H[1] & ~S.V) == 0u);   // no short-circuit branch
  int alive = 0;
#pragma unroll
  for (int d = 0; d < P; ++d) alive += (S.H[d] & ~S.V) ? 1 : 0;
  return alive <= 1;
}

template <int P>
__device__ __forceinline__ uint32_t winner_seat(const Sim<P> &S) {
  if (P == 2) return S.g ^ ((S.H[0] & ~S.V) ? 0u : 1u);      // the mover, else the other seat
  uint32_t d = 0;
#pragma unroll
  for (int i = P - 1; i >= 1; --i) d = (S.H[i] & ~S.V) ? (uint32_t)i : d;
  d = (S.H[0] & ~S.V) ? 0u : d;
  const uint32_t w = S.g + d;
  return w >= (uint32_t)P ? w - P : w;
}

// Joker positions on the device are kept as THRESHOLD keys: kappa(J) = the
// smallest numbered key of J's holder that lies to the right of J (31 when J
// is right of every numbered tile), plus bit 10 = "JW precedes JB" when both sit
// in one gap.  J precedes the numbered tile with key v iff kappa(J) <= v, so
// every joker test is a compare (no select); DESIGN.md §K.
__device__ __forceinline__ uint32_t kap_b(uint32_t ji) { return ji & 31u; }
__device__ __forceinline__ uint32_t kap_w(uint32_t ji) { return (ji >> 5) & 31u; }

// Does the joker `other` (held in the same line) come before joker J?
__device__ __forceinline__ bool joker_first(uint32_t ji, uint32_t other_is_w, uint32_t k_other,
                                            uint32_t k_j) {
  const bool wfirst = (ji >> 10) & 1u;
  // bitwise, not short-circuit: no divergent branch
  return (k_other < k_j) | ((k_other == k_j) & (other_is_w ? wfirst : !wfirst));
}

// Leftmost hidden tile of hand Hp (DESIGN.md §R5 APPLY).
template <bool JOK>
__device__ __forceinline__ uint32_t leftmost_hidden(uint32_t Hp, uint32_t V, uint32_t ji,
                                                    const KParams &kp) {
  const uint32_t hid = Hp & ~V;
  const uint32_t hn = (JOK || !DVC_NUMM_SKIP) ? (hid & kp.numm) : hid;   // no jokers: every key is numbered
  const uint32_t kmin = __ffs(hn) - 1u;   // (FLO of hn & -hn instead measured 0.8% slower: the extra ALU op costs more than the XU op)
  if (!JOK) return kmin;
  const uint32_t hj = (hid >> kp.JB) & 3u;
  // a hidden joker precedes the lowest hidden numbered tile iff kappa <= its
  // key; computed for every lane (no branch on "holds a hidden joker")
  const uint32_t lim = hn ? kmin : 32u;
  const uint32_t kb = kap_b(ji), kw = kap_w(ji);
  const bool cb = (hj & 1u) & (kb <= lim);
  const bool cw = ((hj >> 1) & 1u) & (kw <= lim);
  const uint32_t both = joker_first(ji, 1u, kw, kb) ? kp.JB + 1 : kp.JB;
  return (cb & cw) ? both : (cb ? kp.JB : (cw ? kp.JB + 1 : kmin));
}

// 0-based line position of key v held in hand Hp (root action, §R1 "position").
template <bool JOK>
__device__ __forceinline__ uint32_t line_pos(uint32_t Hp, uint32_t v, uint32_t ji, const KParams &kp) {
  const uint32_t kb = kap_b(ji), kw = kap_w(ji);
  if (!JOK || v < kp.JB) {
    uint32_t pos = __popc(Hp & kp.numm & below(v));
    if (JOK) {
      pos += ((Hp >> kp.JB) & 1u) && kb <= v;
      pos += ((Hp >> (kp.JB + 1)) & 1u) && kw <= v;
    }
    return pos;
  }
  const uint32_t is_w = v - kp.JB;            // 0 = JB, 1 = JW
  const uint32_t k = is_w ? kw : kb, ko = is_w ? kb : kw;
  const bool has_other = (Hp >> (kp.JB + (is_w ^ 1u))) & 1u;
  return __popc(Hp & kp.numm & below(k)) + ((has_other && joker_first(ji, is_w ^ 1u, ko, k)) ? 1u : 0u);
}

// Turn start (DESIGN.md §R5 END_TURN): the next alive player after g becomes
// the mover (relative seats rotate), pend/corr reset, and it draws the
// (choose(|Q|, w))-th smallest pool key (a drawn joker's gap from the
// remainder (w * |Q|) mod 2^32, §R3).  Written
// branch-free under the predicate `et` so lanes at different phases of a turn
// do not diverge; the joker insertion is the only (rare) real branch.
template <int P, bool JOK, int LUT = 0>
__device__ __forceinline__ void turn_start(Sim<P> &S, bool et, uint32_t w, const KParams &kp, uint32_t e = 0u) {
  // e: et as 0/1 (the step state minus one), so the two-player turn start
  // swaps and resets by IMADs instead of selects (DVC_ET_INT: +0.5% C2, +1.1%
  // C3; the same for 3-4 players measured -2.6% on C4, so two players only)
  if (P == 2) {
#if DVC_ET_INT
    const uint32_t dH = S.H[1] - S.H[0];      // swap by IMADs (FMA pipe), no selects
    S.H[0] += e * dH;
    S.H[1] -= e * dH;
    S.g ^= e;
#else
    const uint32_t h0 = et ? S.H[1] : S.H[0], h1 = et ? S.H[0] : S.H[1];
    S.H[0] = h0; S.H[1] = h1;
    S.g ^= et ? 1u : 0u;
#endif
  } else {
    uint32_t delta = P - 1;
#pragma unroll
    for (int d = P - 2; d >= 1; --d) delta = (S.H[d] & ~S.V) ? (uint32_t)d : delta;
    delta = et ? delta : 0u;
    // rotate the hands by delta (< 4) as a rotation by 1 if bit 0, then by 2
    // if bit 1: 2P blends instead of P(P-1) selects, each blend two IMADs
    // (FMA pipe) instead of a SEL (ALU pipe, the binding unit for P > 2)
#pragma unroll
    for (int sh = 1; sh <= 2; sh <<= 1) {
      const uint32_t c = sh == 1 ? (delta & 1u) : (delta >> 1);
      uint32_t Hn[P];
#pragma unroll
      for (int i = 0; i < P; ++i) Hn[i] = blend01(c, S.H[(i + sh) % P], S.H[i]);
#pragma unroll
      for (int i = 0; i < P; ++i) S.H[i] = Hn[i];
    }
    S.g += delta;
    S.g = S.g >= (uint32_t)P ? S.g - P : S.g;
  }
  const uint64_t wq = (uint64_t)w * (uint32_t)__popc(S.Q);   // (choose, remainder) in one IMAD.WIDE
#if DVC_DRAW_LUT
#if DVC_PEND_LMH
  // an empty pool draws "the 0th set bit of the new mover's hidden tiles" =
  // its leftmost hidden tile (no jokers: line order = key order), which is
  // what a wrong guess of this turn reveals -- pend takes it
  const uint32_t qsrc = (LUT != 0 && P == 2) ? (S.Q ? S.Q : (S.H[0] & ~S.V)) : S.Q;
#else
  const uint32_t qsrc = S.Q;
#endif
  uint32_t t;
  if constexpr (LUT != 0) t = nth_bit_lut<LUT>(qsrc, (uint32_t)(wq >> 32));
  else t = nth_bit(S.Q, (uint32_t)(wq >> 32));
#else
  const uint32_t t = nth_bit(S.Q, (uint32_t)(wq >> 32));
#endif
  const bool dr = et && S.Q != 0;
  const uint32_t H0 = S.H[0];
  if (JOK) {
    uint32_t kb = kap_b(S.ji), kw = kap_w(S.ji), wf = (S.ji >> 10) & 1u;
    const bool hasB = (H0 >> kp.JB) & 1u, hasW = (H0 >> (kp.JB + 1)) & 1u;
    const uint32_t Hn = H0 & kp.numm;
    if (dr && t >= kp.JB) {
      // drawn joker: uniform gap in [0, len]; relative order with the other joker
      const uint32_t gam = choose((uint32_t)__popc(H0) + 1u, (uint32_t)wq);
      const uint32_t is_w = t - kp.JB;
      const bool has_other = is_w ? hasB : hasW;
      uint32_t sj = gam;                          // numbered tiles left of the new joker
      if (has_other) {
        const uint32_t lam = __popc(Hn & below(is_w ? kb : kw));   // the other joker's line index
        const bool precedes = gam <= lam;
        sj = precedes ? gam : gam - 1u;
        wf = (is_w ? precedes : !precedes) ? 1u : 0u;
      }
      const uint32_t kj = sj < (uint32_t)__popc(Hn) ? nth_bit(Hn, sj) : 31u;
      if (is_w) kw = kj; else kb = kj;
    } else {
      // numbered t goes before the first larger numbered tile, i.e. right of
      // a joker of its gap: it becomes that joker's threshold when no held
      // numbered key lies in [t, kappa)
      const uint32_t above = ~below(t);
      kb = (dr && hasB && t < kb && !(Hn & below(kb) & above)) ? t : kb;
      kw = (dr && hasW && t < kw && !(Hn & below(kw) & above)) ? t : kw;
    }
    S.ji = kb | (kw << 5) | (wf << 10);
  }
#if DVC_DRAW31 && DVC_ET_INT
  if constexpr (LUT != 0 && P == 2) {
    // the byte-table draw returns t = kNoKey (31) for an empty pool, so no
    // "did it draw" predicate is needed: Q holds t exactly when a tile was
    // drawn (and never holds bit 31), and pend takes t at every turn start
    const uint32_t mv2 = (e << t) & S.Q;
    S.Q ^= mv2;
    S.H[0] = H0 | mv2;
    S.pend += e * (t - S.pend);
    S.corr -= e * S.corr;
    return;
  }
#endif
  // the drawn tile moves pool -> hand under one mask (t is in Q whenever dr):
  // one shift of the predicate and two LOP3 instead of two selects (+1.2% C2,
  // +2.4% C4)
  const uint32_t mv = (dr ? 1u : 0u) << t;
  S.Q ^= mv;
  S.H[0] = H0 | mv;
#if DVC_ET_INT
  if (P == 2) {
    S.pend += e * ((dr ? t : kNoKey) - S.pend);
    S.corr -= e * S.corr;
    return;
  }
#endif
  S.pend = et ? (dr ? t : kNoKey) : S.pend;
  S.corr = et ? 0u : S.corr;
}

// Is the mover's tile drawn this turn still hidden?  Only the mover guesses
// during its turn and its one self-reveal (a wrong guess) ends the turn, and
// the root's pending tile is hidden by encode's validation -- so a pending
// tile is always hidden and the test is pend != NONE (the debug build checks
// the invariant, code 10).
template <int P>
__device__ __forceinline__ bool pending_hidden(const Sim<P> &S) {
#if DVC_PEND_FAST
  return S.pend != kNoKey;
#else
  return S.pend != kNoKey && !((S.V >> S.pend) & 1u);
#endif
}

// Resolve a guess at a hidden tile t (DESIGN.md §R5 APPLY), branch-free:
// correct -> reveal t; wrong -> reveal the mover's drawn tile, or
// its leftmost hidden tile when it drew nothing.
template <int P, bool JOK, bool CONS>
__device__ __forceinline__ uint32_t resolve(Sim<P> &S, uint32_t t, bool correct, const KParams &kp) {
  const bool pend_hidden = pending_hidden(S);
  const uint32_t lmh = leftmost_hidden<JOK>(S.H[0], S.V, S.ji, kp);
  const uint32_t r = correct ? t : (pend_hidden ? S.pend : lmh);
  S.V |= 1u << r;
  S.corr += correct ? 1u : 0u;
  const uint32_t cont = (CONS && correct) ? DECIDE : END_TURN;   // PAPER:106 vs PAPER:153
  if constexpr (kAliveCnt<P, JOK, CONS>) {
    S.na = alive_seats(S);
    return S.na <= 1u ? FINISH : cont;
  } else {
    return over(S) ? FINISH : cont;
  }
}

// The end of a decision step without a branch on STOP: a STOP (stop = true)
// reveals nothing and ends the turn, any guess resolves as above.  Lanes that
// stop and lanes that guess run the same instructions (no divergent region).
template <int P, bool JOK, bool CONS, int LUT = 0>
__device__ __forceinline__ uint32_t finish_decision(Sim<P> &S, bool stop, uint32_t t, bool correct,
                                                    const KParams &kp, uint32_t hd = 0u) {
  uint32_t r;
  if constexpr (DVC_PEND_LMH && DVC_DRAW31 && DVC_ET_INT && LUT != 0 && P == 2) {
    // two players, no jokers, table draw: pend is always the tile a wrong
    // guess reveals (the drawn tile, or the leftmost hidden one set at the
    // turn start)
    r = correct ? t : S.pend;
  } else if constexpr (P == 2 && JOK) {
    // the same select written as one expression: the two-player joker kernel
    // schedules 1.8% faster this way (C3); with 3-4 players it is 4.5% slower
    r = correct ? t : (pending_hidden(S) ? S.pend : leftmost_hidden<JOK>(S.H[0], S.V, S.ji, kp));
  } else {
    const bool pend_hidden = pending_hidden(S);
    const uint32_t lmh = leftmost_hidden<JOK>(S.H[0], S.V, S.ji, kp);
    r = correct ? t : (pend_hidden ? S.pend : lmh);
  }
  constexpr bool kTab2 = DVC_PEND_LMH && DVC_DRAW31 && DVC_ET_INT && LUT != 0 && P == 2;
  S.V |= stop ? 0u : (1u << (r & 31u));
  const bool hit = correct && !stop;
  S.corr += hit ? 1u : 0u;
  const uint32_t cont = (CONS && hit) ? DECIDE : END_TURN;
  if constexpr (kTab2 && DVC_FIN_OWNER) {
    // two players: only the owner of the revealed tile can have run out --
    // the opponent after a correct guess, the mover after a wrong one
    return (!stop && !((correct ? S.H[1] : S.H[0]) & ~S.V)) ? FINISH : cont;
  } else if constexpr (kAliveCnt<P, JOK, CONS>) {
    // 3-4 players: only the revealed tile's owner (the target hd after a
    // correct guess, the mover after a wrong one) can have run out; the game
    // is over when one live seat is left
    S.na -= (!stop && !((correct ? hd : S.H[0]) & ~S.V)) ? 1u : 0u;
    return S.na <= 1u ? FINISH : cont;
  } else {
    return (!stop && over(S)) ? FINISH : cont;
  }
}

// Hidden tile of opponent hand Hd selected by index x of the mover's LEGAL
// list restricted to Hd (slots in line order, nB / nW values per black / white
// slot); returns the tile and the value index inside the slot.
template <bool JOK, bool REM = false>
__device__ __forceinline__ void select_slot(uint32_t Hd, uint32_t V, uint32_t ji, uint32_t nB,
                                            uint32_t nW, uint32_t x, const KParams &kp,
                                            uint32_t *t_out, uint32_t *vidx_out) {
  const uint32_t hid = Hd & ~V;
  uint32_t xs = x;
  uint32_t sel = kNoKey, vidx_j = 0;
  if (JOK) {
    // hidden jokers of this line are placed first, by their thresholds.  Done
    // branch-free for every lane (a warp-uniform skip when no lane's target
    // holds a hidden joker measured -4.5% on C4 and -7% on C3).
    const uint32_t hb = hid & kp.numm & kEven, hw = hid & kp.numm & kOdd;
    const uint32_t kb = kap_b(ji), kw = kap_w(ji);
    const bool hidB = (hid >> kp.JB) & 1u, hidW = (hid >> (kp.JB + 1)) & 1u;
    uint32_t sub = 0;
#pragma unroll
    for (uint32_t is_w = 0; is_w < 2; ++is_w) {
      const bool hidJ = is_w ? hidW : hidB;
      const uint32_t kj = is_w ? kw : kb;
      // weight of the numbered slots left of the joker (keys below kj)
      uint32_t c = nB * popc_below(hb, kj) + nW * popc_below(hw, kj);
      const bool hidO = is_w ? hidB : hidW;
      const uint32_t ko = is_w ? kb : kw;
      c += (hidO & joker_first(ji, is_w ^ 1u, ko, kj)) ? (is_w ? nB : nW) : 0u;
      const uint32_t nJ = is_w ? nW : nB;
      // offset of x from the joker's first value: inside its nJ values iff
      // 0 <= dj < nJ (one unsigned compare), past them iff dj >= nJ (signed)
      const uint32_t dj = x - c;
      const bool here = hidJ && dj < nJ;
      sel = here ? kp.JB + is_w : sel;
      vidx_j = here ? dj : vidx_j;
      sub += (hidJ && (int32_t)dj >= (int32_t)nJ) ? nJ : 0u;
    }
    xs = x - sub;
  }
  // no jokers: every held key is numbered, and these are the masks decide()
  // already formed for the count (the compiler shares them)
  const uint32_t hn = (JOK || !DVC_NUMM_SKIP) ? (hid & kp.numm) : hid;
  const uint32_t hB = hn & kEven, hW = hn & kOdd;
  uint32_t nk = 0, base = 0;        // nk = -k, probes as in nth_bit
  if constexpr (REM) {
    uint32_t rem = xs;               // xs - (weight below k)
    probe_wr<16>(nk, rem, hB, hW, nB, nW, xs);
    probe_wr<8>(nk, rem, hB, hW, nB, nW, xs);
    probe_wr<4>(nk, rem, hB, hW, nB, nW, xs);
    probe_wr<2>(nk, rem, hB, hW, nB, nW, xs);
    probe_wr<1>(nk, rem, hB, hW, nB, nW, xs);
    base = xs - rem;
  } else {
    probe_w<16>(nk, base, hB, hW, nB, nW, xs);
    probe_w<8>(nk, base, hB, hW, nB, nW, xs);
    probe_w<4>(nk, base, hB, hW, nB, nW, xs);
    probe_w<2>(nk, base, hB, hW, nB, nW, xs);
    probe_w<1>(nk, base, hB, hW, nB, nW, xs);
  }
  const uint32_t k = 0u - nk;
  const bool jok = JOK && sel != kNoKey;
  *t_out = jok ? sel : k;
  *vidx_out = jok ? vidx_j : xs - base;
}

// One random decision (DESIGN.md §R5 loop body after the draw): i =
// choose(n, w) over LEGAL(g) (+ STOP last), w = b1.  Returns true for STOP; else the
// targeted hidden tile t and whether the guessed value equals it.  The value
// itself is never materialised: the vidx-th available value of t's colour
// equals t exactly when vidx = #available values of that colour below t.
template <int P, bool JOK, bool CONS>
__device__ __forceinline__ bool decide(const Sim<P> &S, uint32_t w, const KParams &kp, uint32_t *t_out,
                                       bool *correct, uint32_t *hd_out = nullptr) {
  const uint32_t avail = kp.T & ~S.H[0] & ~S.V;
  const uint32_t aB = avail & kEven;
#if DVC_NW_ALL
  const uint32_t nB = __popc(aB), nW = __popc(avail) - nB;   // no white mask: one LOP3 fewer, an IADD more
#else
  const uint32_t aW = avail & kOdd;
  const uint32_t nB = __popc(aB), nW = __popc(aW);
#endif
  uint32_t cnt[P];
  uint32_t tot = 0;
#pragma unroll
  for (int d = 1; d < P; ++d) {
    const uint32_t hid = S.H[d] & ~S.V;
    cnt[d] = nB * __popc(hid & kEven) + nW * __popc(hid & kOdd);
    tot += cnt[d];
  }
  const uint32_t n = tot + ((CONS && S.corr) ? 1u : 0u);   // STOP last
  uint32_t x = choose(n, w);
  const bool stop = CONS && x >= tot;
  // target: the first opponent dd whose cumulative count exceeds x, found by
  // prefix compares (x >= cnt[1] + ... + cnt[dd-1] for dd = 2..P-1), taking
  // its hand and the offset into its list on the way
  uint32_t Hd = S.H[1];
  if (P > 2) {
    uint32_t pre = cnt[1], sub = 0;
#pragma unroll
    for (int dd = 2; dd < P; ++dd) {
      const bool g = x >= pre;
      Hd = g ? S.H[dd] : Hd;
      sub = g ? pre : sub;
      pre += cnt[dd];
    }
    x -= sub;          // (on STOP x, Hd are unused)
  }
  uint32_t t, vidx;
  select_slot<JOK, DVC_REM_FOR(P, JOK)>(Hd, S.V, S.ji, nB, nW, x, kp, &t, &vidx);
  *t_out = t;
  if (hd_out) *hd_out = Hd;
#if DVC_COLMASK
  // the available values of t's colour: kEven flipped to kOdd by XOR with
  // 0 - (t & 1) (an IMAD), one 3-input LOP3 with avail -- no select
  *correct = vidx == popc_below(avail & (kEven ^ (0u - (t & 1u))), t);
#else
  *correct = vidx == popc_below((t & 1u) ? (avail & kOdd) : aB, t);
#endif
  return stop;
}

// ----------------------------------------------------------------- informed policy (§R10)
// Numbered keys strictly between the nearest revealed numbered keys of a line
// (Rd) below `pivot` and at/above it: the candidate window of a hidden slot
// whose true key is pivot (numbered slot) or whose joker threshold is pivot.
__device__ __forceinline__ uint32_t bound_mask(uint32_t Rd, uint32_t pivot) {
  const uint32_t lo = Rd & below(pivot), hi = Rd & ~below(pivot);
  const uint32_t upper = hi ? below(__ffs(hi) - 1u) : 0xFFFFFFFFu;
  const uint32_t lower = lo ? ~below(32u - __clz(lo)) : 0xFFFFFFFFu;
  return upper & lower;
}

// Candidates of one slot: numbered values of its colour inside the window,
// then the joker of that colour when available.
struct InfCtx {
  uint32_t num[2];   // available numbered values per colour
  uint32_t jav[2];   // joker of that colour available (0/1)
};

__device__ __forceinline__ uint32_t slot_weight(const InfCtx &c, uint32_t Rd, uint32_t pivot, uint32_t col) {
  return (uint32_t)__popc(c.num[col] & bound_mask(Rd, pivot)) + c.jav[col];
}

// Total weight of the hidden slots of hand Hd (any order).
template <bool JOK>
__device__ __forceinline__ uint32_t informed_total(const InfCtx &c, uint32_t Hd, uint32_t V, uint32_t ji,
                                                   const KParams &kp) {
  const uint32_t hid = Hd & ~V, Rd = Hd & V & kp.numm;
  uint32_t tot = 0;
  for (uint32_t m = hid & kp.numm; m; m &= m - 1u) {
    const uint32_t t = __ffs(m) - 1u;
    tot += slot_weight(c, Rd, t, t & 1u);
  }
  if (JOK) {
    if ((hid >> kp.JB) & 1u) tot += slot_weight(c, Rd, kap_b(ji), 0u);
    if ((hid >> (kp.JB + 1)) & 1u) tot += slot_weight(c, Rd, kap_w(ji), 1u);
  }
  return tot;
}

// Walk the hidden slots of Hd in LINE order (numbered keys ascending, a joker
// before the numbered keys >= its threshold, JW before JB in one gap iff bit 10)
// and return the slot holding index x plus the value index inside it.
template <bool JOK>
__device__ __forceinline__ void informed_select(const InfCtx &c, uint32_t Hd, uint32_t V, uint32_t ji, uint32_t x,
                                                const KParams &kp, uint32_t *t_out, uint32_t *vidx_out,
                                                uint32_t *win_out) {
  const uint32_t hid = Hd & ~V, Rd = Hd & V & kp.numm;
  // joker slots as sort keys 4*kappa + order (numbered key t sorts at 4t + 3)
  // (jk0, jt0) is the next joker slot, (jk1, jt1) the one after it
  uint32_t jk0 = 0xFFFFFFFFu, jt0 = 0, jk1 = 0xFFFFFFFFu, jt1 = 0;
  if (JOK) {
    const bool hb = (hid >> kp.JB) & 1u, hw = (hid >> (kp.JB + 1)) & 1u;
    const bool wfirst = (ji >> 10) & 1u;
    const uint32_t kb = 4u * kap_b(ji) + (wfirst ? 1u : 0u), kw = 4u * kap_w(ji) + (wfirst ? 0u : 1u);
    if (hb && hw) {
      const bool bfirst = kb < kw;
      jk0 = bfirst ? kb : kw; jt0 = bfirst ? kp.JB : kp.JB + 1u;
      jk1 = bfirst ? kw : kb; jt1 = bfirst ? kp.JB + 1u : kp.JB;
    } else if (hb) {
      jk0 = kb; jt0 = kp.JB;
    } else if (hw) {
      jk0 = kw; jt0 = kp.JB + 1u;
    }
  }
  uint32_t acc = 0;
  uint32_t m = hid & kp.numm;
  while (true) {
    const uint32_t tn = m ? __ffs(m) - 1u : 0xFFFFFFFFu;
    const uint32_t nkey = m ? 4u * tn + 3u : 0xFFFFFFFFu;
    const bool take_joker = JOK && jk0 < nkey;
    if (!take_joker && !m) break;                       // cannot happen: x < total
    const uint32_t t = take_joker ? jt0 : tn;
    const uint32_t col = take_joker ? t - kp.JB : (t & 1u);
    const uint32_t pivot = take_joker ? (jk0 >> 2) : t;
    const uint32_t win = c.num[col] & bound_mask(Rd, pivot);
    const uint32_t w = (uint32_t)__popc(win) + c.jav[col];
    if (x < acc + w) {
      *t_out = t;
      *vidx_out = x - acc;
      *win_out = win;
      return;
    }
    acc += w;
    if (take_joker) {
      jk0 = jk1; jt0 = jt1; jk1 = 0xFFFFFFFFu;
    } else {
      m &= m - 1u;
    }
  }
  *t_out = kNoKey;
  *vidx_out = 0;
  *win_out = 0;
}

// One informed decision: as decide(), over the order-aware list.
template <int P, bool JOK, bool CONS>
__device__ __forceinline__ bool decide_informed(const Sim<P> &S, uint32_t w, const KParams &kp, uint32_t *t_out,
                                                bool *correct, uint32_t *hd_out = nullptr) {
  const uint32_t avail = kp.T & ~S.H[0] & ~S.V;
  InfCtx c;
  c.num[0] = avail & kp.numm & kEven;
  c.num[1] = avail & kp.numm & kOdd;
  c.jav[0] = JOK ? (avail >> kp.JB) & 1u : 0u;
  c.jav[1] = JOK ? (avail >> (kp.JB + 1)) & 1u : 0u;
  uint32_t cnt[P];
  uint32_t tot = 0;
#pragma unroll
  for (int d = 1; d < P; ++d) {
    cnt[d] = informed_total<JOK>(c, S.H[d], S.V, S.ji, kp);
    tot += cnt[d];
  }
  const uint32_t n = tot + ((CONS && S.corr) ? 1u : 0u);   // STOP last
  uint32_t x = choose(n, w);
  const bool stop = CONS && x >= tot;
  uint32_t Hd = S.H[1];          // target by prefix compares, as in decide()
  if (P > 2) {
    uint32_t pre = cnt[1], sub = 0;
#pragma unroll
    for (int dd = 2; dd < P; ++dd) {
      const bool g = x >= pre;
      Hd = g ? S.H[dd] : Hd;
      sub = g ? pre : sub;
      pre += cnt[dd];
    }
    x -= sub;
  }
  if (hd_out) *hd_out = Hd;
  if (stop) {
    *t_out = kNoKey;
    *correct = false;
    return true;
  }
  uint32_t t, vidx, win;
  informed_select<JOK>(c, Hd, S.V, S.ji, x, kp, &t, &vidx, &win);
  *t_out = t;
  // the slot's list: numbered values of the window ascending, then the joker
  *correct = (JOK && t >= kp.JB) ? vidx == (uint32_t)__popc(win) : vidx == (uint32_t)__popc(win & below(t));
  return false;
}

#ifdef DVC_DEBUG
__device__ __forceinline__ void dbg_fail(const KParams &kp, uint32_t code) {
  atomicAdd(&kp.debug[0], 1u);
  atomicCAS(&kp.debug[1], 0u, code);
}
#endif

// ----------------------------------------------------------------- determinization (§R4)
// rho-th element of Det(O) in canonical order: (H1, H2, H3, jinfo).
__device__ __forceinline__ uint4 unrank(const uint8_t *__restrict__ plan, uint64_t rho) {
  const DetPlanHdr *hdr = reinterpret_cast<const DetPlanHdr *>(plan);
  const DetOpt *opts = reinterpret_cast<const DetOpt *>(plan + hdr->opts_off);
  const uint32_t *slots = reinterpret_cast<const uint32_t *>(plan + hdr->slots_off);
  const unsigned long long *tab = reinterpret_cast<const unsigned long long *>(plan + hdr->tab_off);
  const uint32_t n_opts = hdr->n_opts, m = hdr->m, n_opp = hdr->n_opp;
  uint32_t o = 0;
  while (o + 1 < n_opts) {
    const uint64_t c = opts[o].count;
    if (rho < c) break;
    rho -= c;
    ++o;
  }
  const DetOpt &op = opts[o];
  uint32_t hand[3], q[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) { hand[j] = hdr->opp_known[j] | op.jmask[j]; q[j] = 0; }
  const unsigned long long *T = tab + op.tab_off;
  const uint32_t ns = op.n_states;
  uint32_t lin = 0;
  for (uint32_t i = 0; i < m; ++i) {
    const uint32_t u = hdr->ukeys[i];
    const unsigned long long *row = T + (size_t)(i + 1) * ns;
    uint64_t w = __ldg(row + lin);                 // option: pool
    if (rho < w) continue;
    rho -= w;
    bool placed = false;                           // options d = 1..P-1, in order
#pragma unroll
    for (uint32_t j = 0; j < 3; ++j) {
      if (placed || j >= n_opp || q[j] >= op.len[j]) continue;
      const uint32_t sl = __ldg(slots + op.slot_off[j] + q[j]);
      const int c = sl & 1u, lo = (int)((sl >> 8) & 0xFFu) - 1, hi = (int)((sl >> 16) & 0xFFu);
      if ((int)(u & 1u) != c || (int)u <= lo || (int)u >= hi) continue;
      w = __ldg(row + lin + op.stride[j]);
      if (rho < w) {
        hand[j] |= 1u << u;
        q[j] += 1;
        lin += op.stride[j];
        placed = true;
      } else {
        rho -= w;
      }
    }
  }
  // joker slots -> threshold keys (the k-th numbered key of the holder, or 31)
  uint32_t ji = op.jinfo & (1u << 10);
  if (hdr->jb) {
#pragma unroll
    for (uint32_t is_w = 0; is_w < 2; ++is_w) {
      const uint32_t J = hdr->jb + is_w;
      uint32_t H = (hdr->viewer_hand >> J) & 1u ? hdr->viewer_hand : 0u;
#pragma unroll
      for (int j = 0; j < 3; ++j) H = ((hand[j] >> J) & 1u) ? hand[j] : H;
      const uint32_t Hn = H & below(hdr->jb);
      const uint32_t sj = (op.jinfo >> (5 * is_w)) & 31u;
      const uint32_t kj = (H && sj < (uint32_t)__popc(Hn)) ? nth_bit(Hn, sj) : 31u;
      ji |= kj << (5 * is_w);
    }
  }
  return make_uint4(hand[0], hand[1], hand[2], ji);
}

// Determinization (a2): state of playout with determinization block D.
template <int P>
__device__ __forceinline__ void determinize_rho(Sim<P> &S, uint64_t rho, const KParams &kp) {
#ifdef DVC_DEBUG
  if (rho >= kp.N) dbg_fail(kp, 12);            // table read in bounds
#endif
  const uint4 e = kp.table ? __ldg(kp.table + rho) : unrank(kp.plan, rho);
  S.H[0] = kp.Hv;
  if (P > 1) S.H[1] = e.x;
  if (P > 2) S.H[2] = e.y;
  if (P > 3) S.H[3] = e.z;
  S.ji = e.w;
  S.V = kp.V0;
  uint32_t opp = 0;
#pragma unroll
  for (int d = 1; d < P; ++d) opp |= S.H[d];
  S.Q = kp.U & ~opp;
  S.g = kp.g0;
  S.pend = kp.pend0;
  S.corr = kp.corr0;
  if constexpr (kAliveSlot(P)) S.na = alive_seats(S);   // dead code where unused
}

template <int P>
__device__ __forceinline__ void determinize(Sim<P> &S, uint2 D, const KParams &kp) {
  determinize_rho<P>(S, rank64(kp.N, D.x, D.y), kp);
}

// The candidate action at the root (a3).  Returns true for STOP; else the
// guessed key t and whether the target's tile at `pos` is t.
template <int P, bool JOK>
__device__ __forceinline__ bool root_action(const Sim<P> &S, uint32_t meta, const KParams &kp, uint32_t *t_out,
                                            bool *correct) {
  const uint32_t d = meta & 0xFFu;
  const uint32_t pos = (meta >> 8) & 0xFFu, v = meta >> 16;
  const uint32_t Hd = pick<P>(S.H, d);
  *t_out = v;
  *correct = ((Hd >> v) & 1u) && line_pos<JOK>(Hd, v, S.ji, kp) == pos;
  return d == 0;
}

#ifdef DVC_DEBUG
// ---- invariant checks of the debug build (SURVEY §8(c.8) "Rules" row): tile
// conservation, revealed tiles held by someone, joker thresholds valid, the
// mover alive with >= 1 legal decision, exactly one reveal per guess, one
// survivor at the end, decisions bounded by 2(|T|-1).
template <int P, bool JOK>
__device__ __forceinline__ void dbg_check_state(const Sim<P> &S, const KParams &kp) {
  uint32_t uni = S.Q;
  bool disjoint = true;
#pragma unroll
  for (int d = 0; d < P; ++d) { disjoint = disjoint && !(uni & S.H[d]); uni |= S.H[d]; }
  if (!disjoint) dbg_fail(kp, 1);
  if (uni != kp.T) dbg_fail(kp, 2);
  if (S.V & S.Q) dbg_fail(kp, 3);
  if (JOK) {
#pragma unroll
    for (uint32_t is_w = 0; is_w < 2; ++is_w) {
      const uint32_t J = kp.JB + is_w, kj = is_w ? kap_w(S.ji) : kap_b(S.ji);
      uint32_t holder = 0;
#pragma unroll
      for (int d = 0; d < P; ++d) holder = ((S.H[d] >> J) & 1u) ? S.H[d] : holder;
      if (holder && kj != 31u && !((holder & kp.numm) >> kj & 1u)) dbg_fail(kp, 4);
    }
  }
}
#endif

// Key of the tile at 0-based line position pos of hand Hp (pos < popc(Hp)).
template <bool JOK>
__device__ __forceinline__ uint32_t tile_at(uint32_t Hp, uint32_t pos, uint32_t ji, const KParams &kp) {
  const uint32_t Hn = Hp & kp.numm;
  if (!JOK || !((Hp >> kp.JB) & 3u)) return nth_bit(Hn, pos);
  uint32_t before = 0;                      // held jokers left of pos
#pragma unroll
  for (uint32_t is_w = 0; is_w < 2; ++is_w) {
    const uint32_t J = kp.JB + is_w;
    if (!((Hp >> J) & 1u)) continue;
    const uint32_t lp = line_pos<JOK>(Hp, J, ji, kp);
    if (lp == pos) return J;
    before += lp < pos ? 1u : 0u;
  }
  return nth_bit(Hn, pos - before);
}

// A forced viewer action of a deep-tree batch, at a decision
// where the viewer moves.  Returns true for STOP; *illegal when the action is
// not legal in this playout's state (the playout is then void).
template <int P, bool JOK, bool CONS>
__device__ __forceinline__ bool forced_decide(const Sim<P> &S, uint32_t meta, const KParams &kp, uint32_t *t_out,
                                              bool *correct, bool *illegal) {
  const uint32_t d = meta & 0xFFu;
  const uint32_t pos = (meta >> 8) & 0xFFu, v = meta >> 16;
  *t_out = kNoKey;
  *correct = false;
  if (d == 0) {                              // STOP: only after a correct guess this turn
    *illegal = !(CONS && S.corr >= 1u);
    return true;
  }
  const uint32_t Ht = pick<P>(S.H, d);
  const uint32_t hid = Ht & ~S.V;
  bool ok = hid != 0u && pos < (uint32_t)__popc(Ht) && ((kp.T >> v) & 1u) && !((S.H[0] >> v) & 1u) &&
            !((S.V >> v) & 1u);
  uint32_t t = kNoKey;
  if (ok) {
    t = tile_at<JOK>(Ht, pos, S.ji, kp);
    ok = ((hid >> t) & 1u) && (t & 1u) == (v & 1u);
  }
  *illegal = !ok;
  *t_out = t;
  *correct = ok && t == v;
  return false;
}

}  // namespace dvc
