// kernels.cu -- the sm_100a kernels of the hot path.
//
//  * rollout_refill_kernel (default): persistent, warp-refilling.  Each lane
//    holds one playout in registers; the loop body is TWO decision steps for
//    every active lane.  When lanes finish, __ballot_sync counts them, one
//    leader atomicAdd on the launch's work counter hands out that many new
//    (action, sim) items and the lanes start them in the same iteration, so
//    playout-length variance does not idle lanes (BASELINE.json north_star;
//    the paper's "threads ... wait until the thread with the most turns
//    ends", is the loss this removes).
//  * rollout_naive_kernel: thread-per-playout grid-stride loop, the paper's
//    CUDA design kept as the comparison point for the C5 sweep.
//  * det_table_kernel: unranks every rho < N once per state into a table of
//    (H1, H2, H3, jinfo) so a playout's determinization is one 16 B load.
//
// Both rollout kernels reduce winners into shared-memory u32 counters
// hist[a][w] and flush them with one global atomicAdd(u64) per non-zero
// counter per block.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include "rollout.cuh"

namespace dvc {

// Register cap of the refill kernel as min resident 256-thread blocks per SM,
// per instantiation (resident 128-thread blocks then follow from the
// registers used; the grid is sized from the occupancy API).  Two players
// without jokers: 4 (64 registers; 8 blocks of 128 per SM), +1.3% on C2
// (56 or 52 registers, 9-10 blocks: -3% / -4%).  Round 2 sweep of 2 / 3 / 4
// (DESIGN.md §M): two players with jokers 2 (80 registers, +2.3% C3 over 3,
// consecutive = 0 +2.6%), three players jokerless consecutive 4 (64
// registers, +1.4%; consecutive = 0 -1.1%), four players jokerless
// consecutive = 0 2 (+0.6%; consecutive -3.1%); otherwise 3 (C4 -0.1% /
// -0.4% at 4 / 2).
#ifndef DVC_REC1_2J
#define DVC_REC1_2J 1   // the two-player joker kernel under consecutive rules records once per iteration too
#endif
#ifndef DVC_STEPS3
#define DVC_STEPS3 1   // two-player jokerless consecutive: a third nested decision step per loop iteration
#endif
#ifndef DVC_REFILL_MINB2
#define DVC_REFILL_MINB2 4
#endif
#ifndef DVC_REFILL_MINB
#define DVC_REFILL_MINB 3
#endif
#ifndef DVC_MINB_PER_INST
#define DVC_MINB_PER_INST 1
#endif
constexpr int refill_minb(int P, bool JOK, bool CONS) {
  if (P == 2 && !JOK) return DVC_REFILL_MINB2;
  if (!DVC_MINB_PER_INST) return DVC_REFILL_MINB;
  if (P == 2) return 2;
  if (P == 3 && !JOK && CONS) return 4;
  if (P == 4 && !JOK && !CONS) return 2;
  return DVC_REFILL_MINB;
}

// Shared memory: hist[A*P] u32 counters, then the action codes and metas
// (read once per playout start; per-lane indexed, so smem beats the param bank).
// hist has P + 1 columns: column P counts void playouts (deep-tree batches).
struct Smem {
  uint32_t *hist, *codes, *meta, *path;
};

template <int LUT = 0>
__device__ __forceinline__ Smem setup_smem(const KParams &kp, int P) {
  extern __shared__ uint32_t sh[];
  Smem m;
  m.hist = sh;
  m.codes = sh + kp.A * (P + 1);
  m.meta = m.codes + kp.A;
  m.path = m.meta + kp.A;
  for (uint32_t i = threadIdx.x; i < kp.A * (P + 1); i += blockDim.x) m.hist[i] = 0;
  for (uint32_t i = threadIdx.x; i < kp.A; i += blockDim.x) {
    m.codes[i] = kp.codes[i];
    m.meta[i] = kp.meta[i];
  }
  if (threadIdx.x < (uint32_t)kMaxPath) m.path[threadIdx.x] = kp.path_meta[threadIdx.x];
#if DVC_DRAW_LUT
  if constexpr (LUT != 0) init_nth8<LUT>();
#endif
  __syncthreads();
  return m;
}

__device__ __forceinline__ void flush_hist(const uint32_t *sh, const KParams &kp, int P) {
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kp.A * (P + 1); i += blockDim.x) {
    const uint32_t v = sh[i];
    if (!v) continue;
    const uint32_t a = i / (P + 1), w = i - a * (P + 1);
    if (w < (uint32_t)P) atomicAdd(kp.hist + a * P + w, (unsigned long long)v);
    else if (kp.voids) atomicAdd(kp.voids + a, (unsigned long long)v);
  }
}

// Winner column of a finished playout: its seat, or P for a void deep-tree
// playout (a forced action was illegal, or the game ended before all forced
// viewer actions were applied).
template <int P, bool PATH>
__device__ __forceinline__ uint32_t outcome(const Sim<P> &S, uint32_t st, const KParams &kp) {
  if (!PATH) return winner_seat(S);
  return (st == VOID || S.fi <= kp.path_len) ? (uint32_t)P : winner_seat(S);
}

// Count a finished playout (and, in the trace mode only, write its winner).
template <int MODE>
__device__ __forceinline__ void record(const Smem &sm, const KParams &kp, int P, uint32_t a, uint32_t s,
                                       uint32_t w) {
#ifdef DVC_DEBUG
  // bounds of every shared / global write a finished playout makes (the
  // stand-in for compute-sanitizer memcheck, which this GPU pool does not run)
  if (a >= kp.A || w > (uint32_t)P) dbg_fail(kp, 11);
  if (MODE == kModeTrace && (s - kp.trace_s0) >= kp.trace_stride) dbg_fail(kp, 13);
#endif
  atomicAdd(&sm.hist[a * (P + 1) + w], 1u);
  if (MODE == kModeTrace) kp.winners[(size_t)a * kp.trace_stride + (s - kp.trace_s0)] = (uint8_t)w;
}

// Start of playout (a, s): determinization block D, table lookup (a2), root
// action (a3).  Returns the step state.  cb = ctr_base(code, node) (§R3).
template <int P, bool JOK, bool CONS, int MODE>
__device__ __forceinline__ uint32_t start_playout(Sim<P> &S, uint32_t s, uint32_t cb, uint32_t meta, uint32_t a,
                                                  const KParams &kp) {
  constexpr bool PATH = MODE == kModePath;
  if (MODE == kModePlain && kp.rho) {
    determinize_rho<P>(S, kp.rho[a], kp);        // md ablation: the child's own determinization (§R11)
  } else {
    // cb = ctr_base(code, node); under CRN the D block takes the CRN word's base
    const uint2 D = philox_rk(s, (kp.crn ? ctr_base(kCrnWord, kp.node) : cb) | kDetStep, kp);
    determinize<P>(S, D, kp);
  }
  uint32_t t;
  bool correct;
  // deep-tree batches apply the path's first action at the root (F[0])
  const bool stop = root_action<P, JOK>(S, PATH ? kp.path_meta[0] : meta, kp, &t, &correct);
  if (PATH) S.fi = 1;
  return stop ? END_TURN : resolve<P, JOK, CONS>(S, t, correct, kp);
}

// Decision step k of a running playout (a4), given its Philox block B_k.
template <int P, bool JOK, bool CONS, int MODE, int LUT = 0>
__device__ __forceinline__ uint32_t step_block(Sim<P> &S, uint32_t st, const uint2 B, uint32_t k,
                                               const uint32_t *meta_of_a, const uint32_t *path_of, uint32_t a,
                                               const KParams &kp, uint32_t plen) {
  constexpr bool PATH = MODE == kModePath;
  turn_start<P, JOK, LUT>(S, st == END_TURN, B.x, kp, st - 1u);   // st is DECIDE (1) or END_TURN (2) here
#ifdef DVC_DEBUG
  dbg_check_state<P, JOK>(S, kp);
  if (!(S.H[0] & ~S.V)) dbg_fail(kp, 5);                       // the mover is alive
  if (k >= 2u * (uint32_t)__popc(kp.T)) dbg_fail(kp, 6);        // decisions <= 2(|T|-1)
  if (S.pend != kNoKey && ((S.V >> S.pend) & 1u)) dbg_fail(kp, 10);   // a pending tile is hidden
  const uint32_t v_before = __popc(S.V);
#endif
  uint32_t t;
  bool correct;
  bool stop;
  uint32_t hd = 0u;   // the target's hand (3-4 players: the live-seat count, DVC_ALIVE_CNT)
  if (PATH && S.fi <= plen && S.g == kp.g0) {
    // deep-tree batch: the viewer's next forced action F[fi] (the batch
    // action itself at fi == path_len) replaces the random decision
    const uint32_t m = S.fi < plen ? path_of[S.fi] : meta_of_a[a];
    bool illegal;
    stop = forced_decide<P, JOK, CONS>(S, m, kp, &t, &correct, &illegal);
    S.fi += 1;
    if (illegal) return VOID;
  } else if constexpr (MODE == kModeInformed) {
    stop = decide_informed<P, JOK, CONS>(S, B.y, kp, &t, &correct, &hd);
  } else {
    stop = decide<P, JOK, CONS>(S, B.y, kp, &t, &correct, &hd);
  }
#ifdef DVC_DEBUG
  const uint32_t r = stop ? END_TURN : resolve<P, JOK, CONS>(S, t, correct, kp);
  if ((uint32_t)__popc(S.V) != v_before + (stop ? 0u : 1u)) dbg_fail(kp, 7);   // one reveal per guess
  if (stop && !(CONS && S.corr >= 1u)) dbg_fail(kp, 8);                        // STOP only after a correct guess
  if (r == FINISH) {
    uint32_t alive = 0;
#pragma unroll
    for (int d = 0; d < P; ++d) alive += (S.H[d] & ~S.V) ? 1u : 0u;
    if (alive != 1u) dbg_fail(kp, 9);                                         // one survivor
    atomicAdd(&kp.debug[2], 1u);
  }
  dbg_check_state<P, JOK>(S, kp);
  return r;
#else
  if (PATH) return stop ? END_TURN : resolve<P, JOK, CONS>(S, t, correct, kp);
  return finish_decision<P, JOK, CONS, LUT>(S, stop, t, correct, kp, hd);
#endif
}

template <int P, bool JOK, bool CONS, int MODE>
__device__ __forceinline__ uint32_t step_playout(Sim<P> &S, uint32_t st, uint32_t k, uint32_t s, uint32_t cb,
                                                 const uint32_t *meta_of_a, const uint32_t *path_of, uint32_t a,
                                                 const KParams &kp) {
  return step_block<P, JOK, CONS, MODE, DVC_LUT_KIND(P, JOK, CONS)>(S, st, philox_rk(s, cb | k, kp), k, meta_of_a, path_of, a,
                                                             kp, kp.path_len);
}

template <int P, bool JOK, bool CONS, int MODE>
__global__ void __launch_bounds__(1024) rollout_naive_kernel(const __grid_constant__ KParams kp) {
  constexpr bool PATH = MODE == kModePath;
  const Smem sm = setup_smem<DVC_LUT_KIND(P, JOK, CONS)>(kp, P);
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < kp.total; w += stride) {
    const uint32_t a = div_per(w, kp);
    const uint32_t s = kp.s0 + (w - a * kp.n_per);
    const uint32_t cb = ctr_base(sm.codes[a], kp.node), meta = sm.meta[a];
    Sim<P> S;
    uint32_t st = start_playout<P, JOK, CONS, MODE>(S, s, cb, meta, a, kp);
    for (uint32_t k = 0; st != FINISH && !(PATH && st == VOID); ++k)
      st = step_playout<P, JOK, CONS, MODE>(S, st, k, s, cb, sm.meta, sm.path, a, kp);
    record<MODE>(sm, kp, P, a, s, outcome<P, PATH>(S, st, kp));
  }
  flush_hist(sm.hist, kp, P);
}

// ---- refill kernel -------------------------------------------------------
// Every warp keeps a ring of kRing STARTED playouts (determinized, root action
// applied) in shared memory.  Whenever the ring holds fewer than 32, the whole
// warp -- converged -- takes 32 new work items and starts them (Philox block D,
// table lookup, root action), pushing the ones still running.  The main loop is
// two (two-player jokerless consecutive: three) nested decision steps for
// every lane; a lane whose playout ends records the
// winner and pops the next started playout from the ring in the same
// iteration, so lanes never idle on playout-length variance and the start
// code never runs with a handful of lanes (BASELINE.json north_star: lanes
// retire via __ballot_sync and pull new playouts from a work counter).
constexpr uint32_t kRing = kRingSlots;

template <int P, bool JOK, bool CONS>
struct RingView {
  // AoS, ring_vecs(P) x 16 B per slot: a pop is 3-4 LDS.128 -- pops run in a
  // divergent region with ~2 lanes, so instructions, not bank conflicts, are
  // what they cost.  Words: H[P], V, Q, ji, g, pend, corr, st | fi << 4, a, s
  // and the playout's Philox counter word c1 for step 0 (ctr_base(code,
  // node), §R3), then the live-seat count na for 3-4 players.  The turn
  // fields are unpacked -- no shifts and masks on a pop;
  // packing them into one word (one vector less for 3-4 players) measured
  // 3.6% (2p), 1.4% (3p) and 1.0% (4p) slower.
  static constexpr int kNW = P + 10 + (kAliveSlot(P) ? 1 : 0);   // words used
  static constexpr uint32_t V = (kNW + 3) / 4;
  static_assert(V == ring_vecs(P), "ring slot size (host smem sizing) out of step");
  uint4 *base;
  template <bool PATH>
  __device__ __forceinline__ void put(uint32_t i, const Sim<P> &S, uint32_t st, uint32_t a, uint32_t s,
                                      uint32_t c1) const {
    uint32_t w[16];
#pragma unroll
    for (int d = 0; d < P; ++d) w[d] = S.H[d];
    w[P + 0] = S.V;
    w[P + 1] = S.Q;
    w[P + 2] = S.ji;
    w[P + 3] = S.g;
    w[P + 4] = S.pend;
    w[P + 5] = S.corr;
    w[P + 6] = PATH ? (st | (S.fi << 4)) : st;   // fi exists in deep-tree batches only
    w[P + 7] = a;
    w[P + 8] = s;
    w[P + 9] = c1;
    if constexpr (kAliveSlot(P)) w[P + 10] = kAliveCnt<P, JOK, CONS> ? S.na : 0u;
#pragma unroll
    for (int q = kNW; q < 16; ++q) w[q] = 0;
    uint4 *b = base + V * i;
#pragma unroll
    for (uint32_t q = 0; q < V; ++q) b[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
  }
  template <bool PATH>
  __device__ __forceinline__ void get(uint32_t i, Sim<P> &S, uint32_t &st, uint32_t &a, uint32_t &s,
                                      uint32_t &c1) const {
    const uint4 *b = base + V * i;
    uint32_t w[16];
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
      const uint4 v = q < V ? b[q] : make_uint4(0, 0, 0, 0);
      w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int d = 0; d < P; ++d) S.H[d] = w[d];
    S.V = w[P + 0];
    S.Q = w[P + 1];
    S.ji = w[P + 2];
    S.g = w[P + 3];
    S.pend = w[P + 4];
    S.corr = w[P + 5];
    st = PATH ? (w[P + 6] & 0xFu) : w[P + 6];
    S.fi = PATH ? (w[P + 6] >> 4) : 0u;
    a = w[P + 7];
    s = w[P + 8];
    c1 = w[P + 9];
    if constexpr (kAliveCnt<P, JOK, CONS>) S.na = w[P + 10];
  }
};

// First 16 B-aligned word of the refill kernel's rings in dynamic smem.
__host__ __device__ __forceinline__ uint32_t ring_word_offset(uint32_t A, int P) {
  return (A * (uint32_t)(P + 3) + (uint32_t)kMaxPath + 3u) & ~3u;
}

template <int P, bool JOK, bool CONS, int MODE>
__global__ void __launch_bounds__(256, refill_minb(P, JOK, CONS))
    rollout_refill_kernel(const __grid_constant__ KParams kp) {
  constexpr bool PATH = MODE == kModePath;
  const Smem sm = setup_smem<DVC_LUT_KIND(P, JOK, CONS)>(kp, P);
  extern __shared__ uint32_t sh_all[];
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const RingView<P, JOK, CONS> ring{reinterpret_cast<uint4 *>(sh_all + ring_word_offset(kp.A, P)) +
                             (threadIdx.x >> 5) * RingView<P, JOK, CONS>::V * kRing};
  // Warp-uniform work batch: sims s0 + [cs, ce) of action ca (kBatch-aligned
  // slices of ONE action, so no per-lane division).  The next batch index is
  // claimed one batch ahead (lane 0's atomicAdd result is only read at the
  // next produce), so the atomic's latency is hidden.
  uint32_t ca = 0, cs = 0, ce = 0, ccb = 0, cmeta = 0;   // ccb = ctr_base(code of ca, node)
  bool drained = false;
  const uint32_t n_batches = kp.A * kp.nb;
  uint32_t pref = 0;
  if (lane == 0) pref = atomicAdd(kp.counter, 1u);
  uint32_t head = 0, count = 0;       // ring (warp-uniform)
  bool active = false;
  // the running playout: action, sim, step state and its Philox counter word
  // c1 = ctr_base(code, node) | k, advanced by one per decision step (§R3)
  uint32_t a = 0, s = 0, st = FINISH, c1 = 0;
  Sim<P> S;
  while (true) {
    // ---- produce: the whole warp starts up to 32 playouts
    while (count < 32u && !(drained && cs >= ce)) {
      uint32_t rem = ce - cs;
      uint32_t na = 0, ns = 0, ne = 0, ncb = 0, nmeta = 0;
      bool got = false;
      if (rem < 32u && !drained) {
        const uint32_t b = __shfl_sync(0xFFFFFFFFu, pref, 0);
        if (b < n_batches) {
          if (lane == 0) pref = atomicAdd(kp.counter, 1u);     // claim the following batch
          na = b / kp.nb;
          ns = (b - na * kp.nb) * kBatch;       // relative to s0 (no u32 overflow at 2^32)
          ne = min(ns + kBatch, kp.n_per);
          ncb = ctr_base(sm.codes[na], kp.node);
          nmeta = sm.meta[na];
          got = true;
        } else {
          drained = true;
        }
      }
      bool valid = false;
      uint32_t pa = 0, ps = 0, pcb = 0, pmeta = 0;
      if (lane < rem) {
        pa = ca; ps = kp.s0 + cs + lane; pcb = ccb; pmeta = cmeta; valid = true;
      } else if (got && ns + (lane - rem) < ne) {
        pa = na; ps = kp.s0 + ns + (lane - rem); pcb = ncb; pmeta = nmeta; valid = true;
      }
      if (got) {
        ca = na; ccb = ncb; cmeta = nmeta; ce = ne;
        cs = min(ns + (32u - rem), ne);
      } else {
        cs = min(cs + 32u, ce);
      }
      Sim<P> T;
      uint32_t pst = FINISH;
      if (valid) {
        pst = start_playout<P, JOK, CONS, MODE>(T, ps, pcb, pmeta, pa, kp);
        if (pst == FINISH) {                    // decided by the root action alone
          record<MODE>(sm, kp, P, pa, ps, outcome<P, PATH>(T, pst, kp));
          valid = false;
        }
      }
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, valid);
      if (valid) ring.template put<PATH>((head + count + __popc(m & lt_mask)) & (kRing - 1u), T, pst, pa, ps, pcb);
      count += __popc(m);
      __syncwarp();
    }
    // ---- two decision steps for every running lane per loop iteration, the
    // second nested in the first (a lane that finishes in the first idles
    // through the second): the ballot / pop / produce checks are paid once
    // per two steps.  DESIGN.md §M: +4.2% C2, +2.4% C4, +6% 2p jokers over one
    // step; two flat `if (active)` blocks measured +2.8%, three steps 0%,
    // four -2% (round 1).  Round 2: three steps in the two-player jokerless
    // consecutive kernel (+0.2..2.2% on C2 deals), not elsewhere.
    if (active) {
      st = step_block<P, JOK, CONS, MODE, DVC_LUT_KIND(P, JOK, CONS)>(S, st, philox_rk(s, c1, kp), c1 & 63u, sm.meta, sm.path, a, kp,
                                          kp.path_len);
      ++c1;
      if constexpr (P == 2 && (!JOK || (DVC_REC1_2J && CONS))) {
        // one record site per iteration: a lane that finishes in the first
        // step skips the second and records after it (one divergent region
        // instead of two): +0.6% on C2, +0.4% on C3; 2p jokers consecutive = 0
        // -0.5%, 3-4 players -0.1% (§M)
        bool fin = st == FINISH || (PATH && st == VOID);   // VOID exists in path batches only
        if (!fin) {
          st = step_block<P, JOK, CONS, MODE, DVC_LUT_KIND(P, JOK, CONS)>(S, st, philox_rk(s, c1, kp), c1 & 63u, sm.meta, sm.path, a, kp,
                                              kp.path_len);
          ++c1;
          fin = st == FINISH || (PATH && st == VOID);
          // consecutive rules (longer turns): a third step nested in the
          // second, +0.2% on c2_d1, +1.1..2.2% on five other C2 deals, -3.8%
          // on the 4-action endgame c2_d8; consecutive = 0 -5% (§M)
          if (DVC_STEPS3 && CONS && !JOK && !fin) {
            st = step_block<P, JOK, CONS, MODE, DVC_LUT_KIND(P, JOK, CONS)>(S, st, philox_rk(s, c1, kp), c1 & 63u, sm.meta, sm.path, a, kp,
                                                kp.path_len);
            ++c1;
            fin = st == FINISH || (PATH && st == VOID);
          }
        }
        if (fin) {
          record<MODE>(sm, kp, P, a, s, outcome<P, PATH>(S, st, kp));
          active = false;
        }
      } else {
        if (st == FINISH || (PATH && st == VOID)) {
          record<MODE>(sm, kp, P, a, s, outcome<P, PATH>(S, st, kp));
          active = false;
        }
        if (active) {
          st = step_block<P, JOK, CONS, MODE, DVC_LUT_KIND(P, JOK, CONS)>(S, st, philox_rk(s, c1, kp), c1 & 63u, sm.meta, sm.path, a, kp,
                                              kp.path_len);
          ++c1;
          if (st == FINISH || (PATH && st == VOID)) {
            record<MODE>(sm, kp, P, a, s, outcome<P, PATH>(S, st, kp));
            active = false;
          }
        }
      }
    }
    // ---- lanes without a playout pop started ones (in the same iteration)
    const uint32_t need = __ballot_sync(0xFFFFFFFFu, !active);
    if (need) {
      const uint32_t take = min((uint32_t)__popc(need), count);
      if (take) {
        const uint32_t rank = __popc(need & lt_mask);
        if (!active && rank < take) {
          ring.template get<PATH>((head + rank) & (kRing - 1u), S, st, a, s, c1);
          active = true;
        }
        head = (head + take) & (kRing - 1u);
        count -= take;
        __syncwarp();
      }
      if (take == (uint32_t)__popc(need)) continue;        // every lane busy again
      if (count == 0 && drained && cs >= ce && !__any_sync(0xFFFFFFFFu, active)) break;
    }
  }
  flush_hist(sm.hist, kp, P);
  // The last block out re-arms the work counter (counter[0]) and its exit
  // count (counter[1]) for the launch that reuses this slot, so no launch
  // needs a memset first.  Every block stopped claiming before it counts out.
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(kp.counter + 1, 1u) == gridDim.x - 1u) {
      atomicExch(kp.counter, 0u);
      atomicExch(kp.counter + 1, 0u);
    }
  }
}

__global__ void det_table_kernel(const uint8_t *__restrict__ plan, uint64_t N, uint4 *__restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += stride)
    out[r] = unrank(plan, r);
}

__global__ void add_u64_kernel(unsigned long long *p, uint32_t n, unsigned long long v) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] += v;
}

// ---- device-resident flat search -------------------------------------------
// The UCB1 loop of dvc_mcts_search (flat = 1) after the root expansion batch,
// run on the GPU as ONE cooperative kernel instead of one blocking host round
// trip per iteration.  Per iteration every block selects the
// same child redundantly from its shared-memory copy of (visits, wins) --
// UCB1 in IEEE double with no contraction (__d*_rn), ln(N) from the host's
// libm table, so the choice is bit-identical to the host loop -- then the grid
// plays sims [visits, visits + n) of that child, one playout per lane, adds
// the viewer's wins into delta[it], and a grid barrier publishes the sum.
__device__ __forceinline__ bool ucb_better(double v, uint32_t code, uint32_t i, double bv, uint32_t bcode,
                                           uint32_t bi) {
  if (i == 0xFFFFFFFFu) return false;
  if (bi == 0xFFFFFFFFu) return true;
  return v > bv || (v == bv && code < bcode);
}

template <int P, bool JOK, bool CONS, bool INF>
__global__ void __launch_bounds__(128) flat_search_kernel(const __grid_constant__ KParams kp,
                                                          const __grid_constant__ SearchArgs sa) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ unsigned long long shs[];
  unsigned long long *vis = shs, *win = shs + kp.A;
  __shared__ double red_v[4];
  __shared__ uint32_t red_i[4], s_best;
  for (uint32_t a = threadIdx.x; a < kp.A; a += blockDim.x) {
    const int32_t bp = sa.batch_pos[a];
    vis[a] = bp >= 0 ? sa.n : 0ull;
    win[a] = bp >= 0 ? sa.first_hist[(size_t)bp * P + kp.g0] : 0ull;
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x, gsize = gridDim.x * blockDim.x;
  for (uint32_t it = 0; it < sa.iters; ++it) {
    // ---- selection (every block, same result)
    const double lnN = sa.lnN[it];
    double bv = 0.0;
    uint32_t bi = 0xFFFFFFFFu, bcode = 0;
    for (uint32_t a = threadIdx.x; a < kp.A; a += blockDim.x) {
      const double v = vis[a] == 0 ? (double)INFINITY
                     : __dadd_rn(__ddiv_rn((double)win[a], (double)vis[a]),
                                 __dmul_rn(sa.c, __dsqrt_rn(__ddiv_rn(lnN, (double)vis[a]))));
      if (ucb_better(v, kp.codes[a], a, bv, bcode, bi)) { bv = v; bi = a; bcode = kp.codes[a]; }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const double ov = __shfl_down_sync(0xFFFFFFFFu, bv, off);
      const uint32_t oi = __shfl_down_sync(0xFFFFFFFFu, bi, off);
      const uint32_t oc = __shfl_down_sync(0xFFFFFFFFu, bcode, off);
      if (ucb_better(ov, oc, oi, bv, bcode, bi)) { bv = ov; bi = oi; bcode = oc; }
    }
    if (lane == 0) { red_v[wid] = bv; red_i[wid] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (uint32_t w = 1; w < (blockDim.x >> 5); ++w) {
        const uint32_t oi = red_i[w];
        if (oi != 0xFFFFFFFFu && ucb_better(red_v[w], kp.codes[oi], oi, bv, bcode, bi)) {
          bv = red_v[w]; bi = oi; bcode = kp.codes[oi];
        }
      }
      s_best = bi;
    }
    __syncthreads();
    const uint32_t best = s_best;
    const uint32_t cb = ctr_base(kp.codes[best], kp.node), meta = kp.meta[best];
    const uint32_t sbase = (uint32_t)vis[best];
    // ---- simulation: sims [visits, visits + n) of the chosen child
    uint32_t cnt = 0;
    for (uint32_t i = gtid; i < sa.n; i += gsize) {
      const uint32_t s = sbase + i;
      Sim<P> S;
      constexpr int MODE = INF ? kModeInformed : kModePlain;
      uint32_t st = start_playout<P, JOK, CONS, MODE>(S, s, cb, meta, best, kp);
      // latency-bound loop: B_{k+1} is independent of the state, so it is
      // generated while step k runs
      uint2 B = philox_rk(s, cb, kp);
      for (uint32_t k = 0; st != FINISH; ++k) {
        const uint2 Bn = philox_rk(s, cb | (k + 1u), kp);
        st = step_block<P, JOK, CONS, MODE>(S, st, B, k, nullptr, nullptr, 0, kp, 0u);
        B = Bn;
      }
      cnt += winner_seat(S) == kp.g0 ? 1u : 0u;
    }
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    if (lane == 0 && cnt) atomicAdd(sa.delta + it, (unsigned long long)cnt);
    // ---- backpropagation, published by the grid barrier
    grid.sync();
    if (threadIdx.x == 0) {
      vis[best] += sa.n;
      win[best] += __ldcg(sa.delta + it);
    }
    __syncthreads();
  }
  if (blockIdx.x == 0)
    for (uint32_t a = threadIdx.x; a < kp.A; a += blockDim.x) {
      sa.out[a] = vis[a];
      sa.out[kp.A + a] = win[a];
    }
}

template <int P, bool JOK, bool CONS>
const void *search_fn(bool inf) {
  return inf ? (const void *)flat_search_kernel<P, JOK, CONS, true> : (const void *)flat_search_kernel<P, JOK, CONS, false>;
}

const void *select_search(int P, bool jok, bool cons, bool inf) {
#define DVC_SCASE(PP)                                                                            \
  if (P == PP) {                                                                                 \
    if (jok) return cons ? search_fn<PP, true, true>(inf) : search_fn<PP, true, false>(inf);    \
    return cons ? search_fn<PP, false, true>(inf) : search_fn<PP, false, false>(inf);           \
  }
  DVC_SCASE(2)
  DVC_SCASE(3)
  DVC_SCASE(4)
#undef DVC_SCASE
  return nullptr;
}

cudaError_t search_occupancy(int P, bool jok, bool cons, bool inf, int block, size_t smem, int *blocks_per_sm) {
  const void *f = select_search(P, jok, cons, inf);
  if (!f) return cudaErrorInvalidValue;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, block, smem);
}

cudaError_t launch_flat_search(const KParams &kp, const SearchArgs &sa, int P, bool jok, bool cons, bool inf,
                               int grid, int block, size_t smem, cudaStream_t stream) {
  const void *f = select_search(P, jok, cons, inf);
  if (!f) return cudaErrorInvalidValue;
  void *args[] = {(void *)&kp, (void *)&sa};
  return cudaLaunchCooperativeKernel(f, grid, block, args, smem, stream);
}

// ---- device-resident depth-capped tree search ----------------------------
// dvc_mcts_search(flat = 0) with search_device = 1: the tree
// lives in global memory and ONE cooperative kernel runs every iteration.
// Block 0's warp 0 is the controller -- backpropagation of the last batch,
// UCB1 descent (lanes score children, warp argmax; ln by ln_series_dev),
// expansion, the next batch descriptor -- and the whole grid plays the batch
// (F = path + [child], Philox keyed by the child's code and the batch node
// word, exactly as dvc_rollout_path_ex) between two grid barriers.
__device__ __forceinline__ double ln_series_dev(unsigned long long N) {
  int e = 0;
  double m = frexp((double)N, &e);
  if (m < 0.7071067811865476) {
    m = __dmul_rn(m, 2.0);
    e -= 1;
  }
  const double z = __ddiv_rn(__dsub_rn(m, 1.0), __dadd_rn(m, 1.0));
  const double z2 = __dmul_rn(z, z);
  // Horner over the correctly rounded constants 1/(2k+1) (folded at compile time)
  double p = 1.0 / 27.0;
#pragma unroll
  for (int k = 12; k >= 0; --k) p = __dadd_rn(__dmul_rn(p, z2), 1.0 / (double)(2 * k + 1));
  return __dadd_rn(__dmul_rn(2.0, __dmul_rn(z, p)), __dmul_rn((double)e, 0.6931471805599453));
}

__device__ __forceinline__ double ucb1_dev(unsigned long long w, unsigned long long v, double lnN, double c) {
  return __dadd_rn(__ddiv_rn((double)w, (double)v), __dmul_rn(c, __dsqrt_rn(__ddiv_rn(lnN, (double)v))));
}

// Controller step, run by ALL threads of block 0 (block-uniform control flow,
// __syncthreads between phases): backprop (thread 0), UCB1 descent (warp 0),
// expansion / batch descriptor (thread 0), new children + zeroed counters (all).
__device__ void control_step(const DeepArgs &da, uint32_t it) {
  const uint32_t tid = threadIdx.x, lane = tid & 31u;
  DNode *T = da.nodes;
  DBatch *B = da.batch;
  const uint32_t n = da.n;
  __shared__ int32_t s_x;
  __shared__ uint32_t s_stop;
  __shared__ unsigned long long s_dv, s_dw;
  // ---- backpropagation of the batch that just ran: the evaluated nodes in
  // parallel, their sums to the ancestors by thread 0
  if (it > 0) {
    if (tid == 0) { s_dv = 0; s_dw = 0; }
    __syncthreads();
    const uint32_t nb = B->nb;
    const int32_t e0 = B->eval0;
    unsigned long long dv = 0, dw = 0;
    for (uint32_t i = tid; i < nb; i += blockDim.x) {
      DNode &e = T[e0 + (int32_t)i];
      const unsigned long long vo = __ldcg(da.voids + i), wi = __ldcg(da.wins + i);
      e.tried += n;
      e.visits += n - vo;
      e.wins += wi;
      dv += n - vo;
      dw += wi;
    }
    if (dv) atomicAdd(&s_dv, dv);
    if (dw) atomicAdd(&s_dw, dw);
    __syncthreads();
    if (tid == 0)
      for (int32_t y = T[e0].parent; y >= 0; y = T[y].parent) {
        T[y].visits += s_dv;
        T[y].wins += s_dw;
      }
  }
  if (tid == 0) s_stop = it >= da.expansions ? 1u : 0u;
  __syncthreads();
  if (s_stop) {
    if (tid == 0) B->stop = 1u;
    __threadfence();
    return;                                          // block-uniform
  }
  // ---- selection (warp 0): UCB1 descent, tried-but-never-non-void children skipped
  if (tid < 32) {
    int32_t x = 0;
    for (int guard = 0; T[x].expanded && guard <= kMaxPath + 1; ++guard) {
      const double lnN = ln_series_dev(T[x].visits);
      double bv = 0.0;
      uint32_t bi = 0xFFFFFFFFu, bcode = 0;
      for (int32_t i = (int32_t)lane; i < T[x].nch; i += 32) {
        const DNode &ch = T[T[x].first + i];
        if (ch.tried > 0 && ch.visits == 0) continue;
        const double v = ch.tried == 0 ? (double)INFINITY : ucb1_dev(ch.wins, ch.visits, lnN, da.c);
        if (ucb_better(v, ch.code, (uint32_t)i, bv, bcode, bi)) { bv = v; bi = (uint32_t)i; bcode = ch.code; }
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        const double ov = __shfl_xor_sync(0xFFFFFFFFu, bv, off);
        const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, bi, off);
        const uint32_t oc = __shfl_xor_sync(0xFFFFFFFFu, bcode, off);
        if (ucb_better(ov, oc, oi, bv, bcode, bi)) { bv = ov; bi = oi; bcode = oc; }
      }
      if (bi == 0xFFFFFFFFu) break;
      x = T[x].first + (int32_t)bi;
    }
    if (tid == 0) s_x = x;
  }
  __syncthreads();
  const int32_t x = s_x;
  // ---- expansion or re-simulation: the batch descriptor (thread 0)
  if (tid == 0) {
    DNode &X = T[x];
    uint32_t pm[kMaxPath + 1];
    uint32_t depth = 0;
    for (int32_t y = x; y > 0 && depth <= kMaxPath; y = T[y].parent) pm[depth++] = T[y].meta;   // reversed
    const bool expand = !X.expanded && X.depth < (int32_t)da.max_depth && (x == 0 || X.visits > 0);
    uint32_t stop = 0u;
    if (expand) {
      const bool root = x == 0;
      const uint32_t A = root ? da.A_r : da.A_d;
      const int32_t first = (int32_t)da.n_nodes[0];
      if ((uint32_t)first + A > da.max_nodes) {
        stop = 1u;
        *da.status = DVC_E_CAPACITY;
      } else {
        X.first = first;
        X.nch = (int32_t)A;
        X.expanded = 1u;
        da.n_nodes[0] = (uint32_t)first + A;
        B->nb = A;
        B->eval0 = first;
        B->node_word = (uint32_t)x;
        B->plen = depth;
        for (uint32_t i = 0; i < depth; ++i) B->path_meta[i] = pm[depth - 1 - i];
        B->list = root ? 0u : 1u;
      }
    } else if (x == 0) {
      stop = 1u;                                     // nothing left to do
    } else {
      B->nb = 1;
      B->eval0 = x;
      B->node_word = (uint32_t)X.parent;
      B->plen = depth - 1;
      for (uint32_t i = 0; i + 1 < depth; ++i) B->path_meta[i] = pm[depth - 1 - i];
      B->list = 2u;
      B->leaf_code = X.code;
      B->leaf_meta = X.meta;
    }
    if (!stop) {
      const unsigned long long s0 = expand ? 0ull : X.tried;     // new children start at sim 0
      if (s0 + n > (1ull << 32)) {
        stop = 1u;
        *da.status = DVC_E_CONFIG;
      }
      B->s0 = (uint32_t)s0;
    }
    B->stop = stop;
    s_stop = stop;
  }
  __syncthreads();
  if (s_stop) {
    __threadfence();
    return;                                          // block-uniform
  }
  // ---- new children (all threads) and zeroed per-batch counters
  const uint32_t nb = B->nb;
  if (B->list != 2u) {
    const bool root = B->list == 0u;
    const uint32_t *codes = root ? da.root_codes : da.deep_codes;
    const uint32_t *metas = root ? da.root_meta : da.deep_meta;
    const int32_t first = B->eval0;
    const int32_t cdepth = T[x].depth + 1;
    for (uint32_t i = tid; i < nb; i += blockDim.x) {
      DNode &c = T[first + (int32_t)i];
      c.visits = 0; c.wins = 0; c.tried = 0;
      c.code = codes[i]; c.meta = metas[i];
      c.parent = x; c.depth = cdepth; c.first = -1; c.nch = 0; c.expanded = 0u;
    }
  }
  for (uint32_t i = tid; i < nb; i += blockDim.x) { da.wins[i] = 0; da.voids[i] = 0; }
  __threadfence();
  __syncthreads();
}

constexpr int32_t kWatchdogBarrier = 101, kWatchdogPlayout = 102;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Grid barrier with a watchdog (cooperative launch => all blocks resident):
// returns false (and records `code` in *status) if the other blocks do not
// arrive within about a minute, so a logic error ends the kernel with an
// error instead of hanging the device.
__device__ bool grid_barrier(unsigned int *bar, int32_t *status, int32_t code) {
  __shared__ int s_ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    s_ok = 1;
    volatile unsigned int *gen = bar + 1;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1u) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      const long long t0 = clock64();
      while (*gen == g) {
        if (clock64() - t0 > 120000000000ll) { atomicCAS(status, 0, code); s_ok = 0; break; }   // ~1 min
      }
    }
    __threadfence();
  }
  __syncthreads();
  return s_ok != 0;
}

template <int P, bool JOK, bool CONS>
__global__ void __launch_bounds__(128) deep_search_kernel(const __grid_constant__ KParams kp,
                                                          const __grid_constant__ DeepArgs da) {
  extern __shared__ uint32_t shd[];
  uint32_t *swin = shd, *svoid = shd + da.max_batch;
  __shared__ uint32_t s_path[kMaxPath];
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x, gsize = gridDim.x * blockDim.x;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    DNode &r = da.nodes[0];
    r.visits = 0; r.wins = 0; r.tried = 0; r.code = 0; r.meta = 0;
    r.parent = -1; r.depth = 0; r.first = -1; r.nch = 0; r.expanded = 0u;
    da.n_nodes[0] = 1u;
    *da.status = 0;
  }
  unsigned long long t_mark = 0;
  for (uint32_t it = 0;; ++it) {
    if (da.prof && blockIdx.x == 0 && threadIdx.x == 0) t_mark = globaltimer_ns();
    if (blockIdx.x == 0) control_step(da, it);
    if (da.prof && blockIdx.x == 0 && threadIdx.x == 0) { const auto t = globaltimer_ns(); da.prof[0] += t - t_mark; t_mark = t; }
    if (!grid_barrier(da.bar, da.status, kWatchdogBarrier)) return;
    if (da.prof && blockIdx.x == 0 && threadIdx.x == 0) { const auto t = globaltimer_ns(); da.prof[1] += t - t_mark; t_mark = t; }
    const DBatch *B = da.batch;
    if (__ldcg(&B->stop)) break;
    // ---- the batch: nb actions x n sims, F = path + [action]
    const uint32_t nb = __ldcg(&B->nb), plen = __ldcg(&B->plen), list = __ldcg(&B->list);
    const uint32_t node = __ldcg(&B->node_word), s0 = __ldcg(&B->s0);
    const uint32_t K = stream_key(kp.seed_lo, kp.seed_hi, node);   // the batch node's stream key (§R3)
    for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) { swin[i] = 0; svoid[i] = 0; }
    if (threadIdx.x < kMaxPath) s_path[threadIdx.x] = __ldcg(&B->path_meta[threadIdx.x]);
    __syncthreads();
    const uint32_t *codes = list == 0u ? da.root_codes : da.deep_codes;
    const uint32_t *metas = list == 0u ? da.root_meta : da.deep_meta;
    const uint32_t lcode = __ldcg(&B->leaf_code), lmeta = __ldcg(&B->leaf_meta);
    const uint32_t total = nb * da.n;
    for (uint32_t w = gtid; w < total; w += gsize) {
      const uint32_t a = w / da.n, s = s0 + (w - a * da.n);
      const uint32_t code = list == 2u ? lcode : codes[a], meta = list == 2u ? lmeta : metas[a];
      Sim<P> S;
      const uint32_t cb = ctr_base(code, node);
      determinize<P>(S, philox2x32_10(s, cb | kDetStep, K), kp);
      uint32_t t;
      bool correct;
      const bool stop = root_action<P, JOK>(S, plen ? s_path[0] : meta, kp, &t, &correct);
      S.fi = 1;
      uint32_t st = stop ? END_TURN : resolve<P, JOK, CONS>(S, t, correct, kp);
      const uint32_t meta_a[1] = {meta};
      for (uint32_t k = 0; st != FINISH && st != VOID; ++k) {
        st = step_block<P, JOK, CONS, kModePath>(S, st, philox2x32_10(s, cb | k, K), k, meta_a, s_path, 0u,
                                                  kp, plen);
        if (k > 4096u) { atomicCAS(da.status, 0, kWatchdogPlayout); st = VOID; }   // never expected
      }
      if (st == VOID || S.fi <= plen) atomicAdd(&svoid[a], 1u);
      else if (winner_seat(S) == kp.g0) atomicAdd(&swin[a], 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) {
      if (swin[i]) atomicAdd(da.wins + i, (unsigned long long)swin[i]);
      if (svoid[i]) atomicAdd(da.voids + i, (unsigned long long)svoid[i]);
    }
    if (da.prof && blockIdx.x == 0 && threadIdx.x == 0) { const auto t = globaltimer_ns(); da.prof[2] += t - t_mark; t_mark = t; }
    if (!grid_barrier(da.bar, da.status, kWatchdogBarrier)) return;
    if (da.prof && blockIdx.x == 0 && threadIdx.x == 0) { const auto t = globaltimer_ns(); da.prof[3] += t - t_mark; da.prof[4] += 1; }
  }
  if (blockIdx.x == 0) {
    // root children (created in LEGAL order by the first expansion)
    const DNode &r = da.nodes[0];
    for (uint32_t i = threadIdx.x; i < da.A_r; i += blockDim.x) {
      const bool has = r.expanded && (int32_t)i < r.nch;
      da.out[i] = has ? da.nodes[r.first + (int32_t)i].visits : 0ull;
      da.out[da.A_r + i] = has ? da.nodes[r.first + (int32_t)i].wins : 0ull;
    }
  }
}

template <int P, bool JOK, bool CONS>
const void *deep_fn() { return (const void *)deep_search_kernel<P, JOK, CONS>; }

const void *select_deep(int P, bool jok, bool cons) {
#define DVC_DCASE(PP)                                                                   \
  if (P == PP) {                                                                        \
    if (jok) return cons ? deep_fn<PP, true, true>() : deep_fn<PP, true, false>();     \
    return cons ? deep_fn<PP, false, true>() : deep_fn<PP, false, false>();            \
  }
  DVC_DCASE(2)
  DVC_DCASE(3)
  DVC_DCASE(4)
#undef DVC_DCASE
  return nullptr;
}

cudaError_t deep_occupancy(int P, bool jok, bool cons, int block, size_t smem, int *blocks_per_sm) {
  const void *f = select_deep(P, jok, cons);
  if (!f) return cudaErrorInvalidValue;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, block, smem);
}

cudaError_t launch_deep_search(const KParams &kp, const DeepArgs &da, int P, bool jok, bool cons, int grid,
                               int block, size_t smem, cudaStream_t stream) {
  const void *f = select_deep(P, jok, cons);
  if (!f) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  void *args[] = {(void *)&kp, (void *)&da};
  return cudaLaunchCooperativeKernel(f, grid, block, args, smem, stream);
}

// ----------------------------------------------------------------- launchers
cudaError_t launch_add_u64(unsigned long long *p, uint32_t n, uint64_t v, cudaStream_t stream) {
  add_u64_kernel<<<(n + 255) / 256, 256, 0, stream>>>(p, n, v);
  return cudaGetLastError();
}

typedef void (*KernelFn)(const KParams);

template <int P, bool JOK, bool CONS, int MODE>
KernelFn pick_mode(int variant) {
  return variant == 1 ? rollout_naive_kernel<P, JOK, CONS, MODE> : rollout_refill_kernel<P, JOK, CONS, MODE>;
}

template <int P, bool JOK, bool CONS>
KernelFn pick_kernel(int variant, int mode) {
  if (mode == kModePath) return pick_mode<P, JOK, CONS, kModePath>(variant);
  if (mode == kModeInformed) return pick_mode<P, JOK, CONS, kModeInformed>(variant);
  if (mode == kModeTrace) return pick_mode<P, JOK, CONS, kModeTrace>(variant);
  return pick_mode<P, JOK, CONS, kModePlain>(variant);
}

KernelFn select_kernel(int P, bool jok, bool cons, int variant, int mode) {
#define DVC_CASE(PP)                                                                                 \
  if (P == PP) {                                                                                     \
    if (jok) return cons ? pick_kernel<PP, true, true>(variant, mode) : pick_kernel<PP, true, false>(variant, mode); \
    return cons ? pick_kernel<PP, false, true>(variant, mode) : pick_kernel<PP, false, false>(variant, mode);       \
  }
  DVC_CASE(2)
  DVC_CASE(3)
  DVC_CASE(4)
#undef DVC_CASE
  return nullptr;
}

cudaError_t kernel_occupancy(int P, bool jok, bool cons, int variant, int mode, int block, size_t smem,
                             int *blocks_per_sm) {
  KernelFn f = select_kernel(P, jok, cons, variant, mode);
  if (!f) return cudaErrorInvalidValue;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, (const void *)f, block, smem);
}

cudaError_t launch_rollout(const KParams &kp, int P, bool jok, bool cons, int variant, int mode, int grid, int block,
                           size_t smem, cudaStream_t stream) {
  KernelFn f = select_kernel(P, jok, cons, variant, mode);
  if (!f) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  f<<<grid, block, smem, stream>>>(kp);
  return cudaGetLastError();
}

cudaError_t launch_table(const uint8_t *plan, uint64_t N, uint4 *out, cudaStream_t stream) {
  const int block = 256;
  uint64_t want = (N + block - 1) / block;
  int grid = (int)(want < 148ull * 16 ? want : 148ull * 16);
  if (grid < 1) grid = 1;
  det_table_kernel<<<grid, block, 0, stream>>>(plan, N, out);
  return cudaGetLastError();
}

}  // namespace dvc
