/*
 * dvc.h -- C-ABI of libdvc.so: batched Da Vinci Code MCTS rollouts on B200.
 *
 * The hot path of arXiv 2403.10720 (BASELINE.json north_star):
 * for every candidate action at an expanded node, n independent playouts run
 * to terminal.  Each playout samples a determinization of the opponents'
 * hidden tiles, applies the action, plays uniformly random
 * decisions (rules PAPER:102-106, variant PAPER:153) and its winner
 * is added to integer per-action counts.  The normative
 * reading of every rule, the RNG contract and the determinization order are in
 * DESIGN.md §R (= SURVEY.md §8(c)).
 *
 * Conventions (all entry points):
 *  - Status: 0 = DVC_OK; a negative DVC_E_* on failure, with a message in
 *    dvc_last_error() (thread-local).  A failing call leaves its outputs
 *    untouched.
 *  - Ownership: the caller owns every buffer passed in.  The library never
 *    hands out memory; its per-device scratch (work counters, determinization
 *    plans and tables, action arrays) is created lazily and freed by
 *    dvc_shutdown().
 *  - Host vs device pointers: every pointer is a HOST pointer except the
 *    d_* arguments of dvc_rollout_batch_async, which are DEVICE pointers on
 *    `device`.
 *  - Determinism: outputs are a pure function of (state, action code, seed,
 *    node_id, sim range); they do not depend on the action-list order, the
 *    device, the grid/block size, the kernel variant or how the sim range is
 *    split.
 *  - No CPU fallback: if no CUDA device is usable, rollout entry points fail
 *    with DVC_E_CUDA.
 */
#ifndef DVC_H_
#define DVC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DVC_OK = 0,
  DVC_E_CONFIG = -1,       /* bad rules / params                     */
  DVC_E_PROTOCOL = -2,     /* not at AwaitGuess / terminal state    */
  DVC_E_ILLEGAL = -3,      /* an action not in LEGAL(viewer) (+STOP) */
  DVC_E_INCONSISTENT = -4, /* no consistent determinization / bad tiles  */
  DVC_E_CAPACITY = -5,     /* caller buffer too small                              */
  DVC_E_CUDA = -6          /* CUDA error or no device                              */
};

/* Rules (SPEC:49-53 plus `ranks` for tiny tests).  players 2..4, ranks 1..12,
 * jokers / consecutive in {0,1}.  consecutive = 1: a correct guess extends the
 * turn (north_star); 0: the paper's simplification. */
typedef struct { int32_t players, ranks, jokers, consecutive; } dvc_rules;

/* One tile as the viewer sees it.  color 0 = Black, 1 = White.  value = rank
 * 0..ranks-1, DVC_JOKER, or DVC_HIDDEN (opponents' hidden tiles only).
 * revealed = 1 if the tile has been revealed to everybody. */
#define DVC_JOKER 0xFE
#define DVC_HIDDEN 0xFF
typedef struct { uint8_t color, value, revealed, _pad; } dvc_tile_obs;

/* The viewer's information set at AwaitGuess (SPEC:63-68 shape + SURVEY §8(b)).
 * Lines are seat-indexed and left to right; the viewer's own line is fully
 * valued.  pending = index in the viewer's line of the tile drawn this turn,
 * -1 if the pool was empty at turn start.  correct_this_turn >= 1 makes STOP
 * legal at the root (consecutive rules only). */
typedef struct {
  dvc_rules rules;
  int32_t viewer;
  int32_t line_len[4];
  dvc_tile_obs line[4][26];
  int32_t pool_size, pending, correct_this_turn;
} dvc_observation;

/* Immutable, pointer-free POD (memcpy/broadcast safe): ranks can build it
 * independently or ship it byte-for-byte. */
typedef struct { uint64_t opaque[128]; } dvc_state;

/* Validate an observation and encode it.  Checks, in
 * order: DVC_E_CONFIG (rules ranges); DVC_E_INCONSISTENT (every tile valid and
 * at most once, own + revealed + hidden opponent slots + pool_size = |T|, the
 * viewer's numbered tiles ascending, each opponent's revealed numbered tiles
 * ascending, N = |Det(O)| >= 1); DVC_E_PROTOCOL (pool_size > 0 => pending >= 0,
 * pending indexes a hidden viewer tile, correct_this_turn >= 1 => consecutive,
 * viewer and at least one opponent alive). */
int dvc_state_encode(const dvc_observation *obs, dvc_state *out);

/* Facts about an encoded state.  n_det = N = |Det(O)|. */
typedef struct {
  int32_t players, ranks, jokers, consecutive, viewer, pool_size;
  int32_t n_legal;          /* |LEGAL(viewer)| + (STOP allowed ? 1 : 0) */
  int32_t _pad;
  uint64_t n_det;
} dvc_state_info;
int dvc_state_query(const dvc_state *s, dvc_state_info *info);

/* The root's legal action codes in LEGAL order (opponents in
 * seat order after the viewer, hidden positions left to right, values of the
 * slot's colour ascending, joker last), then STOP (0xFFFFFFFF) when allowed.
 * Code = target<<24 | position<<16 | value_key (key = 2*rank+colour; jokers
 * 2R (black) and 2R+1 (white)).  DVC_E_CAPACITY (and *n_out set) if cap is
 * too small. */
#define DVC_STOP 0xFFFFFFFFu
int dvc_legal_actions(const dvc_state *s, uint32_t *codes, int32_t cap, int32_t *n_out);

/* Root batch, blocking (node_id 0, sims [0, n_sims)): wins[a] = number of the
 * n_sims playouts of actions[a] won by the viewer.  n_sims in [1, 2^32);
 * any illegal action fails the whole call (DVC_E_ILLEGAL). */
int dvc_rollout_batch(const dvc_state *s, const uint32_t *actions, int32_t n_actions,
                      uint64_t n_sims, uint64_t seed, uint64_t *wins);

/* General blocking form: hist[a*P + w] = #playouts of actions[a] with sim index
 * in [sim_begin, sim_end) won by seat w (HOST array, overwritten);
 * visits[a] = sim_end - sim_begin (HOST, may be NULL).  sim_end <= 2^32,
 * sim_begin < sim_end.  device = CUDA ordinal (-1 = current). */
int dvc_rollout_batch_ex(const dvc_state *s, const uint32_t *actions, int32_t n_actions,
                         uint64_t seed, uint32_t node_id, uint64_t sim_begin, uint64_t sim_end,
                         uint64_t *hist, uint64_t *visits, int32_t device);

/* Deep-tree batch (PAPER:143-170 guess-keyed tree with a
 * depth threshold): each playout of actions[a] first applies the viewer's
 * forced actions F = (path[0], ..., path[path_len-1], actions[a]) -- path[0]
 * as the root action, F[i] at the viewer's i-th later decision (draws and
 * opponents' decisions stay random) -- then plays randomly to the end.  A
 * playout whose forced action is illegal in its state, or whose game ends
 * before all of F is applied, is VOID: counted in voids[a] (HOST, may be NULL),
 * not in hist.  path[0] must be legal at the root; later codes only
 * well-formed.  path_len 0..8 (0 = dvc_rollout_batch_ex).  Keys, sims and
 * node_id as dvc_rollout_batch_ex. */
int dvc_rollout_path_ex(const dvc_state *s, const uint32_t *path, int32_t path_len, const uint32_t *actions,
                        int32_t n_actions, uint64_t seed, uint32_t node_id, uint64_t sim_begin, uint64_t sim_end,
                        uint64_t *hist, uint64_t *voids, int32_t device);

/* Asynchronous form: ADDS the counts into the DEVICE arrays d_hist[A*P] (and
 * d_visits[A] if non-NULL) on `cuda_stream` (a cudaStream_t, NULL = legacy
 * default stream) of `device`; returns after enqueueing.  The caller zeroes
 * d_hist when it wants fresh counts.  Host-side state (plan, action arrays) is
 * staged before return, so the caller may reuse its host buffers at once. */
int dvc_rollout_batch_async(const dvc_state *s, const uint32_t *actions, int32_t n_actions,
                            uint64_t seed, uint32_t node_id, uint64_t sim_begin, uint64_t sim_end,
                            uint64_t *d_hist, uint64_t *d_visits, int32_t device, void *cuda_stream);

/* Batch variants, selected by `flags` (other bits ->
 * DVC_E_CONFIG); otherwise as dvc_rollout_batch_ex (hist HOST, overwritten)
 * and dvc_rollout_batch_async (d_hist DEVICE, added to on cuda_stream):
 *  DVC_FLAG_CRN       common random numbers across actions:
 *                     the determinization block of sim s is D = Philox(ctr =
 *                     (0xFFFFFFFF, s, 0xFFFFFFFE, node_id)) for EVERY action,
 *                     so all actions play against the same hidden-tile
 *                     assignment for each sim index (the decision blocks B_t
 *                     stay keyed by the action code); each action's counts
 *                     keep their distribution, differences get less variance.
 *  DVC_FLAG_INFORMED  order-aware playout policy: every
 *                     playout decision is uniform over the guesses whose value
 *                     lies strictly between the nearest revealed numbered
 *                     tiles left and right of the slot (joker values always
 *                     kept), LEGAL order, STOP last.  Root actions: any LEGAL.
 * Both flags may be combined.  Not available for deep-tree (path) batches. */
#define DVC_FLAG_CRN 1u
#define DVC_FLAG_INFORMED 2u
int dvc_rollout_batch_flags_ex(const dvc_state *s, const uint32_t *actions, int32_t n_actions, uint64_t seed,
                               uint32_t node_id, uint64_t sim_begin, uint64_t sim_end, uint32_t flags,
                               uint64_t *hist, int32_t device);
int dvc_rollout_batch_flags_async(const dvc_state *s, const uint32_t *actions, int32_t n_actions, uint64_t seed,
                                  uint32_t node_id, uint64_t sim_begin, uint64_t sim_end, uint32_t flags,
                                  uint64_t *d_hist, int32_t device, void *cuda_stream);

/* The "md" ablation ("nodes are enriched with
 * information regarding the chosen set of numbers", the vanilla tree PAPER:145
 * discards): child a = (determinization rhos[a], action actions[a]).  Every
 * playout of child a plays the rhos[a]-th element of Det(O) in canonical order
 * (§R4) instead of sampling one; the rest is dvc_rollout_batch_ex (blocking,
 * HOST hist[A*P]; actions may repeat with different rhos).  Errors:
 * DVC_E_CONFIG when rhos is null or some rhos[a] >= N (dvc_state_query's
 * n_det), plus every error of dvc_rollout_batch_ex. */
int dvc_rollout_batch_fixed_ex(const dvc_state *s, const uint32_t *actions, const uint64_t *rhos,
                               int32_t n_actions, uint64_t seed, uint32_t node_id, uint64_t sim_begin,
                               uint64_t sim_end, uint64_t *hist, int32_t device);

/* SPEC:230 sample_determinization: rhos_out[i] = the element of Det(O)
 * (canonical order) that sim s_begin + i of a CRN batch
 * (DVC_FLAG_CRN, seed, node_id) plays, i.e. rank64(N, D) for D the Philox2x32
 * determinization block of that sim under the CRN word (§R3), i = 0..k-1
 * (duplicates possible).  Host-side, no device work.  Errors: DVC_E_CONFIG
 * for a bad state, k < 0, a null buffer or s_begin + k > 2^32. */
int dvc_sample_determinizations(const dvc_state *s, uint64_t seed, uint32_t node_id, uint32_t s_begin, int32_t k,
                                uint64_t *rhos_out);

/* Debug/parity form of the async call: additionally writes the winner seat of
 * every playout to d_winners[a*(sim_end-sim_begin) + (s - sim_begin)] (DEVICE,
 * uint8).  Same kernels and launch configuration as the async call. */
int dvc_rollout_trace_async(const dvc_state *s, const uint32_t *actions, int32_t n_actions,
                            uint64_t seed, uint32_t node_id, uint64_t sim_begin, uint64_t sim_end,
                            uint64_t *d_hist, uint8_t *d_winners, int32_t device, void *cuda_stream);

/* Launch options (process-wide; they never change results):
 *  "kernel"      0 = persistent warp-refill kernel, 1 = naive
 *                thread-per-playout kernel (the paper-style comparison),
 *                2 = auto (default): naive when all of a call's playouts fit in one
 *                resident wave of naive threads (latency-bound small batches: C1
 *                decisions, search batches), refill otherwise; out of range ->
 *                DVC_E_CONFIG
 *  "block"       threads per block (1..1024 for the naive kernel; a multiple of
 *                32 up to 256 for the refill kernel; default 128)
 *  "grid"        blocks (0 = auto: resident blocks per SM x #SM, or fewer when
 *                the launch has less work than that)
 *  "table_cap"   max determinization-table entries (0 = always unrank inline)
 *  "chunk"       max work items (actions x sims) per kernel launch (1..2^31,
 *                default 2^31; larger ranges are split into several launches)
 *  "plan_cache"  1 = reuse a state's plan + table across calls (default);
 *                0 = re-upload the plan and rebuild the table on every call
 *  "search_device" 0 = dvc_mcts_search keeps UCT selection and backprop on
 *                the host tree, one blocking rollout batch per iteration
 *                (default; BASELINE.json north_star); 1 = the whole search
 *                runs in one cooperative GPU kernel per decision -- flat:
 *                the UCB1 iterations after the root expansion (DESIGN.md
 *                §R8); depth-capped: the tree lives in device memory (§R9).
 *                Same selections, same counts; lower single-search latency,
 *                but a search holds the GPU, so concurrent searches serialise
 * Returns DVC_E_CONFIG for an unknown name or a bad value. */
int dvc_set_option(const char *name, int64_t value);
int dvc_get_option(const char *name, int64_t *value);

/* Host MCTS over the GPU rollout batches (
 * PAPER:112-117 four MCTS steps, PAPER:179-186 root-parallel mini-trees).
 * flat = 1 (the paper's implementation, "expands a child node from
 * the root, with subsequent gameplay unfolding randomly"): the root's children
 * are the legal actions; each of `expansions` iterations selects ONE child by
 * UCB1 (c, IEEE double: wins/visits + c*sqrt(ln(N)/visits), unvisited first,
 * ties to the smallest code) and runs `sims_per_child` playouts
 * of it (node 0, sims [visits, visits + n) of that child, so no playout is
 * ever repeated), then backpropagates visits and the viewer's wins.
 * flat = 0: the depth-capped tree over the viewer's guesses (DESIGN.md §R9,
 * PAPER:143-170; max_depth 1..8): UCB1 descent, expansion of the selected
 * leaf with ALL its children in one GPU batch (dvc_rollout_path_ex, node_id =
 * the parent's creation index), re-simulation of leaves at max_depth, void
 * playouts not counted, backpropagation to the root; `expansions` iterations.
 * table[i] receives every root child in LEGAL order
 * (cap >= n_legal, else DVC_E_CAPACITY); *best_code = most visits, then most
 * wins, then smallest code. */
typedef struct {
  double c;                 /* UCB1 exploration constant (sqrt(2)) */
  int32_t max_depth;        /* expansion depth threshold (4)       */
  int32_t expansions;       /* UCB iterations                                 */
  uint64_t sims_per_child;  /* playouts per iteration                         */
  uint64_t seed;            /* Philox seed of every batch                     */
  int32_t flat;             /* 1 = root-only tree                             */
  int32_t device;           /* CUDA ordinal, -1 = current                     */
  uint32_t flags;           /* DVC_FLAG_* for every batch (flat = 1 only)     */
  uint32_t _pad;
} dvc_search_params;
typedef struct { uint32_t code, _pad; uint64_t visits, wins; } dvc_action_stat;
int dvc_mcts_search(const dvc_state *s, const dvc_search_params *p, dvc_action_stat *table, int32_t cap,
                    int32_t *n_out, uint32_t *best_code);

/* The same search with every rollout batch delegated to a caller callback --
 * root parallelism over ranks (SURVEY §8(e) "the tree replicated on
 * every rank"): each rank runs this search; its callback plays the rank's
 * shard of [sim_begin, sim_end) and sums the counts over ranks (dist.py:
 * all_reduce), so every rank sees identical counts and makes identical UCT
 * choices.  The UCB1 arithmetic (ln_series, reading #28) and the move choice
 * stay in this library; the callback only produces counts.
 *   fn(ctx, path, path_len, actions, n_actions, seed, node_id, sim_begin,
 *      sim_end, flags, hist, voids) must write into the zeroed HOST arrays
 *   hist[n_actions * P] (winner histogram) and, when voids != NULL (deep-tree
 *   batches: path_len >= 1), voids[n_actions], exactly what
 *   dvc_rollout_path_ex / dvc_rollout_batch_flags_ex would return for the
 *   whole range, and return 0 (or a DVC_E_* code, which aborts the search
 *   with that code).  path == NULL for flat batches.  search_device is
 *   ignored (the tree stays on the host).  fn == NULL -> DVC_E_CONFIG; other
 *   errors as dvc_mcts_search. */
typedef int (*dvc_batch_fn)(void *ctx, const uint32_t *path, int32_t path_len, const uint32_t *actions,
                            int32_t n_actions, uint64_t seed, uint32_t node_id, uint64_t sim_begin,
                            uint64_t sim_end, uint32_t flags, uint64_t *hist, uint64_t *voids);
int dvc_mcts_search_cb(const dvc_state *s, const dvc_search_params *p, dvc_batch_fn fn, void *ctx,
                       dvc_action_stat *table, int32_t cap, int32_t *n_out, uint32_t *best_code);

/* The "md" ablation search (PAPER:143 vanilla tree, discarded
 * PAPER:145): flat UCT over children (rho_i, a) -- n_det candidate
 * determinizations x LEGAL.  rho_i: all of Det(O) when N <= n_det, else the
 * first n_det distinct values of dvc_sample_determinizations(seed, node 0,
 * sims 0, 1, ...) (at most 64 n_det samples are drawn).  Child j = i*A + a.
 * The first min(expansions, n_det*A) iterations visit the unvisited children
 * in index order (one batch per rho_i, node_id = 1 + i, sims [0, n)); later
 * iterations select the max UCB1 child (unvisited first, ties -> smallest j)
 * and run sims [visits, visits + n) of it (node_id = 1 + i).  table[a] = the
 * per-action sums over rho_i of visits and viewer wins in LEGAL order;
 * *best_code = most visits, then most wins, then smallest code;
 * *n_det_out = the number of candidate determinizations used. */
typedef struct {
  double c;                 /* UCB1 exploration constant                      */
  int32_t n_det;            /* candidate determinizations (1..4096)           */
  int32_t expansions;       /* UCB iterations                                 */
  uint64_t sims_per_child;  /* playouts per iteration                         */
  uint64_t seed;            /* Philox seed of every batch and of the rho_i    */
  int32_t device;           /* CUDA ordinal, -1 = current                     */
  uint32_t _pad;
} dvc_md_params;
int dvc_md_search(const dvc_state *s, const dvc_md_params *p, dvc_action_stat *table, int32_t cap,
                  int32_t *n_out, uint32_t *best_code, int32_t *n_det_out);

/* Debug build only (libdvc_debug.so, compiled with -DDVC_DEBUG): out3 =
 * {invariant violations, code of the first one, finished playouts checked}
 * accumulated on `device` since its scratch was created (codes: 1 hands/pool
 * not disjoint, 2 tiles not conserved, 3 a pool tile revealed, 4 bad joker
 * threshold, 5 mover dead, 6 too many decisions, 7 not exactly one reveal per
 * guess, 8 STOP without a correct guess, 9 not exactly one survivor, 10 a pending
 * (drawn this turn) tile already revealed, 11 a histogram write out of bounds,
 * 12 a determinization-table read out of bounds, 13 a trace write out of
 * bounds).  The
 * release library returns DVC_E_CONFIG. */
int dvc_debug_counters(int32_t device, uint32_t *out3);

/* Number of kernel launches the library enqueued since the last reset
 * (reset = 1 zeroes it); lets callers count GPU launches in a timed region. */
uint64_t dvc_launch_count(int32_t reset);

/* Bytes the library moved since the last reset (reset = 1 zeroes both after
 * reading): *h2d = host -> device copies (determinization plan images, md
 * rho lists, search tables) plus the parameter block of every kernel launch
 * (the rollout kernel's KParams: codes, metas, round keys); *d2h = device ->
 * host copies (histograms of the blocking calls, search results).  Copies the
 * CALLER makes of its own device buffers (the *_async forms) are not counted.
 * Either pointer may be NULL.  Always DVC_OK. */
int dvc_transfer_bytes(int32_t reset, uint64_t *h2d, uint64_t *d2h);

const char *dvc_last_error(void);
void dvc_shutdown(void);

#ifdef __cplusplus
}
#endif
#endif /* DVC_H_ */
