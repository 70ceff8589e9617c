// dvc_internal.h -- product-internal layouts shared by the host encoder
// (host.cpp), the C-ABI (api.cu) and the kernels (rollout.cu).  Nothing here
// is shared with oracle/ (the two implementations are independent).
//
// Bitmask representation: a set of tiles is a u32 over keys
// (key = 2*rank + colour; jokers 2R and 2R+1), so colour masks
// are the even / odd bits and "ascending key order" is bit order.
#pragma once
#include <stdint.h>
#include <vector>
#include "../../include/dvc.h"

#ifndef __CUDACC__
#define __host__
#define __device__
#endif

namespace dvc {

constexpr uint32_t kMagic = 0x31435644u;  // "DVC1"
constexpr uint32_t kEven = 0x55555555u;   // black keys (incl. JB = 2R)
constexpr uint32_t kOdd = 0xAAAAAAAAu;    // white keys (incl. JW = 2R+1)
constexpr uint32_t kNoKey = 31u;          // "NONE" for pend
constexpr uint8_t kHiddenSlot = 0x80u;    // line[][] entry flag: hidden, low bit = colour
constexpr int kMaxPath = 8;               // deep-tree batches: forced viewer actions before the batch action

// Host jinfo word (plan options): jslot(JB) in bits [0,5), jslot(JW) in [5,10),
// bit 10 = JW precedes JB when both sit in one line (only read when their
// jslots are equal).  The device converts jslots to threshold keys when it
// unranks a determinization (rollout.cuh: kap_b / kap_w).
__host__ __device__ inline uint32_t jslot_b(uint32_t ji) { return ji & 31u; }
__host__ __device__ inline uint32_t jslot_w(uint32_t ji) { return (ji >> 5) & 31u; }

// The encoded root (lives inside dvc_state.opaque; plain data, no pointers).
struct State {
  uint32_t magic;
  int32_t P, R, jokers, consecutive;
  int32_t viewer, pool_size, pend_key, corr;
  uint32_t T;          // tile-set mask
  uint32_t V;          // revealed keys (any line)
  uint32_t U;          // unaccounted keys (not the viewer's, not revealed)
  uint32_t known[4];   // seat -> keys the viewer knows that seat holds
  int32_t line_len[4];
  uint8_t line[4][26];    // key, or kHiddenSlot|colour
  uint64_t N;             // |Det(O)|
  int32_t n_legal;        // incl. STOP
  uint32_t hash_lo, hash_hi;  // FNV-1a of the bytes above (plan cache key)
};
static_assert(sizeof(State) <= sizeof(dvc_state), "State must fit dvc_state");

// ---- determinization plan (DESIGN.md §R4 / §K2), one flat device image ----
struct DetOpt {            // one joint joker option (o_JB major, o_JW minor)
  uint64_t count;          // # numbered completions under this option
  uint32_t tab_off;        // u64 offset of this option's N(i, q) table
  uint32_t n_states;       // prod(len_j + 1)
  uint32_t jinfo;          // jslots of every held joker at the root, jw_first
  uint32_t jmask[3];       // jokers this option puts in opponent d = 1..3
  uint32_t stride[3];      // linear-state stride of q_j
  uint32_t len[3];         // chain length (remaining hidden non-joker slots)
  uint32_t slot_off[3];    // offset into slots[] (packed c | lo<<8 | hi<<16)
};

struct DetPlanHdr {
  uint32_t n_opts, m, n_opp, bytes;
  uint32_t viewer_hand;    // the viewer's tiles (jokers' thresholds need the holder's hand)
  uint32_t jb;             // 2R when jokers are on, else 0
  uint32_t _pad2[2];
  uint32_t ukeys[28];      // numbered keys of U ascending
  uint32_t opp_known[4];   // keys revealed in opponent d's line (d = 1..3 at [d-1])
  uint32_t opts_off, slots_off, tab_off, _pad;  // byte offsets in the image
  uint64_t N;
};

// Action as the kernel reads it: d (relative target seat, 0 = STOP) | pos<<8 | v<<16
__host__ __device__ inline uint32_t act_meta(uint32_t d, uint32_t pos, uint32_t v) {
  return d | (pos << 8) | (v << 16);
}

// ---- error reporting (api.cu): sets dvc_last_error(), returns code ----
int set_error(int code, const char *msg);
// ln N for UCB1 (mcts.cpp; DESIGN.md §R8 reading #28).
double ln_series(uint64_t N);
// Device flat search (api.cu): option "search_device", and the call itself.
bool search_on_device();
int deep_search_gpu(const dvc_state *s, const dvc_search_params *p, const uint32_t *root_codes, int32_t A_r,
                    const uint32_t *deep_codes, int32_t A_d, uint64_t *visits, uint64_t *wins);
int flat_search_gpu(const dvc_state *s, const uint32_t *codes, int32_t A, const uint32_t *first, int32_t k,
                    const int32_t *batch_pos, const double *lnN, int32_t iters, const dvc_search_params *p,
                    uint64_t *visits, uint64_t *wins);

// ---- host functions (host.cpp) ----
int encode(const dvc_observation *obs, State *st, const char **err);
int legal_actions(const State &st, uint32_t *codes, int32_t cap, int32_t *n_out);
// validates codes against LEGAL; fills meta[] for the kernel
int decode_actions(const State &st, const uint32_t *codes, int32_t n, uint32_t *meta,
                   const char **err);
// structural validation of deep-tree path / batch codes (legality is per playout)
int decode_deep(const State &st, const uint32_t *codes, int32_t n, uint32_t *meta, const char **err);
// builds the plan image into `img` (resized); returns N
uint64_t build_plan(const State &st, std::vector<uint8_t> *img);

}  // namespace dvc
