// api.cu -- the C-ABI of include/dvc.h: argument checks,
// per-device scratch (work counters, determinization plan + table cache keyed
// by the state hash), sim-range chunking (<= 2^31 work items per launch so
// the kernels' u32 counters cannot overflow) and kernel launches.  Every step
// of the path runs in kernels.cu; this file only marshals.
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <list>
#include <mutex>
#include <thread>
#include <string>
#include <unordered_map>
#include <vector>

#include "dvc_internal.h"
#include "rollout.cuh"

namespace dvc {
cudaError_t launch_rollout(const KParams &kp, int P, bool jok, bool cons, int variant, int mode, int grid, int block,
                           size_t smem, cudaStream_t stream);
cudaError_t launch_table(const uint8_t *plan, uint64_t N, uint4 *out, cudaStream_t stream);
constexpr size_t kTableArgBytes = sizeof(const uint8_t *) + sizeof(uint64_t) + sizeof(uint4 *);   // det_table_kernel params
cudaError_t launch_add_u64(unsigned long long *p, uint32_t n, uint64_t v, cudaStream_t stream);
cudaError_t kernel_occupancy(int P, bool jok, bool cons, int variant, int mode, int block, size_t smem,
                             int *blocks_per_sm);
cudaError_t search_occupancy(int P, bool jok, bool cons, bool inf, int block, size_t smem, int *blocks_per_sm);
cudaError_t deep_occupancy(int P, bool jok, bool cons, int block, size_t smem, int *blocks_per_sm);
cudaError_t launch_deep_search(const KParams &kp, const DeepArgs &da, int P, bool jok, bool cons, int grid,
                               int block, size_t smem, cudaStream_t stream);
cudaError_t launch_flat_search(const KParams &kp, const SearchArgs &sa, int P, bool jok, bool cons, bool inf,
                               int grid, int block, size_t smem, cudaStream_t stream);

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_kernel{2}, g_block{128}, g_grid{0}, g_table_cap{1ll << 26}, g_plan_cache{1},
    g_chunk{1ll << 31}, g_search_device{0};
std::atomic<uint64_t> g_launches{0};
// bytes the library moved host -> device (copies + kernel parameter blocks)
// and device -> host since the last dvc_transfer_bytes(reset = 1)
std::atomic<uint64_t> g_h2d{0}, g_d2h{0};

int set_err(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

struct PlanEntry {
  uint64_t hash;
  uint8_t *d_plan = nullptr;
  size_t plan_cap = 0;
  uint4 *d_table = nullptr;   // null if N > table_cap when built
  size_t table_cap = 0;
  uint64_t N = 0;
  cudaEvent_t ready = nullptr;  // recorded after plan upload + table build
  // the last launch reading this plan on each stream: an evicted plan's
  // buffers are reused only once all of these have completed
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;
  std::vector<uint8_t> host_img;
};

constexpr int kCounterSlots = 4096;
constexpr size_t kPlanCacheMax = 16;

// Stream + device histogram used by the BLOCKING entry points of one host
// thread, so threads (e.g. concurrent self-play games) overlap on the GPU.
struct HostLane {
  cudaStream_t stream = nullptr;
  unsigned long long *d_hist = nullptr;
  unsigned long long *h_hist = nullptr;  // pinned staging for the blocking calls' read-back
  size_t hist_cap = 0;
  unsigned char *d_search = nullptr;     // device flat search: lnN, delta, out, batch_pos
  size_t search_cap = 0;
  unsigned long long *d_rho = nullptr;   // md ablation batches: per-action determinization (kMaxActions)
  unsigned long long *h_rho = nullptr;   // pinned staging for its upload
};

struct DeviceScratch {
  int device = -1;
  int num_sms = 0;
  uint32_t *d_counters = nullptr;
  uint32_t next_counter = 0;
  // per work-counter slot: the event recorded after the last launch that used
  // it; a launch taking the slot waits on it, so launches on different streams
  // never share a live slot (> kCounterSlots launches in flight)
  std::vector<cudaEvent_t> counter_ev;
  uint32_t *d_debug = nullptr;           // DVC_DEBUG builds: invariant counters
  std::unordered_map<std::thread::id, HostLane> lanes;
  std::list<PlanEntry> plans;            // LRU, front = most recent
  std::list<PlanEntry> zombies;          // evicted, possibly still read by in-flight launches
  std::vector<std::pair<void *, size_t>> pool;   // reclaimed device buffers (best fit)
  std::vector<cudaEvent_t> events;       // reclaimed events
  std::unordered_map<uint64_t, int> occupancy;   // resident blocks per SM per launch shape
};

std::mutex g_mu;
std::unordered_map<int, DeviceScratch *> g_dev;

// Public entry points select their device (get_scratch -> cudaSetDevice);
// this restores the caller's current device on return, so a call on device k
// never changes which device the caller (e.g. torch) is on.
struct DeviceRestore {
  int prev = -1;
  DeviceRestore() { if (cudaGetDevice(&prev) != cudaSuccess) { prev = -1; cudaGetLastError(); } }
  ~DeviceRestore() { if (prev >= 0) cudaSetDevice(prev); }
};

int cuda_fail(cudaError_t e, const char *where) {
  return set_err(DVC_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

int get_scratch(int device, DeviceScratch **out) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return set_err(DVC_E_CUDA, "no CUDA device available (no CPU fallback)");
  if (device < 0) {
    e = cudaGetDevice(&device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  }
  if (device >= ndev) return set_err(DVC_E_CONFIG, "device ordinal out of range");
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  auto it = g_dev.find(device);
  if (it != g_dev.end()) { *out = it->second; return DVC_OK; }
  DeviceScratch *d = new DeviceScratch();
  d->device = device;
  e = cudaDeviceGetAttribute(&d->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) { delete d; return cuda_fail(e, "cudaDeviceGetAttribute"); }
  // slot i = (work counter, exit count) at d_counters[2i]; zero once here, the
  // refill kernel re-arms its slot on exit (kernels.cu)
  e = cudaMalloc(&d->d_counters, 2 * kCounterSlots * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(d->d_counters, 0, 2 * kCounterSlots * sizeof(uint32_t));
  if (e != cudaSuccess) { delete d; return cuda_fail(e, "cudaMalloc(counters)"); }
#ifdef DVC_DEBUG
  e = cudaMalloc(&d->d_debug, 4 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(d->d_debug, 0, 4 * sizeof(uint32_t));
  if (e != cudaSuccess) { delete d; return cuda_fail(e, "cudaMalloc(debug)"); }
#endif
  g_dev[device] = d;
  *out = d;
  return DVC_OK;
}

// The calling thread's lane on device d with a histogram of >= n counters
// (caller holds g_mu).
int get_lane(DeviceScratch *d, size_t n, HostLane **out) {
  HostLane &L = d->lanes[std::this_thread::get_id()];
  if (!L.stream) {
    cudaError_t e = cudaStreamCreateWithFlags(&L.stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) { L.stream = nullptr; return cuda_fail(e, "cudaStreamCreate"); }
  }
  if (L.hist_cap < n) {
    if (L.d_hist) cudaFree(L.d_hist);
    if (L.h_hist) cudaFreeHost(L.h_hist);
    L.d_hist = nullptr;
    L.h_hist = nullptr;
    L.hist_cap = 0;
    cudaError_t e = cudaMalloc(&L.d_hist, n * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMallocHost(&L.h_hist, n * sizeof(unsigned long long));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(hist)");
    L.hist_cap = n;
  }
  *out = &L;
  return DVC_OK;
}

// ---- plan memory: pooled device buffers and events, reclaimed by completion
// events instead of a device-wide synchronisation (concurrent host threads'
// launches keep running while a plan is evicted).
constexpr size_t kPoolMaxBytes = 512ull << 20;
constexpr size_t kZombieMax = 8;

void *pool_get(DeviceScratch *d, size_t bytes, size_t *cap, cudaError_t *err) {
  size_t bi = d->pool.size();
  for (size_t i = 0; i < d->pool.size(); ++i) {
    const size_t c = d->pool[i].second;
    if (c >= bytes && c <= 4 * bytes + 4096 && (bi == d->pool.size() || c < d->pool[bi].second)) bi = i;
  }
  if (bi < d->pool.size()) {
    void *p = d->pool[bi].first;
    *cap = d->pool[bi].second;
    d->pool.erase(d->pool.begin() + (long)bi);
    *err = cudaSuccess;
    return p;
  }
  void *p = nullptr;
  *err = cudaMalloc(&p, bytes);
  *cap = bytes;
  return *err == cudaSuccess ? p : nullptr;
}

void pool_put(DeviceScratch *d, void *p, size_t cap) {
  if (!p) return;
  d->pool.push_back({p, cap});
  size_t total = 0;
  for (auto &b : d->pool) total += b.second;
  while (total > kPoolMaxBytes && !d->pool.empty()) {
    size_t li = 0;
    for (size_t i = 1; i < d->pool.size(); ++i) if (d->pool[i].second > d->pool[li].second) li = i;
    total -= d->pool[li].second;
    cudaFree(d->pool[li].first);
    d->pool.erase(d->pool.begin() + (long)li);
  }
}

cudaError_t event_get(DeviceScratch *d, cudaEvent_t *ev) {
  if (!d->events.empty()) {
    *ev = d->events.back();
    d->events.pop_back();
    return cudaSuccess;
  }
  return cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
}

bool plan_idle(const PlanEntry &p) {
  if (p.ready && cudaEventQuery(p.ready) == cudaErrorNotReady) return false;
  for (auto &u : p.uses)
    if (cudaEventQuery(u.second) == cudaErrorNotReady) return false;
  return true;
}

void reclaim(DeviceScratch *d, PlanEntry &p) {
  pool_put(d, p.d_plan, p.plan_cap);
  pool_put(d, p.d_table, p.table_cap);
  if (p.ready) d->events.push_back(p.ready);
  for (auto &u : p.uses) d->events.push_back(u.second);
  p.d_plan = nullptr; p.d_table = nullptr; p.ready = nullptr;
  p.uses.clear();
}

// Reclaim evicted plans whose launches have finished; past kZombieMax, wait
// for the oldest one's own events (not the whole device).
void reap(DeviceScratch *d) {
  for (auto it = d->zombies.begin(); it != d->zombies.end();) {
    if (plan_idle(*it)) { reclaim(d, *it); it = d->zombies.erase(it); } else { ++it; }
  }
  while (d->zombies.size() > kZombieMax) {
    PlanEntry &p = d->zombies.back();
    if (p.ready) cudaEventSynchronize(p.ready);
    for (auto &u : p.uses) cudaEventSynchronize(u.second);
    reclaim(d, p);
    d->zombies.pop_back();
  }
}

// Record that a launch just enqueued on `stream` reads plan p (caller holds g_mu).
int note_use(DeviceScratch *d, PlanEntry *p, cudaStream_t stream) {
  for (auto &u : p->uses)
    if (u.first == stream) {
      cudaError_t e = cudaEventRecord(u.second, stream);
      return e == cudaSuccess ? DVC_OK : cuda_fail(e, "cudaEventRecord(use)");
    }
  cudaEvent_t ev;
  cudaError_t e = event_get(d, &ev);
  if (e == cudaSuccess) e = cudaEventRecord(ev, stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord(use)");
  p->uses.push_back({stream, ev});
  return DVC_OK;
}

void free_plan_now(PlanEntry &p) {                 // shutdown only (device already synchronised)
  if (p.d_plan) cudaFree(p.d_plan);
  if (p.d_table) cudaFree(p.d_table);
  if (p.ready) cudaEventDestroy(p.ready);
  for (auto &u : p.uses) cudaEventDestroy(u.second);
  p.d_plan = nullptr; p.d_table = nullptr; p.ready = nullptr;
  p.uses.clear();
}

// Plan (+ table) for this state on this device; built on `stream` on first use,
// other streams wait on its event.
int get_plan(DeviceScratch *d, const State &st, cudaStream_t stream, PlanEntry **out) {
  const uint64_t h = ((uint64_t)st.hash_hi << 32) | st.hash_lo;
  const uint64_t cap = (uint64_t)g_table_cap.load();
  for (auto it = d->plans.begin(); it != d->plans.end(); ++it) {
    if (it->hash == h && ((it->d_table != nullptr) == (it->N <= cap))) {
      d->plans.splice(d->plans.begin(), d->plans, it);
      PlanEntry &p = d->plans.front();
      cudaError_t e = cudaStreamWaitEvent(stream, p.ready, 0);
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent");
      if (!g_plan_cache.load()) {
        // recompute per call (no cross-call reuse): plan upload + table build,
        // after every launch that still reads the old contents
        for (auto &u : p.uses)
          if (u.first != stream && (e = cudaStreamWaitEvent(stream, u.second, 0)) != cudaSuccess)
            return cuda_fail(e, "cudaStreamWaitEvent(use)");
        e = cudaMemcpyAsync(p.d_plan, p.host_img.data(), p.host_img.size(), cudaMemcpyHostToDevice, stream);
        g_h2d += p.host_img.size();
        if (e == cudaSuccess && p.d_table) {
          e = launch_table(p.d_plan, p.N, p.d_table, stream);
          g_launches++;
          g_h2d += kTableArgBytes;
        }
        if (e == cudaSuccess) e = cudaEventRecord(p.ready, stream);
        if (e != cudaSuccess) return cuda_fail(e, "plan rebuild");
      }
      *out = &p;
      return DVC_OK;
    }
  }
  reap(d);
  PlanEntry p;
  p.hash = h;
  p.N = build_plan(st, &p.host_img);
  if (p.N != st.N) return set_err(DVC_E_INCONSISTENT, "determinization count changed (corrupt state?)");
  cudaError_t e;
  p.d_plan = static_cast<uint8_t *>(pool_get(d, p.host_img.size(), &p.plan_cap, &e));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(plan)");
  e = cudaMemcpyAsync(p.d_plan, p.host_img.data(), p.host_img.size(), cudaMemcpyHostToDevice, stream);
  g_h2d += p.host_img.size();
  if (e != cudaSuccess) { reclaim(d, p); return cuda_fail(e, "cudaMemcpyAsync(plan)"); }
  if (p.N <= cap) {
    p.d_table = static_cast<uint4 *>(pool_get(d, p.N * sizeof(uint4), &p.table_cap, &e));
    if (e != cudaSuccess) { reclaim(d, p); return cuda_fail(e, "cudaMalloc(table)"); }
    e = launch_table(p.d_plan, p.N, p.d_table, stream);
    g_launches++;
    g_h2d += kTableArgBytes;
    if (e != cudaSuccess) { reclaim(d, p); return cuda_fail(e, "det_table_kernel"); }
  }
  e = event_get(d, &p.ready);
  if (e == cudaSuccess) e = cudaEventRecord(p.ready, stream);
  if (e != cudaSuccess) { reclaim(d, p); return cuda_fail(e, "cudaEventRecord"); }
  d->plans.push_front(std::move(p));
  while (d->plans.size() > kPlanCacheMax) {
    // evicted plans may still be read by launches on other host threads'
    // streams: they wait in `zombies` until their use events complete
    d->zombies.splice(d->zombies.begin(), d->plans, std::prev(d->plans.end()));
  }
  *out = &d->plans.front();
  return DVC_OK;
}

const State *as_state(const dvc_state *s) {
  const State *st = reinterpret_cast<const State *>(s);
  return st->magic == kMagic ? st : nullptr;
}

// Batch-invariant KParams fields: stream key K(seed, node) as Philox2x32 round
// keys (§R3), root state, plan/table.
void fill_kparams(KParams &kp, const State *st, uint64_t seed, uint32_t node_id, uint32_t n_actions,
                  const PlanEntry *plan, const DeviceScratch *d) {
  kp.seed_lo = (uint32_t)seed; kp.seed_hi = (uint32_t)(seed >> 32);
  const uint32_t K = stream_key(kp.seed_lo, kp.seed_hi, node_id);
  for (int r = 0; r < 10; ++r) kp.rk[r] = K + (uint32_t)r * kPhiloxW;
  kp.node = node_id;
  kp.A = n_actions;
  kp.g0 = (uint32_t)st->viewer;
  kp.Hv = st->known[st->viewer];
  kp.V0 = st->V;
  kp.U = st->U;
  kp.T = st->T;
  kp.numm = (1u << (2 * st->R)) - 1u;
  kp.JB = (uint32_t)(2 * st->R);
  // the tile a wrong root guess reveals: the viewer's pending drawn tile, or
  // -- nothing drawn -- its leftmost hidden tile; the viewer's
  // hidden tiles cannot change before its own wrong guess, so this is the
  // same tile the device would find at the reveal
  kp.pend0 = kNoKey;
  if (st->pend_key >= 0) {
    kp.pend0 = (uint32_t)st->pend_key;
  } else {
    for (int32_t i = 0; i < st->line_len[st->viewer]; ++i) {
      const uint32_t k = st->line[st->viewer][i];
      if (!((st->V >> k) & 1u)) { kp.pend0 = k; break; }
    }
  }
  kp.corr0 = (uint32_t)st->corr;
  kp.N = st->N;
  kp.debug = d->d_debug;
  kp.table = plan->d_table;
  kp.plan = plan->d_plan;
}

// Core enqueue: adds hist for [sim_begin, sim_end) into d_hist on stream.
// BatchOpts: a deep-tree forced path (§R9) or the root-batch flags (§R3 CRN, §R10).
struct BatchOpts {
  const uint32_t *codes = nullptr;
  int32_t len = 0;
  unsigned long long *d_voids = nullptr;
  bool crn = false;         // common random numbers across actions (root batches only)
  bool informed = false;    // informed playout policy (root batches only)
  const unsigned long long *d_rho = nullptr;   // md ablation: fixed determinization per action (§R11)
};

int enqueue(const dvc_state *s, const uint32_t *actions, int32_t n_actions, uint64_t seed, uint32_t node_id,
            uint64_t sim_begin, uint64_t sim_end, unsigned long long *d_hist, uint8_t *d_winners,
            int32_t device, cudaStream_t stream, DeviceScratch **dev_out, const BatchOpts &path = BatchOpts()) {
  const State *st = as_state(s);
  if (!st) return set_err(DVC_E_CONFIG, "state was not produced by dvc_state_encode");
  if (!actions || n_actions < 1 || n_actions > kMaxActions)
    return set_err(DVC_E_CONFIG, "n_actions must be in [1, 768]");
  if (sim_begin >= sim_end || sim_end > (1ull << 32))
    return set_err(DVC_E_CONFIG, "need sim_begin < sim_end <= 2^32");
  KParams kp;
  std::memset(&kp, 0, sizeof(kp));
  const char *err = nullptr;
  int rc;
  if (path.len > 0) {
    // deep-tree batch: F[0] = path[0] must be legal at the root; the rest of
    // the path and the batch actions are applied at later viewer decisions
    if (path.len > kMaxPath || !path.codes) return set_err(DVC_E_CONFIG, "path length must be 1..8");
    rc = decode_actions(*st, path.codes, 1, kp.path_meta, &err);
    if (rc == DVC_OK && path.len > 1) rc = decode_deep(*st, path.codes + 1, path.len - 1, kp.path_meta + 1, &err);
    if (rc == DVC_OK) rc = decode_deep(*st, actions, n_actions, kp.meta, &err);
    kp.path_len = (uint32_t)path.len;
    kp.voids = path.d_voids;
  } else {
    rc = decode_actions(*st, actions, n_actions, kp.meta, &err);
  }
  if (rc) return set_err(rc, err ? err : "illegal action");
  std::memcpy(kp.codes, actions, sizeof(uint32_t) * n_actions);

  std::lock_guard<std::mutex> lock(g_mu);
  DeviceScratch *d = nullptr;
  rc = get_scratch(device, &d);
  if (rc) return rc;
  if (dev_out) *dev_out = d;
  PlanEntry *plan = nullptr;
  rc = get_plan(d, *st, stream, &plan);
  if (rc) return rc;

  const int P = st->P;
  fill_kparams(kp, st, seed, node_id, (uint32_t)n_actions, plan, d);
  kp.hist = d_hist;
  kp.winners = d_winners;
  kp.crn = path.crn ? 1u : 0u;
  kp.rho = path.d_rho;
  kp.trace_stride = (uint32_t)(sim_end - sim_begin);
  kp.trace_s0 = (uint32_t)sim_begin;

  int variant = (int)g_kernel.load();
  const int block = (int)g_block.load();
  const int mode = kp.path_len > 0 ? kModePath
                 : path.informed  ? kModeInformed
                 : d_winners      ? kModeTrace
                                  : kModePlain;
  // hist + codes + meta (+ the refill kernel's per-warp rings of started playouts)
  auto smem_of = [&](int v) {
    if (v != 0 && v != 3) return ((size_t)n_actions * (P + 3) + kMaxPath) * sizeof(uint32_t);   // hist[A][P+1], codes, metas, path
    // + the per-warp rings: kRingSlots x ring_vecs(P) x 16 B, 16 B aligned (kernels.cu RingView)
    return (((size_t)n_actions * (P + 3) + kMaxPath + 3) & ~(size_t)3) * sizeof(uint32_t) +
           (size_t)(block / 32) * kRingSlots * ring_vecs(P) * 16;
  };
  // resident blocks per SM, cached per (kernel instance, block, smem)
  auto per_sm_of = [&](int v, size_t sm, int *out) -> int {
    const uint64_t okey = ((uint64_t)v << 60) | ((uint64_t)P << 56) | ((uint64_t)(st->jokers != 0) << 55) |
                          ((uint64_t)(st->consecutive != 0) << 54) | ((uint64_t)mode << 51) |
                          ((uint64_t)block << 32) | (uint64_t)sm;
    auto it = d->occupancy.find(okey);
    if (it != d->occupancy.end()) { *out = it->second; return DVC_OK; }
    cudaError_t e = kernel_occupancy(P, st->jokers != 0, st->consecutive != 0, v, mode, block, sm, out);
    if (e != cudaSuccess) return cuda_fail(e, "occupancy");
    d->occupancy[okey] = *out;
    return DVC_OK;
  };
  if (variant == 2) {
    // auto: a call whose playouts all fit in one resident wave of naive
    // threads is latency-bound -- one playout per thread finishes with the
    // longest playout, where refill warps that claim a second batch finish
    // later (C1: 33 us vs 51 us device span) -- anything larger takes the
    // refill kernel's throughput
    int ps = 0;
    rc = per_sm_of(1, smem_of(1), &ps);
    if (rc) return rc;
    const uint64_t total = (uint64_t)n_actions * (sim_end - sim_begin);
    variant = total <= (uint64_t)ps * (uint64_t)d->num_sms * (uint64_t)block ? 1 : 0;
  }
  const size_t smem = smem_of(variant);
  if (variant == 0 && block % 32) return set_err(DVC_E_CONFIG, "the refill kernel needs whole warps (block % 32 == 0)");
  const int grid_opt = (int)g_grid.load();
  int grid_full = grid_opt;
  if (grid_opt <= 0) {
    int per_sm = 0;
    rc = per_sm_of(variant, smem, &per_sm);
    if (rc) return rc;
    if (per_sm < 1) return set_err(DVC_E_CONFIG, "kernel cannot launch with this block size");
    grid_full = per_sm * d->num_sms;
  }
  // chunk the sim range so each launch has <= 2^31 work items
  uint64_t per_launch = (uint64_t)g_chunk.load() / (uint64_t)n_actions;
  if (per_launch < 1) per_launch = 1;
  for (uint64_t b = sim_begin; b < sim_end;) {
    const uint64_t e_ = (sim_end - b > per_launch) ? b + per_launch : sim_end;
    kp.s0 = (uint32_t)b;
    kp.n_per = (uint32_t)(e_ - b);
    kp.total = kp.n_per * kp.A;
    kp.nb = (kp.n_per + kBatch - 1u) / kBatch;   // refill work batches per action
    // ceil(2^64 / n_per) for the kernels' division-free item -> (action, sim)
    kp.div_magic = kp.n_per == 1 ? 0ull
                 : (uint64_t)(((unsigned __int128)1 << 64) / kp.n_per) + ((((unsigned __int128)1 << 64) % kp.n_per) ? 1 : 0);
    const uint32_t slot = d->next_counter++ % kCounterSlots;
    kp.counter = d->d_counters + 2 * slot;
    cudaError_t e;
    if (variant == 0) {
      if (d->counter_ev.empty()) d->counter_ev.assign(kCounterSlots, nullptr);
      cudaEvent_t &sev = d->counter_ev[slot];
      if (sev) {
        e = cudaStreamWaitEvent(stream, sev, 0);
      } else {
        e = cudaEventCreateWithFlags(&sev, cudaEventDisableTiming);
      }
      if (e != cudaSuccess) return cuda_fail(e, "work-counter slot");
    }
    // auto grid: the resident maximum, or fewer blocks for a small launch (each
    // refill warp starts 32 playouts at a time; each naive thread plays one)
    int grid = grid_full;
    if (grid_opt <= 0) {
      const uint64_t per_block = variant == 0 ? (uint64_t)(block / 32) * 32u : (uint64_t)block;
      const uint64_t need = ((uint64_t)kp.total + per_block - 1) / per_block;
      if (need < (uint64_t)grid) grid = (int)need;
    }
    e = launch_rollout(kp, P, st->jokers != 0, st->consecutive != 0, variant, mode, grid, block, smem, stream);
    g_launches++;
    g_h2d += sizeof(KParams);             // the kernel's parameter block
    if (e == cudaSuccess && variant == 0) e = cudaEventRecord(d->counter_ev[slot], stream);
    if (e != cudaSuccess) return cuda_fail(e, "rollout kernel launch");
    b = e_;
  }
  return note_use(d, plan, stream);
}

// Device-resident flat search: the root-expansion batch (the
// first k children, sims [0, n)) and then ONE cooperative flat_search_kernel
// for the remaining `iters` UCB1 iterations, all on this thread's stream with
// a single synchronisation at the end.
int flat_search_gpu_impl(const dvc_state *s, const uint32_t *codes, int32_t A, const uint32_t *first, int32_t k,
                         const int32_t *batch_pos, const double *lnN, int32_t iters, const dvc_search_params *p,
                         uint64_t *visits, uint64_t *wins) {
  const State *st = as_state(s);
  if (!st) return set_err(DVC_E_CONFIG, "bad state");
  const int P = st->P;
  const uint64_t n = p->sims_per_child;
  const size_t nh = (size_t)k * P;
  const size_t off_delta = (size_t)iters * 8, off_out = off_delta + (size_t)iters * 8,
               off_bp = off_out + (size_t)A * 16, bytes = off_bp + (size_t)A * 4;
  DeviceScratch *d = nullptr;
  HostLane *L = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    int rc = get_scratch(p->device, &d);
    if (rc) return rc;
    rc = get_lane(d, nh, &L);
    if (rc) return rc;
    if (L->search_cap < bytes) {
      if (L->d_search) cudaFree(L->d_search);
      L->d_search = nullptr;
      L->search_cap = 0;
      cudaError_t e = cudaMalloc(&L->d_search, bytes);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(search)");
      L->search_cap = bytes;
    }
    cudaError_t e = cudaMemsetAsync(L->d_hist, 0, nh * sizeof(unsigned long long), L->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(L->d_search + off_delta, 0, (size_t)iters * 8, L->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(L->d_search, lnN, (size_t)iters * 8, cudaMemcpyHostToDevice, L->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(L->d_search + off_bp, batch_pos, (size_t)A * 4, cudaMemcpyHostToDevice, L->stream);
    if (e != cudaSuccess) return cuda_fail(e, "search setup");
  }
  BatchOpts opt;
  opt.crn = (p->flags & DVC_FLAG_CRN) != 0;
  opt.informed = (p->flags & DVC_FLAG_INFORMED) != 0;
  int rc = enqueue(s, first, k, p->seed, 0u, 0, n, L->d_hist, nullptr, d->device, L->stream, nullptr, opt);
  if (rc) return rc;
  KParams kp;
  std::memset(&kp, 0, sizeof(kp));
  const char *err = nullptr;
  rc = decode_actions(*st, codes, A, kp.meta, &err);
  if (rc) return set_err(rc, err ? err : "illegal action");
  std::memcpy(kp.codes, codes, sizeof(uint32_t) * A);
  std::vector<unsigned long long> out((size_t)A * 2);
  {
    std::lock_guard<std::mutex> lock(g_mu);
    PlanEntry *plan = nullptr;
    rc = get_plan(d, *st, L->stream, &plan);
    if (rc) return rc;
    fill_kparams(kp, st, p->seed, 0u, (uint32_t)A, plan, d);
    kp.crn = opt.crn ? 1u : 0u;
    SearchArgs sa;
    sa.lnN = reinterpret_cast<const double *>(L->d_search);
    sa.delta = reinterpret_cast<unsigned long long *>(L->d_search + off_delta);
    sa.out = reinterpret_cast<unsigned long long *>(L->d_search + off_out);
    sa.batch_pos = reinterpret_cast<const int32_t *>(L->d_search + off_bp);
    sa.first_hist = L->d_hist;
    sa.c = p->c;
    sa.n = (uint32_t)n;
    sa.iters = (uint32_t)iters;
    const int block = 128;
    const size_t smem = (size_t)A * 16;
    const uint64_t okey = (3ull << 60) | ((uint64_t)P << 56) | ((uint64_t)(st->jokers != 0) << 55) |
                          ((uint64_t)(st->consecutive != 0) << 54) | ((uint64_t)opt.informed << 53) |
                          ((uint64_t)block << 32) | (uint64_t)smem;
    int per_sm = 0;
    auto it = d->occupancy.find(okey);
    if (it != d->occupancy.end()) {
      per_sm = it->second;
    } else {
      cudaError_t e = search_occupancy(P, st->jokers != 0, st->consecutive != 0, opt.informed, block, smem, &per_sm);
      if (e != cudaSuccess) return cuda_fail(e, "occupancy");
      d->occupancy[okey] = per_sm;
    }
    if (per_sm < 1) return set_err(DVC_E_CONFIG, "search kernel cannot launch");
    uint64_t grid = (n + block - 1) / block;
    if (grid > (uint64_t)per_sm * d->num_sms) grid = (uint64_t)per_sm * d->num_sms;
    cudaError_t e = launch_flat_search(kp, sa, P, st->jokers != 0, st->consecutive != 0, opt.informed, (int)grid,
                                       block, smem, L->stream);
    g_launches++;
    if (e != cudaSuccess) return cuda_fail(e, "flat_search_kernel launch");
    rc = note_use(d, plan, L->stream);
    if (rc) return rc;
    e = cudaMemcpyAsync(out.data(), sa.out, out.size() * 8, cudaMemcpyDeviceToHost, L->stream);
    if (e != cudaSuccess) return cuda_fail(e, "search readback");
  }
  cudaError_t e = cudaStreamSynchronize(L->stream);
  if (e != cudaSuccess) return cuda_fail(e, "flat search");
  for (int32_t a = 0; a < A; ++a) {
    visits[a] = out[a];
    wins[a] = out[(size_t)A + a];
  }
  return DVC_OK;
}

// Device-resident depth-capped tree search: one cooperative
// deep_search_kernel runs all `expansions` iterations; the host uploads the
// candidate lists and reads back the root children's (visits, wins).
int deep_search_gpu_impl(const dvc_state *s, const dvc_search_params *p, const uint32_t *root_codes, int32_t A_r,
                         const uint32_t *deep_codes, int32_t A_d, uint64_t *visits, uint64_t *wins) {
  const State *st = as_state(s);
  if (!st) return set_err(DVC_E_CONFIG, "bad state");
  const int P = st->P;
  std::vector<uint32_t> lists((size_t)2 * (A_r + A_d));
  const char *err = nullptr;
  int rc = decode_actions(*st, root_codes, A_r, lists.data() + A_r, &err);
  if (rc == DVC_OK && A_d > 0) rc = decode_deep(*st, deep_codes, A_d, lists.data() + 2 * A_r + A_d, &err);
  if (rc) return set_err(rc, err ? err : "illegal action");
  std::memcpy(lists.data(), root_codes, sizeof(uint32_t) * A_r);
  std::memcpy(lists.data() + 2 * A_r, deep_codes, sizeof(uint32_t) * A_d);
  const uint32_t max_batch = (uint32_t)(A_r > A_d ? A_r : A_d);
  const uint64_t max_nodes = 1 + (uint64_t)p->expansions * max_batch;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t off_nn = al(max_nodes * sizeof(DNode)), off_b = off_nn + 256, off_l = off_b + al(sizeof(DBatch)),
               off_w = off_l + al(lists.size() * 4), off_v = off_w + al(max_batch * 8),
               off_o = off_v + al(max_batch * 8), off_st = off_o + al((size_t)A_r * 16), bytes = off_st + 256;
  DeviceScratch *d = nullptr;
  HostLane *L = nullptr;
  std::vector<unsigned long long> out((size_t)2 * A_r);
  int32_t status = 0;
  // the lock covers scratch / lane / plan setup, the launch and the async
  // readbacks; the (long) synchronize below runs without it so other host
  // threads' calls proceed (the lane and its buffers belong to this thread)
  std::unique_lock<std::mutex> lock(g_mu);
  rc = get_scratch(p->device, &d);
  if (rc) return rc;
  rc = get_lane(d, 1, &L);
  if (rc) return rc;
  if (L->search_cap < bytes) {
    if (L->d_search) cudaFree(L->d_search);
    L->d_search = nullptr;
    L->search_cap = 0;
    cudaError_t e = cudaMalloc(&L->d_search, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(search)");
    L->search_cap = bytes;
  }
  unsigned char *base = L->d_search;
  cudaError_t e = cudaMemcpyAsync(base + off_l, lists.data(), lists.size() * 4, cudaMemcpyHostToDevice, L->stream);
  if (e != cudaSuccess) return cuda_fail(e, "search setup");
  PlanEntry *plan = nullptr;
  rc = get_plan(d, *st, L->stream, &plan);
  if (rc) return rc;
  KParams kp;
  std::memset(&kp, 0, sizeof(kp));
  fill_kparams(kp, st, p->seed, 0u, 0u, plan, d);
  DeepArgs da;
  da.nodes = reinterpret_cast<DNode *>(base);
  da.n_nodes = reinterpret_cast<uint32_t *>(base + off_nn);
  da.batch = reinterpret_cast<DBatch *>(base + off_b);
  const uint32_t *dl = reinterpret_cast<const uint32_t *>(base + off_l);
  da.root_codes = dl;
  da.root_meta = dl + A_r;
  da.deep_codes = dl + 2 * A_r;
  da.deep_meta = dl + 2 * A_r + A_d;
  da.wins = reinterpret_cast<unsigned long long *>(base + off_w);
  da.voids = reinterpret_cast<unsigned long long *>(base + off_v);
  da.out = reinterpret_cast<unsigned long long *>(base + off_o);
  da.status = reinterpret_cast<int32_t *>(base + off_st);
  da.bar = reinterpret_cast<unsigned int *>(base + off_st + 64);
  da.prof = std::getenv("DVC_DEEP_PROF") ? reinterpret_cast<unsigned long long *>(base + off_st + 128) : nullptr;
  e = cudaMemsetAsync(base + off_st, 0, 256, L->stream);
  if (e != cudaSuccess) return cuda_fail(e, "search setup");
  da.c = p->c;
  da.n = (uint32_t)p->sims_per_child;
  da.expansions = (uint32_t)p->expansions;
  da.max_depth = (uint32_t)p->max_depth;
  da.A_r = (uint32_t)A_r;
  da.A_d = (uint32_t)A_d;
  da.max_batch = max_batch;
  da.max_nodes = (uint32_t)max_nodes;
  const int block = 128;
  const size_t smem = (size_t)max_batch * 8;
  const uint64_t okey = (4ull << 60) | ((uint64_t)P << 56) | ((uint64_t)(st->jokers != 0) << 55) |
                        ((uint64_t)(st->consecutive != 0) << 54) | ((uint64_t)block << 32) | (uint64_t)smem;
  int per_sm = 0;
  auto it = d->occupancy.find(okey);
  if (it != d->occupancy.end()) {
    per_sm = it->second;
  } else {
    e = deep_occupancy(P, st->jokers != 0, st->consecutive != 0, block, smem, &per_sm);
    if (e != cudaSuccess) return cuda_fail(e, "occupancy");
    d->occupancy[okey] = per_sm;
  }
  if (per_sm < 1) return set_err(DVC_E_CONFIG, "deep search kernel cannot launch");
  uint64_t grid = ((uint64_t)max_batch * da.n + block - 1) / block;
  if (grid > (uint64_t)per_sm * d->num_sms) grid = (uint64_t)per_sm * d->num_sms;
  e = launch_deep_search(kp, da, P, st->jokers != 0, st->consecutive != 0, (int)grid, block, smem, L->stream);
  g_launches++;
  if (e != cudaSuccess) return cuda_fail(e, "deep_search_kernel launch");
  rc = note_use(d, plan, L->stream);
  if (rc) return rc;
  e = cudaMemcpyAsync(out.data(), da.out, out.size() * 8, cudaMemcpyDeviceToHost, L->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&status, da.status, 4, cudaMemcpyDeviceToHost, L->stream);
  lock.unlock();
  if (e == cudaSuccess) e = cudaStreamSynchronize(L->stream);
  if (e != cudaSuccess) return cuda_fail(e, "deep search");
  if (da.prof) {
    unsigned long long pr[5];
    if (cudaMemcpy(pr, da.prof, sizeof(pr), cudaMemcpyDeviceToHost) == cudaSuccess && pr[4])
      std::fprintf(stderr, "deep search per iteration (us): control %.1f barrier %.1f playouts %.1f barrier %.1f (%llu it, grid %d)\n",
                   pr[0] / 1e3 / pr[4], pr[1] / 1e3 / pr[4], pr[2] / 1e3 / pr[4], pr[3] / 1e3 / pr[4], pr[4], (int)grid);
  }
  if (status == DVC_E_CONFIG) return set_err(status, "a node's sim index range would pass 2^32");
  if (status == DVC_E_CAPACITY) return set_err(status, "deep search tree capacity");
  if (status) return set_err(DVC_E_CUDA, "deep search kernel watchdog " + std::to_string(status));
  for (int32_t a = 0; a < A_r; ++a) {
    visits[a] = out[a];
    wins[a] = out[(size_t)A_r + a];
  }
  return DVC_OK;
}

}  // namespace

int set_error(int code, const char *msg) { return set_err(code, msg ? msg : ""); }

bool search_on_device() { return g_search_device.load() != 0; }

int deep_search_gpu(const dvc_state *s, const dvc_search_params *p, const uint32_t *root_codes, int32_t A_r,
                    const uint32_t *deep_codes, int32_t A_d, uint64_t *visits, uint64_t *wins) {
  return deep_search_gpu_impl(s, p, root_codes, A_r, deep_codes, A_d, visits, wins);
}

int flat_search_gpu(const dvc_state *s, const uint32_t *codes, int32_t A, const uint32_t *first, int32_t k,
                    const int32_t *batch_pos, const double *lnN, int32_t iters, const dvc_search_params *p,
                    uint64_t *visits, uint64_t *wins) {
  return flat_search_gpu_impl(s, codes, A, first, k, batch_pos, lnN, iters, p, visits, wins);
}

}  // namespace dvc

using namespace dvc;

extern "C" {

int dvc_state_encode(const dvc_observation *obs, dvc_state *out) {
  if (!obs || !out) return set_err(DVC_E_CONFIG, "null argument");
  State st;
  const char *err = nullptr;
  int rc = encode(obs, &st, &err);
  if (rc) return set_err(rc, err ? err : "encode failed");
  std::memset(out, 0, sizeof(*out));
  std::memcpy(out, &st, sizeof(st));
  return DVC_OK;
}

int dvc_state_query(const dvc_state *s, dvc_state_info *info) {
  const State *st = s ? as_state(s) : nullptr;
  if (!st || !info) return set_err(DVC_E_CONFIG, "bad state");
  info->players = st->P; info->ranks = st->R; info->jokers = st->jokers;
  info->consecutive = st->consecutive; info->viewer = st->viewer; info->pool_size = st->pool_size;
  info->n_legal = st->n_legal; info->_pad = 0; info->n_det = st->N;
  return DVC_OK;
}

int dvc_legal_actions(const dvc_state *s, uint32_t *codes, int32_t cap, int32_t *n_out) {
  const State *st = s ? as_state(s) : nullptr;
  if (!st || !n_out || (cap > 0 && !codes)) return set_err(DVC_E_CONFIG, "bad arguments");
  int rc = legal_actions(*st, codes ? codes : nullptr, cap, n_out);
  if (rc) return set_err(rc, "capacity too small for the legal-action list");
  return DVC_OK;
}

}  // extern "C"

namespace dvc {
namespace {
int rollout_blocking(const dvc_state *s, const uint32_t *actions, int32_t n_actions, uint64_t seed,
                     uint32_t node_id, uint64_t sim_begin, uint64_t sim_end, uint64_t *hist, uint64_t *visits,
                     int32_t device, uint32_t flags, const uint64_t *rhos = nullptr) {
  if (flags & ~(uint32_t)(DVC_FLAG_CRN | DVC_FLAG_INFORMED)) return set_err(DVC_E_CONFIG, "unknown batch flag");
  if (!hist) return set_err(DVC_E_CONFIG, "hist is null");
  const State *st = s ? as_state(s) : nullptr;
  if (!st) return set_err(DVC_E_CONFIG, "bad state");
  if (n_actions < 1 || n_actions > kMaxActions) return set_err(DVC_E_CONFIG, "n_actions must be in [1, 768]");
  if (!actions) return set_err(DVC_E_CONFIG, "actions is null");
  if (sim_begin >= sim_end || sim_end > (1ull << 32))
    return set_err(DVC_E_CONFIG, "need sim_begin < sim_end <= 2^32");
  {
    // validate the action list before touching any device (errors leave outputs untouched)
    std::vector<uint32_t> meta((size_t)n_actions);
    const char *err = nullptr;
    int rc = decode_actions(*st, actions, n_actions, meta.data(), &err);
    if (rc) return set_err(rc, err ? err : "illegal action");
    if (rhos)
      for (int32_t a = 0; a < n_actions; ++a)
        if (rhos[a] >= st->N) return set_err(DVC_E_CONFIG, "rho must be < N (the determinization count)");
  }
  const size_t n = (size_t)n_actions * st->P;
  DeviceScratch *d = nullptr;
  HostLane *L = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    int rc = get_scratch(device, &d);
    if (rc) return rc;
    rc = get_lane(d, n, &L);
    if (rc) return rc;
    cudaError_t e = cudaMemsetAsync(L->d_hist, 0, n * sizeof(unsigned long long), L->stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(hist)");
    if (rhos) {
      if (!L->d_rho) {
        e = cudaMalloc(&L->d_rho, kMaxActions * sizeof(unsigned long long));
        if (e == cudaSuccess) e = cudaMallocHost(&L->h_rho, kMaxActions * sizeof(unsigned long long));
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(rho)");
      }
      // the previous call on this lane has completed (blocking calls end with a sync)
      for (int32_t a = 0; a < n_actions; ++a) L->h_rho[a] = rhos[a];
      e = cudaMemcpyAsync(L->d_rho, L->h_rho, (size_t)n_actions * sizeof(unsigned long long),
                          cudaMemcpyHostToDevice, L->stream);
      g_h2d += (size_t)n_actions * sizeof(unsigned long long);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(rho)");
    }
  }
  BatchOpts opt;
  opt.crn = (flags & DVC_FLAG_CRN) != 0;
  opt.informed = (flags & DVC_FLAG_INFORMED) != 0;
  opt.d_rho = rhos ? L->d_rho : nullptr;
  int rc = enqueue(s, actions, n_actions, seed, node_id, sim_begin, sim_end, L->d_hist, nullptr, d->device,
                   L->stream, nullptr, opt);
  if (rc) return rc;
  cudaError_t e = cudaMemcpyAsync(L->h_hist, L->d_hist, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                  L->stream);
  g_d2h += n * sizeof(unsigned long long);
  if (e == cudaSuccess) e = cudaStreamSynchronize(L->stream);
  if (e != cudaSuccess) return cuda_fail(e, "rollout");
  for (size_t i = 0; i < n; ++i) hist[i] = L->h_hist[i];
  if (visits)
    for (int a = 0; a < n_actions; ++a) visits[a] = sim_end - sim_begin;
  return DVC_OK;
}

int rollout_async(const dvc_state *s, const uint32_t *actions, int32_t n_actions, uint64_t seed,
                  uint32_t node_id, uint64_t sim_begin, uint64_t sim_end, uint64_t *d_hist, uint64_t *d_visits,
                  int32_t device, void *cuda_stream, uint32_t flags) {
  if (!d_hist) return set_err(DVC_E_CONFIG, "d_hist is null");
  if (flags & ~(uint32_t)(DVC_FLAG_CRN | DVC_FLAG_INFORMED)) return set_err(DVC_E_CONFIG, "unknown batch flag");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  BatchOpts opt;
  opt.crn = (flags & DVC_FLAG_CRN) != 0;
  opt.informed = (flags & DVC_FLAG_INFORMED) != 0;
  int rc = enqueue(s, actions, n_actions, seed, node_id, sim_begin, sim_end,
                   reinterpret_cast<unsigned long long *>(d_hist), nullptr, device, stream, nullptr, opt);
  if (rc) return rc;
  if (d_visits) {
    cudaError_t e = launch_add_u64(reinterpret_cast<unsigned long long *>(d_visits), (uint32_t)n_actions,
                                   sim_end - sim_begin, stream);
    g_launches++;
    if (e != cudaSuccess) return cuda_fail(e, "visits");
  }
  return DVC_OK;
}
}  // namespace
}  // namespace dvc

extern "C" {

int dvc_rollout_batch_ex(const dvc_state *s, const uint32_t *actions, int32_t n_actions, uint64_t seed,
                         uint32_t node_id, uint64_t sim_begin, uint64_t sim_end, uint64_t *hist,
                         uint64_t *visits, int32_t device) {
  DeviceRestore restore_device;
  return rollout_blocking(s, actions, n_actions, seed, node_id, sim_begin, sim_end, hist, visits, device, 0u);
}

int dvc_rollout_batch_flags_ex(const dvc_state *s, const uint32_t *actions, int32_t n_actions, uint64_t seed,
                               uint32_t node_id, uint64_t sim_begin, uint64_t sim_end, uint32_t flags,
                               uint64_t *hist, int32_t device) {
  DeviceRestore restore_device;
  return rollout_blocking(s, actions, n_actions, seed, node_id, sim_begin, sim_end, hist, nullptr, device, flags);
}

int dvc_sample_determinizations(const dvc_state *s, uint64_t seed, uint32_t node_id, uint32_t s_begin, int32_t k,
                                uint64_t *rhos_out) {
  DeviceRestore restore_device;
  const State *st = s ? as_state(s) : nullptr;
  if (!st) return set_err(DVC_E_CONFIG, "bad state");
  if (k < 0 || (k > 0 && !rhos_out)) return set_err(DVC_E_CONFIG, "need k >= 0 and an output buffer");
  if ((uint64_t)s_begin + (uint64_t)k > (1ull << 32)) return set_err(DVC_E_CONFIG, "sim indices are 32-bit");
  // the determinization block D of sim s under common random numbers (§R3),
  // rho = rank64(N, d0, d1): the element of Det(O) a CRN batch plays at sim s
  const uint32_t K = stream_key((uint32_t)seed, (uint32_t)(seed >> 32), node_id);
  const uint32_t c1 = ctr_base(kCrnWord, node_id) | kDetStep;
  for (int32_t i = 0; i < k; ++i) {
    const uint2 D = philox2x32_10(s_begin + (uint32_t)i, c1, K);
    const unsigned __int128 x = ((unsigned __int128)D.y << 32) | D.x;
    rhos_out[i] = (uint64_t)((x * st->N) >> 64);
  }
  return DVC_OK;
}

int dvc_rollout_batch_fixed_ex(const dvc_state *s, const uint32_t *actions, const uint64_t *rhos,
                               int32_t n_actions, uint64_t seed, uint32_t node_id, uint64_t sim_begin,
                               uint64_t sim_end, uint64_t *hist, int32_t device) {
  DeviceRestore restore_device;
  if (!rhos) return set_err(DVC_E_CONFIG, "rhos is null");
  return rollout_blocking(s, actions, n_actions, seed, node_id, sim_begin, sim_end, hist, nullptr, device, 0u, rhos);
}

int dvc_rollout_batch_flags_async(const dvc_state *s, const uint32_t *actions, int32_t n_actions, uint64_t seed,
                                  uint32_t node_id, uint64_t sim_begin, uint64_t sim_end, uint32_t flags,
                                  uint64_t *d_hist, int32_t device, void *cuda_stream) {
  DeviceRestore restore_device;
  return rollout_async(s, actions, n_actions, seed, node_id, sim_begin, sim_end, d_hist, nullptr, device,
                       cuda_stream, flags);
}

int dvc_rollout_path_ex(const dvc_state *s, const uint32_t *path, int32_t path_len, const uint32_t *actions,
                        int32_t n_actions, uint64_t seed, uint32_t node_id, uint64_t sim_begin, uint64_t sim_end,
                        uint64_t *hist, uint64_t *voids, int32_t device) {
  DeviceRestore restore_device;
  if (path_len == 0) {
    int rc = dvc_rollout_batch_ex(s, actions, n_actions, seed, node_id, sim_begin, sim_end, hist, nullptr, device);
    if (rc == DVC_OK && voids)
      for (int a = 0; a < n_actions; ++a) voids[a] = 0;
    return rc;
  }
  if (!hist || !actions || !path) return set_err(DVC_E_CONFIG, "null argument");
  const State *st = s ? as_state(s) : nullptr;
  if (!st) return set_err(DVC_E_CONFIG, "bad state");
  if (n_actions < 1 || n_actions > kMaxActions) return set_err(DVC_E_CONFIG, "n_actions must be in [1, 768]");
  if (path_len < 0 || path_len > kMaxPath) return set_err(DVC_E_CONFIG, "path length must be 0..8");
  if (sim_begin >= sim_end || sim_end > (1ull << 32)) return set_err(DVC_E_CONFIG, "need sim_begin < sim_end <= 2^32");
  {
    std::vector<uint32_t> meta((size_t)(n_actions > path_len ? n_actions : path_len));
    const char *err = nullptr;
    int rc = decode_actions(*st, path, 1, meta.data(), &err);
    if (rc == DVC_OK && path_len > 1) rc = decode_deep(*st, path + 1, path_len - 1, meta.data(), &err);
    if (rc == DVC_OK) rc = decode_deep(*st, actions, n_actions, meta.data(), &err);
    if (rc) return set_err(rc, err ? err : "illegal action");
  }
  const size_t n = (size_t)n_actions * st->P;
  DeviceScratch *d = nullptr;
  HostLane *L = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    int rc = get_scratch(device, &d);
    if (rc) return rc;
    rc = get_lane(d, n + (size_t)n_actions, &L);
    if (rc) return rc;
    cudaError_t e = cudaMemsetAsync(L->d_hist, 0, (n + n_actions) * sizeof(unsigned long long), L->stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(hist)");
  }
  BatchOpts pa;
  pa.codes = path;
  pa.len = path_len;
  pa.d_voids = L->d_hist + n;
  int rc = enqueue(s, actions, n_actions, seed, node_id, sim_begin, sim_end, L->d_hist, nullptr, d->device,
                   L->stream, nullptr, pa);
  if (rc) return rc;
  cudaError_t e = cudaMemcpyAsync(L->h_hist, L->d_hist, (n + n_actions) * sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, L->stream);
  g_d2h += (n + n_actions) * sizeof(unsigned long long);
  if (e == cudaSuccess) e = cudaStreamSynchronize(L->stream);
  if (e != cudaSuccess) return cuda_fail(e, "rollout");
  for (size_t i = 0; i < n; ++i) hist[i] = L->h_hist[i];
  if (voids)
    for (int a = 0; a < n_actions; ++a) voids[a] = L->h_hist[n + a];
  return DVC_OK;
}

int dvc_rollout_batch(const dvc_state *s, const uint32_t *actions, int32_t n_actions, uint64_t n_sims,
                      uint64_t seed, uint64_t *wins) {
  DeviceRestore restore_device;
  const State *st = s ? as_state(s) : nullptr;
  if (!st || !wins) return set_err(DVC_E_CONFIG, "bad arguments");
  if (n_sims == 0 || n_sims >= (1ull << 32)) return set_err(DVC_E_CONFIG, "n_sims must be in [1, 2^32)");
  if (n_actions < 1 || n_actions > kMaxActions) return set_err(DVC_E_CONFIG, "n_actions must be in [1, 768]");
  std::vector<uint64_t> hist((size_t)n_actions * st->P);
  int rc = dvc_rollout_batch_ex(s, actions, n_actions, seed, 0, 0, n_sims, hist.data(), nullptr, -1);
  if (rc) return rc;
  for (int a = 0; a < n_actions; ++a) wins[a] = hist[(size_t)a * st->P + st->viewer];
  return DVC_OK;
}

int dvc_rollout_batch_async(const dvc_state *s, const uint32_t *actions, int32_t n_actions, uint64_t seed,
                            uint32_t node_id, uint64_t sim_begin, uint64_t sim_end, uint64_t *d_hist,
                            uint64_t *d_visits, int32_t device, void *cuda_stream) {
  DeviceRestore restore_device;
  return rollout_async(s, actions, n_actions, seed, node_id, sim_begin, sim_end, d_hist, d_visits, device,
                       cuda_stream, 0u);
}

int dvc_rollout_trace_async(const dvc_state *s, const uint32_t *actions, int32_t n_actions, uint64_t seed,
                            uint32_t node_id, uint64_t sim_begin, uint64_t sim_end, uint64_t *d_hist,
                            uint8_t *d_winners, int32_t device, void *cuda_stream) {
  DeviceRestore restore_device;
  if (!d_hist || !d_winners) return set_err(DVC_E_CONFIG, "null device pointer");
  return enqueue(s, actions, n_actions, seed, node_id, sim_begin, sim_end,
                 reinterpret_cast<unsigned long long *>(d_hist), d_winners, device,
                 reinterpret_cast<cudaStream_t>(cuda_stream), nullptr);
}

int dvc_set_option(const char *name, int64_t value) {
  if (!name) return set_err(DVC_E_CONFIG, "null option name");
  std::string n(name);
  if (n == "kernel") {
    if (value < 0 || value > 2) return set_err(DVC_E_CONFIG, "kernel must be 0 (refill), 1 (naive) or 2 (auto)");
    g_kernel = value;
  } else if (n == "block") {
    if (value < 1 || value > 1024) return set_err(DVC_E_CONFIG, "block must be 1..1024");
    g_block = value;
  } else if (n == "grid") {
    if (value < 0 || value > (1 << 20)) return set_err(DVC_E_CONFIG, "grid out of range");
    g_grid = value;
  } else if (n == "table_cap") {
    if (value < 0) return set_err(DVC_E_CONFIG, "table_cap must be >= 0");
    g_table_cap = value;
  } else if (n == "chunk") {
    if (value < 1 || value > (1ll << 31)) return set_err(DVC_E_CONFIG, "chunk must be 1..2^31 work items");
    g_chunk = value;
  } else if (n == "plan_cache") {
    if (value != 0 && value != 1) return set_err(DVC_E_CONFIG, "plan_cache must be 0 or 1");
    g_plan_cache = value;
  } else if (n == "search_device") {
    if (value != 0 && value != 1) return set_err(DVC_E_CONFIG, "search_device must be 0 or 1");
    g_search_device = value;
  } else {
    return set_err(DVC_E_CONFIG, "unknown option " + n);
  }
  return DVC_OK;
}

int dvc_get_option(const char *name, int64_t *value) {
  if (!name || !value) return set_err(DVC_E_CONFIG, "null argument");
  std::string n(name);
  if (n == "kernel") *value = g_kernel;
  else if (n == "block") *value = g_block;
  else if (n == "grid") *value = g_grid;
  else if (n == "table_cap") *value = g_table_cap;
  else if (n == "plan_cache") *value = g_plan_cache;
  else if (n == "chunk") *value = g_chunk;
  else if (n == "search_device") *value = g_search_device;
  else return set_err(DVC_E_CONFIG, "unknown option " + n);
  return DVC_OK;
}

int dvc_debug_counters(int32_t device, uint32_t *out3) {
  DeviceRestore restore_device;
#ifdef DVC_DEBUG
  if (!out3) return set_err(DVC_E_CONFIG, "null argument");
  std::lock_guard<std::mutex> lock(g_mu);
  DeviceScratch *d = nullptr;
  int rc = get_scratch(device, &d);
  if (rc) return rc;
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(out3, d->d_debug, 3 * sizeof(uint32_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "debug counters");
  return DVC_OK;
#else
  (void)device; (void)out3;
  return set_err(DVC_E_CONFIG, "not a DVC_DEBUG build (libdvc_debug.so has the invariant checks)");
#endif
}

int dvc_transfer_bytes(int32_t reset, uint64_t *h2d, uint64_t *d2h) {
  if (h2d) *h2d = g_h2d.load();
  if (d2h) *d2h = g_d2h.load();
  if (reset) { g_h2d = 0; g_d2h = 0; }
  return DVC_OK;
}

uint64_t dvc_launch_count(int32_t reset) {
  uint64_t v = g_launches.load();
  if (reset) g_launches = 0;
  return v;
}

const char *dvc_last_error(void) { return g_err.c_str(); }

void dvc_shutdown(void) {
  std::lock_guard<std::mutex> lock(g_mu);
  for (auto &kv : g_dev) {
    DeviceScratch *d = kv.second;
    cudaSetDevice(d->device);
    cudaDeviceSynchronize();
    for (auto &p : d->plans) free_plan_now(p);
    for (auto &p : d->zombies) free_plan_now(p);
    for (auto &b : d->pool) cudaFree(b.first);
    for (auto ev : d->events) cudaEventDestroy(ev);
    for (auto ev : d->counter_ev) if (ev) cudaEventDestroy(ev);
    if (d->d_counters) cudaFree(d->d_counters);
    for (auto &kv2 : d->lanes) {
      if (kv2.second.d_hist) cudaFree(kv2.second.d_hist);
      if (kv2.second.h_hist) cudaFreeHost(kv2.second.h_hist);
      if (kv2.second.d_search) cudaFree(kv2.second.d_search);
      if (kv2.second.d_rho) cudaFree(kv2.second.d_rho);
      if (kv2.second.h_rho) cudaFreeHost(kv2.second.h_rho);
      if (kv2.second.stream) cudaStreamDestroy(kv2.second.stream);
    }
    delete d;
  }
  g_dev.clear();
}

}  // extern "C"
