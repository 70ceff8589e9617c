// kernels.cu -- the sm_100a kernels of the hot path.
//
//  * rollout_refill_kernel (default): persistent, warp-refilling.  Each lane
//    holds one playout in registers; the loop body is ONE decision step for
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
#include <cuda_runtime.h>
#include "rollout.cuh"

namespace dvc {

__device__ __forceinline__ void record(uint32_t *sh_hist, const KParams &kp, uint32_t a, uint32_t s,
                                       uint32_t w, int P) {
  atomicAdd(&sh_hist[a * P + w], 1u);
  if (kp.winners) kp.winners[(size_t)a * kp.trace_stride + (s - kp.trace_s0)] = (uint8_t)w;
}

__device__ __forceinline__ void zero_hist(uint32_t *sh, uint32_t n) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) sh[i] = 0;
  __syncthreads();
}

__device__ __forceinline__ void flush_hist(const uint32_t *sh, uint32_t n, unsigned long long *g) {
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t v = sh[i];
    if (v) atomicAdd(g + i, (unsigned long long)v);
  }
}

template <int P, bool JOK, bool CONS>
__global__ void __launch_bounds__(1024) rollout_naive_kernel(const __grid_constant__ KParams kp) {
  extern __shared__ uint32_t sh_hist[];
  zero_hist(sh_hist, kp.A * P);
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < kp.total; w += stride) {
    const uint32_t a = w / kp.n_per;
    const uint32_t s = kp.s0 + (w - a * kp.n_per);
    const uint32_t code = kp.codes[a];
    Sim<P> S;
    uint32_t st = init_playout<P, JOK, CONS>(S, a, s, kp);
    uint32_t k = 0;
    while (st != FINISH) {
      const uint4 B = philox4x32_10(k, s, code, kp.node, kp.k0, kp.k1);
      st = step<P, JOK, CONS>(S, st, B, kp);
      ++k;
    }
    record(sh_hist, kp, a, s, winner_seat(S), P);
  }
  flush_hist(sh_hist, kp.A * P, kp.hist);
}

template <int P, bool JOK, bool CONS>
__global__ void __launch_bounds__(1024) rollout_refill_kernel(const __grid_constant__ KParams kp) {
  extern __shared__ uint32_t sh_hist[];
  zero_hist(sh_hist, kp.A * P);
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt_mask = (1u << lane) - 1u;
  bool active = false;
  bool exhausted = false;  // warp-uniform
  uint32_t a = 0, s = 0, code = 0, st = FINISH, k = 0;
  Sim<P> S;
  while (true) {
    // ---- refill idle lanes from the launch's work counter
    const uint32_t need = __ballot_sync(0xFFFFFFFFu, !active);
    if (need && !exhausted) {
      const uint32_t leader = __ffs(need) - 1u;
      const uint32_t cnt = __popc(need);
      uint32_t base = 0;
      if (lane == leader) base = atomicAdd(kp.counter, cnt);
      base = __shfl_sync(0xFFFFFFFFu, base, leader);
      exhausted = base + cnt >= kp.total;
      if (!active) {
        const uint32_t w = base + __popc(need & lt_mask);
        if (w < kp.total) {
          a = w / kp.n_per;
          s = kp.s0 + (w - a * kp.n_per);
          code = kp.codes[a];
          st = init_playout<P, JOK, CONS>(S, a, s, kp);
          k = 0;
          active = true;
          if (st == FINISH) {
            record(sh_hist, kp, a, s, winner_seat(S), P);
            active = false;
          }
        }
      }
    }
    if (!__any_sync(0xFFFFFFFFu, active)) {
      if (exhausted) break;
      continue;
    }
    // ---- one decision step for every active lane
    if (active) {
      const uint4 B = philox4x32_10(k, s, code, kp.node, kp.k0, kp.k1);
      st = step<P, JOK, CONS>(S, st, B, kp);
      ++k;
      if (st == FINISH) {
        record(sh_hist, kp, a, s, winner_seat(S), P);
        active = false;
      }
    }
  }
  flush_hist(sh_hist, kp.A * P, kp.hist);
}

__global__ void det_table_kernel(const uint8_t *__restrict__ plan, uint64_t N, uint4 *__restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += stride)
    out[r] = unrank(plan, r);
}

__global__ void add_u64_kernel(unsigned long long *p, uint32_t n, unsigned long long v) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] += v;
}

// ----------------------------------------------------------------- launchers
cudaError_t launch_add_u64(unsigned long long *p, uint32_t n, uint64_t v, cudaStream_t stream) {
  add_u64_kernel<<<(n + 255) / 256, 256, 0, stream>>>(p, n, v);
  return cudaGetLastError();
}

typedef void (*KernelFn)(const KParams);

template <int P, bool JOK, bool CONS>
KernelFn pick_kernel(int variant) {
  return variant == 1 ? rollout_naive_kernel<P, JOK, CONS> : rollout_refill_kernel<P, JOK, CONS>;
}

KernelFn select_kernel(int P, bool jok, bool cons, int variant) {
#define DVC_CASE(PP)                                                                     \
  if (P == PP) {                                                                         \
    if (jok) return cons ? pick_kernel<PP, true, true>(variant) : pick_kernel<PP, true, false>(variant); \
    return cons ? pick_kernel<PP, false, true>(variant) : pick_kernel<PP, false, false>(variant);       \
  }
  DVC_CASE(2)
  DVC_CASE(3)
  DVC_CASE(4)
#undef DVC_CASE
  return nullptr;
}

cudaError_t kernel_occupancy(int P, bool jok, bool cons, int variant, int block, size_t smem, int *blocks_per_sm) {
  KernelFn f = select_kernel(P, jok, cons, variant);
  if (!f) return cudaErrorInvalidValue;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, (const void *)f, block, smem);
}

cudaError_t launch_rollout(const KParams &kp, int P, bool jok, bool cons, int variant, int grid, int block,
                           size_t smem, cudaStream_t stream) {
  KernelFn f = select_kernel(P, jok, cons, variant);
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
