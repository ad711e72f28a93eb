// Grid-wide synchronisation helpers for persistent cooperative kernels.
#pragma once

#include "q1.cuh"

namespace tb {

struct GridBarrier {
  unsigned int count;
  unsigned int gen;
};

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// All CTAs of the (co-resident) grid meet here.  Thread 0 arrives with release semantics and
// spins with acquire; the gpu-scope fence after the spin also invalidates this SM's L1 so the
// plain (L1-cached) loads that follow see other CTAs' writes.
__device__ __forceinline__ void grid_barrier(GridBarrier* gb, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int g = ld_acquire(&gb->gen);
    __threadfence();
    const unsigned int arrived = atomicAdd(&gb->count, 1u);
    if (arrived == nblocks - 1) {
      gb->count = 0u;
      __threadfence();
      st_release(&gb->gen, g + 1u);
    } else {
      while (ld_acquire(&gb->gen) == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// fixed-order sum of nb partials by warp 0, broadcast through shared memory
template <int NV>
__device__ __forceinline__ void sum_partials(const double* part, int nb, double (&out)[NV]) {
  __shared__ double bc[NV];
  if (threadIdx.x < 32) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double s = 0.0;
      for (int b = threadIdx.x; b < nb; b += 32) s += __ldcg(part + v * nb + b);
      s = warp_sum(s);
      if (threadIdx.x == 0) bc[v] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int v = 0; v < NV; ++v) out[v] = bc[v];
  __syncthreads();
}

}  // namespace tb
