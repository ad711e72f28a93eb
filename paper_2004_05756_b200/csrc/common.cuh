// Shared internals of libtopo_b200: error plumbing, grid geometry, deterministic
// block reductions and the device-resident pCG scalar state.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "topo_b200.h"

namespace tb {

void set_error(const char* fmt, ...);
// host-side count of kernels issued by this library (tb_launch_count)
void launched(int64_t n = 1);

#define TB_CUDA(call)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      ::tb::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__,     \
                      __LINE__);                                                            \
      return TB_ERR_CUDA;                                                                   \
    }                                                                                       \
  } while (0)

#define TB_CHECK_LAUNCH() TB_CUDA(cudaGetLastError())

#define TB_TRY(expr)            \
  do {                          \
    int rc_ = (expr);           \
    if (rc_ != TB_OK) return rc_; \
  } while (0)

constexpr int kBlock = 256;

// Structured grid geometry (reference fem.py:154-229; Hex8 extension in include/topo_b200.h).
struct Grid {
  int dim, nx, ny, nz;  // nz = 1 in 2D for uniform indexing
  int nnx, nny, nnz;    // node counts per axis
  double h;
  int64_t n_elems, n_nodes;
};

// Element matrices travel as kernel parameters (constant bank; CUDA >= 12.1 allows 32 KB).
template <int N>
struct Mat {
  double v[N * N];
};

// Device-resident pCG scalars.  Written by the last block of each fused kernel, read by
// every block of the next one; nothing crosses to the host inside the iteration loop.
struct PcgState {
  double rz;     // r^T z of the current residual
  double pq;     // p^T K p
  double alpha;  // rz / pq
  double beta;   // rz_new / rz_old  (consumed by the next direction update)
  double rr;     // ||r||^2 (recursive residual)
  double tol2;   // (rtol ||b||)^2
  double bb;     // ||Z b||^2
  int iters;
  int maxit;
  int done;      // 0 running, 1 converged, 2 maxit, 3 breakdown
  int pad;
  unsigned int count_a, count_b, count_c, pad2;
  // distributed (slab) mode: kernels only publish rank-local sums in red[] (pq; rz, rr) and
  // the host allreduces them before tb_pcg_dist_alpha / tb_pcg_dist_beta
  int dist;
  int dot_k0, dot_k1;  // node planes [k0, k1) that own their rows (reductions, contractions)
  int pad3;
  double red[4];
  int cg_init;  // single-reduction sweep (sweep.cu): the next sweep is a (re)start sweep
  int pad4;
  double cg_beta;  // distributed single-reduction pCG (phases 10-13): beta of the p/s recurrences
  double alpha_lag;  // sweep.cu: alpha of the x update a lagging sweep left pending on p (0: none)
};

// ---------------------------------------------------------------------------------------
// deterministic reductions: fixed shuffle tree inside a block, fixed-order final sum in
// the last block to arrive (no floating-point atomics anywhere).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Sum of NV values over the block; result valid in every thread.  blockDim.x % 32 == 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV]) {
  __shared__ double red[NV][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x * blockDim.y * blockDim.z) >> 5;
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int l = tid & 31, w = tid >> 5;
  (void)lane; (void)warp;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (l == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) red[i][w] = v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double s = (l < nw) ? red[i][l] : 0.0;
    v[i] = warp_sum(s);
  }
  __syncthreads();
}

__device__ __forceinline__ int flat_tid() {
  return threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
}
__device__ __forceinline__ int flat_bid() {
  return blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
}
__device__ __forceinline__ int n_blocks() { return gridDim.x * gridDim.y * gridDim.z; }
__device__ __forceinline__ int n_threads() { return blockDim.x * blockDim.y * blockDim.z; }

// Publish this block's NV partials and report whether it is the last block to arrive.
// partials layout: [NV][n_blocks].
template <int NV>
__device__ __forceinline__ bool publish_partials(const double (&v)[NV], double* partials,
                                                 unsigned int* counter) {
  __shared__ bool last;
  const int tid = flat_tid(), bid = flat_bid(), nb = n_blocks();
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) partials[i * nb + bid] = v[i];
    __threadfence();
    unsigned int t = atomicAdd(counter, 1u);
    last = (t == (unsigned int)(nb - 1));
  }
  __syncthreads();
  return last;
}

// In the last block: fixed-order sum of the published partials (every thread gets the sum).
template <int NV>
__device__ __forceinline__ void gather_partials(double (&v)[NV], const double* partials,
                                                unsigned int* counter) {
  __threadfence();
  const int tid = flat_tid(), nb = n_blocks(), nt = n_threads();
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double s = 0.0;
    for (int b = tid; b < nb; b += nt) s += __ldcg(partials + i * nb + b);
    v[i] = s;
  }
  block_sum<NV>(v);
  if (tid == 0) *counter = 0u;
}

// ---- mbarrier + 1D bulk copy (async proxy) primitives shared by the TMA/bulk-staged kernels ----
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nMBW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra MBW_%=;\n}\n" ::"r"(
          smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// 1D bulk copy global -> shared, completion counted on `bar`; addresses and size 16-byte aligned
__device__ __forceinline__ void bulk_g2s(double* dst, const double* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
// generic-proxy writes (this or other CTAs, ordered by a barrier) -> later async-proxy reads
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;\n" ::: "memory"); }

inline int grid_for(int64_t n, int per_block = kBlock, int cap = 148 * 8) {
  int64_t b = (n + per_block - 1) / per_block;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

// 8-byte asynchronous global -> shared copy (LDGSTS), zero-filling when !valid
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 8 : 0;  // src-size 0 zero-fills the destination
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}
// 16-byte variant: copies src_bytes (0, 8 or 16) and zero-fills the rest of the 16 bytes
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

}  // namespace tb
