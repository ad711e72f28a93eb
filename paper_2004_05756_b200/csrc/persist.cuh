// Persistent cooperative Jacobi-pCG for latency-bound (L2-resident) problems.
//
// One cooperative launch runs the whole iteration: every CTA owns a contiguous node range,
// the direction update is folded into the operator gather (p = z + beta p_old, double
// buffered), and the two reductions per iteration (p.q, then r.z and r.r) are exchanged
// through per-CTA partials behind a software grid barrier.  Every CTA sums the partials in
// the same fixed order, so all CTAs take identical, deterministic decisions.  Two barriers per
// iteration replace the two kernel boundaries of the graph path.
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

struct PersistArgs {
  double *x, *r, *z, *pa, *pb, *q;
  const double* dinv;
  double* part;  // [3][gridDim.x]
  PcgState* st;
  GridBarrier* gb;
};

constexpr int kPersistThreads = 512;

template <int D, int NC, bool SCALED>
__global__ void __launch_bounds__(kPersistThreads) k_pcg_persistent(Grid g, Mat<Q1<D>::NN * NC> K,
                                                                     const double* __restrict__ alpha, PersistArgs a) {
  const unsigned int nb = gridDim.x;
  const int tid = threadIdx.x;
  // element matrix in shared memory: read as broadcast operands, and not hoisted into 64+
  // registers across the persistent loop (constant-bank operands would be)
  __shared__ Mat<Q1<D>::NN * NC> Ks;
  for (int o = tid; o < Q1<D>::NN * NC * Q1<D>::NN * NC; o += blockDim.x) Ks.v[o] = K.v[o];
  __syncthreads();
  const int64_t per = (g.n_nodes + nb - 1) / nb;
  const int64_t n0 = (int64_t)blockIdx.x * per;
  const int64_t n1 = min(g.n_nodes, n0 + per);
  double rz = a.st->rz, beta = a.st->beta, rr = a.st->rr;
  const double tol2 = a.st->tol2;
  int it = a.st->iters;
  const int maxit = a.st->maxit;
  int done = a.st->done;
  double* pold = a.pa;
  double* pnew = a.pb;
  constexpr int self = (D == 3) ? 13 : 4;
  while (done == 0) {
    // ---- phase 1: p = z + beta p_old ; q = K p ; p.q ----
    double acc[1] = {0.0};
    for (int64_t n = n0 + tid; n < n1; n += blockDim.x) {
      int i, j, k;
      node_coords(g, n, i, j, k);
      double P[Q1<D>::NB][NC];
      double sc[Q1<D>::NN];
#pragma unroll
      for (int dz = 0; dz < (D == 3 ? 3 : 1); ++dz)
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) {
            const int nbh = (dz * 3 + dy) * 3 + dx;
            const int ii = i + dx - 1, jj = j + dy - 1, kk = (D == 3) ? k + dz - 1 : 0;
            const bool ok = ii >= 0 && ii < g.nnx && jj >= 0 && jj < g.nny && kk >= 0 && kk < g.nnz;
            const int64_t node = ((int64_t)kk * g.nny + jj) * g.nnx + ii;
#pragma unroll
            for (int c = 0; c < NC; ++c)
              P[nbh][c] = ok ? fma(beta, pold[NC * node + c], a.z[NC * node + c]) : 0.0;
          }
      slot_scales<D, SCALED>(g, i, j, k, alpha, sc);
      double out[NC];
      node_rows<D, NC>(Ks, P, sc, out);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        pnew[NC * n + c] = P[self][c];
        a.q[NC * n + c] = out[c];
        acc[0] = fma(P[self][c], out[c], acc[0]);
      }
    }
    block_sum<1>(acc);
    if (tid == 0) a.part[blockIdx.x] = acc[0];
    grid_barrier(a.gb, nb);
    double pq[1];
    sum_partials<1>(a.part, nb, pq);
    if (!(pq[0] > 0.0) || !isfinite(pq[0])) {
      done = 3;
      break;
    }
    const double al = rz / pq[0];
    // ---- phase 2: x += al p ; r -= al q ; z = D^-1 r ; r.z, r.r ----
    double acc2[2] = {0.0, 0.0};
    for (int64_t d = NC * n0 + tid; d < NC * n1; d += blockDim.x) {
      const double di = a.dinv[d];
      if (di != 0.0) {
        a.x[d] = fma(al, pnew[d], a.x[d]);
        const double ri = fma(-al, a.q[d], a.r[d]);
        const double zi = di * ri;
        a.r[d] = ri;
        a.z[d] = zi;
        acc2[0] = fma(ri, zi, acc2[0]);
        acc2[1] = fma(ri, ri, acc2[1]);
      }
    }
    block_sum<2>(acc2);
    if (tid == 0) {
      a.part[nb + blockIdx.x] = acc2[0];
      a.part[2 * nb + blockIdx.x] = acc2[1];
    }
    grid_barrier(a.gb, nb);
    double red[2];
    sum_partials<2>(a.part + nb, nb, red);
    ++it;
    beta = red[0] / rz;
    rz = red[0];
    rr = red[1];
    double* t = pold;
    pold = pnew;
    pnew = t;
    if (!isfinite(red[0]) || !isfinite(red[1])) done = 3;
    else if (rr <= tol2) done = 1;
    else if (it >= maxit) done = 2;
  }
  if (blockIdx.x == 0 && tid == 0) {
    a.st->rz = rz;
    a.st->rr = rr;
    a.st->beta = beta;
    a.st->iters = it;
    a.st->done = done;
  }
}

}  // namespace tb
