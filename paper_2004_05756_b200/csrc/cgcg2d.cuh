// Single-reduction persistent Jacobi-pCG for 2D structured grids (Chronopoulos-Gear CG).
//
// Why: on BASELINE cfg 1-2 the whole working set (< 20 MB) sits in L2 and a Jacobi-pCG
// iteration is worth ~3 us of memory traffic, so kernel boundaries and grid-wide reductions
// dominate.  This kernel runs the entire solve in one cooperative launch with ONE grid
// barrier per iteration:
//
//   CG-CG recurrences (x, r, u = D^-1 r, w = A u, p, s = A p):
//     p_i = u_i + b_i p_{i-1};  s_i = w_i + b_i s_{i-1}
//     x_{i+1} = x_i + a_i p_i;  r_{i+1} = r_i - a_i s_i;  u_{i+1} = D^-1 r_{i+1};  w_{i+1} = A u_{i+1}
//     g_{i+1} = (r,u), d_{i+1} = (w,u), rho_{i+1} = (r,r)       <- the only reduction
//     b_{i+1} = g_{i+1}/g_i;  a_{i+1} = g_{i+1} / (d_{i+1} - b_{i+1} g_{i+1}/a_i)
//
// Each CTA owns a contiguous node range and keeps x, r, p, s, w, D^-1 of it in shared memory.
// The matvec needs u_{i+1} on a one-node halo; instead of a second barrier the CTA recomputes
// the halo's u_{i+1} = D^-1 (r_i - a_i (w_i + b_i s_{i-1})) from vectors its neighbours
// published before the previous barrier (parity double-buffered in global memory).  Partials
// are summed by every CTA in the same fixed order: deterministic, identical decisions.
#pragma once

#include "q1.cuh"

namespace tb {

#ifdef TB_CGCG_PROF
__device__ __forceinline__ unsigned long long gtime() { return (unsigned long long)clock64(); }
#define PROF_MARK(k)                                  \
  do {                                                \
    if (blockIdx.x == 0 && threadIdx.x == 0) {        \
      const unsigned long long t_ = gtime();          \
      prof[k] += t_ - prof_last;                      \
      prof_last = t_;                                 \
    }                                                 \
  } while (0)
#else
#define PROF_MARK(k) \
  do {               \
  } while (0)
#endif

// Grid barrier: one atomic per CTA, bit 31 flips when all have arrived.  The CTA's writes are
// ordered before thread 0's arrival by bar.sync and the arrival is a RELEASE atomic
// (cumulative over them); the spin is an ACQUIRE load and the closing bar.sync orders the rest
// of the CTA after it.  Every cross-CTA read after the barrier is an L2 load (__ldcg) of
// parity-buffered data, so no trailing fence is needed to drop stale L1 lines.
__device__ __forceinline__ void grid_sync_flip(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int nb = gridDim.x;
    const unsigned int add = (blockIdx.x == 0) ? (0x80000000u - (nb - 1u)) : 1u;
    unsigned int old, cur;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(add) : "memory");
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
    } while (((old ^ cur) & 0x80000000u) == 0u);
  }
  __syncthreads();
}

// End of an iteration of the persistent kernels: this CTA's NV dot partials (same fixed-order
// sum as block_sum) are published to part[i * nbk + blockIdx.x] and the grid barrier is
// crossed, with 2 CTA barriers instead of block_sum's 3 plus the grid barrier's 2.  Only warp 0
// needs the CTA sum; the single bar.sync before it also orders every thread's ring
// publications before thread 0's release arrival.  `red` is reused next iteration only after the
// closing bar.sync, which warp 0 reaches after reading it.
template <int NV>
__device__ __forceinline__ void publish_partials_grid_sync(double (&v)[NV], double* part, unsigned int* bar,
                                                           bool skip_barrier = false) {
  __shared__ double red[NV][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) red[i][w] = v[i];
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = warp_sum((lane < nw) ? red[i][lane] : 0.0);
    if (lane == 0) {
      const unsigned int nb = gridDim.x;
#pragma unroll
      for (int i = 0; i < NV; ++i) part[i * nb + blockIdx.x] = v[i];
      if (!skip_barrier) {
        const unsigned int add = (blockIdx.x == 0) ? (0x80000000u - (nb - 1u)) : 1u;
        unsigned int old, cur;
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(add) : "memory");
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
        } while (((old ^ cur) & 0x80000000u) == 0u);
      }
    }
  }
  __syncthreads();
}

struct CgcgArgs {
  const double* b;     // unused (restart state comes from r, x)
  double* x;           // in: x0 ; out: solution
  const double* r0;    // r0 = Z (b - K x0) (k_pcg_start)
  const double* dinv;  // Jacobi inverse diagonal, 0 on fixed dofs
  double* pub;         // published vectors [2 parities][3 (r, w, s)][n_dofs]
  double* part;        // [2 parities][3][gridDim.x]
  PcgState* st;
  unsigned int* bar;
  int own_max;         // max nodes owned by a CTA
  int dbg;             // profiling builds only: bit0 skip barrier, bit1 skip apply, bit2 skip halo
};

constexpr int kCgcgThreads = 512;

// PAT: K follows the reference's Q4 value pattern (q4_pat); the node rows use its distinct
// values (kernel parameters) instead of reading K from shared memory.
template <int NC, bool SCALED, bool PAT>
__global__ void __launch_bounds__(kCgcgThreads, 1) k_pcg2d_cgcg(Grid g, Mat<4 * NC> K, Q4Pat kp,
                                                               const double* __restrict__ alpha, CgcgArgs a) {
  extern __shared__ double sm[];
  __shared__ __align__(16) Mat<4 * NC> Ks;
  __shared__ double bc[2][3];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nbk = gridDim.x;
  const int64_t N = g.n_nodes, ND = (int64_t)NC * N;
  const int64_t per = (N + nbk - 1) / nbk;
  const int64_t n0 = (int64_t)blockIdx.x * per;
  const int64_t n1 = min(N, n0 + per);
  const int no = (int)max((int64_t)0, n1 - n0);
  const int64_t h0 = max((int64_t)0, n0 - g.nnx - 1);
  const int64_t h1 = min(N, n1 + g.nnx + 1);
  const int ne_ext = (int)(h1 - h0);
  // element rows touching own nodes
  const int j_lo = (int)(n0 / g.nnx), j_hi = (int)((max(n1, n0 + 1) - 1) / g.nnx);
  const int64_t e0 = (int64_t)max(0, j_lo - 1) * g.nx;
  const int64_t e1 = (int64_t)min(g.ny, j_hi + 1) * g.nx;
  // shared-memory carve-up
  double* u_ext = sm;                          // (h1-h0)*NC
  double* dext = u_ext + (size_t)ne_ext * NC;  // D^-1 over own + halo (constant over the solve)
  double* xs = dext + (size_t)ne_ext * NC;     // own: x, r, p, s, w
  double* rs = xs + (size_t)no * NC;
  double* ps = rs + (size_t)no * NC;
  double* ss = ps + (size_t)no * NC;
  double* ws = ss + (size_t)no * NC;
  double* as = ws + (size_t)no * NC;           // alpha of elements [e0, e1)
  double* ds = dext + (n0 - h0) * NC;          // own part of dext
  if (!PAT)
    for (int o = tid; o < 16 * NC * NC; o += nt) Ks.v[o] = K.v[o];
  for (int64_t e = e0 + tid; e < e1; e += nt) as[e - e0] = SCALED ? alpha[e] : 1.0;

  const int64_t d0 = (int64_t)NC * n0;
  const int nod = no * NC;
  // ---- prologue: x, r, D^-1 from global; u on own + halo; s_{-1} = p_{-1} = 0 ----
  for (int o = tid; o < nod; o += nt) {
    xs[o] = a.x[d0 + o];
    rs[o] = a.r0[d0 + o];
    ps[o] = 0.0;
    ss[o] = 0.0;
  }
  for (int64_t o = tid; o < (int64_t)ne_ext * NC; o += nt) {
    const int64_t d = h0 * NC + o;
    dext[o] = a.dinv[d];
    u_ext[o] = a.dinv[d] * a.r0[d];
  }
  __syncthreads();

  double* pubr[2] = {a.pub, a.pub + 3 * ND};
  const int nnx = g.nnx, h0i = (int)h0, e0i = (int)e0, n0i = (int)n0;
  const int nx_e = g.nx, nny = g.nny;
  auto node_apply = [&](int n, double (&out)[NC]) {
    const int j = n / nnx, i = n - j * nnx;
    double P[9][NC];
    double sc[4];
    if (i > 0 && i < nnx - 1 && j > 0 && j < nny - 1) {
      // interior node: all 9 neighbours and 4 elements exist -- constant offsets, no checks
      const double* u0 = u_ext + (n - nnx - 1 - h0i) * NC;
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx)
#pragma unroll
          for (int c = 0; c < NC; ++c) P[dy * 3 + dx][c] = u0[(dy * nnx + dx) * NC + c];
      const double* a0 = as + ((j - 1) * nx_e + i - 1 - e0i);
      sc[0] = a0[0];
      sc[1] = a0[1];
      sc[2] = a0[nx_e];
      sc[3] = a0[nx_e + 1];
    } else {
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const int ii = i + dx - 1, jj = j + dy - 1;
          const bool ok = ii >= 0 && ii < g.nnx && jj >= 0 && jj < g.nny;
          const int m = jj * nnx + ii - h0i;
#pragma unroll
          for (int c = 0; c < NC; ++c) P[dy * 3 + dx][c] = ok ? u_ext[m * NC + c] : 0.0;
        }
#pragma unroll
      for (int sl = 0; sl < 4; ++sl) {
        const int ei = i - 1 + (sl & 1), ej = j - 1 + (sl >> 1);
        const bool ok = ei >= 0 && ei < g.nx && ej >= 0 && ej < g.ny;
        sc[sl] = ok ? as[ej * g.nx + ei - e0i] : 0.0;
      }
    }
    if (PAT)
      node_rows_pat<NC>(kp, P, sc, out);
    else
      node_rows<2, NC>(Ks, P, sc, out);
  };

  // w_0 = A u_0 ; partials ; publish r_0, w_0, s_{-1}
  double acc[3] = {0.0, 0.0, 0.0};
  for (int o = tid; o < no; o += nt) {
    const int n = n0i + o;
    double out[NC];
    node_apply(n, out);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int od = o * NC + c;
      const double u = u_ext[(n - h0i) * NC + c];
      ws[od] = out[c];
      acc[0] = fma(rs[od], u, acc[0]);
      acc[1] = fma(out[c], u, acc[1]);
      acc[2] = fma(rs[od], rs[od], acc[2]);
      pubr[0][d0 + od] = rs[od];
      pubr[0][ND + d0 + od] = out[c];
      pubr[0][2 * ND + d0 + od] = 0.0;
    }
  }
  block_sum<3>(acc);
  // Partials are parity-buffered like the published vectors: a CTA that races ahead writes
  // iteration i+1's partials into the other buffer while slower CTAs still read iteration i's
  // (a single buffer let them sum a mix, branch differently and deadlock at the next barrier).
  if (tid == 0) {
    a.part[blockIdx.x] = acc[0];
    a.part[nbk + blockIdx.x] = acc[1];
    a.part[2 * nbk + blockIdx.x] = acc[2];
  }
  grid_sync_flip(a.bar);

#ifdef TB_CGCG_PROF
  unsigned long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long prof_last = gtime();
#endif
  double gam = 0.0, al = 0.0, be = 0.0, rr = 0.0;
  int it = a.st->iters, done = 0;
  const int maxit = a.st->maxit;
  const double tol2 = a.st->tol2;
  int par = 0;  // parity of the buffer holding (r_i, w_i, s_{i-1})
  // halo geometry (dofs below / above the own range that the stencil of own nodes touches)
  const int64_t lo_len = d0 - h0 * NC;
  const int64_t hi_beg = d0 + nod;
  const int64_t halo = lo_len + (h1 * NC - hi_beg);
  constexpr int kHB = 6;                 // halo loads in flight per thread (warps 1..15)
  const int ht = tid - 32, hnt = nt - 32;  // halo thread index / count (warp 0 reduces partials)
  for (bool first = true;; first = false) {
    // ---- after the barrier: two independent L2 round trips issued together ----
    // warps 1..15: the first batch of the neighbours' published (r, w, s) plus D^-1 for the halo;
    // warp 0: every CTA's partials (fixed-order sum, identical in every CTA).
    const double* pr = pubr[par];
    double rv[kHB], wv[kHB], sv[kHB];
    int mm[kHB];  // halo entry relative to h0 * NC (2D grids: < 2^31 dofs)
    auto halo_load = [&](int64_t base) {
#pragma unroll
      for (int q = 0; q < kHB; ++q) {
        const int64_t t = base + ht + (int64_t)q * hnt;
        const int64_t m = (t < lo_len) ? h0 * NC + t : hi_beg + (t - lo_len);
        mm[q] = (ht >= 0 && t < halo) ? (int)(m - h0 * NC) : -1;
        if (mm[q] >= 0) {
          rv[q] = __ldcg(pr + m);
          wv[q] = __ldcg(pr + ND + m);
          sv[q] = __ldcg(pr + 2 * ND + m);
        }
      }
    };
    if (tid >= 32) halo_load(0);
    if (tid < 32) {
      constexpr int kPB = 8;  // supports up to 256 CTAs
      double v[3][kPB];
#pragma unroll
      for (int q = 0; q < kPB; ++q) {
        const int b = tid + 32 * q;
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c][q] = (b < nbk) ? __ldcg(a.part + (par * 3 + c) * nbk + b) : 0.0;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < kPB; ++q) s += v[c][q];
        s = warp_sum(s);
        if (tid == 0) bc[par][c] = s;  // parity-buffered: no second barrier before reuse
      }
    }
    __syncthreads();
    PROF_MARK(0);
    const double gnew = bc[par][0], dnew = bc[par][1];
    rr = bc[par][2];
#if defined(TB_CGCG_ABL)
    if (a.dbg & 8) {  // ablation timing: run exactly maxit iterations whatever the numbers say
      if (!first && ++it >= maxit) {
        done = 2;
        break;
      }
      be = first ? 0.0 : 0.5;
      al = 0.5;
      gam = 1.0;
      goto abl_continue;
    }
#endif
    if (!isfinite(gnew) || !isfinite(dnew) || !isfinite(rr)) {
      done = 3;
      break;
    }
    if (!first) {
      ++it;
      if (rr <= tol2) {
        done = 1;
        break;
      }
      if (it >= maxit) {
        done = 2;
        break;
      }
    } else if (rr == 0.0 || rr <= tol2) {
      done = 1;
      break;
    }
    if (first) {
      be = 0.0;
      if (!(dnew > 0.0)) {
        done = 3;
        break;
      }
      al = gnew / dnew;
    } else {
      be = gnew / gam;
      const double pap = dnew - be * gnew / al;  // p^T A p
      if (!(pap > 0.0)) {
        done = 3;
        break;
      }
      al = gnew / pap;
    }
    gam = gnew;
#if defined(TB_CGCG_ABL)
  abl_continue:
#endif

    // ---- halo: u_{i+1} = D^-1 (r_i - al (w_i + be s_{i-1})) from the loaded publication ----
    auto halo_store = [&]() {
#pragma unroll
      for (int q = 0; q < kHB; ++q) {
        if (mm[q] < 0) continue;
        const double di = dext[mm[q]];
        double r = rv[q];
        if (di != 0.0) r = fma(-al, fma(be, sv[q], wv[q]), r);
        u_ext[mm[q]] = di * r;
      }
    };
    // ---- own: p, s, x, r and u_{i+1} = D^-1 r (each thread touches only its own entries) ----
    const int own_off = (n0i - h0i) * NC;  // own block inside u_ext
    for (int o = tid; o < nod; o += nt) {
      const double di = ds[o];
      const double u = u_ext[own_off + o];
      const double p = fma(be, ps[o], u);
      const double s = fma(be, ss[o], ws[o]);
      ps[o] = p;
      ss[o] = s;
      double r = rs[o];
      if (di != 0.0) {
        xs[o] = fma(al, p, xs[o]);
        r = fma(-al, s, r);
      }
      rs[o] = r;
      u_ext[own_off + o] = di * r;
    }
    PROF_MARK(1);
#if defined(TB_CGCG_PROF) || defined(TB_CGCG_ABL)
    if (!(a.dbg & 4))
#endif
    if (tid >= 32) {
      halo_store();
      for (int64_t base = (int64_t)kHB * hnt; base < halo; base += (int64_t)kHB * hnt) {
        halo_load(base);
        halo_store();
      }
    }
    __syncthreads();
    PROF_MARK(2);
    PROF_MARK(3);
    // ---- own: w_{i+1} = A u_{i+1}; partials; publish (r_{i+1}, w_{i+1}, s_i) ----
    double* pw = pubr[par ^ 1];
    double acc3[3] = {0.0, 0.0, 0.0};
    for (int o = tid; o < no; o += nt) {
      const int n = n0i + o;
      double out[NC];
#if defined(TB_CGCG_PROF) || defined(TB_CGCG_ABL)
      if (a.dbg & 2) {
        for (int c = 0; c < NC; ++c) out[c] = u_ext[(n - h0i) * NC + c];
      } else
#endif
      node_apply(n, out);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int od = o * NC + c;
        const double u = u_ext[(n - h0i) * NC + c];
        ws[od] = out[c];
        acc3[0] = fma(rs[od], u, acc3[0]);
        acc3[1] = fma(out[c], u, acc3[1]);
        acc3[2] = fma(rs[od], rs[od], acc3[2]);
        pw[d0 + od] = rs[od];
        pw[ND + d0 + od] = out[c];
        pw[2 * ND + d0 + od] = ss[od];
      }
    }
    PROF_MARK(4);
    block_sum<3>(acc3);
    PROF_MARK(5);
    if (tid == 0) {
      double* pp = a.part + (par ^ 1) * 3 * nbk;
      pp[blockIdx.x] = acc3[0];
      pp[nbk + blockIdx.x] = acc3[1];
      pp[2 * nbk + blockIdx.x] = acc3[2];
    }
    par ^= 1;
#if defined(TB_CGCG_PROF) || defined(TB_CGCG_ABL)
    if (!(a.dbg & 1))
#endif
      grid_sync_flip(a.bar);
    PROF_MARK(6);
  }
#ifdef TB_CGCG_PROF
  if (blockIdx.x == 0 && tid == 0)
    printf("cgcg prof (cycles/iter over %d its): sums %.0f own %.0f halo %.0f ownu %.0f apply %.0f bsum %.0f barrier %.0f\n",
           it, prof[0] / (double)it, prof[1] / (double)it, prof[2] / (double)it, prof[3] / (double)it,
           prof[4] / (double)it, prof[5] / (double)it, prof[6] / (double)it);
#endif
  for (int o = tid; o < nod; o += nt) a.x[d0 + o] = xs[o];
  if (blockIdx.x == 0 && tid == 0) {
    a.st->rr = rr;
    a.st->iters = it;
    a.st->done = done;
  }
}

// dynamic shared memory of one CTA for a given ownership size
inline size_t cgcg_smem_bytes(int NC, int64_t own, int64_t nnx, int64_t nx) {
  const int64_t ext = own + 2 * (nnx + 1);
  const int64_t rows = own / nnx + 3;
  return sizeof(double) * (size_t)(2 * ext * NC + 5 * own * NC + (rows + 1) * nx);
}

}  // namespace tb
