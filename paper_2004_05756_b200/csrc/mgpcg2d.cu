// Multigrid-preconditioned CG for 2D plans in ONE persistent cooperative launch.
//
// Why: on BASELINE cfg 1-2 the whole hierarchy (< 25 MB) sits in L2, and the graph-launched
// V-cycle of mg.cu is ~55 kernels of ~3.4 us each per pCG iteration (~190 us at cfg 2), nearly
// all of it launch and drain latency.  Here every phase is a grid-stride pass over one level,
// separated by a software grid barrier:
//
//   A  (level 0)   p = z + beta p_old (p double-buffered), q = K(rho) p, partial p.q   | barrier
//   B  (level 0)   alpha = rz / pq; x += alpha p; r -= alpha q (free dofs), partial r.r;
//                  first pre-smoothing sweep x0 = omega D^-1 r                          | barrier
//   down, l = 0 .. L-2:  [restriction + first sweep of l] | sweep 2 | residual           |
//   coarsest:            restriction | x = Ainv b (one warp per row over the grid)       |
//   up, l = L-2 .. 0:    prolongation | post sweep 1 | post sweep 2 (level 0: + r.z)     |
//
// Measured (profiles/mg_prof.py, TB_MGP_PROF build): a phase costs ~4 us whatever the level
// size (L2 round trips of the neighbour loads, store drain, barrier), so cfg 2 runs ~160 us per
// iteration against ~190 us for the graph: 5.1 vs 6.2 ms per solve.  Running the levels below
// ~6k dofs inside one CTA with CTA barriers was slower (~5.7 us per phase: one SM's serial L2
// latency), as was a 128-dof coarsest level kept in shared memory (27 -> 32 iterations).
//
// The arithmetic per dof is that of the graph path (same V(2,2) cycle, damped Jacobi, full
// weighting, linear prolongation, dense coarsest inverse), term by term, so the iterates agree
// with it to round-off (the dot products are summed in a different fixed order; the level-0
// operator uses the Q4 pattern values, as the persistent Jacobi kernel does).  Every reduction
// is a fixed-order sum of per-CTA partials that every CTA evaluates identically, so all CTAs
// take the same convergence branch.  Cross-CTA data written inside the kernel is read with
// ld.cg (L2); the constant operator data (stencils, D^-1, masks, alpha, inverse) with ld.nc.
#include <atomic>
#include <cooperative_groups.h>

#include "cgcg2d.cuh"
#include "mg.cuh"
#include "plan.cuh"

namespace tb {

constexpr int kMgpThreads = 512;
constexpr int kMgpMaxLv = 16;

struct MgpLevel {
  Grid g;
  const double* st;       // half stencil (levels >= 1)
  const uint8_t* fixed;   // Dirichlet mask
  const double* dinv;     // Jacobi inverse diagonal (0 on fixed)
  double *xa, *xb, *b, *res;  // sweep ping-pong (final iterate in xb), right-hand side, residual
};

struct MgpArgs {
  MgpLevel L[kMgpMaxLv];
  int nlev, nu;  // levels; smoothing sweeps per side (1 or 2)
  int fused;     // V(1,1) in tiled fused phases (TB_MGP_UNFUSED=1: one phase per operation)
  int64_t ncoarse;
  double omega;
  const double* ainv;   // coarsest dense inverse
  const double* alpha;  // level-0 element scales
  double *x, *r, *pa, *pb, *q;
  PcgState* st;
  double* part;         // [3][gridDim.x]: p.q, r.r, r.z partials
  unsigned int* bar;
};

// Diagnostics (TB_MGP_PROF builds): CTA 0 accumulates %globaltimer spans per phase class.
__device__ unsigned long long g_mgp_prof[32];
#ifdef TB_MGP_PROF
__device__ __forceinline__ unsigned long long mgp_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define MGP_MARK(k)                                  \
  do {                                               \
    if (blockIdx.x == 0 && threadIdx.x == 0) {       \
      const unsigned long long t_ = mgp_now();       \
      g_mgp_prof[k] += t_ - prof_last;               \
      prof_last = t_;                                \
    }                                                \
  } while (0)
#else
#define MGP_MARK(k) \
  do {              \
  } while (0)
#endif

struct Rng {
  int64_t start, stride;
};

__device__ __forceinline__ Rng grid_rng() {
  return {(int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x};
}
__device__ __forceinline__ Rng cta_rng() { return {threadIdx.x, blockDim.x}; }

// y_n = (A_l v)_n.  Level 0: matrix-free alpha_e K_e (node-owner slots, as k_node_apply);
// coarse levels: half stencil (as k_mg_sapply).  v was written inside this kernel: L2 loads.
// Every load is unconditional (out-of-grid neighbours read a clamped in-range address) and
// only the accumulation is predicated, so all loads of a node are in flight together; the sums
// are those of the graph path term by term.
// (The operand comes from a functor V(dx, dy, node, out[2]) -- offsets in {0,1,2} around
// (i, j) -- reading the stored vector or, in the fused phases, a shared-memory tile.)
template <bool L0, class VF>
__device__ __forceinline__ void mgp_apply_f(const MgpLevel& L, const Q4Pat& K, const double* __restrict__ alpha,
                                            int n, const VF& V, double (&out)[2]) {
  const Grid& g = L.g;
  const int i = (int)(n % g.nnx), j = (int)(n / g.nnx);
  if (L0) {
    double P[9][2];
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const int ii = i + dx - 1, jj = j + dy - 1;
        const bool ok = ii >= 0 && ii < g.nnx && jj >= 0 && jj < g.nny;
        const int64_t node = ok ? (int64_t)jj * g.nnx + ii : n;
        double vv[2];
        V(dx, dy, node, vv);
        P[dy * 3 + dx][0] = ok ? vv[0] : 0.0;
        P[dy * 3 + dx][1] = ok ? vv[1] : 0.0;
      }
    double a[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int ei = i - 1 + (s & 1), ej = j - 1 + (s >> 1);
      const bool ok = ei >= 0 && ei < g.nx && ej >= 0 && ej < g.ny;
      const double av = __ldg(alpha + (ok ? (int64_t)ej * g.nx + ei : 0));
      a[s] = ok ? av : 0.0;
    }
    node_rows_pat<2>(K, P, a, out);
  } else {
    out[0] = out[1] = 0.0;
    const int64_t N = g.n_nodes;
#pragma unroll
    for (int m = 0; m < 9; ++m) {
      const int ni = i + m % 3 - 1, nj = j + m / 3 - 1;
      const bool ok = ni >= 0 && ni < g.nnx && nj >= 0 && nj < g.nny;
      const int64_t nbn = ok ? (int64_t)nj * g.nnx + ni : n;
      double vv[2];
      V(m % 3, m / 3, nbn, vv);
      const double v0 = vv[0], v1 = vv[1];
      const double* s = (m >= 4) ? L.st + (int64_t)(m - 4) * 4 * N + n : L.st + (int64_t)(4 - m) * 4 * N + nbn;
      const double s0 = __ldg(s), s1 = __ldg(s + N), s2 = __ldg(s + 2 * N), s3 = __ldg(s + 3 * N);
      if (ok) {
        if (m >= 4) {
          out[0] = fma(s1, v1, fma(s0, v0, out[0]));
          out[1] = fma(s3, v1, fma(s2, v0, out[1]));
        } else {  // transpose of the neighbour's block towards this node
          out[0] = fma(s2, v1, fma(s0, v0, out[0]));
          out[1] = fma(s3, v1, fma(s1, v0, out[1]));
        }
      }
    }
  }
}

// y_n = (A_l v)_n for a stored vector v (written inside this kernel: L2 loads)
template <bool L0>
__device__ __forceinline__ void mgp_apply(const MgpLevel& L, const Q4Pat& K, const double* __restrict__ alpha,
                                          int n, const double* v, double (&out)[2]) {
  auto V = [v](int, int, int64_t node, double (&vv)[2]) {
    vv[0] = __ldcg(v + 2 * node);
    vv[1] = __ldcg(v + 2 * node + 1);
  };
  mgp_apply_f<L0>(L, K, alpha, n, V, out);
}

// out = in + omega D^-1 (b - A in)   (in == nullptr: out = omega D^-1 b)
template <bool L0>
__device__ __noinline__ void mgp_sweep(const MgpLevel& L, const Q4Pat K, const double* alpha, double omega,
                                       const double* in, double* out, Rng rg) {
#pragma unroll(L0 ? 2 : 1)
  for (int n = (int)rg.start; n < (int)L.g.n_nodes; n += (int)rg.stride) {
    double y[2] = {0.0, 0.0};
    if (in != nullptr) mgp_apply<L0>(L, K, alpha, n, in, y);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int64_t d = 2 * n + c;
      const double bd = __ldcg(L.b + d);
      const double di = __ldg(L.dinv + d);
      out[d] = (in != nullptr) ? __ldcg(in + d) + omega * di * (bd - y[c]) : omega * di * bd;
    }
  }
}

// res = b - A x on free dofs, 0 on fixed
template <bool L0>
__device__ __noinline__ void mgp_resid(const MgpLevel& L, const Q4Pat K, const double* alpha, const double* x,
                                       Rng rg) {
#pragma unroll(L0 ? 2 : 1)
  for (int n = (int)rg.start; n < (int)L.g.n_nodes; n += (int)rg.stride) {
    double y[2];
    mgp_apply<L0>(L, K, alpha, n, x, y);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int64_t d = 2 * n + c;
      L.res[d] = (__ldg(L.dinv + d) != 0.0) ? __ldcg(L.b + d) - y[c] : 0.0;
    }
  }
}

__device__ __forceinline__ double mgp_pw(int i, int I, int nf) {
  if (i < 0 || i > nf) return 0.0;
  if (!(i & 1)) return (i >> 1) == I ? 1.0 : 0.0;
  if (i == nf) return ((nf + 1) >> 1) == I ? 1.0 : 0.0;
  return ((i >> 1) == I || (i >> 1) + 1 == I) ? 0.5 : 0.0;
}

// b_c = P~^T res_f (full weighting, 0 on coarse fixed dofs); sweep1: xa_c = omega D_c^-1 b_c.
// Zero-weight taps read a clamped address and add w * r = +0 (the graph path skips them).
__device__ __noinline__ void mgp_restrict(const MgpLevel& C, const MgpLevel& F, double omega, bool sweep1,
                                          Rng rg) {
  const Grid& gc = C.g;
  const Grid& gf = F.g;
#pragma unroll 1
  for (int n = (int)rg.start; n < (int)gc.n_nodes; n += (int)rg.stride) {
    const int I = (int)(n % gc.nnx), J = (int)(n / gc.nnx);
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int fi = 2 * I + dx, fj = 2 * J + dy;
        const double w = mgp_pw(fi, I, gf.nx) * mgp_pw(fj, J, gf.ny);
        const int ci = min(max(fi, 0), gf.nx), cj = min(max(fj, 0), gf.ny);
        const int64_t fd = 2 * ((int64_t)cj * gf.nnx + ci);
        const double r0 = __ldcg(F.res + fd), r1 = __ldcg(F.res + fd + 1);
        if (w != 0.0) {
          acc[0] = fma(w, r0, acc[0]);
          acc[1] = fma(w, r1, acc[1]);
        }
      }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int64_t d = 2 * n + c;
      const double bc = __ldg(C.fixed + d) ? 0.0 : acc[c];
      C.b[d] = bc;
      if (sweep1) C.xa[d] = omega * __ldg(C.dinv + d) * bc;
    }
  }
}

// x_f += P~ xb_c on free fine dofs (bilinear interpolation; same summation order as
// k_mg_prolong_add, all four candidate coarse values loaded up front); xb_c = C's final iterate
__device__ __noinline__ void mgp_prolong(const MgpLevel& F, double* xf, const MgpLevel& C, Rng rg) {
  const Grid& gf = F.g;
  const Grid& gc = C.g;
#pragma unroll 1
  for (int n = (int)rg.start; n < (int)gf.n_nodes; n += (int)rg.stride) {
    const int i = (int)(n % gf.nnx), j = (int)(n / gf.nnx);
    int i0, ni, j0, nj;
    if (!(i & 1)) { i0 = i >> 1; ni = 1; } else if (i == gf.nx) { i0 = (gf.nx + 1) >> 1; ni = 1; } else { i0 = i >> 1; ni = 2; }
    if (!(j & 1)) { j0 = j >> 1; nj = 1; } else if (j == gf.ny) { j0 = (gf.ny + 1) >> 1; nj = 1; } else { j0 = j >> 1; nj = 2; }
    const double w = (ni == 2 ? 0.5 : 1.0) * (nj == 2 ? 0.5 : 1.0);
    const int i1 = min(i0 + 1, gc.nnx - 1), j1 = min(j0 + 1, gc.nny - 1);
    const int64_t c00 = 2 * ((int64_t)j0 * gc.nnx + i0), c01 = 2 * ((int64_t)j0 * gc.nnx + i1);
    const int64_t c10 = 2 * ((int64_t)j1 * gc.nnx + i0), c11 = 2 * ((int64_t)j1 * gc.nnx + i1);
    double v[4][2];
    v[0][0] = __ldcg(C.xb + c00), v[0][1] = __ldcg(C.xb + c00 + 1);
    v[1][0] = __ldcg(C.xb + c01), v[1][1] = __ldcg(C.xb + c01 + 1);
    v[2][0] = __ldcg(C.xb + c10), v[2][1] = __ldcg(C.xb + c10 + 1);
    v[3][0] = __ldcg(C.xb + c11), v[3][1] = __ldcg(C.xb + c11 + 1);
    const double x0 = __ldcg(xf + 2 * n), x1 = __ldcg(xf + 2 * n + 1);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      double acc = v[0][c];
      if (ni == 2) acc += v[1][c];
      if (nj == 2) {
        acc += v[2][c];
        if (ni == 2) acc += v[3][c];
      }
      const int64_t d = 2 * n + c;
      if (!__ldg(F.fixed + d)) xf[d] = fma(w, acc, c ? x1 : x0);
    }
  }
}

// ---------------------------------------------------------------------------------------
// Tiled fused phases of the V(1,1) cycle (one grid barrier fewer per level and direction).
// R: residual of level F + restriction to level C.  A CTA takes a tile of kRtX x kRtY coarse
//    nodes, stages the fine iterate around it in shared memory, evaluates the fine residuals of
//    the tile's (2 kRtX + 1) x (2 kRtY + 1) restriction taps from there (~10% recomputed at tile
//    seams), then restricts.
// PS: prolongation + post-smoothing sweep.  A CTA takes a tile of kPtX x kPtY fine nodes, stages
//    the prolongated iterate x + P~ xb_c on the tile and its halo, then sweeps from there.
// The per-dof arithmetic is that of mgp_resid / mgp_restrict / mgp_prolong / mgp_sweep, so the
// iterates are bitwise those of the phase-per-operation form.
#ifndef TB_MGP_RTY
#define TB_MGP_RTY 8
#endif
#ifndef TB_MGP_PTY
#define TB_MGP_PTY 16
#endif
constexpr int kRtX = 16, kRtY = TB_MGP_RTY;              // coarse tile of R
constexpr int kRfX = 2 * kRtX + 1, kRfY = 2 * kRtY + 1;  // fine residual taps (33 x 17)
constexpr int kRxX = kRfX + 2, kRxY = kRfY + 2;          // fine iterate around them (35 x 19)
constexpr int kPtX = 32, kPtY = TB_MGP_PTY;              // fine tile of PS (one node per thread at 16)
constexpr int kPiX = kPtX + 2, kPiY = kPtY + 2;          // prolongated iterate incl. halo
constexpr int kTileX = (kRxX * kRxY > kPiX * kPiY) ? kRxX * kRxY : kPiX * kPiY;  // doubles x 2

template <bool L0F>
__device__ __noinline__ void mgp_tile_R(const MgpLevel& C, const MgpLevel& F, const Q4Pat K, const double* alpha,
                                        const double* xf, double omega, bool sweep1, double* tx, double* tr) {
  const Grid& gc = C.g;
  const Grid& gf = F.g;
  const int ntx = (gc.nnx + kRtX - 1) / kRtX, nty = (gc.nny + kRtY - 1) / kRtY;
  const int t = threadIdx.x, nt = blockDim.x;
#pragma unroll 1
  for (int tile = blockIdx.x; tile < ntx * nty; tile += gridDim.x) {
    const int I0 = (tile % ntx) * kRtX, J0 = (tile / ntx) * kRtY;
    const int fx0 = 2 * I0 - 1, fy0 = 2 * J0 - 1;  // fine origin of the taps
    for (int q = t; q < kRxX * kRxY; q += nt) {
      const int gi = fx0 - 1 + q % kRxX, gj = fy0 - 1 + q / kRxX;
      const bool ok = gi >= 0 && gi < gf.nnx && gj >= 0 && gj < gf.nny;
      const int64_t node = ok ? (int64_t)gj * gf.nnx + gi : 0;
      tx[2 * q] = ok ? __ldcg(xf + 2 * node) : 0.0;
      tx[2 * q + 1] = ok ? __ldcg(xf + 2 * node + 1) : 0.0;
    }
    __syncthreads();
    for (int q = t; q < kRfX * kRfY; q += nt) {
      const int li = q % kRfX, lj = q / kRfX;
      const int gi = fx0 + li, gj = fy0 + lj;
      double r[2] = {0.0, 0.0};
      if (gi >= 0 && gi < gf.nnx && gj >= 0 && gj < gf.nny) {
        const int fn = gj * gf.nnx + gi;
        auto V = [&](int dx, int dy, int64_t, double (&vv)[2]) {
          const int idx = 2 * ((lj + dy) * kRxX + li + dx);
          vv[0] = tx[idx];
          vv[1] = tx[idx + 1];
        };
        double y[2];
        mgp_apply_f<L0F>(F, K, alpha, fn, V, y);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int64_t d = 2 * (int64_t)fn + c;
          r[c] = (__ldg(F.dinv + d) != 0.0) ? __ldcg(F.b + d) - y[c] : 0.0;
        }
      }
      tr[2 * q] = r[0];
      tr[2 * q + 1] = r[1];
    }
    __syncthreads();
    for (int q = t; q < kRtX * kRtY; q += nt) {
      const int I = I0 + q % kRtX, J = J0 + q / kRtX;
      if (I < gc.nnx && J < gc.nny) {
        double acc[2] = {0.0, 0.0};
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
          for (int dx = -1; dx <= 1; ++dx) {
            const int fi = 2 * I + dx, fj = 2 * J + dy;
            const double w = mgp_pw(fi, I, gf.nx) * mgp_pw(fj, J, gf.ny);
            if (w != 0.0) {
              const int idx = 2 * ((fj - fy0) * kRfX + fi - fx0);
              acc[0] = fma(w, tr[idx], acc[0]);
              acc[1] = fma(w, tr[idx + 1], acc[1]);
            }
          }
        const int64_t n = (int64_t)J * gc.nnx + I;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int64_t d = 2 * n + c;
          const double bc = __ldg(C.fixed + d) ? 0.0 : acc[c];
          C.b[d] = bc;
          if (sweep1) C.xa[d] = omega * __ldg(C.dinv + d) * bc;
        }
      }
    }
    __syncthreads();  // the tiles are reused by the next tile
  }
}

// prolongated iterate at fine node (i, j): x_f + P~ xb_c on free dofs (mgp_prolong's arithmetic)
__device__ __forceinline__ void mgp_prolonged(const MgpLevel& F, const double* xf, const MgpLevel& C, int i, int j,
                                              double (&out)[2]) {
  const Grid& gf = F.g;
  const Grid& gc = C.g;
  const int64_t m = (int64_t)j * gf.nnx + i;
  int i0, ni, j0, nj;
  if (!(i & 1)) { i0 = i >> 1; ni = 1; } else if (i == gf.nx) { i0 = (gf.nx + 1) >> 1; ni = 1; } else { i0 = i >> 1; ni = 2; }
  if (!(j & 1)) { j0 = j >> 1; nj = 1; } else if (j == gf.ny) { j0 = (gf.ny + 1) >> 1; nj = 1; } else { j0 = j >> 1; nj = 2; }
  const double w = (ni == 2 ? 0.5 : 1.0) * (nj == 2 ? 0.5 : 1.0);
  const int i1 = min(i0 + 1, gc.nnx - 1), j1 = min(j0 + 1, gc.nny - 1);
  const int64_t c00 = 2 * ((int64_t)j0 * gc.nnx + i0), c01 = 2 * ((int64_t)j0 * gc.nnx + i1);
  const int64_t c10 = 2 * ((int64_t)j1 * gc.nnx + i0), c11 = 2 * ((int64_t)j1 * gc.nnx + i1);
  double v[4][2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    v[0][c] = __ldcg(C.xb + c00 + c);
    v[1][c] = __ldcg(C.xb + c01 + c);
    v[2][c] = __ldcg(C.xb + c10 + c);
    v[3][c] = __ldcg(C.xb + c11 + c);
  }
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const double x0 = __ldcg(xf + 2 * m + c);
    double acc = v[0][c];
    if (ni == 2) acc += v[1][c];
    if (nj == 2) {
      acc += v[2][c];
      if (ni == 2) acc += v[3][c];
    }
    out[c] = __ldg(F.fixed + 2 * m + c) ? x0 : fma(w, acc, x0);
  }
}

// RZ: level 0 (z = out): accumulate r.z of the dofs written (the reduction that follows)
template <bool L0F>
__device__ __noinline__ void mgp_tile_PS(const MgpLevel& F, const double* xf, double* out, const MgpLevel& C,
                                         const Q4Pat K, const double* alpha, double omega, double* tin,
                                         double* rz) {
  const Grid& gf = F.g;
  const int ntx = (gf.nnx + kPtX - 1) / kPtX, nty = (gf.nny + kPtY - 1) / kPtY;
  const int t = threadIdx.x, nt = blockDim.x;
#pragma unroll 1
  for (int tile = blockIdx.x; tile < ntx * nty; tile += gridDim.x) {
    const int i0 = (tile % ntx) * kPtX, j0 = (tile / ntx) * kPtY;
    for (int q = t; q < kPiX * kPiY; q += nt) {
      const int gi = i0 - 1 + q % kPiX, gj = j0 - 1 + q / kPiX;
      double v[2] = {0.0, 0.0};
      if (gi >= 0 && gi < gf.nnx && gj >= 0 && gj < gf.nny) mgp_prolonged(F, xf, C, gi, gj, v);
      tin[2 * q] = v[0];
      tin[2 * q + 1] = v[1];
    }
    __syncthreads();
    for (int q = t; q < kPtX * kPtY; q += nt) {
      const int li = q % kPtX, lj = q / kPtX;
      const int gi = i0 + li, gj = j0 + lj;
      if (gi < gf.nnx && gj < gf.nny) {
        const int n = gj * gf.nnx + gi;
        auto V = [&](int dx, int dy, int64_t, double (&vv)[2]) {
          const int idx = 2 * ((lj + dy) * kPiX + li + dx);
          vv[0] = tin[idx];
          vv[1] = tin[idx + 1];
        };
        double y[2];
        mgp_apply_f<L0F>(F, K, alpha, n, V, y);
        const int self = 2 * ((lj + 1) * kPiX + li + 1);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int64_t d = 2 * (int64_t)n + c;
          const double o = tin[self + c] + omega * __ldg(F.dinv + d) * (__ldcg(F.b + d) - y[c]);
          out[d] = o;
          if (rz != nullptr) *rz = fma(__ldcg(F.b + d), o, *rz);
        }
      }
    }
    __syncthreads();
  }
}

// xb_c = Ainv b_c, one warp per row over the grid (fixed-order lane partials)
__device__ __forceinline__ void mgp_dense(const MgpLevel& C, const double* __restrict__ ainv, int64_t n) {
  const int lane = threadIdx.x & 31;
  const int w = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), nw = (int)((gridDim.x * blockDim.x) >> 5);
  const double* A = ainv;
#pragma unroll 1
  for (int r = w; r < (int)n; r += nw) {
    double s = 0.0;
#pragma unroll 4
    for (int c = lane; c < (int)n; c += 32) s = fma(A[r * n + c], __ldcg(C.b + c), s);
    s = warp_sum(s);
    if (lane == 0) C.xb[r] = s;
  }
}

// fixed-order sum of the per-CTA partials of slot k; every warp computes it identically
__device__ __forceinline__ double mgp_sum(const double* part, int k) {
  // warp 0 alone reads the partials (every warp reading them made 16x the L2 requests on the
  // same lines) and broadcasts the fixed-order sum through shared memory
  __shared__ double bc;
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += __ldcg(part + k * gridDim.x + b);
    s = warp_sum(s);
    if (threadIdx.x == 0) bc = s;
  }
  __syncthreads();
  const double v = bc;
  __syncthreads();  // bc is rewritten by the next reduction
  return v;
}

__global__ void __launch_bounds__(kMgpThreads, 1) k_mgpcg2d(Q4Pat K, MgpArgs a) {
  __shared__ MgpLevel sL[kMgpMaxLv];
  __shared__ double s_tx[2 * kTileX];            // fused phases: staged fine iterate
  __shared__ double s_tr[2 * kRfX * kRfY];       // fused restriction: fine residual taps
  for (int l = threadIdx.x; l < a.nlev; l += blockDim.x) sL[l] = a.L[l];
  __syncthreads();
  PcgState* st = a.st;
  if (st->done != 0) return;
  const double omega = a.omega, tol2 = st->tol2;
  const int maxit = st->maxit;
  int it = st->iters;
  double rz = 0.0, rr = st->rr, beta = 0.0, alpha = 0.0, pq = 0.0;
  int done = 0;
  const int nlev = a.nlev, lg = nlev - 1;  // grid levels 0 .. nlev-2, then the dense coarsest
  const int nu = a.nu;
  const bool fused = a.fused != 0;
  const double* alpha_e = a.alpha;
  double* x = a.x;
  double* r = a.r;
  double* q = a.q;
  double* part = a.part;
  unsigned int* bar = a.bar;
  const Rng G = grid_rng();
  const Grid g0 = sL[0].g;
  const double* dinv0 = sL[0].dinv;
  double* xa0 = sL[0].xa;
  double* z = sL[0].xb;
  const int64_t N0 = g0.n_nodes;
#ifdef TB_MGP_PROF
  unsigned long long prof_last = (blockIdx.x == 0 && threadIdx.x == 0) ? mgp_now() : 0ull;
#endif

  for (bool first = true;; first = false) {
    if (first) {
      // initial preconditioned residual: first sweep from zero on b = r (k_pcg_start set pa = 0)
      mgp_sweep<true>(sL[0], K, alpha_e, omega, nullptr, xa0, G);
      grid_sync_flip(bar);
    } else {
      const double* pold = (it & 1) ? a.pb : a.pa;
      double* pnew = (it & 1) ? a.pa : a.pb;
      // ---- A: p = z + beta p_old, q = K p, p.q
      double acc[1] = {0.0};
#pragma unroll 2
      for (int n = (int)G.start; n < (int)N0; n += (int)G.stride) {
        const int i = (int)(n % g0.nnx), j = (int)(n / g0.nnx);
        double P[9][2];
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) {
            const int ii = i + dx - 1, jj = j + dy - 1;
            const bool ok = ii >= 0 && ii < g0.nnx && jj >= 0 && jj < g0.nny;
            const int64_t node = (int64_t)jj * g0.nnx + ii;
#pragma unroll
            for (int c = 0; c < 2; ++c)
              P[dy * 3 + dx][c] = ok ? fma(beta, __ldcg(pold + 2 * node + c), __ldcg(z + 2 * node + c)) : 0.0;
          }
        double sc[4], out[2];
        slot_scales<2, true>(g0, i, j, 0, alpha_e, sc);
        node_rows_pat<2>(K, P, sc, out);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          pnew[2 * n + c] = P[4][c];
          q[2 * n + c] = out[c];
          acc[0] = fma(P[4][c], out[c], acc[0]);
        }
      }
      publish_partials_grid_sync<1>(acc, part, bar, false);
      pq = mgp_sum(part, 0);
      MGP_MARK(0);
      if (!(pq > 0.0) || !isfinite(pq)) {
        done = 3;
        break;
      }
      alpha = rz / pq;
      // ---- B: x, r update, r.r, first pre-smoothing sweep of level 0 (b = r)
      acc[0] = 0.0;
#pragma unroll 2
      for (int n = (int)G.start; n < (int)N0; n += (int)G.stride)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int64_t d = 2 * n + c;
          const double di = __ldg(dinv0 + d);
          double rd = __ldcg(r + d);
          if (di != 0.0) {
            x[d] = fma(alpha, __ldcg(pnew + d), __ldcg(x + d));
            rd = fma(-alpha, __ldcg(q + d), rd);
            r[d] = rd;
            acc[0] = fma(rd, rd, acc[0]);
          }
          xa0[d] = omega * di * rd;
        }
      publish_partials_grid_sync<1>(acc, part + gridDim.x, bar, false);
      rr = mgp_sum(part, 1);
      MGP_MARK(1);
      ++it;
      if (!isfinite(rr)) done = 3;
      else if (rr <= tol2) done = 1;
      else if (it >= maxit) done = 2;
      if (done) break;
    }
    // ---- rest of the V-cycle: z = M^-1 r.  V(nu, nu), nu in {1, 2}: the pre-smoothed iterate
    // is xa (nu = 1) or xb (nu = 2); the final iterate of every level ends in xb.
    double rzn;
    if (nu == 1 && fused) {
      // V(1,1) in tiled fused phases (see mgp_tile_R / mgp_tile_PS): 12 grid barriers per
      // iteration instead of 19
      for (int l = 1; l <= lg; ++l) {  // level lg = the dense coarsest (no pre-smoothing there)
        if (l == 1) mgp_tile_R<true>(sL[1], sL[0], K, alpha_e, sL[0].xa, omega, l < lg, s_tx, s_tr);
        else mgp_tile_R<false>(sL[l], sL[l - 1], K, alpha_e, sL[l - 1].xa, omega, l < lg, s_tx, s_tr);
        grid_sync_flip(bar);
        MGP_MARK(8 + l - 1);
      }
      mgp_dense(sL[nlev - 1], a.ainv, a.ncoarse);
      MGP_MARK(3);
      grid_sync_flip(bar);
      double rzp[1] = {0.0};
      for (int l = lg - 1; l >= 0; --l) {
        MgpLevel& L = sL[l];
        if (l == 0) {
          mgp_tile_PS<true>(L, L.xa, L.xb, sL[1], K, alpha_e, omega, s_tx, &rzp[0]);  // z = xb of level 0
        } else {
          mgp_tile_PS<false>(L, L.xa, L.xb, sL[l + 1], K, alpha_e, omega, s_tx, nullptr);
          grid_sync_flip(bar);
        }
        MGP_MARK(16 + l);
      }
      publish_partials_grid_sync<1>(rzp, part + 2 * gridDim.x, bar, false);
      rzn = mgp_sum(part, 2);
    } else {
    // ---- rest of the V-cycle: z = M^-1 r.  V(nu, nu), nu in {1, 2}: the pre-smoothed iterate
    // is xa (nu = 1) or xb (nu = 2); the final iterate of every level ends in xb.
    for (int l = 0; l < lg; ++l) {
      MgpLevel& L = sL[l];
      if (l > 0) {
        mgp_restrict(L, sL[l - 1], omega, true, G);
        grid_sync_flip(bar);
      }
      if (nu == 2) {
        if (l == 0) mgp_sweep<true>(L, K, alpha_e, omega, L.xa, L.xb, G);
        else mgp_sweep<false>(L, K, alpha_e, omega, L.xa, L.xb, G);
        grid_sync_flip(bar);
      }
      const double* pre = (nu == 2) ? L.xb : L.xa;
      if (l == 0) mgp_resid<true>(L, K, alpha_e, pre, G);
      else mgp_resid<false>(L, K, alpha_e, pre, G);
      grid_sync_flip(bar);
      MGP_MARK(8 + l);
    }
    // coarsest: restriction, then x = Ainv b with one warp per row over the whole grid
    mgp_restrict(sL[nlev - 1], sL[nlev - 2], omega, false, G);
    grid_sync_flip(bar);
    mgp_dense(sL[nlev - 1], a.ainv, a.ncoarse);
    MGP_MARK(3);
    grid_sync_flip(bar);
    for (int l = lg - 1; l >= 0; --l) {
      MgpLevel& L = sL[l];
      double* pre = (nu == 2) ? L.xb : L.xa;
      mgp_prolong(L, pre, sL[l + 1], G);
      grid_sync_flip(bar);
      if (nu == 2) {
        if (l == 0) mgp_sweep<true>(L, K, alpha_e, omega, L.xb, L.xa, G);
        else mgp_sweep<false>(L, K, alpha_e, omega, L.xb, L.xa, G);
        grid_sync_flip(bar);
      }
      if (l == 0) {
        mgp_sweep<true>(L, K, alpha_e, omega, L.xa, L.xb, G);  // z = xb of level 0
      } else {
        mgp_sweep<false>(L, K, alpha_e, omega, L.xa, L.xb, G);
        grid_sync_flip(bar);
      }
      MGP_MARK(16 + l);
    }
    // ---- r.z (z = xb of level 0, this thread's own dofs)
    double rzp[1] = {0.0};
#pragma unroll 1
    for (int n = (int)G.start; n < (int)N0; n += (int)G.stride)
#pragma unroll
      for (int c = 0; c < 2; ++c) rzp[0] = fma(__ldcg(r + 2 * n + c), __ldcg(z + 2 * n + c), rzp[0]);
    publish_partials_grid_sync<1>(rzp, part + 2 * gridDim.x, bar, false);
    rzn = mgp_sum(part, 2);
    }
    MGP_MARK(16);
    beta = first ? 0.0 : rzn / rz;
    rz = rzn;
    if (!(rzn > 0.0)) done = (rzn == 0.0 && rr == 0.0) ? 1 : 3;
    if (done) break;
  }
#ifdef TB_MGP_PROF
  if (blockIdx.x == 0 && threadIdx.x == 0) g_mgp_prof[31] += 1;
#endif
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->iters = it;
    st->rr = rr;
    st->rz = rz;
    st->pq = pq;
    st->alpha = alpha;
    st->beta = beta;
    st->done = done;
  }
}

// Launch for the plan's current hierarchy (after mg_setup) from the state k_pcg_start left:
// x, r, pa = 0, st (tol2, maxit, iters, rr).  Returns false when the device cannot co-schedule
// the grid (caller uses the graph path).
bool mg_pcg2d_persistent(tb_plan_impl* P, PcgWork& w, cudaStream_t s) {
  Mg& mg = P->mg;
  if (P->g.dim != 2 || !P->pat_ok || mg.lv.size() < 2 || (int)mg.lv.size() > kMgpMaxLv) return false;
  if (mg.nu != 1 && mg.nu != 2) return false;
  if (getenv("TB_NO_PERSIST") != nullptr) return false;  // tests: the graph path
  // co-residency grid per device (a process may hold plans on several GPUs); racing first
  // calls compute the same value
  static std::atomic<int> grids[64];  // grid + 1; 0 = not computed yet
  const int dev = (P->device >= 0 && P->device < 64) ? P->device : 0;
  int grid = grids[dev].load() - 1;
  if (grid < 0) {
    int sms = 0, coop = 0, occ = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mgpcg2d, kMgpThreads, 0);
    grid = (coop && occ >= 1) ? sms : 0;
    grids[dev].store(grid + 1);
  }
  if (grid <= 0 || 2 * w.part_stride < 3 * grid) return false;
  MgpArgs a{};
  a.nlev = (int)mg.lv.size();
  a.nu = mg.nu;
  a.fused = getenv("TB_MGP_UNFUSED") == nullptr ? 1 : 0;
  for (int l = 0; l < a.nlev; ++l) {
    const MgLevel& L = mg.lv[l];
    MgpLevel& d = a.L[l];
    d.g = L.g;
    d.st = L.st;
    d.fixed = L.fixed;
    d.dinv = L.dinv;
    d.xa = L.x;
    d.xb = L.t;
    d.b = L.b;
    d.res = L.r;
  }
  a.L[0].b = w.r;   // the V-cycle's level-0 right-hand side is the pCG residual
  a.L[0].xb = w.z;  // and its result is z
  a.L[0].dinv = w.dinv;
  a.ncoarse = mg.ncoarse;
  a.omega = mg.omega;
  a.ainv = mg.ainv;
  a.alpha = P->d_alpha;
  a.x = w.x;
  a.r = w.r;
  a.pa = w.pa;
  a.pb = w.pb;
  a.q = w.q;
  a.st = w.st;
  a.part = w.part;
  a.bar = reinterpret_cast<unsigned int*>(w.barrier);
  void* args[] = {(void*)&P->pat, (void*)&a};
  if (cudaLaunchCooperativeKernel((const void*)k_mgpcg2d, grid, kMgpThreads, args, 0, s) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  launched(1);
  return true;
}

}  // namespace tb

// Diagnostics: read and clear the per-phase timers of a TB_MGP_PROF build (zeros otherwise).
extern "C" int tb_mgp_prof_read(unsigned long long* out32) {
  if (out32 == nullptr) return 1;
  if (cudaMemcpyFromSymbol(out32, tb::g_mgp_prof, sizeof(unsigned long long) * 32) != cudaSuccess) return 2;
  static const unsigned long long zeros[32] = {};
  if (cudaMemcpyToSymbol(tb::g_mgp_prof, zeros, sizeof(zeros)) != cudaSuccess) return 2;
  return 0;
}
