// Matrix-free structured-grid Q1 kernels (Q4 in 2D, Hex8 in 3D), fp64.
//
// Node-owner gather formulation: thread t owns node n and sums, in a fixed slot
// order, the rows of every adjacent element's  a_e * K_e * v_e  that belong to n.
// No atomics, no assembled matrix, bit-reproducible.  Replaces the reference's
// element scatter  np.bincount(elem_dofs, (v[elem_dofs] @ K_e^T) * alpha)
// (hdm.py:224-233, rom.py:309-317) and the assembled-CSC SpMV behind SuperLU
// (fem.py:357-409).
#pragma once

#include "common.cuh"

namespace tb {

// Local node numbering inside an element (fem.py:225; 3D: bottom face then top face).
__host__ __device__ constexpr int loc_of(int ox, int oy, int oz) {
  return (oy ? (ox ? 2 : 3) : (ox ? 1 : 0)) + 4 * oz;
}
__host__ __device__ constexpr int offx(int b) { return ((b & 3) == 1 || (b & 3) == 2) ? 1 : 0; }
__host__ __device__ constexpr int offy(int b) { return ((b & 3) >= 2) ? 1 : 0; }
__host__ __device__ constexpr int offz(int b) { return b >> 2; }

template <int D>
struct Q1 {
  static constexpr int NN = 1 << D;              // nodes per element
  static constexpr int NB = (D == 2) ? 9 : 27;   // node neighbourhood
};

__device__ __forceinline__ void node_coords(const Grid& g, int64_t n, int& i, int& j, int& k) {
  i = (int)(n % g.nnx);
  int64_t t = n / g.nnx;
  j = (int)(t % g.nny);
  k = (int)(t / g.nny);
}

// Gather the 3^D neighbourhood of node (i,j,k) of a vector with NC interleaved components.
// Out-of-grid neighbours read as 0.  When FUSED: value = z + beta * pold (the pCG
// direction update folded into the operator pass).
template <int D, int NC, bool FUSED>
__device__ __forceinline__ void gather_nbhd(const Grid& g, int i, int j, int k, const double* __restrict__ v,
                                            const double* __restrict__ pold, double beta,
                                            double (&P)[Q1<D>::NB][NC]) {
#pragma unroll
  for (int dz = 0; dz < (D == 3 ? 3 : 1); ++dz)
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const int nb = (dz * 3 + dy) * 3 + dx;
        const int ii = i + dx - 1, jj = j + dy - 1, kk = (D == 3) ? k + dz - 1 : 0;
        const bool ok = ii >= 0 && ii < g.nnx && jj >= 0 && jj < g.nny && kk >= 0 && kk < g.nnz;
        const int64_t node = ((int64_t)kk * g.nny + jj) * g.nnx + ii;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          double val = 0.0;
          if (ok) {
            val = __ldg(v + NC * node + c);
            if (FUSED) val = fma(beta, __ldg(pold + NC * node + c), val);
          }
          P[nb][c] = val;
        }
      }
}

// Per-slot element scale: alpha_e (SCALED) or 1, and 0 for slots outside the grid.
template <int D, bool SCALED>
__device__ __forceinline__ void slot_scales(const Grid& g, int i, int j, int k, const double* __restrict__ alpha,
                                            double (&a)[Q1<D>::NN]) {
#pragma unroll
  for (int s = 0; s < Q1<D>::NN; ++s) {
    const int ei = i - 1 + (s & 1), ej = j - 1 + ((s >> 1) & 1), ek = (D == 3) ? k - 1 + (s >> 2) : 0;
    const bool ok = ei >= 0 && ei < g.nx && ej >= 0 && ej < g.ny && ek >= 0 && ek < g.nz;
    double val = 0.0;
    if (ok) val = SCALED ? __ldg(alpha + ((int64_t)ek * g.ny + ej) * g.nx + ei) : 1.0;
    a[s] = val;
  }
}

// out[c] = sum_slots a_s * (K_e P_e)[row of this node, component c]
template <int D, int NC>
__device__ __forceinline__ void node_rows(const Mat<Q1<D>::NN * NC>& K, const double (&P)[Q1<D>::NB][NC],
                                          const double (&a)[Q1<D>::NN], double (&out)[NC]) {
  constexpr int NN = Q1<D>::NN, NE = NN * NC;
#pragma unroll
  for (int c = 0; c < NC; ++c) out[c] = 0.0;
#pragma unroll
  for (int s = 0; s < NN; ++s) {
    const int sx = s & 1, sy = (s >> 1) & 1, sz = s >> 2;
    const int L = loc_of(1 - sx, 1 - sy, (D == 3) ? 1 - sz : 0);
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
#pragma unroll
    for (int b = 0; b < NN; ++b) {
      const int nb = ((sz + offz(b)) * 3 + (sy + offy(b))) * 3 + (sx + offx(b));
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int cp = 0; cp < NC; ++cp) acc[c] = fma(K.v[(L * NC + c) * NE + b * NC + cp], P[nb][cp], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) out[c] = fma(a[s], acc[c], out[c]);
  }
}

// Q4 element matrices of the reference have a fixed value pattern (fem.py:41-70 elasticity:
// 6 distinct magnitudes for any nu; filtering.py Helmholtz r^2 S + M: 3 values).  With the
// pattern known at compile time the node rows need only the distinct values (kernel
// parameters) instead of 64 shared-memory reads of K per node.  Entry = sign(p) v[|p| - 1].
__host__ __device__ constexpr int q4_pat(int nc, int r, int q) {
  if (nc == 1) {
    const int d = r ^ q;  // corner pairs: 0 same, 1 / 3 edge-adjacent, 2 opposite
    return d == 0 ? 1 : (d == 2 ? 3 : 2);
  }
  constexpr int t[8][8] = {{1, 2, 3, 4, 5, -2, 6, -4},  {2, 1, -4, 6, -2, 5, 4, 3},
                           {3, -4, 1, -2, 6, 4, 5, 2},  {4, 6, -2, 1, -4, 3, 2, 5},
                           {5, -2, 6, -4, 1, 2, 3, 4},  {-2, 5, 4, 3, 2, 1, -4, 6},
                           {6, 4, 5, 2, 3, -4, 1, -2},  {-4, 3, 2, 5, 4, 6, -2, 1}};
  return t[r][q];
}
struct Q4Pat {
  double v[6];
};

// As node_rows<2, NC>, with K given by its pattern values.
template <int NC>
__device__ __forceinline__ void node_rows_pat(const Q4Pat& kp, const double (&P)[9][NC], const double (&a)[4],
                                              double (&out)[NC]) {
#pragma unroll
  for (int c = 0; c < NC; ++c) out[c] = 0.0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int sx = s & 1, sy = s >> 1;
    const int L = loc_of(1 - sx, 1 - sy, 0);
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int nb = (sy + offy(b)) * 3 + (sx + offx(b));
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int cp = 0; cp < NC; ++cp) {
          const int pt = q4_pat(NC, L * NC + c, b * NC + cp);
          acc[c] = pt > 0 ? fma(kp.v[pt - 1], P[nb][cp], acc[c]) : fma(-kp.v[-pt - 1], P[nb][cp], acc[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) out[c] = fma(a[s], acc[c], out[c]);
  }
}

// Host: extract the pattern values of a Q4 element matrix; false if K does not follow it.
inline bool q4_pattern_values(int nc, const double* K, Q4Pat* out) {
  const int ne = 4 * nc;
  double v[6] = {0, 0, 0, 0, 0, 0};
  bool set[6] = {false, false, false, false, false, false};
  double scale = 0.0;
  for (int i = 0; i < ne * ne; ++i) scale = fmax(scale, fabs(K[i]));
  for (int r = 0; r < ne; ++r)
    for (int q = 0; q < ne; ++q) {
      const int p = q4_pat(nc, r, q), k = (p > 0 ? p : -p) - 1;
      const double val = p > 0 ? K[r * ne + q] : -K[r * ne + q];
      if (!set[k]) {
        v[k] = val;
        set[k] = true;
      } else if (fabs(val - v[k]) > 1e-13 * scale) {
        return false;
      }
    }
  for (int k = 0; k < 6; ++k) out->v[k] = v[k];
  return true;
}

// y = K v  (rows with fixed[dof] != 0 zeroed when fixed != nullptr)
template <int D, int NC, bool SCALED, bool SIMP = false>
__global__ void __launch_bounds__(kBlock) k_node_apply(Grid g, Mat<Q1<D>::NN * NC> K, const double* __restrict__ alpha,
                                                       const double* __restrict__ v, double* __restrict__ y,
                                                       const uint8_t* __restrict__ fixed, double rho_l = 0.0) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.n_nodes) return;
  int i, j, k;
  node_coords(g, n, i, j, k);
  double P[Q1<D>::NB][NC];
  double a[Q1<D>::NN];
  gather_nbhd<D, NC, false>(g, i, j, k, v, nullptr, 0.0, P);
  slot_scales<D, SCALED>(g, i, j, k, alpha, a);
  if (SIMP) {  // `alpha` holds rho: alpha = rho_l + (1 - rho_l) rho^3 (k_material's operation order)
#pragma unroll
    for (int s = 0; s < Q1<D>::NN; ++s) {
      const int ei = i - 1 + (s & 1), ej = j - 1 + ((s >> 1) & 1), ek = (D == 3) ? k - 1 + (s >> 2) : 0;
      const bool ok = ei >= 0 && ei < g.nx && ej >= 0 && ej < g.ny && ek >= 0 && ek < g.nz;
      const double r = a[s];
      a[s] = ok ? rho_l + (1.0 - rho_l) * ((r * r) * r) : 0.0;
    }
  }
  double out[NC];
  node_rows<D, NC>(K, P, a, out);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double val = out[c];
    if (fixed != nullptr && fixed[NC * n + c]) val = 0.0;
    y[NC * n + c] = val;
  }
}

// pCG kernel A: pnew = z + beta*pold; q = K pnew (unmasked rows; pnew is 0 on fixed dofs);
// pq = pnew.q reduced deterministically; the last block sets alpha = rz/pq or flags breakdown.
template <int D, int NC, bool SCALED>
__global__ void __launch_bounds__(kBlock) k_pcg_fused(Grid g, Mat<Q1<D>::NN * NC> K, const double* __restrict__ alpha,
                                                      const double* __restrict__ z, const double* __restrict__ pold,
                                                      double* __restrict__ pnew, double* __restrict__ q,
                                                      PcgState* st, double* partials) {
  if (st->done) return;
  const double beta = st->beta;
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double pq[1] = {0.0};
  if (n < g.n_nodes) {
    int i, j, k;
    node_coords(g, n, i, j, k);
    double P[Q1<D>::NB][NC];
    double a[Q1<D>::NN];
    gather_nbhd<D, NC, true>(g, i, j, k, z, pold, beta, P);
    slot_scales<D, SCALED>(g, i, j, k, alpha, a);
    double out[NC];
    node_rows<D, NC>(K, P, a, out);
    constexpr int self = (D == 3) ? 13 : 4;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      pnew[NC * n + c] = P[self][c];
      q[NC * n + c] = out[c];
      if (k >= st->dot_k0 && k < st->dot_k1) pq[0] = fma(P[self][c], out[c], pq[0]);
    }
  }
  block_sum<1>(pq);
  if (publish_partials<1>(pq, partials, &st->count_a)) {
    gather_partials<1>(pq, partials, &st->count_a);
    if (threadIdx.x == 0) {
      const double v = pq[0];
      if (st->dist) {
        st->red[0] = v;
      } else if (!(v > 0.0) || !isfinite(v)) {
        st->done = 3;
      } else {
        st->pq = v;
        st->alpha = st->rz / v;
      }
    }
  }
}

// Jacobi inverse diagonal; 0 on fixed dofs (which also serves as the Dirichlet mask of the
// pCG update kernel).
template <int D, int NC, bool SCALED>
__global__ void __launch_bounds__(kBlock) k_node_dinv(Grid g, Mat<Q1<D>::NN * NC> K, const double* __restrict__ alpha,
                                                      const uint8_t* __restrict__ fixed, double* __restrict__ dinv) {
  constexpr int NN = Q1<D>::NN, NE = NN * NC;
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.n_nodes) return;
  int i, j, k;
  node_coords(g, n, i, j, k);
  double a[NN];
  slot_scales<D, SCALED>(g, i, j, k, alpha, a);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double d = 0.0;
#pragma unroll
    for (int s = 0; s < NN; ++s) {
      const int L = loc_of(1 - (s & 1), 1 - ((s >> 1) & 1), (D == 3) ? 1 - (s >> 2) : 0);
      d = fma(a[s], K.v[(L * NC + c) * NE + L * NC + c], d);
    }
    const bool fx = (fixed != nullptr) && fixed[NC * n + c];
    dinv[NC * n + c] = fx ? 0.0 : 1.0 / d;
  }
}

// element -> its 2^D node ids
template <int D>
__device__ __forceinline__ void elem_nodes(const Grid& g, int64_t e, int64_t (&nodes)[Q1<D>::NN]) {
  const int i = (int)(e % g.nx);
  const int64_t t = e / g.nx;
  const int j = (int)(t % g.ny);
  const int k = (int)(t / g.ny);
  const int64_t n0 = ((int64_t)k * g.nny + j) * g.nnx + i;
#pragma unroll
  for (int b = 0; b < Q1<D>::NN; ++b)
    nodes[b] = n0 + offx(b) + (int64_t)offy(b) * g.nnx + (int64_t)offz(b) * g.nnx * g.nny;
}

// s_e = drho_e - alpha'(rho_e) * u_e^T K_e lam_e   (hdm.py:211-222)
template <int D>
__global__ void __launch_bounds__(kBlock) k_elem_sensitivity(Grid g, Mat<Q1<D>::NN * D> K, double rho_l, double p,
                                                             const double* __restrict__ rho, const double* __restrict__ u,
                                                             const double* __restrict__ lam, const double* __restrict__ drho,
                                                             double* __restrict__ s) {
  constexpr int NN = Q1<D>::NN, NE = NN * D;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= g.n_elems) return;
  int64_t nodes[NN];
  elem_nodes<D>(g, e, nodes);
  double ue[NE], le[NE];
#pragma unroll
  for (int b = 0; b < NN; ++b)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      ue[b * D + c] = __ldg(u + D * nodes[b] + c);
      le[b * D + c] = __ldg(lam + D * nodes[b] + c);
    }
  // (u_e^T K_e) lam_e, column by column like the reference's (u_loc @ K_e) * lam_loc
  double c_ = 0.0;
#pragma unroll
  for (int b = 0; b < NE; ++b) {
    double col = 0.0;
#pragma unroll
    for (int a = 0; a < NE; ++a) col = fma(ue[a], K.v[a * NE + b], col);
    c_ = fma(col, le[b], c_);
  }
  const double r = rho[e];
  const double da = (1.0 - rho_l) * p * ((p == 3.0) ? r * r : pow(r, p - 1.0));
  const double base = (drho != nullptr) ? drho[e] : 0.0;
  s[e] = base - da * c_;
}

// Filter transfers (filtering.py:73-114): node value = scale * sum_{e∋n} val_e, and
// element value = scale * sum_{n∈e} val_n, both in fixed order.
template <int D>
__global__ void __launch_bounds__(kBlock) k_elem_to_node(Grid g, const double* __restrict__ ev, double pre, double post,
                                                         double* __restrict__ nv) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.n_nodes) return;
  int i, j, k;
  node_coords(g, n, i, j, k);
  double acc = 0.0;
#pragma unroll
  for (int s = 0; s < Q1<D>::NN; ++s) {
    const int ei = i - 1 + (s & 1), ej = j - 1 + ((s >> 1) & 1), ek = (D == 3) ? k - 1 + (s >> 2) : 0;
    if (ei >= 0 && ei < g.nx && ej >= 0 && ej < g.ny && ek >= 0 && ek < g.nz)
      acc += __ldg(ev + ((int64_t)ek * g.ny + ej) * g.nx + ei) * pre;
  }
  nv[n] = acc * post;
}

template <int D>
__global__ void __launch_bounds__(kBlock) k_node_to_elem(Grid g, const double* __restrict__ nv, double post,
                                                         double* __restrict__ ev) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= g.n_elems) return;
  const int i = (int)(e % g.nx);
  const int64_t t = e / g.nx;
  const int j = (int)(t % g.ny);
  const int k = (int)(t / g.ny);
  const int64_t n0 = ((int64_t)k * g.nny + j) * g.nnx + i;
  // ascending node-id order, the summation order of the reference's incidence^T matvec
  double acc = 0.0;
#pragma unroll
  for (int b = 0; b < Q1<D>::NN; ++b)
    acc += __ldg(nv + n0 + (b & 1) + (int64_t)((b >> 1) & 1) * g.nnx + (int64_t)(b >> 2) * g.nnx * g.nny);
  ev[e] = acc * post;
}

}  // namespace tb
