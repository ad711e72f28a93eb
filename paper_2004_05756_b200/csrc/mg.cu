// Geometric multigrid preconditioner (see mg.cuh).
#include <cusolverDn.h>

#include "cgcg2d.cuh"  // grid_sync_flip
#include "mg.cuh"
#include <utility>

#include "plan.cuh"

namespace tb {

static inline int nblk(int64_t n) { return (int)((n + kBlock - 1) / kBlock); }
constexpr int64_t kMgMinDofs = 600;     // stop coarsening below this many dofs (3D)
constexpr int64_t kMgMinDofs2D = 1200;  // 2D: cfg 2 stops at 1,092 dofs (19 V(1,1) iterations instead of 30
                                        // with a 320-dof coarsest level); its inverse comes from the
                                        // blocked Gauss-Jordan kernel below (cuSOLVER needed ~2 ms)
constexpr int kGjB = 16;                // Gauss-Jordan block size
constexpr int kGjMaxN = 1700;           // row block K (kGjB x n doubles) fits in shared memory
constexpr int64_t kMgMaxDense = 6144;   // coarsest level solved densely up to this size

__device__ __forceinline__ int64_t dof_of(const Grid& g, int i, int j, int k, int nc, int c) {
  return (((int64_t)k * g.nny + j) * g.nnx + i) * nc + c;
}

// Per-axis coarsening of nf fine elements into nc = (nf + 1) / 2 coarse ones: coarse node I sits
// on fine node min(2I, nf); when nf is odd the last coarse element spans a single fine element.
__host__ __device__ __forceinline__ int cnode(int I, int nf) { return 2 * I < nf ? 2 * I : nf; }
// position in [0,1] of fine node i inside coarse element I (i in [2I, 2I+2])
__host__ __device__ __forceinline__ double tpos(int i, int I, int nf) {
  return (i == nf && (nf & 1)) ? 1.0 : 0.5 * (i - 2 * I);
}
// prolongation weight of coarse node I at fine node i
__device__ __forceinline__ double pw(int i, int I, int nf) {
  if (i < 0 || i > nf) return 0.0;
  if (!(i & 1)) return (i >> 1) == I ? 1.0 : 0.0;
  if (i == nf) return ((nf + 1) >> 1) == I ? 1.0 : 0.0;
  return ((i >> 1) == I || (i >> 1) + 1 == I) ? 0.5 : 0.0;
}
// coarse nodes interpolated at fine node i: lo (and lo+1 when n == 2, weights 1/2)
__device__ __forceinline__ void pmap(int i, int nf, int& lo, int& n) {
  if (!(i & 1)) { lo = i >> 1; n = 1; }
  else if (i == nf) { lo = (nf + 1) >> 1; n = 1; }
  else { lo = i >> 1; n = 2; }
}

// ---------------------------------------------------------------------------------------
// Galerkin coarse element matrices.  One CTA per coarse element E; children e in {0,1}^D.
// R[o][O] = prod_d w((c_d + o_d)/2, O_d), w(t,0) = 1-t, w(t,1) = t (corners in local order).
// ---------------------------------------------------------------------------------------
template <int D, bool FIRST>
__global__ void __launch_bounds__(256) k_mg_aggregate(Grid gc, Grid gf, Mat<Q1<D>::NN * D> Ku,
                                                      const double* __restrict__ alpha,
                                                      const double* __restrict__ ke_f,
                                                      const uint8_t* __restrict__ fixed_f,
                                                      const uint8_t* __restrict__ fixed_c,
                                                      const uint8_t* __restrict__ dirty, double* __restrict__ ke_c) {
  constexpr int NN = Q1<D>::NN, NE = NN * D;
  __shared__ double Ke[NE * NE], T[NE * NE], Acc[NE * NE], R[NN * NN];
  __shared__ uint8_t mf[NE];
  const int t = threadIdx.x;
  const int64_t E = blockIdx.x;
  if (dirty != nullptr && !dirty[E]) return;  // done by the fast path
  const int I = (int)(E % gc.nx);
  const int J = (int)((E / gc.nx) % gc.ny);
  const int K = (D == 3) ? (int)(E / ((int64_t)gc.nx * gc.ny)) : 0;
  for (int o = t; o < NE * NE; o += blockDim.x) Acc[o] = 0.0;
  for (int ch = 0; ch < NN; ++ch) {
    const int cx = ch & 1, cy = (ch >> 1) & 1, cz = ch >> 2;
    const int fi = 2 * I + cx, fj = 2 * J + cy, fk = (D == 3) ? 2 * K + cz : 0;
    if (fi >= gf.nx || fj >= gf.ny || fk >= gf.nz) continue;  // short last coarse element
    const int64_t fe = ((int64_t)fk * gf.ny + fj) * gf.nx + fi;
    __syncthreads();
    // interpolation weights of this child (fine local corner b <- coarse local corner B)
    for (int o = t; o < NN * NN; o += blockDim.x) {
      const int b = o / NN, B = o % NN;
      const double tx = tpos(fi + offx(b), I, gf.nx), ty = tpos(fj + offy(b), J, gf.ny);
      const double tz = (D == 3) ? tpos(fk + offz(b), K, gf.nz) : 0.0;
      double w = (offx(B) ? tx : 1.0 - tx) * (offy(B) ? ty : 1.0 - ty);
      if (D == 3) w *= offz(B) ? tz : 1.0 - tz;
      R[o] = w;
    }
    for (int o = t; o < NE; o += blockDim.x) {
      const int b = o / D, c = o % D;
      mf[o] = fixed_f[dof_of(gf, fi + offx(b), fj + offy(b), fk + (D == 3 ? offz(b) : 0), D, c)];
    }
    __syncthreads();
    const double a = FIRST ? alpha[fe] : 1.0;
    for (int o = t; o < NE * NE; o += blockDim.x) {
      const int r = o / NE, q = o % NE;
      const double v = FIRST ? a * Ku.v[o] : ke_f[fe * NE * NE + o];
      Ke[o] = (mf[r] || mf[q]) ? 0.0 : v;
    }
    __syncthreads();
    // T = Ke (R (x) I_D)
    for (int o = t; o < NE * NE; o += blockDim.x) {
      const int r = o / NE, q = o % NE, B = q / D, cq = q % D;
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < NN; ++b) s = fma(Ke[r * NE + b * D + cq], R[b * NN + B], s);
      T[o] = s;
    }
    __syncthreads();
    // Acc += (R (x) I_D)^T T
    for (int o = t; o < NE * NE; o += blockDim.x) {
      const int r = o / NE, q = o % NE, B = r / D, cr = r % D;
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < NN; ++b) s = fma(R[b * NN + B], T[(b * D + cr) * NE + q], s);
      Acc[o] += s;
    }
  }
  __syncthreads();
  for (int o = t; o < NE; o += blockDim.x) {
    const int B = o / D, c = o % D;
    mf[o] = fixed_c[dof_of(gc, I + offx(B), J + offy(B), K + (D == 3 ? offz(B) : 0), D, c)];
  }
  __syncthreads();
  for (int o = t; o < NE * NE; o += blockDim.x) {
    const int r = o / NE, q = o % NE;
    ke_c[E * NE * NE + o] = (mf[r] || mf[q]) ? 0.0 : Acc[o];
  }
}

// coarse Dirichlet mask: coarse node (I,J,K) coincides with fine node (2I,2J,2K)
template <int D>
__global__ void k_mg_coarse_fixed(Grid gc, Grid gf, const uint8_t* __restrict__ ff, uint8_t* __restrict__ fc) {
  const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= gc.n_nodes * D) return;
  const int64_t n = d / D;
  const int c = (int)(d % D);
  const int I = (int)(n % gc.nnx), J = (int)((n / gc.nnx) % gc.nny), K = (int)(n / ((int64_t)gc.nnx * gc.nny));
  fc[d] = ff[dof_of(gf, cnode(I, gf.nx), cnode(J, gf.ny), (D == 3) ? cnode(K, gf.nz) : 0, D, c)];
}

// Coarse operators are applied as assembled 3^D-point node stencils.  The operator is
// symmetric, so only the centre block and the upper half (offsets m > centre) are stored, SoA
// over nodes:  st[((u D + c) D + c') n_nodes + n],  u = m - centre,  couples dof (n, c) with dof
// (n + off(m), c'),  off(m) = (m % 3 - 1, m / 3 % 3 - 1, m / 9 - 1).  The lower blocks are the
// transposes stored at the neighbour (off(NB-1-m) = -off(m)), which also makes the applied
// operator exactly symmetric.  Built once per set-up from the element matrices in fixed order.
template <int D>
__global__ void __launch_bounds__(kBlock) k_mg_stencil(Grid g, const double* __restrict__ ke, double* __restrict__ st) {
  constexpr int NN = Q1<D>::NN, NE = NN * D, NB = Q1<D>::NB, MC = NB / 2;
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.n_nodes) return;
  int i, j, k;
  node_coords(g, n, i, j, k);
  for (int m = MC; m < NB; ++m) {
    const int dx = m % 3 - 1, dy = (m / 3) % 3 - 1, dz = (D == 3) ? m / 9 - 1 : 0;
    double a[D][D];
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int cp = 0; cp < D; ++cp) a[c][cp] = 0.0;
#pragma unroll
    for (int s = 0; s < NN; ++s) {
      const int sx = s & 1, sy = (s >> 1) & 1, sz = s >> 2;
      const int ei = i - 1 + sx, ej = j - 1 + sy, ek = (D == 3) ? k - 1 + sz : 0;
      if (ei < 0 || ei >= g.nx || ej < 0 || ej >= g.ny || ek < 0 || ek >= g.nz) continue;
      const int ox = 1 - sx, oy = 1 - sy, oz = (D == 3) ? 1 - sz : 0;
      const int bx = ox + dx, by = oy + dy, bz = oz + dz;
      if (bx < 0 || bx > 1 || by < 0 || by > 1 || bz < 0 || bz > 1) continue;
      const int64_t e = ((int64_t)ek * g.ny + ej) * g.nx + ei;
      const int L = loc_of(ox, oy, oz), b = loc_of(bx, by, bz);
      const double* kr = ke + e * NE * NE;
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int cp = 0; cp < D; ++cp) a[c][cp] += kr[(L * D + c) * NE + b * D + cp];
    }
    const int u = m - MC;
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int cp = 0; cp < D; ++cp) st[((int64_t)(u * D + c) * D + cp) * g.n_nodes + n] = a[c][cp];
  }
}

// y = A v on a coarse level from its half stencil (node-owner, fixed neighbour order).
// EPI 1: y = v + omega ed (eb - A v) (damped-Jacobi sweep), EPI 2: y = ed != 0 ? eb - A v : 0
// (masked residual); y must not alias v.
template <int D, int EPI = 0>
__global__ void __launch_bounds__(kBlock) k_mg_sapply(Grid g, const double* __restrict__ st,
                                                      const double* __restrict__ v, double* __restrict__ y,
                                                      const double* __restrict__ eb = nullptr,
                                                      const double* __restrict__ ed = nullptr, double omega = 0.0) {
  constexpr int NB = Q1<D>::NB, MC = NB / 2;
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.n_nodes) return;
  int i, j, k;
  node_coords(g, n, i, j, k);
  double out[D];
#pragma unroll
  for (int c = 0; c < D; ++c) out[c] = 0.0;
#pragma unroll
  for (int m = 0; m < NB; ++m) {
    const int dx = m % 3 - 1, dy = (m / 3) % 3 - 1, dz = (D == 3) ? m / 9 - 1 : 0;
    const int ni = i + dx, nj = j + dy, nk = k + dz;
    if (ni < 0 || ni >= g.nnx || nj < 0 || nj >= g.nny || nk < 0 || nk >= g.nnz) continue;
    const int64_t nbn = ((int64_t)nk * g.nny + nj) * g.nnx + ni;
    double vv[D];
#pragma unroll
    for (int cp = 0; cp < D; ++cp) vv[cp] = __ldg(v + nbn * D + cp);
    if (m >= MC) {  // stored here
      const int u = m - MC;
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int cp = 0; cp < D; ++cp)
          out[c] = fma(__ldg(st + ((int64_t)(u * D + c) * D + cp) * g.n_nodes + n), vv[cp], out[c]);
    } else {  // transpose of the neighbour's block towards this node
      const int u = NB - 1 - m - MC;
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int cp = 0; cp < D; ++cp)
          out[c] = fma(__ldg(st + ((int64_t)(u * D + cp) * D + c) * g.n_nodes + nbn), vv[cp], out[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < D; ++c) {
    double o = out[c];
    if (EPI == 1) o = v[n * D + c] + omega * ed[n * D + c] * (eb[n * D + c] - o);
    if (EPI == 2) o = (ed[n * D + c] != 0.0) ? eb[n * D + c] - o : 0.0;
    y[n * D + c] = o;
  }
}

template <int D>
__global__ void k_mg_dinv(Grid g, const double* __restrict__ st, const uint8_t* __restrict__ fixed,
                          double* __restrict__ dinv) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.n_nodes) return;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const double d = st[((int64_t)c * D + c) * g.n_nodes + n];  // centre block (u = 0)
    dinv[n * D + c] = (fixed[n * D + c] || !(d > 0.0)) ? 0.0 : 1.0 / d;
  }
}

// Level-1 fast path.  A coarse element whose 2^D children all exist and whose fine nodes carry
// no Dirichlet dof has  K_E = sum_ch alpha_ch G_ch,  G_ch = R_ch^T K_unit R_ch  (host-built).
template <int D>
__global__ void k_mg_dirty(Grid gc, Grid gf, const uint8_t* __restrict__ fixed_f, uint8_t* __restrict__ dirty) {
  const int64_t E = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (E >= gc.n_elems) return;
  const int I = (int)(E % gc.nx), J = (int)((E / gc.nx) % gc.ny);
  const int K = (D == 3) ? (int)(E / ((int64_t)gc.nx * gc.ny)) : 0;
  bool d = 2 * I + 1 >= gf.nx || 2 * J + 1 >= gf.ny || (D == 3 && 2 * K + 1 >= gf.nz);
  for (int z = 0; z < (D == 3 ? 3 : 1) && !d; ++z)
    for (int y = 0; y < 3 && !d; ++y)
      for (int x = 0; x < 3 && !d; ++x)
        for (int c = 0; c < D; ++c)
          if (fixed_f[dof_of(gf, 2 * I + x, 2 * J + y, (D == 3) ? 2 * K + z : 0, D, c)]) d = true;
  dirty[E] = d ? 1 : 0;
}

constexpr int kAggBatch = 16;
template <int D>
__global__ void __launch_bounds__(256) k_mg_agg_fast(Grid gc, Grid gf, const double* __restrict__ G,
                                                     const double* __restrict__ alpha,
                                                     const uint8_t* __restrict__ dirty, double* __restrict__ ke_c) {
  constexpr int NN = Q1<D>::NN, NE = NN * D, NE2 = NE * NE;
  __shared__ double a[kAggBatch][NN];
  const int64_t E0 = (int64_t)blockIdx.x * kAggBatch;
  for (int q = threadIdx.x; q < kAggBatch * NN; q += blockDim.x) {
    const int b = q / NN, ch = q % NN;
    const int64_t E = E0 + b;
    double v = 0.0;
    if (E < gc.n_elems && !dirty[E]) {
      const int I = (int)(E % gc.nx), J = (int)((E / gc.nx) % gc.ny);
      const int K = (D == 3) ? (int)(E / ((int64_t)gc.nx * gc.ny)) : 0;
      const int fi = 2 * I + (ch & 1), fj = 2 * J + ((ch >> 1) & 1), fk = (D == 3) ? 2 * K + (ch >> 2) : 0;
      v = alpha[((int64_t)fk * gf.ny + fj) * gf.nx + fi];
    }
    a[b][ch] = v;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < kAggBatch * NE2; q += blockDim.x) {
    const int b = q / NE2, o = q % NE2;
    const int64_t E = E0 + b;
    if (E >= gc.n_elems || dirty[E]) continue;
    double v = 0.0;
#pragma unroll
    for (int ch = 0; ch < NN; ++ch) v = fma(a[b][ch], __ldg(G + ch * NE2 + o), v);
    ke_c[E * NE2 + o] = v;
  }
}

// x_out = x_in + omega D^-1 (b - y)   (x_in may be null: x_in = 0, y ignored)
__global__ void k_mg_jacobi(int64_t n, double omega, const double* __restrict__ dinv, const double* __restrict__ b,
                            const double* __restrict__ y, const double* __restrict__ x_in, double* __restrict__ x_out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double r = x_in ? b[i] - y[i] : b[i];
    x_out[i] = (x_in ? x_in[i] : 0.0) + omega * dinv[i] * r;
  }
}

// r = b - y on free dofs (dinv != 0), 0 elsewhere
__global__ void k_mg_resid(int64_t n, const double* __restrict__ dinv, const double* __restrict__ b,
                           const double* __restrict__ y, double* __restrict__ r) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = (dinv[i] != 0.0) ? b[i] - y[i] : 0.0;
}

// b_c = P~^T r_f : full weighting over the 3^D fine neighbours of the coincident fine node
template <int D>
__global__ void k_mg_restrict(Grid gc, Grid gf, const double* __restrict__ rf, const uint8_t* __restrict__ fc,
                              double* __restrict__ bc) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= gc.n_nodes) return;
  int I, J, K;
  node_coords(gc, n, I, J, K);
  double acc[D];
#pragma unroll
  for (int c = 0; c < D; ++c) acc[c] = 0.0;
#pragma unroll
  for (int dz = (D == 3 ? -1 : 0); dz <= (D == 3 ? 1 : 0); ++dz)
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int fi = 2 * I + dx, fj = 2 * J + dy, fk = 2 * K + dz;
        const double w = pw(fi, I, gf.nx) * pw(fj, J, gf.ny) * ((D == 3) ? pw(fk, K, gf.nz) : 1.0);
        if (w == 0.0) continue;
        const int64_t fd = dof_of(gf, fi, fj, fk, D, 0);
#pragma unroll
        for (int c = 0; c < D; ++c) acc[c] = fma(w, __ldg(rf + fd + c), acc[c]);
      }
#pragma unroll
  for (int c = 0; c < D; ++c) bc[n * D + c] = fc[n * D + c] ? 0.0 : acc[c];
}

// x_f += P~ x_c : (tri)linear interpolation, fixed fine dofs untouched
template <int D>
__global__ void k_mg_prolong_add(Grid gf, Grid gc, const double* __restrict__ xc, const uint8_t* __restrict__ ff,
                                 double* __restrict__ xf) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= gf.n_nodes) return;
  int i, j, k;
  node_coords(gf, n, i, j, k);
  int i0, j0, k0 = 0, ni, nj, nk = 1;
  pmap(i, gf.nx, i0, ni);
  pmap(j, gf.ny, j0, nj);
  if (D == 3) pmap(k, gf.nz, k0, nk);
  const double w = (ni == 2 ? 0.5 : 1.0) * (nj == 2 ? 0.5 : 1.0) * (nk == 2 ? 0.5 : 1.0);
  double acc[D];
#pragma unroll
  for (int c = 0; c < D; ++c) acc[c] = 0.0;
  for (int a = 0; a < nk; ++a)
    for (int b = 0; b < nj; ++b)
      for (int q = 0; q < ni; ++q) {
        const int64_t cd = dof_of(gc, i0 + q, j0 + b, k0 + a, D, 0);
#pragma unroll
        for (int c = 0; c < D; ++c) acc[c] += __ldg(xc + cd + c);
      }
#pragma unroll
  for (int c = 0; c < D; ++c)
    if (!ff[n * D + c]) xf[n * D + c] = fma(w, acc[c], xf[n * D + c]);
}

// dense coarsest matrix, one row per thread (deterministic); fixed rows -> identity
template <int D>
__global__ void k_mg_dense(Grid g, const double* __restrict__ ke, const uint8_t* __restrict__ fixed,
                           double* __restrict__ A) {
  constexpr int NN = Q1<D>::NN, NE = NN * D;
  const int64_t nd = g.n_nodes * D;
  const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= nd) return;
  const int64_t n = d / D;
  const int c = (int)(d % D);
  if (fixed[d]) {
    A[d * nd + d] = 1.0;
    return;
  }
  int i, j, k;
  node_coords(g, n, i, j, k);
  for (int s = 0; s < NN; ++s) {
    const int sx = s & 1, sy = (s >> 1) & 1, sz = s >> 2;
    const int ei = i - 1 + sx, ej = j - 1 + sy, ek = (D == 3) ? k - 1 + sz : 0;
    if (ei < 0 || ei >= g.nx || ej < 0 || ej >= g.ny || ek < 0 || ek >= g.nz) continue;
    const int64_t e = ((int64_t)ek * g.ny + ej) * g.nx + ei;
    const int L = loc_of(1 - sx, 1 - sy, (D == 3) ? 1 - sz : 0);
    for (int b = 0; b < NN; ++b) {
      const int64_t col0 = dof_of(g, ei + offx(b), ej + offy(b), ek + (D == 3 ? offz(b) : 0), D, 0);
      for (int cp = 0; cp < D; ++cp) A[d * nd + col0 + cp] += ke[e * NE * NE + (L * D + c) * NE + b * D + cp];
    }
  }
}

// row-major upper triangle (cuSOLVER column-major lower) -> full symmetric
__global__ void k_mg_symmetrize(int64_t n, double* __restrict__ A) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * n) return;
  const int64_t r = t / n, c = t % n;
  if (r > c) A[r * n + c] = A[c * n + r];
}

// x = Ainv b, warp per row, fixed-order lane partials
__global__ void k_mg_gemv(int64_t n, const double* __restrict__ A, const double* __restrict__ b,
                          double* __restrict__ x) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < n; r += nw) {
    double s = 0.0;
    for (int64_t c = lane; c < n; c += 32) s = fma(A[r * n + c], b[c], s);
    s = warp_sum(s);
    if (lane == 0) x[r] = s;
  }
}

// ---------------------------------------------------------------------------------------
// Coarsest inverse by blocked Gauss-Jordan elimination (SPD: no pivoting), one cooperative
// launch.  CTA c owns row block c (kGjB rows).  Step K: every CTA loads row block K (kGjB x n)
// into shared memory and inverts its diagonal block P in one warp (registers + shuffles).  The
// new row block R = P^-1 [row block K] (R[:, K cols] = P^-1) is formed column-slice by slice
// across all CTAs and parked in a scratch buffer (double-buffered by step parity: other CTAs
// may still be reading row block K), from which owner K takes its rows at the next step.
// Every other owner updates its rows with Gm = F P^-1 (F = its K columns):
// A[i, :] <- A[i, :] - Gm_i [row block K] off the K columns, -Gm_i on them.  One grid barrier
// per step.
// ---------------------------------------------------------------------------------------
// Shared-memory layout of k_mg_gj_inverse (host and device compute it identically): the row
// block K is staged compactly -- this CTA's R slice (LS columns) then its update part (LU) --
// and, when `stg`, this CTA's own rows (update part) and their K columns as well, so the step
// needs no L2 round trip after the staging.
#ifdef TB_GJ_PROF
__device__ unsigned long long g_gj_prof[2][8];
#define GJ_MARK(k)                                                               \
  do {                                                                           \
    if ((blockIdx.x == 0 || blockIdx.x == 100) && threadIdx.x == 0) {            \
      unsigned long long t_;                                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
      g_gj_prof[blockIdx.x ? 1 : 0][k] += t_ - prof_last;                        \
      prof_last = t_;                                                            \
    }                                                                            \
  } while (0)
#else
#define GJ_MARK(k) \
  do {             \
  } while (0)
#endif

struct GjLayout {
  int cols_per, cps, ucols, LS, LU, LW;
  __host__ __device__ GjLayout(int n, int grid) {
    const int nb = (n + kGjB - 1) / kGjB;
    cols_per = (n + grid - 1) / grid;
    cps = grid / nb > 1 ? grid / nb : 1;
    ucols = (n + cps - 1) / cps;
    LS = (cols_per + 1) / 2 * 2;
    LU = (ucols + 1) / 2 * 2;
    LW = LS + LU;
  }
  // bulk copies need 16-byte aligned global rows and ranges
  __host__ __device__ bool bulk(int n) const { return !(n & 1) && !(cols_per & 1) && !(ucols & 1); }
  __host__ __device__ size_t smem(bool stg) const {
    return sizeof(double) * ((size_t)kGjB * LW + (stg ? (size_t)kGjB * LU + kGjB * kGjB : 0));
  }
};

__global__ void __launch_bounds__(512, 1) k_mg_gj_inverse(int n, double* __restrict__ A, double* __restrict__ G,
                                                          unsigned int* bar, int* info, int stg) {
  extern __shared__ __align__(16) double gj_sm[];
  __shared__ double Pi[kGjB][kGjB];  // P^-1
  __shared__ double Gm[kGjB][kGjB];  // F P^-1 for this CTA's rows
  __shared__ int bad;
  __shared__ __align__(8) uint64_t wbar;  // bulk copies of the step's operands
  const int nb = (n + kGjB - 1) / kGjB;
  const int c = blockIdx.x, t = threadIdx.x, nt = blockDim.x, lane = t & 31;
  const GjLayout Lo(n, (int)gridDim.x);
  double* Ws = gj_sm;                           // [kGjB][LW]: row block K, R slice then update part
  double* Os = gj_sm + kGjB * Lo.LW;            // [kGjB][LU]: own rows, update part (stg)
  double* Fs = Os + kGjB * Lo.LU;               // [kGjB][kGjB]: own rows, K columns (stg)
  const int j0 = c * Lo.cols_per, j1 = min(n, j0 + Lo.cols_per);  // this CTA's slice of R
  // row block rbk of the matrix, column part cpart of cps (several CTAs per row block when the
  // grid is at least twice the block count, so more SMs share the rank-16 updates)
  const int rbk = c / Lo.cps, cpart = c % Lo.cps;
  const int u0 = cpart * Lo.ucols, u1 = min(n, u0 + Lo.ucols);
  const bool bulk = Lo.bulk(n);
  if (t == 0) {
    bad = 0;
    mb_init(&wbar, 1);
  }
  __syncthreads();
  uint32_t wphase = 0;
#ifdef TB_GJ_PROF
  unsigned long long prof_last = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prof_last));
#endif
  for (int K = 0; K < nb; ++K) {
    const int k0 = K * kGjB, kb = min(kGjB, n - k0);
    const bool own = (rbk < nb && rbk != K);
    const int r0 = rbk * kGjB, rb = own ? min(kGjB, n - r0) : 0;
    const bool parked = own && (rbk == K - 1);  // rows of block K-1 live in G[(K-1) & 1]
    const double* rows = parked ? G + (int64_t)((K - 1) & 1) * kGjB * n : A + (int64_t)r0 * n;
    const int ns = max(0, j1 - j0), nsu = own ? max(0, u1 - u0) : 0;
    // operands -> shared memory, in flight while P^-1 is formed: row block K (R slice + update
    // part) and, stg, this CTA's own rows; one bulk copy per row and range by one thread (the
    // per-element cp.async loops were ~40% of the kernel's instructions), else 8-byte cp.async
    const bool ownst = stg && own && rb > 0;
    const uint32_t bytes = (uint32_t)(sizeof(double) * (kb * (ns + nsu) + (ownst ? rb * (nsu + kb) : 0)));
    if (bulk) {
      // warp 0 issues: lane 0 arms the barrier, then lane r copies row r of every operand
      // (one thread issuing all ~64 copies took ~3.5 us per step)
      if (t < 32 && bytes > 0) {
        fence_proxy_async();  // operands were written (generic proxy) before the grid barrier
        if (t == 0) mb_expect_tx(&wbar, bytes);
        __syncwarp();
        const int r = t & (kGjB - 1);
        if (t < kGjB && r < kb) {
          const double* src = A + (int64_t)(k0 + r) * n;
          if (ns) bulk_g2s(Ws + r * Lo.LW, src + j0, (uint32_t)(sizeof(double) * ns), &wbar);
          if (nsu) bulk_g2s(Ws + r * Lo.LW + Lo.LS, src + u0, (uint32_t)(sizeof(double) * nsu), &wbar);
        }
        if (ownst && t >= kGjB && r < rb) {
          bulk_g2s(Os + r * Lo.LU, rows + (int64_t)r * n + u0, (uint32_t)(sizeof(double) * nsu), &wbar);
          bulk_g2s(Fs + r * kGjB, rows + (int64_t)r * n + k0, (uint32_t)(sizeof(double) * kb), &wbar);
        }
      }
    } else {
      for (int r = 0; r < kb; ++r) {
        const double* src = A + (int64_t)(k0 + r) * n;
        for (int q = t; q < ns + nsu; q += nt) {
          const bool sl = q < ns;
          const int j = sl ? j0 + q : u0 + (q - ns);
          cp_async8(Ws + r * Lo.LW + (sl ? q : Lo.LS + (q - ns)), src + j, true);
        }
      }
      cp_async_commit();
    }
    GJ_MARK(0);
    // P^-1 in warp 0: lane l holds column l of [P | I] (rows in registers), Gauss-Jordan by
    // shuffles (SPD pivots, no pivoting; a short last block is padded with identity rows)
    if (t < 32) {
      double col[kGjB];
#pragma unroll
      for (int r = 0; r < kGjB; ++r) {
        double v;
        if (lane < kGjB) v = (r < kb && lane < kb) ? __ldcg(A + (int64_t)(k0 + r) * n + k0 + lane) : (r == lane ? 1.0 : 0.0);
        else v = (lane - kGjB == r) ? 1.0 : 0.0;
        col[r] = v;
      }
#pragma unroll
      for (int m = 0; m < kGjB; ++m) {
        const double piv = __shfl_sync(0xffffffffu, col[m], m);
        if (lane == 0 && !(piv > 0.0) && bad == 0) bad = k0 + m + 1;
        col[m] = col[m] * __drcp_rn(piv);
#pragma unroll
        for (int r = 0; r < kGjB; ++r) {
          if (r == m) continue;
          const double f = __shfl_sync(0xffffffffu, col[r], m);
          col[r] = fma(-f, col[m], col[r]);
        }
      }
      if (lane >= kGjB) {
#pragma unroll
        for (int r = 0; r < kGjB; ++r) Pi[r][lane - kGjB] = col[r];
      }
    }
    GJ_MARK(1);
    if (!bulk) {
      cp_async_wait<0>();
    } else if (bytes > 0) {
      mb_wait(&wbar, wphase);
      wphase ^= 1u;
    }
    GJ_MARK(2);
    __syncthreads();
    GJ_MARK(3);
    // Gm = F P^-1, F = this row block's K columns (old)
    if (own && t < kGjB * kGjB) {
      const int r = t / kGjB, p = t % kGjB;
      double f[kGjB];
#pragma unroll
      for (int m = 0; m < kGjB; ++m)
        f[m] = (r < rb && m < kb) ? (ownst ? Fs[r * kGjB + m] : __ldcg(rows + (int64_t)r * n + k0 + m)) : 0.0;
      double acc = 0.0;
#pragma unroll
      for (int m = 0; m < kGjB; ++m) acc = fma(f[m], Pi[m][p], acc);
      Gm[r][p] = (p < kb) ? acc : 0.0;
    }
    // this CTA's slice of R = P^-1 [row block K] (R[:, K cols] = P^-1), parked for owner K
    if (ns > 0) {
      double* g = G + (int64_t)(K & 1) * kGjB * n;
      for (int q = t; q < kGjB * ns; q += nt) {
        const int r = q / ns, jj = q - r * ns, j = j0 + jj;
        if (r >= kb) continue;
        double acc;
        if (j >= k0 && j < k0 + kb) {
          acc = Pi[r][j - k0];
        } else {
          acc = 0.0;
#pragma unroll
          for (int m = 0; m < kGjB; ++m)
            if (m < kb) acc = fma(Pi[r][m], Ws[m * Lo.LW + jj], acc);
        }
        g[(int64_t)r * n + j] = acc;
      }
    }
    GJ_MARK(4);
    __syncthreads();  // Gm
    GJ_MARK(5);
    // row i <- row i - Gm_i [row block K] off the K columns, -Gm_i on them (columns u0 .. u1).
    // The rank-16 update runs on the FP64 tensor cores: 8x8 output tiles (2 row tiles x the
    // column tiles of [u0, u1)) spread over the warps, D = old + (-Gm) W by 4 m8n8k4 k-steps;
    // the K columns are overwritten with -Gm afterwards (the general formula would give 0 there).
    if (own) {
      const int warp = t >> 5, nwarp = nt >> 5;
      const int ntile = (nsu + 7) / 8;
      const int ar = lane >> 2, ak = lane & 3;  // A fragment (row, k); B fragment (k, col) = (ak, ar)
      double ga[2][4];                          // -Gm fragments: [row tile][k-step]
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) ga[mt][ks] = -Gm[mt * 8 + ar][ks * 4 + ak];
      // a warp takes column tiles (both row tiles of a column tile share the B fragments), two
      // independent DMMA chains in flight
      for (int ct = warp; ct < ntile; ct += nwarp) {
        const int jt = ct * 8;            // column tile, relative to u0
        const int jc = jt + 2 * ak;       // D fragment columns jc, jc + 1
        const int jb = jt + ar;           // B fragment column
        double d[2][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int r = mt * 8 + ar;      // D fragment row
#pragma unroll
          for (int e = 0; e < 2; ++e)
            d[mt][e] = (r < rb && jc + e < nsu)
                           ? (ownst ? Os[r * Lo.LU + jc + e] : __ldcg(rows + (int64_t)r * n + u0 + jc + e))
                           : 0.0;
        }
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int m = ks * 4 + ak;
          const double b = (m < kb && jb < nsu) ? Ws[m * Lo.LW + Lo.LS + jb] : 0.0;
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(d[mt][0]), "+d"(d[mt][1])
                         : "d"(ga[mt][ks]), "d"(b));
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int r = mt * 8 + ar;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = u0 + jc + e;
            if (r < rb && jc + e < nsu) A[(int64_t)(r0 + r) * n + j] = (j >= k0 && j < k0 + kb) ? -Gm[r][j - k0] : d[mt][e];
          }
        }
      }
    }
    GJ_MARK(6);
    grid_sync_flip(bar);
    GJ_MARK(7);
  }
  // the last pivot block's rows are still parked in G
  if (c == 0) {
    const int k0 = (nb - 1) * kGjB, kb = n - k0;
    const double* g = G + (int64_t)((nb - 1) & 1) * kGjB * n;
    for (int q = t; q < kb * n; q += nt) A[(int64_t)k0 * n + q] = __ldcg(g + q);
  }
  if (t == 0 && bad) atomicMax(info, bad);
}

#ifdef TB_GJ_PROF
}  // namespace tb
extern "C" int tb_gj_prof_read(unsigned long long* out16) {
  if (cudaMemcpyFromSymbol(out16, tb::g_gj_prof, sizeof(unsigned long long) * 16) != cudaSuccess) return 2;
  static const unsigned long long zeros[16] = {};
  return cudaMemcpyToSymbol(tb::g_gj_prof, zeros, sizeof(zeros)) != cudaSuccess ? 2 : 0;
}
namespace tb {
#endif

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
int mg_build(tb_plan_impl* P) {
  Mg& mg = P->mg;
  if (mg.built) return TB_OK;
  const int D = P->g.dim;
  // 2D: V(1,1), omega 0.7 (cfg 2: 30 iterations of ~23 persistent-kernel phases against 27 of
  // ~33 for V(2,2) with 0.6).  3D: V(2,2), omega 0.5 (V(1,1) with 0.6 was faster on a raw
  // uniform design but slower on the pre-filtered cfg 3 design: 33.4 vs 27.9 ms per
  // evaluation).  profiles/r1_mg_nu.txt.
  mg.nu = (D == 2) ? 1 : 2;
  mg.omega = (D == 2) ? 0.7 : 0.5;
  if (const char* e = getenv("TB_MG_NU")) mg.nu = atoi(e);         // experiments
  if (const char* e = getenv("TB_MG_OMEGA")) mg.omega = atof(e);
  MgLevel l0;
  l0.g = P->g;
  l0.nc = D;
  l0.n = P->n_dofs;
  l0.fixed = P->d_fixed;
  l0.dinv = P->work.dinv;  // stable pointer: graphs capture it before the first set-up
  mg.lv.push_back(l0);
  // TB_MG_MIN_DOFS (experiments): a 1,092-dof coarsest level at cfg 2 needs 15 instead of 27
  // iterations, but cuSOLVER's potrf/potri then costs ~2 ms per set-up (profiles/mg_levels.sh)
  int64_t min_dofs = (D == 2) ? kMgMinDofs2D : kMgMinDofs;
  if (const char* e = getenv("TB_MG_MIN_DOFS")) min_dofs = atoll(e);
  while (mg.lv.back().n > min_dofs) {
    const Grid& gf = mg.lv.back().g;
    const int cx = (gf.nx + 1) / 2, cy = (gf.ny + 1) / 2, cz = (D == 3) ? (gf.nz + 1) / 2 : 1;
    if (cx == gf.nx && cy == gf.ny && cz == gf.nz) break;  // nothing left to coarsen
    MgLevel c;
    c.g = make_grid(D, cx, cy, (D == 3) ? cz : 0, gf.h * 2.0);
    c.nc = D;
    c.n = (int64_t)D * c.g.n_nodes;
    mg.lv.push_back(c);
  }
  if (mg.lv.size() < 2 || mg.lv.back().n > kMgMaxDense) {
    set_error("multigrid needs at least one coarsening and a coarsest level <= %lld dofs (got %zu levels, %lld dofs)",
              (long long)kMgMaxDense, mg.lv.size(), (long long)mg.lv.back().n);
    mg.lv.clear();
    return TB_ERR_INVALID;
  }
  const int NE = (1 << D) * D;
  for (size_t l = 0; l < mg.lv.size(); ++l) {
    MgLevel& L = mg.lv[l];
    double** vecs[] = {&L.x, &L.b, &L.r, &L.t};
    for (double** v : vecs) TB_CUDA(cudaMalloc(v, sizeof(double) * (size_t)L.n));
    if (l > 0) {
      TB_CUDA(cudaMalloc(&L.fixed, (size_t)L.n));
      TB_CUDA(cudaMalloc(&L.dinv, sizeof(double) * (size_t)L.n));
      TB_CUDA(cudaMalloc(&L.ke, sizeof(double) * (size_t)L.g.n_elems * NE * NE));
      TB_CUDA(cudaMalloc(&L.st, sizeof(double) * (size_t)L.g.n_nodes * (D == 2 ? 5 : 14) * D * D));
      const MgLevel& F = mg.lv[l - 1];
      if (D == 2)
        { k_mg_coarse_fixed<2><<<nblk(L.n), kBlock>>>(L.g, F.g, F.fixed, L.fixed); tb::launched(); }
      else
        { k_mg_coarse_fixed<3><<<nblk(L.n), kBlock>>>(L.g, F.g, F.fixed, L.fixed); tb::launched(); }
      TB_CHECK_LAUNCH();
    }
  }
  // level-1 fast-path tables: G_ch = R_ch^T K_unit R_ch for the 2^D children of a full coarse element
  {
    const int NN = 1 << D;
    const double* Ku = (D == 2) ? P->K2.v : P->K3.v;
    std::vector<double> G((size_t)NN * NE * NE, 0.0), R((size_t)NN * NN);
    for (int ch = 0; ch < NN; ++ch) {
      const int c3[3] = {ch & 1, (ch >> 1) & 1, ch >> 2};
      for (int b = 0; b < NN; ++b)
        for (int B = 0; B < NN; ++B) {
          const int ob[3] = {offx(b), offy(b), offz(b)}, oB[3] = {offx(B), offy(B), offz(B)};
          double w = 1.0;
          for (int d = 0; d < D; ++d) {
            const double t = 0.5 * (c3[d] + ob[d]);
            w *= oB[d] ? t : 1.0 - t;
          }
          R[(size_t)b * NN + B] = w;
        }
      double* Gc = G.data() + (size_t)ch * NE * NE;
      for (int r = 0; r < NE; ++r)
        for (int q = 0; q < NE; ++q) {
          const int Br = r / D, cr = r % D, Bq = q / D, cq = q % D;
          double acc = 0.0;
          for (int b = 0; b < NN; ++b) {
            const double rb = R[(size_t)b * NN + Br];
            if (rb == 0.0) continue;
            for (int bp = 0; bp < NN; ++bp) acc += rb * Ku[(b * D + cr) * NE + bp * D + cq] * R[(size_t)bp * NN + Bq];
          }
          Gc[(size_t)r * NE + q] = acc;
        }
    }
    TB_CUDA(cudaMalloc(&mg.G, sizeof(double) * G.size()));
    TB_CUDA(cudaMemcpy(mg.G, G.data(), sizeof(double) * G.size(), cudaMemcpyHostToDevice));
    TB_CUDA(cudaMalloc(&mg.dirty, (size_t)mg.lv[1].g.n_elems));
  }
  mg.ncoarse = mg.lv.back().n;
  TB_CUDA(cudaMalloc(&mg.dense, sizeof(double) * (size_t)mg.ncoarse * mg.ncoarse));
  cusolverDnHandle_t h;
  if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) {
    set_error("cusolverDnCreate failed");
    return TB_ERR_CUDA;
  }
  mg.solver = h;
  int l1 = 0, l2 = 0;
  cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, (int)mg.ncoarse, mg.dense, (int)mg.ncoarse, &l1);
  cusolverDnDpotri_bufferSize(h, CUBLAS_FILL_MODE_LOWER, (int)mg.ncoarse, mg.dense, (int)mg.ncoarse, &l2);
  mg.lwork = l1 > l2 ? l1 : l2;
  TB_CUDA(cudaMalloc(&mg.work, sizeof(double) * (size_t)(mg.lwork + 1)));
  TB_CUDA(cudaMalloc(&mg.info, sizeof(int)));
  mg.ainv = mg.dense;  // potri (or Gauss-Jordan) overwrites the matrix with its inverse in place
  // Gauss-Jordan gives each row block to its own CTA(s) (k_mg_gj_inverse: rbk = c / cps), so it
  // needs at least ceil(n / kGjB) co-resident CTAs at its shared-memory size, one per SM;
  // otherwise (MIG slice, MPS limits, large n) the cuSOLVER path is taken.
  // 2D and 3D alike (round 2: the 3D set-up no longer calls cuSOLVER's potrf/potri)
  bool gj_ok = mg.ncoarse <= kGjMaxN && getenv("TB_MG_CUSOLVER") == nullptr;
  if (gj_ok) {
    int sms = 0, coop = 0, occ = 0;
    TB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->device));
    TB_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, P->device));
    const GjLayout lo((int)mg.ncoarse, sms);
    mg.gj_stg = lo.bulk((int)mg.ncoarse) && lo.smem(true) <= 200 * 1024;  // stage own rows when they fit
    const size_t smem = lo.smem(mg.gj_stg);
    mg.gj_smem = smem;
    TB_CUDA(cudaFuncSetAttribute(k_mg_gj_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    TB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mg_gj_inverse, 512, smem));
    const int64_t nblocks = (mg.ncoarse + kGjB - 1) / kGjB;
    gj_ok = coop && occ >= 1 && nblocks <= sms;
  }
  if (gj_ok) {
    TB_CUDA(cudaMalloc(&mg.gj, sizeof(double) * 2 * kGjB * (size_t)mg.ncoarse));
    TB_CUDA(cudaMalloc(&mg.gj_bar, 64));
    TB_CUDA(cudaMallocHost(&mg.h_info, sizeof(int)));
    TB_CUDA(cudaMemset(mg.gj_bar, 0, 64));
  }
  mg.built = true;
  return TB_OK;
}

void mg_release(Mg& mg) {
  for (size_t l = 0; l < mg.lv.size(); ++l) {
    MgLevel& L = mg.lv[l];
    void* bufs[] = {L.x, L.b, L.r, L.t};
    for (void* b : bufs)
      if (b) cudaFree(b);
    if (l > 0) {
      if (L.fixed) cudaFree(L.fixed);
      if (L.dinv) cudaFree(L.dinv);
      if (L.ke) cudaFree(L.ke);
      if (L.st) cudaFree(L.st);
    }
  }
  mg.lv.clear();
  if (mg.dense) cudaFree(mg.dense);
  if (mg.gj) cudaFree(mg.gj);
  if (mg.gj_bar) cudaFree(mg.gj_bar);
  if (mg.h_info) cudaFreeHost(mg.h_info);
  if (mg.G) cudaFree(mg.G);
  if (mg.dirty) cudaFree(mg.dirty);
  if (mg.work) cudaFree(mg.work);
  if (mg.info) cudaFree(mg.info);
  if (mg.solver) cusolverDnDestroy((cusolverDnHandle_t)mg.solver);
  mg = Mg();
}

int mg_setup(tb_plan_impl* P, cudaStream_t s) {
  Mg& mg = P->mg;
  TB_TRY(mg_build(P));
  const int D = P->g.dim;
  for (size_t l = 1; l < mg.lv.size(); ++l) {
    MgLevel& C = mg.lv[l];
    const MgLevel& F = mg.lv[l - 1];
    const unsigned grid = (unsigned)C.g.n_elems;
    const unsigned fast = (unsigned)((C.g.n_elems + kAggBatch - 1) / kAggBatch);
    if (D == 2) {
      if (l == 1) {
        { k_mg_dirty<2><<<nblk(C.g.n_elems), kBlock, 0, s>>>(C.g, F.g, F.fixed, mg.dirty); tb::launched(); }
        { k_mg_agg_fast<2><<<fast, 256, 0, s>>>(C.g, F.g, mg.G, P->d_alpha, mg.dirty, C.ke); tb::launched(); }
        { k_mg_aggregate<2, true><<<grid, 256, 0, s>>>(C.g, F.g, P->K2, P->d_alpha, nullptr, F.fixed, C.fixed, mg.dirty, C.ke); tb::launched(); }
      } else {
        { k_mg_aggregate<2, false><<<grid, 256, 0, s>>>(C.g, F.g, P->K2, nullptr, F.ke, F.fixed, C.fixed, nullptr, C.ke); tb::launched(); }
      }
      { k_mg_stencil<2><<<nblk(C.g.n_nodes), kBlock, 0, s>>>(C.g, C.ke, C.st); tb::launched(); }
      { k_mg_dinv<2><<<nblk(C.g.n_nodes), kBlock, 0, s>>>(C.g, C.st, C.fixed, C.dinv); tb::launched(); }
    } else {
      if (l == 1) {
        { k_mg_dirty<3><<<nblk(C.g.n_elems), kBlock, 0, s>>>(C.g, F.g, F.fixed, mg.dirty); tb::launched(); }
        { k_mg_agg_fast<3><<<fast, 256, 0, s>>>(C.g, F.g, mg.G, P->d_alpha, mg.dirty, C.ke); tb::launched(); }
        { k_mg_aggregate<3, true><<<grid, 256, 0, s>>>(C.g, F.g, P->K3, P->d_alpha, nullptr, F.fixed, C.fixed, mg.dirty, C.ke); tb::launched(); }
      } else {
        { k_mg_aggregate<3, false><<<grid, 256, 0, s>>>(C.g, F.g, P->K3, nullptr, F.ke, F.fixed, C.fixed, nullptr, C.ke); tb::launched(); }
      }
      { k_mg_stencil<3><<<nblk(C.g.n_nodes), kBlock, 0, s>>>(C.g, C.ke, C.st); tb::launched(); }
      { k_mg_dinv<3><<<nblk(C.g.n_nodes), kBlock, 0, s>>>(C.g, C.st, C.fixed, C.dinv); tb::launched(); }
    }
    TB_CHECK_LAUNCH();
  }
  // coarsest: dense assembly, Cholesky, inverse
  const MgLevel& Lc = mg.lv.back();
  const int64_t n = mg.ncoarse;
  TB_CUDA(cudaMemsetAsync(mg.dense, 0, sizeof(double) * (size_t)n * n, s));
  if (D == 2)
    { k_mg_dense<2><<<nblk(n), kBlock, 0, s>>>(Lc.g, Lc.ke, Lc.fixed, mg.dense); tb::launched(); }
  else
    { k_mg_dense<3><<<nblk(n), kBlock, 0, s>>>(Lc.g, Lc.ke, Lc.fixed, mg.dense); tb::launched(); }
  TB_CHECK_LAUNCH();
  if (mg.gj != nullptr) {  // 2D: blocked Gauss-Jordan, one cooperative launch
    TB_CUDA(cudaMemsetAsync(mg.info, 0, sizeof(int), s));
    int nn = (int)n;
    double* A = mg.dense;
    int stg = mg.gj_stg ? 1 : 0;
    void* args[] = {(void*)&nn, (void*)&A, (void*)&mg.gj, (void*)&mg.gj_bar, (void*)&mg.info, (void*)&stg};
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    TB_CUDA(cudaLaunchCooperativeKernel((const void*)k_mg_gj_inverse, sms, 512, args, mg.gj_smem, s));
    tb::launched();
    // the pivot check is read after the solve's own stream sync (mg_check): no bubble here
    TB_CUDA(cudaMemcpyAsync(mg.h_info, mg.info, sizeof(int), cudaMemcpyDeviceToHost, s));
    mg.info_pending = true;
    { k_mg_symmetrize<<<nblk(n * n), kBlock, 0, s>>>(n, mg.dense); tb::launched(); }
    TB_CHECK_LAUNCH();
    return TB_OK;
  }
  cusolverDnHandle_t h = (cusolverDnHandle_t)mg.solver;
  cusolverDnSetStream(h, s);
  // potrf's status is read before potri runs: potri overwrites info and usually reports 0 on
  // a partially factored matrix
  if (cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, (int)n, mg.dense, (int)n, mg.work, mg.lwork, mg.info) !=
      CUSOLVER_STATUS_SUCCESS) {
    set_error("cuSOLVER Cholesky of the coarsest multigrid level failed");
    return TB_ERR_CUDA;
  }
  int info = 0;
  TB_CUDA(cudaMemcpyAsync(&info, mg.info, sizeof(int), cudaMemcpyDeviceToHost, s));
  TB_CUDA(cudaStreamSynchronize(s));
  if (info != 0) {
    set_error("coarsest multigrid operator is not positive definite (potrf info %d)", info);
    return TB_ERR_INDEFINITE;
  }
  if (cusolverDnDpotri(h, CUBLAS_FILL_MODE_LOWER, (int)n, mg.dense, (int)n, mg.work, mg.lwork, mg.info) !=
      CUSOLVER_STATUS_SUCCESS) {
    set_error("cuSOLVER inverse of the coarsest multigrid level failed");
    return TB_ERR_CUDA;
  }
  { k_mg_symmetrize<<<nblk(n * n), kBlock, 0, s>>>(n, mg.dense); tb::launched(); }
  TB_CHECK_LAUNCH();
  return TB_OK;
}

// level operator y = A_l v
static void level_apply(tb_plan_impl* P, size_t l, const double* v, double* y, cudaStream_t s) {
  const MgLevel& L = P->mg.lv[l];
  if (l == 0) {
    P->apply_alpha(P->d_alpha, v, y, false, s);
  } else if (L.g.dim == 2) {
    { k_mg_sapply<2><<<nblk(L.g.n_nodes), kBlock, 0, s>>>(L.g, L.st, v, y); tb::launched(); }
  } else {
    { k_mg_sapply<3><<<nblk(L.g.n_nodes), kBlock, 0, s>>>(L.g, L.st, v, y); tb::launched(); }
  }
}

// x = V-cycle(b) on level l (x, b are level-sized device vectors; uses the level's r, t)
static void vcycle(tb_plan_impl* P, size_t l, const double* b, double* x, cudaStream_t s) {
  Mg& mg = P->mg;
  const MgLevel& L = mg.lv[l];
  const int nb = grid_for(L.n);
  if (l + 1 == mg.lv.size()) {
    { k_mg_gemv<<<148 * 4, kBlock, 0, s>>>(L.n, mg.ainv, b, x); tb::launched(); }
    return;
  }
  // Level 0 of a Hex8 grid: the smoothing sweeps and the residual run as epilogues of the
  // operator kernel (k_hex8 EPI; TB_MG_NOFUSE=1 keeps the separate update kernels).  A sweep
  // cannot update in place (other CTAs read the halo of its input), so the iterate alternates
  // between L.t and x; it starts in L.t and, after (nu - 1) + nu sweeps, ends in x.
  // The same on the coarse levels through the stencil kernel's epilogue (k_mg_sapply EPI).
  static const bool nofuse = getenv("TB_MG_NOFUSE") != nullptr;
  if ((l > 0 || P->hex8_epi) && !nofuse) {
    // out = epilogue(A_l cur): epi 1 one smoothing sweep, epi 2 the masked residual
    auto level_epi = [&](int epi, const double* cur, double* out) {
      if (l == 0) {
        P->apply_alpha_epi(epi, P->d_alpha, cur, out, b, L.dinv, mg.omega, s);
        return;
      }
      const int blocks = nblk(L.g.n_nodes);
      if (L.g.dim == 2) {
        if (epi == 1) k_mg_sapply<2, 1><<<blocks, kBlock, 0, s>>>(L.g, L.st, cur, out, b, L.dinv, mg.omega);
        else k_mg_sapply<2, 2><<<blocks, kBlock, 0, s>>>(L.g, L.st, cur, out, b, L.dinv, mg.omega);
      } else {
        if (epi == 1) k_mg_sapply<3, 1><<<blocks, kBlock, 0, s>>>(L.g, L.st, cur, out, b, L.dinv, mg.omega);
        else k_mg_sapply<3, 2><<<blocks, kBlock, 0, s>>>(L.g, L.st, cur, out, b, L.dinv, mg.omega);
      }
      tb::launched();
    };
    double* cur = L.t;
    double* oth = x;
    { k_mg_jacobi<<<nb, kBlock, 0, s>>>(L.n, mg.omega, L.dinv, b, nullptr, nullptr, cur); tb::launched(); }
    for (int it = 1; it < mg.nu; ++it) {
      level_epi(1, cur, oth);
      std::swap(cur, oth);
    }
    level_epi(2, cur, L.r);
    const MgLevel& C0 = mg.lv[l + 1];
    if (L.g.dim == 2) {
      { k_mg_restrict<2><<<nblk(C0.g.n_nodes), kBlock, 0, s>>>(C0.g, L.g, L.r, C0.fixed, C0.b); tb::launched(); }
    } else {
      { k_mg_restrict<3><<<nblk(C0.g.n_nodes), kBlock, 0, s>>>(C0.g, L.g, L.r, C0.fixed, C0.b); tb::launched(); }
    }
    vcycle(P, l + 1, C0.b, C0.x, s);
    if (L.g.dim == 2) {
      { k_mg_prolong_add<2><<<nblk(L.g.n_nodes), kBlock, 0, s>>>(L.g, C0.g, C0.x, L.fixed, cur); tb::launched(); }
    } else {
      { k_mg_prolong_add<3><<<nblk(L.g.n_nodes), kBlock, 0, s>>>(L.g, C0.g, C0.x, L.fixed, cur); tb::launched(); }
    }
    for (int it = 0; it < mg.nu; ++it) {
      level_epi(1, cur, oth);
      std::swap(cur, oth);
    }
    return;  // cur == x
  }
  // pre-smoothing: nu damped-Jacobi sweeps from x = 0
  { k_mg_jacobi<<<nb, kBlock, 0, s>>>(L.n, mg.omega, L.dinv, b, nullptr, nullptr, x); tb::launched(); }
  for (int it = 1; it < mg.nu; ++it) {
    level_apply(P, l, x, L.t, s);
    { k_mg_jacobi<<<nb, kBlock, 0, s>>>(L.n, mg.omega, L.dinv, b, L.t, x, x); tb::launched(); }
  }
  // residual, restriction, coarse correction, prolongation
  level_apply(P, l, x, L.t, s);
  { k_mg_resid<<<nb, kBlock, 0, s>>>(L.n, L.dinv, b, L.t, L.r); tb::launched(); }
  const MgLevel& C = mg.lv[l + 1];
  if (L.g.dim == 2) {
    { k_mg_restrict<2><<<nblk(C.g.n_nodes), kBlock, 0, s>>>(C.g, L.g, L.r, C.fixed, C.b); tb::launched(); }
  } else {
    { k_mg_restrict<3><<<nblk(C.g.n_nodes), kBlock, 0, s>>>(C.g, L.g, L.r, C.fixed, C.b); tb::launched(); }
  }
  vcycle(P, l + 1, C.b, C.x, s);
  if (L.g.dim == 2) {
    { k_mg_prolong_add<2><<<nblk(L.g.n_nodes), kBlock, 0, s>>>(L.g, C.g, C.x, L.fixed, x); tb::launched(); }
  } else {
    { k_mg_prolong_add<3><<<nblk(L.g.n_nodes), kBlock, 0, s>>>(L.g, C.g, C.x, L.fixed, x); tb::launched(); }
  }
  // post-smoothing (same sweeps: the cycle is symmetric)
  for (int it = 0; it < mg.nu; ++it) {
    level_apply(P, l, x, L.t, s);
    { k_mg_jacobi<<<nb, kBlock, 0, s>>>(L.n, mg.omega, L.dinv, b, L.t, x, x); tb::launched(); }
  }
}

int mg_check(tb_plan_impl* P) {
  Mg& mg = P->mg;
  if (!mg.info_pending) return TB_OK;
  mg.info_pending = false;
  if (*mg.h_info != 0) {
    set_error("coarsest multigrid operator is not positive definite (pivot %d)", *mg.h_info);
    return TB_ERR_INDEFINITE;
  }
  return TB_OK;
}

int mg_apply(tb_plan_impl* P, const double* r, double* z, cudaStream_t s) {
  vcycle(P, 0, r, z, s);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

}  // namespace tb
