// Geometric multigrid preconditioner (see mg.cuh).
#include <cusolverDn.h>

#include "mg.cuh"
#include "plan.cuh"

namespace tb {

static inline int nblk(int64_t n) { return (int)((n + kBlock - 1) / kBlock); }
constexpr int64_t kMgMinDofs = 600;     // stop coarsening below this many dofs
constexpr int64_t kMgMaxDense = 6144;   // coarsest level solved densely up to this size

__device__ __forceinline__ int64_t dof_of(const Grid& g, int i, int j, int k, int nc, int c) {
  return (((int64_t)k * g.nny + j) * g.nnx + i) * nc + c;
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
                                                      const uint8_t* __restrict__ fixed_c, double* __restrict__ ke_c) {
  constexpr int NN = Q1<D>::NN, NE = NN * D;
  __shared__ double Ke[NE * NE], T[NE * NE], Acc[NE * NE], R[NN * NN];
  __shared__ uint8_t mf[NE];
  const int t = threadIdx.x;
  const int64_t E = blockIdx.x;
  const int I = (int)(E % gc.nx);
  const int J = (int)((E / gc.nx) % gc.ny);
  const int K = (D == 3) ? (int)(E / ((int64_t)gc.nx * gc.ny)) : 0;
  for (int o = t; o < NE * NE; o += blockDim.x) Acc[o] = 0.0;
  for (int ch = 0; ch < NN; ++ch) {
    const int cx = ch & 1, cy = (ch >> 1) & 1, cz = ch >> 2;
    const int fi = 2 * I + cx, fj = 2 * J + cy, fk = (D == 3) ? 2 * K + cz : 0;
    const int64_t fe = ((int64_t)fk * gf.ny + fj) * gf.nx + fi;
    __syncthreads();
    // interpolation weights of this child (fine local corner b <- coarse local corner B)
    for (int o = t; o < NN * NN; o += blockDim.x) {
      const int b = o / NN, B = o % NN;
      const double tx = 0.5 * (cx + offx(b)), ty = 0.5 * (cy + offy(b)), tz = 0.5 * (cz + offz(b));
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
  fc[d] = ff[dof_of(gf, 2 * I, 2 * J, 2 * K, D, c)];
}

// y = A v on a coarse level (dense element matrices), node-owner gather in fixed slot order
template <int D>
__global__ void __launch_bounds__(kBlock) k_mg_apply(Grid g, const double* __restrict__ ke, const double* __restrict__ v,
                                                     double* __restrict__ y) {
  constexpr int NN = Q1<D>::NN, NE = NN * D;
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.n_nodes) return;
  int i, j, k;
  node_coords(g, n, i, j, k);
  double out[D];
#pragma unroll
  for (int c = 0; c < D; ++c) out[c] = 0.0;
#pragma unroll
  for (int s = 0; s < NN; ++s) {
    const int sx = s & 1, sy = (s >> 1) & 1, sz = s >> 2;
    const int ei = i - 1 + sx, ej = j - 1 + sy, ek = (D == 3) ? k - 1 + sz : 0;
    if (ei < 0 || ei >= g.nx || ej < 0 || ej >= g.ny || ek < 0 || ek >= g.nz) continue;
    const int64_t e = ((int64_t)ek * g.ny + ej) * g.nx + ei;
    const int L = loc_of(1 - sx, 1 - sy, (D == 3) ? 1 - sz : 0);
    const double* kr = ke + e * NE * NE;
#pragma unroll
    for (int b = 0; b < NN; ++b) {
      const int64_t nb = dof_of(g, ei + offx(b), ej + offy(b), ek + (D == 3 ? offz(b) : 0), D, 0);
#pragma unroll
      for (int cp = 0; cp < D; ++cp) {
        const double vv = __ldg(v + nb + cp);
#pragma unroll
        for (int c = 0; c < D; ++c) out[c] = fma(__ldg(kr + (L * D + c) * NE + b * D + cp), vv, out[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < D; ++c) y[n * D + c] = out[c];
}

template <int D>
__global__ void k_mg_dinv(Grid g, const double* __restrict__ ke, const uint8_t* __restrict__ fixed,
                          double* __restrict__ dinv) {
  constexpr int NN = Q1<D>::NN, NE = NN * D;
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.n_nodes) return;
  int i, j, k;
  node_coords(g, n, i, j, k);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    double d = 0.0;
#pragma unroll
    for (int s = 0; s < NN; ++s) {
      const int sx = s & 1, sy = (s >> 1) & 1, sz = s >> 2;
      const int ei = i - 1 + sx, ej = j - 1 + sy, ek = (D == 3) ? k - 1 + sz : 0;
      if (ei < 0 || ei >= g.nx || ej < 0 || ej >= g.ny || ek < 0 || ek >= g.nz) continue;
      const int64_t e = ((int64_t)ek * g.ny + ej) * g.nx + ei;
      const int L = loc_of(1 - sx, 1 - sy, (D == 3) ? 1 - sz : 0);
      d += ke[e * NE * NE + (L * D + c) * NE + L * D + c];
    }
    dinv[n * D + c] = (fixed[n * D + c] || !(d > 0.0)) ? 0.0 : 1.0 / d;
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
        if (fi < 0 || fi >= gf.nnx || fj < 0 || fj >= gf.nny || fk < 0 || fk >= gf.nnz) continue;
        const double w = (dx ? 0.5 : 1.0) * (dy ? 0.5 : 1.0) * (dz ? 0.5 : 1.0);
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
  const int i0 = i >> 1, j0 = j >> 1, k0 = k >> 1;
  const int ni = (i & 1) ? 2 : 1, nj = (j & 1) ? 2 : 1, nk = (D == 3 && (k & 1)) ? 2 : 1;
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
// host side
// ---------------------------------------------------------------------------------------
int mg_build(tb_plan_impl* P) {
  Mg& mg = P->mg;
  if (mg.built) return TB_OK;
  const int D = P->g.dim;
  mg.omega = (D == 2) ? 0.6 : 0.5;
  MgLevel l0;
  l0.g = P->g;
  l0.nc = D;
  l0.n = P->n_dofs;
  l0.fixed = P->d_fixed;
  l0.dinv = P->work.dinv;  // stable pointer: graphs capture it before the first set-up
  mg.lv.push_back(l0);
  while (true) {
    const Grid& gf = mg.lv.back().g;
    const bool even = (gf.nx % 2 == 0) && (gf.ny % 2 == 0) && (D == 2 || gf.nz % 2 == 0);
    if (!even || mg.lv.back().n <= kMgMinDofs || gf.nx < 2 || gf.ny < 2) break;
    MgLevel c;
    c.g = make_grid(D, gf.nx / 2, gf.ny / 2, (D == 3) ? gf.nz / 2 : 0, gf.h * 2.0);
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
      const MgLevel& F = mg.lv[l - 1];
      if (D == 2)
        { k_mg_coarse_fixed<2><<<nblk(L.n), kBlock>>>(L.g, F.g, F.fixed, L.fixed); tb::launched(); }
      else
        { k_mg_coarse_fixed<3><<<nblk(L.n), kBlock>>>(L.g, F.g, F.fixed, L.fixed); tb::launched(); }
      TB_CHECK_LAUNCH();
    }
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
  mg.ainv = mg.dense;  // potri overwrites the factor with the inverse in place
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
    }
  }
  mg.lv.clear();
  if (mg.dense) cudaFree(mg.dense);
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
    if (D == 2) {
      if (l == 1)
        { k_mg_aggregate<2, true><<<grid, 256, 0, s>>>(C.g, F.g, P->K2, P->d_alpha, nullptr, F.fixed, C.fixed, C.ke); tb::launched(); }
      else
        { k_mg_aggregate<2, false><<<grid, 256, 0, s>>>(C.g, F.g, P->K2, nullptr, F.ke, F.fixed, C.fixed, C.ke); tb::launched(); }
      { k_mg_dinv<2><<<nblk(C.g.n_nodes), kBlock, 0, s>>>(C.g, C.ke, C.fixed, C.dinv); tb::launched(); }
    } else {
      if (l == 1)
        { k_mg_aggregate<3, true><<<grid, 256, 0, s>>>(C.g, F.g, P->K3, P->d_alpha, nullptr, F.fixed, C.fixed, C.ke); tb::launched(); }
      else
        { k_mg_aggregate<3, false><<<grid, 256, 0, s>>>(C.g, F.g, P->K3, nullptr, F.ke, F.fixed, C.fixed, C.ke); tb::launched(); }
      { k_mg_dinv<3><<<nblk(C.g.n_nodes), kBlock, 0, s>>>(C.g, C.ke, C.fixed, C.dinv); tb::launched(); }
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
  cusolverDnHandle_t h = (cusolverDnHandle_t)mg.solver;
  cusolverDnSetStream(h, s);
  if (cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, (int)n, mg.dense, (int)n, mg.work, mg.lwork, mg.info) !=
          CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDpotri(h, CUBLAS_FILL_MODE_LOWER, (int)n, mg.dense, (int)n, mg.work, mg.lwork, mg.info) !=
          CUSOLVER_STATUS_SUCCESS) {
    set_error("cuSOLVER factorisation of the coarsest multigrid level failed");
    return TB_ERR_CUDA;
  }
  int info = 0;
  TB_CUDA(cudaMemcpyAsync(&info, mg.info, sizeof(int), cudaMemcpyDeviceToHost, s));
  TB_CUDA(cudaStreamSynchronize(s));
  if (info != 0) {
    set_error("coarsest multigrid operator is not positive definite (info %d)", info);
    return TB_ERR_INDEFINITE;
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
    { k_mg_apply<2><<<nblk(L.g.n_nodes), kBlock, 0, s>>>(L.g, L.ke, v, y); tb::launched(); }
  } else {
    { k_mg_apply<3><<<nblk(L.g.n_nodes), kBlock, 0, s>>>(L.g, L.ke, v, y); tb::launched(); }
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

int mg_apply(tb_plan_impl* P, const double* r, double* z, cudaStream_t s) {
  vcycle(P, 0, r, z, s);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

}  // namespace tb
