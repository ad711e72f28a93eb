// Classical cone ("linear hat") density filter on the element grid.
//
//   rho_e = sum_j w(e, j) psi_j / W_e,   w(e, j) = max(0, R - |c_e - c_j|),   W_e = sum_j w(e, j)
//
// over elements j of the grid (the stencil is truncated at the boundary, W_e renormalises it).
// The reference only has the Helmholtz filter (filtering.py); BASELINE's "linear density
// filter" wording is this classical one, so there is no reference parity: tests/test_gpu_cone.py
// checks it against oracle/filters.py.  The weights depend only on the integer offset between
// element centres, so both maps are gather stencils over a fixed offset list (kernel parameter,
// fixed summation order: deterministic and atomic-free).  The adjoint is
// w_j = sum_e w(e, j) v_e / W_e  with the same symmetric weights.
#include "common.cuh"

namespace tb {

constexpr int kConeMax = 512;  // offsets per stencil (3D: R <= ~4.9 h)

struct ConeStencil {
  int n;
  signed char off[kConeMax][3];
  double w[kConeMax];
};

}  // namespace tb

struct tb_cone {
  tb::Grid g{};
  int device = 0;
  double radius = 0.0;
  tb::ConeStencil st{};
  double* d_wsum = nullptr;  // W_e
  double* d_tmp = nullptr;   // v_e / W_e (adjoint)
};

namespace tb {

static inline int nblk(int64_t n) { return (int)((n + kBlock - 1) / kBlock); }

__device__ __forceinline__ void elem_coords(const Grid& g, int64_t e, int& i, int& j, int& k) {
  i = (int)(e % g.nx);
  const int64_t t = e / g.nx;
  j = (int)(t % g.ny);
  k = (int)(t / g.ny);
}

// out_e = sum_o w_o in[e + o] (in-grid offsets only), optionally divided by W_e; or W_e itself
template <int MODE>  // 0: W_e ; 1: (sum w psi) / W_e ; 2: plain sum (adjoint gather)
__global__ void __launch_bounds__(kBlock) k_cone(Grid g, ConeStencil st, const double* __restrict__ in,
                                                 const double* __restrict__ wsum, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= g.n_elems) return;
  int i, j, k;
  elem_coords(g, e, i, j, k);
  double s = 0.0;
  for (int o = 0; o < st.n; ++o) {
    const int ii = i + st.off[o][0], jj = j + st.off[o][1], kk = k + st.off[o][2];
    if (ii < 0 || ii >= g.nx || jj < 0 || jj >= g.ny || kk < 0 || kk >= g.nz) continue;
    const double w = st.w[o];
    if (MODE == 0) {
      s += w;
    } else {
      s = fma(w, __ldg(in + ((int64_t)kk * g.ny + jj) * g.nx + ii), s);
    }
  }
  out[e] = (MODE == 1) ? s / wsum[e] : s;
}

__global__ void k_cone_scale(int64_t n, const double* __restrict__ v, const double* __restrict__ wsum,
                             double* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = v[e] / wsum[e];
}

Grid make_grid(int dim, int nx, int ny, int nz, double h);  // plan.cu

}  // namespace tb

using namespace tb;

extern "C" {

int tb_cone_create(int dim, int nx, int ny, int nz, double h, double radius, int device, tb_cone** out) {
  if (out == nullptr || (dim != 2 && dim != 3) || nx < 1 || ny < 1 || (dim == 3 && nz < 1) || !(h > 0.0) ||
      !(radius >= 0.0)) {
    set_error("tb_cone_create: bad arguments (dim %d, nx %d, ny %d, nz %d, h %g, radius %g)", dim, nx, ny, nz, h,
              radius);
    return TB_ERR_INVALID;
  }
  TB_CUDA(cudaSetDevice(device));
  auto* F = new tb_cone();
  F->g = make_grid(dim, nx, ny, nz, h);
  F->device = device;
  F->radius = radius;
  // offsets with |d| h < R (the centre always: a zero radius is the identity)
  const int m = (int)ceil(radius / h);
  int n = 0;
  for (int dz = (dim == 3 ? -m : 0); dz <= (dim == 3 ? m : 0); ++dz)
    for (int dy = -m; dy <= m; ++dy)
      for (int dx = -m; dx <= m; ++dx) {
        const double dist = h * sqrt((double)(dx * dx + dy * dy + dz * dz));
        double w = radius - dist;
        if (dx == 0 && dy == 0 && dz == 0 && !(w > 0.0)) w = 1.0;  // R = 0: identity
        if (!(w > 0.0)) continue;
        if (n >= kConeMax) {
          delete F;
          set_error("cone filter radius %g too large for the %d-offset stencil", radius, kConeMax);
          return TB_ERR_INVALID;
        }
        F->st.off[n][0] = (signed char)dx;
        F->st.off[n][1] = (signed char)dy;
        F->st.off[n][2] = (signed char)dz;
        F->st.w[n] = w;
        ++n;
      }
  F->st.n = n;
  const size_t bytes = sizeof(double) * (size_t)F->g.n_elems;
  cudaError_t e1 = cudaMalloc(&F->d_wsum, bytes), e2 = cudaMalloc(&F->d_tmp, bytes);
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    if (F->d_wsum) cudaFree(F->d_wsum);
    if (F->d_tmp) cudaFree(F->d_tmp);
    delete F;
    set_error("cudaMalloc failed for the cone filter");
    return TB_ERR_CUDA;
  }
  { k_cone<0><<<nblk(F->g.n_elems), kBlock>>>(F->g, F->st, nullptr, nullptr, F->d_wsum); tb::launched(); }
  TB_CUDA(cudaDeviceSynchronize());
  *out = F;
  return TB_OK;
}

int tb_cone_destroy(tb_cone* f) {
  if (f == nullptr) return TB_OK;
  cudaFree(f->d_wsum);
  cudaFree(f->d_tmp);
  delete f;
  return TB_OK;
}

int tb_cone_apply(tb_cone* f, const double* psi, double* rho, void* stream) {
  if (f == nullptr || psi == nullptr || rho == nullptr) {
    set_error("tb_cone_apply: null argument");
    return TB_ERR_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  { k_cone<1><<<nblk(f->g.n_elems), kBlock, 0, s>>>(f->g, f->st, psi, f->d_wsum, rho); tb::launched(); }
  TB_CHECK_LAUNCH();
  return TB_OK;
}

int tb_cone_adjoint(tb_cone* f, const double* v, double* w, void* stream) {
  if (f == nullptr || v == nullptr || w == nullptr) {
    set_error("tb_cone_adjoint: null argument");
    return TB_ERR_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  { k_cone_scale<<<grid_for(f->g.n_elems), kBlock, 0, s>>>(f->g.n_elems, v, f->d_wsum, f->d_tmp); tb::launched(); }
  { k_cone<2><<<nblk(f->g.n_elems), kBlock, 0, s>>>(f->g, f->st, f->d_tmp, nullptr, w); tb::launched(); }
  TB_CHECK_LAUNCH();
  return TB_OK;
}

}  // extern "C"
