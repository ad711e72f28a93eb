// Direct solve of the Helmholtz filter system H phi = b on the uniform grid (filtering.py:59-76:
// H = sum_e (r^2 S_e + M_e), pure Neumann), replacing the pCG of the whole-grid filter.
//
// The Q1 element on a uniform grid is a tensor product, so with the 1D assembled stiffness S and
// consistent mass M of each axis
//     H = r^2 (Mz (x) My (x) Sx + Mz (x) Sy (x) Mx + Sz (x) My (x) Mx) + Mz (x) My (x) Mx .
// In 1D, M = h D - (h^2/6) S with D = diag(1/2, 1, ..., 1, 1/2), and the cosine vectors
// v_k(j) = cos(pi j k / (n-1)) satisfy S v_k = mu_k D v_k, mu_k = (2/h)(1 - cos(pi k/(n-1))): one
// D-orthonormal basis V diagonalises both, V^T S V = diag(mu), V^T M V = diag(m),
// m_k = h (2 + cos(pi k/(n-1))) / 3.  With W = Vz (x) Vy (x) Vx:  W^T H W = Lambda (diagonal), so
//     phi = W Lambda^-1 W^T b :
// three mode products with the n x n matrices V^T (one per axis), a pointwise scaling and three
// mode products back.  The mode products are dense FP64 contractions (2 n flops per entry and
// axis: 2.8 GFLOP per solve at cfg 3) and run on the FP64 tensor cores (DMMA m8n8k4); the result
// is the solution to round-off, as the reference's sparse direct solve, where pCG stopped at
// its tolerance.  cfg 3: 1.54 -> 0.27 ms per filter call, cfg 2: 0.18 -> 0.08 ms.
//
// tb_filter_create verifies the factorisation against the filter's own operator kernel on a
// random vector (||H phi - b|| <= 1e-11 ||b||) and keeps pCG otherwise.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "plan.cuh"

namespace tb {

namespace {

constexpr int kSgT = 64, kSgK = 16, kSgLd = kSgT + 4;  // 64 x 64 x 16 tiles; row pad: conflict-free fragments

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// C_b(m, n) = sum_k A_b(m, k) B_b(k, n) for b < gridDim.z: A(m, k) at A + b a_sb + m a_sm + k a_sk
// (A_MC: a_sm == 1, else a_sk == 1), B(k, n) at B + b b_sb + k b_sk + n, C(m, n) at
// C + b c_sb + m c_sm + n.  256 threads: warp (wm, wn) of 4 x 2 owns a 16 x 32 block of the tile.
// ksplit > 0 (2D grids: too few output tiles to fill the GPU and a long serial K loop): blockIdx.z
// is not a batch index but a slice [z ksplit, (z + 1) ksplit) of K, and slice z writes its partial
// product to C + z c_sb; k_spec_sum adds the slices in fixed order.
template <bool A_MC>
__global__ void __launch_bounds__(256) k_spec_gemm(int M, int N, int K, const double* __restrict__ A, int64_t a_sm,
                                                   int64_t a_sk, int64_t a_sb, const double* __restrict__ B, int64_t b_sk,
                                                   int64_t b_sb, double* __restrict__ C, int64_t c_sm, int64_t c_sb,
                                                   int ksplit) {
  __shared__ double As[kSgK][kSgLd];  // [k][m]
  __shared__ double Bs[kSgK][kSgLd];  // [k][n]
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int wm = w & 3, wn = w >> 2;
  const int m0 = blockIdx.y * kSgT, n0 = blockIdx.x * kSgT;
  int kbeg = 0;
  if (ksplit > 0) {
    kbeg = (int)blockIdx.z * ksplit;
    K = min(K, kbeg + ksplit);
  } else {
    A += (int64_t)blockIdx.z * a_sb;
    B += (int64_t)blockIdx.z * b_sb;
  }
  C += (int64_t)blockIdx.z * c_sb;
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int g4 = lane >> 2, l4 = lane & 3;
  for (int k0 = kbeg; k0 < K; k0 += kSgK) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int m, k;
      if (A_MC) {
        m = t & 63;
        k = (t >> 6) + 4 * j;
      } else {
        k = t & 15;
        m = (t >> 4) + 16 * j;
      }
      const bool ok = m0 + m < M && k0 + k < K;
      As[k][m] = ok ? A[(int64_t)(m0 + m) * a_sm + (int64_t)(k0 + k) * a_sk] : 0.0;
      const int n = t & 63, kb = (t >> 6) + 4 * j;
      const bool okb = n0 + n < N && k0 + kb < K;
      Bs[kb][n] = okb ? B[(int64_t)(k0 + kb) * b_sk + (n0 + n)] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kSgK; kk += 4) {
      double a[2], b[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = As[kk + l4][wm * 16 + i * 8 + g4];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk + l4][wn * 32 + j * 8 + g4];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int m = m0 + wm * 16 + i * 8 + g4;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + wn * 32 + j * 8 + 2 * l4;
      double* c = C + (int64_t)m * c_sm + n;
      if (n < N) c[0] = acc[i][j][0];
      if (n + 1 < N) c[1] = acc[i][j][1];
    }
  }
}

// x(k, j, i) *= 1 / (r2 (mu_i m_j m_k + m_i mu_j m_k + m_i m_j mu_k) + m_i m_j m_k)
// ev: [mu_x | m_x | mu_y | m_y | mu_z | m_z]; 2D: nnz = 1 with mu_z = 0, m_z = 1
__global__ void __launch_bounds__(kBlock) k_spec_scale(int nnx, int nny, int nnz, double r2,
                                                      const double* __restrict__ ev, double* __restrict__ x) {
  const int64_t n = (int64_t)nnx * nny * nnz;
  const double *mux = ev, *mx = ev + nnx, *muy = mx + nnx, *my = muy + nny, *muz = my + nny, *mz = muz + nnz;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(q % nnx);
    const int64_t rest = q / nnx;
    const int j = (int)(rest % nny), k = (int)(rest / nny);
    const double lam = r2 * (mux[i] * my[j] * mz[k] + mx[i] * muy[j] * mz[k] + mx[i] * my[j] * muz[k]) +
                       mx[i] * my[j] * mz[k];
    x[q] = x[q] / lam;
  }
}

// out = sum over the K slices of a split mode product, in slice order
__global__ void __launch_bounds__(kBlock) k_spec_sum(int64_t n, int ns, const double* __restrict__ part,
                                                    double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = part[i];
    for (int z = 1; z < ns; ++z) s += part[(int64_t)z * n + i];
    out[i] = s;
  }
}

__global__ void __launch_bounds__(kBlock) k_spec_resid(int64_t n, const double* __restrict__ y,
                                                      const double* __restrict__ b, double* __restrict__ part) {
  double acc[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = y[i] - b[i];
    acc[0] = fma(d, d, acc[0]);
    acc[1] = fma(b[i], b[i], acc[1]);
  }
  block_sum<2>(acc);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = acc[0];
    part[2 * blockIdx.x + 1] = acc[1];
  }
}

// D-orthonormal cosine basis of one axis: V[j * n + k] = v_k(j) / ||v_k||_D, mu, m (see the top)
void axis_basis(int n, double h, std::vector<double>* V, std::vector<double>* mu, std::vector<double>* m) {
  V->assign((size_t)n * n, 0.0);
  mu->assign(n, 0.0);
  m->assign(n, 0.0);
  const int p = n - 1;  // elements along the axis (>= 1)
  for (int k = 0; k < n; ++k) {
    const double ck = cos(M_PI * k / p);
    (*mu)[k] = (2.0 / h) * (1.0 - ck);
    (*m)[k] = h * (2.0 + ck) / 3.0;
    const double nrm = (k == 0 || k == p) ? (double)p : 0.5 * p;  // v_k^T D v_k
    const double sc = 1.0 / sqrt(nrm);
    for (int j = 0; j < n; ++j) {
      const long long jk = ((long long)j * k) % (2LL * p);  // cos(pi j k / p), argument reduced exactly
      (*V)[(size_t)j * n + k] = sc * cos(M_PI * (double)jk / p);
    }
  }
}

}  // namespace

struct SpectralFilter {
  double* d_V[3] = {nullptr, nullptr, nullptr};   // V  (row j, column k)
  double* d_Vt[3] = {nullptr, nullptr, nullptr};  // V^T
  double* d_ev = nullptr;                         // [mu_x | m_x | mu_y | m_y | mu_z | m_z]
  double* d_t[2] = {nullptr, nullptr};            // ping-pong scratch (n_nodes each)
  double* d_part = nullptr;                       // 2D: K-slice partial products (kSgSplit x n_nodes)
};

constexpr int kSgSplit = 8;

void spectral_release(tb_filter_impl* F) {
  SpectralFilter* S = F->spec;
  if (S == nullptr) return;
  for (int a = 0; a < 3; ++a) {
    if (S->d_V[a]) cudaFree(S->d_V[a]);
    if (S->d_Vt[a]) cudaFree(S->d_Vt[a]);
  }
  if (S->d_ev) cudaFree(S->d_ev);
  for (auto* p : S->d_t)
    if (p) cudaFree(p);
  if (S->d_part) cudaFree(S->d_part);
  delete S;
  F->spec = nullptr;
}

// Y(o, a, q) = sum_i Q[i][a] X(o, i, q) over the array viewed as [outer][n][inner].  part != null
// (2D, outer or inner == 1 with a single batch): K split into slices, partials in `part`, summed into Y.
static void mode_product(int64_t outer, int n, int64_t inner, const double* Q, const double* X, double* Y,
                         double* part, cudaStream_t s) {
  const int64_t total = outer * n * inner;
  int ksplit = 0, ns = 1;
  if (part != nullptr && (inner == 1 || outer == 1)) {
    ksplit = ((n + kSgSplit - 1) / kSgSplit + kSgK - 1) / kSgK * kSgK;
    ns = (n + ksplit - 1) / ksplit;
    if (ns < 2) ksplit = 0, ns = 1;
  }
  double* C = ksplit ? part : Y;
  if (inner == 1) {  // x axis: Y (outer x n) = X (outer x n) Q
    dim3 grid((unsigned)((n + kSgT - 1) / kSgT), (unsigned)((outer + kSgT - 1) / kSgT), (unsigned)ns);
    k_spec_gemm<false><<<grid, 256, 0, s>>>((int)outer, n, n, X, n, 1, 0, Q, n, 0, C, n, ksplit ? total : 0, ksplit);
  } else {  // Y_o (n x inner) = Q^T X_o
    dim3 grid((unsigned)((inner + kSgT - 1) / kSgT), (unsigned)((n + kSgT - 1) / kSgT),
              (unsigned)(ksplit ? ns : outer));
    k_spec_gemm<true><<<grid, 256, 0, s>>>(n, (int)inner, n, Q, 1, n, 0, X, inner, (int64_t)n * inner, C, inner,
                                           ksplit ? total : (int64_t)n * inner, ksplit);
  }
  launched();
  if (ksplit) {
    k_spec_sum<<<grid_for(total), kBlock, 0, s>>>(total, ns, part, Y);
    launched();
  }
}

// phi = H^-1 b (b and phi may not alias the scratch; b == phi is allowed)
int spectral_solve(tb_filter_impl* F, const double* b, double* phi, cudaStream_t s) {
  SpectralFilter& S = *F->spec;
  const Grid& g = F->g;
  const int nx = g.nnx, ny = g.nny, nz = g.nnz;
  double *t0 = S.d_t[0], *t1 = S.d_t[1];
  double* part = S.d_part;  // null in 3D
  mode_product((int64_t)nz * ny, nx, 1, S.d_V[0], b, t0, part, s);
  mode_product(nz, ny, nx, S.d_V[1], t0, t1, part, s);
  double* cur = t1;
  double* oth = t0;
  if (g.dim == 3) {
    mode_product(1, nz, (int64_t)ny * nx, S.d_V[2], t1, t0, nullptr, s);
    cur = t0;
    oth = t1;
  }
  k_spec_scale<<<grid_for(g.n_nodes), kBlock, 0, s>>>(nx, ny, nz, F->r * F->r, S.d_ev, cur);
  launched();
  if (g.dim == 3) {
    mode_product(1, nz, (int64_t)ny * nx, S.d_Vt[2], cur, oth, nullptr, s);
    double* tmp = cur;
    cur = oth;
    oth = tmp;
  }
  mode_product(nz, ny, nx, S.d_Vt[1], cur, oth, part, s);
  mode_product((int64_t)nz * ny, nx, 1, S.d_Vt[0], oth, phi, part, s);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

// Build the factorisation and check it against the filter's operator; on any failure the filter
// keeps its pCG solver (F->spec stays null).  TB_FILTER_PCG=1 skips it (A/B measurements).
void spectral_init(tb_filter_impl* F) {
  const char* e = getenv("TB_FILTER_PCG");
  if (e != nullptr && e[0] != '\0' && e[0] != '0') return;
  const Grid& g = F->g;
  // 2D as well (same code, nnz = 1): the mode products there have too few output tiles to fill the
  // GPU, so K is split into up to 8 slices summed in fixed order (cfg 2: 0.18 -> 0.08 ms per filter
  // call against the persistent pCG kernel; without the split the direct solve was no faster)
  auto* S = new SpectralFilter();
  F->spec = S;
  const int n[3] = {g.nnx, g.nny, g.dim == 3 ? g.nnz : 1};
  std::vector<double> ev;
  bool ok = true;
  for (int a = 0; a < 3 && ok; ++a) {
    std::vector<double> V, Vt, mu, m;
    if (a < g.dim) {
      axis_basis(n[a], g.h, &V, &mu, &m);
      Vt.resize(V.size());
      for (int j = 0; j < n[a]; ++j)
        for (int k = 0; k < n[a]; ++k) Vt[(size_t)k * n[a] + j] = V[(size_t)j * n[a] + k];
      const size_t bytes = sizeof(double) * V.size();
      ok = cudaMalloc(&S->d_V[a], bytes) == cudaSuccess && cudaMalloc(&S->d_Vt[a], bytes) == cudaSuccess &&
           cudaMemcpy(S->d_V[a], V.data(), bytes, cudaMemcpyHostToDevice) == cudaSuccess &&
           cudaMemcpy(S->d_Vt[a], Vt.data(), bytes, cudaMemcpyHostToDevice) == cudaSuccess;
    } else {
      mu.assign(1, 0.0);
      m.assign(1, 1.0);
    }
    ev.insert(ev.end(), mu.begin(), mu.end());
    ev.insert(ev.end(), m.begin(), m.end());
  }
  const size_t nb = sizeof(double) * (size_t)g.n_nodes;
  ok = ok && cudaMalloc(&S->d_ev, sizeof(double) * ev.size()) == cudaSuccess &&
       cudaMemcpy(S->d_ev, ev.data(), sizeof(double) * ev.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMalloc(&S->d_t[0], nb) == cudaSuccess && cudaMalloc(&S->d_t[1], nb) == cudaSuccess &&
       (g.dim == 3 || cudaMalloc(&S->d_part, nb * kSgSplit) == cudaSuccess);
  // self-check: b = pseudo-random, phi = solve(b), ||H phi - b|| / ||b||
  double rel = 1.0;
  if (ok) {
    std::vector<double> hb((size_t)g.n_nodes);
    uint64_t st = 0x9E3779B97F4A7C15ull;
    for (auto& v : hb) {
      st = st * 6364136223846793005ull + 1442695040888963407ull;
      v = (double)(st >> 11) / 9007199254740992.0 - 0.3;
    }
    const int blocks = grid_for(g.n_nodes);
    double *db = nullptr, *dphi = nullptr, *dy = nullptr, *dpart = nullptr;
    ok = cudaMalloc(&db, nb) == cudaSuccess && cudaMalloc(&dphi, nb) == cudaSuccess &&
         cudaMalloc(&dy, nb) == cudaSuccess && cudaMalloc(&dpart, sizeof(double) * 2 * blocks) == cudaSuccess &&
         cudaMemcpy(db, hb.data(), nb, cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok) ok = spectral_solve(F, db, dphi, nullptr) == TB_OK;
    if (ok) {
      F->op.launch_apply(dphi, dy, nullptr);
      k_spec_resid<<<blocks, kBlock>>>(g.n_nodes, dy, db, dpart);
      std::vector<double> hp((size_t)2 * blocks);
      ok = cudaMemcpy(hp.data(), dpart, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost) == cudaSuccess;
      double rr = 0.0, bb = 0.0;
      for (int i = 0; i < blocks; ++i) {
        rr += hp[2 * i];
        bb += hp[2 * i + 1];
      }
      rel = (bb > 0.0) ? sqrt(rr / bb) : 1.0;
    }
    if (db) cudaFree(db);
    if (dphi) cudaFree(dphi);
    if (dy) cudaFree(dy);
    if (dpart) cudaFree(dpart);
  }
  if (getenv("TB_FILTER_DEBUG") != nullptr)
    fprintf(stderr, "[tb] spectral filter %dD %dx%dx%d: ok=%d self-check residual %.3e\n", g.dim, g.nnx, g.nny, g.nnz,
            (int)ok, rel);
  if (!ok || !(rel <= 1e-11)) {
    cudaGetLastError();
    spectral_release(F);
  }
}

}  // namespace tb
