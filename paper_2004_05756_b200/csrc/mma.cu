// Method of Moving Asymptotes step on the device (reference mma.py:45-175, MmaOptimizer.step).
//
// The step is elementwise except for the volume multiplier, which the reference finds by a
// bracket (lam *= 10) and a bisection on  w . primal(lam) = V.  Here the whole step is ONE
// cooperative persistent kernel: every probe of lam is one grid-stride pass over the elements,
// a fixed-order block reduction, a published partial per CTA and one grid barrier; every CTA
// then sums the partials in the same order and takes the same branch.  Per-element arithmetic
// uses explicit _rn intrinsics so no FMA contraction changes its rounding: it is bit-identical
// to the reference's numpy expressions, and only the dot products differ in summation order.
#include "common.cuh"

namespace tb {

struct MmaArgs {
  int64_t n;
  const double *x, *grad, *lower, *upper, *w;
  double cap, move_cap;  // move_cap < 0: none
  int it, has1, has2;    // step counter after increment; xold1 / xold2 present
  tb_mma_config cfg;
  double *xold1, *xold2, *low, *upp;  // state, updated on success
  double* sc;                         // scratch [7][n]: lowN, uppN, alpha, beta, p0, sq, p1
  double* part;                       // [2][4][gridDim.x]
  unsigned int* bar;
  double* x_new;
  int* status;  // device: 0 ok, 1 grad, 2 box, 3 volume, 4 bracket
};

__device__ __forceinline__ void mma_barrier(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int nb = gridDim.x;
    const unsigned int add = (blockIdx.x == 0) ? (0x80000000u - (nb - 1u)) : 1u;
    __threadfence();
    const unsigned int old = atomicAdd(bar, add);
    unsigned int cur;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
    } while (((old ^ cur) & 0x80000000u) == 0u);
    __threadfence();
  }
  __syncthreads();
}

// grid-wide fixed-order sums of NV per-thread values (identical result in every CTA)
template <int NV>
__device__ __forceinline__ void mma_allsum(double (&v)[NV], double* part, int& par, unsigned int* bar) {
  block_sum<NV>(v);
  double* p = part + (size_t)par * 4 * gridDim.x;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) p[(size_t)i * gridDim.x + blockIdx.x] = v[i];
  }
  mma_barrier(bar);
  __shared__ double bc[NV];
  if (threadIdx.x < 32) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = 0.0;
      for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += __ldcg(p + (size_t)i * gridDim.x + b);
      s = warp_sum(s);
      if (threadIdx.x == 0) bc[i] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = bc[i];
  __syncthreads();
  par ^= 1;
}

__device__ __forceinline__ double clipd(double v, double lo, double hi) { return fmin(fmax(v, lo), hi); }

// primal(lam)_i = clip((low sp + upp sq) / (sp + sq), alpha, beta),  sp = sqrt(p0 + lam p1)
__device__ __forceinline__ double mma_primal(const MmaArgs& a, int64_t i, double lam) {
  const int64_t n = a.n;
  const double* sc = a.sc;
  const double sp = __dsqrt_rn(__dadd_rn(sc[4 * n + i], __dmul_rn(lam, sc[6 * n + i])));
  const double sq = sc[5 * n + i];
  const double num = __dadd_rn(__dmul_rn(sc[0 * n + i], sp), __dmul_rn(sc[1 * n + i], sq));
  return clipd(__ddiv_rn(num, __dadd_rn(sp, sq)), sc[2 * n + i], sc[3 * n + i]);
}

__device__ double mma_volume(const MmaArgs& a, double lam, int& par) {
  double v[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x)
    v[0] = fma(a.w[i], mma_primal(a, i, lam), v[0]);
  mma_allsum<1>(v, a.part, par, a.bar);
  return v[0];
}

__global__ void __launch_bounds__(512) k_mma_step(MmaArgs a) {
  const int64_t n = a.n;
  const int64_t gs = (int64_t)gridDim.x * blockDim.x, i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const tb_mma_config& c = a.cfg;
  int par = 0;
  // ---- validation (mma.py:112-119) + per-element set-up (mma.py:120-146) ----
  double chk[3] = {0.0, 0.0, 0.0};  // non-finite grads, out-of-box, w . x
  for (int64_t i = i0; i < n; i += gs) {
    const double x = a.x[i], g = a.grad[i], lo = a.lower[i], up = a.upper[i];
    if (!isfinite(g)) chk[0] += 1.0;
    if (x < __dsub_rn(lo, 1e-12) || x > __dadd_rn(up, 1e-12)) chk[1] += 1.0;
    chk[2] = fma(a.w[i], x, chk[2]);
    const double range = __dsub_rn(up, lo);
    // asymptotes (mma.py:71-89)
    double low, upp;
    if (a.it <= 2 || !a.has1 || !a.has2) {
      low = __dsub_rn(x, __dmul_rn(c.asy_init, range));
      upp = __dadd_rn(x, __dmul_rn(c.asy_init, range));
    } else {
      const double x1 = a.xold1[i], x2 = a.xold2[i];
      const double sign = __dmul_rn(__dsub_rn(x, x1), __dsub_rn(x1, x2));
      const double f = sign > 0.0 ? c.asy_incr : (sign < 0.0 ? c.asy_decr : 1.0);
      low = __dsub_rn(x, __dmul_rn(f, __dsub_rn(x1, a.low[i])));
      upp = __dadd_rn(x, __dmul_rn(f, __dsub_rn(a.upp[i], x1)));
    }
    low = clipd(low, __dsub_rn(x, __dmul_rn(c.asy_max_frac, range)), __dsub_rn(x, __dmul_rn(c.asy_min_frac, range)));
    upp = clipd(upp, __dadd_rn(x, __dmul_rn(c.asy_min_frac, range)), __dadd_rn(x, __dmul_rn(c.asy_max_frac, range)));
    double move = __dmul_rn(c.move, range);
    if (a.move_cap >= 0.0) move = fmin(move, a.move_cap);
    const double alpha = fmax(fmax(lo, __dadd_rn(low, __dmul_rn(c.albefa, __dsub_rn(x, low)))), __dsub_rn(x, move));
    const double beta = fmin(fmin(up, __dsub_rn(upp, __dmul_rn(c.albefa, __dsub_rn(upp, x)))), __dadd_rn(x, move));
    const double gp = fmax(g, 0.0), gm = fmax(-g, 0.0);
    const double curv = __ddiv_rn(c.raa0, range);
    const double ux = __dsub_rn(upp, x), xl = __dsub_rn(x, low);
    const double ux2 = __dmul_rn(ux, ux), xl2 = __dmul_rn(xl, xl);
    const double p0 = __dmul_rn(ux2, __dadd_rn(__dadd_rn(__dmul_rn(1.001, gp), __dmul_rn(0.001, gm)), curv));
    const double q0 = __dmul_rn(xl2, __dadd_rn(__dadd_rn(__dmul_rn(0.001, gp), __dmul_rn(1.001, gm)), curv));
    const double p1 = __dmul_rn(ux2, a.w[i]);
    double* sc = a.sc;
    sc[0 * n + i] = low;
    sc[1 * n + i] = upp;
    sc[2 * n + i] = alpha;
    sc[3 * n + i] = beta;
    sc[4 * n + i] = p0;
    sc[5 * n + i] = __dsqrt_rn(q0);
    sc[6 * n + i] = p1;
  }
  mma_allsum<3>(chk, a.part, par, a.bar);
  int bad = 0;
  if (chk[0] > 0.0)
    bad = 1;
  else if (chk[1] > 0.0)
    bad = 2;
  else if (chk[2] > __dadd_rn(__dmul_rn(a.cap, 1.0 + 1e-9), 1e-12))
    bad = 3;
  if (bad) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.status = bad;
    return;  // uniform across the grid: nothing was committed
  }
  // ---- volume multiplier (mma.py:148-170) ----
  const double V = a.cap, tol = c.bisect_rtol * fmax(fabs(a.cap), 1.0);
  double lam_final = 0.0;
  const double s0 = mma_volume(a, 0.0, par);
  if (!(s0 <= V + tol)) {
    double lo = 0.0, hi = 1.0;
    double shi = mma_volume(a, hi, par);
    while (shi > V) {
      lo = hi;
      hi *= 10.0;
      if (hi > 1e40) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *a.status = 4;
        return;
      }
      shi = mma_volume(a, hi, par);
    }
    double lam_new = hi, s_new = shi;
    for (int k = 0; k < c.bisect_max_iter; ++k) {
      const double mid = 0.5 * (lo + hi);
      const double sm = mma_volume(a, mid, par);
      if (sm > V) {
        lo = mid;
      } else {
        hi = mid;
        lam_new = mid;
        s_new = sm;
      }
      if (fabs(s_new - V) <= tol) break;
    }
    lam_final = lam_new;
  }
  // ---- commit: x_new and the asymptote memory (mma.py:172-175) ----
  for (int64_t i = i0; i < n; i += gs) {
    a.x_new[i] = mma_primal(a, i, lam_final);
    if (a.has1) a.xold2[i] = a.xold1[i];
    a.xold1[i] = a.x[i];
    a.low[i] = a.sc[0 * n + i];
    a.upp[i] = a.sc[1 * n + i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.status = 0;
}

static int mma_grid() {
  static int g = 0;
  if (g == 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_mma_step, 512, 0);
    g = sms * (per < 1 ? 1 : (per > 2 ? 2 : per));
  }
  return g;
}

}  // namespace tb

using namespace tb;

extern "C" {

size_t tb_mma_workspace_bytes(int64_t n) {
  const int g = 148 * 2;  // upper bound of the cooperative grid
  return sizeof(double) * ((size_t)7 * (size_t)(n > 0 ? n : 0) + (size_t)2 * 4 * g) + 64;
}

int tb_mma_step(int64_t n, const double* x, const double* grad, const double* lower, const double* upper,
                const double* w, double volume_cap, double move_cap, int it, int has_xold1, int has_xold2,
                const tb_mma_config* cfg, double* xold1, double* xold2, double* low, double* upp, void* workspace,
                double* x_new, void* stream) {
  if (n < 1 || !x || !grad || !lower || !upper || !w || !cfg || !xold1 || !xold2 || !low || !upp || !workspace ||
      !x_new) {
    set_error("tb_mma_step: bad arguments");
    return TB_ERR_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  MmaArgs a;
  a.n = n;
  a.x = x;
  a.grad = grad;
  a.lower = lower;
  a.upper = upper;
  a.w = w;
  a.cap = volume_cap;
  a.move_cap = move_cap;
  a.it = it;
  a.has1 = has_xold1;
  a.has2 = has_xold2;
  a.cfg = *cfg;
  a.xold1 = xold1;
  a.xold2 = xold2;
  a.low = low;
  a.upp = upp;
  char* ws = static_cast<char*>(workspace);
  a.bar = reinterpret_cast<unsigned int*>(ws);  // caller zeroes the workspace once
  a.status = reinterpret_cast<int*>(ws + 16);
  a.part = reinterpret_cast<double*>(ws + 64);
  const int grid = mma_grid();
  a.sc = a.part + (size_t)2 * 4 * 148 * 2;
  a.x_new = x_new;
  void* args[] = {&a};
  TB_CUDA(cudaMemsetAsync(a.status, 0xff, sizeof(int), s));  // -1 until the kernel reports
  TB_CUDA(cudaLaunchCooperativeKernel((const void*)k_mma_step, grid, 512, args, 0, s));
  tb::launched();
  int st = -1;
  TB_CUDA(cudaMemcpyAsync(&st, a.status, sizeof(int), cudaMemcpyDeviceToHost, s));
  TB_CUDA(cudaStreamSynchronize(s));
  switch (st) {
    case 0:
      return TB_OK;
    case 1:
      set_error("gradient must be finite");
      return TB_ERR_INVALID;
    case 2:
      set_error("iterate outside box bounds");
      return TB_ERR_INVALID;
    case 3:
      set_error("iterate violates the volume constraint");
      return TB_ERR_INVALID;
    case 4:
      set_error("volume multiplier bracket failed");
      return TB_ERR_RUNTIME;
    default:
      set_error("tb_mma_step: kernel did not report a status");
      return TB_ERR_CUDA;
  }
}

}  // extern "C"
