// libtopo_b200: plan, SIMP elasticity operator, Helmholtz filter, HDM entry points.
#include <stdarg.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <string>

#include "pcg.cuh"
#include "plan.cuh"
#include "cgcg2d.cuh"
#include "cgtile2d.cuh"
#include "q1.cuh"

namespace tb {

static thread_local char g_err[1024] = "";
static std::atomic<int64_t> g_launches{0};

void launched(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// ---------------------------------------------------------------------------------------
// elementwise kernels
// ---------------------------------------------------------------------------------------
// alpha = rho_l + (1-rho_l) rho^p ; alpha' = (1-rho_l) p rho^(p-1)   (hdm.py:40-55)
__global__ void k_material(int64_t n, double rho_l, double p, const double* __restrict__ rho,
                           double* __restrict__ alpha, double* __restrict__ dalpha) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const double r = rho[e];
    // p = 3 (BASELINE's SIMP exponent): multiplies, not the ~100-instruction double pow
    const double rp1 = (p == 3.0) ? r * r : pow(r, p - 1.0);
    const double rp = (p == 3.0) ? rp1 * r : pow(r, p);
    if (alpha) alpha[e] = rho_l + (1.0 - rho_l) * rp;
    if (dalpha) dalpha[e] = (1.0 - rho_l) * p * rp1;
  }
}

// rho = clip(raw, rho_l, 1); block maxima of |rho - raw| (hdm.py:152-153)
__global__ void k_clamp(int64_t n, double lo, const double* __restrict__ raw, double* __restrict__ rho,
                        double* __restrict__ part) {
  double m = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const double r = raw[e];
    // np.clip keeps NaN (the following solve then reports a breakdown); fmin/fmax would not
    const double c = (r != r) ? r : fmin(fmax(r, lo), 1.0);
    rho[e] = c;
    // a NaN entry reports an infinite clamp width (fmax-based reductions drop NaN)
    m = fmax(m, (r != r) ? __longlong_as_double(0x7ff0000000000000LL) : fabs(c - r));
  }
  m = warp_max(m);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    v = warp_max(v);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

// block partial sums of a.b
__global__ void k_dot_part(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ part) {
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc[0] = fma(a[i], b[i], acc[0]);
  block_sum<1>(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
}

// fixed-order final sum (one block) of nb partials, with optional max instead of sum
__global__ void k_finish(int nb, const double* __restrict__ part, double* __restrict__ out, int take_max) {
  double acc[1] = {0.0};
  if (take_max) {
    double m = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) m = fmax(m, part[b]);
    m = warp_max(m);
    __shared__ double red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
      double v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
      v = warp_max(v);
      if (threadIdx.x == 0) *out = v;
    }
    return;
  }
  for (int b = threadIdx.x; b < nb; b += blockDim.x) acc[0] += part[b];
  block_sum<1>(acc);
  if (threadIdx.x == 0) *out = acc[0];
}

void finish_sum(int nb, const double* part, double* out, cudaStream_t s) {
  { k_finish<<<1, kBlock, 0, s>>>(nb, part, out, 0); tb::launched(); }
}

int device_dot(const double* a, const double* b, int64_t n, double* scratch, double* out_dev, cudaStream_t s) {
  const int nb = grid_for(n);
  { k_dot_part<<<nb, kBlock, 0, s>>>(n, a, b, scratch); tb::launched(); }
  { k_finish<<<1, kBlock, 0, s>>>(nb, scratch, out_dev, 0); tb::launched(); }
  TB_CHECK_LAUNCH();
  return TB_OK;
}

// ---------------------------------------------------------------------------------------
// operators
// ---------------------------------------------------------------------------------------
static inline int nblk(int64_t n) { return (int)((n + kBlock - 1) / kBlock); }

void ElastOp::launch_fused(const PcgWork& w, const double* pold, double* pnew, cudaStream_t s) const {
  const Grid& g = plan->g;
  if (g.dim == 2)
    k_pcg_fused<2, 2, true><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, plan->K2, plan->d_alpha, w.z, pold, pnew, w.q,
                                                                w.st, w.partA());
  else if (plan->hex8)
    k_hex8<true><<<hex8_grid(g, plan->zchunk), kHT, kHex8Smem, s>>>(g, plan->hiso, plan->d_alpha, w.z, pold, pnew,
                                                                    w.q, w.st, w.partA(), plan->zchunk);
  else
    k_pcg_fused<3, 3, true><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, plan->K3, plan->d_alpha, w.z, pold, pnew, w.q,
                                                                w.st, w.partA());
}
void ElastOp::launch_apply(const double* v, double* y, cudaStream_t s) const {
  plan->apply_alpha(plan->d_alpha, v, y, true, s);
}
void ElastOp::launch_dinv(double* dinv, cudaStream_t s) const {
  const Grid& g = plan->g;
  if (g.dim == 2)
    { k_node_dinv<2, 2, true><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, plan->K2, plan->d_alpha, plan->d_fixed, dinv); tb::launched(); }
  else
    { k_node_dinv<3, 3, true><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, plan->K3, plan->d_alpha, plan->d_fixed, dinv); tb::launched(); }
}
bool ElastOp::launch_persistent_pc(PcgWork& w, cudaStream_t s) const {
  return plan->precond == 1 && plan->g.dim == 2 && mg_pcg2d_persistent(plan, w, s);
}
int ElastOp::fused_blocks() const {
  if (plan->g.dim == 3 && plan->hex8) {
    const dim3 gr = hex8_grid(plan->g, plan->zchunk);
    return (int)(gr.x * gr.y * gr.z);
  }
  return nblk(plan->g.n_nodes);
}

void HelmOp::launch_fused(const PcgWork& w, const double* pold, double* pnew, cudaStream_t s) const {
  const Grid& g = filt->g;
  if (g.dim == 2)
    k_pcg_fused<2, 1, false><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, filt->H2, nullptr, w.z, pold, pnew, w.q, w.st,
                                                                 w.partA());
  else if (!(filt->iso3 && helm3d_launch_fused(g, filt->h4, w, pold, pnew, s)))
    k_pcg_fused<3, 1, false><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, filt->H3, nullptr, w.z, pold, pnew, w.q, w.st,
                                                                 w.partA());
}
void HelmOp::launch_apply(const double* v, double* y, cudaStream_t s) const {
  const Grid& g = filt->g;
  if (g.dim == 2)
    { k_node_apply<2, 1, false><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, filt->H2, nullptr, v, y, nullptr); tb::launched(); }
  else if (!(filt->iso3 && helm3d_launch_apply(g, filt->h4, v, y, s)))
    { k_node_apply<3, 1, false><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, filt->H3, nullptr, v, y, nullptr); tb::launched(); }
}
void HelmOp::launch_dinv(double* dinv, cudaStream_t s) const {
  const Grid& g = filt->g;
  if (g.dim == 2)
    { k_node_dinv<2, 1, false><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, filt->H2, nullptr, nullptr, dinv); tb::launched(); }
  else
    { k_node_dinv<3, 1, false><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, filt->H3, nullptr, filt->d_fixed, dinv); tb::launched(); }
}
int HelmOp::fused_blocks() const { return nblk(filt->g.n_nodes); }

// Grid of the single-reduction persistent kernel (one CTA per SM, every CTA co-resident), or 0
// when the device cannot launch it cooperatively or a CTA's node range exceeds shared memory.
template <int NC, bool SCALED>
static int persist_grid_for(const Grid& g, TileSpec* ts) {
  int dev = 0, sms = 0, coop = 0, occ = 0, smem_max = 0;
  if (g.dim != 2 || cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (!coop || sms < 1 || getenv("TB_NO_PERSIST") != nullptr) return 0;  // env: graph path (tests)
  // at most one CTA per SM, at least ~128 nodes per CTA (fewer CTAs = cheaper barriers)
  const int64_t want = (g.n_nodes + 127) / 128;
  // partials: 2 parities x 3 sums x grid must fit PcgWork::partA (2 x >= 592 doubles)
  const int cap = sms < 192 ? sms : 192;
  int grid = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  if (getenv("TB_CG_STRIP") == nullptr) {  // 2D node tiles (cgtile2d.cuh); strips for A/B only
    *ts = choose_tiles(g.nnx, g.nny, grid);
    grid = ts->tx * ts->ty;
    // register-resident state pays off once a tile has more nodes than threads (cfg 2: 841
    // nodes, 6.5 vs 6.8 us/iteration); small tiles (cfg 1: ~128 nodes) are faster with SMEM state
    const int64_t tn = (int64_t)ts->tw * ts->th;
    if (tn > kCgcgThreads && tn <= (int64_t)kTregSlots * kTregThreads && getenv("TB_CG_SMEMSTATE") == nullptr) {
      const size_t rsm = treg_smem_bytes(NC, *ts);
      int r1 = 0, r2 = 0;
      if (rsm + 2048 <= (size_t)smem_max &&
          cudaFuncSetAttribute(k_pcg2d_treg<NC, SCALED, false, kTregSlots, kTregThreads>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm) == cudaSuccess &&
          cudaFuncSetAttribute(k_pcg2d_treg<NC, SCALED, true, kTregSlots, kTregThreads>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm) == cudaSuccess &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r1, k_pcg2d_treg<NC, SCALED, false, kTregSlots, kTregThreads>,
                                                        kTregThreads, rsm) == cudaSuccess &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r2, k_pcg2d_treg<NC, SCALED, true, kTregSlots, kTregThreads>,
                                                        kTregThreads, rsm) == cudaSuccess &&
          r1 >= 1 && r2 >= 1 && grid <= sms) {
        ts->reg = 1;
        return grid;
      }
    }
    const size_t tsm = tile_smem_bytes(NC, *ts);
    int o1 = 0, o2 = 0;
    if (tsm + 2048 <= (size_t)smem_max &&
        cudaFuncSetAttribute(k_pcg2d_tile<NC, SCALED, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tsm) == cudaSuccess &&
        cudaFuncSetAttribute(k_pcg2d_tile<NC, SCALED, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tsm) == cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_pcg2d_tile<NC, SCALED, false>, kCgcgThreads, tsm) ==
            cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_pcg2d_tile<NC, SCALED, true>, kCgcgThreads, tsm) ==
            cudaSuccess &&
        o1 >= 1 && o2 >= 1 && grid <= sms)
      return grid;
    grid = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  }
  ts->tx = 0;  // row strips
  const int64_t own = (g.n_nodes + grid - 1) / grid;
  const size_t smem = cgcg_smem_bytes(NC, own, g.nnx, g.nx);
  if (smem + 2048 > (size_t)smem_max) return 0;
  if (cudaFuncSetAttribute(k_pcg2d_cgcg<NC, SCALED, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess ||
      cudaFuncSetAttribute(k_pcg2d_cgcg<NC, SCALED, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
    return 0;
  int occ2 = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_pcg2d_cgcg<NC, SCALED, false>, kCgcgThreads, smem) !=
          cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_pcg2d_cgcg<NC, SCALED, true>, kCgcgThreads, smem) !=
          cudaSuccess ||
      occ < 1 || occ2 < 1)
    return 0;
  return grid;
}

template <int NC, bool SCALED>
static void launch_cgcg(const Grid& g, const Mat<4 * NC>& K, const Q4Pat* pat, const double* alpha,
                        const PcgWork& w, int grid, const TileSpec& tiles, cudaStream_t s) {
  const int64_t own = (g.n_nodes + grid - 1) / grid;
  const size_t smem = tiles.tx > 0 ? tile_smem_bytes(NC, tiles) : cgcg_smem_bytes(NC, own, g.nnx, g.nx);
  CgcgArgs a{nullptr, w.x, w.r, w.dinv, w.pub, w.partA(), w.st, reinterpret_cast<unsigned int*>(w.barrier),
             (int)own, 0};
#if defined(TB_CGCG_PROF) || defined(TB_CGCG_ABL)
  if (const char* e = getenv("TB_CGCG_DBG")) a.dbg = (NC == 2) ? atoi(e) : 0;
#endif
  Grid gg = g;
  Mat<4 * NC> KK = K;
  Q4Pat kp = pat ? *pat : Q4Pat{};
  const double* al = alpha;
  TileSpec ts = tiles;
  if (tiles.tx > 0 && tiles.reg) {
    void* targs[] = {&gg, &KK, &kp, &al, &a, &ts};
    const size_t rsm = treg_smem_bytes(NC, tiles);
    if (pat)
      cudaLaunchCooperativeKernel((const void*)k_pcg2d_treg<NC, SCALED, true, kTregSlots, kTregThreads>, grid, kTregThreads,
                                  targs, rsm, s);
    else
      cudaLaunchCooperativeKernel((const void*)k_pcg2d_treg<NC, SCALED, false, kTregSlots, kTregThreads>, grid, kTregThreads,
                                  targs, rsm, s);
    return;
  }
  if (tiles.tx > 0) {
    void* targs[] = {&gg, &KK, &kp, &al, &a, &ts};
    if (pat)
      cudaLaunchCooperativeKernel((const void*)k_pcg2d_tile<NC, SCALED, true>, grid, kCgcgThreads, targs, smem, s);
    else
      cudaLaunchCooperativeKernel((const void*)k_pcg2d_tile<NC, SCALED, false>, grid, kCgcgThreads, targs, smem, s);
    return;
  }
  void* args[] = {&gg, &KK, &kp, &al, &a};
  if (pat)
    cudaLaunchCooperativeKernel((const void*)k_pcg2d_cgcg<NC, SCALED, true>, grid, kCgcgThreads, args, smem, s);
  else
    cudaLaunchCooperativeKernel((const void*)k_pcg2d_cgcg<NC, SCALED, false>, grid, kCgcgThreads, args, smem, s);
}

void ElastOp::launch_persistent(const PcgWork& w, cudaStream_t s) const {
  launch_cgcg<2, true>(plan->g, plan->K2, plan->pat_ok ? &plan->pat : nullptr, plan->d_alpha, w, persist_grid, tiles,
                       s);
}

void HelmOp::launch_persistent(const PcgWork& w, cudaStream_t s) const {
  launch_cgcg<1, false>(filt->g, filt->H2, filt->pat_ok ? &filt->pat : nullptr, nullptr, w, persist_grid, tiles, s);
}

void tb_plan_impl::apply_alpha(const double* alpha, const double* v, double* y, bool mask, cudaStream_t s) const {
  const uint8_t* fx = mask ? d_fixed : nullptr;
  if (g.dim == 2)
    { k_node_apply<2, 2, true><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, K2, alpha, v, y, fx); tb::launched(); }
  else if (hex8) {
    { k_hex8<false><<<hex8_grid(g, zchunk), kHT, kHex8Smem, s>>>(g, hiso, alpha, v, nullptr, nullptr, y, nullptr, nullptr, zchunk, 0.0, 3.0, mask ? d_fixed_idx : nullptr, mask ? d_fixed_off : nullptr); tb::launched(); }
  } else
    { k_node_apply<3, 3, true><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, K3, alpha, v, y, fx); tb::launched(); }
}

// Hex8 operator with an epilogue on the owned nodes (k_hex8 EPI): epi 1: out = v + omega dinv (b - K v),
// epi 2: out = dinv != 0 ? b - K v : 0.  out must not alias v (other CTAs read v's halo).
bool tb_plan_impl::apply_alpha_epi(int epi, const double* alpha, const double* v, double* out, const double* b,
                                   const double* dinv, double omega, cudaStream_t s) const {
  if (g.dim != 3 || !hex8 || !hex8_epi) return false;
  if (epi == 1)
    k_hex8<false, false, 1><<<hex8_grid(g, zchunk), kHT, kHex8Smem, s>>>(g, hiso, alpha, v, nullptr, nullptr, out,
                                                                         nullptr, nullptr, zchunk, 0.0, 3.0, nullptr,
                                                                         nullptr, 0, 0, b, dinv, omega);
  else
    k_hex8<false, false, 2><<<hex8_grid(g, zchunk), kHT, kHex8Smem, s>>>(g, hiso, alpha, v, nullptr, nullptr, out,
                                                                         nullptr, nullptr, zchunk, 0.0, 3.0, nullptr,
                                                                         nullptr, 0, 0, b, dinv, omega);
  tb::launched();
  return true;
}

int tb_plan_impl::material(const double* rho, double* alpha, double* dalpha, cudaStream_t s) const {
  { k_material<<<grid_for(g.n_elems), kBlock, 0, s>>>(g.n_elems, rho_l, p, rho, alpha, dalpha); tb::launched(); }
  TB_CHECK_LAUNCH();
  return TB_OK;
}

}  // namespace tb

using namespace tb;

// =========================================================================================
// C ABI
// =========================================================================================
extern "C" {

int tb_version(void) { return 100; }
const char* tb_last_error(void) { return g_err; }

#define TB_GUARD(cond, ...)        \
  do {                             \
    if (!(cond)) {                 \
      set_error(__VA_ARGS__);      \
      return TB_ERR_INVALID;       \
    }                              \
  } while (0)

int tb_plan_create(int dim, int nx, int ny, int nz, double h, const double* k_e, double rho_l, double p,
                   const uint8_t* fixed, int device, tb_plan** out) {
  TB_GUARD(out != nullptr && k_e != nullptr && fixed != nullptr, "null argument");
  TB_GUARD(dim == 2 || dim == 3, "dim must be 2 or 3, got %d", dim);
  TB_GUARD(nx >= 1 && ny >= 1 && (dim == 2 || nz >= 1), "element counts must be >= 1");
  TB_GUARD(h > 0.0, "element size must be positive, got %g", h);
  TB_GUARD(rho_l > 0.0 && rho_l < 1.0 && p >= 1.0, "material parameters out of range");
  TB_CUDA(cudaSetDevice(device));
  auto* P = new tb_plan_impl();
  P->g = make_grid(dim, nx, ny, nz, h);
  const Grid& g = P->g;
  P->n_dofs = (int64_t)dim * g.n_nodes;
  P->device = device;
  P->rho_l = rho_l;
  P->p = p;
  const int ne = (dim == 2) ? 8 : 24;
  if (dim == 2) {
    memcpy(P->K2.v, k_e, sizeof(double) * ne * ne);
    P->pat_ok = q4_pattern_values(2, P->K2.v, &P->pat) && getenv("TB_NO_Q4PAT") == nullptr;
  } else {
    memcpy(P->K3.v, k_e, sizeof(double) * ne * ne);
  }
  P->op.plan = P;
  if (dim == 3) {
    P->hex8 = hex8_blocks(P->K3.v, &P->hiso);
    P->zchunk = hex8_zchunk(P->g);
    if (P->hex8) {
      cudaError_t e1 = cudaFuncSetAttribute(k_hex8<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHex8Smem);
      cudaError_t e2 = cudaFuncSetAttribute(k_hex8<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHex8Smem);
      cudaError_t e3 = cudaFuncSetAttribute(k_hex8<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHex8Smem);
      if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess)
        P->hex8 = false;
      P->hex8_epi = P->hex8 &&
                    cudaFuncSetAttribute(k_hex8<false, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kHex8Smem) == cudaSuccess &&
                    cudaFuncSetAttribute(k_hex8<false, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kHex8Smem) == cudaSuccess;
    }
  }
  if (dim == 2) P->op.persist_grid = persist_grid_for<2, true>(P->g, &P->op.tiles);
  int rc = P->init(fixed);
  if (rc != TB_OK) {
    P->release();
    delete P;
    return rc;
  }
  *out = reinterpret_cast<tb_plan*>(P);
  return TB_OK;
}

int tb_plan_destroy(tb_plan* plan) {
  if (!plan) return TB_OK;
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  cudaSetDevice(P->device);
  P->release();
  delete P;
  return TB_OK;
}

int tb_plan_sizes(const tb_plan* plan, int64_t* n_elems, int64_t* n_nodes, int64_t* n_dofs) {
  TB_GUARD(plan != nullptr, "null plan");
  auto* P = reinterpret_cast<const tb_plan_impl*>(plan);
  if (n_elems) *n_elems = P->g.n_elems;
  if (n_nodes) *n_nodes = P->g.n_nodes;
  if (n_dofs) *n_dofs = P->n_dofs;
  return TB_OK;
}

int tb_material(tb_plan* plan, const double* rho, double* alpha, double* dalpha, void* stream) {
  TB_GUARD(plan && rho, "null argument");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  return P->material(rho, alpha, dalpha, (cudaStream_t)stream);
}

int tb_clamp_density(tb_plan* plan, const double* rho_raw, double* rho, double* clamp_width, void* stream) {
  TB_GUARD(plan && rho_raw && rho, "null argument");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = grid_for(P->g.n_elems);
  { k_clamp<<<nb, kBlock, 0, s>>>(P->g.n_elems, P->rho_l, rho_raw, rho, P->d_scratch); tb::launched(); }
  { k_finish<<<1, kBlock, 0, s>>>(nb, P->d_scratch, P->d_scalar, 1); tb::launched(); }
  TB_CHECK_LAUNCH();
  if (clamp_width) {
    TB_CUDA(cudaMemcpyAsync(P->h_scalar, P->d_scalar, sizeof(double), cudaMemcpyDeviceToHost, s));
    TB_CUDA(cudaStreamSynchronize(s));
    *clamp_width = *P->h_scalar;
  }
  return TB_OK;
}

int tb_apply_stiffness(tb_plan* plan, const double* rho, const double* v, double* y, int mask_rows, void* stream) {
  TB_GUARD(plan && rho && v && y, "null argument");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  cudaStream_t s = (cudaStream_t)stream;
  if (P->g.dim == 2 && P->p == 3.0) {  // alpha(rho) inside the node apply: one launch
    { k_node_apply<2, 2, true, true><<<nblk(P->g.n_nodes), kBlock, 0, s>>>(P->g, P->K2, rho, v, y, mask_rows ? P->d_fixed : nullptr, P->rho_l); tb::launched(); }
    TB_CHECK_LAUNCH();
    return TB_OK;
  }
  if (P->g.dim == 3 && P->hex8 && P->p == 3.0) {  // alpha(rho) inside the operator pass
    const Grid& g = P->g;
    { k_hex8<false, true><<<hex8_grid(g, P->zchunk), kHT, kHex8Smem, s>>>(g, P->hiso, rho, v, nullptr, nullptr, y, nullptr, nullptr, P->zchunk, P->rho_l, P->p, mask_rows ? P->d_fixed_idx : nullptr, mask_rows ? P->d_fixed_off : nullptr); tb::launched(); }
    TB_CHECK_LAUNCH();
    return TB_OK;
  }
  TB_TRY(P->material(rho, P->d_alpha2, nullptr, s));
  P->apply_alpha(P->d_alpha2, v, y, mask_rows != 0, s);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

int tb_element_sensitivity(tb_plan* plan, const double* rho, const double* u, const double* lam, const double* drho,
                           double* s_out, void* stream) {
  TB_GUARD(plan && rho && u && lam && s_out, "null argument");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  cudaStream_t s = (cudaStream_t)stream;
  const Grid& g = P->g;
  if (g.dim == 2)
    { k_elem_sensitivity<2><<<nblk(g.n_elems), kBlock, 0, s>>>(g, P->K2, P->rho_l, P->p, rho, u, lam, drho, s_out); tb::launched(); }
  else
    { k_elem_sensitivity<3><<<nblk(g.n_elems), kBlock, 0, s>>>(g, P->K3, P->rho_l, P->p, rho, u, lam, drho, s_out); tb::launched(); }
  TB_CHECK_LAUNCH();
  return TB_OK;
}

int tb_pcg_solve(tb_plan* plan, const double* rho, const double* b, double* x, double rtol, int maxit, int* iters,
                 double* relres, void* stream) {
  TB_GUARD(plan && rho && b && x, "null argument");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  cudaStream_t s = (cudaStream_t)stream;
  if (P->dist) {
    P->dist = 0;
    TB_TRY(P->work.set_fields(0, P->own_k0, P->own_k1));
  }
  TB_TRY(P->material(rho, P->d_alpha, nullptr, s));
  if (sweep_enabled(P)) return pcg_solve_sweep(P, b, x, rtol, maxit, iters, relres, s);
  return pcg_solve(P->op, P->work, b, x, rtol, maxit, iters, relres, s);
}

int tb_pcg_path(tb_plan* plan) {
  if (plan == nullptr) return -1;
  return sweep_enabled(reinterpret_cast<tb_plan_impl*>(plan)) ? 1 : 0;
}

int tb_pcg_kernel_time(tb_plan* plan, float* ms, int* launches) {
  TB_GUARD(plan && ms && launches, "null argument");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  *ms = 0.0f;
  *launches = P->work.klaunches;
  if (P->work.klaunches > 0) {
    TB_CUDA(cudaEventSynchronize(P->work.kev1));
    TB_CUDA(cudaEventElapsedTime(ms, P->work.kev0, P->work.kev1));
  }
  return TB_OK;
}

int tb_pcg_profile(tb_plan* plan, const double* rho, const double* b, int nrep, double* ms_fused, double* ms_update,
                   void* stream) {
  TB_GUARD(plan && rho && b && ms_fused && ms_update && nrep >= 1, "bad arguments");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  cudaStream_t s = (cudaStream_t)stream;
  TB_TRY(P->material(rho, P->d_alpha, nullptr, s));
  if (sweep_enabled(P)) {
    *ms_update = 0.0;
    return pcg_profile_sweep(P, b, nrep, ms_fused, s);
  }
  return pcg_profile(P->op, P->work, b, nrep, ms_fused, ms_update, s);
}

int tb_pcg_iter_time(tb_plan* plan, int reset, double* ms, int64_t* iters) {
  TB_GUARD(plan && ms && iters, "null argument");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  TB_GUARD(sweep_enabled(P), "iteration timing is kept by the single-sweep path only (tb_pcg_path == 1)");
  return pcg_iter_time_sweep(P, reset, ms, iters);
}

int64_t tb_launch_count(void) { return g_launches.load(); }

int tb_plan_set_preconditioner(tb_plan* plan, int kind) {
  TB_GUARD(plan != nullptr, "null plan");
  TB_GUARD(kind == 0 || kind == 1, "preconditioner must be 0 (Jacobi) or 1 (multigrid), got %d", kind);
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  if (kind == 1) TB_TRY(mg_build(P));
  P->precond = kind;
  return TB_OK;
}

int tb_plan_set_owned_planes(tb_plan* plan, int k0, int k1) {
  TB_GUARD(plan != nullptr, "null plan");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  TB_GUARD(0 <= k0 && k0 <= k1 && k1 <= P->g.nnz, "owned node planes [%d, %d) outside [0, %d]", k0, k1, P->g.nnz);
  P->own_k0 = k0;
  P->own_k1 = k1;
  const int64_t pd = (int64_t)P->g.dim * P->g.nnx * P->g.nny;
  P->work.plane = pd;
  P->work.own0 = k0 * pd;
  P->work.own1 = k1 * pd;
  return P->work.set_fields(P->dist, k0, k1);
}

int tb_plan_set_halo_peers(tb_plan* plan, double* lo_dst, double* hi_dst) {
  TB_GUARD(plan != nullptr, "null plan");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  TB_GUARD(P->work.plane > 0, "tb_plan_set_halo_peers needs tb_plan_set_owned_planes first");
  TB_GUARD(lo_dst == nullptr || P->own_k0 > 0, "no lower neighbour: owned planes start at 0");
  TB_GUARD(hi_dst == nullptr || P->own_k1 < P->g.nnz, "no upper neighbour: owned planes reach the top");
  P->work.halo_lo = lo_dst;
  P->work.halo_hi = hi_dst;
  return TB_OK;
}

int tb_ipc_get_handle(const void* dptr, void* handle) {
  TB_GUARD(dptr != nullptr && handle != nullptr, "null argument");
  cudaIpcMemHandle_t h;
  TB_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)));
  memcpy(handle, &h, sizeof(h));
  return TB_OK;
}

int tb_ipc_open(const void* handle, int device, void** dptr) {
  TB_GUARD(dptr != nullptr && handle != nullptr, "null argument");
  TB_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  TB_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return TB_OK;
}

int tb_ipc_close(void* dptr) {
  if (dptr != nullptr) TB_CUDA(cudaIpcCloseMemHandle(dptr));
  return TB_OK;
}

int tb_pcg_dist_phase(tb_plan* plan, int phase, const double* rho, const double* b, double rtol, int maxit,
                      int parity, void* stream) {
  TB_GUARD(plan != nullptr, "null plan");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  cudaStream_t s = (cudaStream_t)stream;
  if (phase == 0 || phase == 10) {
    TB_GUARD(rho && b, "phase %d needs rho and b", phase);
    TB_GUARD(rtol > 0.0 && maxit >= 1, "rtol must be > 0 and maxit >= 1");
    TB_GUARD(phase == 0 || (P->g.dim == 3 && P->hex8), "single-reduction phases need a Hex8 plan");
    if (!P->dist) {
      P->dist = 1;
      TB_TRY(P->work.set_fields(1, P->own_k0, P->own_k1));
    }
    TB_TRY(P->material(rho, P->d_alpha, nullptr, s));
  }
  return pcg_dist_phase(P->op, P->work, phase, b, rtol, maxit, parity, s);
}

int tb_pcg_dist_buffers(tb_plan* plan, double** x, double** z, double** red) {
  TB_GUARD(plan != nullptr, "null plan");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  if (x) *x = P->work.x;
  if (z) *z = P->work.z;
  if (red) *red = P->work.st->red;
  return TB_OK;
}

int tb_pcg_dist_state(tb_plan* plan, int* iters, int* done, double* rr, double* bb, void* stream) {
  TB_GUARD(plan != nullptr, "null plan");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  cudaStream_t s = (cudaStream_t)stream;
  TB_CUDA(cudaMemcpyAsync(P->work.h_st, P->work.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  TB_CUDA(cudaStreamSynchronize(s));
  const PcgState& h = *P->work.h_st;
  if (iters) *iters = h.iters;
  if (done) *done = h.done;
  if (rr) *rr = h.rr;
  if (bb) *bb = h.bb;
  return TB_OK;
}

int tb_dot(tb_plan* plan, const double* a, const double* b, int64_t n, double* out, void* stream) {
  TB_GUARD(plan && a && b && out, "null argument");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  cudaStream_t s = (cudaStream_t)stream;
  TB_TRY(device_dot(a, b, n, P->d_scratch, P->d_scalar, s));
  TB_CUDA(cudaMemcpyAsync(P->h_scalar, P->d_scalar, sizeof(double), cudaMemcpyDeviceToHost, s));
  TB_CUDA(cudaStreamSynchronize(s));
  *out = *P->h_scalar;
  return TB_OK;
}

// ---------------------------------------------------------------------------------------
// Helmholtz filter
// ---------------------------------------------------------------------------------------
int tb_filter_create(int dim, int nx, int ny, int nz, double h, double radius, int device, tb_filter** out) {
  TB_GUARD(out != nullptr, "null argument");
  TB_GUARD(dim == 2 || dim == 3, "dim must be 2 or 3, got %d", dim);
  TB_GUARD(nx >= 1 && ny >= 1 && (dim == 2 || nz >= 1), "element counts must be >= 1");
  TB_GUARD(h > 0.0, "element size must be positive, got %g", h);
  TB_GUARD(radius >= 0.0, "filter radius must be nonnegative, got %g", radius);
  TB_CUDA(cudaSetDevice(device));
  auto* F = new tb_filter_impl();
  F->g = make_grid(dim, nx, ny, nz, h);
  F->device = device;
  F->radius = radius;
  F->r = (1.0 / (2.0 * sqrt(3.0))) * radius;  // LENGTH_SCALE_FACTOR * R (filtering.py:29-32,59)
  const Grid& g = F->g;
  const int nn = (g.dim == 2) ? 4 : 8;
  double S[64], M[64], s_div, m_mul;
  scalar_element_matrices(g.dim, g.h, S, M, &s_div, &m_mul);
  // H_e = r^2 S_e + M_e in the reference's operation order (fem.py:135)
  const double r2 = (g.dim == 2) ? F->r * F->r : F->r * F->r * g.h;
  for (int i = 0; i < nn * nn; ++i) {
    const double hv = r2 * S[i] / s_div + m_mul * M[i];
    if (g.dim == 2)
      F->H2.v[i] = hv;
    else
      F->H3.v[i] = hv;
  }
  F->vol_share = pow(g.h, g.dim) / nn;  // b_e entries = h^d / 2^d (filtering.py:75-76)
  if (g.dim == 2) F->pat_ok = q4_pattern_values(1, F->H2.v, &F->pat);
  if (g.dim == 3) F->iso3 = helm3d_iso(F->H3.v, F->h4);
  F->op.filt = F;
  F->op.persist_grid = (g.dim == 2) ? persist_grid_for<1, false>(g, &F->op.tiles) : 0;  // 3D: graph loop
  int rc = F->work.alloc(g.n_nodes, F->op.fused_blocks(), F->op.persist_grid > 0);
  if (rc == TB_OK) rc = F->work.set_fields(0, 0, g.nnz);
  if (rc == TB_OK) {
    cudaError_t e = cudaMalloc(&F->d_b, sizeof(double) * g.n_nodes);
    if (e != cudaSuccess) {
      set_error("cudaMalloc: %s", cudaGetErrorString(e));
      rc = TB_ERR_CUDA;
    }
  }
  if (rc != TB_OK) {
    F->work.release();
    delete F;
    return rc;
  }
  spectral_init(F);
  *out = reinterpret_cast<tb_filter*>(F);
  return TB_OK;
}

int tb_filter_destroy(tb_filter* filt) {
  if (!filt) return TB_OK;
  auto* F = reinterpret_cast<tb_filter_impl*>(filt);
  cudaSetDevice(F->device);
  spectral_release(F);
  F->work.release();
  if (F->d_b) cudaFree(F->d_b);
  if (F->d_fixed) cudaFree(F->d_fixed);
  delete F;
  return TB_OK;
}

int tb_filter_load_vector(tb_filter* filt, const double* psi, double* b, void* stream) {
  TB_GUARD(filt && psi && b, "null argument");
  auto* F = reinterpret_cast<tb_filter_impl*>(filt);
  const Grid& g = F->g;
  cudaStream_t s = (cudaStream_t)stream;
  if (g.dim == 2)
    { k_elem_to_node<2><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, psi, F->vol_share, 1.0, b); tb::launched(); }
  else
    { k_elem_to_node<3><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, psi, F->vol_share, 1.0, b); tb::launched(); }
  TB_CHECK_LAUNCH();
  return TB_OK;
}

}  // extern "C"

// a whole-grid solve after slab phases: dots over every node plane again
static int filter_single_mode(tb_filter_impl* F) {
  if (!F->dist) return TB_OK;
  F->dist = 0;
  return F->work.set_fields(0, F->own_k0, F->own_k1);
}

// whole-grid H x = d_b into work.x: direct (spectral.cu, 0 iterations) or pCG
static int filter_solve(tb_filter_impl* F, double rtol, int* iters, cudaStream_t s) {
  if (F->spec != nullptr) {
    if (iters) *iters = 0;
    return spectral_solve(F, F->d_b, F->work.x, s);
  }
  TB_TRY(filter_single_mode(F));
  return pcg_solve(F->op, F->work, F->d_b, F->work.x, rtol, 10000, iters, nullptr, s);
}

extern "C" {

int tb_filter_apply(tb_filter* filt, const double* psi, double* phi, double* rho, double rtol, int* iters,
                    void* stream) {
  TB_GUARD(filt && psi && rho, "null argument");
  auto* F = reinterpret_cast<tb_filter_impl*>(filt);
  const Grid& g = F->g;
  cudaStream_t s = (cudaStream_t)stream;
  TB_TRY(tb_filter_load_vector(filt, psi, F->d_b, stream));
  TB_TRY(filter_solve(F, rtol, iters, s));
  const double inv_nn = (g.dim == 2) ? 0.25 : 0.125;
  if (g.dim == 2)
    { k_node_to_elem<2><<<nblk(g.n_elems), kBlock, 0, s>>>(g, F->work.x, inv_nn, rho); tb::launched(); }
  else
    { k_node_to_elem<3><<<nblk(g.n_elems), kBlock, 0, s>>>(g, F->work.x, inv_nn, rho); tb::launched(); }
  TB_CHECK_LAUNCH();
  if (phi) TB_CUDA(cudaMemcpyAsync(phi, F->work.x, sizeof(double) * g.n_nodes, cudaMemcpyDeviceToDevice, s));
  return TB_OK;
}

int tb_filter_adjoint(tb_filter* filt, const double* v, double* w, double rtol, int* iters, void* stream) {
  TB_GUARD(filt && v && w, "null argument");
  auto* F = reinterpret_cast<tb_filter_impl*>(filt);
  const Grid& g = F->g;
  cudaStream_t s = (cudaStream_t)stream;
  const double inv_nn = (g.dim == 2) ? 0.25 : 0.125;
  if (g.dim == 2)
    { k_elem_to_node<2><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, v, inv_nn, 1.0, F->d_b); tb::launched(); }
  else
    { k_elem_to_node<3><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, v, inv_nn, 1.0, F->d_b); tb::launched(); }
  TB_CHECK_LAUNCH();
  TB_TRY(filter_solve(F, rtol, iters, s));
  if (g.dim == 2)
    { k_node_to_elem<2><<<nblk(g.n_elems), kBlock, 0, s>>>(g, F->work.x, F->vol_share, w); tb::launched(); }
  else
    { k_node_to_elem<3><<<nblk(g.n_elems), kBlock, 0, s>>>(g, F->work.x, F->vol_share, w); tb::launched(); }
  TB_CHECK_LAUNCH();
  return TB_OK;
}

// ---- slab-distributed Helmholtz filter (BASELINE cfg 4; same phases as tb_pcg_dist_phase) ----
int tb_filter_set_owned_planes(tb_filter* filt, int k0, int k1) {
  TB_GUARD(filt != nullptr, "null filter");
  auto* F = reinterpret_cast<tb_filter_impl*>(filt);
  const Grid& g = F->g;
  TB_GUARD(g.dim == 3, "slab filters are 3D");
  TB_GUARD(0 <= k0 && k0 < k1 && k1 <= g.nnz, "owned node planes [%d, %d) outside [0, %d]", k0, k1, g.nnz);
  const int64_t pd = (int64_t)g.nnx * g.nny;
  if (F->d_fixed == nullptr) TB_CUDA(cudaMalloc(&F->d_fixed, (size_t)g.n_nodes));
  // ghost node planes are rows this rank never updates: Dirichlet-masked like the slab plan's
  TB_CUDA(cudaMemset(F->d_fixed, 0, (size_t)g.n_nodes));
  if (k0 > 0) TB_CUDA(cudaMemset(F->d_fixed, 1, (size_t)(k0 * pd)));
  if (k1 < g.nnz) TB_CUDA(cudaMemset(F->d_fixed + k1 * pd, 1, (size_t)((g.nnz - k1) * pd)));
  F->own_k0 = k0;
  F->own_k1 = k1;
  F->work.plane = pd;
  F->work.own0 = k0 * pd;
  F->work.own1 = k1 * pd;
  return F->work.set_fields(F->dist, k0, k1);
}

int tb_filter_dist_phase(tb_filter* filt, int phase, const double* b, double rtol, int maxit, int parity,
                         void* stream) {
  TB_GUARD(filt != nullptr, "null filter");
  auto* F = reinterpret_cast<tb_filter_impl*>(filt);
  TB_GUARD(F->work.plane > 0, "tb_filter_dist_phase needs tb_filter_set_owned_planes first");
  if (phase == 0) {
    TB_GUARD(b != nullptr, "phase 0 needs b");
    TB_GUARD(rtol > 0.0 && maxit >= 1, "rtol must be > 0 and maxit >= 1");
    if (!F->dist) {
      F->dist = 1;
      TB_TRY(F->work.set_fields(1, F->own_k0, F->own_k1));
    }
  }
  return pcg_dist_phase(F->op, F->work, phase, b, rtol, maxit, parity, (cudaStream_t)stream);
}

int tb_filter_dist_buffers(tb_filter* filt, double** x, double** z, double** red) {
  TB_GUARD(filt != nullptr, "null filter");
  auto* F = reinterpret_cast<tb_filter_impl*>(filt);
  if (x) *x = F->work.x;
  if (z) *z = F->work.z;
  if (red) *red = F->work.st->red;
  return TB_OK;
}

int tb_filter_dist_state(tb_filter* filt, int* iters, int* done, double* rr, double* bb, void* stream) {
  TB_GUARD(filt != nullptr, "null filter");
  auto* F = reinterpret_cast<tb_filter_impl*>(filt);
  cudaStream_t s = (cudaStream_t)stream;
  TB_CUDA(cudaMemcpyAsync(F->work.h_st, F->work.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  TB_CUDA(cudaStreamSynchronize(s));
  const PcgState& h = *F->work.h_st;
  if (iters) *iters = h.iters;
  if (done) *done = h.done;
  if (rr) *rr = h.rr;
  if (bb) *bb = h.bb;
  return TB_OK;
}

int tb_filter_set_halo_peers(tb_filter* filt, double* lo_dst, double* hi_dst) {
  TB_GUARD(filt != nullptr, "null filter");
  auto* F = reinterpret_cast<tb_filter_impl*>(filt);
  TB_GUARD(F->work.plane > 0, "tb_filter_set_halo_peers needs tb_filter_set_owned_planes first");
  TB_GUARD(lo_dst == nullptr || F->own_k0 > 0, "no lower neighbour: owned planes start at 0");
  TB_GUARD(hi_dst == nullptr || F->own_k1 < F->g.nnz, "no upper neighbour: owned planes reach the top");
  F->work.halo_lo = lo_dst;
  F->work.halo_hi = hi_dst;
  return TB_OK;
}

int tb_filter_transfer(tb_filter* filt, int mode, const double* in, double scale, double* out, void* stream) {
  TB_GUARD(filt && in && out, "null argument");
  TB_GUARD(mode == 0 || mode == 1, "mode must be 0 (element -> node) or 1 (node -> element), got %d", mode);
  auto* F = reinterpret_cast<tb_filter_impl*>(filt);
  const Grid& g = F->g;
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 0) {
    if (g.dim == 2)
      { k_elem_to_node<2><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, in, scale, 1.0, out); tb::launched(); }
    else
      { k_elem_to_node<3><<<nblk(g.n_nodes), kBlock, 0, s>>>(g, in, scale, 1.0, out); tb::launched(); }
  } else {
    if (g.dim == 2)
      { k_node_to_elem<2><<<nblk(g.n_elems), kBlock, 0, s>>>(g, in, scale, out); tb::launched(); }
    else
      { k_node_to_elem<3><<<nblk(g.n_elems), kBlock, 0, s>>>(g, in, scale, out); tb::launched(); }
  }
  TB_CHECK_LAUNCH();
  return TB_OK;
}

}  // extern "C"
