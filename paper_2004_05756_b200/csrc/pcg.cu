// pCG engine implementation (see pcg.cuh).
#include <stddef.h>
#include <stdlib.h>

#include "pcg.cuh"

namespace tb {

int PcgWork::alloc(int64_t n_, int max_blocks, bool with_pub, int64_t cap) {
  n = n_;
  part_stride = max_blocks > kUpdateBlocks ? max_blocks : kUpdateBlocks;
  const size_t vb = sizeof(double) * (size_t)(cap > n ? cap : n);
  double** vecs[] = {&x, &r, &z, &pa, &pb, &q, &dinv, &tmp};
  for (double** p : vecs) TB_CUDA(cudaMalloc(p, vb));
  TB_CUDA(cudaMalloc(&part, sizeof(double) * 6 * (size_t)part_stride));
  TB_CUDA(cudaMalloc(&st, sizeof(PcgState)));
  TB_CUDA(cudaMemset(st, 0, sizeof(PcgState)));
  TB_CUDA(cudaMallocHost(&h_st, sizeof(PcgState)));
  TB_CUDA(cudaMalloc(&barrier, 64));
  TB_CUDA(cudaMemset(barrier, 0, 64));
  if (with_pub) TB_CUDA(cudaMalloc(&pub, sizeof(double) * 6 * (size_t)n));
  return TB_OK;
}

int PcgWork::set_fields(int dist, int dot_k0, int dot_k1) {
  const int v[3] = {dist, dot_k0, dot_k1};
  TB_CUDA(cudaMemcpy(reinterpret_cast<char*>(st) + offsetof(PcgState, dist), v, sizeof(v), cudaMemcpyHostToDevice));
  return TB_OK;
}

void PcgWork::release() {
  double* vecs[] = {x, r, z, pa, pb, q, dinv, tmp, part};
  for (double* p : vecs)
    if (p) cudaFree(p);
  if (st) cudaFree(st);
  if (h_st) cudaFreeHost(h_st);
  if (barrier) cudaFree(barrier);
  if (pub) cudaFree(pub);
  if (exec) cudaGraphExecDestroy(exec);
  if (exec_pc) cudaGraphExecDestroy(exec_pc);
  if (kev0) cudaEventDestroy(kev0);
  if (kev1) cudaEventDestroy(kev1);
  *this = PcgWork();
}

// Kernel B: x += alpha p ; r -= alpha q ; z = D^-1 r on free dofs (dinv != 0); rz, rr.
// Pure streaming (8 vector passes): each thread handles 4 x 2 consecutive dofs per trip with
// 16-byte loads so ~40 independent loads are in flight per thread.
__device__ __forceinline__ void upd2(double a, double2 p, double2 q, double2 d, double2& x, double2& r, double2& z,
                                     double (&acc)[2]) {
  if (d.x != 0.0) {
    x.x = fma(a, p.x, x.x);
    r.x = fma(-a, q.x, r.x);
    z.x = d.x * r.x;
    acc[0] = fma(r.x, z.x, acc[0]);
    acc[1] = fma(r.x, r.x, acc[1]);
  } else {
    z.x = 0.0;
  }
  if (d.y != 0.0) {
    x.y = fma(a, p.y, x.y);
    r.y = fma(-a, q.y, r.y);
    z.y = d.y * r.y;
    acc[0] = fma(r.y, z.y, acc[0]);
    acc[1] = fma(r.y, r.y, acc[1]);
  } else {
    z.y = 0.0;
  }
}

__global__ void __launch_bounds__(kBlock) k_pcg_update(int64_t n, const double* __restrict__ p,
                                                       const double* __restrict__ q, const double* __restrict__ dinv,
                                                       double* __restrict__ x, double* __restrict__ r,
                                                       double* __restrict__ z, PcgState* st, double* partials) {
  if (st->done) return;
  const double a = st->alpha;
  double acc[2] = {0.0, 0.0};
  constexpr int U = 4;
  const int64_t n2 = n / 2;  // double2 count (vectors are 16-byte aligned cudaMalloc buffers)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double2* p2 = reinterpret_cast<const double2*>(p);
  const double2* q2 = reinterpret_cast<const double2*>(q);
  const double2* d2 = reinterpret_cast<const double2*>(dinv);
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* r2 = reinterpret_cast<double2*>(r);
  double2* z2 = reinterpret_cast<double2*>(z);
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 pv[U], qv[U], dv[U], xv[U], rv[U], zv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + u * stride;
      pv[u] = __ldcs(p2 + j);
      qv[u] = __ldcs(q2 + j);
      dv[u] = __ldg(d2 + j);
      xv[u] = x2[j];
      rv[u] = r2[j];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      upd2(a, pv[u], qv[u], dv[u], xv[u], rv[u], zv[u], acc);
      const int64_t j = i + u * stride;
      x2[j] = xv[u];
      r2[j] = rv[u];
      z2[j] = zv[u];
    }
  }
  for (; i < n2; i += stride) {
    double2 pv = p2[i], qv = q2[i], dv = d2[i], xv = x2[i], rv = r2[i], zv;
    upd2(a, pv, qv, dv, xv, rv, zv, acc);
    x2[i] = xv;
    r2[i] = rv;
    z2[i] = zv;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd tail dof
    const int64_t k = n - 1;
    const double di = dinv[k];
    if (di != 0.0) {
      x[k] = fma(a, p[k], x[k]);
      const double ri = fma(-a, q[k], r[k]);
      r[k] = ri;
      z[k] = di * ri;
      acc[0] = fma(ri, z[k], acc[0]);
      acc[1] = fma(ri, ri, acc[1]);
    } else {
      z[k] = 0.0;
    }
  }
  block_sum<2>(acc);
  if (publish_partials<2>(acc, partials, &st->count_b)) {
    gather_partials<2>(acc, partials, &st->count_b);
    if (threadIdx.x == 0 && st->dist) {
      st->red[1] = acc[0];
      st->red[2] = acc[1];
    } else if (threadIdx.x == 0) {
      const int it = st->iters + 1;
      st->iters = it;
      st->beta = acc[0] / st->rz;
      st->rz = acc[0];
      st->rr = acc[1];
      if (!isfinite(acc[0]) || !isfinite(acc[1])) st->done = 3;
      else if (acc[1] <= st->tol2) st->done = 1;
      else if (it >= st->maxit) st->done = 2;
    }
  }
}

// (Re)start: r = Z(b - Kx) (Kx = tmp, or x = 0 when tmp == nullptr), z = D^-1 r, p_old = 0,
// rz, rr; on init also sets tol2 from ||Z b||.
__global__ void __launch_bounds__(kBlock) k_pcg_start(int64_t n, const double* __restrict__ b,
                                                      const double* __restrict__ kx, const double* __restrict__ dinv,
                                                      double* __restrict__ x, double* __restrict__ r,
                                                      double* __restrict__ z, double* __restrict__ pa,
                                                      PcgState* st, double* partials, int init, double rtol,
                                                      int maxit) {
  double acc[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double di = dinv[i];
    double ri = 0.0;
    if (di != 0.0) ri = (kx != nullptr) ? b[i] - kx[i] : b[i];
    if (init) x[i] = 0.0;
    const double zi = di * ri;
    r[i] = ri;
    z[i] = zi;
    pa[i] = 0.0;
    acc[0] = fma(ri, zi, acc[0]);
    acc[1] = fma(ri, ri, acc[1]);
  }
  block_sum<2>(acc);
  if (publish_partials<2>(acc, partials, &st->count_c)) {
    gather_partials<2>(acc, partials, &st->count_c);
    if (threadIdx.x == 0 && st->dist) {
      st->red[1] = acc[0];
      st->red[2] = acc[1];
      if (init) {
        st->iters = 0;
        st->maxit = maxit;
        st->beta = 0.0;
        st->alpha = 0.0;
        st->done = 0;
        st->pq = rtol;  // stashed until tb_pcg_dist_init2 has the global norm
      }
    } else if (threadIdx.x == 0 && !(init == 0 && st->done == 3)) {  // a breakdown stays reported
      if (init) {
        st->tol2 = rtol * rtol * acc[1];
        st->iters = 0;
        st->maxit = maxit;
        st->bb = acc[1];
      }
      st->rz = acc[0];
      st->rr = acc[1];
      st->beta = 0.0;
      st->alpha = 0.0;
      const bool conv = init ? (acc[1] == 0.0) : (acc[1] <= st->tol2);
      st->done = conv ? 1 : (!isfinite(acc[1]) ? 3 : (st->iters >= st->maxit ? 2 : 0));
    }
  }
}

__global__ void k_pcg_cond(cudaGraphConditionalHandle h, const PcgState* st) {
  cudaGraphSetConditional(h, st->done == 0 ? 1u : 0u);
}

static int build_graph(const PcgOp& op, PcgWork& w) {
  cudaStream_t cs;
  TB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaGraph_t g;
  TB_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  TB_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  TB_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  TB_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  for (int it = 0; it < kIters; ++it) {
    double* pold = (it & 1) ? w.pb : w.pa;
    double* pnew = (it & 1) ? w.pa : w.pb;
    op.launch_fused(w, pold, pnew, cs);
    k_pcg_update<<<kUpdateBlocks, kBlock, 0, cs>>>(w.n, pnew, w.q, w.dinv, w.x, w.r, w.z, w.st, w.partB());
  }
  k_pcg_cond<<<1, 1, 0, cs>>>(h, w.st);
  cudaGraph_t captured;
  TB_CUDA(cudaStreamEndCapture(cs, &captured));
  TB_CUDA(cudaGraphInstantiate(&w.exec, g, 0));
  TB_CUDA(cudaGraphDestroy(g));
  TB_CUDA(cudaStreamDestroy(cs));
  return TB_OK;
}

// ---- general preconditioner (multigrid): the update kernel leaves z to M^-1 ----
__global__ void __launch_bounds__(kBlock) k_pcg_update_pc(int64_t n, const double* __restrict__ p,
                                                          const double* __restrict__ q, const double* __restrict__ dinv,
                                                          double* __restrict__ x, double* __restrict__ r, PcgState* st,
                                                          double* partials) {
  if (st->done) return;
  const double a = st->alpha;
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (dinv[i] != 0.0) {
      x[i] = fma(a, p[i], x[i]);
      const double ri = fma(-a, q[i], r[i]);
      r[i] = ri;
      acc[0] = fma(ri, ri, acc[0]);
    }
  }
  block_sum<1>(acc);
  if (publish_partials<1>(acc, partials, &st->count_b)) {
    gather_partials<1>(acc, partials, &st->count_b);
    if (threadIdx.x == 0) {
      const int it = st->iters + 1;
      st->iters = it;
      st->rr = acc[0];
      if (!isfinite(acc[0])) st->done = 3;
      else if (acc[0] <= st->tol2) st->done = 1;
      else if (it >= st->maxit) st->done = 2;
    }
  }
}

// rz = r.z of z = M^-1 r; beta = rz / rz_old (init: beta = 0)
__global__ void __launch_bounds__(kBlock) k_pcg_rz(int64_t n, const double* __restrict__ r, const double* __restrict__ z,
                                                   PcgState* st, double* partials, int init) {
  if (!init && st->done) return;
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc[0] = fma(r[i], z[i], acc[0]);
  block_sum<1>(acc);
  if (publish_partials<1>(acc, partials, &st->count_c)) {
    gather_partials<1>(acc, partials, &st->count_c);
    if (threadIdx.x == 0) {
      st->beta = init ? 0.0 : acc[0] / st->rz;
      st->rz = acc[0];
      if (!(acc[0] > 0.0) && !(st->done)) st->done = (acc[0] == 0.0 && st->rr == 0.0) ? 1 : 3;
    }
  }
}

static void pc_body(const PcgOp& op, PcgWork& w, cudaStream_t s) {
  op.launch_fused(w, w.pa, w.pb, s);
  k_pcg_update_pc<<<kUpdateBlocks, kBlock, 0, s>>>(w.n, w.pb, w.q, w.dinv, w.x, w.r, w.st, w.partB());
  op.precond_apply(w.r, w.z, s);
  k_pcg_rz<<<kUpdateBlocks, kBlock, 0, s>>>(w.n, w.r, w.z, w.st, w.partC(), 0);
  // p is double buffered by copy here (one iteration per body): pb -> pa
  cudaMemcpyAsync(w.pa, w.pb, sizeof(double) * w.n, cudaMemcpyDeviceToDevice, s);
}

static int build_graph_pc(const PcgOp& op, PcgWork& w) {
  cudaStream_t cs;
  TB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaGraph_t g;
  TB_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  TB_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  TB_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  TB_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  pc_body(op, w, cs);
  k_pcg_cond<<<1, 1, 0, cs>>>(h, w.st);
  cudaGraph_t captured;
  TB_CUDA(cudaStreamEndCapture(cs, &captured));
  TB_CUDA(cudaGraphInstantiate(&w.exec_pc, g, 0));
  TB_CUDA(cudaGraphDestroy(g));
  TB_CUDA(cudaStreamDestroy(cs));
  return TB_OK;
}

// TB_PCG_NOGRAPH=1 issues the same kernels as plain stream launches (ncu cannot profile kernel
// nodes of graphs that contain conditional nodes); results are identical.
static bool no_graph() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TB_PCG_NOGRAPH");
    v = (e != nullptr && e[0] != '\0' && e[0] != '0') ? 1 : 0;
  }
  return v == 1;
}

static int run_loop_plain(const PcgOp& op, PcgWork& w, cudaStream_t s) {
  for (;;) {
    for (int it = 0; it < kIters; ++it) {
      double* pold = (it & 1) ? w.pb : w.pa;
      double* pnew = (it & 1) ? w.pa : w.pb;
      op.launch_fused(w, pold, pnew, s);
      k_pcg_update<<<kUpdateBlocks, kBlock, 0, s>>>(w.n, pnew, w.q, w.dinv, w.x, w.r, w.z, w.st, w.partB());
    }
    TB_CHECK_LAUNCH();
    TB_CUDA(cudaMemcpyAsync(w.h_st, w.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    TB_CUDA(cudaStreamSynchronize(s));
    if (w.h_st->done != 0) return TB_OK;
  }
}

// pCG with a general SPD preconditioner (multigrid V-cycle); one iteration per graph body.
static int pcg_solve_pc(const PcgOp& op, PcgWork& w, const double* b, double* x_out, double rtol, int maxit,
                        int* iters, double* relres, cudaStream_t s, double accept) {
  const bool plain = no_graph();
  if (!plain && !w.exec_pc) TB_TRY(build_graph_pc(op, w));
  const int nb = kUpdateBlocks;
  op.launch_dinv(w.dinv, s);
  k_pcg_start<<<nb, kBlock, 0, s>>>(w.n, b, nullptr, w.dinv, w.x, w.r, w.z, w.pa, w.st, w.partC(), 1, rtol, maxit);
  launched(1);
  TB_CHECK_LAUNCH();
  TB_TRY(op.precond_setup(s));
  int rc = TB_OK, stalls = 0, it_before = 0;
  double best_rr = -1.0;
  w.klaunches = 0;
  if (!w.kev0) {
    TB_CUDA(cudaEventCreate(&w.kev0));
    TB_CUDA(cudaEventCreate(&w.kev1));
  }
  for (int restart = 0;; ++restart) {
    if (w.klaunches == 0) TB_CUDA(cudaEventRecord(w.kev0, s));
    const bool persistent = !plain && op.launch_persistent_pc(w, s);
    if (persistent) {
      TB_CHECK_LAUNCH();
      TB_CUDA(cudaEventRecord(w.kev1, s));
      ++w.klaunches;
    } else {
    TB_TRY(op.precond_apply(w.r, w.z, s));
    k_pcg_rz<<<nb, kBlock, 0, s>>>(w.n, w.r, w.z, w.st, w.partC(), 1);
    launched(1);
    if (plain) {
      for (;;) {
        pc_body(op, w, s);
        TB_CHECK_LAUNCH();
        TB_CUDA(cudaMemcpyAsync(w.h_st, w.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
        TB_CUDA(cudaStreamSynchronize(s));
        if (w.h_st->done != 0) break;
      }
    } else {
      TB_CUDA(cudaGraphLaunch(w.exec_pc, s));
    }
    }
    op.launch_apply(w.x, w.tmp, s);
    k_pcg_start<<<nb, kBlock, 0, s>>>(w.n, b, w.tmp, w.dinv, w.x, w.r, w.z, w.pa, w.st, w.partC(), 0, rtol, maxit);
    launched(1);
    TB_CHECK_LAUNCH();
    TB_CUDA(cudaMemcpyAsync(w.h_st, w.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    TB_CUDA(cudaStreamSynchronize(s));
    TB_TRY(op.precond_check());
    const PcgState& h = *w.h_st;
    if (!persistent) launched((int64_t)(h.iters - it_before) * 40);  // approximate: kernels per V-cycle iteration
    it_before = h.iters;
    if (h.done == 1) break;
    if (h.done == 3) {
      set_error("preconditioned pCG breakdown after %d iterations", h.iters);
      rc = TB_ERR_INDEFINITE;
      break;
    }
    if (best_rr >= 0.0 && h.rr > 0.25 * best_rr) ++stalls;
    else stalls = 0;
    if (best_rr < 0.0 || h.rr < best_rr) best_rr = h.rr;
    if (stalls >= 3 && accept > 0.0 && h.rr <= accept * accept * h.bb) break;  // round-off mode: at the floor
    if (h.done == 2 || h.iters >= maxit || stalls >= 3 || restart >= 64) {
      set_error("preconditioned pCG did not reach rtol=%g in %d iterations (relative residual %.3e)", rtol, h.iters,
                sqrt(h.rr / (h.bb > 0 ? h.bb : 1.0)));
      rc = TB_ERR_NOT_CONVERGED;
      break;
    }
  }
  const PcgState& h = *w.h_st;
  if (iters) *iters = h.iters;
  if (relres) *relres = (h.bb > 0.0) ? sqrt(h.rr / h.bb) : 0.0;
  if (x_out != w.x) TB_CUDA(cudaMemcpyAsync(x_out, w.x, sizeof(double) * w.n, cudaMemcpyDeviceToDevice, s));
  return rc;
}

// rtol < 0 selects round-off mode (include/topo_b200.h): target |rtol|, and a solve whose true
// residual stagnates (restarts stop paying off) at or below max(100 |rtol|, 1e-7) counts as
// converged -- the attainable accuracy of Jacobi-pCG on an ill-conditioned SIMP design.
int pcg_solve(const PcgOp& op, PcgWork& w, const double* b, double* x_out, double rtol, int maxit, int* iters,
              double* relres, cudaStream_t s) {
  double accept = 0.0;
  if (rtol < 0.0) {
    rtol = -rtol;
    accept = fmax(100.0 * rtol, 1e-7);
  }
  if (!(rtol > 0.0) || maxit < 1) {
    set_error("pcg: rtol must be nonzero and maxit >= 1 (got %g, %d)", rtol, maxit);
    return TB_ERR_INVALID;
  }
  if (op.has_precond()) return pcg_solve_pc(op, w, b, x_out, rtol, maxit, iters, relres, s, accept);
  const bool plain = no_graph();
  const bool persistent = !plain && op.has_persistent();
  if (!plain && !persistent && !w.exec) TB_TRY(build_graph(op, w));
  const int nb = kUpdateBlocks;
  op.launch_dinv(w.dinv, s);
  k_pcg_start<<<nb, kBlock, 0, s>>>(w.n, b, nullptr, w.dinv, w.x, w.r, w.z, w.pa, w.st, w.partC(), 1, rtol, maxit);
  launched(1);
  TB_CHECK_LAUNCH();
  int rc = TB_OK;
  int iters_before = 0, stalls = 0;
  double best_rr = -1.0;
  for (int restart = 0;; ++restart) {
    if (plain) {
      TB_TRY(run_loop_plain(op, w, s));
    } else if (persistent) {
      op.launch_persistent(w, s);
      TB_CHECK_LAUNCH();
    } else {
      TB_CUDA(cudaGraphLaunch(w.exec, s));
    }
    // true residual check at exit
    op.launch_apply(w.x, w.tmp, s);
    k_pcg_start<<<nb, kBlock, 0, s>>>(w.n, b, w.tmp, w.dinv, w.x, w.r, w.z, w.pa, w.st, w.partC(), 0, rtol, maxit);
    launched(1);
    TB_CHECK_LAUNCH();
    TB_CUDA(cudaMemcpyAsync(w.h_st, w.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    TB_CUDA(cudaStreamSynchronize(s));
    const PcgState& h = *w.h_st;
    const int delta = h.iters - iters_before;
    iters_before = h.iters;
    if (persistent) launched(1);
    else launched((int64_t)(delta > 0 ? (delta + kIters - 1) / kIters : 1) * (2 * kIters + 1));
    if (h.done == 1) break;  // true residual within tolerance
    if (h.done == 3) {
      set_error("pCG breakdown after %d iterations: p^T K p <= 0 or non-finite; matrix is not positive definite",
                h.iters);
      rc = TB_ERR_INDEFINITE;
      break;
    }
    // the recursive residual met rtol but the true one did not: restart from the true residual,
    // unless restarts have stopped paying off (rtol below the attainable accuracy)
    if (best_rr >= 0.0 && h.rr > 0.25 * best_rr) ++stalls;
    else stalls = 0;
    if (best_rr < 0.0 || h.rr < best_rr) best_rr = h.rr;
    if (stalls >= 3 && accept > 0.0 && h.rr <= accept * accept * h.bb) break;  // round-off mode: at the floor
    if (h.done == 2 || h.iters >= maxit || stalls >= 3 || restart >= 64) {
      set_error("pCG did not reach rtol=%g in %d iterations (relative residual %.3e)", rtol, h.iters,
                sqrt(h.rr / (h.bb > 0 ? h.bb : 1.0)));
      rc = TB_ERR_NOT_CONVERGED;
      break;
    }
  }
  const PcgState& h = *w.h_st;
  if (iters) *iters = h.iters;
  if (relres) *relres = (h.bb > 0.0) ? sqrt(h.rr / h.bb) : 0.0;
  if (x_out != w.x) TB_CUDA(cudaMemcpyAsync(x_out, w.x, sizeof(double) * w.n, cudaMemcpyDeviceToDevice, s));
  return rc;
}

int pcg_profile(const PcgOp& op, PcgWork& w, const double* b, int nrep, double* ms_fused, double* ms_update,
                cudaStream_t s) {
  const int nb = kUpdateBlocks;
  op.launch_dinv(w.dinv, s);
  // rtol = 0 (tol2 = 0) and maxit = INT_MAX keep every iteration live
  k_pcg_start<<<nb, kBlock, 0, s>>>(w.n, b, nullptr, w.dinv, w.x, w.r, w.z, w.pa, w.st, w.partC(), 1, 0.0,
                                    0x7fffffff);
  launched(1);
  TB_CHECK_LAUNCH();
  cudaEvent_t ev[3];
  for (auto& e : ev) TB_CUDA(cudaEventCreate(&e));
  double tf = 0.0, tu = 0.0;
  for (int it = 0; it < nrep; ++it) {
    double* pold = (it & 1) ? w.pb : w.pa;
    double* pnew = (it & 1) ? w.pa : w.pb;
    cudaEventRecord(ev[0], s);
    op.launch_fused(w, pold, pnew, s);
    cudaEventRecord(ev[1], s);
    k_pcg_update<<<kUpdateBlocks, kBlock, 0, s>>>(w.n, pnew, w.q, w.dinv, w.x, w.r, w.z, w.st, w.partB());
    cudaEventRecord(ev[2], s);
    launched(2);
    TB_CUDA(cudaEventSynchronize(ev[2]));
    float a = 0.f, c = 0.f;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&c, ev[1], ev[2]);
    tf += a;
    tu += c;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  TB_CUDA(cudaMemcpy(w.h_st, w.st, sizeof(PcgState), cudaMemcpyDeviceToHost));
  if (w.h_st->done != 0) {
    set_error("profile run stopped early (state %d after %d iterations)", w.h_st->done, w.h_st->iters);
    return TB_ERR_INVALID;
  }
  *ms_fused = tf / nrep;
  *ms_update = tu / nrep;
  return TB_OK;
}

// ---- distributed (slab) mode: rank-local phases, scalars finished after host allreduce ----
__global__ void k_dist_init2(PcgState* st) {
  const double rtol = st->pq;
  st->rz = st->red[1];
  st->bb = st->red[2];
  st->rr = st->red[2];
  st->tol2 = rtol * rtol * st->red[2];
  st->beta = 0.0;
  st->done = (st->red[2] == 0.0) ? 1 : (isfinite(st->red[2]) ? 0 : 3);
}
__global__ void k_dist_alpha(PcgState* st) {
  if (st->done) return;
  const double v = st->red[0];
  if (!(v > 0.0) || !isfinite(v)) {
    st->done = 3;
  } else {
    st->pq = v;
    st->alpha = st->rz / v;
  }
}
__global__ void k_dist_beta(PcgState* st) {
  if (st->done) return;
  const int it = st->iters + 1;
  st->iters = it;
  st->beta = st->red[1] / st->rz;
  st->rz = st->red[1];
  st->rr = st->red[2];
  if (!isfinite(st->red[1]) || !isfinite(st->red[2])) st->done = 3;
  else if (st->red[2] <= st->tol2) st->done = 1;
  else if (it >= st->maxit) st->done = 2;
}

// Halo push fused into the kernels that produce z: a value of the first owned node plane goes
// to the lower neighbour's ghost-above plane, one of the last owned plane to the upper
// neighbour's ghost-below plane.  The destinations are peer memory (IPC-mapped over NVLink) or
// local buffers.  No flag or wait is needed: the push happens in phases 0 and 4, each followed
// on every rank by the allreduce of `red`, and a neighbour reads its ghost planes only in its
// next operator phase, after that allreduce (RAW).  It overwrites them again only after the
// allreduce that follows that operator phase (WAR).  Ghost planes of z are therefore written
// by the neighbour alone; the dist kernels never touch them.
struct HaloPush {
  int64_t own0, own1, plane;
  double *lo, *hi;
  __device__ __forceinline__ bool push(int64_t i, double zi) const {
    bool any = false;
    if (lo != nullptr && i < own0 + plane) {
      lo[i - own0] = zi;
      any = true;
    }
    if (hi != nullptr && i >= own1 - plane) {
      hi[i - (own1 - plane)] = zi;
      any = true;
    }
    return any;
  }
};

// phase 0: r = Z b, x = 0, p_old = 0 everywhere; z = D^-1 r on owned dofs (+ push); local r.z, r.r
__global__ void __launch_bounds__(kBlock) k_dist_start(int64_t n, HaloPush hp, const double* __restrict__ b,
                                                       const double* __restrict__ dinv, double* __restrict__ x,
                                                       double* __restrict__ r, double* __restrict__ z,
                                                       double* __restrict__ pa, PcgState* st, double* partials,
                                                       double rtol, int maxit) {
  double acc[2] = {0.0, 0.0};
  bool pushed = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double di = dinv[i];
    const double ri = (di != 0.0) ? b[i] : 0.0;
    x[i] = 0.0;
    r[i] = ri;
    pa[i] = 0.0;
    if (i >= hp.own0 && i < hp.own1) {
      const double zi = di * ri;
      z[i] = zi;
      pushed |= hp.push(i, zi);
      acc[0] = fma(ri, zi, acc[0]);
      acc[1] = fma(ri, ri, acc[1]);
    }
  }
  if (pushed) __threadfence_system();
  block_sum<2>(acc);
  if (publish_partials<2>(acc, partials, &st->count_c)) {
    gather_partials<2>(acc, partials, &st->count_c);
    if (threadIdx.x == 0) {
      st->red[1] = acc[0];
      st->red[2] = acc[1];
      st->iters = 0;
      st->maxit = maxit;
      st->beta = 0.0;
      st->alpha = 0.0;
      st->done = 0;
      st->pq = rtol;  // stashed until k_dist_init2 has the global norm
    }
  }
}

// phase 4: x += alpha p, r -= alpha q, z = D^-1 r over the owned dofs only (+ push); local r.z, r.r
__global__ void __launch_bounds__(kBlock) k_dist_update(HaloPush hp, const double* __restrict__ p,
                                                        const double* __restrict__ q, const double* __restrict__ dinv,
                                                        double* __restrict__ x, double* __restrict__ r,
                                                        double* __restrict__ z, PcgState* st, double* partials) {
  if (st->done) return;
  const double a = st->alpha;
  double acc[2] = {0.0, 0.0};
  bool pushed = false;
  // 16-byte accesses over the even-aligned interior [v0, v1) of the owned range; the (at most
  // two) odd end dofs go to the first two threads of block 0
  const int64_t v0 = (hp.own0 + 1) & ~int64_t(1), v1 = hp.own1 & ~int64_t(1);
  constexpr int U = 4;
  const int64_t n2 = v1 > v0 ? (v1 - v0) / 2 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double2* p2 = reinterpret_cast<const double2*>(p + v0);
  const double2* q2 = reinterpret_cast<const double2*>(q + v0);
  const double2* d2 = reinterpret_cast<const double2*>(dinv + v0);
  double2* x2 = reinterpret_cast<double2*>(x + v0);
  double2* r2 = reinterpret_cast<double2*>(r + v0);
  double2* z2 = reinterpret_cast<double2*>(z + v0);
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 pv[U], qv[U], dv[U], xv[U], rv[U], zv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + u * stride;
      pv[u] = __ldcs(p2 + j);
      qv[u] = __ldcs(q2 + j);
      dv[u] = __ldg(d2 + j);
      xv[u] = x2[j];
      rv[u] = r2[j];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      upd2(a, pv[u], qv[u], dv[u], xv[u], rv[u], zv[u], acc);
      const int64_t j = i + u * stride;
      x2[j] = xv[u];
      r2[j] = rv[u];
      z2[j] = zv[u];
      pushed |= hp.push(v0 + 2 * j, zv[u].x);
      pushed |= hp.push(v0 + 2 * j + 1, zv[u].y);
    }
  }
  for (; i < n2; i += stride) {
    double2 pv = p2[i], qv = q2[i], dv = d2[i], xv = x2[i], rv = r2[i], zv;
    upd2(a, pv, qv, dv, xv, rv, zv, acc);
    x2[i] = xv;
    r2[i] = rv;
    z2[i] = zv;
    pushed |= hp.push(v0 + 2 * i, zv.x);
    pushed |= hp.push(v0 + 2 * i + 1, zv.y);
  }
  if (blockIdx.x == 0 && threadIdx.x < 2) {  // odd end dofs
    const int64_t k = threadIdx.x == 0 ? hp.own0 : v1;
    const bool live = threadIdx.x == 0 ? (hp.own0 & 1) != 0 && hp.own0 < hp.own1 : v1 < hp.own1 && v1 >= v0;
    if (live) {
      double zv = 0.0;
      const double di = dinv[k];
      if (di != 0.0) {
        x[k] = fma(a, p[k], x[k]);
        const double ri = fma(-a, q[k], r[k]);
        r[k] = ri;
        zv = di * ri;
        acc[0] = fma(ri, zv, acc[0]);
        acc[1] = fma(ri, ri, acc[1]);
      }
      z[k] = zv;
      pushed |= hp.push(k, zv);
    }
  }
  if (pushed) __threadfence_system();
  block_sum<2>(acc);
  if (publish_partials<2>(acc, partials, &st->count_b)) {
    gather_partials<2>(acc, partials, &st->count_b);
    if (threadIdx.x == 0) {
      st->red[1] = acc[0];
      st->red[2] = acc[1];
    }
  }
}

// ---- distributed single-reduction pCG (Chronopoulos-Gear; phases 10-13) ----------------
// Vectors: u = D^-1 r lives in w.z (so the halo machinery of z -- copies or IPC peer pushes --
// carries it unchanged), w = K u in w.q, p in w.pa, s in w.tmp, scratch w.pb.  One iteration:
//   13 update (p, s, x, r, u on owned dofs; local g = r.u, r.r; push u) -> halo -> 11 operator
//   (w = K u, local d = w.u) -> ONE allreduce of (d, g, r.r) -> 12 scalars (alpha, beta, done).
// phase 10: r = Z b, x = p = s = 0, u = D^-1 r on owned dofs (+ push); local g, r.r
__global__ void __launch_bounds__(kBlock) k_dist_cg_start(int64_t n, HaloPush hp, const double* __restrict__ b,
                                                          const double* __restrict__ dinv, double* __restrict__ x,
                                                          double* __restrict__ r, double* __restrict__ u,
                                                          double* __restrict__ p, double* __restrict__ sv,
                                                          double* __restrict__ scratch, PcgState* st,
                                                          double* partials, double rtol, int maxit) {
  double acc[2] = {0.0, 0.0};
  bool pushed = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double di = dinv[i];
    const double ri = (di != 0.0) ? b[i] : 0.0;
    x[i] = 0.0;
    r[i] = ri;
    p[i] = 0.0;
    sv[i] = 0.0;
    scratch[i] = 0.0;
    if (i >= hp.own0 && i < hp.own1) {
      const double ui = di * ri;
      u[i] = ui;
      pushed |= hp.push(i, ui);
      acc[0] = fma(ri, ui, acc[0]);
      acc[1] = fma(ri, ri, acc[1]);
    }
  }
  if (pushed) __threadfence_system();
  block_sum<2>(acc);
  if (publish_partials<2>(acc, partials, &st->count_c)) {
    gather_partials<2>(acc, partials, &st->count_c);
    if (threadIdx.x == 0) {
      st->red[1] = acc[0];
      st->red[2] = acc[1];
      st->iters = 0;
      st->maxit = maxit;
      st->beta = 0.0;  // the fused operator forms p = u + 0 p_old: it applies K to u
      st->alpha = 0.0;
      st->cg_beta = 0.0;
      st->cg_init = 1;
      st->done = 0;
      st->pq = rtol;  // stashed until phase 12 has the global ||Z b||
    }
  }
}

// phase 12 (one thread, after the host allreduce of red = (d, g, r.r))
__global__ void k_dist_cg_scalars(PcgState* st) {
  if (st->done) return;
  const double del = st->red[0], gam = st->red[1], rr = st->red[2];
  st->rr = rr;
  if (!isfinite(del) || !isfinite(gam) || !isfinite(rr)) {
    st->done = 3;
  } else if (st->cg_init) {
    st->cg_init = 0;
    st->bb = rr;
    st->tol2 = st->pq * st->pq * rr;  // rtol stashed by phase 10
    if (rr == 0.0 || gam == 0.0) {
      st->done = 1;
    } else if (!(del > 0.0)) {
      st->done = 3;
    } else {
      st->alpha = gam / del;
      st->cg_beta = 0.0;
      st->rz = gam;
    }
  } else {
    const int it = st->iters + 1;
    st->iters = it;
    if (rr <= st->tol2) {
      st->done = 1;
    } else {
      const double beta = gam / st->rz;
      const double den = del - beta * gam / st->alpha;
      if (!(den > 0.0)) {
        st->done = 3;
      } else {
        st->cg_beta = beta;
        st->alpha = gam / den;
        st->rz = gam;
        if (it >= st->maxit) st->done = 2;
      }
    }
  }
}

// phase 13: p = u + b p ; s = w + b s ; x += a p ; r -= a s ; u = D^-1 r (owned, free dofs; + push)
__global__ void __launch_bounds__(kBlock) k_dist_cg_update(HaloPush hp, const double* __restrict__ dinv,
                                                           const double* __restrict__ w, double* __restrict__ u,
                                                           double* __restrict__ p, double* __restrict__ sv,
                                                           double* __restrict__ x, double* __restrict__ r,
                                                           PcgState* st, double* partials) {
  if (st->done) return;
  const double a = st->alpha, bt = st->cg_beta;
  double acc[2] = {0.0, 0.0};
  bool pushed = false;
  for (int64_t i = hp.own0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hp.own1;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double di = dinv[i];
    double un = 0.0;
    if (di != 0.0) {
      const double pi = fma(bt, p[i], u[i]);
      const double si = fma(bt, sv[i], w[i]);
      p[i] = pi;
      sv[i] = si;
      x[i] = fma(a, pi, x[i]);
      const double ri = fma(-a, si, r[i]);
      r[i] = ri;
      un = di * ri;
      acc[0] = fma(ri, un, acc[0]);
      acc[1] = fma(ri, ri, acc[1]);
    }
    u[i] = un;
    pushed |= hp.push(i, un);
  }
  if (pushed) __threadfence_system();
  block_sum<2>(acc);
  if (publish_partials<2>(acc, partials, &st->count_b)) {
    gather_partials<2>(acc, partials, &st->count_b);
    if (threadIdx.x == 0) {
      st->red[1] = acc[0];
      st->red[2] = acc[1];
    }
  }
}

int pcg_dist_phase(const PcgOp& op, PcgWork& w, int phase, const double* b, double rtol, int maxit, int parity,
                   cudaStream_t s) {
  const int nb = kUpdateBlocks;
  double* pold = (parity & 1) ? w.pb : w.pa;
  double* pnew = (parity & 1) ? w.pa : w.pb;
  const int64_t o1 = (w.own1 < 0 || w.own1 > w.n) ? w.n : w.own1;
  const int64_t pl = (w.plane > 0 && w.plane <= o1 - w.own0) ? w.plane : o1 - w.own0;
  const HaloPush hp{w.own0, o1, pl, w.halo_lo, w.halo_hi};
  switch (phase) {
    case 0:  // init: D^-1, r = Z b, z, local r.z and r.r
      op.launch_dinv(w.dinv, s);
      k_dist_start<<<nb, kBlock, 0, s>>>(w.n, hp, b, w.dinv, w.x, w.r, w.z, w.pa, w.st, w.partC(), rtol, maxit);
      launched(1);
      break;
    case 1:
      k_dist_init2<<<1, 1, 0, s>>>(w.st);
      launched(1);
      break;
    case 2:  // operator + local p.q
      op.launch_fused(w, pold, pnew, s);
      launched(1);
      break;
    case 3:
      k_dist_alpha<<<1, 1, 0, s>>>(w.st);
      launched(1);
      break;
    case 4:  // update + local r.z, r.r (+ halo push)
      k_dist_update<<<kUpdateBlocks, kBlock, 0, s>>>(hp, pnew, w.q, w.dinv, w.x, w.r, w.z, w.st, w.partB());
      launched(1);
      break;
    case 5:
      k_dist_beta<<<1, 1, 0, s>>>(w.st);
      launched(1);
      break;
    case 10:  // single reduction: init (D^-1, r = Z b, u = D^-1 r, local g and r.r)
      op.launch_dinv(w.dinv, s);
      k_dist_cg_start<<<nb, kBlock, 0, s>>>(w.n, hp, b, w.dinv, w.x, w.r, w.z, w.pa, w.tmp, w.pb, w.st, w.partC(),
                                            rtol, maxit);
      launched(2);
      break;
    case 11:  // w = K u (fused operator with beta = 0: p = u, q = K u) + local d = u.w
      op.launch_fused(w, w.pb, w.pb, s);
      launched(1);
      break;
    case 12:
      k_dist_cg_scalars<<<1, 1, 0, s>>>(w.st);
      launched(1);
      break;
    case 13:  // update + local g, r.r (+ halo push of u)
      k_dist_cg_update<<<kUpdateBlocks, kBlock, 0, s>>>(hp, w.dinv, w.q, w.z, w.pa, w.tmp, w.x, w.r, w.st, w.partB());
      launched(1);
      break;
    default:
      set_error("unknown distributed pCG phase %d", phase);
      return TB_ERR_INVALID;
  }
  TB_CHECK_LAUNCH();
  return TB_OK;
}

}  // namespace tb
