// Jacobi-preconditioned CG engine, device-resident.
//
// One iteration = two kernels:
//   A (operator-specific, fused):  p = z + beta p_old ; q = K p ; pq  -> alpha
//   B (generic, per dof):          x += alpha p ; r -= alpha q ; z = D^-1 r ; rz, rr -> beta, done
// The loop runs inside ONE CUDA graph whose body (kIters iterations + a condition kernel)
// sits under a conditional WHILE node, so a whole solve is a single graph launch with no
// host round trip; convergence is re-checked on the TRUE residual at exit
// (reference SpdFactorization.solve, fem.py:324-333, is a direct solve; the survey's
// Appendix A requires the true residual <= rtol).
#pragma once

#include "common.cuh"

namespace tb {

struct PcgWork;

struct PcgOp {
  virtual ~PcgOp() = default;
  virtual int64_t size() const = 0;     // vector length (dofs)
  virtual int fused_blocks() const = 0; // grid of kernel A
  // kernel A on stream s
  virtual void launch_fused(const PcgWork& w, const double* pold, double* pnew, cudaStream_t s) const = 0;
  // y = Z K v (fixed rows zeroed)
  virtual void launch_apply(const double* v, double* y, cudaStream_t s) const = 0;
  // Jacobi inverse diagonal (0 on fixed dofs)
  virtual void launch_dinv(double* dinv, cudaStream_t s) const = 0;
  // Whole iteration loop in one persistent cooperative launch (operators without a persistent
  // variant use the conditional-graph loop).
  virtual bool has_persistent() const { return false; }
  // optional preconditioner replacing Jacobi (multigrid): set-up per operator, z = M^-1 r
  virtual bool has_precond() const { return false; }
  virtual int precond_setup(cudaStream_t s) const { (void)s; return TB_OK; }
  virtual int precond_apply(const double* r, double* z, cudaStream_t s) const { (void)r; (void)z; (void)s; return TB_OK; }
  // deferred set-up checks, called after a stream synchronisation
  virtual int precond_check() const { return TB_OK; }
  virtual void launch_persistent(const PcgWork& w, cudaStream_t s) const { (void)w; (void)s; }
  // preconditioned loop (from r, pa = 0) in one persistent launch; false: use the graph loop
  virtual bool launch_persistent_pc(PcgWork& w, cudaStream_t s) const { (void)w; (void)s; return false; }
};

struct PcgWork {
  int64_t n = 0;
  double *x = nullptr, *r = nullptr, *z = nullptr, *pa = nullptr, *pb = nullptr, *q = nullptr,
         *dinv = nullptr, *tmp = nullptr, *part = nullptr;
  int part_stride = 0;  // doubles per partial region
  PcgState* st = nullptr;
  PcgState* h_st = nullptr;  // pinned
  void* barrier = nullptr;   // grid-barrier word of the persistent kernel
  double* pub = nullptr;     // persistent kernel's published vectors [2][3][n]
  cudaGraphExec_t exec = nullptr;
  cudaGraphExec_t exec_pc = nullptr;  // graph of the preconditioned (multigrid) loop
  // span of the persistent preconditioned launches of the last solve (tb_pcg_kernel_time)
  cudaEvent_t kev0 = nullptr, kev1 = nullptr;
  int klaunches = 0;
  // distributed (slab) mode: owned dof range [own0, own1) (own1 < 0: n), dofs per node plane,
  // and where the first / last owned plane of z is pushed (neighbours' ghost planes, possibly
  // peer memory over NVLink; nullptr: the caller exchanges the halo)
  int64_t own0 = 0, own1 = -1, plane = 0;
  double *halo_lo = nullptr, *halo_hi = nullptr;
  double* partA() const { return part; }
  double* partB() const { return part + 2 * part_stride; }
  double* partC() const { return part + 4 * part_stride; }
  int alloc(int64_t n_, int max_blocks, bool with_pub = false, int64_t cap = 0);  // cap: vector capacity >= n_
  int set_fields(int dist, int dot_k0, int dot_k1);  // distributed mode + owned node planes
  void release();
};

constexpr int kIters = 8;  // pCG iterations per while-loop body
constexpr int kUpdateBlocks = 148 * 4;

int pcg_solve(const PcgOp& op, PcgWork& w, const double* b, double* x_out, double rtol, int maxit,
              int* iters, double* relres, cudaStream_t stream);
// one phase of the distributed (slab) pCG: 0 init, 1 finish init, 2 operator, 3 alpha, 4 update, 5 beta
int pcg_dist_phase(const PcgOp& op, PcgWork& w, int phase, const double* b, double rtol, int maxit, int parity,
                   cudaStream_t stream);
int pcg_profile(const PcgOp& op, PcgWork& w, const double* b, int nrep, double* ms_fused, double* ms_update,
                cudaStream_t stream);

}  // namespace tb
