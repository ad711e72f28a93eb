/*
 * topo_b200.h — C ABI of the B200-native FE-evaluation hot path of the
 * reference `romtopt` package (arXiv 2004.05756), built for sm_100a.
 *
 * Plain C: opaque handles, plain pointers and sizes, `int` status codes, a
 * thread-local message from tb_last_error().  No torch types.  All array
 * arguments of compute calls are DEVICE pointers on the plan's device,
 * caller-owned, fp64 unless stated; `stream` is a cudaStream_t passed as
 * void* (0 = legacy default stream).  Plans are not safe for concurrent calls
 * from several threads; distinct plans are independent.
 *
 * Layout (reference fem.py:154-229, extended to Hex8):
 *   node id   n = (k*(ny+1) + j)*(nx+1) + i     (k = 0 in 2D)
 *   element   e = (k*ny + j)*nx + i
 *   dof       d*n + c  (interleaved components, d = 2 or 3)
 *   element nodes: CCW from the bottom-left corner (2D, fem.py:225);
 *                  3D: bottom face (z=k) CCW, then top face (z=k+1) CCW.
 *
 * Each entry point names the reference interface it replaces (file:line in
 * /root/reference/pkg/src/romtopt).
 */
#ifndef TOPO_B200_H
#define TOPO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define TB_OK 0
#define TB_ERR_INVALID 1        /* bad argument  -> Python ValueError                      */
#define TB_ERR_CUDA 2           /* CUDA runtime failure                                    */
#define TB_ERR_INDEFINITE 3     /* pCG breakdown p^T K p <= 0 / non-finite -> IndefiniteMatrixError (fem.py:33-38) */
#define TB_ERR_NOT_CONVERGED 4  /* maxit reached before rtol                               */
#define TB_ERR_DEGENERATE 5     /* reduced stiffness not SPD -> DegenerateBasisError (rom.py:49-50) */
#define TB_ERR_DENSITY 6        /* density outside [rho_l, 1] -> ValueError (hdm.py:156-162) */
#define TB_ERR_RUNTIME 7        /* numerical failure the reference raises RuntimeError for (mma.py:158) */

typedef struct tb_plan tb_plan;
typedef struct tb_filter tb_filter;

int tb_version(void);
const char* tb_last_error(void);

/* ---- plan: one structured mesh + unit element stiffness + SIMP law + Dirichlet set ----
 * Replaces HdmSolver.__init__ (hdm.py:120-142) and PatternAssembler (fem.py:357-396):
 * no matrix is assembled; the operator is applied matrix-free.
 *   dim       2 (Q4) or 3 (Hex8); nz ignored for dim 2
 *   k_e       HOST pointer, (8x8) or (24x24) row-major unit-density element stiffness
 *   rho_l, p  MaterialModel (hdm.py:40-55)
 *   fixed     HOST pointer, n_dofs bytes, nonzero = Dirichlet dof (hdm.py:139-141)      */
int tb_plan_create(int dim, int nx, int ny, int nz, double h, const double* k_e,
                   double rho_l, double p, const uint8_t* fixed, int device, tb_plan** out);
int tb_plan_destroy(tb_plan* plan);
int tb_plan_sizes(const tb_plan* plan, int64_t* n_elems, int64_t* n_nodes, int64_t* n_dofs);

/* alpha(rho) and alpha'(rho) per element (hdm.py:40-55). */
int tb_material(tb_plan* plan, const double* rho, double* alpha, double* dalpha, void* stream);

/* Clamp a raw filtered density into [rho_l, 1] and return the largest adjustment
 * (hdm.py:144-154); *clamp_width is a HOST pointer (synchronises the stream). */
int tb_clamp_density(tb_plan* plan, const double* rho_raw, double* rho, double* clamp_width,
                     void* stream);

/* y = Z K(rho) v (fixed ROWS zeroed when mask_rows != 0): HdmSolver.apply_stiffness
 * (hdm.py:224-233).  mask_rows = 0 gives the unmasked K(rho) v of rom.py:309-317. */
int tb_apply_stiffness(tb_plan* plan, const double* rho, const double* v, double* y,
                       int mask_rows, void* stream);

/* s_e = drho_e - alpha'(rho_e) u_e^T K_e lam_e: HdmSolver.element_sensitivity
 * (hdm.py:211-222).  drho may be NULL (compliance: dj/drho = 0, hdm.py:95-96). */
int tb_element_sensitivity(tb_plan* plan, const double* rho, const double* u, const double* lam,
                           const double* drho, double* s, void* stream);

/* Jacobi-preconditioned CG on Z K(rho) Z x = Z b (replaces PatternAssembler.factorize +
 * SpdFactorization.solve, fem.py:283-333, 406-409; fixed dofs of x stay 0).  Stops when the
 * TRUE residual ||Z(b - K x)|| <= rtol ||Z b||.  x is output only (x0 = 0).
 * *iters, *relres are HOST pointers (may be NULL).  Returns TB_ERR_INDEFINITE on breakdown,
 * TB_ERR_NOT_CONVERGED at maxit (x holds the last iterate).  rtol < 0 selects round-off mode:
 * target |rtol|, and a true residual that stagnates at <= max(100 |rtol|, 1e-7) is accepted (the
 * reference solves directly; this is "as exact as the arithmetic allows").  The same convention holds for
 * tb_filter_apply / tb_filter_adjoint. */
int tb_pcg_solve(tb_plan* plan, const double* rho, const double* b, double* x, double rtol,
                 int maxit, int* iters, double* relres, void* stream);

/* Preconditioner of tb_pcg_solve: 0 Jacobi (default), 1 geometric multigrid (Galerkin element
 * aggregation, damped-Jacobi V-cycle, dense coarsest solve; needs even element counts down to a
 * coarsest level of <= 6144 dofs, else TB_ERR_INVALID). */
int tb_plan_set_preconditioner(tb_plan* plan, int kind);

/* Diagnostics: time the pCG kernels in situ.  Starts a solve of K(rho) x = b and runs
 * nrep iterations with a CUDA event pair around every kernel on `stream`; returns the mean
 * duration (ms) of the fused operator kernel and of the update kernel (HOST pointers).  On the
 * single-sweep path (tb_pcg_path == 1) ms_fused is the whole iteration and ms_update is 0. */
int tb_pcg_profile(tb_plan* plan, const double* rho, const double* b, int nrep, double* ms_fused,
                   double* ms_update, void* stream);
/* Diagnostics: device time (CUDA events on the solve's stream) spanned by the persistent
 * multigrid-pCG launches of the plan's last tb_pcg_solve (2D, preconditioner 1), and how many
 * there were (restarts after a true-residual check add one each); 0 launches when the solve ran
 * the graph path.  Synchronises on the last launch. */
int tb_pcg_kernel_time(tb_plan* plan, float* ms, int* launches);
/* Diagnostics: in-situ iteration timing of the single-sweep path (tb_pcg_path == 1).  reset != 0
 * starts (or restarts) accumulating: every later tb_pcg_solve brackets its iteration-graph
 * launches with CUDA events on the solve's stream.  Returns the accumulated device time (ms)
 * and the number of sweeps it covered (HOST pointers), i.e. the mean sweep duration of real
 * solves.  Replaces nothing in the reference (diagnostic). */
int tb_pcg_iter_time(tb_plan* plan, int reset, double* ms, int64_t* iters);
/* Which Jacobi-pCG iteration tb_pcg_solve runs for this plan: 1 = the 3D single-sweep
 * Chronopoulos-Gear kernel (Hex8, TMA-staged, one reduction per iteration), 0 = the two-kernel
 * iteration (2D / multigrid / distributed), -1 = null plan.  Replaces nothing in the reference
 * (diagnostic; the reference solve is fem.py:270-349). */
int tb_pcg_path(tb_plan* plan);
/* Diagnostics: 1 when tb_rom_reduced_stiffness(plan, ., k, ., nd, ...) runs the fused
 * element-form kernel (Hex8 plans, even k <= 64: S_e = C_e^T C_e on FP64 tensor cores, weighted
 * into all nd designs in one pass over Phi), with the tensor flops it executes in *flops; 0
 * otherwise.  The reference computes the same sum in rom.py:254-262. */
int tb_rom_fused_info(tb_plan* plan, int k, int nd, double* flops);
/* Diagnostics: per-phase %globaltimer sums (ns) of the persistent 2D multigrid pCG kernel in a
 * build with -DTB_MGP_PROF (tools/build_prof.sh); zeros in the product build.  Reads and clears
 * 32 counters into a HOST array. */
int tb_mgp_prof_read(unsigned long long* out32);
/* Number of kernels this library has launched so far (graph-body kernels included). */
int64_t tb_launch_count(void);

/* ---- slab-distributed pCG: the plan covers one z-slab; ghost node planes are
 * Dirichlet-masked in `fixed`.  Reductions, the operator's p.q and the rows contracted by
 * tb_rom_reduced_stiffness run over the owned node planes [k0, k1) only. */
int tb_plan_set_owned_planes(tb_plan* plan, int k0, int k1);
/* One phase of a distributed Jacobi-pCG iteration on this rank.  Phases: 0 init (needs rho, b,
 * rtol, maxit; publishes local r.z, r.r), 1 finish init (after the host allreduce), 2 operator
 * (publishes local p.q; `parity` = iteration index), 3 alpha (after allreduce), 4 update
 * (publishes local r.z, r.r), 5 beta/convergence (after allreduce).  Between phases the caller
 * allreduces the 4-double `red` buffer and, after phase 4, refreshes the ghost planes of z.
 * Single-reduction form (Chronopoulos-Gear, Hex8 plans): 10 init (needs rho, b, rtol, maxit;
 * u = D^-1 r in the z buffer, publishes local r.u, r.r), 13 update (p, s, x, r, u; publishes
 * local r.u, r.r), 11 operator (w = K u; publishes local w.u), 12 scalars (after the allreduce).
 * Iteration: 13 -> z halo -> 11 -> ONE allreduce of red[0..2] -> 12; start: 10 -> halo -> 11 ->
 * allreduce -> 12.  Replaces the two per-iteration reductions of phases 2-5. */
int tb_pcg_dist_phase(tb_plan* plan, int phase, const double* rho, const double* b, double rtol,
                      int maxit, int parity, void* stream);
/* Device pointers of this rank's solution x, preconditioned residual z and reduction buffer. */
int tb_pcg_dist_buffers(tb_plan* plan, double** x, double** z, double** red);
/* Host read of the iteration state (synchronises the stream). */
int tb_pcg_dist_state(tb_plan* plan, int* iters, int* done, double* rr, double* bb, void* stream);
/* Fused halo exchange: phases 0 and 4 store this rank's first owned plane of z to `lo_dst` (the
 * lower neighbour's ghost-above plane) and its last owned plane to `hi_dst` (the upper
 * neighbour's ghost-below plane), 3(nx+1)(ny+1) doubles each, while they compute z.  The
 * pointers are usually a neighbour's memory mapped with tb_ipc_open (NVLink peer stores); NULL
 * leaves that side to the caller's halo exchange.  The allreduce that follows phases 0 and 4 on
 * every rank orders the stores against the neighbour's reads, so no other synchronisation is
 * needed.  Requires tb_plan_set_owned_planes. */
int tb_plan_set_halo_peers(tb_plan* plan, double* lo_dst, double* hi_dst);
/* CUDA IPC of a device allocation (e.g. tb_pcg_dist_buffers' z) between the ranks' processes:
 * `handle` is 64 bytes (cudaIpcMemHandle_t); tb_ipc_open maps a peer's allocation on `device`. */
int tb_ipc_get_handle(const void* dptr, void* handle);
int tb_ipc_open(const void* handle, int device, void** dptr);
int tb_ipc_close(void* dptr);

/* Deterministic fp64 dot product of two device vectors; *out is a HOST pointer. */
int tb_dot(tb_plan* plan, const double* a, const double* b, int64_t n, double* out, void* stream);

/* ---- Helmholtz PDE density filter (filtering.py:47-114); HelmholtzFilter.__init__(mesh, R) ----
 * radius R -> PDE length r = R/(2 sqrt 3) (filtering.py:29-32,59); pure Neumann;
 * solved matrix-free by Jacobi-PCG to rtol (relative to the load vector norm). */
int tb_filter_create(int dim, int nx, int ny, int nz, double h, double radius, int device,
                     tb_filter** out);
int tb_filter_destroy(tb_filter* filt);
/* b(psi) = (h^d/2^d) sum_{e∋n} psi_e  (filtering.py:73-76) */
int tb_filter_load_vector(tb_filter* filt, const double* psi, double* b, void* stream);
/* phi = H^-1 b(psi); rho_e = mean of phi over the element nodes (filtering.py:78-97);
 * phi may be NULL.  *iters HOST (may be NULL).  A whole-grid filter solves H phi = b DIRECTLY in
 * the tensor-product cosine basis of the uniform grid (csrc/spectral.cu: the solution to round-off,
 * as the reference's sparse direct solve; rtol is not used and *iters = 0); the pCG path with the
 * rtol convention of tb_pcg_solve remains for slab phases and under TB_FILTER_PCG=1. */
int tb_filter_apply(tb_filter* filt, const double* psi, double* phi, double* rho, double rtol,
                    int* iters, void* stream);
/* w = (h^d/2^d) Q^T H^-1 Q (v/2^d): exact transpose of psi->rho (filtering.py:99-114) */
int tb_filter_adjoint(tb_filter* filt, const double* v, double* w, double rtol, int* iters,
                      void* stream);

/* ---- slab-distributed filter (BASELINE cfg 4): the filter covers one z-slab's
 * local grid (owned node planes plus one ghost plane per interior side), as tb_plan_* do for
 * the elasticity solve.  Ghost node planes are masked (never updated); reductions run over the
 * owned planes [k0, k1).  Phases, `red` and the halo contract are those of tb_pcg_dist_phase
 * (phase 0 takes the load vector b instead of rho).  Replaces, per rank, the factor-once /
 * solve pair of HelmholtzFilter (filtering.py:54-71, 78-97, 99-114). */
int tb_filter_set_owned_planes(tb_filter* filt, int k0, int k1);
int tb_filter_dist_phase(tb_filter* filt, int phase, const double* b, double rtol, int maxit,
                         int parity, void* stream);
int tb_filter_dist_buffers(tb_filter* filt, double** x, double** z, double** red);
int tb_filter_dist_state(tb_filter* filt, int* iters, int* done, double* rr, double* bb,
                         void* stream);
int tb_filter_set_halo_peers(tb_filter* filt, double* lo_dst, double* hi_dst);
/* Grid transfers of the filter (filtering.py:73-76, 95-97, 106-114): mode 0 element -> node,
 * out_n = scale * sum_{e∋n} in_e; mode 1 node -> element, out_e = scale * sum_{n∈e} in_n
 * (same summation order as tb_filter_apply / tb_filter_adjoint). */
int tb_filter_transfer(tb_filter* filt, int mode, const double* in, double scale, double* out,
                       void* stream);

/* ---- reduced-order model (rom.py:182-390); phi is (n_dofs x k) ROW-major ---- */
/* out[k*d + j] = sum_i phi[i*k + j] * vec[d*n + i] for nvec stacked vectors of length n (16 per pass over Phi)
 * (Phi^T f, rom.py:251, 289; also Q^T S of the POD) */
int tb_rom_project(int64_t n, const double* phi, int k, const double* vec, int nvec, double* out,
                   void* stream);
/* khat[d] = Phi^T K(rho_d) Phi (k x k, row-major) for nd designs stacked in rho (nd x n_elems):
 * RomModel.reduced_stiffness (rom.py:254-262), node-form contraction on FP64 tensor cores. */
int tb_rom_reduced_stiffness(tb_plan* plan, const double* phi, int k, const double* rho, int nd,
                             double* khat, void* stream);
/* out (k x k, row-major) = A^T B for column-major A, B (k columns, leading dimension ld, rows
 * [0, n)): the DMMA contraction of tb_rom_reduced_stiffness on its own (also a Gram matrix).
 * symmetric != 0: the caller guarantees A^T B is symmetric (Phi^T K Phi, a Gram matrix); only
 * the upper 8x8 tiles are computed and mirrored, as tb_rom_reduced_stiffness does. */
int tb_rom_gram_colmajor(int64_t n, int k, const double* A, const double* B, int64_t ld, int symmetric,
                         double* out, void* stream);
/* Batched Cholesky solve khat[d] X = rhs[d] (nrhs right-hand sides per design, row-major
 * nd x nrhs x k) for rom.py:280-291.  status is a HOST int array of nd entries: 0 ok,
 * 1 = not SPD (cho_factor LinAlgError -> DegenerateBasisError). */
int tb_rom_cholesky_solve(int k, int nd, int nrhs, const double* khat, const double* rhs,
                          double* x, int* status, void* stream);
/* u[d] = Phi uhat[d] (length n) for nd coefficient vectors (16 per pass over Phi; rom.py:285) */
int tb_rom_reconstruct(int64_t n, const double* phi, int k, const double* uhat, int nd, double* u,
                       void* stream);
/* norms[d] = || Z (K(rho_d) Phi uhat_d - g_d) ||_2 (rom.py:309-335); g is (nd x n_dofs) or a
 * single shared vector when g_stride == 0.  norms is a HOST array of nd doubles. */
int tb_rom_residual_norms(tb_plan* plan, const double* phi, int k, const double* rho,
                          const double* uhat, int nd, const double* g, int64_t g_stride,
                          double* norms, void* stream);

/* Gram-Schmidt with one re-orthogonalisation pass and relative drop tolerance (rom.py:76-97):
 * block classical GS in panels of 8 (Q^T W on DMMA), decisions on the device, one host sync.  vectors: m COLUMN vectors of length n (column-major n x m, device);
 * q: output (n x kept) ROW-major, compact (buffer of n*m doubles). *kept HOST.
 * Returns TB_ERR_INVALID when no vector survives ("no independent vectors supplied"). */
int tb_gram_schmidt(int64_t n, int m, const double* vectors, double drop_tol, double* q,
                    int* kept, void* stream);

/* ---- Cone ("linear hat") density filter (the reference has only the
 * Helmholtz filter, filtering.py): rho_e = sum_j w(e,j) psi_j / sum_j w(e,j) with
 * w(e,j) = max(0, R - |c_e - c_j|) over the element grid, and its exact transpose. ---- */
typedef struct tb_cone tb_cone;
int tb_cone_create(int dim, int nx, int ny, int nz, double h, double radius, int device, tb_cone** out);
int tb_cone_destroy(tb_cone* filt);
/* rho = cone(psi); psi, rho: n_elems device doubles */
int tb_cone_apply(tb_cone* filt, const double* psi, double* rho, void* stream);
/* w = cone^T v (exact transpose of tb_cone_apply) */
int tb_cone_adjoint(tb_cone* filt, const double* v, double* w, void* stream);

/* ---- Method of Moving Asymptotes (the trust-region subproblem engine) ---- */
/* MmaConfig (mma.py:25-38), same fields and defaults on the Python side. */
typedef struct tb_mma_config {
  double asy_init, asy_incr, asy_decr, asy_min_frac, asy_max_frac;
  double move, albefa, raa0, bisect_rtol;
  int bisect_max_iter;
} tb_mma_config;
/* Device workspace for tb_mma_step on n variables; zero it once before the first step. */
size_t tb_mma_workspace_bytes(int64_t n);
/* One MmaOptimizer.step (mma.py:91-175) on device arrays of n doubles: x_new from x and grad
 * under box [lower, upper] and w . x <= volume_cap; move_cap < 0 means none.  it = step count
 * after increment; has_xold1/has_xold2 say whether the asymptote history exists.  On success
 * the state (xold1, xold2, low, upp) advances as in mma.py:172-175; on TB_ERR_INVALID ("gradient
 * must be finite", "iterate outside box bounds", "iterate violates the volume constraint") it is
 * untouched.  TB_ERR_RUNTIME: "volume multiplier bracket failed".  Synchronises the stream. */
int tb_mma_step(int64_t n, const double* x, const double* grad, const double* lower, const double* upper,
                const double* w, double volume_cap, double move_cap, int it, int has_xold1, int has_xold2,
                const tb_mma_config* cfg, double* xold1, double* xold2, double* low, double* upp,
                void* workspace, double* x_new, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TOPO_B200_H */
