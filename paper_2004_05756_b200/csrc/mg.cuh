// Geometric multigrid preconditioner for the SIMP elasticity operator.
//
// Hierarchy: vertex-centred coarsening by 2 in every direction (an odd element count leaves a
// last coarse element spanning one fine element) until the level has few enough dofs.  Coarse operators are exact Galerkin products, built element by element: a coarse
// element E covers 2^d fine elements e, and with the (tri)linear interpolation R_e from E's
// corners to e's corners,
//     K_E = sum_{e in E} R_e^T (Z_e K_e Z_e) R_e ,  then rows/cols of fixed coarse dofs zeroed,
// where Z masks Dirichlet dofs and K_e = alpha_e K_unit on the finest level.  The interpolation
// is element-local inside a coarse element, so sum_E P_E K_E P_E^T equals P^T Z A Z P exactly.
//
// V-cycle (symmetric, so the preconditioner is SPD and plain pCG applies): nu damped-Jacobi
// sweeps, residual, restriction P^T, recursive coarse correction, prolongation P, nu sweeps.
// The coarsest level is solved exactly with a dense inverse (cuSOLVER potrf/potri at set-up).
// Coarse levels are applied from assembled 3^D-point node stencils (fewer bytes per apply than
// the element matrices they are built from).
#pragma once

#include <vector>

#include "q1.cuh"

namespace tb {

struct MgLevel {
  Grid g{};
  int nc = 2;                  // components
  double* ke = nullptr;        // level >= 1: dense element matrices (n_elems x NE x NE), set-up only
  double* st = nullptr;        // level >= 1: half node stencil ((3^D+1)/2 D^2 x n_nodes), applies
  uint8_t* fixed = nullptr;    // Dirichlet mask of this level
  double* dinv = nullptr;      // Jacobi inverse diagonal (0 on fixed)
  double *x = nullptr, *b = nullptr, *r = nullptr, *t = nullptr;  // work vectors
  int64_t n = 0;               // dofs
};

struct Mg {
  std::vector<MgLevel> lv;     // lv[0] = fine level (operator = alpha K_unit, matrix-free)
  double* ainv = nullptr;      // coarsest dense inverse (n x n)
  double* G = nullptr;         // level-1 fast path: R_ch^T K_unit R_ch per child (2^D x NE x NE)
  uint8_t* dirty = nullptr;    // level-1 coarse elements that need the general aggregation
  double* dense = nullptr;     // coarsest dense matrix scratch
  double* gj = nullptr;        // 2D: Gauss-Jordan parked pivot rows (2 x kGjB x n)
  bool gj_stg = false;         // Gauss-Jordan stages the CTA's own rows in shared memory
  size_t gj_smem = 0;          // its dynamic shared memory per CTA
  int* h_info = nullptr;       // pinned copy of the Gauss-Jordan pivot flag, read after the solve
  bool info_pending = false;
  unsigned int* gj_bar = nullptr;  // its grid barrier
  int64_t ncoarse = 0;
  int nu = 2;                  // smoothing sweeps
  double omega = 0.6;          // Jacobi damping
  void* solver = nullptr;      // cusolverDnHandle_t
  double* work = nullptr;      // cuSOLVER workspace
  int lwork = 0;
  int* info = nullptr;
  bool built = false;
};

struct tb_plan_impl;
int mg_build(tb_plan_impl* P);                          // allocate the hierarchy (once per plan)
int mg_setup(tb_plan_impl* P, cudaStream_t s);          // operators for the current alpha
int mg_apply(tb_plan_impl* P, const double* r, double* z, cudaStream_t s);  // z = M^-1 r
int mg_check(tb_plan_impl* P);  // after a stream sync: the deferred set-up check (SPD coarsest level)
struct PcgWork;
// 2D: the whole MG-preconditioned pCG loop in one persistent cooperative launch (mgpcg2d.cu);
// false when unavailable (3D, TB_NO_PERSIST, no co-residency) -> graph path
bool mg_pcg2d_persistent(tb_plan_impl* P, PcgWork& w, cudaStream_t s);
void mg_release(Mg& mg);

}  // namespace tb
