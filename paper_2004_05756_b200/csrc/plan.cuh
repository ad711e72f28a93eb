// Plan / filter objects behind the opaque C handles.
#pragma once

#include "hex8.cuh"
#include "mg.cuh"
#include "pcg.cuh"
#include "cgtile2d.cuh"

namespace tb {

struct tb_plan_impl;
struct tb_filter_impl;
struct SweepState;
struct SpectralFilter;

// SIMP elasticity operator  Z K(rho) Z  (alpha from the plan's d_alpha)
struct ElastOp final : PcgOp {
  tb_plan_impl* plan = nullptr;
  int64_t size() const override;
  int fused_blocks() const override;
  void launch_fused(const PcgWork& w, const double* pold, double* pnew, cudaStream_t s) const override;
  void launch_apply(const double* v, double* y, cudaStream_t s) const override;
  void launch_dinv(double* dinv, cudaStream_t s) const override;
  bool has_persistent() const override { return persist_grid > 0; }
  void launch_persistent(const PcgWork& w, cudaStream_t s) const override;
  bool has_precond() const override;
  int precond_setup(cudaStream_t s) const override;
  int precond_apply(const double* r, double* z, cudaStream_t s) const override;
  bool launch_persistent_pc(PcgWork& w, cudaStream_t s) const override;
  int precond_check() const override;
  int persist_grid = 0;
  TileSpec tiles{0, 0, 0, 0, 0};  // 2D persistent pCG decomposition (tx = 0: row strips)
};

// Helmholtz operator  H = sum_e (r^2 S_e + M_e)  (pure Neumann)
struct HelmOp final : PcgOp {
  tb_filter_impl* filt = nullptr;
  int64_t size() const override;
  int fused_blocks() const override;
  void launch_fused(const PcgWork& w, const double* pold, double* pnew, cudaStream_t s) const override;
  void launch_apply(const double* v, double* y, cudaStream_t s) const override;
  void launch_dinv(double* dinv, cudaStream_t s) const override;
  bool has_persistent() const override { return persist_grid > 0; }
  void launch_persistent(const PcgWork& w, cudaStream_t s) const override;
  int persist_grid = 0;
  TileSpec tiles{0, 0, 0, 0, 0};  // 2D persistent pCG decomposition (tx = 0: row strips)
};

struct tb_plan_impl {
  Grid g{};
  int64_t n_dofs = 0;
  int device = 0;
  double rho_l = 1e-3, p = 3.0;
  Mat<8> K2{};
  Q4Pat pat{};       // 2D: pattern values of K2 (q4_pat)
  bool pat_ok = false;
  Mat<24> K3{};
  Hex8Iso hiso{};        // WHT block values of K3 (3D)
  bool hex8 = false;     // K3 has the isotropic WHT block structure -> element-centric kernel
  bool hex8_epi = false; // the epilogue instances of k_hex8 (multigrid level 0) are usable
  int zchunk = 8;
  int dist = 0;              // distributed (slab) pCG mode
  int precond = 0;           // 0 Jacobi, 1 geometric multigrid
  Mg mg;
  int own_k0 = 0, own_k1 = 1 << 30;  // owned node planes (set by tb_plan_set_owned_planes); ROM rows
  uint8_t* d_fixed = nullptr;
  int64_t* d_fixed_idx = nullptr;  // 3D Hex8: fixed dofs bucketed by the k_hex8 CTA owning them
  int* d_fixed_off = nullptr;      // bucket offsets (CTAs + 1)
  int64_t n_fixed = 0;
  double* d_alpha = nullptr;   // alpha of the design being solved (read by the pCG graph)
  double* d_alpha2 = nullptr;  // alpha scratch for one-off applies
  double* d_scratch = nullptr; // reduction partials
  double* d_scalar = nullptr;
  double* h_scalar = nullptr;  // pinned
  double* d_rom = nullptr;     // ROM scratch (grown on demand)
  size_t rom_bytes = 0;
  ElastOp op;
  PcgWork work;
  SweepState* sweep = nullptr;  // 3D single-sweep Jacobi-pCG (sweep.cu), created on first use

  int init(const uint8_t* fixed_host);
  void release();
  void apply_alpha(const double* alpha, const double* v, double* y, bool mask, cudaStream_t s) const;
  bool apply_alpha_epi(int epi, const double* alpha, const double* v, double* out, const double* b,
                       const double* dinv, double omega, cudaStream_t s) const;
  int material(const double* rho, double* alpha, double* dalpha, cudaStream_t s) const;
  int rom_scratch(size_t bytes);
};

struct tb_filter_impl {
  Grid g{};
  int device = 0;
  double radius = 0.0, r = 0.0, vol_share = 0.0;
  Mat<4> H2{};
  Q4Pat pat{};       // 2D: pattern values of H2
  bool pat_ok = false;
  Mat<8> H3{};
  bool iso3 = false;    // 3D: H3 has the cube symmetry -> 27-point stencil kernel (helm3d.cu)
  double h4[4] = {0, 0, 0, 0};
  double* d_b = nullptr;
  // slab mode (tb_filter_set_owned_planes): ghost node planes masked (dinv 0), owned [k0, k1)
  uint8_t* d_fixed = nullptr;
  int dist = 0, own_k0 = 0, own_k1 = 1 << 30;
  HelmOp op;
  PcgWork work;
  // direct solve of the whole-grid filter system by the tensor-product cosine basis
  // (spectral.cu); null: pCG (slab phases, TB_FILTER_PCG=1, or a failed self-check)
  SpectralFilter* spec = nullptr;
};

// direct Helmholtz filter solve (spectral.cu)
void spectral_init(tb_filter_impl* F);
void spectral_release(tb_filter_impl* F);
int spectral_solve(tb_filter_impl* F, const double* b, double* phi, cudaStream_t s);

// Integer Laplacian / mass tables of the scalar Q1 element: S_e = (h^(d-2)) S/s_div,
// M_e = m_mul * M  (2D: S/6, h^2/36 M, fem.py:72-92; 3D: h S/12, h^3/216 M).
// Isotropic WHT block values of a Hex8 element matrix; false if K lacks that structure.
bool hex8_blocks(const double* K, Hex8Iso* B);
void scalar_element_matrices(int dim, double h, double* S, double* M, double* s_div, double* m_mul);
Grid make_grid(int dim, int nx, int ny, int nz, double h);
void finish_sum(int nb, const double* part, double* out, cudaStream_t s);
int device_dot(const double* a, const double* b, int64_t n, double* scratch, double* out_dev, cudaStream_t s);

// 3D Helmholtz operator as a constant-coefficient 27-point stencil (helm3d.cu)
bool helm3d_iso(const double* H3, double* h4);
bool helm3d_launch_fused(const Grid& g, const double* h4, const PcgWork& w, const double* pold, double* pnew,
                         cudaStream_t s);
bool helm3d_launch_apply(const Grid& g, const double* h4, const double* v, double* y, cudaStream_t s);
int64_t helm3d_max_ctas(const Grid& g);

// single-sweep 3D Jacobi-pCG (sweep.cu)
int64_t sweep_size(const Grid& g);
bool sweep_enabled(const tb_plan_impl* P);
void sweep_release(tb_plan_impl* P);
int pcg_solve_sweep(tb_plan_impl* P, const double* b, double* x_out, double rtol, int maxit, int* iters,
                    double* relres, cudaStream_t s);
int pcg_profile_sweep(tb_plan_impl* P, const double* b, int nrep, double* ms_iter, cudaStream_t s);
int pcg_iter_time_sweep(tb_plan_impl* P, int reset, double* ms, int64_t* iters);

// element-form reduced stiffness on DMMA for Hex8 plans (romfused.cu)
bool rom_fused_eligible(const tb_plan_impl* P, int k);
double rom_fused_flops(const tb_plan_impl* P, int k, int nd);
size_t rom_fused_scratch_bytes(const tb_plan_impl* P, int k, int nd);
int rom_fused_khat(tb_plan_impl* P, const double* phi, int k, const double* alpha, int nd, int kb0, int kb1,
                   double* part_scratch, size_t part_bytes, double* khat, cudaStream_t s);

}  // namespace tb
