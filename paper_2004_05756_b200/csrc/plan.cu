// Plan lifetime, element tables and workspace management.
#include <vector>

#include "plan.cuh"

namespace tb {

int64_t ElastOp::size() const { return plan->n_dofs; }
int64_t HelmOp::size() const { return filt->g.n_nodes; }

// Hamming distance between two local corner nodes of the Q1 element.
static int corner_dist(int a, int b) {
  auto ox = [](int t) { return ((t & 3) == 1 || (t & 3) == 2) ? 1 : 0; };
  auto oy = [](int t) { return ((t & 3) >= 2) ? 1 : 0; };
  auto oz = [](int t) { return t >> 2; };
  return (ox(a) != ox(b)) + (oy(a) != oy(b)) + (oz(a) != oz(b));
}

void scalar_element_matrices(int dim, double h, double* S, double* M, double* s_div, double* m_mul) {
  const int nn = (dim == 2) ? 4 : 8;
  // 2D (fem.py:72-92): Laplacian 6*S = {4 | -1 edge | -2 diagonal}, mass 36/h^2*M = {4 | 2 | 1}
  // 3D: Laplacian 12/h*S = {4 | 0 edge | -1 face diag | -1 body diag}, mass 216/h^3*M = {8|4|2|1}
  static const double s2[3] = {4.0, -1.0, -2.0}, m2[3] = {4.0, 2.0, 1.0};
  static const double s3[4] = {4.0, 0.0, -1.0, -1.0}, m3[4] = {8.0, 4.0, 2.0, 1.0};
  for (int a = 0; a < nn; ++a)
    for (int b = 0; b < nn; ++b) {
      const int d = corner_dist(a, b);
      S[a * nn + b] = (dim == 2) ? s2[d] : s3[d];
      M[a * nn + b] = (dim == 2) ? m2[d] : m3[d];
    }
  *s_div = (dim == 2) ? 6.0 : 12.0;
  *m_mul = (dim == 2) ? h * h / 36.0 : h * h * h / 216.0;
}

bool hex8_blocks(const double* K, Hex8Iso* B) {
  auto loc = [](int t) {  // corner t = ox + 2 oy + 4 oz -> local node (CCW faces)
    const int ox = t & 1, oy = (t >> 1) & 1, oz = t >> 2;
    return (oy ? (ox ? 2 : 3) : (ox ? 1 : 0)) + 4 * oz;
  };
  auto sgn = [](int s, int t) { return (__builtin_popcount(s & t) & 1) ? -1.0 : 1.0; };
  double Mf[24][24];  // (s, c) x (s', c')
  double kmax = 0.0;
  for (int s = 0; s < 8; ++s)
    for (int c = 0; c < 3; ++c)
      for (int s2 = 0; s2 < 8; ++s2)
        for (int c2 = 0; c2 < 3; ++c2) {
          double acc = 0.0;
          for (int t = 0; t < 8; ++t)
            for (int t2 = 0; t2 < 8; ++t2)
              acc += sgn(s, t) * K[(loc(t) * 3 + c) * 24 + loc(t2) * 3 + c2] * sgn(s2, t2);
          Mf[s * 3 + c][s2 * 3 + c2] = acc / 64.0;
          kmax = fmax(kmax, fabs(acc / 64.0));
        }
  double off = 0.0;
  for (int r = 0; r < 24; ++r)
    for (int q = 0; q < 24; ++q) {
      const int kr = (r / 3) ^ (1 << (r % 3)), kq = (q / 3) ^ (1 << (q % 3));
      if (kr != kq) off = fmax(off, fabs(Mf[r][q]));
    }
  double m[8][3][3];
  for (int k = 0; k < 8; ++k)
    for (int c = 0; c < 3; ++c)
      for (int c2 = 0; c2 < 3; ++c2) m[k][c][c2] = Mf[(k ^ (1 << c)) * 3 + c][(k ^ (1 << c2)) * 3 + c2];
  B->a = m[0][0][0];
  B->b = m[0][0][1];
  B->c = m[1][1][1];
  B->d = m[1][1][2];
  B->e = m[3][0][0];
  B->f = m[3][2][2];
  B->g = m[7][0][0];
  B->h = m[7][0][1];
  const double a = B->a, b = B->b, c = B->c, d = B->d, e = B->e, f = B->f, g = B->g, h = B->h;
  const double pat[8][3][3] = {
      {{a, b, b}, {b, a, b}, {b, b, a}}, {{0, 0, 0}, {0, c, d}, {0, d, c}}, {{c, 0, d}, {0, 0, 0}, {d, 0, c}},
      {{e, e, 0}, {e, e, 0}, {0, 0, f}}, {{c, d, 0}, {d, c, 0}, {0, 0, 0}}, {{e, 0, e}, {0, f, 0}, {e, 0, e}},
      {{f, 0, 0}, {0, e, e}, {0, e, e}}, {{g, h, h}, {h, g, h}, {h, h, g}}};
  double dev = off;
  for (int k = 0; k < 8; ++k)
    for (int c2 = 0; c2 < 3; ++c2)
      for (int c3 = 0; c3 < 3; ++c3) dev = fmax(dev, fabs(m[k][c2][c3] - pat[k][c2][c3]));
  return dev <= 1e-13 * kmax;
}

Grid make_grid(int dim, int nx, int ny, int nz, double h) {
  Grid g{};
  g.dim = dim;
  g.nx = nx;
  g.ny = ny;
  g.nz = (dim == 3) ? nz : 1;
  g.nnx = nx + 1;
  g.nny = ny + 1;
  g.nnz = (dim == 3) ? nz + 1 : 1;
  g.h = h;
  g.n_elems = (int64_t)nx * ny * g.nz;
  g.n_nodes = (int64_t)g.nnx * g.nny * g.nnz;
  return g;
}

int tb_plan_impl::init(const uint8_t* fixed_host) {
  const size_t ne = (size_t)g.n_elems;
  TB_CUDA(cudaMalloc(&d_fixed, (size_t)n_dofs));
  TB_CUDA(cudaMemcpy(d_fixed, fixed_host, (size_t)n_dofs, cudaMemcpyHostToDevice));
  if (g.dim == 3 && hex8) {  // Dirichlet rows per owning k_hex8 CTA (counting sort)
    const dim3 gr = hex8_grid(g, zchunk);
    const int64_t nb = (int64_t)gr.x * gr.y * gr.z;
    std::vector<int> off(nb + 1, 0);
    for (int64_t d = 0; d < n_dofs; ++d)
      if (fixed_host[d]) ++off[hex8_owner(g, zchunk, d) + 1];
    for (int64_t b = 0; b < nb; ++b) off[b + 1] += off[b];
    n_fixed = off[nb];
    std::vector<int64_t> idx(n_fixed > 0 ? n_fixed : 1);
    std::vector<int> pos(off.begin(), off.end() - 1);
    for (int64_t d = 0; d < n_dofs; ++d)
      if (fixed_host[d]) idx[pos[hex8_owner(g, zchunk, d)]++] = d;
    TB_CUDA(cudaMalloc(&d_fixed_idx, sizeof(int64_t) * idx.size()));
    TB_CUDA(cudaMemcpy(d_fixed_idx, idx.data(), sizeof(int64_t) * idx.size(), cudaMemcpyHostToDevice));
    TB_CUDA(cudaMalloc(&d_fixed_off, sizeof(int) * off.size()));
    TB_CUDA(cudaMemcpy(d_fixed_off, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice));
  }
  TB_CUDA(cudaMalloc(&d_alpha, sizeof(double) * ne));
  TB_CUDA(cudaMalloc(&d_alpha2, sizeof(double) * ne));
  TB_CUDA(cudaMalloc(&d_scratch, sizeof(double) * 8 * 148 * 8));
  TB_CUDA(cudaMalloc(&d_scalar, sizeof(double) * 16));
  TB_CUDA(cudaMallocHost(&h_scalar, sizeof(double) * 16));
  // Hex8 plans: vectors large enough for the pitched layout of the single-sweep pCG
  TB_TRY(work.alloc(n_dofs, op.fused_blocks(), op.persist_grid > 0, (g.dim == 3 && hex8) ? sweep_size(g) : 0));
  TB_TRY(work.set_fields(0, 0, g.nnz));
  return TB_OK;
}

bool ElastOp::has_precond() const { return plan->precond == 1 && !plan->dist; }
int ElastOp::precond_setup(cudaStream_t s) const { return mg_setup(plan, s); }
int ElastOp::precond_apply(const double* r, double* z, cudaStream_t s) const { return mg_apply(plan, r, z, s); }
int ElastOp::precond_check() const { return plan->precond == 1 ? mg_check(plan) : TB_OK; }

void tb_plan_impl::release() {
  sweep_release(this);
  mg_release(mg);
  work.release();
  void* bufs[] = {d_fixed, d_fixed_idx, d_fixed_off, d_alpha, d_alpha2, d_scratch, d_scalar, d_rom};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (h_scalar) cudaFreeHost(h_scalar);
  d_fixed = nullptr;
  d_fixed_idx = nullptr;
  d_fixed_off = nullptr;
  n_fixed = 0;
  d_alpha = d_alpha2 = d_scratch = d_scalar = d_rom = h_scalar = nullptr;
}

int tb_plan_impl::rom_scratch(size_t bytes) {
  if (bytes <= rom_bytes) return TB_OK;
  if (d_rom) cudaFree(d_rom);
  d_rom = nullptr;
  rom_bytes = 0;
  TB_CUDA(cudaMalloc(&d_rom, bytes));
  rom_bytes = bytes;
  return TB_OK;
}

}  // namespace tb
