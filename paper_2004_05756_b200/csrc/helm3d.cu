// 3D Helmholtz filter operator (reference filtering.py:47-114, H = sum_e r^2 S_e + M_e on a
// uniform Hex8 grid) as a constant-coefficient 27-point stencil with a shared-memory z-sweep.
//
// On a cube both S_e and M_e are invariant under the cube's reflections, so H_e[a][b] depends
// only on the Hamming distance between corners a and b: four values h0..h3.  The node-owner
// sum y_n = sum_{e at n} sum_b H_e[n][b] x_b then collapses to
//   y_n = sum_d h_|d| cx(dx) cy(dy) cz(dz) x_{n+d},   d in {-1,0,1}^3,
// where c(-1) = [element below exists], c(+1) = [element above exists], c(0) = their sum counts
// the elements on that axis that contain both nodes (the domain boundary removes elements).
// The generic node-owner kernel (q1.cuh: 27 gathered neighbours, each p = z + beta p_old built
// from two global loads, 64 FMA over 8 element rows) took ~97 us per call at cfg 3 (1.79M
// nodes, 2.7% of the headline evaluation); this one stages node planes of p in shared memory.
//
// A CTA owns a 32 x 8 node tile and sweeps a z-chunk: node plane kp arrives (z and p_old by
// cp.async, zero-filled outside the grid), p = z + beta p_old goes into a 3-plane ring (and to
// pnew on owned nodes), then the plane below is finished from the ring.  FUSED also reduces
// p.q over the planes [dot_k0, dot_k1) and, in the last CTA, sets alpha = rz / pq (the contract
// of k_pcg_fused); !FUSED is y = H x.
#include "plan.cuh"

namespace tb {

namespace {

constexpr int kHzX = 32, kHzY = 8, kHzT = kHzX * kHzY;  // owned node tile, one node per thread
constexpr int kHzPX = kHzX + 2, kHzPY = kHzY + 2;        // plane tile with halo
constexpr int kHzPlane = kHzPX * kHzPY;                   // 340

struct HelmIso {
  double h[4];  // H_e entries by corner Hamming distance 0..3
};

template <bool FUSED>
__global__ void __launch_bounds__(kHzT) k_helm3d(Grid g, HelmIso H, const double* __restrict__ z,
                                                 const double* __restrict__ pold, double* __restrict__ pnew,
                                                 double* __restrict__ q, PcgState* st, double* partials,
                                                 int zchunk) {
  __shared__ double stg[2][2][kHzPlane];  // [buffer][z, p_old] raw planes
  __shared__ double ring[3][kHzPlane];    // p planes
  double beta = 0.0;
  int dk0 = 0, dk1 = 0;
  if (FUSED) {
    if (st->done) return;
    beta = st->beta;
    dk0 = st->dot_k0;
    dk1 = st->dot_k1;
  }
  const int t = threadIdx.x;
  const int i0 = blockIdx.x * kHzX, j0 = blockIdx.y * kHzY;
  const int K0 = blockIdx.z * zchunk, K1 = min(g.nnz, K0 + zchunk);
  const int ox = t % kHzX, oy = t / kHzX;
  const int i = i0 + ox, j = j0 + oy;
  const bool own = i < g.nnx && j < g.nny;
  const int64_t pn = (int64_t)g.nnx * g.nny;
  // per-axis element-existence factors of this thread's node (c(-1), c(0), c(+1))
  const double xm = i > 0 ? 1.0 : 0.0, xp = i < g.nx ? 1.0 : 0.0;
  const double ym = j > 0 ? 1.0 : 0.0, yp = j < g.ny ? 1.0 : 0.0;
  // x-row weights for |dy| + |dz| = m: centre cx(0) h_m, sides cx(-1) h_{m+1}, cx(+1) h_{m+1}
  double wc[3], wl[3], wr[3];
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    wc[m] = (xm + xp) * H.h[m];
    wl[m] = xm * H.h[m + 1];
    wr[m] = xp * H.h[m + 1];
  }
  const double cy[3] = {ym, ym + yp, yp};
  // fetch slots: halo plane index f = t + s kHzT (two slots cover 340); the in-plane offset,
  // validity and ownership of each slot are fixed for the whole sweep
  int64_t soff[2];
  unsigned sok = 0, sown = 0;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int f = t + s * kHzT;
    const int lx = f % kHzPX, ly = f / kHzPX;
    const int ni = i0 - 1 + lx, nj = j0 - 1 + ly;
    const bool ok = f < kHzPlane && ni >= 0 && ni < g.nnx && nj >= 0 && nj < g.nny;
    soff[s] = ok ? (int64_t)nj * g.nnx + ni : 0;
    if (ok) sok |= 1u << s;
    if (ok && lx >= 1 && lx <= kHzX && ly >= 1 && ly <= kHzY) sown |= 1u << s;
  }
  auto issue = [&](int kp, int buf) {
    const bool zok = kp >= 0 && kp < g.nnz;
    const int64_t po = zok ? (int64_t)kp * pn : 0;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int f = t + s * kHzT;
      if (f < kHzPlane) {
        const bool ok = zok && (sok >> s & 1u);
        const int64_t off = ok ? po + soff[s] : 0;
        cp_async8(&stg[buf][0][f], z + off, ok);
        if (FUSED) cp_async8(&stg[buf][1][f], pold + off, ok);
      }
    }
    cp_async_commit();
  };
  // plane kp landed in stg[buf] -> p into ring slot, owned p to pnew
  auto land = [&](int kp, int buf, int slot) {
    const bool pown = kp >= K0 && kp < K1;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int f = t + s * kHzT;
      if (f < kHzPlane) {
        const double p = FUSED ? fma(beta, stg[buf][1][f], stg[buf][0][f]) : stg[buf][0][f];
        ring[slot][f] = p;
        if (FUSED && pown && (sown >> s & 1u)) pnew[(int64_t)kp * pn + soff[s]] = p;
      }
    }
  };
  double acc[1] = {0.0};
  // planes m = 0 .. S are node planes K0-1 .. K1 (zero outside the grid); output plane
  // ko = K0 + m - 2 is finished once plane m has landed (it needs ko-1, ko, ko+1)
  const int S = K1 - K0 + 1;
  issue(K0 - 1, 0);
  issue(K0, 1);
  for (int m = 0; m <= S; ++m) {
    if (m + 1 <= S) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();  // plane m landed for everyone; ring slot m % 3 no longer read
    land(K0 - 1 + m, m & 1, m % 3);
    __syncthreads();
    if (m + 2 <= S) issue(K0 + 1 + m, m & 1);  // into the staging buffer just consumed
    if (m >= 2 && own) {
      const int ko = K0 + m - 2;
      const double zm = ko > 0 ? 1.0 : 0.0, zp = ko < g.nz ? 1.0 : 0.0;
      const double cz[3] = {zm, zm + zp, zp};
      double y = 0.0;
#pragma unroll
      for (int dz = 0; dz < 3; ++dz) {
        const double* P = ring[(m - 2 + dz) % 3];
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) {
          const int mm = (dz != 1) + (dy != 1);
          const double* row = P + (oy + dy) * kHzPX + ox;
          const double sx = fma(wl[mm], row[0], fma(wc[mm], row[1], wr[mm] * row[2]));
          y = fma(cz[dz] * cy[dy], sx, y);
        }
      }
      q[(int64_t)ko * pn + (int64_t)j * g.nnx + i] = y;
      if (FUSED && ko >= dk0 && ko < dk1) acc[0] = fma(ring[(m - 1) % 3][(oy + 1) * kHzPX + ox + 1], y, acc[0]);
    }
  }
  if (FUSED) {
    block_sum<1>(acc);
    if (publish_partials<1>(acc, partials, &st->count_a)) {
      gather_partials<1>(acc, partials, &st->count_a);
      if (threadIdx.x == 0) {
        const double v = acc[0];
        if (st->dist) {
          st->red[0] = v;
        } else if (!(v > 0.0) || !isfinite(v)) {
          st->done = 3;
        } else {
          st->pq = v;
          st->alpha = st->rz / v;
        }
      }
    }
  }
}

inline dim3 helm3d_grid(const Grid& g, int zc) {
  return dim3((g.nnx + kHzX - 1) / kHzX, (g.nny + kHzY - 1) / kHzY, (g.nnz + zc - 1) / zc);
}

// z-chunk: a whole number of waves at 6 resident CTAs per SM, chunks of >= 8 planes
inline int helm3d_zchunk(const Grid& g) {
  const int64_t xy = (int64_t)((g.nnx + kHzX - 1) / kHzX) * ((g.nny + kHzY - 1) / kHzY);
  const int64_t slots = 148 * 6;
  int best = g.nnz;
  double bc = 1e30;
  for (int zc = 8; zc <= g.nnz + 7; ++zc) {
    const int64_t ctas = xy * ((g.nnz + zc - 1) / zc);
    const double cost = (double)((ctas + slots - 1) / slots) * (zc + 2.0);
    if (cost < bc - 1e-9) {
      bc = cost;
      best = zc;
    }
  }
  return best;
}

}  // namespace

// H3 (8 x 8, local corner order of q1.cuh) -> the four Hamming-distance values, or false when H3
// lacks that symmetry (the generic node-owner kernel is used then)
bool helm3d_iso(const double* H3, double* h4) {
  double hv[4] = {0, 0, 0, 0};
  bool seen[4] = {false, false, false, false};
  double scale = 0.0;
  for (int a = 0; a < 64; ++a) scale = fmax(scale, fabs(H3[a]));
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) {
      const int d = (offx(a) != offx(b)) + (offy(a) != offy(b)) + (offz(a) != offz(b));
      const double v = H3[a * 8 + b];
      if (!seen[d]) {
        hv[d] = v;
        seen[d] = true;
      } else if (fabs(v - hv[d]) > 1e-14 * scale) {
        return false;
      }
    }
  for (int d = 0; d < 4; ++d) h4[d] = hv[d];
  return true;
}

static bool helm3d_off() {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("TB_HELM3D_GENERIC");
    off = (e != nullptr && e[0] != '\0' && e[0] != '0') ? 1 : 0;
  }
  return off == 1;
}

bool helm3d_launch_fused(const Grid& g, const double* h4, const PcgWork& w, const double* pold, double* pnew,
                         cudaStream_t s) {
  if (helm3d_off()) return false;
  HelmIso H;
  for (int d = 0; d < 4; ++d) H.h[d] = h4[d];
  const int zc = helm3d_zchunk(g);
  k_helm3d<true><<<helm3d_grid(g, zc), kHzT, 0, s>>>(g, H, w.z, pold, pnew, w.q, w.st, w.partA(), zc);
  return true;  // counted by the pCG driver, as the generic kernel
}

bool helm3d_launch_apply(const Grid& g, const double* h4, const double* v, double* y, cudaStream_t s) {
  if (helm3d_off()) return false;
  HelmIso H;
  for (int d = 0; d < 4; ++d) H.h[d] = h4[d];
  const int zc = helm3d_zchunk(g);
  k_helm3d<false><<<helm3d_grid(g, zc), kHzT, 0, s>>>(g, H, v, nullptr, nullptr, y, nullptr, nullptr, zc);
  launched(1);
  return true;
}

int64_t helm3d_max_ctas(const Grid& g) {
  const dim3 gr = helm3d_grid(g, helm3d_zchunk(g));
  return (int64_t)gr.x * gr.y * gr.z;
}

}  // namespace tb
