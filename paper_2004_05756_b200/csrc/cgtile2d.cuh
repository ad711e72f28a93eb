// Persistent single-reduction Jacobi-pCG for 2D grids on square-ish node TILES.
//
// Same algorithm as k_pcg2d_cgcg (cgcg2d.cuh: Chronopoulos-Gear pCG, state in shared memory,
// one grid barrier per iteration, redundant halo recomputation of u = D^-1 r from the
// neighbours' published (r, w, s)), but a CTA owns a tw x th block of nodes instead of a run
// of node ids.  A row strip of ~1.4 node rows (cfg 2) has a halo of two full rows -- larger
// than what it owns -- and publishes every own value; a 29 x 29 tile reads a ring of ~120
// halo nodes and publishes only its own boundary ring, ~10x less L2 traffic per iteration.
#pragma once

#include "cgcg2d.cuh"

// TB_CGCG_ABL builds: TB_CGCG_DBG bits skip phases for timing (results meaningless)
#if defined(TB_CGCG_ABL)
#define TILE_SKIP(bit) (a.dbg & (bit))
#else
#define TILE_SKIP(bit) false
#endif

namespace tb {

struct TileSpec {
  int tx, ty;  // tiles along x / y (gridDim.x = tx * ty)
  int tw, th;  // tile width / height in nodes (last tiles may be smaller)
  int reg;     // host: 1 = register-resident kernel (k_pcg2d_treg)
};

template <int NC, bool SCALED, bool PAT>
__global__ void __launch_bounds__(kCgcgThreads, 1) k_pcg2d_tile(Grid g, Mat<4 * NC> K, Q4Pat kp,
                                                               const double* __restrict__ alpha, CgcgArgs a,
                                                               TileSpec ts) {
  extern __shared__ double sm[];
  __shared__ __align__(16) Mat<4 * NC> Ks;
  __shared__ double bc[2][3];
  const int tid = threadIdx.x, nt = blockDim.x, nbk = gridDim.x;
  const int nnx = g.nnx, nny = g.nny;
  const int64_t ND = (int64_t)NC * g.n_nodes;
  const int bx = blockIdx.x % ts.tx, by = blockIdx.x / ts.tx;
  const int ox0 = bx * ts.tw, ox1 = min(nnx, ox0 + ts.tw);
  const int oy0 = by * ts.th, oy1 = min(nny, oy0 + ts.th);
  const int owx = max(0, ox1 - ox0), owy = max(0, oy1 - oy0), no = owx * owy;
  // extended tile: own nodes plus the one-node ring the stencil touches (clipped to the grid)
  const int ex0 = max(ox0 - 1, 0), ex1 = min(ox1 + 1, nnx), ey0 = max(oy0 - 1, 0), ey1 = min(oy1 + 1, nny);
  const int W = max(0, ex1 - ex0), H = max(0, ey1 - ey0), ne_ext = W * H;
  // elements touching own nodes
  const int ax0 = max(ox0 - 1, 0), ax1 = min(ox1, g.nx), ay0 = max(oy0 - 1, 0), ay1 = min(oy1, g.ny);
  const int AW = max(0, ax1 - ax0), AH = max(0, ay1 - ay0);
  double* u_ext = sm;                          // [H][W][NC]
  double* dext = u_ext + (size_t)ne_ext * NC;  // D^-1 over the extended tile (constant)
  double* xs = dext + (size_t)ne_ext * NC;     // own [no][NC]: x, r, p, s, w
  double* rs = xs + (size_t)no * NC;
  double* ps = rs + (size_t)no * NC;
  double* ss = ps + (size_t)no * NC;
  double* ws = ss + (size_t)no * NC;
  double* as = ws + (size_t)no * NC;           // alpha [AH][AW]
  const int offx = ox0 - ex0, offy = oy0 - ey0;
  if (!PAT)
    for (int o = tid; o < 16 * NC * NC; o += nt) Ks.v[o] = K.v[o];
  for (int q = tid; q < AW * AH; q += nt) {
    const int ey = ay0 + q / AW, exx = ax0 + q % AW;
    as[q] = SCALED ? alpha[(int64_t)ey * g.nx + exx] : 1.0;
  }
  for (int q = tid; q < ne_ext * NC; q += nt) {
    const int node = q / NC, c = q % NC;
    const int y = ey0 + node / W, x = ex0 + node % W;
    const int64_t d = ((int64_t)y * nnx + x) * NC + c;
    dext[q] = a.dinv[d];
    u_ext[q] = a.dinv[d] * a.r0[d];
  }
  for (int o = tid; o < no; o += nt) {
    const int ly = o / owx, lx = o - ly * owx;
    const int64_t d = ((int64_t)(oy0 + ly) * nnx + ox0 + lx) * NC;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      xs[o * NC + c] = a.x[d + c];
      rs[o * NC + c] = a.r0[d + c];
      ps[o * NC + c] = 0.0;
      ss[o * NC + c] = 0.0;
    }
  }
  __syncthreads();

  double* pubr[2] = {a.pub, a.pub + 3 * ND};
  // out = rows of K(alpha) for own node (x, y) at extended index ei
  auto node_apply = [&](int x, int y, int ei, double (&out)[NC]) {
    double P[9][NC];
    double sc[4];
    if (x > 0 && x < nnx - 1 && y > 0 && y < nny - 1) {
      const double* u0 = u_ext + (ei - W - 1) * NC;
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx)
#pragma unroll
          for (int c = 0; c < NC; ++c) P[dy * 3 + dx][c] = u0[(dy * W + dx) * NC + c];
      const double* a0 = as + ((y - 1 - ay0) * AW + x - 1 - ax0);
      sc[0] = a0[0];
      sc[1] = a0[1];
      sc[2] = a0[AW];
      sc[3] = a0[AW + 1];
    } else {
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const int ii = x + dx - 1, jj = y + dy - 1;
          const bool ok = ii >= 0 && ii < nnx && jj >= 0 && jj < nny;
          const int m = (jj - ey0) * W + ii - ex0;
#pragma unroll
          for (int c = 0; c < NC; ++c) P[dy * 3 + dx][c] = ok ? u_ext[m * NC + c] : 0.0;
        }
#pragma unroll
      for (int sl = 0; sl < 4; ++sl) {
        const int ei_ = x - 1 + (sl & 1), ej = y - 1 + (sl >> 1);
        const bool ok = ei_ >= 0 && ei_ < g.nx && ej >= 0 && ej < g.ny;
        sc[sl] = ok ? as[(ej - ay0) * AW + ei_ - ax0] : 0.0;
      }
    }
    if (PAT)
      node_rows_pat<NC>(kp, P, sc, out);
    else
      node_rows<2, NC>(Ks, P, sc, out);
  };

  // w_0 = A u_0; partials; publish the own boundary ring of (r_0, w_0, s_{-1} = 0)
  double acc[3] = {0.0, 0.0, 0.0};
  for (int o = tid; o < no; o += nt) {
    const int ly = o / owx, lx = o - ly * owx, x = ox0 + lx, y = oy0 + ly;
    const int ei = (ly + offy) * W + lx + offx;
    double out[NC];
    node_apply(x, y, ei, out);
    const bool ring = lx == 0 || lx == owx - 1 || ly == 0 || ly == owy - 1;
    const int64_t d = ((int64_t)y * nnx + x) * NC;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int od = o * NC + c;
      const double u = u_ext[ei * NC + c];
      ws[od] = out[c];
      acc[0] = fma(rs[od], u, acc[0]);
      acc[1] = fma(out[c], u, acc[1]);
      acc[2] = fma(rs[od], rs[od], acc[2]);
      if (ring) {
        pubr[0][d + c] = rs[od];
        pubr[0][ND + d + c] = out[c];
        pubr[0][2 * ND + d + c] = 0.0;
      }
    }
  }
  // partials parity-buffered (see cgcg2d.cuh); the non-pattern variant keeps the separate block
  // sum and barrier (ptxas spills ~800 B there otherwise)
  if constexpr (PAT) {
    publish_partials_grid_sync<3>(acc, a.part, a.bar);
  } else {
    block_sum<3>(acc);
    if (tid == 0) {
      a.part[blockIdx.x] = acc[0];
      a.part[nbk + blockIdx.x] = acc[1];
      a.part[2 * nbk + blockIdx.x] = acc[2];
    }
    grid_sync_flip(a.bar);
  }

  double gam = 0.0, al = 0.0, be = 0.0, rr = 0.0;
  int it = a.st->iters, done = 0;
  const int maxit = a.st->maxit;
  const double tol2 = a.st->tol2;
  int par = 0;
  // halo ring of the extended tile: bottom row, top row, left column, right column
  const int nb_b = (ey0 < oy0) ? W : 0, nb_t = (ey1 > oy1) ? W : 0;
  const int nb_l = (ex0 < ox0) ? owy : 0, nb_r = (ex1 > ox1) ? owy : 0;
  const int halo = (nb_b + nb_t + nb_l + nb_r) * NC;
  constexpr int kHB = 2;
  const int ht = tid - 32, hnt = nt - 32;
  auto ring_xy = [&](int t, int& x, int& y) {
    if (t < nb_b) { x = ex0 + t; y = ey0; return; }
    t -= nb_b;
    if (t < nb_t) { x = ex0 + t; y = ey1 - 1; return; }
    t -= nb_t;
    if (t < nb_l) { x = ex0; y = oy0 + t; return; }
    t -= nb_l;
    x = ex1 - 1;
    y = oy0 + t;
  };
  for (bool first = true;; first = false) {
    const double* pr = pubr[par];
    double rv[kHB], wv[kHB], sv[kHB];
    int mm[kHB];
    auto halo_load = [&](int base) {
#pragma unroll
      for (int q = 0; q < kHB; ++q) {
        const int e = base + ht + q * hnt;
        mm[q] = -1;
        if (ht >= 0 && e < halo) {
          int x, y;
          ring_xy(e / NC, x, y);
          const int c = e % NC;
          const int64_t m = ((int64_t)y * nnx + x) * NC + c;
          mm[q] = ((y - ey0) * W + x - ex0) * NC + c;
          rv[q] = __ldcg(pr + m);
          wv[q] = __ldcg(pr + ND + m);
          sv[q] = __ldcg(pr + 2 * ND + m);
        }
      }
    };
    if (tid >= 32 && !TILE_SKIP(4)) halo_load(0);
    if (tid < 32 && !TILE_SKIP(16)) {
      constexpr int kPB = 8;  // up to 256 CTAs
      double v[3][kPB];
#pragma unroll
      for (int q = 0; q < kPB; ++q) {
        const int b = tid + 32 * q;
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c][q] = (b < nbk) ? __ldcg(a.part + (par * 3 + c) * nbk + b) : 0.0;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < kPB; ++q) s += v[c][q];
        s = warp_sum(s);
        if (tid == 0) bc[par][c] = s;
      }
    }
    __syncthreads();
    const double gnew = bc[par][0], dnew = bc[par][1];
    rr = bc[par][2];
#if defined(TB_CGCG_ABL)
    if (a.dbg & 8) {  // run exactly maxit iterations
      if (!first && ++it >= maxit) {
        done = 2;
        break;
      }
      be = first ? 0.0 : 0.5;
      al = 0.5;
      gam = 1.0;
      goto tile_continue;
    }
#endif
    if (!isfinite(gnew) || !isfinite(dnew) || !isfinite(rr)) {
      done = 3;
      break;
    }
    if (!first) {
      ++it;
      if (rr <= tol2) {
        done = 1;
        break;
      }
      if (it >= maxit) {
        done = 2;
        break;
      }
    } else if (rr == 0.0 || rr <= tol2) {
      done = 1;
      break;
    }
    if (first) {
      be = 0.0;
      if (!(dnew > 0.0)) {
        done = 3;
        break;
      }
      al = gnew / dnew;
    } else {
      be = gnew / gam;
      const double pap = dnew - be * gnew / al;
      if (!(pap > 0.0)) {
        done = 3;
        break;
      }
      al = gnew / pap;
    }
    gam = gnew;
#if defined(TB_CGCG_ABL)
  tile_continue:
#endif
    auto halo_store = [&]() {
#pragma unroll
      for (int q = 0; q < kHB; ++q) {
        if (mm[q] < 0) continue;
        const double di = dext[mm[q]];
        double r = rv[q];
        if (di != 0.0) r = fma(-al, fma(be, sv[q], wv[q]), r);
        u_ext[mm[q]] = di * r;
      }
    };
    // own: p, s, x, r and u = D^-1 r
    for (int o = tid; o < (TILE_SKIP(32) ? 0 : no); o += nt) {
      const int ly = o / owx, lx = o - ly * owx;
      const int ei = (ly + offy) * W + lx + offx;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int od = o * NC + c;
        const double di = dext[ei * NC + c];
        const double p = fma(be, ps[od], u_ext[ei * NC + c]);
        const double s = fma(be, ss[od], ws[od]);
        ps[od] = p;
        ss[od] = s;
        double r = rs[od];
        if (di != 0.0) {
          xs[od] = fma(al, p, xs[od]);
          r = fma(-al, s, r);
        }
        rs[od] = r;
        u_ext[ei * NC + c] = di * r;
      }
    }
    if (tid >= 32 && !TILE_SKIP(4)) {
      halo_store();
      for (int base = kHB * hnt; base < halo; base += kHB * hnt) {
        halo_load(base);
        halo_store();
      }
    }
    __syncthreads();
    // own: w = A u; partials; publish the boundary ring of (r, w, s)
    double* pw = pubr[par ^ 1];
    double acc3[3] = {0.0, 0.0, 0.0};
    for (int o = tid; o < no; o += nt) {
      const int ly = o / owx, lx = o - ly * owx, x = ox0 + lx, y = oy0 + ly;
      const int ei = (ly + offy) * W + lx + offx;
      double out[NC];
      if (TILE_SKIP(2)) {
        for (int c = 0; c < NC; ++c) out[c] = u_ext[ei * NC + c];
      } else {
        node_apply(x, y, ei, out);
      }
      const bool ring = lx == 0 || lx == owx - 1 || ly == 0 || ly == owy - 1;
      const int64_t d = ((int64_t)y * nnx + x) * NC;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int od = o * NC + c;
        const double u = u_ext[ei * NC + c];
        ws[od] = out[c];
        acc3[0] = fma(rs[od], u, acc3[0]);
        acc3[1] = fma(out[c], u, acc3[1]);
        acc3[2] = fma(rs[od], rs[od], acc3[2]);
        if (ring) {
          pw[d + c] = rs[od];
          pw[ND + d + c] = out[c];
          pw[2 * ND + d + c] = ss[od];
        }
      }
    }
    if constexpr (PAT) {
      publish_partials_grid_sync<3>(acc3, a.part + (par ^ 1) * 3 * nbk, a.bar, TILE_SKIP(1));
    } else {
      if (!TILE_SKIP(64)) block_sum<3>(acc3);
      if (tid == 0) {
        double* pp = a.part + (par ^ 1) * 3 * nbk;
        pp[blockIdx.x] = acc3[0];
        pp[nbk + blockIdx.x] = acc3[1];
        pp[2 * nbk + blockIdx.x] = acc3[2];
      }
      if (!TILE_SKIP(1)) grid_sync_flip(a.bar);
    }
    par ^= 1;
  }
  for (int o = tid; o < no; o += nt) {
    const int ly = o / owx, lx = o - ly * owx;
    const int64_t d = ((int64_t)(oy0 + ly) * nnx + ox0 + lx) * NC;
#pragma unroll
    for (int c = 0; c < NC; ++c) a.x[d + c] = xs[o * NC + c];
  }
  if (blockIdx.x == 0 && tid == 0) {
    a.st->rr = rr;
    a.st->iters = it;
    a.st->done = done;
  }
}

// Register-resident variant (tiles of at most NS * kCgcgThreads nodes).  Shared-memory
// bandwidth was the next bound: with x, r, p, s, w and D^-1 in shared memory, every dof cost
// ~26 64-bit shared accesses per iteration (~1.4 us per SM at cfg 2).  Here thread t owns tile
// nodes o = t + k * blockDim (k < NS) for the whole solve and keeps their x, r, p, s, w, u in
// registers; shared memory holds only the stencil inputs (u over the extended tile, alpha) and
// D^-1.  Same arithmetic in the same order as k_pcg2d_tile.
template <int NC, bool SCALED, bool PAT, int NS, int NT>
__global__ void __launch_bounds__(NT, 1) k_pcg2d_treg(Grid g, Mat<4 * NC> K, Q4Pat kp,
                                                               const double* __restrict__ alpha, CgcgArgs a,
                                                               TileSpec ts) {
  extern __shared__ double sm[];
  __shared__ __align__(16) Mat<4 * NC> Ks;
  __shared__ double bc[2][3];
  const int tid = threadIdx.x, nt = blockDim.x, nbk = gridDim.x;
  const int nnx = g.nnx, nny = g.nny;
  const int64_t ND = (int64_t)NC * g.n_nodes;
  const int bx = blockIdx.x % ts.tx, by = blockIdx.x / ts.tx;
  const int ox0 = bx * ts.tw, ox1 = min(nnx, ox0 + ts.tw);
  const int oy0 = by * ts.th, oy1 = min(nny, oy0 + ts.th);
  const int owx = max(0, ox1 - ox0), owy = max(0, oy1 - oy0), no = owx * owy;
  const int ex0 = max(ox0 - 1, 0), ex1 = min(ox1 + 1, nnx), ey0 = max(oy0 - 1, 0), ey1 = min(oy1 + 1, nny);
  const int W = max(0, ex1 - ex0), H = max(0, ey1 - ey0), ne_ext = W * H;
  const int ax0 = max(ox0 - 1, 0), ax1 = min(ox1, g.nx), ay0 = max(oy0 - 1, 0), ay1 = min(oy1, g.ny);
  const int AW = max(0, ax1 - ax0), AH = max(0, ay1 - ay0);
  double* u_ext = sm;                          // [H][W][NC]
  double* dext = u_ext + (size_t)ne_ext * NC;  // D^-1 over the extended tile
  double* as = dext + (size_t)ne_ext * NC;     // alpha [AH][AW]
  double* xs = as + (size_t)AW * AH;           // own x [NS][nt][NC] (read + written once per iteration)
  const int offx = ox0 - ex0, offy = oy0 - ey0;
  if (!PAT)
    for (int o = tid; o < 16 * NC * NC; o += nt) Ks.v[o] = K.v[o];
  for (int q = tid; q < AW * AH; q += nt) {
    const int ey = ay0 + q / AW, exx = ax0 + q % AW;
    as[q] = SCALED ? alpha[(int64_t)ey * g.nx + exx] : 1.0;
  }
  for (int q = tid; q < ne_ext * NC; q += nt) {
    const int node = q / NC, c = q % NC;
    const int y = ey0 + node / W, x = ex0 + node % W;
    const int64_t d = ((int64_t)y * nnx + x) * NC + c;
    dext[q] = a.dinv[d];
    u_ext[q] = a.dinv[d] * a.r0[d];
  }
  // per-thread nodes and their state
  int sx[NS], sy[NS], sei[NS];
  bool has[NS], ring[NS];
  double rv_[NS][NC], pv[NS][NC], sv_[NS][NC], wv_[NS][NC], uv[NS][NC];
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    const int o = tid + k * nt;
    has[k] = o < no;
    const int ly = has[k] ? o / owx : 0, lx = has[k] ? o - ly * owx : 0;
    sx[k] = ox0 + lx;
    sy[k] = oy0 + ly;
    sei[k] = (ly + offy) * W + lx + offx;
    ring[k] = lx == 0 || lx == owx - 1 || ly == 0 || ly == owy - 1;
    const int64_t d = ((int64_t)sy[k] * nnx + sx[k]) * NC;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      xs[(k * nt + tid) * NC + c] = has[k] ? a.x[d + c] : 0.0;
      rv_[k][c] = has[k] ? a.r0[d + c] : 0.0;
      uv[k][c] = has[k] ? a.dinv[d + c] * a.r0[d + c] : 0.0;
      pv[k][c] = 0.0;
      sv_[k][c] = 0.0;
      wv_[k][c] = 0.0;
    }
  }
  __syncthreads();

  auto node_apply = [&](int x, int y, int ei, double (&out)[NC]) {
    double P[9][NC];
    double sc[4];
    if (x > 0 && x < nnx - 1 && y > 0 && y < nny - 1) {
      const double* u0 = u_ext + (ei - W - 1) * NC;
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx)
#pragma unroll
          for (int c = 0; c < NC; ++c) P[dy * 3 + dx][c] = u0[(dy * W + dx) * NC + c];
      const double* a0 = as + ((y - 1 - ay0) * AW + x - 1 - ax0);
      sc[0] = a0[0];
      sc[1] = a0[1];
      sc[2] = a0[AW];
      sc[3] = a0[AW + 1];
    } else {
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const int ii = x + dx - 1, jj = y + dy - 1;
          const bool ok = ii >= 0 && ii < nnx && jj >= 0 && jj < nny;
          const int m = (jj - ey0) * W + ii - ex0;
#pragma unroll
          for (int c = 0; c < NC; ++c) P[dy * 3 + dx][c] = ok ? u_ext[m * NC + c] : 0.0;
        }
#pragma unroll
      for (int sl = 0; sl < 4; ++sl) {
        const int ei_ = x - 1 + (sl & 1), ej = y - 1 + (sl >> 1);
        const bool ok = ei_ >= 0 && ei_ < g.nx && ej >= 0 && ej < g.ny;
        sc[sl] = ok ? as[(ej - ay0) * AW + ei_ - ax0] : 0.0;
      }
    }
    if (PAT)
      node_rows_pat<NC>(kp, P, sc, out);
    else
      node_rows<2, NC>(Ks, P, sc, out);
  };
  // w = A u for own nodes, the three dot partials, publication of the boundary ring
  auto apply_dots_publish = [&](double* pw, double (&acc)[3]) {
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      if (!has[k]) continue;
      double out[NC];
      node_apply(sx[k], sy[k], sei[k], out);
      const int64_t d = ((int64_t)sy[k] * nnx + sx[k]) * NC;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        wv_[k][c] = out[c];
        acc[0] = fma(rv_[k][c], uv[k][c], acc[0]);
        acc[1] = fma(out[c], uv[k][c], acc[1]);
        acc[2] = fma(rv_[k][c], rv_[k][c], acc[2]);
        if (ring[k]) {
          pw[d + c] = rv_[k][c];
          pw[ND + d + c] = out[c];
          pw[2 * ND + d + c] = sv_[k][c];
        }
      }
    }
  };

  {
    double acc[3] = {0.0, 0.0, 0.0};
    apply_dots_publish(a.pub, acc);
    publish_partials_grid_sync<3>(acc, a.part, a.bar);  // partials parity-buffered (see cgcg2d.cuh)
  }

  double gam = 0.0, al = 0.0, be = 0.0, rr = 0.0;
  int it = a.st->iters, done = 0;
  const int maxit = a.st->maxit;
  const double tol2 = a.st->tol2;
  int par = 0;
  const int nb_b = (ey0 < oy0) ? W : 0, nb_t = (ey1 > oy1) ? W : 0;
  const int nb_l = (ex0 < ox0) ? owy : 0, nb_r = (ex1 > ox1) ? owy : 0;
  const int halo = (nb_b + nb_t + nb_l + nb_r) * NC;
  (void)nb_r;
  constexpr int kHB = 1;
  const int ht = tid - 32, hnt = nt - 32;
  auto ring_xy = [&](int t, int& x, int& y) {
    if (t < nb_b) { x = ex0 + t; y = ey0; return; }
    t -= nb_b;
    if (t < nb_t) { x = ex0 + t; y = ey1 - 1; return; }
    t -= nb_t;
    if (t < nb_l) { x = ex0; y = oy0 + t; return; }
    t -= nb_l;
    x = ex1 - 1;
    y = oy0 + t;
  };
  for (bool first = true;; first = false) {
    const double* pr = a.pub + par * 3 * ND;
    double hr[kHB], hw[kHB], hs[kHB];
    int mm[kHB];
    auto halo_load = [&](int base) {
#pragma unroll
      for (int q = 0; q < kHB; ++q) {
        const int e = base + ht + q * hnt;
        mm[q] = -1;
        if (ht >= 0 && e < halo) {
          int x, y;
          ring_xy(e / NC, x, y);
          const int c = e % NC;
          const int64_t m = ((int64_t)y * nnx + x) * NC + c;
          mm[q] = ((y - ey0) * W + x - ex0) * NC + c;
          hr[q] = __ldcg(pr + m);
          hw[q] = __ldcg(pr + ND + m);
          hs[q] = __ldcg(pr + 2 * ND + m);
        }
      }
    };
    if (tid >= 32 && !TILE_SKIP(4)) halo_load(0);
    if (tid < 32 && !TILE_SKIP(16)) {
      constexpr int kPB = 8;  // up to 256 CTAs
      double v[3][kPB];
#pragma unroll
      for (int q = 0; q < kPB; ++q) {
        const int b = tid + 32 * q;
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c][q] = (b < nbk) ? __ldcg(a.part + (par * 3 + c) * nbk + b) : 0.0;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < kPB; ++q) s += v[c][q];
        s = warp_sum(s);
        if (tid == 0) bc[par][c] = s;
      }
    }
    __syncthreads();
    const double gnew = bc[par][0], dnew = bc[par][1];
    rr = bc[par][2];
#if defined(TB_CGCG_ABL)
    if (a.dbg & 8) {
      if (!first && ++it >= maxit) {
        done = 2;
        break;
      }
      be = first ? 0.0 : 0.5;
      al = 0.5;
      gam = 1.0;
      goto treg_continue;
    }
#endif
    if (!isfinite(gnew) || !isfinite(dnew) || !isfinite(rr)) {
      done = 3;
      break;
    }
    if (!first) {
      ++it;
      if (rr <= tol2) {
        done = 1;
        break;
      }
      if (it >= maxit) {
        done = 2;
        break;
      }
    } else if (rr == 0.0 || rr <= tol2) {
      done = 1;
      break;
    }
    if (first) {
      be = 0.0;
      if (!(dnew > 0.0)) {
        done = 3;
        break;
      }
      al = gnew / dnew;
    } else {
      be = gnew / gam;
      const double pap = dnew - be * gnew / al;
      if (!(pap > 0.0)) {
        done = 3;
        break;
      }
      al = gnew / pap;
    }
    gam = gnew;
#if defined(TB_CGCG_ABL)
  treg_continue:
#endif
    // own: p, s, x, r, u in registers; u also to shared memory for the stencils
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      if (!has[k] || TILE_SKIP(32)) continue;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double di = dext[sei[k] * NC + c];
        pv[k][c] = fma(be, pv[k][c], uv[k][c]);
        sv_[k][c] = fma(be, sv_[k][c], wv_[k][c]);
        double r = rv_[k][c];
        if (di != 0.0) {
          double* xp = xs + (k * nt + tid) * NC + c;
          *xp = fma(al, pv[k][c], *xp);
          r = fma(-al, sv_[k][c], r);
        }
        rv_[k][c] = r;
        uv[k][c] = di * r;
        u_ext[sei[k] * NC + c] = uv[k][c];
      }
    }
    if (tid >= 32 && !TILE_SKIP(4)) {
      auto halo_store = [&]() {
#pragma unroll
        for (int q = 0; q < kHB; ++q) {
          if (mm[q] < 0) continue;
          const double di = dext[mm[q]];
          double r = hr[q];
          if (di != 0.0) r = fma(-al, fma(be, hs[q], hw[q]), r);
          u_ext[mm[q]] = di * r;
        }
      };
      halo_store();
      for (int base = kHB * hnt; base < halo; base += kHB * hnt) {
        halo_load(base);
        halo_store();
      }
    }
    __syncthreads();
    double acc3[3] = {0.0, 0.0, 0.0};
    if (!TILE_SKIP(2)) apply_dots_publish(a.pub + (par ^ 1) * 3 * ND, acc3);
    publish_partials_grid_sync<3>(acc3, a.part + (par ^ 1) * 3 * nbk, a.bar, TILE_SKIP(1));
    par ^= 1;
  }
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    if (!has[k]) continue;
    const int64_t d = ((int64_t)sy[k] * nnx + sx[k]) * NC;
#pragma unroll
    for (int c = 0; c < NC; ++c) a.x[d + c] = xs[(k * nt + tid) * NC + c];
  }
  if (blockIdx.x == 0 && tid == 0) {
    a.st->rr = rr;
    a.st->iters = it;
    a.st->done = done;
  }
}

#ifndef TB_TREG_NT
#define TB_TREG_NT 512
#endif
#ifndef TB_TREG_NS
#define TB_TREG_NS 2
#endif
constexpr int kTregThreads = TB_TREG_NT;  // threads per CTA of the register-resident kernel
constexpr int kTregSlots = TB_TREG_NS;    // nodes per thread

inline size_t treg_smem_bytes(int NC, const TileSpec& ts) {
  const size_t ext = (size_t)(ts.tw + 2) * (ts.th + 2);
  return sizeof(double) * (2 * ext * NC + (size_t)(ts.tw + 1) * (ts.th + 1) +
                           (size_t)kTregSlots * kTregThreads * NC);
}

inline size_t tile_smem_bytes(int NC, const TileSpec& ts) {
  const size_t ext = (size_t)(ts.tw + 2) * (ts.th + 2), own = (size_t)ts.tw * ts.th;
  return sizeof(double) * (2 * ext * NC + 5 * own * NC + (size_t)(ts.tw + 1) * (ts.th + 1));
}

// tiles for at most `ctas` CTAs: smallest per-CTA node count, then smallest perimeter
inline TileSpec choose_tiles(int nnx, int nny, int ctas) {
  TileSpec best{1, 1, nnx, nny, 0};
  double best_cost = 1e300;
  for (int ty = 1; ty <= ctas && ty <= nny; ++ty) {
    const int tx0 = ctas / ty;
    if (tx0 < 1) break;
    const int tw = (nnx + tx0 - 1) / tx0, th = (nny + ty - 1) / ty;
    const int tx = (nnx + tw - 1) / tw, tyr = (nny + th - 1) / th;
    const double cost = (double)tw * th + 2.0 * (tw + th);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = TileSpec{tx, tyr, tw, th, 0};
    }
  }
  return best;
}

}  // namespace tb
