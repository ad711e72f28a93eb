// Element-centric Hex8 SIMP operator (3D), z-sweep with shared-memory node planes.
//
// The unit-density Hex8 stiffness of a cube is invariant under the reflections of the cube,
// so a per-component Walsh-Hadamard transform H over the 8 corners block-diagonalises it:
// K_e = H M H with M = 8 blocks of 3x3 (character k couples (component c, frequency k^e_c)).
// One element costs 2 x 72 add/sub (forward + inverse WHT) + 72 FMA (blocks) + 24 MUL
// (alpha) = ~240 FP64 instructions instead of 576 FMA for the dense 24x24 product, which
// brings the 3D operator to the HBM/FP64 ridge.
//
// Data movement: a CTA owns a 31 x 7 column of nodes and sweeps it along z.  Each step stages
// one node plane (+1 halo ring) of the input in shared memory (SoA per component), computes
// the 32 x 8 elements of one element plane (one per thread), stages their 8 x 3 corner
// outputs, and every owned node sums its 4 bottom-corner contributions plus the 4 top-corner
// contributions carried in registers from the previous plane: deterministic, atomic-free.
#pragma once

#include "q1.cuh"

namespace tb {

struct Hex8Blocks {
  double m[8][9];  // M_k (3x3 row-major), H K H / 64
};

constexpr int kHX = 32, kHY = 8;            // element tile per plane (one element per thread)
constexpr int kHT = kHX * kHY;              // 256 threads
constexpr int kPX = kHX + 1, kPY = kHY + 1;  // node-plane tile incl. halo ring
constexpr int kPN = kPX * kPY;
constexpr int kOX = kHX - 1, kOY = kHY - 1;  // owned nodes per plane (31 x 7)

__device__ __forceinline__ void wht8(double (&v)[8]) {
#pragma unroll
  for (int bit = 1; bit < 8; bit <<= 1)
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (!(t & bit)) {
        const double a = v[t], b = v[t | bit];
        v[t] = a + b;
        v[t | bit] = a - b;
      }
}

// y (corner-ordered, 8 x 3) = alpha * K_e u  via  H M H
__device__ __forceinline__ void hex8_element(const Hex8Blocks& B, double alpha, double (&u)[3][8],
                                             double (&y)[3][8]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) wht8(u[c]);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double v0 = u[0][k ^ 1], v1 = u[1][k ^ 2], v2 = u[2][k ^ 4];
    const double* m = B.m[k];
    y[0][k ^ 1] = alpha * fma(m[0], v0, fma(m[1], v1, m[2] * v2));
    y[1][k ^ 2] = alpha * fma(m[3], v0, fma(m[4], v1, m[5] * v2));
    y[2][k ^ 4] = alpha * fma(m[6], v0, fma(m[7], v1, m[8] * v2));
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) wht8(y[c]);
}

// FUSED: in = z, in2 = p_old, out = q, writes pnew, reduces p.q (pCG kernel A).
// !FUSED: in = v, out = y = K v (fixed rows zeroed when `fixed` != nullptr).
template <bool FUSED>
__global__ void __launch_bounds__(kHT) k_hex8(Grid g, Hex8Blocks B, const double* __restrict__ alpha,
                                              const double* __restrict__ in, const double* __restrict__ in2,
                                              double* __restrict__ pnew, double* __restrict__ out,
                                              const uint8_t* __restrict__ fixed, PcgState* st, double* partials,
                                              int zchunk) {
  extern __shared__ double hsm[];  // plane[2][3][kPN] then stage[8][3][kHT]
  double (*plane)[3][kPN] = reinterpret_cast<double (*)[3][kPN]>(hsm);
  double (*stage)[3][kHT] = reinterpret_cast<double (*)[3][kHT]>(hsm + 2 * 3 * kPN);
  double beta = 0.0;
  if (FUSED) {
    if (st->done) return;
    beta = st->beta;
  }
  const int t = threadIdx.x;
  const int i0 = blockIdx.x * kOX, j0 = blockIdx.y * kOY;
  const int K0 = blockIdx.z * zchunk;
  const int K1 = min(g.nnz, K0 + zchunk);
  const int ex = t % kHX, ey = t / kHX;                   // element in the tile
  const int gei = i0 - 1 + ex, gej = j0 - 1 + ey;         // global element column
  const bool own = t < kOX * kOY;
  const int onx = t % kOX, ony = t / kOX;                 // owned node in the tile
  const int gni = i0 + onx, gnj = j0 + ony;
  const bool own_ok = own && gni < g.nnx && gnj < g.nny;
  const int px = onx + 1, py = ony + 1;                   // its position in the plane tile
  const int64_t plane_stride = (int64_t)g.nnx * g.nny;

  auto load_plane = [&](int kp, int buf) {
    for (int idx = t; idx < kPN; idx += kHT) {
      const int lx = idx % kPX, ly = idx / kPX;
      const int ni = i0 - 1 + lx, nj = j0 - 1 + ly;
      const bool ok = kp >= 0 && kp < g.nnz && ni >= 0 && ni < g.nnx && nj >= 0 && nj < g.nny;
      const int64_t node = (int64_t)kp * plane_stride + (int64_t)nj * g.nnx + ni;
      const bool owned = FUSED && ok && kp >= K0 && kp < K1 && lx >= 1 && lx <= kOX && ly >= 1 && ly <= kOY;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double v = 0.0;
        if (ok) {
          v = __ldg(in + 3 * node + c);
          if (FUSED) v = fma(beta, __ldg(in2 + 3 * node + c), v);
        }
        plane[buf][c][idx] = v;
        if (owned) pnew[3 * node + c] = v;
      }
    }
  };

  int lo = 0;
  load_plane(K0 - 1, lo);
  load_plane(K0, lo ^ 1);
  double carry[3] = {0.0, 0.0, 0.0};
  double acc[1] = {0.0};
  for (int ez = K0 - 1; ez < K1; ++ez) {
    __syncthreads();
    // ---- element (gei, gej, ez) ----
    {
      const bool ok = gei >= 0 && gei < g.nx && gej >= 0 && gej < g.ny && ez >= 0 && ez < g.nz;
      double u[3][8], y[3][8];
      const double a = ok ? __ldg(alpha + ((int64_t)ez * g.ny + gej) * g.nx + gei) : 0.0;
#pragma unroll
      for (int tc = 0; tc < 8; ++tc) {
        const int b = (tc >> 2) ? lo ^ 1 : lo;
        const int idx = (ey + ((tc >> 1) & 1)) * kPX + ex + (tc & 1);
#pragma unroll
        for (int c = 0; c < 3; ++c) u[c][tc] = plane[b][c][idx];
      }
      hex8_element(B, a, u, y);
#pragma unroll
      for (int tc = 0; tc < 8; ++tc)
#pragma unroll
        for (int c = 0; c < 3; ++c) stage[tc][c][t] = y[c][tc];
    }
    __syncthreads();
    // ---- owned node: finalize plane ez (bottom corners now + top corners carried) ----
    if (own) {
      double bot[3], top[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) bot[c] = top[c] = 0.0;
#pragma unroll
      for (int s = 0; s < 4; ++s) {  // elements (px-1+sx, py-1+sy) of the tile
        const int sx = s & 1, sy = s >> 1;
        const int et = (py - 1 + sy) * kHX + (px - 1 + sx);
        const int corner = (1 - sx) + 2 * (1 - sy);  // this node's corner in that element (z = 0)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          bot[c] += stage[corner][c][et];
          top[c] += stage[corner + 4][c][et];
        }
      }
      if (ez >= K0 && own_ok) {
        const int64_t node = (int64_t)ez * plane_stride + (int64_t)gnj * g.nnx + gni;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double v = carry[c] + bot[c];
          if (FUSED) {
            acc[0] = fma(plane[lo][c][py * kPX + px], v, acc[0]);
          } else if (fixed != nullptr && fixed[3 * node + c]) {
            v = 0.0;
          }
          out[3 * node + c] = v;
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) carry[c] = top[c];
    }
    __syncthreads();
    if (ez + 2 <= K1) load_plane(ez + 2, lo);  // next element plane needs node plane ez+2
    lo ^= 1;
  }
  if (FUSED) {
    block_sum<1>(acc);
    if (publish_partials<1>(acc, partials, &st->count_a)) {
      gather_partials<1>(acc, partials, &st->count_a);
      if (threadIdx.x == 0) {
        const double v = acc[0];
        if (!(v > 0.0) || !isfinite(v)) {
          st->done = 3;
        } else {
          st->pq = v;
          st->alpha = st->rz / v;
        }
      }
    }
  }
}

constexpr size_t kHex8Smem = sizeof(double) * (2 * 3 * kPN + 8 * 3 * kHT);

// z-chunk giving ~6 CTAs per SM of work (3 resident) without much plane-halo redundancy
inline int hex8_zchunk(const Grid& g) {
  const int64_t xy = (int64_t)((g.nnx + kOX - 1) / kOX) * ((g.nny + kOY - 1) / kOY);
  int64_t chunks = (148 * 6 + xy - 1) / xy;
  if (chunks < 1) chunks = 1;
  int zc = (int)((g.nnz + chunks - 1) / chunks);
  return zc < 4 ? 4 : (zc > 64 ? 64 : zc);
}

inline dim3 hex8_grid(const Grid& g, int zchunk) {
  return dim3((g.nnx + kOX - 1) / kOX, (g.nny + kOY - 1) / kOY, (g.nnz + zchunk - 1) / zchunk);
}

}  // namespace tb
