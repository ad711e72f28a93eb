// Element-centric Hex8 SIMP operator (3D), z-sweep with shared-memory node planes.
//
// The unit-density Hex8 stiffness of a cube is invariant under the reflections of the cube,
// so a per-component Walsh-Hadamard transform H over the 8 corners block-diagonalises it:
// K_e = H M H with M = 8 blocks of 3x3 (character k couples (component c, frequency k^e_c)).
// For an isotropic material the 72 block entries take only 8 distinct values (a..h below);
// the block product then costs ~33 flops, the two transforms ~120 add/sub, and alpha scales
// the 8 constants once: ~190 FP64 instructions per element instead of 576 FMA for the dense
// 24x24 product.  Non-isotropic element matrices use the dense
// node-owner kernel of q1.cuh instead.
//
// Data movement: a CTA owns a 31 x 7 column of nodes and sweeps it along z.  Each step
//  * prefetches node plane ez+2 into registers (its global latency overlaps the step),
//  * computes the 32 x 8 elements of element plane ez (one per thread): only the top face
//    (plane ez+1) is read from shared memory; the bottom face's xy-transformed values are
//    carried in registers from the previous step,
//  * sums each element's corner outputs with its x-neighbour by warp shuffle (one warp = one
//    element row), stages them, and every owned node adds its two staged rows plus the top
//    contributions carried from the previous step.  Deterministic and atomic-free.
#pragma once

#include "q1.cuh"

namespace tb {

// the 8 distinct WHT-block values of an isotropic Hex8 element (H K H / 64)
struct Hex8Iso {
  double a, b, c, d, e, f, g, h;
};

constexpr int kHX = 32, kHY = 8;            // element tile per plane (one element per thread)
constexpr int kHT = kHX * kHY;              // 256 threads
constexpr int kPX = kHX + 1, kPY = kHY + 1;  // node-plane tile incl. halo ring
constexpr int kPN = kPX * kPY;
constexpr int kOX = kHX - 1, kOY = kHY - 1;  // owned nodes per plane (31 x 7)

// in-place 4-point WHT over a face (corner index ox + 2 oy)
__device__ __forceinline__ void wht4(double (&v)[4]) {
  const double a0 = v[0] + v[1], a1 = v[0] - v[1], a2 = v[2] + v[3], a3 = v[2] - v[3];
  v[0] = a0 + a2;
  v[2] = a0 - a2;
  v[1] = a1 + a3;
  v[3] = a1 - a3;
}

// Block product  u <- (alpha M) u  on the full WHT spectrum u[c][s] (s = sxy + 4 sz), in place.
__device__ __forceinline__ void hex8_iso_blocks(const Hex8Iso& K, double alpha, double (&u)[3][8]) {
  const double amb = alpha * (K.a - K.b), bb = alpha * K.b, c = alpha * K.c, d = alpha * K.d;
  const double e = alpha * K.e, f = alpha * K.f, gmh = alpha * (K.g - K.h), hh = alpha * K.h;
  // k = 0: (u0[1], u1[2], u2[4]) with [[a,b,b],[b,a,b],[b,b,a]]
  {
    const double v0 = u[0][1], v1 = u[1][2], v2 = u[2][4];
    const double s = bb * (v0 + v1 + v2);
    u[0][1] = fma(amb, v0, s);
    u[1][2] = fma(amb, v1, s);
    u[2][4] = fma(amb, v2, s);
  }
  // k = 7: (u0[6], u1[5], u2[3]) with [[g,h,h],[h,g,h],[h,h,g]]
  {
    const double v0 = u[0][6], v1 = u[1][5], v2 = u[2][3];
    const double s = hh * (v0 + v1 + v2);
    u[0][6] = fma(gmh, v0, s);
    u[1][5] = fma(gmh, v1, s);
    u[2][3] = fma(gmh, v2, s);
  }
  // k = 1: (u0[0], u1[3], u2[5]) with [[0,0,0],[0,c,d],[0,d,c]]
  {
    const double v1 = u[1][3], v2 = u[2][5];
    u[0][0] = 0.0;
    u[1][3] = fma(c, v1, d * v2);
    u[2][5] = fma(d, v1, c * v2);
  }
  // k = 2: (u0[3], u1[0], u2[6]) with [[c,0,d],[0,0,0],[d,0,c]]
  {
    const double v0 = u[0][3], v2 = u[2][6];
    u[1][0] = 0.0;
    u[0][3] = fma(c, v0, d * v2);
    u[2][6] = fma(d, v0, c * v2);
  }
  // k = 4: (u0[5], u1[6], u2[0]) with [[c,d,0],[d,c,0],[0,0,0]]
  {
    const double v0 = u[0][5], v1 = u[1][6];
    u[2][0] = 0.0;
    u[0][5] = fma(c, v0, d * v1);
    u[1][6] = fma(d, v0, c * v1);
  }
  // k = 3: (u0[2], u1[1], u2[7]) with [[e,e,0],[e,e,0],[0,0,f]]
  {
    const double s = e * (u[0][2] + u[1][1]);
    u[0][2] = s;
    u[1][1] = s;
    u[2][7] = f * u[2][7];
  }
  // k = 5: (u0[4], u1[7], u2[1]) with [[e,0,e],[0,f,0],[e,0,e]]
  {
    const double s = e * (u[0][4] + u[2][1]);
    u[0][4] = s;
    u[2][1] = s;
    u[1][7] = f * u[1][7];
  }
  // k = 6: (u0[7], u1[4], u2[2]) with [[f,0,0],[0,e,e],[0,e,e]]
  {
    const double s = e * (u[1][4] + u[2][2]);
    u[1][4] = s;
    u[2][2] = s;
    u[0][7] = f * u[0][7];
  }
}

// FUSED: in = z, in2 = p_old, out = q, writes pnew, reduces p.q (pCG kernel A).
// !FUSED: in = v, out = y = K v (fixed rows zeroed when `fixed` != nullptr).
template <bool FUSED>
__global__ void __launch_bounds__(kHT, 2) k_hex8(Grid g, Hex8Iso K, const double* __restrict__ alpha,
                                                 const double* __restrict__ in, const double* __restrict__ in2,
                                                 double* __restrict__ pnew, double* __restrict__ out,
                                                 const uint8_t* __restrict__ fixed, PcgState* st, double* partials,
                                                 int zchunk) {
  // plane[4][3][kPN]: node planes, buffer = plane index mod 4 (SoA per component).
  // stage[2][4][3][kHT]: corner outputs (q = oy + 2 oz) already summed over the two
  // x-neighbour elements, double buffered by step parity.  With 4 plane buffers and 2 stage
  // buffers a step needs ONE barrier: no thread can be more than one step ahead of another.
  extern __shared__ double hsm[];
  double (*plane)[3][kPN] = reinterpret_cast<double (*)[3][kPN]>(hsm);
  double (*stage2)[4][3][kHT] = reinterpret_cast<double (*)[4][3][kHT]>(hsm + 4 * 3 * kPN);
  double beta = 0.0;
  if (FUSED) {
    if (st->done) return;
    beta = st->beta;
  }
  const int t = threadIdx.x;
  const int i0 = blockIdx.x * kOX, j0 = blockIdx.y * kOY;
  const int K0 = blockIdx.z * zchunk;
  const int K1 = min(g.nnz, K0 + zchunk);
  const int ex = t % kHX, ey = t / kHX;                   // element in the tile (ex == lane)
  const int gei = i0 - 1 + ex, gej = j0 - 1 + ey;         // global element column
  const bool col_ok = gei >= 0 && gei < g.nx && gej >= 0 && gej < g.ny;
  const bool own = t < kOX * kOY;
  const int onx = t % kOX, ony = t / kOX;                 // owned node in the tile
  const int gni = i0 + onx, gnj = j0 + ony;
  const bool own_ok = own && gni < g.nnx && gnj < g.nny;
  const int px = onx + 1, py = ony + 1;                   // its position in the plane tile
  const int64_t plane_stride = (int64_t)g.nnx * g.nny;
  constexpr int kPF = (kPN + kHT - 1) / kHT;              // plane entries per thread (2)
  int lxs[kPF], lys[kPF];
#pragma unroll
  for (int q = 0; q < kPF; ++q) {
    lxs[q] = (t + q * kHT) % kPX;
    lys[q] = (t + q * kHT) / kPX;
  }

  double pf[kPF][3];
#define HEX8_FETCH(kp_)                                                                                     \
  _Pragma("unroll") for (int q = 0; q < kPF; ++q) {                                                         \
    const int ni = i0 - 1 + lxs[q], nj = j0 - 1 + lys[q];                                                   \
    const bool ok = (t + q * kHT) < kPN && (kp_) >= 0 && (kp_) < g.nnz && ni >= 0 && ni < g.nnx && nj >= 0 && \
                    nj < g.nny;                                                                             \
    const int64_t node = (int64_t)(kp_) * plane_stride + (int64_t)nj * g.nnx + ni;                          \
    _Pragma("unroll") for (int c = 0; c < 3; ++c) {                                                         \
      double v = 0.0;                                                                                       \
      if (ok) {                                                                                             \
        v = __ldg(in + 3 * node + c);                                                                       \
        if (FUSED) v = fma(beta, __ldg(in2 + 3 * node + c), v);                                             \
      }                                                                                                     \
      pf[q][c] = v;                                                                                         \
    }                                                                                                       \
  }
#define HEX8_STORE(kp_, buf_)                                                                               \
  _Pragma("unroll") for (int q = 0; q < kPF; ++q) {                                                         \
    const int idx = t + q * kHT;                                                                            \
    if (idx < kPN) {                                                                                        \
      _Pragma("unroll") for (int c = 0; c < 3; ++c) plane[(buf_)][c][idx] = pf[q][c];                       \
      if (FUSED && (kp_) >= K0 && (kp_) < K1 && lxs[q] >= 1 && lxs[q] <= kOX && lys[q] >= 1 &&              \
          lys[q] <= kOY) {                                                                                  \
        const int ni = i0 - 1 + lxs[q], nj = j0 - 1 + lys[q];                                               \
        if (ni < g.nnx && nj < g.nny) {                                                                     \
          const int64_t node = (int64_t)(kp_) * plane_stride + (int64_t)nj * g.nnx + ni;                    \
          _Pragma("unroll") for (int c = 0; c < 3; ++c) pnew[3 * node + c] = pf[q][c];                      \
        }                                                                                                   \
      }                                                                                                     \
    }                                                                                                       \
  }
#define HEX8_FACE(buf_, f_)                                                                                 \
  _Pragma("unroll") for (int cc = 0; cc < 4; ++cc) {                                                        \
    const int idx = (ey + (cc >> 1)) * kPX + ex + (cc & 1);                                                 \
    _Pragma("unroll") for (int c = 0; c < 3; ++c) f_[c][cc] = plane[(buf_)][c][idx];                        \
  }                                                                                                         \
  _Pragma("unroll") for (int c = 0; c < 3; ++c) wht4(f_[c]);

  auto pbuf = [](int kp) { return (kp + 4) & 3; };  // kp >= -1
  HEX8_FETCH(K0 - 1);
  HEX8_STORE(K0 - 1, pbuf(K0 - 1));
  HEX8_FETCH(K0);
  HEX8_STORE(K0, pbuf(K0));
  HEX8_FETCH(K0 + 1);  // plane of the second step, stored at the top of the first
  double a_next = (col_ok && K0 - 1 >= 0) ? __ldg(alpha + ((int64_t)(K0 - 1) * g.ny + gej) * g.nx + gei) : 0.0;
  __syncthreads();
  // xy-WHT of the 4 corner nodes of the current bottom face of this element column
  double fb[3][4];
  HEX8_FACE(pbuf(K0 - 1), fb);
  double carry[3] = {0.0, 0.0, 0.0};
  double acc[1] = {0.0};
  for (int ez = K0 - 1; ez < K1; ++ez) {
    const int sb = (ez + 1) & 1;  // stage buffer of this step
    // store node plane ez+2 (fetched last step; read from the next step on) and fetch ez+3
    if (ez + 2 <= K1) {
      HEX8_STORE(ez + 2, pbuf(ez + 2));
    }
    if (ez + 3 <= K1) {
      HEX8_FETCH(ez + 3);
    }
    const double a = a_next;
    a_next = (col_ok && ez + 1 < g.nz && ez + 1 < K1) ? __ldg(alpha + ((int64_t)(ez + 1) * g.ny + gej) * g.nx + gei)
                                                       : 0.0;
    // ---- element (gei, gej, ez): spectrum from carried bottom face + new top face ----
    {
      double ft[3][4];
      HEX8_FACE(pbuf(ez + 1), ft);
      double u[3][8];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          u[c][s] = fb[c][s] + ft[c][s];
          u[c][s + 4] = fb[c][s] - ft[c][s];
          fb[c][s] = ft[c][s];  // this top face is the next element's bottom face
        }
      hex8_iso_blocks(K, a, u);
      // inverse: z stage, then xy stage per face -> corner outputs (ox + 2 oy + 4 oz)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double bot[4], top[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          bot[s] = u[c][s] + u[c][s + 4];
          top[s] = u[c][s] - u[c][s + 4];
        }
        wht4(bot);
        wht4(top);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          u[c][s] = bot[s];
          u[c][s + 4] = top[s];
        }
      }
      // node column ex+1 of this row: corner ox=1 of this element + ox=0 of the next
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // q = oy + 2 oz
        const int base = 2 * (q & 1) + 4 * (q >> 1);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double right = __shfl_down_sync(0xffffffffu, u[c][base], 1);
          stage2[sb][q][c][t] = u[c][base + 1] + (ex < kHX - 1 ? right : 0.0);
        }
      }
    }
    __syncthreads();
    // ---- owned node (px, py): rows ey = py-1 (its corner oy=1) and ey = py (oy=0) ----
    if (own) {
      const int e_dn = (py - 1) * kHX + (px - 1), e_up = py * kHX + (px - 1);
      double bot[3], top[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        bot[c] = stage2[sb][1][c][e_dn] + stage2[sb][0][c][e_up];
        top[c] = stage2[sb][3][c][e_dn] + stage2[sb][2][c][e_up];
      }
      if (ez >= K0 && own_ok) {
        const int64_t node = (int64_t)ez * plane_stride + (int64_t)gnj * g.nnx + gni;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double v = carry[c] + bot[c];
          if (FUSED) {
            if (ez >= st->dot_k0 && ez < st->dot_k1) acc[0] = fma(plane[pbuf(ez)][c][py * kPX + px], v, acc[0]);
          } else if (fixed != nullptr && fixed[3 * node + c]) {
            v = 0.0;
          }
          out[3 * node + c] = v;
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) carry[c] = top[c];
    }
  }
#undef HEX8_FETCH
#undef HEX8_STORE
#undef HEX8_FACE
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

constexpr size_t kHex8Smem = sizeof(double) * (4 * 3 * kPN + 2 * 4 * 3 * kHT);

// z-chunk giving ~8 CTAs of work per SM (2 resident) without much plane-halo redundancy
inline int hex8_zchunk(const Grid& g) {
  const int64_t xy = (int64_t)((g.nnx + kOX - 1) / kOX) * ((g.nny + kOY - 1) / kOY);
  int64_t chunks = (148 * 8 + xy - 1) / xy;
  if (chunks < 1) chunks = 1;
  const int zc = (int)((g.nnz + chunks - 1) / chunks);
  return zc < 4 ? 4 : (zc > 64 ? 64 : zc);
}

inline dim3 hex8_grid(const Grid& g, int zchunk) {
  return dim3((g.nnx + kOX - 1) / kOX, (g.nny + kOY - 1) / kOY, (g.nnz + zchunk - 1) / zchunk);
}

}  // namespace tb
