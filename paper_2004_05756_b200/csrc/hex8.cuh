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

#ifndef TB_HEX8_HY
#define TB_HEX8_HY 8
#endif
constexpr int kHX = 32, kHY = TB_HEX8_HY;   // element tile per plane (one element per thread)
constexpr int kHT = kHX * kHY;              // 256 threads
constexpr int kHexCtas = 512 / kHT;         // resident CTAs per SM (128 registers per thread)
#ifndef TB_HEX8_UNROLL
#define TB_HEX8_UNROLL 2
#endif
constexpr int kHex8Unroll = TB_HEX8_UNROLL;  // z-sweep unrolled by 2: no loop-carried register moves (apply 50.4 -> 48.9 us at cfg3)
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

// Shared/global tile geometry.  A node-plane tile is kPY rows of kPX nodes; with the dof
// layout 3 n + c each row is kRow = 3 kPX contiguous doubles in global memory, so a plane is
// fetched as kPY coalesced row segments and kept in shared memory in the same (AoS) order.
constexpr int kRow = 3 * kPX;                          // 99 doubles per node row
constexpr int kPlane = kRow * kPY;                     // 891 doubles per node plane
constexpr int kSlots = (kPlane + kHT - 1) / kHT;       // 4 fetch slots per thread
constexpr int kORow = 3 * kOX;                         // 93 owned doubles per row
constexpr int kOPlane = kORow * kOY;                   // 651 owned doubles per plane
constexpr int kOSlots = (kOPlane + kHT - 1) / kHT;     // 3 store slots per thread

// FUSED: in = z, in2 = p_old, out = q, writes pnew, reduces p.q (pCG kernel A).
// !FUSED: in = v, out = y = K v.  Dirichlet rows: when `zoff` is given, CTA b zeroes
// out[zidx[zoff[b] .. zoff[b+1])] (the fixed dofs it owns, bucketed per CTA at plan creation)
// after its last flush.  Mask bytes read inside the sweep cost registers (spills) and ~8 us.
// SIMP (!FUSED only, p = 3): `alpha` holds rho; alpha = rho_l + (1 - rho_l) rho^3 is formed per
// element as it is loaded (same operation order as k_material), saving the material pass.
// EPI (!FUSED only): epilogue on the owned nodes instead of out = K in (multigrid level 0, mg.cu):
//   1: out = in + omega * ed * (eb - K in)   (damped-Jacobi sweep, ed = D^-1 with 0 on fixed dofs)
//   2: out = ed != 0 ? eb - K in : 0          (masked residual)
// eb / ed of the node plane gathered next travel by cp.async into the (otherwise unused) p_old
// staging area one step ahead; `in` at the node is read from the staged plane.  This saves the
// separate update kernel's pass over 5 (3) vectors per smoothing sweep (residual).
template <bool FUSED, bool SIMP = false, int EPI = 0>
__global__ void __launch_bounds__(kHT, kHexCtas) k_hex8(Grid g, Hex8Iso K, const double* __restrict__ alpha,
                                                 const double* __restrict__ in, const double* __restrict__ in2,
                                                 double* __restrict__ pnew, double* __restrict__ out,
                                                 PcgState* st, double* partials,
                                                 int zchunk, double rho_l = 0.0, double p_simp = 3.0,
                                                 const int64_t* __restrict__ zidx = nullptr,
                                                 const int* __restrict__ zoff = nullptr,
                                                 int64_t col_stride = 0, int zblocks = 0,
                                                 const double* __restrict__ eb = nullptr,
                                                 const double* __restrict__ ed = nullptr, double omega = 0.0) {
  static_assert(EPI == 0 || !FUSED, "the epilogue modes belong to the plain operator");
  // plane[4][kPlane]: node planes (buffer = plane index mod 4), AoS rows as in global memory.
  // stage[2][2][3][kHT]: node-plane corner outputs (oy) already summed over the two
  // x-neighbour elements, double buffered by step parity.  ostg[2][kOPlane]: finished owned
  // node values of a plane, stored to global memory (coalesced) one step later; pstg[2][kPlane]:
  // p_old staging (FUSED).  With 4 plane
  // buffers and 2 stage/output buffers a step needs ONE barrier.
  extern __shared__ double hsm[];
  double* plane = hsm;
  double (*stage2)[2][3][kHT] = reinterpret_cast<double (*)[2][3][kHT]>(hsm + 4 * kPlane);
  double* ostg = hsm + 4 * kPlane + 2 * 2 * 3 * kHT;
  double beta = 0.0;
  if (FUSED) {
    if (st->done) return;
    beta = st->beta;
  }
  const int t = threadIdx.x;
  const int i0 = blockIdx.x * kOX, j0 = blockIdx.y * kOY;
  // several columns in one launch (ROM, !FUSED): blockIdx.z = column * zblocks + z-chunk
  int zb = (int)blockIdx.z;
  if (!FUSED && zblocks > 0) {
    const int col = (int)blockIdx.z / zblocks;
    zb = (int)blockIdx.z - col * zblocks;
    in += col * col_stride;
    out += col * col_stride;
  }
  const int K0 = zb * zchunk;
  const int K1 = min(g.nnz, K0 + zchunk);
  const int ex = t % kHX, ey = t / kHX;                   // element in the tile (ex == lane)
  const int gei = i0 - 1 + ex, gej = j0 - 1 + ey;         // global element column
  const bool col_ok = gei >= 0 && gei < g.nx && gej >= 0 && gej < g.ny;
  const bool own = t < kOX * kOY;
  const int onx = t % kOX, ony = t / kOX;                 // owned node in the tile
  const int px = onx + 1, py = ony + 1;                   // its position in the plane tile
  const int plane_dofs = 3 * g.nnx * g.nny;               // < 2^31 for every supported grid
  // fetch slots: flat tile index f = t + s kHT -> (row f / kRow, double f % kRow)
  int goff[kSlots];
  unsigned fok = 0, fown = 0;                              // slot valid / slot is an owned node
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    const int f = t + s * kHT, ly = f / kRow, d = f % kRow, lx = d / 3;
    const int ni = i0 - 1 + lx, nj = j0 - 1 + ly;
    goff[s] = 3 * (nj * g.nnx + ni) + d % 3;
    if (f < kPlane && ni >= 0 && ni < g.nnx && nj >= 0 && nj < g.nny) {
      fok |= 1u << s;
      if (lx >= 1 && lx <= kOX && ly >= 1 && ly <= kOY) fown |= 1u << s;
    }
  }
  // store slots: flat owned index o = t + s kHT -> (row o / kORow, double o % kORow)
  int ooff[kOSlots];
  unsigned ook = 0;
#pragma unroll
  for (int s = 0; s < kOSlots; ++s) {
    const int o = t + s * kHT, r = o / kORow, d = o % kORow;
    const int ni = i0 + d / 3, nj = j0 + r;
    ooff[s] = 3 * (nj * g.nnx + ni) + d % 3;
    if (o < kOPlane && ni < g.nnx && nj < g.nny) ook |= 1u << s;
  }

  // Node planes move global -> shared with cp.async (no register staging): plane kp goes to
  // plane buffer pbuf(kp); in FUSED mode p_old goes to pstg and, once landed, each thread turns
  // its own slots into p = z + beta p_old in place (and writes owned p to pnew).
#define HEX8_ISSUE(kp_, boff_, pst_)                                                                        \
  {                                                                                                         \
    const bool zok = (kp_) >= 0 && (kp_) < g.nnz;                                                           \
    const double* src = in + (int64_t)(zok ? (kp_) : 0) * plane_dofs;                                       \
    const double* src2 = FUSED ? in2 + (int64_t)(zok ? (kp_) : 0) * plane_dofs : nullptr;                   \
    double* dst = plane + (boff_);                                                                          \
    _Pragma("unroll") for (int s = 0; s < kSlots; ++s) {                                                    \
      if (s < kSlots - 1 || t < kPlane - (kSlots - 1) * kHT) {                                              \
        const bool ok = zok && (fok >> s & 1u);                                                             \
        const int off = ok ? goff[s] : 0;                                                                   \
        cp_async8(dst + t + s * kHT, src + off, ok);                                                        \
        if (FUSED) cp_async8((pst_) + t + s * kHT, src2 + off, ok);                                         \
      }                                                                                                     \
    }                                                                                                       \
    cp_async_commit();                                                                                      \
  }
#define HEX8_LAND(kp_, boff_, pst_)                                                                         \
  if (FUSED) {                                                                                              \
    double* dst = plane + (boff_);                                                                          \
    const bool pown = (kp_) >= K0 && (kp_) < K1;                                                            \
    double* pdst = pnew + (int64_t)(kp_) * plane_dofs;                                                      \
    _Pragma("unroll") for (int s = 0; s < kSlots; ++s) {                                                    \
      if (s < kSlots - 1 || t < kPlane - (kSlots - 1) * kHT) {                                              \
        const int f = t + s * kHT;                                                                          \
        const double v = fma(beta, (pst_)[f], dst[f]);                                                      \
        dst[f] = v;                                                                                         \
        if (pown && (fown >> s & 1u)) pdst[goff[s]] = v;                                                    \
      }                                                                                                     \
    }                                                                                                       \
  }
#define HEX8_FACE(boff_, f_)                                                                                \
  _Pragma("unroll") for (int cc = 0; cc < 4; ++cc) {                                                        \
    const double* src = plane + (boff_) + (ey + (cc >> 1)) * kRow + 3 * (ex + (cc & 1));                    \
    _Pragma("unroll") for (int c = 0; c < 3; ++c) f_[c][cc] = src[c];                                       \
  }                                                                                                         \
  _Pragma("unroll") for (int c = 0; c < 3; ++c) wht4(f_[c]);
  // coalesced store of the finished owned plane kp_ (staged in ostg[(kp_) & 1])
#define HEX8_FLUSH(kp_, par_)                                                                               \
  {                                                                                                         \
    const double* srcs = ostg + (par_) * kOPlane;                                                           \
    double* dst = out + (int64_t)(kp_) * plane_dofs;                                                        \
    _Pragma("unroll") for (int s = 0; s < kOSlots; ++s) {                                                   \
      if ((s < kOSlots - 1 || t < kOPlane - (kOSlots - 1) * kHT) && (ook >> s & 1u)) {                      \
        dst[ooff[s]] = srcs[t + s * kHT];                                                                   \
      }                                                                                                     \
    }                                                                                                       \
  }

  // Ring buffers are indexed by the plane's position relative to the first plane of this CTA
  // (K0 - 1).
  double* pstg = ostg + 2 * kOPlane;  // [2][kPlane] p_old staging (FUSED)
  // EPI: eb, ed of this thread's owned node on the plane gathered next: estg[2][3][kHT] in pstg
  double* estg = pstg;
  static_assert(2 * 3 * kHT <= 2 * kPlane, "epilogue staging must fit the p_old staging area");
  const bool own_in = own && i0 + onx < g.nnx && j0 + ony < g.nny;
  const int gnode = 3 * ((j0 + ony) * g.nnx + (i0 + onx));
  auto epi_issue = [&](int kp) {  // own group: the plane issue that may follow commits its own
    if (EPI != 0) {
      if (own) {
        const bool ok = own_in && kp >= K0 && kp < K1;
        const int64_t off = ok ? (int64_t)kp * plane_dofs + gnode : 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          cp_async8(estg + c * kHT + t, eb + off + c, ok);
          cp_async8(estg + (3 + c) * kHT + t, ed + off + c, ok);
        }
      }
      cp_async_commit();
    }
  };
#define HEX8_PB(rel_) (((rel_) & 3) * kPlane)
#define HEX8_PS(rel_) (pstg + ((rel_) & 1) * kPlane)
  HEX8_ISSUE(K0 - 1, HEX8_PB(0), HEX8_PS(0));
  HEX8_ISSUE(K0, HEX8_PB(1), HEX8_PS(1));
  // p_old of plane K0+1 is staged in the (still unused) buffer of plane K0+2
  HEX8_ISSUE(K0 + 1, HEX8_PB(2), plane + HEX8_PB(3));
  epi_issue(K0);
  cp_async_wait<0>();
  HEX8_LAND(K0 - 1, HEX8_PB(0), HEX8_PS(0));
  HEX8_LAND(K0, HEX8_PB(1), HEX8_PS(1));
  HEX8_LAND(K0 + 1, HEX8_PB(2), plane + HEX8_PB(3));
  const double* a_ptr = alpha + ((int64_t)gej * g.nx + gei);  // element column base (valid iff col_ok)
  const int64_t a_stride = (int64_t)g.nx * g.ny;
  (void)p_simp;  // SIMP launches are p = 3 only (host checks), the BASELINE exponent
  auto simp = [&](double r) { return SIMP ? rho_l + (1.0 - rho_l) * ((r * r) * r) : r; };
  // the element's alpha (or rho, SIMP) is loaded one step ahead and used raw; SIMP turns it into
  // alpha only in the step that consumes it, so the load latency hides behind a whole step
  bool a_ok = col_ok && K0 - 1 >= 0;
  double a_next = a_ok ? __ldg(a_ptr + (K0 - 1) * a_stride) : 0.0;
  __syncthreads();
  // xy-WHT of the 4 corner nodes of the current bottom face of this element column
  double fb[3][4];
  HEX8_FACE(HEX8_PB(0), fb);
  double tc[3][4];  // top-face spectrum of the previous element (its share of node plane ez)
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int s = 0; s < 4; ++s) tc[c][s] = 0.0;
  double acc[1] = {0.0};
  const bool dot_any = FUSED && st->dot_k1 > st->dot_k0;
  const int dk0 = FUSED ? st->dot_k0 : 0, dk1 = FUSED ? st->dot_k1 : 0;
  const int steps = K1 - (K0 - 1);  // element planes ez = K0-1 .. K1-1
  // (a 4-way unrolled sweep makes the ring offsets constants but spills and runs slower)
#pragma unroll kHex8Unroll
  for (int rel = 0; rel < steps; ++rel) {
    {
      const int r = rel & 3;
      const int ez = K0 - 1 + rel;
      const double a_raw = a_next;
      const bool a_cur = a_ok;
      a_ok = col_ok && ez + 1 < g.nz && ez + 1 < K1;
      a_next = a_ok ? __ldg(a_ptr + (ez + 1) * a_stride) : 0.0;
      // ---- element (gei, gej, ez): spectrum from carried bottom face + new top face ----
      {
        double ft[3][4];
        HEX8_FACE(HEX8_PB(r + 1), ft);
        double u[3][8];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            u[c][s] = fb[c][s] + ft[c][s];
            u[c][s + 4] = fb[c][s] - ft[c][s];
            fb[c][s] = ft[c][s];  // this top face is the next element's bottom face
          }
        hex8_iso_blocks(K, SIMP ? (a_cur ? simp(a_raw) : 0.0) : a_raw, u);
        // inverse z stage: bottom-face spectrum joins the previous element's top-face spectrum
        // (both land on node plane ez), so the xy inverse runs once per node plane
        double fq[3][4];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            fq[c][s] = tc[c][s] + (u[c][s] + u[c][s + 4]);
            tc[c][s] = u[c][s] - u[c][s + 4];
          }
          if (FUSED) {
            wht4(fq[c]);  // -> corner values (ox + 2 oy) of node plane ez from this element column
          } else {
            // x stage only: sums feed corner ox = 0, differences ox = 1 (y stage after the combine)
            const double s0 = fq[c][0] + fq[c][1], d0 = fq[c][0] - fq[c][1];
            const double s1 = fq[c][2] + fq[c][3], d1 = fq[c][2] - fq[c][3];
            fq[c][0] = s0;
            fq[c][1] = d0;
            fq[c][2] = s1;
            fq[c][3] = d1;
          }
        }
        // node column ex+1 of this row = corner ox=1 of this element + ox=0 of the next (lane
        // 31's value is never read: node column 32 of the tile is not owned).  Non-fused: the y
        // stage is linear, so the x-stage outputs are combined first and the y stage runs once
        // on the sums (P + Q, P - Q): 6 fewer DADD per element; in the fused pCG kernel the
        // longer dependency chain measured slower (127.9 vs 125.7 us/iteration at cfg 3).
        if (FUSED) {
#pragma unroll
          for (int oy = 0; oy < 2; ++oy)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const double right = __shfl_down_sync(0xffffffffu, fq[c][2 * oy], 1);
              stage2[r & 1][oy][c][t] = fq[c][2 * oy + 1] + right;
            }
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double pp = fq[c][1] + __shfl_down_sync(0xffffffffu, fq[c][0], 1);
            const double qq = fq[c][3] + __shfl_down_sync(0xffffffffu, fq[c][2], 1);
            stage2[r & 1][0][c][t] = pp + qq;
            stage2[r & 1][1][c][t] = pp - qq;
          }
        }
      }
      // node plane ez+2 (issued at the end of the last step; the prologue landed plane K0+1)
      // must have landed before the barrier: it is read from the next step on
      if (rel >= 1 && ez + 2 <= K1) {
        cp_async_wait<0>();
        HEX8_LAND(ez + 2, HEX8_PB(r + 2), HEX8_PS(r + 2));
      } else if (EPI != 0) {
        cp_async_wait<0>();  // this step's eb, ed
      }
      __syncthreads();
      if (rel >= 2) HEX8_FLUSH(ez - 1, (r + 1) & 1);  // plane ez-1 was staged before this barrier
      // ---- owned node (px, py) of plane ez: rows ey = py-1 (corner oy=1) and ey = py (oy=0) ----
      if (own && rel >= 1) {
        const int e_dn = (py - 1) * kHX + (px - 1), e_up = py * kHX + (px - 1);
        double* o = ostg + (r & 1) * kOPlane + ony * kORow + 3 * onx;
        const double* pp = plane + HEX8_PB(r) + py * kRow + 3 * px;
        const bool dot_here = dot_any && ez >= dk0 && ez < dk1;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double v = stage2[r & 1][1][c][e_dn] + stage2[r & 1][0][c][e_up];
          if (FUSED && dot_here) acc[0] = fma(pp[c], v, acc[0]);  // p is 0 outside the grid
          if (EPI == 1) v = pp[c] + omega * estg[(3 + c) * kHT + t] * (estg[c * kHT + t] - v);
          if (EPI == 2) v = (estg[(3 + c) * kHT + t] != 0.0) ? estg[c * kHT + t] - v : 0.0;
          o[c] = v;
        }
      }
      // plane ez+3 reuses the buffer of plane ez-1, which every thread finished with before
      // this step's barrier
      epi_issue(ez + 1);  // after this step's gather has read the staging slots (same thread)
      if (ez + 3 <= K1) HEX8_ISSUE(ez + 3, HEX8_PB(r + 3), HEX8_PS(r + 3));
    }
  }
  __syncthreads();
  if (steps >= 2) HEX8_FLUSH(K1 - 1, (steps - 1) & 1);
  if (!FUSED && zoff != nullptr) {  // Dirichlet rows this CTA owns, after its own flushes
    __syncthreads();
    const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    for (int i = zoff[b] + t; i < zoff[b + 1]; i += kHT) out[zidx[i]] = 0.0;
  }
#undef HEX8_ISSUE
#undef HEX8_LAND
#undef HEX8_FACE
#undef HEX8_FLUSH
#undef HEX8_PB
#undef HEX8_PS
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

constexpr size_t kHex8Smem = sizeof(double) * (4 * kPlane + 2 * 2 * 3 * kHT + 2 * kOPlane + 2 * kPlane);

// z-chunk: as few chunks per xy column as possible (each chunk recomputes one element plane
// and refetches two node planes) while filling the resident CTA slots in whole waves.
inline int hex8_zchunk(const Grid& g) {
  const int64_t xy = (int64_t)((g.nnx + kOX - 1) / kOX) * ((g.nny + kOY - 1) / kOY);
  const int64_t slots = (int64_t)kHexCtas * 148;
  double best = 1e30;
  int best_zc = g.nnz;
  for (int64_t c = 1; c <= 64 && c <= g.nnz; ++c) {
    const int zc = (int)((g.nnz + c - 1) / c);
    const int64_t ctas = xy * ((g.nnz + zc - 1) / zc);
    const int64_t waves = (ctas + slots - 1) / slots;
    // cost ~ waves x per-CTA work (zc owned planes + ~1.5 planes of chunk overhead)
    const double cost = (double)waves * (zc + 1.5);
    if (cost < best - 1e-9) {
      best = cost;
      best_zc = zc;
    }
  }
  return best_zc;
}

// z-chunk for ncol columns in one launch (blockIdx.z = column * chunks + chunk): the waves are
// shared by all columns, so long chunks (little recomputation) pack as well as short ones.
inline int hex8_zchunk_cols(const Grid& g, int ncol) {
  const int64_t xy = (int64_t)((g.nnx + kOX - 1) / kOX) * ((g.nny + kOY - 1) / kOY);
  const int64_t slots = (int64_t)kHexCtas * 148;
  double best = 1e30;
  int best_zc = g.nnz;
  for (int64_t c = 1; c <= 64 && c <= g.nnz; ++c) {
    const int zc = (int)((g.nnz + c - 1) / c);
    const int64_t chunks = (g.nnz + zc - 1) / zc;
    if (chunks * ncol > 65535) continue;
    const int64_t ctas = xy * chunks * ncol;
    const double waves = (double)((ctas + slots - 1) / slots);
    const double cost = waves * (zc + 1.5);
    if (cost < best - 1e-9) {
      best = cost;
      best_zc = zc;
    }
  }
  return best_zc;
}

inline dim3 hex8_grid(const Grid& g, int zchunk) {
  return dim3((g.nnx + kOX - 1) / kOX, (g.nny + kOY - 1) / kOY, (g.nnz + zchunk - 1) / zchunk);
}

// CTA of k_hex8's grid that owns (flushes) dof d
inline int64_t hex8_owner(const Grid& g, int zchunk, int64_t d) {
  const int64_t n = d / 3, i = n % g.nnx, j = (n / g.nnx) % g.nny, k = n / ((int64_t)g.nnx * g.nny);
  const dim3 gr = hex8_grid(g, zchunk);
  return i / kOX + (int64_t)gr.x * (j / kOY + (int64_t)gr.y * (k / zchunk));
}

}  // namespace tb
