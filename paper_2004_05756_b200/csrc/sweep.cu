// 3D Jacobi-pCG in ONE z-sweep per iteration (Chronopoulos-Gear single-reduction CG), with
// TMA node-plane staging.  Replaces, for Hex8 plans, the two-kernel iteration of pcg.cu
// (k_hex8<true> + k_pcg_update: 12 N_u + N_e doubles and two grid-wide reductions).
//
// Recurrences (Chronopoulos & Gear; u = D^-1 r, w = A u):
//   p_i = u_i + b_i p_{i-1}       s_i = w_i + b_i s_{i-1}        (s = A p)
//   x_{i+1} = x_i + a_i p_i       r_{i+1} = r_i - a_i s_i
//   u_{i+1} = D^-1 r_{i+1}        w_{i+1} = A u_{i+1}
//   g = (r, u), d = (w, u):  b_{i+1} = g_{i+1}/g_i,  a_{i+1} = g_{i+1} / (d_{i+1} - b_{i+1} g_{i+1}/a_i)
// One sweep does all of it: when node plane k lands in shared memory (TMA, one instruction per
// array, two planes in flight per CTA), every thread updates its slots pointwise (s, r, then
// u = D^-1 r into the operator's plane ring; x, p and the stores on owned slots), then the
// element-centric WHT-block Hex8 operator of hex8.cuh runs on the u planes and its owned outputs
// are w.  The halo ring and the two ghost planes of u are recomputed from r, s, w, D^-1 (bitwise
// identical to the owner's).  Per iteration: read x r p s w + D^-1 (one double per node) +
// alpha, write x r p s w: ~10.3 N_u + N_e doubles and ONE reduction of (g, r.r, d) (the textbook
// iteration is 9 N_u + N_e over two sweeps and two reductions; the two-kernel path moved 12 N_u).
//
// Lagged x: x is needed only at the exit, so every other sweep (parity 0, kModeCgLag) leaves
// x alone and records its alpha in st->alpha_lag; the next sweep (parity 1) reads p_i and forms
// x_{i+2} = fma(a_{i+1}, p_{i+1}, fma(a_i, p_i, x_i)) -- the same operations, in the same order,
// as two consecutive updates, so the iterates are bitwise those of the unlagged form.  A solve
// that stops after a lagging sweep applies the pending update once (k_sweep_xfix).  This takes
// the x read and write out of half the sweeps: ~9.3 instead of ~10.3 N_u doubles per iteration.
//
// Layout: the solver's vectors are PITCHED: dof (i, j, k, c) at (k nny + j) P + 3 i + c with the
// row pitch P >= 3 nnx a multiple of 4 doubles, so the tensor-map strides are legal (3 nnx is odd
// for every BASELINE grid).  b comes in and x goes out in the reference's compact layout
// (conversion kernels below, once per solve).
//
// r, s and w are read at halo nodes (neighbour CTAs, ghost planes of the z-chunks) while their
// owners write the next iterate, so they are double-buffered by iteration parity q: a sweep reads
// set q and writes set 1 - q.  x and p are read and written by their owner only (in place).
//
// Jacobi: for the isotropic Hex8 element every diagonal entry of K_e is the same k_d, so
// D_n = k_d sum_{e at n} alpha_e is one value per NODE; it is stored as 1/D_n with the node's
// three Dirichlet flags in the three lowest mantissa bits (a relative perturbation < 1e-15 of a
// preconditioner, which changes nothing CG relies on).  Fixed dofs get u = 0 and s = r = 0, so
// w's fixed rows (never masked) are never read: the solve is the reference's Z K Z system
// (fem.py:291-294, 378-382).
#include <cuda.h>
#include <stdlib.h>

#include "plan.cuh"

namespace tb {

namespace {

constexpr int kTRow = 100;                              // node-plane tile row: 3 x 33 doubles + 1 (16 B multiple)
constexpr int kTRows = kPY;                             // 9 node rows
constexpr int kTPlane = kTRow * kTRows;                 // 900 doubles
constexpr int kTPlaneS = (kTPlane + 15) / 16 * 16;      // smem stride: 128-byte multiple (912)
constexpr int kTORow = 94;                              // owned tile row: 3 x 31 + 1
constexpr int kTOPlane = kTORow * kOY;                  // 658
constexpr int kTOPlaneS = (kTOPlane + 15) / 16 * 16;    // 672
constexpr int kTNRow = 34;                              // per-node D^-1 tile row: 33 nodes + 1
constexpr int kTNPlane = kTNRow * kTRows;               // 306
constexpr int kTNPlaneS = (kTNPlane + 15) / 16 * 16;    // 320
// one staged plane: r, s, w (halo tiles), D^-1 (node tile), x, p (owned tiles)
constexpr int kStage = 3 * kTPlaneS + kTNPlaneS + 2 * kTOPlaneS;   // 4400 doubles
constexpr uint32_t kHaloBytes = sizeof(double) * kTPlane;
constexpr uint32_t kNodeBytes = sizeof(double) * kTNPlane;
constexpr uint32_t kOwnBytes = sizeof(double) * kTOPlane;
constexpr int kSmemDoubles = 2 * kStage + 3 * kTPlaneS + 2 * 3 * kHT + 3 * kHT + kHT;  // + LAND slot table
constexpr size_t kSweepSmem = sizeof(double) * kSmemDoubles + 2 * sizeof(uint64_t) + 128;  // + mbarriers + align

enum { kModeCg = 0, kModeApply = 1, kModeCgLag = 2 };

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA: 3D tile of a pitched vector -> shared memory, completion counted on `bar`; coordinates
// outside the tensor (negative included) are zero-filled by the hardware.  The first inner
// coordinate must be 16-byte aligned (an odd double index faults with an illegal instruction
// on B200, tools/tma_probe.cu), so callers round tile starts down and shift their indices.
__device__ __forceinline__ void tma_load3(double* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// Stores of the new iterate carry an L2 evict_last policy: an iteration writes ~200 MB at cfg 3
// into a 126 MB L2 that the sweep's own reads (r, s, w of the old set: dead once read) stream
// through as well; with the hint the planes written last survive until the next, reversed sweep
// reads them first.  (evict_first on the dead loads instead evicts halo rows before the
// neighbour CTA re-reads them: 100.2 against 93.5 us per sweep.)
__device__ __forceinline__ void st_keep(double2* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

}  // namespace

// Tensor maps of one plan's pitched vectors: halo tiles [100 x 9 x 1] of r, s, w (both parity
// sets) and x (for the true-residual apply), the node tile [34 x 9 x 1] of D^-1, owned tiles
// [94 x 7 x 1] of x and p.
struct SweepMaps {
  CUtensorMap r[2], s[2], w[2], dn, xh, x, p;
};

struct SweepVecs {
  double *x, *p;
  double *r[2], *s[2], *w[2];
  double* y;       // APPLY output y = K x
  int64_t pitch;   // P (doubles per node row)
  int64_t plane;   // P nny (doubles per node plane)
};

// One Chronopoulos-Gear iteration of parity q (MODE kModeCg / kModeCgLag (x untouched, see the
// top); st->cg_init: the start sweep with a = b = 0 that forms u_0, w_0, g_0, d_0) or
// y = K(alpha) x (kModeApply, no reductions).
template <int MODE>
__global__ void __launch_bounds__(kHT, kHexCtas)
    k_hex8_cg(const __grid_constant__ SweepMaps maps, Grid g, Hex8Iso K, const double* __restrict__ alpha,
              SweepVecs V, PcgState* st, double* partials, int zchunk, int q) {
  extern __shared__ __align__(128) double sm_raw[];
  // 128-byte aligned TMA destinations; the offset is applied to the __shared__ array itself so
  // the compiler keeps shared-space (LDS/STS) accesses instead of generic ones
  double* sm = sm_raw + (((smem_u32(sm_raw) + 127u) & ~127u) - smem_u32(sm_raw)) / sizeof(double);
  double* STG = sm;                                    // [2][kStage] staged planes (APPLY: x halo tile only)
  double* U = STG + 2 * kStage;                        // [3][kTPlaneS] u node-plane ring
  double(*stage2)[3][kHT] = reinterpret_cast<double(*)[3][kHT]>(U + 3 * kTPlaneS);
  double* aring = U + 3 * kTPlaneS + 2 * 3 * kHT;      // [3][kHT] alpha of element planes ez .. ez+2
  uint32_t* lsl = reinterpret_cast<uint32_t*>(aring + 3 * kHT);  // [2][kHT] LAND slot descriptors
  uint64_t* bar = reinterpret_cast<uint64_t*>(aring + 4 * kHT);  // [2]

  constexpr bool CG = MODE != kModeApply;
  // Sweep direction.  The lagging sweeps run bottom-up, the catch-up sweeps top-down: a sweep then
  // starts on the node planes its predecessor wrote last, which are still in the 126 MB L2 (an
  // iteration writes ~200 MB at cfg 3), instead of on the ones written longest ago.  The top-down
  // sweep is the mirror image: sweep plane m is node plane K1 - m, the carried face is the
  // element's upper one, and the z stage swaps roles (same operands in every sum: node values
  // bitwise those of the bottom-up sweep; the dot products add the planes in reverse order).
  constexpr bool DOWN = MODE == kModeCg;
  uint64_t kpol;  // L2 policy of the stores (see st_keep)
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(kpol));
  double a_cg = 0.0, b_cg = 0.0, a_lag = 0.0;
  if (CG) {
    if (st->done) return;
    if (!st->cg_init) {
      a_cg = st->alpha;
      b_cg = st->beta;
      if (MODE == kModeCg) a_lag = st->alpha_lag;
    }
  }
  const int t = threadIdx.x;
  const int i0 = blockIdx.x * kOX, j0 = blockIdx.y * kOY;
  const int K0 = blockIdx.z * zchunk;
  const int K1 = min(g.nnz, K0 + zchunk);
  const int ex = t % kHX, ey = t / kHX;
  const int gei = i0 - 1 + ex, gej = j0 - 1 + ey;
  const bool col_ok = gei >= 0 && gei < g.nx && gej >= 0 && gej < g.ny;
  const bool own = t < kOX * kOY;
  const int onx = t % kOX, ony = t / kOX;
  const int px = onx + 1, py = ony + 1;
  // 16-byte aligned tile starts: the halo tile begins at dof 3 (i0 - 1) - shh, the owned tile at
  // 3 i0 - sho, the node tile at node i0 - 1 - shn; shared-memory indices carry the shifts
  const int shh = (3 * (i0 - 1)) & 1, sho = (3 * i0) & 1, shn = (i0 - 1) & 1;
  // LAND pairs: even box index f = 2h -> (row f / kTRow, tile doubles d0 = f % kTRow - shh, d0 + 1);
  // owned tile doubles [3, dlim) of rows [1, oylim] (inside the grid)
  const int dlim = min(3 * (kOX + 1), 3 * (g.nnx - (i0 - 1)));
  const int oylim = min(kOY, g.nny - j0);
  // singles pass (see land): lane l < 2 kOY of the last warp owns the unpaired owned dof at the
  // low (even l) or high (odd l) end of owned row 1 + l/2, if that row end is unpaired
  bool single = false;
  if (t >= kHT - 32 && t < kHT - 32 + 2 * kOY) {
    const int l = t - (kHT - 32), d = (l & 1) ? dlim - 1 : 3;
    const int mate = ((d - shh) & 1) ? d - 1 : d + 1;  // pairs start at tile doubles = shh (mod 2)
    single = 1 + (l >> 1) <= oylim && (mate < 3 || mate >= dlim);
  }
  const int64_t gbase = (int64_t)(j0 - 1) * V.pitch + 3 * (i0 - 1);  // pitched offset of tile (0, 0)
  // LAND slot descriptors, loop-invariant (pairs h = t and t + kHT of every plane), packed so the
  // per-plane pass does no index division: bits 0-8 h, 9-17 D^-1 tile index of the node of double
  // f = 2h plus 1, 18-19 its component, 20 owned pair, 21-24 node row ly, 25-31 tile double d0 + 1
  auto lslot = [&](int h) -> uint32_t {
    const int f = 2 * h, ly = f / kTRow, d0 = f - ly * kTRow - shh;  // tile doubles d0, d0 + 1 of row ly
    const int lx0 = (d0 + 3) / 3 - 1, c0 = d0 - 3 * lx0;               // d0 = -1 -> lx0 = -1 (unused slot)
    const bool ow = ly >= 1 && ly <= oylim && d0 >= 3 && d0 + 1 < dlim;  // owned, inside the grid
    return (uint32_t)h | (uint32_t)(ly * kTNRow + shn + lx0 + 1) << 9 | (uint32_t)c0 << 18 | (uint32_t)ow << 20 |
           (uint32_t)ly << 21 | (uint32_t)(d0 + 1) << 25;
  };
  // kept in shared memory (one LDS per pair): as two more live registers they made the sweep spill
  lsl[t] = lslot(t);
  lsl[kHT + t] = lslot(min(t + kHT, kTPlane / 2 - 1));
  const bool own_in = own && i0 + onx < g.nnx && j0 + ony < g.nny;
  const int64_t obase = (int64_t)(j0 + ony) * V.pitch + 3 * (i0 + onx);  // this thread's owned node
  if (t == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // Plane m of the sweep is node plane K0 - 1 + m; it is staged in buffer m & 1, whose barrier
  // completes once per use, so plane m waits on parity (m >> 1) & 1.
  auto issue = [&](int m) {
    if (t == 0) {
      const int kp = DOWN ? K1 - m : K0 - 1 + m;
      double* B = STG + (m & 1) * kStage;
      uint64_t* bb = bar + (m & 1);
      const int cx = 3 * (i0 - 1) - shh, cy = j0 - 1;
      if (CG) {
        mbar_expect_tx(bb, 3 * kHaloBytes + kNodeBytes + (MODE == kModeCg ? 2 : 1) * kOwnBytes);
        tma_load3(B, &maps.r[q], cx, cy, kp, bb);
        tma_load3(B + kTPlaneS, &maps.s[q], cx, cy, kp, bb);
        tma_load3(B + 2 * kTPlaneS, &maps.w[q], cx, cy, kp, bb);
        tma_load3(B + 3 * kTPlaneS, &maps.dn, i0 - 1 - shn, cy, kp, bb);
        if (MODE == kModeCg) tma_load3(B + 3 * kTPlaneS + kTNPlaneS, &maps.x, 3 * i0 - sho, j0, kp, bb);
        tma_load3(B + 3 * kTPlaneS + kTNPlaneS + kTOPlaneS, &maps.p, 3 * i0 - sho, j0, kp, bb);
      } else {
        mbar_expect_tx(bb, kHaloBytes);
        tma_load3(B, &maps.xh, cx, cy, kp, bb);
      }
    }
  };
  double acc[3] = {0.0, 0.0, 0.0};  // g = r.u, r.r (free, owned), d = w.u
  // (selects, not V.r[q ^ 1]: dynamic indexing would copy the parameter struct to local memory)
  double* rout = q ? V.r[0] : V.r[1];
  double* sout = q ? V.s[0] : V.s[1];
  // plane m landed -> u into ring slot m % 3; owned slots of owned planes: x, r, p, s out
  auto land = [&](int m) {
    mbar_wait(bar + (m & 1), (m >> 1) & 1);
    const double* B = STG + (m & 1) * kStage;
    double* ub = U + (m % 3) * kTPlaneS;
    const int kp = DOWN ? K1 - m : K0 - 1 + m;
    const bool pown = kp >= K0 && kp < K1;
    const int64_t pl = (int64_t)kp * V.plane;
    // one pair of tile doubles (f, f + 1) from its packed slot descriptor (see lslot)
    auto pair = [&](uint32_t pk) {
      const int f = 2 * (int)(pk & 511u);  // even box index: 16-byte aligned pairs in every tile
      if (MODE == kModeApply) {
        *reinterpret_cast<double2*>(ub + f) = *reinterpret_cast<const double2*>(B + f);
      } else {
        const int c0 = (int)(pk >> 18) & 3, c1 = c0 == 2 ? 0 : c0 + 1;  // components of f, f + 1
        const double* dnr = B + 3 * kTPlaneS + (int)((pk >> 9) & 511u) - 1;  // node of double f
        const double dn0 = dnr[0], dn1 = dnr[c0 == 2 ? 1 : 0];
        const bool fr0 = !((__double2loint(dn0) >> c0) & 1), fr1 = !((__double2loint(dn1) >> c1) & 1);
        const double2 r = *reinterpret_cast<const double2*>(B + f);
        const double2 so = *reinterpret_cast<const double2*>(B + kTPlaneS + f);
        const double2 w = *reinterpret_cast<const double2*>(B + 2 * kTPlaneS + f);
        // fixed dofs: r = s = 0 in every stored iterate (k_sweep_prep/restart, and this update
        // keeps them), so masking w alone gives s = r = u = 0 there -- bitwise the values of
        // masking s, r and D^-1 separately, with 8 fewer selects per pair
        const double sn0 = fma(b_cg, so.x, fr0 ? w.x : 0.0), sn1 = fma(b_cg, so.y, fr1 ? w.y : 0.0);
        const double rn0 = fma(-a_cg, sn0, r.x), rn1 = fma(-a_cg, sn1, r.y);
        const double un0 = dn0 * rn0, un1 = dn1 * rn1;
        *reinterpret_cast<double2*>(ub + f) = make_double2(un0, un1);
        // owned pairs: vector stores; the one or two unpaired owned dofs of a row go to the
        // singles pass below (93 owned doubles per row: odd)
        if (pown && ((pk >> 20) & 1u)) {
          const int ly = (int)(pk >> 21) & 15, d0 = (int)(pk >> 25) - 1;  // node row, tile double of f
          // owned-tile index and pitched offset are even: f even and sho - shh odd (see shh/sho)
          const int fo = 3 * kTPlaneS + kTNPlaneS + (ly - 1) * kTORow + (d0 - 3 + sho);
          const double2 po = *reinterpret_cast<const double2*>(B + fo + kTOPlaneS);
          const double pn0 = fma(b_cg, po.x, dn0 * r.x), pn1 = fma(b_cg, po.y, dn1 * r.y);
          const int64_t go = pl + gbase + (int64_t)ly * V.pitch + d0;
          if (MODE == kModeCg) {
            const double2 xo = *reinterpret_cast<const double2*>(B + fo);
            const double xn0 = fma(a_cg, pn0, fma(a_lag, po.x, xo.x)), xn1 = fma(a_cg, pn1, fma(a_lag, po.y, xo.y));
            st_keep(reinterpret_cast<double2*>(V.x + go), make_double2(xn0, xn1), kpol);
          }
          st_keep(reinterpret_cast<double2*>(rout + go), make_double2(rn0, rn1), kpol);
          st_keep(reinterpret_cast<double2*>(V.p + go), make_double2(pn0, pn1), kpol);
          st_keep(reinterpret_cast<double2*>(sout + go), make_double2(sn0, sn1), kpol);
          acc[0] = fma(rn0, un0, acc[0]);
          acc[1] = fma(rn0, rn0, acc[1]);
          acc[0] = fma(rn1, un1, acc[0]);
          acc[1] = fma(rn1, rn1, acc[1]);
        }
      }
    };
    pair(lsl[t]);
    if (t < kTPlane / 2 - kHT) pair(lsl[kHT + t]);
    // singles: lanes 0..13 of the last warp (one pair each above) redo the pointwise update of
    // the unpaired owned dof at the low (even lane) or high (odd lane) end of owned row 1 + l/2
    // (same inputs, bitwise the same s, r, u as the pair pass) and store it
    if (CG && pown && single) {
      // the lane index is re-read here (volatile) so the compiler does not hoist this rare
      // branch's index math out of the sweep loop: hoisted, it was spilled to local memory and
      // reloaded after every barrier (k_hex8_cg<2>: 5.8% of the stall samples)
      int tv;
      asm volatile("mov.u32 %0, %%laneid;" : "=r"(tv));
      const int l = tv, ly = 1 + (l >> 1);
      const int d = (l & 1) ? dlim - 1 : 3;
      const int f = ly * kTRow + d + shh, lx = d / 3, c = d - 3 * lx;
      const double dn = B[3 * kTPlaneS + ly * kTNRow + shn + lx];
      const bool fr = !((__double2loint(dn) >> c) & 1);
      const double r = B[f];
      const double sn = fma(b_cg, B[kTPlaneS + f], fr ? B[2 * kTPlaneS + f] : 0.0);  // as the pairs
      const double rn = fma(-a_cg, sn, r);
      const int fo = 3 * kTPlaneS + kTNPlaneS + (ly - 1) * kTORow + (d - 3 + sho);
      const double po = B[fo + kTOPlaneS];
      const double pn = fma(b_cg, po, dn * r);
      const int64_t go = pl + gbase + (int64_t)ly * V.pitch + d;
      if (MODE == kModeCg) st_keep(V.x + go, fma(a_cg, pn, fma(a_lag, po, B[fo])), kpol);
      st_keep(rout + go, rn, kpol);
      st_keep(V.p + go, pn, kpol);
      st_keep(sout + go, sn, kpol);
      acc[0] = fma(rn, dn * rn, acc[0]);
      acc[1] = fma(rn, rn, acc[1]);
    }
  };
#define SW_FACE(boff_, f_)                                                                                   \
  _Pragma("unroll") for (int cc = 0; cc < 4; ++cc) {                                                         \
    const double* src = U + (boff_) + (ey + (cc >> 1)) * kTRow + shh + 3 * (ex + (cc & 1));                  \
    _Pragma("unroll") for (int c = 0; c < 3; ++c) f_[c][cc] = src[c];                                        \
  }                                                                                                          \
  _Pragma("unroll") for (int c = 0; c < 3; ++c) wht4(f_[c]);

  // planes m = 0 .. steps (node planes K0-1 .. K1); two in flight ahead of the one landing
  const int steps = K1 - (K0 - 1);  // element planes ez = K0-1 .. K1-1  (steps >= 2)
  issue(0);
  issue(1);
  land(0);
  __syncthreads();
  issue(2);
  land(1);
  __syncthreads();
  if (steps >= 3) issue(3);
  land(2);
  __syncthreads();
  if (steps >= 4) issue(4);
  // alpha of element plane ez travels global -> shared by cp.async two steps ahead of its use
  // (a register prefetch was sunk by the compiler next to its use: one DRAM latency per step)
  const double* a_ptr = alpha + ((int64_t)gej * g.nx + gei);
  const int64_t a_stride = (int64_t)g.nx * g.ny;
  auto alpha_fetch = [&](int e, int slot) {  // element plane e (zero outside the grid / chunk)
    const bool ok = col_ok && e >= 0 && e < g.nz && e < K1 && e >= K0 - 1;
    cp_async8(aring + slot * kHT + t, ok ? a_ptr + (int64_t)e * a_stride : alpha, ok);
    cp_async_commit();
  };
  alpha_fetch(DOWN ? K1 - 1 : K0 - 1, 0);
  alpha_fetch(DOWN ? K1 - 2 : K0, 1);
  double fb[3][4];
  SW_FACE(0, fb);
  double tc[3][4];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int s = 0; s < 4; ++s) tc[c][s] = 0.0;
  double* outv = (MODE == kModeApply) ? V.y : (q ? V.w[0] : V.w[1]);
  // one step: element plane ez = K0 - 1 + rel from the carried bottom face `bot` and the top
  // face (node plane rel + 1) loaded into `top`; unrolled by two below so the faces swap roles
  // instead of being copied
  auto step = [&](int rel, const double(&bot)[3][4], double(&top)[3][4]) {
    const int ez = DOWN ? K1 - 1 - rel : K0 - 1 + rel;  // element plane between sweep planes rel, rel + 1
    const int kpo = DOWN ? K1 - rel : K0 - 1 + rel;     // node plane completed by this step (sweep plane rel)
    cp_async_wait<1>();  // this thread's alpha of plane ez (group rel) has landed
    const double a_cur = aring[(rel % 3) * kHT + t];
    alpha_fetch(DOWN ? ez - 2 : ez + 2, (rel + 2) % 3);
    {  // ---- element (gei, gej, ez): spectrum from the bottom face + top face (plane rel+1) ----
      SW_FACE(((rel + 1) % 3) * kTPlaneS, top);
      double u[3][8];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          u[c][s] = bot[c][s] + top[c][s];
          u[c][s + 4] = DOWN ? top[c][s] - bot[c][s] : bot[c][s] - top[c][s];  // lower face - upper face
        }
      hex8_iso_blocks(K, a_cur, u);
      double fq[3][4];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          // share of the completed plane (the element's lower face going up, upper going down)
          // joins the neighbour element's carried share; the other face's share is carried on
          fq[c][s] = tc[c][s] + (DOWN ? u[c][s] - u[c][s + 4] : u[c][s] + u[c][s + 4]);
          tc[c][s] = DOWN ? u[c][s] + u[c][s + 4] : u[c][s] - u[c][s + 4];
        }
        const double s0 = fq[c][0] + fq[c][1], d0 = fq[c][0] - fq[c][1];
        const double s1 = fq[c][2] + fq[c][3], d1 = fq[c][2] - fq[c][3];
        fq[c][0] = s0;
        fq[c][1] = d0;
        fq[c][2] = s1;
        fq[c][3] = d1;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double pp = fq[c][1] + __shfl_down_sync(0xffffffffu, fq[c][0], 1);
        const double qq = fq[c][3] + __shfl_down_sync(0xffffffffu, fq[c][2], 1);
        stage2[0][c][t] = pp + qq;
        stage2[1][c][t] = pp - qq;
      }
    }
    __syncthreads();
    if (own_in && rel >= 1) {  // owned node (px, py) of plane ez: w out, d = w.u
      const int e_dn = (py - 1) * kHX + (px - 1), e_up = py * kHX + (px - 1);
      const double* up = U + (rel % 3) * kTPlaneS + py * kTRow + shh + 3 * px;
      double* dst = outv + (int64_t)kpo * V.plane + obase;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double v = stage2[1][c][e_dn] + stage2[0][c][e_up];
        if (CG) acc[2] = fma(up[c], v, acc[2]);
        st_keep(dst + c, v, kpol);
      }
    }
    // plane rel + 2 (in flight for two steps) -> ring slot (rel + 2) % 3 = slot of plane rel - 1
    if (rel >= 1 && rel + 2 <= steps) land(rel + 2);
    __syncthreads();
    // its stage buffer is free again: plane rel + 4 in flight
    if (rel >= 1 && rel + 4 <= steps) issue(rel + 4);
  };
  double ft[3][4];
  int rel = 0;
#pragma unroll 1
  for (; rel + 2 <= steps; rel += 2) {
    step(rel, fb, ft);
    step(rel + 1, ft, fb);
  }
  if (rel < steps) step(rel, fb, ft);
#undef SW_FACE
  if (CG) {
    block_sum<3>(acc);
    if (publish_partials<3>(acc, partials, &st->count_a)) {
      gather_partials<3>(acc, partials, &st->count_a);
      if (threadIdx.x == 0) {
        const double gam = acc[0], rr = acc[1], del = acc[2];
        st->rr = rr;
        st->alpha_lag = (MODE == kModeCgLag) ? a_cg : 0.0;  // this sweep's x update, pending on p
        if (!isfinite(gam) || !isfinite(rr) || !isfinite(del)) {
          st->done = 3;
        } else if (st->cg_init) {
          st->cg_init = 0;
          if (rr <= st->tol2 || gam == 0.0) {
            st->done = 1;
          } else if (!(del > 0.0)) {
            st->done = 3;
          } else {
            st->rz = gam;
            st->pq = del;
            st->alpha = gam / del;
            st->beta = 0.0;
          }
        } else {
          const int it = st->iters + 1;
          st->iters = it;
          if (rr <= st->tol2) {
            st->done = 1;
          } else {
            const double beta = gam / st->rz;
            const double den = del - beta * gam / st->alpha;
            if (!(den > 0.0)) {
              st->done = 3;
            } else {
              st->beta = beta;
              st->alpha = gam / den;
              st->rz = gam;
              st->pq = del;
              if (it >= st->maxit) st->done = 2;
            }
          }
        }
      }
    }
  }
}

// pitched index of compact dof i
__device__ __forceinline__ int64_t pitched(const Grid& g, int64_t pitch, int64_t i) {
  const int64_t node = i / 3, c = i - 3 * node;
  const int64_t ni = node % g.nnx, rest = node / g.nnx;
  return rest * pitch + 3 * ni + c;
}

// Per-node Jacobi inverse with the node's Dirichlet flags in the low mantissa bits (see top).
__global__ void __launch_bounds__(kBlock) k_sweep_dinv(Grid g, double kd, const double* __restrict__ alpha,
                                                      const uint8_t* __restrict__ fixed, int64_t npitch,
                                                      double* __restrict__ dn) {
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < g.n_nodes;
       n += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(n % g.nnx);
    const int64_t rest = n / g.nnx;
    const int j = (int)(rest % g.nny), k = (int)(rest / g.nny);
    double a = 0.0;
    for (int dz = -1; dz <= 0; ++dz)
      for (int dy = -1; dy <= 0; ++dy)
        for (int dx = -1; dx <= 0; ++dx) {
          const int ei = i + dx, ej = j + dy, ek = k + dz;
          if (ei >= 0 && ei < g.nx && ej >= 0 && ej < g.ny && ek >= 0 && ek < g.nz)
            a += alpha[((int64_t)ek * g.ny + ej) * g.nx + ei];
        }
    const double dinv = 1.0 / (kd * a);
    const long long m = (fixed[3 * n] ? 1 : 0) | (fixed[3 * n + 1] ? 2 : 0) | (fixed[3 * n + 2] ? 4 : 0);
    dn[rest * npitch + i] = __longlong_as_double((__double_as_longlong(dinv) & ~7LL) | m);
  }
}

// start: r = Z b, x = p = s = w = 0 (parity set 0, which the next sweep reads);
// tol2 = rtol^2 ||Z b||^2
__global__ void __launch_bounds__(kBlock) k_sweep_prep(Grid g, int64_t n, int64_t pitch, const double* __restrict__ b,
                                                      const uint8_t* __restrict__ fixed, SweepVecs V, PcgState* st,
                                                      double* partials, double rtol, int maxit) {
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = pitched(g, pitch, i);
    const double r = fixed[i] ? 0.0 : b[i];
    V.r[0][q] = r;
    V.x[q] = 0.0;
    V.p[q] = 0.0;
    V.s[0][q] = 0.0;
    V.w[0][q] = 0.0;
    acc[0] = fma(r, r, acc[0]);
  }
  block_sum<1>(acc);
  if (publish_partials<1>(acc, partials, &st->count_c)) {
    gather_partials<1>(acc, partials, &st->count_c);
    if (threadIdx.x == 0) {
      st->bb = acc[0];
      st->rr = acc[0];
      st->tol2 = rtol * rtol * acc[0];
      st->iters = 0;
      st->maxit = maxit;
      st->alpha = st->beta = 0.0;
      st->alpha_lag = 0.0;
      st->cg_init = 1;
      st->done = (acc[0] == 0.0) ? 1 : (isfinite(acc[0]) ? 0 : 3);
    }
  }
}

// restart from the true residual: r = Z(b - y), y = K x (pitched); p = s = w = 0; converged when
// ||r||^2 <= tol2
__global__ void __launch_bounds__(kBlock) k_sweep_restart(Grid g, int64_t n, int64_t pitch, const double* __restrict__ b,
                                                         const double* __restrict__ y, const uint8_t* __restrict__ fixed,
                                                         SweepVecs V, PcgState* st, double* partials) {
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = pitched(g, pitch, i);
    const double r = fixed[i] ? 0.0 : b[i] - y[q];
    V.r[0][q] = r;
    V.p[q] = 0.0;
    V.s[0][q] = 0.0;
    V.w[0][q] = 0.0;
    acc[0] = fma(r, r, acc[0]);
  }
  block_sum<1>(acc);
  if (publish_partials<1>(acc, partials, &st->count_c)) {
    gather_partials<1>(acc, partials, &st->count_c);
    if (threadIdx.x == 0) {
      st->rr = acc[0];
      st->cg_init = 1;
      st->alpha_lag = 0.0;
      if (st->done != 3) st->done = !isfinite(acc[0]) ? 3 : (acc[0] <= st->tol2 ? 1 : 0);
    }
  }
}

// the x update a lagging sweep left pending: x += alpha_lag p (before x is read; the restart
// kernel that follows clears alpha_lag)
__global__ void __launch_bounds__(kBlock) k_sweep_xfix(Grid g, int64_t n, int64_t pitch, SweepVecs V,
                                                      const PcgState* st) {
  const double al = st->alpha_lag;
  if (al == 0.0) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = pitched(g, pitch, i);
    V.x[q] = fma(al, V.p[q], V.x[q]);
  }
}

__global__ void __launch_bounds__(kBlock) k_sweep_unpitch(Grid g, int64_t n, int64_t pitch, const double* __restrict__ xP,
                                                         double* __restrict__ x) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = xP[pitched(g, pitch, i)];
}

__global__ void k_sweep_cond(cudaGraphConditionalHandle h, const PcgState* st) {
  cudaGraphSetConditional(h, st->done == 0 ? 1u : 0u);
}

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 3D map over a pitched array: inner dimension `inner` elements, row pitch `pitch` doubles
static int encode(CUtensorMap* m, double* base, const Grid& g, int64_t inner, int64_t pitch, int bx, int by) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) {
    set_error("cuTensorMapEncodeTiled is unavailable from the driver");
    return TB_ERR_CUDA;
  }
  const cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)g.nny, (cuuint64_t)g.nnz};
  const cuuint64_t strides[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)pitch * g.nny * 8};
  const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult rc = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)rc);
    return TB_ERR_CUDA;
  }
  return TB_OK;
}

// Hex8 Jacobi solves (not distributed, no multigrid) take the sweep; TB_NO_SWEEP=1 keeps the
// two-kernel iteration of pcg.cu (A/B measurements)
bool sweep_enabled(const tb_plan_impl* P) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("TB_NO_SWEEP");
    off = (e != nullptr && e[0] != '\0' && e[0] != '0') ? 1 : 0;
  }
  return off == 0 && P->g.dim == 3 && P->hex8 && P->precond == 0 && !P->dist;
}

int64_t sweep_pitch(const Grid& g) { return ((int64_t)3 * g.nnx + 3) / 4 * 4; }
int64_t sweep_size(const Grid& g) { return sweep_pitch(g) * g.nny * g.nnz; }
static int64_t node_pitch(const Grid& g) { return ((int64_t)g.nnx + 1) / 2 * 2; }

struct SweepState {
  SweepMaps maps;
  SweepVecs vecs;
  double* dn = nullptr;                // per-node D^-1 + Dirichlet bits (pitched)
  double* w1 = nullptr;                // w[1] (w[0] reuses the plan's dinv vector)
  cudaGraphExec_t exec = nullptr;
  // in-situ iteration timing (tb_pcg_iter_time): events around every iteration-graph launch
  bool timing = false;
  cudaEvent_t tev[2] = {nullptr, nullptr};
  double t_ms = 0.0;
  int64_t t_iters = 0;
};

// The plan's PcgWork vectors are allocated with sweep_size() doubles for Hex8 plans and reused
// (pitched) here: x -> x, pa -> p, r/z -> r[0]/r[1], pb/q -> s[0]/s[1], dinv -> w[0], tmp -> y.
int sweep_init(tb_plan_impl* P) {
  if (P->sweep != nullptr) return TB_OK;
  const Grid& g = P->g;
  PcgWork& w = P->work;
  auto* S = new SweepState();
  const int64_t pitch = sweep_pitch(g);
  int rc = TB_OK;
  if (cudaMalloc(&S->w1, sizeof(double) * (size_t)sweep_size(g)) != cudaSuccess ||
      cudaMalloc(&S->dn, sizeof(double) * (size_t)(node_pitch(g) * g.nny * g.nnz)) != cudaSuccess) {
    set_error("sweep pCG: cudaMalloc failed");
    rc = TB_ERR_CUDA;
  }
  S->vecs.x = w.x;
  S->vecs.p = w.pa;
  S->vecs.r[0] = w.r;
  S->vecs.r[1] = w.z;
  S->vecs.s[0] = w.pb;
  S->vecs.s[1] = w.q;
  S->vecs.w[0] = w.dinv;
  S->vecs.w[1] = S->w1;
  S->vecs.y = w.tmp;
  S->vecs.pitch = pitch;
  S->vecs.plane = pitch * g.nny;
  const int64_t in3 = 3 * (int64_t)g.nnx;
  for (int k = 0; k < 2 && rc == TB_OK; ++k) {
    rc = encode(&S->maps.r[k], S->vecs.r[k], g, in3, pitch, kTRow, kTRows);
    if (rc == TB_OK) rc = encode(&S->maps.s[k], S->vecs.s[k], g, in3, pitch, kTRow, kTRows);
    if (rc == TB_OK) rc = encode(&S->maps.w[k], S->vecs.w[k], g, in3, pitch, kTRow, kTRows);
  }
  if (rc == TB_OK) rc = encode(&S->maps.dn, S->dn, g, g.nnx, node_pitch(g), kTNRow, kTRows);
  if (rc == TB_OK) rc = encode(&S->maps.xh, w.x, g, in3, pitch, kTRow, kTRows);
  if (rc == TB_OK) rc = encode(&S->maps.x, w.x, g, in3, pitch, kTORow, kOY);
  if (rc == TB_OK) rc = encode(&S->maps.p, w.pa, g, in3, pitch, kTORow, kOY);
  if (rc == TB_OK) {
    cudaError_t e1 = cudaFuncSetAttribute(k_hex8_cg<kModeCg>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
    cudaError_t e2 = cudaFuncSetAttribute(k_hex8_cg<kModeApply>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
    cudaError_t e3 = cudaFuncSetAttribute(k_hex8_cg<kModeCgLag>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
      set_error("k_hex8_cg shared memory attribute: %s",
                cudaGetErrorString(e1 != cudaSuccess ? e1 : (e2 != cudaSuccess ? e2 : e3)));
      rc = TB_ERR_CUDA;
    }
  }
  if (rc != TB_OK) {
    if (S->w1) cudaFree(S->w1);
    if (S->dn) cudaFree(S->dn);
    delete S;
    return rc;
  }
  P->sweep = S;
  return TB_OK;
}

void sweep_release(tb_plan_impl* P) {
  if (P->sweep == nullptr) return;
  if (P->sweep->exec) cudaGraphExecDestroy(P->sweep->exec);
  for (auto& e : P->sweep->tev)
    if (e) cudaEventDestroy(e);
  if (P->sweep->w1) cudaFree(P->sweep->w1);
  if (P->sweep->dn) cudaFree(P->sweep->dn);
  delete P->sweep;
  P->sweep = nullptr;
}

// sweep of parity q: reads r, s, w set q, writes set 1 - q (a solve starts on set 0); parity 0
// lags the x update, parity 1 catches up (see the top)
static void launch_iter(tb_plan_impl* P, int q, cudaStream_t s) {
  SweepState& S = *P->sweep;
  if (q == 0)
    k_hex8_cg<kModeCgLag><<<hex8_grid(P->g, P->zchunk), kHT, kSweepSmem, s>>>(
        S.maps, P->g, P->hiso, P->d_alpha, S.vecs, P->work.st, P->work.partA(), P->zchunk, q);
  else
    k_hex8_cg<kModeCg><<<hex8_grid(P->g, P->zchunk), kHT, kSweepSmem, s>>>(
        S.maps, P->g, P->hiso, P->d_alpha, S.vecs, P->work.st, P->work.partA(), P->zchunk, q);
}

static void launch_apply_x(tb_plan_impl* P, cudaStream_t s) {
  SweepState& S = *P->sweep;
  k_hex8_cg<kModeApply><<<hex8_grid(P->g, P->zchunk), kHT, kSweepSmem, s>>>(S.maps, P->g, P->hiso, P->d_alpha,
                                                                            S.vecs, P->work.st, P->work.partA(),
                                                                            P->zchunk, 0);
}

static int build_sweep_graph(tb_plan_impl* P) {
  SweepState& S = *P->sweep;
  cudaStream_t cs;
  TB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaGraph_t gr;
  TB_CUDA(cudaGraphCreate(&gr, 0));
  cudaGraphConditionalHandle h;
  TB_CUDA(cudaGraphConditionalHandleCreate(&h, gr, 1u, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  TB_CUDA(cudaGraphAddNode(&node, gr, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  TB_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  static_assert(kIters % 2 == 0, "the graph body must end on parity 0");
  for (int it = 0; it < kIters; ++it) launch_iter(P, it & 1, cs);
  k_sweep_cond<<<1, 1, 0, cs>>>(h, P->work.st);
  cudaGraph_t captured;
  TB_CUDA(cudaStreamEndCapture(cs, &captured));
  TB_CUDA(cudaGraphInstantiate(&S.exec, gr, 0));
  TB_CUDA(cudaGraphDestroy(gr));
  TB_CUDA(cudaStreamDestroy(cs));
  return TB_OK;
}

static bool sweep_no_graph() {
  const char* e = getenv("TB_PCG_NOGRAPH");
  return e != nullptr && e[0] != '\0' && e[0] != '0';
}

static int sweep_start(tb_plan_impl* P, const double* b, double rtol, int maxit, cudaStream_t s) {
  SweepState& S = *P->sweep;
  PcgWork& w = P->work;
  k_sweep_dinv<<<grid_for(P->g.n_nodes), kBlock, 0, s>>>(P->g, P->K3.v[0], P->d_alpha, P->d_fixed, node_pitch(P->g),
                                                          S.dn);
  k_sweep_prep<<<kUpdateBlocks, kBlock, 0, s>>>(P->g, P->n_dofs, S.vecs.pitch, b, P->d_fixed, S.vecs, w.st, w.partC(),
                                                rtol, maxit);
  launched(2);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

int pcg_solve_sweep(tb_plan_impl* P, const double* b, double* x_out, double rtol, int maxit, int* iters,
                    double* relres, cudaStream_t s) {
  double accept = 0.0;  // round-off mode (rtol < 0), as pcg_solve
  if (rtol < 0.0) {
    rtol = -rtol;
    accept = fmax(100.0 * rtol, 1e-7);
  }
  if (!(rtol > 0.0) || maxit < 1) {
    set_error("pcg: rtol must be nonzero and maxit >= 1 (got %g, %d)", rtol, maxit);
    return TB_ERR_INVALID;
  }
  TB_TRY(sweep_init(P));
  SweepState& S = *P->sweep;
  PcgWork& w = P->work;
  const bool plain = sweep_no_graph();
  if (!plain && !S.exec) TB_TRY(build_sweep_graph(P));
  TB_TRY(sweep_start(P, b, rtol, maxit, s));
  int rc = TB_OK, stalls = 0, it_before = 0;
  double best_rr = -1.0;
  for (int restart = 0;; ++restart) {
    if (plain) {
      for (;;) {
        for (int k = 0; k < kIters; ++k) launch_iter(P, k & 1, s);
        launched(kIters);
        TB_CHECK_LAUNCH();
        TB_CUDA(cudaMemcpyAsync(w.h_st, w.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
        TB_CUDA(cudaStreamSynchronize(s));
        if (w.h_st->done != 0) break;
      }
    } else {
      if (S.timing) TB_CUDA(cudaEventRecord(S.tev[0], s));
      TB_CUDA(cudaGraphLaunch(S.exec, s));
      if (S.timing) TB_CUDA(cudaEventRecord(S.tev[1], s));
    }
    // true residual at exit: y = K x, r = Z(b - y); converged if ||r|| <= rtol ||Z b||
    k_sweep_xfix<<<kUpdateBlocks, kBlock, 0, s>>>(P->g, P->n_dofs, S.vecs.pitch, S.vecs, w.st);
    launched(1);
    launch_apply_x(P, s);
    k_sweep_restart<<<kUpdateBlocks, kBlock, 0, s>>>(P->g, P->n_dofs, S.vecs.pitch, b, S.vecs.y, P->d_fixed, S.vecs,
                                                     w.st, w.partC());
    launched(2);
    TB_CHECK_LAUNCH();
    TB_CUDA(cudaMemcpyAsync(w.h_st, w.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    TB_CUDA(cudaStreamSynchronize(s));
    const PcgState& h = *w.h_st;
    if (!plain) launched((int64_t)((h.iters - it_before + kIters) / kIters) * (kIters + 1));
    if (!plain && S.timing) {  // the stream sync above has passed tev[1]
      float ms = 0.f;
      TB_CUDA(cudaEventElapsedTime(&ms, S.tev[0], S.tev[1]));
      S.t_ms += ms;
      S.t_iters += h.iters - it_before + 1;  // + the start sweep of this (re)start
    }
    it_before = h.iters;
    if (h.done == 1) break;
    if (h.done == 3) {
      set_error("pCG breakdown after %d iterations: p^T K p <= 0 or non-finite; matrix is not positive definite",
                h.iters);
      rc = TB_ERR_INDEFINITE;
      break;
    }
    if (best_rr >= 0.0 && h.rr > 0.25 * best_rr) ++stalls;
    else stalls = 0;
    if (best_rr < 0.0 || h.rr < best_rr) best_rr = h.rr;
    if (stalls >= 3 && accept > 0.0 && h.rr <= accept * accept * h.bb) break;  // round-off mode: at the floor
    if (h.iters >= maxit || stalls >= 3 || restart >= 64) {
      set_error("pCG did not reach rtol=%g in %d iterations (relative residual %.3e)", rtol, h.iters,
                sqrt(h.rr / (h.bb > 0 ? h.bb : 1.0)));
      rc = TB_ERR_NOT_CONVERGED;
      break;
    }
    // not converged on the true residual: the restart kernel left done = 0 and cg_init = 1
  }
  const PcgState& h = *w.h_st;
  if (iters) *iters = h.iters;
  if (relres) *relres = (h.bb > 0.0) ? sqrt(h.rr / h.bb) : 0.0;
  k_sweep_unpitch<<<kUpdateBlocks, kBlock, 0, s>>>(P->g, P->n_dofs, S.vecs.pitch, S.vecs.x, x_out);
  launched(1);
  TB_CHECK_LAUNCH();
  return rc;
}

int pcg_iter_time_sweep(tb_plan_impl* P, int reset, double* ms, int64_t* iters) {
  TB_TRY(sweep_init(P));
  SweepState& S = *P->sweep;
  if (reset) {
    if (!S.tev[0]) {
      TB_CUDA(cudaEventCreate(&S.tev[0]));
      TB_CUDA(cudaEventCreate(&S.tev[1]));
    }
    S.timing = true;
    S.t_ms = 0.0;
    S.t_iters = 0;
  }
  *ms = S.t_ms;
  *iters = S.t_iters;
  return TB_OK;
}

// per-launch CUDA-event time of the sweep (iterations kept live with rtol = 0)
int pcg_profile_sweep(tb_plan_impl* P, const double* b, int nrep, double* ms_iter, cudaStream_t s) {
  TB_TRY(sweep_init(P));
  PcgWork& w = P->work;
  TB_TRY(sweep_start(P, b, 0.0, 0x7fffffff, s));
  launch_iter(P, 0, s);  // start sweep
  launched(1);
  cudaEvent_t ev[2];
  for (auto& e : ev) TB_CUDA(cudaEventCreate(&e));
  double tot = 0.0;
  for (int it = 0; it < nrep; ++it) {
    cudaEventRecord(ev[0], s);
    launch_iter(P, (it + 1) & 1, s);
    cudaEventRecord(ev[1], s);
    launched(1);
    TB_CUDA(cudaEventSynchronize(ev[1]));
    float a = 0.f;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    tot += a;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  TB_CUDA(cudaMemcpy(w.h_st, w.st, sizeof(PcgState), cudaMemcpyDeviceToHost));
  if (w.h_st->done != 0) {
    set_error("profile run stopped early (state %d after %d iterations)", w.h_st->done, w.h_st->iters);
    return TB_ERR_INVALID;
  }
  *ms_iter = tot / nrep;
  return TB_OK;
}

}  // namespace tb
