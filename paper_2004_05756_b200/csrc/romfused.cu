// Batched reduced stiffness for Hex8 plans in ONE pass over Phi, element form on FP64 tensor
// cores (reference rom.py:254-262):
//
//   K_hat_d = sum_e alpha_{e,d} Phi_e^T K_e Phi_e          for all designs d of the batch.
//
// The isotropic Hex8 matrix is K_e = H M H (H the per-component Walsh-Hadamard transform over
// the element's corners, M = 8 blocks of 3x3; hex8.cuh).  Each PSD block factors into <= 3
// scaled rows, so K_e = G^T G with G = L^T H of rank 18 (24 - 6 rigid modes), and
//
//   Phi_e^T K_e Phi_e = C_e^T C_e,   C_e = G Phi_e   (18 x k, padded to 20 rows).
//
// S_e = C_e^T C_e is DESIGN-INDEPENDENT: it is formed once per element on DMMA (mma.sync
// m8n8k4 f64, K = 20 rows in 5 steps per 8x8 tile) and then weighted into every design's
// accumulator (16 designs x 2 FMAs per lane per tile).  Per element this is 2 * 20 * k^2
// tensor flops + 2 * nd * k^2 / 2 vector flops, against 16 k^2 * 24 (element form per design,
// PAPER.md:664) or 2 N_u k^2 / N_e (node form per design) -- the designs share the tensor work.
// Y = K Phi is never materialised and Phi is streamed once (the four CTA groups that cover
// the 36 upper 8x8 tiles of a k = 64 basis run on the same element columns, so they share it
// through L2).
//
// Layout: a CTA walks element columns (4 consecutive elements in x at one y, every z) and
// stages node planes of Phi (2 rows x 5 nodes x 3 dofs x k columns, contiguous in the
// row-major Phi) with cp.async.bulk + mbarrier, two planes ahead.  Per z step: 256 threads
// build C for the 4 elements (one (element, column) each: 3 eight-point WHTs, 18 rows), then
// each of the 12 consumer warps contracts its 8x8 tile of S for the 4 elements and accumulates it,
// alpha-weighted, for all designs.  Deterministic: fixed per-CTA element order, partials summed
// in CTA order by k_rom_fused_reduce.
#include "plan.cuh"

namespace tb {

namespace {

constexpr int kRfEB = 4;                 // elements per step (x)
constexpr int kRfNodes = kRfEB + 1;      // nodes per staged row
constexpr int kRfWarps = 12;             // one 8x8 tile of S per consumer warp (3 per SM sub-partition)
constexpr int kRfThreads = 32 * kRfWarps;
constexpr int kRfMaxK = 64;
constexpr int kRfMaxD = 16;              // designs per launch
constexpr int kRfCtasPerSm = 1;          // 162 registers per thread (16 designs x 2 accumulators live)
constexpr int kRfRows = 20;              // rows of C (18 + 2 zero)
constexpr int kRfCStride = kRfMaxK + 4;  // 68: the 4 rows of a DMMA k-step fall in distinct banks
constexpr int kRfPlane = 2 * kRfNodes * 3 * kRfMaxK;   // staged node plane (doubles), k = 64
constexpr int kRfSbStride = 68;         // per-warp S staging: element stride (bank-conflict free B reads)
constexpr int kRfSmemDoubles = 3 * kRfPlane + 2 * kRfEB * kRfRows * kRfCStride + 4 * kRfMaxD * kRfEB +
                               kRfWarps * kRfEB * kRfSbStride;
constexpr size_t kRfSmem = sizeof(double) * kRfSmemDoubles + 3 * sizeof(uint64_t) + 128;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nRFW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra RFW_%=;\n}\n" ::"r"(
          su32(bar)),
      "r"(parity)
      : "memory");
}
// 1D bulk copy global -> shared (UBLKCP); addresses and size 16-byte aligned
__device__ __forceinline__ void bulk_load(double* dst, const double* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

}  // namespace

// Row scales of the rank-18 factor G (see the top comment; hex8_blocks gives a..h).
struct RomRows {
  double q1, q2, q3;  // block (a, b): (v0+v1+v2), (v0-v1), (v0+v1-2v2)
  double q4, q5, q6;  // block (g, h): same rows
  double qp, qm;      // blocks (c, d): (v1+v2), (v1-v2)
  double qe, qf;      // blocks (e, f): (v0+v1), v2
};

// Warp-specialised: warps 0..8 (consumers) each own one 8x8 tile (I, J) of S and the
// accumulators of every design; warps 9..16 (producers) stream Phi node planes (cp.async.bulk),
// fetch alpha and build C for the next element step into the other half of a double buffer.
// Named barriers hand buffers over (FULL: producers -> consumers, EMPTY: back), so building C
// overlaps the tensor-core work instead of alternating with it.
// grid: blockIdx.x = column-chunk * ngroups + group; group -> tiles [12 group, 12 group + 12).
// KC: the basis size at compile time (64, BASELINE cfg 5) or 0 (runtime k).
constexpr int kRfCons = kRfWarps * 32;           // consumer threads
constexpr int kRfProd = kRfEB * kRfMaxK;         // producer threads: one (element, column) each
constexpr int kRfAll = kRfCons + kRfProd;        // 544
constexpr int kRfCBuf = kRfEB * kRfRows * kRfCStride;  // C of one step
constexpr int kRfAlpha = kRfMaxD * kRfEB;               // alpha of one element plane [d][el]

__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

template <int KC>
__global__ void __launch_bounds__(kRfAll, 1)
    k_rom_fused(Grid g, RomRows R, const double* __restrict__ phi, int k_rt, const double* __restrict__ alpha,
                int nd, int ngroups, int kb0, int kb1, double* __restrict__ part) {
  const int k = KC > 0 ? KC : k_rt;
  extern __shared__ __align__(128) double rf_raw[];
  double* sm = rf_raw + (((su32(rf_raw) + 127u) & ~127u) - su32(rf_raw)) / sizeof(double);
  double* PH = sm;                                        // [3][2][5][3k] node planes of Phi
  double* CB = PH + 3 * kRfPlane;                         // [2] C [EB][20][68]
  double* AR = CB + 2 * kRfCBuf;                          // [4] alpha ring [16][EB], two planes ahead
  double* SB = AR + 4 * kRfAlpha;                         // [consumer warps][EB][68] S tiles
  uint64_t* bar = reinterpret_cast<uint64_t*>(SB + kRfWarps * kRfEB * kRfSbStride);  // [3]

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int group = blockIdx.x % ngroups, chunk = blockIdx.x / ngroups, nchunks = gridDim.x / ngroups;
  const int rowd = 3 * k;                                 // doubles per node of row-major Phi
  const int nxb = (g.nx + kRfEB - 1) / kRfEB;             // element batches per x row
  const int ncols = nxb * g.ny;                           // element columns (x batch, y)
  if (t == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(bar + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // named barriers: 1, 2 FULL[buffer]; 3, 4 EMPTY[buffer]; 5 producers only
  if (warp < kRfWarps) {
    // ===================================== consumers =====================================
    const int nbk = (k + 7) / 8, ntile = nbk * (nbk + 1) / 2;
    const int tile = group * kRfWarps + warp;
    int I = 0, J = 0;
    {
      int rem = tile;
      while (I < nbk && rem >= nbk - I) {
        rem -= nbk - I;
        ++I;
      }
      J = I + rem;
    }
    const bool live = tile < ntile;
    // K_hat tile (I, J) of 16 designs as DMMA accumulators: acc[m][r] = designs 8m..8m+7 x
    // entries (8I + r, 8J + 0..7)
    double acc[2][8][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int r = 0; r < 8; ++r) acc[m][r][0] = acc[m][r][1] = 0.0;
    double* sb = SB + warp * kRfEB * kRfSbStride;
    int buf = 0, gstep = 0;
    for (int col = chunk; col < ncols; col += nchunks)
      for (int ez = 0; ez < g.nz; ++ez) {
        nb_sync(1 + buf, kRfAll);  // FULL[buf]
        const double* C = CB + buf * kRfCBuf;
        const double* al = AR + (gstep & 3) * kRfAlpha;  // [d][el]
        if (live) {
          // S tile (I, J) of each element on DMMA (K = 20 rows of C), staged in this warp's sb
#pragma unroll
          for (int el = 0; el < kRfEB; ++el) {
            const double* ce = C + el * kRfRows * kRfCStride + (lane & 3) * kRfCStride + (lane >> 2);
            double s[2] = {0.0, 0.0};
#pragma unroll
            for (int kk = 0; kk < kRfRows / 4; ++kk) {
              const double a = ce[4 * kk * kRfCStride + 8 * I];
              const double b = ce[4 * kk * kRfCStride + 8 * J];
              dmma(s, a, b);
            }
            *reinterpret_cast<double2*>(sb + el * kRfSbStride + (lane >> 2) * 8 + 2 * (lane & 3)) =
                make_double2(s[0], s[1]);  // S_e[lane/4][2(lane%4) + h]
          }
          __syncwarp();
          // K_hat[d] += sum_e alpha[d][e] S_e: ONE DMMA k-step over the 4 elements per (m, r)
          const double a0 = al[lane], a1 = al[32 + lane];  // A[m = design][k = element]
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const double b = sb[(lane & 3) * kRfSbStride + r * 8 + (lane >> 2)];  // B[k = element][n] = S_e[r][n]
            dmma(acc[0][r], a0, b);
            dmma(acc[1][r], a1, b);
          }
          __syncwarp();
        }
        nb_arrive(3 + buf, kRfAll);  // EMPTY[buf]
        buf ^= 1;
        ++gstep;
      }
    // partials: part[(chunk * ntile + tile) * nd + d][64 entries]; thread holds designs
    // 8m + lane/4, entries (r, 2(lane%4) + h)
    if (live) {
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int d = 8 * m + (lane >> 2);
        if (d < nd) {
          double* o = part + ((int64_t)(chunk * ntile + tile) * nd + d) * 64 + 2 * (lane & 3);
#pragma unroll
          for (int r = 0; r < 8; ++r) *reinterpret_cast<double2*>(o + r * 8) = make_double2(acc[m][r][0], acc[m][r][1]);
        }
      }
    }
    return;
  }
  // ====================================== producers ======================================
  const int pt = t - kRfCons;                  // 0 .. 255
  const int el = pt / kRfMaxK, c = pt % kRfMaxK;
  uint32_t phase = 0;                          // bit s: parity of ring slot s's next completion
  double fb[3][4];                             // xy-WHT of this (element, column)'s bottom face
  int buf = 0, produced = 0;
  for (int col = chunk; col < ncols; col += nchunks) {
    const int xb = col % nxb, ej = col / nxb;
    const int ei0 = xb * kRfEB;
    const int nn = min(kRfNodes, g.nnx - ei0);  // nodes of the staged rows
    const uint32_t rbytes = (uint32_t)(sizeof(double) * nn * rowd);
    // node plane m (0..nz) of this column -> slot m % 3: rows j = ej, ej + 1 of nodes ei0..
    auto issue = [&](int m) {
      if (pt == 0) {
        uint64_t* b = bar + (m % 3);
        double* dst = PH + (m % 3) * kRfPlane;
        mbar_expect_tx(b, 2 * rbytes);
#pragma unroll
        for (int oy = 0; oy < 2; ++oy) {
          const int64_t node = ((int64_t)m * g.nny + (ej + oy)) * g.nnx + ei0;
          bulk_load(dst + oy * kRfNodes * rowd, phi + node * rowd, rbytes, b);
        }
      }
    };
    auto wait_plane = [&](int m) {
      const int s = m % 3;
      mbar_wait(bar + s, (phase >> s) & 1u);
      phase ^= 1u << s;
    };
    // xy-WHT (corner ox + 2 oy -> frequency fx + 2 fy) of this thread's element face on node
    // plane m, column c, per component
    auto face = [&](int m, double (&f)[3][4]) {
      const double* pl = PH + (m % 3) * kRfPlane;
#pragma unroll
      for (int oy = 0; oy < 2; ++oy)
#pragma unroll
        for (int ox = 0; ox < 2; ++ox) {
          const int nidx = el + ox;
          const bool in = nidx < nn && c < k;
          const double* src = pl + (oy * kRfNodes + nidx) * rowd + c;
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) f[cc][ox + 2 * oy] = in ? src[cc * k] : 0.0;
        }
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) wht4(f[cc]);
    };
    // alpha of element plane e (designs x elements; the DMMA A fragment is al[lane]) -> ring
    // slot (global step) & 3; one commit group per call, empty past the top, so the group count
    // is regular.  Slot reuse: step G + 2 overwrites step G - 2, which the consumers released
    // before the producers passed EMPTY at step G (and G0 - 4, G0 - 3 at a column start).
    const int gcol0 = produced;
    auto alpha_fetch = [&](int e) {
      if (pt < kRfEB * kRfMaxD && e < g.nz) {
        const int d = pt / kRfEB, ae = pt % kRfEB;
        const int ei = ei0 + ae;
        const bool ok = d < nd && ei < g.nx && e >= kb0 && e < kb1;
        const double* src = ok ? alpha + (int64_t)d * g.n_elems + ((int64_t)e * g.ny + ej) * g.nx + ei : alpha;
        cp_async8(AR + ((gcol0 + e) & 3) * kRfAlpha + pt, src, ok);
      }
      cp_async_commit();
    };
    issue(0);
    issue(1);
    if (g.nz >= 2) issue(2);
    alpha_fetch(0);
    alpha_fetch(1);
    wait_plane(0);
    face(0, fb);
    for (int ez = 0; ez < g.nz; ++ez) {
      if (produced >= 2) nb_sync(3 + buf, kRfAll);  // EMPTY[buf]: the consumers are done with it
      double* C = CB + buf * kRfCBuf;
      alpha_fetch(ez + 2);  // two planes ahead
      wait_plane(ez + 1);
      // C of this thread's (element, column): bottom face carried, top face (plane ez + 1) new
      double ft[3][4];
      face(ez + 1, ft);
      double v[3][8];
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          v[cc][q] = fb[cc][q] + ft[cc][q];
          v[cc][q + 4] = fb[cc][q] - ft[cc][q];
          fb[cc][q] = ft[cc][q];
        }
      // blocks of hex8_iso_blocks: (v0, v1, v2) per block as there
      const double a0 = v[0][1], a1 = v[1][2], a2 = v[2][4];   // (a, b)
      const double g0 = v[0][6], g1 = v[1][5], g2 = v[2][3];   // (g, h)
      double* cp = C + el * kRfRows * kRfCStride + c;
      cp[0 * kRfCStride] = R.q1 * (a0 + a1 + a2);
      cp[1 * kRfCStride] = R.q2 * (a0 - a1);
      cp[2 * kRfCStride] = R.q3 * (a0 + a1 - 2.0 * a2);
      cp[3 * kRfCStride] = R.q4 * (g0 + g1 + g2);
      cp[4 * kRfCStride] = R.q5 * (g0 - g1);
      cp[5 * kRfCStride] = R.q6 * (g0 + g1 - 2.0 * g2);
      cp[6 * kRfCStride] = R.qp * (v[1][3] + v[2][5]);   // k = 1: (u1[3], u2[5])
      cp[7 * kRfCStride] = R.qm * (v[1][3] - v[2][5]);
      cp[8 * kRfCStride] = R.qp * (v[0][3] + v[2][6]);   // k = 2: (u0[3], u2[6])
      cp[9 * kRfCStride] = R.qm * (v[0][3] - v[2][6]);
      cp[10 * kRfCStride] = R.qp * (v[0][5] + v[1][6]);  // k = 4: (u0[5], u1[6])
      cp[11 * kRfCStride] = R.qm * (v[0][5] - v[1][6]);
      cp[12 * kRfCStride] = R.qe * (v[0][2] + v[1][1]);  // k = 3: (u0[2], u1[1]), f: u2[7]
      cp[13 * kRfCStride] = R.qf * v[2][7];
      cp[14 * kRfCStride] = R.qe * (v[0][4] + v[2][1]);  // k = 5: (u0[4], u2[1]), f: u1[7]
      cp[15 * kRfCStride] = R.qf * v[1][7];
      cp[16 * kRfCStride] = R.qe * (v[1][4] + v[2][2]);  // k = 6: (u1[4], u2[2]), f: u0[7]
      cp[17 * kRfCStride] = R.qf * v[0][7];
      cp[18 * kRfCStride] = 0.0;
      cp[19 * kRfCStride] = 0.0;
      cp_async_wait<2>();          // alpha of plane ez (two newer groups may be in flight)
      nb_arrive(1 + buf, kRfAll);  // FULL[buf]
      buf ^= 1;
      ++produced;
      nb_sync(5, kRfProd);  // every producer is done with ring slot ez % 3
      if (ez + 3 <= g.nz) issue(ez + 3);
    }
  }
}

// khat[d][8I + r][8J + c] = sum over chunks (fixed order), mirrored to the lower triangle
__global__ void k_rom_fused_reduce(int nchunks, int ntile, int nbk, int nd, int k, const double* __restrict__ part,
                                   double* __restrict__ khat) {
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (tile, d, entry)
  if (o >= (int64_t)ntile * nd * 64) return;
  const int entry = (int)(o % 64), d = (int)((o / 64) % nd), tile = (int)(o / (64 * nd));
  double s = 0.0;
  for (int c = 0; c < nchunks; ++c) s += part[((int64_t)(c * ntile + tile) * nd + d) * 64 + entry];
  int I = 0, rem = tile;
  while (rem >= nbk - I) {
    rem -= nbk - I;
    ++I;
  }
  const int J = I + rem;
  const int row = 8 * I + entry / 8, colm = 8 * J + entry % 8;
  if (row < k && colm < k) {
    double* kd = khat + (int64_t)d * k * k;
    kd[(int64_t)row * k + colm] = s;
    kd[(int64_t)colm * k + row] = s;  // I == J: the tile's own transpose writes the same sum
  }
}

bool rom_fused_rows(const Hex8Iso& h, RomRows* R) {
  const double l1 = h.a + 2 * h.b, l2 = h.a - h.b, l3 = h.g + 2 * h.h, l4 = h.g - h.h;
  const double lp = h.c + h.d, lm = h.c - h.d, le = h.e, lf = h.f;
  const double ls[8] = {l1, l2, l3, l4, lp, lm, le, lf};
  double mx = 0.0;
  for (double l : ls) mx = fmax(mx, fabs(l));
  for (double l : ls)
    if (l < -1e-12 * mx) return false;  // not positive semidefinite: no real factor
  auto sq = [](double x) { return sqrt(x > 0.0 ? x : 0.0); };
  R->q1 = sq(l1 / 3.0);
  R->q2 = sq(l2 / 2.0);
  R->q3 = sq(l2 / 6.0);
  R->q4 = sq(l3 / 3.0);
  R->q5 = sq(l4 / 2.0);
  R->q6 = sq(l4 / 6.0);
  R->qp = sq(lp / 2.0);
  R->qm = sq(lm / 2.0);
  R->qe = sq(le);
  R->qf = sq(lf);
  return true;
}

bool rom_fused_eligible(const tb_plan_impl* P, int k) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("TB_NO_ROM_FUSED");
    off = (e != nullptr && e[0] != '\0' && e[0] != '0') ? 1 : 0;
  }
  RomRows R;
  return off == 0 && P->g.dim == 3 && P->hex8 && k >= 2 && k <= kRfMaxK && (k % 2) == 0 &&
         rom_fused_rows(P->hiso, &R);
}

// K_hat for nd designs (alpha of each design precomputed, nd x N_e), element planes [kb0, kb1)
int rom_fused_khat(tb_plan_impl* P, const double* phi, int k, const double* alpha, int nd, int kb0, int kb1,
                   double* part_scratch, size_t part_bytes, double* khat, cudaStream_t s) {
  RomRows R;
  if (!rom_fused_rows(P->hiso, &R)) {
    set_error("element matrix has no real rank factor (not PSD)");
    return TB_ERR_INVALID;
  }
  static bool attr = false;
  if (!attr) {
    TB_CUDA(cudaFuncSetAttribute(k_rom_fused<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRfSmem));
    TB_CUDA(cudaFuncSetAttribute(k_rom_fused<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRfSmem));
    attr = true;
  }
  const int nbk = (k + 7) / 8, ntile = nbk * (nbk + 1) / 2;
  const int ngroups = (ntile + kRfWarps - 1) / kRfWarps;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->device);
  // one wave: every CTA resident at once (a partial second wave would double the time)
  const int nchunks = (kRfCtasPerSm * sms / ngroups) > 0 ? (kRfCtasPerSm * sms / ngroups) : 1;
  if ((size_t)nchunks * ntile * nd * 64 * sizeof(double) > part_bytes) {
    set_error("ROM fused scratch too small");
    return TB_ERR_INVALID;
  }
  for (int d0 = 0; d0 < nd; d0 += kRfMaxD) {
    const int n = nd - d0 < kRfMaxD ? nd - d0 : kRfMaxD;
    if (k == 64)
      k_rom_fused<64><<<nchunks * ngroups, kRfAll, kRfSmem, s>>>(P->g, R, phi, k, alpha + (int64_t)d0 * P->g.n_elems,
                                                                     n, ngroups, kb0, kb1, part_scratch);
    else
      k_rom_fused<0><<<nchunks * ngroups, kRfAll, kRfSmem, s>>>(P->g, R, phi, k, alpha + (int64_t)d0 * P->g.n_elems,
                                                                    n, ngroups, kb0, kb1, part_scratch);
    const int64_t outs = (int64_t)ntile * n * 64;
    k_rom_fused_reduce<<<(int)((outs + 255) / 256), 256, 0, s>>>(nchunks, ntile, nbk, n, k, part_scratch,
                                                                  khat + (int64_t)d0 * k * k);
    launched(2);
    TB_CHECK_LAUNCH();
  }
  return TB_OK;
}

size_t rom_fused_scratch_bytes(const tb_plan_impl* P, int k, int nd) {
  const int nbk = (k + 7) / 8, ntile = nbk * (nbk + 1) / 2;
  const int ngroups = (ntile + kRfWarps - 1) / kRfWarps;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->device);
  const int nchunks = (kRfCtasPerSm * sms / ngroups) > 0 ? (kRfCtasPerSm * sms / ngroups) : 1;
  return (size_t)nchunks * ntile * (nd < kRfMaxD ? nd : kRfMaxD) * 64 * sizeof(double) + 4096;
}

// executed tensor flops of one tb_rom_reduced_stiffness call on the fused path: per owned
// element and 8x8 tile, 5 DMMA (S = C_I^T C_J, K = 20) + 8 ceil(nd / 8) per 4 elements (weighting:
// one DMMA per S row and 8-design m-tile, K = the 4 elements)
double rom_fused_flops(const tb_plan_impl* P, int k, int nd) {
  const int nbk = (k + 7) / 8, ntile = nbk * (nbk + 1) / 2;
  const int kb1 = P->own_k1 < P->g.nz ? P->own_k1 : P->g.nz;
  const double ne = (double)P->g.nx * P->g.ny * (kb1 - P->own_k0);
  double per = 0.0;
  for (int d0 = 0; d0 < nd; d0 += kRfMaxD) {
    const int n = nd - d0 < kRfMaxD ? nd - d0 : kRfMaxD;
    per += 5.0 + (double)((n + 7) / 8) * 8 / kRfEB;
  }
  return ne * ntile * per * 512.0;
}

}  // namespace tb

extern "C" int tb_rom_fused_info(tb_plan* plan, int k, int nd, double* flops) {
  if (plan == nullptr || flops == nullptr) return TB_ERR_INVALID;
  auto* P = reinterpret_cast<tb::tb_plan_impl*>(plan);
  *flops = 0.0;
  if (!tb::rom_fused_eligible(P, k)) return 0;
  *flops = tb::rom_fused_flops(P, k, nd);
  return 1;
}
