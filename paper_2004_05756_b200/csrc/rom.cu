// Reduced-order-model kernels (reference rom.py:76-390).
//
// Reduced stiffness uses the node-form identity  Phi^T K(rho) Phi = Phi^T Y,  Y = K(rho) Phi
// (reference PAPER.md:444; rom.py:254-262 evaluates the same sum element by element).
// Y rows are produced by the node-owner operator over k columns; the k x k contraction
// Phi^T Y runs on the FP64 tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA) with a
// deterministic two-level reduction.
#include <string.h>

#include "plan.cuh"
#include "q1.cuh"

namespace tb {

static inline int nblk(int64_t n) { return (int)((n + kBlock - 1) / kBlock); }

// ---------------------------------------------------------------------------------------
// out[d][j] = sum_i phi[i][j] vec[d][i]     (Phi^T f, rom.py:251)
// ---------------------------------------------------------------------------------------
constexpr int kMaxVec = 16;

// NV >= nvec is the compile-time vector count (1, 2, 4, 8 or 16): with the loop over kMaxVec
// predicated at run time a single vector cost ~190 instructions per row and warp (issue-bound,
// 0.55 TB/s at cfg 5 size).  4 rows of Phi in flight per thread.
template <int NV>
__global__ void __launch_bounds__(kBlock) k_project_part(int64_t n, int k, const double* __restrict__ phi,
                                                         const double* __restrict__ vec, int nvec,
                                                         double* __restrict__ part) {
  extern __shared__ double sh[];  // [groups][nvec][k]
  const int groups = kBlock / k;
  const int t = threadIdx.x, j = t % k, rg = t / k;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * per, i1 = min(n, i0 + per);
  double acc[NV];
#pragma unroll
  for (int d = 0; d < NV; ++d) acc[d] = 0.0;
  if (rg < groups) {
    constexpr int U = 4;
    int64_t i = i0 + rg;
    for (; i + (int64_t)(U - 1) * groups < i1; i += (int64_t)U * groups) {
      double pv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) pv[u] = __ldg(phi + (i + (int64_t)u * groups) * k + j);
#pragma unroll
      for (int u = 0; u < U; ++u)  // rows in increasing order, as the rolled loop
#pragma unroll
        for (int d = 0; d < NV; ++d)
          if (NV == 1 || d < nvec) acc[d] = fma(pv[u], __ldg(vec + (int64_t)d * n + i + (int64_t)u * groups), acc[d]);
    }
    for (; i < i1; i += groups) {
      const double pv = phi[i * k + j];
#pragma unroll
      for (int d = 0; d < NV; ++d)
        if (NV == 1 || d < nvec) acc[d] = fma(pv, __ldg(vec + (int64_t)d * n + i), acc[d]);
    }
#pragma unroll
    for (int d = 0; d < NV; ++d)
      if (d < nvec) sh[(rg * nvec + d) * k + j] = acc[d];
  }
  __syncthreads();
  for (int o = t; o < nvec * k; o += blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < groups; ++g) s += sh[g * nvec * k + o];
    part[(int64_t)blockIdx.x * nvec * k + o] = s;
  }
}

// Several vectors: the NV values of a row are needed by every column thread, so a chunk of kPtR
// rows of the vectors is staged in shared memory (coalesced loads, transposed to [row][NV]) and
// read back as broadcast 16-byte loads; the per-thread global loads of the kernel above (NV per
// row and thread, the same address in all lanes) ran 16 vectors at 0.6 TB/s at cfg 5 size.
// Same partition and the same row order per thread as k_project_part: bitwise the same sums.
constexpr int kPtR = 64;
template <int NV>
__global__ void __launch_bounds__(kBlock) k_project_tile(int64_t n, int k, const double* __restrict__ phi,
                                                         const double* __restrict__ vec, int nvec,
                                                         double* __restrict__ part) {
  extern __shared__ double sh[];  // [groups][nvec][k] for the final reduction
  __shared__ __align__(16) double vt[kPtR * NV];
  const int groups = kBlock / k;
  const int t = threadIdx.x, j = t % k, rg = t / k;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * per, i1 = min(n, i0 + per);
  double acc[NV];
#pragma unroll
  for (int d = 0; d < NV; ++d) acc[d] = 0.0;
  // chunks start at multiples of `groups` rows from i0, so thread rg keeps rows i0 + rg + m groups
  const int rows_per = kPtR / groups * groups;  // >= groups: the host launches this kernel for groups <= kPtR only
  for (int64_t base = i0; base < i1; base += rows_per) {
    const int rows = (int)min((int64_t)rows_per, i1 - base);
    __syncthreads();  // the previous chunk's tile has been read
    for (int idx = t; idx < NV * rows_per; idx += kBlock) {
      const int d = idx / rows_per, r = idx - d * rows_per;
      vt[r * NV + d] = (d < nvec && r < rows) ? __ldg(vec + (int64_t)d * n + base + r) : 0.0;
    }
    __syncthreads();
    if (rg < groups) {
      constexpr int U = 4;
      int r = rg;
      for (; r + (U - 1) * groups < rows; r += U * groups) {
        double pv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) pv[u] = __ldg(phi + (base + r + u * groups) * k + j);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const double2* vr = reinterpret_cast<const double2*>(vt + (r + u * groups) * NV);
#pragma unroll
          for (int d2 = 0; d2 < NV / 2; ++d2) {
            const double2 v = vr[d2];
            acc[2 * d2] = fma(pv[u], v.x, acc[2 * d2]);
            acc[2 * d2 + 1] = fma(pv[u], v.y, acc[2 * d2 + 1]);
          }
        }
      }
      for (; r < rows; r += groups) {
        const double pv = __ldg(phi + (base + r) * k + j);
#pragma unroll
        for (int d = 0; d < NV; ++d) acc[d] = fma(pv, vt[r * NV + d], acc[d]);
      }
    }
  }
  if (rg < groups) {
#pragma unroll
    for (int d = 0; d < NV; ++d)
      if (d < nvec) sh[(rg * nvec + d) * k + j] = acc[d];
  }
  __syncthreads();
  for (int o = t; o < nvec * k; o += blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < groups; ++g) s += sh[g * nvec * k + o];
    part[(int64_t)blockIdx.x * nvec * k + o] = s;
  }
}

// out[o] = sum_b part[b][o]  (fixed order), o < len
__global__ void k_sum_parts(int nb, int len, const double* __restrict__ part, double* __restrict__ out) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= len) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[(int64_t)b * len + o];
  out[o] = s;
}

// ---------------------------------------------------------------------------------------
// Y = K(alpha) Phi  for all k columns: thread per (node, column), column fastest so the
// neighbourhood loads of a warp are contiguous rows of Phi.
// ---------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(kBlock) k_apply_cols(Grid g, Mat<Q1<D>::NN * D> K, const double* __restrict__ alpha,
                                                       const double* __restrict__ phi, int k, double* __restrict__ y) {
  constexpr int NC = D;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = t / k;
  const int col = (int)(t % k);
  if (n >= g.n_nodes) return;
  int i, j, kk;
  node_coords(g, n, i, j, kk);
  double P[Q1<D>::NB][NC];
#pragma unroll
  for (int dz = 0; dz < (D == 3 ? 3 : 1); ++dz)
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const int nb = (dz * 3 + dy) * 3 + dx;
        const int ii = i + dx - 1, jj = j + dy - 1, k3 = (D == 3) ? kk + dz - 1 : 0;
        const bool ok = ii >= 0 && ii < g.nnx && jj >= 0 && jj < g.nny && k3 >= 0 && k3 < g.nnz;
        const int64_t node = ((int64_t)k3 * g.nny + jj) * g.nnx + ii;
#pragma unroll
        for (int c = 0; c < NC; ++c) P[nb][c] = ok ? __ldg(phi + (NC * node + c) * k + col) : 0.0;
      }
  double a[Q1<D>::NN];
  slot_scales<D, true>(g, i, j, kk, alpha, a);
  double out[NC];
  node_rows<D, NC>(K, P, a, out);
#pragma unroll
  for (int c = 0; c < NC; ++c) y[(NC * n + c) * k + col] = out[c];
}

// ---------------------------------------------------------------------------------------
// C_part[block] = A^T B over a row range, A,B: n x k row-major, on DMMA (m8n8k4 f64).
// ---------------------------------------------------------------------------------------
constexpr int kRows = 32;       // rows staged per step
constexpr int kGemmThreads = 256;

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// COLMAJOR: A and B are k contiguous columns with leading dimension ld (A[c*ld + row]);
// otherwise row-major (A[row*k + c]).
template <int KP, bool COLMAJOR>
__global__ void __launch_bounds__(kGemmThreads) k_atb_dmma(int64_t n, int k, const double* __restrict__ A,
                                                           const double* __restrict__ B, double* __restrict__ part,
                                                           int64_t ld) {
  constexpr int LD = KP + 8;  // padded smem row (bank-conflict-free fragment reads)
  constexpr int TILES = (KP / 8) * (KP / 8);
  constexpr int NW = kGemmThreads / 32;
  constexpr int TPW = (TILES + NW - 1) / NW;
  __shared__ double sa[kRows * LD];
  __shared__ double sb[kRows * LD];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t per = ((n + gridDim.x - 1) / gridDim.x + kRows - 1) / kRows * kRows;
  const int64_t i0 = (int64_t)blockIdx.x * per, i1 = min(n, i0 + per);
  double acc[TPW][2];
#pragma unroll
  for (int t = 0; t < TPW; ++t) acc[t][0] = acc[t][1] = 0.0;
  for (int64_t base = i0; base < i1; base += kRows) {
    __syncthreads();
    for (int o = tid; o < kRows * KP; o += kGemmThreads) {
      const int r = COLMAJOR ? o % kRows : o / KP, c = COLMAJOR ? o / kRows : o % KP;
      const int64_t row = base + r;
      const bool ok = row < i1 && c < k;
      const int64_t at = COLMAJOR ? c * ld + row : row * k + c;
      sa[r * LD + c] = ok ? A[at] : 0.0;
      sb[r * LD + c] = ok ? B[at] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      const int tile = warp + t * NW;
      if (tile < TILES) {
        const int m0 = (tile / (KP / 8)) * 8, n0 = (tile % (KP / 8)) * 8;
#pragma unroll
        for (int r0 = 0; r0 < kRows; r0 += 4) {
          const double a = sa[(r0 + (lane & 3)) * LD + m0 + (lane >> 2)];
          const double b = sb[(r0 + (lane & 3)) * LD + n0 + (lane >> 2)];
          dmma_8x8x4(acc[t], a, b);
        }
      }
    }
  }
  // D fragment: row = lane>>2, cols = 2*(lane&3) + {0,1}
  double* out = part + (int64_t)blockIdx.x * k * k;
#pragma unroll
  for (int t = 0; t < TPW; ++t) {
    const int tile = warp + t * NW;
    if (tile < TILES) {
      const int m = (tile / (KP / 8)) * 8 + (lane >> 2);
      const int c0 = (tile % (KP / 8)) * 8 + 2 * (lane & 3);
      if (m < k && c0 < k) out[m * k + c0] = acc[t][0];
      if (m < k && c0 + 1 < k) out[m * k + c0 + 1] = acc[t][1];
    }
  }
}

// ---------------------------------------------------------------------------------------
// Column-major A^T B on DMMA with a double-buffered cp.async pipeline (3D ROM path).
// A, B: k columns with leading dimension ld; rows [r0, r1) are contracted.
// Stage = 32 rows x KP columns of both matrices in shared memory as [col][row] (+pad);
// warp w owns output row block(s) so its A fragment feeds 8 DMMAs per k-step.
// ---------------------------------------------------------------------------------------
#ifndef TB_CM_STAGES
#define TB_CM_STAGES 2
#endif
constexpr int kCmRows = 32, kCmLd = kCmRows + 4;
constexpr int kCmStages = TB_CM_STAGES;                       // cp.async ring depth
constexpr int kCmCtas = (kCmStages <= 2) ? 3 : (kCmStages == 3 ? 2 : 1);  // resident CTAs per SM (KP = 64)


// SYM: A^T B is known to be symmetric (Phi^T K Phi): only the MB(MB+1)/2 upper 8x8 tiles are
// computed and the lower triangle is mirrored on output (exactly symmetric result).
template <int KP, bool SYM, bool V16>
__global__ void __launch_bounds__(kGemmThreads) k_atb_cm(int64_t r0, int64_t r1, int k,
                                                         const double* __restrict__ A, const double* __restrict__ B,
                                                         double* __restrict__ part, int64_t ld) {
  constexpr int MB = KP / 8, TILES = SYM ? MB * (MB + 1) / 2 : MB * MB, NW = kGemmThreads / 32;
  constexpr int TPW = (TILES + NW - 1) / NW;
  constexpr int STAGE = 2 * KP * kCmLd;  // doubles per stage (A then B)
  extern __shared__ __align__(16) double smc[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = r1 - r0;
  const int64_t per = ((n + gridDim.x - 1) / gridDim.x + kCmRows - 1) / kCmRows * kCmRows;
  const int64_t i0 = r0 + (int64_t)blockIdx.x * per, i1 = min(r1, i0 + per);
  const int nstages = (int)((max(i1 - i0, (int64_t)0) + kCmRows - 1) / kCmRows);
  auto load = [&](int stg, int buf) {
    const int64_t base = i0 + (int64_t)stg * kCmRows;
    double* sbuf = smc + buf * STAGE;
    if (V16) {  // row pairs: base and ld are even, so every pair is 16-byte aligned
      for (int idx = tid; idx < KP * kCmRows; idx += kGemmThreads) {
        const int mat = idx / (KP * kCmRows / 2), rem = idx % (KP * kCmRows / 2);
        const int c = rem / (kCmRows / 2), r = 2 * (rem % (kCmRows / 2));
        const int64_t row = base + r;
        const int bytes = (c < k && row < i1) ? (row + 1 < i1 ? 16 : 8) : 0;
        const double* src = (mat ? B : A) + (bytes ? (int64_t)c * ld + row : 0);
        cp_async16(sbuf + mat * KP * kCmLd + c * kCmLd + r, src, bytes);
      }
    } else {
      for (int idx = tid; idx < 2 * KP * kCmRows; idx += kGemmThreads) {
        const int mat = idx / (KP * kCmRows), rem = idx % (KP * kCmRows);
        const int c = rem / kCmRows, r = rem % kCmRows;
        const int64_t row = base + r;
        const bool ok = c < k && row < i1;
        const double* src = (mat ? B : A) + (ok ? (int64_t)c * ld + row : 0);
        cp_async8(sbuf + mat * KP * kCmLd + c * kCmLd + r, src, ok);
      }
    }
    cp_async_commit();
  };
  double acc[TPW][2];
  int tm[TPW], tn[TPW];  // tile origin (row block, column block) of this warp's tiles
#pragma unroll
  for (int t = 0; t < TPW; ++t) {
    acc[t][0] = acc[t][1] = 0.0;
    int u = warp * TPW + t, mb = 0;
    if (SYM) {
      while (mb < MB && u >= MB - mb) u -= MB - mb++;
      tm[t] = mb * 8;
      tn[t] = (mb + u) * 8;
    } else {
      tm[t] = (u / MB) * 8;
      tn[t] = (u % MB) * 8;
    }
  }
  // ring of kCmStages buffers; stage st + kCmStages - 1 is issued while stage st is consumed
#pragma unroll
  for (int p = 0; p < kCmStages - 1; ++p) {
    if (p < nstages)
      load(p, p);
    else
      cp_async_commit();  // empty group keeps the wait count uniform
  }
  for (int st = 0; st < nstages; ++st) {
    cp_async_wait<kCmStages - 2>();
    __syncthreads();  // stage st visible to all; every warp is done with stage st-1's buffer
    {
      const int nx = st + kCmStages - 1;
      if (nx < nstages)
        load(nx, nx % kCmStages);
      else
        cp_async_commit();
    }
    const double* sa = smc + (st % kCmStages) * STAGE;
    const double* sb = sa + KP * kCmLd;
#pragma unroll
    for (int r0 = 0; r0 < kCmRows; r0 += 4) {
      const int rr = r0 + (lane & 3), cc = lane >> 2;
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        const int tile = warp * TPW + t;
        if (tile < TILES) {
          const double a = sa[(tm[t] + cc) * kCmLd + rr];
          const double b = sb[(tn[t] + cc) * kCmLd + rr];
          dmma_8x8x4(acc[t], a, b);
        }
      }
    }
  }
  cp_async_wait<0>();
  double* out = part + (int64_t)blockIdx.x * k * k;
#pragma unroll
  for (int t = 0; t < TPW; ++t) {
    const int tile = warp * TPW + t;
    if (tile < TILES) {
      const int m = tm[t] + (lane >> 2);
      const int c0 = tn[t] + 2 * (lane & 3);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = c0 + h;
        if (m >= k || c >= k) continue;
        if (!SYM) {
          out[m * k + c] = acc[t][h];
        } else if (c >= m) {  // upper entry (diagonal tiles: their lower half is dropped)
          out[m * k + c] = acc[t][h];
          out[c * k + m] = acc[t][h];
        }
      }
    }
  }
}

template <int KP, bool SYM>
static int launch_cm(int64_t r0, int64_t r1, int k, const double* A, const double* B, double* part, int nb,
                     int64_t ld, cudaStream_t s) {
  const size_t smem = sizeof(double) * kCmStages * 2 * KP * kCmLd;
  const bool v16 = ((r0 | ld) & 1) == 0 && ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
  if (v16) {
    TB_CUDA(cudaFuncSetAttribute(k_atb_cm<KP, SYM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    { k_atb_cm<KP, SYM, true><<<nb, kGemmThreads, smem, s>>>(r0, r1, k, A, B, part, ld); tb::launched(); }
  } else {
    TB_CUDA(cudaFuncSetAttribute(k_atb_cm<KP, SYM, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    { k_atb_cm<KP, SYM, false><<<nb, kGemmThreads, smem, s>>>(r0, r1, k, A, B, part, ld); tb::launched(); }
  }
  TB_CHECK_LAUNCH();
  return TB_OK;
}

template <bool SYM>
static int launch_atb_colmajor(int64_t r0, int64_t r1, int k, const double* A, const double* B, double* part,
                               int nb, int64_t ld, cudaStream_t s) {
  const int kp = (k + 7) / 8 * 8;
  if (kp <= 16) return launch_cm<16, SYM>(r0, r1, k, A, B, part, nb, ld, s);
  if (kp <= 32) return launch_cm<32, SYM>(r0, r1, k, A, B, part, nb, ld, s);
  if (kp <= 64) return launch_cm<64, SYM>(r0, r1, k, A, B, part, nb, ld, s);
  set_error("reduced basis size k=%d exceeds 64", k);
  return TB_ERR_INVALID;
}

template <bool CM>
static int launch_atb_t(int64_t n, int k, const double* A, const double* B, double* part, int nb, int64_t ld,
                        cudaStream_t s) {
  const int kp = (k + 7) / 8 * 8;
  if (kp <= 8)
    { k_atb_dmma<8, CM><<<nb, kGemmThreads, 0, s>>>(n, k, A, B, part, ld); tb::launched(); }
  else if (kp <= 16)
    { k_atb_dmma<16, CM><<<nb, kGemmThreads, 0, s>>>(n, k, A, B, part, ld); tb::launched(); }
  else if (kp <= 32)
    { k_atb_dmma<32, CM><<<nb, kGemmThreads, 0, s>>>(n, k, A, B, part, ld); tb::launched(); }
  else if (kp <= 64)
    { k_atb_dmma<64, CM><<<nb, kGemmThreads, 0, s>>>(n, k, A, B, part, ld); tb::launched(); }
  else {
    set_error("reduced basis size k=%d exceeds 64", k);
    return TB_ERR_INVALID;
  }
  TB_CHECK_LAUNCH();
  return TB_OK;
}

static int launch_atb(int64_t n, int k, const double* A, const double* B, double* part, int nb, cudaStream_t s) {
  return launch_atb_t<false>(n, k, A, B, part, nb, 0, s);
}

// row-major (n x k) -> column-major (k columns, leading dimension ld >= n), 32 x 32 tiles
__global__ void k_transpose_rm_cm(int64_t n, int k, const double* __restrict__ rm, double* __restrict__ cm,
                                  int64_t ld) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + y;
    const int c = c0 + threadIdx.x;
    tile[y][threadIdx.x] = (r < n && c < k) ? rm[r * k + c] : 0.0;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int c = c0 + y;
    const int64_t r = r0 + threadIdx.x;
    if (c < k && r < ld) cm[(int64_t)c * ld + r] = (r < n) ? tile[threadIdx.x][y] : 0.0;
  }
}

// ---------------------------------------------------------------------------------------
// batched Cholesky  A = U^T U  (upper triangle, as scipy.linalg.cho_factor(lower=False))
// and solve for nrhs right-hand sides.  One CTA per design.
// ---------------------------------------------------------------------------------------
__global__ void k_cholesky_solve(int k, int nrhs, const double* __restrict__ khat, const double* __restrict__ rhs,
                                 double* __restrict__ x, int* __restrict__ status) {
  extern __shared__ double U[];  // k*k
  const int d = blockIdx.x, t = threadIdx.x, nt = blockDim.x;
  const double* A = khat + (int64_t)d * k * k;
  for (int o = t; o < k * k; o += nt) U[o] = A[o];
  __shared__ int bad;
  if (t == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    if (t == 0) {
      const double piv = U[j * k + j];
      const double ref = fabs(A[j * k + j]);
      // non-positive pivot, or one lost in round-off: numerically singular (rom.py:49-50)
      if (!(piv > (double)k * 2.220446049250313e-16 * ref) || !isfinite(piv)) bad = 1;
      else U[j * k + j] = sqrt(piv);
    }
    __syncthreads();
    if (bad) break;
    const double ujj = U[j * k + j];
    for (int c = j + 1 + t; c < k; c += nt) U[j * k + c] /= ujj;
    __syncthreads();
    const int m = k - j - 1;
    for (int o = t; o < m * m; o += nt) {
      const int r = j + 1 + o / m, c = j + 1 + o % m;
      if (c >= r) U[r * k + c] -= U[j * k + r] * U[j * k + c];
    }
    __syncthreads();
  }
  if (t == 0) status[d] = bad;
  if (bad) return;
  // U^T y = b ; U x = y
  for (int q = t; q < nrhs; q += nt) {
    const double* b = rhs + ((int64_t)d * nrhs + q) * k;
    double* xv = x + ((int64_t)d * nrhs + q) * k;
    for (int i = 0; i < k; ++i) {
      double s = b[i];
      for (int l = 0; l < i; ++l) s -= U[l * k + i] * xv[l];
      xv[i] = s / U[i * k + i];
    }
    for (int i = k - 1; i >= 0; --i) {
      double s = xv[i];
      for (int l = i + 1; l < k; ++l) s -= U[i * k + l] * xv[l];
      xv[i] = s / U[i * k + i];
    }
  }
}

// u[d][i] = sum_j phi[i][j] uhat[d][j]  (warp per row, lanes over j)
__global__ void __launch_bounds__(kBlock) k_reconstruct(int64_t n, int k, const double* __restrict__ phi,
                                                        const double* __restrict__ uhat, int nd, double* __restrict__ u) {
  extern __shared__ double su[];  // nd*k
  for (int o = threadIdx.x; o < nd * k; o += blockDim.x) su[o] = uhat[o];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    double acc[kMaxVec];
#pragma unroll
    for (int d = 0; d < kMaxVec; ++d) acc[d] = 0.0;
    for (int j = lane; j < k; j += 32) {
      const double pv = phi[i * k + j];
#pragma unroll
      for (int d = 0; d < kMaxVec; ++d)
        if (d < nd) acc[d] = fma(pv, su[d * k + j], acc[d]);
    }
#pragma unroll
    for (int d = 0; d < kMaxVec; ++d)
      if (d < nd) {
        const double v = warp_sum(acc[d]);
        if (lane == 0) u[(int64_t)d * n + i] = v;
      }
  }
}

// Same product on FP64 tensor cores: U^T (n x nd) = Phi (n x k) Uhat^T (k x nd) as m8n8k4 DMMA
// tiles -- a warp per 8 rows of Phi, the nd <= 16 designs as two 8-wide n-tiles whose B
// fragments (Uhat) stay in registers for the whole kernel.  Phi is streamed once.
__global__ void __launch_bounds__(kBlock) k_reconstruct_dmma(int64_t n, int k, const double* __restrict__ phi,
                                                             const double* __restrict__ uhat, int nd,
                                                             double* __restrict__ u) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int kSteps = 16;  // k <= 64
  double b[2][kSteps];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int st = 0; st < kSteps; ++st) {
      const int d = 8 * t + (lane >> 2), j = 4 * st + (lane & 3);
      b[t][st] = (d < nd && j < k) ? uhat[(int64_t)d * k + j] : 0.0;
    }
  // the A fragments of the next 8 rows are loaded (all 16 k-steps, unconditionally issued) before
  // the DMMA chain of the current ones: ncu of the load-then-use loop showed 4 warps per
  // scheduler stalled 22 cycles per issue on the long scoreboard (2.25 TB/s at cfg 5 size; now
  // 4.5 TB/s)
  auto load_tile = [&](int64_t i0, double (&a)[kSteps]) {
    const int64_t row = i0 + (lane >> 2);
    const double* pr = phi + row * k;
#pragma unroll
    for (int st = 0; st < kSteps; ++st) {
      const int j = 4 * st + (lane & 3);
      a[st] = (row < n && j < k) ? __ldg(pr + j) : 0.0;
    }
  };
  double a[kSteps];
  if (warp * 8 < n) load_tile(warp * 8, a);
  for (int64_t i0 = warp * 8; i0 < n; i0 += nwarps * 8) {
    double an[kSteps];
    const int64_t inext = i0 + nwarps * 8;
    if (inext < n) load_tile(inext, an);
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int st = 0; st < kSteps; ++st) {
      dmma_8x8x4(acc[0], a[st], b[0][st]);
      dmma_8x8x4(acc[1], a[st], b[1][st]);
    }
#pragma unroll
    for (int st = 0; st < kSteps; ++st) a[st] = an[st];
    // thread holds U^T[row i0 + lane/4][design 8t + 2(lane%4) + h]
    const int64_t ri = i0 + (lane >> 2);
    if (ri < n) {
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int d = 8 * t + 2 * (lane & 3) + h;
          if (d < nd) u[(int64_t)d * n + ri] = acc[t][h];
        }
    }
  }
}

// block partials of || mask * (y - g) ||^2
__global__ void __launch_bounds__(kBlock) k_resid_part(int64_t n, const double* __restrict__ y,
                                                       const double* __restrict__ g, const uint8_t* __restrict__ fixed,
                                                       double* __restrict__ part) {
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!fixed[i]) {
      const double r = y[i] - g[i];
      acc[0] = fma(r, r, acc[0]);
    }
  }
  block_sum<1>(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
}

}  // namespace tb

using namespace tb;

extern "C" {

#define TB_GUARD(cond, ...)   \
  do {                        \
    if (!(cond)) {            \
      set_error(__VA_ARGS__); \
      return TB_ERR_INVALID;  \
    }                         \
  } while (0)

int tb_rom_project(int64_t n, const double* phi, int k, const double* vec, int nvec, double* out, void* stream) {
  TB_GUARD(phi && vec && out && n >= 1, "bad arguments");
  TB_GUARD(k >= 1 && k <= kBlock, "basis size k=%d out of range [1, %d]", k, kBlock);
  TB_GUARD(nvec >= 1, "nvec=%d must be >= 1", nvec);
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = n >= (int64_t)1 << 20 ? 148 * 8 : 148 * 2;  // large bases: every resident CTA slot streams
  double* part = nullptr;
  const int nv0 = nvec < kMaxVec ? nvec : kMaxVec;
  TB_CUDA(cudaMallocAsync(&part, sizeof(double) * (size_t)nb * nv0 * k, s));
  const int groups = kBlock / k;
  for (int v0 = 0; v0 < nvec; v0 += kMaxVec) {  // kMaxVec vectors per pass over Phi
    const int nv = nvec - v0 < kMaxVec ? nvec - v0 : kMaxVec;
    const size_t sm = sizeof(double) * groups * nv * k;
    const double* v = vec + (int64_t)v0 * n;
    if (nv == 1) k_project_part<1><<<nb, kBlock, sm, s>>>(n, k, phi, v, nv, part);
    else if (groups > kPtR) {  // k < 4: a row chunk of the tile kernel would be empty
      if (nv == 2) k_project_part<2><<<nb, kBlock, sm, s>>>(n, k, phi, v, nv, part);
      else if (nv <= 4) k_project_part<4><<<nb, kBlock, sm, s>>>(n, k, phi, v, nv, part);
      else if (nv <= 8) k_project_part<8><<<nb, kBlock, sm, s>>>(n, k, phi, v, nv, part);
      else k_project_part<16><<<nb, kBlock, sm, s>>>(n, k, phi, v, nv, part);
    }
    else if (nv == 2) k_project_tile<2><<<nb, kBlock, sm, s>>>(n, k, phi, v, nv, part);
    else if (nv <= 4) k_project_tile<4><<<nb, kBlock, sm, s>>>(n, k, phi, v, nv, part);
    else if (nv <= 8) k_project_tile<8><<<nb, kBlock, sm, s>>>(n, k, phi, v, nv, part);
    else k_project_tile<16><<<nb, kBlock, sm, s>>>(n, k, phi, v, nv, part);
    tb::launched();
    { k_sum_parts<<<nblk(nv * k), kBlock, 0, s>>>(nb, nv * k, part, out + (int64_t)v0 * k); tb::launched(); }
  }
  TB_CHECK_LAUNCH();
  TB_CUDA(cudaFreeAsync(part, s));
  return TB_OK;
}

int tb_rom_reduced_stiffness(tb_plan* plan, const double* phi, int k, const double* rho, int nd, double* khat,
                             void* stream) {
  TB_GUARD(plan && phi && rho && khat, "null argument");
  TB_GUARD(k >= 1 && k <= 64, "basis size k=%d out of range [1, 64]", k);
  TB_GUARD(nd >= 1, "nd must be >= 1");
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  cudaStream_t s = (cudaStream_t)stream;
  const Grid& g = P->g;
  const int64_t n = P->n_dofs;
  const int nb = 148 * 2;
  // contract only the rows of owned node planes (a slab's ghost rows belong to a neighbour)
  const int64_t pd = (int64_t)g.dim * g.nnx * g.nny;
  const int64_t r0 = (int64_t)P->own_k0 * pd;
  const int64_t r1 = P->own_k1 >= g.nnz ? n : (int64_t)P->own_k1 * pd;
  const bool hex8 = (g.dim == 3 && P->hex8);
  if (hex8 && rom_fused_eligible(P, k)) {
    // element form, all designs per pass over Phi (romfused.cu); owned element planes of a slab
    const int kb0 = P->own_k0, kb1 = P->own_k1 < g.nz ? P->own_k1 : g.nz;
    const size_t na = ((size_t)nd * g.n_elems + 31) / 32 * 32;  // partials start 256-byte aligned
    const size_t pbytes = rom_fused_scratch_bytes(P, k, nd);
    TB_TRY(P->rom_scratch(sizeof(double) * na + pbytes));
    double* al = P->d_rom;
    for (int d = 0; d < nd; ++d) TB_TRY(P->material(rho + (int64_t)d * g.n_elems, al + (int64_t)d * g.n_elems, nullptr, s));
    return rom_fused_khat(P, phi, k, al, nd, kb0, kb1, P->d_rom + na, pbytes, khat, s);
  }
  // 3D: one WHT Hex8 launch per column on a column-major copy of Phi; 2D: node-owner over
  // all k columns of the row-major Phi
  const int nbc = hex8 ? 148 * kCmCtas : nb;        // column-major DMMA: one wave of resident CTAs
  const int64_t ldp = hex8 ? (n + 1) / 2 * 2 : n;    // even leading dimension (16-byte columns)
  const size_t ybytes = sizeof(double) * (size_t)ldp * k * (hex8 ? 2 : 1);
  const size_t pbytes = sizeof(double) * (size_t)nbc * k * k;
  TB_TRY(P->rom_scratch(ybytes + pbytes));
  double* Y = P->d_rom;
  double* PhiT = hex8 ? P->d_rom + (size_t)ldp * k : nullptr;
  double* part = P->d_rom + (size_t)ldp * k * (hex8 ? 2 : 1);
  if (hex8) {
    dim3 tg((unsigned)((n + 31) / 32), (unsigned)((k + 31) / 32));
    { k_transpose_rm_cm<<<tg, dim3(32, 8), 0, s>>>(n, k, phi, PhiT, ldp); tb::launched(); }
  }
  for (int d = 0; d < nd; ++d) {
    TB_TRY(P->material(rho + (int64_t)d * g.n_elems, P->d_alpha2, nullptr, s));
    if (hex8) {
      // Y = K(rho) Phi: all k columns in ONE launch (blockIdx.z = column * chunks + chunk)
      const int zc = hex8_zchunk_cols(g, k);
      dim3 gr = hex8_grid(g, zc);
      const int zblocks = (int)gr.z;
      gr.z *= (unsigned)k;
      { k_hex8<false><<<gr, kHT, kHex8Smem, s>>>(g, P->hiso, P->d_alpha2, PhiT, nullptr, nullptr, Y, nullptr, nullptr, zc, 0.0, 3.0, nullptr, nullptr, ldp, zblocks); tb::launched(); }
      TB_CHECK_LAUNCH();
      TB_TRY(launch_atb_colmajor<true>(r0, r1, k, PhiT, Y, part, nbc, ldp, s));  // Phi^T (K Phi) is symmetric
    } else {
      const int64_t threads = g.n_nodes * k;
      const int blocks = (int)((threads + kBlock - 1) / kBlock);
      if (g.dim == 2)
        { k_apply_cols<2><<<blocks, kBlock, 0, s>>>(g, P->K2, P->d_alpha2, phi, k, Y); tb::launched(); }
      else
        { k_apply_cols<3><<<blocks, kBlock, 0, s>>>(g, P->K3, P->d_alpha2, phi, k, Y); tb::launched(); }
      TB_CHECK_LAUNCH();
      TB_TRY(launch_atb(r1 - r0, k, phi + r0 * k, Y + r0 * k, part, nb, s));
    }
    { k_sum_parts<<<nblk(k * k), kBlock, 0, s>>>(hex8 ? nbc : nb, k * k, part, khat + (int64_t)d * k * k); tb::launched(); }
    TB_CHECK_LAUNCH();
  }
  return TB_OK;
}

int tb_rom_gram_colmajor(int64_t n, int k, const double* A, const double* B, int64_t ld, int symmetric,
                         double* out, void* stream) {
  TB_GUARD(A && B && out && n >= 1 && ld >= n, "bad arguments");
  TB_GUARD(k >= 1 && k <= 64, "k=%d out of range [1, 64]", k);
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = 148 * kCmCtas;
  double* part = nullptr;
  TB_CUDA(cudaMallocAsync(&part, sizeof(double) * (size_t)nb * k * k, s));
  if (symmetric)
    TB_TRY(launch_atb_colmajor<true>(0, n, k, A, B, part, nb, ld, s));
  else
    TB_TRY(launch_atb_colmajor<false>(0, n, k, A, B, part, nb, ld, s));
  { k_sum_parts<<<nblk(k * k), kBlock, 0, s>>>(nb, k * k, part, out); tb::launched(); }
  TB_CHECK_LAUNCH();
  TB_CUDA(cudaFreeAsync(part, s));
  return TB_OK;
}

int tb_rom_cholesky_solve(int k, int nd, int nrhs, const double* khat, const double* rhs, double* x, int* status,
                          void* stream) {
  TB_GUARD(khat && rhs && x && status, "null argument");
  TB_GUARD(k >= 1 && k <= 128 && nd >= 1 && nrhs >= 1, "bad sizes k=%d nd=%d nrhs=%d", k, nd, nrhs);
  cudaStream_t s = (cudaStream_t)stream;
  int* d_status = nullptr;
  TB_CUDA(cudaMallocAsync(&d_status, sizeof(int) * nd, s));
  const size_t sm = sizeof(double) * k * k;
  if (sm > 48 * 1024) TB_CUDA(cudaFuncSetAttribute(k_cholesky_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  { k_cholesky_solve<<<nd, 256, sm, s>>>(k, nrhs, khat, rhs, x, d_status); tb::launched(); }
  TB_CHECK_LAUNCH();
  TB_CUDA(cudaMemcpyAsync(status, d_status, sizeof(int) * nd, cudaMemcpyDeviceToHost, s));
  TB_CUDA(cudaFreeAsync(d_status, s));
  TB_CUDA(cudaStreamSynchronize(s));
  for (int d = 0; d < nd; ++d)
    if (status[d]) {
      set_error("reduced stiffness of design %d is not positive definite", d);
      return TB_ERR_DEGENERATE;
    }
  return TB_OK;
}

int tb_rom_reconstruct(int64_t n, const double* phi, int k, const double* uhat, int nd, double* u, void* stream) {
  TB_GUARD(phi && uhat && u && n >= 1, "bad arguments");
  TB_GUARD(k >= 1 && nd >= 1, "bad sizes k=%d nd=%d", k, nd);
  cudaStream_t s = (cudaStream_t)stream;
  for (int d0 = 0; d0 < nd; d0 += kMaxVec) {  // kMaxVec designs per pass over Phi
    const int m = nd - d0 < kMaxVec ? nd - d0 : kMaxVec;
    const double* uh = uhat + (int64_t)d0 * k;
    double* ud = u + (int64_t)d0 * n;
    if (k <= 64)
      { k_reconstruct_dmma<<<148 * 8, kBlock, 0, s>>>(n, k, phi, uh, m, ud); tb::launched(); }
    else
      { k_reconstruct<<<148 * 8, kBlock, sizeof(double) * m * k, s>>>(n, k, phi, uh, m, ud); tb::launched(); }
  }
  TB_CHECK_LAUNCH();
  return TB_OK;
}

int tb_rom_residual_norms(tb_plan* plan, const double* phi, int k, const double* rho, const double* uhat, int nd,
                          const double* g, int64_t g_stride, double* norms, void* stream) {
  TB_GUARD(plan && phi && rho && uhat && g && norms, "null argument");
  TB_GUARD(k >= 1 && nd >= 1 && nd <= kMaxVec, "bad sizes k=%d nd=%d", k, nd);
  auto* P = reinterpret_cast<tb_plan_impl*>(plan);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = P->n_dofs;
  const int nb = grid_for(n);
  TB_TRY(P->rom_scratch(sizeof(double) * ((size_t)(nd + 1) * n + nb + 16)));
  double* U = P->d_rom;
  double* Y = U + (size_t)nd * n;
  double* part = Y + n;
  TB_TRY(tb_rom_reconstruct(n, phi, k, uhat, nd, U, stream));
  for (int d = 0; d < nd; ++d) {
    TB_TRY(P->material(rho + (int64_t)d * P->g.n_elems, P->d_alpha2, nullptr, s));
    P->apply_alpha(P->d_alpha2, U + (int64_t)d * n, Y, false, s);
    { k_resid_part<<<nb, kBlock, 0, s>>>(n, Y, g + d * g_stride, P->d_fixed, part); tb::launched(); }
    finish_sum(nb, part, P->d_scalar + d, s);
  }
  TB_CHECK_LAUNCH();
  TB_CUDA(cudaMemcpyAsync(P->h_scalar, P->d_scalar, sizeof(double) * nd, cudaMemcpyDeviceToHost, s));
  TB_CUDA(cudaStreamSynchronize(s));
  for (int d = 0; d < nd; ++d) norms[d] = sqrt(P->h_scalar[d]);
  return TB_OK;
}

}  // extern "C"
