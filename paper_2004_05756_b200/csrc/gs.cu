// Block Gram-Schmidt with a drop tolerance (reference rom.py:76-97), entirely on the device.
//
// The reference orthonormalises vector by vector (MGS, two passes over every kept vector) and
// drops a vector whose residual falls below drop_tol times its original norm.  Here the vectors
// go in panels of 8 (block classical Gram-Schmidt, BCGS2 form):
//   1. norms   : ||v_j|| of the panel's original vectors (the drop reference);
//   2. pass 1  : C = Q^T W on the FP64 tensor cores (mma m8n8k4 -> DMMA), W -= Q C;
//   3. intra   : per panel vector, CGS2 against the vectors this panel already kept (<= 7
//                columns), then the drop decision and the append -- all decided on the device;
//   4. pass 2  : C = Q^T Q_b (DMMA), Q_b -= Q C on the panel's new columns, which removes the
//                components along the earlier basis that the intra step's rounding reintroduced
//                (their size is eps ||v|| / ||w||, so the orthonormality error left is its square).
// Q is read four times per panel instead of 2-3 times per vector, the Gram products run on DMMA,
// and nothing waits on the host: the column counts live in device memory (GsCtl) and the host
// reads the final count once.  Deterministic (fixed-order reductions, no atomics on values).
#include "plan.cuh"

namespace tb {

namespace {

constexpr int kGsB = 8;            // panel width (one DMMA n-tile)
constexpr int kGsThreads = 256;
constexpr int kGsWarps = kGsThreads / 32;
constexpr int kGsRows = 32;        // rows staged per step
constexpr int kGsLd = kGsRows + 4; // padded staging row
constexpr int kGsTpw = 2;          // A tiles per warp
constexpr int kGsChunk = kGsTpw * kGsWarps * 8;  // Q columns per DMMA launch (128)
constexpr int kGsCtas = 148 * 2;
constexpr size_t kGsAtbSmem = sizeof(double) * 2 * (kGsChunk + kGsB) * kGsLd;  // 78 KB

struct GsCtl {
  int nk;              // committed basis columns
  int nk0;             // basis columns before the current panel
  int keep;            // decision for the current vector
  unsigned int count;  // last-block counter
  double nrm0[kGsB];   // original norms of the panel's vectors
  double c[2][kGsB];   // intra coefficients (double-buffered by pass)
  double rr;           // ||w||^2 of the current vector
  double scale;        // 1 / ||w||
};

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Last block to arrive (after a fence) -> true in every thread of that block.
__device__ __forceinline__ bool last_block(unsigned int* counter) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
    if (last) *counter = 0u;
  }
  __syncthreads();
  return last;
}

// panel norms: nrm0[j] = ||W[:, j]||, j < nb; the last block also opens the panel (nk0 = nk)
__global__ void __launch_bounds__(kGsThreads) k_gs_norms(int64_t n, int nb, const double* __restrict__ W, GsCtl* ctl,
                                                         double* part) {
  double acc[kGsB];
#pragma unroll
  for (int j = 0; j < kGsB; ++j) acc[j] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int j = 0; j < kGsB; ++j)
      if (j < nb) {
        const double v = W[(int64_t)j * n + i];
        acc[j] = fma(v, v, acc[j]);
      }
  }
  block_sum<kGsB>(acc);
  if (publish_partials<kGsB>(acc, part, &ctl->count)) {
    gather_partials<kGsB>(acc, part, &ctl->count);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int j = 0; j < kGsB; ++j) ctl->nrm0[j] = sqrt(acc[j]);
      ctl->nk0 = ctl->nk;
    }
  }
}

// Partial C[c0 + m][j] = sum_r Q[r][c0 + m] B[r][j] over this CTA's row range, m < 128, on DMMA.
// Q: basis columns [0, nk0) (ld n).  B: the panel W (nB = nb) or, PANEL_Q, the basis columns
// [nk0, nk) this panel added.  part: [cta][kGsChunk][8].
template <bool PANEL_Q>
__global__ void __launch_bounds__(kGsThreads) k_gs_atb(int64_t n, int c0, const double* __restrict__ Q,
                                                       const double* __restrict__ W, int nb, const GsCtl* ctl,
                                                       double* __restrict__ part) {
  extern __shared__ __align__(16) double gs_sm[];  // [2][kGsChunk * kGsLd] A, then [2][kGsB * kGsLd] B
  auto sA = [&](int buf) { return gs_sm + buf * kGsChunk * kGsLd; };
  auto sB = [&](int buf) { return gs_sm + 2 * kGsChunk * kGsLd + buf * kGsB * kGsLd; };
  const int nA = min(kGsChunk, ctl->nk0 - c0);
  const int nB = PANEL_Q ? ctl->nk - ctl->nk0 : nb;
  const double* B = PANEL_Q ? Q + (int64_t)ctl->nk0 * n : W;
  const double* A = Q + (int64_t)c0 * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* out = part + (int64_t)blockIdx.x * kGsChunk * kGsB;
  if (nA <= 0 || nB <= 0) {  // nothing to project (uniform over the grid): zero partials
    for (int o = tid; o < kGsChunk * kGsB; o += kGsThreads) out[o] = 0.0;
    return;
  }
  const int64_t per = ((n + gridDim.x - 1) / gridDim.x + kGsRows - 1) / kGsRows * kGsRows;
  const int64_t i0 = (int64_t)blockIdx.x * per, i1 = min(n, i0 + per);
  const int nst = (int)((max(i1 - i0, (int64_t)0) + kGsRows - 1) / kGsRows);
  const int nA8 = (nA + 7) / 8 * 8;  // staged A columns: the valid ones, zero-filled to a whole tile
  auto load = [&](int stg, int buf) {
    const int64_t base = i0 + (int64_t)stg * kGsRows;
    for (int idx = tid; idx < (nA8 + kGsB) * kGsRows; idx += kGsThreads) {
      const int c = idx / kGsRows, r = idx % kGsRows;
      const int64_t row = base + r;
      const bool isA = c < nA8;
      const int cc = isA ? c : c - nA8;
      const bool ok = row < i1 && cc < (isA ? nA : nB);
      const double* src = (isA ? A : B) + (ok ? (int64_t)cc * n + row : 0);
      cp_async8((isA ? sA(buf) : sB(buf)) + cc * kGsLd + r, src, ok);
    }
    cp_async_commit();
  };
  double acc[kGsTpw][2];
#pragma unroll
  for (int t = 0; t < kGsTpw; ++t) acc[t][0] = acc[t][1] = 0.0;
  if (nst > 0) load(0, 0);
  for (int s = 0; s < nst; ++s) {
    if (s + 1 < nst) {
      load(s + 1, (s + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* a_s = sA(s & 1);
    const double* b_s = sB(s & 1);
#pragma unroll
    for (int t = 0; t < kGsTpw; ++t) {
      const int m0 = (warp + t * kGsWarps) * 8;
      if (m0 < nA) {
#pragma unroll
        for (int r0 = 0; r0 < kGsRows; r0 += 4) {
          const double a = a_s[(m0 + (lane >> 2)) * kGsLd + r0 + (lane & 3)];
          const double b = b_s[(lane >> 2) * kGsLd + r0 + (lane & 3)];
          dmma884(acc[t], a, b);
        }
      }
    }
    __syncthreads();
  }
  // D fragment: row m0 + lane/4, columns 2 (lane % 4) + {0, 1}
#pragma unroll
  for (int t = 0; t < kGsTpw; ++t) {
    const int m = (warp + t * kGsWarps) * 8 + (lane >> 2), j = 2 * (lane & 3);
    out[m * kGsB + j] = acc[t][0];
    out[m * kGsB + j + 1] = acc[t][1];
  }
}

// C[c0 + o] = sum_cta part[cta][o] (fixed order)
__global__ void k_gs_sum(int c0, int nparts, const double* __restrict__ part, double* __restrict__ C) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= kGsChunk * kGsB) return;
  double s = 0.0;
  for (int b = 0; b < nparts; ++b) s += part[(int64_t)b * kGsChunk * kGsB + o];
  C[(int64_t)c0 * kGsB + o] = s;
}

// B[:, j] -= sum_{l < nk0} Q[:, l] C[l][j], j < nB (B = W or, PANEL_Q, the panel's basis columns);
// C rows in shared memory (dynamic: nk0 x 8 doubles), four Q loads in flight per thread
template <bool PANEL_Q>
__global__ void __launch_bounds__(kGsThreads) k_gs_update(int64_t n, const double* __restrict__ Q, double* W, int nb,
                                                          const double* __restrict__ C, const GsCtl* ctl) {
  extern __shared__ __align__(16) double gs_c[];
  const int nA = ctl->nk0;
  const int nB = PANEL_Q ? ctl->nk - ctl->nk0 : nb;
  double* B = PANEL_Q ? const_cast<double*>(Q) + (int64_t)nA * n : W;
  if (nA <= 0 || nB <= 0) return;
  for (int o = threadIdx.x; o < nA * kGsB; o += blockDim.x) gs_c[o] = C[o];
  __syncthreads();
  const double2* c2 = reinterpret_cast<const double2*>(gs_c);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc[kGsB];
#pragma unroll
    for (int j = 0; j < kGsB; ++j) acc[j] = 0.0;
    int l = 0;
    for (; l + 4 <= nA; l += 4) {
      double q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = Q[(int64_t)(l + u) * n + i];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < kGsB / 2; ++j) {
          const double2 c = c2[(l + u) * (kGsB / 2) + j];
          acc[2 * j] = fma(q[u], c.x, acc[2 * j]);
          acc[2 * j + 1] = fma(q[u], c.y, acc[2 * j + 1]);
        }
    }
    for (; l < nA; ++l) {
      const double q = Q[(int64_t)l * n + i];
#pragma unroll
      for (int j = 0; j < kGsB / 2; ++j) {
        const double2 c = c2[l * (kGsB / 2) + j];
        acc[2 * j] = fma(q, c.x, acc[2 * j]);
        acc[2 * j + 1] = fma(q, c.y, acc[2 * j + 1]);
      }
    }
#pragma unroll
    for (int j = 0; j < kGsB; ++j)
      if (j < nB) B[(int64_t)j * n + i] -= acc[j];
  }
}

enum { kGsUpdate = 1, kGsDots = 2, kGsDecide = 4 };

// Intra-panel CGS step for panel vector j against the columns the panel kept before it
// (basis columns [nk0, nk)): optionally w -= Q_b c_in, then c_out = Q_b^T w and ||w||^2;
// kGsDecide: keep = ||v_j|| > 0 and ||w|| >= drop ||v_j||, scale = 1 / ||w||.
__global__ void __launch_bounds__(kGsThreads) k_gs_intra(int64_t n, const double* __restrict__ Q, double* __restrict__ w,
                                                         int j, int mode, int par, double drop, GsCtl* ctl,
                                                         double* part) {
  const int nq = ctl->nk - ctl->nk0;  // <= j < 8
  const double* Qb = Q + (int64_t)ctl->nk0 * n;
  double cin[kGsB - 1];
#pragma unroll
  for (int l = 0; l < kGsB - 1; ++l) cin[l] = (mode & kGsUpdate) && l < nq ? ctl->c[par][l] : 0.0;
  double acc[kGsB];  // c_out[0..6], ||w||^2
#pragma unroll
  for (int l = 0; l < kGsB; ++l) acc[l] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double q[kGsB - 1];
#pragma unroll
    for (int l = 0; l < kGsB - 1; ++l) q[l] = l < nq ? Qb[(int64_t)l * n + i] : 0.0;
    double v = w[i];
    if (mode & kGsUpdate) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < kGsB - 1; ++l) s = fma(q[l], cin[l], s);
      v -= s;
      w[i] = v;
    }
    if (mode & kGsDots) {
#pragma unroll
      for (int l = 0; l < kGsB - 1; ++l) acc[l] = fma(q[l], v, acc[l]);
    }
    acc[kGsB - 1] = fma(v, v, acc[kGsB - 1]);
  }
  block_sum<kGsB>(acc);
  if (publish_partials<kGsB>(acc, part, &ctl->count)) {
    gather_partials<kGsB>(acc, part, &ctl->count);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int l = 0; l < kGsB - 1; ++l) ctl->c[par ^ 1][l] = acc[l];
      const double rr = acc[kGsB - 1];
      ctl->rr = rr;
      if (mode & kGsDecide) {
        const double n0 = ctl->nrm0[j], nw = sqrt(rr);
        ctl->keep = (n0 > 0.0 && nw >= drop * n0) ? 1 : 0;
        ctl->scale = 1.0 / nw;
      }
    }
  }
}

// kept -> basis column nk = w * scale; the last block commits nk
__global__ void __launch_bounds__(kGsThreads) k_gs_append(int64_t n, double* __restrict__ Q, const double* __restrict__ w,
                                                          GsCtl* ctl) {
  const int keep = ctl->keep;
  if (keep) {
    const double sc = ctl->scale;
    double* dst = Q + (int64_t)ctl->nk * n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      dst[i] = w[i] * sc;
  }
  if (last_block(&ctl->count) && threadIdx.x == 0) ctl->nk += keep;
}

// column-major (n x m, ld n) -> row-major (n x m)
__global__ void k_gs_transpose(int64_t n, int m, const double* __restrict__ cm, double* __restrict__ rm) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k;
    const int64_t r = r0 + threadIdx.x;
    tile[k][threadIdx.x] = (c < m && r < n) ? cm[(int64_t)c * n + r] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k;
    const int c = c0 + threadIdx.x;
    if (c < m && r < n) rm[r * m + c] = tile[threadIdx.x][k];
  }
}

}  // namespace

}  // namespace tb

using namespace tb;

extern "C" int tb_gram_schmidt(int64_t n, int m, const double* vectors, double drop_tol, double* q, int* kept,
                               void* stream) {
  if (!(vectors && q && kept && n >= 1 && m >= 1)) {
    set_error("gram_schmidt: bad arguments");
    return TB_ERR_INVALID;
  }
  if (m > 2048) {
    set_error("gram_schmidt: at most 2048 vectors per call (got %d)", m);
    return TB_ERR_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  {  // keep up to 16 GB of freed workspace in the stream-ordered pool between calls: re-mapping
     // cfg 5's 6.6 GB basis workspace on every call cost more than the orthogonalisation
    static bool done[64] = {};
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && dev < 64 && !done[dev] &&
        cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = 16ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      done[dev] = true;
    }
  }
  const int mcap = (m + kGsChunk - 1) / kGsChunk * kGsChunk;
  double *Q = nullptr, *W = nullptr, *C = nullptr, *part = nullptr;
  GsCtl* ctl = nullptr;
  const size_t npart = (size_t)kGsCtas * kGsChunk * kGsB;
  TB_CUDA(cudaMallocAsync(&Q, sizeof(double) * (size_t)n * m, s));
  TB_CUDA(cudaMallocAsync(&W, sizeof(double) * (size_t)n * kGsB, s));
  TB_CUDA(cudaMallocAsync(&C, sizeof(double) * (size_t)mcap * kGsB, s));
  TB_CUDA(cudaMallocAsync(&part, sizeof(double) * npart, s));
  TB_CUDA(cudaMallocAsync(&ctl, sizeof(GsCtl), s));
  TB_CUDA(cudaMemsetAsync(ctl, 0, sizeof(GsCtl), s));
  const int nbk = grid_for(n, kGsThreads, kGsCtas);
  TB_CUDA(cudaFuncSetAttribute(k_gs_atb<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGsAtbSmem));
  TB_CUDA(cudaFuncSetAttribute(k_gs_atb<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGsAtbSmem));
  const size_t usm = sizeof(double) * (size_t)m * kGsB;  // C rows of k_gs_update
  if (usm > 48 * 1024) {
    TB_CUDA(cudaFuncSetAttribute(k_gs_update<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm));
    TB_CUDA(cudaFuncSetAttribute(k_gs_update<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm));
  }
  for (int i0 = 0; i0 < m; i0 += kGsB) {
    const int nb = m - i0 < kGsB ? m - i0 : kGsB;
    cudaMemcpyAsync(W, vectors + (int64_t)i0 * n, sizeof(double) * (size_t)n * nb, cudaMemcpyDeviceToDevice, s);
    k_gs_norms<<<nbk, kGsThreads, 0, s>>>(n, nb, W, ctl, part);
    launched(1);
    // pass 1: W -= Q (Q^T W) against the basis kept before this panel (at most i0 columns)
    if (i0 > 0) {
      for (int c0 = 0; c0 < i0; c0 += kGsChunk) {
        k_gs_atb<false><<<kGsCtas, kGsThreads, kGsAtbSmem, s>>>(n, c0, Q, W, nb, ctl, part);
        k_gs_sum<<<(kGsChunk * kGsB + 255) / 256, 256, 0, s>>>(c0, kGsCtas, part, C);
        launched(2);
      }
      k_gs_update<false><<<nbk, kGsThreads, usm, s>>>(n, Q, W, nb, C, ctl);
      launched(1);
    }
    // intra-panel CGS2 + drop decision + append, vector by vector (decisions stay on the device)
    for (int j = 0; j < nb; ++j) {
      double* w = W + (int64_t)j * n;
      k_gs_intra<<<nbk, kGsThreads, 0, s>>>(n, Q, w, j, kGsDots, 0, drop_tol, ctl, part);
      k_gs_intra<<<nbk, kGsThreads, 0, s>>>(n, Q, w, j, kGsUpdate | kGsDots, 1, drop_tol, ctl, part);
      k_gs_intra<<<nbk, kGsThreads, 0, s>>>(n, Q, w, j, kGsUpdate | kGsDecide, 0, drop_tol, ctl, part);
      k_gs_append<<<nbk, kGsThreads, 0, s>>>(n, Q, w, ctl);
      launched(4);
    }
    // pass 2: the panel's new columns against the earlier basis
    if (i0 > 0) {
      for (int c0 = 0; c0 < i0; c0 += kGsChunk) {
        k_gs_atb<true><<<kGsCtas, kGsThreads, kGsAtbSmem, s>>>(n, c0, Q, W, nb, ctl, part);
        k_gs_sum<<<(kGsChunk * kGsB + 255) / 256, 256, 0, s>>>(c0, kGsCtas, part, C);
        launched(2);
      }
      k_gs_update<true><<<nbk, kGsThreads, usm, s>>>(n, Q, W, nb, C, ctl);
      launched(1);
    }
  }
  int rc = TB_OK;
  GsCtl h;
  if (cudaMemcpyAsync(&h, ctl, sizeof(GsCtl), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    set_error("CUDA failure in gram_schmidt");
    rc = TB_ERR_CUDA;
  }
  if (rc == TB_OK && h.nk == 0) {
    set_error("no independent vectors supplied");
    rc = TB_ERR_INVALID;
  }
  if (rc == TB_OK) {
    dim3 tg((unsigned)((n + 31) / 32), (unsigned)((h.nk + 31) / 32));
    k_gs_transpose<<<tg, dim3(32, 8), 0, s>>>(n, h.nk, Q, q);
    launched(1);
  }
  *kept = rc == TB_OK ? h.nk : 0;
  cudaFreeAsync(Q, s);
  cudaFreeAsync(W, s);
  cudaFreeAsync(C, s);
  cudaFreeAsync(part, s);
  cudaFreeAsync(ctl, s);
  if (rc == TB_OK && cudaGetLastError() != cudaSuccess) {
    set_error("CUDA failure in gram_schmidt");
    rc = TB_ERR_CUDA;
  }
  return rc;
}
