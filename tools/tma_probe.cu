// Probe of the TMA pattern used by csrc/sweep.cu (one case per process: a fault is sticky).
//   case 0: mbarrier only (plain arrive, no TMA)
//   case 1: 1D bulk copy (cp.async.bulk, non-tensor) + mbarrier tx
//   case 2: 3D FLOAT64 tensor map, small box 16x4 at (0,0,0), map as __grid_constant__ param
//   case 3: same map, box 100x9 at (-3,-1,0) (the sweep's halo tile)
//   case 4: case 2 with the map in global memory
//   case 5: case 2 with a 2D map over the same data
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void wait0(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(su32(bar))
      : "memory");
}

__global__ void k_probe(const __grid_constant__ CUtensorMap m, const CUtensorMap* gm, int mode, int c0, int c1,
                        int c2, int n, const double* src, double* out) {
  extern __shared__ __align__(128) double s[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (mode == 0) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&bar)) : "memory");
    } else {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar)), "r"(n * 8) : "memory");
      if (mode == 1) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         su32(s)),
                     "l"(src), "r"(n * 8), "r"(su32(&bar))
                     : "memory");
      } else if (mode == 5) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];\n" ::"r"(su32(s)),
            "l"(&m), "r"(c0), "r"(c1), "r"(su32(&bar))
            : "memory");
      } else {
        const void* mp = (mode == 4) ? (const void*)gm : (const void*)&m;
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];\n" ::"r"(su32(s)),
            "l"(mp), "r"(c0), "r"(c1), "r"(c2), "r"(su32(&bar))
            : "memory");
      }
    }
  }
  wait0(&bar);
  if (mode != 0)
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = s[i];
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 2;
  const int nnx = 193, nny = 97, nnz = 97;
  const int64_t P = ((int64_t)3 * nnx + 3) / 4 * 4;
  const int64_t N = P * nny * nnz;
  std::vector<double> h(N);
  for (int64_t i = 0; i < N; ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, N * 8);
  cudaMalloc(&o, 1 << 20);
  cudaMemcpy(d, h.data(), N * 8, cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t ge = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  printf("entry point: %s, query %d, fn %p\n", cudaGetErrorString(ge), (int)q, fp);
  Enc enc = (Enc)fp;
  int bx = 16, by = 4, c0 = 0, c1 = 0, c2 = 0;
  if (mode == 3) bx = 100, by = 9, c0 = -3, c1 = -1;
  if (argc > 5) bx = atoi(argv[2]), by = atoi(argv[3]), c0 = atoi(argv[4]), c1 = atoi(argv[5]);
  CUtensorMap m;
  CUresult r1;
  const cuuint32_t es[3] = {1, 1, 1};
  if (mode == 5) {
    const cuuint64_t dims[2] = {(cuuint64_t)3 * nnx, (cuuint64_t)nny * nnz};
    const cuuint64_t str[1] = {(cuuint64_t)P * 8};
    const cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by};
    r1 = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[3] = {(cuuint64_t)3 * nnx, (cuuint64_t)nny, (cuuint64_t)nnz};
    const cuuint64_t str[2] = {(cuuint64_t)P * 8, (cuuint64_t)P * nny * 8};
    const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    r1 = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  CUtensorMap* gm;
  cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
  const int n = (mode == 1) ? 256 : bx * by;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k_probe<<<1, 128, 16 * 1024>>>(m, gm, mode, c0, c1, c2, n, d, o);
  cudaError_t e = cudaDeviceSynchronize();
  int bad = 0;
  if (e == cudaSuccess && mode != 0) {
    std::vector<double> got(n);
    cudaMemcpy(got.data(), o, n * 8, cudaMemcpyDeviceToHost);
    for (int y = 0; y < (mode == 1 ? 1 : by); ++y)
      for (int x = 0; x < (mode == 1 ? n : bx); ++x) {
        const int gx = c0 + x, gy = c1 + y;
        const double want = (gx >= 0 && gy >= 0) ? (double)(gy * P + gx) : 0.0;
        if (got[y * bx + x] != want) ++bad;
      }
  }
  printf("mode %d: encode %d, kernel %s, mismatches %d\n", mode, (int)r1, cudaGetErrorString(e), bad);
  return e == cudaSuccess && bad == 0 ? 0 : 1;
}
