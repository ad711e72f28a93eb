// Probe: can a cooperative launch carry a thread-block cluster dimension on B200, and what do a
// hardware cluster barrier, a software barrier among one cluster's CTAs and the software grid
// barrier cost?  (Design input for running the small multigrid levels inside one cluster.)
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void grid_bar(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int nb = gridDim.x;
    const unsigned int add = (blockIdx.x == 0) ? (0x80000000u - (nb - 1u)) : 1u;
    unsigned int old, cur;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(add) : "memory");
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
    } while (((old ^ cur) & 0x80000000u) == 0u);
  }
  __syncthreads();
}

template <int MODE>
__global__ void kprobe(unsigned int* bar, int iters, double* out) {
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
      grid_bar(bar);
    } else if (MODE == 1) {  // hardware cluster barrier
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else {  // cluster 0 only: hardware cluster barrier, other clusters idle
      if (blockIdx.x < 8)
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    acc += it;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

int main() {
  unsigned int* bar;
  cudaMalloc(&bar, 64);
  cudaMemset(bar, 0, 64);
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cs : {8, 16}) {
    for (int threads : {512}) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeCooperative;
      at[1].val.cooperative = 1;
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = 100 * 1024;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      if (cs == 16) cudaFuncSetAttribute(kprobe<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (cs == 16) cudaFuncSetAttribute(kprobe<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(kprobe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
      cudaFuncSetAttribute(kprobe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
      cfg.gridDim = dim3(cs);
      int ncl = 0;
      cudaError_t eo = cudaOccupancyMaxActiveClusters(&ncl, (void*)kprobe<0>, &cfg);
      printf("cluster %d threads %d: max active clusters %d (%s), sms %d\n", cs, threads, ncl, cudaGetErrorString(eo), sms);
      if (ncl <= 0) continue;
      cfg.gridDim = dim3(ncl * cs);
      int iters = 20000;
      for (int mode = 0; mode < 2; ++mode) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaError_t e1 = mode == 0 ? cudaLaunchKernelEx(&cfg, kprobe<0>, bar, iters, out) : cudaLaunchKernelEx(&cfg, kprobe<1>, bar, iters, out);
        cudaEventRecord(a);
        cudaError_t e2 = mode == 0 ? cudaLaunchKernelEx(&cfg, kprobe<0>, bar, iters, out) : cudaLaunchKernelEx(&cfg, kprobe<1>, bar, iters, out);
        cudaEventRecord(b);
        cudaError_t e3 = cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("  grid %d mode %s: %.3f us/barrier (%s / %s / %s)\n", ncl * cs, mode == 0 ? "grid-sw" : "cluster-hw",
               ms * 1e3 / iters, cudaGetErrorString(e1), cudaGetErrorString(e2), cudaGetErrorString(e3));
      }
    }
  }
  return 0;
}
