// Microbenchmark: cost of a software grid barrier (148 co-resident CTAs) on B200.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

struct GB { unsigned int count, gen; };
__device__ __forceinline__ unsigned int ld_acq(const unsigned int* p) { unsigned int v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_rel(unsigned int* p, unsigned int v) { asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ unsigned int atom_add_acqrel(unsigned int* p, unsigned int v) { unsigned int o; asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory"); return o; }

template <int MODE>
__global__ void kbar(GB* gb, int iters, double* part, double* out) {
  const unsigned nb = gridDim.x;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 3) { cg::this_grid().sync(); continue; }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (MODE == 4) part[blockIdx.x] = it;  // write a partial
      unsigned g = ld_acq(&gb->gen);
      if (MODE == 0) __threadfence();
      unsigned a = (MODE == 0) ? atomicAdd(&gb->count, 1u) : atom_add_acqrel(&gb->count, 1u);
      if (a == nb - 1) { gb->count = 0; if (MODE == 0) __threadfence(); st_rel(&gb->gen, g + 1); }
      else { while (ld_acq(&gb->gen) == g) {} }
      if (MODE == 0) __threadfence();
    }
    __syncthreads();
    if (MODE == 4 && threadIdx.x < 32) {  // read all partials
      double s = 0; for (int b = threadIdx.x; b < nb; b += 32) s += __ldcg(part + b);
      acc += s;
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

int main() {
  GB* gb; cudaMalloc(&gb, 64); cudaMemset(gb, 0, 64);
  double *part, *out; cudaMalloc(&part, 8 * 1024); cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 20000;
  for (int mode = 0; mode < 5; ++mode) {
    for (int threads : {256, 512}) {
      void* args[] = {&gb, &iters, &part, &out};
      const void* f = mode == 0 ? (const void*)kbar<0> : mode == 1 ? (const void*)kbar<1> : mode == 3 ? (const void*)kbar<3> : (const void*)kbar<4>;
      if (mode == 2) continue;
      cudaLaunchCooperativeKernel(f, sms, threads, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel(f, sms, threads, args, 0, 0);
      cudaEventRecord(b);
      cudaError_t e = cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("mode %d threads %d: %.3f us/barrier (%s)\n", mode, threads, ms * 1e3 / iters, cudaGetErrorString(e));
    }
  }
  return 0;
}
