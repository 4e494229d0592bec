// Micro-benchmark: cost of a software grid barrier (atomic arrive + acquire spin)
// for small cooperative grids.  nvcc -O3 -arch=sm_100a gridbar.cu -o gridbar
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int SLEEP>
__global__ void k_bar(unsigned* bar, int iters) {
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned gen = ld_acquire(bar + 1);
      __threadfence();
      if (atomicAdd(bar, 1u) == gridDim.x - 1) {
        bar[0] = 0;
        __threadfence();
        st_release(bar + 1, gen + 1);
      } else {
        while (ld_acquire(bar + 1) == gen) {
          if (SLEEP) __nanosleep(SLEEP);
        }
      }
    }
    __syncthreads();
  }
}

int main() {
  unsigned* bar;
  cudaMalloc(&bar, 8);
  for (int grid : {11, 54, 148}) {
    for (int sleep : {0, 32}) {
      cudaMemset(bar, 0, 8);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      int iters = 20000;
      void* args[] = {&bar, &iters};
      auto k = sleep ? (void*)k_bar<32> : (void*)k_bar<0>;
      cudaLaunchCooperativeKernel(k, grid, 224, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel(k, grid, 224, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %3d sleep %2d: %.3f us per barrier (%s)\n", grid, sleep, 1e3 * ms / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
