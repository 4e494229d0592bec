// Micro-benchmark: L2 (LTS) throughput of the whole chip on B200, the ceiling of
// the gather-heavy stage kernels.  Every SM streams 16-byte loads (ld.global.cg:
// L1 bypassed, every request served by L2) over a buffer that fits in L2, and
// optionally a 16-byte-granular random gather pattern like k_mm4's link loads.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a l2bw.cu -o l2bw && ./l2bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_stream(const double2* __restrict__ a, size_t n, int reps, double* out) {
  double acc = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      const double2 v = __ldcg(a + i);
      acc += v.x + v.y;
    }
  if (acc == 12345.678) out[0] = acc;  // keep the loads
}

// each thread gathers 16-byte pairs at pseudo-random pair indices (a 32-byte
// sector holds two of them, as in the Hermitian tile layout)
__global__ void k_gather(const double2* __restrict__ a, size_t n, int reps, double* out) {
  double acc = 0.0;
  unsigned x = 2463534242u ^ (blockIdx.x * 9781u + threadIdx.x * 6271u);
  for (int r = 0; r < reps; ++r) {
#pragma unroll 8
    for (int k = 0; k < 64; ++k) {
      x ^= x << 13;
      x ^= x >> 17;
      x ^= x << 5;
      const double2 v = __ldcg(a + (x % n));
      acc += v.x + v.y;
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 48ull << 20;  // well inside the 126 MB L2
  const size_t n = bytes / sizeof(double2);
  double2* a;
  double* out;
  cudaMalloc(&a, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bpsm : {4, 8, 16}) {
    const int grid = sms * bpsm, block = 256;
    const int reps = 40;
    k_stream<<<grid, block>>>(a, n, 2, out);
    cudaEventRecord(e0);
    k_stream<<<grid, block>>>(a, n, reps, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("stream  %2d CTAs/SM x 256: %.0f GB/s\n", bpsm, (double)bytes * reps / (ms * 1e6));
    const int greps = 40;
    k_gather<<<grid, block>>>(a, n, 2, out);
    cudaEventRecord(e0);
    k_gather<<<grid, block>>>(a, n, greps, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double gb = (double)grid * block * greps * 64 * 16;
    printf("gather  %2d CTAs/SM x 256: %.0f GB/s useful (16 B of each 32-B sector)\n", bpsm,
           gb / (ms * 1e6));
  }
  return 0;
}
