// Shared pieces of the production kernel (hb_mm4.cu) and the halo kernels:
// the Hermitian-packed plane map and the mbarrier / bulk-copy (TMA) helpers.
#pragma once
#include <cstdint>
#include "hb_internal.h"

namespace hb {

template <int D>
struct Pk {  // Hermitian packed planes: diagonal i -> i, upper (i<j) -> D + 2*off
  __host__ __device__ static constexpr int off(int i, int j) {
    int e = 0;
    for (int r = 0; r < i; ++r) e += D - 1 - r;
    return e + (j - i - 1);
  }
  __host__ __device__ static constexpr int re(int i, int j) {
    return i == j ? i : D + 2 * off(i < j ? i : j, i < j ? j : i);
  }
  __host__ __device__ static constexpr int im(int i, int j) {
    return D + 2 * off(i < j ? i : j, i < j ? j : i) + 1;
  }
};

// sigma_{ij} from the packed register copy (i, j compile-time after unrolling)
template <class T, int D>
__device__ __forceinline__ T sre(const T (&s)[D * D], int i, int j) {
  return s[Pk<D>::re(i, j)];
}
template <class T, int D>
__device__ __forceinline__ T sim(const T (&s)[D * D], int i, int j) {
  return i == j ? (T)0 : (i < j ? s[Pk<D>::im(i, j)] : -s[Pk<D>::im(i, j)]);
}
template <int D>
__device__ __forceinline__ double sre(const double (&s)[D * D], int i, int j) {
  return sre<double, D>(s, i, j);
}
template <int D>
__device__ __forceinline__ double sim(const double (&s)[D * D], int i, int j) {
  return sim<double, D>(s, i, j);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "HB_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HB_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace hb
