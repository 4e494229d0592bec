// Compressed halo exchange for sharded propagation.
//
// A shard's stage kernel reads, from a neighbour ADO reached through mode m,
// only the cross of site(m): the 2d-1 Hermitian-packed planes of row/column
// site(m) (_kernels.py:41-57 reads element (i,j) of a neighbour only when i or
// j is that mode's site).  So instead of whole tiles (32 ADOs x d^2 planes) a
// consumer needs, per halo ADO, just the crosses of the sites it reaches it
// through: entries (device position t, site s), 13 doubles each at d = 7.
// At N_max = 8, K = 1 that cuts the halo ~3.7x (62.5 -> 17 MB per
// stage per GPU at P = 8).
//   pack   : owner, entries of one send segment -> contiguous [entry][plane]
//   unpack : consumer, contiguous -> the same planes of its full-size buffer
// Positions are shard-local slots: the owner packs from its owned slots, the
// consumer unpacks into its halo slots (both list a segment's entries in the
// same order).
#include "hb_internal.h"

namespace hb {

template <class T>
__global__ void k_halo_pack(const T* __restrict__ buf, int n, const int32_t* __restrict__ pos,
                            const int32_t* __restrict__ site, const int16_t* __restrict__ planes,
                            int nc, int n_planes, int d, T* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * nc) return;
  const int e = (int)(idx / nc), q = (int)(idx % nc);
  const int t = pos[e];
  const int p = planes[site[e] * nc + q];
  HB_CHECK(t >= 0 && p >= 0 && p < n_planes);
  out[idx] = buf[(size_t)(t >> 5) * n_planes * TILE + herm_off(d, p, t & 31)];
}

template <class T>
__global__ void k_halo_unpack(T* __restrict__ buf, int n, const int32_t* __restrict__ pos,
                              const int32_t* __restrict__ site, const int16_t* __restrict__ planes,
                              int nc, int n_planes, int d, const T* __restrict__ in) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * nc) return;
  const int e = (int)(idx / nc), q = (int)(idx % nc);
  const int t = pos[e];
  const int p = planes[site[e] * nc + q];
  HB_CHECK(t >= 0 && p >= 0 && p < n_planes);
  buf[(size_t)(t >> 5) * n_planes * TILE + herm_off(d, p, t & 31)] = in[idx];
}

// in-process shards: the divergence max over the shards' control blocks (the
// bit patterns of non-negative doubles order like the doubles), written back to
// every block so that each shard's step bookkeeping sees the global value
struct GuardPtrs {
  unsigned long long* p[64];
  int n;
};

__global__ void k_guard_max(GuardPtrs g) {
  if (threadIdx.x != 0) return;
  unsigned long long m = 0;
  for (int i = 0; i < g.n; ++i) {
    const unsigned long long v = *(volatile unsigned long long*)g.p[i];
    m = v > m ? v : m;
  }
  for (int i = 0; i < g.n; ++i) *(volatile unsigned long long*)g.p[i] = m;
}

cudaError_t launch_guard_max(unsigned long long* const* bits, int n, cudaStream_t s) {
  if (n < 1 || n > 64) return cudaErrorInvalidValue;
  GuardPtrs g{};
  for (int i = 0; i < n; ++i) g.p[i] = bits[i];
  g.n = n;
  k_guard_max<<<1, 32, 0, s>>>(g);
  return cudaGetLastError();
}

static unsigned blocks(int n, int nc) { return (unsigned)(((int64_t)n * nc + 255) / 256); }

cudaError_t launch_halo(int op, bool single, void* dst, const void* src, int n, const int32_t* pos,
                        const int32_t* site, const int16_t* planes, int nc, int n_planes,
                        void* packed, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int d = (nc + 1) / 2;  // nc = 2d - 1 planes per cross (Hermitian layout)
  const unsigned g = blocks(n, nc);
  if (single) {
    using T = float;
    if (op == 0) k_halo_pack<T><<<g, 256, 0, s>>>((const T*)src, n, pos, site, planes, nc, n_planes, d, (T*)packed);
    if (op == 1) k_halo_unpack<T><<<g, 256, 0, s>>>((T*)dst, n, pos, site, planes, nc, n_planes, d, (const T*)packed);
  } else {
    using T = double;
    if (op == 0) k_halo_pack<T><<<g, 256, 0, s>>>((const T*)src, n, pos, site, planes, nc, n_planes, d, (T*)packed);
    if (op == 1) k_halo_unpack<T><<<g, 256, 0, s>>>((T*)dst, n, pos, site, planes, nc, n_planes, d, (const T*)packed);
  }
  return cudaGetLastError();
}

}  // namespace hb
