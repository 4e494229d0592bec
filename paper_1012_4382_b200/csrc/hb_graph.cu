// Device hierarchy builder: multi-index enumeration and raise/lower neighbour
// tables (replaces hierarchy.py:59-105 enumerate_hierarchy).
//
// Instead of the reference's tuple dictionary every thread ranks / unranks its
// multi-index with a binomial table (combinatorial number system), so the
// tables are built in O(n_tot * modes * n_max) fully parallel work.
//
// Two orders exist:
//  * reference order -- tier-major, lexicographic ascending within a tier
//    (hierarchy.py:71-78); the exported tables are always in this order and must
//    match the reference bit for bit;
//  * device order HB_ORDER_LEX -- pure lexicographic over all tiers.  Adding e_m
//    preserves lexicographic order, so every raise/lower map is monotone, and
//    the neighbour via the last modes is a few positions away: gathers of a warp
//    stay inside a few sectors and the reuse distance of a gathered ADO is far
//    shorter than in tier-major order (hard part 1).
//  * device order HB_ORDER_LEX_SPLIT -- the same tiles as HB_ORDER_LEX, but
//    inside every tile the ADOs below the top tier come first and the top-tier
//    ones (whose raise links are all TRUNCATED) after them, each group in
//    lexicographic order (ADO 0 stays at position 0).  A warp's valid raise
//    (and, mostly, lower) links then sit on adjacent lanes, so a gathered plane
//    of its 32 neighbours touches fewer 32-byte sectors: 3.9 instead of 5.1 per
//    ADO and plane load at N_max = 8, K = 1 (65 % instead of 50 % useful).
#include <vector>
#include <cstring>
#include "hb_internal.h"

namespace hb {

int64_t hierarchy_size(int modes, int n_max) {
  if (modes < 0 || n_max < 0) return 0;
  // C(modes + n_max, modes) with overflow detection
  __int128 r = 1;
  int k = modes < n_max ? modes : n_max;
  int64_t n = (int64_t)modes + n_max;
  for (int i = 1; i <= k; ++i) {
    r = r * (n - k + i) / i;
    if (r > (__int128)INT64_MAX) return -1;
  }
  return (int64_t)r;
}

// S(q, B) = C(q + B, q) = |{n in N^q : |n| <= B}|, table [q][B]
static std::vector<int64_t> simplex_table(int modes, int n_max) {
  std::vector<int64_t> S((size_t)(modes + 1) * (n_max + 1));
  for (int q = 0; q <= modes; ++q)
    for (int B = 0; B <= n_max; ++B) {
      int64_t v = hierarchy_size(q, B);
      S[(size_t)q * (n_max + 1) + B] = v < 0 ? INT64_MAX : v;
    }
  return S;
}

struct Comb {
  const int64_t* S;
  int M, N1;
  __device__ int64_t s(int q, int B) const { return B < 0 ? 0 : S[q * N1 + B]; }
  // compositions of x into q parts
  __device__ int64_t comp(int x, int q) const {
    if (x < 0) return 0;
    if (q == 0) return x == 0 ? 1 : 0;
    return s(q - 1, x);
  }
  __device__ int64_t graded_offset(int t) const { return t == 0 ? 0 : s(M, t - 1); }

  __device__ void lex_unrank(int64_t r, int N, int* n) const {
    int B = N;
    for (int i = 0; i < M - 1; ++i) {
      int v = 0;
      for (;; ++v) {
        int64_t c = s(M - i - 1, B - v);
        if (r < c) break;
        r -= c;
      }
      n[i] = v;
      B -= v;
    }
    n[M - 1] = (int)r;
  }
  __device__ int64_t lex_rank(const int* n, int N) const {
    int64_t r = 0;
    int B = N;
    for (int i = 0; i < M; ++i) {
      for (int v = 0; v < n[i]; ++v) r += s(M - i - 1, B - v);
      B -= n[i];
    }
    return r;
  }
  __device__ void graded_unrank(int64_t k, int N, int* n) const {
    int t = 0;
    while (t < N && graded_offset(t + 1) <= k) ++t;
    int64_t r = k - graded_offset(t);
    int R = t;
    for (int i = 0; i < M - 1; ++i) {
      int v = 0;
      for (;; ++v) {
        int64_t c = comp(R - v, M - i - 1);
        if (r < c) break;
        r -= c;
      }
      n[i] = v;
      R -= v;
    }
    n[M - 1] = R;
  }
  __device__ int64_t graded_rank(const int* n) const {
    int t = 0;
    for (int i = 0; i < M; ++i) t += n[i];
    int64_t r = graded_offset(t);
    int R = t;
    for (int i = 0; i < M - 1; ++i) {
      for (int v = 0; v < n[i]; ++v) r += comp(R - v, M - i - 1);
      R -= n[i];
    }
    return r;
  }
};

__global__ void k_build_ref(Comb cb, int N, int n_tot, int32_t* indices, int32_t* tiers,
                            int32_t* plus, int32_t* minus, int32_t* ref2dev) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_tot) return;
  const int M = cb.M;
  int n[MAX_MODES];
  cb.graded_unrank(k, N, n);
  int t = 0;
  for (int m = 0; m < M; ++m) t += n[m];
  if (tiers) tiers[k] = t;
  for (int m = 0; m < M; ++m) {
    if (indices) indices[(int64_t)k * M + m] = n[m];
    int32_t p = -1, q = -2;   // TRUNCATED / ABSENT (hierarchy.py:18-21)
    if (t < N) {
      n[m] += 1;
      p = (int32_t)cb.graded_rank(n);
      n[m] -= 1;
    }
    if (n[m] > 0) {
      n[m] -= 1;
      q = (int32_t)cb.graded_rank(n);
      n[m] += 1;
    }
    if (plus) plus[(int64_t)k * M + m] = p;
    if (minus) minus[(int64_t)k * M + m] = q;
  }
  if (ref2dev) ref2dev[k] = (int32_t)cb.lex_rank(n, N);
}

// HB_ORDER_LEX_SPLIT: per tile, the lexicographic lanes that are real ADOs and
// the subset of those on the top tier (one warp = one tile of lex positions)
__global__ void k_split_masks(Comb cb, int N, int n_tot, int n_pad, uint32_t* real_mask,
                              uint32_t* top_mask) {
  const int L = blockIdx.x * blockDim.x + threadIdx.x;
  if (L >= n_pad) return;  // n_pad is a multiple of 32: whole warps return
  bool top = false;
  const bool real = L < n_tot;
  if (real) {
    int n[MAX_MODES];
    cb.lex_unrank(L, N, n);
    int t = 0;
    for (int m = 0; m < cb.M; ++m) t += n[m];
    top = t == N;
  }
  const uint32_t rm = __ballot_sync(0xffffffffu, real), tm = __ballot_sync(0xffffffffu, top);
  if ((threadIdx.x & 31) == 0) {
    real_mask[L >> 5] = rm;
    top_mask[L >> 5] = tm;
  }
}

struct SplitOrder {
  const uint32_t* real;
  const uint32_t* top;
  // lexicographic position -> device position
  __device__ int dev(int L) const {
    const int T = L >> 5, l = L & 31;
    const uint32_t below = (1u << l) - 1u;
    const uint32_t lo = real[T] & ~top[T], hi = top[T];
    const int nlo = __popc(lo);
    const int lane = (lo >> l) & 1u ? __popc(lo & below) : nlo + __popc(hi & below);
    return T * 32 + lane;
  }
  // device position -> lexicographic position (-1: padding)
  __device__ int lex(int r) const {
    const int T = r >> 5, j = r & 31;
    const uint32_t lo = real[T] & ~top[T], hi = top[T];
    const int nlo = __popc(lo), nhi = __popc(hi);
    if (j < nlo) return T * 32 + (__fns(lo, 0, j + 1));
    if (j < nlo + nhi) return T * 32 + (__fns(hi, 0, j - nlo + 1));
    return -1;
  }
};

__global__ void k_build_dev(Comb cb, int N, int n_tot, int n_pad, int ordering, SplitOrder so,
                            int32_t* plus_t, int32_t* minus_t, uint8_t* nvec_t, int32_t* dev2ref) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_pad) return;
  const int M = cb.M;
  const int64_t base = (int64_t)(r >> 5) * M * TILE + (r & 31);
  const bool split = ordering == HB_ORDER_LEX_SPLIT;
  const int L = split ? so.lex(r) : r;  // the ADO at device position r, lex rank
  if (r >= n_tot || L < 0) {  // padding lanes: no links, n = 0 -> the state stays zero
    for (int m = 0; m < M; ++m) {
      plus_t[base + m * TILE] = -1;
      minus_t[base + m * TILE] = -2;
      nvec_t[base + m * TILE] = 0;
    }
    dev2ref[r] = -1;
    return;
  }
  int n[MAX_MODES];
  const bool lex = ordering == HB_ORDER_LEX || split;
  if (lex) cb.lex_unrank(L, N, n); else cb.graded_unrank(r, N, n);
  auto pos = [&](const int* v) -> int32_t {
    if (!lex) return (int32_t)cb.graded_rank(v);
    const int64_t lr = cb.lex_rank(v, N);
    return split ? (int32_t)so.dev((int)lr) : (int32_t)lr;
  };
  int t = 0;
  for (int m = 0; m < M; ++m) t += n[m];
  for (int m = 0; m < M; ++m) {
    int32_t p = -1, q = -2;
    if (t < N) {
      n[m] += 1;
      p = pos(n);
      n[m] -= 1;
    }
    if (n[m] > 0) {
      n[m] -= 1;
      q = pos(n);
      n[m] += 1;
    }
    plus_t[base + m * TILE] = p;
    minus_t[base + m * TILE] = q;
    nvec_t[base + m * TILE] = (uint8_t)n[m];
  }
  dev2ref[r] = (int32_t)cb.graded_rank(n);
}

void free_graph(GraphTables* gt) {
  if (!gt) return;
  cudaFree(gt->plus_t);
  cudaFree(gt->minus_t);
  cudaFree(gt->nvec_t);
  cudaFree(gt->dev2ref);
  gt->plus_t = gt->minus_t = nullptr;
  gt->nvec_t = nullptr;
  gt->dev2ref = nullptr;
}

#define HB_TRY(x)                      \
  do {                                 \
    cudaError_t e_ = (x);              \
    if (e_ != cudaSuccess) return e_;  \
  } while (0)

cudaError_t build_graph(int modes, int n_max, int ordering, cudaStream_t s, int32_t* h_indices,
                        int32_t* h_tiers, int32_t* h_plus, int32_t* h_minus, int32_t* h_perm,
                        GraphTables* gt) {
  const int64_t n_tot64 = hierarchy_size(modes, n_max);
  const int n_tot = (int)n_tot64;
  std::vector<int64_t> S = simplex_table(modes, n_max);
  int64_t* dS = nullptr;
  HB_TRY(cudaMalloc(&dS, S.size() * sizeof(int64_t)));
  HB_TRY(cudaMemcpyAsync(dS, S.data(), S.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  Comb cb{dS, modes, n_max + 1};
  const int threads = 128;
  cudaError_t err = cudaSuccess;
  if (h_indices || h_tiers || h_plus || h_minus || h_perm) {
    const size_t tab = (size_t)n_tot * modes * sizeof(int32_t);
    int32_t *d_ind = nullptr, *d_tiers = nullptr, *d_plus = nullptr, *d_minus = nullptr,
            *d_perm = nullptr;
    if (h_indices) err = err ? err : cudaMalloc(&d_ind, tab);
    if (h_tiers) err = err ? err : cudaMalloc(&d_tiers, (size_t)n_tot * sizeof(int32_t));
    if (h_plus) err = err ? err : cudaMalloc(&d_plus, tab);
    if (h_minus) err = err ? err : cudaMalloc(&d_minus, tab);
    if (h_perm) err = err ? err : cudaMalloc(&d_perm, (size_t)n_tot * sizeof(int32_t));
    if (!err) {
      k_build_ref<<<(n_tot + threads - 1) / threads, threads, 0, s>>>(
          cb, n_max, n_tot, d_ind, d_tiers, d_plus, d_minus, d_perm);
      err = cudaGetLastError();
    }
    if (!err && h_indices) err = cudaMemcpyAsync(h_indices, d_ind, tab, cudaMemcpyDeviceToHost, s);
    if (!err && h_tiers)
      err = cudaMemcpyAsync(h_tiers, d_tiers, (size_t)n_tot * 4, cudaMemcpyDeviceToHost, s);
    if (!err && h_plus) err = cudaMemcpyAsync(h_plus, d_plus, tab, cudaMemcpyDeviceToHost, s);
    if (!err && h_minus) err = cudaMemcpyAsync(h_minus, d_minus, tab, cudaMemcpyDeviceToHost, s);
    if (!err && h_perm)
      err = cudaMemcpyAsync(h_perm, d_perm, (size_t)n_tot * 4, cudaMemcpyDeviceToHost, s);
    if (!err) err = cudaStreamSynchronize(s);
    cudaFree(d_ind);
    cudaFree(d_tiers);
    cudaFree(d_plus);
    cudaFree(d_minus);
    cudaFree(d_perm);
  }
  if (!err && gt) {
    gt->modes = modes;
    gt->n_max = n_max;
    gt->n_tot = n_tot;
    gt->n_tiles = (n_tot + TILE - 1) / TILE;
    const int n_pad = gt->n_tiles * TILE;
    const size_t tab = (size_t)n_pad * modes;
    err = cudaMalloc(&gt->plus_t, tab * sizeof(int32_t));
    if (!err) err = cudaMalloc(&gt->minus_t, tab * sizeof(int32_t));
    if (!err) err = cudaMalloc(&gt->nvec_t, tab);
    if (!err) err = cudaMalloc(&gt->dev2ref, (size_t)n_pad * sizeof(int32_t));
    uint32_t* masks = nullptr;
    SplitOrder so{nullptr, nullptr};
    if (!err && ordering == HB_ORDER_LEX_SPLIT) {
      err = cudaMalloc(&masks, (size_t)2 * gt->n_tiles * sizeof(uint32_t));
      if (!err) {
        so = SplitOrder{masks, masks + gt->n_tiles};
        k_split_masks<<<(n_pad + threads - 1) / threads, threads, 0, s>>>(
            cb, n_max, n_tot, n_pad, masks, masks + gt->n_tiles);
        err = cudaGetLastError();
      }
    }
    if (!err) {
      k_build_dev<<<(n_pad + threads - 1) / threads, threads, 0, s>>>(
          cb, n_max, n_tot, n_pad, ordering, so, gt->plus_t, gt->minus_t, gt->nvec_t,
          gt->dev2ref);
      err = cudaGetLastError();
    }
    if (!err) err = cudaStreamSynchronize(s);
    cudaFree(masks);
  }
  cudaFree(dS);
  return err;
}

cudaError_t upload_tables(int modes, int n_tot, const int32_t* plus, const int32_t* minus,
                          const uint8_t* nvec, cudaStream_t s, GraphTables* gt) {
  gt->modes = modes;
  gt->n_tot = n_tot;
  gt->n_tiles = (n_tot + TILE - 1) / TILE;
  const int n_pad = gt->n_tiles * TILE;
  const size_t tab = (size_t)n_pad * modes;
  std::vector<int32_t> p(tab), q(tab), perm(n_pad);
  std::vector<uint8_t> nv(tab);
  for (int r = 0; r < n_pad; ++r) {
    const size_t base = (size_t)(r >> 5) * modes * TILE + (r & 31);
    perm[r] = r < n_tot ? r : -1;
    for (int m = 0; m < modes; ++m) {
      const bool ok = r < n_tot;
      p[base + (size_t)m * TILE] = ok ? plus[(size_t)r * modes + m] : -1;
      q[base + (size_t)m * TILE] = ok ? minus[(size_t)r * modes + m] : -2;
      nv[base + (size_t)m * TILE] = ok ? nvec[(size_t)r * modes + m] : 0;
    }
  }
  HB_TRY(cudaMalloc(&gt->plus_t, tab * sizeof(int32_t)));
  HB_TRY(cudaMalloc(&gt->minus_t, tab * sizeof(int32_t)));
  HB_TRY(cudaMalloc(&gt->nvec_t, tab));
  HB_TRY(cudaMalloc(&gt->dev2ref, (size_t)n_pad * sizeof(int32_t)));
  HB_TRY(cudaMemcpyAsync(gt->plus_t, p.data(), tab * 4, cudaMemcpyHostToDevice, s));
  HB_TRY(cudaMemcpyAsync(gt->minus_t, q.data(), tab * 4, cudaMemcpyHostToDevice, s));
  HB_TRY(cudaMemcpyAsync(gt->nvec_t, nv.data(), tab, cudaMemcpyHostToDevice, s));
  HB_TRY(cudaMemcpyAsync(gt->dev2ref, perm.data(), (size_t)n_pad * 4, cudaMemcpyHostToDevice, s));
  return cudaStreamSynchronize(s);
}

}  // namespace hb
