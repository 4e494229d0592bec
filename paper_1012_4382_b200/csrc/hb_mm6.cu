// Experimental stage kernel (variant 9, k_mm6): k_mm4's arithmetic in CTAs of
// W warps that own a CONTIGUOUS tile range (HB_MM6_R tiles per warp, or
// persistent: one CTA per SM).
//
// The no-gather timing experiment (k_mm4 VAR 5, profiles/) put the streamed
// part of a step at the HBM floor (0.26 ms) and the neighbour gathers at
// +0.17 ms: ~1.6 KB per ADO and stage of L2->SM sectors, 20% L1 hits.  With
// one-warp CTAs the hardware scatters consecutive tiles over all SMs, so the
// links that stay close in the lexicographic order (the last ~5 of the 14
// modes reach < 128 ADOs = 4 tiles away) land in another SM's L1.  Here one
// CTA of W warps owns tiles [t0, t1) of the stage; warp w takes t0 + w,
// t0 + w + W, ...: the W warps of an SM sweep the range side by side, so a
// near neighbour is the SM's own current or recent tile -- an L1 hit.
// Per warp and tile: bulk copy of links + base (one mbarrier, phase flips per
// tile), phase A (commutator, damping), phase B (site crosses), phase C
// (store); the last CTA of stage 4 runs the step bookkeeping.
#include <algorithm>
#include <cstdlib>
#include "hb_device.cuh"
#include "hb_fast.cuh"
#include "hb_mm_common.cuh"

namespace hb {

// dynamic shared memory of one CTA: per warp the base tile, the link tables, n
template <int D, int KP1, int STAGE, int W>
struct Mm6Smem {
  static constexpr int M = D * KP1, NB = STAGE >= 2 ? D * D : 1;
  static constexpr size_t BASE = 0;
  static constexpr size_t UP = BASE + (size_t)W * NB * TILE * 8;
  static constexpr size_t DN = UP + (size_t)W * M * TILE * 4;
  static constexpr size_t N = DN + (size_t)W * M * TILE * 4;
  static constexpr size_t BAR = (N + (size_t)W * M * TILE + 15) / 16 * 16;
  static constexpr size_t BYTES = BAR + 8 * W;
};

template <int D, int KP1, int STAGE, int W>
__global__ void __launch_bounds__(32 * W, 8 / W) k_mm6(const KParams P) {
  constexpr int NP = D * D;
  constexpr int M = D * KP1;
  constexpr int TB = NP * TILE;
  using L = Mm6Smem<D, KP1, STAGE, W>;
  extern __shared__ __align__(128) unsigned char smem[];
  auto sBase = reinterpret_cast<double(*)[L::NB][TILE]>(smem + L::BASE);
  auto sUp = reinterpret_cast<int32_t(*)[M][TILE]>(smem + L::UP);
  auto sDn = reinterpret_cast<int32_t(*)[M][TILE]>(smem + L::DN);
  auto sN = reinterpret_cast<uint8_t(*)[M][TILE]>(smem + L::N);
  auto bar = reinterpret_cast<uint64_t*>(smem + L::BAR);

  volatile Ctl* ctl = P.ctl;
  if (ctl->status != ST_RUNNING) return;
  const long long step_next = ctl->step + 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t0 = (int)((long long)P.n_tiles * blockIdx.x / gridDim.x);
  const int t1 = (int)((long long)P.n_tiles * (blockIdx.x + 1) / gridDim.x);
  const double c = STAGE == 4 ? P.dt / 6.0 : P.coef;
  double maxa2 = 0.0;
  unsigned it = 0;
  for (int t = t0 + w; t < t1; t += W, ++it) {
    const int tile = P.tile_begin + t;
    const int own = tile * TB + lane;
    tile_prologue<double, D, KP1, STAGE>(P, tile, &sBase[w][0][0], &sUp[w][0][0], &sDn[w][0][0],
                                 &sN[w][0][0], &bar[w], it == 0);
    double acc[NP];
    phase_a<double, D, KP1, STAGE>(P, tile, lane, own, c, sBase[w], sN[w], &bar[w], acc, it & 1u);
    phase_b_sites<double, D, KP1>(P, lane, c, sUp[w], sDn[w], sN[w], acc);
    phase_c_store<double, D, STAGE>(P, lane, own, sBase[w], acc, maxa2);
    __syncwarp();  // every lane done with this tile's shared memory before the refill
  }
  if (STAGE == 4) stage4_finish<D>(P, step_next, maxa2);
}

static int num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <int D, int KP1, int STAGE, int W>
static cudaError_t mm6_go(int grid, const KParams& p, cudaStream_t s) {
  constexpr size_t bytes = Mm6Smem<D, KP1, STAGE, W>::BYTES;
  static const cudaError_t attr = cudaFuncSetAttribute(
      k_mm6<D, KP1, STAGE, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (attr != cudaSuccess) return attr;
  k_mm6<D, KP1, STAGE, W><<<grid, 32 * W, bytes, s>>>(p);
  return cudaGetLastError();
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

template <int D, int KP1, int W>
static cudaError_t mm6_launch_w(int stage, const KParams& p, cudaStream_t s) {
  // HB_MM6_R (experiments): tiles per warp; 0 = persistent, one CTA per SM
  static const int r = env_int("HB_MM6_R", 1);
  const int grid = r > 0 ? std::max(1, (p.n_tiles + W * r - 1) / (W * r))
                         : std::max(1, std::min(num_sms(), (p.n_tiles + W - 1) / W));
  switch (stage) {
    case 1: return mm6_go<D, KP1, 1, W>(grid, p, s);
    case 2: return mm6_go<D, KP1, 2, W>(grid, p, s);
    case 3: return mm6_go<D, KP1, 3, W>(grid, p, s);
    case 4: return mm6_go<D, KP1, 4, W>(grid, p, s);
  }
  return cudaErrorInvalidValue;
}

template <int D, int KP1>
static cudaError_t mm6_launch_t(int stage, const KParams& p, cudaStream_t s) {
  // HB_MM6_W (experiments): warps (adjacent tiles) per CTA
  static const int w = env_int("HB_MM6_W", 4);
  if constexpr (D == 7 && KP1 == 2) {
    if (w == 2) return mm6_launch_w<D, KP1, 2>(stage, p, s);
    if (w == 8) return mm6_launch_w<D, KP1, 8>(stage, p, s);
  }
  return mm6_launch_w<D, KP1, 4>(stage, p, s);
}

cudaError_t launch_mm6(int stage, const KParams& p, cudaStream_t s) {
  // experiment: instantiated for the FMO shape only (others run k_mm4)
  if (p.d == 7 && p.kp1 == 2 && !p.single) return mm6_launch_t<7, 2>(stage, p, s);
  return launch_mm4(stage, p, s);
}

}  // namespace hb
