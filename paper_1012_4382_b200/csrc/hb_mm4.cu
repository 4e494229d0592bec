// Production stage kernel (variant 7, k_mm4): k_mm3's 12-pass RK bookkeeping
// and register accumulator, re-cut for occupancy and FP64 issue.
//
// What the k_mm3 ncu capture (profiles/r1_ncu_k_mm3.json) showed: 254
// registers -> 8 warps per SM, long-scoreboard stalls ~2.5 per issue, and
// 1,878 FP64 instructions per tile-stage of which 679 DADD and 469 DMUL (the
// `a*b - c*d` forms were not contracted), plus 350 CS2R zeroing the
// predicated-off gathers.  Here:
//   * every RHS term is one explicit DFMA into the register accumulator: the
//     RK stage coefficient c is folded into the link coefficients once per link
//     (c*n*b_k, c*n*a_k, and c for a raise link), so nothing is scaled twice;
//   * an absent link (TRUNCATED raise at the top tier, ABSENT lower where
//     n_m = 0) is predicated off (measured: redirecting it to the own ADO with
//     a zero coefficient, or prefetching the next site into L1, is slower);
//   * the tile's base operand (sigma, or B at stage 4) and its three link
//     tables ([mode][32] int32 raise/lower, uint8 n) arrive by one bulk copy
//     group (cp.async.bulk, one mbarrier) at kernel start: no per-lane table
//     LDG/STS round trip, the raw positions are decoded to element offsets
//     where they are used;
//   * a tile none of whose lanes has a raise link (every top-tier tile of the
//     tier-major order) gathers two sites' lower links per round trip
//     (phase_b_sites<PAIRED>): 4 dependent L2 round trips instead of 7.
// T = double (HB_PREC_DOUBLE) or float (HB_PREC_SINGLE: float state, float RHS,
// heom.py:93-94; bookkeeping, sinks and records stay double).
// The arithmetic is the reference RHS (_kernels.py:23-58 generalised to K+1
// modes per site); the stage combinations are k_mm2's (hb_fast.cu):
//   stage 1: Y2 = s + h/2 k1;  2: Y3 = s + h/2 k2, B = (Y2 - s)/3 + 2/3 Y3;
//   stage 3: Y4 = s + h k3;    4: s = B + Y4/3 + h/6 k4          (heom.py:370-381)
#include <cstdlib>
#include "hb_device.cuh"
#include "hb_fast.cuh"
#include "hb_mm_common.cuh"

namespace hb {

// VAR (experiments, HB_MM4_VAR): 1 = production; 5 = skip the neighbour crosses
// (timing experiment for the streamed part alone; wrong results); 6 = production
// with an idle second warp per CTA (half the resident working warps, same L1);
// 7 = base operands read in phase C instead of bulk-copied to shared memory;
// 8 = registers capped for 12 resident warps per SM (float path);
// 9 = production (paired-site rounds for tiles without raise links are part of
// every production variant; 7 runs without them; three sites per round measured
// the same as two).
template <class T, int D, int KP1, int STAGE, int VAR>
__global__ void __launch_bounds__(VAR == 6 ? 64 : 32, VAR == 8 ? 12 : 1) k_mm4(const KParams P) {
  constexpr int NP = D * D;
  constexpr int M = D * KP1;
  constexpr int TB = NP * TILE;
  constexpr bool kInc = kIncScheme<T>;
  constexpr bool kLate = VAR == 7 && !kInc;  // base operands in phase C (no smem tile)
  __shared__ __align__(128) T sBase[(STAGE >= 2 && !kLate) || kInc ? NP : 1][TILE];
  __shared__ __align__(128) T sInc[kInc && (STAGE == 2 || STAGE == 4) ? NP : 1][TILE];
  __shared__ __align__(16) int32_t sUp[M][TILE];
  __shared__ __align__(16) int32_t sDn[M][TILE];
  __shared__ __align__(16) uint8_t sN[M][TILE];
  __shared__ __align__(8) uint64_t bar;

  volatile Ctl* ctl = P.ctl;
  if (VAR == 6 && threadIdx.x >= 32) {  // occupancy experiment: an idle 2nd warp
    if (STAGE == 4) {
      pdl_wait();
      if (ctl->status == ST_RUNNING) stage4_finish<D>(P, ctl->step + 1, 0.0);
    }
    return;
  }
  const int lane = threadIdx.x;
  const int tile = P.tile_begin + blockIdx.x;
  const int own = tile * TB + lane;  // element offset of this lane's ADO, plane 0
  const T c = (T)(STAGE == 4 ? P.dt / 6.0 : P.coef);

  // operands no running kernel writes, before the grid dependency (PDL, see
  // hb_mm_common.cuh); the float increment tile (written by stage 1) after it
  tile_prologue<T, D, KP1, kLate ? 1 : STAGE>(P, tile, &sBase[0][0], &sUp[0][0], &sDn[0][0],
                                               &sN[0][0], &bar, true, &sInc[0][0], true);
  pdl_wait();
  tile_prologue_late<T, D, STAGE>(P, tile, &sInc[0][0], &bar);
  if (ctl->status != ST_RUNNING) {
    mbar_wait(&bar, 0);  // no bulk copy may land after the CTA has exited
    return;
  }
  pdl_release();
  const long long step_next = ctl->step + 1;
  T acc[NP];
  phase_a<T, D, KP1, STAGE, kLate>(P, tile, lane, own, c, sBase, sN, &bar, acc);
  if (VAR != 5) phase_b_sites<T, D, KP1, VAR != 7>(P, lane, c, sUp, sDn, sN, acc);
  double maxa2 = 0.0;
  phase_c_store<T, D, STAGE, kLate>(P, lane, own, sBase, acc, maxa2, sInc);
  if (STAGE == 4) {
    if (VAR == 6) {
      stage4_finish<D>(P, step_next, maxa2);
    } else if (step_next % 25 == 0) {  // the step bookkeeping runs in k_step_finish
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
      if (lane == 0)
        atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                  (unsigned long long)__double_as_longlong(maxa2));
    }
  }
}

// Split CTAs for grids under about one wave (small hierarchies, where a stage is
// the latency of one tile's chain of dependent round trips, not bandwidth): two
// warps per tile.  Warp 0 runs phase A (own ADO, commutator, damping) and the
// crosses of sites [0, D/2); warp 1 gathers sites [D/2, D) into its own
// accumulator and hands it over through shared memory; warp 0 stores.  Same
// arithmetic as k_mm4 (the second accumulator is added once per element before
// the store, so the sum order differs from k_mm4's by that one regrouping).
template <class T, int D, int KP1, int STAGE>
__global__ void __launch_bounds__(64, 1) k_mm4s(const KParams P) {
  constexpr int NP = D * D;
  constexpr int M = D * KP1;
  constexpr int SPLIT = D / 2;
  constexpr bool kInc = kIncScheme<T>;
  __shared__ __align__(128) T sBase[STAGE >= 2 || kInc ? NP : 1][TILE];
  __shared__ __align__(128) T sInc[kInc && (STAGE == 2 || STAGE == 4) ? NP : 1][TILE];
  __shared__ __align__(128) T sX[NP][TILE];
  __shared__ __align__(16) int32_t sUp[M][TILE];
  __shared__ __align__(16) int32_t sDn[M][TILE];
  __shared__ __align__(16) uint8_t sN[M][TILE];
  __shared__ __align__(8) uint64_t bar;

  volatile Ctl* ctl = P.ctl;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tile = P.tile_begin + blockIdx.x;
  const int own = tile * (NP * TILE) + lane;
  const T c = (T)(STAGE == 4 ? P.dt / 6.0 : P.coef);

  if (warp == 0)
    tile_prologue<T, D, KP1, STAGE>(P, tile, &sBase[0][0], &sUp[0][0], &sDn[0][0], &sN[0][0],
                                    &bar, true, &sInc[0][0], true);
  __syncthreads();  // barrier initialised before warp 1 waits on it
  pdl_wait();
  if (warp == 0) tile_prologue_late<T, D, STAGE>(P, tile, &sInc[0][0], &bar);
  if (ctl->status != ST_RUNNING) {
    mbar_wait(&bar, 0);  // no bulk copy may land after the CTA has exited
    return;
  }
  pdl_release();
  const long long step_next = ctl->step + 1;
  T acc[NP];
  if (warp == 0) {
    phase_a<T, D, KP1, STAGE>(P, tile, lane, own, c, sBase, sN, &bar, acc);
    phase_b_sites<T, D, KP1, true, 2, 0, SPLIT>(P, lane, c, sUp, sDn, sN, acc);
  } else {
#pragma unroll
    for (int p = 0; p < NP; ++p) acc[p] = 0;
    mbar_wait(&bar, 0);
    phase_b_sites<T, D, KP1, true, 2, SPLIT, D>(P, lane, c, sUp, sDn, sN, acc);
#pragma unroll
    for (int p = 0; p < NP; ++p) sX[p][lane] = acc[p];
  }
  __syncthreads();
  if (warp != 0) return;
#pragma unroll
  for (int p = 0; p < NP; ++p) acc[p] += sX[p][lane];
  double maxa2 = 0.0;
  phase_c_store<T, D, STAGE, false>(P, lane, own, sBase, acc, maxa2, sInc);
  if (STAGE == 4 && step_next % 25 == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
    if (lane == 0)
      atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                (unsigned long long)__double_as_longlong(maxa2));
  }
}

// The per-step bookkeeping (sinks heom.py:382-383, guard heom.py:386-389,
// records, stop policy) as its own one-warp kernel after stage 4, chained by
// PDL: it waits for the stage-4 grid to complete and flush, so the stage
// kernels need no per-CTA fence and no contended last-CTA election counter
// (each of those cost every CTA a round trip before it could retire).
template <int D>
__global__ void __launch_bounds__(32, 1) k_step_finish(const KParams P) {
  volatile Ctl* ctl = P.ctl;
  pdl_wait();
  if (ctl->status != ST_RUNNING) return;
  pdl_release();
  const long long step_next = ctl->step + 1;
  if (threadIdx.x == 0) ctl->launches = ctl->launches + 5;
  finish_step_warp<D, true>(P, step_next);
}

template <int D>
static cudaError_t finish_go(const KParams& p, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_step_finish<D>, p);
}

// HB_MM4_PAD (experiments): unused dynamic shared memory per CTA, to lower the
// resident warps per SM (occupancy-sensitivity measurements)
static int mm4_pad() {
  static const int v = [] {
    const char* e = getenv("HB_MM4_PAD");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// HB_PDL (experiments): 0 disables programmatic dependent launch
static bool mm4_pdl() {
  static const bool v = [] {
    const char* e = getenv("HB_PDL");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

template <class T, int D, int KP1, int STAGE, int VAR>
static cudaError_t mm4_go(const KParams& p, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.n_tiles);
  cfg.blockDim = dim3(VAR == 6 ? 64 : 32);
  cfg.dynamicSmemBytes = (size_t)mm4_pad();
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = mm4_pdl() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_mm4<T, D, KP1, STAGE, VAR>, p);
}

template <class T, int D, int KP1, int STAGE>
static cudaError_t mm4s_go(const KParams& p, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.n_tiles);
  cfg.blockDim = dim3(64);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = mm4_pdl() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_mm4s<T, D, KP1, STAGE>, p);
}

// HB_SPLIT_TILES (experiment): grids of at most this many tiles run the split CTAs
// (k_mm4s); off by default (measured no faster)
static int split_tiles() {
  static const int v = [] {
    const char* e = getenv("HB_SPLIT_TILES");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <class T, int D, int KP1>
static cudaError_t mm4s_launch(int stage, const KParams& p, cudaStream_t s) {
  switch (stage) {
    case 1: return mm4s_go<T, D, KP1, 1>(p, s);
    case 2: return mm4s_go<T, D, KP1, 2>(p, s);
    case 3: return mm4s_go<T, D, KP1, 3>(p, s);
    case 4: {
      const cudaError_t e = mm4s_go<T, D, KP1, 4>(p, s);
      if (e != cudaSuccess) return e;
      return finish_go<D>(p, s);
    }
  }
  return cudaErrorInvalidValue;
}

template <class T, int D, int KP1, int VAR>
static cudaError_t mm4_launch_b(int stage, const KParams& p, cudaStream_t s) {
  if (VAR == 1 && D >= 2 && p.n_tiles <= split_tiles()) return mm4s_launch<T, D, KP1>(stage, p, s);
  switch (stage) {
    case 1: return mm4_go<T, D, KP1, 1, VAR>(p, s);
    case 2: return mm4_go<T, D, KP1, 2, VAR>(p, s);
    case 3: return mm4_go<T, D, KP1, 3, VAR>(p, s);
    case 4: {
      const cudaError_t e = mm4_go<T, D, KP1, 4, VAR>(p, s);
      if (e != cudaSuccess || VAR == 6) return e;
      return finish_go<D>(p, s);
    }
  }
  return cudaErrorInvalidValue;
}

template <int D, int KP1>
static cudaError_t mm4_launch_t(int stage, const KParams& p, cudaStream_t s) {
  if (p.single) {
    // float state: 168 registers (12 warps/SM) fit without spills; stages 1 and 3
    // (10 KB of shared memory per CTA) gain from it, stages 2 and 4 (17 KB: L1 is
    // squeezed to ~40 KB at 12 CTAs) do not.  HB_MM4_FVAR (experiments): 1 = never
    // capped, 8 = capped at every stage, default = stages 1 and 3
    static const int fvar = [] {
      const char* e = getenv("HB_MM4_FVAR");
      return e ? atoi(e) : 0;
    }();
    const bool cap = fvar == 8 || (fvar == 0 && (stage == 1 || stage == 3));
    if (cap) return mm4_launch_b<float, D, KP1, 8>(stage, p, s);
    return mm4_launch_b<float, D, KP1, 1>(stage, p, s);
  }
  if constexpr (D == 7 && KP1 == 2) {
    static const int var = [] {
      const char* e = getenv("HB_MM4_VAR");
      return e ? atoi(e) : 1;
    }();
    if (var == 5) return mm4_launch_b<double, D, KP1, 5>(stage, p, s);
    if (var == 6) return mm4_launch_b<double, D, KP1, 6>(stage, p, s);
    if (var == 7) return mm4_launch_b<double, D, KP1, 7>(stage, p, s);
    if (var == 9) return mm4_launch_b<double, D, KP1, 9>(stage, p, s);
  }
  return mm4_launch_b<double, D, KP1, 1>(stage, p, s);
}

template <int D>
static cudaError_t mm4_kp1(int stage, const KParams& p, cudaStream_t s) {
  return p.kp1 == 1 ? mm4_launch_t<D, 1>(stage, p, s) : mm4_launch_t<D, 2>(stage, p, s);
}

cudaError_t launch_mm4(int stage, const KParams& p, cudaStream_t s) {
  switch (p.d) {
    case 1: return mm4_kp1<1>(stage, p, s);
    case 2: return mm4_kp1<2>(stage, p, s);
    case 3: return mm4_kp1<3>(stage, p, s);
    case 4: return mm4_kp1<4>(stage, p, s);
    case 5: return mm4_kp1<5>(stage, p, s);
    case 6: return mm4_kp1<6>(stage, p, s);
    case 7: return mm4_kp1<7>(stage, p, s);
    case 8: return mm4_kp1<8>(stage, p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hb
