// Production stage kernel k_mm4: one launch per RK4 stage evaluates the RHS of
// the reference (_kernels.py:23-58, generalised to K+1 modes per site) for its
// tiles and writes the next stage input, folding add_scaled / rk4_update
// (_kernels.py:61-72, heom.py:370-381); see hb_mm_common.cuh for the phases and
// the 12-pass (double) / increment (float) RK bookkeeping.
//
// One warp = one CTA = one tile of 32 ADOs (lane = ADO), fully unrolled for
// (d, K+1), the ADO and the accumulator in registers:
//   * the run's status is read first: a replay past the stop exits before it
//     issues any copy (graph steps enqueued after the stop cost a CTA launch);
//   * the tile's base operand (sigma, or B at stage 4) and its link tables
//     ([mode][32] int32 raise/lower, uint8 n) arrive by one bulk copy group
//     (cp.async.bulk, one mbarrier); a top-tier tile (no raise links; every tile
//     past P.top_tile in the tier-major order) does not copy its raise table;
//   * every RHS term is one explicit FMA, the RK stage coefficient c folded into
//     the link coefficients once per link;
//   * absent links (TRUNCATED raise, ABSENT lower) are predicated off;
//   * a tile with no raise link gathers two sites' lower links per round trip:
//     4 dependent L2 round trips instead of 7.
// T = double (HB_PREC_DOUBLE) or float (HB_PREC_SINGLE: float state, float RHS,
// heom.py:93-94; bookkeeping, sinks and records stay double).
//
// Small hierarchies (KParams::split) use k_mm4ab below instead: the same phases
// on separate warps of one CTA per tile, and in CUDA graphs the previous step's
// bookkeeping folded into stage 1 as an extra CTA (KParams::fold).
#include "hb_device.cuh"
#include "hb_mm_common.cuh"

namespace hb {

// CAP: registers capped for 12 resident warps per SM (float stages 1 and 3)
template <class T, int D, int KP1, int STAGE, bool CAP>
__global__ void __launch_bounds__(32, CAP ? 12 : 1) k_mm4(const KParams P) {
  constexpr int NP = D * D;
  constexpr int M = D * KP1;
  constexpr int TB = NP * TILE;
  constexpr bool kInc = kIncScheme<T>;
  __shared__ __align__(128) T sBase[(STAGE >= 2 || kInc ? NP : 1) * TILE];
  __shared__ __align__(128) T sInc[(kInc && (STAGE == 2 || STAGE == 4) ? NP : 1) * TILE];
  __shared__ __align__(16) int32_t sUp[M][TILE];
  __shared__ __align__(16) int32_t sDn[M][TILE];
  __shared__ __align__(16) uint8_t sN[M][TILE];
  __shared__ __align__(8) uint64_t bar;

  volatile Ctl* ctl = P.ctl;
  // a status other than RUNNING is final for the run (only the host restarts
  // it), so a stale read can only be a stale RUNNING, caught after pdl_wait
  if (ctl->status != ST_RUNNING) return;
  const int lane = threadIdx.x;
  const int tile = P.tile_list ? P.tile_list[blockIdx.x] : P.tile_begin + blockIdx.x;
  HB_CHECK(tile >= 0 && tile < P.n_tiles_total);
  const size_t tb = (size_t)tile * TB;  // element offset of the tile
  const T c = (T)(STAGE == 4 ? P.dt / 6.0 : P.coef);
  const bool top = tile >= P.top_tile;

  // operands no running kernel writes, before the grid dependency (PDL); the
  // float increment tile (written by stage 1) after it
  tile_prologue<T, D, KP1, STAGE>(P, tile, sBase, &sUp[0][0], &sDn[0][0], &sN[0][0], &bar, !top,
                                  sInc, true);
  pdl_wait();
  tile_prologue_late<T, D, STAGE>(P, tile, sInc, &bar);
  // the status after the grid dependency is tested before the stores only, so
  // the loads below do not wait for it (replays after the stop already exited
  // at the first test; this one catches a stop landing while the CTA started)
  const int status = ctl->status;
  pdl_release();
  const long long step_next = ctl->step + 1;
  T acc[NP];
  phase_a<T, D, KP1, STAGE>(P, tile, lane, c, sBase, sN, &bar, acc);
  bool no_up = top;
  if (!top) {
    bool up_any = false;
#pragma unroll
    for (int m = 0; m < M; ++m) up_any |= sUp[m][lane] >= 0;
    no_up = !__any_sync(0xffffffffu, up_any);
  }
  phase_b_sites<T, D, KP1>(P, lane, c, no_up, sUp, sDn, sN, acc);
  if (status != ST_RUNNING) return;  // past the bulk-copy wait (phase A)
  double maxa2 = 0.0;
  phase_c_store<T, D, STAGE>(P, lane, tb, sBase, acc, maxa2, sInc);
  if (STAGE == 4 && step_next % 25 == 0) {  // whole-state guard (heom.py:386-389)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
    if (lane == 0)
      atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                (unsigned long long)__double_as_longlong(maxa2));
  }
}


// k_mm4ab: the stage kernel for small hierarchies (KParams::split; at most a
// few tiles per SM).  There one warp per tile leaves three of an SM's four
// sub-partitions idle and the tile's chain is the stage time: phase A (the
// commutator, ~850 instructions, FP64-issue bound in one warp) then phase B (the
// link crosses, 4-7 dependent gather rounds).  Here NA warps run phase A on
// disjoint row ranges of the ADO while NB warps run phase B on disjoint site
// ranges, each from its own zeroed accumulator; the last warp adds the partial
// sums from shared memory, (A + B_lo) + B_hi, and stores as k_mm4.  The same
// phase functions as k_mm4 (hb_mm_common.cuh), so every element's RHS terms are
// the reference's; only the grouping of the final sum differs from k_mm4 (equal
// to the last bits).  The split is chosen from the size of the whole hierarchy,
// so all shards of a run and the unsharded run use the same one.
// Row ranges balance the commutator's cost; sites split at an even index so
// the paired rounds of top-tier tiles stay pairs.  Measured (us per step, vs
// k_mm4): config-3 K = 0 twin, 54 tiles, 3 + 2 warps: 17.5 vs 25.5; K = 1,
// N_max = 4, 96 tiles, 2 + 2: 25.6 vs 37; N_max = 5, 364 tiles, 1 + 1: 36 vs 43;
// above ~4 tiles per SM one warp per tile wins (N_max = 6, 1,211 tiles: 58 vs
// 51).  2 + 1 / 1 + 2 / 4 + 1 / 4 + 2 warps were measured too (within 5 %).
// rows [row_bound(w), row_bound(w + 1)) of the ADO for phase-A warp w of NA:
// the partition minimising the largest part, row i costing ~3 (d - 1 - i) + 1
// (off-diagonal elements ~3x a diagonal one)
template <int D, int NA>
struct RowSplit {
  int b[5];
  __host__ __device__ constexpr RowSplit() : b{0, D, D, D, D} {
    int best = 1 << 30;
    auto cost = [](int r0, int r1) {
      int c = 0;
      for (int i = r0; i < r1; ++i) c += 3 * (D - 1 - i) + 1;
      return c;
    };
    auto mx = [](int x, int y) { return x > y ? x : y; };
    for (int x = 0; x <= D; ++x)
      for (int y = x; y <= D; ++y)
        for (int z = y; z <= D; ++z) {
          const int c1 = NA >= 2 ? x : D, c2 = NA >= 3 ? y : D, c3 = NA >= 4 ? z : D;
          if ((NA < 2 && x) || (NA < 3 && y != x) || (NA < 4 && z != y)) continue;
          const int m = mx(mx(cost(0, c1), cost(c1, c2)), mx(cost(c2, c3), cost(c3, D)));
          if (m < best) {
            best = m;
            b[1] = c1;
            b[2] = c2;
            b[3] = c3;
          }
        }
    b[NA] = D;
  }
};
template <int D>
__host__ __device__ constexpr int site_split() { return ((D + 1) / 2 + 1) / 2 * 2 < D ? ((D + 1) / 2 + 1) / 2 * 2 : D; }

template <class T, int D, int KP1, int STAGE, int NA, int NB, bool FOLD = false>
__global__ void __launch_bounds__(32 * (NA + NB), 1) k_mm4ab(const KParams P) {
  constexpr int NP = D * D;
  constexpr int M = D * KP1;
  constexpr int TB = NP * TILE;
  constexpr bool kInc = kIncScheme<T>;
  constexpr RowSplit<D, NA> RB{};
  constexpr int SS = NB == 2 ? site_split<D>() : D;
  __shared__ __align__(128) T sBase[(STAGE >= 2 || kInc ? NP : 1) * TILE];
  __shared__ __align__(128) T sInc[(kInc && (STAGE == 2 || STAGE == 4) ? NP : 1) * TILE];
  __shared__ __align__(128) T sXA[NP * TILE];
  __shared__ __align__(128) T sXB[(NB == 2 ? NP : 1) * TILE];
  __shared__ __align__(16) int32_t sUp[M][TILE];
  __shared__ __align__(16) int32_t sDn[M][TILE];
  __shared__ __align__(16) uint8_t sN[M][TILE];
  __shared__ __align__(8) uint64_t bar;
  volatile Ctl* ctl = P.ctl;
  // the early exit must be one decision per CTA: the status can change while
  // the CTA starts (the previous step's bookkeeping runs concurrently under PDL,
  // or in this very launch when folded), and a warp that went on alone would
  // wait on a barrier nobody initialised
  __shared__ int s_stopped;
  if (threadIdx.x == 0) s_stopped = ctl->status != ST_RUNNING;
  __syncthreads();
  if (s_stopped) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // a separate instantiation: the bookkeeping code (~20 KB of SASS) in every
  // stage-1 kernel costs ~5 % through the instruction cache when unused
  if constexpr (FOLD) {
    if (blockIdx.x == gridDim.x - 1) {
      // the extra CTA of a folded stage 1: the previous step's bookkeeping, on
      // an SM of its own, while the tiles compute
      pdl_wait();
      pdl_release();
      if (warp == 0) fold_finish_warp<D>(P);
      return;
    }
  }
  const int tile = P.tile_list ? P.tile_list[blockIdx.x] : P.tile_begin + blockIdx.x;
  HB_CHECK(tile >= 0 && tile < P.n_tiles_total);
  const size_t tb = (size_t)tile * TB;
  const T c = (T)(STAGE == 4 ? P.dt / 6.0 : P.coef);
  const bool top = tile >= P.top_tile;
  if (warp == 0)
    tile_prologue<T, D, KP1, STAGE>(P, tile, sBase, &sUp[0][0], &sDn[0][0], &sN[0][0], &bar, !top,
                                    sInc, true);
  __syncthreads();
  pdl_wait();
  if (warp == 0) tile_prologue_late<T, D, STAGE>(P, tile, sInc, &bar);
  // the status after the grid dependency is only tested before the stores, so
  // the tile's loads do not wait for it (a stopped run's replays compute and
  // discard; the sink rates written by tile 0 are only read while running)
  const int status = ctl->status;
  pdl_release();
  const long long step_next = ctl->step + 1;
  T acc[NP];
  auto put_rows = [&](auto r0, auto r1) {
#pragma unroll
    for (int i = decltype(r0)::value; i < decltype(r1)::value; ++i) {
      sXA[i * TILE + lane] = acc[i];
#pragma unroll
      for (int j = i + 1; j < D; ++j) {
        sXA[Pk<D>::re(i, j) * TILE + lane] = acc[Pk<D>::re(i, j)];
        sXA[Pk<D>::im(i, j) * TILE + lane] = acc[Pk<D>::im(i, j)];
      }
    }
  };
  auto phase_b_part = [&](auto s0, auto s1) {
    mbar_wait(&bar, 0);
#pragma unroll
    for (int e = 0; e < NP; ++e) acc[e] = 0;
    bool no_up = top;
    if (!top) {
      bool up_any = false;
#pragma unroll
      for (int m = 0; m < M; ++m) up_any |= sUp[m][lane] >= 0;
      no_up = !__any_sync(0xffffffffu, up_any);
    }
    phase_b_sites<T, D, KP1, 2, decltype(s0)::value, decltype(s1)::value>(P, lane, c, no_up, sUp,
                                                                            sDn, sN, acc);
  };
  using Z = std::integral_constant<int, 0>;
  using Dc = std::integral_constant<int, D>;
  using SSc = std::integral_constant<int, SS>;
  if (warp < NA) {
    auto part_a = [&](auto w) {
      constexpr int W = decltype(w)::value;
      if constexpr (W < NA) {
        if (warp == W) {
          phase_a<T, D, KP1, STAGE, RB.b[W], RB.b[W + 1]>(P, tile, lane, c, sBase, sN, &bar, acc);
          put_rows(std::integral_constant<int, RB.b[W]>(), std::integral_constant<int, RB.b[W + 1]>());
        }
      }
    };
    part_a(std::integral_constant<int, 0>());
    part_a(std::integral_constant<int, 1>());
    part_a(std::integral_constant<int, 2>());
    part_a(std::integral_constant<int, 3>());
  } else if (NB == 2 && warp == NA) {
    phase_b_part(Z(), SSc());
#pragma unroll
    for (int e = 0; e < NP; ++e) sXB[e * TILE + lane] = acc[e];
  } else {
    if constexpr (NB == 2) phase_b_part(SSc(), Dc());
    else phase_b_part(Z(), Dc());
  }
  __syncthreads();
  if (status != ST_RUNNING) return;  // every warp is past its bulk-copy wait
  if (warp == NA + NB - 1) {
#pragma unroll
    for (int e = 0; e < NP; ++e)
      acc[e] = NB == 2 ? (sXA[e * TILE + lane] + sXB[e * TILE + lane]) + acc[e]
                       : sXA[e * TILE + lane] + acc[e];
    double maxa2 = 0.0;
    phase_c_store<T, D, STAGE>(P, lane, tb, sBase, acc, maxa2, sInc);
    if (STAGE == 4 && step_next % 25 == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
      if (lane == 0)
        atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                  (unsigned long long)__double_as_longlong(maxa2));
    }
  }
}

// The per-step bookkeeping (sinks heom.py:382-383, guard heom.py:386-389,
// records, stop policy heom.py:359-368) as its own one-warp kernel after stage
// 4, chained by PDL: it waits for the stage-4 grid to complete and flush, so the
// stage kernels need no per-CTA fence and no last-CTA election counter.
// The finish kernel of the last step of a CUDA-graph WHILE body (P.set_cond)
// also decides whether the body runs again: while the run is RUNNING and fewer
// than P.loop_iters iterations of this launch have run (the record buffer is
// sized for that many).
template <int D>
__global__ void __launch_bounds__(32, 1) k_step_finish(const KParams P) {
  // released only once stage 4 has completed: released earlier, the next
  // step's stage-1 CTAs would take SM slots from stage 4's last waves
  pdl_wait();
  pdl_release();
  volatile Ctl* ctl = P.ctl;
  int status;
  long long loop_iter;
  if (!P.root) {  // non-root shard (hb_device.cuh finish_step_shard)
    if (ctl->status == ST_RUNNING) {
      const long long step_next = ctl->step + 1;
      if (threadIdx.x == 0) ctl->launches = ctl->launches + 5;
      finish_step_warp<D, true>(P, step_next);
    }
    __syncwarp();
    status = ctl->status;
    loop_iter = ctl->loop_iter;
  } else {
    // the control block and sigma^0 in one round trip (both are read even when
    // the run has stopped: a replay past the stop then writes nothing)
    __shared__ Sig0 s0;
    __shared__ Ctl cs;
    ctl_load_warp(P.ctl, cs);
    sig0_warp<D, true>(P, s0);
    if (cs.status == ST_RUNNING) {
      if (threadIdx.x == 0) cs.launches += 5;
      finish_step_loaded<D>(P, cs.step + 1, s0, cs, P.rpar);
      ctl_store_warp(P.ctl, cs);
    }
    status = cs.status;
    loop_iter = cs.loop_iter;
  }
  if (P.set_cond && threadIdx.x == 0) {
    const long long it = loop_iter + 1;
    const bool again = status == ST_RUNNING && it < P.loop_iters;
    ctl->loop_iter = again ? it : 0;
    cudaGraphSetConditional(P.cond, again ? 1u : 0u);
  }
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

template <class T, int D, int KP1, int STAGE, bool CAP>
static cudaError_t mm4_go(const KParams& p, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.n_tiles);
  cfg.blockDim = dim3(32);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  int n = 1;
  if (p.apw_tiles > 0) {  // the gather targets of the stage input kept in L2
    const size_t tb = (size_t)D * D * TILE * sizeof(T);
    attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[1].val.accessPolicyWindow.base_ptr =
        (void*)(reinterpret_cast<const char*>(p.Yin) + p.apw_first_tile * tb);
    attr[1].val.accessPolicyWindow.num_bytes = (size_t)p.apw_tiles * tb;
    attr[1].val.accessPolicyWindow.hitRatio = p.apw_hit;
    attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    n = 2;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  if constexpr (D <= 7) {  // (41.5 KB of static shared memory at d = 7, 2 + 2 warps)
    constexpr bool kFold = STAGE == 1;
    const bool fold = kFold && p.fold;
    if (fold) cfg.gridDim.x += 1;  // the folded bookkeeping CTA
    if (p.split == 1) {
      cfg.blockDim = dim3(64);
      return cudaLaunchKernelEx(&cfg, fold ? k_mm4ab<T, D, KP1, STAGE, 1, 1, kFold>
                                           : k_mm4ab<T, D, KP1, STAGE, 1, 1>, p);
    }
    if (p.split == 2) {  // K = 0: 3 + 2 warps; K >= 1 (twice the link crosses): 2 + 2
      constexpr int NA = KP1 == 1 ? 3 : 2;
      cfg.blockDim = dim3(32 * (NA + 2));
      return cudaLaunchKernelEx(&cfg, fold ? k_mm4ab<T, D, KP1, STAGE, NA, 2, kFold>
                                           : k_mm4ab<T, D, KP1, STAGE, NA, 2>, p);
    }
  }
  return cudaLaunchKernelEx(&cfg, k_mm4<T, D, KP1, STAGE, CAP>, p);
}

// float state: 168 registers (12 warps/SM) fit without spills; stages 1 and 3
// (10 KB of shared memory per CTA) gain from it, stages 2 and 4 (17 KB: L1 is
// squeezed to ~40 KB at 12 CTAs) do not
template <class T, int D, int KP1>
static cudaError_t mm4_stage(int stage, const KParams& p, cudaStream_t s) {
  constexpr bool F = std::is_same<T, float>::value;
  switch (stage) {
    case 1: return mm4_go<T, D, KP1, 1, F>(p, s);
    case 2: return mm4_go<T, D, KP1, 2, false>(p, s);
    case 3: return mm4_go<T, D, KP1, 3, F>(p, s);
    case 4: return mm4_go<T, D, KP1, 4, false>(p, s);
  }
  return cudaErrorInvalidValue;
}

// stage 4 is followed by the step bookkeeping kernel
template <int D, int KP1>
static cudaError_t mm4_t(int stage, const KParams& p, cudaStream_t s) {
  const cudaError_t e = p.single ? mm4_stage<float, D, KP1>(stage, p, s)
                                 : mm4_stage<double, D, KP1>(stage, p, s);
  if (e != cudaSuccess || stage != 4 || p.fold) return e;  // folded: the next stage 1 finishes
  return finish_go<D>(p, s);
}

template <int D>
static cudaError_t mm4_kp1(int stage, const KParams& p, cudaStream_t s) {
  return p.kp1 == 1 ? mm4_t<D, 1>(stage, p, s) : mm4_t<D, 2>(stage, p, s);
}

// the stage kernel alone (sharded runs launch a stage as several tile groups and
// the step bookkeeping once after the last); a group that is one contiguous
// ascending run of tiles is launched as a range (no per-CTA tile-list load)
template <int D, int KP1>
static cudaError_t mm4_only_t(int stage, const KParams& p, cudaStream_t s) {
  return p.single ? mm4_stage<float, D, KP1>(stage, p, s) : mm4_stage<double, D, KP1>(stage, p, s);
}
template <int D>
static cudaError_t mm4_only_kp1(int stage, const KParams& p, cudaStream_t s) {
  if (stage == 5) return finish_go<D>(p, s);
  return p.kp1 == 1 ? mm4_only_t<D, 1>(stage, p, s) : mm4_only_t<D, 2>(stage, p, s);
}

cudaError_t launch_mm4_only(int stage, const KParams& p, cudaStream_t s) {
  switch (p.d) {
    case 1: return mm4_only_kp1<1>(stage, p, s);
    case 2: return mm4_only_kp1<2>(stage, p, s);
    case 3: return mm4_only_kp1<3>(stage, p, s);
    case 4: return mm4_only_kp1<4>(stage, p, s);
    case 5: return mm4_only_kp1<5>(stage, p, s);
    case 6: return mm4_only_kp1<6>(stage, p, s);
    case 7: return mm4_only_kp1<7>(stage, p, s);
    case 8: return mm4_only_kp1<8>(stage, p, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_step_finish(const KParams& p, cudaStream_t s) { return launch_mm4_only(5, p, s); }

bool mm4_supported(int d, int kp1) { return d >= 1 && d <= 8 && kp1 >= 1 && kp1 <= 2; }

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
