// Experimental stage kernel (variant 13, k_mm9): k_mm8's tensor-memory
// accumulator used to PIPELINE the neighbour gathers instead of raising the
// occupancy.
//
// The step is bound by the chain of dependent L2 round trips per tile (own
// ADO, then one round per site -- or per site pair on top-tier tiles).  With
// the accumulator in TMEM a thread holds only gathered values: at 255
// registers (8 warps per SM) two rounds fit, so round r+1's loads are issued
// before round r is consumed (TMEM read, FMA, TMEM write), and round 0's loads
// go out with the own-ADO loads, before the commutator.  The tile's chain
// shrinks from (1 + rounds) round trips to ~1 + rounds/2 of exposed latency.
// Arithmetic, stage combinations and base handling are k_mm8's (LATE).
#include <cstdlib>
#include "hb_device.cuh"
#include "hb_fast.cuh"
#include "hb_mm_common.cuh"

namespace hb {

namespace mm9 {

constexpr int kWarps = 4;   // one warpgroup per CTA (TMEM lane quarters)
constexpr int kCols = 128;  // TMEM columns per CTA

__device__ __forceinline__ void st2(uint32_t ta, double v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(ta),
               "r"(__double2loint(v)), "r"(__double2hiint(v))
               : "memory");
}
__device__ __forceinline__ void st4(uint32_t ta, double a, double b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ta),
               "r"(__double2loint(a)), "r"(__double2hiint(a)), "r"(__double2loint(b)),
               "r"(__double2hiint(b))
               : "memory");
}
__device__ __forceinline__ double ld2(uint32_t ta) {
  int lo, hi;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
               : "=r"(lo), "=r"(hi)
               : "r"(ta)
               : "memory");
  return __hiloint2double(hi, lo);
}
__device__ __forceinline__ void ld4(uint32_t ta, double& a, double& b) {
  int a0, a1, b0, b1;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(b0), "=r"(b1)
               : "r"(ta)
               : "memory");
  a = __hiloint2double(a1, a0);
  b = __hiloint2double(b1, b0);
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <int D, int KP1>
struct Smem {
  static constexpr int M = D * KP1;
  static constexpr size_t UP = 0;
  static constexpr size_t DN = UP + (size_t)kWarps * M * TILE * 4;
  static constexpr size_t N = DN + (size_t)kWarps * M * TILE * 4;
  static constexpr size_t BAR = (N + (size_t)kWarps * M * TILE + 15) / 16 * 16;
  static constexpr size_t TADDR = BAR + 8 * kWarps;
  static constexpr size_t BYTES = TADDR + 16;
};

// One round = 2 * KP1 link slots; slot j of round R:
//   normal : site R, raise (j < KP1) or lower (j >= KP1), k = j % KP1
//   paired : lower links only, site 2R + j / KP1, k = j % KP1
template <int D, int KP1, bool PAIR, int R, int J>
struct Slot {
  static constexpr int site = PAIR ? 2 * R + J / KP1 : R;
  static constexpr bool lower = PAIR ? true : J >= KP1;
  static constexpr int k = J % KP1;
  static constexpr bool exists = site < D;
};

template <int D>
__device__ __forceinline__ constexpr int cross_plane(int st, int q) {
  // q = 0: diagonal; then (re, im) of (st, o) for o != st ascending
  if (q == 0) return st;
  const int idx = (q - 1) / 2;
  const int o = idx < st ? idx : idx + 1;
  return Pk<D>::re(st, o) + ((q - 1) & 1);
}

template <int D, int KP1, bool PAIR, int R>
__device__ __forceinline__ void load_round(const KParams& P, int lane, const int32_t (*sUp)[TILE],
                                           const int32_t (*sDn)[TILE],
                                           double (&g)[2 * KP1][2 * D - 1]) {
  constexpr int TB = D * D * TILE, NC = 2 * D - 1;
#pragma unroll
  for (int j = 0; j < 2 * KP1; ++j) {
    const int site = PAIR ? 2 * R + j / KP1 : R;
    const bool lower = PAIR ? true : j >= KP1;
    const int k = j % KP1;
    if (site >= D) continue;
    const int m = site * KP1 + k;
    const int p = lower ? sDn[m][lane] : sUp[m][lane];
    const double* q = P.Yin + ((p >> 5) * TB + (p & 31));
#pragma unroll
    for (int e = 0; e < NC; ++e) {
      double v = 0.0;
      if (p >= 0) v = __ldg(q + cross_plane<D>(site, e) * TILE);
      g[j][e] = v;
    }
  }
}

template <int D, int KP1, bool PAIR, int R>
__device__ __forceinline__ void consume_round(const KParams& P, int lane, uint32_t tm, double c,
                                              const int32_t (*sUp)[TILE],
                                              const int32_t (*sDn)[TILE],
                                              const uint8_t (*sN)[TILE],
                                              const double (&g)[2 * KP1][2 * D - 1]) {
  constexpr int NP = D * D, NC = 2 * D - 1;
  constexpr int NSITES = PAIR ? 2 : 1;
#pragma unroll
  for (int si = 0; si < NSITES; ++si) {
    const int st = PAIR ? 2 * R + si : R;
    if (st >= D) continue;
    auto col = [&](int plane) { return tm + 2u * (uint32_t)plane; };
    double x[NP];
    x[st] = ld2(col(st));
#pragma unroll
    for (int o = 0; o < D; ++o)
      if (o != st) ld4(col(Pk<D>::re(st, o)), x[Pk<D>::re(st, o)], x[Pk<D>::re(st, o) + 1]);
    wait_ld();
#pragma unroll
    for (int j = 0; j < 2 * KP1; ++j) {
      const int site = PAIR ? 2 * R + j / KP1 : R;
      if (site != st) continue;
      const bool lower = PAIR ? true : j >= KP1;
      const int k = j % KP1;
      const int m = st * KP1 + k;
      double cb = 0.0, ca = 0.0, cu = 0.0;
      if (lower) {
        const double n = sDn[m][lane] >= 0 ? (double)sN[m][lane] : 0.0;
        cb = n * c * P.b[k];
        ca = n * c * P.a[k];
        x[st] = fma(2.0 * cb, g[j][0], x[st]);
      } else {
        cu = sUp[m][lane] >= 0 ? c : 0.0;
      }
#pragma unroll
      for (int o = 0; o < D; ++o) {
        if (o == st) continue;
        const int idx = o < st ? o : o - 1;
        const int pr = Pk<D>::re(st, o), pim = pr + 1;
        const double vr = g[j][1 + 2 * idx], vi = g[j][2 + 2 * idx];
        if (lower) {
          if (o > st) {
            x[pr] = fma(cb, vr, fma(-ca, vi, x[pr]));
            x[pim] = fma(cb, vi, fma(ca, vr, x[pim]));
          } else {
            x[pr] = fma(cb, vr, fma(ca, vi, x[pr]));
            x[pim] = fma(cb, vi, fma(-ca, vr, x[pim]));
          }
        } else {
          if (o > st) {  // -i x
            x[pr] = fma(-cu, vi, x[pr]);
            x[pim] = fma(cu, vr, x[pim]);
          } else {       // +i x
            x[pr] = fma(cu, vi, x[pr]);
            x[pim] = fma(-cu, vr, x[pim]);
          }
        }
      }
    }
    st2(col(st), x[st]);
#pragma unroll
    for (int o = 0; o < D; ++o)
      if (o != st) st4(col(Pk<D>::re(st, o)), x[Pk<D>::re(st, o)], x[Pk<D>::re(st, o) + 1]);
    wait_st();
  }
}

// rounds R .. NR-1 with a one-round-deep prefetch; `cur` holds round R's loads
template <int D, int KP1, bool PAIR, int R, int NR>
__device__ __forceinline__ void pipeline(const KParams& P, int lane, uint32_t tm, double c,
                                         const int32_t (*sUp)[TILE], const int32_t (*sDn)[TILE],
                                         const uint8_t (*sN)[TILE],
                                         double (&cur)[2 * KP1][2 * D - 1]) {
  if constexpr (R < NR) {
    double nxt[2 * KP1][2 * D - 1];
    if constexpr (R + 1 < NR) load_round<D, KP1, PAIR, R + 1>(P, lane, sUp, sDn, nxt);
    consume_round<D, KP1, PAIR, R>(P, lane, tm, c, sUp, sDn, sN, cur);
    if constexpr (R + 1 < NR) pipeline<D, KP1, PAIR, R + 1, NR>(P, lane, tm, c, sUp, sDn, sN, nxt);
  }
}

}  // namespace mm9

template <int D, int KP1, int STAGE>
__global__ void __launch_bounds__(32 * mm9::kWarps, 2) k_mm9(const KParams P) {
  using namespace mm9;
  constexpr int NP = D * D;
  constexpr int M = D * KP1;
  constexpr int TB = NP * TILE;
  constexpr int NC = 2 * D - 1;
  using L = Smem<D, KP1>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t(*sUp)[TILE] = reinterpret_cast<int32_t(*)[M][TILE]>(smem + L::UP)[w];
  int32_t(*sDn)[TILE] = reinterpret_cast<int32_t(*)[M][TILE]>(smem + L::DN)[w];
  uint8_t(*sN)[TILE] = reinterpret_cast<uint8_t(*)[M][TILE]>(smem + L::N)[w];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::BAR) + w;
  uint32_t* s_taddr = reinterpret_cast<uint32_t*>(smem + L::TADDR);

  volatile Ctl* ctl = P.ctl;
  const int t = blockIdx.x * kWarps + w;
  const bool active = t < P.n_tiles;
  const int tile = P.tile_begin + (active ? t : 0);
  const int own = tile * TB + lane;
  const double c = STAGE == 4 ? P.dt / 6.0 : P.coef;

  if (active)  // link tables only; the base operands are read in phase C
    tile_prologue<double, D, KP1, 1>(P, tile, nullptr, &sUp[0][0], &sDn[0][0], &sN[0][0], bar);
  pdl_wait();
  if (ctl->status != ST_RUNNING) {
    if (active) mbar_wait(bar, 0);
    return;
  }
  pdl_release();
  const long long step_next = ctl->step + 1;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(s_taddr)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = *s_taddr + ((uint32_t)(32 * w) << 16);
  auto col = [&](int plane) { return tm + 2u * (uint32_t)plane; };

  double maxa2 = 0.0;
  if (active) {
    double s[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) s[p] = __ldg(P.Yin + own + p * TILE);
    if (tile == 0 && lane == 0) {  // sink rates of this stage input (heom.py:282-283)
      int q = 0;
      for (int sk = 0; sk < P.n_sinks; ++sk) {
        double a = 0.0;
        for (int cc = 0; cc < P.sink_nterms[sk]; ++cc, ++q) {
          const double v = P.sink_rate[q] * __ldg(P.Yin + P.sink_pos[q] * TILE);
          a = cc == 0 ? v : a + v;
        }
        ctl->r[STAGE - 1][sk] = a;
      }
    }
    mbar_wait(bar, 0);
    bool up_any = false;
#pragma unroll
    for (int m = 0; m < M; ++m) up_any |= sUp[m][lane] >= 0;
    const bool pair = !__any_sync(0xffffffffu, up_any);
    double g0[2 * KP1][NC];  // round 0's gathers go out with the own-ADO loads
    if (pair) load_round<D, KP1, true, 0>(P, lane, sUp, sDn, g0);
    else load_round<D, KP1, false, 0>(P, lane, sUp, sDn, g0);
    {  // ---- phase A: the increment (k_mm8 LATE), streamed to TMEM
      int tk[KP1];
#pragma unroll
      for (int k = 0; k < KP1; ++k) tk[k] = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) tk[m % KP1] += sN[m][lane];
      double damp = 0.0;
#pragma unroll
      for (int k = 0; k < KP1; ++k) damp = fma((double)tk[k], P.nu[k], damp);
      auto base = [&](int p) -> double {
        return STAGE == 4 ? s[p] * (1.0 / 3.0) : (STAGE == 1 ? s[p] : 0.0);
      };
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double cm = 0.0;
#pragma unroll
        for (int l = 0; l < D; ++l)
          if (l != i) cm = fma(P.h[i * MAXD + l], sim<D>(s, i, l), cm);
        const double fi = -(damp + P.decay[i]);
        st2(col(i), fma(c, fma(fi, s[i], -2.0 * cm), base(i)));
#pragma unroll
        for (int j = i + 1; j < D; ++j) {
          const int pr = Pk<D>::re(i, j), pim = Pk<D>::im(i, j);
          const double dh = P.h[i * MAXD + i] - P.h[j * MAXD + j], hij = P.h[i * MAXD + j];
          double cr = fma(hij, s[j], fma(-hij, s[i], dh * s[pr]));
          double ci = dh * s[pim];
#pragma unroll
          for (int l = 0; l < D; ++l) {
            if (l == i || l == j) continue;
            const double hil = P.h[i * MAXD + l], hlj = P.h[l * MAXD + j];
            cr = fma(hil, sre<D>(s, l, j), cr);
            cr = fma(-hlj, sre<D>(s, i, l), cr);
            ci = fma(hil, sim<D>(s, l, j), ci);
            ci = fma(-hlj, sim<D>(s, i, l), ci);
          }
          const double f = -(damp + 0.5 * (P.decay[i] + P.decay[j]));
          st4(col(pr), fma(c, fma(f, s[pr], ci), base(pr)), fma(c, fma(f, s[pim], -cr), base(pim)));
        }
      }
    }
    wait_st();
    // ---- phase B: pipelined rounds
    if (pair) pipeline<D, KP1, true, 0, (D + 1) / 2>(P, lane, tm, c, sUp, sDn, sN, g0);
    else pipeline<D, KP1, false, 0, D>(P, lane, tm, c, sUp, sDn, sN, g0);
    // ---- phase C: TMEM + base operands -> global (stage 2 also B)
    auto emit = [&](int p, double y) {
      if (STAGE >= 2) {
        const double sg = __ldg((STAGE == 4 ? P.Bbuf : P.sig) + own + p * TILE);
        y += sg;
        if (STAGE == 2) {
          const double y2 = __ldg(P.Yin + own + p * TILE);
          P.Bbuf[own + p * TILE] = fma(2.0 / 3.0, y, (y2 - sg) * (1.0 / 3.0));
        }
      }
      P.Yout[own + p * TILE] = y;
      return y;
    };
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const double y = ld2(col(i));
      wait_ld();
      const double yo = emit(i, y);
      if (STAGE == 4) maxa2 = fmax(maxa2, yo * yo);
    }
#pragma unroll
    for (int pr = D; pr < NP; pr += 2) {
      double yr, yi;
      ld4(col(pr), yr, yi);
      wait_ld();
      yr = emit(pr, yr);
      yi = emit(pr + 1, yi);
      if (STAGE == 4) maxa2 = fmax(maxa2, fma(yr, yr, yi * yi));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*s_taddr),
                 "n"(kCols)
                 : "memory");
  }
  if (STAGE == 4) stage4_finish<D>(P, step_next, maxa2);
}

template <int STAGE>
static cudaError_t mm9_go(const KParams& p, cudaStream_t s) {
  constexpr size_t bytes = mm9::Smem<7, 2>::BYTES;
  static const cudaError_t attr = cudaFuncSetAttribute(
      k_mm9<7, 2, STAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (attr != cudaSuccess) return attr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((p.n_tiles + mm9::kWarps - 1) / mm9::kWarps));
  cfg.blockDim = dim3(32 * mm9::kWarps);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = s;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_mm9<7, 2, STAGE>, p);
}

cudaError_t launch_mm9(int stage, const KParams& p, cudaStream_t s) {
  if (p.d != 7 || p.kp1 != 2 || p.single) return launch_mm4(stage, p, s);
  switch (stage) {
    case 1: return mm9_go<1>(p, s);
    case 2: return mm9_go<2>(p, s);
    case 3: return mm9_go<3>(p, s);
    case 4: return mm9_go<4>(p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hb
