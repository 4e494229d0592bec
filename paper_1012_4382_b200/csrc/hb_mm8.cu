// Experimental stage kernel (variant 11, k_mm8): the accumulator in TENSOR
// MEMORY, so the thread-per-ADO kernel fits 168 registers and an SM keeps 12
// warps resident instead of 8.
//
// Why: k_mm4 holds the ADO (98 registers) and its accumulator (98) in
// registers, 255 per thread, and the register file is split per SM
// sub-partition, so 8 warps per SM; the idle-warp experiment (HB_MM4_VAR=6,
// 4 working warps) is 1.42x slower, i.e. the gathers are occupancy bound.
// Here the accumulator lives in TMEM (512 columns x 128 lanes x 32 bit per SM):
// a CTA is one warpgroup (4 warps = 4 adjacent tiles), warp w owns TMEM lanes
// 32w..32w+31 (lane = ADO), plane p of the accumulator is columns 2p, 2p+1
// (the two halves of a double).  Phase A streams each finished element to TMEM
// (tcgen05.st), phase B reads one site's cross (13 elements, tcgen05.ld),
// adds the gathered links and writes it back, phase C reads it out and stores.
// TMEM traffic uses its own datapath, not the LSU/L1 path the gathers need.
// Arithmetic and stage combinations are k_mm4's (double, 12 passes).
#include <algorithm>
#include <cstdlib>
#include "hb_device.cuh"
#include "hb_fast.cuh"
#include "hb_mm_common.cuh"

namespace hb {

constexpr int kMm8Warps = 4;      // one warpgroup per CTA (TMEM lane quarters)
constexpr int kMm8Cols = 128;     // TMEM columns per CTA (>= 2 * 8 * 8 planes)

__device__ __forceinline__ void tm_st2(uint32_t ta, double v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(ta),
               "r"(__double2loint(v)), "r"(__double2hiint(v))
               : "memory");
}
__device__ __forceinline__ void tm_st4(uint32_t ta, double a, double b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ta),
               "r"(__double2loint(a)), "r"(__double2hiint(a)), "r"(__double2loint(b)),
               "r"(__double2hiint(b))
               : "memory");
}
__device__ __forceinline__ double tm_ld2(uint32_t ta) {
  int lo, hi;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
               : "=r"(lo), "=r"(hi)
               : "r"(ta)
               : "memory");
  return __hiloint2double(hi, lo);
}
__device__ __forceinline__ void tm_ld4(uint32_t ta, double& a, double& b) {
  int a0, a1, b0, b1;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(b0), "=r"(b1)
               : "r"(ta)
               : "memory");
  a = __hiloint2double(a1, a0);
  b = __hiloint2double(b1, b0);
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <int D, int KP1, int STAGE, bool LATE>
struct Mm8Smem {
  static constexpr int M = D * KP1, NB = STAGE >= 2 && !LATE ? D * D : 1;
  static constexpr size_t BASE = 0;
  static constexpr size_t UP = BASE + (size_t)kMm8Warps * NB * TILE * 8;
  static constexpr size_t DN = UP + (size_t)kMm8Warps * M * TILE * 4;
  static constexpr size_t N = DN + (size_t)kMm8Warps * M * TILE * 4;
  static constexpr size_t BAR = (N + (size_t)kMm8Warps * M * TILE + 15) / 16 * 16;
  static constexpr size_t TADDR = BAR + 8 * kMm8Warps;
  static constexpr size_t BYTES = TADDR + 16;
};

// LATE: the base operands (sigma; Y2 again at stage 2; B at stage 4) are read in
// phase C with plain loads instead of a bulk copy into shared memory at kernel
// start, so a CTA needs 16 KB of shared memory instead of 66 KB and L1 keeps
// ~200 KB for the gathers; phase A then accumulates only the increment.
// PAIRED: tiles without raise links gather two sites' lower links per round trip
template <int D, int KP1, int STAGE, int MINB, bool LATE, bool PAIRED = true>
__global__ void __launch_bounds__(32 * kMm8Warps, MINB) k_mm8(const KParams P) {
  constexpr int NP = D * D;
  constexpr int M = D * KP1;
  constexpr int TB = NP * TILE;
  constexpr int PSTAGE = LATE ? 1 : STAGE;  // what the prologue bulk-copies
  using L = Mm8Smem<D, KP1, STAGE, LATE>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double(*sBase)[TILE] = reinterpret_cast<double(*)[L::NB][TILE]>(smem + L::BASE)[w];
  int32_t(*sUp)[TILE] = reinterpret_cast<int32_t(*)[M][TILE]>(smem + L::UP)[w];
  int32_t(*sDn)[TILE] = reinterpret_cast<int32_t(*)[M][TILE]>(smem + L::DN)[w];
  uint8_t(*sN)[TILE] = reinterpret_cast<uint8_t(*)[M][TILE]>(smem + L::N)[w];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::BAR) + w;
  uint32_t* s_taddr = reinterpret_cast<uint32_t*>(smem + L::TADDR);

  volatile Ctl* ctl = P.ctl;
  const int t = blockIdx.x * kMm8Warps + w;
  const bool active = t < P.n_tiles;
  const int tile = P.tile_begin + (active ? t : 0);
  const int own = tile * TB + lane;
  const double c = STAGE == 4 ? P.dt / 6.0 : P.coef;

  if (active)
    tile_prologue<double, D, KP1, PSTAGE>(P, tile, &sBase[0][0], &sUp[0][0], &sDn[0][0],
                                          &sN[0][0], bar);
  pdl_wait();
  if (ctl->status != ST_RUNNING) {  // the same for every warp (set only by a finished grid)
    if (active) mbar_wait(bar, 0);
    return;
  }
  pdl_release();
  const long long step_next = ctl->step + 1;
  // TMEM: warp 0 allocates the CTA's columns; warp w addresses lanes 32w..32w+31
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(s_taddr)),
                 "n"(kMm8Cols)
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
    // ---- phase A: acc = base + c * (damping + commutator), streamed to TMEM
    {
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
      int tk[KP1];
#pragma unroll
      for (int k = 0; k < KP1; ++k) tk[k] = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) tk[m % KP1] += sN[m][lane];
      double damp = 0.0;
#pragma unroll
      for (int k = 0; k < KP1; ++k) damp = fma((double)tk[k], P.nu[k], damp);
      constexpr double third = 1.0 / 3.0;
      auto base = [&](int p) -> double {
        if (LATE) return STAGE == 4 ? s[p] * third : (STAGE == 1 ? s[p] : 0.0);
        if (STAGE == 1) return s[p];
        const double b = sBase[p][lane];
        if (STAGE == 2) sBase[p][lane] = (s[p] - b) * third;  // park (Y2 - s)/3 for B
        if (STAGE == 4) return fma(s[p], third, b);
        return b;
      };
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double cm = 0.0;
#pragma unroll
        for (int l = 0; l < D; ++l)
          if (l != i) cm = fma(P.h[i * MAXD + l], sim<D>(s, i, l), cm);
        const double fi = -(damp + P.decay[i]);
        tm_st2(col(i), fma(c, fma(fi, s[i], -2.0 * cm), base(i)));
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
          tm_st4(col(pr), fma(c, fma(f, s[pr], ci), base(pr)),
                 fma(c, fma(f, s[pim], -cr), base(pim)));  // pim == pr + 1
        }
      }
    }
    tm_wait_st();
    // ---- phase B: one site's cross at a time: TMEM -> registers, + links, -> TMEM
    const double cbk0 = c * P.b[0], cak0 = c * P.a[0];
    const double cbk1 = KP1 > 1 ? c * P.b[KP1 - 1] : 0.0, cak1 = KP1 > 1 ? c * P.a[KP1 - 1] : 0.0;
    bool up_any = false;
#pragma unroll
    for (int m = 0; m < M; ++m) up_any |= sUp[m][lane] >= 0;
    if (PAIRED && !__any_sync(0xffffffffu, up_any)) {
      // no lane has a raise link (a top-tier tile): two sites' lower links per
      // round trip -- all 4(2d-1) loads issued first, then each site's cross is
      // read from TMEM, updated and written back
      constexpr int NC = 2 * D - 1;
#pragma unroll
      for (int s0 = 0; s0 < D; s0 += 2) {
        double g[2][KP1][NC];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int st = s0 + j;
          if (st >= D) continue;
#pragma unroll
          for (int k = 0; k < KP1; ++k) {
            const int pd = sDn[st * KP1 + k][lane];
            const double* dn = P.Yin + ((pd >> 5) * TB + (pd & 31));
            int q = 0;
#pragma unroll
            for (int o = 0; o < D; ++o) {
              const int p0 = o == st ? st : Pk<D>::re(st, o);
              double v0 = 0.0, v1 = 0.0;
              if (pd >= 0) v0 = __ldg(dn + p0 * TILE);
              if (o != st && pd >= 0) v1 = __ldg(dn + (p0 + 1) * TILE);
              g[j][k][q++] = v0;
              if (o != st) g[j][k][q++] = v1;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int st = s0 + j;
          if (st >= D) continue;
          double x[NP];
          x[st] = tm_ld2(col(st));
#pragma unroll
          for (int o = 0; o < D; ++o)
            if (o != st) tm_ld4(col(Pk<D>::re(st, o)), x[Pk<D>::re(st, o)], x[Pk<D>::re(st, o) + 1]);
          tm_wait_ld();
#pragma unroll
          for (int k = 0; k < KP1; ++k) {
            const int m = st * KP1 + k;
            const double n = sDn[m][lane] >= 0 ? (double)sN[m][lane] : 0.0;
            const double cb = n * (k == 0 ? cbk0 : cbk1), ca = n * (k == 0 ? cak0 : cak1);
            int q = 0;
#pragma unroll
            for (int o = 0; o < D; ++o) {
              if (o == st) {
                x[st] = fma(2.0 * cb, g[j][k][q++], x[st]);
                continue;
              }
              const int pr = Pk<D>::re(st, o), pim = pr + 1;
              const double dr = g[j][k][q], di = g[j][k][q + 1];
              q += 2;
              if (o > st) {
                x[pr] = fma(cb, dr, fma(-ca, di, x[pr]));
                x[pim] = fma(cb, di, fma(ca, dr, x[pim]));
              } else {
                x[pr] = fma(cb, dr, fma(ca, di, x[pr]));
                x[pim] = fma(cb, di, fma(-ca, dr, x[pim]));
              }
            }
          }
          tm_st2(col(st), x[st]);
#pragma unroll
          for (int o = 0; o < D; ++o)
            if (o != st) tm_st4(col(Pk<D>::re(st, o)), x[Pk<D>::re(st, o)], x[Pk<D>::re(st, o) + 1]);
          tm_wait_st();
        }
      }
    } else
#pragma unroll
    for (int st = 0; st < D; ++st) {
      double x[NP];  // only the 2D-1 cross planes of st are touched (compile-time indices)
      x[st] = tm_ld2(col(st));
#pragma unroll
      for (int o = 0; o < D; ++o) {
        if (o == st) continue;
        const int pr = Pk<D>::re(st, o);
        tm_ld4(col(pr), x[pr], x[pr + 1]);
      }
#pragma unroll
      for (int k = 0; k < KP1; ++k) {
        const int m = st * KP1 + k;
        const int pu = sUp[m][lane], pd = sDn[m][lane];
        const bool vu = pu >= 0, vd = pd >= 0;
        const double* up = P.Yin + ((pu >> 5) * TB + (pu & 31));
        const double* dn = P.Yin + ((pd >> 5) * TB + (pd & 31));
        const double n = vd ? (double)sN[m][lane] : 0.0;
        const double cb = n * (k == 0 ? cbk0 : cbk1), ca = n * (k == 0 ? cak0 : cak1);
        const double cu = vu ? c : 0.0;
        auto ld = [](const double* q, bool v) -> double {
          double r = 0.0;
          if (v) r = __ldg(q);
          return r;
        };
        if (k == 0) tm_wait_ld();
        x[st] = fma(2.0 * cb, ld(dn + st * TILE, vd), x[st]);
#pragma unroll
        for (int o = 0; o < D; ++o) {
          if (o == st) continue;
          const int pr = Pk<D>::re(st, o), pim = Pk<D>::im(st, o);
          const double ur = ld(up + pr * TILE, vu), ui = ld(up + pim * TILE, vu);
          const double dr = ld(dn + pr * TILE, vd), di = ld(dn + pim * TILE, vd);
          if (o > st) {
            x[pr] = fma(cb, dr, fma(-ca, di, fma(-cu, ui, x[pr])));
            x[pim] = fma(cb, di, fma(ca, dr, fma(cu, ur, x[pim])));
          } else {
            x[pr] = fma(cb, dr, fma(ca, di, fma(cu, ui, x[pr])));
            x[pim] = fma(cb, di, fma(-ca, dr, fma(-cu, ur, x[pim])));
          }
        }
      }
      tm_st2(col(st), x[st]);
#pragma unroll
      for (int o = 0; o < D; ++o) {
        if (o == st) continue;
        const int pr = Pk<D>::re(st, o);
        tm_st4(col(pr), x[pr], x[pr + 1]);
      }
      tm_wait_st();  // the next site's cross overlaps this one
    }
    // ---- phase C: TMEM -> global (stage 2 also B = (Y2 - s)/3 + 2/3 Y3)
    auto emit = [&](int p, double y) {
      if (LATE && STAGE >= 2) {
        const double sg = __ldg((STAGE == 4 ? P.Bbuf : P.sig) + own + p * TILE);
        if (STAGE == 2) {
          const double y2 = __ldg(P.Yin + own + p * TILE);
          y += sg;
          P.Bbuf[own + p * TILE] = fma(2.0 / 3.0, y, (y2 - sg) * (1.0 / 3.0));
        } else {
          y += sg;
        }
      } else if (STAGE == 2) {
        P.Bbuf[own + p * TILE] = fma(2.0 / 3.0, y, sBase[p][lane]);
      }
      P.Yout[own + p * TILE] = y;
      return y;
    };
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const double y = tm_ld2(col(i));
      tm_wait_ld();
      const double yo = emit(i, y);
      if (STAGE == 4) maxa2 = fmax(maxa2, yo * yo);
    }
#pragma unroll
    for (int pr = D; pr < NP; pr += 2) {
      double yr, yi;
      tm_ld4(col(pr), yr, yi);
      tm_wait_ld();
      yr = emit(pr, yr);
      yi = emit(pr + 1, yi);
      if (STAGE == 4) maxa2 = fmax(maxa2, fma(yr, yr, yi * yi));
    }
  }
  // ---- TMEM release (all warps done), then the stage-4 bookkeeping
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*s_taddr),
                 "n"(kMm8Cols)
                 : "memory");
  }
  if (STAGE == 4) stage4_finish<D>(P, step_next, maxa2);
}

template <int D, int KP1, int STAGE, int MINB, bool LATE>
static cudaError_t mm8_go(const KParams& p, cudaStream_t s) {
  constexpr size_t bytes = Mm8Smem<D, KP1, STAGE, LATE>::BYTES;
  static const cudaError_t attr = cudaFuncSetAttribute(
      k_mm8<D, KP1, STAGE, MINB, LATE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (attr != cudaSuccess) return attr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((p.n_tiles + kMm8Warps - 1) / kMm8Warps));
  cfg.blockDim = dim3(32 * kMm8Warps);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = s;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_mm8<D, KP1, STAGE, MINB, LATE>, p);
}

template <int MINB, bool LATE>
static cudaError_t mm8_stage(int stage, const KParams& p, cudaStream_t s) {
  switch (stage) {
    case 1: return mm8_go<7, 2, 1, MINB, LATE>(p, s);
    case 2: return mm8_go<7, 2, 2, MINB, LATE>(p, s);
    case 3: return mm8_go<7, 2, 3, MINB, LATE>(p, s);
    case 4: return mm8_go<7, 2, 4, MINB, LATE>(p, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_mm8(int stage, const KParams& p, cudaStream_t s) {
  // HB_MM8_MINB (experiments): CTAs (warpgroups) per SM the registers are cut for
  static const int minb = [] {
    const char* e = getenv("HB_MM8_MINB");
    return e ? atoi(e) : 3;
  }();
  // HB_MM8_LATE (experiments): 1 = base operands in phase C (default), 0 = bulk copy
  static const bool late = [] {
    const char* e = getenv("HB_MM8_LATE");
    return e ? atoi(e) != 0 : true;
  }();
  if (p.d != 7 || p.kp1 != 2 || p.single) return cudaErrorInvalidValue;
  if (minb == 2) return late ? mm8_stage<2, true>(stage, p, s) : mm8_stage<2, false>(stage, p, s);
  return late ? mm8_stage<3, true>(stage, p, s) : mm8_stage<3, false>(stage, p, s);
}

}  // namespace hb
