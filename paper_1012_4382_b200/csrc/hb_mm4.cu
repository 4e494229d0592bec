// Production stage kernel (variant 7, k_mm4): k_mm3's 12-pass RK bookkeeping
// and register accumulator, re-cut for occupancy and FP64 issue.
//
// What the k_mm3 ncu capture (profiles/r1_ncu_k_mm3_*.csv) showed: 254
// registers -> 8 warps per SM, long-scoreboard stalls ~2.5 per issue, and
// 1,878 FP64 instructions per tile-stage of which 679 DADD and 469 DMUL (the
// `a*b - c*d` forms were not contracted), plus 350 CS2R zeroing the
// predicated-off gathers.  Here:
//   * every RHS term is one explicit DFMA into the register accumulator: the
//     RK stage coefficient c is folded into the link coefficients once per link
//     (c*n*b_k, c*n*a_k, and c for a raise link), so nothing is scaled twice;
//   * an absent link (TRUNCATED raise at the top tier, ABSENT lower where
//     n_m = 0) is redirected to the lane's OWN ADO (an L1 hit, loaded in phase
//     A) with coefficient 0 -- no zeroing moves, no zero tile, no L2 traffic;
//   * the tile's base operand (sigma, or B at stage 4) and its three link
//     tables ([mode][32] int32 raise/lower, uint8 n) arrive by one bulk copy
//     group (cp.async.bulk, one mbarrier) at kernel start: no per-lane table
//     LDG/STS round trip, the raw positions are decoded to element offsets
//     where they are used.
// The arithmetic is the reference RHS (_kernels.py:23-58 generalised to K+1
// modes per site); the stage combinations are k_mm2's (hb_fast.cu):
//   stage 1: Y2 = s + h/2 k1;  2: Y3 = s + h/2 k2, B = (Y2 - s)/3 + 2/3 Y3;
//   stage 3: Y4 = s + h k3;    4: s = B + Y4/3 + h/6 k4          (heom.py:370-381)
#include <cstdlib>
#include "hb_device.cuh"
#include "hb_fast.cuh"
#include "hb_mm_common.cuh"

namespace hb {

__device__ __forceinline__ void pf_l1(const double* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// VAR (experiments, HB_MM4_VAR): bit 0 = predicate absent links off (zero) instead
// of redirecting them to the own ADO; bit 1 = prefetch the next site's crosses
// into L1 while the current site is gathered; bit 2 = skip the neighbour
// crosses (timing experiment only, wrong results).
template <int D, int KP1, int STAGE, int MINB, int VAR>
__global__ void __launch_bounds__(32, MINB) k_mm4(const KParams P) {
  constexpr bool kPred = VAR & 1, kPf = VAR & 2, kNoB = VAR & 4;
  constexpr int NP = D * D;
  constexpr int M = D * KP1;
  constexpr int TB = NP * TILE;
  constexpr bool kBase = STAGE >= 2;
  __shared__ __align__(128) double sBase[kBase ? NP : 1][TILE];
  __shared__ __align__(16) int32_t sUp[M][TILE];
  __shared__ __align__(16) int32_t sDn[M][TILE];
  __shared__ __align__(16) uint8_t sN[M][TILE];
  __shared__ __align__(8) uint64_t bar;

  volatile Ctl* ctl = P.ctl;
  if (ctl->status != ST_RUNNING) return;
  const long long step_next = ctl->step + 1;
  const int lane = threadIdx.x;
  const int tile = P.tile_begin + blockIdx.x;
  const size_t toff = (size_t)tile * TB;
  const int own = (int)toff + lane;  // element offset of this lane's ADO, plane 0
  const double c = STAGE == 4 ? P.dt / 6.0 : P.coef;

  tile_prologue<D, KP1, STAGE>(P, tile, &sBase[0][0], &sUp[0][0], &sDn[0][0], &sN[0][0], &bar);

  double acc[NP];
  phase_a<D, KP1, STAGE>(P, tile, lane, own, c, sBase, sN, &bar, acc);
  // ---- phase B: neighbour crosses, one site at a time, straight into acc
  double cbk[KP1], cak[KP1];
#pragma unroll
  for (int k = 0; k < KP1; ++k) {
    cbk[k] = c * P.b[k];
    cak[k] = c * P.a[k];
  }
  auto prefetch_site = [&](int st) {
#pragma unroll
    for (int k = 0; k < KP1; ++k) {
      const int m = st * KP1 + k;
      const int pu = sUp[m][lane], pd = sDn[m][lane];
      const double* up = P.Yin + ((pu >> 5) * TB + (pu & 31));
      const double* dn = P.Yin + ((pd >> 5) * TB + (pd & 31));
#pragma unroll
      for (int o = 0; o < D; ++o) {
        const int pr = Pk<D>::re(st, o);
        if (pd >= 0) pf_l1(dn + pr * TILE);
        if (o != st && pu >= 0) pf_l1(up + pr * TILE);
        if (o != st) {
          const int pim = Pk<D>::im(st, o);
          if (pd >= 0) pf_l1(dn + pim * TILE);
          if (pu >= 0) pf_l1(up + pim * TILE);
        }
      }
    }
  };
  if (kPf) prefetch_site(0);
#pragma unroll
  for (int st = 0; st < (kNoB ? 0 : D); ++st) {
    if (kPf && st + 1 < D) prefetch_site(st + 1);
#pragma unroll
    for (int k = 0; k < KP1; ++k) {
      const int m = st * KP1 + k;
      const int pu = sUp[m][lane], pd = sDn[m][lane];
      const bool vu = pu >= 0, vd = pd >= 0;
      const double* up = P.Yin + (vu ? (pu >> 5) * TB + (pu & 31) : own);
      const double* dn = P.Yin + (vd ? (pd >> 5) * TB + (pd & 31) : own);
      const double n = vd ? (double)sN[m][lane] : 0.0;
      const double cb = n * cbk[k], ca = n * cak[k];
      const double cu = vu ? c : 0.0;
      auto ld = [&](const double* q, bool v) -> double {
        if (!kPred) return __ldg(q);
        double r = 0.0;
        if (v) r = __ldg(q);
        return r;
      };
      acc[st] = fma(2.0 * cb, ld(dn + st * TILE, vd), acc[st]);
#pragma unroll
      for (int o = 0; o < D; ++o) {
        if (o == st) continue;
        const int pr = Pk<D>::re(st, o), pim = Pk<D>::im(st, o);
        const double ur = ld(up + pr * TILE, vu), ui = ld(up + pim * TILE, vu);
        const double dr = ld(dn + pr * TILE, vd), di = ld(dn + pim * TILE, vd);
        if (o > st) {  // element (st, o): row st
          acc[pr] = fma(cb, dr, fma(-ca, di, fma(-cu, ui, acc[pr])));
          acc[pim] = fma(cb, di, fma(ca, dr, fma(cu, ur, acc[pim])));
        } else {       // element (o, st): column st
          acc[pr] = fma(cb, dr, fma(ca, di, fma(cu, ui, acc[pr])));
          acc[pim] = fma(cb, di, fma(-ca, dr, fma(-cu, ur, acc[pim])));
        }
      }
    }
  }
  phase_c<D, STAGE>(P, lane, own, step_next, sBase, acc);
}

template <int D, int KP1, int MINB, int VAR>
static cudaError_t mm4_launch_b(int stage, const KParams& p, cudaStream_t s) {
  switch (stage) {
    case 1: k_mm4<D, KP1, 1, MINB, VAR><<<p.n_tiles, 32, 0, s>>>(p); break;
    case 2: k_mm4<D, KP1, 2, MINB, VAR><<<p.n_tiles, 32, 0, s>>>(p); break;
    case 3: k_mm4<D, KP1, 3, MINB, VAR><<<p.n_tiles, 32, 0, s>>>(p); break;
    case 4: k_mm4<D, KP1, 4, MINB, VAR><<<p.n_tiles, 32, 0, s>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

template <int D, int KP1>
static cudaError_t mm4_launch_t(int stage, const KParams& p, cudaStream_t s) {
  // HB_MM4_VAR (experiments): see k_mm4's VAR bits
  static const int var = env_int("HB_MM4_VAR", 1);
  if constexpr (D == 7) {
    switch (var) {
      case 0: return mm4_launch_b<D, KP1, 1, 0>(stage, p, s);
      case 1: return mm4_launch_b<D, KP1, 1, 1>(stage, p, s);
      case 2: return mm4_launch_b<D, KP1, 1, 2>(stage, p, s);
      case 5: return mm4_launch_b<D, KP1, 1, 5>(stage, p, s);
      default: break;
    }
  }
  return mm4_launch_b<D, KP1, 1, 3>(stage, p, s);
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
