// Phases shared by the register-accumulator stage kernels k_mm4 / k_mm5:
//   tile_prologue  -- one elected lane bulk-copies the tile's link tables
//                     ([mode][32] raise / lower int32, n uint8) and, at stages 2-4,
//                     its base operand (sigma, or B at stage 4) into shared memory;
//   phase_a        -- acc = base + c * (-(damping) s - i[H, s]), the ADO in
//                     registers, H from the constant bank; also the sink rates
//                     of the stage input (heom.py:282-283) on tile 0;
//   phase_c        -- store (stage 2 also B), stage-4 max|x|^2 and the
//                     last-CTA step bookkeeping (heom.py:381-394).
// The stage combinations (12 state passes per step) are k_mm2's (hb_fast.cu) for
// T = double.  For T = float (precision='single') that scheme's differences of
// rounded stage values ((Y2 - s)/3 ...) cost several float ulps of sigma per step,
// so the float path carries the RK increment instead (kInc, 15 float passes):
//   stage 1: Y2 = s + a1,          Binc = a1 / 3            (a1 = h/2 k1)
//   stage 2: Y3 = s + a2,          Binc += 2/3 a2           (a2 = h/2 k2)
//   stage 3: Y4 = s + a3                                    (a3 = h k3)
//   stage 4: s  = s + (Binc + a4 + (Y4 - s)/3)             (a4 = h/6 k4)
// acc holds the increment a_s (never the rounded sum), so sigma is rounded once
// per step like the reference's rk4_update (_kernels.py:68-72, heom.py:381).
#pragma once
#include <type_traits>
#include "hb_device.cuh"
#include "hb_fast.cuh"

namespace hb {

// operands in the kernel's arithmetic type (HB_PREC_SINGLE: float copies in KParams)
template <class T> struct Opd;
template <> struct Opd<double> {
  static __device__ __forceinline__ double h(const KParams& P, int i) { return P.h[i]; }
  static __device__ __forceinline__ double decay(const KParams& P, int i) { return P.decay[i]; }
  static __device__ __forceinline__ double nu(const KParams& P, int k) { return P.nu[k]; }
  static __device__ __forceinline__ double a(const KParams& P, int k) { return P.a[k]; }
  static __device__ __forceinline__ double b(const KParams& P, int k) { return P.b[k]; }
};
template <> struct Opd<float> {
  static __device__ __forceinline__ float h(const KParams& P, int i) { return P.hf[i]; }
  static __device__ __forceinline__ float decay(const KParams& P, int i) { return P.decayf[i]; }
  static __device__ __forceinline__ float nu(const KParams& P, int k) { return P.nuf[k]; }
  static __device__ __forceinline__ float a(const KParams& P, int k) { return P.af[k]; }
  static __device__ __forceinline__ float b(const KParams& P, int k) { return P.bf[k]; }
};
// state buffers of the stage (KParams keeps them as double*; float when single)
template <class T> __device__ __forceinline__ const T* st_in(const KParams& P) {
  return reinterpret_cast<const T*>(P.Yin);
}
template <class T> __device__ __forceinline__ T* st_out(const KParams& P) {
  return reinterpret_cast<T*>(P.Yout);
}
template <class T> __device__ __forceinline__ T* st_b(const KParams& P) {
  return reinterpret_cast<T*>(P.Bbuf);
}
template <class T> __device__ __forceinline__ const T* st_sig(const KParams& P) {
  return reinterpret_cast<const T*>(P.sig);
}

template <int D, int KP1>
struct MmSmem {
  static constexpr int NP = D * D, M = D * KP1;
};

// float state: increment scheme (see the header)
template <class T>
constexpr bool kIncScheme = std::is_same<T, float>::value;

// HB_TBL_KEEP (build-time experiment): link-table bulk copies with an L2
// evict-last policy
#ifndef HB_TBL_KEEP
#define HB_TBL_KEEP 0
#endif

template <class T, int D, int KP1, int STAGE>
__device__ __forceinline__ void tile_prologue(const KParams& P, int tile, T* sBase,
                                              int32_t* sUp, int32_t* sDn, uint8_t* sN,
                                              uint64_t* bar, bool init = true,
                                              T* sInc = nullptr, bool defer_inc = false) {
  constexpr int NP = D * D, M = D * KP1, TB = NP * TILE;
  constexpr bool kInc = kIncScheme<T>;
  constexpr bool kLoadInc = kInc && (STAGE == 2 || STAGE == 4);
  if ((threadIdx.x & 31) == 0) {
    constexpr unsigned LB = M * TILE * 4u, NB = M * TILE;
    if (init) {
      mbar_init(bar, 1);
    } else {  // the warp's generic-proxy reads of the previous tile precede the refill
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    mbar_expect_tx(bar, 2 * LB + NB + (STAGE >= 2 ? TB * (unsigned)sizeof(T) : 0u) +
                            (kLoadInc ? TB * (unsigned)sizeof(T) : 0u));
    const size_t gt = (size_t)tile * M * TILE;
#if HB_TBL_KEEP
    bulk_g2s_keep(sUp, P.plus + gt, LB, bar);
    bulk_g2s_keep(sDn, P.minus + gt, LB, bar);
    bulk_g2s_keep(sN, P.nvec + gt, NB, bar);
#else
    bulk_g2s(sUp, P.plus + gt, LB, bar);
    bulk_g2s(sDn, P.minus + gt, LB, bar);
    bulk_g2s(sN, P.nvec + gt, NB, bar);
#endif
    if (STAGE >= 2)
      bulk_g2s(sBase, (STAGE == 4 && !kInc ? st_b<T>(P) : st_sig<T>(P)) + (size_t)tile * TB,
               TB * (unsigned)sizeof(T), bar);
    if (kLoadInc && !defer_inc)
      bulk_g2s(sInc, st_b<T>(P) + (size_t)tile * TB, TB * (unsigned)sizeof(T), bar);
  }
  __syncwarp();  // barrier initialised before any lane waits on it
}

// the increment tile copy held back by tile_prologue(defer_inc): issued once the
// kernel that writes it (stage 1 of the float scheme) is known to be complete
template <class T, int D, int STAGE>
__device__ __forceinline__ void tile_prologue_late(const KParams& P, int tile, T* sInc,
                                                   uint64_t* bar) {
  constexpr int TB = D * D * TILE;
  if (kIncScheme<T> && (STAGE == 2 || STAGE == 4) && (threadIdx.x & 31) == 0)
    bulk_g2s(sInc, st_b<T>(P) + (size_t)tile * TB, TB * (unsigned)sizeof(T), bar);
}

// Programmatic dependent launch (PDL).  A stage kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while the previous
// stage's last wave drains: it issues the bulk copies of operands no running
// kernel writes (link tables; sigma, or B at stage 4, whose writers finished two
// launches back), then waits for the previous grid to complete and flush
// (griddepcontrol.wait) before touching its stage input or the control block,
// and releases its own dependent right after that wait.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// status: the run's status read at kernel start (its load overlaps the tile's);
// returns false -- after draining the bulk copy, before any global write --
// when the run is no longer RUNNING (graph replays past the stop are no-ops)
// LATE (double scheme): the base operand is added in phase C (phase_c_store<LATE>)
// instead of coming from shared memory here; acc holds s at stage 1, s/3 at
// stage 4 and 0 otherwise, plus the increment
template <class T, int D, int KP1, int STAGE, bool LATE = false>
__device__ __forceinline__ bool phase_a(const KParams& P, int tile, int lane, int own, T c,
                                        T (*sBase)[TILE], const uint8_t (*sN)[TILE],
                                        uint64_t* bar, T (&acc)[D * D],
                                        unsigned parity = 0, int status = ST_RUNNING) {
  constexpr int NP = D * D, M = D * KP1;
  volatile Ctl* ctl = P.ctl;
  {  // ---- phase A: base + c * (damping + commutator), ADO in registers
    T s[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) s[p] = __ldg(st_in<T>(P) + own + p * TILE);
    if (status != ST_RUNNING) {
      mbar_wait(bar, parity);
      return false;
    }
    if (tile == 0 && lane == 0) {  // sink rates of this stage input (heom.py:282-283)
      int q = 0;
      for (int sk = 0; sk < P.n_sinks; ++sk) {
        double a = 0.0;
        for (int cc = 0; cc < P.sink_nterms[sk]; ++cc, ++q) {
          const double v = P.sink_rate[q] * (double)__ldg(st_in<T>(P) + P.sink_pos[q] * TILE);
          a = cc == 0 ? v : a + v;
        }
        ctl->r[STAGE - 1][sk] = a;
      }
    }
    mbar_wait(bar, parity);
    // damping sum_k nu_k sum_j n_jk (heom.py:275, generalised), pre-scaled by c
    int tk[KP1];
#pragma unroll
    for (int k = 0; k < KP1; ++k) tk[k] = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) tk[m % KP1] += sN[m][lane];
    T damp = 0;
#pragma unroll
    for (int k = 0; k < KP1; ++k) damp = fma((T)tk[k], Opd<T>::nu(P, k), damp);
    constexpr T third = (T)(1.0 / 3.0);
    auto base = [&](int p) -> T {
      if (kIncScheme<T>) {  // acc = increment; sigma kept (stage 1) or TMA'd in sBase
        if (STAGE == 1) sBase[p][lane] = s[p];
        if (STAGE == 4) return (s[p] - sBase[p][lane]) * third;  // (Y4 - s)/3
        return (T)0;
      }
      if (STAGE == 1) return s[p];
      if (LATE) return STAGE == 4 ? s[p] * third : (T)0;
      const T b = sBase[p][lane];
      if (STAGE == 2) sBase[p][lane] = (s[p] - b) * third;  // park (Y2 - s)/3 for B
      if (STAGE == 4) return fma(s[p], third, b);
      return b;
    };
#pragma unroll
    for (int i = 0; i < D; ++i) {
      // diagonal: Re(-i[H,s])_ii = 2 sum_{l != i} h_il Im s_il
      T cm = 0;
#pragma unroll
      for (int l = 0; l < D; ++l)
        if (l != i) cm = fma(Opd<T>::h(P, i * MAXD + l), sim<T, D>(s, i, l), cm);
      const T fi = -(damp + Opd<T>::decay(P, i));
      acc[i] = fma(c, fma(fi, s[i], (T)-2 * cm), base(i));
#pragma unroll
      for (int j = i + 1; j < D; ++j) {
        const int pr = Pk<D>::re(i, j), pim = Pk<D>::im(i, j);
        // [H,s]_ij = sum_l h_il s_lj - s_il h_lj; the l = i and l = j terms pair up:
        // (h_ii - h_jj) s_ij + h_ij (s_jj - s_ii)  (s_ii, s_jj real)
        const T dh = Opd<T>::h(P, i * MAXD + i) - Opd<T>::h(P, j * MAXD + j);
        const T hij = Opd<T>::h(P, i * MAXD + j);
        T cr = fma(hij, s[j], fma(-hij, s[i], dh * s[pr]));
        T ci = dh * s[pim];
#pragma unroll
        for (int l = 0; l < D; ++l) {
          if (l == i || l == j) continue;
          const T hil = Opd<T>::h(P, i * MAXD + l), hlj = Opd<T>::h(P, l * MAXD + j);
          cr = fma(hil, sre<T, D>(s, l, j), cr);
          cr = fma(-hlj, sre<T, D>(s, i, l), cr);
          ci = fma(hil, sim<T, D>(s, l, j), ci);
          ci = fma(-hlj, sim<T, D>(s, i, l), ci);
        }
        const T f = -(damp + (T)0.5 * (Opd<T>::decay(P, i) + Opd<T>::decay(P, j)));
        acc[pr] = fma(c, fma(f, s[pr], ci), base(pr));   // -1j * [H,s]
        acc[pim] = fma(c, fma(f, s[pim], -cr), base(pim));
      }
    }
  }
  return true;
}

// phase B: the neighbour crosses, one site at a time (2(K+1) links, 2d-1 planes
// each, all loads of a site independent), absent links predicated off, every
// term one DFMA into the register accumulator (c folded into the coefficients)
// PAIRED: a tile none of whose lanes has a raise link (every ADO on the top
// tier -- whole tiles only in the tier-major order) gathers two sites' lower
// links per round trip (the same 4(2d-1) loads as one full site), halving the
// rounds of that tile
// [S0, S1): the sites this warp gathers (k_mm4's split CTAs give a tile's sites
// to two warps)
template <class T, int D, int KP1, bool PAIRED = false, int GROUP = 2, int S0 = 0, int S1 = D>
__device__ __forceinline__ void phase_b_sites(const KParams& P, int lane, T c,
                                              const int32_t (*sUp)[TILE],
                                              const int32_t (*sDn)[TILE],
                                              const uint8_t (*sN)[TILE], T (&acc)[D * D]) {
  constexpr int TB = D * D * TILE;
  const T* yin = st_in<T>(P);
  T cbk[KP1], cak[KP1];
#pragma unroll
  for (int k = 0; k < KP1; ++k) {
    cbk[k] = c * Opd<T>::b(P, k);
    cak[k] = c * Opd<T>::a(P, k);
  }
  if (PAIRED) {
    bool up_any = false;
#pragma unroll
    for (int m = 0; m < D * KP1; ++m) up_any |= sUp[m][lane] >= 0;
    if (!__any_sync(0xffffffffu, up_any)) {
#pragma unroll
      for (int s0 = S0; s0 < S1; s0 += GROUP) {
#pragma unroll
        for (int st = s0; st < (s0 + GROUP < S1 ? s0 + GROUP : S1); ++st) {
#pragma unroll
          for (int k = 0; k < KP1; ++k) {
            const int m = st * KP1 + k;
            const int pd = sDn[m][lane];
            const bool vd = pd >= 0;
            const T* dn = yin + ((pd >> 5) * TB + (pd & 31));
            const T n = vd ? (T)sN[m][lane] : (T)0;
            const T cb = n * cbk[k], ca = n * cak[k];
            auto ld = [](const T* q, bool v) -> T {
              T r = 0;
              if (v) r = __ldg(q);
              return r;
            };
            acc[st] = fma((T)2 * cb, ld(dn + st * TILE, vd), acc[st]);
#pragma unroll
            for (int o = 0; o < D; ++o) {
              if (o == st) continue;
              const int pr = Pk<D>::re(st, o), pim = Pk<D>::im(st, o);
              const T dr = ld(dn + pr * TILE, vd), di = ld(dn + pim * TILE, vd);
              if (o > st) {
                acc[pr] = fma(cb, dr, fma(-ca, di, acc[pr]));
                acc[pim] = fma(cb, di, fma(ca, dr, acc[pim]));
              } else {
                acc[pr] = fma(cb, dr, fma(ca, di, acc[pr]));
                acc[pim] = fma(cb, di, fma(-ca, dr, acc[pim]));
              }
            }
          }
        }
      }
      return;
    }
  }
#pragma unroll
  for (int st = S0; st < S1; ++st) {
#pragma unroll
    for (int k = 0; k < KP1; ++k) {
      const int m = st * KP1 + k;
      const int pu = sUp[m][lane], pd = sDn[m][lane];
      const bool vu = pu >= 0, vd = pd >= 0;
      const T* up = yin + ((pu >> 5) * TB + (pu & 31));
      const T* dn = yin + ((pd >> 5) * TB + (pd & 31));
      const T n = vd ? (T)sN[m][lane] : (T)0;
      const T cb = n * cbk[k], ca = n * cak[k];
      const T cu = vu ? c : (T)0;
      auto ld = [](const T* q, bool v) -> T {
        T r = 0;
        if (v) r = __ldg(q);
        return r;
      };
      acc[st] = fma((T)2 * cb, ld(dn + st * TILE, vd), acc[st]);
#pragma unroll
      for (int o = 0; o < D; ++o) {
        if (o == st) continue;
        const int pr = Pk<D>::re(st, o), pim = Pk<D>::im(st, o);
        const T ur = ld(up + pr * TILE, vu), ui = ld(up + pim * TILE, vu);
        const T dr = ld(dn + pr * TILE, vd), di = ld(dn + pim * TILE, vd);
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
}

// HB_ST_CS (build-time experiment): 1 = B (read two stages later) stored
// evict-first (st.global.cs); 2 = the stage output too; 0 = plain stores
#ifndef HB_ST_CS
#define HB_ST_CS 0
#endif
template <class T> __device__ __forceinline__ void st_y(T* q, T v) {
  if (HB_ST_CS >= 2) __stcs(q, v); else *q = v;
}
template <class T> __device__ __forceinline__ void st_bb(T* q, T v) {
  if (HB_ST_CS >= 1) __stcs(q, v); else *q = v;
}

template <class T, int D, int STAGE, bool LATE = false>
__device__ __forceinline__ void phase_c_store(const KParams& P, int lane, int own,
                                              T (*sBase)[TILE], T (&acc)[D * D],
                                              double& maxa2, T (*sInc)[TILE] = nullptr) {
  constexpr int NP = D * D;
  constexpr T third = (T)(1.0 / 3.0), two3 = (T)(2.0 / 3.0);
  if (LATE && STAGE >= 2) {  // base operands now: sigma (2, 3), B (4); stage 2 re-reads Y2
    const T* bs = STAGE == 4 ? st_b<T>(P) : st_sig<T>(P);
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const T sg = __ldg(bs + own + p * TILE);
      if (STAGE == 2) {
        const T y2 = __ldg(st_in<T>(P) + own + p * TILE);
        acc[p] += sg;
        st_b<T>(P)[own + p * TILE] = fma(two3, acc[p], (y2 - sg) * third);
      } else {
        acc[p] += sg;
      }
    }
  }
  // ---- phase C: store (stage 2 also B = (Y2 - s)/3 + 2/3 Y3; float: see header)
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    if (LATE) {
      st_out<T>(P)[own + p * TILE] = acc[p];
    } else if (kIncScheme<T>) {
      const T a = acc[p], sg = sBase[p][lane];
      if (STAGE == 1) st_b<T>(P)[own + p * TILE] = a * third;
      if (STAGE == 2) st_b<T>(P)[own + p * TILE] = fma(two3, a, sInc[p][lane]);
      acc[p] = STAGE == 4 ? sg + (sInc[p][lane] + a) : sg + a;
      st_out<T>(P)[own + p * TILE] = acc[p];
    } else {
      st_y(st_out<T>(P) + own + p * TILE, acc[p]);
      if (STAGE == 2) st_bb(st_b<T>(P) + own + p * TILE, fma(two3, acc[p], sBase[p][lane]));
    }
  }
  if (STAGE == 4) {  // max |y|^2 per element (diagonal planes are real)
#pragma unroll
    for (int i = 0; i < D; ++i) {
      maxa2 = fmax(maxa2, (double)acc[i] * (double)acc[i]);
#pragma unroll
      for (int j = i + 1; j < D; ++j) {
        const double yr = acc[Pk<D>::re(i, j)], yi = acc[Pk<D>::im(i, j)];
        maxa2 = fmax(maxa2, fma(yr, yr, yi * yi));
      }
    }
  }
}

// stage 4, after every warp of the CTA has stored: the divergence max (every 25
// steps, heom.py:323) and the last-CTA election that runs the step bookkeeping
template <int D>
__device__ __forceinline__ void stage4_finish(const KParams& P, long long step_next, double maxa2) {
  volatile Ctl* ctl = P.ctl;
  const int lane = threadIdx.x & 31;
  __shared__ int s_last;
  if (step_next % 25 == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
    if (lane == 0)
      atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                (unsigned long long)__double_as_longlong(maxa2));
  }
  // the last CTA's bookkeeping reads sigma^0 and the stage-4 sink rates (both
  // written by the CTA holding tile 0) and, every 25 steps, the max|x|^2 atomics:
  // only those writes must be visible before the election counter moves
  if (step_next % 25 == 0 || (P.tile_begin == 0 && blockIdx.x == 0)) __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(const_cast<unsigned*>(&ctl->blocks_done), 1u);
    s_last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x < 32) {
    __threadfence();
    if (lane == 0) ctl->launches = ctl->launches + 4;
    finish_step_warp<D, true>(P, step_next);
  }
}

template <class T, int D, int STAGE>
__device__ __forceinline__ void phase_c(const KParams& P, int lane, int own, long long step_next,
                                        T (*sBase)[TILE], T (&acc)[D * D],
                                        T (*sInc)[TILE] = nullptr) {
  double maxa2 = 0.0;
  phase_c_store<T, D, STAGE>(P, lane, own, sBase, acc, maxa2, sInc);
  if (STAGE == 4) stage4_finish<D>(P, step_next, maxa2);
}

}  // namespace hb
