// Phases shared by the register-accumulator stage kernels k_mm4 / k_mm5:
//   tile_prologue  -- one elected lane bulk-copies the tile's link tables
//                     ([mode][32] raise / lower int32, n uint8) and, at stages 2-4,
//                     its base operand (sigma, or B at stage 4) into shared memory;
//   phase_a        -- acc = base + c * (-(damping) s - i[H, s]), the ADO in
//                     registers, H from the constant bank; also the sink rates
//                     of the stage input (heom.py:282-283) on tile 0;
//   phase_c        -- store (stage 2 also B), stage-4 max|x|^2 and the
//                     last-CTA step bookkeeping (heom.py:381-394).
// The stage combinations (12 state passes per step) are k_mm2's (hb_fast.cu).
#pragma once
#include "hb_device.cuh"
#include "hb_fast.cuh"

namespace hb {

template <int D, int KP1>
struct MmSmem {
  static constexpr int NP = D * D, M = D * KP1;
};

template <int D, int KP1, int STAGE>
__device__ __forceinline__ void tile_prologue(const KParams& P, int tile, double* sBase,
                                              int32_t* sUp, int32_t* sDn, uint8_t* sN,
                                              uint64_t* bar, bool init = true) {
  constexpr int NP = D * D, M = D * KP1, TB = NP * TILE;
  if ((threadIdx.x & 31) == 0) {
    constexpr unsigned LB = M * TILE * 4u, NB = M * TILE;
    if (init) {
      mbar_init(bar, 1);
    } else {  // the warp's generic-proxy reads of the previous tile precede the refill
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    mbar_expect_tx(bar, 2 * LB + NB + (STAGE >= 2 ? TB * 8u : 0u));
    const size_t gt = (size_t)tile * M * TILE;
    bulk_g2s(sUp, P.plus + gt, LB, bar);
    bulk_g2s(sDn, P.minus + gt, LB, bar);
    bulk_g2s(sN, P.nvec + gt, NB, bar);
    if (STAGE >= 2) bulk_g2s(sBase, (STAGE == 4 ? P.Bbuf : P.sig) + (size_t)tile * TB, TB * 8u, bar);
  }
  __syncwarp();  // barrier initialised before any lane waits on it
}

// status: the run's status read at kernel start (its load overlaps the tile's);
// returns false -- after draining the bulk copy, before any global write --
// when the run is no longer RUNNING (graph replays past the stop are no-ops)
template <int D, int KP1, int STAGE>
__device__ __forceinline__ bool phase_a(const KParams& P, int tile, int lane, int own, double c,
                                        double (*sBase)[TILE], const uint8_t (*sN)[TILE],
                                        uint64_t* bar, double (&acc)[D * D],
                                        unsigned parity = 0, int status = ST_RUNNING) {
  constexpr int NP = D * D, M = D * KP1;
  volatile Ctl* ctl = P.ctl;
  {  // ---- phase A: base + c * (damping + commutator), ADO in registers
    double s[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) s[p] = __ldg(P.Yin + own + p * TILE);
    if (status != ST_RUNNING) {
      mbar_wait(bar, parity);
      return false;
    }
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
    mbar_wait(bar, parity);
    // damping sum_k nu_k sum_j n_jk (heom.py:275, generalised), pre-scaled by c
    int tk[KP1];
#pragma unroll
    for (int k = 0; k < KP1; ++k) tk[k] = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) tk[m % KP1] += sN[m][lane];
    double damp = 0.0;
#pragma unroll
    for (int k = 0; k < KP1; ++k) damp = fma((double)tk[k], P.nu[k], damp);
    auto base = [&](int p) -> double {
      if (STAGE == 1) return s[p];
      const double b = sBase[p][lane];
      if (STAGE == 2) sBase[p][lane] = (s[p] - b) * (1.0 / 3.0);  // park (Y2 - s)/3 for B
      if (STAGE == 4) return fma(s[p], 1.0 / 3.0, b);
      return b;
    };
#pragma unroll
    for (int i = 0; i < D; ++i) {
      // diagonal: Re(-i[H,s])_ii = 2 sum_{l != i} h_il Im s_il
      double cm = 0.0;
#pragma unroll
      for (int l = 0; l < D; ++l)
        if (l != i) cm = fma(P.h[i * MAXD + l], sim<D>(s, i, l), cm);
      const double fi = -(damp + P.decay[i]);
      acc[i] = fma(c, fma(fi, s[i], -2.0 * cm), base(i));
#pragma unroll
      for (int j = i + 1; j < D; ++j) {
        const int pr = Pk<D>::re(i, j), pim = Pk<D>::im(i, j);
        // [H,s]_ij = sum_l h_il s_lj - s_il h_lj; the l = i and l = j terms pair up:
        // (h_ii - h_jj) s_ij + h_ij (s_jj - s_ii)  (s_ii, s_jj real)
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
template <int D, int KP1>
__device__ __forceinline__ void phase_b_sites(const KParams& P, int lane, double c,
                                              const int32_t (*sUp)[TILE],
                                              const int32_t (*sDn)[TILE],
                                              const uint8_t (*sN)[TILE], double (&acc)[D * D]) {
  constexpr int TB = D * D * TILE;
  double cbk[KP1], cak[KP1];
#pragma unroll
  for (int k = 0; k < KP1; ++k) {
    cbk[k] = c * P.b[k];
    cak[k] = c * P.a[k];
  }
#pragma unroll
  for (int st = 0; st < D; ++st) {
#pragma unroll
    for (int k = 0; k < KP1; ++k) {
      const int m = st * KP1 + k;
      const int pu = sUp[m][lane], pd = sDn[m][lane];
      const bool vu = pu >= 0, vd = pd >= 0;
      const double* up = P.Yin + ((pu >> 5) * TB + (pu & 31));
      const double* dn = P.Yin + ((pd >> 5) * TB + (pd & 31));
      const double n = vd ? (double)sN[m][lane] : 0.0;
      const double cb = n * cbk[k], ca = n * cak[k];
      const double cu = vu ? c : 0.0;
      auto ld = [](const double* q, bool v) -> double {
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
}

template <int D, int STAGE>
__device__ __forceinline__ void phase_c_store(const KParams& P, int lane, int own,
                                              double (*sBase)[TILE], const double (&acc)[D * D],
                                              double& maxa2) {
  constexpr int NP = D * D;
  // ---- phase C: store (stage 2 also B = (Y2 - s)/3 + 2/3 Y3)
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    P.Yout[own + p * TILE] = acc[p];
    if (STAGE == 2) P.Bbuf[own + p * TILE] = fma(2.0 / 3.0, acc[p], sBase[p][lane]);
  }
  if (STAGE == 4) {  // max |y|^2 per element (diagonal planes are real)
#pragma unroll
    for (int i = 0; i < D; ++i) {
      maxa2 = fmax(maxa2, acc[i] * acc[i]);
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
  __threadfence();
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

template <int D, int STAGE>
__device__ __forceinline__ void phase_c(const KParams& P, int lane, int own, long long step_next,
                                        double (*sBase)[TILE], const double (&acc)[D * D]) {
  double maxa2 = 0.0;
  phase_c_store<D, STAGE>(P, lane, own, sBase, acc, maxa2);
  if (STAGE == 4) stage4_finish<D>(P, step_next, maxa2);
}

}  // namespace hb
