// Phases of the production stage kernel k_mm4 (hb_mm4.cu):
//   tile_prologue  -- one elected lane bulk-copies the tile's link tables
//                     ([mode][32] raise / lower int32, n uint8) and, at stages 2-4,
//                     its base operand (sigma, or B at stage 4) into shared memory;
//                     a tile of the top tier (no raise links) skips the raise table;
//   phase_a        -- acc = base + c * (-(damping) s - i[H, s]), the ADO in
//                     registers, H from the constant bank; also the sink rates
//                     of the stage input (heom.py:282-283) on tile 0;
//   phase_b_sites  -- the neighbour crosses (_kernels.py:41-57);
//   phase_c_store  -- store (stage 2 also B), stage-4 max|x|^2.
// The stage combinations (12 state passes per step) for T = double:
//   stage 1: Y2 = s + h/2 k1;  2: Y3 = s + h/2 k2, B = (Y2 - s)/3 + 2/3 Y3;
//   stage 3: Y4 = s + h k3;    4: s = B + Y4/3 + h/6 k4          (heom.py:370-381)
// For T = float (precision='single') that scheme's differences of rounded stage
// values ((Y2 - s)/3 ...) cost several float ulps of sigma per step, so the float
// path carries the RK increment instead (kInc, 15 float passes):
//   stage 1: Y2 = s + a1,          Binc = a1 / 3            (a1 = h/2 k1)
//   stage 2: Y3 = s + a2,          Binc += 2/3 a2           (a2 = h/2 k2)
//   stage 3: Y4 = s + a3                                    (a3 = h k3)
//   stage 4: s  = s + (Binc + a4 + (Y4 - s)/3)             (a4 = h/6 k4)
// acc holds the increment a_s (never the rounded sum), so sigma is rounded once
// per step like the reference's rk4_update (_kernels.py:68-72, heom.py:381).
#pragma once
#include <type_traits>
#include "hb_device.cuh"
#include "hb_tma.cuh"

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

// float state: increment scheme (see the header)
template <class T>
constexpr bool kIncScheme = std::is_same<T, float>::value;

// (re, im) pairs of the Hermitian tile layout (herm_off, hb_internal.h)
template <class T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };
template <class T> using v2_t = typename Vec2<T>::type;
template <class T> __device__ __forceinline__ v2_t<T> ldg2(const T* p) {
  return __ldg(reinterpret_cast<const v2_t<T>*>(p));
}
template <class T> __device__ __forceinline__ void st2(T* p, T x, T y) {
  v2_t<T> v;
  v.x = x;
  v.y = y;
  *reinterpret_cast<v2_t<T>*>(p) = v;
}
template <class T> __device__ __forceinline__ v2_t<T>& sm2(T* p) {
  return *reinterpret_cast<v2_t<T>*>(p);
}

// load_up = false: the tile has no raise links (top tier), its raise table is
// not copied
template <class T, int D, int KP1, int STAGE>
__device__ __forceinline__ void tile_prologue(const KParams& P, int tile, T* sBase,
                                              int32_t* sUp, int32_t* sDn, uint8_t* sN,
                                              uint64_t* bar, bool load_up, T* sInc = nullptr,
                                              bool defer_inc = false) {
  constexpr int NP = D * D, M = D * KP1, TB = NP * TILE;
  constexpr bool kInc = kIncScheme<T>;
  constexpr bool kLoadInc = kInc && (STAGE == 2 || STAGE == 4);
  if ((threadIdx.x & 31) == 0) {
    constexpr unsigned LB = M * TILE * 4u, NB = M * TILE;
    mbar_init(bar, 1);
    mbar_expect_tx(bar, (load_up ? 2 * LB : LB) + NB +
                            (STAGE >= 2 ? TB * (unsigned)sizeof(T) : 0u) +
                            (kLoadInc ? TB * (unsigned)sizeof(T) : 0u));
    const size_t gt = (size_t)tile * M * TILE;
    if (load_up) bulk_g2s(sUp, P.plus + gt, LB, bar);
    bulk_g2s(sDn, P.minus + gt, LB, bar);
    bulk_g2s(sN, P.nvec + gt, NB, bar);
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

// phase A: acc = base + c (damping + commutator) with the ADO in registers.
// sBase: the tile's base operand (flat, Hermitian tile layout).
template <class T, int D, int KP1, int STAGE, int R0 = 0, int R1 = D>
__device__ __forceinline__ void phase_a(const KParams& P, int tile, int lane, T c, T* sBase,
                                        const uint8_t (*sN)[TILE], uint64_t* bar,
                                        T (&acc)[D * D]) {
  constexpr int NP = D * D, M = D * KP1, DIAG = D * TILE, E = D * (D - 1) / 2;
  volatile Ctl* ctl = P.ctl;
  const T* yo = st_in<T>(P) + (size_t)tile * NP * TILE;
  T s[NP];
#pragma unroll
  for (int i = 0; i < D; ++i) s[i] = __ldg(yo + i * TILE + lane);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const v2_t<T> v = ldg2(yo + DIAG + e * 2 * TILE + 2 * lane);
    s[D + 2 * e] = v.x;
    s[D + 2 * e + 1] = v.y;
  }
  if (R0 == 0 && tile == 0 && lane == 0) {  // sink rates of this stage input (heom.py:282-283)
    int q = 0;
    for (int sk = 0; sk < P.n_sinks; ++sk) {
      double a = 0.0;
      for (int cc = 0; cc < P.sink_nterms[sk]; ++cc, ++q) {
        const double v = P.sink_rate[q] * (double)__ldg(st_in<T>(P) + P.sink_pos[q] * TILE);
        a = cc == 0 ? v : a + v;
      }
      ctl->r[P.rpar][STAGE - 1][sk] = a;
    }
  }
  mbar_wait(bar, 0);
  // damping sum_k nu_k sum_j n_jk (heom.py:275, generalised)
  int tk[KP1];
#pragma unroll
  for (int k = 0; k < KP1; ++k) tk[k] = 0;
#pragma unroll
  for (int m = 0; m < M; ++m) tk[m % KP1] += sN[m][lane];
  T damp = 0;
#pragma unroll
  for (int k = 0; k < KP1; ++k) damp = fma((T)tk[k], Opd<T>::nu(P, k), damp);
  constexpr T third = (T)(1.0 / 3.0);
  constexpr bool kInc = kIncScheme<T>;
#pragma unroll
  for (int i = R0; i < R1; ++i) {
    // diagonal: Re(-i[H,s])_ii = 2 sum_{l != i} h_il Im s_il
    T cm = 0;
#pragma unroll
    for (int l = 0; l < D; ++l)
      if (l != i) cm = fma(Opd<T>::h(P, i * MAXD + l), sim<T, D>(s, i, l), cm);
    const T fi = -(damp + Opd<T>::decay(P, i));
    // the RK base term (see the header): sigma / B from shared memory
    T* bs = sBase + i * TILE + lane;
    T bv;
    if constexpr (kInc) {
      if (STAGE == 1) *bs = s[i];
      bv = STAGE == 4 ? (s[i] - *bs) * third : (T)0;
    } else if constexpr (STAGE == 1) {
      bv = s[i];
    } else {
      const T b = *bs;
      if (STAGE == 2) *bs = (s[i] - b) * third;  // park (Y2 - s)/3 for B
      bv = STAGE == 4 ? fma(s[i], third, b) : b;
    }
    acc[i] = fma(c, fma(fi, s[i], (T)-2 * cm), bv);
#pragma unroll
    for (int j = i + 1; j < D; ++j) {
      const int pr = Pk<D>::re(i, j), pim = Pk<D>::im(i, j), e = Pk<D>::off(i, j);
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
      T* bp = sBase + DIAG + e * 2 * TILE + 2 * lane;
      T br, bi;
      if constexpr (kInc) {
        if (STAGE == 1) st2(bp, s[pr], s[pim]);
        if (STAGE == 4) {
          const v2_t<T> b = sm2<T>(bp);
          br = (s[pr] - b.x) * third;
          bi = (s[pim] - b.y) * third;
        } else {
          br = bi = (T)0;
        }
      } else if constexpr (STAGE == 1) {
        br = s[pr];
        bi = s[pim];
      } else {
        const v2_t<T> b = sm2<T>(bp);
        if (STAGE == 2) st2(bp, (s[pr] - b.x) * third, (s[pim] - b.y) * third);
        br = STAGE == 4 ? fma(s[pr], third, b.x) : b.x;
        bi = STAGE == 4 ? fma(s[pim], third, b.y) : b.y;
      }
      acc[pr] = fma(c, fma(f, s[pr], ci), br);   // -1j * [H,s]
      acc[pim] = fma(c, fma(f, s[pim], -cr), bi);
    }
  }
}

// phase B: the neighbour crosses (_kernels.py:41-57), every term one FMA into the
// register accumulator with the RK coefficient c folded into the link
// coefficients (c n b_k, c n a_k, c); absent links are predicated off.  Each
// off-diagonal element of a cross is one (re, im) pair load.
// no_up (warp-uniform): no lane of the tile has a raise link (the top tier) --
// the lower links of GROUP sites are gathered per round trip (the same loads as
// one full site), halving the dependent rounds of the tile.
template <class T, int D, int KP1, int GROUP = 2, int S0 = 0, int S1 = D>
__device__ __forceinline__ void phase_b_sites(const KParams& P, int lane, T c, bool no_up,
                                              const int32_t (*sUp)[TILE],
                                              const int32_t (*sDn)[TILE],
                                              const uint8_t (*sN)[TILE], T (&acc)[D * D]) {
  constexpr int TB = D * D * TILE, DIAG = D * TILE;
  const T* yin = st_in<T>(P);
  T cbk[KP1], cak[KP1];
#pragma unroll
  for (int k = 0; k < KP1; ++k) {
    cbk[k] = c * Opd<T>::b(P, k);
    cak[k] = c * Opd<T>::a(P, k);
  }
  auto ld = [](const T* q, bool v) -> T {
    T r = 0;
    if (v) r = __ldg(q);
    return r;
  };
  auto ld2 = [](const T* q, bool v) -> v2_t<T> {
    v2_t<T> r;
    r.x = 0;
    r.y = 0;
    if (v) r = ldg2(q);
    return r;
  };
  // link target t (position): its tile base and its lane
  auto tbase = [&](int t) -> const T* {
    HB_CHECK(t < 0 || t < P.n_tiles_total * TILE);
    return yin + (size_t)(t >> 5) * TB;
  };
  if (no_up) {
#pragma unroll
    for (int s0 = S0; s0 < S1; s0 += GROUP) {
#pragma unroll
      for (int st = s0; st < (s0 + GROUP < S1 ? s0 + GROUP : S1); ++st) {
#pragma unroll
        for (int k = 0; k < KP1; ++k) {
          const int m = st * KP1 + k;
          const int pd = sDn[m][lane];
          const bool vd = pd >= 0;
          const T* dn = tbase(pd);
          const int ld_ = pd & 31;
          const T n = vd ? (T)sN[m][lane] : (T)0;
          const T cb = n * cbk[k], ca = n * cak[k];
          acc[st] = fma((T)2 * cb, ld(dn + st * TILE + ld_, vd), acc[st]);
#pragma unroll
          for (int o = 0; o < D; ++o) {
            if (o == st) continue;
            const int pr = Pk<D>::re(st, o), pim = Pk<D>::im(st, o);
            const int e = Pk<D>::off(st < o ? st : o, st < o ? o : st);
            const v2_t<T> dv = ld2(dn + DIAG + e * 2 * TILE + 2 * ld_, vd);
            if (o > st) {
              acc[pr] = fma(cb, dv.x, fma(-ca, dv.y, acc[pr]));
              acc[pim] = fma(cb, dv.y, fma(ca, dv.x, acc[pim]));
            } else {
              acc[pr] = fma(cb, dv.x, fma(ca, dv.y, acc[pr]));
              acc[pim] = fma(cb, dv.y, fma(-ca, dv.x, acc[pim]));
            }
          }
        }
      }
    }
    return;
  }
#pragma unroll
  for (int st = S0; st < S1; ++st) {
#pragma unroll
    for (int k = 0; k < KP1; ++k) {
      const int m = st * KP1 + k;
      const int pu = sUp[m][lane], pd = sDn[m][lane];
      const bool vu = pu >= 0, vd = pd >= 0;
      const T* up = tbase(pu);
      const T* dn = tbase(pd);
      const int lu = pu & 31, ld_ = pd & 31;
      const T n = vd ? (T)sN[m][lane] : (T)0;
      const T cb = n * cbk[k], ca = n * cak[k];
      const T cu = vu ? c : (T)0;
      acc[st] = fma((T)2 * cb, ld(dn + st * TILE + ld_, vd), acc[st]);
#pragma unroll
      for (int o = 0; o < D; ++o) {
        if (o == st) continue;
        const int pr = Pk<D>::re(st, o), pim = Pk<D>::im(st, o);
        const int e = Pk<D>::off(st < o ? st : o, st < o ? o : st);
        const v2_t<T> uv = ld2(up + DIAG + e * 2 * TILE + 2 * lu, vu);
        const v2_t<T> dv = ld2(dn + DIAG + e * 2 * TILE + 2 * ld_, vd);
        if (o > st) {  // element (st, o): row st
          acc[pr] = fma(cb, dv.x, fma(-ca, dv.y, fma(-cu, uv.y, acc[pr])));
          acc[pim] = fma(cb, dv.y, fma(ca, dv.x, fma(cu, uv.x, acc[pim])));
        } else {       // element (o, st): column st
          acc[pr] = fma(cb, dv.x, fma(ca, dv.y, fma(cu, uv.y, acc[pr])));
          acc[pim] = fma(cb, dv.y, fma(-ca, dv.x, fma(-cu, uv.x, acc[pim])));
        }
      }
    }
  }
}

// phase C: store (stage 2 also B = (Y2 - s)/3 + 2/3 Y3; float: see the header);
// stage 4 also max|y|^2 over the lane's elements (diagonal planes are real).
// tb: element offset of the tile; sBase / sInc flat (Hermitian tile layout).
template <class T, int D, int STAGE>
__device__ __forceinline__ void phase_c_store(const KParams& P, int lane, size_t tb, T* sBase,
                                              T (&acc)[D * D], double& maxa2, T* sInc) {
  constexpr int DIAG = D * TILE, E = D * (D - 1) / 2;
  constexpr T third = (T)(1.0 / 3.0), two3 = (T)(2.0 / 3.0);
  T* out = st_out<T>(P) + tb;
  T* bo = st_b<T>(P) + tb;
  // one element: slot offset o (diagonal) -> value stored, B store as a side effect
  auto fin = [&](T a, int o) -> T {
    if (kIncScheme<T>) {
      const T sg = sBase[o];
      if (STAGE == 1) bo[o] = a * third;
      if (STAGE == 2) bo[o] = fma(two3, a, sInc[o]);
      return STAGE == 4 ? sg + (sInc[o] + a) : sg + a;
    }
    if (STAGE == 2) bo[o] = fma(two3, a, sBase[o]);
    return a;
  };
#pragma unroll
  for (int i = 0; i < D; ++i) {
    acc[i] = fin(acc[i], i * TILE + lane);
    out[i * TILE + lane] = acc[i];
  }
  // the upper triangle, element e = planes D + 2e (re), D + 2e + 1 (im)
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int pr = D + 2 * e, pim = pr + 1;
    const int o = DIAG + e * 2 * TILE + 2 * lane;
    if (kIncScheme<T>) {
      const v2_t<T> sg = sm2<T>(sBase + o);
      v2_t<T> in;
      in.x = 0;
      in.y = 0;
      if (STAGE == 2 || STAGE == 4) in = sm2<T>(sInc + o);
      if (STAGE == 1) st2(bo + o, acc[pr] * third, acc[pim] * third);
      if (STAGE == 2) st2(bo + o, fma(two3, acc[pr], in.x), fma(two3, acc[pim], in.y));
      acc[pr] = STAGE == 4 ? sg.x + (in.x + acc[pr]) : sg.x + acc[pr];
      acc[pim] = STAGE == 4 ? sg.y + (in.y + acc[pim]) : sg.y + acc[pim];
    } else if (STAGE == 2) {
      const v2_t<T> b = sm2<T>(sBase + o);
      st2(bo + o, fma(two3, acc[pr], b.x), fma(two3, acc[pim], b.y));
    }
    st2(out + o, acc[pr], acc[pim]);
  }
  if (STAGE == 4) {
#pragma unroll
    for (int i = 0; i < D; ++i) maxa2 = fmax(maxa2, (double)acc[i] * (double)acc[i]);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const double yr = acc[D + 2 * e], yi = acc[D + 2 * e + 1];
      maxa2 = fmax(maxa2, fma(yr, yr, yi * yi));
    }
  }
}

}  // namespace hb
