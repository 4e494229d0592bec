// Element-parallel stage kernel for small grids (k_el).  At config 3's K = 0
// twin (54 tiles on 148 SMs) a stage is latency bound, and a globaltimer
// timeline of k_mm4 (one warp per tile) shows where: ~0.9 us for the grid
// dependency to release, ~2.3 us for phase A -- one warp issuing the ~2,000
// FP64 instructions of the commutator alone on its SM -- ~1.7 us of gathers and
// ~0.4 us of stores per 5.2 us stage.  Here a tile gets a CTA of 4 warps and the
// 28 elements of the Hermitian-packed ADO (7 diagonal, 21 upper) are dealt to
// the warps, 7 each: every warp computes phase A (commutator, damping, RK base)
// and phase B (its elements' entries of the linked ADOs: all loads of one round
// issued together) for its own elements and stores them.  The own tile arrives
// by one bulk copy into shared memory right after the grid dependency; the link
// tables and the base tile before it (PDL), as in k_mm4.
//
// Per element the FMA sequence is k_mm4's (hb_mm_common.cuh phase_a /
// phase_b_sites: phase A, then the links of site i, then those of site j, modes
// in order), so the results are bit-identical to k_mm4.  FP64, Hermitian
// layout, every block level a site.
#include "hb_device.cuh"
#include "hb_mm_common.cuh"

namespace hb {

constexpr int kElWarps = 4;

// element q of the ADO: q < D the diagonal q, else upper-triangle e = q - D
template <int D>
struct ElIdx {
  __host__ __device__ static constexpr int i(int q) {
    if (q < D) return q;
    int e = q - D, r = 0;
    while (e >= D - 1 - r) {
      e -= D - 1 - r;
      ++r;
    }
    return r;
  }
  __host__ __device__ static constexpr int j(int q) {
    if (q < D) return q;
    int e = q - D, r = 0;
    while (e >= D - 1 - r) {
      e -= D - 1 - r;
      ++r;
    }
    return r + 1 + e;
  }
};

// warp W's elements q = W, W + NW, ...: phase A, phase B, store
template <int D, int KP1, int STAGE, int W, int NW>
__device__ __forceinline__ double el_warp(const KParams& P, int lane, int tile, double c, double damp,
                                          const double* sS, const double* sBase,
                                          const int32_t (*sUp)[TILE], const int32_t (*sDn)[TILE],
                                          const uint8_t (*sN)[TILE], bool has_up) {
  using T = double;
  constexpr int NP = D * D, TB = NP * TILE, DIAG = D * TILE, NQ = D + D * (D - 1) / 2;
  constexpr int NMY = W < NQ ? (NQ - 1 - W) / NW + 1 : 0;
  constexpr T third = (T)(1.0 / 3.0), two3 = (T)(2.0 / 3.0);
  auto S = [&](int p) -> T { return sS[herm_off(D, p, lane)]; };
  auto sre_ = [&](int i, int j) -> T { return S(Pk<D>::re(i, j)); };
  auto sim_ = [&](int i, int j) -> T {
    return i == j ? (T)0 : (i < j ? S(Pk<D>::im(i, j)) : -S(Pk<D>::im(i, j)));
  };
  auto base = [&](int p, T x) -> T {  // k_mm4 phase_a's base term (12-pass scheme)
    if (STAGE == 1) return x;
    const T b = sBase[herm_off(D, p, lane)];
    if (STAGE == 4) return fma(x, third, b);
    return b;
  };
  const T* yin = st_in<T>(P);
  T cbk[KP1], cak[KP1];
#pragma unroll
  for (int k = 0; k < KP1; ++k) {
    cbk[k] = c * P.b[k];
    cak[k] = c * P.a[k];
  }
  T re[NMY > 0 ? NMY : 1], im[NMY > 0 ? NMY : 1];
  // ---- gathers first (one round): the entries of the linked ADOs this warp needs
  T gdn[NMY > 0 ? NMY : 1][2][KP1][2], gup[NMY > 0 ? NMY : 1][2][KP1][2];
#pragma unroll
  for (int u = 0; u < NMY; ++u) {
    const int q = W + u * NW, i = ElIdx<D>::i(q), j = ElIdx<D>::j(q);
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int st = side == 0 ? i : j;
#pragma unroll
      for (int k = 0; k < KP1; ++k) {
        const int m = st * KP1 + k;
        const int pd = sDn[m][lane], pu = has_up ? sUp[m][lane] : -1;
        T dr = 0, di = 0, ur = 0, ui = 0;
        if (i == j) {
          if (side == 0 && pd >= 0) dr = __ldg(yin + (size_t)(pd >> 5) * TB + i * TILE + (pd & 31));
        } else {
          const int off = DIAG + Pk<D>::off(i, j) * 2 * TILE;
          if (pd >= 0) {
            const v2_t<T> v = ldg2(yin + (size_t)(pd >> 5) * TB + off + 2 * (pd & 31));
            dr = v.x;
            di = v.y;
          }
          if (pu >= 0) {
            const v2_t<T> v = ldg2(yin + (size_t)(pu >> 5) * TB + off + 2 * (pu & 31));
            ur = v.x;
            ui = v.y;
          }
        }
        gdn[u][side][k][0] = dr;
        gdn[u][side][k][1] = di;
        gup[u][side][k][0] = ur;
        gup[u][side][k][1] = ui;
      }
    }
  }
  // ---- phase A (k_mm4 phase_a, element by element)
#pragma unroll
  for (int u = 0; u < NMY; ++u) {
    const int q = W + u * NW, i = ElIdx<D>::i(q), j = ElIdx<D>::j(q);
    if (i == j) {
      T cm = 0;
#pragma unroll
      for (int l = 0; l < D; ++l)
        if (l != i) cm = fma(P.h[i * MAXD + l], sim_(i, l), cm);
      re[u] = fma(c, fma(-(damp + P.decay[i]), S(i), (T)-2 * cm), base(i, S(i)));
    } else {
      const int pr = Pk<D>::re(i, j), pim = Pk<D>::im(i, j);
      const T dh = P.h[i * MAXD + i] - P.h[j * MAXD + j], hij = P.h[i * MAXD + j];
      T cr = fma(hij, S(j), fma(-hij, S(i), dh * S(pr)));
      T ci = dh * S(pim);
#pragma unroll
      for (int l = 0; l < D; ++l) {
        if (l == i || l == j) continue;
        const T hil = P.h[i * MAXD + l], hlj = P.h[l * MAXD + j];
        cr = fma(hil, sre_(l, j), cr);
        cr = fma(-hlj, sre_(i, l), cr);
        ci = fma(hil, sim_(l, j), ci);
        ci = fma(-hlj, sim_(i, l), ci);
      }
      const T f = -(damp + (T)0.5 * (P.decay[i] + P.decay[j]));
      re[u] = fma(c, fma(f, S(pr), ci), base(pr, S(pr)));
      im[u] = fma(c, fma(f, S(pim), -cr), base(pim, S(pim)));
    }
  }
  // ---- phase B (k_mm4 phase_b_sites: site i, then site j, modes in order)
#pragma unroll
  for (int u = 0; u < NMY; ++u) {
    const int q = W + u * NW, i = ElIdx<D>::i(q), j = ElIdx<D>::j(q);
#pragma unroll
    for (int side = 0; side < (i == j ? 1 : 2); ++side) {
      const int st = side == 0 ? i : j;
#pragma unroll
      for (int k = 0; k < KP1; ++k) {
        const int m = st * KP1 + k;
        const bool vd = sDn[m][lane] >= 0, vu = has_up && sUp[m][lane] >= 0;
        const T n = vd ? (T)sN[m][lane] : (T)0;
        const T cb = n * cbk[k], ca = n * cak[k];
        const T cu = vu ? c : (T)0;
        const T dr = gdn[u][side][k][0], di = gdn[u][side][k][1];
        const T ur = gup[u][side][k][0], ui = gup[u][side][k][1];
        if (i == j) {
          re[u] = fma((T)2 * cb, dr, re[u]);
        } else if (side == 0) {  // element (st, o > st): row st
          re[u] = fma(cb, dr, fma(-ca, di, fma(-cu, ui, re[u])));
          im[u] = fma(cb, di, fma(ca, dr, fma(cu, ur, im[u])));
        } else {                 // element (o < st, st): column st
          re[u] = fma(cb, dr, fma(ca, di, fma(cu, ui, re[u])));
          im[u] = fma(cb, di, fma(-ca, dr, fma(-cu, ur, im[u])));
        }
      }
    }
  }
  // ---- phase C (k_mm4 phase_c_store, double): store, stage 2 also B
  T* out = st_out<T>(P) + (size_t)tile * TB;
  T* bo = st_b<T>(P) + (size_t)tile * TB;
  double m2 = 0.0;
#pragma unroll
  for (int u = 0; u < NMY; ++u) {
    const int q = W + u * NW, i = ElIdx<D>::i(q), j = ElIdx<D>::j(q);
    if (i == j) {
      const int o = i * TILE + lane;
      if (STAGE == 2) bo[o] = fma(two3, re[u], (S(i) - sBase[o]) * third);
      out[o] = re[u];
      if (STAGE == 4) m2 = fmax(m2, re[u] * re[u]);
    } else {
      const int e = Pk<D>::off(i, j), o = DIAG + e * 2 * TILE + 2 * lane;
      if (STAGE == 2) {
        const v2_t<T> b = sm2<T>(const_cast<T*>(sBase) + o);
        const v2_t<T> x = sm2<T>(const_cast<T*>(sS) + o);
        st2(bo + o, fma(two3, re[u], (x.x - b.x) * third), fma(two3, im[u], (x.y - b.y) * third));
      }
      st2(out + o, re[u], im[u]);
      if (STAGE == 4) m2 = fmax(m2, fma(re[u], re[u], im[u] * im[u]));
    }
  }
  return m2;
}

template <int D, int KP1, int STAGE>
__global__ void __launch_bounds__(32 * kElWarps, 1) k_el(const KParams P) {
  using T = double;
  constexpr int NP = D * D, M = D * KP1, TB = NP * TILE;
  __shared__ __align__(128) T sS[NP * TILE];                        // the own tile
  __shared__ __align__(128) T sBase[(STAGE >= 2 ? NP : 1) * TILE];  // sigma, or B at stage 4
  __shared__ __align__(16) int32_t sUp[M][TILE];
  __shared__ __align__(16) int32_t sDn[M][TILE];
  __shared__ __align__(16) uint8_t sN[M][TILE];
  __shared__ double sMax[kElWarps];
  __shared__ __align__(8) uint64_t bar[2];

  volatile Ctl* ctl = P.ctl;
  if (ctl->status != ST_RUNNING) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = P.tile_begin + blockIdx.x;
  HB_CHECK(tile >= 0 && tile < P.n_tiles_total);
  const double c = STAGE == 4 ? P.dt / 6.0 : P.coef;
  const bool top = tile >= P.top_tile;
  // link tables and the base tile before the grid dependency (nothing running
  // writes them), the stage input after it
  if (threadIdx.x == 0) {
    constexpr unsigned LB = M * TILE * 4u, NB = M * TILE;
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_expect_tx(&bar[0], (top ? LB : 2 * LB) + NB + (STAGE >= 2 ? TB * 8u : 0u));
    const size_t gt = (size_t)tile * M * TILE;
    if (!top) bulk_g2s(&sUp[0][0], P.plus + gt, LB, &bar[0]);
    bulk_g2s(&sDn[0][0], P.minus + gt, LB, &bar[0]);
    bulk_g2s(&sN[0][0], P.nvec + gt, NB, &bar[0]);
    if (STAGE >= 2)
      bulk_g2s(sBase, (STAGE == 4 ? st_b<T>(P) : st_sig<T>(P)) + (size_t)tile * TB, TB * 8u, &bar[0]);
  }
  __syncthreads();  // barriers initialised before any warp waits on them
  pdl_wait();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar[1], TB * 8u);
    bulk_g2s(sS, st_in<T>(P) + (size_t)tile * TB, TB * 8u, &bar[1]);
  }
  if (ctl->status != ST_RUNNING) {
    if (threadIdx.x == 0) {  // no bulk copy may land after the CTA has exited
      mbar_wait(&bar[0], 0);
      mbar_wait(&bar[1], 0);
    }
    __syncthreads();
    return;
  }
  pdl_release();
  const long long step_next = ctl->step + 1;
  mbar_wait(&bar[0], 0);
  // damping sum_k nu_k sum_j n_jk (heom.py:275, generalised)
  T damp = 0;
  {
    int tk[KP1];
#pragma unroll
    for (int k = 0; k < KP1; ++k) tk[k] = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) tk[m % KP1] += sN[m][lane];
#pragma unroll
    for (int k = 0; k < KP1; ++k) damp = fma((T)tk[k], P.nu[k], damp);
  }
  mbar_wait(&bar[1], 0);
  if (tile == 0 && threadIdx.x == 0) {  // sink rates of this stage input (heom.py:282-283)
    int q = 0;
    for (int sk = 0; sk < P.n_sinks; ++sk) {
      double a = 0.0;
      for (int cc = 0; cc < P.sink_nterms[sk]; ++cc, ++q) {
        const double v = P.sink_rate[q] * sS[P.sink_pos[q] * TILE];
        a = cc == 0 ? v : a + v;
      }
      ctl->r[STAGE - 1][sk] = a;
    }
  }
  double m2 = 0.0;
  switch (warp) {
    case 0: m2 = el_warp<D, KP1, STAGE, 0, kElWarps>(P, lane, tile, c, damp, sS, sBase, sUp, sDn, sN, !top); break;
    case 1: m2 = el_warp<D, KP1, STAGE, 1, kElWarps>(P, lane, tile, c, damp, sS, sBase, sUp, sDn, sN, !top); break;
    case 2: m2 = el_warp<D, KP1, STAGE, 2, kElWarps>(P, lane, tile, c, damp, sS, sBase, sUp, sDn, sN, !top); break;
    case 3: m2 = el_warp<D, KP1, STAGE, 3, kElWarps>(P, lane, tile, c, damp, sS, sBase, sUp, sDn, sN, !top); break;
  }
  if (STAGE == 4 && step_next % 25 == 0) {  // whole-state guard (heom.py:386-389)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m2 = fmax(m2, __shfl_xor_sync(0xffffffffu, m2, o));
    if (lane == 0) sMax[warp] = m2;
    __syncthreads();
    if (threadIdx.x == 0) {
      double mx = sMax[0];
#pragma unroll
      for (int w = 1; w < kElWarps; ++w) mx = fmax(mx, sMax[w]);
      atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                (unsigned long long)__double_as_longlong(mx));
    }
  }
}

template <int D, int KP1, int STAGE>
static cudaError_t el_go(const KParams& p, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.n_tiles);
  cfg.blockDim = dim3(32 * kElWarps);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_el<D, KP1, STAGE>, p);
}

template <int D, int KP1>
static cudaError_t el_stage(int stage, const KParams& p, cudaStream_t s) {
  switch (stage) {
    case 1: return el_go<D, KP1, 1>(p, s);
    case 2: return el_go<D, KP1, 2>(p, s);
    case 3: return el_go<D, KP1, 3>(p, s);
    case 4: return el_go<D, KP1, 4>(p, s);
  }
  return cudaErrorInvalidValue;
}

template <int D>
static cudaError_t el_kp1(int stage, const KParams& p, cudaStream_t s) {
  return p.kp1 == 1 ? el_stage<D, 1>(stage, p, s) : el_stage<D, 2>(stage, p, s);
}

// the stage kernel alone (the caller launches the step bookkeeping after stage 4)
cudaError_t launch_el(int stage, const KParams& p, cudaStream_t s) {
  switch (p.d) {
    case 1: return el_kp1<1>(stage, p, s);
    case 2: return el_kp1<2>(stage, p, s);
    case 3: return el_kp1<3>(stage, p, s);
    case 4: return el_kp1<4>(stage, p, s);
    case 5: return el_kp1<5>(stage, p, s);
    case 6: return el_kp1<6>(stage, p, s);
    case 7: return el_kp1<7>(stage, p, s);
    case 8: return el_kp1<8>(stage, p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hb
