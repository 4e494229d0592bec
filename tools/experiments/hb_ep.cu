// Element-parallel stage kernel k_ep (double): one tile of 32 ADOs per CTA of
// NW = 4 warps; lane = ADO as in k_mm4, but the d(d+1)/2 elements of the
// Hermitian ADO are dealt to the warps, so a tile's FP64 work and its link
// gathers run on the four SM sub-partitions at once instead of one.
//
// The same code runs in every warp: a warp's elements are runtime (i, j) pairs,
// the tile's stage input sits in shared memory (one bulk copy after the grid
// dependency) and is read with runtime offsets, H and the decay rates are staged
// in shared memory too.  Every element is evaluated with exactly the FMA sequence
// of k_mm4 (hb_mm_common.cuh: phase_a, phase_b_sites, phase_c_store), so the two
// kernels are bitwise interchangeable -- a sharded run (k_mm4 over tile lists)
// and an unsharded one agree to the bit whichever kernel each uses.
//
// Each warp owns only its elements' accumulators (a few registers), so all of a
// warp's link gathers are issued as one round instead of the 4-7 dependent
// rounds of k_mm4, and 4 warps x up to 7 tiles share an SM.
// RHS: _kernels.py:23-58 (generalised to K+1 modes per site); RK folding as k_mm4.
#include "hb_device.cuh"
#include "hb_mm_common.cuh"

namespace hb {

namespace {

constexpr int NW = 4;  // warps per tile

template <int D>
__device__ __forceinline__ int hoff(int a, int b) {  // a < b: packed pair index
  return a * (2 * D - a - 1) / 2 + (b - a - 1);
}

// the a-th upper-triangle element (row-major over i < j)
template <int D>
__device__ __forceinline__ void pair_of(int e, int& i, int& j) {
  int r = 0;
#pragma unroll
  for (int q = 0; q < D - 1; ++q) {
    if (e >= D - 1 - r) {
      e -= D - 1 - r;
      ++r;
    }
  }
  i = r;
  j = r + 1 + e;
}

}  // namespace

template <int D, int KP1, int STAGE>
__global__ void __launch_bounds__(NW * 32) k_ep(const KParams P) {
  using T = double;
  constexpr int NP = D * D, M = D * KP1, DIAG = D * TILE, TB = NP * TILE;
  constexpr int NO = D * (D - 1) / 2;           // off-diagonal elements
  constexpr int QO = (NO + NW - 1) / NW;        // per warp
  constexpr int QD = (D + NW - 1) / NW;         // diagonal elements per warp
  constexpr T third = 1.0 / 3.0, two3 = 2.0 / 3.0;
  __shared__ __align__(128) T sS[TB];
  __shared__ __align__(128) T sBase[(STAGE >= 2 ? NP : 1) * TILE];
  __shared__ __align__(16) int32_t sUp[M][TILE];
  __shared__ __align__(16) int32_t sDn[M][TILE];
  __shared__ __align__(16) uint8_t sN[M][TILE];
  __shared__ T sH[NP];
  __shared__ T sDec[D];
  __shared__ __align__(8) uint64_t bar[2];

  volatile Ctl* ctl = P.ctl;
  if (ctl->status != ST_RUNNING) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = P.tile_list ? P.tile_list[blockIdx.x] : P.tile_begin + blockIdx.x;
  HB_CHECK(tile >= 0 && tile < P.n_tiles_total);
  const size_t tb = (size_t)tile * TB;
  const T c = STAGE == 4 ? P.dt / 6.0 : P.coef;
  const bool top = tile >= P.top_tile;

  if (tid == 0) {  // operands no running kernel writes, before the grid dependency
    constexpr unsigned LB = M * TILE * 4u, NB = M * TILE;
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_expect_tx(&bar[0], (top ? LB : 2 * LB) + NB + (STAGE >= 2 ? TB * 8u : 0u));
    const size_t gt = (size_t)tile * M * TILE;
    if (!top) bulk_g2s(&sUp[0][0], P.plus + gt, LB, &bar[0]);
    bulk_g2s(&sDn[0][0], P.minus + gt, LB, &bar[0]);
    bulk_g2s(&sN[0][0], P.nvec + gt, NB, &bar[0]);
    if (STAGE >= 2) bulk_g2s(sBase, (STAGE == 4 ? P.Bbuf : P.sig) + tb, TB * 8u, &bar[0]);
  }
  if (warp == 1) {
#pragma unroll
    for (int q = 0; q < (NP + 31) / 32; ++q) {
      const int e = q * 32 + lane;
      if (e < NP) sH[e] = P.h[(e / D) * MAXD + e % D];
    }
    if (lane < D) sDec[lane] = P.decay[lane];
  }
  __syncthreads();  // barriers initialised, H staged
  pdl_wait();
  if (ctl->status != ST_RUNNING) {
    mbar_wait(&bar[0], 0);  // no bulk copy may land after the CTA has exited
    return;
  }
  if (tid == 0) {  // the stage input tile, written by the previous kernel
    mbar_expect_tx(&bar[1], TB * 8u);
    bulk_g2s(sS, P.Yin + tb, TB * 8u, &bar[1]);
  }
  pdl_release();
  const long long step_next = ctl->step + 1;
  if (tile == 0 && tid == 0) {  // sink rates of this stage input (heom.py:282-283)
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
  mbar_wait(&bar[0], 0);

  // damping sum_k nu_k sum_j n_jk (heom.py:275, generalised)
  int tk[KP1];
#pragma unroll
  for (int k = 0; k < KP1; ++k) tk[k] = 0;
#pragma unroll
  for (int m = 0; m < M; ++m) tk[m % KP1] += sN[m][lane];
  T damp = 0;
#pragma unroll
  for (int k = 0; k < KP1; ++k) damp = fma((T)tk[k], P.nu[k], damp);
  T cbk[KP1], cak[KP1];
#pragma unroll
  for (int k = 0; k < KP1; ++k) {
    cbk[k] = c * P.b[k];
    cak[k] = c * P.a[k];
  }
  bool no_up = top;
  if (!top) {
    bool up_any = false;
#pragma unroll
    for (int m = 0; m < M; ++m) up_any |= sUp[m][lane] >= 0;
    no_up = !__syncthreads_or(up_any);
  }

  // ---- the link gathers of this warp's elements, issued before the stage input
  // lands (they read other tiles of the same stage input: complete after pdl_wait)
  const T* yin = P.Yin;
  auto nbr = [&](int p) -> const T* {
    HB_CHECK(p < 0 || p < P.n_tiles_total * TILE);
    return yin + (size_t)(p >> 5) * TB + (p & 31);
  };
  using V2 = double2;
  auto ld2z = [](const T* q, bool v) -> V2 {
    V2 r;
    r.x = 0;
    r.y = 0;
    if (v) r = __ldg(reinterpret_cast<const V2*>(q));
    return r;
  };
  // off-diagonal elements: gathered pairs [q][site i/j][k][dn/up]
  int oi[QO], oj[QO];
  V2 gd[QO][2][KP1], gu[QO][2][KP1];
#pragma unroll
  for (int q = 0; q < QO; ++q) {
    const int e = warp + NW * q;
    int i = 0, j = 1;
    if (e < NO) pair_of<D>(e, i, j);
    oi[q] = i;
    oj[q] = j;
    const int po = DIAG + hoff<D>(i, j) * 2 * TILE;
#pragma unroll
    for (int sd = 0; sd < 2; ++sd) {
      const int st = sd == 0 ? i : j;
#pragma unroll
      for (int k = 0; k < KP1; ++k) {
        const int m = st * KP1 + k;
        const int pd = sDn[m][lane];
        gd[q][sd][k] = ld2z(nbr(pd) + po + (pd & 31), e < NO && pd >= 0);
        if (!no_up) {
          const int pu = sUp[m][lane];
          gu[q][sd][k] = ld2z(nbr(pu) + po + (pu & 31), e < NO && pu >= 0);
        }
      }
    }
  }
  T gdd[QD][KP1];
#pragma unroll
  for (int q = 0; q < QD; ++q) {
    const int i = warp + NW * q;
#pragma unroll
    for (int k = 0; k < KP1; ++k) {
      const int pd = i < D ? sDn[i * KP1 + k][lane] : -1;
      gdd[q][k] = 0;
      if (pd >= 0) gdd[q][k] = __ldg(nbr(pd) + i * TILE);
    }
  }

  mbar_wait(&bar[1], 0);
  const T* S = sS;
  auto pr = [&](int a, int b) -> V2 {  // a < b
    return *reinterpret_cast<const V2*>(S + DIAG + hoff<D>(a, b) * 2 * TILE + 2 * lane);
  };

  double maxa2 = 0.0;
  T* out = P.Yout + tb;
  T* bo = P.Bbuf + tb;
  // ---- off-diagonal elements: phase A (k_mm4 phase_a), B (phase_b_sites), C
#pragma unroll
  for (int q = 0; q < QO; ++q) {
    const int e = warp + NW * q;
    if (e >= NO) break;
    const int i = oi[q], j = oj[q];
    const int po = DIAG + hoff<D>(i, j) * 2 * TILE + 2 * lane;
    const V2 sij = *reinterpret_cast<const V2*>(S + po);
    const T sii = S[i * TILE + lane], sjj = S[j * TILE + lane];
    const T dh = sH[i * D + i] - sH[j * D + j];
    const T hij = sH[i * D + j];
    T cr = fma(hij, sjj, fma(-hij, sii, dh * sij.x));
    T ci = dh * sij.y;
#pragma unroll
    for (int l = 0; l < D; ++l) {
      if (l == i || l == j) continue;
      const T hil = sH[i * D + l], hlj = sH[l * D + j];
      const V2 plj = l < j ? pr(l, j) : pr(j, l);
      const V2 pil = i < l ? pr(i, l) : pr(l, i);
      const T imlj = l < j ? plj.y : -plj.y;
      const T imil = i < l ? pil.y : -pil.y;
      cr = fma(hil, plj.x, cr);
      cr = fma(-hlj, pil.x, cr);
      ci = fma(hil, imlj, ci);
      ci = fma(-hlj, imil, ci);
    }
    const T f = -(damp + (T)0.5 * (sDec[i] + sDec[j]));
    T* bp = sBase + po;
    T br, bi;
    if (STAGE == 1) {
      br = sij.x;
      bi = sij.y;
    } else {
      const V2 b = *reinterpret_cast<const V2*>(bp);
      if (STAGE == 2) {
        V2 pk;
        pk.x = (sij.x - b.x) * third;
        pk.y = (sij.y - b.y) * third;
        *reinterpret_cast<V2*>(bp) = pk;  // park (Y2 - s)/3 for B
      }
      br = STAGE == 4 ? fma(sij.x, third, b.x) : b.x;
      bi = STAGE == 4 ? fma(sij.y, third, b.y) : b.y;
    }
    T re = fma(c, fma(f, sij.x, ci), br);
    T im = fma(c, fma(f, sij.y, -cr), bi);
    // link crosses: site i (element (st, o), o > st), then site j ((o, st), o < st)
#pragma unroll
    for (int sd = 0; sd < 2; ++sd) {
      const int st = sd == 0 ? i : j;
#pragma unroll
      for (int k = 0; k < KP1; ++k) {
        const int m = st * KP1 + k;
        const bool vd = sDn[m][lane] >= 0;
        const T n = vd ? (T)sN[m][lane] : (T)0;
        const T cb = n * cbk[k], ca = n * cak[k];
        const V2 dv = gd[q][sd][k];
        if (no_up) {
          if (sd == 0) {
            re = fma(cb, dv.x, fma(-ca, dv.y, re));
            im = fma(cb, dv.y, fma(ca, dv.x, im));
          } else {
            re = fma(cb, dv.x, fma(ca, dv.y, re));
            im = fma(cb, dv.y, fma(-ca, dv.x, im));
          }
        } else {
          const T cu = sUp[m][lane] >= 0 ? c : (T)0;
          const V2 uv = gu[q][sd][k];
          if (sd == 0) {
            re = fma(cb, dv.x, fma(-ca, dv.y, fma(-cu, uv.y, re)));
            im = fma(cb, dv.y, fma(ca, dv.x, fma(cu, uv.x, im)));
          } else {
            re = fma(cb, dv.x, fma(ca, dv.y, fma(cu, uv.y, re)));
            im = fma(cb, dv.y, fma(-ca, dv.x, fma(-cu, uv.x, im)));
          }
        }
      }
    }
    if (STAGE == 2) {
      const V2 b = *reinterpret_cast<const V2*>(bp);
      st2(bo + po, fma(two3, re, b.x), fma(two3, im, b.y));
    }
    st2(out + po, re, im);
    if (STAGE == 4) maxa2 = fmax(maxa2, fma(re, re, im * im));
  }
  // ---- diagonal elements
#pragma unroll
  for (int q = 0; q < QD; ++q) {
    const int i = warp + NW * q;
    if (i >= D) break;
    T cm = 0;
#pragma unroll
    for (int l = 0; l < D; ++l) {
      if (l == i) continue;
      const V2 p = i < l ? pr(i, l) : pr(l, i);
      cm = fma(sH[i * D + l], i < l ? p.y : -p.y, cm);
    }
    const T fi = -(damp + sDec[i]);
    const int o = i * TILE + lane;
    const T si = S[o];
    T bv;
    if (STAGE == 1) {
      bv = si;
    } else {
      const T b = sBase[o];
      if (STAGE == 2) sBase[o] = (si - b) * third;
      bv = STAGE == 4 ? fma(si, third, b) : b;
    }
    T a = fma(c, fma(fi, si, (T)-2 * cm), bv);
#pragma unroll
    for (int k = 0; k < KP1; ++k) {
      const int m = i * KP1 + k;
      const bool vd = sDn[m][lane] >= 0;
      const T n = vd ? (T)sN[m][lane] : (T)0;
      const T cb = n * cbk[k];
      a = fma((T)2 * cb, gdd[q][k], a);
    }
    if (STAGE == 2) bo[o] = fma(two3, a, sBase[o]);
    out[o] = a;
    if (STAGE == 4) maxa2 = fmax(maxa2, (double)a * (double)a);
  }
  if (STAGE == 4 && step_next % 25 == 0) {  // whole-state guard (heom.py:386-389)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
    if (lane == 0)
      atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                (unsigned long long)__double_as_longlong(maxa2));
  }
}

template <int D, int KP1, int STAGE>
static cudaError_t ep_go(const KParams& p, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.n_tiles);
  cfg.blockDim = dim3(NW * 32);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  int n = 1;
  if (p.apw_tiles > 0) {
    const size_t tb = (size_t)D * D * TILE * sizeof(double);
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
  return cudaLaunchKernelEx(&cfg, k_ep<D, KP1, STAGE>, p);
}

template <int D, int KP1>
static cudaError_t ep_stage(int stage, const KParams& p, cudaStream_t s) {
  switch (stage) {
    case 1: return ep_go<D, KP1, 1>(p, s);
    case 2: return ep_go<D, KP1, 2>(p, s);
    case 3: return ep_go<D, KP1, 3>(p, s);
    case 4: return ep_go<D, KP1, 4>(p, s);
  }
  return cudaErrorInvalidValue;
}

bool ep_supported(int d, int kp1) { return d == 7 && kp1 >= 1 && kp1 <= 2; }

// one stage of the element-parallel kernel (double, d = 7); stage 4 is followed
// by the caller's step bookkeeping launch
cudaError_t launch_ep(int stage, const KParams& p, cudaStream_t s) {
  if (p.single || p.d != 7) return cudaErrorInvalidValue;
  return p.kp1 == 1 ? ep_stage<7, 1>(stage, p, s) : ep_stage<7, 2>(stage, p, s);
}

}  // namespace hb
