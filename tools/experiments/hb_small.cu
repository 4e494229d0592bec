// Persistent kernel for small hierarchies (at most one tile per SM): one launch
// runs many RK4 steps, the four stages separated by grid-wide barriers, the
// per-step bookkeeping (sinks heom.py:382-383, guard heom.py:386-389, records,
// stop policy heom.py:359-368) done by the CTA that arrives last at the barrier
// after stage 4.  At these sizes (config 3's K = 0 twin: 1,716 ADOs = 54 tiles,
// config 2: 11 tiles) a stage is the latency of one tile's chain of dependent
// memory round trips plus a kernel boundary, not bandwidth; so
//   * a tile gets one CTA of D warps instead of one warp: warp w gathers the
//     crosses of site w (all 2(K+1) links in ONE round trip) and owns a share of
//     the elements for the commutator and the store;
//   * the link tables, n and the damping are loaded once per launch;
//   * no kernel boundary between stages, only a grid barrier.
// Same arithmetic as k_mm4 / the reference RHS (_kernels.py:23-58, K+1 modes
// per site), summed in a different order (within 1e-15 of k_mm4).  Hermitian
// tile layout (herm_off), FP64 only, every block level a site.
#include "hb_device.cuh"
#include "hb_mm_common.cuh"

namespace hb {

namespace {

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Grid barrier over all CTAs (co-resident: cooperative launch).  bar[0] counts
// arrivals, bar[1] is the generation.  With `book`, the last CTA to arrive runs
// the step bookkeeping (one warp) before it releases the others.
template <int D>
__device__ __forceinline__ void grid_barrier(unsigned* bar, const KParams& P, bool book,
                                             long long step_next) {
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned gen = 0;
    int last = 0;
    if (threadIdx.x == 0) {
      gen = ld_acquire(bar + 1);
      __threadfence();
      last = atomicAdd(bar, 1u) == gridDim.x - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      if (threadIdx.x == 0) bar[0] = 0;
      __threadfence();
      if (book) finish_step_warp<D, true>(P, step_next);
      __syncwarp();
      if (threadIdx.x == 0) {
        __threadfence();
        st_release(bar + 1, gen + 1);
      }
    } else if (threadIdx.x == 0) {
      while (ld_acquire(bar + 1) == gen) __nanosleep(32);
    }
  }
  __syncthreads();
}

}  // namespace

// Element ownership: warp W owns diagonal W and the upper-triangle elements
// e = W, W + D, W + 2D, ... (row-major over i < j); its phase-A and store code
// is instantiated per W so that every index is a compile-time constant.
template <int D>
struct Upper {  // upper element e -> (i, j)
  __host__ __device__ static constexpr int i(int e) {
    int r = 0;
    while (e >= D - 1 - r) {
      e -= D - 1 - r;
      ++r;
    }
    return r;
  }
  __host__ __device__ static constexpr int j(int e) {
    int r = 0;
    while (e >= D - 1 - r) {
      e -= D - 1 - r;
      ++r;
    }
    return r + 1 + e;
  }
};

// phase A of warp W: -(damping) s - i[H, s] of its elements -> sAcc
template <int D, int W>
__device__ __forceinline__ void small_phase_a(const KParams& P, const double* sS, double* sAcc,
                                              int lane, double damp) {
  using T = double;
  constexpr int E = D * (D - 1) / 2;
  auto S = [&](int p) -> T { return sS[herm_off(D, p, lane)]; };
  auto sre_ = [&](int i, int j) -> T { return S(Pk<D>::re(i, j)); };
  auto sim_ = [&](int i, int j) -> T {
    return i == j ? (T)0 : (i < j ? S(Pk<D>::im(i, j)) : -S(Pk<D>::im(i, j)));
  };
  if (W < D) {
    constexpr int i = W;
    T cm = 0;
#pragma unroll
    for (int l = 0; l < D; ++l)
      if (l != i) cm = fma(P.h[i * MAXD + l], sim_(i, l), cm);
    sAcc[i * TILE + lane] = fma(-(damp + P.decay[i]), S(i), (T)-2 * cm);
  }
#pragma unroll
  for (int e = W; e < E; e += D) {
    const int i = Upper<D>::i(e), j = Upper<D>::j(e);
    const int pr = D + 2 * e, pim = pr + 1;
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
    sAcc[herm_off(D, pr, lane)] = fma(f, S(pr), ci);   // -1j * [H,s]
    sAcc[herm_off(D, pim, lane)] = fma(f, S(pim), -cr);
  }
}

// the RK stage combination of warp W's elements (the 12-pass scheme of
// hb_mm_common.cuh: Y2 = s + h/2 f, Y3 = sigma + h/2 f, B = (Y2 - sigma)/3 +
// 2/3 Y3, Y4 = sigma + h f, sigma = B + Y4/3 + h/6 f); returns max|y|^2.
// The base operands (sigma or B) of all owned elements are loaded before the
// first store: the stores may alias them as far as the compiler knows, and a
// load after each store would serialise one L2 round trip per element.
template <int D, int W>
__device__ __forceinline__ double small_store(const double* sS, const double* sAcc,
                                              double* const* bufs, double* yout, size_t tb,
                                              int lane, int stage, double c) {
  using T = double;
  constexpr int E = D * (D - 1) / 2;
  constexpr int NE = (W < E ? (E - 1 - W) / D + 1 : 0);  // owned upper elements
  constexpr int NV = 1 + 2 * NE;                         // owned planes
  int off[NV];
  off[0] = herm_off(D, W, lane);
#pragma unroll
  for (int u = 0; u < NE; ++u) {
    off[1 + 2 * u] = herm_off(D, D + 2 * (W + u * D), lane);
    off[2 + 2 * u] = off[1 + 2 * u] + 1;
  }
  T base[NV];
  if (stage >= 2) {
    const T* bsrc = (stage == 4 ? bufs[4] : bufs[0]) + tb;
#pragma unroll
    for (int v = 0; v < NV; ++v) base[v] = __ldcg(bsrc + off[v]);
  }
  T y[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const T f = sAcc[off[v]], x = sS[off[v]];
    if (stage == 1) {
      y[v] = fma(c, f, x);
    } else if (stage == 4) {
      y[v] = fma(c, f, fma(x, (T)(1.0 / 3.0), base[v]));
    } else {
      y[v] = fma(c, f, base[v]);
      if (stage == 2) bufs[4][tb + off[v]] = fma((T)(2.0 / 3.0), y[v], (x - base[v]) * (T)(1.0 / 3.0));
    }
    yout[tb + off[v]] = y[v];
  }
  double m2 = y[0] * y[0];
#pragma unroll
  for (int u = 0; u < NE; ++u) m2 = fmax(m2, fma(y[1 + 2 * u], y[1 + 2 * u], y[2 + 2 * u] * y[2 + 2 * u]));
  return m2;
}

#define HB_SMALL_WARPS(X) \
  switch (w) {            \
    case 0: X(0); break;  \
    case 1: X(1); break;  \
    case 2: X(2); break;  \
    case 3: X(3); break;  \
    case 4: X(4); break;  \
    case 5: X(5); break;  \
    case 6: X(6); break;  \
    case 7: X(7); break;  \
  }

template <int D, int KP1>
__global__ void __launch_bounds__(D * 32, 1) k_small(const KParams P, unsigned* bar,
                                                     long long max_steps) {
  using T = double;
  constexpr int NP = D * D, TB = NP * TILE, DIAG = D * TILE;
  __shared__ __align__(16) T sS[TB];    // the tile's stage input
  __shared__ __align__(16) T sAcc[TB];  // the tile's right-hand side
  __shared__ double sMax[D];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const size_t tb = (size_t)tile * TB;
  volatile Ctl* ctl = P.ctl;
  double* const bufs[5] = {const_cast<T*>(P.sig), const_cast<T*>(P.Y2), const_cast<T*>(P.Y3),
                           const_cast<T*>(P.Yin), P.Bbuf};  // sigma, Y2, Y3, Y4, B (stage-4 params)
  const double dt = P.dt;

  // ---- once per launch: this lane's links through site w, n, damping, and the
  // tile offsets of the cross elements (w, o) / (o, w)
  int up[KP1], dn[KP1];
  T nn[KP1];
#pragma unroll
  for (int k = 0; k < KP1; ++k) {
    const int m = w * KP1 + k;
    const size_t g = (size_t)tile * P.modes * TILE + (size_t)m * TILE + lane;
    up[k] = __ldcg(P.plus + g);
    dn[k] = __ldcg(P.minus + g);
    nn[k] = (T)__ldcg(P.nvec + g);
  }
  T damp = 0;
  {
    int tk[KP1];
#pragma unroll
    for (int k = 0; k < KP1; ++k) tk[k] = 0;
    for (int m = 0; m < D * KP1; ++m)
      tk[m % KP1] += __ldcg(P.nvec + (size_t)tile * P.modes * TILE + (size_t)m * TILE + lane);
#pragma unroll
    for (int k = 0; k < KP1; ++k) damp = fma((T)tk[k], P.nu[k], damp);
  }
  int xo[D];  // pair offset (elements) of cross element o inside a tile, lane 0
#pragma unroll
  for (int o = 0; o < D; ++o) {
    const int a = w < o ? w : o, b = w < o ? o : w;
    int e = 0;
    for (int r = 0; r < a; ++r) e += D - 1 - r;
    xo[o] = DIAG + (e + b - a - 1) * 2 * TILE;
  }

  for (long long it = 0; it < max_steps; ++it) {
    if (ctl->status != ST_RUNNING) break;  // set by the bookkeeping behind a barrier
    const long long step_next = ctl->step + 1;
#pragma unroll 1
    for (int stage = 1; stage <= 4; ++stage) {
      const T* yin = bufs[stage - 1];           // sigma, Y2, Y3, Y4
      T* yout = bufs[stage % 4];                // Y2, Y3, Y4, sigma
      // -- the site-w crosses of the 2(K+1) links (one round trip) and the own
      // tile into shared memory
      T gd[KP1], gr[2 * KP1][D], gi[2 * KP1][D];
#pragma unroll
      for (int l = 0; l < 2 * KP1; ++l) {
        const int t = l < KP1 ? dn[l] : up[l - KP1];
        const bool v = t >= 0;
        const T* base = yin + (size_t)(t >> 5) * TB + 2 * (t & 31);
        if (l < KP1) gd[l] = v ? __ldcg(yin + (size_t)(t >> 5) * TB + w * TILE + (t & 31)) : (T)0;
#pragma unroll
        for (int o = 0; o < D; ++o) {
          double2 x = make_double2(0.0, 0.0);
          if (v && o != w) x = __ldcg(reinterpret_cast<const double2*>(base + xo[o]));
          gr[l][o] = x.x;
          gi[l][o] = x.y;
        }
      }
      for (int i = threadIdx.x; i < TB / 2; i += D * 32)
        reinterpret_cast<double2*>(sS)[i] = __ldcg(reinterpret_cast<const double2*>(yin + tb) + i);
      if (tile == 0 && threadIdx.x == 0) {  // sink rates of this stage input (heom.py:282-283)
        int q = 0;
        for (int sk = 0; sk < P.n_sinks; ++sk) {
          double a = 0.0;
          for (int cc = 0; cc < P.sink_nterms[sk]; ++cc, ++q) {
            const double v = P.sink_rate[q] * __ldcg(yin + P.sink_pos[q] * TILE);
            a = cc == 0 ? v : a + v;
          }
          ctl->r[stage - 1][sk] = a;
        }
      }
      __syncthreads();
#define HB_PA(W) small_phase_a<D, (W < D ? W : 0)>(P, sS, sAcc, lane, damp)
      HB_SMALL_WARPS(HB_PA)
#undef HB_PA
      // -- phase B: site w's links; the row part (elements (w, o > w) and the
      // diagonal), then, after a barrier, the column part (elements (o < w, w))
      T rd = 0, rr[D], ri[D];
#pragma unroll
      for (int o = 0; o < D; ++o) rr[o] = ri[o] = 0;
#pragma unroll
      for (int k = 0; k < KP1; ++k) {
        const T n = dn[k] >= 0 ? nn[k] : (T)0;
        const T cb = n * P.b[k], ca = n * P.a[k];
        const T cu = up[k] >= 0 ? (T)1 : (T)0;
        rd = fma((T)2 * cb, gd[k], rd);
#pragma unroll
        for (int o = 0; o < D; ++o) {
          const T dr = gr[k][o], di = gi[k][o], ur = gr[KP1 + k][o], ui = gi[KP1 + k][o];
          if (o > w) {
            rr[o] = fma(cb, dr, fma(-ca, di, fma(-cu, ui, rr[o])));
            ri[o] = fma(cb, di, fma(ca, dr, fma(cu, ur, ri[o])));
          } else {
            rr[o] = fma(cb, dr, fma(ca, di, fma(cu, ui, rr[o])));
            ri[o] = fma(cb, di, fma(-ca, dr, fma(-cu, ur, ri[o])));
          }
        }
      }
      __syncthreads();
      sAcc[w * TILE + lane] += rd;
#pragma unroll
      for (int o = 0; o < D; ++o)
        if (o > w) {
          sAcc[xo[o] + 2 * lane] += rr[o];
          sAcc[xo[o] + 2 * lane + 1] += ri[o];
        }
      __syncthreads();
#pragma unroll
      for (int o = 0; o < D; ++o)
        if (o < w) {
          sAcc[xo[o] + 2 * lane] += rr[o];
          sAcc[xo[o] + 2 * lane + 1] += ri[o];
        }
      __syncthreads();
      // -- store the owned elements
      const T c = stage == 4 ? dt / 6.0 : (stage == 3 ? dt : 0.5 * dt);
      double maxa2 = 0.0;
#define HB_ST(W) maxa2 = small_store<D, (W < D ? W : 0)>(sS, sAcc, bufs, yout, tb, lane, stage, c)
      HB_SMALL_WARPS(HB_ST)
#undef HB_ST
      if (stage == 4 && step_next % 25 == 0) {  // whole-state guard (heom.py:386-389)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
        if (lane == 0) sMax[w] = maxa2;
        __syncthreads();
        if (threadIdx.x == 0) {
          double m = sMax[0];
          for (int q = 1; q < D; ++q) m = fmax(m, sMax[q]);
          atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                    (unsigned long long)__double_as_longlong(m));
        }
      }
      grid_barrier<D>(bar, P, stage == 4, step_next);
    }
  }
}

bool small_supported(int d, int kp1) { return d >= 1 && d <= 8 && kp1 >= 1 && kp1 <= 2; }

template <int D, int KP1>
static cudaError_t small_go(const KParams& p, unsigned* bar, long long steps, cudaStream_t s,
                            int* max_ctas) {
  if (max_ctas) {
    int per_sm = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const cudaError_t e =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_small<D, KP1>, D * 32, 0);
    *max_ctas = e == cudaSuccess ? per_sm * sms : 0;
    return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.n_tiles);
  cfg.blockDim = dim3(D * 32);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_small<D, KP1>, p, bar, steps);
}

template <int D>
static cudaError_t small_kp1(const KParams& p, unsigned* bar, long long steps, cudaStream_t s,
                             int* max_ctas) {
  return p.kp1 == 1 ? small_go<D, 1>(p, bar, steps, s, max_ctas)
                    : small_go<D, 2>(p, bar, steps, s, max_ctas);
}

// max_ctas != null: only report how many CTAs can be co-resident
cudaError_t launch_small(const KParams& p, unsigned* bar, long long steps, cudaStream_t s,
                         int* max_ctas) {
  switch (p.d) {
    case 1: return small_kp1<1>(p, bar, steps, s, max_ctas);
    case 2: return small_kp1<2>(p, bar, steps, s, max_ctas);
    case 3: return small_kp1<3>(p, bar, steps, s, max_ctas);
    case 4: return small_kp1<4>(p, bar, steps, s, max_ctas);
    case 5: return small_kp1<5>(p, bar, steps, s, max_ctas);
    case 6: return small_kp1<6>(p, bar, steps, s, max_ctas);
    case 7: return small_kp1<7>(p, bar, steps, s, max_ctas);
    case 8: return small_kp1<8>(p, bar, steps, s, max_ctas);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hb
