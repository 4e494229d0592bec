// Small hierarchies resident in the distributed shared memory of ONE thread-block
// cluster (up to 16 CTAs on 16 SMs): the whole state -- sigma, the two rotating
// stage buffers and B -- lives in shared memory for the whole run, the RK4
// stages are separated by hardware cluster barriers (barrier.cluster, a few
// hundred ns) instead of kernel boundaries or software grid barriers (~2 us on
// B200, tools/micro/gridbar.cu), and a neighbour's cross is gathered from the
// shared memory of the CTA that owns it (mapa + ld.shared::cluster) instead of
// from L2.  One launch runs many steps; the step bookkeeping (sinks
// heom.py:382-383, guard heom.py:386-389, records, stop policy heom.py:359-368)
// is done by CTA 0 behind a fifth barrier.
//
// At config 3's K = 0 twin (1,716 ADOs = 54 tiles) the state is 5 x 0.67 MB:
// 14 CTAs of 4 warps (one tile per warp, lane = ADO), 4 tiles and 4 buffers
// (sigma, P = Y2 / Y4, Q = Y3, B) per CTA = 201 KB of shared memory each.
// Arithmetic: the reference RHS (_kernels.py:23-58, K+1 modes per site) and the
// 12-pass RK4 bookkeeping of k_mm4 (hb_mm_common.cuh), term for term.
#include <cstring>
#include "hb_device.cuh"
#include "hb_mm_common.cuh"

namespace hb {

namespace {

constexpr int kClTpc = 4;        // tiles (= warps) per CTA
constexpr int kClMaxCtas = 16;   // non-portable cluster size limit

__device__ __forceinline__ uint32_t cl_map(uint32_t saddr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ double cl_ld(uint32_t a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ double2 cl_ld2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ int cl_rank() {
  int r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int D, int KP1>
struct ClSmem {
  static constexpr int NP = D * D, M = D * KP1, TB = NP * TILE;
  static constexpr size_t BUF = (size_t)kClTpc * TB * 8;      // one state buffer, 4 tiles
  static constexpr size_t TAB = (size_t)kClTpc * M * TILE * 4;
  static constexpr size_t UP = 4 * BUF, DN = UP + TAB, NV = DN + TAB;
  static constexpr size_t MAXW = (NV + (size_t)kClTpc * M * TILE + 15) / 16 * 16;
  static constexpr size_t BYTES = MAXW + 16 * 8;
};

}  // namespace

template <int D, int KP1>
__global__ void __launch_bounds__(kClTpc * 32, 1) k_cluster(const KParams P, long long max_steps) {
  using T = double;
  using L = ClSmem<D, KP1>;
  constexpr int NP = D * D, M = D * KP1, TB = NP * TILE, DIAG = D * TILE;
  extern __shared__ __align__(128) unsigned char smem[];
  T* const sb = reinterpret_cast<T*>(smem);  // buffers [4][kClTpc][TB]: sigma, P, Q, B
  int32_t(*sUp)[TILE] = reinterpret_cast<int32_t(*)[TILE]>(smem + L::UP);
  int32_t(*sDn)[TILE] = reinterpret_cast<int32_t(*)[TILE]>(smem + L::DN);
  uint8_t(*sN)[TILE] = reinterpret_cast<uint8_t(*)[TILE]>(smem + L::NV);
  double* sMax = reinterpret_cast<double*>(smem + L::MAXW);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = cl_rank();
  const int tile = cta * kClTpc + w;
  const bool active = tile < P.n_tiles;
  volatile Ctl* ctl = P.ctl;
  T* const gsig = const_cast<T*>(P.sig);  // sigma in global memory (stage-4 params: Yout too)
  const uint32_t sbase = smem_u32(sb);
  auto buf = [&](int b, int lt) -> T* { return sb + ((size_t)b * kClTpc + lt) * TB; };
  // this warp's tables ([mode][32] of its tile) and its tile of sigma, once per launch
  int32_t(*up)[TILE] = sUp + w * M;
  int32_t(*dn)[TILE] = sDn + w * M;
  uint8_t(*nv)[TILE] = sN + w * M;
  if (active) {
    const size_t g = (size_t)tile * M * TILE;
    for (int m = 0; m < M; ++m) {
      up[m][lane] = __ldg(P.plus + g + m * TILE + lane);
      dn[m][lane] = __ldg(P.minus + g + m * TILE + lane);
      nv[m][lane] = __ldg(P.nvec + g + m * TILE + lane);
    }
    for (int i = lane; i < TB; i += 32) buf(0, w)[i] = __ldcg(P.sig + (size_t)tile * TB + i);
  }
  T damp = 0;
  {
    int tk[KP1];
#pragma unroll
    for (int k = 0; k < KP1; ++k) tk[k] = 0;
    if (active) {
#pragma unroll
      for (int m = 0; m < M; ++m) tk[m % KP1] += nv[m][lane];
    }
#pragma unroll
    for (int k = 0; k < KP1; ++k) damp = fma((T)tk[k], P.nu[k], damp);
  }
  cl_sync();
  constexpr T third = (T)(1.0 / 3.0), two3 = (T)(2.0 / 3.0);
  // buffer roles: stage s reads bin, writes bout; sigma = 0, P = 1, Q = 2, B = 3

  long long it = 0;
  for (; it < max_steps; ++it) {
    if (ctl->status != ST_RUNNING) break;
    const long long step_next = ctl->step + 1;
    double maxa2 = 0.0;
#pragma unroll 1
    for (int stage = 1; stage <= 4; ++stage) {
      const int bin = stage == 1 ? 0 : (stage == 4 ? 1 : stage - 1);  // sigma, P, Q, P
      const int bout = stage == 4 ? 0 : (stage == 3 ? 1 : stage);     // P, Q, P, sigma
      const T c = stage == 4 ? P.dt / 6.0 : (stage == 3 ? P.dt : 0.5 * P.dt);
      if (active) {
        const T* own = buf(bin, w);
        if (tile == 0 && lane == 0) {  // sink rates of this stage input (heom.py:282-283)
          int q = 0;
          for (int sk = 0; sk < P.n_sinks; ++sk) {
            double a = 0.0;
            for (int cc = 0; cc < P.sink_nterms[sk]; ++cc, ++q) {
              const double v = P.sink_rate[q] * own[P.sink_pos[q] * TILE];
              a = cc == 0 ? v : a + v;
            }
            ctl->r[stage - 1][sk] = a;
          }
        }
        // ---- phase A: the ADO from shared memory, base + c (damping + commutator)
        T s[NP];
#pragma unroll
        for (int i = 0; i < D; ++i) s[i] = own[i * TILE + lane];
#pragma unroll
        for (int e = 0; e < D * (D - 1) / 2; ++e) {
          const double2 v = *reinterpret_cast<const double2*>(own + DIAG + e * 2 * TILE + 2 * lane);
          s[D + 2 * e] = v.x;
          s[D + 2 * e + 1] = v.y;
        }
        const T* bse = stage == 4 ? buf(3, w) : buf(0, w);  // sigma, or B at stage 4
        T acc[NP];
        auto base = [&](int p, T x) -> T {  // the 12-pass RK base term of plane p
          if (stage == 1) return x;
          const T b = bse[herm_off(D, p, lane)];
          if (stage == 4) return fma(x, third, b);
          return b;
        };
#pragma unroll
        for (int i = 0; i < D; ++i) {
          T cm = 0;
#pragma unroll
          for (int l = 0; l < D; ++l)
            if (l != i) cm = fma(P.h[i * MAXD + l], sim<T, D>(s, i, l), cm);
          acc[i] = fma(c, fma(-(damp + P.decay[i]), s[i], (T)-2 * cm), base(i, s[i]));
#pragma unroll
          for (int j = i + 1; j < D; ++j) {
            const int pr = Pk<D>::re(i, j), pim = Pk<D>::im(i, j);
            const T dh = P.h[i * MAXD + i] - P.h[j * MAXD + j], hij = P.h[i * MAXD + j];
            T cr = fma(hij, s[j], fma(-hij, s[i], dh * s[pr]));
            T ci = dh * s[pim];
#pragma unroll
            for (int l = 0; l < D; ++l) {
              if (l == i || l == j) continue;
              const T hil = P.h[i * MAXD + l], hlj = P.h[l * MAXD + j];
              cr = fma(hil, sre<T, D>(s, l, j), cr);
              cr = fma(-hlj, sre<T, D>(s, i, l), cr);
              ci = fma(hil, sim<T, D>(s, l, j), ci);
              ci = fma(-hlj, sim<T, D>(s, i, l), ci);
            }
            const T f = -(damp + (T)0.5 * (P.decay[i] + P.decay[j]));
            acc[pr] = fma(c, fma(f, s[pr], ci), base(pr, s[pr]));
            acc[pim] = fma(c, fma(f, s[pim], -cr), base(pim, s[pim]));
          }
        }
        // ---- phase B: the neighbour crosses from the owners' shared memory
        T cbk[KP1], cak[KP1];
#pragma unroll
        for (int k = 0; k < KP1; ++k) {
          cbk[k] = c * P.b[k];
          cak[k] = c * P.a[k];
        }
        // remote address of (plane offset o) of link target t in buffer bin
        auto raddr = [&](int t) -> uint32_t {
          const int g = t >> 5;
          const uint32_t local = sbase + (uint32_t)((((size_t)bin * kClTpc + g % kClTpc) * TB) * 8);
          return cl_map(local, g / kClTpc);
        };
#pragma unroll
        for (int st = 0; st < D; ++st) {
#pragma unroll
          for (int k = 0; k < KP1; ++k) {
            const int m = st * KP1 + k;
            const int pu = up[m][lane], pd = dn[m][lane];
            const bool vu = pu >= 0, vd = pd >= 0;
            const uint32_t au = vu ? raddr(pu) + (uint32_t)((pu & 31) * 16) : 0u;
            const uint32_t ad = vd ? raddr(pd) + (uint32_t)((pd & 31) * 16) : 0u;
            const uint32_t ad1 = vd ? raddr(pd) + (uint32_t)((pd & 31) * 8) : 0u;
            const T n = vd ? (T)nv[m][lane] : (T)0;
            const T cb = n * cbk[k], ca = n * cak[k];
            const T cu = vu ? c : (T)0;
            if (vd) acc[st] = fma((T)2 * cb, cl_ld(ad1 + (uint32_t)(st * TILE * 8)), acc[st]);
#pragma unroll
            for (int o = 0; o < D; ++o) {
              if (o == st) continue;
              const int pr = Pk<D>::re(st, o), pim = Pk<D>::im(st, o);
              const int e = Pk<D>::off(st < o ? st : o, st < o ? o : st);
              const uint32_t eo = (uint32_t)((DIAG + e * 2 * TILE) * 8);
              double2 uv = make_double2(0.0, 0.0), dv = make_double2(0.0, 0.0);
              if (vu) uv = cl_ld2(au + eo);
              if (vd) dv = cl_ld2(ad + eo);
              if (o > st) {
                acc[pr] = fma(cb, dv.x, fma(-ca, dv.y, fma(-cu, uv.y, acc[pr])));
                acc[pim] = fma(cb, dv.y, fma(ca, dv.x, fma(cu, uv.x, acc[pim])));
              } else {
                acc[pr] = fma(cb, dv.x, fma(ca, dv.y, fma(cu, uv.y, acc[pr])));
                acc[pim] = fma(cb, dv.y, fma(-ca, dv.x, fma(-cu, uv.x, acc[pim])));
              }
            }
          }
        }
        // every CTA has gathered this stage's input before anyone overwrites it:
        // the outputs go to OUT[stage] != IN[stage], and B / P are rewritten only
        // behind at least one more barrier
        T* out = buf(bout, w);
        T* bb = buf(3, w);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const int o = herm_off(D, p, lane);
          if (stage == 2) bb[o] = fma(two3, acc[p], (s[p] - buf(0, w)[o]) * third);
          out[o] = acc[p];
        }
        if (stage == 4) {
#pragma unroll
          for (int i = 0; i < D; ++i) maxa2 = fmax(maxa2, acc[i] * acc[i]);
#pragma unroll
          for (int e = 0; e < D * (D - 1) / 2; ++e)
            maxa2 = fmax(maxa2, fma(acc[D + 2 * e], acc[D + 2 * e], acc[D + 2 * e + 1] * acc[D + 2 * e + 1]));
        }
      }
      if (stage == 4 && step_next % 25 == 0) {  // whole-state guard (heom.py:386-389)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
        if (lane == 0) sMax[w] = maxa2;
        __syncthreads();
        if (threadIdx.x == 0) {
          double mx = sMax[0];
          for (int q = 1; q < kClTpc; ++q) mx = fmax(mx, sMax[q]);
          atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                    (unsigned long long)__double_as_longlong(mx));
        }
      }
      cl_sync();
    }
    // ---- the step bookkeeping: CTA 0, sigma^0 published to global first
    if (cta == 0 && w == 0) {
      if (lane == 0)
        for (int p = 0; p < NP; ++p) gsig[herm_off(D, p, 0)] = buf(0, 0)[herm_off(D, p, 0)];
      __syncwarp();
      __threadfence();
      finish_step_warp<D, true>(P, step_next);
      __threadfence();
    }
    cl_sync();
  }
  // the state back to global memory (hb_get_state / hb_get_sigma0 / the next launch)
  if (active)
    for (int i = lane; i < TB; i += 32) gsig[(size_t)tile * TB + i] = buf(0, w)[i];
}

bool cluster_supported(int d, int kp1) { return d >= 1 && d <= 8 && kp1 >= 1 && kp1 <= 2; }

template <int D, int KP1>
static cudaError_t cluster_go(const KParams& p, long long steps, cudaStream_t s, int* max_tiles) {
  using L = ClSmem<D, KP1>;
  auto kern = k_cluster<D, KP1>;
  if (max_tiles) {  // what fits: shared memory per CTA and the cluster size
    int dev = 0, smem_optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    *max_tiles = (size_t)smem_optin >= L::BYTES ? kClMaxCtas * kClTpc : 0;
    return cudaSuccess;
  }
  const int ctas = (p.n_tiles + kClTpc - 1) / kClTpc;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
  if (!e) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ctas);
  cfg.blockDim = dim3(kClTpc * 32);
  cfg.dynamicSmemBytes = L::BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)ctas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p, steps);
}

template <int D>
static cudaError_t cluster_kp1(const KParams& p, long long steps, cudaStream_t s, int* mt) {
  return p.kp1 == 1 ? cluster_go<D, 1>(p, steps, s, mt) : cluster_go<D, 2>(p, steps, s, mt);
}

// p = stage-4 params (sigma in p.sig).  max_tiles != null: only report the
// largest hierarchy (in tiles) the cluster holds, 0 if none.
cudaError_t launch_cluster(const KParams& p, long long steps, cudaStream_t s, int* max_tiles) {
  switch (p.d) {
    case 1: return cluster_kp1<1>(p, steps, s, max_tiles);
    case 2: return cluster_kp1<2>(p, steps, s, max_tiles);
    case 3: return cluster_kp1<3>(p, steps, s, max_tiles);
    case 4: return cluster_kp1<4>(p, steps, s, max_tiles);
    case 5: return cluster_kp1<5>(p, steps, s, max_tiles);
    case 6: return cluster_kp1<6>(p, steps, s, max_tiles);
    case 7: return cluster_kp1<7>(p, steps, s, max_tiles);
    case 8: return cluster_kp1<8>(p, steps, s, max_tiles);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hb
