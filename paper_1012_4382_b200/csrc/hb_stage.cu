// Fused RK4 stage kernels of the HEOM propagator (sm_100a).
//
// Replaces, per RK4 stage, the reference's hierarchy_rhs_kernel + add_scaled /
// rk4_update passes (_kernels.py:23-72, driven from heom.py:370-383) with ONE
// kernel that evaluates the right-hand side of a tile of 32 ADOs and writes the
// next stage input directly:
//
//   stage 1: Y2 = s + dt/2 f(s)          reads s,            writes Y2
//   stage 2: Y3 = s + dt/2 f(Y2)         reads Y2, s,        writes Y3
//   stage 3: Y4 = s + dt   f(Y3)         reads Y3, s,        writes Y4
//   stage 4: s  = s + [(Y2-s) + 2(Y3-s) + (Y4-s)]/3 + dt/6 f(Y4)
//                                        reads Y4, s, Y2, Y3, writes s (in place)
//
// which is algebraically the reference's k1..k4 combination (heom.py:381) with
// 13 state passes per step instead of 23 (no k buffers).  Stage 4 also folds in
// the sink integration (heom.py:382-383), the divergence guard (heom.py:386-389),
// recording (heom.py:390-394) and the stop policy for the next step
// (heom.py:359-368): the last CTA to finish (atomic election) does the scalar
// bookkeeping, so the host only syncs once per CUDA-graph chunk.
//
// Layout: AoSoA, [tile][plane][32] float64.  HERMITIAN layout stores the real
// diagonal and the upper triangle (d*d planes, 392 B per ADO at d=7): every ADO
// of the hierarchy stays Hermitian because a, b, nu and H are real
// (heom.py:7-20), so the lower triangle is the conjugate.  GENERAL layout
// stores all d*d complex entries (2*d*d planes) for non-Hermitian inputs and the
// Level-2 kernel shim.
//
// Mapping: one CTA = one tile of 32 ADOs, d warps; lane = ADO, warp w handles
// elements w, w+d, ... (each warp gets one diagonal + (d-1)/2 off-diagonals in
// the Hermitian layout).  The tile is staged unpacked in shared memory (the
// commutator needs a full row and column), the 2*modes neighbour links of the
// tile are staged too; neighbour elements are gathered with read-only loads
// (the neighbour maps are monotone so a warp's 32 gathers touch few sectors).
#include "hb_device.cuh"

namespace hb {

// tile slot idx (0 .. NP*32-1, in memory order) -> (plane, lane)
template <int D, bool HERM>
__device__ __forceinline__ void slot_info(int idx, int& p, int& l) {
  if (!HERM || idx < D * TILE) {
    p = idx >> 5;
    l = idx & 31;
    return;
  }
  const int r = idx - D * TILE;
  p = D + 2 * (r >> 6) + (r & 1);
  l = (r >> 1) & 31;
}

// ---------------------------------------------------------------------------
// the stage kernel

template <int D, bool HERM, int STAGE>  // STAGE 1..4; 0 = right-hand side only
__global__ void __launch_bounds__(D * 32) k_stage(const KParams P) {
  constexpr int NP = Lay<D, HERM>::NP;
  constexpr int NE = Lay<D, HERM>::NE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double s_re[D][D][TILE];
  __shared__ double s_im[D][D][TILE];
  __shared__ double s_red[D];
  __shared__ int s_last;

  volatile Ctl* ctl = P.ctl;
  long long step_next = 0;
  if (STAGE != 0) {
    if (ctl->status != ST_RUNNING) return;
    step_next = ctl->step + 1;
  }
  const int tile = P.tile_begin + blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  HB_CHECK(tile < P.n_tiles_total);
  const int M = P.modes;
  int32_t* s_plus = reinterpret_cast<int32_t*>(smem_raw);
  int32_t* s_minus = s_plus + M * TILE;
  uint8_t* s_nv = reinterpret_cast<uint8_t*>(s_minus + M * TILE);

  const size_t tbase = (size_t)tile * NP * TILE;
  for (int idx = threadIdx.x; idx < NP * TILE; idx += D * 32) {
    int p, l;
    slot_info<D, HERM>(idx, p, l);
    const double v = __ldg(P.Yin + tbase + idx);
    int i, j, part;
    plane_info<D, HERM>(p, i, j, part);
    if (HERM) {
      if (i == j) {
        s_re[i][i][l] = v;
        s_im[i][i][l] = 0.0;
      } else if (part == 0) {
        s_re[i][j][l] = v;
        s_re[j][i][l] = v;
      } else {
        s_im[i][j][l] = v;
        s_im[j][i][l] = -v;
      }
    } else {
      if (part == 0) s_re[i][j][l] = v; else s_im[i][j][l] = v;
    }
  }
  const size_t gbase = (size_t)tile * M * TILE;
  for (int idx = threadIdx.x; idx < M * TILE; idx += D * 32) {
    s_plus[idx] = __ldg(P.plus + gbase + idx);
    s_minus[idx] = __ldg(P.minus + gbase + idx);
    s_nv[idx] = __ldg(P.nvec + gbase + idx);
  }
  __syncthreads();

  // sink rates on this stage's input sigma^0 (heom.py:282-283, 371-380)
  if (STAGE != 0 && tile == 0 && threadIdx.x == 0) {
    int t = 0;
    for (int s = 0; s < P.n_sinks; ++s) {
      double acc = 0.0;
      for (int cc = 0; cc < P.sink_nterms[s]; ++cc, ++t) {
        const int p = P.sink_pos[t];
        const double v = P.sink_rate[t] * s_re[p][p][0];
        acc = cc == 0 ? v : acc + v;
      }
      ctl->r[P.rpar][STAGE - 1][s] = acc;
    }
  }

  double damp;
  if (P.damp_plane) {
    damp = P.damp_plane[(size_t)tile * TILE + lane];
  } else {  // heom.py:275 tiers*gamma, generalised: sum_k nu_k * sum_j n_jk
    damp = 0.0;
    for (int kk = 0; kk < P.kp1; ++kk) {
      int tk = 0;
      for (int jj = 0; jj < P.n_sites; ++jj) tk += s_nv[(jj * P.kp1 + kk) * TILE + lane];
      damp += (double)tk * P.nu[kk];
    }
  }

  double maxa2 = 0.0;
  auto at = [&](int plane, int ln) -> int { return plane_off(HERM, D, plane, ln); };
  for (int e = warp; e < NE; e += D) {
    int i, j, pr, pim;
    elem_info<D, HERM>(e, i, j, pr, pim);
    const bool diag = HERM && (i == j);  // real element, raise terms cancel
    const double sr = s_re[i][j][lane], si = s_im[i][j][lane];
    const double f = -(damp + 0.5 * (P.decay[i] + P.decay[j]));
    double ar = f * sr, ai = f * si;
    double cr = 0.0, ci = 0.0;
#pragma unroll
    for (int l = 0; l < D; ++l) {
      const double hil = P.h[i * MAXD + l], hlj = P.h[l * MAXD + j];
      cr += hil * s_re[l][j][lane] - s_re[i][l][lane] * hlj;
      ci += hil * s_im[l][j][lane] - s_im[i][l][lane] * hlj;
    }
    ar += ci;  // acc += -1j * cm
    ai -= cr;
    const int mi = P.site_of[i], mj = P.site_of[j];
    if (mi >= 0) {
      for (int kk = 0; kk < P.kp1; ++kk) {
        const int m = mi * P.kp1 + kk;
        const int p = s_plus[m * TILE + lane];
        HB_CHECK(p < P.n_tiles_total * TILE);
        if (!diag && p >= 0) {  // + 1j * sig[p][i,j]
          const double* nb = P.Yin + (size_t)(p >> 5) * NP * TILE;
          const double xr = __ldg(nb + at(pr, p & 31)), xi = __ldg(nb + at(pim, p & 31));
          ar -= xi;
          ai += xr;
        }
        const int q = s_minus[m * TILE + lane];
        HB_CHECK(q < P.n_tiles_total * TILE);
        if (q >= 0) {  // + n (b + 1j a) sig[q][i,j]
          const double n = (double)s_nv[m * TILE + lane];
          const double cb = n * P.b[kk], ca = n * P.a[kk];
          const double* nb = P.Yin + (size_t)(q >> 5) * NP * TILE;
          const double xr = __ldg(nb + at(pr, q & 31));
          const double xi = diag ? 0.0 : __ldg(nb + at(pim, q & 31));
          ar += cb * xr - ca * xi;
          ai += cb * xi + ca * xr;
        }
      }
    }
    if (mj >= 0) {
      for (int kk = 0; kk < P.kp1; ++kk) {
        const int m = mj * P.kp1 + kk;
        const int p = s_plus[m * TILE + lane];
        if (!diag && p >= 0) {  // - 1j * sig[p][i,j]
          const double* nb = P.Yin + (size_t)(p >> 5) * NP * TILE;
          const double xr = __ldg(nb + at(pr, p & 31)), xi = __ldg(nb + at(pim, p & 31));
          ar += xi;
          ai -= xr;
        }
        const int q = s_minus[m * TILE + lane];
        if (q >= 0) {  // + n (b - 1j a) sig[q][i,j]
          const double n = (double)s_nv[m * TILE + lane];
          const double cb = n * P.b[kk], ca = n * P.a[kk];
          const double* nb = P.Yin + (size_t)(q >> 5) * NP * TILE;
          const double xr = __ldg(nb + at(pr, q & 31));
          const double xi = diag ? 0.0 : __ldg(nb + at(pim, q & 31));
          ar += cb * xr + ca * xi;
          ai += cb * xi - ca * xr;
        }
      }
    }

    if (i == j) {  // Lindblad refill of sink levels (dense path, heom.py:146)
      for (int q = 0; q < P.n_refill; ++q)
        if (P.refill_dst[q] == i) {
          const int src = P.refill_src[q];
          ar += P.refill_rate[q] * s_re[src][src][lane];
          ai += P.refill_rate[q] * s_im[src][src][lane];
        }
    }
    double yr, yi;
    if (STAGE == 0) {
      yr = ar;
      yi = ai;
    } else if (STAGE == 1) {
      yr = sr + P.coef * ar;
      yi = si + P.coef * ai;
    } else if (STAGE == 2 || STAGE == 3) {
      const double gr = P.sig[tbase + at(pr, lane)];
      const double gi = diag ? 0.0 : P.sig[tbase + at(pim, lane)];
      yr = gr + P.coef * ar;
      yi = gi + P.coef * ai;
    } else {
      const double gr = P.sig[tbase + at(pr, lane)];
      const double gi = diag ? 0.0 : P.sig[tbase + at(pim, lane)];
      const double y2r = P.Y2[tbase + at(pr, lane)], y3r = P.Y3[tbase + at(pr, lane)];
      const double y2i = diag ? 0.0 : P.Y2[tbase + at(pim, lane)];
      const double y3i = diag ? 0.0 : P.Y3[tbase + at(pim, lane)];
      const double w = P.dt / 6.0, third = 1.0 / 3.0;
      yr = gr + ((y2r - gr) + 2.0 * (y3r - gr) + (sr - gr)) * third + w * ar;
      yi = gi + ((y2i - gi) + 2.0 * (y3i - gi) + (si - gi)) * third + w * ai;
      const double a2 = yr * yr + yi * yi;
      maxa2 = fmax(maxa2, a2);
    }
    P.Yout[tbase + at(pr, lane)] = yr;
    if (!diag) P.Yout[tbase + at(pim, lane)] = yi;
  }

  if (STAGE == 4) {
    if (step_next % 25 == 0) {  // whole-state guard every 25 steps (heom.py:387)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
      if (lane == 0) s_red[warp] = maxa2;
      __syncthreads();
      if (threadIdx.x == 0) {
        double m = s_red[0];
        for (int w = 1; w < D; ++w) m = fmax(m, s_red[w]);
        atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                  (unsigned long long)__double_as_longlong(m));
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned prev = atomicAdd(const_cast<unsigned*>(&ctl->blocks_done), 1u);
      s_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && (threadIdx.x >> 5) == 0) {
      __threadfence();
      if (threadIdx.x == 0) ctl->launches = ctl->launches + 4;
      finish_step_warp<D, HERM>(P, step_next);
    }
  }
}

template <int D, bool HERM>
__global__ void k_init(const KParams P) {
  init_warp<D, HERM>(P);
}

// ---------------------------------------------------------------------------
// layout conversion: reference order (n_tot,d,d) complex <-> AoSoA planes

template <int D, bool HERM>
__global__ void k_pack(const KParams P, const double* __restrict__ ref, const int32_t* dev2ref,
                       double* __restrict__ dst) {
  constexpr int NP = Lay<D, HERM>::NP;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)P.n_tiles * TILE * NP;
  if (idx >= total) return;
  const int64_t tile = idx / (NP * TILE);
  int p, lane;
  slot_info<D, HERM>((int)(idx % (NP * TILE)), p, lane);
  const int64_t r = tile * TILE + lane;
  double v = 0.0;
  if (r < P.n_tot) {
    const int64_t k = dev2ref[r];
    int i, j, part;
    plane_info<D, HERM>(p, i, j, part);
    v = ref[(k * D * D + i * D + j) * 2 + part];
  }
  if (P.single)  // float state (HB_PREC_SINGLE): rounded once, like the reference's astype
    reinterpret_cast<float*>(dst)[idx] = (float)v;
  else
    dst[idx] = v;
}

template <int D, bool HERM>
__global__ void k_unpack(const KParams P, const double* __restrict__ src, const int32_t* dev2ref,
                         double* __restrict__ ref) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // over n_tot*D*D
  if (idx >= (int64_t)P.n_tot * D * D) return;
  const int64_t r = idx / (D * D);
  const int e = idx % (D * D);
  const int i = e / D, j = e % D;
  const int64_t k = dev2ref[r];
  const int64_t s0 = (r >> 5) * Lay<D, HERM>::NP * TILE;
  const int ln = (int)(r & 31);
  auto s = [&](int plane) -> double {  // float state when HB_PREC_SINGLE
    const int64_t o = s0 + plane_off(HERM, D, plane, ln);
    return P.single ? (double)reinterpret_cast<const float*>(src)[o] : src[o];
  };
  double re, im;
  if (HERM) {
    if (i == j) {
      re = s(i);
      im = 0.0;
    } else {
      const int a = i < j ? i : j, b = i < j ? j : i;
      int ee = D;
      for (int rr = 0; rr < a; ++rr) ee += D - 1 - rr;
      ee += b - a - 1;
      const int pr = D + 2 * (ee - D);
      re = s(pr);
      im = s(pr + 1);
      if (i > j) im = -im;
    }
  } else {
    re = s(2 * e);
    im = s(2 * e + 1);
  }
  ref[(k * D * D + e) * 2] = re;
  ref[(k * D * D + e) * 2 + 1] = im;
}

// ---------------------------------------------------------------------------
// Level-2 elementwise kernels (_kernels.py:61-84)

__global__ void k_elementwise(int op, int64_t n2, double* __restrict__ out,
                              const double* __restrict__ x, const double* __restrict__ y,
                              const double* __restrict__ z, const double* __restrict__ w, double c) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (op == 0) out[i] = x[i] + c * y[i];                            // add_scaled
    else out[i] = out[i] + c * (x[i] + 2.0 * (y[i] + z[i]) + w[i]);  // rk4_update
  }
}

__global__ void k_max_abs2(int64_t n, const double* __restrict__ x, unsigned long long* bits) {
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double a = x[2 * i] * x[2 * i] + x[2 * i + 1] * x[2 * i + 1];
    if (a > m) m = a;  // NaN never wins, as in the reference
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(bits, (unsigned long long)__double_as_longlong(m));
}

// ---------------------------------------------------------------------------
// launchers

static size_t dyn_smem(int modes) {
  return ((size_t)modes * TILE * (4 + 4 + 1) + 15) & ~(size_t)15;
}

template <int D, bool HERM, int STAGE>
static cudaError_t launch_one(const KParams& p, cudaStream_t s, int grid) {
  k_stage<D, HERM, STAGE><<<grid, D * 32, dyn_smem(p.modes), s>>>(p);
  return cudaGetLastError();
}

template <int D, bool HERM>
static cudaError_t configure_impl(const KParams&) {
  // allow the dynamic link tables beyond the 48 KB default (large d and modes);
  // not a stream operation, so it must run before graph capture
  const int lim = 64 * 1024;
  cudaError_t e = cudaFuncSetAttribute(k_stage<D, HERM, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (!e) e = cudaFuncSetAttribute(k_stage<D, HERM, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (!e) e = cudaFuncSetAttribute(k_stage<D, HERM, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (!e) e = cudaFuncSetAttribute(k_stage<D, HERM, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (!e) e = cudaFuncSetAttribute(k_stage<D, HERM, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  return e;
}

template <int D, bool HERM>
static cudaError_t dispatch_stage(int stage, const KParams& p, cudaStream_t s) {
  const int grid = p.n_tiles;
  switch (stage) {
    case 0: return launch_one<D, HERM, 0>(p, s, grid);
    case 1: return launch_one<D, HERM, 1>(p, s, grid);
    case 2: return launch_one<D, HERM, 2>(p, s, grid);
    case 3: return launch_one<D, HERM, 3>(p, s, grid);
    case 4: return launch_one<D, HERM, 4>(p, s, grid);
  }
  return cudaErrorInvalidValue;
}

#define HB_DISPATCH_D(FN, ...)                                                   \
  switch (p.d) {                                                                 \
    case 1: return p.hermitian ? FN<1, true>(__VA_ARGS__) : FN<1, false>(__VA_ARGS__); \
    case 2: return p.hermitian ? FN<2, true>(__VA_ARGS__) : FN<2, false>(__VA_ARGS__); \
    case 3: return p.hermitian ? FN<3, true>(__VA_ARGS__) : FN<3, false>(__VA_ARGS__); \
    case 4: return p.hermitian ? FN<4, true>(__VA_ARGS__) : FN<4, false>(__VA_ARGS__); \
    case 5: return p.hermitian ? FN<5, true>(__VA_ARGS__) : FN<5, false>(__VA_ARGS__); \
    case 6: return p.hermitian ? FN<6, true>(__VA_ARGS__) : FN<6, false>(__VA_ARGS__); \
    case 7: return p.hermitian ? FN<7, true>(__VA_ARGS__) : FN<7, false>(__VA_ARGS__); \
    case 8: return p.hermitian ? FN<8, true>(__VA_ARGS__) : FN<8, false>(__VA_ARGS__); \
    case 9: return p.hermitian ? FN<9, true>(__VA_ARGS__) : FN<9, false>(__VA_ARGS__); \
  }                                                                              \
  return cudaErrorInvalidValue;

cudaError_t launch_stage(int stage, const KParams& p, cudaStream_t s) {
  if (p.fast && stage >= 1) return launch_mm4(stage, p, s);
  HB_DISPATCH_D(dispatch_stage, stage, p, s)
}

cudaError_t launch_rhs_only(const KParams& p, cudaStream_t s) { return launch_stage(0, p, s); }

cudaError_t configure_stages(const KParams& p) { HB_DISPATCH_D(configure_impl, p) }

template <int D, bool HERM>
static cudaError_t init_impl(const KParams& p, cudaStream_t s) {
  k_init<D, HERM><<<1, 32, 0, s>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_init(const KParams& p, cudaStream_t s) { HB_DISPATCH_D(init_impl, p, s) }

template <int D, bool HERM>
static cudaError_t pack_impl(const KParams& p, const double* ref, const int32_t* d2r, double* dst,
                             cudaStream_t s) {
  const int64_t total = (int64_t)p.n_tiles * TILE * Lay<D, HERM>::NP;
  k_pack<D, HERM><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(p, ref, d2r, dst);
  return cudaGetLastError();
}
cudaError_t launch_pack(const KParams& p, const double* ref_sig, const int32_t* dev2ref,
                        double* dst, cudaStream_t s) {
  HB_DISPATCH_D(pack_impl, p, ref_sig, dev2ref, dst, s)
}

template <int D, bool HERM>
static cudaError_t unpack_impl(const KParams& p, const double* src, const int32_t* d2r,
                               double* ref, cudaStream_t s) {
  const int64_t total = (int64_t)p.n_tot * D * D;
  k_unpack<D, HERM><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(p, src, d2r, ref);
  return cudaGetLastError();
}
cudaError_t launch_unpack(const KParams& p, const double* src, const int32_t* dev2ref,
                          double* ref_sig, cudaStream_t s) {
  HB_DISPATCH_D(unpack_impl, p, src, dev2ref, ref_sig, s)
}

cudaError_t launch_elementwise(int op, int64_t n, double* out, const double* x, const double* y,
                               const double* z, const double* w, double c, cudaStream_t s) {
  const int64_t n2 = 2 * n;
  int grid = (int)((n2 + 255) / 256);
  if (grid > 148 * 16) grid = 148 * 16;
  if (grid < 1) grid = 1;
  k_elementwise<<<grid, 256, 0, s>>>(op, n2, out, x, y, z, w, c);
  return cudaGetLastError();
}

cudaError_t launch_max_abs2(int64_t n, const double* x, unsigned long long* bits, cudaStream_t s) {
  int grid = (int)((n + 255) / 256);
  if (grid > 148 * 16) grid = 148 * 16;
  if (grid < 1) grid = 1;
  k_max_abs2<<<grid, 256, 0, s>>>(n, x, bits);
  return cudaGetLastError();
}

}  // namespace hb
