// Production stage kernel: one thread per ADO, fully unrolled at compile time.
//
// Same arithmetic and the same fused-RK4 stage structure as k_stage
// (hb_stage.cu, whose header describes the stages), specialised for the shape
// every production run has: Hermitian-packed state, every block level is a
// site (site_of == identity, as for FMO and the dimer), d and K+1 known at
// compile time.  The generic kernel spends ~70% of its issue slots on runtime
// element decoding, parameter indexing and link branches (ncu, profiles/);
// here:
//   * the thread's own ADO (d*d doubles) lives in registers, so the commutator
//     -i[H, s] reads no memory and H comes from the constant bank with
//     immediate offsets;
//   * plane offsets of every element are compile-time immediates of the LDG;
//   * absent links (TRUNCATED / ABSENT) point at a zero tile, so the 4(K+1)
//     gathers of an element are unconditional and can all be in flight;
//   * per-link base pointers and the lower coefficients n_m (b_k, a_k) are
//     staged once per thread in shared memory (the thread's own column).
#include <cstdlib>
#include <type_traits>
#include "hb_device.cuh"
#include "hb_fast.cuh"

namespace hb {

constexpr int FT = 64;  // threads (ADOs) per CTA

template <int STAGE>
__device__ __forceinline__ void epilogue(const KParams& P, size_t tb, int pr, int pim, double sr,
                                         double si, double ar, double ai, double& maxa2) {
  double yr, yi = 0.0;
  if (STAGE == 1) {
    yr = sr + P.coef * ar;
    yi = si + P.coef * ai;
  } else if (STAGE == 2 || STAGE == 3) {
    const double gr = P.sig[tb + pr * TILE];
    const double gi = pim >= 0 ? P.sig[tb + pim * TILE] : 0.0;
    yr = gr + P.coef * ar;
    yi = gi + P.coef * ai;
  } else {
    const double gr = P.sig[tb + pr * TILE];
    const double y2r = P.Y2[tb + pr * TILE], y3r = P.Y3[tb + pr * TILE];
    const double w = P.dt / 6.0, third = 1.0 / 3.0;
    yr = gr + ((y2r - gr) + 2.0 * (y3r - gr) + (sr - gr)) * third + w * ar;
    if (pim >= 0) {
      const double gi = P.sig[tb + pim * TILE];
      const double y2i = P.Y2[tb + pim * TILE], y3i = P.Y3[tb + pim * TILE];
      yi = gi + ((y2i - gi) + 2.0 * (y3i - gi) + (si - gi)) * third + w * ai;
    }
    maxa2 = fmax(maxa2, yr * yr + yi * yi);
  }
  P.Yout[tb + pr * TILE] = yr;
  if (pim >= 0) P.Yout[tb + pim * TILE] = yi;
}

template <int D, int KP1, int STAGE, int MINB>
__global__ void __launch_bounds__(FT, MINB) k_fast(const KParams P) {
  constexpr int NP = D * D;
  constexpr int M = D * KP1;
  __shared__ double2 s_coef[M][FT];          // n_m * (b_k, a_k)
  __shared__ const double* s_up[M][FT];      // base of the raise neighbour (or zero tile)
  __shared__ const double* s_dn[M][FT];      // base of the lower neighbour (or zero tile)
  __shared__ double s_red[FT / 32];
  __shared__ int s_last;

  volatile Ctl* ctl = P.ctl;
  if (ctl->status != ST_RUNNING) return;
  const long long step_next = ctl->step + 1;
  const int t = threadIdx.x;
  const int r = blockIdx.x * FT + t;
  const int tile = P.tile_begin + (r >> 5), lane = r & 31;
  const bool active = (r >> 5) < P.n_tiles;
  double maxa2 = 0.0;

  if (active && lane == 0 && P.prefetch) {
    prefetch_epilogue<STAGE>(P, (size_t)tile * NP * TILE, NP * TILE * sizeof(double));
    if (P.pf_dist > 0) prefetch_tile<STAGE>(P, tile + P.pf_dist);
  }
  if (active) {
    const size_t tb = (size_t)tile * NP * TILE + lane;
    double s[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) s[p] = __ldg(P.Yin + tb + p * TILE);

    // links and lower coefficients of this ADO
    const size_t gb = (size_t)tile * M * TILE + lane;
    int tk[KP1];
#pragma unroll
    for (int k = 0; k < KP1; ++k) tk[k] = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int up = __ldg(P.plus + gb + m * TILE);
      const int dn = __ldg(P.minus + gb + m * TILE);
      const int n = __ldg(P.nvec + gb + m * TILE);
      tk[m % KP1] += n;
      const double nd = (double)n;
      s_coef[m][t] = make_double2(nd * P.b[m % KP1], nd * P.a[m % KP1]);
      s_up[m][t] = up >= 0 ? P.Yin + (size_t)(up >> 5) * NP * TILE + (up & 31) : P.zero_tile;
      s_dn[m][t] = dn >= 0 ? P.Yin + (size_t)(dn >> 5) * NP * TILE + (dn & 31) : P.zero_tile;
    }
    // heom.py:275 (tiers * gamma), generalised: sum_k nu_k * sum_j n_jk
    double damp = 0.0;
#pragma unroll
    for (int k = 0; k < KP1; ++k) damp += (double)tk[k] * P.nu[k];

    // sink rates of this stage input (heom.py:282-283, 371-380): ADO 0 only
    if (tile == 0 && lane == 0) {
      int q = 0;
      for (int sk = 0; sk < P.n_sinks; ++sk) {
        double acc = 0.0;
        for (int cc = 0; cc < P.sink_nterms[sk]; ++cc, ++q) {
          const double v = P.sink_rate[q] * __ldg(P.Yin + P.sink_pos[q] * TILE);
          acc = cc == 0 ? v : acc + v;
        }
        ctl->r[STAGE - 1][sk] = acc;
      }
    }

#pragma unroll
    for (int i = 0; i < D; ++i) {
      const double* rup[KP1];
      const double* rdn[KP1];
      double2 rco[KP1];
#pragma unroll
      for (int k = 0; k < KP1; ++k) {
        rup[k] = s_up[i * KP1 + k][t];
        rdn[k] = s_dn[i * KP1 + k][t];
        rco[k] = s_coef[i * KP1 + k][t];
      }
      // ---- diagonal (i, i): real; raise terms cancel, lower terms add twice
      {
        double cm_im = 0.0;  // Im sum_l (h_il s_li - s_il h_li) = -2 sum_l h_il Im s_il
#pragma unroll
        for (int l = 0; l < D; ++l)
          if (l != i) cm_im += P.h[i * MAXD + l] * sim<D>(s, i, l);
        double ar = -(damp + P.decay[i]) * s[i] - 2.0 * cm_im;
#pragma unroll
        for (int k = 0; k < KP1; ++k) ar += 2.0 * rco[k].x * __ldg(rdn[k] + i * TILE);
        epilogue<STAGE>(P, tb, i, -1, s[i], 0.0, ar, 0.0, maxa2);
      }
      // ---- upper off-diagonals (i, j > i)
#pragma unroll
      for (int j = i + 1; j < D; ++j) {
        const int pr = Pk<D>::re(i, j), pim = Pk<D>::im(i, j);
        const double sr = s[pr], si = s[pim];
        const double f = -(damp + 0.5 * (P.decay[i] + P.decay[j]));
        double cr = 0.0, ci = 0.0;
#pragma unroll
        for (int l = 0; l < D; ++l) {
          const double hil = P.h[i * MAXD + l], hlj = P.h[l * MAXD + j];
          cr += hil * sre<D>(s, l, j) - sre<D>(s, i, l) * hlj;
          ci += hil * sim<D>(s, l, j) - sim<D>(s, i, l) * hlj;
        }
        double ar = f * sr + ci;  // acc += -1j * cm
        double ai = f * si - cr;
        // row site i: + 1j s_up, + n (b + 1j a) s_dn
#pragma unroll
        for (int k = 0; k < KP1; ++k) {
          const double ur = __ldg(rup[k] + pr * TILE), ui = __ldg(rup[k] + pim * TILE);
          const double dr = __ldg(rdn[k] + pr * TILE), di = __ldg(rdn[k] + pim * TILE);
          ar += rco[k].x * dr - rco[k].y * di - ui;
          ai += rco[k].x * di + rco[k].y * dr + ur;
        }
        // column site j: - 1j s_up, + n (b - 1j a) s_dn
#pragma unroll
        for (int k = 0; k < KP1; ++k) {
          const double* cu = s_up[j * KP1 + k][t];
          const double* cd = s_dn[j * KP1 + k][t];
          const double2 cc = s_coef[j * KP1 + k][t];
          const double ur = __ldg(cu + pr * TILE), ui = __ldg(cu + pim * TILE);
          const double dr = __ldg(cd + pr * TILE), di = __ldg(cd + pim * TILE);
          ar += cc.x * dr + cc.y * di + ui;
          ai += cc.x * di - cc.y * dr - ur;
        }
        epilogue<STAGE>(P, tb, pr, pim, sr, si, ar, ai, maxa2);
      }
    }
  }

  if (STAGE == 4) {
    const int lane_id = t & 31, warp = t >> 5;
    if (step_next % 25 == 0) {  // whole-state guard every 25 steps (heom.py:387)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
      if (lane_id == 0) s_red[warp] = maxa2;
      __syncthreads();
      if (t == 0) {
        double m = s_red[0];
        for (int w = 1; w < FT / 32; ++w) m = fmax(m, s_red[w]);
        atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                  (unsigned long long)__double_as_longlong(m));
      }
    }
    __threadfence();
    __syncthreads();
    if (t == 0) {
      const unsigned prev = atomicAdd(const_cast<unsigned*>(&ctl->blocks_done), 1u);
      s_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && (t >> 5) == 0) {
      __threadfence();
      if (t == 0) ctl->launches = ctl->launches + 4;
      finish_step_warp<D, true>(P, step_next);
    }
  }
}


// Column-streamed variant: the commutator via X = H sigma computed one column
// of sigma at a time, so only one column of sigma, one column of X and the
// not-yet-consumed lower half of X are live (instead of all of sigma):
//   cm_ij = (H s - s H)_ij = X_ij - conj(X_ji)   (s Hermitian, H real symmetric)
// Element (i, j <= ... ) of the upper triangle is finished while column j is
// live (X_ji was parked at column i < j).  Links are int offsets into the
// state buffer; absent links point at the zero tile appended to every buffer.
template <int D, int KP1, int STAGE, int MINB>
__global__ void __launch_bounds__(FT, MINB) k_col(const KParams P) {
  constexpr int NP = D * D;
  constexpr int M = D * KP1;
  constexpr int NL = D * (D - 1) / 2 > 0 ? D * (D - 1) / 2 : 1;
  __shared__ double2 s_coef[M][FT];  // n_m * (b_k, a_k)
  __shared__ int s_up[M][FT];        // element offset of the raise neighbour (or zero tile)
  __shared__ int s_dn[M][FT];        // element offset of the lower neighbour (or zero tile)
  __shared__ double s_red[FT / 32];
  __shared__ int s_last;

  volatile Ctl* ctl = P.ctl;
  if (ctl->status != ST_RUNNING) return;
  const long long step_next = ctl->step + 1;
  const int t = threadIdx.x;
  const int r = blockIdx.x * FT + t;
  const int tile = P.tile_begin + (r >> 5), lane = r & 31;
  const bool active = (r >> 5) < P.n_tiles;
  double maxa2 = 0.0;

  if (active && lane == 0 && P.prefetch) {
    prefetch_epilogue<STAGE>(P, (size_t)tile * NP * TILE, NP * TILE * sizeof(double));
    if (P.pf_dist > 0) prefetch_tile<STAGE>(P, tile + P.pf_dist);
  }
  if (active) {
    const size_t tb = (size_t)tile * NP * TILE + lane;
    const double* own = P.Yin + tb;
    const int zero_off = P.n_tiles_total * NP * TILE;
    const size_t gb = (size_t)tile * M * TILE + lane;
    int tk[KP1];
#pragma unroll
    for (int k = 0; k < KP1; ++k) tk[k] = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int up = __ldg(P.plus + gb + m * TILE);
      const int dn = __ldg(P.minus + gb + m * TILE);
      const int n = __ldg(P.nvec + gb + m * TILE);
      tk[m % KP1] += n;
      const double nd = (double)n;
      s_coef[m][t] = make_double2(nd * P.b[m % KP1], nd * P.a[m % KP1]);
      s_up[m][t] = up >= 0 && !P.debug ? (up >> 5) * NP * TILE + (up & 31) : zero_off;
      s_dn[m][t] = dn >= 0 && !P.debug ? (dn >> 5) * NP * TILE + (dn & 31) : zero_off;
    }
    double damp = 0.0;  // heom.py:275, generalised: sum_k nu_k * sum_j n_jk
#pragma unroll
    for (int k = 0; k < KP1; ++k) damp += (double)tk[k] * P.nu[k];

    if (tile == 0 && lane == 0) {  // sink rates of this stage input (heom.py:282-283)
      int q = 0;
      for (int sk = 0; sk < P.n_sinks; ++sk) {
        double acc = 0.0;
        for (int cc = 0; cc < P.sink_nterms[sk]; ++cc, ++q) {
          const double v = P.sink_rate[q] * __ldg(P.Yin + P.sink_pos[q] * TILE);
          acc = cc == 0 ? v : acc + v;
        }
        ctl->r[STAGE - 1][sk] = acc;
      }
    }

    double lxr[NL], lxi[NL];  // parked lower half of X: (row, col) with row > col
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double cre[D], cim[D];  // column j of sigma
#pragma unroll
      for (int l = 0; l < D; ++l) {
        if (l == j) {
          cre[l] = __ldg(own + l * TILE);
          cim[l] = 0.0;
        } else if (l < j) {
          cre[l] = __ldg(own + Pk<D>::re(l, j) * TILE);
          cim[l] = __ldg(own + Pk<D>::im(l, j) * TILE);
        } else {
          cre[l] = __ldg(own + Pk<D>::re(j, l) * TILE);
          cim[l] = -__ldg(own + Pk<D>::im(j, l) * TILE);
        }
      }
      double xr[D], xi[D];  // column j of X = H sigma
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double ar = 0.0, ai = 0.0;
#pragma unroll
        for (int l = 0; l < D; ++l) {
          ar += P.h[i * MAXD + l] * cre[l];
          ai += P.h[i * MAXD + l] * cim[l];
        }
        xr[i] = ar;
        xi[i] = ai;
      }
      int cu[KP1], cd[KP1];
      double2 cco[KP1];
#pragma unroll
      for (int k = 0; k < KP1; ++k) {
        cu[k] = s_up[j * KP1 + k][t];
        cd[k] = s_dn[j * KP1 + k][t];
        cco[k] = s_coef[j * KP1 + k][t];
      }
      {  // diagonal (j, j): -i (X_jj - conj X_jj) = 2 Im X_jj; lower terms twice
        double ar = -(damp + P.decay[j]) * cre[j] + 2.0 * xi[j];
#pragma unroll
        for (int k = 0; k < KP1; ++k) ar += 2.0 * cco[k].x * __ldg(P.Yin + cd[k] + j * TILE);
        epilogue<STAGE>(P, tb, j, -1, cre[j], 0.0, ar, 0.0, maxa2);
      }
#pragma unroll
      for (int i = 0; i < j; ++i) {  // upper element (i, j)
        const int pr = Pk<D>::re(i, j), pim = Pk<D>::im(i, j);
        const int li = (j * (j - 1)) / 2 + i;  // parked X_ji
        const double cmr = xr[i] - lxr[li], cmi = xi[i] + lxi[li];
        const double f = -(damp + 0.5 * (P.decay[i] + P.decay[j]));
        double ar = f * cre[i] + cmi;  // acc += -1j * cm
        double ai = f * cim[i] - cmr;
#pragma unroll
        for (int k = 0; k < KP1; ++k) {  // row site i: + 1j up, + n (b + 1j a) dn
          const int ru = s_up[i * KP1 + k][t], rd = s_dn[i * KP1 + k][t];
          const double2 rc = s_coef[i * KP1 + k][t];
          const double ur = __ldg(P.Yin + ru + pr * TILE), ui = __ldg(P.Yin + ru + pim * TILE);
          const double dr = __ldg(P.Yin + rd + pr * TILE), di = __ldg(P.Yin + rd + pim * TILE);
          ar += rc.x * dr - rc.y * di - ui;
          ai += rc.x * di + rc.y * dr + ur;
        }
#pragma unroll
        for (int k = 0; k < KP1; ++k) {  // column site j: - 1j up, + n (b - 1j a) dn
          const double ur = __ldg(P.Yin + cu[k] + pr * TILE), ui = __ldg(P.Yin + cu[k] + pim * TILE);
          const double dr = __ldg(P.Yin + cd[k] + pr * TILE), di = __ldg(P.Yin + cd[k] + pim * TILE);
          ar += cco[k].x * dr + cco[k].y * di + ui;
          ai += cco[k].x * di - cco[k].y * dr - ur;
        }
        epilogue<STAGE>(P, tb, pr, pim, cre[i], cim[i], ar, ai, maxa2);
      }
#pragma unroll
      for (int rr = j + 1; rr < D; ++rr) {  // park X_rj (rr > j) for column rr
        lxr[(rr * (rr - 1)) / 2 + j] = xr[rr];
        lxi[(rr * (rr - 1)) / 2 + j] = xi[rr];
      }
    }
  }

  if (STAGE == 4) {
    const int lane_id = t & 31, warp = t >> 5;
    if (step_next % 25 == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
      if (lane_id == 0) s_red[warp] = maxa2;
      __syncthreads();
      if (t == 0) {
        double m = s_red[0];
        for (int w = 1; w < FT / 32; ++w) m = fmax(m, s_red[w]);
        atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                  (unsigned long long)__double_as_longlong(m));
      }
    }
    __threadfence();
    __syncthreads();
    if (t == 0) {
      const unsigned prev = atomicAdd(const_cast<unsigned*>(&ctl->blocks_done), 1u);
      s_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && (t >> 5) == 0) {
      __threadfence();
      if (t == 0) ctl->launches = ctl->launches + 4;
      finish_step_warp<D, true>(P, step_next);
    }
  }
}


// Warp-split variant: one CTA = one tile of 32 ADOs, NW warps, lane = ADO.
//   phase 0: links, lower coefficients and damping of the tile -> shared memory
//   phase 1: warp w computes the columns c = w, w+NW, ... of X = H sigma for its
//            lane's ADO (sigma column from the own tile, conj for the lower half)
//            and parks them in shared memory ([element][lane], conflict-free)
//   phase 2: warp w finishes the packed elements e = w, w+NW, ... :
//            cm_ij = X_ij - conj(X_ji), damping, 4(K+1) gathers, RK epilogue.
// Every element set is compile-time per warp (switch on the warp index), so
// planes, H operands and shared-memory offsets are immediates, and the
// per-thread live state is a column instead of a whole ADO.
constexpr int NW = 4;

template <int D, int KP1, int STAGE, int W>
__device__ __forceinline__ void split_phase1(const KParams& P, const double* own, int lane,
                                             double2 (*sX)[TILE]) {
#pragma unroll
  for (int j = W; j < D; j += NW) {
    double cre[D], cim[D];
#pragma unroll
    for (int l = 0; l < D; ++l) {
      if (l == j) {
        cre[l] = __ldg(own + l * TILE);
        cim[l] = 0.0;
      } else if (l < j) {
        cre[l] = __ldg(own + Pk<D>::re(l, j) * TILE);
        cim[l] = __ldg(own + Pk<D>::im(l, j) * TILE);
      } else {
        cre[l] = __ldg(own + Pk<D>::re(j, l) * TILE);
        cim[l] = -__ldg(own + Pk<D>::im(j, l) * TILE);
      }
    }
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double ar = 0.0, ai = 0.0;
#pragma unroll
      for (int l = 0; l < D; ++l) {
        ar += P.h[i * MAXD + l] * cre[l];
        ai += P.h[i * MAXD + l] * cim[l];
      }
      sX[i * D + j][lane] = make_double2(ar, ai);
    }
  }
}

// packed element e -> (i, j): e < D diagonal, then the upper triangle row-major
template <int D>
__host__ __device__ constexpr int elem_i(int e) {
  if (e < D) return e;
  int o = e - D, r = 0, cnt = D - 1;
  while (o >= cnt) { o -= cnt; ++r; cnt = D - 1 - r; }
  return r;
}
template <int D>
__host__ __device__ constexpr int elem_j(int e) {
  if (e < D) return e;
  int o = e - D, r = 0, cnt = D - 1;
  while (o >= cnt) { o -= cnt; ++r; cnt = D - 1 - r; }
  return r + 1 + o;
}

template <int D, int KP1, int STAGE, int W>
__device__ __forceinline__ void split_phase2(const KParams& P, size_t tb, int lane, double damp,
                                             const double2 (*sX)[TILE], const double2 (*sC)[TILE],
                                             const int (*sU)[TILE], const int (*sD)[TILE],
                                             double& maxa2) {
  constexpr int NE = D * (D + 1) / 2;
  const double* own = P.Yin + tb;
#pragma unroll
  for (int e = W; e < NE; e += NW) {
    const int i = elem_i<D>(e), j = elem_j<D>(e);
    if (i == j) {  // diagonal: 2 Im X_ii, lower terms twice, raise terms cancel
      const double sr = __ldg(own + i * TILE);
      double ar = -(damp + P.decay[i]) * sr + 2.0 * sX[i * D + i][lane].y;
#pragma unroll
      for (int k = 0; k < KP1; ++k)
        ar += 2.0 * sC[i * KP1 + k][lane].x * __ldg(P.Yin + sD[i * KP1 + k][lane] + i * TILE);
      epilogue<STAGE>(P, tb, i, -1, sr, 0.0, ar, 0.0, maxa2);
    } else {
      const int pr = Pk<D>::re(i, j), pim = Pk<D>::im(i, j);
      const double sr = __ldg(own + pr * TILE), si = __ldg(own + pim * TILE);
      const double2 xij = sX[i * D + j][lane], xji = sX[j * D + i][lane];
      const double cmr = xij.x - xji.x, cmi = xij.y + xji.y;  // X_ij - conj(X_ji)
      const double f = -(damp + 0.5 * (P.decay[i] + P.decay[j]));
      double ar = f * sr + cmi;  // acc += -1j * cm
      double ai = f * si - cmr;
#pragma unroll
      for (int k = 0; k < KP1; ++k) {  // row site i: + 1j up, + n (b + 1j a) dn
        const int ru = sU[i * KP1 + k][lane], rd = sD[i * KP1 + k][lane];
        const double2 rc = sC[i * KP1 + k][lane];
        const double ur = __ldg(P.Yin + ru + pr * TILE), ui = __ldg(P.Yin + ru + pim * TILE);
        const double dr = __ldg(P.Yin + rd + pr * TILE), di = __ldg(P.Yin + rd + pim * TILE);
        ar += rc.x * dr - rc.y * di - ui;
        ai += rc.x * di + rc.y * dr + ur;
      }
#pragma unroll
      for (int k = 0; k < KP1; ++k) {  // column site j: - 1j up, + n (b - 1j a) dn
        const int cu = sU[j * KP1 + k][lane], cd = sD[j * KP1 + k][lane];
        const double2 cc = sC[j * KP1 + k][lane];
        const double ur = __ldg(P.Yin + cu + pr * TILE), ui = __ldg(P.Yin + cu + pim * TILE);
        const double dr = __ldg(P.Yin + cd + pr * TILE), di = __ldg(P.Yin + cd + pim * TILE);
        ar += cc.x * dr + cc.y * di + ui;
        ai += cc.x * di - cc.y * dr - ur;
      }
      epilogue<STAGE>(P, tb, pr, pim, sr, si, ar, ai, maxa2);
    }
  }
}

template <int D, int KP1, int STAGE, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB) k_split(const KParams P) {
  constexpr int NP = D * D;
  constexpr int M = D * KP1;
  __shared__ double2 sX[D * D][TILE];
  __shared__ double2 sC[M][TILE];
  __shared__ int sU[M][TILE];
  __shared__ int sD[M][TILE];
  __shared__ double sDamp[TILE];
  __shared__ double s_red[NW];
  __shared__ int s_last;

  volatile Ctl* ctl = P.ctl;
  if (ctl->status != ST_RUNNING) return;
  const long long step_next = ctl->step + 1;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int tile = P.tile_begin + blockIdx.x;
  const size_t tb = (size_t)tile * NP * TILE + lane;
  const int zero_off = P.n_tiles_total * NP * TILE;
  if (t == 0 && P.prefetch) {
    prefetch_epilogue<STAGE>(P, (size_t)tile * NP * TILE, NP * TILE * sizeof(double));
    if (P.pf_dist > 0) prefetch_tile<STAGE>(P, tile + P.pf_dist);
  }

  // phase 0: links and coefficients of the tile (coalesced [tile][mode][32])
  const size_t gb = (size_t)tile * M * TILE;
  for (int idx = t; idx < M * TILE; idx += NW * 32) {
    const int m = idx >> 5, l = idx & 31;
    const int up = __ldg(P.plus + gb + idx);
    const int dn = __ldg(P.minus + gb + idx);
    const double nd = (double)__ldg(P.nvec + gb + idx);
    sC[m][l] = make_double2(nd * P.b[m % KP1], nd * P.a[m % KP1]);
    sU[m][l] = up >= 0 && !P.debug ? (up >> 5) * NP * TILE + (up & 31) : zero_off;
    sD[m][l] = dn >= 0 && !P.debug ? (dn >> 5) * NP * TILE + (dn & 31) : zero_off;
  }
  if (warp == 0) {  // heom.py:275, generalised: sum_k nu_k * sum_j n_jk
    double damp = 0.0;
#pragma unroll
    for (int k = 0; k < KP1; ++k) {
      int tk = 0;
#pragma unroll
      for (int jj = 0; jj < D; ++jj) tk += __ldg(P.nvec + gb + (jj * KP1 + k) * TILE + lane);
      damp += (double)tk * P.nu[k];
    }
    sDamp[lane] = damp;
    if (tile == 0 && lane == 0) {  // sink rates of this stage input (heom.py:282-283)
      int q = 0;
      for (int sk = 0; sk < P.n_sinks; ++sk) {
        double acc = 0.0;
        for (int cc = 0; cc < P.sink_nterms[sk]; ++cc, ++q) {
          const double v = P.sink_rate[q] * __ldg(P.Yin + P.sink_pos[q] * TILE);
          acc = cc == 0 ? v : acc + v;
        }
        ctl->r[STAGE - 1][sk] = acc;
      }
    }
  }
  // phase 1: columns of X = H sigma
  const double* own = P.Yin + tb;
  switch (warp) {
    case 0: split_phase1<D, KP1, STAGE, 0>(P, own, lane, sX); break;
    case 1: split_phase1<D, KP1, STAGE, 1>(P, own, lane, sX); break;
    case 2: split_phase1<D, KP1, STAGE, 2>(P, own, lane, sX); break;
    default: split_phase1<D, KP1, STAGE, 3>(P, own, lane, sX); break;
  }
  __syncthreads();
  // phase 2: packed elements
  double maxa2 = 0.0;
  const double damp = sDamp[lane];
  switch (warp) {
    case 0: split_phase2<D, KP1, STAGE, 0>(P, tb, lane, damp, sX, sC, sU, sD, maxa2); break;
    case 1: split_phase2<D, KP1, STAGE, 1>(P, tb, lane, damp, sX, sC, sU, sD, maxa2); break;
    case 2: split_phase2<D, KP1, STAGE, 2>(P, tb, lane, damp, sX, sC, sU, sD, maxa2); break;
    default: split_phase2<D, KP1, STAGE, 3>(P, tb, lane, damp, sX, sC, sU, sD, maxa2); break;
  }

  if (STAGE == 4) {
    if (step_next % 25 == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
      if (lane == 0) s_red[warp] = maxa2;
      __syncthreads();
      if (t == 0) {
        double m = s_red[0];
        for (int w = 1; w < NW; ++w) m = fmax(m, s_red[w]);
        atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                  (unsigned long long)__double_as_longlong(m));
      }
    }
    __threadfence();
    __syncthreads();
    if (t == 0) {
      const unsigned prev = atomicAdd(const_cast<unsigned*>(&ctl->blocks_done), 1u);
      s_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && (t >> 5) == 0) {
      __threadfence();
      if (t == 0) ctl->launches = ctl->launches + 4;
      finish_step_warp<D, true>(P, step_next);
    }
  }
}


// ---------------------------------------------------------------------------
// TMA variant (default): the tile's streamed operands -- own stage input, the
// epilogue operands (sigma; Y2, Y3 at stage 4) and the three link tables --
// are fetched with cp.async.bulk into shared memory behind one mbarrier, so
// all streamed bytes of a CTA are in flight at once without holding registers
// (the register-fed variants above stay latency bound at ~3 TB/s).  Compute is
// the warp-split scheme (X = H sigma columns in shared memory, compile-time
// element sets per warp); only the neighbour gathers remain LDGs.

template <int D, int KP1, int STAGE>
struct TmaLayout {
  static constexpr int NP = D * D, M = D * KP1, TB = NP * TILE;
  static constexpr int NOPS = STAGE == 4 ? 3 : (STAGE >= 2 ? 1 : 0);
  static constexpr size_t OWN = 0;
  static constexpr size_t OPS = OWN + (size_t)TB * 8;
  static constexpr size_t UP = OPS + (size_t)NOPS * TB * 8;
  static constexpr size_t DN = UP + (size_t)M * TILE * 4;
  static constexpr size_t NV = DN + (size_t)M * TILE * 4;
  static constexpr size_t X = (NV + (size_t)M * TILE + 15) & ~(size_t)15;
  static constexpr size_t BYTES = X + (size_t)NP * TILE * 16;
  static constexpr unsigned TX = (unsigned)(NV + (size_t)M * TILE);  // bytes delivered by TMA
};

template <int D, int KP1, int STAGE, int W, int TNW>
__device__ __forceinline__ void tma_phase1(const KParams& P, const double* sOwn, int lane,
                                           double2* sX) {
#pragma unroll
  for (int j = W; j < D; j += TNW) {
    double cre[D], cim[D];
#pragma unroll
    for (int l = 0; l < D; ++l) {
      if (l == j) {
        cre[l] = sOwn[l * TILE + lane];
        cim[l] = 0.0;
      } else if (l < j) {
        cre[l] = sOwn[Pk<D>::re(l, j) * TILE + lane];
        cim[l] = sOwn[Pk<D>::im(l, j) * TILE + lane];
      } else {
        cre[l] = sOwn[Pk<D>::re(j, l) * TILE + lane];
        cim[l] = -sOwn[Pk<D>::im(j, l) * TILE + lane];
      }
    }
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double ar = 0.0, ai = 0.0;
#pragma unroll
      for (int l = 0; l < D; ++l) {
        ar += P.h[i * MAXD + l] * cre[l];
        ai += P.h[i * MAXD + l] * cim[l];
      }
      sX[(i * D + j) * TILE + lane] = make_double2(ar, ai);
    }
  }
}

template <int STAGE>
__device__ __forceinline__ void tma_epilogue(const KParams& P, size_t tb, const double* sOps,
                                             int lane, int pr, int pim, double sr, double si,
                                             double ar, double ai, double& maxa2) {
  constexpr int TBQ = 0;  // operand stride is passed through sOps layout below
  (void)TBQ;
  double yr, yi = 0.0;
  if (STAGE == 1) {
    yr = sr + P.coef * ar;
    yi = si + P.coef * ai;
  } else if (STAGE == 2 || STAGE == 3) {
    const double gr = sOps[pr * TILE + lane];
    const double gi = pim >= 0 ? sOps[pim * TILE + lane] : 0.0;
    yr = gr + P.coef * ar;
    yi = gi + P.coef * ai;
  } else {
    const int TB = P.n_planes * TILE;
    const double gr = sOps[pr * TILE + lane];
    const double y2r = sOps[TB + pr * TILE + lane], y3r = sOps[2 * TB + pr * TILE + lane];
    const double w = P.dt / 6.0, third = 1.0 / 3.0;
    yr = gr + ((y2r - gr) + 2.0 * (y3r - gr) + (sr - gr)) * third + w * ar;
    if (pim >= 0) {
      const double gi = sOps[pim * TILE + lane];
      const double y2i = sOps[TB + pim * TILE + lane], y3i = sOps[2 * TB + pim * TILE + lane];
      yi = gi + ((y2i - gi) + 2.0 * (y3i - gi) + (si - gi)) * third + w * ai;
    }
    maxa2 = fmax(maxa2, yr * yr + yi * yi);
  }
  P.Yout[tb + pr * TILE] = yr;
  if (pim >= 0) P.Yout[tb + pim * TILE] = yi;
}

template <int D, int KP1, int STAGE, int W, int TNW>
__device__ __forceinline__ void tma_phase2(const KParams& P, size_t tb, int lane, double damp,
                                           const double* sOwn, const double* sOps,
                                           const double2* sX, const int* sUp, const int* sDn,
                                           const uint8_t* sNv, double& maxa2) {
  constexpr int NE = D * (D + 1) / 2;
#pragma unroll
  for (int e = W; e < NE; e += TNW) {
    const int i = elem_i<D>(e), j = elem_j<D>(e);
    if (i == j) {  // diagonal: 2 Im X_ii, lower terms twice, raise terms cancel
      const double sr = sOwn[i * TILE + lane];
      double ar = -(damp + P.decay[i]) * sr + 2.0 * sX[(i * D + i) * TILE + lane].y;
#pragma unroll
      for (int k = 0; k < KP1; ++k) {
        const int m = i * KP1 + k;
        const double cb = (double)sNv[m * TILE + lane] * P.b[k];
        ar += 2.0 * cb * __ldg(P.Yin + sDn[m * TILE + lane] + i * TILE);
      }
      tma_epilogue<STAGE>(P, tb, sOps, lane, i, -1, sr, 0.0, ar, 0.0, maxa2);
    } else {
      const int pr = Pk<D>::re(i, j), pim = Pk<D>::im(i, j);
      const double sr = sOwn[pr * TILE + lane], si = sOwn[pim * TILE + lane];
      const double2 xij = sX[(i * D + j) * TILE + lane], xji = sX[(j * D + i) * TILE + lane];
      const double cmr = xij.x - xji.x, cmi = xij.y + xji.y;  // X_ij - conj(X_ji)
      const double f = -(damp + 0.5 * (P.decay[i] + P.decay[j]));
      double ar = f * sr + cmi;  // acc += -1j * cm
      double ai = f * si - cmr;
#pragma unroll
      for (int k = 0; k < KP1; ++k) {  // row site i: + 1j up, + n (b + 1j a) dn
        const int m = i * KP1 + k;
        const int ru = sUp[m * TILE + lane], rd = sDn[m * TILE + lane];
        const double n = (double)sNv[m * TILE + lane];
        const double cb = n * P.b[k], ca = n * P.a[k];
        const double ur = __ldg(P.Yin + ru + pr * TILE), ui = __ldg(P.Yin + ru + pim * TILE);
        const double dr = __ldg(P.Yin + rd + pr * TILE), di = __ldg(P.Yin + rd + pim * TILE);
        ar += cb * dr - ca * di - ui;
        ai += cb * di + ca * dr + ur;
      }
#pragma unroll
      for (int k = 0; k < KP1; ++k) {  // column site j: - 1j up, + n (b - 1j a) dn
        const int m = j * KP1 + k;
        const int cu = sUp[m * TILE + lane], cd = sDn[m * TILE + lane];
        const double n = (double)sNv[m * TILE + lane];
        const double cb = n * P.b[k], ca = n * P.a[k];
        const double ur = __ldg(P.Yin + cu + pr * TILE), ui = __ldg(P.Yin + cu + pim * TILE);
        const double dr = __ldg(P.Yin + cd + pr * TILE), di = __ldg(P.Yin + cd + pim * TILE);
        ar += cb * dr + ca * di + ui;
        ai += cb * di - ca * dr - ur;
      }
      tma_epilogue<STAGE>(P, tb, sOps, lane, pr, pim, sr, si, ar, ai, maxa2);
    }
  }
}

// compile-time warp index: calls f(integral_constant<W>) for the runtime warp
template <int W, int TNW, class F>
__device__ __forceinline__ void warp_switch(int warp, F&& f) {
  if constexpr (W < TNW) {
    if (warp == W) f(std::integral_constant<int, W>{});
    else warp_switch<W + 1, TNW>(warp, f);
  }
}

template <int D, int KP1, int STAGE, int TNW>
__global__ void __launch_bounds__(TNW * 32) k_tma(const KParams P) {
  using L = TmaLayout<D, KP1, STAGE>;
  constexpr int NP = L::NP, M = L::M, TB = L::TB;
  extern __shared__ __align__(128) unsigned char smem[];
  double* sOwn = reinterpret_cast<double*>(smem + L::OWN);
  double* sOps = reinterpret_cast<double*>(smem + L::OPS);
  int* sUp = reinterpret_cast<int*>(smem + L::UP);
  int* sDn = reinterpret_cast<int*>(smem + L::DN);
  uint8_t* sNv = smem + L::NV;
  double2* sX = reinterpret_cast<double2*>(smem + L::X);
  __shared__ __align__(8) uint64_t bar;
  __shared__ double sDamp[TILE];
  __shared__ double s_red[TNW];
  __shared__ int s_last;

  volatile Ctl* ctl = P.ctl;
  if (ctl->status != ST_RUNNING) return;
  const long long step_next = ctl->step + 1;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int tile = P.tile_begin + blockIdx.x;
  const size_t toff = (size_t)tile * TB;
  const size_t goff = (size_t)tile * M * TILE;

  if (t == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, L::TX);
    bulk_g2s(sOwn, P.Yin + toff, TB * 8, &bar);
    if (L::NOPS >= 1) bulk_g2s(sOps, P.sig + toff, TB * 8, &bar);
    if (L::NOPS == 3) {
      bulk_g2s(sOps + TB, P.Y2 + toff, TB * 8, &bar);
      bulk_g2s(sOps + 2 * TB, P.Y3 + toff, TB * 8, &bar);
    }
    bulk_g2s(sUp, P.plus + goff, M * TILE * 4, &bar);
    bulk_g2s(sDn, P.minus + goff, M * TILE * 4, &bar);
    bulk_g2s(sNv, P.nvec + goff, M * TILE, &bar);
  }
  __syncthreads();  // barrier initialised before anyone waits on it
  mbar_wait(&bar, 0);

  // phase 0: links -> element offsets (absent -> zero tile), damping, sink rates
  const int zero_off = P.n_tiles_total * TB;
  for (int idx = t; idx < M * TILE; idx += TNW * 32) {
    const int up = sUp[idx], dn = sDn[idx];
    sUp[idx] = up >= 0 && !P.debug ? (up >> 5) * TB + (up & 31) : zero_off;
    sDn[idx] = dn >= 0 && !P.debug ? (dn >> 5) * TB + (dn & 31) : zero_off;
  }
  if (warp == 0) {  // heom.py:275, generalised: sum_k nu_k * sum_j n_jk
    double damp = 0.0;
#pragma unroll
    for (int k = 0; k < KP1; ++k) {
      int tk = 0;
#pragma unroll
      for (int jj = 0; jj < D; ++jj) tk += sNv[(jj * KP1 + k) * TILE + lane];
      damp += (double)tk * P.nu[k];
    }
    sDamp[lane] = damp;
    if (tile == 0 && lane == 0) {  // sink rates of this stage input (heom.py:282-283)
      int q = 0;
      for (int sk = 0; sk < P.n_sinks; ++sk) {
        double acc = 0.0;
        for (int cc = 0; cc < P.sink_nterms[sk]; ++cc, ++q) {
          const double v = P.sink_rate[q] * sOwn[P.sink_pos[q] * TILE];
          acc = cc == 0 ? v : acc + v;
        }
        ctl->r[STAGE - 1][sk] = acc;
      }
    }
  }
  // phase 1: columns of X = H sigma (reads only sOwn)
  warp_switch<0, TNW>(warp, [&](auto wc) {
    tma_phase1<D, KP1, STAGE, decltype(wc)::value, TNW>(P, sOwn, lane, sX);
  });
  __syncthreads();
  double maxa2 = 0.0;
  const double damp = sDamp[lane];
  const size_t tb = toff + lane;
  warp_switch<0, TNW>(warp, [&](auto wc) {
    tma_phase2<D, KP1, STAGE, decltype(wc)::value, TNW>(P, tb, lane, damp, sOwn, sOps, sX, sUp,
                                                        sDn, sNv, maxa2);
  });

  if (STAGE == 4) {
    if (step_next % 25 == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
      if (lane == 0) s_red[warp] = maxa2;
      __syncthreads();
      if (t == 0) {
        double m = s_red[0];
        for (int w = 1; w < TNW; ++w) m = fmax(m, s_red[w]);
        atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                  (unsigned long long)__double_as_longlong(m));
      }
    }
    __threadfence();
    __syncthreads();
    if (t == 0) {
      const unsigned prev = atomicAdd(const_cast<unsigned*>(&ctl->blocks_done), 1u);
      s_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && (t >> 5) == 0) {
      __threadfence();
      if (t == 0) ctl->launches = ctl->launches + 4;
      finish_step_warp<D, true>(P, step_next);
    }
  }
}

template <int D, int KP1, int TNW>
static cudaError_t tma_configure_nw() {
  cudaError_t e = cudaFuncSetAttribute(k_tma<D, KP1, 1, TNW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)TmaLayout<D, KP1, 1>::BYTES);
  if (!e) e = cudaFuncSetAttribute(k_tma<D, KP1, 2, TNW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)TmaLayout<D, KP1, 2>::BYTES);
  if (!e) e = cudaFuncSetAttribute(k_tma<D, KP1, 3, TNW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)TmaLayout<D, KP1, 3>::BYTES);
  if (!e) e = cudaFuncSetAttribute(k_tma<D, KP1, 4, TNW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)TmaLayout<D, KP1, 4>::BYTES);
  return e;
}

// warps per tile of the TMA kernel (HB_TMA_NW in {4, 8, 16}; experiments)
static int tma_nw() {
  static int v = [] {
    const char* e = getenv("HB_TMA_NW");
    const int n = e ? atoi(e) : 8;
    return (n == 4 || n == 16) ? n : 8;
  }();
  return v;
}

template <int D, int KP1>
static cudaError_t tma_configure() {
  if constexpr (D == 7) {
    switch (tma_nw()) {
      case 4: return tma_configure_nw<D, KP1, 4>();
      case 16: return tma_configure_nw<D, KP1, 16>();
      default: return tma_configure_nw<D, KP1, 8>();
    }
  }
  return cudaSuccess;  // only d = 7 instantiates the TMA variant
}

template <int D, int KP1, int TNW>
static cudaError_t tma_launch(int stage, const KParams& p, cudaStream_t s) {
  switch (stage) {
    case 1: k_tma<D, KP1, 1, TNW><<<p.n_tiles, TNW * 32, TmaLayout<D, KP1, 1>::BYTES, s>>>(p); break;
    case 2: k_tma<D, KP1, 2, TNW><<<p.n_tiles, TNW * 32, TmaLayout<D, KP1, 2>::BYTES, s>>>(p); break;
    case 3: k_tma<D, KP1, 3, TNW><<<p.n_tiles, TNW * 32, TmaLayout<D, KP1, 3>::BYTES, s>>>(p); break;
    case 4: k_tma<D, KP1, 4, TNW><<<p.n_tiles, TNW * 32, TmaLayout<D, KP1, 4>::BYTES, s>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <int D>
static cudaError_t tma_configure_d(int kp1) {
  return kp1 == 1 ? tma_configure<D, 1>() : tma_configure<D, 2>();
}

cudaError_t configure_fast(const KParams& p) {
  switch (p.d) {
    case 1: return tma_configure_d<1>(p.kp1);
    case 2: return tma_configure_d<2>(p.kp1);
    case 3: return tma_configure_d<3>(p.kp1);
    case 4: return tma_configure_d<4>(p.kp1);
    case 5: return tma_configure_d<5>(p.kp1);
    case 6: return tma_configure_d<6>(p.kp1);
    case 7: return tma_configure_d<7>(p.kp1);
    case 8: return tma_configure_d<8>(p.kp1);
  }
  return cudaErrorInvalidValue;
}


// ---------------------------------------------------------------------------
// Mode-major variant: per warp one tile (lane = ADO).
//   A: damping + commutator from the ADO held in registers -> accumulator in
//      shared memory ([plane][lane], the packed layout of the state);
//   B: for each site s, all 2(K+1) link crosses of s are gathered at once (13
//      elements each, independent loads, nothing else live), summed in
//      registers and added to the accumulator with one read-modify-write per
//      cross element -- the gathers of a site are all in flight together
//      instead of one element at a time;
//   C: RK epilogue from the accumulator (epilogue tiles were bulk-prefetched
//      into L2 at kernel start).
// Per-element term order equals the reference's (row site before column site,
// raise before lower for each k); only the grouping of the additions differs.
template <int D, int KP1, int STAGE, int MM_WPC, int MINB>
__global__ void __launch_bounds__(MM_WPC * 32, MINB) k_mm(const KParams P) {
  constexpr int NP = D * D;
  constexpr int M = D * KP1;
  constexpr int TB = NP * TILE;
  __shared__ double sAcc[MM_WPC][NP][TILE];
  __shared__ int sU[MM_WPC][M][TILE];
  __shared__ int sD[MM_WPC][M][TILE];
  __shared__ unsigned char sN[MM_WPC][M][TILE];
  __shared__ double s_red[MM_WPC];
  __shared__ int s_last;

  volatile Ctl* ctl = P.ctl;
  if (ctl->status != ST_RUNNING) return;
  const long long step_next = ctl->step + 1;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int local_tile = blockIdx.x * MM_WPC + w;
  const bool active = local_tile < P.n_tiles;
  const int tile = P.tile_begin + local_tile;
  double maxa2 = 0.0;

  if (active) {
    const size_t toff = (size_t)tile * TB;
    if (lane == 0 && P.prefetch) prefetch_epilogue<STAGE>(P, toff, TB * sizeof(double));
    const size_t tb = toff + lane;
    double (*acc)[TILE] = sAcc[w];
    // ---- links, n, damping
    const int zero_off = P.n_tiles_total * TB;
    const size_t gb = (size_t)tile * M * TILE + lane;
    int tk[KP1];
#pragma unroll
    for (int k = 0; k < KP1; ++k) tk[k] = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int up = __ldg(P.plus + gb + m * TILE);
      const int dn = __ldg(P.minus + gb + m * TILE);
      const int n = __ldg(P.nvec + gb + m * TILE);
      tk[m % KP1] += n;
      sU[w][m][lane] = up >= 0 && !P.debug ? (up >> 5) * TB + (up & 31) : zero_off;
      sD[w][m][lane] = dn >= 0 && !P.debug ? (dn >> 5) * TB + (dn & 31) : zero_off;
      sN[w][m][lane] = (unsigned char)n;
    }
    double damp = 0.0;  // heom.py:275, generalised: sum_k nu_k * sum_j n_jk
#pragma unroll
    for (int k = 0; k < KP1; ++k) damp += (double)tk[k] * P.nu[k];

    {  // ---- phase A: damping + commutator, ADO in registers
      double s[NP];
#pragma unroll
      for (int p = 0; p < NP; ++p) s[p] = __ldg(P.Yin + tb + p * TILE);
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
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double cm_im = 0.0;
#pragma unroll
        for (int l = 0; l < D; ++l)
          if (l != i) cm_im += P.h[i * MAXD + l] * sim<D>(s, i, l);
        acc[i][lane] = -(damp + P.decay[i]) * s[i] - 2.0 * cm_im;
#pragma unroll
        for (int j = i + 1; j < D; ++j) {
          const int pr = Pk<D>::re(i, j), pim = Pk<D>::im(i, j);
          const double f = -(damp + 0.5 * (P.decay[i] + P.decay[j]));
          double cr = 0.0, ci = 0.0;
#pragma unroll
          for (int l = 0; l < D; ++l) {
            const double hil = P.h[i * MAXD + l], hlj = P.h[l * MAXD + j];
            cr += hil * sre<D>(s, l, j) - sre<D>(s, i, l) * hlj;
            ci += hil * sim<D>(s, l, j) - sim<D>(s, i, l) * hlj;
          }
          acc[pr][lane] = f * s[pr] + ci;  // acc += -1j * cm
          acc[pim][lane] = f * s[pim] - cr;
        }
      }
    }
    __syncwarp();
    // ---- phase B: neighbour crosses, one site at a time
#pragma unroll
    for (int st = 0; st < D; ++st) {
      double cre[D], cim[D];
#pragma unroll
      for (int o = 0; o < D; ++o) cre[o] = cim[o] = 0.0;
#pragma unroll
      for (int k = 0; k < KP1; ++k) {
        const int m = st * KP1 + k;
        const double* up = P.Yin + sU[w][m][lane];
        const double* dn = P.Yin + sD[w][m][lane];
        const double n = (double)sN[w][m][lane];
        const double cb = n * P.b[k], ca = n * P.a[k];
        cre[st] += 2.0 * cb * __ldg(dn + st * TILE);  // diagonal: lower terms twice
#pragma unroll
        for (int o = 0; o < D; ++o) {
          if (o == st) continue;
          const int a = st < o ? st : o, b = st < o ? o : st;
          const int pr = Pk<D>::re(a, b), pim = Pk<D>::im(a, b);
          const double ur = __ldg(up + pr * TILE), ui = __ldg(up + pim * TILE);
          const double dr = __ldg(dn + pr * TILE), di = __ldg(dn + pim * TILE);
          if (o > st) {  // element (st, o): st is its row site
            cre[o] += cb * dr - ca * di - ui;
            cim[o] += cb * di + ca * dr + ur;
          } else {       // element (o, st): st is its column site
            cre[o] += cb * dr + ca * di + ui;
            cim[o] += cb * di - ca * dr - ur;
          }
        }
      }
      acc[st][lane] += cre[st];
#pragma unroll
      for (int o = 0; o < D; ++o) {
        if (o == st) continue;
        const int a = st < o ? st : o, b = st < o ? o : st;
        acc[Pk<D>::re(a, b)][lane] += cre[o];
        acc[Pk<D>::im(a, b)][lane] += cim[o];
      }
    }
    __syncwarp();
    // ---- phase C: RK epilogue
    const double* own = P.Yin + tb;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      epilogue<STAGE>(P, tb, i, -1, STAGE == 1 || STAGE == 4 ? __ldg(own + i * TILE) : 0.0, 0.0,
                      acc[i][lane], 0.0, maxa2);
#pragma unroll
      for (int j = i + 1; j < D; ++j) {
        const int pr = Pk<D>::re(i, j), pim = Pk<D>::im(i, j);
        const double sr = STAGE == 1 || STAGE == 4 ? __ldg(own + pr * TILE) : 0.0;
        const double si = STAGE == 1 || STAGE == 4 ? __ldg(own + pim * TILE) : 0.0;
        epilogue<STAGE>(P, tb, pr, pim, sr, si, acc[pr][lane], acc[pim][lane], maxa2);
      }
    }
  }

  if (STAGE == 4) {
    if (step_next % 25 == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
      if (lane == 0) s_red[w] = maxa2;
      __syncthreads();
      if (t == 0) {
        double m = s_red[0];
        for (int q = 1; q < MM_WPC; ++q) m = fmax(m, s_red[q]);
        atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                  (unsigned long long)__double_as_longlong(m));
      }
    }
    __threadfence();
    __syncthreads();
    if (t == 0) {
      const unsigned prev = atomicAdd(const_cast<unsigned*>(&ctl->blocks_done), 1u);
      s_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && w == 0) {
      __threadfence();
      if (t == 0) ctl->launches = ctl->launches + 4;
      finish_step_warp<D, true>(P, step_next);
    }
  }
}

template <int D, int KP1, int WPC, int MINB>
static cudaError_t mm_launch_w(int stage, const KParams& p, cudaStream_t s) {
  const int grid = (p.n_tiles + WPC - 1) / WPC;
  switch (stage) {
    case 1: k_mm<D, KP1, 1, WPC, MINB><<<grid, WPC * 32, 0, s>>>(p); break;
    case 2: k_mm<D, KP1, 2, WPC, MINB><<<grid, WPC * 32, 0, s>>>(p); break;
    case 3: k_mm<D, KP1, 3, WPC, MINB><<<grid, WPC * 32, 0, s>>>(p); break;
    case 4: k_mm<D, KP1, 4, WPC, MINB><<<grid, WPC * 32, 0, s>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// HB_MM_CFG (experiments): 1 = 1 warp/CTA (default, fastest measured), 0 = 2 warps,
// 3 = 2 warps capped at 128 registers
static int mm_cfg() {
  static int v = [] {
    const char* e = getenv("HB_MM_CFG");
    return e ? atoi(e) : 1;
  }();
  return v;
}

template <int D, int KP1>
static cudaError_t mm_launch(int stage, const KParams& p, cudaStream_t s) {
  switch (mm_cfg()) {
    case 1: return mm_launch_w<D, KP1, 1, 1>(stage, p, s);
    case 3: return mm_launch_w<D, KP1, 2, 8>(stage, p, s);
    default: return mm_launch_w<D, KP1, 2, 1>(stage, p, s);
  }
}


// ---------------------------------------------------------------------------
// Production kernel (variant 5): mode-major + the RK base tile delivered by TMA.
// The stage epilogue needs one base tile per ADO besides its own input; it is
// bulk-copied (cp.async.bulk, one mbarrier) straight into the shared-memory
// accumulator at kernel start, so phase A starts from acc = base and every
// contribution is added pre-scaled by the stage coefficient:
//   stage 1: Y2 = s + h/2 k1          base = s (own input, from registers)
//   stage 2: Y3 = s + h/2 k2          base = s;  also B = (Y2 - s)/3 + 2/3 Y3
//   stage 3: Y4 = s + h k3            base = s
//   stage 4: s  = B + Y4/3 + h/6 k4   base = B
// B + Y4/3 = (Y2 + 2Y3 - s + Y4)/3, so s_new = s + h/6 (k1 + 2k2 + 2k3 + k4)
// (heom.py:381).  B is formed where Y2 is the thread's own input, so the
// scheme moves 12 state passes per step (2 + 4 + 3 + 3) and no epilogue waits
// on a load.
template <int D, int KP1, int STAGE, int MINB>
__global__ void __launch_bounds__(32, MINB) k_mm2(const KParams P) {
  constexpr int NP = D * D;
  constexpr int M = D * KP1;
  constexpr int TB = NP * TILE;
  constexpr bool kE1 = STAGE == 2;  // stage 2 parks (Y2 - s)/3 for B
  __shared__ __align__(128) double sAcc[NP][TILE];
  __shared__ __align__(128) double sE1[kE1 ? NP : 1][TILE];
  __shared__ int sU[M][TILE];
  __shared__ int sD[M][TILE];
  __shared__ unsigned char sN[M][TILE];
  __shared__ __align__(8) uint64_t bar;

  volatile Ctl* ctl = P.ctl;
  if (ctl->status != ST_RUNNING) return;
  const long long step_next = ctl->step + 1;
  const int lane = threadIdx.x;
  const int tile = P.tile_begin + blockIdx.x;
  const size_t toff = (size_t)tile * TB;
  const size_t tb = toff + lane;
  double maxa2 = 0.0;
  // RK coefficient of this stage's right-hand side
  const double c = STAGE == 4 ? P.dt / 6.0 : P.coef;

  if (STAGE >= 2 && lane == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, TB * 8u);
    bulk_g2s(&sAcc[0][0], (STAGE == 4 ? P.Bbuf : P.sig) + toff, TB * 8, &bar);
  }
  __syncwarp();  // barrier initialised before any lane waits on it
  // ---- links, n, damping
  const int zero_off = P.n_tiles_total * TB;
  const size_t gb = (size_t)tile * M * TILE + lane;
  int tk[KP1];
#pragma unroll
  for (int k = 0; k < KP1; ++k) tk[k] = 0;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int up = __ldg(P.plus + gb + m * TILE);
    const int dn = __ldg(P.minus + gb + m * TILE);
    const int n = __ldg(P.nvec + gb + m * TILE);
    tk[m % KP1] += n;
    sU[m][lane] = up >= 0 && !P.debug ? (up >> 5) * TB + (up & 31) : zero_off;
    sD[m][lane] = dn >= 0 && !P.debug ? (dn >> 5) * TB + (dn & 31) : zero_off;
    sN[m][lane] = (unsigned char)n;
  }
  double damp = 0.0;  // heom.py:275, generalised: sum_k nu_k * sum_j n_jk
#pragma unroll
  for (int k = 0; k < KP1; ++k) damp += (double)tk[k] * P.nu[k];

  {  // ---- phase A: damping + commutator from the ADO in registers
    double s[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) s[p] = __ldg(P.Yin + tb + p * TILE);
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
    if (STAGE >= 2) mbar_wait(&bar, 0);
    // base of plane p: own input (stage 1), sigma (2, 3), B + Y4/3 (4)
    auto base = [&](int p) -> double {
      if (STAGE == 1) return s[p];
      if (STAGE == 4) return sAcc[p][lane] + s[p] * (1.0 / 3.0);
      return sAcc[p][lane];
    };
    auto emit_b = [&](int p) {  // stage 2: park (Y2 - s)/3 (own input minus base)
      if (STAGE == 2) sE1[p][lane] = (s[p] - sAcc[p][lane]) * (1.0 / 3.0);
    };
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double cm_im = 0.0;
#pragma unroll
      for (int l = 0; l < D; ++l)
        if (l != i) cm_im += P.h[i * MAXD + l] * sim<D>(s, i, l);
      emit_b(i);
      sAcc[i][lane] = base(i) + c * (-(damp + P.decay[i]) * s[i] - 2.0 * cm_im);
#pragma unroll
      for (int j = i + 1; j < D; ++j) {
        const int pr = Pk<D>::re(i, j), pim = Pk<D>::im(i, j);
        const double f = -(damp + 0.5 * (P.decay[i] + P.decay[j]));
        double cr = 0.0, ci = 0.0;
#pragma unroll
        for (int l = 0; l < D; ++l) {
          const double hil = P.h[i * MAXD + l], hlj = P.h[l * MAXD + j];
          cr += hil * sre<D>(s, l, j) - sre<D>(s, i, l) * hlj;
          ci += hil * sim<D>(s, l, j) - sim<D>(s, i, l) * hlj;
        }
        emit_b(pr);
        emit_b(pim);
        sAcc[pr][lane] = base(pr) + c * (f * s[pr] + ci);  // -1j * cm
        sAcc[pim][lane] = base(pim) + c * (f * s[pim] - cr);
      }
    }
  }
  __syncwarp();
  // ---- phase B: neighbour crosses, one site at a time, added pre-scaled by c
#pragma unroll
  for (int st = 0; st < D; ++st) {
    double cre[D], cim[D];
#pragma unroll
    for (int o = 0; o < D; ++o) cre[o] = cim[o] = 0.0;
#pragma unroll
    for (int k = 0; k < KP1; ++k) {
      const int m = st * KP1 + k;
      const double* up = P.Yin + sU[m][lane];
      const double* dn = P.Yin + sD[m][lane];
      const double n = (double)sN[m][lane];
      const double cb = n * P.b[k], ca = n * P.a[k];
      cre[st] += 2.0 * cb * __ldg(dn + st * TILE);
#pragma unroll
      for (int o = 0; o < D; ++o) {
        if (o == st) continue;
        const int a = st < o ? st : o, b = st < o ? o : st;
        const int pr = Pk<D>::re(a, b), pim = Pk<D>::im(a, b);
        const double ur = __ldg(up + pr * TILE), ui = __ldg(up + pim * TILE);
        const double dr = __ldg(dn + pr * TILE), di = __ldg(dn + pim * TILE);
        if (o > st) {
          cre[o] += cb * dr - ca * di - ui;
          cim[o] += cb * di + ca * dr + ur;
        } else {
          cre[o] += cb * dr + ca * di + ui;
          cim[o] += cb * di - ca * dr - ur;
        }
      }
    }
    sAcc[st][lane] += c * cre[st];
#pragma unroll
    for (int o = 0; o < D; ++o) {
      if (o == st) continue;
      const int a = st < o ? st : o, b = st < o ? o : st;
      sAcc[Pk<D>::re(a, b)][lane] += c * cre[o];
      sAcc[Pk<D>::im(a, b)][lane] += c * cim[o];
    }
  }
  __syncwarp();
  // ---- phase C: store (stage 2 also B = (Y2 - s)/3 + 2/3 Y3)
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const double y = sAcc[p][lane];
    P.Yout[tb + p * TILE] = y;
    if (STAGE == 2) P.Bbuf[tb + p * TILE] = sE1[p][lane] + (2.0 / 3.0) * y;
    if (STAGE == 4) maxa2 = fmax(maxa2, y * y);
  }
  if (STAGE == 4) {
    // |y|^2 per element: diagonal planes are real; an off-diagonal pair adds up
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = i + 1; j < D; ++j) {
        const double yr = sAcc[Pk<D>::re(i, j)][lane], yi = sAcc[Pk<D>::im(i, j)][lane];
        maxa2 = fmax(maxa2, yr * yr + yi * yi);
      }
    __shared__ int s_last;
    if (step_next % 25 == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
      if (lane == 0)
        atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                  (unsigned long long)__double_as_longlong(maxa2));
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) {
      const unsigned prev = atomicAdd(const_cast<unsigned*>(&ctl->blocks_done), 1u);
      s_last = prev == gridDim.x - 1;
    }
    __syncwarp();
    if (s_last) {
      __threadfence();
      if (lane == 0) ctl->launches = ctl->launches + 4;
      finish_step_warp<D, true>(P, step_next);
    }
  }
}

template <int D, int KP1, int MINB>
static cudaError_t mm2_launch_b(int stage, const KParams& p, cudaStream_t s) {
  switch (stage) {
    case 1: k_mm2<D, KP1, 1, MINB><<<p.n_tiles, 32, 0, s>>>(p); break;
    case 2: k_mm2<D, KP1, 2, MINB><<<p.n_tiles, 32, 0, s>>>(p); break;
    case 3: k_mm2<D, KP1, 3, MINB><<<p.n_tiles, 32, 0, s>>>(p); break;
    case 4: k_mm2<D, KP1, 4, MINB><<<p.n_tiles, 32, 0, s>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// HB_MM2_MINB (experiments): register cap via min resident warps per SM
static int mm2_minb() {
  static int v = [] {
    const char* e = getenv("HB_MM2_MINB");
    return e ? atoi(e) : 1;
  }();
  return v;
}

template <int D, int KP1>
static cudaError_t mm2_launch(int stage, const KParams& p, cudaStream_t s) {
  if constexpr (D == 7) {
    switch (mm2_minb()) {
      case 10: return mm2_launch_b<D, KP1, 10>(stage, p, s);
      case 12: return mm2_launch_b<D, KP1, 12>(stage, p, s);
      case 16: return mm2_launch_b<D, KP1, 16>(stage, p, s);
      default: break;
    }
  }
  return mm2_launch_b<D, KP1, 1>(stage, p, s);
}

// ---------------------------------------------------------------------------
// Production kernel (variant 6): k_mm2's 12-pass bookkeeping with the
// accumulator in registers and predicated gathers.
//   * The shared-memory accumulator of k_mm2 cost ~700 L1 wavefronts per tile
//     and stage (ncu: 22-28% of the LSU data pipe); here acc[] lives in
//     registers: phase A builds it from the ADO (registers) and the TMA'd base
//     tile, phase B adds the neighbour crosses straight into it, phase C stores
//     it.  The base tile's shared memory is reused for stage 2's (Y2 - s)/3.
//   * Absent links (TRUNCATED raise at the top tier, ABSENT lower where
//     n_m = 0) are predicated off per lane instead of reading a zero tile, so
//     they generate no L1 wavefronts; with the reference (tier-major) order the
//     top-tier tiles -- 64% of the ADOs at N_max = 8, K = 1 -- issue no raise
//     traffic at all, and lower links of a tile land on ~2 lines per request.
template <int D, int KP1, int STAGE, int MINB>
__global__ void __launch_bounds__(32, MINB) k_mm3(const KParams P) {
  constexpr int NP = D * D;
  constexpr int M = D * KP1;
  constexpr int TB = NP * TILE;
  __shared__ __align__(128) double sBase[STAGE >= 2 ? NP : 1][TILE];
  __shared__ int sU[M][TILE];
  __shared__ int sD[M][TILE];
  __shared__ unsigned char sN[M][TILE];
  __shared__ __align__(8) uint64_t bar;

  volatile Ctl* ctl = P.ctl;
  if (ctl->status != ST_RUNNING) return;
  const long long step_next = ctl->step + 1;
  const int lane = threadIdx.x;
  const int tile = P.tile_begin + blockIdx.x;
  const size_t toff = (size_t)tile * TB;
  const size_t tb = toff + lane;
  double maxa2 = 0.0;
  const double c = STAGE == 4 ? P.dt / 6.0 : P.coef;

  if (STAGE >= 2 && lane == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, TB * 8u);
    bulk_g2s(&sBase[0][0], (STAGE == 4 ? P.Bbuf : P.sig) + toff, TB * 8, &bar);
  }
  __syncwarp();
  // ---- links (element offsets, -1 = absent), n, damping
  const size_t gb = (size_t)tile * M * TILE + lane;
  int tk[KP1];
#pragma unroll
  for (int k = 0; k < KP1; ++k) tk[k] = 0;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int up = __ldg(P.plus + gb + m * TILE);
    const int dn = __ldg(P.minus + gb + m * TILE);
    const int n = __ldg(P.nvec + gb + m * TILE);
    tk[m % KP1] += n;
    sU[m][lane] = up >= 0 && !P.debug ? (up >> 5) * TB + (up & 31) : -1;
    sD[m][lane] = dn >= 0 && !P.debug ? (dn >> 5) * TB + (dn & 31) : -1;
    sN[m][lane] = (unsigned char)n;
  }
  double damp = 0.0;  // heom.py:275, generalised: sum_k nu_k * sum_j n_jk
#pragma unroll
  for (int k = 0; k < KP1; ++k) damp += (double)tk[k] * P.nu[k];

  double acc[NP];
  {  // ---- phase A: base + c * (damping + commutator), ADO in registers
    double s[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) s[p] = __ldg(P.Yin + tb + p * TILE);
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
    if (STAGE >= 2) mbar_wait(&bar, 0);
    auto base = [&](int p) -> double {
      if (STAGE == 1) return s[p];
      const double b = sBase[p][lane];
      if (STAGE == 2) sBase[p][lane] = (s[p] - b) * (1.0 / 3.0);  // park (Y2 - s)/3 for B
      if (STAGE == 4) return b + s[p] * (1.0 / 3.0);
      return b;
    };
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double cm_im = 0.0;
#pragma unroll
      for (int l = 0; l < D; ++l)
        if (l != i) cm_im += P.h[i * MAXD + l] * sim<D>(s, i, l);
      acc[i] = base(i) + c * (-(damp + P.decay[i]) * s[i] - 2.0 * cm_im);
#pragma unroll
      for (int j = i + 1; j < D; ++j) {
        const int pr = Pk<D>::re(i, j), pim = Pk<D>::im(i, j);
        const double f = -(damp + 0.5 * (P.decay[i] + P.decay[j]));
        double cr = 0.0, ci = 0.0;
#pragma unroll
        for (int l = 0; l < D; ++l) {
          const double hil = P.h[i * MAXD + l], hlj = P.h[l * MAXD + j];
          cr += hil * sre<D>(s, l, j) - sre<D>(s, i, l) * hlj;
          ci += hil * sim<D>(s, l, j) - sim<D>(s, i, l) * hlj;
        }
        acc[pr] = base(pr) + c * (f * s[pr] + ci);  // -1j * cm
        acc[pim] = base(pim) + c * (f * s[pim] - cr);
      }
    }
  }
  __syncwarp();
  // ---- phase B: neighbour crosses, one site at a time, predicated per lane
#pragma unroll
  for (int st = 0; st < D; ++st) {
    double cre[D], cim[D];
#pragma unroll
    for (int o = 0; o < D; ++o) cre[o] = cim[o] = 0.0;
#pragma unroll
    for (int k = 0; k < KP1; ++k) {
      const int m = st * KP1 + k;
      const int ou = sU[m][lane], od = sD[m][lane];
      const bool vu = ou >= 0, vd = od >= 0;
      const double* up = P.Yin + (vu ? ou : 0);
      const double* dn = P.Yin + (vd ? od : 0);
      const double n = (double)sN[m][lane];
      const double cb = n * P.b[k], ca = n * P.a[k];
      auto ld = [](const double* q, bool v) {
        double r = 0.0;
        if (v) r = __ldg(q);
        return r;
      };
      cre[st] += 2.0 * cb * ld(dn + st * TILE, vd);
#pragma unroll
      for (int o = 0; o < D; ++o) {
        if (o == st) continue;
        const int a = st < o ? st : o, b = st < o ? o : st;
        const int pr = Pk<D>::re(a, b), pim = Pk<D>::im(a, b);
        const double ur = ld(up + pr * TILE, vu), ui = ld(up + pim * TILE, vu);
        const double dr = ld(dn + pr * TILE, vd), di = ld(dn + pim * TILE, vd);
        if (o > st) {
          cre[o] += cb * dr - ca * di - ui;
          cim[o] += cb * di + ca * dr + ur;
        } else {
          cre[o] += cb * dr + ca * di + ui;
          cim[o] += cb * di - ca * dr - ur;
        }
      }
    }
    acc[st] += c * cre[st];
#pragma unroll
    for (int o = 0; o < D; ++o) {
      if (o == st) continue;
      const int a = st < o ? st : o, b = st < o ? o : st;
      acc[Pk<D>::re(a, b)] += c * cre[o];
      acc[Pk<D>::im(a, b)] += c * cim[o];
    }
  }
  // ---- phase C: store (stage 2 also B = (Y2 - s)/3 + 2/3 Y3)
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    P.Yout[tb + p * TILE] = acc[p];
    if (STAGE == 2) P.Bbuf[tb + p * TILE] = sBase[p][lane] + (2.0 / 3.0) * acc[p];
  }
  if (STAGE == 4) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      maxa2 = fmax(maxa2, acc[i] * acc[i]);
#pragma unroll
      for (int j = i + 1; j < D; ++j) {
        const double yr = acc[Pk<D>::re(i, j)], yi = acc[Pk<D>::im(i, j)];
        maxa2 = fmax(maxa2, yr * yr + yi * yi);
      }
    }
    __shared__ int s_last;
    if (step_next % 25 == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxa2 = fmax(maxa2, __shfl_xor_sync(0xffffffffu, maxa2, o));
      if (lane == 0)
        atomicMax(const_cast<unsigned long long*>(&ctl->maxabs2_bits),
                  (unsigned long long)__double_as_longlong(maxa2));
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) {
      const unsigned prev = atomicAdd(const_cast<unsigned*>(&ctl->blocks_done), 1u);
      s_last = prev == gridDim.x - 1;
    }
    __syncwarp();
    if (s_last) {
      __threadfence();
      if (lane == 0) ctl->launches = ctl->launches + 4;
      finish_step_warp<D, true>(P, step_next);
    }
  }
}

template <int D, int KP1, int MINB>
static cudaError_t mm3_launch_b(int stage, const KParams& p, cudaStream_t s) {
  switch (stage) {
    case 1: k_mm3<D, KP1, 1, MINB><<<p.n_tiles, 32, 0, s>>>(p); break;
    case 2: k_mm3<D, KP1, 2, MINB><<<p.n_tiles, 32, 0, s>>>(p); break;
    case 3: k_mm3<D, KP1, 3, MINB><<<p.n_tiles, 32, 0, s>>>(p); break;
    case 4: k_mm3<D, KP1, 4, MINB><<<p.n_tiles, 32, 0, s>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <int D, int KP1>
static cudaError_t mm3_launch(int stage, const KParams& p, cudaStream_t s) {
  if constexpr (D == 7) {
    switch (mm2_minb()) {
      case 10: return mm3_launch_b<D, KP1, 10>(stage, p, s);
      case 12: return mm3_launch_b<D, KP1, 12>(stage, p, s);
      case 16: return mm3_launch_b<D, KP1, 16>(stage, p, s);
      default: break;
    }
  }
  return mm3_launch_b<D, KP1, 1>(stage, p, s);
}

bool fast_supported(int d, int kp1) { return d >= 1 && d <= 8 && kp1 >= 1 && kp1 <= 2; }

// HB_FAST_VARIANT (experiments): 7 = k_mm4 (hb_mm4.cu, default); 12 = k_mm4
// stage 1 + k_mm8 (TMEM accumulator, hb_mm8.cu) stages 2-4 for d = 7, K + 1 = 2;
// 11 = k_mm8 everywhere;
// 6 = register accumulator + predicated gathers,
// 5 = mode-major + TMA base tile, 12-pass RK,
// 4 = mode-major, 1 = sigma in registers, 3 = TMA, 2 = warp-split, 0 = column-streamed
static int fast_variant() {
  static int v = [] {
    const char* e = getenv("HB_FAST_VARIANT");
    return e ? atoi(e) : 7;
  }();
  return v;
}

// Variant dispatch.  Only d = 7 (FMO) instantiates all variants (for the
// measurements in DESIGN.md); HB_FAST_MINB = register cap of the legacy ones.
template <int D, int KP1, int MINB>
static cudaError_t legacy_dispatch(int variant, int stage, const KParams& p, cudaStream_t s) {
  const int grid = (p.n_tiles * TILE + FT - 1) / FT;
  switch (variant * 8 + stage) {
    case 2 * 8 + 1: k_split<D, KP1, 1, MINB><<<p.n_tiles, NW * 32, 0, s>>>(p); break;
    case 2 * 8 + 2: k_split<D, KP1, 2, MINB><<<p.n_tiles, NW * 32, 0, s>>>(p); break;
    case 2 * 8 + 3: k_split<D, KP1, 3, MINB><<<p.n_tiles, NW * 32, 0, s>>>(p); break;
    case 2 * 8 + 4: k_split<D, KP1, 4, MINB><<<p.n_tiles, NW * 32, 0, s>>>(p); break;
    case 0 * 8 + 1: k_col<D, KP1, 1, MINB><<<grid, FT, 0, s>>>(p); break;
    case 0 * 8 + 2: k_col<D, KP1, 2, MINB><<<grid, FT, 0, s>>>(p); break;
    case 0 * 8 + 3: k_col<D, KP1, 3, MINB><<<grid, FT, 0, s>>>(p); break;
    case 0 * 8 + 4: k_col<D, KP1, 4, MINB><<<grid, FT, 0, s>>>(p); break;
    case 1 * 8 + 1: k_fast<D, KP1, 1, MINB><<<grid, FT, 0, s>>>(p); break;
    case 1 * 8 + 2: k_fast<D, KP1, 2, MINB><<<grid, FT, 0, s>>>(p); break;
    case 1 * 8 + 3: k_fast<D, KP1, 3, MINB><<<grid, FT, 0, s>>>(p); break;
    case 1 * 8 + 4: k_fast<D, KP1, 4, MINB><<<grid, FT, 0, s>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

static int fast_minb() {
  static int v = [] {
    const char* e = getenv("HB_FAST_MINB");
    return e ? atoi(e) : 1;
  }();
  return v;
}

template <int D, int KP1>
static cudaError_t fast_dispatch(int stage, const KParams& p, cudaStream_t s) {
  if constexpr (D == 7) {
    const int v = fast_variant();
    if (v == 13) return launch_mm9(stage, p, s);
    if (v == 12)  // k_mm4 for stage 1, the TMEM-accumulator k_mm8 for 2-4
      return KP1 == 2 && stage >= 2 ? launch_mm8(stage, p, s) : launch_mm4(stage, p, s);
    if (v == 11) return KP1 == 2 ? launch_mm8(stage, p, s) : launch_mm4(stage, p, s);
    if (v == 9) return launch_mm6(stage, p, s);
    if (v == 8) return launch_mm5(stage, p, s);
    if (v == 7) return launch_mm4(stage, p, s);
    if (v == 6) return mm3_launch<D, KP1>(stage, p, s);
    if (v == 5) return mm2_launch<D, KP1>(stage, p, s);
    if (v == 4) return mm_launch<D, KP1>(stage, p, s);
    if (v != 3) {
      return fast_minb() == 4 ? legacy_dispatch<D, KP1, 4>(v, stage, p, s)
                              : legacy_dispatch<D, KP1, 1>(v, stage, p, s);
    }
    switch (tma_nw()) {
      case 4: return tma_launch<D, KP1, 4>(stage, p, s);
      case 16: return tma_launch<D, KP1, 16>(stage, p, s);
      default: return tma_launch<D, KP1, 8>(stage, p, s);
    }
  } else {  // other d: the production kernel only
    return launch_mm4(stage, p, s);
  }
}

template <int D>
static cudaError_t fast_kp1(int stage, const KParams& p, cudaStream_t s) {
  return p.kp1 == 1 ? fast_dispatch<D, 1>(stage, p, s) : fast_dispatch<D, 2>(stage, p, s);
}

cudaError_t launch_fast(int stage, const KParams& p, cudaStream_t s) {
  if (p.single) return launch_mm4(stage, p, s);  // the float state has one kernel
  switch (p.d) {
    case 1: return fast_kp1<1>(stage, p, s);
    case 2: return fast_kp1<2>(stage, p, s);
    case 3: return fast_kp1<3>(stage, p, s);
    case 4: return fast_kp1<4>(stage, p, s);
    case 5: return fast_kp1<5>(stage, p, s);
    case 6: return fast_kp1<6>(stage, p, s);
    case 7: return fast_kp1<7>(stage, p, s);
    case 8: return fast_kp1<8>(stage, p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hb
