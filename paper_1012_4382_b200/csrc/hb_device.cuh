// Device-side helpers shared by the stage kernels (hb_stage.cu, hb_mm4.cu):
// packed-plane bookkeeping, numpy-compatible summation and the scalar per-step
// bookkeeping done by the last CTA of a stage-4 launch (sinks, guard, records,
// stop policy -- heom.py:355-394).
#pragma once
#include "hb_internal.h"

namespace hb {

template <int D, bool HERM>
struct Lay {
  static constexpr int NP = HERM ? D * D : 2 * D * D;      // float64 planes per ADO
  static constexpr int NE = HERM ? D * (D + 1) / 2 : D * D;  // elements per ADO
};

// element e -> (i, j) and its planes; Hermitian: e < D diagonal (real),
// then the upper triangle row-major.
template <int D, bool HERM>
__device__ __forceinline__ void elem_info(int e, int& i, int& j, int& pr, int& pim) {
  if (HERM) {
    if (e < D) {
      i = j = e;
      pr = e;
      pim = -1;
      return;
    }
    int o = e - D, r = 0, cnt = D - 1;
    while (o >= cnt) {
      o -= cnt;
      ++r;
      cnt = D - 1 - r;
    }
    i = r;
    j = r + 1 + o;
    pr = D + 2 * (e - D);
    pim = pr + 1;
  } else {
    i = e / D;
    j = e % D;
    pr = 2 * e;
    pim = 2 * e + 1;
  }
}

// plane p -> (i, j, part) for the unpack into shared memory
template <int D, bool HERM>
__device__ __forceinline__ void plane_info(int p, int& i, int& j, int& part) {
  if (HERM) {
    if (p < D) {
      i = j = p;
      part = 0;
      return;
    }
    int e = D + ((p - D) >> 1);
    int pr, pim;
    elem_info<D, HERM>(e, i, j, pr, pim);
    part = (p - D) & 1;
  } else {
    const int e = p >> 1;
    i = e / D;
    j = e % D;
    part = p & 1;
  }
}

// sigma^0 entry (i, j) straight from global memory (tile 0, lane 0)
template <int D, bool HERM>
__device__ __forceinline__ void load_sig0(const double* s, int i, int j, double& re, double& im,
                                          bool single = false) {
  if (single) {  // float state (HB_PREC_SINGLE): Hermitian-packed only
    const float* f = reinterpret_cast<const float*>(s);
    if (i == j) {
      re = (double)__ldcg(f + i * TILE);
      im = 0.0;
      return;
    }
    const int a = i < j ? i : j, b = i < j ? j : i;
    int e = D;
    for (int r = 0; r < a; ++r) e += D - 1 - r;
    e += b - a - 1;
    const int pr = D + 2 * (e - D);
    re = (double)__ldcg(f + herm_off(D, pr, 0));
    im = (double)__ldcg(f + herm_off(D, pr + 1, 0));
    if (i > j) im = -im;
    return;
  }
  if (HERM) {
    if (i == j) {
      re = __ldcg(s + i * TILE);
      im = 0.0;
      return;
    }
    const int a = i < j ? i : j, b = i < j ? j : i;
    int e = D;
    for (int r = 0; r < a; ++r) e += D - 1 - r;
    e += b - a - 1;
    const int pr = D + 2 * (e - D);
    re = __ldcg(s + herm_off(D, pr, 0));
    im = __ldcg(s + herm_off(D, pr + 1, 0));
    if (i > j) im = -im;
  } else {
    const int e = i * D + j;
    re = __ldcg(s + 2 * e * TILE);
    im = __ldcg(s + (2 * e + 1) * TILE);
  }
}

// numpy add.reduce of a short float64 vector (pairwise_sum), see or_np_sum
__device__ inline double np_sum(const double* x, int m) {
  double rest;
  if (m < 8) {
    rest = -0.0;
    for (int i = 0; i < m; ++i) rest += x[i];
  } else {
    double r[8];
    for (int jj = 0; jj < 8; ++jj) r[jj] = x[jj];
    int i;
    for (i = 8; i < m - (m % 8); i += 8)
      for (int jj = 0; jj < 8; ++jj) r[jj] += x[i + jj];
    rest = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < m; ++i) rest += x[i];
  }
  return rest;
}

// ---------------------------------------------------------------------------
// per-step bookkeeping, done by ONE WARP of the last CTA of a stage-4 launch
// (and by the init kernel): sigma^0 is fetched once, in parallel, into shared
// memory; records, guard and stop policy read it from there.

struct Sig0 {
  double re[MAXD * MAXD];
  double im[MAXD * MAXD];
};

template <int D, bool HERM>
__device__ void sig0_warp(const KParams& P, Sig0& s0) {
  const int lane = threadIdx.x & 31;
  for (int f = lane; f < D * D; f += 32)
    load_sig0<D, HERM>(P.sig, f / D, f % D, s0.re[f], s0.im[f], P.single != 0);
  __syncwarp();
}

template <int D>
__device__ void record_warp(const KParams& P, long long step, const Sig0& s0, volatile Ctl* c) {
  const int lane = threadIdx.x & 31;
  const long long idx = c->n_rec;
  if (idx >= P.rec_cap) return;  // host sizes the buffer for a whole chunk
  const int df = P.d_full;
  double* pops = P.rec_pops + idx * df;
  for (int f = lane; f < df; f += 32) {
    const int b = P.full2blk[f], sk = P.full2sink[f];
    pops[f] = b >= 0 ? s0.re[b * D + b] : (sk >= 0 ? c->sink_pops[sk] : 0.0);
  }
  if (P.record_matrices) {
    double* m = P.rec_mats + idx * df * df * 2;
    for (int f = lane; f < df * df; f += 32) {
      const int fi = f / df, fj = f % df;
      const int bi = P.full2blk[fi], bj = P.full2blk[fj];
      double re = 0.0, im = 0.0;
      if (bi >= 0 && bj >= 0) {
        re = s0.re[bi * D + bj];
        im = s0.im[bi * D + bj];
      } else if (fi == fj && P.full2sink[fi] >= 0) {
        re = c->sink_pops[P.full2sink[fi]];
      }
      m[2 * f] = re;
      m[2 * f + 1] = im;
    }
  }
  __syncwarp();
  if (lane == 0) {
    P.rec_step[idx] = step;
    c->n_rec = idx + 1;
  }
  __syncwarp();
}

// stop policy evaluated before step `step` (heom.py:359-368)
template <int D>
__device__ void check_stop_warp(const KParams& P, long long step, const Sig0& s0, volatile Ctl* c) {
  const int lane = threadIdx.x & 31;
  int st = ST_RUNNING;
  if (lane == 0) {
    const double t = (double)step * P.dt;
    if (P.has_t_end && t >= P.t_end - 1e-9) {
      st = ST_T_END;
    } else if (P.has_residual) {
      double diag[MAXD];
      for (int k = 0; k < P.n_site_pos; ++k) diag[k] = s0.re[P.site_pos[k] * (D + 1)];
      if (np_sum(diag, P.n_site_pos) <= P.residual) st = ST_RESIDUAL;
    }
    if (st == ST_RUNNING && !P.has_t_end && t >= P.hard_cap) st = ST_HARDCAP;
  }
  st = __shfl_sync(0xffffffffu, st, 0);
  if (st == ST_RUNNING) return;
  if (st != ST_HARDCAP && step % P.stride != 0) record_warp<D>(P, step, s0, c);
  if (lane == 0) c->status = st;
}

// non-root shard: advance the step, own-range guard every 25 steps, t_end only
__device__ inline void finish_step_shard(const KParams& P, long long step) {
  if ((threadIdx.x & 31) != 0) return;
  volatile Ctl* c = P.ctl;
  c->blocks_done = 0;
  c->step = step;
  if (step % 25 == 0) {
    const double mall = __longlong_as_double((long long)c->maxabs2_bits);
    c->maxabs2_bits = 0ull;
    if (mall > P.blow2) {
      c->status = ST_DIVERGED;
      return;
    }
  }
  const double t = (double)step * P.dt;
  if (P.has_t_end && t >= P.t_end - 1e-9) c->status = ST_T_END;
}

// The control block is read once, in parallel with sigma^0, into a shared
// copy (one round trip instead of a chain of dependent volatile accesses), the
// bookkeeping works on the copy, and the copy is written back at the end.  No
// other CTA touches the block meanwhile: this is the last CTA of the step (or
// the init kernel).
__device__ __forceinline__ void ctl_load_warp(const Ctl* g, Ctl& cs) {
  constexpr int NW = sizeof(Ctl) / 8;
  static_assert(sizeof(Ctl) % 8 == 0, "Ctl is copied in 8-byte words");
  __syncwarp();  // lane 0's last writes to the block are ordered before the copy
  const int lane = threadIdx.x & 31;
  for (int w = lane; w < NW; w += 32)
    reinterpret_cast<unsigned long long*>(&cs)[w] =
        __ldcg(reinterpret_cast<const unsigned long long*>(g) + w);
}
__device__ __forceinline__ void ctl_store_warp(Ctl* g, const Ctl& cs) {
  constexpr int NW = sizeof(Ctl) / 8;
  __syncwarp();
  const int lane = threadIdx.x & 31;
  for (int w = lane; w < NW; w += 32)
    __stcg(reinterpret_cast<unsigned long long*>(g) + w,
           reinterpret_cast<const unsigned long long*>(&cs)[w]);
  __syncwarp();
}

// the root bookkeeping on copies already in shared memory (cs: the control
// block, s0: sigma^0 of the new state); the caller writes cs back
template <int D>
__device__ void finish_step_loaded(const KParams& P, long long step, const Sig0& s0, Ctl& cs,
                                   int par) {
  const int lane = threadIdx.x & 31;
  volatile Ctl* c = &cs;
  double m0 = 0.0;
  for (int f = lane; f < D * D; f += 32) m0 = fmax(m0, s0.re[f] * s0.re[f] + s0.im[f] * s0.im[f]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m0 = fmax(m0, __shfl_xor_sync(0xffffffffu, m0, o));
  int diverged = 0;
  if (lane == 0) {
    c->blocks_done = 0;
    c->step = step;
    for (int s = 0; s < P.n_sinks; ++s)
      c->sink_pops[s] += (P.dt / 6.0) * (c->r[par][0][s] + 2.0 * (c->r[par][1][s] + c->r[par][2][s]) +
                                         c->r[par][3][s]);
    const bool full = step % 25 == 0;
    double mall = 0.0;
    if (full) {
      mall = __longlong_as_double((long long)c->maxabs2_bits);
      c->maxabs2_bits = 0ull;
    }
    diverged = (m0 > P.blow2 || (full && mall > P.blow2));
    if (diverged) c->status = ST_DIVERGED;
  }
  diverged = __shfl_sync(0xffffffffu, diverged, 0);
  __syncwarp();
  if (!diverged) {
    if (step % P.stride == 0) record_warp<D>(P, step, s0, c);
    check_stop_warp<D>(P, step, s0, c);
  }
}

template <int D, bool HERM>
__device__ void finish_step_warp(const KParams& P, long long step) {
  if (!P.root) {
    finish_step_shard(P, step);
    return;
  }
  __shared__ Sig0 s0;
  __shared__ Ctl cs;
  ctl_load_warp(P.ctl, cs);
  sig0_warp<D, HERM>(P, s0);  // ends with __syncwarp: cs is complete too
  finish_step_loaded<D>(P, step, s0, cs, P.rpar);
  ctl_store_warp(P.ctl, cs);
}

// The bookkeeping of the previous step done by the extra CTA of a stage-1 launch
// (KParams::fold), while the tiles compute that stage: it reads the
// control block and sigma^0 as k_step_finish does, takes the sink rates of the
// previous step's parity, and writes back only the fields the bookkeeping owns
// (tile 0 of this launch writes this step's sink rates concurrently).
template <int D>
__device__ void fold_finish_warp(const KParams& P) {
  __shared__ Sig0 s0;
  __shared__ Ctl cs;
  ctl_load_warp(P.ctl, cs);
  sig0_warp<D, true>(P, s0);
  if (cs.status != ST_RUNNING) return;
  if ((threadIdx.x & 31) == 0) cs.launches += 4;  // this step's four stage kernels
  finish_step_loaded<D>(P, cs.step + 1, s0, cs, P.rpar ^ 1);
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    Ctl* g = P.ctl;
    for (int s = 0; s < MAXS; ++s) __stcg(&g->sink_pops[s], cs.sink_pops[s]);
    __stcg(&g->maxabs2_bits, cs.maxabs2_bits);
    __stcg(&g->n_rec, cs.n_rec);
    __stcg(&g->launches, cs.launches);
    __stcg(&g->step, cs.step);
    __stcg(&g->status, cs.status);
  }
}

// t = 0 sample + stop policy before the first step (heom.py:355-368); 1 warp
template <int D, bool HERM>
__device__ void init_warp(const KParams& P) {
  if (!P.root) {
    if ((threadIdx.x & 31) == 0 && P.has_t_end && 0.0 >= P.t_end - 1e-9) P.ctl->status = ST_T_END;
    return;
  }
  __shared__ Sig0 s0;
  __shared__ Ctl cs;
  ctl_load_warp(P.ctl, cs);
  sig0_warp<D, HERM>(P, s0);
  record_warp<D>(P, 0, s0, &cs);
  check_stop_warp<D>(P, 0, s0, &cs);
  ctl_store_warp(P.ctl, cs);
}

}  // namespace hb
