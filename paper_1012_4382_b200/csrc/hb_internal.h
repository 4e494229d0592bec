// Internal interfaces shared by the CUDA translation units of libheomb200.so.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "heom_b200.h"

// HB_CHECKED (build target libheomb200_checked.so, tests only): device-side
// bounds checks on every gathered position, tile index and halo slot -- the
// substitute for compute-sanitizer, which is closed on the GPU pool.
#ifdef HB_CHECKED
#include <cassert>
#define HB_CHECK(cond) assert(cond)
#else
#define HB_CHECK(cond) ((void)0)
#endif

namespace hb {

constexpr int TILE = 32;          // ADOs per tile (AoSoA inner extent = one warp)
constexpr int MAXD = HB_MAX_D;
constexpr int MAXKP1 = HB_MAX_KP1;
constexpr int MAXS = HB_MAX_SINKS;
constexpr int MAXT = HB_MAX_SINK_TERMS;
constexpr int MAX_MODES = 64;
constexpr int MAXFULL = 16;       // full basis (block + sinks) for records

// Hermitian-packed tile (HB_LAYOUT_HERMITIAN), 32 ADOs: the d real diagonal
// planes [d][32], then the d(d-1)/2 upper-triangle elements as (re, im) pairs
// [e][32][2], so a gathered complex element is one 16-byte load (8 for float).
// Plane p < d is diagonal element p; plane d + 2e (+1) is the real (imaginary)
// part of upper-triangle element e (row-major over i < j).  Returns the offset
// of (plane p, lane) inside the tile, in elements.
__host__ __device__ inline int herm_off(int d, int p, int lane) {
  return p < d ? p * TILE + lane : d * TILE + ((p - d) >> 1) * 2 * TILE + 2 * lane + ((p - d) & 1);
}
// the generic (GENERAL) layout: plane-major [2 d^2][32]
__host__ __device__ inline int plane_off(bool herm, int d, int p, int lane) {
  return herm ? herm_off(d, p, lane) : p * TILE + lane;
}

enum Status : int {
  ST_RUNNING = 0,
  ST_T_END = 1,
  ST_RESIDUAL = 2,
  ST_DIVERGED = 3,
  ST_HARDCAP = 4,
};

// Device-resident control block of one run (one per handle).
struct Ctl {
  int status;
  int pad0;
  long long step;
  double sink_pops[MAXS];
  double r[2][4][MAXS];               // sink rates of the four stage inputs, by step parity
                                      // (KParams::rpar; the folded bookkeeping reads the last step's)
  unsigned long long maxabs2_bits;    // max |x|^2 over all ADOs (every 25 steps)
  unsigned int blocks_done;           // last-block election counter
  unsigned int pad1;
  long long n_rec;                    // records in the device record buffer
  long long launches;                 // product-kernel launches that did work
  long long loop_iter;                // WHILE-body iterations of the current graph launch
};

// Everything a stage kernel needs; passed by value (lives in the constant bank).
struct KParams {
  // operands
  double h[MAXD * MAXD];
  double decay[MAXD];
  int site_of[MAXD];
  double nu[MAXKP1], a[MAXKP1], b[MAXKP1];
  int d, n_sites, kp1, modes;
  int n_tot, n_tiles, tile_begin, n_planes;
  int n_tiles_total;     // tiles per state buffer (a zero tile follows the last one)
  int root;              // this launch owns tile 0 (ADO 0): sinks, records, stop policy
  // state (AoSoA: [tile][plane][32] doubles)
  const double* Yin;     // stage input: own tile + gathers
  const double* sig;     // sigma (stages 2-4)
  const double* Y2;      // stage 4
  const double* Y3;      // stage 4
  double* Yout;          // Y_{s+1} (stages 1-3), sigma (stage 4), k (rhs-only)
  double* Bbuf;          // B-scheme kernels: B = (Y2 - s)/3 + 2/3 Y3 (written at stage 2)
  // tables (AoSoA: [tile][mode][32])
  const int32_t* plus;
  const int32_t* minus;
  const uint8_t* nvec;
  const double* damp_plane;  // optional per-ADO damping (Level-2 shim), else null
  int fast;                  // production kernel k_mm4 (hb_mm4.cu), else the generic k_stage
  int rpar;                  // step parity of this launch: which ctl->r the stage writes
  int fold;                  // k_mm4ab graphs: stage 1 also does the previous step's
                             // bookkeeping (an extra warp of CTA 0); stage 4 then has no
                             // k_step_finish after it
  int split;                 // small hierarchies (fast path, d <= 7): a tile's phase A and
                             // phase B on separate warps, k_mm4ab: 1 = 1 + 1 warps,
                             // 2 = 2 + 2 warps; 0 = k_mm4 (one warp per tile)
  int top_tile;              // first tile whose ADOs all sit on the top tier (no raise
                             // links; tier-major order), n_tiles_total if none
  const int32_t* tile_list;  // if set: block b computes tile tile_list[b] (sharded
                             // boundary / interior launches), else tile_begin + b
  long long apw_first_tile;  // L2 persisting window over tiles [first, first + n) of the
  long long apw_tiles;       // stage input (0 tiles: none), hit ratio apw_hit
  float apw_hit;
  int set_cond;              // k_step_finish of the last step of a WHILE-node body
  long long loop_iters;      // WHILE-body iterations per graph launch
  unsigned long long cond;   // cudaGraphConditionalHandle of that WHILE node
  int single;                // HB_PREC_SINGLE: the state buffers hold float (production
                             // kernel only); the operands below in float for its RHS
  float hf[MAXD * MAXD], decayf[MAXD], nuf[MAXKP1], af[MAXKP1], bf[MAXKP1];
  double coef;               // dt/2, dt/2, dt for stages 1-3
  double dt;
  // bookkeeping
  Ctl* ctl;
  int n_sinks;
  int sink_nterms[MAXS];
  double sink_rate[MAXT];
  int sink_pos[MAXT];
  int n_site_pos;
  int site_pos[MAXD];
  int d_full;
  int block_full[MAXD];
  int sink_full[MAXS];
  int full2blk[MAXFULL];     // full index -> block position or -1
  int full2sink[MAXFULL];    // full index -> sink slot or -1
  int n_refill;              // dense path only: out[dst,dst] += rate * sig[src,src]
  int refill_dst[MAXT], refill_src[MAXT];
  double refill_rate[MAXT];
  int has_t_end, has_residual, record_matrices, hermitian;
  double t_end, residual, hard_cap, blow2;
  long long stride;
  long long rec_cap;
  long long* rec_step;
  double* rec_pops;
  double* rec_mats;
};

// hb_mm4.cu: production stage kernel for the Hermitian layout with every block
// level a site (site_of == identity), d <= 8, K + 1 <= 2; stage 4 launches the
// step bookkeeping kernel after it
bool mm4_supported(int d, int kp1);
cudaError_t launch_mm4(int stage, const KParams& p, cudaStream_t s);
cudaError_t launch_mm4_only(int stage, const KParams& p, cudaStream_t s);  // no bookkeeping
cudaError_t launch_step_finish(const KParams& p, cudaStream_t s);         // k_step_finish
// hb_halo.cu: the divergence max of n shards' control blocks, written back to all
cudaError_t launch_guard_max(unsigned long long* const* bits, int n, cudaStream_t s);

// hb_stage.cu
cudaError_t launch_stage(int stage, const KParams& p, cudaStream_t s);
cudaError_t launch_rhs_only(const KParams& p, cudaStream_t s);
cudaError_t configure_stages(const KParams& p);
cudaError_t launch_init(const KParams& p, cudaStream_t s);
cudaError_t launch_pack(const KParams& p, const double* ref_sig, const int32_t* dev2ref,
                        double* dst, cudaStream_t s);
cudaError_t launch_unpack(const KParams& p, const double* src, const int32_t* dev2ref,
                          double* ref_sig, cudaStream_t s);
cudaError_t launch_elementwise(int op, int64_t n, double* out, const double* x,
                               const double* y, const double* z, const double* w, double c,
                               cudaStream_t s);
cudaError_t launch_max_abs2(int64_t n, const double* x, unsigned long long* bits,
                            cudaStream_t s);

// hb_halo.cu: compressed (cross-only) halo exchange; op 0 = pack src -> packed,
// 1 = unpack packed -> dst
cudaError_t launch_halo(int op, bool single, void* dst, const void* src, int n, const int32_t* pos,
                        const int32_t* site, const int16_t* planes, int nc, int n_planes,
                        void* packed, cudaStream_t s);

// hb_graph.cu
struct GraphTables {
  int modes, n_max, n_tot, n_tiles;
  int32_t* plus_t = nullptr;    // device, AoSoA [tile][mode][32], device ordering
  int32_t* minus_t = nullptr;
  uint8_t* nvec_t = nullptr;
  int32_t* dev2ref = nullptr;   // device position -> reference position
};
int64_t hierarchy_size(int modes, int n_max);
// builds the reference-order tables (host outputs may be null) and, if gt != null,
// the device-order AoSoA tables.  ordering: HB_ORDER_*.
cudaError_t build_graph(int modes, int n_max, int ordering, cudaStream_t s,
                        int32_t* h_indices, int32_t* h_tiers, int32_t* h_plus, int32_t* h_minus,
                        int32_t* h_perm, GraphTables* gt);
void free_graph(GraphTables* gt);
// converts caller tables in reference order (n_tot, modes) into AoSoA device tables
cudaError_t upload_tables(int modes, int n_tot, const int32_t* plus, const int32_t* minus,
                          const uint8_t* nvec, cudaStream_t s, GraphTables* gt);

}  // namespace hb
