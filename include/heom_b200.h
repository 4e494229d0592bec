/*
 * heom_b200.h -- C ABI of the B200-native HEOM propagator (libheomb200.so).
 *
 * Plain pointers and sizes only; complex arrays are interleaved (re, im) float64
 * in C order, i.e. exactly numpy complex128.  Host buffers are owned by the
 * caller; device buffers, the CUDA stream and the CUDA graph are owned by the
 * handle.  Distinct handles may be driven from different threads concurrently
 * (ctypes releases the GIL); one handle must not be used by two threads at once.
 *
 * Every entry point cites the reference interface it replaces
 * (/root/reference/pkg/src/excitonflow/...).
 *
 * Return codes: HB_OK, or one of the HB_ERR_* / HB_DIVERGED / HB_HARDCAP codes;
 * the message of the last failure on the calling thread is hb_last_error().
 */
#ifndef HEOM_B200_H
#define HEOM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HB_OK 0
#define HB_ERR_ARG 1      /* bad argument -> ValueError            */
#define HB_ERR_CUDA 2     /* CUDA failure / no device             */
#define HB_DIVERGED 3     /* heom.py:386-389 PropagationDiverged  */
#define HB_HARDCAP 4      /* heom.py:366-368 ConvergenceFailure   */
#define HB_ERR_RANGE 5    /* hierarchy.py:66-69 index range       */

/* stop reasons (Trajectory.stop_reason, observables.py:33) */
#define HB_STOP_NONE 0
#define HB_STOP_T_END 1
#define HB_STOP_RESIDUAL 2

/* state layouts on the device */
#define HB_LAYOUT_AUTO 0       /* Hermitian-packed if rho0 is exactly Hermitian */
#define HB_LAYOUT_HERMITIAN 1  /* d*d real planes per ADO (upper triangle)     */
#define HB_LAYOUT_GENERAL 2    /* 2*d*d real planes per ADO                     */

/* ADO orderings on the device (the tables exported are always reference order) */
#define HB_ORDER_LEX 0         /* pure lexicographic over all tiers (locality)  */
#define HB_ORDER_REFERENCE 1   /* tier-major lexicographic (hierarchy.py:71-78) */
#define HB_ORDER_LEX_SPLIT 2   /* lexicographic tiles, top tier last inside a tile */

/* stage-kernel variants */
#define HB_KERNEL_AUTO 0       /* unrolled thread-per-ADO kernel when the shape allows */
#define HB_KERNEL_GENERIC 1    /* runtime-shaped tile kernel (any d, K, layout)        */

/* state precision (heom.py:74 PropagationConfig.precision, heom.py:93-94 dtype) */
#define HB_PREC_DOUBLE 0       /* complex128 state, FP64 arithmetic                     */
#define HB_PREC_SINGLE 1       /* complex64 state, FP32 RHS arithmetic, FP64 bookkeeping;
                                  needs the production shape (Hermitian rho0, every block
                                  level a site, d <= 8, K + 1 <= 2)                     */

#define HB_MAX_D 9
#define HB_MAX_KP1 8
#define HB_MAX_SINKS 4
#define HB_MAX_SINK_TERMS 32

/* Operands + stop policy of one propagation (heom.py:57-94 PropagationConfig,
 * heom.py:235-275 _BlockPropagator.__init__, heom.py:121-134 loss channels). */
typedef struct {
    int d;                    /* block dimension (non-sink levels), 1..HB_MAX_D   */
    int n_sites;              /* site slots (len(system.site_indices))            */
    int kp1;                  /* modes per site = n_matsubara + 1                 */
    int n_max;                /* truncation tier                                  */
    const double* h;          /* d*d, rad/fs, mean-diagonal shifted (heom.py:251-255) */
    const int32_t* site_of;   /* d: block position -> site slot or -1             */
    const double* decay;      /* d: summed loss rate out of each position         */
    const double* nu;         /* kp1: damping rate of Matsubara index k (fs^-1)   */
    const double* a;          /* kp1: commutator weight of theta_k (fs^-2)        */
    const double* b;          /* kp1: anticommutator weight of theta_k (fs^-2)    */
    int n_sinks;              /* sinks integrated alongside (heom.py:282-283)     */
    const int32_t* sink_nterms;   /* n_sinks                                      */
    const double* sink_rate;      /* concatenated (rate, pos) terms, channel order */
    const int32_t* sink_pos;
    int n_site_pos;           /* residual sum positions (heom.py:352-353)         */
    const int32_t* site_pos;
    int d_full;               /* full basis dimension for records                 */
    const int32_t* block_full;    /* d: full index of each block position          */
    const int32_t* sink_full;     /* n_sinks: full index of each sink              */
    double dt;
    int has_t_end;
    double t_end;
    int has_residual;
    double residual;
    double hard_cap;
    int64_t record_stride;
    int record_matrices;
    double blowup_norm;
    int device;               /* CUDA device ordinal                              */
    int layout;               /* HB_LAYOUT_*                                      */
    int ordering;             /* HB_ORDER_*                                       */
    int chunk_steps;          /* RK4 steps per CUDA-graph launch (0 = default)    */
    int kernel_variant;       /* HB_KERNEL_*                                      */
    int precision;            /* HB_PREC_*                                        */
} hb_params;

typedef struct {
    int stop_reason;          /* HB_STOP_*                                        */
    int layout;               /* layout actually used                             */
    int64_t steps;            /* RK4 steps taken                                  */
    int64_t n_records;        /* records available via hb_get_records             */
    int64_t n_tot;            /* hierarchy size                                   */
} hb_result;

typedef struct hb_handle hb_handle;

/* Last error message of the calling thread ("" if none). */
const char* hb_last_error(void);

/* Number of visible CUDA devices (0 when none / no driver). */
int hb_device_count(void);

/* hierarchy.py:27-29 hierarchy_size; -1 if the count overflows int64. */
int64_t hb_hierarchy_size(int modes, int n_max);

/* hierarchy.py:59-105 enumerate_hierarchy, built on the device.  All outputs in
 * the reference order (tier-major lexicographic), int32, caller-allocated:
 * indices/plus/minus (n_tot, modes), tiers (n_tot).  perm_or_null (n_tot)
 * receives the device (HB_ORDER_LEX) position of every reference position.
 * Errors: HB_ERR_ARG (modes < 1 or n_max < 0), HB_ERR_RANGE (n_tot > INT32_MAX). */
int hb_graph_build(int modes, int n_max, int device, int32_t* indices, int32_t* tiers,
                   int32_t* plus, int32_t* minus, int32_t* perm_or_null);

/* ---- Level-2 kernel ABI (_kernels.py), host buffers, copies inside ---- */

/* _kernels.py:23-58 hierarchy_rhs_kernel(out, sig, h, site_of, plus, minus, nvec,
 * tier_damp, a_comm, b_anti, decay): sig/out (n_tot,d,d) complex128, plus/minus/
 * nvec (n_tot,modes) with modes = number of site slots (one mode per site),
 * nvec holding integers 0..255 (as float64, like the reference). */
int hb_rhs(double* out, const double* sig, int64_t n_tot, int d, const double* h,
           const int32_t* site_of, const int32_t* plus, const int32_t* minus, int modes,
           const double* nvec, const double* tier_damp, double a_comm, double b_anti,
           const double* decay, int device);

/* heom.py:175-204 heom_rhs: the dense semantic definition on the FULL basis
 * (sinks included): hb_rhs plus the Lindblad refill of the sink populations,
 * out[dst,dst] += rate * sig[src,src] for every (rate, src, dst) channel
 * (heom.py:146).  d up to HB_MAX_D (9 = the FMO basis). */
int hb_heom_rhs(double* out, const double* sig, int64_t n_tot, int d, const double* h,
                const int32_t* site_of, const int32_t* plus, const int32_t* minus, int modes,
                const double* nvec, const double* tier_damp, double a_comm, double b_anti,
                const double* decay, int n_refill, const int32_t* refill_dst,
                const int32_t* refill_src, const double* refill_rate, int device);

/* _kernels.py:61-65 add_scaled: out = x + c*y over n complex elements. */
int hb_add_scaled(double* out, const double* x, const double* y, double c, int64_t n,
                  int device);
/* _kernels.py:68-72 rk4_update: sig += w*(k1 + 2*(k2+k3) + k4). */
int hb_rk4_update(double* sig, const double* k1, const double* k2, const double* k3,
                  const double* k4, double w, int64_t n, int device);
/* _kernels.py:75-84 max_abs2 -> *result. */
int hb_max_abs2(const double* x, int64_t n, double* result, int device);

/* ---- Level-1 propagator (heom.py:286-406 propagate_from) ---- */

/* Allocate device state, build the hierarchy tables on the device. */
int hb_create(const hb_params* params, hb_handle** out);
void hb_destroy(hb_handle* h);

/* rho0_block: d*d complex (block part of rho0), sink_pops: n_sinks.  Resets the
 * run (step 0, auxiliaries 0), records the t=0 sample and evaluates the stop
 * policy for step 0.  layout AUTO picks HERMITIAN when rho0_block is exactly
 * Hermitian (diagonal imaginary parts zero), else GENERAL. */
int hb_set_rho0(hb_handle* h, const double* rho0_block, const double* sink_pops);

/* The whole hierarchy state instead of rho0 (auxiliaries included): sig is
 * (n_tot,d,d) complex in the reference order (hierarchy.py:71-78), sink_pops
 * n_sinks.  Otherwise as hb_set_rho0 (layout AUTO: HERMITIAN if every ADO is
 * exactly Hermitian).  The reference's propagate_from accepts only rho0
 * (heom.py:286-311, auxiliaries zero); this entry point is its state-restart
 * counterpart, used to pin the production kernel on every ADO against the
 * oracle (the full-state check of test_heom.py:120-130).  Unsharded handles only. */
int hb_set_state(hb_handle* h, const double* sig, const double* sink_pops);

/* Run until a stop policy fires (heom.py:358-391).  Returns HB_OK with
 * res->stop_reason set, HB_DIVERGED (res->steps = step whose guard fired) or
 * HB_HARDCAP. */
int hb_run(hb_handle* h, hb_result* res);

/* Records collected by hb_set_rho0 + hb_run: steps (n), pops (n*d_full),
 * mats_or_null (n*d_full*d_full complex; requires record_matrices).  cap = room. */
int hb_get_records(hb_handle* h, int64_t* steps, double* pops, double* mats_or_null,
                   int64_t cap);

/* Number of records collected so far (what hb_get_records will return). */
int64_t hb_record_count(hb_handle* h);

/* Current state in the reference order and layout: sig (n_tot,d,d) complex,
 * sink_pops (n_sinks). */
int hb_get_state(hb_handle* h, double* sig, double* sink_pops);

/* sigma^0 only (the reduced density matrix block, d*d complex) and the sinks:
 * what Trajectory.final_rho needs (heom.py:343-350) without copying the state. */
int hb_get_sigma0(hb_handle* h, double* sig0, double* sink_pops);

/* Benchmark / profiling helpers (bench.py).  Run exactly n_steps RK4 steps on
 * the resident state ignoring the stop policy; *ms = CUDA-event time on the
 * handle's stream.  stage_ms_or_null[4] (optional) receives the average time of
 * each stage kernel, measured with events around individual launches. */
int hb_time_steps(hb_handle* h, int64_t n_steps, double* ms, double* stage_ms_or_null);

/* Product kernels that did work since hb_create: host-launched ones plus the
 * step kernels counted on the device (as of the handle's last synchronisation). */
int64_t hb_launch_count(hb_handle* h);

/* Frees the idle device buffers the library pools between handles (state
 * buffers of finished runs are kept per (device, size) up to 24 GiB so that a
 * repeated propagate() of the same shape skips cudaMalloc; an allocation that
 * fails also trims the pool and retries).  Live handles are untouched. */
void hb_pool_trim(void);

/* Cumulative host->device and device->host bytes copied by the library since it
 * was loaded (all handles and shims): the end-to-end benchmark's transfer count. */
void hb_io_bytes(int64_t* h2d, int64_t* d2h);

/* ---- Sharding (new, no reference counterpart: SPEC.md:277) ----
 * One hierarchy split over several handles (one per GPU over NCCL, or several
 * in one process on one GPU for verification).  A shard numbers its ADO slots
 * locally: its owned ADOs first -- those below the top tier, then the top-tier
 * ones in whole tiles (no raise links: k_mm4's paired gather rounds) -- then
 * halo slots for the neighbours owned by other shards; the buffers hold only
 * owned + halo slots.  The host side (shard.py) builds the local tables, the
 * halo plan and four launch groups partitioning the owned tiles.  The shard
 * whose slot 0 holds ADO 0 (the root) does sinks, records and the stop policy;
 * sharded runs use the t_end policy. */
typedef struct {
    int n_local;            /* ADO slots (a multiple of 32): owned tiles, then halo   */
    int own_tiles;          /* tiles [0, own_tiles) are computed by this shard         */
    int top_tile;           /* first owned tile whose ADOs all sit on the top tier      */
    int root;               /* local slot 0 holds ADO 0                                  */
    const int32_t* plus;    /* (n_local, modes) local raise links, -1 = none            */
    const int32_t* minus;   /* (n_local, modes) local lower links, -2 = none            */
    const uint8_t* nvec;    /* (n_local, modes) n_m                                      */
    const int32_t* groups;  /* owned tiles of the four launch groups, concatenated:      */
    int group_count[4];     /* send-only, interior, send+halo, halo-only (a partition)  */
} hb_shard_tables;
int hb_create_shard(const hb_params* params, const hb_shard_tables* tables, hb_handle** out);
/* wait for the handle's work, drain records, read the status / step */
int hb_sync(hb_handle* h, int* status, int64_t* step);
/* NCCL (libnccl loaded at run time); id = ncclUniqueId (128 bytes) */
int hb_nccl_unique_id(char* id128);
int hb_nccl_init(hb_handle* h, const char* id128, int nranks, int rank);
/* Compressed halos: a consumer reads from a halo ADO only the cross of the site
 * it reaches it through (2d-1 Hermitian-packed planes, _kernels.py:41-57), so
 * the plan lists (local slot, site) entries.  Segment i has count[i] consecutive
 * entries of pos/site exchanged with shard peer[i]: is_send[i] = 1 packs them
 * from this shard's owned slots, 0 unpacks them into its halo slots; owner and
 * consumer list a segment's entries in the same order.  After hb_set_rho0. */
int hb_halo_set(hb_handle* h, int n_seg, const int32_t* peer, const int32_t* is_send,
                const int32_t* count, const int32_t* pos, const int32_t* site);
/* Enqueue n_steps RK4 steps of this shard (NCCL): per stage the send-only and
 * interior tiles, then -- once the halo of the stage input has arrived -- the
 * send+halo tiles; the output crosses go out on a second stream (pack, grouped
 * ncclSend/ncclRecv, unpack) while the halo-only tiles compute.  Every 25th
 * step the divergence max is all-reduced (ncclAllReduce MAX) so all shards stop
 * together (heom.py:386-389).  ms_or_null: CUDA-event time (synchronises). */
int hb_shard_steps(hb_handle* h, int64_t n_steps, double* ms_or_null);
/* The same for n in-process shards on one device, the exchange as device
 * copies of the packed crosses, every stage serialised (the bit-exactness check
 * of partition, local numbering and halo plan). */
int hb_shard_steps_local(hb_handle** shards, int n, int64_t n_steps, double* ms_or_null);

#ifdef __cplusplus
}
#endif
#endif /* HEOM_B200_H */
