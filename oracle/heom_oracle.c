/*
 * heom_oracle.c -- CPU restatement of the reference HEOM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library,
 * and only as the checker (or the timed CPU baseline), never as the product.
 *
 * Pinned: tests/test_oracle.py checks every function below against the golden
 * vectors produced by running the reference itself (tests/golden/make_golden.py).
 *
 * Restated reference (paths relative to /root/reference/pkg/src/excitonflow):
 *   or_enumerate      hierarchy.py:59-105 (+ _compositions :32-39, sentinels :18-21)
 *   or_rhs            _kernels.py:23-58  (hierarchy_rhs_kernel), generalised from one
 *                     exponential per site to (K+1) modes per site, mode m = j*(K+1)+k
 *                     ("recommended K>=1 convention"); K=0 is the reference.
 *   or_add_scaled     _kernels.py:61-65
 *   or_rk4_update     _kernels.py:68-72
 *   or_max_abs2       _kernels.py:75-84
 *   or_propagate      heom.py:286-406 (RK4 loop, sink integration heom.py:282-283 and
 *                     :382-383, stop policy :359-368, divergence guard :386-389,
 *                     records :390-394)
 *
 * Complex arrays are interleaved (re, im) float64, C order (n_tot, d, d), exactly
 * the reference's complex128 layout.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define OR_TRUNCATED (-1)
#define OR_ABSENT (-2)

static int64_t binom(int64_t n, int64_t k) {
    if (k < 0 || k > n) return 0;
    if (k > n - k) k = n - k;
    /* exact for the sizes accepted below (result checked against INT32 range) */
    __int128 r = 1;
    for (int64_t i = 1; i <= k; ++i) {
        r = r * (n - k + i) / i;
        if (r > ((__int128)1 << 100)) return INT64_MAX;
    }
    return r > INT64_MAX ? INT64_MAX : (int64_t)r;
}

/* hierarchy.py:27-29 */
int64_t or_hierarchy_size(int modes, int n_max) {
    return binom((int64_t)modes + n_max, modes);
}

/* lexicographic compare of two rows of length m */
static int row_cmp(const int32_t* a, const int32_t* b, int m) {
    for (int i = 0; i < m; ++i) {
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    }
    return 0;
}

/* _compositions (hierarchy.py:32-39): all tuples of `parts` non-negative ints
 * summing to `total`, lexicographic ascending.  Writes rows into out, returns count. */
static int64_t compositions(int total, int parts, int32_t* prefix, int depth,
                            int32_t* out, int64_t cursor, int modes) {
    if (depth == modes - 1) {
        prefix[depth] = total;
        memcpy(out + cursor * modes, prefix, sizeof(int32_t) * modes);
        return cursor + 1;
    }
    for (int head = 0; head <= total; ++head) {
        prefix[depth] = head;
        cursor = compositions(total - head, parts - 1, prefix, depth + 1, out, cursor, modes);
    }
    return cursor;
}

/* position lookup: rows of one tier are lexicographically sorted, so a binary
 * search inside the tier block plays the role of the reference's tuple dict
 * (hierarchy.py:84). */
static int64_t lookup(const int32_t* rows, const int64_t* tier_start, int modes,
                      int tier, const int32_t* key) {
    int64_t lo = tier_start[tier], hi = tier_start[tier + 1] - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        int c = row_cmp(rows + mid * modes, key, modes);
        if (c == 0) return mid;
        if (c < 0) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

/* hierarchy.py:59-105.  Returns 0 on success, 1 on bad parameters, 2 when the
 * count exceeds int32 (hierarchy.py:66-69).  Outputs are caller-allocated. */
int or_enumerate(int modes, int n_max, int32_t* indices, int32_t* tiers,
                 int32_t* plus, int32_t* minus) {
    if (modes < 1 || n_max < 0) return 1;
    int64_t n_tot = or_hierarchy_size(modes, n_max);
    if (n_tot > INT32_MAX) return 2;
    int64_t* tier_start = (int64_t*)malloc(sizeof(int64_t) * (n_max + 2));
    int32_t* prefix = (int32_t*)calloc(modes, sizeof(int32_t));
    int64_t cursor = 0;
    for (int t = 0; t <= n_max; ++t) {
        tier_start[t] = cursor;
        cursor = compositions(t, modes, prefix, 0, indices, cursor, modes);
        for (int64_t k = tier_start[t]; k < cursor; ++k) tiers[k] = t;
    }
    tier_start[n_max + 1] = cursor;
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n_tot; ++k) {
        int32_t key[256];
        const int32_t* row = indices + k * modes;
        memcpy(key, row, sizeof(int32_t) * modes);
        for (int m = 0; m < modes; ++m) {
            plus[k * modes + m] = OR_TRUNCATED;
            minus[k * modes + m] = OR_ABSENT;
            if (tiers[k] < n_max) {
                key[m] += 1;
                plus[k * modes + m] = (int32_t)lookup(indices, tier_start, modes, tiers[k] + 1, key);
                key[m] -= 1;
            }
            if (row[m] > 0) {
                key[m] -= 1;
                minus[k * modes + m] = (int32_t)lookup(indices, tier_start, modes, tiers[k] - 1, key);
                key[m] += 1;
            }
        }
    }
    free(tier_start);
    free(prefix);
    return 0;
}

/* Operands of the block right-hand side (heom.py:235-275 generalised to modes). */
typedef struct {
    int64_t n_tot;
    int d;             /* block dimension */
    int n_sites;       /* number of site slots */
    int kp1;           /* modes per site (K+1) */
    const double* h;   /* d*d real, rad/fs (mean-diagonal shifted) */
    const int32_t* site_of;  /* d: block position -> site slot or -1 */
    const double* decay;     /* d */
    const int32_t* plus;     /* n_tot*modes */
    const int32_t* minus;    /* n_tot*modes */
    const int32_t* indices;  /* n_tot*modes (the multi-index n) */
    const double* nu;        /* kp1: damping rate of Matsubara index k */
    const double* a;         /* kp1: commutator weight of theta_k */
    const double* b;         /* kp1: anticommutator weight of theta_k */
} or_ops;

/* _kernels.py:23-58.  tier damping is sum_k nu_k * (sum_j n_{jk}); at K=0 that
 * is tiers*gamma exactly as heom.py:275. */
void or_rhs(const or_ops* op, const double* sig, double* out) {
    const int d = op->d, kp1 = op->kp1, modes = op->n_sites * op->kp1;
    const int64_t n_tot = op->n_tot;
    const int64_t mat = (int64_t)d * d;
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n_tot; ++k) {
        const double* s = sig + 2 * mat * k;
        double* o = out + 2 * mat * k;
        const int32_t* nk = op->indices + k * modes;
        double damp = 0.0;
        for (int kk = 0; kk < kp1; ++kk) {
            int64_t tk = 0;
            for (int j = 0; j < op->n_sites; ++j) tk += nk[j * kp1 + kk];
            damp += (double)tk * op->nu[kk];
        }
        for (int i = 0; i < d; ++i) {
            const int mi = op->site_of[i];
            const double di = op->decay[i];
            for (int j = 0; j < d; ++j) {
                const double f = -(damp + 0.5 * (di + op->decay[j]));
                double ar = f * s[2 * (i * d + j)];
                double ai = f * s[2 * (i * d + j) + 1];
                double cr = 0.0, ci = 0.0;
                for (int l = 0; l < d; ++l) {
                    const double hil = op->h[i * d + l], hlj = op->h[l * d + j];
                    cr += hil * s[2 * (l * d + j)] - s[2 * (i * d + l)] * hlj;
                    ci += hil * s[2 * (l * d + j) + 1] - s[2 * (i * d + l) + 1] * hlj;
                }
                /* acc += -1j * cm */
                ar += ci;
                ai -= cr;
                if (mi >= 0) {
                    for (int kk = 0; kk < kp1; ++kk) {
                        const int m = mi * kp1 + kk;
                        const int32_t p = op->plus[k * modes + m];
                        if (p >= 0) {  /* acc += 1j * sig[p][i,j] */
                            const double* sp = sig + 2 * mat * p + 2 * (i * d + j);
                            ar -= sp[1];
                            ai += sp[0];
                        }
                        const int32_t q = op->minus[k * modes + m];
                        if (q >= 0) {  /* acc += (n b + 1j n a) * sig[q][i,j] */
                            const double n = (double)nk[m];
                            const double cb = n * op->b[kk], ca = n * op->a[kk];
                            const double* sq = sig + 2 * mat * q + 2 * (i * d + j);
                            ar += cb * sq[0] - ca * sq[1];
                            ai += cb * sq[1] + ca * sq[0];
                        }
                    }
                }
                const int mj = op->site_of[j];
                if (mj >= 0) {
                    for (int kk = 0; kk < kp1; ++kk) {
                        const int m = mj * kp1 + kk;
                        const int32_t p = op->plus[k * modes + m];
                        if (p >= 0) {  /* acc -= 1j * sig[p][i,j] */
                            const double* sp = sig + 2 * mat * p + 2 * (i * d + j);
                            ar += sp[1];
                            ai -= sp[0];
                        }
                        const int32_t q = op->minus[k * modes + m];
                        if (q >= 0) {  /* acc += (n b - 1j n a) * sig[q][i,j] */
                            const double n = (double)nk[m];
                            const double cb = n * op->b[kk], ca = n * op->a[kk];
                            const double* sq = sig + 2 * mat * q + 2 * (i * d + j);
                            ar += cb * sq[0] + ca * sq[1];
                            ai += cb * sq[1] - ca * sq[0];
                        }
                    }
                }
                o[2 * (i * d + j)] = ar;
                o[2 * (i * d + j) + 1] = ai;
            }
        }
    }
}

/* _kernels.py:61-65, flat complex arrays of n elements */
void or_add_scaled(int64_t n, double* out, const double* x, const double* y, double c) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < 2 * n; ++i) out[i] = x[i] + c * y[i];
}

/* _kernels.py:68-72 */
void or_rk4_update(int64_t n, double* sig, const double* k1, const double* k2,
                   const double* k3, const double* k4, double w) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < 2 * n; ++i)
        sig[i] = sig[i] + w * (k1[i] + 2.0 * (k2[i] + k3[i]) + k4[i]);
}

/* _kernels.py:75-84 (serial; NaN never compares greater) */
double or_max_abs2(int64_t n, const double* x) {
    double m = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double a = x[2 * i] * x[2 * i] + x[2 * i + 1] * x[2 * i + 1];
        if (a > m) m = a;
    }
    return m;
}

/* numpy's add.reduce over a short contiguous float64 vector (pairwise_sum:
 * sequential from -0.0 below 8 elements, 8 interleaved accumulators up to 128;
 * checked empirically against ndarray.sum).  Used for the residual test
 * (heom.py:352-353) so the stop step follows the reference's rounding. */
double or_np_sum(const double* x, int m) {
    double rest;
    if (m < 8) {
        rest = -0.0;
        for (int i = 0; i < m; ++i) rest += x[i];
    } else {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = x[j];
        int i;
        for (i = 8; i < m - (m % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += x[i + j];
        rest = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < m; ++i) rest += x[i];
    }
    return rest;
}

/* Stop / run parameters of propagate_from (heom.py:57-94, 286-406). */
typedef struct {
    double dt;
    int has_t_end;
    double t_end;
    int has_residual;
    double residual;
    double hard_cap;
    int64_t stride;
    double blowup_norm;
    int n_sinks;
    const int32_t* sink_nterms;   /* n_sinks */
    const double* sink_rate;      /* concatenated terms, channel order */
    const int32_t* sink_pos;      /* concatenated terms: block position */
    int n_site_pos;
    const int32_t* site_pos;      /* block positions of the sites (residual sum) */
    int64_t max_steps;            /* safety bound for the caller's buffers */
} or_run;

enum { OR_OK = 0, OR_T_END = 1, OR_RESIDUAL = 2, OR_DIVERGED = 3, OR_HARDCAP = 4,
       OR_CAPACITY = 5 };

static void sink_rates(const or_run* rp, const double* sig0, int d, double* r) {
    int t = 0;
    for (int s = 0; s < rp->n_sinks; ++s) {
        double acc = 0.0;  /* python sum() starts from int 0: 0 + x == x */
        for (int c = 0; c < rp->sink_nterms[s]; ++c, ++t) {
            const int p = rp->sink_pos[t];
            const double v = rp->sink_rate[t] * sig0[2 * (p * d + p)];
            acc = (c == 0) ? v : acc + v;
        }
        r[s] = acc;
    }
}

static double system_population(const or_run* rp, const double* sig0, int d) {
    double diag[256];
    for (int i = 0; i < rp->n_site_pos; ++i) {
        const int p = rp->site_pos[i];
        diag[i] = sig0[2 * (p * d + p)];
    }
    return or_np_sum(diag, rp->n_site_pos);
}

/*
 * heom.py:286-406.  sig: (n_tot,d,d) complex state, sig[0] = rho0 block, rest 0,
 * updated in place.  sink_pops: n_sinks, updated in place.  Records: rec_step[r],
 * rec_sig0[r] (d*d complex), rec_sinks[r] (n_sinks); rec_cap records at most.
 * Returns the stop code; *n_rec and *n_steps report what happened.  A diverged
 * run returns OR_DIVERGED with *n_steps = the step whose guard fired.
 */
int or_propagate(const or_ops* op, const or_run* rp, double* sig, double* sink_pops,
                 int64_t rec_cap, int64_t* rec_step, double* rec_sig0, double* rec_sinks,
                 int64_t* n_rec, int64_t* n_steps) {
    const int d = op->d;
    const int64_t n = op->n_tot * d * d;  /* complex elements */
    const int64_t mat2 = 2LL * d * d;
    double* k1 = (double*)malloc(sizeof(double) * 2 * n);
    double* k2 = (double*)malloc(sizeof(double) * 2 * n);
    double* k3 = (double*)malloc(sizeof(double) * 2 * n);
    double* k4 = (double*)malloc(sizeof(double) * 2 * n);
    double* tmp = (double*)malloc(sizeof(double) * 2 * n);
    const double dt = rp->dt;
    const double blow2 = rp->blowup_norm * rp->blowup_norm;
    double r1[16], r2[16], r3[16], r4[16];
    int64_t nr = 0, step = 0;
    int code = OR_OK;

#define RECORD()                                                               \
    do {                                                                       \
        if (nr >= rec_cap) { code = OR_CAPACITY; goto done; }                  \
        rec_step[nr] = step;                                                   \
        memcpy(rec_sig0 + nr * mat2, sig, sizeof(double) * mat2);              \
        for (int s_ = 0; s_ < rp->n_sinks; ++s_)                               \
            rec_sinks[nr * rp->n_sinks + s_] = sink_pops[s_];                  \
        ++nr;                                                                  \
    } while (0)

    RECORD();
    for (;;) {
        const double t = (double)step * dt;
        if (rp->has_t_end && t >= rp->t_end - 1e-9) { code = OR_T_END; break; }
        if (rp->has_residual && system_population(rp, sig, d) <= rp->residual) {
            code = OR_RESIDUAL; break;
        }
        if (!rp->has_t_end && t >= rp->hard_cap) { code = OR_HARDCAP; goto done; }
        if (step >= rp->max_steps) { code = OR_CAPACITY; goto done; }

        or_rhs(op, sig, k1);
        sink_rates(rp, sig, d, r1);
        or_add_scaled(n, tmp, sig, k1, 0.5 * dt);
        or_rhs(op, tmp, k2);
        sink_rates(rp, tmp, d, r2);
        or_add_scaled(n, tmp, sig, k2, 0.5 * dt);
        or_rhs(op, tmp, k3);
        sink_rates(rp, tmp, d, r3);
        or_add_scaled(n, tmp, sig, k3, dt);
        or_rhs(op, tmp, k4);
        sink_rates(rp, tmp, d, r4);
        or_rk4_update(n, sig, k1, k2, k3, k4, dt / 6.0);
        for (int s = 0; s < rp->n_sinks; ++s)
            sink_pops[s] += (dt / 6.0) * (r1[s] + 2.0 * (r2[s] + r3[s]) + r4[s]);
        step += 1;
        if (or_max_abs2(d * d, sig) > blow2 ||
            (step % 25 == 0 && or_max_abs2(n, sig) > blow2)) {
            code = OR_DIVERGED; goto done;
        }
        if (step % rp->stride == 0) RECORD();
    }
    if (step % rp->stride != 0) RECORD();
done:
#undef RECORD
    *n_rec = nr;
    *n_steps = step;
    free(k1); free(k2); free(k3); free(k4); free(tmp);
    return code;
}
