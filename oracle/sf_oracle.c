/*
 * sf_oracle.c -- CPU restatement (f64) of the reference's wave-propagator hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  The product (paper_1808_01995_b200/) never links or calls it.
 *
 * Parity status: PINNED.  The functions below are checked (tests/test_oracle_pins.py)
 * against every known-answer the reference's own tests hold for this path
 * and against outputs of the reference's own sources compiled
 * in place (oracle/_ref, fixtures under tests/golden/, generator oracle/make_golden.py).
 * The TTI functions at the bottom have NO reference counterpart: parity unpinned.
 *
 * Each function cites the reference file:line (relative to /root/reference/proj) whose
 * meaning it follows.  Nothing here is copied: the reference describes its operators
 * symbolically and generates loop nests at run time; this file writes those loop nests
 * out by hand from the pinned closed form (tests/test_compiler.cpp:80-91).
 *
 * Conventions (reference): axes d0,d1,d2 = x,y,z row-major, d2 contiguous
 * (include/sf/function.hpp:15-17); metres, milliseconds, m/ms.  Ranks 1..3 are
 * embedded in 3-D by prepending unit axes, so axis a of a rank-r grid is internal
 * axis 3-r+a.  Corner index c uses reference axis 0 as least-significant bit
 * (include/sf/sparse.hpp:23-25).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

typedef struct {
    int ndim;          /* 1..3 */
    long n[3];         /* computational (padded) extents, reference axis order */
    double h[3];       /* spacing per reference axis */
    int space_order;   /* k, even */
    double dt;
    long nt;
    const double *w2;  /* second-derivative weights w_0..w_K (centre first) */
} sfo_grid;

int sfo_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void sfo_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ---- internal 3-D embedding ------------------------------------------------------- */

typedef struct {
    long N[3];     /* internal extents (unit for absent axes) */
    double ih2[3]; /* 1/h^2, 0 for absent axes */
    int act[3];
    int K;
    long P[3];     /* haloed extents */
    long s0, s1;   /* haloed strides */
    size_t total;  /* haloed element count */
} emb3;

static void embed(const sfo_grid *g, emb3 *e) {
    int off = 3 - g->ndim;
    e->K = g->space_order / 2;
    for (int d = 0; d < 3; ++d) {
        e->N[d] = 1;
        e->ih2[d] = 0.0;
        e->act[d] = 0;
    }
    for (int a = 0; a < g->ndim; ++a) {
        e->N[off + a] = g->n[a];
        e->ih2[off + a] = 1.0 / (g->h[a] * g->h[a]);
        e->act[off + a] = 1;
    }
    for (int d = 0; d < 3; ++d) e->P[d] = e->N[d] + (e->act[d] ? 2 * e->K : 0);
    e->s1 = e->P[2];
    e->s0 = e->P[1] * e->P[2];
    e->total = (size_t)e->P[0] * (size_t)e->P[1] * (size_t)e->P[2];
}

static inline size_t hidx(const emb3 *e, long i, long j, long l) {
    return (size_t)(i + (e->act[0] ? e->K : 0)) * (size_t)e->s0 +
           (size_t)(j + (e->act[1] ? e->K : 0)) * (size_t)e->s1 +
           (size_t)(l + (e->act[2] ? e->K : 0));
}

/* ---- model: include/sf/model.hpp, src/model.cpp ------------------------------------ */

/* Edge-clamped extension of physical velocities into the absorbing layer, m = 1/v^2.
 * Follows src/model.cpp:80-101 (set_velocity).  Output is compact [N0][N1][N2] with
 * N_d = n_d + 2*nbl.  Returns 0, or 1 if a velocity is not positive. */
int sfo_pad_slowness(int ndim, const long *nphys, long nbl, const double *vel,
                     double *m_out, double *vmin, double *vmax) {
    long np[3] = {1, 1, 1}, N[3] = {1, 1, 1};
    int off = 3 - ndim;
    size_t cnt = 1;
    for (int a = 0; a < ndim; ++a) {
        np[off + a] = nphys[a];
        N[off + a] = nphys[a] + 2 * nbl;
        cnt *= (size_t)nphys[a];
    }
    double lo = vel[0], hi = vel[0];
    for (size_t i = 0; i < cnt; ++i) {
        if (!(vel[i] > 0.0)) return 1;
        if (vel[i] < lo) lo = vel[i];
        if (vel[i] > hi) hi = vel[i];
    }
    if (vmin) *vmin = lo;
    if (vmax) *vmax = hi;
    long pad[3];
    for (int d = 0; d < 3; ++d) pad[d] = (d >= off) ? nbl : 0;
#pragma omp parallel for collapse(2) schedule(static)
    for (long i = 0; i < N[0]; ++i)
        for (long j = 0; j < N[1]; ++j) {
            long pi = i - pad[0], pj = j - pad[1];
            pi = pi < 0 ? 0 : (pi > np[0] - 1 ? np[0] - 1 : pi);
            pj = pj < 0 ? 0 : (pj > np[1] - 1 ? np[1] - 1 : pj);
            for (long l = 0; l < N[2]; ++l) {
                long pl = l - pad[2];
                pl = pl < 0 ? 0 : (pl > np[2] - 1 ? np[2] - 1 : pl);
                double v = vel[((size_t)pi * np[1] + pj) * np[2] + pl];
                m_out[((size_t)i * N[1] + j) * N[2] + l] = 1.0 / (v * v);
            }
        }
    return 0;
}

/* Same extension applied to squared-slowness values stored verbatim
 * (src/model.cpp:124-147, set_physical_m). */
void sfo_pad_m(int ndim, const long *nphys, long nbl, const double *m_phys, double *m_out) {
    long np[3] = {1, 1, 1}, N[3] = {1, 1, 1};
    int off = 3 - ndim;
    for (int a = 0; a < ndim; ++a) {
        np[off + a] = nphys[a];
        N[off + a] = nphys[a] + 2 * nbl;
    }
    long pad[3];
    for (int d = 0; d < 3; ++d) pad[d] = (d >= off) ? nbl : 0;
    for (long i = 0; i < N[0]; ++i)
        for (long j = 0; j < N[1]; ++j)
            for (long l = 0; l < N[2]; ++l) {
                long pi = i - pad[0], pj = j - pad[1], pl = l - pad[2];
                pi = pi < 0 ? 0 : (pi > np[0] - 1 ? np[0] - 1 : pi);
                pj = pj < 0 ? 0 : (pj > np[1] - 1 ? np[1] - 1 : pj);
                pl = pl < 0 ? 0 : (pl > np[2] - 1 ? np[2] - 1 : pl);
                m_out[((size_t)i * N[1] + j) * N[2] + l] =
                    m_phys[((size_t)pi * np[1] + pj) * np[2] + pl];
            }
}

/* Absorbing mask, src/model.cpp:35-56 (build_damping): separable sum over axes of
 * eta_max_d * ramp((nbl - dist)/nbl) where dist < nbl; ramp = w (linear=1) or w^2.
 * Returns 1 when nbl violates nbl < (N_d+1)/2 (src/model.cpp:40-42). */
int sfo_build_damping(int ndim, const long *N, const double *h, long nbl, double v_max,
                      int linear, double *damp_out) {
    if (nbl < 0) return 1;
    for (int a = 0; a < ndim; ++a)
        if (nbl >= (N[a] + 1) / 2) return 1;
    long M[3] = {1, 1, 1};
    double hh[3] = {1, 1, 1};
    int act[3] = {0, 0, 0};
    int off = 3 - ndim;
    for (int a = 0; a < ndim; ++a) {
        M[off + a] = N[a];
        hh[off + a] = h[a];
        act[off + a] = 1;
    }
    size_t cnt = (size_t)M[0] * M[1] * M[2];
    if (nbl == 0) {
        memset(damp_out, 0, cnt * sizeof(double));
        return 0;
    }
    const double eta_gain = v_max * log(1000.0);
    for (long i = 0; i < M[0]; ++i)
        for (long j = 0; j < M[1]; ++j)
            for (long l = 0; l < M[2]; ++l) {
                long idx[3] = {i, j, l};
                double eta = 0.0;
                for (int d = 0; d < 3; ++d) {
                    if (!act[d]) continue;
                    double eta_max = eta_gain / ((double)nbl * hh[d]);
                    long dist = idx[d] < M[d] - 1 - idx[d] ? idx[d] : M[d] - 1 - idx[d];
                    if (dist < nbl) {
                        double w = (double)(nbl - dist) / (double)nbl;
                        eta += eta_max * (linear ? w : w * w);
                    }
                }
                damp_out[((size_t)i * M[1] + j) * M[2] + l] = eta;
            }
    return 0;
}

/* CFL bound, src/model.cpp:103-111: gamma*h_min*sqrt(1/vmax^2)/sqrt(ndim*sum|w|/2),
 * w = all 2K+1 second-derivative weights. */
double sfo_critical_dt(int ndim, const double *h, double v_max, int space_order,
                       const double *w2, double gamma) {
    int K = space_order / 2;
    double wsum = fabs(w2[0]);
    for (int j = 1; j <= K; ++j) wsum += 2.0 * fabs(w2[j]);
    double h_min = h[0];
    for (int a = 1; a < ndim; ++a)
        if (h[a] < h_min) h_min = h[a];
    double m_min = 1.0 / (v_max * v_max);
    return gamma * h_min * sqrt(m_min) / sqrt((double)ndim * wsum / 2.0);
}

/* ---- wavelet / geometry: include/sf/wavelet.hpp:12-24, src/geometry.cpp:26-33 ------ */

void sfo_ricker(double f0, double t0, double dt, long nt, double *out) {
    for (long i = 0; i < nt; ++i) {
        double tau = (t0 + (double)i * dt) - 1.0 / f0;
        double a = M_PI * M_PI * f0 * f0 * tau * tau;
        out[i] = (1.0 - 2.0 * a) * exp(-a);
    }
}

long sfo_num_samples(double t0, double tn, double dt) { /* src/geometry.cpp:26 */
    return (long)floor((tn - t0) / dt) + 1;
}

/* ---- sparse points: src/sparse.cpp:36-70 (locate) ---------------------------------- */

/* coords [np][ndim]; base [np][ndim]; w [np][2^ndim].  Returns 0, or 1+p for the
 * first point outside the domain (LocationError in the reference). */
long sfo_locate(int ndim, const long *N, const double *h, const double *origin, long np,
                const double *coords, long *base, double *w) {
    int nc = 1 << ndim;
    for (long p = 0; p < np; ++p) {
        double frac[3];
        for (int d = 0; d < ndim; ++d) {
            double rel = (coords[p * ndim + d] - origin[d]) / h[d];
            double last = (double)(N[d] - 1);
            double tol = 1e-9 * (last > 1.0 ? last : 1.0);
            if (rel < -tol || rel > last + tol) return 1 + p;
            if (rel < 0) rel = 0;
            if (rel > last) rel = last;
            long b = (long)floor(rel);
            if (b > N[d] - 2) b = N[d] - 2;
            base[p * ndim + d] = b;
            frac[d] = rel - (double)b;
        }
        for (int c = 0; c < nc; ++c) {
            double ww = 1.0;
            for (int d = 0; d < ndim; ++d) ww *= ((c >> d) & 1) ? frac[d] : 1.0 - frac[d];
            w[p * nc + c] = ww;
        }
    }
    return 0;
}

/* ---- time stepping ------------------------------------------------------------------ */

/* One dense update, all computational nodes: the closed form pinned at
 * tests/test_compiler.cpp:80,84 and restated in SURVEY.md Appendix B step 1.
 *   out = ( L(cur) - m*(old - 2 cur)/dt^2 + 1/2 damp*old/dt ) * inv0
 * cur/old/out are haloed arrays (zero halo = the reference's Dirichlet reads,
 * include/sf/function.hpp:17); m/damp/inv0 are compact. */
/* one row of the dense update with the halo width known at compile time (inlined into the
 * switch below, so gcc unrolls the stencil and vectorises along the contiguous axis; the
 * summation order per node is unchanged: centre, then neighbours K..1, axis by axis) */
static inline __attribute__((always_inline)) void dense_row(
    const int K, const long N2, const long s0, const long s1, const int a0, const int a1,
    const int a2, const double *ih2, const double *w2, const double s0dt, const double s1dt,
    const double *restrict cur, const double *restrict old, double *restrict out,
    const double *restrict m, const double *restrict damp, const double *restrict inv0) {
#pragma omp simd
    for (long l = 0; l < N2; ++l) {
        double lap = 0.0;
        if (a0) {
            double acc = w2[0] * cur[l];
            for (int jj = K; jj >= 1; --jj) acc += w2[jj] * (cur[l - jj * s0] + cur[l + jj * s0]);
            lap += acc * ih2[0];
        }
        if (a1) {
            double acc = w2[0] * cur[l];
            for (int jj = K; jj >= 1; --jj) acc += w2[jj] * (cur[l - jj * s1] + cur[l + jj * s1]);
            lap += acc * ih2[1];
        }
        if (a2) {
            double acc = w2[0] * cur[l];
            for (int jj = K; jj >= 1; --jj) acc += w2[jj] * (cur[l - jj] + cur[l + jj]);
            lap += acc * ih2[2];
        }
        double v = -1.0 * (-1.0 * lap + m[l] * (old[l] + (-2.0) * cur[l]) * s1dt +
                           (-0.5) * damp[l] * old[l] * s0dt);
        out[l] = v * inv0[l];
    }
}

static void dense_update(const emb3 *e, const double *w2, double dt, const double *cur,
                         const double *old, double *out, const double *m,
                         const double *damp, const double *inv0) {
    const int K = e->K;
    const double s0 = 1.0 / dt, s1 = 1.0 / (dt * dt);
    const long N0 = e->N[0], N1 = e->N[1], N2 = e->N[2];
#pragma omp parallel for collapse(2) schedule(static)
    for (long i = 0; i < N0; ++i)
        for (long j = 0; j < N1; ++j) {
            size_t row = hidx(e, i, j, 0);
            size_t crow = ((size_t)i * N1 + j) * N2;
#define SFO_ROW(KK)                                                                          \
    dense_row(KK, N2, e->s0, e->s1, e->act[0], e->act[1], e->act[2], e->ih2, w2, s0, s1,     \
              cur + row, old + row, out + row, m + crow, damp + crow, inv0 + crow)
            switch (K) {
            case 1: SFO_ROW(1); break;
            case 2: SFO_ROW(2); break;
            case 3: SFO_ROW(3); break;
            case 4: SFO_ROW(4); break;
            case 5: SFO_ROW(5); break;
            case 6: SFO_ROW(6); break;
            case 7: SFO_ROW(7); break;
            case 8: SFO_ROW(8); break;
            default: SFO_ROW(K); break;
            }
#undef SFO_ROW
        }
}

/* Scatter: src/sparse.cpp:138-150 as used at src/seismic_ops.cpp:74-76; serial,
 * point-major / corner-minor (src/lower.cpp:198); weight dt^2/m at the corner node
 * (tests/test_compiler.cpp:86-89). */
static void inject_points(const emb3 *e, int ndim, double dt, long np, const long *base,
                          const double *w, const double *trace_row, double *field,
                          const double *m) {
    const int nc = 1 << ndim, off = 3 - ndim;
    const double s4 = dt * dt;
    for (long p = 0; p < np; ++p)
        for (int c = 0; c < nc; ++c) {
            long id[3] = {0, 0, 0};
            for (int a = 0; a < ndim; ++a) id[off + a] = base[p * ndim + a] + ((c >> a) & 1);
            size_t cm = ((size_t)id[0] * e->N[1] + id[1]) * e->N[2] + id[2];
            field[hidx(e, id[0], id[1], id[2])] += trace_row[p] * w[p * nc + c] * s4 * (1.0 / m[cm]);
        }
}

/* Gather: src/sparse.cpp:130-136 as used at src/seismic_ops.cpp:77. */
static void sample_points(const emb3 *e, int ndim, long np, const long *base, const double *w,
                          const double *field, double *trace_row) {
    const int nc = 1 << ndim, off = 3 - ndim;
#pragma omp parallel for schedule(static) if (np > 4096)
    for (long p = 0; p < np; ++p) {
        double s = 0.0;
        for (int c = 0; c < nc; ++c) {
            long id[3] = {0, 0, 0};
            for (int a = 0; a < ndim; ++a) id[off + a] = base[p * ndim + a] + ((c >> a) & 1);
            s += w[p * nc + c] * field[hidx(e, id[0], id[1], id[2])];
        }
        trace_row[p] = s;
    }
}

static void compact_copy(const emb3 *e, const double *haloed, double *compact) {
    for (long i = 0; i < e->N[0]; ++i)
        for (long j = 0; j < e->N[1]; ++j)
            memcpy(compact + ((size_t)i * e->N[1] + j) * e->N[2], haloed + hidx(e, i, j, 0),
                   (size_t)e->N[2] * sizeof(double));
}

static int all_finite(const double *p, size_t n) {
    int ok = 1;
#pragma omp parallel for reduction(&& : ok) schedule(static)
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(p[i])) ok = 0;
    return ok;
}

/* hoisted invariant of src/passes.cpp:168-183: inv0 = 1/(m/dt^2 + damp/(2dt)) */
static double *make_inv0(const emb3 *e, double dt, const double *m, const double *damp) {
    size_t cnt = (size_t)e->N[0] * e->N[1] * e->N[2];
    double *inv0 = (double *)malloc(cnt * sizeof(double));
    if (!inv0) return NULL;
    const double s0 = 1.0 / dt, s1 = 1.0 / (dt * dt);
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < cnt; ++i) inv0[i] = 1.0 / (m[i] * s1 + 0.5 * damp[i] * s0);
    return inv0;
}

/*
 * Forward / adjoint sweep: src/seismic_ops.cpp:58-107 + run_wave :137-141 +
 * run_window :44-54 (window [1, nt-1)), time slots t mod 3 (src/execute.cpp:187-199).
 *
 * direction = +1: forward_operator.  for t = 1..nt-2:  u[t+1] = update(u[t], u[t-1]);
 *                 inject inj_tr[t] at the inj cloud into u[t+1]; smp_tr[t] = P u[t].
 * direction = -1: adjoint_operator.  for t = nt-2..1:  v[t-1] = update(v[t], v[t+1]);
 *                 inject inj_tr[t] (receiver traces) into v[t-1]; smp_tr[t] = P v[t].
 * (the adjoint PDE flips the damping sign and solves for t-1, which yields the same
 *  algebraic update with the roles of the outer levels swapped: SURVEY.md a10.)
 *
 * smp_tr [nt][nsmp] is zeroed first.  Optional outputs (may be NULL):
 *   final_a  compact copy of the last level written (forward: level nt-1; adjoint: 0)
 *   final_b  compact copy of the level before it    (forward: nt-2;       adjoint: 1)
 *   snaps    forward only: compact copies of levels t with t % save_every == 0,
 *            stored at index t / save_every  (save_every = 1 is the reference's
 *            save=true history, src/seismic_ops.cpp:66-68); needs
 *            ((nt-1)/save_every + 1) slots.
 * Returns 0, 2 on a non-finite field (StabilityError, src/emit.cpp:333-341),
 * 3 on allocation failure.
 */
int sfo_propagate(const sfo_grid *g, int direction, const double *m, const double *damp,
                  long ninj, const long *inj_base, const double *inj_w, const double *inj_tr,
                  long nsmp, const long *smp_base, const double *smp_w, double *smp_tr,
                  double *final_a, double *final_b, double *snaps, long save_every) {
    emb3 e;
    embed(g, &e);
    const long nt = g->nt;
    size_t cnt = (size_t)e.N[0] * e.N[1] * e.N[2];
    double *buf[3];
    for (int s = 0; s < 3; ++s) {
        buf[s] = (double *)calloc(e.total, sizeof(double));
        if (!buf[s]) return 3;
    }
    double *inv0 = make_inv0(&e, g->dt, m, damp);
    if (!inv0) return 3;
    memset(smp_tr, 0, (size_t)nt * (size_t)nsmp * sizeof(double));
    if (snaps && direction > 0) {
        long nslots = (nt - 1) / save_every + 1;
        memset(snaps, 0, (size_t)nslots * cnt * sizeof(double));
    }
    if (direction > 0) {
        for (long t = 1; t < nt - 1; ++t) {
            double *cur = buf[t % 3], *old = buf[(t - 1) % 3], *out = buf[(t + 1) % 3];
            dense_update(&e, g->w2, g->dt, cur, old, out, m, damp, inv0);
            inject_points(&e, g->ndim, g->dt, ninj, inj_base, inj_w, inj_tr + (size_t)t * ninj,
                          out, m);
            sample_points(&e, g->ndim, nsmp, smp_base, smp_w, cur, smp_tr + (size_t)t * nsmp);
            if (snaps && (t + 1) % save_every == 0)
                compact_copy(&e, out, snaps + (size_t)((t + 1) / save_every) * cnt);
        }
        if (final_a) compact_copy(&e, buf[(nt - 1) % 3], final_a);
        if (final_b) compact_copy(&e, buf[(nt - 2) % 3], final_b);
    } else {
        for (long t = nt - 2; t >= 1; --t) {
            double *cur = buf[t % 3], *old = buf[(t + 1) % 3], *out = buf[(t - 1) % 3];
            dense_update(&e, g->w2, g->dt, cur, old, out, m, damp, inv0);
            inject_points(&e, g->ndim, g->dt, ninj, inj_base, inj_w, inj_tr + (size_t)t * ninj,
                          out, m);
            sample_points(&e, g->ndim, nsmp, smp_base, smp_w, cur, smp_tr + (size_t)t * nsmp);
        }
        if (final_a) compact_copy(&e, buf[0], final_a);
        if (final_b) compact_copy(&e, buf[1 % 3], final_b);
    }
    int ok = 1;
    for (int s = 0; s < 3; ++s) ok = ok && all_finite(buf[s], e.total);
    for (int s = 0; s < 3; ++s) free(buf[s]);
    free(inv0);
    return ok ? 0 : 2;
}

/*
 * Gradient sweep: src/seismic_ops.cpp:109-135 + run_gradient :143-147.
 * for t = nt-2..1: v[t-1] = update(v[t], v[t+1]); inject resid[t] into v[t-1]; then, in
 * a separate dense nest that sees the injected v[t-1] (src/lower.cpp:136-142):
 *     grad -= u_saved[t] * (v[t-1] - 2 v[t] + v[t+1]) / dt^2        (:132)
 * snaps holds forward levels t % save_every == 0 at index t/save_every; imaging runs
 * on those levels only (save_every = 1 is the reference).  grad_out: compact padded
 * grid [N0][N1][N2], zeroed first.
 */
int sfo_gradient(const sfo_grid *g, const double *m, const double *damp, long nrec,
                 const long *rec_base, const double *rec_w, const double *resid,
                 const double *snaps, long save_every, double *grad_out) {
    emb3 e;
    embed(g, &e);
    const long nt = g->nt;
    size_t cnt = (size_t)e.N[0] * e.N[1] * e.N[2];
    double *buf[3];
    for (int s = 0; s < 3; ++s) {
        buf[s] = (double *)calloc(e.total, sizeof(double));
        if (!buf[s]) return 3;
    }
    double *inv0 = make_inv0(&e, g->dt, m, damp);
    if (!inv0) return 3;
    memset(grad_out, 0, cnt * sizeof(double));
    const double s1 = 1.0 / (g->dt * g->dt);
    for (long t = nt - 2; t >= 1; --t) {
        double *cur = buf[t % 3], *old = buf[(t + 1) % 3], *out = buf[(t - 1) % 3];
        dense_update(&e, g->w2, g->dt, cur, old, out, m, damp, inv0);
        inject_points(&e, g->ndim, g->dt, nrec, rec_base, rec_w, resid + (size_t)t * nrec, out, m);
        if (t % save_every != 0) continue;
        const double *us = snaps + (size_t)(t / save_every) * cnt;
#pragma omp parallel for collapse(2) schedule(static)
        for (long i = 0; i < e.N[0]; ++i)
            for (long j = 0; j < e.N[1]; ++j) {
                size_t row = hidx(&e, i, j, 0);
                size_t crow = ((size_t)i * e.N[1] + j) * e.N[2];
                for (long l = 0; l < e.N[2]; ++l) {
                    size_t q = row + l;
                    grad_out[crow + l] -= us[crow + l] * ((out[q] - 2.0 * cur[q] + old[q]) * s1);
                }
            }
    }
    int ok = 1;
    for (int s = 0; s < 3; ++s) ok = ok && all_finite(buf[s], e.total);
    for (int s = 0; s < 3; ++s) free(buf[s]);
    free(inv0);
    return ok ? 0 : 2;
}

/* src/seismic_ops.cpp:149-160 */
double sfo_objective(long n, const double *pred, const double *observed) {
    double phi = 0.0;
    for (long i = 0; i < n; ++i) {
        double r = pred[i] - observed[i];
        phi += 0.5 * r * r;
    }
    return phi;
}

/* Adjoint of the edge extension, src/seismic_ops.cpp:166-193: every padded cell's value
 * is summed onto clamp(idx - nbl, 0, n-1), visiting padded cells in row-major order. */
void sfo_fold_gradient(int ndim, const long *nphys, long nbl, const double *grad_padded,
                       double *out) {
    long np[3] = {1, 1, 1}, N[3] = {1, 1, 1}, pad[3] = {0, 0, 0};
    int off = 3 - ndim;
    size_t cnt = 1;
    for (int a = 0; a < ndim; ++a) {
        np[off + a] = nphys[a];
        N[off + a] = nphys[a] + 2 * nbl;
        pad[off + a] = nbl;
        cnt *= (size_t)nphys[a];
    }
    memset(out, 0, cnt * sizeof(double));
    for (long i = 0; i < N[0]; ++i)
        for (long j = 0; j < N[1]; ++j)
            for (long l = 0; l < N[2]; ++l) {
                long pi = i - pad[0], pj = j - pad[1], pl = l - pad[2];
                pi = pi < 0 ? 0 : (pi > np[0] - 1 ? np[0] - 1 : pi);
                pj = pj < 0 ? 0 : (pj > np[1] - 1 ? np[1] - 1 : pj);
                pl = pl < 0 ? 0 : (pl > np[2] - 1 ? np[2] - 1 : pl);
                out[((size_t)pi * np[1] + pj) * np[2] + pl] +=
                    grad_padded[((size_t)i * N[1] + j) * N[2] + l];
            }
}

/*
 * Bare dense stepping for the CPU throughput baseline (the recipe of
 * src/verify.cpp:338-376 `bench`: update only, no points).  Runs `steps` updates on a
 * seeded non-zero state and returns nothing; the caller times it.
 */
int sfo_dense_steps(const sfo_grid *g, const double *m, const double *damp, long steps,
                    double *state_cur, double *state_old) {
    emb3 e;
    embed(g, &e);
    double *buf[3];
    for (int s = 0; s < 3; ++s) {
        buf[s] = (double *)calloc(e.total, sizeof(double));
        if (!buf[s]) return 3;
    }
    for (long i = 0; i < e.N[0]; ++i)
        for (long j = 0; j < e.N[1]; ++j) {
            size_t c = ((size_t)i * e.N[1] + j) * e.N[2];
            memcpy(buf[1] + hidx(&e, i, j, 0), state_cur + c, (size_t)e.N[2] * sizeof(double));
            memcpy(buf[0] + hidx(&e, i, j, 0), state_old + c, (size_t)e.N[2] * sizeof(double));
        }
    double *inv0 = make_inv0(&e, g->dt, m, damp);
    if (!inv0) return 3;
    for (long t = 1; t <= steps; ++t)
        dense_update(&e, g->w2, g->dt, buf[t % 3], buf[(t - 1) % 3], buf[(t + 1) % 3], m, damp,
                     inv0);
    compact_copy(&e, buf[(steps + 1) % 3], state_cur);
    compact_copy(&e, buf[steps % 3], state_old);
    for (int s = 0; s < 3; ++s) free(buf[s]);
    free(inv0);
    return 0;
}

/* ====================================================================================
 * TTI forward (pseudo-acoustic, rotated Laplacian).  NO REFERENCE COUNTERPART: the
 * reference has no anisotropic operator, so this restates the builder's
 * own formulation and its parity is UNPINNED by the reference.
 *
 *   m p_tt + damp p_t = (1+2 eps) H0(p) + sqrt(1+2 delta) Hz(r)
 *   m r_tt + damp r_t = sqrt(1+2 delta) H0(p) + Hz(r)
 *   g(f)  = a D0 f + b D1 f + c D2 f,      (a,b,c) = (sin th cos ph, sin th sin ph, cos th)
 *   Hz(f) = D0(a g) + D1(b g) + D2(c g)    ( = -Dbar^T Dbar f: negative semi-definite )
 *   H0(f) = L(f) - Hz(f),                   L = the acoustic order-k Laplacian
 * D_i = centred order-k first derivative on axis i (weights w1_1..w1_K, antisymmetric),
 * every field restricted to the grid with zero outside (the reference's halo convention).
 * Time discretisation, damping, injection (into p and r, weight dt^2/m) and sampling (of
 * p) are the acoustic operator's (Appendix B).  With eps = delta = theta = phi = 0 the
 * two equations coincide and p = r follows the acoustic update exactly.
 * ==================================================================================== */

typedef struct {
    const double *eps, *delta, *theta, *phi; /* compact [N0][N1][N2] */
    const double *w1;                        /* first-derivative weights w1_1..w1_K */
} sfo_tti;

static void tti_g(const emb3 *e, const double *w1, const double *f, const double *a,
                  const double *b, const double *c, double *g /* haloed */) {
    const int K = e->K;
    const long st[3] = {e->s0, e->s1, 1};
    const double ih[3] = {sqrt(e->ih2[0]), sqrt(e->ih2[1]), sqrt(e->ih2[2])};
#pragma omp parallel for collapse(2) schedule(static)
    for (long i = 0; i < e->N[0]; ++i)
        for (long j = 0; j < e->N[1]; ++j) {
            size_t row = hidx(e, i, j, 0), crow = ((size_t)i * e->N[1] + j) * e->N[2];
            for (long l = 0; l < e->N[2]; ++l) {
                size_t q = row + l;
                double d[3] = {0, 0, 0};
                for (int ax = 0; ax < 3; ++ax) {
                    if (!e->act[ax]) continue;
                    double s = 0.0;
                    for (int jj = 1; jj <= K; ++jj)
                        s += w1[jj - 1] * (f[q + jj * st[ax]] - f[q - jj * st[ax]]);
                    d[ax] = s * ih[ax];
                }
                g[q] = a[crow + l] * d[0] + b[crow + l] * d[1] + c[crow + l] * d[2];
            }
        }
}

/* hz = D0(a g) + D1(b g) + D2(c g); abc are haloed copies so neighbours outside read 0 */
static void tti_hz(const emb3 *e, const double *w1, const double *g, const double *ah,
                   const double *bh, const double *ch, double *hz /* compact */) {
    const int K = e->K;
    const long st[3] = {e->s0, e->s1, 1};
    const double ih[3] = {sqrt(e->ih2[0]), sqrt(e->ih2[1]), sqrt(e->ih2[2])};
    const double *n[3] = {ah, bh, ch};
#pragma omp parallel for collapse(2) schedule(static)
    for (long i = 0; i < e->N[0]; ++i)
        for (long j = 0; j < e->N[1]; ++j) {
            size_t row = hidx(e, i, j, 0), crow = ((size_t)i * e->N[1] + j) * e->N[2];
            for (long l = 0; l < e->N[2]; ++l) {
                size_t q = row + l;
                double acc = 0.0;
                for (int ax = 0; ax < 3; ++ax) {
                    if (!e->act[ax]) continue;
                    double s = 0.0;
                    for (int jj = 1; jj <= K; ++jj) {
                        size_t qp = q + jj * st[ax], qm = q - jj * st[ax];
                        s += w1[jj - 1] * (n[ax][qp] * g[qp] - n[ax][qm] * g[qm]);
                    }
                    acc += s * ih[ax];
                }
                hz[crow + l] = acc;
            }
        }
}

static void to_haloed(const emb3 *e, const double *compact, double *haloed) {
    memset(haloed, 0, e->total * sizeof(double));
    for (long i = 0; i < e->N[0]; ++i)
        for (long j = 0; j < e->N[1]; ++j)
            memcpy(haloed + hidx(e, i, j, 0), compact + ((size_t)i * e->N[1] + j) * e->N[2],
                   (size_t)e->N[2] * sizeof(double));
}

/* TTI forward sweep over [1, nt-1).  src [nt][nsrc] injected into p and r, rec [nt][nrec]
 * samples p.  Optional outputs: final_p / final_r = level nt-1 (compact); energy [nt] =
 * sum p^2 + r^2 per level written (growth / dissipation checks).  Returns 0 / 2 / 3. */
int sfo_tti_forward(const sfo_grid *g, const sfo_tti *t, const double *m, const double *damp,
                    long nsrc, const long *src_base, const double *src_w, const double *src_tr,
                    long nrec, const long *rec_base, const double *rec_w, double *rec_tr,
                    double *final_p, double *final_r, double *energy) {
    emb3 e;
    embed(g, &e);
    const int K = e.K;
    const long nt = g->nt;
    size_t cnt = (size_t)e.N[0] * e.N[1] * e.N[2];
    double *P[3], *R[3];
    for (int s = 0; s < 3; ++s) {
        P[s] = (double *)calloc(e.total, sizeof(double));
        R[s] = (double *)calloc(e.total, sizeof(double));
        if (!P[s] || !R[s]) return 3;
    }
    double *gp = (double *)calloc(e.total, sizeof(double)), *gr = (double *)calloc(e.total, sizeof(double));
    double *ah = (double *)malloc(e.total * sizeof(double)), *bh = (double *)malloc(e.total * sizeof(double));
    double *ch = (double *)malloc(e.total * sizeof(double));
    double *a = (double *)malloc(cnt * sizeof(double)), *b = (double *)malloc(cnt * sizeof(double));
    double *c = (double *)malloc(cnt * sizeof(double));
    double *hzp = (double *)malloc(cnt * sizeof(double)), *hzr = (double *)malloc(cnt * sizeof(double));
    double *inv0 = make_inv0(&e, g->dt, m, damp);
    if (!gp || !gr || !ah || !bh || !ch || !a || !b || !c || !hzp || !hzr || !inv0) return 3;
    for (size_t i = 0; i < cnt; ++i) {
        a[i] = sin(t->theta[i]) * cos(t->phi[i]);
        b[i] = sin(t->theta[i]) * sin(t->phi[i]);
        c[i] = cos(t->theta[i]);
    }
    to_haloed(&e, a, ah);
    to_haloed(&e, b, bh);
    to_haloed(&e, c, ch);
    memset(rec_tr, 0, (size_t)nt * (size_t)nrec * sizeof(double));
    if (energy) memset(energy, 0, (size_t)nt * sizeof(double));
    const double s0 = 1.0 / g->dt, s1 = 1.0 / (g->dt * g->dt);
    const long st[3] = {e.s0, e.s1, 1};
    for (long tt = 1; tt < nt - 1; ++tt) {
        double *pc = P[tt % 3], *po = P[(tt - 1) % 3], *pn = P[(tt + 1) % 3];
        double *rc = R[tt % 3], *ro = R[(tt - 1) % 3], *rn = R[(tt + 1) % 3];
        tti_g(&e, t->w1, pc, a, b, c, gp);
        tti_g(&e, t->w1, rc, a, b, c, gr);
        tti_hz(&e, t->w1, gp, ah, bh, ch, hzp);
        tti_hz(&e, t->w1, gr, ah, bh, ch, hzr);
        double en = 0.0;
#pragma omp parallel for collapse(2) schedule(static) reduction(+ : en)
        for (long i = 0; i < e.N[0]; ++i)
            for (long j = 0; j < e.N[1]; ++j) {
                size_t row = hidx(&e, i, j, 0), crow = ((size_t)i * e.N[1] + j) * e.N[2];
                for (long l = 0; l < e.N[2]; ++l) {
                    size_t q = row + l, k = crow + l;
                    double lap = 0.0;
                    for (int d = 0; d < 3; ++d) {
                        if (!e.act[d]) continue;
                        double acc = g->w2[0] * pc[q];
                        for (int jj = K; jj >= 1; --jj)
                            acc += g->w2[jj] * (pc[q - jj * st[d]] + pc[q + jj * st[d]]);
                        lap += acc * e.ih2[d];
                    }
                    const double h0 = lap - hzp[k];
                    const double e1 = 1.0 + 2.0 * t->eps[k], e2 = sqrt(1.0 + 2.0 * t->delta[k]);
                    const double rhs_p = e1 * h0 + e2 * hzr[k];
                    const double rhs_r = e2 * h0 + hzr[k];
                    pn[q] = (rhs_p - m[k] * (po[q] - 2.0 * pc[q]) * s1 + 0.5 * damp[k] * po[q] * s0) * inv0[k];
                    rn[q] = (rhs_r - m[k] * (ro[q] - 2.0 * rc[q]) * s1 + 0.5 * damp[k] * ro[q] * s0) * inv0[k];
                    en += pn[q] * pn[q] + rn[q] * rn[q];
                }
            }
        inject_points(&e, g->ndim, g->dt, nsrc, src_base, src_w, src_tr + (size_t)tt * nsrc, pn, m);
        inject_points(&e, g->ndim, g->dt, nsrc, src_base, src_w, src_tr + (size_t)tt * nsrc, rn, m);
        sample_points(&e, g->ndim, nrec, rec_base, rec_w, pc, rec_tr + (size_t)tt * nrec);
        if (energy) energy[tt + 1] = en;
    }
    if (final_p) compact_copy(&e, P[(nt - 1) % 3], final_p);
    if (final_r) compact_copy(&e, R[(nt - 1) % 3], final_r);
    int ok = 1;
    for (int s = 0; s < 3; ++s) ok = ok && all_finite(P[s], e.total) && all_finite(R[s], e.total);
    for (int s = 0; s < 3; ++s) {
        free(P[s]);
        free(R[s]);
    }
    free(gp); free(gr); free(ah); free(bh); free(ch); free(a); free(b); free(c);
    free(hzp); free(hzr); free(inv0);
    return ok ? 0 : 2;
}
