/*
 * boris_oracle.c -- TEST INFRASTRUCTURE ONLY (see boris_oracle.h).
 *
 * Scalar double-precision reference for the relativistic Boris push of
 * arXiv 2104.04579 §2.  Each function cites the PAPER.md lines it restates.
 * Deliberately naive: one particle at a time, the paper's p-form, the paper's
 * order of operations, no blocking, no fusion, no vectorisation hints.
 */
#include "boris_oracle.h"

#include <math.h>
#include <stddef.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static void cross(const double a[3], const double b[3], double out[3]) {
    out[0] = a[1] * b[2] - a[2] * b[1];
    out[1] = a[2] * b[0] - a[0] * b[2];
    out[2] = a[0] * b[1] - a[1] * b[0];
}

static double dot(const double a[3], const double b[3]) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

/*
 * Paper §2, "Summarizing, in this method the particle motion is performed in
 * a following procedure" (L175-186), with equations (5), (7), (9), (10), (12),
 * (13).  SURVEY.md §8(c) steps 3-9.
 */
void oracle_boris_step(double r[3], double p[3], double *gamma, double q, double m,
                       double c, const double E[3], const double B[3], double dt) {
    double p_minus[3], p_prime[3], p_plus[3], t[3], s[3], tmp[3];
    double mc = m * c;
    int k;

    /* Step 1, eq. (9): p^- = p^{n-1/2} + qE dt/2. */
    for (k = 0; k < 3; ++k) p_minus[k] = p[k] + q * E[k] * dt / 2.0;

    /* gamma_n = gamma(p^-) = (1 + p^2/(m^2 c^2))^{1/2}  (L162, reading c2). */
    double gamma_n = sqrt(1.0 + dot(p_minus, p_minus) / (mc * mc));

    /* Eq. (13): t = qB/(gamma_n m c) * dt/2;  s = 2t/(1 + t^2). */
    for (k = 0; k < 3; ++k) t[k] = q * B[k] / (gamma_n * m * c) * dt / 2.0;
    double t2 = dot(t, t);
    for (k = 0; k < 3; ++k) s[k] = 2.0 * t[k] / (1.0 + t2);

    /* Step 2, eq. (12): p' = p^- + p^- x t;  p^+ = p^- + p' x s. */
    cross(p_minus, t, tmp);
    for (k = 0; k < 3; ++k) p_prime[k] = p_minus[k] + tmp[k];
    cross(p_prime, s, tmp);
    for (k = 0; k < 3; ++k) p_plus[k] = p_minus[k] + tmp[k];

    /* Step 3, eq. (10): p^{n+1/2} = p^+ + qE dt/2. */
    for (k = 0; k < 3; ++k) p[k] = p_plus[k] + q * E[k] * dt / 2.0;

    /* Step 4: gamma^{n+1/2} from eq. (5) L106-109 (reading c3), v = p/(gamma m),
     * and eq. (7): r^{n+1} = r^n + dt v^{n+1/2}. */
    double g = sqrt(1.0 + dot(p, p) / (mc * mc));
    *gamma = g;
    for (k = 0; k < 3; ++k) r[k] = r[k] + dt * p[k] / (g * m);
}

/* gamma_new of Vay (2008) / Higuera-Cary (2017): the positive root of
 * gamma^4 - sigma gamma^2 - (tau^2 + ustar^2) = 0, sigma = gamma_v^2 - tau^2. */
static double alt_gamma_new(const double v[3], const double tau[3]) {
    double g2 = 1.0 + dot(v, v);
    double tau2 = dot(tau, tau);
    double us = dot(v, tau);
    double sigma = g2 - tau2;
    return sqrt((sigma + sqrt(sigma * sigma + 4.0 * (tau2 + us * us))) / 2.0);
}

/* x = s [v + (v.t) t + v x t], s = 1/(1 + t^2): the solution of x = v + x x t. */
static void alt_implicit_rotation(const double v[3], const double t[3], double x[3]) {
    double s = 1.0 / (1.0 + dot(t, t));
    double vt = dot(v, t), vxt[3];
    int k;
    cross(v, t, vxt);
    for (k = 0; k < 3; ++k) x[k] = s * (v[k] + vt * t[k] + vxt[k]);
}

void oracle_vay_step(double r[3], double p[3], double *gamma, double q, double m, double c,
                     const double E[3], const double B[3], double dt) {
    double u[3], tau[3], uxt[3], up[3], t[3], un[3];
    double mc = m * c;
    int k;
    for (k = 0; k < 3; ++k) {
        u[k] = p[k] / mc;
        tau[k] = q * B[k] * dt / (2.0 * mc);
    }
    double g_old = sqrt(1.0 + dot(u, u));
    double beta[3] = {u[0] / g_old, u[1] / g_old, u[2] / g_old};
    cross(beta, tau, uxt);
    for (k = 0; k < 3; ++k) up[k] = u[k] + q * E[k] * dt / mc + uxt[k];
    double g_new = alt_gamma_new(up, tau);
    for (k = 0; k < 3; ++k) t[k] = tau[k] / g_new;
    alt_implicit_rotation(up, t, un);
    double g = sqrt(1.0 + dot(un, un));
    *gamma = g;
    for (k = 0; k < 3; ++k) {
        p[k] = un[k] * mc;
        r[k] = r[k] + dt * c * un[k] / g;
    }
}

void oracle_hc_step(double r[3], double p[3], double *gamma, double q, double m, double c,
                    const double E[3], const double B[3], double dt) {
    double um[3], tau[3], eps[3], t[3], ub[3], ubxt[3];
    double mc = m * c;
    int k;
    for (k = 0; k < 3; ++k) {
        eps[k] = q * E[k] * dt / (2.0 * mc);
        um[k] = p[k] / mc + eps[k];
        tau[k] = q * B[k] * dt / (2.0 * mc);
    }
    double g_new = alt_gamma_new(um, tau);
    for (k = 0; k < 3; ++k) t[k] = tau[k] / g_new;
    alt_implicit_rotation(um, t, ub);
    cross(ub, t, ubxt);
    double un[3];
    for (k = 0; k < 3; ++k) un[k] = ub[k] + eps[k] + ubxt[k];
    double g = sqrt(1.0 + dot(un, un));
    *gamma = g;
    for (k = 0; k < 3; ++k) {
        p[k] = un[k] * mc;
        r[k] = r[k] + dt * c * un[k] / g;
    }
}

static int g_pusher = ORACLE_PUSHER_BORIS;
void oracle_set_pusher(int pusher) { g_pusher = pusher; }

void oracle_field_uniform(const double *params, double E[3], double B[3]) {
    int k;
    for (k = 0; k < 3; ++k) {
        E[k] = params[k];
        B[k] = params[3 + k];
    }
}

/* Plane wave, reading c-PW: phi = k (khat.r) - omega t + phase0,
 * E = E0 ehat cos(phi), B = khat x E. */
void oracle_field_plane_wave(const double *params, const double r[3], double t,
                             double E[3], double B[3]) {
    double E0 = params[0];
    const double *khat = params + 1;
    const double *ehat = params + 4;
    double omega = params[7], k = params[8], phase0 = params[9];
    double phi = k * dot(khat, r) - omega * t + phase0;
    double a = E0 * cos(phi);
    int i;
    for (i = 0; i < 3; ++i) E[i] = a * ehat[i];
    cross(khat, E, B);
}

/*
 * Radial functions of eq. (15) L418-426 in reading c11/c13.
 *   f1 = sin(xi)/xi^2 - cos(xi)/xi                       (= j1)
 *   f2 = (3/xi^3 - 1/xi) sin(xi) - 3 cos(xi)/xi^2         (= 3 j1/xi - j0)
 *   f3 = (1/xi - 1/xi^3) sin(xi) + cos(xi)/xi^2           (= j0 - j1/xi)
 * Returned: g1 = f1/xi, g2 = f2/xi^2, f3.
 * For xi < xi_star: j0 = sum_n (-1)^n xi^{2n}/(2n+1)!,
 *                   j1/xi = sum_n (-1)^n 2(n+1) xi^{2n}/(2n+3)!, n < n_terms,
 *   g1 = j1/xi,  f3 = j0 - j1/xi,
 *   g2 = sum_{n=1}^{n_terms-1} (-1)^n [6(n+1)/(2n+3)! - 1/(2n+1)!] xi^{2n-2}.
 */
void oracle_mdipole_radial(double xi, double xi_star, int n_terms, double *g1,
                           double *g2, double *f3) {
    if (xi >= xi_star) {
        double sn = sin(xi), cs = cos(xi);
        double f1 = sn / (xi * xi) - cs / xi;
        double f2 = (3.0 / (xi * xi * xi) - 1.0 / xi) * sn - 3.0 * cs / (xi * xi);
        *f3 = (1.0 / xi - 1.0 / (xi * xi * xi)) * sn + cs / (xi * xi);
        *g1 = f1 / xi;
        *g2 = f2 / (xi * xi);
        return;
    }
    double x2 = xi * xi;
    double j0 = 0.0, j1x = 0.0, s2 = 0.0;
    double pw = 1.0; /* xi^{2n} */
    int n;
    for (n = 0; n < n_terms; ++n) {
        /* (2n+1)! and (2n+3)! computed directly, no recurrences shared. */
        double f_2n1 = 1.0, f_2n3;
        int j;
        for (j = 2; j <= 2 * n + 1; ++j) f_2n1 *= (double)j;
        f_2n3 = f_2n1 * (double)(2 * n + 2) * (double)(2 * n + 3);
        double sign = (n % 2 == 0) ? 1.0 : -1.0;
        j0 += sign * pw / f_2n1;
        j1x += sign * 2.0 * (double)(n + 1) * pw / f_2n3;
        pw *= x2;
    }
    /* g2 = (3 j1/xi - j0)/xi^2 term by term (the n = 0 term is exactly 0). */
    pw = 1.0; /* xi^{2n-2} for n = 1 */
    for (n = 1; n < n_terms; ++n) {
        double f_2n1 = 1.0, f_2n3;
        int j;
        for (j = 2; j <= 2 * n + 1; ++j) f_2n1 *= (double)j;
        f_2n3 = f_2n1 * (double)(2 * n + 2) * (double)(2 * n + 3);
        double sign = (n % 2 == 0) ? 1.0 : -1.0;
        s2 += sign * (6.0 * (double)(n + 1) / f_2n3 - 1.0 / f_2n1) * pw;
        pw *= x2;
    }
    *g1 = j1x;
    *g2 = s2;
    *f3 = j0 - j1x;
}

/*
 * Eq. (14) L398-411 in the corrected reading c9/c10, c12 (A0 passed in):
 *   E = 2 A0 cos(w0 t) (f1/R) (-y, x, 0)
 *   Bx = -2 A0 sin(w0 t) (x z/R^2) f2,  By = -2 A0 sin(w0 t) (y z/R^2) f2,
 *   Bz = -2 A0 sin(w0 t) [(z^2/R^2) f2 + f3],
 * evaluated without R in a denominator (c13): f1/R = k g1, f2/R^2 = k^2 g2.
 */
void oracle_field_mdipole(const double *params, const double r[3], double t,
                          double E[3], double B[3]) {
    double A0 = params[0], omega0 = params[1], k = params[2];
    double xi_star = params[3];
    int n_terms = (int)params[4];
    double x = r[0], y = r[1], z = r[2];
    double R = sqrt(x * x + y * y + z * z);
    double g1, g2, f3;
    oracle_mdipole_radial(k * R, xi_star, n_terms, &g1, &g2, &f3);
    double ce = 2.0 * A0 * cos(omega0 * t);
    double sb = -2.0 * A0 * sin(omega0 * t);
    E[0] = ce * k * g1 * (-y);
    E[1] = ce * k * g1 * x;
    E[2] = 0.0;
    B[0] = sb * k * k * g2 * x * z;
    B[1] = sb * k * k * g2 * y * z;
    B[2] = sb * (k * k * g2 * z * z + f3);
}

/* Reading c-grid: CIC (cloud-in-cell, first-order) form factor on a periodic
 * collocated grid.  Along each axis: xi = (x - x0)/dx, i0 = floor(xi), f = xi - i0,
 * weights (1 - f, f) on nodes (i0 mod n, i0 + 1 mod n); the 3D weight of node
 * (a, b, c) is the product of the three 1D weights. */
static int64_t wrap_index(double i, int64_t n) {
    double m = fmod(i, (double)n);
    if (m < 0) m += (double)n;
    return (int64_t)m;
}

void oracle_field_grid(const double *params, const double *gridE, const double *gridB,
                       const double r[3], double E[3], double B[3]) {
    int64_t n[3], idx[3][2];
    double w[3][2];
    int d, a, b, c;
    for (d = 0; d < 3; ++d) {
        n[d] = (int64_t)params[6 + d];
        double xi = (r[d] - params[d]) / params[3 + d];
        double i0 = floor(xi);
        double f = xi - i0;
        w[d][0] = 1.0 - f;
        w[d][1] = f;
        idx[d][0] = wrap_index(i0, n[d]);
        idx[d][1] = wrap_index(i0 + 1.0, n[d]);
    }
    int64_t ncell = n[0] * n[1] * n[2];
    for (d = 0; d < 3; ++d) E[d] = B[d] = 0.0;
    for (c = 0; c < 2; ++c)
        for (b = 0; b < 2; ++b)
            for (a = 0; a < 2; ++a) {
                int64_t node = (idx[2][c] * n[1] + idx[1][b]) * n[0] + idx[0][a];
                double wt = w[0][a] * w[1][b] * w[2][c];
                for (d = 0; d < 3; ++d) {
                    E[d] += wt * gridE[d * ncell + node];
                    B[d] += wt * gridB[d * ncell + node];
                }
            }
}

/* Reading c-dep: direct CIC current deposition at the half-step position. */
void oracle_deposit_current(int64_t n, const double *pos, const double *mom,
                            const double *weight, const int16_t *type, const double *type_q,
                            const double *type_m, double c, double dt, const double *params,
                            double *J) {
    int64_t nn[3], i, node;
    int d, a, b, cc;
    for (d = 0; d < 3; ++d) nn[d] = (int64_t)params[6 + d];
    int64_t ncell = nn[0] * nn[1] * nn[2];
    double vol = params[3] * params[4] * params[5];
    for (i = 0; i < 3 * ncell; ++i) J[i] = 0.0;
    for (i = 0; i < n; ++i) {
        const double *p = mom + 3 * i;
        double m = type_m[type[i]], q = type_q[type[i]];
        double g = sqrt(1.0 + dot(p, p) / (m * c * m * c));
        double v[3], rh[3], w[3][2];
        int64_t idx[3][2];
        for (d = 0; d < 3; ++d) {
            v[d] = p[d] / (g * m);
            rh[d] = pos[3 * i + d] - 0.5 * dt * v[d];
            double xi = (rh[d] - params[d]) / params[3 + d];
            double i0 = floor(xi);
            double f = xi - i0;
            w[d][0] = 1.0 - f;
            w[d][1] = f;
            idx[d][0] = wrap_index(i0, nn[d]);
            idx[d][1] = wrap_index(i0 + 1.0, nn[d]);
        }
        double qw = q * weight[i] / vol;
        for (cc = 0; cc < 2; ++cc)
            for (b = 0; b < 2; ++b)
                for (a = 0; a < 2; ++a) {
                    node = (idx[2][cc] * nn[1] + idx[1][b]) * nn[0] + idx[0][a];
                    double wt = w[0][a] * w[1][b] * w[2][cc];
                    for (d = 0; d < 3; ++d) J[d * ncell + node] += qw * wt * v[d];
                }
    }
}

void oracle_field_at(int kind, const double *params, const double *fieldE,
                     const double *fieldB, int64_t i, const double r[3], double t,
                     double E[3], double B[3]) {
    int k;
    switch (kind) {
    case ORACLE_FIELD_ARRAYS:
        for (k = 0; k < 3; ++k) {
            E[k] = fieldE[3 * i + k];
            B[k] = fieldB[3 * i + k];
        }
        break;
    case ORACLE_FIELD_UNIFORM:
        oracle_field_uniform(params, E, B);
        break;
    case ORACLE_FIELD_PLANE_WAVE:
        oracle_field_plane_wave(params, r, t, E, B);
        break;
    case ORACLE_FIELD_GRID:
        oracle_field_grid(params, fieldE, fieldB, r, E, B);
        break;
    default:
        oracle_field_mdipole(params, r, t, E, B);
        break;
    }
}

/* Paper §4.1 (L256-269): the step loop outside, the particle loop inside,
 * `#pragma omp parallel for` over particles. */
int oracle_push(int64_t n, double *pos, double *mom, double *gamma,
                const int16_t *type, const double *type_q, const double *type_m,
                int32_t n_types, double c, int field_kind, const double *params,
                const double *fieldE, const double *fieldB, double t0, double dt,
                int64_t n_steps, int n_threads) {
    int64_t i, step;
    for (i = 0; i < n; ++i)
        if (type[i] < 0 || type[i] >= n_types) return -1;
#ifdef _OPENMP
    if (n_threads <= 0) n_threads = omp_get_max_threads();
#else
    (void)n_threads;
#endif
    for (step = 0; step < n_steps; ++step) {
        /* t_n = t0 + n dt, computed, not accumulated (c5). */
        double t_n = t0 + (double)step * dt;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(n_threads)
#endif
        for (i = 0; i < n; ++i) {
            double E[3], B[3];
            int j = type[i];
            oracle_field_at(field_kind, params, fieldE, fieldB, i, pos + 3 * i, t_n, E, B);
            if (g_pusher == ORACLE_PUSHER_VAY)
                oracle_vay_step(pos + 3 * i, mom + 3 * i, gamma + i, type_q[j], type_m[j], c, E,
                                B, dt);
            else if (g_pusher == ORACLE_PUSHER_HIGUERA_CARY)
                oracle_hc_step(pos + 3 * i, mom + 3 * i, gamma + i, type_q[j], type_m[j], c, E,
                               B, dt);
            else
                oracle_boris_step(pos + 3 * i, mom + 3 * i, gamma + i, type_q[j], type_m[j], c,
                                  E, B, dt);
        }
    }
    return 0;
}

/* Neumaier, "Rundungsfehleranalyse einiger Verfahren zur Summation endlicher
 * Summen" (1974): compensated summation; deterministic, serial. */
double oracle_neumaier_sum(int64_t n, const double *x) {
    double sum = 0.0, comp = 0.0;
    int64_t i;
    for (i = 0; i < n; ++i) {
        double t = sum + x[i];
        if (fabs(sum) >= fabs(x[i]))
            comp += (sum - t) + x[i];
        else
            comp += (x[i] - t) + sum;
        sum = t;
    }
    return sum + comp;
}

/* c17: KE = sum_i w_i (gamma_i - 1) m_i c^2 evaluated as
 * w m c^2 |u|^2/(gamma + 1), u = p/(mc), gamma as stored. */
double oracle_kinetic_energy(int64_t n, const double *mom, const double *gamma,
                             const double *weight, const int16_t *type,
                             const double *type_m, double c) {
    double sum = 0.0, comp = 0.0;
    int64_t i;
    for (i = 0; i < n; ++i) {
        double m = type_m[type[i]];
        double mc = m * c;
        double u2 = (mom[3 * i] * mom[3 * i] + mom[3 * i + 1] * mom[3 * i + 1] +
                     mom[3 * i + 2] * mom[3 * i + 2]) / (mc * mc);
        double ke = weight[i] * m * c * c * u2 / (gamma[i] + 1.0);
        double t = sum + ke;
        if (fabs(sum) >= fabs(ke))
            comp += (sum - t) + ke;
        else
            comp += (ke - t) + sum;
        sum = t;
    }
    return sum + comp;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
