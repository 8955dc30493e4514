/*
 * boris_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the relativistic Boris push of
 * arXiv 2104.04579 (Volokitin et al.), written in scalar double precision C.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It shares no code, header, table or
 * constant with the CUDA path (paper_2104_04579_b200/csrc, include/libboris.h).
 *
 * Citations "Lnnn" are lines of /root/reference/PAPER.md (the paper text);
 * "c<k>" are the readings listed in SURVEY.md §8(c) / DESIGN.md §3.
 *
 * Every function here follows the paper's p-form (momentum p, not p/(mc)),
 * step by step in the paper's order (L175-186), with no fusion or reordering.
 *
 * Parity pins: see DESIGN.md §4.  All functions below are pinned by
 * `-m "not gpu"` tests in tests/test_oracle_pins.py; oracle_push's sampling of
 * r- and t-dependent fields at (r^n, t0 + n dt) by tests/test_oracle_driver_pins.py
 * (exact invariants of plane-wave, m-dipole and grid motion at O(dt^2), each shown to
 * reject a driver that samples at t_{n+1/2}, at r^{n+1} or ignores t0).  No function
 * is "parity unpinned".
 */
#ifndef BORIS_ORACLE_H
#define BORIS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Field source kinds understood by oracle_push (the oracle's own numbering). */
enum {
    ORACLE_FIELD_ARRAYS = 0,     /* per-particle E,B, constant over steps (L369-371, c6)   */
    ORACLE_FIELD_UNIFORM = 1,    /* params = {Ex,Ey,Ez,Bx,By,Bz}                            */
    ORACLE_FIELD_PLANE_WAVE = 2, /* params = {E0, kx,ky,kz (unit), ex,ey,ez (unit), omega, k, phase0} */
    ORACLE_FIELD_MDIPOLE = 3,    /* params = {A0, omega0, k, xi_star, n_terms}  eq.14-15, c9-c13 */
    ORACLE_FIELD_GRID = 4        /* params = {x0,y0,z0, dx,dy,dz, nx,ny,nz}; fieldE/fieldB =
                                    Ex|Ey|Ez and Bx|By|Bz node values, 3*nx*ny*nz each
                                    (component-major, node (i,j,k) at (k*ny+j)*nx+i);
                                    reading c-grid, SURVEY §8(f) row 3 */
};

/* Field on a periodic collocated Cartesian grid gathered with CIC (trilinear)
 * weights (reading c-grid; "each particle interacts with a
 * set of nearby grid values of the electromagnetic field, depending on the form
 * factor").  Node (i,j,k) sits at origin + (i dx, j dy, k dz); the grid repeats
 * with period (nx dx, ny dy, nz dz). */
void oracle_field_grid(const double *params, const double *gridE, const double *gridB,
                       const double r[3], double E[3], double B[3]);

/*
 * One Boris step of one particle, paper §2 (L147-186), p-form, double.
 *   r[3]    in: r^n          out: r^{n+1}
 *   p[3]    in: p^{n-1/2}    out: p^{n+1/2}
 *   gamma   out: gamma^{n+1/2} = sqrt(1 + |p^{n+1/2}|^2/(mc)^2)      (c3)
 *   q, m    charge and rest mass of the particle's type (L202-205)
 *   c       light velocity (Gaussian units, eq. 4; c1)
 *   E, B    field at (r^n, t_n) (eq. 6, c5)
 *   dt      time step
 */
void oracle_boris_step(double r[3], double p[3], double *gamma, double q, double m,
                       double c, const double E[3], const double B[3], double dt);

/*
 * Current deposition ("the step after the push"; PAPER.md
 * L89-92: "The grid values of the current J are computed and added to Maxwell's
 * equations"; reading c-dep): direct CIC deposition of every particle's current
 * q w v^{n+1/2} at its half-step position r^{n+1/2} = r^{n+1} - (dt/2) v^{n+1/2}
 * onto the nodes of the periodic collocated grid `params` (as ORACLE_FIELD_GRID),
 * divided by the cell volume: J[d*ncell + node] += q w v_d S(r - r_node)/(hx hy hz).
 * pos/mom are the state AFTER the push (r^{n+1}, p^{n+1/2}); J is zeroed first.
 */
void oracle_deposit_current(int64_t n, const double *pos, const double *mom,
                            const double *weight, const int16_t *type, const double *type_q,
                            const double *type_m, double c, double dt, const double *params,
                            double *J);

/* Pusher selector for oracle_push (PAPER.md L111-113,
 * L137-140 cite alternative relativistic pushers (ref. [11]) without giving them;
 * readings c-vay / c-hc in DESIGN.md follow their original papers). */
enum { ORACLE_PUSHER_BORIS = 0, ORACLE_PUSHER_VAY = 1, ORACLE_PUSHER_HIGUERA_CARY = 2 };

/* Vay (Phys. Plasmas 15, 056701, 2008), in u = p/(mc) (reading c-vay):
 *   u' = u + (q dt/(mc)) E + (u/gamma(u)) x tau,        tau = q B dt/(2 m c)
 *   sigma = gamma'^2 - tau^2, u* = u'.tau,
 *   gamma_new = sqrt((sigma + sqrt(sigma^2 + 4 (tau^2 + u*^2)))/2),
 *   t = tau/gamma_new, s = 1/(1+t^2),  u_new = s [u' + (u'.t) t + u' x t],
 *   then gamma = gamma(u_new), r += dt c u_new / gamma (eq. 7). */
void oracle_vay_step(double r[3], double p[3], double *gamma, double q, double m, double c,
                     const double E[3], const double B[3], double dt);

/* Higuera & Cary (Phys. Plasmas 24, 052104, 2017), in u = p/(mc) (reading c-hc):
 *   u- = u + eps, eps = q E dt/(2 m c);  gamma_new from (u-, tau) as in Vay;
 *   t = tau/gamma_new, s = 1/(1+t^2), ubar = s [u- + (u-.t) t + u- x t],
 *   u_new = ubar + eps + ubar x t,  gamma = gamma(u_new), r += dt c u_new / gamma. */
void oracle_hc_step(double r[3], double p[3], double *gamma, double q, double m, double c,
                    const double E[3], const double B[3], double dt);

/* Select the pusher used by oracle_push (default ORACLE_PUSHER_BORIS). */
void oracle_set_pusher(int pusher);

/* Uniform field: E, B constant (SURVEY §8(c) "Analytic fields"). */
void oracle_field_uniform(const double *params, double E[3], double B[3]);

/* Plane wave (north_star; not defined in the paper, reading c-PW in DESIGN.md):
 * phi = k (khat . r) - omega t + phase0;  E = E0 ehat cos(phi);  B = khat x E. */
void oracle_field_plane_wave(const double *params, const double r[3], double t,
                             double E[3], double B[3]);

/* Standing magnetic-dipole wave, eq. 14-15 (L398-426) in the corrected reading
 * c9-c12, with the Taylor branch c13 for xi = kR < xi_star (n_terms terms). */
void oracle_field_mdipole(const double *params, const double r[3], double t,
                          double E[3], double B[3]);

/* Radial functions of eq. 15 (c11, c13): g1 = f1/xi, g2 = f2/xi^2, f3.
 * Closed forms for xi >= xi_star, Taylor series (n_terms) otherwise. */
void oracle_mdipole_radial(double xi, double xi_star, int n_terms,
                           double *g1, double *g2, double *f3);

/* Field at particle i, position r, time t, for any field kind. */
void oracle_field_at(int kind, const double *params, const double *fieldE,
                     const double *fieldB, int64_t i, const double r[3], double t,
                     double E[3], double B[3]);

/*
 * Push an ensemble n_steps steps (paper §4.1 shape, L261-269: steps outside,
 * particles inside).  Arrays are canonical double, xyz-interleaved:
 *   pos[3n], mom[3n], gamma[n] (written), type[n] in [0, n_types).
 *   type_q[n_types], type_m[n_types]: the per-type table (L202-205).
 *   fieldE/fieldB[3n]: per-particle field (kind ARRAYS), else NULL.
 *   t0: time of r^0 for analytic fields; step n samples t_n = t0 + n*dt (c5).
 *   n_threads: OpenMP threads (1 = serial); used only for CPU-baseline timing.
 * Returns 0, or -1 on an out-of-range type index (nothing is written then).
 */
int oracle_push(int64_t n, double *pos, double *mom, double *gamma,
                const int16_t *type, const double *type_q, const double *type_m,
                int32_t n_types, double c, int field_kind, const double *params,
                const double *fieldE, const double *fieldB, double t0, double dt,
                int64_t n_steps, int n_threads);

/* Kinetic energy sum_i w_i m_i c^2 |u_i|^2/(gamma_i+1), u = p/(mc), which is
 * w (gamma-1) m c^2 without cancellation (c17); Neumaier-compensated sum. */
double oracle_kinetic_energy(int64_t n, const double *mom, const double *gamma,
                             const double *weight, const int16_t *type,
                             const double *type_m, double c);

/* Neumaier (improved Kahan-Babuska) sum of x[0..n). */
double oracle_neumaier_sum(int64_t n, const double *x);

/* Number of OpenMP threads the oracle would use for n_threads <= 0. */
int oracle_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif
