/*
 * libboris.h -- C ABI of the B200-native relativistic Boris particle pusher.
 *
 * Method: arXiv 2104.04579 (Volokitin et al., "High Performance Implementation
 * of Boris Particle Pusher on DPC++"), §2.  Citations "Lnnn" are lines of the
 * paper text; "c<k>" are the readings of DESIGN.md §3 (= SURVEY.md
 * §8(c)).  Every entry point is `extern "C"`, takes plain pointers and sizes,
 * and returns a boris_status; no C++ or torch type crosses this boundary.
 *
 * Conventions (apply to every function below)
 * -------------------------------------------
 * Status:     BORIS_OK (0) or an error code; details in boris_last_error()
 *             (thread-local, valid until the next libboris call on that thread).
 *             Out-parameters are written only on BORIS_OK.
 * Streams:    `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *             stream).  Work is enqueued on it; functions documented as
 *             "asynchronous" return without a host sync, so kernel faults
 *             surface at the caller's next synchronisation.
 * Devices:    every handle is bound to one CUDA device; libboris switches to it
 *             internally and restores the caller's current device on return.
 * Units:      Gaussian CGS (eq. 1-5; reading c1) with the speed of
 *             light `light_velocity` a parameter (29979245800 for CGS, 1 for
 *             normalised units).  Momentum is p = gamma m v (eq. 5).
 * State:      positions r^n and momenta p^{n-1/2} (leapfrog, eq. 6-7,
 *             L117-136; reading c4: the initial p is p^{-1/2}, no back-step).
 *             gamma stored per particle is gamma(p^{n-1/2}) (reading c3).
 * Ordering:   particle order, weights and types are never modified by a push.
 * Threading:  a handle may be used by one host thread at a time.
 */
#ifndef LIBBORIS_H
#define LIBBORIS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LIBBORIS_ABI_VERSION 1

typedef int32_t boris_status;
#define BORIS_OK 0
#define BORIS_E_INVALID_ARG 1       /* NULL handle/pointer, n < 0, non-finite dt, bad enum ... */
#define BORIS_E_OUT_OF_MEMORY 2     /* device or pinned-host allocation failed                 */
#define BORIS_E_CUDA 3              /* a CUDA runtime call or kernel launch failed             */
#define BORIS_E_TYPE_OUT_OF_RANGE 4 /* a particle type index is outside [0, n_types)           */
#define BORIS_E_MISMATCH 5          /* field/ensemble precision, layout, size or device differ */
#define BORIS_E_UNSUPPORTED 6       /* valid request this build does not implement             */
#define BORIS_E_NO_DEVICE 7         /* no CUDA device / device index out of range              */

/* Particle layout (paper §3). */
typedef int32_t boris_layout;
#define BORIS_LAYOUT_AOS 0 /* array of 36 B (fp32) / 72 B (fp64) records, see below */
#define BORIS_LAYOUT_SOA 1 /* one array per component                             */

/* Floating-point type FP (paper §3). */
typedef int32_t boris_precision;
#define BORIS_FP32 0
#define BORIS_FP64 1

/* Residency of an ensemble's arrays. */
#define BORIS_MEMORY_DEVICE 0 /* arrays in device memory (HBM)                          */
#define BORIS_MEMORY_HOST 1   /* arrays in (preferably pinned) host memory: push streams */

/*
 * Per-type constants (paper §3: "parameters ... corresponding to
 * particles of different types, are stored in a separate table in a single
 * copy").  charge q (statC) and rest mass m (g); m > 0, q any finite value.
 * At most BORIS_MAX_TYPES entries.
 */
typedef struct boris_particle_type {
    double charge;
    double mass;
} boris_particle_type;
#define BORIS_MAX_TYPES 256

/* Largest particle count of one ensemble handle (2^40). */
#define BORIS_MAX_PARTICLES ((int64_t)1 << 40)

/*
 * AoS record layouts (paper §3: "Particle { FP3 position; FP3
 * momentum; FP weight; FP gamma; short type; }", 34 B -> 36 B aligned in
 * single precision, 66 B -> 72 B in double precision).  Byte offsets:
 *   fp32: position 0, momentum 12, weight 24, gamma 28, type 32, pad 34..35
 *   fp64: position 0, momentum 24, weight 48, gamma 56, type 64, pad 66..71
 * Field records for AoS ensembles: { FP3 E; FP3 B; } = 24 B / 48 B.
 */
#define BORIS_AOS_RECORD_BYTES_FP32 36
#define BORIS_AOS_RECORD_BYTES_FP64 72
#define BORIS_AOS_FIELD_BYTES_FP32 24
#define BORIS_AOS_FIELD_BYTES_FP64 48

typedef struct boris_ensemble boris_ensemble; /* opaque */
typedef struct boris_field boris_field;       /* opaque */

/* ------------------------------------------------------------------------ */
/* Library                                                                   */
/* ------------------------------------------------------------------------ */

int32_t boris_abi_version(void);
const char *boris_status_string(boris_status status);
const char *boris_last_error(void);

/*
 * Process-wide options.  The library reads no environment variables; the knobs
 * tests and tools need are set here.
 *   BORIS_OPT_FUSED_GENERIC (0 or 1, default 0): 1 turns off the axis-aligned
 *     specialisation of the register-fused kernels (uniform E on y and B on z;
 *     plane wave along x polarised along y), so those pushes run the generic
 *     kernel.  Results are bitwise identical (the specialisation only skips
 *     products with exact zeros); for tests that cover both kernels.
 *   BORIS_OPT_HOST_CHUNK (particles, default 4194304): chunk size of the
 *     host-resident (BORIS_MEMORY_HOST) push pipeline; must be >= 1024, used
 *     rounded down to a multiple of 8.
 *   BORIS_OPT_MD_ORDER (0 or 1, default 1): 1 lets a fused m-dipole push
 *     schedule the particles by radial branch (Taylor ones first, reading c13;
 *     a scratch index list of 4 n bytes); 0 pushes them in storage order.
 *     Scheduling only: results are bitwise identical; for tests.
 * A new value applies to pushes issued after the call.  Errors: INVALID_ARG
 * (unknown option, value out of range, NULL out-pointer).
 */
#define BORIS_OPT_FUSED_GENERIC 1
#define BORIS_OPT_HOST_CHUNK 2
#define BORIS_OPT_MD_ORDER 3
boris_status boris_set_option(int32_t option, int64_t value);
boris_status boris_get_option(int32_t option, int64_t *value);

/* ------------------------------------------------------------------------ */
/* Ensembles (paper §3 "Data Structures", L193-254)                           */
/* ------------------------------------------------------------------------ */

/*
 * Allocate an owned ensemble of n particles on `device` (all components zero,
 * types 0, gamma 1, weight 1, time 0).  SoA arrays are 256 B aligned and padded
 * to a multiple of 8 particles; padding is never downloaded or counted.
 * `types[0..n_types)` is copied.  n == 0 is allowed.
 * Errors: INVALID_ARG (n outside [0, BORIS_MAX_PARTICLES] — also for the wrap
 * functions —, n_types not in [1, BORIS_MAX_TYPES], mass <= 0,
 * non-finite values, light_velocity <= 0), NO_DEVICE, OUT_OF_MEMORY, CUDA.
 */
boris_status boris_ensemble_create(int32_t device, boris_layout layout,
                                   boris_precision precision, int64_t n,
                                   const boris_particle_type *types, int32_t n_types,
                                   double light_velocity, boris_ensemble **out);

/*
 * Wrap caller-owned SoA arrays (e.g. torch tensors) without copying.
 * x..pz, gamma: n elements of FP each; weight: n FP (may be NULL: weight 1 in
 * diagnostics); type: n int16 (may be NULL iff n_types == 1).  `memory` is
 * BORIS_MEMORY_DEVICE (arrays on `device`) or BORIS_MEMORY_HOST (host arrays,
 * pinned for full copy bandwidth; pushes stream them through the GPU in
 * chunks, see boris_push).  Any alignment is accepted; 16 B aligned arrays take
 * the vectorised path, others a scalar path with identical arithmetic.
 * The arrays must outlive the handle and every push enqueued on it.
 * The push never reads gamma (it is an output, reading c3); its contents are
 * the caller's until the first push.
 * Type indices are validated (synchronously) here; if the caller later changes
 * them it must call boris_ensemble_validate_types.
 * Errors: INVALID_ARG, NO_DEVICE, TYPE_OUT_OF_RANGE, CUDA.
 */
boris_status boris_ensemble_wrap_soa(int32_t device, int32_t memory, boris_precision precision,
                                     int64_t n, void *x, void *y, void *z, void *px, void *py,
                                     void *pz, void *weight, void *gamma, int16_t *type,
                                     const boris_particle_type *types, int32_t n_types,
                                     double light_velocity, boris_ensemble **out);

/*
 * Wrap caller-owned AoS records (n x 36 B fp32 or n x 72 B fp64, layout
 * above) without copying.  `records` must be 16 B aligned (fp32 records are 36
 * B, so 4 B aligned records are rejected with INVALID_ARG).  Otherwise as
 * boris_ensemble_wrap_soa.
 */
boris_status boris_ensemble_wrap_aos(int32_t device, int32_t memory, boris_precision precision,
                                     int64_t n, void *records,
                                     const boris_particle_type *types, int32_t n_types,
                                     double light_velocity, boris_ensemble **out);

/* Free an ensemble (and owned memory).  NULL is a no-op.  The caller must make
 * sure no enqueued push still uses it (synchronise the stream first). */
boris_status boris_ensemble_destroy(boris_ensemble *ens);

/*
 * Copy particles [first, first+count) from canonical HOST arrays into the
 * ensemble, converting to its layout and precision:
 *   pos3, mom3: count x 3 double, xyz interleaved (required)
 *   weight:     count double (NULL: leave unchanged)
 *   type:       count int16  (NULL: leave unchanged); validated, and nothing is
 *               written if any index is out of range (TYPE_OUT_OF_RANGE)
 *   gamma:      count double (NULL: recompute gamma = sqrt(1+|p|^2/(mc)^2),
 *               reading c3)
 * Synchronous: returns after the data is in place (`stream` orders it).
 */
boris_status boris_ensemble_upload(boris_ensemble *ens, int64_t first, int64_t count,
                                   const double *pos3, const double *mom3, const double *weight,
                                   const int16_t *type, const double *gamma, void *stream);

/* Copy particles [first, first+count) out to canonical HOST arrays (any output
 * pointer may be NULL to skip it).  Synchronous. */
boris_status boris_ensemble_download(const boris_ensemble *ens, int64_t first, int64_t count,
                                     double *pos3, double *mom3, double *weight, double *gamma,
                                     int16_t *type, void *stream);

/* Re-check all type indices (synchronous device check). */
boris_status boris_ensemble_validate_types(boris_ensemble *ens, void *stream);

/* Shape query.  Any out pointer may be NULL. */
boris_status boris_ensemble_get_info(const boris_ensemble *ens, boris_layout *layout,
                                     boris_precision *precision, int64_t *n, int32_t *n_types,
                                     int32_t *device, int32_t *memory);

/* Simulation time of r^n: t0 + (steps pushed) * dt; used for analytic fields
 * (reading c5: step n samples the field at t_n = t0 + n dt). */
boris_status boris_ensemble_get_time(const boris_ensemble *ens, double *t);
boris_status boris_ensemble_set_time(boris_ensemble *ens, double t);

/* ------------------------------------------------------------------------ */
/* Field sources (paper §5.2)                                       */
/* ------------------------------------------------------------------------ */

/*
 * "Precalculated fields" (L369-371, reading c6): one E,B per particle,
 * constant over steps, SoA arrays of n FP in the residency and precision of
 * `like` (an SoA ensemble).  Non-owning; arrays must outlive every push.
 */
boris_status boris_field_create_arrays_soa(const boris_ensemble *like, const void *Ex,
                                           const void *Ey, const void *Ez, const void *Bx,
                                           const void *By, const void *Bz, boris_field **out);

/* Precalculated fields for an AoS ensemble: n records {FP3 E; FP3 B} (24/48 B),
 * 16 B aligned.  Non-owning. */
boris_status boris_field_create_arrays_aos(const boris_ensemble *like, const void *records,
                                           boris_field **out);

/* Analytic uniform field: E, B constant (3 doubles each, statV/cm, G). */
boris_status boris_field_create_uniform(const double E[3], const double B[3],
                                        boris_field **out);

/*
 * Analytic plane wave (north_star; reading c-PW):
 *   phi = k (k_hat . r) - omega t + phase0,  E = E0 e_hat cos(phi),  B = k_hat x E.
 * k_hat, e_hat: unit vectors (|.|-1 <= 1e-12) with k_hat . e_hat <= 1e-12,
 * else INVALID_ARG.  omega, k >= 0 finite.
 */
boris_status boris_field_create_plane_wave(double E0, const double k_hat[3],
                                           const double e_hat[3], double omega, double k,
                                           double phase0, boris_field **out);

/*
 * Analytic standing magnetic-dipole wave, eq. 14-15 (L398-426) in the corrected
 * reading c9-c12 with the Taylor branch c13 (xi = kR < 1 with 9 terms for
 * fp64, xi < 1.5 with 7 terms for fp32):
 *   E  = 2 A0 cos(omega0 t) (f1(kR)/R) (-y, x, 0)
 *   Bx = -2 A0 sin(omega0 t) (xz/R^2) f2,  By = -2 A0 sin(omega0 t) (yz/R^2) f2,
 *   Bz = -2 A0 sin(omega0 t) [(z^2/R^2) f2 + f3].
 * A0 (statV/cm), omega0 (s^-1), k (cm^-1) finite, k > 0.
 */
boris_status boris_field_create_mdipole(double A0, double omega0, double k, boris_field **out);

/*
 * Grid field ("each particle interacts
 * with a set of nearby grid values of the electromagnetic field, depending on the
 * form factor"; reading c-grid): E, B given on the nodes of a periodic collocated
 * Cartesian grid, node (i,j,k) at origin + (i, j, k) * spacing, gathered at each
 * particle's position r^n every step with the CIC (trilinear) form factor.
 * Ex..Bz: DEVICE arrays of nx*ny*nz FP on `device`, node (i,j,k) at
 * (k*ny + j)*nx + i; they are copied (packed into 12-FP x-pair records, node i
 * and its periodic +x neighbour, owned by the handle: 12 FP per node of device
 * memory), so they may be freed after this call returns (synchronous).
 * Errors: INVALID_ARG (n < 1, > 2^31 nodes, spacing <= 0, NULL), NO_DEVICE, CUDA.
 * Ensembles pushed with it must have the same precision and device (MISMATCH).
 */
boris_status boris_field_create_grid(int32_t device, boris_precision precision, int32_t nx,
                                     int32_t ny, int32_t nz, const double origin[3],
                                     const double spacing[3], const void *Ex, const void *Ey,
                                     const void *Ez, const void *Bx, const void *By,
                                     const void *Bz, boris_field **out);

boris_status boris_field_destroy(boris_field *field);

/*
 * Periodic particle sort ("we have to periodically sort the
 * array of particles in order to improve cache locality"): reorder every array
 * of `ens` (positions, momenta, weight, gamma, type; AoS records whole) by the
 * grid cell of `grid` containing each particle.  Stable (particles of one cell
 * keep their relative order), so the result is deterministic.  Per-particle
 * field arrays are NOT permuted (they belong to the caller).  Device ensembles,
 * n < 2^32.  Asynchronous (temporary buffers are stream-ordered allocations).
 * Scratch: 16 B + (SoA) 8 FP + 2 B, or (AoS) one record, per particle, taken from
 * a library-owned per-device memory pool that keeps up to 1/16 of the device
 * memory mapped between calls (repeated sorts do not re-map their scratch).
 */
boris_status boris_ensemble_sort_by_cell(boris_ensemble *ens, const boris_field *grid,
                                         void *stream);

/*
 * Current deposition, the step after the push in a PIC cycle (
 * "The grid values of the current J are computed and added to
 * Maxwell's equations"; reading c-dep): for the state after a push of size dt
 * (r^{n+1}, p^{n+1/2}), deposit q w v^{n+1/2} of every particle at its half-step
 * position r^{n+1/2} = r^{n+1} - (dt/2) v^{n+1/2} onto the nodes of `grid` with the
 * CIC form factor, divided by the cell volume (current density, statA/cm^2).
 * Jx, Jy, Jz: DEVICE arrays of nx*ny*nz FP (node (i,j,k) at (k*ny+j)*nx+i),
 * overwritten with the result.  The atomics accumulate into a stream-ordered
 * scratch of (nx+1)(ny+1)(nz+1) nodes (16 B per node in fp32, 24 B in fp64; the
 * +1 layers are periodic ghosts) from the library's memory pool, folded into J at
 * the end.  Hardware atomics: the summation order varies run to run (results
 * reproducible to rounding, not bitwise).  Device ensembles; grid precision and
 * device must match (MISMATCH); OUT_OF_MEMORY if the scratch cannot be allocated.
 * Asynchronous.
 */
boris_status boris_deposit_current(const boris_ensemble *ens, const boris_field *grid, double dt,
                                   void *Jx, void *Jy, void *Jz, void *stream);

/*
 * Fused PIC particle step (field interpolation to the particles,
 * the push, and the current "computed and added to Maxwell's equations"): one
 * push of size dt with the field gathered from `grid` (as boris_push(ens, grid,
 * dt, 1, stream)) followed by the current deposition of the new state onto the
 * same grid (as boris_deposit_current(ens, grid, dt, Jx, Jy, Jz, stream)), in one
 * kernel for 16 B-aligned SoA ensembles (r, p and w are read once), else as the
 * two launches.  The ensemble state is bitwise the push's; J (DEVICE, nx*ny*nz FP
 * each, overwritten; the same scratch as boris_deposit_current) equals the
 * separate deposition up to the order of its float atomics.  d_diag (DEVICE, 2 doubles, or NULL): {sum KE, N} after the step,
 * as boris_push_diag.  The ensemble time advances by dt.  Errors: INVALID_ARG
 * (NULL ens/grid/J, non-grid field, dt not finite), MISMATCH (precision or
 * device), UNSUPPORTED (host-resident ensemble), OUT_OF_MEMORY (scratch), CUDA.
 * Asynchronous.
 */
boris_status boris_push_deposit(boris_ensemble *ens, const boris_field *grid, double dt,
                                void *Jx, void *Jy, void *Jz, double *d_diag, void *stream);

/*
 * "Precalculated fields" (L369-371, reading c6): evaluate the analytic field
 * `analytic` (uniform / plane wave / m-dipole) at every particle's current
 * position r_i at time t and write it into the per-particle field `out` (arrays
 * created with boris_field_create_arrays_* for `ens`; layout, precision, n,
 * device and residency must match, else MISMATCH).  The values are those the
 * fused push uses at (r_i, t), to rounding: the m-dipole is evaluated with the
 * fused step's radial functions and branch (reading c13), but the single-type
 * Boris fused push works in the scaled variables k r and p/(m c) and folds the
 * type's coefficients into the field's scalar factors instead of forming E and
 * B (a few roundings apart).  Device ensembles only.  Asynchronous.
 */
boris_status boris_field_evaluate(const boris_field *analytic, const boris_ensemble *ens,
                                  double t, const boris_field *out, void *stream);

/* ------------------------------------------------------------------------ */
/* Push (paper §2)                        */
/* ------------------------------------------------------------------------ */

/*
 * Advance every particle n_steps Boris steps of size dt:
 *   p^- = p + qE dt/2                          (eq. 9,  L149-150)
 *   gamma_n = sqrt(1 + |p^-|^2/(mc)^2)          (L162, reading c2)
 *   t = qB dt/(2 gamma_n m c), s = 2t/(1+t^2)   (eq. 13)
 *   p' = p^- + p^- x t, p^+ = p^- + p' x s      (eq. 12)
 *   p^{n+1/2} = p^+ + qE dt/2                   (eq. 10)
 *   gamma = sqrt(1 + |p|^2/(mc)^2)  (stored),  r += dt p/(gamma m)   (eq. 5, 7)
 * with (E, B) the field at (r^n, t_n), t_n = time + n dt (reading c5).
 * Per-particle fields must match the ensemble's layout, precision, n, device
 * and residency (else MISMATCH).  n_steps == 0 is a no-op; dt must be finite.
 * Asynchronous on `stream`; advances the ensemble time by n_steps*dt.
 *
 * Device ensembles: per-particle fields -> one streaming kernel launch per
 * step when n_steps == 1, one register-fused launch otherwise (bitwise the
 * same, see boris_push_ex); analytic fields -> one register-fused launch for
 * all n_steps.
 * Device-ensemble pushes do no host synchronisation and no allocation, so they
 * can be captured into a CUDA graph (after one eager call); note that the field
 * time t0 and dt are baked into the captured kernel parameters, so replays of a
 * captured analytic-field push re-use the captured times.
 * Host ensembles: the ensemble (and per-particle fields) stream through the
 * GPU in chunks with H2D / compute / D2H overlapped; each chunk is pushed all
 * n_steps while resident.  Host arrays must be pinned for asynchrony.
 */
boris_status boris_push(boris_ensemble *ens, const boris_field *field, double dt,
                        int64_t n_steps, void *stream);

/*
 * As boris_push, and additionally write the diagnostic of the state after the
 * last step into d_diag (DEVICE memory, 2 doubles):
 *   d_diag[0] = sum_i w_i (gamma_i - 1) m_i c^2  (evaluated as w m c^2 |u|^2/(gamma+1),
 *               u = p/(mc), reading c17; erg)
 *   d_diag[1] = number of particles (exact in double)
 * The sum is fused into the last step's kernel (per-block fp64 partials, then
 * a deterministic fixed-order finalize): bitwise reproducible run to run.
 * Host-resident ensembles: the diagnostic is reduced per chunk, then over
 * chunks (also deterministic); n_steps must be >= 1 there (else UNSUPPORTED).
 */
boris_status boris_push_diag(boris_ensemble *ens, const boris_field *field, double dt,
                             int64_t n_steps, double *d_diag, void *stream);

/*
 * Push flags for boris_push_ex.
 * BORIS_PUSH_AUTO (0): per-particle fields with n_steps > 1 run register-fused
 *   (E, B read once, the state kept in registers in FP and rounded exactly as
 *   the streaming kernel stores it): bitwise identical to n_steps single steps,
 *   with 1/n_steps of the HBM traffic.  boris_push / boris_push_diag use this.
 * BORIS_PUSH_STREAM_EACH_STEP: one streaming launch per step, re-reading the
 *   field array every step -- the paper's "precalculated fields" benchmark
 *   semantics (L369-371, L497-500).  Same results, HBM-bound.
 */
#define BORIS_PUSH_AUTO 0u
#define BORIS_PUSH_STREAM_EACH_STEP 1u

/*
 * Momentum-update scheme, bits 4-5 of the flags (the paper
 * cites alternative relativistic pushers, L111-113, L137-140, ref. [11], without
 * giving them; readings c-vay / c-hc in DESIGN.md follow their original papers):
 *   BORIS_PUSH_PUSHER_BORIS (default): the paper's conventional Boris (L141-186);
 *   BORIS_PUSH_PUSHER_VAY: Vay, Phys. Plasmas 15, 056701 (2008);
 *   BORIS_PUSH_PUSHER_HIGUERA_CARY: Higuera & Cary, Phys. Plasmas 24, 052104 (2017).
 * Same state, half-kick/position conventions and field sampling as Boris.  The
 * alternatives run in the register-fused kernels (single steps included).
 */
#define BORIS_PUSH_PUSHER_BORIS 0x00u
#define BORIS_PUSH_PUSHER_VAY 0x10u
#define BORIS_PUSH_PUSHER_HIGUERA_CARY 0x20u
#define BORIS_PUSH_PUSHER_MASK 0x30u

/*
 * boris_push / boris_push_diag with explicit flags (see above); d_diag may be
 * NULL (no diagnostic) or a DEVICE buffer of 2 doubles as in boris_push_diag.
 * Unknown flag bits: INVALID_ARG.
 */
boris_status boris_push_ex(boris_ensemble *ens, const boris_field *field, double dt,
                           int64_t n_steps, uint32_t flags, double *d_diag, void *stream);

/* The same diagnostic for the current state, without pushing (asynchronous);
 * gamma is recomputed from p (eq. 5), not read from the stored gamma. */
boris_status boris_kinetic_energy(const boris_ensemble *ens, double *d_diag, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* LIBBORIS_H */
