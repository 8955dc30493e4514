// boris_internal.h -- host-side declarations shared by libboris's translation units.
// Not part of the ABI (include/libboris.h is).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "boris_device.cuh"
#include "grid.cuh"
#include "libboris.h"

namespace boris {

#ifndef BORIS_STREAM_THREADS
#define BORIS_STREAM_THREADS 256
#endif
constexpr int kStreamThreads = BORIS_STREAM_THREADS;  // SoA streaming kernel block size
constexpr int kAosThreads = 256;     // AoS tile kernel block size (one particle / thread / tile)
constexpr int kFusedThreads = 128;   // register-fused multi-step kernel block size
constexpr int kFinalizeThreads = 1024;

enum FieldKind { FK_ARRAYS = 0, FK_UNIFORM = 1, FK_PLANE_WAVE = 2, FK_MDIPOLE = 3, FK_GRID = 4 };

struct SoaPtrs {
    void *x, *y, *z, *px, *py, *pz, *w, *g;
    int16_t *type;
};

struct FieldSoaPtrs {
    const void *Ex, *Ey, *Ez, *Bx, *By, *Bz;
};

// Analytic field parameters prepared on the host for one push (FP = kernel
// precision; phases in double, reading c5: t_n = t0 + n dt, never accumulated).
template <typename FP>
struct AnalyticArgs {
    // uniform
    FP E[3], B[3];
    // plane wave: phi_n = (kvec . r) + ph0 - n * wdt ; E = cE cos(phi), B = cB cos(phi)
    double kvec[3];  // k * k_hat
    double ph0;      // phase0 - omega * t0
    double wdt;      // omega * dt
    FP cE[3];        // E0 * e_hat
    FP cB[3];        // E0 * (k_hat x e_hat)
    FP kf[3];        // kvec in FP (phase increments inside a fused window)
    FP wdtf;         // omega * dt in FP
    // m-dipole (eq. 14-15, readings c9-c13): time phase w0 t_n = w0t0 + n * w0dt
    FP A0, k, k2;
    FP A0k2;         // 2 A0 k
    FP mA02;         // -2 A0
    double w0t0, w0dt;
    int md_order;  // schedule by radial branch (k_md_order; BORIS_OPT_MD_ORDER)
    // single-type Boris m-dipole (k_fused kMdFold; push_view fills these): the step runs
    // in the scaled variables X = k r, u = p/(m c), so that xi^2 = |X|^2 and
    // gamma^2 = 1 + |u|^2 (no k^2, kappa^2 factors in the loop)
    double mdf_k, mdf_ik;        // k, 1/k
    double mdf_kick, mdf_rot;    // (q dt / 2 m c) 2 A0, (q dt / 2 m c) (-2 A0)
    FP mdf_uin, mdf_uout, mdf_cr;  // 1/(m c), m c, k c dt
    // grid (FK_GRID): CIC gather of packed node records (grid.cuh)
    GridArgs<FP> grid;
    // uniform / plane wave with E || y^, B || z^ (k^ = x^): the k_fused YZ
    // specialisation applies (boris_momentum_yz; bitwise identical results)
    int yz;
};

// Per-launch description of an ensemble's storage.
struct EnsView {
    int precision;  // BORIS_FP32 / BORIS_FP64
    int layout;     // BORIS_LAYOUT_*
    int64_t n;
    SoaPtrs soa;    // SoA
    void *aos;      // AoS records
};

// Diagnostic partials: launchers report how many (ke, count) pairs they wrote.
struct DiagOut {
    double *partials;    // device scratch, capacity 2 * cap doubles
    int64_t cap;         // pairs available
    int64_t written;     // pairs written by the launch (0 if no diag)
};

int sm_count(int device);

// Stream-ordered scratch from the library's per-device pool (k_util.cu).
cudaError_t scratch_alloc(void **ptr, size_t bytes, cudaStream_t st);
void scratch_free(void *ptr, cudaStream_t st);

// Grid of a grid-stride launch: min(work blocks, SMs x resident blocks x waves).
#ifndef BORIS_STREAM_WAVES
#define BORIS_STREAM_WAVES 64
#endif
constexpr int kStreamWaves = BORIS_STREAM_WAVES;
int64_t stream_grid(int64_t work_blocks, int blocks_per_sm, int device, int waves = 4);
// Grid of an ALU-bound grid-stride launch: min(work blocks, SMs x the kernel's
// resident blocks per SM) -- one wave, equal work per block.
int64_t resident_grid(const void *kernel, int threads, int64_t work_blocks, int device);

// Grid of the register-fused kernels (k_fused, k_fused_arrays; kFusedThreads
// threads).  BORIS_FUSED_GRID (tuning): 0 one resident wave, 1 the 4-wave
// grid-stride cap of stream_grid, 2 one block per work block (no grid stride).
#ifndef BORIS_FUSED_GRID
#define BORIS_FUSED_GRID 2
#endif
inline int64_t fused_grid(const void *kernel, int64_t work_blocks, int device) {
    if (BORIS_FUSED_GRID == 0) return resident_grid(kernel, kFusedThreads, work_blocks, device);
    if (BORIS_FUSED_GRID == 2) return work_blocks;
    return stream_grid(work_blocks, 2048 / kFusedThreads, device);
}

template <typename FP>
cudaError_t launch_stream_soa(const EnsView &e, const FieldSoaPtrs &f, const Coefs<FP> &co,
                              bool multi, DiagOut *diag, int device, cudaStream_t st);

// Single-step SoA push with a grid-gathered field (cudaErrorNotSupported if the
// arrays are not 16 B aligned).
template <typename FP>
cudaError_t launch_stream_soa_grid(const EnsView &e, const GridArgs<FP> &g, const Coefs<FP> &co,
                                   bool multi, DiagOut *diag, int device, cudaStream_t st);

template <typename FP>
cudaError_t launch_stream_aos(const EnsView &e, const void *field_records, const Coefs<FP> &co,
                              bool multi, DiagOut *diag, int device, cudaStream_t st);

template <typename FP>
cudaError_t launch_fused(const EnsView &e, int field_kind, const AnalyticArgs<FP> &fa,
                         const Coefs<FP> &co, int64_t n_steps, bool multi, int pusher,
                         DiagOut *diag, int device, cudaStream_t st);

// Grid field support (k_grid.cu): pack 6 component arrays (ncell FP each) into
// 8-FP node records; stable sort of an ensemble by grid cell (LSD radix sort of
// (cell, index) pairs + permutation of every particle array).
cudaError_t launch_grid_pack(int precision, int64_t ncell, int nx, const void *const comps[6],
                             void *nodes, cudaStream_t st);
template <typename FP>
cudaError_t sort_by_cell(const EnsView &e, const GridArgs<FP> &g, int device, cudaStream_t st);

// Current deposition (reading c-dep): per-type coefficients.
template <typename FP>
struct DepCoef {
    FP S;       // 2^k ~ 1/(mc): u = S p
    FP kappa2;  // 1/(S m c)^2
    FP inv_Sm;  // 1/(S m): v = u inv_Sm / gamma
    FP q_vol;   // q / (hx hy hz)
};
template <typename FP>
struct DepCoefs {
    int n_types;
    FP half_dt;
    DepCoef<FP> t[kMaxTypes];
};
// Deposition target (deposit.cuh): the padded scratch J4, node (i, j, k) for
// 0 <= i <= nx, 0 <= j <= ny, 0 <= k <= nz with index (k sy + j) sx + i; fp32
// components interleaved (x, y, z, pad per node), fp64 in three planes.  The +1
// layers are ghosts that dep_scratch_end folds onto their periodic images.
template <typename FP>
struct DepOut {
    FP *j4;
    uint32_t sx;     // nx + 1
    uint32_t sxy;    // (nx + 1)(ny + 1)
    uint32_t plane;  // (nx + 1)(ny + 1)(nz + 1): fp64 component plane stride
};
// Allocates and zeroes J4 for grid g (stream-ordered scratch).
template <typename FP>
cudaError_t dep_scratch_begin(const GridArgs<FP> &g, DepOut<FP> &o, cudaStream_t st);
// Folds J4 into the caller's Jx, Jy, Jz (nx*ny*nz each, overwritten) and frees J4.
template <typename FP>
cudaError_t dep_scratch_end(const GridArgs<FP> &g, DepOut<FP> &o, void *Jx, void *Jy, void *Jz,
                            cudaStream_t st);
// Frees J4 without folding (error paths).
template <typename FP>
void dep_scratch_free(DepOut<FP> &o, cudaStream_t st);

// Fused grid-gather push + current deposition into J4 (SoA, 16 B-aligned; else
// cudaErrorNotSupported).
template <typename FP>
cudaError_t launch_push_deposit_soa(const EnsView &e, const GridArgs<FP> &g, const Coefs<FP> &co,
                                    const DepCoefs<FP> &dc, const DepOut<FP> &o, bool multi,
                                    DiagOut *diag, int device, cudaStream_t st);

template <typename FP>
cudaError_t launch_deposit(const EnsView &e, const GridArgs<FP> &g, const DepCoefs<FP> &dc,
                           void *Jx, void *Jy, void *Jz, int device, cudaStream_t st);

// Analytic field at every particle's position (time baked into fa) -> arrays.
template <typename FP>
cudaError_t launch_field_evaluate(const EnsView &e, int field_kind, const AnalyticArgs<FP> &fa,
                                  const FieldSoaPtrs &out, void *out_rec, int device,
                                  cudaStream_t st);

// n_steps in registers with per-particle (constant) fields; bitwise identical to
// n_steps launches of the streaming kernels.
template <typename FP>
cudaError_t launch_fused_arrays(const EnsView &e, const FieldSoaPtrs &f, const void *frec,
                                const Coefs<FP> &co, int64_t n_steps, bool multi, int pusher,
                                DiagOut *diag, int device, cudaStream_t st);

template <typename FP>
cudaError_t launch_kinetic_energy(const EnsView &e, const Coefs<FP> &co, bool multi,
                                  DiagOut *diag, int device, cudaStream_t st);

// Sum `pairs` (ke, count) partials in a fixed order into out[0..1].
cudaError_t launch_diag_finalize(const double *partials, int64_t pairs, double *out,
                                 cudaStream_t st);

// Canonical double <-> layout conversion for upload/download (staging on device).
// Staging layout: pos[3c], mom[3c], weight[c], gamma[c] (doubles), type[c] (int16).
cudaError_t launch_from_canonical(const EnsView &e, int64_t first, int64_t count,
                                  const double *d_pos, const double *d_mom, const double *d_w,
                                  const int16_t *d_type, const double *d_gamma,
                                  const double *d_inv_mc2_by_type, int n_types, int has_w,
                                  int has_type, cudaStream_t st);
cudaError_t launch_to_canonical(const EnsView &e, int64_t first, int64_t count, double *d_pos,
                                double *d_mom, double *d_w, double *d_gamma, int16_t *d_type,
                                cudaStream_t st);
// Count type indices outside [0, n_types) into *d_bad (device int64).
cudaError_t launch_check_types(const int16_t *type, int64_t stride_bytes, int64_t n,
                               int n_types, unsigned long long *d_bad, cudaStream_t st);
cudaError_t launch_fill_defaults(const EnsView &e, cudaStream_t st);

}  // namespace boris
