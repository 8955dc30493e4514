// k_stream_soa.cu -- single-step SoA streaming Boris push ("precalculated
// fields").
//
// HBM-bound: per particle-step fp32 reads r,p,E,B (48 B) and writes r,p,gamma
// (28 B) = 76 B (+4 B weight with the KE diagnostic, +2 B type if multi-type).
// Design: one thread owns 16 B of every component array (4 fp32
// or 2 fp64 particles), so each component moves with one 128-bit access per
// thread and a warp touches 512 contiguous bytes per array; all loads of a
// group are issued before any arithmetic (12 x LDG.128 in flight per thread).
// Grid-stride over groups with a grid sized to the resident-block count.
#include <stdlib.h>

#include "boris_internal.h"
#include "deposit.cuh"

namespace boris {

#ifndef BORIS_STREAM_MINB
#define BORIS_STREAM_MINB 1  // resident blocks per SM requested from ptxas (tuning knob)
#endif

template <typename FP, bool MULTI, bool DIAG>
__global__ void __launch_bounds__(kStreamThreads, BORIS_STREAM_MINB)
    k_stream_soa_vec(SoaPtrs s, FieldSoaPtrs f, const __grid_constant__ KCoefs<FP, MULTI> co,
                     int64_t n_groups, int64_t n, double *partials) {
    constexpr int V = Vec<FP>::N;
    __shared__ TypeCoef<FP> s_t[MULTI ? kMaxTypes : 1];
    if (MULTI) load_type_table(co, s_t);

    FP *__restrict__ X = (FP *)s.x;
    FP *__restrict__ Y = (FP *)s.y;
    FP *__restrict__ Z = (FP *)s.z;
    FP *__restrict__ PX = (FP *)s.px;
    FP *__restrict__ PY = (FP *)s.py;
    FP *__restrict__ PZ = (FP *)s.pz;
    FP *__restrict__ G = (FP *)s.g;
    const FP *__restrict__ W = (const FP *)s.w;
    const FP *__restrict__ EX = (const FP *)f.Ex;
    const FP *__restrict__ EY = (const FP *)f.Ey;
    const FP *__restrict__ EZ = (const FP *)f.Ez;
    const FP *__restrict__ BX = (const FP *)f.Bx;
    const FP *__restrict__ BY = (const FP *)f.By;
    const FP *__restrict__ BZ = (const FP *)f.Bz;

    double ke = 0.0, cnt = 0.0;
    const int64_t stride = (int64_t)gridDim.x * kStreamThreads;
    for (int64_t grp = (int64_t)blockIdx.x * kStreamThreads + threadIdx.x; grp < n_groups;
         grp += stride) {
        const int64_t i0 = grp * V;
        Vec<FP> x, y, z, px, py, pz, ex, ey, ez, bx, by, bz, w, gm;
        // a1/a2: issue every load of the group before any arithmetic
        x.load_state(X + i0);
        y.load_state(Y + i0);
        z.load_state(Z + i0);
        px.load_state(PX + i0);
        py.load_state(PY + i0);
        pz.load_state(PZ + i0);
        ex.load_field(EX + i0);
        ey.load_field(EY + i0);
        ez.load_field(EZ + i0);
        bx.load_field(BX + i0);
        by.load_field(BY + i0);
        bz.load_field(BZ + i0);
        int ty[V];
        if (MULTI) load_types<V>(s.type + i0, ty);
        if (DIAG) {
            if (W) w.load_field(W + i0);
            else {
#pragma unroll
                for (int j = 0; j < V; ++j) w.v[j] = FP(1);
            }
        }
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const TypeCoef<FP> tc = MULTI ? s_t[ty[j]] : co.t[0];
            FP ux, uy, uz;
            push_one<FP>(x.v[j], y.v[j], z.v[j], px.v[j], py.v[j], pz.v[j], gm.v[j], ex.v[j],
                         ey.v[j], ez.v[j], bx.v[j], by.v[j], bz.v[j], tc, ux, uy, uz);
            if (DIAG) {
                ke += (double)kinetic_energy<FP>(ux, uy, uz, gm.v[j], w.v[j], tc);
                cnt += 1.0;
            }
        }
        x.store(X + i0);
        y.store(Y + i0);
        z.store(Z + i0);
        px.store(PX + i0);
        py.store(PY + i0);
        pz.store(PZ + i0);
        gm.store(G + i0);
    }
    // ragged tail: the last n - V*n_groups (< V) particles, scalar loads, same arithmetic
    const int64_t tail0 = n_groups * V;
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x < n - tail0) {
        const int64_t i = tail0 + threadIdx.x;
        const TypeCoef<FP> tc = MULTI ? s_t[s.type[i]] : co.t[0];
        FP ux, uy, uz, gam;
        FP x = X[i], y = Y[i], z = Z[i], px = PX[i], py = PY[i], pz = PZ[i];
        push_one<FP>(x, y, z, px, py, pz, gam, EX[i], EY[i], EZ[i], BX[i], BY[i], BZ[i], tc,
                     ux, uy, uz);
        X[i] = x; Y[i] = y; Z[i] = z; PX[i] = px; PY[i] = py; PZ[i] = pz; G[i] = gam;
        if (DIAG) {
            ke += (double)kinetic_energy<FP>(ux, uy, uz, gam, W ? W[i] : FP(1), tc);
            cnt += 1.0;
        }
    }
    if (DIAG) block_diag_partial<kStreamThreads>(ke, cnt, partials);
}

// Single-step push with the field gathered from a grid (the
// PIC case: the grid field changes between steps, so pushes are single steps).
// Same 128-bit state streaming as k_stream_soa_vec; the V particles of a thread
// gather their 8 nodes each with independent loads (ILP hides the L1/L2 latency).
// 3 resident blocks per SM (<= 80 registers): the gathers are latency-bound, so
// occupancy wins over per-thread registers (measured, 10^7 sorted, 64^3 grid:
// fp32 14.8 -> 12.3 ps, fp64 29.4 -> 23.7 ps vs the unconstrained ~100-register
// build; 4 blocks spill and lose again; profiles/r01/exp_grid_minblocks.txt).
#ifndef BORIS_GRID_MINB
#define BORIS_GRID_MINB 3
#endif
#define BORIS_GRID_BOUNDS __launch_bounds__(kStreamThreads, BORIS_GRID_MINB)
// Preferred shared-memory carveout (percent) of the grid push: -1 leaves the driver's
// choice (tuning).
#ifndef BORIS_GRID_CARVEOUT
#define BORIS_GRID_CARVEOUT -1
#endif
template <typename FP, bool MULTI, bool DIAG>
__global__ void BORIS_GRID_BOUNDS
    k_stream_soa_grid(SoaPtrs s, const __grid_constant__ GridArgs<FP> g,
                      const __grid_constant__ KCoefs<FP, MULTI> co, int64_t n_groups, int64_t n,
                      double *partials) {
    constexpr int V = Vec<FP>::N;
    __shared__ TypeCoef<FP> s_t[MULTI ? kMaxTypes : 1];
    if (MULTI) load_type_table(co, s_t);
    FP *X = (FP *)s.x, *Y = (FP *)s.y, *Z = (FP *)s.z;
    FP *PX = (FP *)s.px, *PY = (FP *)s.py, *PZ = (FP *)s.pz, *G = (FP *)s.g;
    const FP *W = (const FP *)s.w;
    double ke = 0.0, cnt = 0.0;
    const int64_t stride = (int64_t)gridDim.x * kStreamThreads;
    struct State {
        Vec<FP> x, y, z, px, py, pz, w;
        int ty[V];
    };
    auto load = [&](int64_t grp, State &st) {
        const int64_t i0 = grp * V;
        st.x.load_state(X + i0);
        st.y.load_state(Y + i0);
        st.z.load_state(Z + i0);
        st.px.load_state(PX + i0);
        st.py.load_state(PY + i0);
        st.pz.load_state(PZ + i0);
        if (MULTI) load_types<V>(s.type + i0, st.ty);
        if (DIAG) {
            if (W) st.w.load_field(W + i0);
            else {
#pragma unroll
                for (int j = 0; j < V; ++j) st.w.v[j] = FP(1);
            }
        }
    };
    int64_t grp = (int64_t)blockIdx.x * kStreamThreads + threadIdx.x;
    State cur;
    if (grp < n_groups) load(grp, cur);
    for (; grp < n_groups; grp += stride) {
        const int64_t i0 = grp * V;
        Vec<FP> gm;
        FP ex[V], ey[V], ez[V], bx[V], by[V], bz[V];
#pragma unroll
        for (int j = 0; j < V; ++j)
            grid_gather<FP>(g, cur.x.v[j], cur.y.v[j], cur.z.v[j], ex[j], ey[j], ez[j], bx[j],
                            by[j], bz[j]);
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const TypeCoef<FP> tc = MULTI ? s_t[cur.ty[j]] : co.t[0];
            FP ux, uy, uz;
            push_one<FP>(cur.x.v[j], cur.y.v[j], cur.z.v[j], cur.px.v[j], cur.py.v[j],
                         cur.pz.v[j], gm.v[j], ex[j], ey[j], ez[j], bx[j], by[j], bz[j], tc, ux,
                         uy, uz);
            if (DIAG) {
                ke += (double)kinetic_energy<FP>(ux, uy, uz, gm.v[j], cur.w.v[j], tc);
                cnt += 1.0;
            }
        }
        cur.x.store(X + i0);
        cur.y.store(Y + i0);
        cur.z.store(Z + i0);
        cur.px.store(PX + i0);
        cur.py.store(PY + i0);
        cur.pz.store(PZ + i0);
        gm.store(G + i0);
        if (grp + stride < n_groups) load(grp + stride, cur);
    }
    const int64_t tail0 = n_groups * V;
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x < n - tail0) {
        const int64_t i = tail0 + threadIdx.x;
        const TypeCoef<FP> tc = MULTI ? s_t[s.type[i]] : co.t[0];
        FP ux, uy, uz, gam, Ex, Ey, Ez, Bx, By, Bz;
        FP x = X[i], y = Y[i], z = Z[i], px = PX[i], py = PY[i], pz = PZ[i];
        grid_gather<FP>(g, x, y, z, Ex, Ey, Ez, Bx, By, Bz);
        push_one<FP>(x, y, z, px, py, pz, gam, Ex, Ey, Ez, Bx, By, Bz, tc, ux, uy, uz);
        X[i] = x; Y[i] = y; Z[i] = z; PX[i] = px; PY[i] = py; PZ[i] = pz; G[i] = gam;
        if (DIAG) {
            ke += (double)kinetic_energy<FP>(ux, uy, uz, gam, W ? W[i] : FP(1), tc);
            cnt += 1.0;
        }
    }
    if (DIAG) block_diag_partial<kStreamThreads>(ke, cnt, partials);
}

template <typename FP, bool MULTI, bool DIAG>
static cudaError_t dispatch_soa_grid(const EnsView &e, const GridArgs<FP> &g,
                                     const Coefs<FP> &co, DiagOut *diag, int device,
                                     cudaStream_t st) {
    constexpr int V = Vec<FP>::N;
    const int64_t n_groups = e.n / V;
    const int64_t blocks = (n_groups + kStreamThreads - 1) / kStreamThreads;
    int64_t grid = stream_grid(blocks > 0 ? blocks : 1, 2048 / kStreamThreads, device);
    if (DIAG && grid > diag->cap) grid = diag->cap;
    if (BORIS_GRID_CARVEOUT >= 0) {  // L1 / shared split of the SM (the gathers live in L1)
        static const cudaError_t once = cudaFuncSetAttribute(
            k_stream_soa_grid<FP, MULTI, DIAG>, cudaFuncAttributePreferredSharedMemoryCarveout,
            BORIS_GRID_CARVEOUT);
        if (once != cudaSuccess) return once;
    }
    k_stream_soa_grid<FP, MULTI, DIAG><<<(unsigned)grid, kStreamThreads, 0, st>>>(
        e.soa, g, kcoefs<MULTI>(co), n_groups, e.n, diag ? diag->partials : nullptr);
    if (diag) diag->written = DIAG ? grid : 0;
    return cudaGetLastError();
}

static bool aligned16(const void *p);

// Returns cudaErrorNotSupported when the arrays are not 16 B aligned (the caller
// then uses the fused kernel).
template <typename FP>
cudaError_t launch_stream_soa_grid(const EnsView &e, const GridArgs<FP> &g, const Coefs<FP> &co,
                                   bool multi, DiagOut *diag, int device, cudaStream_t st) {
    constexpr int V = Vec<FP>::N;
    if (e.n == 0) {
        if (diag) diag->written = 0;
        return cudaSuccess;
    }
    const bool al = aligned16(e.soa.x) && aligned16(e.soa.y) && aligned16(e.soa.z) &&
                    aligned16(e.soa.px) && aligned16(e.soa.py) && aligned16(e.soa.pz) &&
                    aligned16(e.soa.g) && (!diag || !e.soa.w || aligned16(e.soa.w)) &&
                    (!multi || ((uintptr_t)e.soa.type & (2 * V - 1)) == 0);
    if (!al) return cudaErrorNotSupported;
    const bool d = diag != nullptr;
    if (multi)
        return d ? dispatch_soa_grid<FP, true, true>(e, g, co, diag, device, st)
                 : dispatch_soa_grid<FP, true, false>(e, g, co, diag, device, st);
    return d ? dispatch_soa_grid<FP, false, true>(e, g, co, diag, device, st)
             : dispatch_soa_grid<FP, false, false>(e, g, co, diag, device, st);
}

template cudaError_t launch_stream_soa_grid<float>(const EnsView &, const GridArgs<float> &,
                                                   const Coefs<float> &, bool, DiagOut *, int,
                                                   cudaStream_t);
template cudaError_t launch_stream_soa_grid<double>(const EnsView &, const GridArgs<double> &,
                                                    const Coefs<double> &, bool, DiagOut *, int,
                                                    cudaStream_t);

// ---------------------------------------------------------------------------
// Fused PIC particle step: grid-gather push (as k_stream_soa_grid) followed, in the
// same thread and registers, by the CIC current deposition of the new state (as
// k_deposit_runs): r, p, w are not re-read and the deposition costs no launch.
// The state is bitwise the push's; J differs from push + deposit only in the
// order of its float atomics.  Warp-uniform grid-stride loop (every lane takes
// part in the end-of-group segmented merge).
// ---------------------------------------------------------------------------
#ifndef BORIS_PD_PREP
#define BORIS_PD_PREP 1
#endif
#ifndef BORIS_PD_MINB
#define BORIS_PD_MINB 2
#endif
template <typename FP, bool MULTI, bool DIAG, bool HAS_W>
__global__ void __launch_bounds__(kStreamThreads, BORIS_PD_MINB)
    k_push_deposit_soa(SoaPtrs s, const __grid_constant__ GridArgs<FP> g,
                       const __grid_constant__ KCoefs<FP, MULTI> co,
                       const __grid_constant__ DepCoefs<FP> dc,
                       const DepOut<FP> o, int64_t n_groups, int64_t n, double *partials) {
    constexpr int V = Vec<FP>::N;
    __shared__ TypeCoef<FP> s_t[MULTI ? kMaxTypes : 1];
    __shared__ DepCoef<FP> s_d[MULTI ? kMaxTypes : 1];
    __shared__ typename DepositRun<FP>::MergeSmem
        s_merge[kTransposedMergePD<FP> ? kStreamThreads / 32 : 1];
    if (MULTI) {
        for (int k = threadIdx.x; k < dc.n_types; k += blockDim.x) s_d[k] = dc.t[k];
        load_type_table(co, s_t);  // ends with __syncthreads
    }
    const int lane = threadIdx.x & 31;
    FP *X = (FP *)s.x, *Y = (FP *)s.y, *Z = (FP *)s.z;
    FP *PX = (FP *)s.px, *PY = (FP *)s.py, *PZ = (FP *)s.pz, *G = (FP *)s.g;
    const FP *W = (const FP *)s.w;
    double ke = 0.0, cnt = 0.0;
    const int64_t stride = (int64_t)gridDim.x * kStreamThreads;
    for (int64_t g0 = (int64_t)blockIdx.x * kStreamThreads + (threadIdx.x & ~31); g0 < n_groups;
         g0 += stride) {
        const int64_t grp = g0 + lane;
        const bool valid = grp < n_groups;
        DepositRun<FP> run;
        run.reset();
        if (valid) {
            const int64_t i0 = grp * V;
            Vec<FP> x, y, z, px, py, pz, w, gm;
            x.load_state(X + i0);
            y.load_state(Y + i0);
            z.load_state(Z + i0);
            px.load_state(PX + i0);
            py.load_state(PY + i0);
            pz.load_state(PZ + i0);
            int ty[V];
            if (MULTI) load_types<V>(s.type + i0, ty);
            if constexpr (HAS_W) {
                w.load_field(W + i0);
            } else {
#pragma unroll
                for (int j = 0; j < V; ++j) w.v[j] = FP(1);
            }
            FP ex[V], ey[V], ez[V], bx[V], by[V], bz[V];
#pragma unroll
            for (int j = 0; j < V; ++j)
                grid_gather<FP, true>(g, x.v[j], y.v[j], z.v[j], ex[j], ey[j], ez[j], bx[j],
                                      by[j],
                                bz[j]);
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const TypeCoef<FP> tc = MULTI ? s_t[ty[j]] : co.t[0];
                FP ux, uy, uz;
                push_one<FP>(x.v[j], y.v[j], z.v[j], px.v[j], py.v[j], pz.v[j], gm.v[j], ex[j],
                             ey[j], ez[j], bx[j], by[j], bz[j], tc, ux, uy, uz);
                if (DIAG) {
                    ke += (double)kinetic_energy<FP>(ux, uy, uz, gm.v[j], w.v[j], tc);
                    cnt += 1.0;
                }
            }
            x.store(X + i0);
            y.store(Y + i0);
            z.store(Z + i0);
            px.store(PX + i0);
            py.store(PY + i0);
            pz.store(PZ + i0);
            gm.store(G + i0);
            // deposition of the new state (measured: recomputing 1/gamma from the
            // stored p after the stores beats carrying the push's u and 1/gamma)
#if BORIS_PD_PREP
            {   // the V particles' weights first (independent chains), then accumulate
                typename DepositRun<FP>::Part pp[V];
#pragma unroll
                for (int j = 0; j < V; ++j)
                    DepositRun<FP>::prepare(g, MULTI ? s_d[ty[j]] : dc.t[0], dc.half_dt, x.v[j],
                                         y.v[j], z.v[j], px.v[j], py.v[j], pz.v[j], w.v[j], pp[j]);
#pragma unroll
                for (int j = 0; j < V; ++j) run.add_part(g, o, pp[j]);
            }
#else
#pragma unroll
            for (int j = 0; j < V; ++j)
                run.add(g, o, MULTI ? s_d[ty[j]] : dc.t[0], dc.half_dt, x.v[j], y.v[j], z.v[j],
                        px.v[j], py.v[j], pz.v[j], w.v[j]);
#endif
        }
        if constexpr (kTransposedMergePD<FP>) {
            run.merge_flush(o, s_merge[threadIdx.x >> 5], lane);
        } else {
            run.warp_merge(lane);
            run.flush<true>(o);
        }
    }
    // ragged tail (n mod V particles): push then deposit directly
    const int64_t tail0 = n_groups * V;
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x < n - tail0) {
        const int64_t i = tail0 + threadIdx.x;
        const int ty = MULTI ? s.type[i] : 0;
        const TypeCoef<FP> tc = MULTI ? s_t[ty] : co.t[0];
        FP ux, uy, uz, gam, Ex, Ey, Ez, Bx, By, Bz;
        FP x = X[i], y = Y[i], z = Z[i], px = PX[i], py = PY[i], pz = PZ[i];
        const FP w = HAS_W ? W[i] : FP(1);
        grid_gather<FP>(g, x, y, z, Ex, Ey, Ez, Bx, By, Bz);
        push_one<FP>(x, y, z, px, py, pz, gam, Ex, Ey, Ez, Bx, By, Bz, tc, ux, uy, uz);
        X[i] = x; Y[i] = y; Z[i] = z; PX[i] = px; PY[i] = py; PZ[i] = pz; G[i] = gam;
        if (DIAG) {
            ke += (double)kinetic_energy<FP>(ux, uy, uz, gam, w, tc);
            cnt += 1.0;
        }
        DepositRun<FP> run;
        run.reset();
        run.add(g, o, MULTI ? s_d[ty] : dc.t[0], dc.half_dt, x, y, z, px, py, pz, w);
        run.flush(o);
    }
    if (DIAG) block_diag_partial<kStreamThreads>(ke, cnt, partials);
}

template <typename FP, bool MULTI, bool DIAG>
static cudaError_t dispatch_push_deposit(const EnsView &e, const GridArgs<FP> &g,
                                         const Coefs<FP> &co, const DepCoefs<FP> &dc,
                                         const DepOut<FP> &o, DiagOut *diag, int device,
                                         cudaStream_t st) {
    constexpr int V = Vec<FP>::N;
    const int64_t n_groups = e.n / V;
    const int64_t blocks = (n_groups + kStreamThreads - 1) / kStreamThreads;
    int64_t grid = stream_grid(blocks > 0 ? blocks : 1, BORIS_PD_MINB, device);
    if (DIAG && grid > diag->cap) grid = diag->cap;
    if (e.soa.w)
        k_push_deposit_soa<FP, MULTI, DIAG, true><<<(unsigned)grid, kStreamThreads, 0, st>>>(
            e.soa, g, kcoefs<MULTI>(co), dc, o, n_groups, e.n, diag ? diag->partials : nullptr);
    else
        k_push_deposit_soa<FP, MULTI, DIAG, false><<<(unsigned)grid, kStreamThreads, 0, st>>>(
            e.soa, g, kcoefs<MULTI>(co), dc, o, n_groups, e.n, diag ? diag->partials : nullptr);
    if (diag) diag->written = DIAG ? grid : 0;
    return cudaGetLastError();
}

// Returns cudaErrorNotSupported when the state arrays are not 16 B aligned (the
// caller then runs the push and the deposition as two launches).
template <typename FP>
cudaError_t launch_push_deposit_soa(const EnsView &e, const GridArgs<FP> &g, const Coefs<FP> &co,
                                    const DepCoefs<FP> &dc, const DepOut<FP> &o, bool multi,
                                    DiagOut *diag, int device, cudaStream_t st) {
    constexpr int V = Vec<FP>::N;
    if (e.n == 0) {
        if (diag) diag->written = 0;
        return cudaSuccess;
    }
    const bool al = aligned16(e.soa.x) && aligned16(e.soa.y) && aligned16(e.soa.z) &&
                    aligned16(e.soa.px) && aligned16(e.soa.py) && aligned16(e.soa.pz) &&
                    aligned16(e.soa.g) && (!e.soa.w || aligned16(e.soa.w)) &&
                    (!multi || ((uintptr_t)e.soa.type & (2 * V - 1)) == 0);
    if (!al) return cudaErrorNotSupported;
    const bool d = diag != nullptr;
    if (multi)
        return d ? dispatch_push_deposit<FP, true, true>(e, g, co, dc, o, diag, device, st)
                 : dispatch_push_deposit<FP, true, false>(e, g, co, dc, o, diag, device, st);
    return d ? dispatch_push_deposit<FP, false, true>(e, g, co, dc, o, diag, device, st)
             : dispatch_push_deposit<FP, false, false>(e, g, co, dc, o, diag, device, st);
}

template cudaError_t launch_push_deposit_soa<float>(const EnsView &, const GridArgs<float> &,
                                                    const Coefs<float> &, const DepCoefs<float> &,
                                                    const DepOut<float> &, bool, DiagOut *, int,
                                                    cudaStream_t);
template cudaError_t launch_push_deposit_soa<double>(const EnsView &, const GridArgs<double> &,
                                                     const Coefs<double> &,
                                                     const DepCoefs<double> &,
                                                     const DepOut<double> &, bool, DiagOut *, int,
                                                     cudaStream_t);

// Unaligned inputs (e.g. sliced torch tensors): one particle per thread, scalar
// accesses, the same push_one arithmetic.
template <typename FP, bool MULTI, bool DIAG>
__global__ void __launch_bounds__(kStreamThreads)
    k_stream_soa_scalar(SoaPtrs s, FieldSoaPtrs f, const __grid_constant__ KCoefs<FP, MULTI> co,
                        int64_t n, double *partials) {
    __shared__ TypeCoef<FP> s_t[MULTI ? kMaxTypes : 1];
    if (MULTI) load_type_table(co, s_t);
    FP *X = (FP *)s.x, *Y = (FP *)s.y, *Z = (FP *)s.z;
    FP *PX = (FP *)s.px, *PY = (FP *)s.py, *PZ = (FP *)s.pz, *G = (FP *)s.g;
    const FP *W = (const FP *)s.w;
    const FP *EX = (const FP *)f.Ex, *EY = (const FP *)f.Ey, *EZ = (const FP *)f.Ez;
    const FP *BX = (const FP *)f.Bx, *BY = (const FP *)f.By, *BZ = (const FP *)f.Bz;
    double ke = 0.0, cnt = 0.0;
    const int64_t stride = (int64_t)gridDim.x * kStreamThreads;
    for (int64_t i = (int64_t)blockIdx.x * kStreamThreads + threadIdx.x; i < n; i += stride) {
        const int ty = MULTI ? s.type[i] : 0;
        const TypeCoef<FP> tc = MULTI ? s_t[ty] : co.t[0];
        FP ux, uy, uz, gam;
        FP x = X[i], y = Y[i], z = Z[i], px = PX[i], py = PY[i], pz = PZ[i];
        push_one<FP>(x, y, z, px, py, pz, gam, EX[i], EY[i], EZ[i], BX[i], BY[i], BZ[i], tc,
                     ux, uy, uz);
        X[i] = x; Y[i] = y; Z[i] = z; PX[i] = px; PY[i] = py; PZ[i] = pz; G[i] = gam;
        if (DIAG) {
            ke += (double)kinetic_energy<FP>(ux, uy, uz, gam, W ? W[i] : FP(1), tc);
            cnt += 1.0;
        }
    }
    if (DIAG) block_diag_partial<kStreamThreads>(ke, cnt, partials);
}

static bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

template <typename FP, bool MULTI, bool DIAG>
static cudaError_t dispatch_soa(const EnsView &e, const FieldSoaPtrs &f, const Coefs<FP> &co,
                                DiagOut *diag, int device, cudaStream_t st) {
    constexpr int V = Vec<FP>::N;
    const bool vec = aligned16(e.soa.x) && aligned16(e.soa.y) && aligned16(e.soa.z) &&
                     aligned16(e.soa.px) && aligned16(e.soa.py) && aligned16(e.soa.pz) &&
                     aligned16(e.soa.g) && aligned16(f.Ex) && aligned16(f.Ey) &&
                     aligned16(f.Ez) && aligned16(f.Bx) && aligned16(f.By) && aligned16(f.Bz) &&
                     (!DIAG || e.soa.w == nullptr || aligned16(e.soa.w)) &&
                     (!MULTI || ((uintptr_t)e.soa.type & (2 * V - 1)) == 0);
    double *partials = diag ? diag->partials : nullptr;
    int64_t grid;
    if (vec) {
        const int64_t n_groups = e.n / V;
        const int64_t blocks = (n_groups + kStreamThreads - 1) / kStreamThreads;
        grid = stream_grid(blocks > 0 ? blocks : 1, 2048 / kStreamThreads, device, kStreamWaves);
        if (DIAG && grid > diag->cap) grid = diag->cap;
        k_stream_soa_vec<FP, MULTI, DIAG>
            <<<(unsigned)grid, kStreamThreads, 0, st>>>(e.soa, f, kcoefs<MULTI>(co), n_groups, e.n,
                                                        partials);
    } else {
        const int64_t blocks = (e.n + kStreamThreads - 1) / kStreamThreads;
        grid = stream_grid(blocks > 0 ? blocks : 1, 2048 / kStreamThreads, device, kStreamWaves);
        if (DIAG && grid > diag->cap) grid = diag->cap;
        k_stream_soa_scalar<FP, MULTI, DIAG>
            <<<(unsigned)grid, kStreamThreads, 0, st>>>(e.soa, f, kcoefs<MULTI>(co), e.n, partials);
    }
    if (diag) diag->written = DIAG ? grid : 0;
    return cudaGetLastError();
}

template <typename FP>
cudaError_t launch_stream_soa(const EnsView &e, const FieldSoaPtrs &f, const Coefs<FP> &co,
                              bool multi, DiagOut *diag, int device, cudaStream_t st) {
    if (e.n == 0) {
        if (diag) diag->written = 0;
        return cudaSuccess;
    }
    const bool d = diag != nullptr;
    if (multi)
        return d ? dispatch_soa<FP, true, true>(e, f, co, diag, device, st)
                 : dispatch_soa<FP, true, false>(e, f, co, diag, device, st);
    return d ? dispatch_soa<FP, false, true>(e, f, co, diag, device, st)
             : dispatch_soa<FP, false, false>(e, f, co, diag, device, st);
}

template cudaError_t launch_stream_soa<float>(const EnsView &, const FieldSoaPtrs &,
                                              const Coefs<float> &, bool, DiagOut *, int,
                                              cudaStream_t);
template cudaError_t launch_stream_soa<double>(const EnsView &, const FieldSoaPtrs &,
                                               const Coefs<double> &, bool, DiagOut *, int,
                                               cudaStream_t);

}  // namespace boris
