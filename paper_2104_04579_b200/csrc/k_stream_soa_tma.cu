// k_stream_soa_tma.cu -- single-step SoA streaming Boris push with TMA bulk-copy
// staging (alternative to the LDG.128 kernel of k_stream_soa.cu; same push_one
// arithmetic, so bitwise-identical results).
//
// Persistent CTAs; one elected thread streams tiles of TP particles of every
// component array (6 state + 6 field arrays, + weight / type when needed) into
// shared memory with 1-D bulk copies completing on one mbarrier per stage,
// STAGES tiles in flight; 256 threads push the tile out of shared memory and the
// elected thread writes the 7 output slices (r, p, gamma) back with bulk stores.
// No per-thread global loads or stores: the LSU and register file are idle, the
// copy engines move the bytes (HBM-bound, 76-80 B per particle-step).
#include "boris_internal.h"
#include "tma.cuh"

namespace boris {

namespace {

template <typename FP>
struct SoaTma {
    static constexpr int THREADS = 256;
    static constexpr int TP = sizeof(FP) == 4 ? 512 : 256;  // particles per tile
    static constexpr int PPT = TP / THREADS;                  // per thread per tile
    static constexpr int ARR = TP * (int)sizeof(FP);          // 2 KiB per array slice
    static constexpr int NSLOT = 14;  // 0-5 state, 6-11 E B, 12 weight, 13 gamma (out)
    static constexpr int STAGE = NSLOT * ARR + TP * 2;        // + int16 type slice
    static constexpr int STAGES = 3;
    static constexpr int SMEM = STAGES * STAGE + STAGES * 8;
    static constexpr int ALIGN = 8;  // tiles cover multiples of 8 particles (16 B int16 slices)
};

}  // namespace

template <typename FP, bool MULTI, bool DIAG>
__global__ void __launch_bounds__(SoaTma<FP>::THREADS)
    k_stream_soa_tma(SoaPtrs s, FieldSoaPtrs f, const __grid_constant__ Coefs<FP> co,
                     int64_t n_tiles, int64_t n_main, int64_t n, double *partials) {
    using G = SoaTma<FP>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bar = (uint64_t *)(smem + G::STAGES * G::STAGE);
    __shared__ TypeCoef<FP> s_t[MULTI ? kMaxTypes : 1];

    const FP *src[12] = {(const FP *)s.x,  (const FP *)s.y,  (const FP *)s.z,
                         (const FP *)s.px, (const FP *)s.py, (const FP *)s.pz,
                         (const FP *)f.Ex, (const FP *)f.Ey, (const FP *)f.Ez,
                         (const FP *)f.Bx, (const FP *)f.By, (const FP *)f.Bz};
    const bool has_w = DIAG && s.w != nullptr;

    if (threadIdx.x == 0) {
        for (int k = 0; k < G::STAGES; ++k) mbar_init(&bar[k], 1);
        fence_proxy_async_smem();
    }
    if (MULTI) load_type_table(co, s_t);
    else __syncthreads();

    auto slot = [&](int stage, int k) -> FP * {
        return (FP *)(smem + stage * G::STAGE + k * G::ARR);
    };
    auto tslot = [&](int stage) -> int16_t * {
        return (int16_t *)(smem + stage * G::STAGE + G::NSLOT * G::ARR);
    };
    auto tile_count = [&](int64_t t) -> int {
        const int64_t c = n_main - t * G::TP;
        return c < G::TP ? (int)c : G::TP;
    };
    auto issue = [&](int64_t t, int stage) {
        const int c = tile_count(t);
        const uint32_t b = (uint32_t)c * sizeof(FP);
        const int64_t i0 = t * G::TP;
        uint32_t tx = 12 * b + (has_w ? b : 0) + (MULTI ? 2u * c : 0u);
        mbar_arrive_expect_tx(&bar[stage], tx);
        for (int k = 0; k < 12; ++k) bulk_g2s(slot(stage, k), src[k] + i0, b, &bar[stage]);
        if (has_w) bulk_g2s(slot(stage, 12), (const FP *)s.w + i0, b, &bar[stage]);
        if (MULTI) bulk_g2s(tslot(stage), s.type + i0, 2u * c, &bar[stage]);
    };

    if (threadIdx.x == 0)
        for (int k = 0; k < G::STAGES; ++k) {
            const int64_t t = blockIdx.x + (int64_t)k * gridDim.x;
            if (t < n_tiles) issue(t, k);
        }

    double ke = 0.0, cnt = 0.0;
    for (int64_t it = 0;; ++it) {
        const int64_t t = blockIdx.x + it * gridDim.x;
        if (t >= n_tiles) break;
        const int stage = (int)(it % G::STAGES);
        mbar_wait(&bar[stage], (uint32_t)((it / G::STAGES) & 1));
        const int c = tile_count(t);
#pragma unroll
        for (int q = 0; q < G::PPT; ++q) {
            const int j = threadIdx.x + q * G::THREADS;
            if (j < c) {
                FP *X = slot(stage, 0), *Y = slot(stage, 1), *Z = slot(stage, 2);
                FP *PX = slot(stage, 3), *PY = slot(stage, 4), *PZ = slot(stage, 5);
                const int ty = MULTI ? tslot(stage)[j] : 0;
                const TypeCoef<FP> tc = MULTI ? s_t[ty] : co.t[0];
                FP x = X[j], y = Y[j], z = Z[j], px = PX[j], py = PY[j], pz = PZ[j];
                FP ux, uy, uz, gam;
                push_one<FP>(x, y, z, px, py, pz, gam, slot(stage, 6)[j], slot(stage, 7)[j],
                             slot(stage, 8)[j], slot(stage, 9)[j], slot(stage, 10)[j],
                             slot(stage, 11)[j], tc, ux, uy, uz);
                X[j] = x; Y[j] = y; Z[j] = z; PX[j] = px; PY[j] = py; PZ[j] = pz;
                slot(stage, 13)[j] = gam;
                if (DIAG) {
                    ke += (double)kinetic_energy<FP>(ux, uy, uz, gam,
                                                     has_w ? slot(stage, 12)[j] : FP(1), tc);
                    cnt += 1.0;
                }
            }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t b = (uint32_t)c * sizeof(FP);
            const int64_t i0 = t * G::TP;
            FP *dst[7] = {(FP *)s.x, (FP *)s.y, (FP *)s.z, (FP *)s.px, (FP *)s.py, (FP *)s.pz,
                          (FP *)s.g};
            for (int k = 0; k < 6; ++k) bulk_s2g(dst[k] + i0, slot(stage, k), b);
            bulk_s2g(dst[6] + i0, slot(stage, 13), b);
            bulk_commit();
            const int64_t tn = t + (int64_t)G::STAGES * gridDim.x;
            if (tn < n_tiles) {
                bulk_wait_read_all();
                issue(tn, stage);
            }
        }
    }
    // ragged tail (< ALIGN particles): direct global access, same arithmetic
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x < n - n_main) {
        const int64_t i = n_main + threadIdx.x;
        FP *X = (FP *)s.x, *Y = (FP *)s.y, *Z = (FP *)s.z;
        FP *PX = (FP *)s.px, *PY = (FP *)s.py, *PZ = (FP *)s.pz;
        const TypeCoef<FP> tc = MULTI ? s_t[s.type[i]] : co.t[0];
        FP x = X[i], y = Y[i], z = Z[i], px = PX[i], py = PY[i], pz = PZ[i];
        FP ux, uy, uz, gam;
        push_one<FP>(x, y, z, px, py, pz, gam, src[6][i], src[7][i], src[8][i], src[9][i],
                     src[10][i], src[11][i], tc, ux, uy, uz);
        X[i] = x; Y[i] = y; Z[i] = z; PX[i] = px; PY[i] = py; PZ[i] = pz;
        ((FP *)s.g)[i] = gam;
        if (DIAG) {
            ke += (double)kinetic_energy<FP>(ux, uy, uz, gam, has_w ? ((const FP *)s.w)[i] : FP(1),
                                             tc);
            cnt += 1.0;
        }
    }
    if (threadIdx.x == 0) bulk_wait_all();
    if (DIAG) block_diag_partial<SoaTma<FP>::THREADS>(ke, cnt, partials);
}

template <typename FP, bool MULTI, bool DIAG>
static cudaError_t dispatch_tma(const EnsView &e, const FieldSoaPtrs &f, const Coefs<FP> &co,
                                DiagOut *diag, int device, cudaStream_t st) {
    using G = SoaTma<FP>;
    auto kern = k_stream_soa_tma<FP, MULTI, DIAG>;
    static bool attr_set[64] = {};
    if (device >= 0 && device < 64 && !attr_set[device]) {
        cudaError_t err =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        if (err != cudaSuccess) return err;
        attr_set[device] = true;
    }
    int per_sm = 0;
    cudaError_t err =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::THREADS, G::SMEM);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) per_sm = 1;
    const int64_t n_main = e.n / G::ALIGN * G::ALIGN;
    const int64_t n_tiles = (n_main + G::TP - 1) / G::TP;
    int64_t grid = (int64_t)sm_count(device) * per_sm;
    if (grid > n_tiles) grid = n_tiles > 0 ? n_tiles : 1;
    if (DIAG && grid > diag->cap) grid = diag->cap;
    kern<<<(unsigned)grid, G::THREADS, G::SMEM, st>>>(e.soa, f, co, n_tiles, n_main, e.n,
                                                     diag ? diag->partials : nullptr);
    if (diag) diag->written = DIAG ? grid : 0;
    return cudaGetLastError();
}

template <typename FP>
cudaError_t launch_stream_soa_tma(const EnsView &e, const FieldSoaPtrs &f, const Coefs<FP> &co,
                                  bool multi, DiagOut *diag, int device, cudaStream_t st) {
    if (e.n == 0) {
        if (diag) diag->written = 0;
        return cudaSuccess;
    }
    const bool d = diag != nullptr;
    if (multi)
        return d ? dispatch_tma<FP, true, true>(e, f, co, diag, device, st)
                 : dispatch_tma<FP, true, false>(e, f, co, diag, device, st);
    return d ? dispatch_tma<FP, false, true>(e, f, co, diag, device, st)
             : dispatch_tma<FP, false, false>(e, f, co, diag, device, st);
}

// ---------------------------------------------------------------------------
// Grid-gather single step with TMA-staged particle state.
// The CIC gather makes this kernel latency-bound rather than copy-bound: with
// per-thread LDG the HBM wait for the state and the L1/L2 gathers serialise
// inside every thread.  Here one elected thread keeps STAGES tiles of the state
// (x y z px py pz [w] [type]) in flight with 1-D bulk copies while the 256
// threads gather and push the resident tile; results go back by bulk stores.
// Same push_one / grid_gather arithmetic as k_stream_soa_grid: bitwise equal.
// ---------------------------------------------------------------------------
template <typename FP>
struct GridTma {
    static constexpr int THREADS = 256;
#ifdef BORIS_GRID_TMA_TP
    static constexpr int TP = BORIS_GRID_TMA_TP / (sizeof(FP) / 4);
#else
    static constexpr int TP = sizeof(FP) == 4 ? 512 : 256;  // particles per tile
#endif
    static constexpr int PPT = TP / THREADS;
    static constexpr int ARR = TP * (int)sizeof(FP);
    static constexpr int NSLOT = 8;  // 0-5 state, 6 weight, 7 gamma (out)
    static constexpr int STAGE = NSLOT * ARR + TP * 2;
#ifdef BORIS_GRID_TMA_STAGES
    static constexpr int STAGES = BORIS_GRID_TMA_STAGES;
#else
    static constexpr int STAGES = 4;
#endif
    static constexpr int SMEM = STAGES * STAGE + STAGES * 8;
    static constexpr int ALIGN = 8;
};

template <typename FP, bool MULTI, bool DIAG>
__global__ void __launch_bounds__(GridTma<FP>::THREADS)
    k_stream_soa_grid_tma(SoaPtrs s, const __grid_constant__ GridArgs<FP> g,
                          const __grid_constant__ Coefs<FP> co, int64_t n_tiles, int64_t n_main,
                          int64_t n, double *partials) {
    using G = GridTma<FP>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bar = (uint64_t *)(smem + G::STAGES * G::STAGE);
    __shared__ TypeCoef<FP> s_t[MULTI ? kMaxTypes : 1];
    const FP *src[6] = {(const FP *)s.x,  (const FP *)s.y,  (const FP *)s.z,
                        (const FP *)s.px, (const FP *)s.py, (const FP *)s.pz};
    const bool has_w = DIAG && s.w != nullptr;

    if (threadIdx.x == 0) {
        for (int k = 0; k < G::STAGES; ++k) mbar_init(&bar[k], 1);
        fence_proxy_async_smem();
    }
    if (MULTI) load_type_table(co, s_t);
    else __syncthreads();

    auto slot = [&](int stage, int k) -> FP * {
        return (FP *)(smem + stage * G::STAGE + k * G::ARR);
    };
    auto tslot = [&](int stage) -> int16_t * {
        return (int16_t *)(smem + stage * G::STAGE + G::NSLOT * G::ARR);
    };
    auto tile_count = [&](int64_t t) -> int {
        const int64_t c = n_main - t * G::TP;
        return c < G::TP ? (int)c : G::TP;
    };
    auto issue = [&](int64_t t, int stage) {
        const int c = tile_count(t);
        const uint32_t b = (uint32_t)c * sizeof(FP);
        const int64_t i0 = t * G::TP;
        const uint32_t tx = 6 * b + (has_w ? b : 0) + (MULTI ? 2u * c : 0u);
        mbar_arrive_expect_tx(&bar[stage], tx);
        for (int k = 0; k < 6; ++k) bulk_g2s(slot(stage, k), src[k] + i0, b, &bar[stage]);
        if (has_w) bulk_g2s(slot(stage, 6), (const FP *)s.w + i0, b, &bar[stage]);
        if (MULTI) bulk_g2s(tslot(stage), s.type + i0, 2u * c, &bar[stage]);
    };

    if (threadIdx.x == 0)
        for (int k = 0; k < G::STAGES; ++k) {
            const int64_t t = blockIdx.x + (int64_t)k * gridDim.x;
            if (t < n_tiles) issue(t, k);
        }

    double ke = 0.0, cnt = 0.0;
    for (int64_t it = 0;; ++it) {
        const int64_t t = blockIdx.x + it * gridDim.x;
        if (t >= n_tiles) break;
        const int stage = (int)(it % G::STAGES);
        mbar_wait(&bar[stage], (uint32_t)((it / G::STAGES) & 1));
        const int c = tile_count(t);
        FP *X = slot(stage, 0), *Y = slot(stage, 1), *Z = slot(stage, 2);
        FP *PX = slot(stage, 3), *PY = slot(stage, 4), *PZ = slot(stage, 5);
        FP ex[G::PPT], ey[G::PPT], ez[G::PPT], bx[G::PPT], by[G::PPT], bz[G::PPT];
#pragma unroll
        for (int q = 0; q < G::PPT; ++q) {  // independent gathers first (ILP)
            const int j = threadIdx.x + q * G::THREADS;
            if (j < c) grid_gather<FP>(g, X[j], Y[j], Z[j], ex[q], ey[q], ez[q], bx[q], by[q], bz[q]);
        }
#pragma unroll
        for (int q = 0; q < G::PPT; ++q) {
            const int j = threadIdx.x + q * G::THREADS;
            if (j < c) {
                const TypeCoef<FP> tc = MULTI ? s_t[tslot(stage)[j]] : co.t[0];
                FP x = X[j], y = Y[j], z = Z[j], px = PX[j], py = PY[j], pz = PZ[j];
                FP ux, uy, uz, gam;
                push_one<FP>(x, y, z, px, py, pz, gam, ex[q], ey[q], ez[q], bx[q], by[q], bz[q],
                             tc, ux, uy, uz);
                X[j] = x; Y[j] = y; Z[j] = z; PX[j] = px; PY[j] = py; PZ[j] = pz;
                slot(stage, 7)[j] = gam;
                if (DIAG) {
                    ke += (double)kinetic_energy<FP>(ux, uy, uz, gam,
                                                     has_w ? slot(stage, 6)[j] : FP(1), tc);
                    cnt += 1.0;
                }
            }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t b = (uint32_t)c * sizeof(FP);
            const int64_t i0 = t * G::TP;
            FP *dst[7] = {(FP *)s.x, (FP *)s.y, (FP *)s.z, (FP *)s.px, (FP *)s.py, (FP *)s.pz,
                          (FP *)s.g};
            for (int k = 0; k < 6; ++k) bulk_s2g(dst[k] + i0, slot(stage, k), b);
            bulk_s2g(dst[6] + i0, slot(stage, 7), b);
            bulk_commit();
            const int64_t tn = t + (int64_t)G::STAGES * gridDim.x;
            if (tn < n_tiles) {
                bulk_wait_read_all();
                issue(tn, stage);
            }
        }
    }
    // ragged tail (< ALIGN particles): direct global access, same arithmetic
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x < n - n_main) {
        const int64_t i = n_main + threadIdx.x;
        FP *X = (FP *)s.x, *Y = (FP *)s.y, *Z = (FP *)s.z;
        FP *PX = (FP *)s.px, *PY = (FP *)s.py, *PZ = (FP *)s.pz;
        const TypeCoef<FP> tc = MULTI ? s_t[s.type[i]] : co.t[0];
        FP x = X[i], y = Y[i], z = Z[i], px = PX[i], py = PY[i], pz = PZ[i];
        FP ux, uy, uz, gam, Ex, Ey, Ez, Bx, By, Bz;
        grid_gather<FP>(g, x, y, z, Ex, Ey, Ez, Bx, By, Bz);
        push_one<FP>(x, y, z, px, py, pz, gam, Ex, Ey, Ez, Bx, By, Bz, tc, ux, uy, uz);
        X[i] = x; Y[i] = y; Z[i] = z; PX[i] = px; PY[i] = py; PZ[i] = pz;
        ((FP *)s.g)[i] = gam;
        if (DIAG) {
            ke += (double)kinetic_energy<FP>(ux, uy, uz, gam, has_w ? ((const FP *)s.w)[i] : FP(1),
                                             tc);
            cnt += 1.0;
        }
    }
    if (threadIdx.x == 0) bulk_wait_all();
    if (DIAG) block_diag_partial<GridTma<FP>::THREADS>(ke, cnt, partials);
}

template <typename FP, bool MULTI, bool DIAG>
static cudaError_t dispatch_grid_tma(const EnsView &e, const GridArgs<FP> &g, const Coefs<FP> &co,
                                     DiagOut *diag, int device, cudaStream_t st) {
    using G = GridTma<FP>;
    auto kern = k_stream_soa_grid_tma<FP, MULTI, DIAG>;
    static bool attr_set[64] = {};
    if (device >= 0 && device < 64 && !attr_set[device]) {
        cudaError_t err =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        if (err != cudaSuccess) return err;
        attr_set[device] = true;
    }
    int per_sm = 0;
    cudaError_t err =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::THREADS, G::SMEM);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) per_sm = 1;
    const int64_t n_main = e.n / G::ALIGN * G::ALIGN;
    const int64_t n_tiles = (n_main + G::TP - 1) / G::TP;
    int64_t grid = (int64_t)sm_count(device) * per_sm;
    if (grid > n_tiles) grid = n_tiles > 0 ? n_tiles : 1;
    if (DIAG && grid > diag->cap) grid = diag->cap;
    kern<<<(unsigned)grid, G::THREADS, G::SMEM, st>>>(e.soa, g, co, n_tiles, n_main, e.n,
                                                     diag ? diag->partials : nullptr);
    if (diag) diag->written = DIAG ? grid : 0;
    return cudaGetLastError();
}

// Requires 16 B-aligned state arrays (bulk copies); the caller checks.
template <typename FP>
cudaError_t launch_stream_soa_grid_tma(const EnsView &e, const GridArgs<FP> &g,
                                       const Coefs<FP> &co, bool multi, DiagOut *diag,
                                       int device, cudaStream_t st) {
    if (e.n == 0) {
        if (diag) diag->written = 0;
        return cudaSuccess;
    }
    const bool d = diag != nullptr;
    if (multi)
        return d ? dispatch_grid_tma<FP, true, true>(e, g, co, diag, device, st)
                 : dispatch_grid_tma<FP, true, false>(e, g, co, diag, device, st);
    return d ? dispatch_grid_tma<FP, false, true>(e, g, co, diag, device, st)
             : dispatch_grid_tma<FP, false, false>(e, g, co, diag, device, st);
}

template cudaError_t launch_stream_soa_grid_tma<float>(const EnsView &, const GridArgs<float> &,
                                                       const Coefs<float> &, bool, DiagOut *, int,
                                                       cudaStream_t);
template cudaError_t launch_stream_soa_grid_tma<double>(const EnsView &, const GridArgs<double> &,
                                                        const Coefs<double> &, bool, DiagOut *,
                                                        int, cudaStream_t);

template cudaError_t launch_stream_soa_tma<float>(const EnsView &, const FieldSoaPtrs &,
                                                  const Coefs<float> &, bool, DiagOut *, int,
                                                  cudaStream_t);
template cudaError_t launch_stream_soa_tma<double>(const EnsView &, const FieldSoaPtrs &,
                                                   const Coefs<double> &, bool, DiagOut *, int,
                                                   cudaStream_t);

}  // namespace boris
