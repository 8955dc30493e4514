// k_util.cu -- diagnostics (kinetic energy + finalize), canonical <-> layout
// conversion for upload/download, type-index validation, defaults.
#include <mutex>

#include "boris_internal.h"

namespace boris {

int sm_count(int device) {
    static int cache[64] = {};
    if (device >= 0 && device < 64 && cache[device] > 0) return cache[device];
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0)
        v = 148;
    if (device >= 0 && device < 64) cache[device] = v;
    return v;
}

// Stream-ordered scratch (sort keys, permutation blocks, staging) comes from one
// library-owned pool per device whose release threshold keeps up to 1/16 of the
// device memory cached across synchronisations: repeated sorts/uploads then reuse
// mapped memory instead of re-mapping hundreds of MB per call.  The process's
// default pool is left untouched.
static cudaMemPool_t scratch_pool(int device) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    if (device < 0 || device >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[device]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        cudaMemPool_t p = nullptr;
        if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        size_t total = 0, free_b = 0;
        uint64_t keep = 1ull << 32;
        if (cudaMemGetInfo(&free_b, &total) == cudaSuccess) keep = total / 16;
        cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
        pools[device] = p;
    }
    return pools[device];
}

cudaError_t scratch_alloc(void **ptr, size_t bytes, cudaStream_t st) {
    int dev = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err != cudaSuccess) return err;
    cudaMemPool_t pool = scratch_pool(dev);
    if (!pool) return cudaMallocAsync(ptr, bytes, st);
    return cudaMallocFromPoolAsync(ptr, bytes, pool, st);
}

void scratch_free(void *ptr, cudaStream_t st) {
    if (ptr) cudaFreeAsync(ptr, st);
}

int64_t stream_grid(int64_t work_blocks, int blocks_per_sm, int device, int waves) {
    // Grid-stride kernels: up to `waves` waves of `blocks_per_sm` resident blocks per SM.
    // The pure HBM streams (k_stream_soa_*) take kStreamWaves = 64: many short-lived
    // blocks beat few looping ones there, fresh blocks issuing their loads while retiring
    // blocks store (C2 fp32 SoA at 1e8: 4 waves 11.66 ps, 16: 11.36, 64: 11.12 = 6.83
    // TB/s; C5 bench 0.97 -> 1.00 of copy).  The gather / deposition kernels keep 4
    // (64 measured slower: grid push 11.4 -> 11.9 ps, PIC 25.3 -> 28.7,
    // profiles/r02/exp_stream_waves.jsonl).
    const int64_t cap = (int64_t)sm_count(device) * blocks_per_sm * waves;
    return work_blocks < cap ? work_blocks : cap;
}

int64_t resident_grid(const void *kernel, int threads, int64_t work_blocks, int device) {
    // ALU-bound grid-stride kernels: exactly the blocks that are resident at once
    // (occupancy of this instantiation), so every block starts in the first wave
    // and all do the same work -- no partial tail wave.
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) !=
            cudaSuccess ||
        per_sm < 1) {
        (void)cudaGetLastError();
        per_sm = 1;
    }
    const int64_t cap = (int64_t)sm_count(device) * per_sm;
    return work_blocks < cap ? work_blocks : cap;
}

// ---------------------------------------------------------------------------
// Kinetic-energy diagnostic of the current state (reading c17).
// ---------------------------------------------------------------------------
template <typename FP, int LAYOUT, bool MULTI>
__global__ void __launch_bounds__(kStreamThreads)
    k_kinetic_energy(EnsView e, const __grid_constant__ KCoefs<FP, MULTI> co, double *partials) {
    __shared__ TypeCoef<FP> s_t[MULTI ? kMaxTypes : 1];
    if (MULTI) load_type_table(co, s_t);
    double ke = 0.0, cnt = 0.0;
    const int64_t stride = (int64_t)gridDim.x * kStreamThreads;
    for (int64_t i = (int64_t)blockIdx.x * kStreamThreads + threadIdx.x; i < e.n; i += stride) {
        FP px, py, pz, g, w;
        int ty;
        if (LAYOUT == BORIS_LAYOUT_SOA) {
            px = ((const FP *)e.soa.px)[i];
            py = ((const FP *)e.soa.py)[i];
            pz = ((const FP *)e.soa.pz)[i];
            w = e.soa.w ? ((const FP *)e.soa.w)[i] : FP(1);
            ty = (MULTI && e.soa.type) ? e.soa.type[i] : 0;
        } else {
            constexpr int RB = sizeof(FP) == 4 ? 36 : 72;
            const unsigned char *rec = (const unsigned char *)e.aos + i * RB;
            const FP *r = (const FP *)rec;
            px = r[3]; py = r[4]; pz = r[5]; w = r[6];
            ty = MULTI ? *(const int16_t *)(rec + 8 * sizeof(FP)) : 0;
        }
        const TypeCoef<FP> tc = MULTI ? s_t[ty] : co.t[0];
        // gamma from p (eq. 5), so the diagnostic does not depend on a stored gamma
        const FP ux = b_mul(px, tc.S), uy = b_mul(py, tc.S), uz = b_mul(pz, tc.S);
        g = b_sqrt(b_fma(tc.kappa2, b_norm2(ux, uy, uz), FP(1)));
        ke += (double)kinetic_energy<FP>(ux, uy, uz, g, w, tc);
        cnt += 1.0;
    }
    block_diag_partial<kStreamThreads>(ke, cnt, partials);
}

template <typename FP>
cudaError_t launch_kinetic_energy(const EnsView &e, const Coefs<FP> &co, bool multi,
                                  DiagOut *diag, int device, cudaStream_t st) {
    const int64_t blocks = (e.n + kStreamThreads - 1) / kStreamThreads;
    int64_t grid = stream_grid(blocks > 0 ? blocks : 1, 2048 / kStreamThreads, device, kStreamWaves);
    if (grid > diag->cap) grid = diag->cap;
    const bool soa = e.layout == BORIS_LAYOUT_SOA;
    if (soa && multi)
        k_kinetic_energy<FP, BORIS_LAYOUT_SOA, true><<<(unsigned)grid, kStreamThreads, 0, st>>>(e, kcoefs<true>(co), diag->partials);
    else if (soa)
        k_kinetic_energy<FP, BORIS_LAYOUT_SOA, false><<<(unsigned)grid, kStreamThreads, 0, st>>>(e, kcoefs<false>(co), diag->partials);
    else if (multi)
        k_kinetic_energy<FP, BORIS_LAYOUT_AOS, true><<<(unsigned)grid, kStreamThreads, 0, st>>>(e, kcoefs<true>(co), diag->partials);
    else
        k_kinetic_energy<FP, BORIS_LAYOUT_AOS, false><<<(unsigned)grid, kStreamThreads, 0, st>>>(e, kcoefs<false>(co), diag->partials);
    diag->written = grid;
    return cudaGetLastError();
}
template cudaError_t launch_kinetic_energy<float>(const EnsView &, const Coefs<float> &, bool,
                                                  DiagOut *, int, cudaStream_t);
template cudaError_t launch_kinetic_energy<double>(const EnsView &, const Coefs<double> &, bool,
                                                   DiagOut *, int, cudaStream_t);

// Fixed-order reduction of (ke, count) partials: thread t sums pairs t, t+T, ...
// in index order, then a fixed tree.  Deterministic for a given partial count.
__global__ void __launch_bounds__(kFinalizeThreads)
    k_diag_finalize(const double *partials, int64_t pairs, double *out) {
    __shared__ double s_ke[kFinalizeThreads], s_cnt[kFinalizeThreads];
    double ke = 0.0, cnt = 0.0;
    for (int64_t i = threadIdx.x; i < pairs; i += kFinalizeThreads) {
        ke += partials[2 * i];
        cnt += partials[2 * i + 1];
    }
    s_ke[threadIdx.x] = ke;
    s_cnt[threadIdx.x] = cnt;
    __syncthreads();
    for (int h = kFinalizeThreads / 2; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) {
            s_ke[threadIdx.x] += s_ke[threadIdx.x + h];
            s_cnt[threadIdx.x] += s_cnt[threadIdx.x + h];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = s_ke[0];
        out[1] = s_cnt[0];
    }
}

cudaError_t launch_diag_finalize(const double *partials, int64_t pairs, double *out,
                                 cudaStream_t st) {
    k_diag_finalize<<<1, kFinalizeThreads, 0, st>>>(partials, pairs, out);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Upload / download conversion (canonical double, xyz interleaved <-> layout).
// ---------------------------------------------------------------------------
template <typename FP>
__global__ void k_from_canonical(EnsView e, int64_t first, int64_t count, const double *pos,
                                 const double *mom, const double *w, const int16_t *type,
                                 const double *gamma, const double *inv_mc2, int has_w,
                                 int has_type) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride) {
        const int64_t i = first + j;
        int ty;
        FP *rec = nullptr;
        if (e.layout == BORIS_LAYOUT_SOA) {
            if (has_type && e.soa.type) e.soa.type[i] = type[j];
            ty = e.soa.type ? e.soa.type[i] : 0;
        } else {
            constexpr int RB = sizeof(FP) == 4 ? 36 : 72;
            unsigned char *r = (unsigned char *)e.aos + i * RB;
            rec = (FP *)r;
            int16_t *tp = (int16_t *)(r + 8 * sizeof(FP));
            if (has_type) tp[0] = type[j];
            ty = tp[0];
        }
        const double px = mom[3 * j], py = mom[3 * j + 1], pz = mom[3 * j + 2];
        // reading c3: gamma = sqrt(1 + |p|^2/(mc)^2) unless given
        const double g = gamma ? gamma[j]
                               : sqrt(1.0 + (px * px + py * py + pz * pz) * inv_mc2[ty]);
        if (e.layout == BORIS_LAYOUT_SOA) {
            ((FP *)e.soa.x)[i] = (FP)pos[3 * j];
            ((FP *)e.soa.y)[i] = (FP)pos[3 * j + 1];
            ((FP *)e.soa.z)[i] = (FP)pos[3 * j + 2];
            ((FP *)e.soa.px)[i] = (FP)px;
            ((FP *)e.soa.py)[i] = (FP)py;
            ((FP *)e.soa.pz)[i] = (FP)pz;
            ((FP *)e.soa.g)[i] = (FP)g;
            if (has_w && e.soa.w) ((FP *)e.soa.w)[i] = (FP)w[j];
        } else {
            rec[0] = (FP)pos[3 * j]; rec[1] = (FP)pos[3 * j + 1]; rec[2] = (FP)pos[3 * j + 2];
            rec[3] = (FP)px; rec[4] = (FP)py; rec[5] = (FP)pz;
            if (has_w) rec[6] = (FP)w[j];
            rec[7] = (FP)g;
        }
    }
}

template <typename FP>
__global__ void k_to_canonical(EnsView e, int64_t first, int64_t count, double *pos,
                               double *mom, double *w, double *gamma, int16_t *type) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride) {
        const int64_t i = first + j;
        if (e.layout == BORIS_LAYOUT_SOA) {
            pos[3 * j] = ((const FP *)e.soa.x)[i];
            pos[3 * j + 1] = ((const FP *)e.soa.y)[i];
            pos[3 * j + 2] = ((const FP *)e.soa.z)[i];
            mom[3 * j] = ((const FP *)e.soa.px)[i];
            mom[3 * j + 1] = ((const FP *)e.soa.py)[i];
            mom[3 * j + 2] = ((const FP *)e.soa.pz)[i];
            w[j] = e.soa.w ? (double)((const FP *)e.soa.w)[i] : 1.0;
            gamma[j] = ((const FP *)e.soa.g)[i];
            type[j] = e.soa.type ? e.soa.type[i] : 0;
        } else {
            constexpr int RB = sizeof(FP) == 4 ? 36 : 72;
            const unsigned char *r = (const unsigned char *)e.aos + i * RB;
            const FP *rec = (const FP *)r;
            pos[3 * j] = rec[0]; pos[3 * j + 1] = rec[1]; pos[3 * j + 2] = rec[2];
            mom[3 * j] = rec[3]; mom[3 * j + 1] = rec[4]; mom[3 * j + 2] = rec[5];
            w[j] = rec[6];
            gamma[j] = rec[7];
            type[j] = *(const int16_t *)(r + 8 * sizeof(FP));
        }
    }
}

static unsigned conv_grid(int64_t count) {
    int64_t b = (count + 255) / 256;
    if (b > 65535) b = 65535;
    return (unsigned)(b > 0 ? b : 1);
}

cudaError_t launch_from_canonical(const EnsView &e, int64_t first, int64_t count,
                                  const double *d_pos, const double *d_mom, const double *d_w,
                                  const int16_t *d_type, const double *d_gamma,
                                  const double *d_inv_mc2_by_type, int /*n_types*/, int has_w,
                                  int has_type, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    if (e.precision == BORIS_FP32)
        k_from_canonical<float><<<conv_grid(count), 256, 0, st>>>(
            e, first, count, d_pos, d_mom, d_w, d_type, d_gamma, d_inv_mc2_by_type, has_w,
            has_type);
    else
        k_from_canonical<double><<<conv_grid(count), 256, 0, st>>>(
            e, first, count, d_pos, d_mom, d_w, d_type, d_gamma, d_inv_mc2_by_type, has_w,
            has_type);
    return cudaGetLastError();
}

cudaError_t launch_to_canonical(const EnsView &e, int64_t first, int64_t count, double *d_pos,
                                double *d_mom, double *d_w, double *d_gamma, int16_t *d_type,
                                cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    if (e.precision == BORIS_FP32)
        k_to_canonical<float><<<conv_grid(count), 256, 0, st>>>(e, first, count, d_pos, d_mom,
                                                                 d_w, d_gamma, d_type);
    else
        k_to_canonical<double><<<conv_grid(count), 256, 0, st>>>(e, first, count, d_pos, d_mom,
                                                                  d_w, d_gamma, d_type);
    return cudaGetLastError();
}

__global__ void k_check_types(const unsigned char *type, int64_t stride, int64_t n, int n_types,
                              unsigned long long *bad) {
    unsigned long long local = 0;
    const int64_t s = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += s) {
        const int t = *(const int16_t *)(type + i * stride);
        local += (t < 0 || t >= n_types) ? 1ull : 0ull;
    }
    if (local) atomicAdd(bad, local);
}

cudaError_t launch_check_types(const int16_t *type, int64_t stride_bytes, int64_t n, int n_types,
                               unsigned long long *d_bad, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_check_types<<<conv_grid(n), 256, 0, st>>>((const unsigned char *)type, stride_bytes, n,
                                                n_types, d_bad);
    return cudaGetLastError();
}

template <typename FP>
__global__ void k_fill_defaults(EnsView e) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e.n; i += stride) {
        if (e.layout == BORIS_LAYOUT_SOA) {
            ((FP *)e.soa.w)[i] = FP(1);
            ((FP *)e.soa.g)[i] = FP(1);
        } else {
            constexpr int RB = sizeof(FP) == 4 ? 36 : 72;
            FP *rec = (FP *)((unsigned char *)e.aos + i * RB);
            rec[6] = FP(1);
            rec[7] = FP(1);
        }
    }
}

cudaError_t launch_fill_defaults(const EnsView &e, cudaStream_t st) {
    if (e.n == 0) return cudaSuccess;
    if (e.precision == BORIS_FP32)
        k_fill_defaults<float><<<conv_grid(e.n), 256, 0, st>>>(e);
    else
        k_fill_defaults<double><<<conv_grid(e.n), 256, 0, st>>>(e);
    return cudaGetLastError();
}

}  // namespace boris
