// k_stream_aos.cu -- single-step AoS Boris push with TMA bulk-copy tile staging
// (paper §3 "Particle" records; AoS vs SoA L237-250;
// SURVEY §8(a) rows a1-a13, Appendix A "AoS kernel").
//
// Records are 36 B (fp32) / 72 B (fp64): per-thread global loads would be
// stride-36/72 and uncoalesced.  Instead each CTA is a persistent pipeline:
// one elected thread streams tiles of kAosThreads records (+ their {E,B} field
// records) HBM -> shared memory with 1-D TMA bulk copies
// (cp.async.bulk ... mbarrier::complete_tx), STAGES tiles in flight; every
// thread pushes one particle in shared memory (record stride 9 words fp32 /
// 18 words fp64: bank-conflict free), then the elected thread writes the whole
// tile back with one bulk store (cp.async.bulk.global.shared::cta).  Writing
// full records keeps every DRAM sector fully written (no read-modify-write).
// Layout-implied traffic: fp32 36+24 read + 36 write = 96 B/particle-step.
#include "boris_internal.h"
#include "tma.cuh"

// fp32: 8 stages (one CTA per SM, 122 KB of tiles in flight) measured best: 14.9 ps at
// 1e8 vs 15.3 with 4 stages x 3 CTAs (6, 10, 12, 14 stages: 15.0-15.7,
// profiles/r02/exp_aos_stages.jsonl); fp64 3 stages (2-14 tried).
#ifndef BORIS_AOS_STAGES32
#define BORIS_AOS_STAGES32 8
#endif
#ifndef BORIS_AOS_STAGES64
#define BORIS_AOS_STAGES64 3
#endif

namespace boris {

namespace {

template <typename FP>
struct AosGeom {
    static constexpr int RB = sizeof(FP) == 4 ? BORIS_AOS_RECORD_BYTES_FP32
                                              : BORIS_AOS_RECORD_BYTES_FP64;
    static constexpr int FB = 6 * (int)sizeof(FP);
    static constexpr int TP = kAosThreads;           // particles per tile
    static constexpr int STAGES = sizeof(FP) == 4 ? BORIS_AOS_STAGES32 : BORIS_AOS_STAGES64;
    static constexpr int TILE_R = TP * RB;           // 9216 / 18432 B
    static constexpr int TILE_F = TP * FB;           // 6144 / 12288 B
    static constexpr int SMEM = STAGES * (TILE_R + TILE_F) + STAGES * 8;
    static constexpr int TYPE_OFF = 8 * (int)sizeof(FP);  // 32 / 64
    // bulk copies move multiples of 16 B: tiles cover a multiple of ALIGN particles
    static constexpr int ALIGN = sizeof(FP) == 4 ? 4 : 2;
};

// Push particle j of a shared-memory record tile (record layout of libboris.h).
template <typename FP, bool MULTI, bool DIAG>
__device__ __forceinline__ void push_record(unsigned char *rec, const FP *fld,
                                            const KCoefs<FP, MULTI> &co, const TypeCoef<FP> *s_t,
                                            double &ke,
                                            double &cnt) {
    FP *r = (FP *)rec;
    const int ty = MULTI ? *(const int16_t *)(rec + AosGeom<FP>::TYPE_OFF) : 0;
    const TypeCoef<FP> tc = MULTI ? s_t[ty] : co.t[0];
    FP ux, uy, uz, gam;
    push_one<FP>(r[0], r[1], r[2], r[3], r[4], r[5], gam, fld[0], fld[1], fld[2], fld[3], fld[4],
                 fld[5], tc, ux, uy, uz);
    r[7] = gam;
    if (DIAG) {
        ke += (double)kinetic_energy<FP>(ux, uy, uz, gam, r[6], tc);
        cnt += 1.0;
    }
}

}  // namespace

template <typename FP, bool MULTI, bool DIAG>
__global__ void __launch_bounds__(kAosThreads)
    k_stream_aos(unsigned char *rec, const unsigned char *frec,
                 const __grid_constant__ KCoefs<FP, MULTI> co, int64_t n_tiles, int64_t n_main,
                 int64_t n, double *partials) {
    using Gm = AosGeom<FP>;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *s_rec = smem;
    unsigned char *s_fld = smem + Gm::STAGES * Gm::TILE_R;
    uint64_t *bar = (uint64_t *)(s_fld + Gm::STAGES * Gm::TILE_F);
    __shared__ TypeCoef<FP> s_t[MULTI ? kMaxTypes : 1];

    if (threadIdx.x == 0) {
        for (int s = 0; s < Gm::STAGES; ++s) mbar_init(&bar[s], 1);
        fence_proxy_async_smem();
    }
    if (MULTI) load_type_table(co, s_t);  // contains __syncthreads
    else __syncthreads();

    auto tile_count = [&](int64_t t) -> int {
        const int64_t c = n_main - t * Gm::TP;
        return c < Gm::TP ? (int)c : Gm::TP;
    };
    auto issue = [&](int64_t t, int s) {
        const int c = tile_count(t);
        const uint32_t br = (uint32_t)c * Gm::RB, bf = (uint32_t)c * Gm::FB;
        mbar_arrive_expect_tx(&bar[s], br + bf);
        bulk_g2s(s_rec + s * Gm::TILE_R, rec + t * Gm::TILE_R, br, &bar[s]);
        bulk_g2s(s_fld + s * Gm::TILE_F, frec + t * Gm::TILE_F, bf, &bar[s]);
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < Gm::STAGES; ++s) {
            const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
            if (t < n_tiles) issue(t, s);
        }
    }

    double ke = 0.0, cnt = 0.0;
    for (int64_t k = 0;; ++k) {
        const int64_t t = blockIdx.x + k * gridDim.x;
        if (t >= n_tiles) break;
        const int s = (int)(k % Gm::STAGES);
        mbar_wait(&bar[s], (uint32_t)((k / Gm::STAGES) & 1));
        const int c = tile_count(t);
        if ((int)threadIdx.x < c)
            push_record<FP, MULTI, DIAG>(s_rec + s * Gm::TILE_R + threadIdx.x * Gm::RB,
                                         (const FP *)(s_fld + s * Gm::TILE_F) + threadIdx.x * 6,
                                         co, s_t, ke, cnt);
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            bulk_s2g(rec + t * Gm::TILE_R, s_rec + s * Gm::TILE_R, (uint32_t)c * Gm::RB);
            bulk_commit();
            const int64_t tn = t + (int64_t)Gm::STAGES * gridDim.x;
            if (tn < n_tiles) {
                bulk_wait_read_all();  // the stage's smem has been read out by the store
                issue(tn, s);
            }
        }
    }
    // ragged tail (< ALIGN particles not covered by 16 B-multiple tiles): direct access
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x < n - n_main) {
        const int64_t i = n_main + threadIdx.x;
        push_record<FP, MULTI, DIAG>(rec + i * Gm::RB, (const FP *)(frec + i * Gm::FB), co, s_t,
                                     ke, cnt);
    }
    if (threadIdx.x == 0) bulk_wait_all();
    if (DIAG) block_diag_partial<kAosThreads>(ke, cnt, partials);
}

template <typename FP, bool MULTI, bool DIAG>
static cudaError_t dispatch_aos(const EnsView &e, const void *frec, const Coefs<FP> &co,
                                DiagOut *diag, int device, cudaStream_t st) {
    using Gm = AosGeom<FP>;
    auto kern = k_stream_aos<FP, MULTI, DIAG>;
    static bool attr_set[64] = {};  // per device
    if (device >= 0 && device < 64 && !attr_set[device]) {
        cudaError_t err =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Gm::SMEM);
        if (err != cudaSuccess) return err;
        attr_set[device] = true;
    }
    int per_sm = 0;
    cudaError_t err =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kAosThreads, Gm::SMEM);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) per_sm = 1;
    const int64_t n_main = e.n / Gm::ALIGN * Gm::ALIGN;
    const int64_t n_tiles = (n_main + Gm::TP - 1) / Gm::TP;
    int64_t grid = (int64_t)sm_count(device) * per_sm;
    if (grid > n_tiles) grid = n_tiles > 0 ? n_tiles : 1;
    if (DIAG && grid > diag->cap) grid = diag->cap;
    kern<<<(unsigned)grid, kAosThreads, Gm::SMEM, st>>>(
        (unsigned char *)e.aos, (const unsigned char *)frec, kcoefs<MULTI>(co), n_tiles, n_main, e.n,
        diag ? diag->partials : nullptr);
    if (diag) diag->written = DIAG ? grid : 0;
    return cudaGetLastError();
}

template <typename FP>
cudaError_t launch_stream_aos(const EnsView &e, const void *field_records, const Coefs<FP> &co,
                              bool multi, DiagOut *diag, int device, cudaStream_t st) {
    if (e.n == 0) {
        if (diag) diag->written = 0;
        return cudaSuccess;
    }
    const bool d = diag != nullptr;
    if (multi)
        return d ? dispatch_aos<FP, true, true>(e, field_records, co, diag, device, st)
                 : dispatch_aos<FP, true, false>(e, field_records, co, diag, device, st);
    return d ? dispatch_aos<FP, false, true>(e, field_records, co, diag, device, st)
             : dispatch_aos<FP, false, false>(e, field_records, co, diag, device, st);
}

template cudaError_t launch_stream_aos<float>(const EnsView &, const void *,
                                              const Coefs<float> &, bool, DiagOut *, int,
                                              cudaStream_t);
template cudaError_t launch_stream_aos<double>(const EnsView &, const void *,
                                               const Coefs<double> &, bool, DiagOut *, int,
                                               cudaStream_t);

}  // namespace boris
