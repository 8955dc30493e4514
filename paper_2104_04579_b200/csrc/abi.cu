// abi.cu -- the C ABI of libboris (include/libboris.h): handles, argument
// validation, error strings, kernel dispatch, and the host-resident streaming
// pipeline.  Every compute step runs in the kernels of k_*.cu; this file only
// validates, prepares per-push coefficients (double on the host, reading a3)
// and enqueues work.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <atomic>

#include "boris_internal.h"

// Process-wide options (boris_set_option); the library reads no environment.
static std::atomic<int64_t> g_opt_fused_generic{0};
static std::atomic<int64_t> g_opt_host_chunk{(int64_t)4 << 20};
static std::atomic<int64_t> g_opt_md_order{1};

using namespace boris;

// ---------------------------------------------------------------------------
// Errors
// ---------------------------------------------------------------------------
namespace {
thread_local std::string g_last_error;

boris_status fail(boris_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}
boris_status ok() {
    g_last_error.clear();
    return BORIS_OK;
}
boris_status cuda_fail(cudaError_t err, const char *what) {
    // The error is reported here, so take it out of the runtime's per-thread
    // last-error slot: a failed cudaMalloc (not sticky) would otherwise surface
    // again at the next launch check and fail an unrelated push.
    (void)cudaGetLastError();
    if (err == cudaErrorMemoryAllocation)
        return fail(BORIS_E_OUT_OF_MEMORY, "%s: %s", what, cudaGetErrorString(err));
    return fail(BORIS_E_CUDA, "%s: %s", what, cudaGetErrorString(err));
}
#define CUDA_TRY(call, what)                                   \
    do {                                                       \
        cudaError_t _e = (call);                               \
        if (_e != cudaSuccess) return cuda_fail(_e, (what));   \
    } while (0)

// Switch to a device for the duration of a call, restore on exit.
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev) {
        err = cudaGetDevice(&prev);
        if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

bool finite3(const double *v) {
    return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]);
}

size_t fp_size(int precision) { return precision == BORIS_FP32 ? 4 : 8; }
size_t record_bytes(int precision) {
    return precision == BORIS_FP32 ? BORIS_AOS_RECORD_BYTES_FP32 : BORIS_AOS_RECORD_BYTES_FP64;
}
size_t field_record_bytes(int precision) {
    return precision == BORIS_FP32 ? BORIS_AOS_FIELD_BYTES_FP32 : BORIS_AOS_FIELD_BYTES_FP64;
}
}  // namespace

// ---------------------------------------------------------------------------
// Handles
// ---------------------------------------------------------------------------
struct HostPipeline {
    static constexpr int kBuffers = 3;  // H2D of chunk k+2 overlaps push k+1 and D2H k
    int64_t chunk = 0;
    void *dev_block[kBuffers] = {};
    SoaPtrs soa[kBuffers] = {};
    void *aos[kBuffers] = {};
    void *fsoa[kBuffers][6] = {};
    void *faos[kBuffers] = {};
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t loaded[kBuffers] = {}, computed[kBuffers] = {}, freed[kBuffers] = {};
    bool with_fields = false;
    double *chunk_diag = nullptr;  // (ke, count) per chunk, summed by the final finalize
    int64_t chunk_diag_cap = 0;
};

struct boris_ensemble {
    int device = 0;
    int memory = BORIS_MEMORY_DEVICE;
    int layout = BORIS_LAYOUT_SOA;
    int precision = BORIS_FP32;
    int64_t n = 0;
    int n_types = 1;
    boris_particle_type types[BORIS_MAX_TYPES];
    double c = 1.0;
    double time = 0.0;
    bool owned = false;
    void *block = nullptr;  // owned device allocation
    SoaPtrs soa = {};
    void *aos = nullptr;
    double *partials = nullptr;  // diag scratch (device)
    int64_t partials_cap = 0;
    unsigned long long *d_bad = nullptr;
    HostPipeline *pipe = nullptr;

    EnsView view() const {
        EnsView v;
        v.precision = precision;
        v.layout = layout;
        v.n = n;
        v.soa = soa;
        v.aos = aos;
        return v;
    }
    bool multi() const { return n_types > 1; }
};

struct boris_field {
    int kind = FK_UNIFORM;
    // per-particle arrays
    int layout = -1, precision = -1, device = -1, memory = -1;
    int64_t n = -1;
    FieldSoaPtrs soa = {};
    const void *aos = nullptr;
    // analytic
    double E[3] = {0, 0, 0}, B[3] = {0, 0, 0};
    double E0 = 0, k_hat[3] = {0, 0, 0}, e_hat[3] = {0, 0, 0}, omega = 0, k = 0, phase0 = 0;
    double A0 = 0, omega0 = 0, kd = 0;
    // grid (FK_GRID): owned packed node records on `device`, in `precision`
    void *nodes = nullptr;
    int gn[3] = {0, 0, 0};
    double org[3] = {0, 0, 0}, h[3] = {0, 0, 0};
};

namespace {

boris_status check_types_table(const boris_particle_type *types, int32_t n_types, double c) {
    if (!types) return fail(BORIS_E_INVALID_ARG, "types is NULL");
    if (n_types < 1 || n_types > BORIS_MAX_TYPES)
        return fail(BORIS_E_INVALID_ARG, "n_types=%d outside [1, %d]", n_types, BORIS_MAX_TYPES);
    if (!(std::isfinite(c) && c > 0)) return fail(BORIS_E_INVALID_ARG, "light_velocity must be > 0");
    for (int i = 0; i < n_types; ++i) {
        if (!std::isfinite(types[i].charge) || !(std::isfinite(types[i].mass) && types[i].mass > 0))
            return fail(BORIS_E_INVALID_ARG, "type %d: charge must be finite and mass > 0", i);
    }
    return BORIS_OK;
}

boris_status check_device(int device) {
    int count = 0;
    cudaError_t err = cudaGetDeviceCount(&count);
    if (err != cudaSuccess || count == 0)
        return fail(BORIS_E_NO_DEVICE, "no CUDA device (%s)", cudaGetErrorString(err));
    if (device < 0 || device >= count)
        return fail(BORIS_E_NO_DEVICE, "device %d outside [0, %d)", device, count);
    return BORIS_OK;
}

boris_status alloc_scratch(boris_ensemble *e) {
    // one (KE, count) pair per block of the largest diagnostic grid (stream_grid at
    // 8 blocks of 256 per SM)
    e->partials_cap = (int64_t)sm_count(e->device) * 8 * kStreamWaves;
    CUDA_TRY(cudaMalloc(&e->partials, (size_t)e->partials_cap * 2 * sizeof(double)),
             "cudaMalloc(diag partials)");
    CUDA_TRY(cudaMalloc(&e->d_bad, sizeof(unsigned long long)), "cudaMalloc(type check)");
    return BORIS_OK;
}

boris_ensemble *new_ensemble(int device, int memory, int layout, int precision, int64_t n,
                             const boris_particle_type *types, int32_t n_types, double c) {
    boris_ensemble *e = new boris_ensemble();
    e->device = device;
    e->memory = memory;
    e->layout = layout;
    e->precision = precision;
    e->n = n;
    e->n_types = n_types;
    for (int i = 0; i < n_types; ++i) e->types[i] = types[i];
    e->c = c;
    return e;
}

void free_pipeline(HostPipeline *p) {
    if (!p) return;
    for (int b = 0; b < HostPipeline::kBuffers; ++b) {
        if (p->dev_block[b]) cudaFree(p->dev_block[b]);
        if (p->loaded[b]) cudaEventDestroy(p->loaded[b]);
        if (p->computed[b]) cudaEventDestroy(p->computed[b]);
        if (p->freed[b]) cudaEventDestroy(p->freed[b]);
    }
    if (p->h2d) cudaStreamDestroy(p->h2d);
    if (p->d2h) cudaStreamDestroy(p->d2h);
    if (p->chunk_diag) cudaFree(p->chunk_diag);
    delete p;
}

void free_ensemble(boris_ensemble *e) {
    if (!e) return;
    if (e->owned && e->block) cudaFree(e->block);
    if (e->partials) cudaFree(e->partials);
    if (e->d_bad) cudaFree(e->d_bad);
    free_pipeline(e->pipe);
    delete e;
}

// Synchronous device check of type indices (strided for AoS records).
boris_status validate_types_device(boris_ensemble *e, cudaStream_t st) {
    if (e->n == 0) return BORIS_OK;
    const int16_t *tp;
    int64_t stride;
    if (e->layout == BORIS_LAYOUT_SOA) {
        if (!e->soa.type) return BORIS_OK;  // n_types == 1, implicit type 0
        tp = e->soa.type;
        stride = 2;
    } else {
        tp = (const int16_t *)((const unsigned char *)e->aos + 8 * fp_size(e->precision));
        stride = (int64_t)record_bytes(e->precision);
    }
    CUDA_TRY(cudaMemsetAsync(e->d_bad, 0, sizeof(unsigned long long), st), "cudaMemsetAsync");
    CUDA_TRY(launch_check_types(tp, stride, e->n, e->n_types, e->d_bad, st), "type check launch");
    unsigned long long bad = 0;
    CUDA_TRY(cudaMemcpyAsync(&bad, e->d_bad, sizeof bad, cudaMemcpyDeviceToHost, st),
             "cudaMemcpyAsync");
    CUDA_TRY(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    if (bad) return fail(BORIS_E_TYPE_OUT_OF_RANGE, "%llu type indices outside [0, %d)", bad, e->n_types);
    return BORIS_OK;
}

boris_status validate_types_host(const boris_ensemble *e) {
    const size_t rb = record_bytes(e->precision);
    for (int64_t i = 0; i < e->n; ++i) {
        int t;
        if (e->layout == BORIS_LAYOUT_SOA) {
            if (!e->soa.type) return BORIS_OK;
            t = e->soa.type[i];
        } else {
            int16_t v;
            memcpy(&v, (const unsigned char *)e->aos + i * rb + 8 * fp_size(e->precision), 2);
            t = v;
        }
        if (t < 0 || t >= e->n_types)
            return fail(BORIS_E_TYPE_OUT_OF_RANGE, "particle %lld: type %d outside [0, %d)",
                        (long long)i, t, e->n_types);
    }
    return BORIS_OK;
}

template <typename FP>
Coefs<FP> make_coefs(const boris_ensemble *e, double dt) {
    Coefs<FP> co;
    memset(&co, 0, sizeof co);
    co.n_types = e->n_types;
    for (int i = 0; i < e->n_types; ++i) {
        const double q = e->types[i].charge, m = e->types[i].mass;
        const double mc = m * e->c;
        // S = 2^k closest to 1/(mc): u = S p is exact in binary floating point
        const double S = std::ldexp(1.0, -(int)std::lround(std::log2(mc)));
        const double kappa = 1.0 / (S * mc);
        co.t[i].aE = (FP)(S * q * dt / 2.0);          // eq. 9-10
        co.t[i].alpha = (FP)(q * dt / (2.0 * mc));    // eq. 13
        co.t[i].kappa2 = (FP)(kappa * kappa);         // eq. 5
        co.t[i].kappa = (FP)kappa;
#ifdef BORIS_TEST_PERTURB_CR
        // test-only tuning build (never the product): a10 off by a relative 1e-4, which
        // the displacement parity check (tests/parity_util.py Displacement) must reject
        co.t[i].cr = (FP)(dt / (S * m) * (1.0 + BORIS_TEST_PERTURB_CR));
#else
        co.t[i].cr = (FP)(dt / (S * m));              // eq. 7
#endif
        co.t[i].S = (FP)S;
        co.t[i].invS = (FP)(1.0 / S);
        co.t[i].ke = (FP)(1.0 / (S * S * m));         // m c^2 kappa^2
    }
    return co;
}

template <typename FP>
GridArgs<FP> make_grid_args(const boris_field *f) {
    GridArgs<FP> g;
    memset(&g, 0, sizeof g);
    g.nodes = (const FP *)f->nodes;
    for (int d = 0; d < 3; ++d) {
        g.org[d] = (FP)f->org[d];
        g.inv_h[d] = (FP)(1.0 / f->h[d]);
        g.nf[d] = (FP)f->gn[d];
        g.inv_nf[d] = (FP)(1.0 / f->gn[d]);
        g.n[d] = f->gn[d];
    }
    return g;
}

template <typename FP>
AnalyticArgs<FP> make_analytic(const boris_field *f, double t0, double dt) {
    AnalyticArgs<FP> a;
    memset(&a, 0, sizeof a);
    for (int i = 0; i < 3; ++i) {
        a.E[i] = (FP)f->E[i];
        a.B[i] = (FP)f->B[i];
    }
    if (f->kind == FK_PLANE_WAVE) {
        for (int i = 0; i < 3; ++i) {
            a.kvec[i] = f->k * f->k_hat[i];
            a.kf[i] = (FP)a.kvec[i];
        }
        a.ph0 = f->phase0 - f->omega * t0;
        a.wdt = f->omega * dt;
        a.wdtf = (FP)a.wdt;
        const double *kh = f->k_hat, *eh = f->e_hat;
        const double kxe[3] = {kh[1] * eh[2] - kh[2] * eh[1], kh[2] * eh[0] - kh[0] * eh[2],
                               kh[0] * eh[1] - kh[1] * eh[0]};
        for (int i = 0; i < 3; ++i) {
            a.cE[i] = (FP)(f->E0 * eh[i]);
            a.cB[i] = (FP)(f->E0 * kxe[i]);
        }
    } else if (f->kind == FK_MDIPOLE) {
        a.A0 = (FP)f->A0;
        a.k = (FP)f->kd;
        a.k2 = (FP)(f->kd * f->kd);
        a.A0k2 = (FP)(2.0 * f->A0 * f->kd);
        a.mA02 = (FP)(-2.0 * f->A0);
        a.w0t0 = f->omega0 * t0;
        a.w0dt = f->omega0 * dt;
        a.md_order = (int)g_opt_md_order.load(std::memory_order_relaxed);
    } else if (f->kind == FK_GRID) {
        a.grid = make_grid_args<FP>(f);
    }
    // exact zeros off the y (E) and z (B) axes -> the YZ fused specialisation;
    // BORIS_OPT_FUSED_GENERIC = 1 forces the generic kernel (tests)
    const bool allow = g_opt_fused_generic.load(std::memory_order_relaxed) == 0;
    if (allow && f->kind == FK_UNIFORM)
        a.yz = a.E[0] == 0 && a.E[2] == 0 && a.B[0] == 0 && a.B[1] == 0;
    else if (allow && f->kind == FK_PLANE_WAVE)
        a.yz = a.cE[0] == 0 && a.cE[2] == 0 && a.cB[0] == 0 && a.cB[1] == 0 &&
               a.kf[1] == 0 && a.kf[2] == 0 && a.kvec[1] == 0 && a.kvec[2] == 0;
    return a;
}

// One step (or n_steps fused) on a device-resident view.
template <typename FP>
cudaError_t push_view(const boris_ensemble *e, const EnsView &v, const boris_field *f,
                      const FieldSoaPtrs &fs, const void *faos, double t0, double dt,
                      int64_t n_steps, uint32_t flags, DiagOut *diag, cudaStream_t st) {
    const Coefs<FP> co = make_coefs<FP>(e, dt);
    const int pusher = (int)((flags & BORIS_PUSH_PUSHER_MASK) >> 4);
    if (f->kind == FK_ARRAYS) {
        const bool each = (flags & BORIS_PUSH_STREAM_EACH_STEP) != 0;
        if (n_steps > 1 && !each)
            return launch_fused_arrays<FP>(v, fs, faos, co, n_steps, e->multi(), pusher, diag,
                                           e->device, st);
        for (int64_t s = 0; s < n_steps; ++s) {
            DiagOut *d = (s == n_steps - 1) ? diag : nullptr;
            cudaError_t err;
            if (pusher != PUSHER_BORIS)  // streaming kernels are Boris-only: 1-step fused launch
                err = launch_fused_arrays<FP>(v, fs, faos, co, 1, e->multi(), pusher, d,
                                              e->device, st);
            else
                err = v.layout == BORIS_LAYOUT_SOA
                          ? launch_stream_soa<FP>(v, fs, co, e->multi(), d, e->device, st)
                          : launch_stream_aos<FP>(v, faos, co, e->multi(), d, e->device, st);
            if (err != cudaSuccess) return err;
        }
        return cudaSuccess;
    }
    AnalyticArgs<FP> fa = make_analytic<FP>(f, t0, dt);
    if (f->kind == FK_MDIPOLE && !e->multi()) {  // k_fused kMdFold scaled variables
        const double q = e->types[0].charge, mc = e->types[0].mass * e->c;
        const double alpha = q * dt / (2.0 * mc);  // eq. 9-10, 13 with u = p/(m c)
        fa.mdf_k = f->kd;
        fa.mdf_ik = 1.0 / f->kd;
        fa.mdf_kick = alpha * 2.0 * f->A0;
        fa.mdf_rot = alpha * -2.0 * f->A0;
        fa.mdf_uin = (FP)(1.0 / mc);
        fa.mdf_uout = (FP)mc;
        fa.mdf_cr = (FP)(f->kd * e->c * dt);  // eq. 7: dX = k c dt u / gamma
    }
    if (f->kind == FK_GRID && n_steps == 1 && v.layout == BORIS_LAYOUT_SOA &&
        pusher == PUSHER_BORIS) {  // the PIC single step: 128-bit streaming + gather
        const cudaError_t err =
            launch_stream_soa_grid<FP>(v, fa.grid, co, e->multi(), diag, e->device, st);
        if (err != cudaErrorNotSupported) return err;
    }
    return launch_fused<FP>(v, f->kind, fa, co, n_steps, e->multi(), pusher, diag, e->device, st);
}

boris_status check_push_args(const boris_ensemble *e, const boris_field *f, double dt,
                             int64_t n_steps) {
    if (!e) return fail(BORIS_E_INVALID_ARG, "ensemble is NULL");
    if (!f) return fail(BORIS_E_INVALID_ARG, "field is NULL");
    if (!std::isfinite(dt)) return fail(BORIS_E_INVALID_ARG, "dt must be finite");
    if (n_steps < 0) return fail(BORIS_E_INVALID_ARG, "n_steps < 0");
    if (f->kind == FK_ARRAYS) {
        if (f->layout != e->layout || f->precision != e->precision || f->n != e->n ||
            f->device != e->device || f->memory != e->memory)
            return fail(BORIS_E_MISMATCH,
                        "per-particle field (layout %d, precision %d, n %lld, device %d, memory %d) "
                        "does not match the ensemble (%d, %d, %lld, %d, %d)",
                        f->layout, f->precision, (long long)f->n, f->device, f->memory, e->layout,
                        e->precision, (long long)e->n, e->device, e->memory);
    }
    if (f->kind == FK_GRID && (f->precision != e->precision || f->device != e->device))
        return fail(BORIS_E_MISMATCH, "grid field (precision %d, device %d) does not match the "
                    "ensemble (%d, %d)", f->precision, f->device, e->precision, e->device);
    return BORIS_OK;
}

// ---------------------------------------------------------------------------
// Host-resident ensembles: chunked H2D -> push -> D2H pipeline (double buffer).
// ---------------------------------------------------------------------------
int64_t host_chunk_particles() { return g_opt_host_chunk.load(std::memory_order_relaxed) / 8 * 8; }

static boris_status build_pipeline(const boris_ensemble *e, bool with_fields, HostPipeline *p);

// The staging pipeline of a host-resident ensemble, created on first use (and
// re-created with field staging when a per-particle-field push first needs it;
// the old one may still be in use by enqueued work, hence the device sync).
// On failure nothing is left half-built.
boris_status ensure_pipeline(boris_ensemble *e, bool with_fields) {
    if (e->pipe && (e->pipe->with_fields || !with_fields)) return BORIS_OK;
    if (e->pipe) {
        cudaDeviceSynchronize();
        free_pipeline(e->pipe);
        e->pipe = nullptr;
    }
    HostPipeline *p = new HostPipeline();
    const boris_status s = build_pipeline(e, with_fields, p);
    if (s != BORIS_OK) {
        free_pipeline(p);
        return s;
    }
    e->pipe = p;
    return BORIS_OK;
}

static boris_status build_pipeline(const boris_ensemble *e, bool with_fields, HostPipeline *p) {
    p->with_fields = with_fields;
    p->chunk = host_chunk_particles();
    if (p->chunk > e->n) p->chunk = (e->n + 7) / 8 * 8;
    const size_t fs = fp_size(e->precision);
    const size_t C = (size_t)p->chunk;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    size_t bytes;
    if (e->layout == BORIS_LAYOUT_SOA)
        bytes = 8 * al(C * fs) + al(C * 2) + (with_fields ? 6 * al(C * fs) : 0);
    else
        bytes = al(C * record_bytes(e->precision)) +
                (with_fields ? al(C * field_record_bytes(e->precision)) : 0);
    CUDA_TRY(cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking), "cudaStreamCreate");
    CUDA_TRY(cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking), "cudaStreamCreate");
    for (int b = 0; b < HostPipeline::kBuffers; ++b) {
        CUDA_TRY(cudaMalloc(&p->dev_block[b], bytes), "cudaMalloc(host pipeline staging)");
        CUDA_TRY(cudaEventCreateWithFlags(&p->loaded[b], cudaEventDisableTiming), "cudaEventCreate");
        CUDA_TRY(cudaEventCreateWithFlags(&p->computed[b], cudaEventDisableTiming), "cudaEventCreate");
        CUDA_TRY(cudaEventCreateWithFlags(&p->freed[b], cudaEventDisableTiming), "cudaEventCreate");
        unsigned char *q = (unsigned char *)p->dev_block[b];
        if (e->layout == BORIS_LAYOUT_SOA) {
            void **slots[8] = {&p->soa[b].x, &p->soa[b].y, &p->soa[b].z, &p->soa[b].px,
                               &p->soa[b].py, &p->soa[b].pz, &p->soa[b].w, &p->soa[b].g};
            for (int i = 0; i < 8; ++i) {
                *slots[i] = q;
                q += al(C * fs);
            }
            p->soa[b].type = (int16_t *)q;
            q += al(C * 2);
            if (with_fields)
                for (int i = 0; i < 6; ++i) {
                    p->fsoa[b][i] = q;
                    q += al(C * fs);
                }
        } else {
            p->aos[b] = q;
            q += al(C * record_bytes(e->precision));
            if (with_fields) p->faos[b] = q;
        }
    }
    return BORIS_OK;
}

template <typename FP>
boris_status push_host(boris_ensemble *e, const boris_field *f, double dt, int64_t n_steps,
                       uint32_t flags, double *d_diag, cudaStream_t st) {
    const bool arrays = f->kind == FK_ARRAYS;
    boris_status s = ensure_pipeline(e, arrays);
    if (s != BORIS_OK) return s;
    HostPipeline *p = e->pipe;
    const size_t fs = sizeof(FP);
    const bool soa = e->layout == BORIS_LAYOUT_SOA;
    const size_t rb = record_bytes(e->precision), frb = field_record_bytes(e->precision);
    const int64_t n_chunks = (e->n + p->chunk - 1) / p->chunk;
    if (d_diag && p->chunk_diag_cap < n_chunks) {
        if (p->chunk_diag) cudaFree(p->chunk_diag);
        p->chunk_diag = nullptr;
        p->chunk_diag_cap = 0;
        CUDA_TRY(cudaMalloc(&p->chunk_diag, (size_t)n_chunks * 2 * sizeof(double)),
                 "cudaMalloc(chunk diag)");
        p->chunk_diag_cap = n_chunks;
    }
    const bool with_w = d_diag && soa && e->soa.w;
    cudaEvent_t entry;
    CUDA_TRY(cudaEventCreateWithFlags(&entry, cudaEventDisableTiming), "cudaEventCreate");
    CUDA_TRY(cudaEventRecord(entry, st), "cudaEventRecord");
    CUDA_TRY(cudaStreamWaitEvent(p->h2d, entry, 0), "cudaStreamWaitEvent");
    cudaEventDestroy(entry);
    for (int64_t k = 0; k < n_chunks; ++k) {
        const int b = (int)(k % HostPipeline::kBuffers);
        const int64_t first = k * p->chunk;
        const int64_t cnt = (first + p->chunk <= e->n) ? p->chunk : e->n - first;
        // H2D (waits until buffer b's previous D2H has drained)
        CUDA_TRY(cudaStreamWaitEvent(p->h2d, p->freed[b], 0), "cudaStreamWaitEvent");
        if (soa) {
            const void *src[6] = {e->soa.x, e->soa.y, e->soa.z, e->soa.px, e->soa.py, e->soa.pz};
            void *dst[6] = {p->soa[b].x, p->soa[b].y, p->soa[b].z,
                            p->soa[b].px, p->soa[b].py, p->soa[b].pz};
            for (int i = 0; i < 6; ++i)
                CUDA_TRY(cudaMemcpyAsync(dst[i], (const unsigned char *)src[i] + first * fs,
                                         cnt * fs, cudaMemcpyHostToDevice, p->h2d), "H2D");
            if (e->multi())
                CUDA_TRY(cudaMemcpyAsync(p->soa[b].type, e->soa.type + first, cnt * 2,
                                         cudaMemcpyHostToDevice, p->h2d), "H2D");
            if (with_w)
                CUDA_TRY(cudaMemcpyAsync(p->soa[b].w, (const unsigned char *)e->soa.w + first * fs,
                                         cnt * fs, cudaMemcpyHostToDevice, p->h2d), "H2D");
            if (arrays) {
                const void *fsrc[6] = {f->soa.Ex, f->soa.Ey, f->soa.Ez,
                                       f->soa.Bx, f->soa.By, f->soa.Bz};
                for (int i = 0; i < 6; ++i)
                    CUDA_TRY(cudaMemcpyAsync(p->fsoa[b][i],
                                             (const unsigned char *)fsrc[i] + first * fs,
                                             cnt * fs, cudaMemcpyHostToDevice, p->h2d), "H2D");
            }
        } else {
            CUDA_TRY(cudaMemcpyAsync(p->aos[b], (const unsigned char *)e->aos + first * rb,
                                     cnt * rb, cudaMemcpyHostToDevice, p->h2d), "H2D");
            if (arrays)
                CUDA_TRY(cudaMemcpyAsync(p->faos[b], (const unsigned char *)f->aos + first * frb,
                                         cnt * frb, cudaMemcpyHostToDevice, p->h2d), "H2D");
        }
        CUDA_TRY(cudaEventRecord(p->loaded[b], p->h2d), "cudaEventRecord");
        // compute on the caller's stream
        CUDA_TRY(cudaStreamWaitEvent(st, p->loaded[b], 0), "cudaStreamWaitEvent");
        EnsView v;
        v.precision = e->precision;
        v.layout = e->layout;
        v.n = cnt;
        v.soa = p->soa[b];
        if (!with_w) v.soa.w = nullptr;
        if (!e->multi()) v.soa.type = nullptr;
        v.aos = p->aos[b];
        FieldSoaPtrs fsp = {p->fsoa[b][0], p->fsoa[b][1], p->fsoa[b][2],
                            p->fsoa[b][3], p->fsoa[b][4], p->fsoa[b][5]};
        DiagOut diag = {e->partials, e->partials_cap, 0};
        CUDA_TRY(push_view<FP>(e, v, f, fsp, p->faos[b], e->time, dt, n_steps, flags,
                               d_diag ? &diag : nullptr, st),
                 "push kernel launch");
        if (d_diag)
            CUDA_TRY(launch_diag_finalize(diag.partials, diag.written, p->chunk_diag + 2 * k, st),
                     "diag finalize");
        CUDA_TRY(cudaEventRecord(p->computed[b], st), "cudaEventRecord");
        // D2H of the pushed state
        CUDA_TRY(cudaStreamWaitEvent(p->d2h, p->computed[b], 0), "cudaStreamWaitEvent");
        if (soa) {
            void *dst[7] = {e->soa.x, e->soa.y, e->soa.z, e->soa.px, e->soa.py, e->soa.pz, e->soa.g};
            const void *src[7] = {p->soa[b].x, p->soa[b].y, p->soa[b].z, p->soa[b].px,
                                  p->soa[b].py, p->soa[b].pz, p->soa[b].g};
            for (int i = 0; i < 7; ++i)
                CUDA_TRY(cudaMemcpyAsync((unsigned char *)dst[i] + first * fs, src[i], cnt * fs,
                                         cudaMemcpyDeviceToHost, p->d2h), "D2H");
        } else {
            CUDA_TRY(cudaMemcpyAsync((unsigned char *)e->aos + first * rb, p->aos[b], cnt * rb,
                                     cudaMemcpyDeviceToHost, p->d2h), "D2H");
        }
        CUDA_TRY(cudaEventRecord(p->freed[b], p->d2h), "cudaEventRecord");
    }
    if (d_diag) CUDA_TRY(launch_diag_finalize(p->chunk_diag, n_chunks, d_diag, st), "diag finalize");
    // the caller's stream completes only after every chunk is back on the host
    for (int b = 0; b < HostPipeline::kBuffers && b < n_chunks; ++b)
        CUDA_TRY(cudaStreamWaitEvent(st, p->freed[b], 0), "cudaStreamWaitEvent");
    return BORIS_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// ABI
// ---------------------------------------------------------------------------
extern "C" {

int32_t boris_abi_version(void) { return LIBBORIS_ABI_VERSION; }

const char *boris_status_string(boris_status s) {
    switch (s) {
    case BORIS_OK: return "BORIS_OK";
    case BORIS_E_INVALID_ARG: return "BORIS_E_INVALID_ARG";
    case BORIS_E_OUT_OF_MEMORY: return "BORIS_E_OUT_OF_MEMORY";
    case BORIS_E_CUDA: return "BORIS_E_CUDA";
    case BORIS_E_TYPE_OUT_OF_RANGE: return "BORIS_E_TYPE_OUT_OF_RANGE";
    case BORIS_E_MISMATCH: return "BORIS_E_MISMATCH";
    case BORIS_E_UNSUPPORTED: return "BORIS_E_UNSUPPORTED";
    case BORIS_E_NO_DEVICE: return "BORIS_E_NO_DEVICE";
    default: return "BORIS_E_UNKNOWN";
    }
}

const char *boris_last_error(void) { return g_last_error.c_str(); }

boris_status boris_set_option(int32_t option, int64_t value) {
    switch (option) {
    case BORIS_OPT_FUSED_GENERIC:
        if (value != 0 && value != 1)
            return fail(BORIS_E_INVALID_ARG, "BORIS_OPT_FUSED_GENERIC must be 0 or 1");
        g_opt_fused_generic.store(value);
        return BORIS_OK;
    case BORIS_OPT_HOST_CHUNK:
        if (value < 1024 || value > BORIS_MAX_PARTICLES)
            return fail(BORIS_E_INVALID_ARG, "BORIS_OPT_HOST_CHUNK = %lld outside [1024, 2^40]",
                        (long long)value);
        g_opt_host_chunk.store(value);
        return BORIS_OK;
    case BORIS_OPT_MD_ORDER:
        if (value != 0 && value != 1)
            return fail(BORIS_E_INVALID_ARG, "BORIS_OPT_MD_ORDER must be 0 or 1");
        g_opt_md_order.store(value);
        return BORIS_OK;
    default:
        return fail(BORIS_E_INVALID_ARG, "unknown option %d", option);
    }
}

boris_status boris_get_option(int32_t option, int64_t *value) {
    if (!value) return fail(BORIS_E_INVALID_ARG, "value is NULL");
    switch (option) {
    case BORIS_OPT_FUSED_GENERIC: *value = g_opt_fused_generic.load(); return BORIS_OK;
    case BORIS_OPT_HOST_CHUNK: *value = g_opt_host_chunk.load(); return BORIS_OK;
    case BORIS_OPT_MD_ORDER: *value = g_opt_md_order.load(); return BORIS_OK;
    default: return fail(BORIS_E_INVALID_ARG, "unknown option %d", option);
    }
}

boris_status boris_ensemble_create(int32_t device, boris_layout layout, boris_precision precision,
                                   int64_t n, const boris_particle_type *types, int32_t n_types,
                                   double light_velocity, boris_ensemble **out) {
    if (!out) return fail(BORIS_E_INVALID_ARG, "out is NULL");
    if (layout != BORIS_LAYOUT_AOS && layout != BORIS_LAYOUT_SOA)
        return fail(BORIS_E_INVALID_ARG, "bad layout %d", layout);
    if (precision != BORIS_FP32 && precision != BORIS_FP64)
        return fail(BORIS_E_INVALID_ARG, "bad precision %d", precision);
    if (n < 0 || n > BORIS_MAX_PARTICLES)
        return fail(BORIS_E_INVALID_ARG, "n = %lld outside [0, 2^40]", (long long)n);
    boris_status s = check_types_table(types, n_types, light_velocity);
    if (s != BORIS_OK) return s;
    if ((s = check_device(device)) != BORIS_OK) return s;
    DeviceGuard g(device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    boris_ensemble *e = new_ensemble(device, BORIS_MEMORY_DEVICE, layout, precision, n, types,
                                     n_types, light_velocity);
    e->owned = true;
    const size_t fs = fp_size(precision);
    const int64_t npad = (n + 7) / 8 * 8;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    size_t bytes = layout == BORIS_LAYOUT_SOA ? 8 * al(npad * fs) + al(npad * 2)
                                              : al(npad * record_bytes(precision));
    if (bytes == 0) bytes = 256;
    cudaError_t err = cudaMalloc(&e->block, bytes);
    if (err != cudaSuccess) {
        free_ensemble(e);
        return cuda_fail(err, "cudaMalloc(ensemble)");
    }
    cudaMemset(e->block, 0, bytes);
    unsigned char *q = (unsigned char *)e->block;
    if (layout == BORIS_LAYOUT_SOA) {
        void **slots[8] = {&e->soa.x, &e->soa.y, &e->soa.z, &e->soa.px,
                           &e->soa.py, &e->soa.pz, &e->soa.w, &e->soa.g};
        for (int i = 0; i < 8; ++i) {
            *slots[i] = q;
            q += al(npad * fs);
        }
        e->soa.type = n_types > 1 ? (int16_t *)q : nullptr;
    } else {
        e->aos = q;
    }
    if ((s = alloc_scratch(e)) != BORIS_OK) {
        free_ensemble(e);
        return s;
    }
    err = launch_fill_defaults(e->view(), 0);
    if (err == cudaSuccess) err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
        free_ensemble(e);
        return cuda_fail(err, "ensemble init");
    }
    *out = e;
    return ok();
}

boris_status boris_ensemble_wrap_soa(int32_t device, int32_t memory, boris_precision precision,
                                     int64_t n, void *x, void *y, void *z, void *px, void *py,
                                     void *pz, void *weight, void *gamma, int16_t *type,
                                     const boris_particle_type *types, int32_t n_types,
                                     double light_velocity, boris_ensemble **out) {
    if (!out) return fail(BORIS_E_INVALID_ARG, "out is NULL");
    if (precision != BORIS_FP32 && precision != BORIS_FP64)
        return fail(BORIS_E_INVALID_ARG, "bad precision %d", precision);
    if (memory != BORIS_MEMORY_DEVICE && memory != BORIS_MEMORY_HOST)
        return fail(BORIS_E_INVALID_ARG, "bad memory kind %d", memory);
    if (n < 0 || n > BORIS_MAX_PARTICLES)
        return fail(BORIS_E_INVALID_ARG, "n = %lld outside [0, 2^40]", (long long)n);
    if (n > 0 && (!x || !y || !z || !px || !py || !pz || !gamma))
        return fail(BORIS_E_INVALID_ARG, "x, y, z, px, py, pz and gamma must be non-NULL");
    boris_status s = check_types_table(types, n_types, light_velocity);
    if (s != BORIS_OK) return s;
    if (n_types > 1 && n > 0 && !type)
        return fail(BORIS_E_INVALID_ARG, "type array required when n_types > 1");
    if ((s = check_device(device)) != BORIS_OK) return s;
    DeviceGuard g(device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    boris_ensemble *e = new_ensemble(device, memory, BORIS_LAYOUT_SOA, precision, n, types,
                                     n_types, light_velocity);
    e->soa = {x, y, z, px, py, pz, weight, gamma, n_types > 1 ? type : nullptr};
    if ((s = alloc_scratch(e)) != BORIS_OK) {
        free_ensemble(e);
        return s;
    }
    s = memory == BORIS_MEMORY_DEVICE ? validate_types_device(e, 0) : validate_types_host(e);
    if (s != BORIS_OK) {
        free_ensemble(e);
        return s;
    }
    *out = e;
    return ok();
}

boris_status boris_ensemble_wrap_aos(int32_t device, int32_t memory, boris_precision precision,
                                     int64_t n, void *records, const boris_particle_type *types,
                                     int32_t n_types, double light_velocity,
                                     boris_ensemble **out) {
    if (!out) return fail(BORIS_E_INVALID_ARG, "out is NULL");
    if (precision != BORIS_FP32 && precision != BORIS_FP64)
        return fail(BORIS_E_INVALID_ARG, "bad precision %d", precision);
    if (memory != BORIS_MEMORY_DEVICE && memory != BORIS_MEMORY_HOST)
        return fail(BORIS_E_INVALID_ARG, "bad memory kind %d", memory);
    if (n < 0 || n > BORIS_MAX_PARTICLES)
        return fail(BORIS_E_INVALID_ARG, "n = %lld outside [0, 2^40]", (long long)n);
    if (n > 0 && !records) return fail(BORIS_E_INVALID_ARG, "records is NULL");
    if (((uintptr_t)records & 15u) != 0)
        return fail(BORIS_E_INVALID_ARG, "AoS records must be 16 B aligned");
    boris_status s = check_types_table(types, n_types, light_velocity);
    if (s != BORIS_OK) return s;
    if ((s = check_device(device)) != BORIS_OK) return s;
    DeviceGuard g(device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    boris_ensemble *e = new_ensemble(device, memory, BORIS_LAYOUT_AOS, precision, n, types,
                                     n_types, light_velocity);
    e->aos = records;
    if ((s = alloc_scratch(e)) != BORIS_OK) {
        free_ensemble(e);
        return s;
    }
    s = memory == BORIS_MEMORY_DEVICE ? validate_types_device(e, 0) : validate_types_host(e);
    if (s != BORIS_OK) {
        free_ensemble(e);
        return s;
    }
    *out = e;
    return ok();
}

boris_status boris_ensemble_destroy(boris_ensemble *e) {
    if (!e) return ok();
    DeviceGuard g(e->device);
    free_ensemble(e);
    return ok();
}

boris_status boris_ensemble_validate_types(boris_ensemble *e, void *stream) {
    if (!e) return fail(BORIS_E_INVALID_ARG, "ensemble is NULL");
    if (e->memory == BORIS_MEMORY_HOST) {
        boris_status s = validate_types_host(e);
        return s == BORIS_OK ? ok() : s;
    }
    DeviceGuard g(e->device);
    boris_status s = validate_types_device(e, (cudaStream_t)stream);
    return s == BORIS_OK ? ok() : s;
}

boris_status boris_ensemble_get_info(const boris_ensemble *e, boris_layout *layout,
                                     boris_precision *precision, int64_t *n, int32_t *n_types,
                                     int32_t *device, int32_t *memory) {
    if (!e) return fail(BORIS_E_INVALID_ARG, "ensemble is NULL");
    if (layout) *layout = e->layout;
    if (precision) *precision = e->precision;
    if (n) *n = e->n;
    if (n_types) *n_types = e->n_types;
    if (device) *device = e->device;
    if (memory) *memory = e->memory;
    return ok();
}

boris_status boris_ensemble_get_time(const boris_ensemble *e, double *t) {
    if (!e || !t) return fail(BORIS_E_INVALID_ARG, "NULL argument");
    *t = e->time;
    return ok();
}

boris_status boris_ensemble_set_time(boris_ensemble *e, double t) {
    if (!e) return fail(BORIS_E_INVALID_ARG, "ensemble is NULL");
    if (!std::isfinite(t)) return fail(BORIS_E_INVALID_ARG, "time must be finite");
    e->time = t;
    return ok();
}

}  // extern "C"

// Host-memory ensembles: canonical <-> layout conversion on the host side of the
// boundary is data movement only (no push arithmetic).
namespace {
template <typename FP>
void host_store(boris_ensemble *e, int64_t i, const double *pos, const double *mom,
                const double *w, const int16_t *type, double g) {
    if (e->layout == BORIS_LAYOUT_SOA) {
        ((FP *)e->soa.x)[i] = (FP)pos[0];
        ((FP *)e->soa.y)[i] = (FP)pos[1];
        ((FP *)e->soa.z)[i] = (FP)pos[2];
        ((FP *)e->soa.px)[i] = (FP)mom[0];
        ((FP *)e->soa.py)[i] = (FP)mom[1];
        ((FP *)e->soa.pz)[i] = (FP)mom[2];
        ((FP *)e->soa.g)[i] = (FP)g;
        if (w && e->soa.w) ((FP *)e->soa.w)[i] = (FP)*w;
        if (type && e->soa.type) e->soa.type[i] = *type;
    } else {
        unsigned char *r = (unsigned char *)e->aos + i * record_bytes(e->precision);
        FP v[8];
        memcpy(v, r, sizeof v);
        for (int k = 0; k < 3; ++k) {
            v[k] = (FP)pos[k];
            v[3 + k] = (FP)mom[k];
        }
        if (w) v[6] = (FP)*w;
        v[7] = (FP)g;
        memcpy(r, v, sizeof v);
        if (type) memcpy(r + 8 * sizeof(FP), type, 2);
    }
}
template <typename FP>
void host_load(const boris_ensemble *e, int64_t i, double *pos, double *mom, double *w,
               double *g, int16_t *type) {
    if (e->layout == BORIS_LAYOUT_SOA) {
        if (pos) {
            pos[0] = ((const FP *)e->soa.x)[i];
            pos[1] = ((const FP *)e->soa.y)[i];
            pos[2] = ((const FP *)e->soa.z)[i];
        }
        if (mom) {
            mom[0] = ((const FP *)e->soa.px)[i];
            mom[1] = ((const FP *)e->soa.py)[i];
            mom[2] = ((const FP *)e->soa.pz)[i];
        }
        if (w) *w = e->soa.w ? (double)((const FP *)e->soa.w)[i] : 1.0;
        if (g) *g = ((const FP *)e->soa.g)[i];
        if (type) *type = e->soa.type ? e->soa.type[i] : 0;
    } else {
        const unsigned char *r = (const unsigned char *)e->aos + i * record_bytes(e->precision);
        FP v[8];
        memcpy(v, r, sizeof v);
        if (pos) for (int k = 0; k < 3; ++k) pos[k] = v[k];
        if (mom) for (int k = 0; k < 3; ++k) mom[k] = v[3 + k];
        if (w) *w = v[6];
        if (g) *g = v[7];
        if (type) memcpy(type, r + 8 * sizeof(FP), 2);
    }
}
}  // namespace

extern "C" {

boris_status boris_ensemble_upload(boris_ensemble *e, int64_t first, int64_t count,
                                   const double *pos3, const double *mom3, const double *weight,
                                   const int16_t *type, const double *gamma, void *stream) {
    if (!e) return fail(BORIS_E_INVALID_ARG, "ensemble is NULL");
    if (first < 0 || count < 0 || first + count > e->n)
        return fail(BORIS_E_INVALID_ARG, "range [%lld, %lld) outside [0, %lld)", (long long)first,
                    (long long)(first + count), (long long)e->n);
    if (count == 0) return ok();
    if (!pos3 || !mom3) return fail(BORIS_E_INVALID_ARG, "pos3 and mom3 are required");
    if (type) {
        if (e->layout == BORIS_LAYOUT_SOA && !e->soa.type && e->n_types == 1) {
            for (int64_t j = 0; j < count; ++j)
                if (type[j] != 0)
                    return fail(BORIS_E_TYPE_OUT_OF_RANGE, "type %d with n_types == 1", type[j]);
            type = nullptr;
        } else {
            for (int64_t j = 0; j < count; ++j)
                if (type[j] < 0 || type[j] >= e->n_types)
                    return fail(BORIS_E_TYPE_OUT_OF_RANGE, "particle %lld: type %d outside [0, %d)",
                                (long long)(first + j), type[j], e->n_types);
        }
    }
    for (int64_t j = 0; j < count; ++j)
        if (!finite3(pos3 + 3 * j) || !finite3(mom3 + 3 * j))
            return fail(BORIS_E_INVALID_ARG, "non-finite position or momentum at %lld",
                        (long long)(first + j));
    if (e->memory == BORIS_MEMORY_HOST) {
        for (int64_t j = 0; j < count; ++j) {
            const int64_t i = first + j;
            int16_t ty = 0;
            if (type) ty = type[j];
            else {
                if (e->precision == BORIS_FP32) host_load<float>(e, i, nullptr, nullptr, nullptr, nullptr, &ty);
                else host_load<double>(e, i, nullptr, nullptr, nullptr, nullptr, &ty);
            }
            const double *p = mom3 + 3 * j;
            const double mc = e->types[ty].mass * e->c;
            const double g = gamma ? gamma[j]
                                   : std::sqrt(1.0 + (p[0] * p[0] + p[1] * p[1] + p[2] * p[2]) / (mc * mc));
            if (e->precision == BORIS_FP32)
                host_store<float>(e, i, pos3 + 3 * j, p, weight ? weight + j : nullptr,
                                  type ? type + j : nullptr, g);
            else
                host_store<double>(e, i, pos3 + 3 * j, p, weight ? weight + j : nullptr,
                                   type ? type + j : nullptr, g);
        }
        return ok();
    }
    DeviceGuard g(e->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t c = (size_t)count;
    const size_t bytes = c * 8 * 8 + c * 2 + 64 * 8 + 256;
    unsigned char *d = nullptr;
    CUDA_TRY(scratch_alloc((void **)&d, bytes, st), "scratch_alloc(upload staging)");
    double *d_pos = (double *)d, *d_mom = d_pos + 3 * c, *d_w = d_mom + 3 * c, *d_g = d_w + c;
    double *d_inv = d_g + c;
    int16_t *d_type = (int16_t *)(d_inv + 64);
    double inv_mc2[64] = {};
    for (int i = 0; i < e->n_types; ++i) {
        const double mc = e->types[i].mass * e->c;
        inv_mc2[i] = 1.0 / (mc * mc);
    }
    cudaError_t err = cudaMemcpyAsync(d_pos, pos3, 3 * c * 8, cudaMemcpyHostToDevice, st);
    if (err == cudaSuccess) err = cudaMemcpyAsync(d_mom, mom3, 3 * c * 8, cudaMemcpyHostToDevice, st);
    if (err == cudaSuccess && weight) err = cudaMemcpyAsync(d_w, weight, c * 8, cudaMemcpyHostToDevice, st);
    if (err == cudaSuccess && gamma) err = cudaMemcpyAsync(d_g, gamma, c * 8, cudaMemcpyHostToDevice, st);
    if (err == cudaSuccess && type) err = cudaMemcpyAsync(d_type, type, c * 2, cudaMemcpyHostToDevice, st);
    if (err == cudaSuccess) err = cudaMemcpyAsync(d_inv, inv_mc2, sizeof inv_mc2, cudaMemcpyHostToDevice, st);
    if (err == cudaSuccess)
        err = launch_from_canonical(e->view(), first, count, d_pos, d_mom, d_w, d_type,
                                    gamma ? d_g : nullptr, d_inv, e->n_types, weight != nullptr,
                                    type != nullptr, st);
    scratch_free(d, st);
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) return cuda_fail(err, "boris_ensemble_upload");
    return ok();
}

boris_status boris_ensemble_download(const boris_ensemble *e, int64_t first, int64_t count,
                                     double *pos3, double *mom3, double *weight, double *gamma,
                                     int16_t *type, void *stream) {
    if (!e) return fail(BORIS_E_INVALID_ARG, "ensemble is NULL");
    if (first < 0 || count < 0 || first + count > e->n)
        return fail(BORIS_E_INVALID_ARG, "range outside the ensemble");
    if (count == 0) return ok();
    if (e->memory == BORIS_MEMORY_HOST) {
        if (e->pipe) {  // pushes run asynchronously on the caller's stream
            DeviceGuard g(e->device);
            cudaStreamSynchronize((cudaStream_t)stream);
        }
        for (int64_t j = 0; j < count; ++j) {
            if (e->precision == BORIS_FP32)
                host_load<float>(e, first + j, pos3 ? pos3 + 3 * j : nullptr,
                                 mom3 ? mom3 + 3 * j : nullptr, weight ? weight + j : nullptr,
                                 gamma ? gamma + j : nullptr, type ? type + j : nullptr);
            else
                host_load<double>(e, first + j, pos3 ? pos3 + 3 * j : nullptr,
                                  mom3 ? mom3 + 3 * j : nullptr, weight ? weight + j : nullptr,
                                  gamma ? gamma + j : nullptr, type ? type + j : nullptr);
        }
        return ok();
    }
    DeviceGuard g(e->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t c = (size_t)count;
    unsigned char *d = nullptr;
    CUDA_TRY(scratch_alloc((void **)&d, c * 8 * 8 + c * 2 + 256, st), "scratch_alloc(download staging)");
    double *d_pos = (double *)d, *d_mom = d_pos + 3 * c, *d_w = d_mom + 3 * c, *d_g = d_w + c;
    int16_t *d_type = (int16_t *)(d_g + c);
    cudaError_t err = launch_to_canonical(e->view(), first, count, d_pos, d_mom, d_w, d_g, d_type, st);
    if (err == cudaSuccess && pos3) err = cudaMemcpyAsync(pos3, d_pos, 3 * c * 8, cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess && mom3) err = cudaMemcpyAsync(mom3, d_mom, 3 * c * 8, cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess && weight) err = cudaMemcpyAsync(weight, d_w, c * 8, cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess && gamma) err = cudaMemcpyAsync(gamma, d_g, c * 8, cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess && type) err = cudaMemcpyAsync(type, d_type, c * 2, cudaMemcpyDeviceToHost, st);
    scratch_free(d, st);
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) return cuda_fail(err, "boris_ensemble_download");
    return ok();
}

// ---------------------------------------------------------------------------
// Fields
// ---------------------------------------------------------------------------
boris_status boris_field_create_arrays_soa(const boris_ensemble *like, const void *Ex,
                                           const void *Ey, const void *Ez, const void *Bx,
                                           const void *By, const void *Bz, boris_field **out) {
    if (!like || !out) return fail(BORIS_E_INVALID_ARG, "NULL argument");
    if (like->layout != BORIS_LAYOUT_SOA)
        return fail(BORIS_E_MISMATCH, "SoA field arrays need an SoA ensemble");
    if (like->n > 0 && (!Ex || !Ey || !Ez || !Bx || !By || !Bz))
        return fail(BORIS_E_INVALID_ARG, "field arrays must be non-NULL");
    boris_field *f = new boris_field();
    f->kind = FK_ARRAYS;
    f->layout = BORIS_LAYOUT_SOA;
    f->precision = like->precision;
    f->device = like->device;
    f->memory = like->memory;
    f->n = like->n;
    f->soa = {Ex, Ey, Ez, Bx, By, Bz};
    *out = f;
    return ok();
}

boris_status boris_field_create_arrays_aos(const boris_ensemble *like, const void *records,
                                           boris_field **out) {
    if (!like || !out) return fail(BORIS_E_INVALID_ARG, "NULL argument");
    if (like->layout != BORIS_LAYOUT_AOS)
        return fail(BORIS_E_MISMATCH, "AoS field records need an AoS ensemble");
    if (like->n > 0 && !records) return fail(BORIS_E_INVALID_ARG, "records is NULL");
    if (((uintptr_t)records & 15u) != 0)
        return fail(BORIS_E_INVALID_ARG, "field records must be 16 B aligned");
    boris_field *f = new boris_field();
    f->kind = FK_ARRAYS;
    f->layout = BORIS_LAYOUT_AOS;
    f->precision = like->precision;
    f->device = like->device;
    f->memory = like->memory;
    f->n = like->n;
    f->aos = records;
    *out = f;
    return ok();
}

boris_status boris_field_create_uniform(const double E[3], const double B[3], boris_field **out) {
    if (!E || !B || !out) return fail(BORIS_E_INVALID_ARG, "NULL argument");
    if (!finite3(E) || !finite3(B)) return fail(BORIS_E_INVALID_ARG, "non-finite field");
    boris_field *f = new boris_field();
    f->kind = FK_UNIFORM;
    for (int i = 0; i < 3; ++i) {
        f->E[i] = E[i];
        f->B[i] = B[i];
    }
    *out = f;
    return ok();
}

boris_status boris_field_create_plane_wave(double E0, const double k_hat[3], const double e_hat[3],
                                           double omega, double k, double phase0,
                                           boris_field **out) {
    if (!k_hat || !e_hat || !out) return fail(BORIS_E_INVALID_ARG, "NULL argument");
    if (!std::isfinite(E0) || !finite3(k_hat) || !finite3(e_hat) || !std::isfinite(omega) ||
        !std::isfinite(k) || !std::isfinite(phase0) || omega < 0 || k < 0)
        return fail(BORIS_E_INVALID_ARG, "plane wave parameters must be finite, omega, k >= 0");
    const double kk = k_hat[0] * k_hat[0] + k_hat[1] * k_hat[1] + k_hat[2] * k_hat[2];
    const double ee = e_hat[0] * e_hat[0] + e_hat[1] * e_hat[1] + e_hat[2] * e_hat[2];
    const double ke = k_hat[0] * e_hat[0] + k_hat[1] * e_hat[1] + k_hat[2] * e_hat[2];
    if (std::fabs(kk - 1) > 1e-12 || std::fabs(ee - 1) > 1e-12 || std::fabs(ke) > 1e-12)
        return fail(BORIS_E_INVALID_ARG, "k_hat, e_hat must be orthogonal unit vectors");
    boris_field *f = new boris_field();
    f->kind = FK_PLANE_WAVE;
    f->E0 = E0;
    for (int i = 0; i < 3; ++i) {
        f->k_hat[i] = k_hat[i];
        f->e_hat[i] = e_hat[i];
    }
    f->omega = omega;
    f->k = k;
    f->phase0 = phase0;
    *out = f;
    return ok();
}

boris_status boris_field_create_mdipole(double A0, double omega0, double k, boris_field **out) {
    if (!out) return fail(BORIS_E_INVALID_ARG, "out is NULL");
    if (!std::isfinite(A0) || !std::isfinite(omega0) || !std::isfinite(k) || !(k > 0))
        return fail(BORIS_E_INVALID_ARG, "m-dipole parameters must be finite, k > 0");
    boris_field *f = new boris_field();
    f->kind = FK_MDIPOLE;
    f->A0 = A0;
    f->omega0 = omega0;
    f->kd = k;
    *out = f;
    return ok();
}

boris_status boris_field_destroy(boris_field *f) {
    if (f && f->nodes) {
        DeviceGuard g(f->device);
        cudaFree(f->nodes);
    }
    delete f;
    return ok();
}

boris_status boris_field_create_grid(int32_t device, boris_precision precision, int32_t nx,
                                     int32_t ny, int32_t nz, const double origin[3],
                                     const double spacing[3], const void *Ex, const void *Ey,
                                     const void *Ez, const void *Bx, const void *By,
                                     const void *Bz, boris_field **out) {
    if (!out || !origin || !spacing) return fail(BORIS_E_INVALID_ARG, "NULL argument");
    if (precision != BORIS_FP32 && precision != BORIS_FP64)
        return fail(BORIS_E_INVALID_ARG, "bad precision %d", precision);
    if (nx < 1 || ny < 1 || nz < 1)
        return fail(BORIS_E_INVALID_ARG, "grid dimensions must be >= 1");
    const int64_t ncell = (int64_t)nx * ny * nz;
    if (ncell > (int64_t)1 << 31) return fail(BORIS_E_INVALID_ARG, "grid larger than 2^31 nodes");
    if (!finite3(origin) || !finite3(spacing) || !(spacing[0] > 0) || !(spacing[1] > 0) ||
        !(spacing[2] > 0))
        return fail(BORIS_E_INVALID_ARG, "origin must be finite and spacing > 0");
    if (!Ex || !Ey || !Ez || !Bx || !By || !Bz)
        return fail(BORIS_E_INVALID_ARG, "grid component arrays must be non-NULL");
    boris_status s = check_device(device);
    if (s != BORIS_OK) return s;
    DeviceGuard g(device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    boris_field *f = new boris_field();
    f->kind = FK_GRID;
    f->precision = precision;
    f->device = device;
    f->gn[0] = nx;
    f->gn[1] = ny;
    f->gn[2] = nz;
    for (int d = 0; d < 3; ++d) {
        f->org[d] = origin[d];
        f->h[d] = spacing[d];
    }
    const size_t rec_fp = precision == BORIS_FP32 ? kGridStride<float> : kGridStride<double>;
    cudaError_t err = cudaMalloc(&f->nodes, (size_t)ncell * rec_fp * fp_size(precision));
    if (err != cudaSuccess) {
        delete f;
        return cuda_fail(err, "cudaMalloc(grid nodes)");
    }
    const void *comps[6] = {Ex, Ey, Ez, Bx, By, Bz};
    err = launch_grid_pack(precision, ncell, nx, comps, f->nodes, 0);
    if (err == cudaSuccess) err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
        cudaFree(f->nodes);
        delete f;
        return cuda_fail(err, "grid packing");
    }
    *out = f;
    return ok();
}

}  // extern "C"

template <typename FP>
static DepCoefs<FP> make_dep_coefs(const boris_ensemble *e, const boris_field *grid, double dt) {
    DepCoefs<FP> dc;
    memset(&dc, 0, sizeof dc);
    dc.n_types = e->n_types;
    dc.half_dt = (FP)(0.5 * dt);
    const double vol = grid->h[0] * grid->h[1] * grid->h[2];
    for (int i = 0; i < e->n_types; ++i) {
        const double q = e->types[i].charge, m = e->types[i].mass, mc = m * e->c;
        const double S = std::ldexp(1.0, -(int)std::lround(std::log2(mc)));
        dc.t[i].S = (FP)S;
        const double kappa = 1.0 / (S * mc);  // as make_coefs: the fused PIC step reuses
        dc.t[i].kappa2 = (FP)(kappa * kappa);  // the push's 1/gamma bitwise
        dc.t[i].inv_Sm = (FP)(1.0 / (S * m));
        dc.t[i].q_vol = (FP)(q / vol);
    }
    return dc;
}

template <typename FP>
static cudaError_t push_deposit_view(boris_ensemble *e, const boris_field *grid, double dt,
                                     void *Jx, void *Jy, void *Jz, DiagOut *dp, cudaStream_t st) {
    const GridArgs<FP> g = make_grid_args<FP>(grid);
    const DepCoefs<FP> dc = make_dep_coefs<FP>(e, grid, dt);
    const EnsView v = e->view();
    if (v.layout == BORIS_LAYOUT_SOA) {
        DepOut<FP> o;
        cudaError_t err = dep_scratch_begin<FP>(g, o, st);
        if (err != cudaSuccess) return err;
        err = launch_push_deposit_soa<FP>(v, g, make_coefs<FP>(e, dt), dc, o, e->multi(), dp,
                                          e->device, st);
        if (err == cudaSuccess) return dep_scratch_end<FP>(g, o, Jx, Jy, Jz, st);
        dep_scratch_free<FP>(o, st);
        if (err != cudaErrorNotSupported) return err;
    }
    // AoS or unaligned: the push, then the deposition (which zeroes J)
    cudaError_t err = push_view<FP>(e, v, grid, grid->soa, grid->aos, e->time, dt, 1,
                                    BORIS_PUSH_AUTO, dp, st);
    if (err != cudaSuccess) return err;
    return launch_deposit<FP>(v, g, dc, Jx, Jy, Jz, e->device, st);
}

extern "C" {

boris_status boris_deposit_current(const boris_ensemble *e, const boris_field *grid, double dt,
                                   void *Jx, void *Jy, void *Jz, void *stream) {
    if (!e || !grid || !Jx || !Jy || !Jz) return fail(BORIS_E_INVALID_ARG, "NULL argument");
    if (grid->kind != FK_GRID) return fail(BORIS_E_INVALID_ARG, "field is not a grid");
    if (!std::isfinite(dt)) return fail(BORIS_E_INVALID_ARG, "dt must be finite");
    if (grid->precision != e->precision || grid->device != e->device)
        return fail(BORIS_E_MISMATCH, "grid and ensemble differ in precision or device");
    if (e->memory != BORIS_MEMORY_DEVICE)
        return fail(BORIS_E_UNSUPPORTED, "deposition needs a device-resident ensemble");
    DeviceGuard g(e->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    cudaError_t err =
        e->precision == BORIS_FP32
            ? launch_deposit<float>(e->view(), make_grid_args<float>(grid),
                                    make_dep_coefs<float>(e, grid, dt), Jx, Jy, Jz, e->device,
                                    (cudaStream_t)stream)
            : launch_deposit<double>(e->view(), make_grid_args<double>(grid),
                                     make_dep_coefs<double>(e, grid, dt), Jx, Jy, Jz, e->device,
                                     (cudaStream_t)stream);
    if (err != cudaSuccess) return cuda_fail(err, "current deposition");
    return ok();
}

boris_status boris_push_deposit(boris_ensemble *e, const boris_field *grid, double dt, void *Jx,
                                void *Jy, void *Jz, double *d_diag, void *stream) {
    if (!e || !grid || !Jx || !Jy || !Jz) return fail(BORIS_E_INVALID_ARG, "NULL argument");
    if (grid->kind != FK_GRID) return fail(BORIS_E_INVALID_ARG, "field is not a grid");
    boris_status s = check_push_args(e, grid, dt, 1);
    if (s != BORIS_OK) return s;
    if (e->memory != BORIS_MEMORY_DEVICE)
        return fail(BORIS_E_UNSUPPORTED, "push + deposition needs a device-resident ensemble");
    DeviceGuard g(e->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    DiagOut diag = {e->partials, e->partials_cap, 0};
    DiagOut *dp = d_diag ? &diag : nullptr;
    cudaError_t err =
        e->precision == BORIS_FP32
            ? push_deposit_view<float>(e, grid, dt, Jx, Jy, Jz, dp, st)
            : push_deposit_view<double>(e, grid, dt, Jx, Jy, Jz, dp, st);
    if (err != cudaSuccess) return cuda_fail(err, "push + deposition launch");
    if (d_diag) {
        err = e->n == 0 ? cudaMemsetAsync(d_diag, 0, 2 * sizeof(double), st)
                        : launch_diag_finalize(diag.partials, diag.written, d_diag, st);
        if (err != cudaSuccess) return cuda_fail(err, "diag finalize");
    }
    e->time += dt;
    return ok();
}

boris_status boris_ensemble_sort_by_cell(boris_ensemble *e, const boris_field *grid,
                                         void *stream) {
    if (!e || !grid) return fail(BORIS_E_INVALID_ARG, "NULL argument");
    if (grid->kind != FK_GRID) return fail(BORIS_E_INVALID_ARG, "field is not a grid");
    if (grid->precision != e->precision || grid->device != e->device)
        return fail(BORIS_E_MISMATCH, "grid and ensemble differ in precision or device");
    if (e->memory != BORIS_MEMORY_DEVICE)
        return fail(BORIS_E_UNSUPPORTED, "sorting needs a device-resident ensemble");
    if (e->n >= ((int64_t)1 << 32)) return fail(BORIS_E_UNSUPPORTED, "n >= 2^32");
    DeviceGuard g(e->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    cudaError_t err = e->precision == BORIS_FP32
                          ? sort_by_cell<float>(e->view(), make_grid_args<float>(grid), e->device,
                                                (cudaStream_t)stream)
                          : sort_by_cell<double>(e->view(), make_grid_args<double>(grid),
                                                 e->device, (cudaStream_t)stream);
    if (err != cudaSuccess) return cuda_fail(err, "sort by cell");
    return ok();
}

boris_status boris_field_evaluate(const boris_field *analytic, const boris_ensemble *e, double t,
                                  const boris_field *out, void *stream) {
    if (!analytic || !e || !out) return fail(BORIS_E_INVALID_ARG, "NULL argument");
    if (analytic->kind == FK_ARRAYS)
        return fail(BORIS_E_INVALID_ARG, "the source field must be analytic or a grid");
    if (analytic->kind == FK_GRID &&
        (analytic->precision != e->precision || analytic->device != e->device))
        return fail(BORIS_E_MISMATCH, "grid and ensemble differ in precision or device");
    if (!std::isfinite(t)) return fail(BORIS_E_INVALID_ARG, "t must be finite");
    if (out->kind != FK_ARRAYS || out->layout != e->layout || out->precision != e->precision ||
        out->n != e->n || out->device != e->device || out->memory != e->memory)
        return fail(BORIS_E_MISMATCH, "output field arrays do not match the ensemble");
    if (e->memory != BORIS_MEMORY_DEVICE)
        return fail(BORIS_E_UNSUPPORTED, "field evaluation needs a device-resident ensemble");
    DeviceGuard g(e->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    cudaError_t err =
        e->precision == BORIS_FP32
            ? launch_field_evaluate<float>(e->view(), analytic->kind,
                                           make_analytic<float>(analytic, t, 0.0), out->soa,
                                           (void *)out->aos, e->device, (cudaStream_t)stream)
            : launch_field_evaluate<double>(e->view(), analytic->kind,
                                            make_analytic<double>(analytic, t, 0.0), out->soa,
                                            (void *)out->aos, e->device, (cudaStream_t)stream);
    if (err != cudaSuccess) return cuda_fail(err, "field evaluate launch");
    return ok();
}

// ---------------------------------------------------------------------------
// Push
// ---------------------------------------------------------------------------
static boris_status push_impl(boris_ensemble *e, const boris_field *f, double dt, int64_t n_steps,
                              uint32_t flags, double *d_diag, cudaStream_t st) {
    boris_status s = check_push_args(e, f, dt, n_steps);
    if (s != BORIS_OK) return s;
    if ((flags & ~(uint32_t)(BORIS_PUSH_STREAM_EACH_STEP | BORIS_PUSH_PUSHER_MASK)) ||
        (flags & BORIS_PUSH_PUSHER_MASK) == BORIS_PUSH_PUSHER_MASK)
        return fail(BORIS_E_INVALID_ARG, "unknown push flags 0x%x", flags);
    if (n_steps == 0 && !d_diag) return ok();
    DeviceGuard g(e->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    if (e->memory == BORIS_MEMORY_HOST) {
        if (n_steps == 0)
            return fail(BORIS_E_UNSUPPORTED, "host-resident diagnostics need n_steps >= 1");
        if (e->n == 0) {
            if (d_diag) CUDA_TRY(cudaMemsetAsync(d_diag, 0, 2 * sizeof(double), st), "cudaMemsetAsync");
            e->time += (double)n_steps * dt;
            return ok();
        }
        s = e->precision == BORIS_FP32 ? push_host<float>(e, f, dt, n_steps, flags, d_diag, st)
                                       : push_host<double>(e, f, dt, n_steps, flags, d_diag, st);
        if (s != BORIS_OK) return s;
        e->time += (double)n_steps * dt;
        return ok();
    }
    DiagOut diag = {e->partials, e->partials_cap, 0};
    DiagOut *dp = d_diag ? &diag : nullptr;
    cudaError_t err;
    const FieldSoaPtrs fs = f->soa;
    if (n_steps == 0) {
        err = e->precision == BORIS_FP32
                  ? launch_kinetic_energy<float>(e->view(), make_coefs<float>(e, dt), e->multi(), dp, e->device, st)
                  : launch_kinetic_energy<double>(e->view(), make_coefs<double>(e, dt), e->multi(), dp, e->device, st);
    } else {
        err = e->precision == BORIS_FP32
                  ? push_view<float>(e, e->view(), f, fs, f->aos, e->time, dt, n_steps, flags, dp, st)
                  : push_view<double>(e, e->view(), f, fs, f->aos, e->time, dt, n_steps, flags, dp, st);
    }
    if (err != cudaSuccess) return cuda_fail(err, "push kernel launch");
    if (d_diag) {
        if (e->n == 0) {
            err = cudaMemsetAsync(d_diag, 0, 2 * sizeof(double), st);
        } else {
            err = launch_diag_finalize(diag.partials, diag.written, d_diag, st);
        }
        if (err != cudaSuccess) return cuda_fail(err, "diag finalize");
    }
    e->time += (double)n_steps * dt;
    return ok();
}

boris_status boris_push(boris_ensemble *e, const boris_field *f, double dt, int64_t n_steps,
                        void *stream) {
    return push_impl(e, f, dt, n_steps, BORIS_PUSH_AUTO, nullptr, (cudaStream_t)stream);
}

boris_status boris_push_diag(boris_ensemble *e, const boris_field *f, double dt, int64_t n_steps,
                             double *d_diag, void *stream) {
    if (!d_diag) return fail(BORIS_E_INVALID_ARG, "d_diag is NULL");
    return push_impl(e, f, dt, n_steps, BORIS_PUSH_AUTO, d_diag, (cudaStream_t)stream);
}

boris_status boris_push_ex(boris_ensemble *e, const boris_field *f, double dt, int64_t n_steps,
                           uint32_t flags, double *d_diag, void *stream) {
    return push_impl(e, f, dt, n_steps, flags, d_diag, (cudaStream_t)stream);
}

boris_status boris_kinetic_energy(const boris_ensemble *e, double *d_diag, void *stream) {
    if (!e || !d_diag) return fail(BORIS_E_INVALID_ARG, "NULL argument");
    if (e->memory == BORIS_MEMORY_HOST)
        return fail(BORIS_E_UNSUPPORTED, "diagnostics need a device-resident ensemble");
    DeviceGuard g(e->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    if (e->n == 0) {
        CUDA_TRY(cudaMemsetAsync(d_diag, 0, 2 * sizeof(double), st), "cudaMemsetAsync");
        return ok();
    }
    DiagOut diag = {e->partials, e->partials_cap, 0};
    cudaError_t err = e->precision == BORIS_FP32
                          ? launch_kinetic_energy<float>(e->view(), make_coefs<float>(e, 0.0), e->multi(), &diag, e->device, st)
                          : launch_kinetic_energy<double>(e->view(), make_coefs<double>(e, 0.0), e->multi(), &diag, e->device, st);
    if (err == cudaSuccess) err = launch_diag_finalize(diag.partials, diag.written, d_diag, st);
    if (err != cudaSuccess) return cuda_fail(err, "kinetic energy launch");
    return ok();
}

}  // extern "C"
