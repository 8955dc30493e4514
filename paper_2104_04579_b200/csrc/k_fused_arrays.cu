// k_fused_arrays.cu -- register-fused multi-step push for per-particle
// ("precalculated", reading c6) fields.
//
// The precalculated field of a particle is constant over steps (c6), so
// n_steps single-step pushes only re-read the same E, B from HBM n_steps times.
// This kernel reads r, p, E, B (and type, weight) once, runs n_steps Boris steps
// in registers with the state kept in FP (rounded exactly as the streaming kernel
// stores it), and writes r, p, gamma once: the result is bitwise identical to
// n_steps launches of k_stream_soa_vec / k_stream_aos (same push_one arithmetic),
// with HBM traffic divided by n_steps (ALU-bound instead of HBM-bound).
#include "boris_internal.h"

namespace boris {

template <typename FP, int LAYOUT, bool MULTI, bool DIAG, int PUSHER>
__global__ void __launch_bounds__(kFusedThreads)
    k_fused_arrays(EnsView e, FieldSoaPtrs f, const void *frec,
                   const __grid_constant__ KCoefs<FP, MULTI> co, int64_t n_steps,
                   double *partials) {
    __shared__ TypeCoef<FP> s_t[MULTI ? kMaxTypes : 1];
    if (MULTI) load_type_table(co, s_t);
    double ke = 0.0, cnt = 0.0;
    constexpr int RB = sizeof(FP) == 4 ? BORIS_AOS_RECORD_BYTES_FP32 : BORIS_AOS_RECORD_BYTES_FP64;
    const int64_t stride = (int64_t)gridDim.x * kFusedThreads;
    for (int64_t i = (int64_t)blockIdx.x * kFusedThreads + threadIdx.x; i < e.n; i += stride) {
        FP x, y, z, px, py, pz, w, Ex, Ey, Ez, Bx, By, Bz;
        int ty = 0;
        FP *rec = nullptr;
        if (LAYOUT == BORIS_LAYOUT_SOA) {
            x = ((const FP *)e.soa.x)[i];
            y = ((const FP *)e.soa.y)[i];
            z = ((const FP *)e.soa.z)[i];
            px = ((const FP *)e.soa.px)[i];
            py = ((const FP *)e.soa.py)[i];
            pz = ((const FP *)e.soa.pz)[i];
            w = (DIAG && e.soa.w) ? ((const FP *)e.soa.w)[i] : FP(1);
            if (MULTI) ty = e.soa.type[i];
            Ex = ((const FP *)f.Ex)[i];
            Ey = ((const FP *)f.Ey)[i];
            Ez = ((const FP *)f.Ez)[i];
            Bx = ((const FP *)f.Bx)[i];
            By = ((const FP *)f.By)[i];
            Bz = ((const FP *)f.Bz)[i];
        } else {
            rec = (FP *)((unsigned char *)e.aos + i * RB);
            x = rec[0]; y = rec[1]; z = rec[2];
            px = rec[3]; py = rec[4]; pz = rec[5];
            w = rec[6];
            if (MULTI) ty = *(const int16_t *)(rec + 8);
            const FP *fr = (const FP *)frec + 6 * i;
            Ex = fr[0]; Ey = fr[1]; Ez = fr[2];
            Bx = fr[3]; By = fr[4]; Bz = fr[5];
        }
        const TypeCoef<FP> tc = MULTI ? s_t[ty] : co.t[0];
        FP ux = FP(0), uy = FP(0), uz = FP(0), gam = FP(1);
        for (int64_t s = 0; s < n_steps; ++s)
            push_one<FP, PUSHER>(x, y, z, px, py, pz, gam, Ex, Ey, Ez, Bx, By, Bz, tc, ux, uy,
                                 uz);
        if (LAYOUT == BORIS_LAYOUT_SOA) {
            ((FP *)e.soa.x)[i] = x;
            ((FP *)e.soa.y)[i] = y;
            ((FP *)e.soa.z)[i] = z;
            ((FP *)e.soa.px)[i] = px;
            ((FP *)e.soa.py)[i] = py;
            ((FP *)e.soa.pz)[i] = pz;
            ((FP *)e.soa.g)[i] = gam;
        } else {
            rec[0] = x; rec[1] = y; rec[2] = z;
            rec[3] = px; rec[4] = py; rec[5] = pz;
            rec[7] = gam;
        }
        if (DIAG) {
            ke += (double)kinetic_energy<FP>(ux, uy, uz, gam, w, tc);
            cnt += 1.0;
        }
    }
    if (DIAG) block_diag_partial<kFusedThreads>(ke, cnt, partials);
}

template <typename FP, int LAYOUT, bool MULTI, bool DIAG, int PUSHER>
static cudaError_t dispatch_fa(const EnsView &e, const FieldSoaPtrs &f, const void *frec,
                               const Coefs<FP> &co, int64_t n_steps, DiagOut *diag, int device,
                               cudaStream_t st) {
    const int64_t blocks = (e.n + kFusedThreads - 1) / kFusedThreads;
    const auto kern = &k_fused_arrays<FP, LAYOUT, MULTI, DIAG, PUSHER>;
    int64_t grid = fused_grid((const void *)kern, blocks > 0 ? blocks : 1, device);
    if (DIAG && grid > diag->cap) grid = diag->cap;
    kern<<<(unsigned)grid, kFusedThreads, 0, st>>>(
        e, f, frec, kcoefs<MULTI>(co), n_steps, diag ? diag->partials : nullptr);
    if (diag) diag->written = DIAG ? grid : 0;
    return cudaGetLastError();
}

template <typename FP, int LAYOUT, int PUSHER>
static cudaError_t dispatch_fa_md(const EnsView &e, const FieldSoaPtrs &f, const void *frec,
                                  const Coefs<FP> &co, int64_t n_steps, bool multi,
                                  DiagOut *diag, int device, cudaStream_t st) {
    if (multi)
        return diag ? dispatch_fa<FP, LAYOUT, true, true, PUSHER>(e, f, frec, co, n_steps, diag,
                                                                   device, st)
                    : dispatch_fa<FP, LAYOUT, true, false, PUSHER>(e, f, frec, co, n_steps, diag,
                                                                    device, st);
    return diag ? dispatch_fa<FP, LAYOUT, false, true, PUSHER>(e, f, frec, co, n_steps, diag,
                                                                device, st)
                : dispatch_fa<FP, LAYOUT, false, false, PUSHER>(e, f, frec, co, n_steps, diag,
                                                                 device, st);
}

template <typename FP, int LAYOUT>
static cudaError_t dispatch_fa_layout(const EnsView &e, const FieldSoaPtrs &f, const void *frec,
                                      const Coefs<FP> &co, int64_t n_steps, bool multi,
                                      int pusher, DiagOut *diag, int device, cudaStream_t st) {
    switch (pusher) {
    case PUSHER_VAY:
        return dispatch_fa_md<FP, LAYOUT, PUSHER_VAY>(e, f, frec, co, n_steps, multi, diag,
                                                      device, st);
    case PUSHER_HIGUERA_CARY:
        return dispatch_fa_md<FP, LAYOUT, PUSHER_HIGUERA_CARY>(e, f, frec, co, n_steps, multi,
                                                               diag, device, st);
    default:
        return dispatch_fa_md<FP, LAYOUT, PUSHER_BORIS>(e, f, frec, co, n_steps, multi, diag,
                                                        device, st);
    }
}

template <typename FP>
cudaError_t launch_fused_arrays(const EnsView &e, const FieldSoaPtrs &f, const void *frec,
                                const Coefs<FP> &co, int64_t n_steps, bool multi, int pusher,
                                DiagOut *diag, int device, cudaStream_t st) {
    if (e.n == 0) {
        if (diag) diag->written = 0;
        return cudaSuccess;
    }
    if (e.layout == BORIS_LAYOUT_SOA)
        return dispatch_fa_layout<FP, BORIS_LAYOUT_SOA>(e, f, frec, co, n_steps, multi, pusher,
                                                        diag, device, st);
    return dispatch_fa_layout<FP, BORIS_LAYOUT_AOS>(e, f, frec, co, n_steps, multi, pusher, diag,
                                                    device, st);
}

template cudaError_t launch_fused_arrays<float>(const EnsView &, const FieldSoaPtrs &,
                                                const void *, const Coefs<float> &, int64_t, bool,
                                                int, DiagOut *, int, cudaStream_t);
template cudaError_t launch_fused_arrays<double>(const EnsView &, const FieldSoaPtrs &,
                                                 const void *, const Coefs<double> &, int64_t,
                                                 bool, int, DiagOut *, int, cudaStream_t);

}  // namespace boris
