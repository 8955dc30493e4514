// boris_device.cuh -- device-side building blocks of the B200 Boris pusher.
//
// The per-particle arithmetic is the paper's procedure (arXiv 2104.04579 §2,
// PAPER.md L175-186) in the normalised momentum u = p/(mc) ("u-form"), which is
// eq. 9, 12, 13, 10, 5, 7 multiplied through by 1/(mc):
//   u^-  = u + alpha E                       alpha = q dt/(2 m c)      (eq. 9)
//   g_n  = sqrt(1 + |u^-|^2)                                            (L162)
//   t    = alpha B / g_n,  s = 2 t/(1 + |t|^2)                          (eq. 13)
//   u'   = u^- + u^- x t,  u^+ = u^- + u' x s                            (eq. 12)
//   u    = u^+ + alpha E                                                 (eq. 10)
//   g    = sqrt(1 + |u|^2),  r += (c dt / g) u                           (eq. 5, 7)
// Storage keeps the paper's momentum p = m c u (L207-212).  The u-form keeps
// every intermediate O(1) so fp32 never under/overflows in CGS or SI units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace boris {

constexpr int kMaxTypes = 32;  // == BORIS_MAX_TYPES

// Per-type coefficients, computed in double on the host for each push and
// cast to FP.
template <typename FP>
struct TypeCoef {
    FP alpha;   // q dt / (2 m c)
    FP inv_mc;  // 1 / (m c)
    FP mc;      // m c
};

template <typename FP>
struct Coefs {
    FP cdt;       // c dt
    int n_types;  // table entries used
    TypeCoef<FP> t[kMaxTypes];
    double ke[kMaxTypes];  // m c^2 for the kinetic-energy diagnostic
};

// ---------------------------------------------------------------------------
// Correctly rounded elementary operations (IEEE round-to-nearest, reading c14).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float b_sqrt(float x) { return __fsqrt_rn(x); }
__device__ __forceinline__ double b_sqrt(double x) { return __dsqrt_rn(x); }
__device__ __forceinline__ float b_rcp(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double b_rcp(double x) { return __drcp_rn(x); }

// One Boris momentum update in u-form for one particle (steps a4-a9).
// Returns 1/gamma^{n+1/2}; writes gamma^{n+1/2} to `gamma`.
template <typename FP>
__device__ __forceinline__ FP boris_momentum(FP &ux, FP &uy, FP &uz, FP Ex, FP Ey, FP Ez, FP Bx,
                                             FP By, FP Bz, FP alpha, FP &gamma) {
    // a4: first electric half kick (eq. 9)
    const FP ex = alpha * Ex, ey = alpha * Ey, ez = alpha * Ez;
    ux += ex;
    uy += ey;
    uz += ez;
    // a5: gamma_n = gamma(u^-) (L162, reading c2)
    const FP gn = b_sqrt(FP(1) + (ux * ux + uy * uy + uz * uz));
    // a6: rotation vectors (eq. 13)
    const FP ta = alpha * b_rcp(gn);
    const FP tx = ta * Bx, ty = ta * By, tz = ta * Bz;
    const FP sf = FP(2) * b_rcp(FP(1) + (tx * tx + ty * ty + tz * tz));
    const FP sx = sf * tx, sy = sf * ty, sz = sf * tz;
    // a7: rotation (eq. 12): u' = u^- + u^- x t ; u^+ = u^- + u' x s
    const FP upx = ux + (uy * tz - uz * ty);
    const FP upy = uy + (uz * tx - ux * tz);
    const FP upz = uz + (ux * ty - uy * tx);
    ux += upy * sz - upz * sy;
    uy += upz * sx - upx * sz;
    uz += upx * sy - upy * sx;
    // a8: second electric half kick (eq. 10)
    ux += ex;
    uy += ey;
    uz += ez;
    // a9: gamma^{n+1/2} (eq. 5, reading c3)
    gamma = b_sqrt(FP(1) + (ux * ux + uy * uy + uz * uz));
    return b_rcp(gamma);
}

// One full Boris step of one particle on stored quantities (rows a1-a11):
// p -> u, boris_momentum, position update, u -> p.  Shared by every streaming
// path (SoA vector/scalar, AoS tiles) so they are bitwise identical.
template <typename FP>
__device__ __forceinline__ void push_one(FP &x, FP &y, FP &z, FP &px, FP &py, FP &pz, FP &g,
                                         FP Ex, FP Ey, FP Ez, FP Bx, FP By, FP Bz,
                                         const TypeCoef<FP> &tc, FP cdt, FP &ux, FP &uy,
                                         FP &uz) {
    ux = px * tc.inv_mc;
    uy = py * tc.inv_mc;
    uz = pz * tc.inv_mc;
    const FP inv_g = boris_momentum<FP>(ux, uy, uz, Ex, Ey, Ez, Bx, By, Bz, tc.alpha, g);
    // a10: r^{n+1} = r^n + (c dt / gamma) u^{n+1/2}   (eq. 7)
    const FP ct = cdt * inv_g;
    x += ct * ux;
    y += ct * uy;
    z += ct * uz;
    // a11: store p = m c u
    px = ux * tc.mc;
    py = uy * tc.mc;
    pz = uz * tc.mc;
}

// Kinetic energy of one macroparticle, w m c^2 |u|^2 / (gamma + 1) (= w (gamma-1) m c^2
// without cancellation, reading c17), accumulated in double.
template <typename FP>
__device__ __forceinline__ double kinetic_energy(FP ux, FP uy, FP uz, FP gamma, FP w,
                                                 double mc2) {
    const double dux = ux, duy = uy, duz = uz;
    const double u2 = dux * dux + duy * duy + duz * duz;
    return (double)w * mc2 * u2 / ((double)gamma + 1.0);
}

// ---------------------------------------------------------------------------
// Streaming global-memory access with cache hints.  State arrays are read once
// and written once per step by the same thread; field arrays are read-only.
// Nothing is reused within a step, so loads bypass L1 and stores are
// evict-first (st.global.cs).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float4 ld_state(const float *p) {
    float4 v;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_state(const double *p) {
    double2 v;
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ld_field(const float *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_field(const double *p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream(float *p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_stream(double *p, double2 v) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// Vector of the particles one thread owns: 4 floats or 2 doubles = 16 B.
template <typename FP>
struct Vec;
template <>
struct Vec<float> {
    static constexpr int N = 4;
    float v[4];
    __device__ __forceinline__ void load_state(const float *p) {
        float4 t = ld_state(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
    __device__ __forceinline__ void load_field(const float *p) {
        float4 t = ld_field(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
    __device__ __forceinline__ void store(float *p) const {
        st_stream(p, make_float4(v[0], v[1], v[2], v[3]));
    }
};
template <>
struct Vec<double> {
    static constexpr int N = 2;
    double v[2];
    __device__ __forceinline__ void load_state(const double *p) {
        double2 t = ld_state(p);
        v[0] = t.x; v[1] = t.y;
    }
    __device__ __forceinline__ void load_field(const double *p) {
        double2 t = ld_field(p);
        v[0] = t.x; v[1] = t.y;
    }
    __device__ __forceinline__ void store(double *p) const {
        st_stream(p, make_double2(v[0], v[1]));
    }
};

// N int16 type indices (8 B for 4 particles, 4 B for 2).
template <int N>
__device__ __forceinline__ void load_types(const int16_t *p, int (&out)[N]);
template <>
__device__ __forceinline__ void load_types<4>(const int16_t *p, int (&out)[4]) {
    unsigned short a, b, c, d;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u16 {%0,%1,%2,%3}, [%4];"
                 : "=h"(a), "=h"(b), "=h"(c), "=h"(d)
                 : "l"(p));
    out[0] = (int16_t)a; out[1] = (int16_t)b; out[2] = (int16_t)c; out[3] = (int16_t)d;
}
template <>
__device__ __forceinline__ void load_types<2>(const int16_t *p, int (&out)[2]) {
    unsigned short a, b;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u16 {%0,%1}, [%2];"
                 : "=h"(a), "=h"(b)
                 : "l"(p));
    out[0] = (int16_t)a; out[1] = (int16_t)b;
}

// ---------------------------------------------------------------------------
// Block reduction of the (KE, count) diagnostic into per-block partials.
// Fixed shuffle/shared-memory tree: deterministic for a fixed launch shape.
// ---------------------------------------------------------------------------
template <int kThreads>
__device__ __forceinline__ void block_diag_partial(double ke, double count, double *partials) {
    static_assert(kThreads % 32 == 0 && kThreads <= 1024, "block size");
    __shared__ double s_ke[kThreads / 32], s_cnt[kThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ke += __shfl_xor_sync(0xffffffffu, ke, o);
        count += __shfl_xor_sync(0xffffffffu, count, o);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        s_ke[warp] = ke;
        s_cnt[warp] = count;
    }
    __syncthreads();
    if (warp == 0) {
        ke = lane < kThreads / 32 ? s_ke[lane] : 0.0;
        count = lane < kThreads / 32 ? s_cnt[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ke += __shfl_xor_sync(0xffffffffu, ke, o);
            count += __shfl_xor_sync(0xffffffffu, count, o);
        }
        if (lane == 0) {
            partials[2 * blockIdx.x] = ke;
            partials[2 * blockIdx.x + 1] = count;
        }
    }
}

// Load the type table into shared memory (multi-type kernels).  Divergent
// indexing into the kernel-parameter bank serialises; shared memory does not.
template <typename FP>
__device__ __forceinline__ void load_type_table(const Coefs<FP> &co, TypeCoef<FP> *s_t,
                                                double *s_ke) {
    for (int i = threadIdx.x; i < co.n_types; i += blockDim.x) {
        s_t[i] = co.t[i];
        s_ke[i] = co.ke[i];
    }
    __syncthreads();
}

}  // namespace boris
