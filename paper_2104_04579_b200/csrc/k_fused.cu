// k_fused.cu -- register-fused multi-step Boris push for analytic fields
// ("Analytical fields"; north_star "an analytic-field
// variant that fuses n_steps iterations in registers so HBM is touched once
// per launch"; SURVEY §8(a) row a12, Appendix A "Fused analytic kernel").
//
// One thread owns one particle for the whole launch: it reads r, p (and type,
// weight) once, runs n_steps Boris steps with the field evaluated at
// (r^n, t_n = t0 + n dt) in registers (reading c5), and writes r, p, gamma once.
// The kernel is ALU-bound (FP32 FMA pipe for fp32, FP64 pipe for fp64).
// fp32 kernels keep r in fp64 registers across steps (3 DADD per step on the
// otherwise idle FP64 pipe) and evaluate the plane-wave phase in fp64 with an
// exact 2-pi range reduction before the fp32 cosine (SURVEY §8(c) "GPU<->oracle,
// fp32": this quadruples the margin under the 1e-5 bar at C4).
#include <type_traits>

#include "boris_internal.h"

namespace boris {

namespace {

// 2 pi split for Cody-Waite range reduction in double.
constexpr double kTwoPiHi = 6.283185307179586;
constexpr double kTwoPiLo = 2.4492935982947064e-16;
constexpr double kInvTwoPi = 0.15915494309189535;

// cos(phi) for |phi| large: reduce in double, evaluate in FP.
__device__ __forceinline__ float cos_reduced(double phi, float) {
    const double q = rint(phi * kInvTwoPi);
    double r = fma(-q, kTwoPiHi, phi);
    r = fma(-q, kTwoPiLo, r);
    return cosf((float)r);
}
__device__ __forceinline__ double cos_reduced(double phi, double) { return cos(phi); }

// phi mod 2 pi in [-pi, pi] (Cody-Waite, exact for |phi| < 2^40).
__device__ __forceinline__ double reduce_2pi(double phi) {
    const double q = rint(phi * kInvTwoPi);
    return fma(-q, kTwoPiLo, fma(-q, kTwoPiHi, phi));
}

// cos of a phase within a few radians of [-pi, pi]: fp32 -> MUFU cos (abs error
// ~2^-21, below the fp32 rounding of the phase itself) unless BORIS_PRECISE_MATH.
__device__ __forceinline__ float cos_small(float x) {
#ifdef BORIS_PRECISE_MATH
    return cosf(x);
#else
    return __cosf(x);
#endif
}
__device__ __forceinline__ double cos_small(double x) { return cos(x); }

// m-dipole radial functions (eq. 15, readings c11, c13): g1 = f1/xi, g2 = f2/xi^2, f3.
// Taylor coefficients generated at compile time from their defining series:
//   j0 = sum (-1)^n xi^{2n}/(2n+1)!,  j1/xi = sum (-1)^n 2(n+1) xi^{2n}/(2n+3)!,
//   g2 = sum_{n>=1} (-1)^n [6(n+1)/(2n+3)! - 1/(2n+1)!] xi^{2n-2}.
// The Horner chains below take them as template constants (FFMA immediates in the
// fp32 SASS: no constant-bank loads, conversions or registers held for them).
constexpr double fact(int k) { return k <= 1 ? 1.0 : k * fact(k - 1); }
constexpr double md_sign(int n) { return (n % 2 == 0) ? 1.0 : -1.0; }
constexpr double md_j0c(int n) { return md_sign(n) / fact(2 * n + 1); }
constexpr double md_j1xc(int n) { return md_sign(n) * 2.0 * (n + 1) / fact(2 * n + 3); }
constexpr double md_g2c(int n) {  // used for n >= 1
    return md_sign(n) * (6.0 * (n + 1) / fact(2 * n + 3) - 1.0 / fact(2 * n + 1));
}
// sum_{n=N}^{T-1} c_n x2^{n-N} by Horner from the top term (WHICH: 0 j0, 1 j1/xi, 2 g2)
template <typename FP, int WHICH, int N, int T>
struct MdHorner {
    static __device__ __forceinline__ FP eval(FP x2) {
        constexpr FP c = FP(WHICH == 0 ? md_j0c(N) : WHICH == 1 ? md_j1xc(N) : md_g2c(N));
        if constexpr (N == T - 1)
            return c;
        else
            return MdHorner<FP, WHICH, N + 1, T>::eval(x2) * x2 + c;
    }
};

template <typename FP>
struct MdBranch;
template <>
struct MdBranch<double> {  // reading c13: fp64 xi* = 1, 9 terms
    static constexpr double xi_star = 1.0;
    static constexpr int terms = 9;
};
template <>
struct MdBranch<float> {  // reading c13: fp32 xi* = 1.5, 7 terms
    static constexpr float xi_star = 1.5f;
    static constexpr int terms = 7;
};

#ifdef BORIS_PRECISE_MATH
// R = |r| for the m-dipole with BORIS_PRECISE_MATH (correctly rounded square roots; the
// default math works with xi^2 and never forms R, md_radial_x2 below).
__device__ __forceinline__ float md_radius(float r2) { return __fsqrt_rn(r2); }
__device__ __forceinline__ double md_radius(double r2) { return __dsqrt_rn(r2); }
#endif

// Closed-form branch of the radial functions (eq. 15, reading c11) from s = sin xi,
// c = cos xi and i = 1/xi, factored so that each product is formed once:
//   P  = i (s i) - c i
//   g1 = f1/xi   = i^2 (s i - c)
//   g2 = f2/xi^2 = i^3 (3 P - s)
//   f3           = i (s - P)
// (f1 = s/xi^2 - c/xi, f2 = (3/xi^3 - 1/xi) s - 3c/xi^2, f3 = (1/xi - 1/xi^3) s + c/xi^2).
template <typename FP>
__device__ __forceinline__ void md_closed(FP sn, FP cs, FP ix, FP &g1, FP &g2, FP &f3) {
    const FP a = b_mul(sn, ix), b = b_mul(cs, ix), i2 = b_mul(ix, ix);
    const FP P = b_fma(ix, a, -b);
    g1 = b_mul(i2, b_add(a, -cs));
    g2 = b_mul(b_mul(i2, ix), b_fma(FP(3), P, -sn));
    f3 = b_mul(ix, b_add(sn, -P));
}

// Taylor branch (reading c13) from xi^2
template <typename FP>
__device__ __forceinline__ void md_taylor_series(FP x2, FP &g1, FP &g2, FP &f3) {
    constexpr int T = MdBranch<FP>::terms;
    const FP j0 = MdHorner<FP, 0, 0, T>::eval(x2);
    const FP j1x = MdHorner<FP, 1, 0, T>::eval(x2);
    g1 = j1x;
    g2 = MdHorner<FP, 2, 1, T>::eval(x2);
    f3 = j0 - j1x;
}

template <typename FP>
__device__ __forceinline__ void md_radial(FP xi, FP &g1, FP &g2, FP &f3) {
    if (xi < MdBranch<FP>::xi_star) {
        md_taylor_series<FP>(xi * xi, g1, g2, f3);
    } else {
        FP sn, cs, ix;
        if constexpr (sizeof(FP) == 4) {
            sincosf(xi, &sn, &cs);
            ix = 1.0f / xi;
        } else {
            sincos(xi, &sn, &cs);
            ix = __drcp_rn(xi);  // == 1.0 / xi (both correctly rounded), no division
        }
        md_closed<FP>(sn, cs, ix, g1, g2, f3);
    }
}

// The radial functions from xi^2 (fp32 / fp64 default math): the Taylor branch is a
// series in xi^2 (no square root), and the closed form takes 1/xi = rsqrt(xi^2) from
// one MUFU rsqrt and xi = xi^2 / xi; the branch test xi < xi* becomes xi^2 < xi*^2
// (reading c13).  fp32 sin and cos of xi straight from the MUFU (sin.approx /
// cos.approx: absolute error 2^-21.4 on [-pi, pi], growing with the 2^-23 relative
// rounding of the argument's revolutions beyond, ~2^-21 at the sphere's xi = 3.8);
// fp64 with the double rsqrt (1 ulp) and sincos.
template <typename FP>
__device__ __forceinline__ void md_radial_x2(FP x2, FP &g1, FP &g2, FP &f3) {
    if (x2 < MdBranch<FP>::xi_star * MdBranch<FP>::xi_star) {
        md_taylor_series<FP>(x2, g1, g2, f3);
    } else {
        FP sn, cs;
        const FP ix = b_rsqrt(x2), xi = b_mul(x2, ix);
        if constexpr (sizeof(FP) == 4)
            __sincosf(xi, &sn, &cs);
        else
            sincos(xi, &sn, &cs);
        md_closed<FP>(sn, cs, ix, g1, g2, f3);
    }
}

// The radial functions from r^2 = |r|^2 (field evaluation, the multi-type and
// alternative-pusher fused steps, the branch ordering k_md_order): xi^2 = k^2 r^2 as above;
// BORIS_PRECISE_MATH uses R = sqrt(r^2), xi = k R with correctly rounded square root
// and reciprocal.
template <typename FP>
__device__ __forceinline__ bool md_taylor(const AnalyticArgs<FP> &fa, FP r2) {
#ifndef BORIS_PRECISE_MATH
    return b_mul(fa.k2, r2) < MdBranch<FP>::xi_star * MdBranch<FP>::xi_star;
#else
    return b_mul(fa.k, md_radius(r2)) < MdBranch<FP>::xi_star;
#endif
}
template <typename FP>
__device__ __forceinline__ void md_radial_r2(const AnalyticArgs<FP> &fa, FP r2, FP &g1, FP &g2,
                                             FP &f3) {
#ifndef BORIS_PRECISE_MATH
    md_radial_x2<FP>(b_mul(fa.k2, r2), g1, g2, f3);
#else
    md_radial<FP>(b_mul(fa.k, md_radius(r2)), g1, g2, f3);
#endif
}

template <typename FP, int FIELD>
__device__ __forceinline__ void analytic_field(const AnalyticArgs<FP> &fa, double rx, double ry,
                                               double rz, int64_t n, FP &Ex, FP &Ey, FP &Ez,
                                               FP &Bx, FP &By, FP &Bz) {
    if constexpr (FIELD == FK_UNIFORM) {
        Ex = fa.E[0]; Ey = fa.E[1]; Ez = fa.E[2];
        Bx = fa.B[0]; By = fa.B[1]; Bz = fa.B[2];
    } else if constexpr (FIELD == FK_PLANE_WAVE) {
        // phi = k (k_hat . r) - omega t_n + phase0, t_n = t0 + n dt (reading c5)
        const double phi = fma(fa.kvec[0], rx, fma(fa.kvec[1], ry, fa.kvec[2] * rz)) +
                           (fa.ph0 - (double)n * fa.wdt);
        const FP c = cos_reduced(phi, FP(0));
        Ex = fa.cE[0] * c; Ey = fa.cE[1] * c; Ez = fa.cE[2] * c;
        Bx = fa.cB[0] * c; By = fa.cB[1] * c; Bz = fa.cB[2] * c;
    } else if constexpr (FIELD == FK_GRID) {
        grid_gather<FP>(fa.grid, (FP)rx, (FP)ry, (FP)rz, Ex, Ey, Ez, Bx, By, Bz);
    } else {  // FK_MDIPOLE, eq. 14 in readings c9, c10, c13
        // the fused step's arithmetic (k_fused below): radial functions from r^2, the
        // time amplitudes rounded as its per-block tables, the same product order
        const FP x = (FP)rx, y = (FP)ry, z = (FP)rz;
        FP g1, g2, f3;
        md_radial_r2<FP>(fa, b_norm2(x, y, z), g1, g2, f3);
        double sn, cs;
        sincos(fa.w0t0 + (double)n * fa.w0dt, &sn, &cs);  // t_n = t0 + n dt (c5)
        const FP ce = b_mul(b_mul(fa.A0k2, (FP)cs), g1);    // 2 A0 k cos(w t) f1/xi
        const FP sb = b_mul(fa.mA02, (FP)sn);               // -2 A0 sin(w t)
        const FP k2g2 = b_mul(fa.k2, g2);                   // f2/R^2
        Ex = -b_mul(ce, y);
        Ey = b_mul(ce, x);
        Ez = FP(0);
        const FP sk = b_mul(sb, k2g2);
        Bx = b_mul(b_mul(sk, x), z);
        By = b_mul(b_mul(sk, y), z);
        Bz = b_mul(sb, b_fma(k2g2, b_mul(z, z), f3));
    }
}

// Position accumulator: double for fp32 state (see header), FP otherwise.
template <typename FP, int LAYOUT>
struct Particle {
    static __device__ __forceinline__ void load(const EnsView &e, int64_t i, double &x, double &y,
                                                double &z, FP &px, FP &py, FP &pz, FP &w,
                                                int &ty) {
        if constexpr (LAYOUT == BORIS_LAYOUT_SOA) {
            x = ((const FP *)e.soa.x)[i];
            y = ((const FP *)e.soa.y)[i];
            z = ((const FP *)e.soa.z)[i];
            px = ((const FP *)e.soa.px)[i];
            py = ((const FP *)e.soa.py)[i];
            pz = ((const FP *)e.soa.pz)[i];
            w = e.soa.w ? ((const FP *)e.soa.w)[i] : FP(1);
            ty = e.soa.type ? e.soa.type[i] : 0;
        } else {
            constexpr int RB = sizeof(FP) == 4 ? 36 : 72;
            const unsigned char *rec = (const unsigned char *)e.aos + i * RB;
            const FP *r = (const FP *)rec;
            x = r[0]; y = r[1]; z = r[2];
            px = r[3]; py = r[4]; pz = r[5];
            w = r[6];
            ty = *(const int16_t *)(rec + 8 * sizeof(FP));
        }
    }
    static __device__ __forceinline__ void store(const EnsView &e, int64_t i, double x, double y,
                                                 double z, FP px, FP py, FP pz, FP g) {
        if constexpr (LAYOUT == BORIS_LAYOUT_SOA) {
            ((FP *)e.soa.x)[i] = (FP)x;
            ((FP *)e.soa.y)[i] = (FP)y;
            ((FP *)e.soa.z)[i] = (FP)z;
            ((FP *)e.soa.px)[i] = px;
            ((FP *)e.soa.py)[i] = py;
            ((FP *)e.soa.pz)[i] = pz;
            ((FP *)e.soa.g)[i] = g;
        } else {
            constexpr int RB = sizeof(FP) == 4 ? 36 : 72;
            FP *r = (FP *)((unsigned char *)e.aos + i * RB);
            r[0] = (FP)x; r[1] = (FP)y; r[2] = (FP)z;
            r[3] = px; r[4] = py; r[5] = pz;
            r[7] = g;
        }
    }
};

// m-dipole branch ordering.  Before the fused launch, k_md_order writes the particle
// indices into `order`: those whose xi = kR is below xi* at the launch's first step
// (Taylor branch, reading c13) from the front, the closed-form ones from the back (each
// warp reserves its runs with one atomic per branch).  The fused kernel then pushes
// order[32 r .. 32 r + 31] in warp-round r, so all warp-rounds but the one at the
// boundary run a single branch (with one particle per thread in storage order, a
// 0.6-lambda sphere puts a Taylor particle in ~87 % of warps, and a divergent warp
// executes both bodies), with no barrier and a work unit of one round.  Scheduling
// only: every particle's arithmetic is unchanged, so results are bitwise identical
// to the unordered kernel; particles keep their storage slots (c18).
template <typename FP, int LAYOUT>
__global__ void __launch_bounds__(256)
    k_md_order(EnsView e, const __grid_constant__ AnalyticArgs<FP> fa, int *order,
               unsigned long long *counts) {
    const int lane = threadIdx.x & 31;
    const unsigned below = (1u << lane) - 1u;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < e.n;
         i0 += stride) {  // warp-uniform
        const int64_t i = i0 + lane;
        bool taylor = false;
        if (i < e.n) {
            FP x, y, z;
            if constexpr (LAYOUT == BORIS_LAYOUT_SOA) {
                x = ((const FP *)e.soa.x)[i];
                y = ((const FP *)e.soa.y)[i];
                z = ((const FP *)e.soa.z)[i];
            } else {
                const FP *r = (const FP *)((const unsigned char *)e.aos +
                                           i * (sizeof(FP) == 4 ? 36 : 72));
                x = r[0]; y = r[1]; z = r[2];
            }
            taylor = md_taylor<FP>(fa, b_norm2(x, y, z));  // k_fused's x = (FP)xa + 0
        }
        const unsigned bt = __ballot_sync(0xffffffffu, i < e.n && taylor);
        const unsigned bc = __ballot_sync(0xffffffffu, i < e.n && !taylor);
        unsigned long long ft = 0, fc = 0;
        if (lane == 0) {
            if (bt) ft = atomicAdd(&counts[0], (unsigned long long)__popc(bt));
            if (bc) fc = atomicAdd(&counts[1], (unsigned long long)__popc(bc));
        }
        ft = __shfl_sync(0xffffffffu, ft, 0);
        fc = __shfl_sync(0xffffffffu, fc, 0);
        if (i < e.n) {
            if (taylor)
                order[ft + __popc(bt & below)] = (int)i;
            else
                order[e.n - 1 - (int64_t)(fc + __popc(bc & below))] = (int)i;
        }
    }
}

}  // namespace

// The fused step loop runs in windows of kFlush steps.  At each window start the
// position anchor r_a (fp64) absorbs the FP displacement accumulated in the
// window (fp32: position effectively kept in fp64, reading c-fp32r, without an
// fp64 op in the inner loop), and the plane-wave phase is re-anchored in fp64
// and reduced mod 2 pi; inside the window
//   phi_n = phi_a + kvec . (r - r_a) - (n - n_a) omega dt      (FP, |.| <~ pi + 0.5)
// which is phi = k (k_hat . r^n) - omega t_n + phase0 (reading c5) re-associated.
// Grid field in the fused kernel: keep the particle's cell records in registers
// across steps (grid_gather_cached); 0 gathers every step from L1/L2.
#ifndef BORIS_GRID_CACHE
#define BORIS_GRID_CACHE 1
#endif

// Window length: fp32 16 steps (8: C4 1.287 ps, 12: 1.217, 16: 1.181 per particle-step;
// parity after 100 steps 4.2e-6 -> 5.2e-6 of the 1e-5 bar, profiles/r01/exp_flush_window/),
// fp64 8 (16 spills in the alternative pushers and is slower).
#ifndef BORIS_FUSED_FLUSH32
#define BORIS_FUSED_FLUSH32 16
#endif
#ifndef BORIS_FUSED_FLUSH64
#define BORIS_FUSED_FLUSH64 8
#endif
// One reciprocal square root for t and s (boris_momentum_*_m): measured 10 % faster
// on the fp64 uniform-field kernel (C3), slower on fp32 and on the generic-orientation
// plane wave (profiles/r01/exp_merged_rsqrt/).  BORIS_MERGED_RSQRT (tuning): 0 never,
// 1 every uniform / plane-wave Boris kernel, 2 fp64 uniform fields only.
#ifndef BORIS_MERGED_RSQRT
#define BORIS_MERGED_RSQRT 2
#endif
template <typename FP, int FIELD>
constexpr bool kMergedRsqrt =
    (FIELD == FK_UNIFORM || FIELD == FK_PLANE_WAVE) &&
    (BORIS_MERGED_RSQRT == 1 ||
     (BORIS_MERGED_RSQRT == 2 && sizeof(FP) == 8 && FIELD == FK_UNIFORM));

template <typename FP>
constexpr int kFlushOf = sizeof(FP) == 4 ? BORIS_FUSED_FLUSH32 : BORIS_FUSED_FLUSH64;
// m-dipole: sin/cos(omega0 t_n) is the same for every particle; each block
// tabulates -2 A0 sin and 2 A0 k cos of it (fp64 sincos, cast to FP, times the FP
// amplitude: the roundings the step would do) once per launch in shared memory.
// Launches are split into chunks of kTimeTab steps on the host.
constexpr int kTimeTab = 1024;

// One Boris step of the single-type m-dipole (kMdFold) in X = k r, u = p/(m c):
// E = 2 A0 cos(w t) g1 (-Y, X, 0), B = -2 A0 sin(w t) (g2 Z X + f3 z^), xi^2 = |X|^2
// (eq. 14 in readings c9, c10, c13).  The kick is (q dt/2mc) E = e (-Y, X, 0) with
// e = tab.y g1, and the rotation vector t = (q dt/2mc) B / gamma_n = a X + b z^ with
// a = (tab.x / gamma_n) g2 Z, b = (tab.x / gamma_n) f3 (eq. 9-13; E_z = 0 exactly);
// 1/gamma = rsqrt(1 + |u|^2) (eq. 5 with kappa = 1); the displacement in the window
// dX += (k c dt / gamma^{n+1/2}) u (eq. 7).  r^n = anchor + d (reading c-fp32r).
template <typename FP, typename FP2>
__device__ __forceinline__ void md_fold_step(const FP2 tab, FP xf, FP yf, FP zf, FP &dx, FP &dy,
                                             FP &dz, FP &ux, FP &uy, FP &uz, FP cr) {
    const FP x = b_add(xf, dx), y = b_add(yf, dy), z = b_add(zf, dz);
    FP g1, g2, f3;
    md_radial_x2<FP>(b_norm2(x, y, z), g1, g2, f3);
    const FP e = b_mul(tab.y, g1);
    ux = b_fma(-e, y, ux);
    uy = b_fma(e, x, uy);
    const FP tsb = b_mul(tab.x, b_rsqrt(b_fma(ux, ux, b_fma(uy, uy, b_fma(uz, uz, FP(1))))));
    const FP al = b_mul(tsb, b_mul(g2, z));
    boris_rotate<FP>(ux, uy, uz, b_mul(al, x), b_mul(al, y), b_fma(al, z, b_mul(tsb, f3)));
    ux = b_fma(-e, y, ux);
    uy = b_fma(e, x, uy);
    const FP ct = b_mul(cr, b_rsqrt(b_fma(ux, ux, b_fma(uy, uy, b_fma(uz, uz, FP(1))))));
    dx = b_fma(ct, ux, dx);
    dy = b_fma(ct, uy, dy);
    dz = b_fma(ct, uz, dz);
}

// Minimum resident blocks per SM in the fused kernels' launch bounds (0: none given).
// m-dipole: a register cap; fp32 single-type m-dipole, 10^7 x 10^3 steps: none (54
// registers) 2.77-2.84 ps, 8 (56) 2.70, 10 (40) 2.79-2.88, 12 (40) 2.71
// (profiles/r02/exp_mdipole_minb_pair.jsonl).  fp32 grid: an explicit 1 lets ptxas take
// 116 instead of 105 registers (100 fused steps, 10^7 sorted: 5.69 vs 5.87 ps); every
// other field keeps none -- an explicit 1 took C4 from 48 to 80 registers (1.18 ->
// 1.24 ps) and the fp64 grid kernel from 158 to 184 (10.9 -> 13.0 ps).  Sweep of the
// tuning knobs below (profiles/r02/exp_fused_minblocks_sweep.jsonl): fp64 m-dipole 5 / 6
// / 10 blocks 7.94 / 7.94 / 8.05 vs 7.86 ps with 8; uniform 1 / 10 C3 2.35 / 2.40 vs
// 2.33; plane wave 1 / 12 C4 1.24 / 1.20 vs 1.18.
#ifndef BORIS_MD_MINB
#define BORIS_MD_MINB 8
#endif
// Particles per thread of the single-type m-dipole kernel (tuning): 2 measured 2.69-2.71
// ps fp32 (72-80 registers), 8.0 fp64, vs 2.70 / 7.97 with 1.
#ifndef BORIS_MD_PAIR
#define BORIS_MD_PAIR 1
#endif
constexpr int kMdPair = BORIS_MD_PAIR;
#ifndef BORIS_MD_MINB64
#define BORIS_MD_MINB64 BORIS_MD_MINB
#endif
#ifndef BORIS_UNIFORM_MINB
#define BORIS_UNIFORM_MINB 0
#endif
#ifndef BORIS_PLANE_MINB
#define BORIS_PLANE_MINB 0
#endif
template <typename FP, int FIELD>
constexpr int kFusedMinBlocks =
    FIELD == FK_MDIPOLE                     ? (sizeof(FP) == 4 ? BORIS_MD_MINB : BORIS_MD_MINB64)
    : (FIELD == FK_GRID && sizeof(FP) == 4) ? 1
    : FIELD == FK_UNIFORM                   ? BORIS_UNIFORM_MINB
    : FIELD == FK_PLANE_WAVE                ? BORIS_PLANE_MINB
                                            : 0;

template <typename FP, int LAYOUT, int FIELD, bool MULTI, bool DIAG, int PUSHER, bool YZ>
__global__ void __launch_bounds__(kFusedThreads, kFusedMinBlocks<FP, FIELD>)
    k_fused(EnsView e, const __grid_constant__ AnalyticArgs<FP> fa,
            const __grid_constant__ KCoefs<FP, MULTI> co, int64_t n_steps, double *partials,
            const int *__restrict__ order) {
    constexpr int kFlush = kFlushOf<FP>;
    constexpr bool kMerged = kMergedRsqrt<FP, FIELD>;
    __shared__ TypeCoef<FP> s_t[MULTI ? kMaxTypes : 1];
    // m-dipole time table: .x the sin(w0 t_j) factor, .y the cos(w0 t_j) factor
    using FP2 = typename std::conditional<sizeof(FP) == 4, float2, double2>::type;
    __shared__ FP2 s_tab[FIELD == FK_MDIPOLE ? kTimeTab : 1];
    if (MULTI) load_type_table(co, s_t);
    // single-type Boris m-dipole (kMdFold): the step runs in X = k r, u = p/(m c)
    // (AnalyticArgs mdf_*), with the type's half-kick and rotation factors folded into
    // the time table (t and the kick come straight from the field's scalar factors, no
    // E, B vectors are formed)
    constexpr bool kMdFold = FIELD == FK_MDIPOLE && !MULTI && PUSHER == PUSHER_BORIS;
    if constexpr (FIELD == FK_MDIPOLE) {
        for (int j = threadIdx.x; j < n_steps; j += kFusedThreads) {
            double sn, cs;
            sincos(fa.w0t0 + (double)j * fa.w0dt, &sn, &cs);  // t_j = t0 + j dt (c5)
            if (kMdFold) {
                s_tab[j].x = (FP)(fa.mdf_rot * sn);   // (q dt / 2mc) (-2 A0 sin(w t_j))
                s_tab[j].y = (FP)(fa.mdf_kick * cs);  // (q dt / 2mc) 2 A0 cos(w t_j)
            } else {
                s_tab[j].x = b_mul(fa.mA02, (FP)sn);  // -2 A0 sin(w t_j)
                s_tab[j].y = b_mul(fa.A0k2, (FP)cs);  // 2 A0 k cos(w t_j)
            }
        }
        __syncthreads();
    }
    double ke = 0.0, cnt = 0.0;
    const int64_t stride = (int64_t)gridDim.x * kFusedThreads;
    auto push_particle = [&](int64_t i) {
        double xa, ya, za;
        FP px, py, pz, w;
        int ty;
        Particle<FP, LAYOUT>::load(e, i, xa, ya, za, px, py, pz, w, ty);
        if (!MULTI) ty = 0;
        const TypeCoef<FP> tc = MULTI ? s_t[ty] : co.t[0];
        FP ux = b_mul(px, tc.S), uy = b_mul(py, tc.S), uz = b_mul(pz, tc.S);
        FP gam = FP(1);
        // uniform / plane wave: E = c e, B = c b with fixed e, b -> per-particle aE e, alpha b
        FP ae[3], ab[3];
        if constexpr (FIELD == FK_UNIFORM || FIELD == FK_PLANE_WAVE) {
            const FP *ev = FIELD == FK_UNIFORM ? fa.E : fa.cE;
            const FP *bv = FIELD == FK_UNIFORM ? fa.B : fa.cB;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                ae[k] = b_mul(tc.aE, ev[k]);
                ab[k] = b_mul(tc.alpha, bv[k]);
            }
        }
        // boris_momentum_*_m operands (exact power-of-two scalings)
        FP abs_[3] = {FP(0), FP(0), FP(0)}, abs2[3] = {FP(0), FP(0), FP(0)};
        if constexpr (kMerged) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                abs_[k] = b_mul(ab[k], FP(1.52587890625e-05));  // 2^-16
                abs2[k] = b_mul(ab[k], FP(3.0517578125e-05));   // 2^-15
            }
        }
        const FP kappa2s = b_mul(tc.kappa2, FP(2.3283064365386963e-10));  // 2^-32
        const FP ones = FP(2.3283064365386963e-10);
#if BORIS_GRID_CACHE
        GridCache<FP> gcache;  // FK_GRID: the particle's cell records (dead code otherwise)
#endif
        for (int64_t s0 = 0; s0 < n_steps; s0 += kFlush) {
            FP phia = FP(0);
            if constexpr (FIELD == FK_PLANE_WAVE)
                phia = (FP)reduce_2pi(fma(fa.kvec[0], xa, fma(fa.kvec[1], ya, fa.kvec[2] * za)) +
                                      (fa.ph0 - (double)s0 * fa.wdt));
            FP dx = FP(0), dy = FP(0), dz = FP(0);
            const int m = (n_steps - s0) < kFlush ? (int)(n_steps - s0) : kFlush;
            auto step = [&](int j) {
                FP inv_g;
                if constexpr (FIELD == FK_UNIFORM) {
                    if constexpr (kMerged && YZ)
                        inv_g = boris_momentum_yz_m<FP, true>(ux, uy, uz, FP(1), ae[1], abs_[2],
                                                              abs2[2], tc.kappa2, kappa2s, ones,
                                                              gam);
                    else if constexpr (kMerged && PUSHER == PUSHER_BORIS)
                        inv_g = boris_momentum_dir_m<FP, true>(ux, uy, uz, FP(1), ae, abs_, abs2,
                                                               tc.kappa2, kappa2s, ones, gam);
                    else if constexpr (YZ)
                        inv_g = boris_momentum_yz<FP, true>(ux, uy, uz, FP(1), ae[1], ab[2],
                                                            tc.kappa2, gam);
                    else if constexpr (PUSHER == PUSHER_BORIS)
                        inv_g = boris_momentum_dir<FP, true>(ux, uy, uz, FP(1), ae, ab, tc.kappa2,
                                                             gam);
                    else
                        inv_g = momentum_update<FP, PUSHER>(ux, uy, uz, fa.E[0], fa.E[1], fa.E[2],
                                                            fa.B[0], fa.B[1], fa.B[2], tc, gam);
                } else if constexpr (FIELD == FK_PLANE_WAVE) {
                    // YZ: kf = (kf0, 0, 0) exactly, the dropped fma terms add signed zeros
                    const FP phi = YZ ? b_fma(fa.kf[0], dx, b_fma(-(FP)j, fa.wdtf, phia))
                                      : b_fma(fa.kf[0], dx, b_fma(fa.kf[1], dy, b_fma(fa.kf[2], dz,
                                        b_fma(-(FP)j, fa.wdtf, phia))));
                    const FP c = cos_small(phi);  // E = E0 e_hat c, B = E0 (k_hat x e_hat) c
                    if constexpr (kMerged && YZ)
                        inv_g = boris_momentum_yz_m<FP, false>(ux, uy, uz, c, ae[1], abs_[2],
                                                               abs2[2], tc.kappa2, kappa2s, ones,
                                                               gam);
                    else if constexpr (kMerged && PUSHER == PUSHER_BORIS)
                        inv_g = boris_momentum_dir_m<FP, false>(ux, uy, uz, c, ae, abs_, abs2,
                                                                tc.kappa2, kappa2s, ones, gam);
                    else if constexpr (YZ)
                        inv_g = boris_momentum_yz<FP, false>(ux, uy, uz, c, ae[1], ab[2],
                                                             tc.kappa2, gam);
                    else if constexpr (PUSHER == PUSHER_BORIS)
                        inv_g = boris_momentum_dir<FP, false>(ux, uy, uz, c, ae, ab, tc.kappa2,
                                                              gam);
                    else
                        inv_g = momentum_update<FP, PUSHER>(
                            ux, uy, uz, b_mul(fa.cE[0], c), b_mul(fa.cE[1], c), b_mul(fa.cE[2], c),
                            b_mul(fa.cB[0], c), b_mul(fa.cB[1], c), b_mul(fa.cB[2], c), tc, gam);
                } else if constexpr (FIELD == FK_GRID) {  // CIC gather (reading c-grid)
                    FP Ex, Ey, Ez, Bx, By, Bz;
#if BORIS_GRID_CACHE
                    grid_gather_cached<FP>(fa.grid, b_add((FP)xa, dx), b_add((FP)ya, dy),
                                           b_add((FP)za, dz), gcache, Ex, Ey, Ez, Bx, By, Bz);
#else
                    grid_gather<FP>(fa.grid, b_add((FP)xa, dx), b_add((FP)ya, dy),
                                    b_add((FP)za, dz), Ex, Ey, Ez, Bx, By, Bz);
#endif
                    inv_g = momentum_update<FP, PUSHER>(ux, uy, uz, Ex, Ey, Ez, Bx, By, Bz, tc, gam);
                } else {  // FK_MDIPOLE, eq. 14 in readings c9, c10, c13
                    FP Ex, Ey, Ez, Bx, By, Bz;
                    const FP x = b_add((FP)xa, dx), y = b_add((FP)ya, dy), z = b_add((FP)za, dz);
                    FP g1, g2, f3;
                    md_radial_r2<FP>(fa, b_norm2(x, y, z), g1, g2, f3);
                    // per-block tables hold the amplitudes (same roundings as in the step)
                    const FP2 tab = s_tab[s0 + j];
                    const FP ce = b_mul(tab.y, g1);  // 2 A0 k cos(w t) f1/xi
                    const FP sb = tab.x;             // -2 A0 sin(w t)
                    const FP k2g2 = b_mul(fa.k2, g2);               // f2/R^2
                    Ex = -b_mul(ce, y);
                    Ey = b_mul(ce, x);
                    Ez = FP(0);
                    const FP sk = b_mul(sb, k2g2);
                    Bx = b_mul(b_mul(sk, x), z);
                    By = b_mul(b_mul(sk, y), z);
                    Bz = b_mul(sb, b_fma(k2g2, b_mul(z, z), f3));
                    if constexpr (PUSHER == PUSHER_BORIS)  // E_z = 0 exactly (eq. 14)
                        inv_g = boris_momentum<FP, true>(ux, uy, uz, Ex, Ey, Ez, Bx, By, Bz, tc,
                                                         gam);
                    else
                        inv_g = momentum_update<FP, PUSHER>(ux, uy, uz, Ex, Ey, Ez, Bx, By, Bz,
                                                            tc, gam);
                }
                // a10 (eq. 7): displacement accumulated in the window
                const FP ct = b_mul(tc.cr, inv_g);
                dx = b_fma(ct, ux, dx);
                dy = b_fma(ct, uy, dy);
                dz = b_fma(ct, uz, dz);
            };
            // full windows of the short-bodied fields run as straight-line code (measured
            // +4 % on C4); the long m-dipole / grid bodies stay rolled (unrolled: -15 %;
            // unrolled by 2: m-dipole -0.5..2 %, grid -5 %).
            constexpr bool kUnroll = FIELD == FK_UNIFORM || FIELD == FK_PLANE_WAVE;
            if (kUnroll && m == kFlush) {
#pragma unroll
                for (int j = 0; j < kFlush; ++j) step(j);
            } else {
                for (int j = 0; j < m; ++j) step(j);
            }
            xa = __dadd_rn(xa, (double)dx);
            ya = __dadd_rn(ya, (double)dy);
            za = __dadd_rn(za, (double)dz);
        }
        const double x = xa, y = ya, z = za;
        if (n_steps == 0) gam = b_sqrt(b_fma(tc.kappa2, b_norm2(ux, uy, uz), FP(1)));
        Particle<FP, LAYOUT>::store(e, i, x, y, z, b_mul(ux, tc.invS), b_mul(uy, tc.invS),
                                    b_mul(uz, tc.invS), gam);
        if (DIAG) {
            ke += (double)kinetic_energy<FP>(ux, uy, uz, gam, w, tc);
            cnt += 1.0;
        }
    };
    // kMdFold: kMdPair particles per thread stepped together (kMdPair = 2: two
    // independent dependency chains per thread, the time-table load and the loop
    // control shared).  i1 < 0: the second chain repeats particle i0, not stored.
    auto push_md = [&](int64_t i0, int64_t i1) {
        constexpr int Q = kMdPair;
        const TypeCoef<FP> tc = co.t[0];
        const int64_t ii[2] = {i0, i1 >= 0 ? i1 : i0};
        double xa[Q], ya[Q], za[Q];
        FP ux[Q], uy[Q], uz[Q], w[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            FP px, py, pz;
            int ty;
            Particle<FP, LAYOUT>::load(e, ii[q], xa[q], ya[q], za[q], px, py, pz, w[q], ty);
            ux[q] = b_mul(px, fa.mdf_uin);  // u = p/(m c)
            uy[q] = b_mul(py, fa.mdf_uin);
            uz[q] = b_mul(pz, fa.mdf_uin);
            xa[q] *= fa.mdf_k;  // X = k r
            ya[q] *= fa.mdf_k;
            za[q] *= fa.mdf_k;
        }
        for (int64_t s0 = 0; s0 < n_steps; s0 += kFlush) {
            FP dx[Q], dy[Q], dz[Q], xf[Q], yf[Q], zf[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                dx[q] = dy[q] = dz[q] = FP(0);
                xf[q] = (FP)xa[q];
                yf[q] = (FP)ya[q];
                zf[q] = (FP)za[q];
            }
            const int m = (n_steps - s0) < kFlush ? (int)(n_steps - s0) : kFlush;
            const FP2 *tab = s_tab + s0;
            for (int j = 0; j < m; ++j) {
                const FP2 tj = tab[j];
#pragma unroll
                for (int q = 0; q < Q; ++q)
                    md_fold_step<FP>(tj, xf[q], yf[q], zf[q], dx[q], dy[q], dz[q], ux[q], uy[q],
                                     uz[q], fa.mdf_cr);
            }
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                xa[q] = __dadd_rn(xa[q], (double)dx[q]);
                ya[q] = __dadd_rn(ya[q], (double)dy[q]);
                za[q] = __dadd_rn(za[q], (double)dz[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            if (q == 1 && i1 < 0) break;
            // back from X = k r, u = p/(m c); then u = S p as in the other kernels
            const FP sx = b_mul(b_mul(ux[q], fa.mdf_uout), tc.S);
            const FP sy = b_mul(b_mul(uy[q], fa.mdf_uout), tc.S);
            const FP sz = b_mul(b_mul(uz[q], fa.mdf_uout), tc.S);
            FP gam;
            if (n_steps == 0)
                gam = b_sqrt(b_fma(tc.kappa2, b_norm2(sx, sy, sz), FP(1)));
            else
                boris_gamma<FP>(sx, sy, sz, tc.kappa2, gam);
            Particle<FP, LAYOUT>::store(e, ii[q], xa[q] * fa.mdf_ik, ya[q] * fa.mdf_ik,
                                        za[q] * fa.mdf_ik, b_mul(sx, tc.invS), b_mul(sy, tc.invS),
                                        b_mul(sz, tc.invS), gam);
            if (DIAG) {
                ke += (double)kinetic_energy<FP>(sx, sy, sz, gam, w[q], tc);
                cnt += 1.0;
            }
        }
    };
    if constexpr (kMdFold) {  // warp-rounds of 32 kMdPair over the branch order
        const int64_t nwarp = (int64_t)gridDim.x * (kFusedThreads / 32);
        constexpr int64_t R = 32 * kMdPair;
        for (int64_t r = (int64_t)blockIdx.x * (kFusedThreads / 32) + (threadIdx.x >> 5);
             r * R < e.n; r += nwarp) {
            const int64_t k = r * R + (threadIdx.x & 31);
            if (k < e.n)
                push_md(order ? order[k] : k,
                        (kMdPair == 2 && k + 32 < e.n) ? (order ? order[k + 32] : k + 32) : -1);
        }
    } else if constexpr (FIELD == FK_MDIPOLE) {  // warp-rounds over the branch order
        const int64_t nwarp = (int64_t)gridDim.x * (kFusedThreads / 32);
        for (int64_t r = (int64_t)blockIdx.x * (kFusedThreads / 32) + (threadIdx.x >> 5);
             r * 32 < e.n; r += nwarp) {
            const int64_t k = r * 32 + (threadIdx.x & 31);
            if (k < e.n) push_particle(order ? order[k] : k);
        }
    } else {
        for (int64_t i = (int64_t)blockIdx.x * kFusedThreads + threadIdx.x; i < e.n; i += stride)
            push_particle(i);
    }
    if (DIAG) block_diag_partial<kFusedThreads>(ke, cnt, partials);
}

template <typename FP, int LAYOUT, int FIELD, bool MULTI, bool DIAG, int PUSHER>
static cudaError_t dispatch_fused(const EnsView &e, const AnalyticArgs<FP> &fa,
                                  const Coefs<FP> &co, int64_t n_steps, DiagOut *diag,
                                  int device, cudaStream_t st) {
    constexpr bool kPair = FIELD == FK_MDIPOLE && !MULTI && PUSHER == PUSHER_BORIS;  // kMdFold
    const int64_t per_block = (kPair ? kMdPair : 1) * (int64_t)kFusedThreads;
    const int64_t blocks = (e.n + per_block - 1) / per_block;
    constexpr bool kHasYZ =
        (FIELD == FK_UNIFORM || FIELD == FK_PLANE_WAVE) && PUSHER == PUSHER_BORIS;
    const auto kern = (kHasYZ && fa.yz) ? &k_fused<FP, LAYOUT, FIELD, MULTI, DIAG, PUSHER, kHasYZ>
                                        : &k_fused<FP, LAYOUT, FIELD, MULTI, DIAG, PUSHER, false>;
    int64_t grid = fused_grid((const void *)kern, blocks > 0 ? blocks : 1, device);
    if (DIAG && grid > diag->cap) grid = diag->cap;
    int *order = nullptr;  // nullptr: storage order
    if constexpr (FIELD == FK_MDIPOLE) {  // branch order (k_md_order), stream-ordered scratch
        // (scheduling only: above 2^31 particles, or without scratch memory, the kernel
        // pushes in storage order)
        if (fa.md_order && e.n <= INT32_MAX &&
            scratch_alloc((void **)&order, (size_t)e.n * sizeof(int) + 64, st) == cudaSuccess) {
            unsigned long long *counts = (unsigned long long *)((char *)order +
                                                                (((size_t)e.n * 4 + 15) / 16) * 16);
            cudaError_t err = cudaMemsetAsync(counts, 0, 2 * sizeof(unsigned long long), st);
            if (err == cudaSuccess) {
                k_md_order<FP, LAYOUT><<<(unsigned)stream_grid((e.n + 255) / 256, 8, device, 4),
                                         256, 0, st>>>(e, fa, order, counts);
                err = cudaGetLastError();
            }
            if (err != cudaSuccess) {
                scratch_free(order, st);
                return err;
            }
        } else {
            (void)cudaGetLastError();  // a failed pool allocation is not sticky
            order = nullptr;
        }
    }
    kern<<<(unsigned)grid, kFusedThreads, 0, st>>>(e, fa, kcoefs<MULTI>(co), n_steps,
                                                  diag ? diag->partials : nullptr, order);
    const cudaError_t kerr = cudaGetLastError();
    if (order) scratch_free(order, st);
    if (diag) diag->written = DIAG ? grid : 0;
    return kerr;
}

template <typename FP, int LAYOUT, int FIELD, int PUSHER>
static cudaError_t dispatch_fused_md(const EnsView &e, const AnalyticArgs<FP> &fa,
                                     const Coefs<FP> &co, int64_t n_steps, bool multi,
                                     DiagOut *diag, int device, cudaStream_t st) {
    if (multi)
        return diag ? dispatch_fused<FP, LAYOUT, FIELD, true, true, PUSHER>(e, fa, co, n_steps,
                                                                             diag, device, st)
                    : dispatch_fused<FP, LAYOUT, FIELD, true, false, PUSHER>(e, fa, co, n_steps,
                                                                              diag, device, st);
    return diag ? dispatch_fused<FP, LAYOUT, FIELD, false, true, PUSHER>(e, fa, co, n_steps, diag,
                                                                          device, st)
                : dispatch_fused<FP, LAYOUT, FIELD, false, false, PUSHER>(e, fa, co, n_steps,
                                                                           diag, device, st);
}

template <typename FP, int LAYOUT, int PUSHER>
static cudaError_t dispatch_fused_field(const EnsView &e, int field_kind,
                                        const AnalyticArgs<FP> &fa, const Coefs<FP> &co,
                                        int64_t n_steps, bool multi, DiagOut *diag, int device,
                                        cudaStream_t st) {
    switch (field_kind) {
    case FK_UNIFORM:
        return dispatch_fused_md<FP, LAYOUT, FK_UNIFORM, PUSHER>(e, fa, co, n_steps, multi, diag,
                                                                 device, st);
    case FK_PLANE_WAVE:
        return dispatch_fused_md<FP, LAYOUT, FK_PLANE_WAVE, PUSHER>(e, fa, co, n_steps, multi,
                                                                    diag, device, st);
    case FK_MDIPOLE:
        return dispatch_fused_md<FP, LAYOUT, FK_MDIPOLE, PUSHER>(e, fa, co, n_steps, multi, diag,
                                                                 device, st);
    case FK_GRID:
        return dispatch_fused_md<FP, LAYOUT, FK_GRID, PUSHER>(e, fa, co, n_steps, multi, diag,
                                                              device, st);
    default:
        return cudaErrorInvalidValue;
    }
}

template <typename FP, int LAYOUT>
static cudaError_t dispatch_fused_pusher(const EnsView &e, int field_kind,
                                         const AnalyticArgs<FP> &fa, const Coefs<FP> &co,
                                         int64_t n_steps, bool multi, int pusher, DiagOut *diag,
                                         int device, cudaStream_t st) {
    switch (pusher) {
    case PUSHER_VAY:
        return dispatch_fused_field<FP, LAYOUT, PUSHER_VAY>(e, field_kind, fa, co, n_steps,
                                                            multi, diag, device, st);
    case PUSHER_HIGUERA_CARY:
        return dispatch_fused_field<FP, LAYOUT, PUSHER_HIGUERA_CARY>(e, field_kind, fa, co,
                                                                     n_steps, multi, diag,
                                                                     device, st);
    default:
        return dispatch_fused_field<FP, LAYOUT, PUSHER_BORIS>(e, field_kind, fa, co, n_steps,
                                                              multi, diag, device, st);
    }
}

template <typename FP>
cudaError_t launch_fused(const EnsView &e, int field_kind, const AnalyticArgs<FP> &fa,
                         const Coefs<FP> &co, int64_t n_steps, bool multi, int pusher,
                         DiagOut *diag, int device, cudaStream_t st) {
    if (e.n == 0) {
        if (diag) diag->written = 0;
        return cudaSuccess;
    }
    // m-dipole launches cover at most kTimeTab steps (the per-block time table);
    // chunk c starts at t0 + c0 dt, omega0 t computed from the step index (c5).
    const int64_t chunk = field_kind == FK_MDIPOLE ? kTimeTab : n_steps;
    for (int64_t c0 = 0; c0 < n_steps; c0 += chunk) {
        const int64_t m = (n_steps - c0) < chunk ? n_steps - c0 : chunk;
        AnalyticArgs<FP> fc = fa;
        fc.w0t0 = fa.w0t0 + (double)c0 * fa.w0dt;
        DiagOut *d = (c0 + m == n_steps) ? diag : nullptr;
        const cudaError_t err =
            e.layout == BORIS_LAYOUT_SOA
                ? dispatch_fused_pusher<FP, BORIS_LAYOUT_SOA>(e, field_kind, fc, co, m, multi,
                                                              pusher, d, device, st)
                : dispatch_fused_pusher<FP, BORIS_LAYOUT_AOS>(e, field_kind, fc, co, m, multi,
                                                              pusher, d, device, st);
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

template cudaError_t launch_fused<float>(const EnsView &, int, const AnalyticArgs<float> &,
                                         const Coefs<float> &, int64_t, bool, int, DiagOut *, int,
                                         cudaStream_t);
template cudaError_t launch_fused<double>(const EnsView &, int, const AnalyticArgs<double> &,
                                          const Coefs<double> &, int64_t, bool, int, DiagOut *,
                                          int, cudaStream_t);

// ---------------------------------------------------------------------------
// "Precalculated fields": an analytic field evaluated at
// every particle's current position at time t0 (fa built with that t0), written
// to per-particle arrays (SoA) or {E,B} records (AoS).  Reads r (12/24 B),
// writes E,B (24/48 B) per particle; same analytic_field as the fused push.
// ---------------------------------------------------------------------------
template <typename FP, int LAYOUT, int FIELD>
__global__ void __launch_bounds__(kFusedThreads)
    k_field_evaluate(EnsView e, const __grid_constant__ AnalyticArgs<FP> fa, FieldSoaPtrs out,
                     void *out_rec) {
    const int64_t stride = (int64_t)gridDim.x * kFusedThreads;
    for (int64_t i = (int64_t)blockIdx.x * kFusedThreads + threadIdx.x; i < e.n; i += stride) {
        double x, y, z;
        FP px, py, pz, w;
        int ty;
        Particle<FP, LAYOUT>::load(e, i, x, y, z, px, py, pz, w, ty);
        FP Ex, Ey, Ez, Bx, By, Bz;
        analytic_field<FP, FIELD>(fa, x, y, z, 0, Ex, Ey, Ez, Bx, By, Bz);
        if (LAYOUT == BORIS_LAYOUT_SOA) {
            ((FP *)out.Ex)[i] = Ex;
            ((FP *)out.Ey)[i] = Ey;
            ((FP *)out.Ez)[i] = Ez;
            ((FP *)out.Bx)[i] = Bx;
            ((FP *)out.By)[i] = By;
            ((FP *)out.Bz)[i] = Bz;
        } else {
            FP *r = (FP *)out_rec + 6 * i;
            r[0] = Ex; r[1] = Ey; r[2] = Ez;
            r[3] = Bx; r[4] = By; r[5] = Bz;
        }
    }
}

template <typename FP, int LAYOUT>
static cudaError_t dispatch_eval(const EnsView &e, int field_kind, const AnalyticArgs<FP> &fa,
                                 const FieldSoaPtrs &out, void *out_rec, int device,
                                 cudaStream_t st) {
    const int64_t blocks = (e.n + kFusedThreads - 1) / kFusedThreads;
    const unsigned grid = (unsigned)stream_grid(blocks > 0 ? blocks : 1, 2048 / kFusedThreads,
                                                device);
    switch (field_kind) {
    case FK_UNIFORM:
        k_field_evaluate<FP, LAYOUT, FK_UNIFORM><<<grid, kFusedThreads, 0, st>>>(e, fa, out, out_rec);
        break;
    case FK_PLANE_WAVE:
        k_field_evaluate<FP, LAYOUT, FK_PLANE_WAVE><<<grid, kFusedThreads, 0, st>>>(e, fa, out, out_rec);
        break;
    case FK_MDIPOLE:
        k_field_evaluate<FP, LAYOUT, FK_MDIPOLE><<<grid, kFusedThreads, 0, st>>>(e, fa, out, out_rec);
        break;
    case FK_GRID:
        k_field_evaluate<FP, LAYOUT, FK_GRID><<<grid, kFusedThreads, 0, st>>>(e, fa, out, out_rec);
        break;
    default:
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <typename FP>
cudaError_t launch_field_evaluate(const EnsView &e, int field_kind, const AnalyticArgs<FP> &fa,
                                  const FieldSoaPtrs &out, void *out_rec, int device,
                                  cudaStream_t st) {
    if (e.n == 0) return cudaSuccess;
    if (e.layout == BORIS_LAYOUT_SOA)
        return dispatch_eval<FP, BORIS_LAYOUT_SOA>(e, field_kind, fa, out, out_rec, device, st);
    return dispatch_eval<FP, BORIS_LAYOUT_AOS>(e, field_kind, fa, out, out_rec, device, st);
}

template cudaError_t launch_field_evaluate<float>(const EnsView &, int,
                                                  const AnalyticArgs<float> &,
                                                  const FieldSoaPtrs &, void *, int,
                                                  cudaStream_t);
template cudaError_t launch_field_evaluate<double>(const EnsView &, int,
                                                   const AnalyticArgs<double> &,
                                                   const FieldSoaPtrs &, void *, int,
                                                   cudaStream_t);

}  // namespace boris
