// boris_device.cuh -- device-side building blocks of the B200 Boris pusher.
//
// The per-particle arithmetic is the paper's procedure (arXiv 2104.04579 §2,
// PAPER.md L175-186) on a power-of-two scaled momentum u = S p, S = 2^k ~ 1/(mc)
// chosen per type on the host, so that p <-> u conversions are EXACT (no
// rounding bias accumulates step after step) while every intermediate stays
// O(1) in fp32 for any unit system.  With kappa = 1/(S m c):
//   u^-  = u + aE E                  aE = S q dt/2                      (eq. 9)
//   g_n  = sqrt(1 + kappa^2 |u^-|^2)                                     (L162)
//   t    = alpha B / g_n             alpha = q dt/(2 m c)                (eq. 13)
//   s    = 2 t/(1 + |t|^2)
//   u'   = u^- + u^- x t,  u^+ = u^- + u' x s                            (eq. 12)
//   u    = u^+ + aE E                                                    (eq. 10)
//   g    = sqrt(1 + kappa^2 |u|^2),  r += (cr / g) u,  cr = dt/(S m)     (eq. 5, 7)
// which is eq. 9-13, 5, 7 multiplied through by S (the rotation is scale-free).
//
// Every operation is an explicit IEEE intrinsic (__fmul_rn, __fadd_rn,
// __fmaf_rn, ...): the compiler can neither contract nor reorder them, so every
// kernel variant (SoA vector / scalar tail / unaligned, AoS tiles, multi-type,
// with or without diagnostics, device- or host-resident) produces bit-identical
// results for the same particle.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "libboris.h"

namespace boris {

#ifndef BORIS_KMAX_TYPES
#define BORIS_KMAX_TYPES BORIS_MAX_TYPES
#endif
constexpr int kMaxTypes = BORIS_KMAX_TYPES;  // == BORIS_MAX_TYPES (tuning builds may shrink it)

// Per-type coefficients, computed in double on the host for each push and
// cast to FP.
template <typename FP>
struct TypeCoef {
    FP aE;      // S q dt / 2       E half kick in scaled units (eq. 9-10)
    FP alpha;   // q dt / (2 m c)   t = alpha B / gamma_n (eq. 13)
    FP kappa2;  // 1 / (S m c)^2    gamma = sqrt(1 + kappa2 |u|^2) (eq. 5)
    FP cr;      // dt / (S m)       r += cr u / gamma (eq. 7)
    FP S;       // 2^k              u = S p (exact)
    FP invS;    // 2^-k             p = invS u (exact)
    FP ke;      // m c^2 kappa^2 = 1/(S^2 m): KE = w ke |u|^2/(gamma+1)
    FP kappa;   // 1 / (S m c)      (alternative pushers: u*.tau in true units)
};

// Momentum update scheme (readings c-vay, c-hc in DESIGN.md).
enum Pusher { PUSHER_BORIS = 0, PUSHER_VAY = 1, PUSHER_HIGUERA_CARY = 2 };

template <typename FP, int NT>
struct CoefsN {
    int n_types;  // table entries used
    TypeCoef<FP> t[NT];
};
// The full per-push table (host side, multi-type kernels).
template <typename FP>
using Coefs = CoefsN<FP, kMaxTypes>;
// A kernel instantiation's parameter block: single-type kernels read t[0] only, so
// they take a one-entry table (a 256-entry fp32 table in every launch's parameter
// block measured +0.4-1.0 us per push on 4096-particle launches).
template <typename FP, bool MULTI>
using KCoefs = CoefsN<FP, MULTI ? kMaxTypes : 1>;
template <bool MULTI, typename FP>
inline KCoefs<FP, MULTI> kcoefs(const Coefs<FP> &co) {
    if constexpr (MULTI) {
        return co;
    } else {
        KCoefs<FP, false> k;
        k.n_types = co.n_types;
        k.t[0] = co.t[0];
        return k;
    }
}

// ---------------------------------------------------------------------------
// Correctly rounded elementary operations (IEEE round-to-nearest, reading c14),
// never contracted or reassociated by the compiler.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float b_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double b_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float b_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double b_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float b_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double b_fma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float b_sqrt(float x) { return __fsqrt_rn(x); }
__device__ __forceinline__ double b_sqrt(double x) { return __dsqrt_rn(x); }
__device__ __forceinline__ float b_rcp(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double b_rcp(double x) { return __drcp_rn(x); }

// Reciprocal square root and reciprocal used by the push.  Default (north_star:
// "fp32 variants using rsqrt/FMA"): fp32 uses the MUFU approximations
// rsqrt.approx / rcp.approx (<= 2 ulp); fp64 uses CUDA's rsqrt (1 ulp) and the
// IEEE reciprocal.  -DBORIS_PRECISE_MATH switches every one of them to
// correctly rounded sqrt + reciprocal.  Either way the operations are
// deterministic, so all kernel variants stay bitwise identical.
#ifdef BORIS_PRECISE_MATH
__device__ __forceinline__ float b_rsqrt(float x) { return __frcp_rn(__fsqrt_rn(x)); }
__device__ __forceinline__ double b_rsqrt(double x) { return __drcp_rn(__dsqrt_rn(x)); }
__device__ __forceinline__ float b_rcpx(float x) { return __frcp_rn(x); }
#else
__device__ __forceinline__ float b_rsqrt(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ double b_rsqrt(double x) { return rsqrt(x); }
__device__ __forceinline__ float b_rcpx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
#endif
__device__ __forceinline__ double b_rcpx(double x) { return __drcp_rn(x); }

// |v|^2 = fma(x, x, fma(y, y, z*z))
template <typename FP>
__device__ __forceinline__ FP b_norm2(FP x, FP y, FP z) {
    return b_fma(x, x, b_fma(y, y, b_mul(z, z)));
}
// a*b - c*d (one component of a cross product)
template <typename FP>
__device__ __forceinline__ FP b_cross(FP a, FP b, FP c, FP d) {
    return b_fma(a, b, -b_mul(c, d));
}

// Steps a6 (s from t, eq. 13) and a7 (rotation, eq. 12) given t.  Each cross
// product component is folded into the addition as two nested FMAs,
// u'_x = fma(u_y, t_z, fma(-u_z, t_y, u_x)), so a zero component of t (the
// axis-aligned fields) drops out exactly: fma(-u_z, 0, u_x) == u_x.
template <typename FP>
__device__ __forceinline__ void boris_rotate(FP &ux, FP &uy, FP &uz, FP tx, FP ty, FP tz) {
    const FP sf = b_mul(FP(2), b_rcpx(b_fma(tx, tx, b_fma(ty, ty, b_fma(tz, tz, FP(1))))));
    const FP sx = b_mul(sf, tx), sy = b_mul(sf, ty), sz = b_mul(sf, tz);
    // u' = u^- + u^- x t ; u^+ = u^- + u' x s
    const FP upx = b_fma(uy, tz, b_fma(-uz, ty, ux));
    const FP upy = b_fma(uz, tx, b_fma(-ux, tz, uy));
    const FP upz = b_fma(ux, ty, b_fma(-uy, tx, uz));
    ux = b_fma(upy, sz, b_fma(-upz, sy, ux));
    uy = b_fma(upz, sx, b_fma(-upx, sz, uy));
    uz = b_fma(upx, sy, b_fma(-upy, sx, uz));
}

// Step a9: gamma^{n+1/2} (eq. 5, reading c3); returns its reciprocal.
template <typename FP>
__device__ __forceinline__ FP boris_gamma(FP ux, FP uy, FP uz, FP kappa2, FP &gamma) {
    const FP g2 = b_fma(kappa2, b_norm2(ux, uy, uz), FP(1));
#ifdef BORIS_PRECISE_MATH
    gamma = b_sqrt(g2);
    return b_rcp(gamma);
#else
    const FP inv_g = b_rsqrt(g2);
    gamma = b_mul(g2, inv_g);
    return inv_g;
#endif
}

// Boris momentum update for a field of fixed directions with a common scalar
// amplitude c: E = c e, B = c b (plane wave: c = cos phi; uniform: c = 1, UNIT).
// ae = aE e and ab = alpha b are precomputed per particle (per type), which
// saves 6 multiplies per step in the register-fused kernels.  Same steps a4-a9.
template <typename FP, bool UNIT>
__device__ __forceinline__ FP boris_momentum_dir(FP &ux, FP &uy, FP &uz, FP c, const FP (&ae)[3],
                                                 const FP (&ab)[3], FP kappa2, FP &gamma) {
    // half kicks: u + c aE e as one FMA (UNIT: c = 1, a plain addition)
    auto kick = [&](FP u, FP a) { return UNIT ? b_add(u, a) : b_fma(c, a, u); };
    ux = kick(ux, ae[0]);
    uy = kick(uy, ae[1]);
    uz = kick(uz, ae[2]);
    const FP inv_gn = b_rsqrt(b_fma(kappa2, b_norm2(ux, uy, uz), FP(1)));
    const FP ta = UNIT ? inv_gn : b_mul(inv_gn, c);
    boris_rotate<FP>(ux, uy, uz, b_mul(ta, ab[0]), b_mul(ta, ab[1]), b_mul(ta, ab[2]));
    ux = kick(ux, ae[0]);
    uy = kick(uy, ae[1]);
    uz = kick(uz, ae[2]);
    return boris_gamma<FP>(ux, uy, uz, kappa2, gamma);
}

// boris_momentum_dir for the axis-aligned orientation E = c aE_y y^, B = c ab_z z^
// (a plane wave with k^ = x^, e^ = y^, or a uniform E || y^, B || z^; either may
// be zero).  It performs exactly the roundings boris_momentum_dir performs when
// ae = (0, aey, 0) and ab = (0, 0, abz) — every product with an exact zero and
// every addition of a signed zero drops out — so results are bitwise identical
// (up to the sign of zero components) with ~40 % fewer instructions per step.
template <typename FP, bool UNIT>
__device__ __forceinline__ FP boris_momentum_yz(FP &ux, FP &uy, FP &uz, FP c, FP aey, FP abz,
                                                FP kappa2, FP &gamma) {
    uy = UNIT ? b_add(uy, aey) : b_fma(c, aey, uy);
    const FP inv_gn = b_rsqrt(b_fma(kappa2, b_norm2(ux, uy, uz), FP(1)));
    const FP ta = UNIT ? inv_gn : b_mul(inv_gn, c);
    const FP tz = b_mul(ta, abz);
    // boris_rotate with t = (0, 0, tz): s = (0, 0, sf tz)
    const FP sz = b_mul(b_mul(FP(2), b_rcpx(b_fma(tz, tz, FP(1)))), tz);
    const FP upx = b_fma(uy, tz, ux);
    const FP upy = b_fma(-ux, tz, uy);
    ux = b_fma(upy, sz, ux);
    uy = b_fma(-upx, sz, uy);
    uy = UNIT ? b_add(uy, aey) : b_fma(c, aey, uy);
    return boris_gamma<FP>(ux, uy, uz, kappa2, gamma);
}

// Merged-reciprocal variants of boris_momentum_dir / _yz (register-fused kernels).
// With tau = alpha B (= c ab) and g2 = gamma_n^2, D = g2 + |tau|^2:
//   t = tau / gamma_n,  s = 2 t / (1 + |t|^2) = 2 tau gamma_n / D,
// and both come from ONE reciprocal square root r = rsqrt(g2 D^2) = 1/(gamma_n D):
//   t = (D r) tau,  s = (2 g2 r) tau,
// instead of rsqrt(g2) and the reciprocal 1/(1 + |t|^2) (eq. 13 re-associated).  The
// operands are pre-scaled by powers of two (exact): g2s = 2^-32 g2 (kappa2s =
// 2^-32 kappa2, ones = 2^-32), taus = 2^-16 tau (abs = 2^-16 ab), taus2 = 2^-15 tau
// (abs2), so X = g2s Ds^2 = 2^-96 g2 D^2 stays a normal fp32 number for
// 1 <= gamma_n, |tau| < 2^37; then Ds r = 2^16/gamma_n and g2s r = 2^16 gamma_n/D.
template <typename FP>
__device__ __forceinline__ void boris_rotate_ts(FP &ux, FP &uy, FP &uz, FP tx, FP ty, FP tz,
                                                FP sx, FP sy, FP sz) {
    const FP upx = b_fma(uy, tz, b_fma(-uz, ty, ux));
    const FP upy = b_fma(uz, tx, b_fma(-ux, tz, uy));
    const FP upz = b_fma(ux, ty, b_fma(-uy, tx, uz));
    ux = b_fma(upy, sz, b_fma(-upz, sy, ux));
    uy = b_fma(upz, sx, b_fma(-upx, sz, uy));
    uz = b_fma(upx, sy, b_fma(-upy, sx, uz));
}

template <typename FP, bool UNIT>
__device__ __forceinline__ FP boris_momentum_dir_m(FP &ux, FP &uy, FP &uz, FP c,
                                                   const FP (&ae)[3], const FP (&abs)[3],
                                                   const FP (&abs2)[3], FP kappa2, FP kappa2s,
                                                   FP ones, FP &gamma) {
    auto kick = [&](FP u, FP a) { return UNIT ? b_add(u, a) : b_fma(c, a, u); };
    ux = kick(ux, ae[0]);
    uy = kick(uy, ae[1]);
    uz = kick(uz, ae[2]);
    const FP g2s = b_fma(kappa2s, b_norm2(ux, uy, uz), ones);
    FP ts[3], ts2[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        ts[k] = UNIT ? abs[k] : b_mul(c, abs[k]);
        ts2[k] = UNIT ? abs2[k] : b_mul(c, abs2[k]);
    }
    const FP Ds = b_fma(ts[0], ts[0], b_fma(ts[1], ts[1], b_fma(ts[2], ts[2], g2s)));
    const FP r = b_rsqrt(b_mul(b_mul(g2s, Ds), Ds));
    const FP ft = b_mul(Ds, r), fs = b_mul(g2s, r);
    boris_rotate_ts<FP>(ux, uy, uz, b_mul(ft, ts[0]), b_mul(ft, ts[1]), b_mul(ft, ts[2]),
                        b_mul(fs, ts2[0]), b_mul(fs, ts2[1]), b_mul(fs, ts2[2]));
    ux = kick(ux, ae[0]);
    uy = kick(uy, ae[1]);
    uz = kick(uz, ae[2]);
    return boris_gamma<FP>(ux, uy, uz, kappa2, gamma);
}

// boris_momentum_dir_m for E || y^, B || z^: the same roundings with the exact
// zeros dropped (fma(0, 0, x) == x), bitwise identical.
template <typename FP, bool UNIT>
__device__ __forceinline__ FP boris_momentum_yz_m(FP &ux, FP &uy, FP &uz, FP c, FP aey, FP absz,
                                                  FP abs2z, FP kappa2, FP kappa2s, FP ones,
                                                  FP &gamma) {
    uy = UNIT ? b_add(uy, aey) : b_fma(c, aey, uy);
    const FP g2s = b_fma(kappa2s, b_norm2(ux, uy, uz), ones);
    const FP ts = UNIT ? absz : b_mul(c, absz);
    const FP ts2 = UNIT ? abs2z : b_mul(c, abs2z);
    const FP Ds = b_fma(ts, ts, g2s);
    const FP r = b_rsqrt(b_mul(b_mul(g2s, Ds), Ds));
    const FP tz = b_mul(b_mul(Ds, r), ts);
    const FP sz = b_mul(b_mul(g2s, r), ts2);
    const FP upx = b_fma(uy, tz, ux);
    const FP upy = b_fma(-ux, tz, uy);
    ux = b_fma(upy, sz, ux);
    uy = b_fma(-upx, sz, uy);
    uy = UNIT ? b_add(uy, aey) : b_fma(c, aey, uy);
    return boris_gamma<FP>(ux, uy, uz, kappa2, gamma);
}

// One Boris momentum update on the scaled momentum u (steps a4-a9).
// Returns 1/gamma^{n+1/2}; writes gamma^{n+1/2} to `gamma`.  EZ0: the caller's
// E_z is exactly zero (the m-dipole, eq. 14), so the z kicks u_z + aE 0 are
// skipped -- the same value up to the sign of a zero u_z.
template <typename FP, bool EZ0 = false>
__device__ __forceinline__ FP boris_momentum(FP &ux, FP &uy, FP &uz, FP Ex, FP Ey, FP Ez, FP Bx,
                                             FP By, FP Bz, const TypeCoef<FP> &tc, FP &gamma) {
    // a4: first electric half kick (eq. 9), u + aE E as one FMA per component
    ux = b_fma(tc.aE, Ex, ux);
    uy = b_fma(tc.aE, Ey, uy);
    if (!EZ0) uz = b_fma(tc.aE, Ez, uz);
    // a5: 1/gamma_n, gamma_n = gamma(u^-) (L162, reading c2)
    const FP inv_gn = b_rsqrt(b_fma(tc.kappa2, b_norm2(ux, uy, uz), FP(1)));
    // a6: rotation vectors (eq. 13)
    const FP ta = b_mul(tc.alpha, inv_gn);
    // a6-a7: s and the rotation (eq. 12-13)
    boris_rotate<FP>(ux, uy, uz, b_mul(ta, Bx), b_mul(ta, By), b_mul(ta, Bz));
    // a8: second electric half kick (eq. 10)
    ux = b_fma(tc.aE, Ex, ux);
    uy = b_fma(tc.aE, Ey, uy);
    if (!EZ0) uz = b_fma(tc.aE, Ez, uz);
    // a9: gamma^{n+1/2} (eq. 5, reading c3) and its reciprocal
    return boris_gamma<FP>(ux, uy, uz, tc.kappa2, gamma);
}

// ---------------------------------------------------------------------------
// Alternative pushers (Vay 2008; Higuera & Cary 2017), same scaled-u units:
// u = S p, u_true = kappa u, tau = alpha B = q B dt/(2mc) (dimensionless).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float b_sqrtx(float x) {
#ifdef BORIS_PRECISE_MATH
    return __fsqrt_rn(x);
#else
    return b_mul(x, b_rsqrt(x));  // x > 0 here
#endif
}
__device__ __forceinline__ double b_sqrtx(double x) { return __dsqrt_rn(x); }

// gamma_new: positive root of g^4 - sigma g^2 - (tau^2 + u*^2) = 0 with
// sigma = 1 + |v_true|^2 - tau^2 and u* = v_true . tau.
template <typename FP>
__device__ __forceinline__ FP alt_gamma(FP vx, FP vy, FP vz, FP tx, FP ty, FP tz, FP tau2,
                                        const TypeCoef<FP> &tc) {
    const FP sigma = b_add(b_fma(tc.kappa2, b_norm2(vx, vy, vz), FP(1)), -tau2);
    const FP us = b_mul(tc.kappa, b_fma(vx, tx, b_fma(vy, ty, b_mul(vz, tz))));
    const FP disc = b_fma(sigma, sigma, b_mul(FP(4), b_fma(us, us, tau2)));
    return b_sqrtx(b_mul(FP(0.5), b_add(sigma, b_sqrtx(disc))));
}

// x = s [v + (v.t) t + v x t], s = 1/(1+t^2): the solution of x = v + x x t.
template <typename FP>
__device__ __forceinline__ void alt_rotate(FP vx, FP vy, FP vz, FP tx, FP ty, FP tz, FP &x,
                                           FP &y, FP &z) {
    const FP s = b_rcpx(b_add(FP(1), b_norm2(tx, ty, tz)));
    const FP vt = b_fma(vx, tx, b_fma(vy, ty, b_mul(vz, tz)));
    x = b_mul(s, b_add(b_fma(vt, tx, vx), b_cross(vy, tz, vz, ty)));
    y = b_mul(s, b_add(b_fma(vt, ty, vy), b_cross(vz, tx, vx, tz)));
    z = b_mul(s, b_add(b_fma(vt, tz, vz), b_cross(vx, ty, vy, tx)));
}

// Higuera-Cary: u- = u + eps; gamma_new(u-, tau); t = tau/gamma_new;
// ubar = implicit rotation of u-; u = ubar + eps + ubar x t.
template <typename FP>
__device__ __forceinline__ FP hc_momentum(FP &ux, FP &uy, FP &uz, FP Ex, FP Ey, FP Ez, FP Bx,
                                          FP By, FP Bz, const TypeCoef<FP> &tc, FP &gamma) {
    const FP ex = b_mul(tc.aE, Ex), ey = b_mul(tc.aE, Ey), ez = b_mul(tc.aE, Ez);
    ux = b_add(ux, ex);
    uy = b_add(uy, ey);
    uz = b_add(uz, ez);
    const FP tx = b_mul(tc.alpha, Bx), ty = b_mul(tc.alpha, By), tz = b_mul(tc.alpha, Bz);
    const FP tau2 = b_norm2(tx, ty, tz);
    const FP ig = b_rcpx(alt_gamma<FP>(ux, uy, uz, tx, ty, tz, tau2, tc));
    const FP sx = b_mul(tx, ig), sy = b_mul(ty, ig), sz = b_mul(tz, ig);
    FP bx, by, bz;
    alt_rotate<FP>(ux, uy, uz, sx, sy, sz, bx, by, bz);
    ux = b_add(b_add(bx, ex), b_cross(by, sz, bz, sy));
    uy = b_add(b_add(by, ey), b_cross(bz, sx, bx, sz));
    uz = b_add(b_add(bz, ez), b_cross(bx, sy, by, sx));
    return boris_gamma<FP>(ux, uy, uz, tc.kappa2, gamma);
}

// Vay: u' = u + 2 eps + (u/gamma(u)) x tau; gamma_new(u', tau); t = tau/gamma_new;
// u = implicit rotation of u'.
template <typename FP>
__device__ __forceinline__ FP vay_momentum(FP &ux, FP &uy, FP &uz, FP Ex, FP Ey, FP Ez, FP Bx,
                                           FP By, FP Bz, const TypeCoef<FP> &tc, FP &gamma) {
    const FP ig0 = b_rsqrt(b_fma(tc.kappa2, b_norm2(ux, uy, uz), FP(1)));
    const FP tx = b_mul(tc.alpha, Bx), ty = b_mul(tc.alpha, By), tz = b_mul(tc.alpha, Bz);
    const FP wx = b_mul(ux, ig0), wy = b_mul(uy, ig0), wz = b_mul(uz, ig0);
    const FP a2 = b_mul(FP(2), tc.aE);
    const FP px = b_add(b_fma(a2, Ex, ux), b_cross(wy, tz, wz, ty));
    const FP py = b_add(b_fma(a2, Ey, uy), b_cross(wz, tx, wx, tz));
    const FP pz = b_add(b_fma(a2, Ez, uz), b_cross(wx, ty, wy, tx));
    const FP tau2 = b_norm2(tx, ty, tz);
    const FP ig = b_rcpx(alt_gamma<FP>(px, py, pz, tx, ty, tz, tau2, tc));
    alt_rotate<FP>(px, py, pz, b_mul(tx, ig), b_mul(ty, ig), b_mul(tz, ig), ux, uy, uz);
    return boris_gamma<FP>(ux, uy, uz, tc.kappa2, gamma);
}

// Steps a4-a9 with the selected scheme.
template <typename FP, int PUSHER>
__device__ __forceinline__ FP momentum_update(FP &ux, FP &uy, FP &uz, FP Ex, FP Ey, FP Ez, FP Bx,
                                              FP By, FP Bz, const TypeCoef<FP> &tc, FP &gamma) {
    if constexpr (PUSHER == PUSHER_VAY)
        return vay_momentum<FP>(ux, uy, uz, Ex, Ey, Ez, Bx, By, Bz, tc, gamma);
    else if constexpr (PUSHER == PUSHER_HIGUERA_CARY)
        return hc_momentum<FP>(ux, uy, uz, Ex, Ey, Ez, Bx, By, Bz, tc, gamma);
    else
        return boris_momentum<FP>(ux, uy, uz, Ex, Ey, Ez, Bx, By, Bz, tc, gamma);
}

// One full Boris step of one particle on stored quantities (rows a1-a11):
// p -> u (exact), boris_momentum, position update, u -> p (exact).  Shared by
// every streaming path so they are bitwise identical.
// Returns 1/gamma^{n+1/2} (the deposition's v = u inv_Sm / gamma reuses it).
template <typename FP, int PUSHER = PUSHER_BORIS>
__device__ __forceinline__ FP push_one(FP &x, FP &y, FP &z, FP &px, FP &py, FP &pz, FP &g,
                                         FP Ex, FP Ey, FP Ez, FP Bx, FP By, FP Bz,
                                         const TypeCoef<FP> &tc, FP &ux, FP &uy, FP &uz) {
    ux = b_mul(px, tc.S);
    uy = b_mul(py, tc.S);
    uz = b_mul(pz, tc.S);
    const FP inv_g = momentum_update<FP, PUSHER>(ux, uy, uz, Ex, Ey, Ez, Bx, By, Bz, tc, g);
    // a10: r^{n+1} = r^n + dt p^{n+1/2}/(gamma m) = r^n + (cr/gamma) u   (eq. 7)
    const FP ct = b_mul(tc.cr, inv_g);
    x = b_fma(ct, ux, x);
    y = b_fma(ct, uy, y);
    z = b_fma(ct, uz, z);
    // a11: store p = u / S
    px = b_mul(ux, tc.invS);
    py = b_mul(uy, tc.invS);
    pz = b_mul(uz, tc.invS);
    return inv_g;
}

// Kinetic energy of one macroparticle, w m c^2 |p/(mc)|^2 / (gamma + 1)
// (= w (gamma-1) m c^2 without cancellation, reading c17), evaluated in FP and
// accumulated by the caller in double; tc.ke = m c^2 kappa^2 converts |u|^2.
template <typename FP>
__device__ __forceinline__ FP kinetic_energy(FP ux, FP uy, FP uz, FP gamma, FP w,
                                             const TypeCoef<FP> &tc) {
    const FP u2 = b_norm2(ux, uy, uz);
    return b_mul(b_mul(w, tc.ke), b_mul(u2, b_rcpx(b_add(gamma, FP(1)))));
}

// ---------------------------------------------------------------------------
// Streaming global-memory access with cache hints.  State arrays are read once
// and written once per step by the same thread; field arrays are read-only.
// Nothing is reused within a step, so loads bypass L1 and stores are
// evict-first (st.global.cs).
// ---------------------------------------------------------------------------
// Tuning knobs (experiments only; defaults are the measured best):
// BORIS_LD_L2PF adds the .L2::256B prefetch-size hint to streaming loads,
// BORIS_ST_WB uses write-back instead of evict-first (.cs) stores.
#ifdef BORIS_LD_L2PF
#define BORIS_LD_PF ".L2::256B"
#else
#define BORIS_LD_PF ""
#endif
#ifdef BORIS_STATE_NC
#define BORIS_STATE_LD "ld.global.nc.L1::no_allocate"
#else
#define BORIS_STATE_LD "ld.global.L1::no_allocate"
#endif
#ifdef BORIS_ST_WB
#define BORIS_ST_Q ""
#else
#define BORIS_ST_Q ".cs"
#endif

__device__ __forceinline__ float4 ld_state(const float *p) {
    float4 v;
    asm volatile(BORIS_STATE_LD BORIS_LD_PF ".v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_state(const double *p) {
    double2 v;
    asm volatile(BORIS_STATE_LD BORIS_LD_PF ".v2.f64 {%0,%1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ld_field(const float *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate" BORIS_LD_PF ".v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_field(const double *p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate" BORIS_LD_PF ".v2.f64 {%0,%1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream(float *p, float4 v) {
    asm volatile("st.global" BORIS_ST_Q ".v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_stream(double *p, double2 v) {
    asm volatile("st.global" BORIS_ST_Q ".v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
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
template <typename FP, int NT>
__device__ __forceinline__ void load_type_table(const CoefsN<FP, NT> &co, TypeCoef<FP> *s_t) {
    for (int i = threadIdx.x; i < co.n_types; i += blockDim.x) s_t[i] = co.t[i];
    __syncthreads();
}

}  // namespace boris
