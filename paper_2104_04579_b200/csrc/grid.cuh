// grid.cuh -- field gather from a periodic collocated Cartesian grid with the
// CIC (cloud-in-cell, first-order) form factor (PAPER.md
// L72-79, L89-91: "each particle interacts with a set of nearby grid values of
// the electromagnetic field, depending on the form factor"; reading c-grid in
// DESIGN.md).  Node (i,j,k) sits at origin + (i hx, j hy, k hz); the grid repeats
// with period (nx hx, ny hy, nz hz).  Nodes are packed as x-pair records of
// kGridRecord = 12 FP: node i followed by its periodic +x neighbour.
#pragma once

#include "boris_device.cuh"

namespace boris {

constexpr int kGridRecord = 12;  // FP per x-pair record: [E B](i) [E B](i+1)

template <typename FP>
struct GridArgs {
    const FP *nodes;  // x-pair records (12 FP, kGridStride apart), record (i,j,k) at (k*ny + j)*nx + i
    FP org[3];        // origin
    FP inv_h[3];      // 1 / spacing
    FP nf[3];         // n as FP
    FP inv_nf[3];     // 1 / n
    int n[3];
};

// One axis of the CIC weights: xi = (x - org)/h, base node floor(xi) wrapped into
// [0, n), upper node base+1 (mod n), weight of the upper node f = xi - floor(xi).
// FAST: a floor inside [0, n) skips the periodic wrap (a branch; the index is the
// same).  Measured: faster in the register-fused grid kernel (6.24 -> 5.86 ps fp32) and
// the fused PIC step (26.0 -> 25.8 ps), slower in the single-step grid push (11.5 ->
// 11.8 ps), which keeps the branch-free wrap.
template <typename FP, bool FAST = false>
__device__ __forceinline__ void grid_axis(FP x, FP org, FP inv_h, FP nf, FP inv_nf, int n,
                                          int &i0, int &i1, FP &f) {
    const FP xi = b_mul(b_add(x, -org), inv_h);
    const FP fl = floor(xi);
    f = b_add(xi, -fl);  // exact, in [0, 1)
    int i;
    if (FAST && fl >= FP(0) && fl < nf) {  // inside the periodic box: no wrap needed
        i = (int)fl;
    } else {
        const FP w = b_fma(-nf, floor(b_mul(fl, inv_nf)), fl);  // fl mod n, up to +-1 rounding
        i = (int)w;
        if (i >= n) i -= n;
        if (i < 0) i += n;
    }
    i0 = i;
    i1 = (i + 1 == n) ? 0 : i + 1;
}

// Linear index of the cell whose base node is (i0, j0, k0): the sort key.
template <typename FP>
__device__ __forceinline__ uint32_t grid_cell(const GridArgs<FP> &g, FP x, FP y, FP z) {
    int i0, i1, j0, j1, k0, k1;
    FP f;
    grid_axis<FP>(x, g.org[0], g.inv_h[0], g.nf[0], g.inv_nf[0], g.n[0], i0, i1, f);
    grid_axis<FP>(y, g.org[1], g.inv_h[1], g.nf[1], g.inv_nf[1], g.n[1], j0, j1, f);
    grid_axis<FP>(z, g.org[2], g.inv_h[2], g.nf[2], g.inv_nf[2], g.n[2], k0, k1, f);
    return ((uint32_t)k0 * (uint32_t)g.n[1] + (uint32_t)j0) * (uint32_t)g.n[0] + (uint32_t)i0;
}

// FP between consecutive records in the nodes buffer.  BORIS_GRID_LDG256 (tuning): a
// record is read with 256-bit loads (sm_100 LDG.256) -- fp32 pads the 48 B record to
// 64 B so every record starts on a 32 B boundary (one 256-bit + one 128-bit load),
// fp64's 96 B records are three 256-bit loads.  Measured (10^7, 64^3): single-step
// push sorted fp32 11.56-11.73 vs 11.52-11.55 ps with 16 B loads, fp64 26.1 vs 22.4, PIC
// cycle 25.3 both (profiles/r02/exp_grid_ldg256.jsonl): off (3 / 6 16 B loads).
#ifndef BORIS_GRID_LDG256
#define BORIS_GRID_LDG256 0
#endif
template <typename FP>
constexpr int kGridStride = (sizeof(FP) == 4 && BORIS_GRID_LDG256) ? 16 : kGridRecord;

// The two x-nodes (i0, i0+1 mod nx) of a cell row: one x-pair record, 12 FP,
// e[0..5] = [E B](i0), e[6..11] = [E B](i0+1): 12 loads per particle with 16 B loads
// (16 with one 8-FP record per node).
__device__ __forceinline__ void load_pair(const float *nodes, uint32_t rec, float (&e)[12]) {
    const float *p = nodes + kGridStride<float> * (size_t)rec;
#if BORIS_GRID_LDG256
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(e[0]), "=f"(e[1]), "=f"(e[2]), "=f"(e[3]), "=f"(e[4]), "=f"(e[5]), "=f"(e[6]),
          "=f"(e[7])
        : "l"(p));
    const float4 c = __ldg(reinterpret_cast<const float4 *>(p + 8));
    e[8] = c.x; e[9] = c.y; e[10] = c.z; e[11] = c.w;
#else
    const float4 *q = reinterpret_cast<const float4 *>(p);
    const float4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
    e[0] = a.x; e[1] = a.y; e[2] = a.z; e[3] = a.w; e[4] = b.x; e[5] = b.y;
    e[6] = b.z; e[7] = b.w; e[8] = c.x; e[9] = c.y; e[10] = c.z; e[11] = c.w;
#endif
}
__device__ __forceinline__ void load_pair(const double *nodes, uint32_t rec, double (&e)[12]) {
    const double *p = nodes + kGridStride<double> * (size_t)rec;
#if BORIS_GRID_LDG256
#pragma unroll
    for (int k = 0; k < 3; ++k)
        asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
            : "=d"(e[4 * k]), "=d"(e[4 * k + 1]), "=d"(e[4 * k + 2]), "=d"(e[4 * k + 3])
            : "l"(p + 4 * k));
#else
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const double2 v = __ldg(reinterpret_cast<const double2 *>(p) + k);
        e[2 * k] = v.x;
        e[2 * k + 1] = v.y;
    }
#endif
}

// E, B at (x, y, z): sum over the 8 nodes of the cell of wx wy wz F_node.
template <typename FP, bool FAST = false>
__device__ __forceinline__ void grid_gather(const GridArgs<FP> &g, FP x, FP y, FP z, FP &Ex,
                                            FP &Ey, FP &Ez, FP &Bx, FP &By, FP &Bz) {
    int ix[2], iy[2], iz[2];
    FP fx, fy, fz;
    grid_axis<FP, FAST>(x, g.org[0], g.inv_h[0], g.nf[0], g.inv_nf[0], g.n[0], ix[0], ix[1], fx);
    grid_axis<FP, FAST>(y, g.org[1], g.inv_h[1], g.nf[1], g.inv_nf[1], g.n[1], iy[0], iy[1], fy);
    grid_axis<FP, FAST>(z, g.org[2], g.inv_h[2], g.nf[2], g.inv_nf[2], g.n[2], iz[0], iz[1], fz);
    const FP wx[2] = {b_add(FP(1), -fx), fx};
    const FP wy[2] = {b_add(FP(1), -fy), fy};
    const FP wz[2] = {b_add(FP(1), -fz), fz};
    FP acc[6] = {FP(0), FP(0), FP(0), FP(0), FP(0), FP(0)};
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const FP wyz = b_mul(wy[b], wz[c]);
            const uint32_t row = ((uint32_t)iz[c] * (uint32_t)g.n[1] + (uint32_t)iy[b]) *
                                 (uint32_t)g.n[0];
            FP pair[12];
            load_pair(g.nodes, row + (uint32_t)ix[0], pair);
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const FP wt = b_mul(wx[a], wyz);
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = b_fma(wt, pair[6 * a + q], acc[q]);
            }
        }
    Ex = acc[0]; Ey = acc[1]; Ez = acc[2];
    Bx = acc[3]; By = acc[4]; Bz = acc[5];
}

// grid_gather for a thread that owns one particle over many steps (the register-
// fused kernel): the cell's four x-pair records stay in registers and are reloaded
// only when the particle's base cell changes (a particle crosses a cell every
// h/(v dt) steps), so the per-step L1 gather requests disappear.  Same arithmetic
// in the same order as grid_gather: bitwise identical.
template <typename FP>
struct GridCache {
    uint32_t key = 0xFFFFFFFFu;  // linear index of the cached base cell (none)
    FP rec[4][12];
};

template <typename FP>
__device__ __forceinline__ void grid_gather_cached(const GridArgs<FP> &g, FP x, FP y, FP z,
                                                   GridCache<FP> &gc, FP &Ex, FP &Ey, FP &Ez,
                                                   FP &Bx, FP &By, FP &Bz) {
    int ix[2], iy[2], iz[2];
    FP fx, fy, fz;
    grid_axis<FP, true>(x, g.org[0], g.inv_h[0], g.nf[0], g.inv_nf[0], g.n[0], ix[0], ix[1], fx);
    grid_axis<FP, true>(y, g.org[1], g.inv_h[1], g.nf[1], g.inv_nf[1], g.n[1], iy[0], iy[1], fy);
    grid_axis<FP, true>(z, g.org[2], g.inv_h[2], g.nf[2], g.inv_nf[2], g.n[2], iz[0], iz[1], fz);
    const uint32_t key =
        ((uint32_t)iz[0] * (uint32_t)g.n[1] + (uint32_t)iy[0]) * (uint32_t)g.n[0] + (uint32_t)ix[0];
    if (key != gc.key) {
        gc.key = key;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int b = 0; b < 2; ++b)
                load_pair(g.nodes,
                          ((uint32_t)iz[c] * (uint32_t)g.n[1] + (uint32_t)iy[b]) *
                                  (uint32_t)g.n[0] + (uint32_t)ix[0],
                          gc.rec[c * 2 + b]);
    }
    const FP wx[2] = {b_add(FP(1), -fx), fx};
    const FP wy[2] = {b_add(FP(1), -fy), fy};
    const FP wz[2] = {b_add(FP(1), -fz), fz};
    FP acc[6] = {FP(0), FP(0), FP(0), FP(0), FP(0), FP(0)};
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const FP wyz = b_mul(wy[b], wz[c]);
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const FP wt = b_mul(wx[a], wyz);
#pragma unroll
                for (int q = 0; q < 6; ++q)
                    acc[q] = b_fma(wt, gc.rec[c * 2 + b][6 * a + q], acc[q]);
            }
        }
    Ex = acc[0]; Ey = acc[1]; Ez = acc[2];
    Bx = acc[3]; By = acc[4]; Bz = acc[5];
}

}  // namespace boris
