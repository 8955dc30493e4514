// deposit.cuh -- run-accumulating CIC current deposition of one lane (SURVEY §8(f)
// row 4; reading c-dep in DESIGN.md): q w v^{n+1/2} at the half-
// step position r^{n+1/2} = r^{n+1} - (dt/2) v^{n+1/2}, divided by the cell volume,
// onto the 8 nodes of the particle's cell.  A lane keeps the 8 x 3 node sums of its
// current cell in registers and issues atomics only when the cell changes
// (`add`), or at the end of a warp tile after merging with the neighbouring lanes
// that hold the same cell (`warp_merge` + `flush`).  Shared by the standalone
// deposition kernel (k_grid.cu) and the fused push + deposit kernel.
#pragma once

#include "boris_internal.h"

namespace boris {

constexpr uint32_t kNoNode = 0xFFFFFFFFu;

// End-of-tile merge of the lanes' open cells: shuffle scan (warp_merge + flush) or
// transposed through shared memory (merge_flush; fp32 only, fp64's 24 x 34 doubles
// per warp would exceed static shared memory).  Standalone deposition (kTransposedMerge)
// and the fused PIC step (kTransposedMergePD) choose separately (measured).
#ifndef BORIS_DEP_MERGE_T
#define BORIS_DEP_MERGE_T 0
#endif
#ifndef BORIS_PD_MERGE_T
#define BORIS_PD_MERGE_T 1
#endif
template <typename FP>
constexpr bool kTransposedMerge = sizeof(FP) == 4 && BORIS_DEP_MERGE_T;
template <typename FP>
constexpr bool kTransposedMergePD = sizeof(FP) == 4 && BORIS_PD_MERGE_T;

template <typename FP>
struct DepositRun {
    FP acc[8][3];
    int cx[2], cy[2], cz[2];  // the open cell's node indices (cx[0] < 0: none)
    FP fl[3];                 // the open cell's unwrapped floor((r - org)/h)

    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q][0] = acc[q][1] = acc[q][2] = FP(0);
        cx[0] = cx[1] = -1;
        cy[0] = cy[1] = cz[0] = cz[1] = 0;
        fl[0] = fl[1] = fl[2] = FP(0);
    }

    // grid_axis split in two: the unwrapped floor and the weight f (every
    // particle), the periodic wrap to node indices (only when the cell changes).
    static __device__ __forceinline__ FP axis_floor(FP x, FP org, FP inv_h, FP &f) {
        const FP xi = b_mul(b_add(x, -org), inv_h);
        const FP l = floor(xi);
        f = b_add(xi, -l);  // exact, in [0, 1)
        return l;
    }
    static __device__ __forceinline__ void axis_wrap(FP l, FP nf, FP inv_nf, int n, int &i0,
                                                     int &i1) {
        const FP w = b_fma(-nf, floor(b_mul(l, inv_nf)), l);  // l mod n, up to +-1 rounding
        int i = (int)w;
        if (i >= n) i -= n;
        if (i < 0) i += n;
        i0 = i;
        i1 = (i + 1 == n) ? 0 : i + 1;
    }

    // Atomics for the open cell (if any), then zero the sums.
    __device__ __forceinline__ void flush(const GridArgs<FP> &g, FP *Jx, FP *Jy, FP *Jz) {
        if (cx[0] < 0) return;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const uint32_t row =
                    ((uint32_t)cz[c] * (uint32_t)g.n[1] + (uint32_t)cy[b]) * (uint32_t)g.n[0];
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const int q = (c * 2 + b) * 2 + a;
                    const uint32_t node = row + (uint32_t)cx[a];
                    atomicAdd(Jx + node, acc[q][0]);
                    atomicAdd(Jy + node, acc[q][1]);
                    atomicAdd(Jz + node, acc[q][2]);
                    acc[q][0] = acc[q][1] = acc[q][2] = FP(0);
                }
            }
    }

    // One particle (state after the push: r^{n+1}, p^{n+1/2}, weight w).
    __device__ __forceinline__ void add(const GridArgs<FP> &g, const DepCoef<FP> &t, FP half_dt,
                                        FP x, FP y, FP z, FP px, FP py, FP pz, FP w, FP *Jx,
                                        FP *Jy, FP *Jz) {
        const FP ux = b_mul(px, t.S), uy = b_mul(py, t.S), uz = b_mul(pz, t.S);
        add_u(g, t, half_dt, x, y, z, ux, uy, uz,
              b_rsqrt(b_fma(t.kappa2, b_norm2(ux, uy, uz), FP(1))), w, Jx, Jy, Jz);
    }

    // The same with u = S p and 1/gamma known (the fused PIC step has both from the
    // push: bitwise the values add() recomputes).
    __device__ __forceinline__ void add_u(const GridArgs<FP> &g, const DepCoef<FP> &t, FP half_dt,
                                          FP x, FP y, FP z, FP ux, FP uy, FP uz, FP inv_g, FP w,
                                          FP *Jx, FP *Jy, FP *Jz) {
        // v = p/(gamma m) = u/(S m gamma)
        const FP vf = b_mul(t.inv_Sm, inv_g);
        const FP vx = b_mul(ux, vf), vy = b_mul(uy, vf), vz = b_mul(uz, vf);
        FP fx, fy, fz;
        const FP lx = axis_floor(b_fma(-half_dt, vx, x), g.org[0], g.inv_h[0], fx);
        const FP ly = axis_floor(b_fma(-half_dt, vy, y), g.org[1], g.inv_h[1], fy);
        const FP lz = axis_floor(b_fma(-half_dt, vz, z), g.org[2], g.inv_h[2], fz);
        // same unwrapped cell -> same nodes; a periodic image of the open cell only
        // costs an extra flush
        if (cx[0] < 0 || lx != fl[0] || ly != fl[1] || lz != fl[2]) {
            flush(g, Jx, Jy, Jz);
            fl[0] = lx; fl[1] = ly; fl[2] = lz;
            axis_wrap(lx, g.nf[0], g.inv_nf[0], g.n[0], cx[0], cx[1]);
            axis_wrap(ly, g.nf[1], g.inv_nf[1], g.n[1], cy[0], cy[1]);
            axis_wrap(lz, g.nf[2], g.inv_nf[2], g.n[2], cz[0], cz[1]);
        }
        const FP wx[2] = {b_add(FP(1), -fx), fx};
        const FP wy[2] = {b_add(FP(1), -fy), fy};
        const FP wz[2] = {b_add(FP(1), -fz), fz};
        const FP qw = b_mul(t.q_vol, w);
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const FP wyz = b_mul(qw, b_mul(wy[b], wz[c]));
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const int q = (c * 2 + b) * 2 + a;
                    const FP sw = b_mul(wx[a], wyz);
                    acc[q][0] = b_fma(sw, vx, acc[q][0]);
                    acc[q][1] = b_fma(sw, vy, acc[q][1]);
                    acc[q][2] = b_fma(sw, vz, acc[q][2]);
                }
            }
    }

    // Per-warp scratch of merge_flush.
    struct MergeSmem {
        static constexpr int RS = sizeof(FP) == 4 ? 36 : 34;  // row stride: conflict-free
        FP red[24 * RS];      // red[t * RS + l] = lane l's sum t = q * 3 + d
        uint32_t rowb[4][32];  // lane l's open cell: row bases ((k*ny + j)*nx) for (b, c)
        int cxs[2][32];        // and its two x node indices
    };

    // End of a warp tile (all 32 lanes), transposed: every lane stashes its 24 sums
    // in shared memory, then lane t < 24 walks component t of the 32 lanes in lane
    // order and adds each run of equal open cells (contiguous when sorted) to J
    // with one atomic at the run's last lane -- one 24-lane atomic instruction per
    // run instead of a shuffle scan over the 24 sums.  The run ends (tails) are
    // warp-uniform, so the walk's branches do not diverge.
    __device__ __forceinline__ void merge_flush(const GridArgs<FP> &g, FP *Jx, FP *Jy, FP *Jz,
                                                MergeSmem &sm, int lane) {
        const unsigned full = 0xffffffffu;
        const bool has = cx[0] >= 0;
        const uint32_t key = has ? ((uint32_t)cz[0] * (uint32_t)g.n[1] + (uint32_t)cy[0]) *
                                           (uint32_t)g.n[0] + (uint32_t)cx[0]
                                 : kNoNode;
        const uint32_t next = __shfl_down_sync(full, key, 1);
        const unsigned tails = __ballot_sync(full, has && (lane == 31 || next != key));
        if (tails == 0) return;
        constexpr int RS = MergeSmem::RS;
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                sm.red[(q * 3 + d) * RS + lane] = acc[q][d];
                acc[q][d] = FP(0);
            }
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int b = 0; b < 2; ++b)
                sm.rowb[c * 2 + b][lane] =
                    ((uint32_t)cz[c] * (uint32_t)g.n[1] + (uint32_t)cy[b]) * (uint32_t)g.n[0];
        sm.cxs[0][lane] = cx[0];
        sm.cxs[1][lane] = cx[1];
        cx[0] = -1;
        __syncwarp();
        if (lane < 24) {
            const int q = lane / 3, d = lane - 3 * (lane / 3);
            FP *J = d == 0 ? Jx : (d == 1 ? Jy : Jz);
            const FP *row = sm.red + lane * RS;
            const uint32_t *rb = sm.rowb[q >> 1];
            const int *xs = sm.cxs[q & 1];
            FP run = FP(0);
            constexpr int VW = 16 / sizeof(FP);  // FP per 16 B vector
#pragma unroll
            for (int l0 = 0; l0 < 32; l0 += VW) {
                FP v[VW];
                if constexpr (VW == 4) {
                    const float4 t = reinterpret_cast<const float4 *>(row)[l0 / 4];
                    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
                } else {
                    const double2 t = reinterpret_cast<const double2 *>(row)[l0 / 2];
                    v[0] = t.x; v[1] = t.y;
                }
#pragma unroll
                for (int k = 0; k < VW; ++k) {
                    run = b_add(run, v[k]);
                    if (tails & (1u << (l0 + k))) {  // warp-uniform
                        atomicAdd(J + rb[l0 + k] + (uint32_t)xs[l0 + k], run);
                        run = FP(0);
                    }
                }
            }
        }
        __syncwarp();
    }

    // End of a warp tile (all 32 lanes): lanes holding the same open cell in
    // consecutive lanes (contiguous when sorted) are summed with a segmented
    // scan; every lane but each segment's last drops its cell, so the following
    // flush() issues one set of atomics per segment.
    __device__ __forceinline__ void warp_merge(const GridArgs<FP> &g, int lane) {
        const unsigned full = 0xffffffffu;
        const uint32_t key = cx[0] < 0 ? kNoNode
                                       : ((uint32_t)cz[0] * (uint32_t)g.n[1] + (uint32_t)cy[0]) *
                                                 (uint32_t)g.n[0] + (uint32_t)cx[0];
        const uint32_t prev = __shfl_up_sync(full, key, 1);
        const uint32_t next = __shfl_down_sync(full, key, 1);
        const unsigned heads = __ballot_sync(full, lane == 0 || prev != key);
        const int seg = 31 - __clz(heads & (full >> (31 - lane)));
        // only as many scan rounds as the longest segment needs (warp-uniform)
        const int span = (int)__reduce_max_sync(full, (unsigned)(lane - seg));
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            if (off > span) break;
            const bool take = lane - off >= seg;
#pragma unroll
            for (int q = 0; q < 8; ++q)
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const FP v = __shfl_up_sync(full, acc[q][d], off);
                    if (take) acc[q][d] = b_add(acc[q][d], v);
                }
        }
        if (!(lane == 31 || next != key)) cx[0] = -1;  // not a segment tail: no flush
    }
};

// ---------------------------------------------------------------------------
// Warp-run deposition (sorted input): the lanes of a warp hold 32 CONSECUTIVE
// particles per round (coalesced 4/8 B loads), so after sorting by cell a round
// almost always lies in one cell.  Every lane accumulates its particles of the
// warp's open cell in 8 x 3 registers; when a round leaves the open cell the 24
// sums are reduced across the warp through shared memory (transposed: lane t < 24
// adds row t = component t of all 32 lanes) and written with ONE 24-lane atomic
// instruction.  Per particle: one all-vote, the CIC weights and 24 FMA; the
// reduction is paid once per cell, not per particle or per lane.  Lanes of a
// round whose cell is neither the open one nor the round's newest cell (unsorted
// input) deposit their own particle with 24 scalar atomics.
// ---------------------------------------------------------------------------
template <typename FP>
struct WarpRunSmem {
    static constexpr int RS = sizeof(FP) == 4 ? 36 : 34;  // row stride (FP): conflict-free
    FP red[24 * RS];
};

template <typename FP>
struct WarpRun {
    FP acc[8][3];
    FP oc[3];   // open cell's unwrapped floor((r - org)/h) (warp-uniform)
    bool open;  // warp-uniform

    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q][0] = acc[q][1] = acc[q][2] = FP(0);
        oc[0] = oc[1] = oc[2] = FP(0);
        open = false;
    }

    // One particle's CIC data: unwrapped cell l, node weights sw (q = (c*2+b)*2+a),
    // and q w v / volume.
    struct Part {
        FP l[3];
        FP sw[8];
        FP qv[3];
    };

    static __device__ __forceinline__ void prepare(const GridArgs<FP> &g, const DepCoef<FP> &t,
                                                   FP half_dt, FP x, FP y, FP z, FP px, FP py,
                                                   FP pz, FP w, Part &p) {
        const FP ux = b_mul(px, t.S), uy = b_mul(py, t.S), uz = b_mul(pz, t.S);
        const FP vf = b_mul(t.inv_Sm, b_rsqrt(b_fma(t.kappa2, b_norm2(ux, uy, uz), FP(1))));
        const FP vx = b_mul(ux, vf), vy = b_mul(uy, vf), vz = b_mul(uz, vf);
        FP f[3];
        p.l[0] = DepositRun<FP>::axis_floor(b_fma(-half_dt, vx, x), g.org[0], g.inv_h[0], f[0]);
        p.l[1] = DepositRun<FP>::axis_floor(b_fma(-half_dt, vy, y), g.org[1], g.inv_h[1], f[1]);
        p.l[2] = DepositRun<FP>::axis_floor(b_fma(-half_dt, vz, z), g.org[2], g.inv_h[2], f[2]);
        const FP qw = b_mul(t.q_vol, w);
        p.qv[0] = b_mul(qw, vx);
        p.qv[1] = b_mul(qw, vy);
        p.qv[2] = b_mul(qw, vz);
        const FP wx[2] = {b_add(FP(1), -f[0]), f[0]};
        const FP wy[2] = {b_add(FP(1), -f[1]), f[1]};
        const FP wz[2] = {b_add(FP(1), -f[2]), f[2]};
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const FP wyz = b_mul(wy[b], wz[c]);
#pragma unroll
                for (int a = 0; a < 2; ++a) p.sw[(c * 2 + b) * 2 + a] = b_mul(wx[a], wyz);
            }
    }

    __device__ __forceinline__ void add(const Part &p) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
            for (int d = 0; d < 3; ++d) acc[q][d] = b_fma(p.sw[q], p.qv[d], acc[q][d]);
    }

    // Nodes of the cell with unwrapped floor l (periodic wrap): corner q = (c*2+b)*2+a
    // is row(b, c) + i[a].
    struct Nodes {
        uint32_t row[4];
        int i[2];
        __device__ __forceinline__ uint32_t operator()(int q) const {
            return row[q >> 1] + (uint32_t)i[q & 1];
        }
    };
    static __device__ __forceinline__ Nodes nodes(const GridArgs<FP> &g, const FP (&l)[3]) {
        Nodes nd;
        int j[2], k[2];
        DepositRun<FP>::axis_wrap(l[0], g.nf[0], g.inv_nf[0], g.n[0], nd.i[0], nd.i[1]);
        DepositRun<FP>::axis_wrap(l[1], g.nf[1], g.inv_nf[1], g.n[1], j[0], j[1]);
        DepositRun<FP>::axis_wrap(l[2], g.nf[2], g.inv_nf[2], g.n[2], k[0], k[1]);
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int b = 0; b < 2; ++b)
                nd.row[c * 2 + b] = ((uint32_t)k[c] * (uint32_t)g.n[1] + (uint32_t)j[b]) *
                                    (uint32_t)g.n[0];
        return nd;
    }

    // Warp-wide: reduce the 24 sums over the lanes and add them to J at the open
    // cell's nodes (one atomic instruction, lanes 0..23); zero the sums.
    __device__ __forceinline__ void flush(const GridArgs<FP> &g, FP *Jx, FP *Jy, FP *Jz,
                                          WarpRunSmem<FP> &sm, int lane) {
        constexpr int RS = WarpRunSmem<FP>::RS;
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                sm.red[(q * 3 + d) * RS + lane] = acc[q][d];
                acc[q][d] = FP(0);
            }
        __syncwarp();
        if (lane < 24) {
            const FP *row = sm.red + lane * RS;
            FP s;
            if constexpr (sizeof(FP) == 4) {
                float4 a = reinterpret_cast<const float4 *>(row)[0];
#pragma unroll
                for (int k = 1; k < 8; ++k) {
                    const float4 v = reinterpret_cast<const float4 *>(row)[k];
                    a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
                }
                s = (a.x + a.y) + (a.z + a.w);
            } else {
                double2 a = reinterpret_cast<const double2 *>(row)[0];
#pragma unroll
                for (int k = 1; k < 16; ++k) {
                    const double2 v = reinterpret_cast<const double2 *>(row)[k];
                    a.x += v.x;
                    a.y += v.y;
                }
                s = a.x + a.y;
            }
            const int q = lane / 3, d = lane - 3 * (lane / 3);
            FP *J = d == 0 ? Jx : (d == 1 ? Jy : Jz);
            if (s != FP(0)) atomicAdd(J + nodes(g, oc)(q), s);
        }
        __syncwarp();
    }

    // One particle straight to J (a lane outside the round's open cells).
    static __device__ __forceinline__ void deposit_single(const GridArgs<FP> &g, const Part &p,
                                                          FP *Jx, FP *Jy, FP *Jz) {
        const Nodes nds = nodes(g, p.l);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t nd = nds(q);
            atomicAdd(Jx + nd, b_mul(p.sw[q], p.qv[0]));
            atomicAdd(Jy + nd, b_mul(p.sw[q], p.qv[1]));
            atomicAdd(Jz + nd, b_mul(p.sw[q], p.qv[2]));
        }
    }

    // One round (all 32 lanes; an invalid lane passes qv = 0 and valid = false).
    __device__ __forceinline__ void round(const GridArgs<FP> &g, const Part &p, bool valid,
                                          FP *Jx, FP *Jy, FP *Jz, WarpRunSmem<FP> &sm,
                                          int lane) {
        const unsigned full = 0xffffffffu;
        const bool in_open =
            !valid || (open && p.l[0] == oc[0] && p.l[1] == oc[1] && p.l[2] == oc[2]);
        if (__all_sync(full, in_open)) {
            add(p);  // invalid lanes add exact zeros
            return;
        }
        if (in_open && valid) add(p);
        if (open) flush(g, Jx, Jy, Jz, sm, lane);
        // the newest cell of the round (highest lane outside the open cell) opens
        const unsigned rest = __ballot_sync(full, !in_open);
        const int leader = 31 - __clz(rest);
        oc[0] = __shfl_sync(full, p.l[0], leader);
        oc[1] = __shfl_sync(full, p.l[1], leader);
        oc[2] = __shfl_sync(full, p.l[2], leader);
        open = true;
        if (!in_open) {
            if (p.l[0] == oc[0] && p.l[1] == oc[1] && p.l[2] == oc[2]) add(p);
            else deposit_single(g, p, Jx, Jy, Jz);
        }
    }
};

}  // namespace boris
