// deposit.cuh -- CIC current deposition helpers (PAPER.md
// L89-92; reading c-dep in DESIGN.md): q w v^{n+1/2} at the half-step position
// r^{n+1/2} = r^{n+1} - (dt/2) v^{n+1/2}, divided by the cell volume, onto the 8
// nodes of the particle's cell.
//
// Target: a padded scratch J4 (DepOut) with one ghost node layer on the +x, +y, +z
// faces: node (i, j, k), 0 <= i <= nx etc., has index (k sy + j) sx + i; fp32
// stores x, y, z, 0 interleaved per node, fp64 three planes.  A cell with base
// node (i0, j0, k0) (wrapped into [0, n)) owns the nodes base + {0, 1} + {0, sx} +
// {0, sxy}: no periodic wrap per corner, and in fp32 one 16 B vector atomic
// (red.global.add.v4.f32) per node instead of three scalar ones.  k_fold_j4
// (k_grid.cu) adds the ghost layers onto their periodic images and writes the
// caller's Jx, Jy, Jz.
//
// Two accumulation schemes share it:
//  * DepositRun (lane runs): a lane deposits consecutive particles, keeping the 8 x 3
//    node sums of its current cell in registers and flushing on a cell change; at
//    the end of a warp tile the lanes' open cells are merged (shuffle scan or
//    transposed through shared memory) so one set of atomics covers each run;
//  * WarpRun (warp runs): the lanes hold 32 consecutive particles per round and
//    accumulate the warp's open cell; a round that leaves it reduces the 24 sums
//    across the warp once.
#pragma once

#include "boris_internal.h"

namespace boris {

constexpr uint32_t kNoNode = 0xFFFFFFFFu;

// End-of-tile merge of the lanes' open cells: shuffle scan (warp_merge + flush) or
// transposed through shared memory (merge_flush; fp32 only, fp64's 24 x 34 doubles
// per warp would exceed static shared memory).  Standalone deposition (kTransposedMerge)
// and the fused PIC step (kTransposedMergePD) can choose separately; both use the
// transposed merge since its walk adds 4-lane groups without a run end as one partial
// sum (standalone 10.5 -> 10.1 ps, PIC 25.8 -> 25.2).
#ifndef BORIS_DEP_MERGE_T
#define BORIS_DEP_MERGE_T 1
#endif
#ifndef BORIS_PD_MERGE_T
#define BORIS_PD_MERGE_T 1
#endif
template <typename FP>
constexpr bool kTransposedMerge = sizeof(FP) == 4 && BORIS_DEP_MERGE_T;
template <typename FP>
constexpr bool kTransposedMergePD = sizeof(FP) == 4 && BORIS_PD_MERGE_T;
// Lane-run sums in moment form (DepositRun; tuning): 1 accumulates q w v times the
// monomials 1, fx, fy, fx fy, fz, fx fz, fy fz, fx fy fz of the particle's in-cell
// offsets (4 products instead of 15 operations for the node weights) and converts the
// run sums to the 8 node sums at each flush / run end (across lanes by shuffles in
// the transposed merge).  Measured slower (10^7 sorted, 64^3: deposition 10.85 vs
// 10.22 ps, fused PIC cycle 28.6 vs 25.3; profiles/r02/exp_deposit_moments.jsonl):
// 0 accumulates q w v times the 8 node weights.
#ifndef BORIS_DEP_MOMENTS
#define BORIS_DEP_MOMENTS 0
#endif
// lanes per group whose 24 sums are added as one partial sum when no run ends in it
#ifndef BORIS_MERGE_GROUP
#define BORIS_MERGE_GROUP 4
#endif

// x, y, z added to J4 node `node`: fp32 nodes are interleaved (x, y, z, 0; one
// 16 B vector reduction), fp64 components are planar (three planes of o.plane
// nodes: three reductions on separate sectors -- interleaved fp64 measured 25 %
// slower on unsorted input, the three reductions serialising on one sector).
__device__ __forceinline__ void red_node(const DepOut<float> &o, uint32_t node, float x, float y,
                                         float z) {
    float *p = o.j4 + 4 * (size_t)node;
    asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(x),
                 "f"(y), "f"(z), "f"(0.f)
                 : "memory");
}
__device__ __forceinline__ void red_node(const DepOut<double> &o, uint32_t node, double x,
                                         double y, double z) {
    double *p = o.j4 + node;
    atomicAdd(p, x);
    atomicAdd(p + o.plane, y);
    atomicAdd(p + 2 * (size_t)o.plane, z);
}

// Per-axis CIC pieces: the unwrapped floor l and weight f of the upper node (every
// particle), and l wrapped into [0, n) (only when the cell changes).
template <typename FP>
__device__ __forceinline__ FP axis_floor(FP x, FP org, FP inv_h, FP &f) {
    const FP xi = b_mul(b_add(x, -org), inv_h);
    const FP l = floor(xi);
    f = b_add(xi, -l);  // exact, in [0, 1)
    return l;
}
template <typename FP>
__device__ __forceinline__ uint32_t axis_wrap(FP l, FP nf, FP inv_nf, int n) {
    const FP w = b_fma(-nf, floor(b_mul(l, inv_nf)), l);  // l mod n, up to +-1 rounding
    int i = (int)w;
    if (i >= n) i -= n;
    if (i < 0) i += n;
    return (uint32_t)i;
}
// J4 node index of the base node of the cell with unwrapped floor l.
template <typename FP>
__device__ __forceinline__ uint32_t base_node(const GridArgs<FP> &g, const DepOut<FP> &o,
                                              const FP (&l)[3]) {
    return axis_wrap(l[2], g.nf[2], g.inv_nf[2], g.n[2]) * o.sxy +
           axis_wrap(l[1], g.nf[1], g.inv_nf[1], g.n[1]) * o.sx +
           axis_wrap(l[0], g.nf[0], g.inv_nf[0], g.n[0]);
}
// Corner q = (c*2 + b)*2 + a of a cell relative to its base node.
template <typename FP>
__device__ __forceinline__ uint32_t corner(const DepOut<FP> &o, int q) {
    return ((q >> 2) ? o.sxy : 0u) + (((q >> 1) & 1) ? o.sx : 0u) + (uint32_t)(q & 1);
}
// Adds s[q][d] to the 8 nodes of the cell at base node nb.
template <typename FP>
__device__ __forceinline__ void red_cell(const DepOut<FP> &o, uint32_t nb, const FP (&s)[8][3]) {
#pragma unroll
    for (int q = 0; q < 8; ++q) red_node(o, nb + corner(o, q), s[q][0], s[q][1], s[q][2]);
}

template <typename FP>
struct DepositRun {
    FP acc[8][3];  // BORIS_DEP_MOMENTS: moment k = (kz*2 + ky)*2 + kx sums; else node q sums
    uint32_t nb;  // J4 base node of the open cell (kNoNode: none)
    FP fl[3];     // the open cell's unwrapped floor((r - org)/h)

    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q][0] = acc[q][1] = acc[q][2] = FP(0);
        nb = kNoNode;
        fl[0] = fl[1] = fl[2] = FP(0);
    }

    // Moment sums -> node sums (in place): per axis, node (offset 0) = M(1) - M(f) and
    // node (offset 1) = M(f), since the CIC weights are (1 - f, f) (reading c-dep);
    // node q = (c*2 + b)*2 + a as corner().
    __device__ __forceinline__ void to_nodes() {
#if BORIS_DEP_MOMENTS
#pragma unroll
        for (int sb = 1; sb < 8; sb <<= 1)
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (!(k & sb))
#pragma unroll
                    for (int d = 0; d < 3; ++d) acc[k][d] = b_add(acc[k][d], -acc[k | sb][d]);
#endif
    }

    // Atomics for the open cell (if any), then zero the sums (LAST: the run ends
    // here and is reset before any reuse, so the sums are left as they are).
    template <bool LAST = false>
    __device__ __forceinline__ void flush(const DepOut<FP> &o) {
        if (nb == kNoNode) return;
        to_nodes();
        red_cell(o, nb, acc);
        if constexpr (!LAST) {
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q][0] = acc[q][1] = acc[q][2] = FP(0);
        }
    }

    // One particle's CIC data: unwrapped cell l, in-cell offsets f and their
    // products (moments) or the 8 node weights, and q w v / cell volume.
    struct Part {
        FP l[3];
        FP m[8];  // moments: 1 (unused), fx, fy, fx fy, fz, fx fz, fy fz, fx fy fz; or weights
        FP qv[3];
    };

    // State after the push: r^{n+1}, p^{n+1/2}, weight w (reading c-dep: r^{n+1/2} =
    // r^{n+1} - (dt/2) v^{n+1/2}).
    static __device__ __forceinline__ void prepare(const GridArgs<FP> &g, const DepCoef<FP> &t,
                                                   FP half_dt, FP x, FP y, FP z, FP px, FP py,
                                                   FP pz, FP w, Part &p) {
        const FP ux = b_mul(px, t.S), uy = b_mul(py, t.S), uz = b_mul(pz, t.S);
        const FP vf = b_mul(t.inv_Sm, b_rsqrt(b_fma(t.kappa2, b_norm2(ux, uy, uz), FP(1))));
        const FP vx = b_mul(ux, vf), vy = b_mul(uy, vf), vz = b_mul(uz, vf);
        FP f[3];
        p.l[0] = axis_floor(b_fma(-half_dt, vx, x), g.org[0], g.inv_h[0], f[0]);
        p.l[1] = axis_floor(b_fma(-half_dt, vy, y), g.org[1], g.inv_h[1], f[1]);
        p.l[2] = axis_floor(b_fma(-half_dt, vz, z), g.org[2], g.inv_h[2], f[2]);
        const FP qw = b_mul(t.q_vol, w);
        p.qv[0] = b_mul(qw, vx);
        p.qv[1] = b_mul(qw, vy);
        p.qv[2] = b_mul(qw, vz);
#if BORIS_DEP_MOMENTS
        p.m[0] = FP(1);
        p.m[1] = f[0];
        p.m[2] = f[1];
        p.m[3] = b_mul(f[0], f[1]);
        p.m[4] = f[2];
        p.m[5] = b_mul(f[0], f[2]);
        p.m[6] = b_mul(f[1], f[2]);
        p.m[7] = b_mul(p.m[3], f[2]);
#else
        const FP wx[2] = {b_add(FP(1), -f[0]), f[0]};
        const FP wy[2] = {b_add(FP(1), -f[1]), f[1]};
        const FP wz[2] = {b_add(FP(1), -f[2]), f[2]};
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const FP wyz = b_mul(wy[b], wz[c]);
#pragma unroll
                for (int a = 0; a < 2; ++a) p.m[(c * 2 + b) * 2 + a] = b_mul(wx[a], wyz);
            }
#endif
    }

    // One particle (state after the push).
    __device__ __forceinline__ void add(const GridArgs<FP> &g, const DepOut<FP> &o,
                                        const DepCoef<FP> &t, FP half_dt, FP x, FP y, FP z,
                                        FP px, FP py, FP pz, FP w) {
        Part p;
        prepare(g, t, half_dt, x, y, z, px, py, pz, w, p);
        add_part(g, o, p);
    }

    // One prepared particle: the cell test and the 24 accumulations only, so a caller
    // can prepare several particles first (independent chains) and accumulate them after.
    __device__ __forceinline__ void add_part(const GridArgs<FP> &g, const DepOut<FP> &o,
                                             const Part &p) {
        // same unwrapped cell -> same nodes; a periodic image of the open cell only
        // costs an extra flush
        if (nb == kNoNode || p.l[0] != fl[0] || p.l[1] != fl[1] || p.l[2] != fl[2]) {
            flush(o);
            fl[0] = p.l[0]; fl[1] = p.l[1]; fl[2] = p.l[2];
            nb = base_node(g, o, p.l);
        }
#pragma unroll
        for (int d = 0; d < 3; ++d)
            acc[0][d] = BORIS_DEP_MOMENTS ? b_add(acc[0][d], p.qv[d])
                                          : b_fma(p.m[0], p.qv[d], acc[0][d]);
#pragma unroll
        for (int q = 1; q < 8; ++q)
#pragma unroll
            for (int d = 0; d < 3; ++d) acc[q][d] = b_fma(p.m[q], p.qv[d], acc[q][d]);
    }

    // End of a warp tile (all 32 lanes): lanes holding the same open cell in
    // consecutive lanes (contiguous when sorted) are summed with a segmented
    // scan; every lane but each segment's last drops its cell, so the following
    // flush() issues one set of atomics per segment.
    __device__ __forceinline__ void warp_merge(int lane) {
        const unsigned full = 0xffffffffu;
        const uint32_t key = nb;
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
        if (!(lane == 31 || next != key)) nb = kNoNode;  // not a segment tail: no flush
    }

    // Per-warp scratch of merge_flush.
    struct MergeSmem {
        static constexpr int RS = sizeof(FP) == 4 ? 36 : 34;  // row stride: conflict-free
        FP red[24 * RS];   // red[t * RS + l] = lane l's sum t = q * 3 + d
        uint32_t nbs[32];  // lane l's open cell (base node)
    };

    // End of a warp tile (all 32 lanes; the run ends), transposed: every lane stashes its 24 sums
    // in shared memory, then lane t < 24 walks component t of the 32 lanes in lane
    // order and closes each run of equal open cells (contiguous when sorted) at its
    // last lane, where lanes 3q..3q+2 pass their components to lane 3q for one node
    // reduction -- one 8-lane vector atomic per run instead of a shuffle scan over
    // the 24 sums.  The run ends (tails) are warp-uniform: no divergent branches.
    __device__ __forceinline__ void merge_flush(const DepOut<FP> &o, MergeSmem &sm, int lane) {
        const unsigned full = 0xffffffffu;
        const bool has = nb != kNoNode;
        const uint32_t next = __shfl_down_sync(full, nb, 1);
        const unsigned tails = __ballot_sync(full, has && (lane == 31 || next != nb));
        if (tails == 0) return;
        constexpr int RS = MergeSmem::RS;
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
            for (int d = 0; d < 3; ++d) sm.red[(q * 3 + d) * RS + lane] = acc[q][d];
        sm.nbs[lane] = nb;
        nb = kNoNode;  // the run ends: reset() before reuse (the sums are left)
        __syncwarp();
        const int t = lane < 24 ? lane : 23;  // lanes 24..31 shadow lane 23 (no atomics)
        const int q = t / 3, d = t - 3 * (t / 3);
        const FP *row = sm.red + t * RS;
        FP run = FP(0);
        constexpr int VW = 16 / sizeof(FP);  // FP per 16 B vector
        constexpr int GV = BORIS_MERGE_GROUP / VW;  // vectors per tested group
#pragma unroll
        for (int g0 = 0; g0 < 32; g0 += GV * VW) {
            FP v[GV][VW];
#pragma unroll
            for (int gv = 0; gv < GV; ++gv) {
                const int l0 = g0 + gv * VW;
                if constexpr (VW == 4) {
                    const float4 w = reinterpret_cast<const float4 *>(row)[l0 / 4];
                    v[gv][0] = w.x; v[gv][1] = w.y; v[gv][2] = w.z; v[gv][3] = w.w;
                } else {
                    const double2 w = reinterpret_cast<const double2 *>(row)[l0 / 2];
                    v[gv][0] = w.x; v[gv][1] = w.y;
                }
            }
            // no run ends in this group of lanes (warp-uniform): one partial sum
            if (((tails >> g0) & ((1u << (GV * VW)) - 1u)) == 0) {
                FP gsum = FP(0);
#pragma unroll
                for (int gv = 0; gv < GV; ++gv) {
                    FP vs = v[gv][0];
#pragma unroll
                    for (int k = 1; k < VW; ++k) vs = b_add(vs, v[gv][k]);
                    gsum = gv == 0 ? vs : b_add(gsum, vs);
                }
                run = b_add(run, gsum);
                continue;
            }
#pragma unroll
            for (int gv = 0; gv < GV; ++gv)
#pragma unroll
                for (int k = 0; k < VW; ++k) {
                    const int l = g0 + gv * VW + k;
                    run = b_add(run, v[gv][k]);
                    if (tails & (1u << l)) {  // warp-uniform
#if BORIS_DEP_MOMENTS
                        // lane 3k + d holds moment k of component d: to node sums
                        // (to_nodes across the lanes)
#pragma unroll
                        for (int sb = 1; sb < 8; sb <<= 1) {
                            const FP other = __shfl_sync(full, run, 3 * (q ^ sb) + d);
                            if (!(q & sb)) run = b_add(run, -other);
                        }
#endif
                        const FP ry = __shfl_down_sync(full, run, 1);
                        const FP rz = __shfl_down_sync(full, run, 2);
                        if (lane < 24 && d == 0)
                            red_node(o, sm.nbs[l] + corner(o, q), run, ry, rz);
                        run = FP(0);
                    }
                }
        }
        __syncwarp();
    }
};

// ---------------------------------------------------------------------------
// Warp-run deposition (sorted input): the lanes of a warp hold 32 CONSECUTIVE
// particles per round (coalesced 4/8 B loads), so after sorting by cell a round
// almost always lies in one cell.  Every lane accumulates its particles of the
// warp's open cell in 8 x 3 registers; when a round leaves the open cell the 24
// sums are reduced across the warp through shared memory (transposed: lane t < 24
// adds row t = component t of all 32 lanes) and lanes 0, 3, .., 21 add one node
// each.  Per particle: one all-vote, the CIC weights and 24 FMA; the reduction is
// paid once per cell, not per particle or per lane.  Lanes of a round whose cell
// is neither the open one nor the round's newest cell (unsorted input) deposit
// their own particle directly.
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
        p.l[0] = axis_floor(b_fma(-half_dt, vx, x), g.org[0], g.inv_h[0], f[0]);
        p.l[1] = axis_floor(b_fma(-half_dt, vy, y), g.org[1], g.inv_h[1], f[1]);
        p.l[2] = axis_floor(b_fma(-half_dt, vz, z), g.org[2], g.inv_h[2], f[2]);
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

    // Warp-wide: reduce the 24 sums over the lanes and add them to the open cell's
    // nodes (lane 3q adds node q with its neighbours' components); zero the sums.
    __device__ __forceinline__ void flush(const GridArgs<FP> &g, const DepOut<FP> &o,
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
        const int t = lane < 24 ? lane : 23;
        const FP *row = sm.red + t * RS;
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
        const FP sy = __shfl_down_sync(0xffffffffu, s, 1);
        const FP sz = __shfl_down_sync(0xffffffffu, s, 2);
        const int q = t / 3;
        if (lane < 24 && lane == 3 * q)
            red_node(o, base_node(g, o, oc) + corner(o, q), s, sy, sz);
        __syncwarp();
    }

    // One particle straight to J4 (a lane outside the round's open cells).
    static __device__ __forceinline__ void deposit_single(const GridArgs<FP> &g,
                                                          const DepOut<FP> &o, const Part &p) {
        FP s[8][3];
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
            for (int d = 0; d < 3; ++d) s[q][d] = b_mul(p.sw[q], p.qv[d]);
        red_cell(o, base_node(g, o, p.l), s);
    }

    // One round (all 32 lanes; an invalid lane passes qv = 0 and valid = false).
    __device__ __forceinline__ void round(const GridArgs<FP> &g, const DepOut<FP> &o,
                                          const Part &p, bool valid, WarpRunSmem<FP> &sm,
                                          int lane) {
        const unsigned full = 0xffffffffu;
        const bool in_open =
            !valid || (open && p.l[0] == oc[0] && p.l[1] == oc[1] && p.l[2] == oc[2]);
        if (__all_sync(full, in_open)) {
            add(p);  // invalid lanes add exact zeros
            return;
        }
        if (in_open && valid) add(p);
        if (open) flush(g, o, sm, lane);
        // the newest cell of the round (highest lane outside the open cell) opens
        const unsigned rest = __ballot_sync(full, !in_open);
        const int leader = 31 - __clz(rest);
        oc[0] = __shfl_sync(full, p.l[0], leader);
        oc[1] = __shfl_sync(full, p.l[1], leader);
        oc[2] = __shfl_sync(full, p.l[2], leader);
        open = true;
        if (!in_open) {
            if (p.l[0] == oc[0] && p.l[1] == oc[1] && p.l[2] == oc[2]) add(p);
            else deposit_single(g, o, p);
        }
    }
};

}  // namespace boris
