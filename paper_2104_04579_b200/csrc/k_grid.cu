// k_grid.cu -- grid-field support: node packing and the
// periodic particle sort by grid cell ("we have to periodically sort the array
// of particles in order to improve cache locality").
//
// The sort is a stable LSD radix sort of (cell, original index) pairs written
// here (8-bit digits, per-tile histograms, a recursive exclusive scan, and a
// stable per-tile scatter using warp match_any ranks), followed by a gather of
// every particle array through the sorted index.  Stable => particles of one
// cell keep their relative order => the result is deterministic.
#include <vector>

#include <type_traits>

#include "boris_internal.h"
#include "deposit.cuh"

namespace boris {

// ---------------------------------------------------------------------------
// Node packing into x-pair records: record i holds node i and its +x neighbour
// (periodic), 12 FP = [E B](i) [E B](i+1) (grid.cuh kGridStride apart): the CIC
// gather loads a cell's two x-nodes with 3 (fp32) / 6 (fp64) 128-bit loads, 12 per
// particle instead of 16 with one record per node.
// ---------------------------------------------------------------------------
template <typename FP>
__global__ void k_grid_pack(int64_t ncell, int nx, const FP *Ex, const FP *Ey, const FP *Ez,
                            const FP *Bx, const FP *By, const FP *Bz, FP *nodes) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ncell; i += stride) {
        const int64_t ix = i % nx;
        const int64_t i1 = i - ix + (ix + 1 == nx ? 0 : ix + 1);
        FP *r = nodes + kGridStride<FP> * i;
        r[0] = Ex[i];  r[1] = Ey[i];  r[2] = Ez[i];
        r[3] = Bx[i];  r[4] = By[i];  r[5] = Bz[i];
        r[6] = Ex[i1]; r[7] = Ey[i1]; r[8] = Ez[i1];
        r[9] = Bx[i1]; r[10] = By[i1]; r[11] = Bz[i1];
#pragma unroll
        for (int k = kGridRecord; k < kGridStride<FP>; ++k) r[k] = FP(0);  // padding
    }
}

static unsigned grid1d(int64_t n, int threads = 256) {
    int64_t b = (n + threads - 1) / threads;
    if (b > 65535 * 8) b = 65535 * 8;
    return (unsigned)(b > 0 ? b : 1);
}

cudaError_t launch_grid_pack(int precision, int64_t ncell, int nx, const void *const c[6],
                             void *nodes, cudaStream_t st) {
    if (precision == BORIS_FP32)
        k_grid_pack<float><<<grid1d(ncell), 256, 0, st>>>(
            ncell, nx, (const float *)c[0], (const float *)c[1], (const float *)c[2],
            (const float *)c[3], (const float *)c[4], (const float *)c[5], (float *)nodes);
    else
        k_grid_pack<double><<<grid1d(ncell), 256, 0, st>>>(
            ncell, nx, (const double *)c[0], (const double *)c[1], (const double *)c[2],
            (const double *)c[3], (const double *)c[4], (const double *)c[5], (double *)nodes);
    return cudaGetLastError();
}

// SoA permutation by particle records.  A permutation from random order gathers
// every array at random indices; a 4 B gather costs a whole DRAM access, so eight
// separate array gathers moved ~740 B per particle (ncu, 10^7, random order).
// Instead: (1) k_pack_soa writes each particle's present arrays as one record of
// RS FP slots (x y z px py pz [w] [g] [type]) with coalesced reads; (2)
// k_unpack_soa reads record perm[i] (RS adjacent slots: 1-2 sectors) and writes
// slot a to array a at i, coalesced, straight into the ensemble's own arrays (the
// records are the only copy, so no copy-back pass).  From sorted order the record
// reads are sequential too, so the traffic is the same as gather + copy-back.
struct PermPlan {
    void *arr[8];  // present FP arrays in record-slot order
    int nf;        // number of FP slots before the type slot
    int16_t *type; // null: no type slot
    int rs;        // record stride in FP slots
};

static PermPlan perm_plan(const SoaPtrs &s) {
    PermPlan p{};
    void *all[8] = {s.x, s.y, s.z, s.px, s.py, s.pz, s.w, s.g};
    for (int a = 0; a < 8; ++a)
        if (all[a]) p.arr[p.nf++] = all[a];
    p.type = s.type;
    p.rs = p.nf + (s.type ? 1 : 0);
    return p;
}

// Records whose size is a multiple of 16 B (x y z px py pz w g without a type slot)
// are written straight from registers with 16 B vector stores by the first radix
// histogram pass (k_rs_hist<.., PACK>).  Otherwise the records of a 256-particle tile
// are assembled in shared memory (thread t writes
// slots t*RS + a; RS = 9 is odd, so fp32 writes are conflict-free) and leave as
// contiguous 16 B vector stores: every written sector is written whole either way
// (scalar stores at a 36 B lane stride took 3x the time of the traffic).
constexpr int kPackTile = 256;
#ifndef BORIS_UNPACK_VEC
#define BORIS_UNPACK_VEC 1
#endif
#ifndef BORIS_UNPACK_NA
#define BORIS_UNPACK_NA 0
#endif

template <typename FP>
__global__ void __launch_bounds__(kPackTile)
    k_pack_soa(const __grid_constant__ PermPlan p, int64_t n, FP *rec) {
    using W = typename std::conditional<sizeof(FP) == 4, uint32_t, unsigned long long>::type;
    extern __shared__ __align__(16) unsigned char pack_smem[];
    FP *tile = reinterpret_cast<FP *>(pack_smem);
    const int64_t ntiles = (n + kPackTile - 1) / kPackTile;
    const int t = threadIdx.x;
    for (int64_t tb = blockIdx.x; tb < ntiles; tb += gridDim.x) {
        const int64_t i0 = tb * kPackTile;
        const int cnt = (int)(n - i0 < kPackTile ? n - i0 : kPackTile);
        if (t < cnt) {
            const int64_t i = i0 + t;
            FP v[8];
#pragma unroll
            for (int a = 0; a < 8; ++a)
                if (a < p.nf) v[a] = ((const FP *)p.arr[a])[i];
            FP *r = tile + t * p.rs;
#pragma unroll
            for (int a = 0; a < 8; ++a)
                if (a < p.nf) r[a] = v[a];
            if (p.type) reinterpret_cast<W *>(r)[p.nf] = (W)(uint16_t)p.type[i];
        }
        __syncthreads();
        // cnt * rs FP values, contiguous at rec + i0 * rs (16 B aligned: i0 * rs * sizeof(FP)
        // is a multiple of 256 * 4 B)
        const int64_t words = (int64_t)cnt * p.rs;
        const int nvec = (int)(words * sizeof(FP) / 16);
        uint4 *dst = reinterpret_cast<uint4 *>(rec + i0 * p.rs);
        const uint4 *src = reinterpret_cast<const uint4 *>(tile);
        for (int k = t; k < nvec; k += kPackTile) dst[k] = src[k];
        for (int64_t k = (int64_t)nvec * 16 / sizeof(FP) + t; k < words; k += kPackTile)
            rec[i0 * p.rs + k] = tile[k];
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Stable LSD radix sort of the particles' cell keys, digits of up to 10 bits
// (a 64^3 grid's 18-bit keys take 2 passes of 9 bits).  Tile = 256 threads x 8
// keys; in round r thread t owns key tile0 + r*256 + t, so (round, thread) order
// is the original order and the per-tile ranking below keeps it (stable).
// Pass 0 computes the keys from the positions (grid_cell, the gather's own base
// node) while histogramming; its values are the implicit indices i; the last
// pass writes only values (the permutation).
// ---------------------------------------------------------------------------
constexpr int kRsThreads = 256;
constexpr int kRsItems = 8;
constexpr int kRsTile = kRsThreads * kRsItems;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsMaxBits = 10;
constexpr int kRsMaxBins = 1 << kRsMaxBits;

// Histogram of one digit per tile, written digit-major: hist[d * nb + tile].
// KEYS: compute the key of particle i from its position and store it.
// PACK (pass 0, SoA records that are a 16 B multiple): the same threads also write
// each particle's packed record (16 B vector stores), so the permutation's pack
// costs no separate read of the positions and no launch.
template <typename FP, bool KEYS, bool PACK = false>
__global__ void __launch_bounds__(kRsThreads)
    k_rs_hist(EnsView e, const __grid_constant__ GridArgs<FP> g, uint32_t *keys, int64_t n,
              int shift, int bins, uint32_t *hist, int64_t nb,
              const __grid_constant__ PermPlan plan, FP *rec) {
    constexpr int RB = sizeof(FP) == 4 ? BORIS_AOS_RECORD_BYTES_FP32 : BORIS_AOS_RECORD_BYTES_FP64;
    __shared__ uint32_t cnt[kRsMaxBins];
    for (int b = threadIdx.x; b < bins; b += kRsThreads) cnt[b] = 0;
    __syncthreads();
    const uint32_t mask = (uint32_t)bins - 1u;
    const int64_t t0 = (int64_t)blockIdx.x * kRsTile;
    const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
    // warp-aggregated: one shared atomic per distinct digit in the warp (sorted input
    // puts a whole warp in one bin, where per-lane atomics serialise)
    auto count_digit = [&](int d) {
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (d < bins && __popc(peers & lt) == 0) atomicAdd(&cnt[d], (uint32_t)__popc(peers));
    };
    // later passes: all rounds' key loads first, then the warp-synchronous counting
    // (pass 1 hist 33 -> 24 us at 1e7); pass 0 counts per round (measured faster with
    // its position loads and record stores)
    int dg[kRsItems];
#pragma unroll
    for (int r = 0; r < kRsItems; ++r) {
        const int64_t i = t0 + r * kRsThreads + threadIdx.x;
        int d = bins;  // out of range: not counted
        if (i < n) {
            uint32_t key;
            if constexpr (KEYS) {
                FP x, y, z;
                if (e.layout == BORIS_LAYOUT_SOA) {
                    x = ((const FP *)e.soa.x)[i];
                    y = ((const FP *)e.soa.y)[i];
                    z = ((const FP *)e.soa.z)[i];
                } else {
                    const FP *rr = (const FP *)((const unsigned char *)e.aos + i * RB);
                    x = rr[0]; y = rr[1]; z = rr[2];
                }
                key = grid_cell<FP>(g, x, y, z);
                keys[i] = key;
                if constexpr (PACK) {  // plan.arr[0..2] are x, y, z
                    constexpr int V = 16 / sizeof(FP);
                    FP v[8];
                    v[0] = x; v[1] = y; v[2] = z;
#pragma unroll
                    for (int a = 3; a < 8; ++a)
                        if (a < plan.nf) v[a] = ((const FP *)plan.arr[a])[i];
                    uint4 *r = reinterpret_cast<uint4 *>(rec + i * plan.rs);
#pragma unroll
                    for (int k = 0; k < 8 / V; ++k)
                        if (k * V < plan.nf) {
                            uint4 u;
                            memcpy(&u, v + k * V, 16);
                            r[k] = u;
                        }
                }
            } else {
                key = keys[i];
            }
            d = (int)((key >> shift) & mask);
        }
        dg[r] = d;
        if constexpr (KEYS) count_digit(d);  // pass 0: count as the keys arrive
    }
    if constexpr (!KEYS) {
#pragma unroll
        for (int r = 0; r < kRsItems; ++r) count_digit(dg[r]);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < bins; b += kRsThreads)
        hist[(int64_t)b * nb + blockIdx.x] = cnt[b];
}

// Scatter one digit: keys_out may be null (last pass), vals_in null (pass 0: i).
// Warp w of a tile owns the contiguous keys [w*256, (w+1)*256) of the tile, in 8
// rounds of 32, so (warp, round, lane) order is the original order (stable).
// Pass 1: per-warp digit counts (match_any leaders, warp-synchronous).  Pass 2:
// per digit, an exclusive scan over the warps starting at the tile's global
// offset.  Pass 3: every key goes to its warp's running position for its digit.
// Three block barriers per tile.
__global__ void __launch_bounds__(kRsThreads)
    k_rs_scatter(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                 uint32_t *vals_out, int64_t n, int shift, int bins, const uint32_t *offs,
                 int64_t nb) {
    __shared__ uint32_t wc[kRsWarps][kRsMaxBins];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b = threadIdx.x; b < bins; b += kRsThreads)
#pragma unroll
        for (int w = 0; w < kRsWarps; ++w) wc[w][b] = 0;
    __syncthreads();
    const uint32_t mask = (uint32_t)bins - 1u;
    const int64_t w0 = (int64_t)blockIdx.x * kRsTile + (int64_t)warp * (kRsItems * 32);
    const unsigned lt = (1u << lane) - 1u;
    uint32_t key[kRsItems], val[kRsItems];
    unsigned peers[kRsItems];
    int dig[kRsItems];
#pragma unroll
    for (int r = 0; r < kRsItems; ++r) {
        const int64_t i = w0 + r * 32 + lane;
        const bool valid = i < n;
        key[r] = valid ? keys_in[i] : 0u;
        val[r] = valid ? (vals_in ? vals_in[i] : (uint32_t)i) : 0u;
        dig[r] = valid ? (int)((key[r] >> shift) & mask) : bins;
    }
#pragma unroll
    for (int r = 0; r < kRsItems; ++r) {
        peers[r] = __match_any_sync(0xffffffffu, dig[r]);
        if (dig[r] < bins && __popc(peers[r] & lt) == 0) wc[warp][dig[r]] += __popc(peers[r]);
        __syncwarp();
    }
    __syncthreads();
    for (int b = threadIdx.x; b < bins; b += kRsThreads) {
        uint32_t run = offs[(int64_t)b * nb + blockIdx.x];
#pragma unroll
        for (int w = 0; w < kRsWarps; ++w) {
            const uint32_t c = wc[w][b];
            wc[w][b] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRsItems; ++r) {
        const int d = dig[r];
        const int rank = __popc(peers[r] & lt);
        if (d < bins) {
            const uint32_t pos = wc[warp][d] + (uint32_t)rank;
            if (keys_out) keys_out[pos] = key[r];
            vals_out[pos] = val[r];
        }
        __syncwarp();
        if (d < bins && rank == 0) wc[warp][d] += __popc(peers[r]);
        __syncwarp();
    }
}

// Exclusive scan of uint32 (64-bit running totals fit: n < 2^32 particles).
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanChunk = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads)
    k_scan_chunks(uint32_t *data, int64_t len, uint32_t *chunk_tot) {
    // thread sums of 4 items, a warp-shuffle inclusive scan, the 32 warp totals
    // scanned by warp 0: two block barriers
    __shared__ uint32_t s_w[kScanThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t c0 = (int64_t)blockIdx.x * kScanChunk + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems], sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = (c0 + k < len) ? data[c0 + k] : 0u;
        sum += v[k];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += t;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = s_w[lane];  // kScanThreads / 32 == 32 warps
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= off) w += t;
        }
        s_w[lane] = w;
    }
    __syncthreads();
    uint32_t run = inc - sum + (warp > 0 ? s_w[warp - 1] : 0u);  // exclusive prefix
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (c0 + k < len) data[c0 + k] = run;
        run += v[k];
    }
    if (threadIdx.x == kScanThreads - 1 && chunk_tot) chunk_tot[blockIdx.x] = s_w[31];
}

__global__ void k_scan_add(uint32_t *data, int64_t len, const uint32_t *chunk_off) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < len) data[i] += chunk_off[i / kScanChunk];
}

// Single-pass exclusive scan (decoupled look-back): chunks of kScanChunk values are
// scanned in the order of a ticket counter (so every predecessor of a running chunk
// has started: forward progress); a chunk publishes its total (flag 1) and then its
// inclusive prefix (flag 2) in one 64-bit status word, and looks back over its
// predecessors (32 per round, one per lane of warp 0), summing totals until it meets
// an inclusive prefix.  One launch (+ a memset of the status words) instead of the
// chunk / chunk-total / add kernels: 26.5 -> 13.7 us per radix pass on the 2.5 M
// histogram entries of 10^7 particles (one-lane look-back: 21.5), sort 41.5 -> 40.4 ps
// presorted, 78 -> 77 random (profiles/r02/exp_sort_lookback_scan.jsonl).
#ifndef BORIS_SCAN_LOOKBACK
#define BORIS_SCAN_LOOKBACK 1
#endif
// look-back chunks: 16 values per thread (a 10^7-particle histogram of 2.5 M entries
// is 153 chunks, one wave)
#ifndef BORIS_SCAN_LB_ITEMS
#define BORIS_SCAN_LB_ITEMS 16
#endif
constexpr int kLbItems = BORIS_SCAN_LB_ITEMS;
constexpr int kLbChunk = kScanThreads * kLbItems;
__global__ void __launch_bounds__(kScanThreads)
    k_scan_lookback(uint32_t *data, int64_t len, unsigned long long *status, unsigned *ticket) {
    __shared__ uint32_t s_w[kScanThreads / 32];
    __shared__ uint32_t s_chunk, s_excl;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_chunk = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t chunk = s_chunk;
    const int64_t c0 = (int64_t)chunk * kLbChunk + (int64_t)threadIdx.x * kLbItems;
    uint32_t v[kLbItems], sum = 0;
    const bool full = c0 + kLbItems <= len && ((uintptr_t)data & 15u) == 0;  // uint4 access
    if (full) {
#pragma unroll
        for (int k = 0; k < kLbItems / 4; ++k) {
            const uint4 q4 = reinterpret_cast<const uint4 *>(data + c0)[k];
            v[4 * k] = q4.x; v[4 * k + 1] = q4.y; v[4 * k + 2] = q4.z; v[4 * k + 3] = q4.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kLbItems; ++k) v[k] = (c0 + k < len) ? data[c0 + k] : 0u;
    }
#pragma unroll
    for (int k = 0; k < kLbItems; ++k) sum += v[k];
    uint32_t inc = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += t;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = s_w[lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= off) w += t;
        }
        s_w[lane] = w;
        // publish and look back, 32 predecessors per round: lane j reads chunk
        // base - j; the nearest inclusive prefix (flag 2) ends the look-back (the chunk
        // total is s_w[31] = w of lane 31)
        const uint32_t total = __shfl_sync(0xffffffffu, w, 31);
        uint32_t excl = 0;
        if (chunk == 0) {
            if (lane == 0) atomicExch(&status[0], (2ull << 32) | total);
        } else {
            if (lane == 0) atomicExch(&status[chunk], (1ull << 32) | total);
            for (int64_t base = (int64_t)chunk - 1;; base -= 32) {
                const int64_t q = base - lane;
                unsigned long long st = 2ull << 32;  // before chunk 0: inclusive 0
                if (q >= 0) {
                    do {
                        st = *((volatile unsigned long long *)&status[q]);
                    } while ((st >> 32) == 0);
                }
                const unsigned incl = __ballot_sync(0xffffffffu, (st >> 32) == 2);
                const int stop = incl ? __ffs(incl) - 1 : 32;  // nearest inclusive lane
                uint32_t v = lane <= stop ? (uint32_t)st : 0u;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                excl += v;
                if (incl) break;
            }
            if (lane == 0) atomicExch(&status[chunk], (2ull << 32) | (uint32_t)(excl + total));
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    uint32_t run = s_excl + inc - sum + (warp > 0 ? s_w[warp - 1] : 0u);  // exclusive prefix
#pragma unroll
    for (int k = 0; k < kLbItems; ++k) {
        const uint32_t x = v[k];
        v[k] = run;
        run += x;
    }
    if (full) {
#pragma unroll
        for (int k = 0; k < kLbItems / 4; ++k)
            reinterpret_cast<uint4 *>(data + c0)[k] =
                make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < kLbItems; ++k)
            if (c0 + k < len) data[c0 + k] = v[k];
    }
}

static cudaError_t exclusive_scan(uint32_t *data, int64_t len, cudaStream_t st) {
    const int64_t chunks = (len + kScanChunk - 1) / kScanChunk;
    if (chunks <= 1) {
        k_scan_chunks<<<1, kScanThreads, 0, st>>>(data, len, nullptr);
        return cudaGetLastError();
    }
    cudaError_t err;
    if (BORIS_SCAN_LOOKBACK) {
        const int64_t lchunks = (len + kLbChunk - 1) / kLbChunk;
        unsigned long long *status = nullptr;
        const size_t bytes = (size_t)(lchunks + 1) * sizeof(unsigned long long);
        if ((err = scratch_alloc((void **)&status, bytes, st)) != cudaSuccess) return err;
        err = cudaMemsetAsync(status, 0, bytes, st);
        if (err == cudaSuccess) {
            k_scan_lookback<<<(unsigned)lchunks, kScanThreads, 0, st>>>(
                data, len, status, (unsigned *)(status + lchunks));
            err = cudaGetLastError();
        }
        scratch_free(status, st);
        return err;
    }
    uint32_t *tot = nullptr;
    err = scratch_alloc((void **)&tot, (size_t)chunks * sizeof(uint32_t), st);
    if (err != cudaSuccess) return err;
    k_scan_chunks<<<(unsigned)chunks, kScanThreads, 0, st>>>(data, len, tot);
    if ((err = exclusive_scan(tot, chunks, st)) == cudaSuccess) {
        k_scan_add<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(data, len, tot);
        err = cudaGetLastError();
    }
    scratch_free(tot, st);
    return err;
}

// ---------------------------------------------------------------------------
// Permutation: out[i] = in[perm[i]] for every particle array.
// ---------------------------------------------------------------------------
template <int BYTES>
__global__ void k_gather_bytes(const unsigned char *in, unsigned char *out, const uint32_t *perm,
                               int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t j = perm[i];
        if constexpr (BYTES % 4 == 0) {
            const uint32_t *s = (const uint32_t *)(in + j * BYTES);
            uint32_t *d = (uint32_t *)(out + i * BYTES);
#pragma unroll
            for (int k = 0; k < BYTES / 4; ++k) d[k] = s[k];
        } else {
            const unsigned short *s = (const unsigned short *)(in + j * BYTES);
            unsigned short *d = (unsigned short *)(out + i * BYTES);
#pragma unroll
            for (int k = 0; k < BYTES / 2; ++k) d[k] = s[k];
        }
    }
}

// Four particles per thread (i = base + k*256 + tid): 4 x RS independent record
// loads in flight, every store warp-coalesced.
// A record read: __ldg by default; BORIS_UNPACK_NA (L1 no-allocate) measured worse
// from random order (126 vs 112 B of DRAM read per particle, 270 vs 236 us at 1e7).
__device__ __forceinline__ uint4 ld_record(const uint4 *p) {
    uint4 v;
#if BORIS_UNPACK_NA
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
#else
    v = __ldg(p);
#endif
    return v;
}

template <typename FP, bool VEC = false>
__global__ void __launch_bounds__(256)
    k_unpack_soa(const __grid_constant__ PermPlan p, const uint32_t *perm, int64_t n,
                 const FP *rec) {
    using W = typename std::conditional<sizeof(FP) == 4, uint32_t, unsigned long long>::type;
    constexpr int U = 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x * U; base < n; base += stride) {
        int64_t j[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int64_t i = base + k * blockDim.x + threadIdx.x;
            j[k] = i < n ? (int64_t)__ldg(perm + i) : -1;
        }
        FP v[U][8];
        W t[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            if (j[k] < 0) continue;
            const FP *r = rec + j[k] * p.rs;
            if constexpr (VEC) {  // record of nf FP slots, a 16 B multiple, no type slot
                constexpr int V = 16 / sizeof(FP);
#pragma unroll
                for (int h = 0; h < 8 / V; ++h)
                    if (h * V < p.nf) {
                        const uint4 u = ld_record(reinterpret_cast<const uint4 *>(r) + h);
                        memcpy(&v[k][h * V], &u, 16);
                    }
            } else {
#pragma unroll
                for (int a = 0; a < 8; ++a)
                    if (a < p.nf) v[k][a] = __ldg(r + a);
                if (p.type) t[k] = __ldg(reinterpret_cast<const W *>(r) + p.nf);
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            if (j[k] < 0) continue;
            const int64_t i = base + k * blockDim.x + threadIdx.x;
#pragma unroll
            for (int a = 0; a < 8; ++a)
                if (a < p.nf) ((FP *)p.arr[a])[i] = v[k][a];
            if (p.type) p.type[i] = (int16_t)(uint16_t)t[k];
        }
    }
}

template <int BYTES>
static cudaError_t permute_array(void *arr, void *tmp, const uint32_t *perm, int64_t n,
                                 cudaStream_t st) {
    k_gather_bytes<BYTES><<<grid1d(n), 256, 0, st>>>((const unsigned char *)arr,
                                                     (unsigned char *)tmp, perm, n);
    cudaError_t err = cudaGetLastError();
    if (err == cudaSuccess)
        err = cudaMemcpyAsync(arr, tmp, (size_t)n * BYTES, cudaMemcpyDeviceToDevice, st);
    return err;
}

template <typename FP>
cudaError_t sort_by_cell(const EnsView &e, const GridArgs<FP> &g, int /*device*/,
                         cudaStream_t st) {
    const int64_t n = e.n;
    if (n <= 1) return cudaSuccess;
    const uint64_t ncell = (uint64_t)g.n[0] * g.n[1] * g.n[2];
    int bits = 1;
    while (bits < 32 && (1ull << bits) < ncell) ++bits;
    const int passes = (bits + kRsMaxBits - 1) / kRsMaxBits;
    const int dbits = (bits + passes - 1) / passes;  // <= kRsMaxBits
    const int bins = 1 << dbits;
    const int64_t nb = (n + kRsTile - 1) / kRsTile;
    constexpr int RB = sizeof(FP) == 4 ? BORIS_AOS_RECORD_BYTES_FP32 : BORIS_AOS_RECORD_BYTES_FP64;
    const size_t tmp_bytes = e.layout == BORIS_LAYOUT_SOA ? 0 : (size_t)n * RB;
    unsigned char *buf = nullptr;
    const int64_t nn = (n + 63) / 64 * 64;  // 256 B-aligned key/value arrays
    const size_t kv = (size_t)nn * sizeof(uint32_t);
    const size_t hist_bytes = (size_t)bins * nb * sizeof(uint32_t);
    cudaError_t err = scratch_alloc((void **)&buf, 4 * kv + hist_bytes + tmp_bytes + 256, st);
    if (err != cudaSuccess) return err;
    uint32_t *k0 = (uint32_t *)buf, *v0 = k0 + nn, *k1 = v0 + nn, *v1 = k1 + nn;
    uint32_t *hist = v1 + nn;
    unsigned char *tmp = (unsigned char *)(hist + (size_t)bins * nb);
    tmp = (unsigned char *)(((uintptr_t)tmp + 255) & ~(uintptr_t)255);

    // SoA: packed particle records for the permutation (PermPlan); written by the
    // first histogram pass when they are a 16 B multiple, else by k_pack_soa
    const bool soa = e.layout == BORIS_LAYOUT_SOA;
    PermPlan plan{};
    FP *rec = nullptr;
    bool fused_pack = false;
    if (soa) {
        plan = perm_plan(e.soa);
        fused_pack = !plan.type && plan.rs * sizeof(FP) % 16 == 0;
        if ((err = scratch_alloc((void **)&rec, (size_t)n * plan.rs * sizeof(FP), st)) !=
            cudaSuccess) {
            scratch_free(buf, st);
            return err;
        }
    }
    for (int p = 0; p < passes && err == cudaSuccess; ++p) {
        const int shift = dbits * p;
        if (p == 0 && fused_pack)
            k_rs_hist<FP, true, true><<<(unsigned)nb, kRsThreads, 0, st>>>(
                e, g, k0, n, shift, bins, hist, nb, plan, rec);
        else if (p == 0)
            k_rs_hist<FP, true><<<(unsigned)nb, kRsThreads, 0, st>>>(e, g, k0, n, shift, bins,
                                                                   hist, nb, plan, rec);
        else
            k_rs_hist<FP, false><<<(unsigned)nb, kRsThreads, 0, st>>>(e, g, k0, n, shift, bins,
                                                                    hist, nb, plan, rec);
        if ((err = cudaGetLastError()) != cudaSuccess) break;
        if ((err = exclusive_scan(hist, (int64_t)bins * nb, st)) != cudaSuccess) break;
        const bool last = p == passes - 1;
        k_rs_scatter<<<(unsigned)nb, kRsThreads, 0, st>>>(k0, p == 0 ? nullptr : v0,
                                                          last ? nullptr : k1, v1, n, shift,
                                                          bins, hist, nb);
        err = cudaGetLastError();
        uint32_t *t;
        t = k0; k0 = k1; k1 = t;
        t = v0; v0 = v1; v1 = t;
    }
    // v0 = sorted original indices: apply to every particle array
    if (err == cudaSuccess) {
        if (soa) {
            // gather the packed records through the permutation into the arrays
            if (!fused_pack) {
                const size_t smem = (size_t)kPackTile * plan.rs * sizeof(FP);
                k_pack_soa<FP><<<grid1d(n), kPackTile, smem, st>>>(plan, n, rec);
                err = cudaGetLastError();
            }
            if (err == cudaSuccess) {
                if (fused_pack && BORIS_UNPACK_VEC)
                    k_unpack_soa<FP, true><<<grid1d((n + 3) / 4), 256, 0, st>>>(plan, v0, n, rec);
                else
                    k_unpack_soa<FP><<<grid1d((n + 3) / 4), 256, 0, st>>>(plan, v0, n, rec);
                err = cudaGetLastError();
            }
        } else {
            err = permute_array<RB>(e.aos, tmp, v0, n, st);
        }
    }
    if (rec) scratch_free(rec, st);
    scratch_free(buf, st);
    return err;
}

// ---------------------------------------------------------------------------
// Current deposition (reading c-dep): direct CIC deposition
// of q w v^{n+1/2} at r^{n+1/2} = r^{n+1} - (dt/2) v^{n+1/2}, divided by the cell
// volume, with hardware atomics (red.global.add) into the padded, interleaved
// scratch J4 (deposit.cuh), folded into Jx, Jy, Jz at the end.
// ---------------------------------------------------------------------------
template <typename FP>
__global__ void k_fold_j4(const DepOut<FP> o, int nx, int ny, int nz, FP *Jx, FP *Jy, FP *Jz) {
    // component d of node m: fp32 interleaved, fp64 planar
    constexpr bool kPlanar = sizeof(FP) == 8;
    const size_t cs = kPlanar ? o.plane : 1, ns = kPlanar ? 1 : 4;
    const int64_t ncell = (int64_t)nx * ny * nz;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += stride) {
        const int i = (int)(c % nx);
        const int j = (int)((c / nx) % ny);
        const int k = (int)(c / ((int64_t)nx * ny));
        FP sx_ = FP(0), sy_ = FP(0), sz_ = FP(0);
        // the node itself and, on the low faces, its ghost images at i + nx etc.
        for (int cc = 0; cc < (k == 0 ? 2 : 1); ++cc)
            for (int bb = 0; bb < (j == 0 ? 2 : 1); ++bb)
                for (int aa = 0; aa < (i == 0 ? 2 : 1); ++aa) {
                    const FP *p = o.j4 + ns * ((size_t)(k + cc * nz) * o.sxy +
                                               (size_t)(j + bb * ny) * o.sx + (size_t)(i + aa * nx));
                    sx_ = b_add(sx_, p[0]);
                    sy_ = b_add(sy_, p[cs]);
                    sz_ = b_add(sz_, p[2 * cs]);
                }
        Jx[c] = sx_;
        Jy[c] = sy_;
        Jz[c] = sz_;
    }
}

template <typename FP>
cudaError_t dep_scratch_begin(const GridArgs<FP> &g, DepOut<FP> &o, cudaStream_t st) {
    o.sx = (uint32_t)g.n[0] + 1u;
    o.sxy = o.sx * ((uint32_t)g.n[1] + 1u);
    o.plane = o.sxy * ((uint32_t)g.n[2] + 1u);
    const size_t bytes = (size_t)o.plane * (sizeof(FP) == 4 ? 4 : 3) * sizeof(FP);
    o.j4 = nullptr;
    cudaError_t err = scratch_alloc((void **)&o.j4, bytes, st);
    if (err != cudaSuccess) return err;
    err = cudaMemsetAsync(o.j4, 0, bytes, st);
    if (err != cudaSuccess) dep_scratch_free(o, st);
    return err;
}

template <typename FP>
void dep_scratch_free(DepOut<FP> &o, cudaStream_t st) {
    if (o.j4) scratch_free(o.j4, st);
    o.j4 = nullptr;
}

template <typename FP>
cudaError_t dep_scratch_end(const GridArgs<FP> &g, DepOut<FP> &o, void *Jx, void *Jy, void *Jz,
                            cudaStream_t st) {
    const int64_t ncell = (int64_t)g.n[0] * g.n[1] * g.n[2];
    k_fold_j4<FP><<<grid1d(ncell), 256, 0, st>>>(o, g.n[0], g.n[1], g.n[2], (FP *)Jx, (FP *)Jy,
                                                 (FP *)Jz);
    const cudaError_t err = cudaGetLastError();
    dep_scratch_free(o, st);
    return err;
}

template cudaError_t dep_scratch_begin<float>(const GridArgs<float> &, DepOut<float> &,
                                              cudaStream_t);
template cudaError_t dep_scratch_begin<double>(const GridArgs<double> &, DepOut<double> &,
                                               cudaStream_t);
template cudaError_t dep_scratch_end<float>(const GridArgs<float> &, DepOut<float> &, void *,
                                            void *, void *, cudaStream_t);
template cudaError_t dep_scratch_end<double>(const GridArgs<double> &, DepOut<double> &, void *,
                                             void *, void *, cudaStream_t);
template void dep_scratch_free<float>(DepOut<float> &, cudaStream_t);
template void dep_scratch_free<double>(DepOut<double> &, cudaStream_t);

// AoS (any order): one particle per thread; for each corner the lanes holding the
// same node in CONTIGUOUS lanes (the common case for particles sorted by cell) are
// summed with a segmented shuffle scan and only each segment's last lane adds the
// node.  Equal nodes in non-contiguous lanes stay separate segments (still correct).
template <typename FP>
__device__ __forceinline__ void warp_scatter_node(const DepOut<FP> &o, uint32_t node, FP vx,
                                                  FP vy, FP vz) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const uint32_t prev = __shfl_up_sync(full, node, 1);
    const uint32_t next = __shfl_down_sync(full, node, 1);
    const unsigned heads = __ballot_sync(full, lane == 0 || prev != node);
    const int seg = 31 - __clz(heads & (full >> (31 - lane)));  // head lane of my segment
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const FP ax = __shfl_up_sync(full, vx, off);
        const FP ay = __shfl_up_sync(full, vy, off);
        const FP az = __shfl_up_sync(full, vz, off);
        if (lane - off >= seg) {
            vx = b_add(vx, ax);
            vy = b_add(vy, ay);
            vz = b_add(vz, az);
        }
    }
    if ((lane == 31 || next != node) && node != kNoNode) red_node(o, node, vx, vy, vz);
}

template <typename FP>
__global__ void __launch_bounds__(256)
    k_deposit_aos(EnsView e, const __grid_constant__ GridArgs<FP> g,
                  const __grid_constant__ DepCoefs<FP> dc, const DepOut<FP> o) {
    constexpr int RB = sizeof(FP) == 4 ? BORIS_AOS_RECORD_BYTES_FP32 : BORIS_AOS_RECORD_BYTES_FP64;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // whole blocks iterate together so every lane takes part in the warp shuffles
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < e.n; base += stride) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < e.n;
        FP x = FP(0), y = FP(0), z = FP(0), px = FP(0), py = FP(0), pz = FP(0), w = FP(0);
        int ty = 0;
        if (valid) {
            const FP *r = (const FP *)((const unsigned char *)e.aos + i * RB);
            x = r[0]; y = r[1]; z = r[2];
            px = r[3]; py = r[4]; pz = r[5];
            w = r[6];
            ty = *(const int16_t *)(r + 8);
        }
        typename WarpRun<FP>::Part p;
        WarpRun<FP>::prepare(g, dc.t[dc.n_types > 1 ? ty : 0], dc.half_dt, x, y, z, px, py, pz,
                             w, p);
        const uint32_t nb = valid ? base_node(g, o, p.l) : kNoNode;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            warp_scatter_node<FP>(o, valid ? nb + corner(o, q) : kNoNode, b_mul(p.sw[q], p.qv[0]),
                                  b_mul(p.sw[q], p.qv[1]), b_mul(p.sw[q], p.qv[2]));
    }
}

// ---------------------------------------------------------------------------
// Lane-run deposition (fp32 SoA, 16 B-aligned arrays): each lane deposits K = 8
// consecutive particles, loaded with two 128-bit loads per array (a warp's loads
// cover its 256-particle tile contiguously), keeping the 8 nodes x 3 components
// of its current cell in registers and issuing atomics only when the cell
// changes.  For particles sorted by cell (boris_ensemble_sort_by_cell) one flush
// covers a whole run; at the end of a tile the lanes' open cells are merged.
// ---------------------------------------------------------------------------
constexpr int kDepK = 8;            // particles per lane per tile
constexpr int kDepWarps = 8;        // warps per block
constexpr int kDepTile = 32 * kDepK;

#ifndef BORIS_DEP_DIRECT_MINB
#define BORIS_DEP_DIRECT_MINB 2
#endif
#ifndef BORIS_DEP_PREP
#define BORIS_DEP_PREP 1
#endif
// MULTI / HAS_W compile-time: no per-tile default-value moves or predicated loads
// for an absent weight array or type table.
template <bool MULTI, bool HAS_W>
__global__ void __launch_bounds__(kDepWarps * 32, BORIS_DEP_DIRECT_MINB)
    k_deposit_runs(EnsView e, const __grid_constant__ GridArgs<float> g,
                   const __grid_constant__ DepCoefs<float> dc, const DepOut<float> o) {
    __shared__ DepositRun<float>::MergeSmem s_merge[kTransposedMerge<float> ? kDepWarps : 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float *arr[7] = {(const float *)e.soa.x, (const float *)e.soa.y, (const float *)e.soa.z,
                           (const float *)e.soa.px, (const float *)e.soa.py,
                           (const float *)e.soa.pz, (const float *)e.soa.w};
    constexpr bool multi = MULTI;
    const int64_t stride = (int64_t)gridDim.x * kDepWarps * kDepTile;
    for (int64_t base = ((int64_t)blockIdx.x * kDepWarps + warp) * kDepTile; base < e.n;
         base += stride) {
        // lane's K = 8 consecutive particles: two 128-bit loads per array (scalar
        // loads in the ragged last tile)
        float rv[7][kDepK];
        int16_t rty[kDepK];
        const int64_t i0 = base + lane * kDepK;
        if (i0 + kDepK <= e.n) {
#pragma unroll
            for (int a = 0; a < 7; ++a)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float4 v = (a < 6 || HAS_W)
                                         ? __ldg(reinterpret_cast<const float4 *>(arr[a] + i0) + h)
                                         : make_float4(1.f, 1.f, 1.f, 1.f);
                    rv[a][4 * h] = v.x; rv[a][4 * h + 1] = v.y;
                    rv[a][4 * h + 2] = v.z; rv[a][4 * h + 3] = v.w;
                }
            if (multi) {
                const uint4 t4 = __ldg(reinterpret_cast<const uint4 *>(e.soa.type + i0));
                const uint32_t tw[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
                for (int j = 0; j < kDepK; ++j) rty[j] = (int16_t)(tw[j >> 1] >> (16 * (j & 1)));
            }
        } else {
#pragma unroll
            for (int j = 0; j < kDepK; ++j) {
                const int64_t i = i0 + j;
#pragma unroll
                for (int a = 0; a < 7; ++a)
                    rv[a][j] = (i < e.n) ? ((a < 6 || HAS_W) ? arr[a][i] : 1.f) : 0.f;
                rty[j] = (multi && i < e.n) ? e.soa.type[i] : (int16_t)0;
            }
        }
        DepositRun<float> run;
        run.reset();
#if BORIS_DEP_PREP
        if (i0 + kDepK <= e.n) {
            // groups of 4: the four particles' weights first (independent chains),
            // then the cell tests and accumulations
#pragma unroll
            for (int h = 0; h < kDepK; h += 4) {
                DepositRun<float>::Part pp[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    DepositRun<float>::prepare(g, dc.t[multi ? rty[h + j] : 0], dc.half_dt,
                                            rv[0][h + j], rv[1][h + j], rv[2][h + j],
                                            rv[3][h + j], rv[4][h + j], rv[5][h + j],
                                            rv[6][h + j], pp[j]);
#pragma unroll
                for (int j = 0; j < 4; ++j) run.add_part(g, o, pp[j]);
            }
        } else
#endif
#pragma unroll
        for (int j = 0; j < kDepK; ++j) {
            if (i0 + j >= e.n) break;
            run.add(g, o, dc.t[multi ? rty[j] : 0], dc.half_dt, rv[0][j], rv[1][j], rv[2][j],
                    rv[3][j], rv[4][j], rv[5][j], rv[6][j]);
        }
        // end of tile: merge lanes holding the same cell, one atomic set per run
        if constexpr (kTransposedMerge<float>) {
            run.merge_flush(o, s_merge[warp], lane);
        } else {
            run.warp_merge(lane);
            run.flush<true>(o);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Warp-run deposition (fp64, or fp32 with unaligned arrays; deposit.cuh WarpRun):
// each warp owns a contiguous chunk of particles and walks it in rounds of 32
// consecutive particles (lane l takes particle base + l: 4/8 B loads,
// warp-coalesced), PD rounds of loads in flight ahead of the arithmetic (register
// ring).  Sorted by cell, a round almost always lies in the warp's open cell: 24
// FMA per particle, one warp reduction + 8 node atomics per cell.
// ---------------------------------------------------------------------------
#ifndef BORIS_DW_PD
#define BORIS_DW_PD 3
#endif
#ifndef BORIS_DW_MINB
#define BORIS_DW_MINB 2
#endif
template <typename FP>
struct DepWarp {
    static constexpr int WARPS = sizeof(FP) == 4 ? 8 : 4;  // warps per block (static smem)
    static constexpr int PD = BORIS_DW_PD;                  // rounds of loads in flight
    static constexpr int MINB = sizeof(FP) == 4 ? BORIS_DW_MINB : 2;  // blocks per SM
};

template <typename FP, bool MULTI>
__global__ void __launch_bounds__(DepWarp<FP>::WARPS * 32, DepWarp<FP>::MINB)
    k_deposit_warp(EnsView e, const __grid_constant__ GridArgs<FP> g,
                   const __grid_constant__ DepCoefs<FP> dc, const DepOut<FP> o, int64_t chunk) {
    using D = DepWarp<FP>;
    constexpr int PD = D::PD;
    __shared__ WarpRunSmem<FP> sm[D::WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t begin = ((int64_t)blockIdx.x * D::WARPS + warp) * chunk;
    if (begin >= e.n) return;  // warp-uniform; no block barrier follows
    const int64_t end = begin + chunk < e.n ? begin + chunk : e.n;
    FP buf[PD][7];
    int ty[PD];
    // array bases stay in the parameter bank (no pointer registers)
    auto load = [&](int k, int64_t i) {
        const bool ok = i < end;
        buf[k][0] = ok ? __ldg((const FP *)e.soa.x + i) : FP(0);
        buf[k][1] = ok ? __ldg((const FP *)e.soa.y + i) : FP(0);
        buf[k][2] = ok ? __ldg((const FP *)e.soa.z + i) : FP(0);
        buf[k][3] = ok ? __ldg((const FP *)e.soa.px + i) : FP(0);
        buf[k][4] = ok ? __ldg((const FP *)e.soa.py + i) : FP(0);
        buf[k][5] = ok ? __ldg((const FP *)e.soa.pz + i) : FP(0);
        buf[k][6] = ok ? (e.soa.w ? __ldg((const FP *)e.soa.w + i) : FP(1)) : FP(0);  // w = 0: no current
        ty[k] = (MULTI && ok) ? (int)__ldg(e.soa.type + i) : 0;
    };
#pragma unroll
    for (int k = 0; k < PD; ++k) load(k, begin + 32 * k + lane);
    WarpRun<FP> run;
    run.reset();
    for (int64_t base = begin; base < end; base += 32 * PD) {
#pragma unroll
        for (int k = 0; k < PD; ++k) {
            if (base + 32 * k >= end) break;  // warp-uniform
            const int64_t i = base + 32 * k + lane;
            FP v[7];
#pragma unroll
            for (int a = 0; a < 7; ++a) v[a] = buf[k][a];
            const int t = ty[k];
            load(k, i + 32 * PD);
            typename WarpRun<FP>::Part part;
            WarpRun<FP>::prepare(g, dc.t[MULTI ? t : 0], dc.half_dt, v[0], v[1], v[2], v[3],
                                 v[4], v[5], v[6], part);
            run.round(g, o, part, i < end, sm[warp], lane);
        }
    }
    if (run.open) run.flush(g, o, sm[warp], lane);
}

template <typename FP>
static cudaError_t launch_deposit_kernel(const EnsView &e, const GridArgs<FP> &g,
                                         const DepCoefs<FP> &dc, const DepOut<FP> &o, int device,
                                         cudaStream_t st) {
    if (e.n == 0) return cudaSuccess;
    if (e.layout == BORIS_LAYOUT_AOS) {
        const int64_t blocks = (e.n + 255) / 256;
        const unsigned grid = (unsigned)stream_grid(blocks, 8, device);
        k_deposit_aos<FP><<<grid, 256, 0, st>>>(e, g, dc, o);
        return cudaGetLastError();
    }
    // fp32 with 16 B-aligned arrays: lane runs (128-bit loads); fp64 or unaligned:
    // warp runs.  Measured on 10^7 sorted particles, 64^3 grid: fp32 11.0 (lane) vs
    // 13.2 ps (warp), fp64 34.0 (lane, staged tiles) vs 22.5 ps (warp).
    if constexpr (sizeof(FP) == 4) {
        auto al16 = [](const void *q) { return ((uintptr_t)q & 15u) == 0; };
        if (al16(e.soa.x) && al16(e.soa.y) && al16(e.soa.z) && al16(e.soa.px) &&
            al16(e.soa.py) && al16(e.soa.pz) && al16(e.soa.w) && al16(e.soa.type)) {
            const int64_t tiles = (e.n + kDepTile - 1) / kDepTile;
            const int64_t blocks = (tiles + kDepWarps - 1) / kDepWarps;
            const unsigned grid = (unsigned)stream_grid(blocks, 4, device);
            const bool multi = dc.n_types > 1 && e.soa.type, w = e.soa.w != nullptr;
            if (multi)
                w ? k_deposit_runs<true, true><<<grid, kDepWarps * 32, 0, st>>>(e, g, dc, o)
                  : k_deposit_runs<true, false><<<grid, kDepWarps * 32, 0, st>>>(e, g, dc, o);
            else
                w ? k_deposit_runs<false, true><<<grid, kDepWarps * 32, 0, st>>>(e, g, dc, o)
                  : k_deposit_runs<false, false><<<grid, kDepWarps * 32, 0, st>>>(e, g, dc, o);
            return cudaGetLastError();
        }
    }
    // one contiguous chunk per warp, a multiple of 32 particles, sized so the
    // resident blocks cover the ensemble in one wave
    using D = DepWarp<FP>;
    const int64_t warps = (int64_t)sm_count(device) * D::MINB * D::WARPS;
    int64_t chunk = (e.n + warps - 1) / warps;
    chunk = (chunk + 31) / 32 * 32;
    const int64_t blocks = ((e.n + chunk - 1) / chunk + D::WARPS - 1) / D::WARPS;
    if (dc.n_types > 1 && e.soa.type)
        k_deposit_warp<FP, true><<<(unsigned)blocks, D::WARPS * 32, 0, st>>>(e, g, dc, o, chunk);
    else
        k_deposit_warp<FP, false><<<(unsigned)blocks, D::WARPS * 32, 0, st>>>(e, g, dc, o, chunk);
    return cudaGetLastError();
}

template <typename FP>
cudaError_t launch_deposit(const EnsView &e, const GridArgs<FP> &g, const DepCoefs<FP> &dc,
                           void *Jx, void *Jy, void *Jz, int device, cudaStream_t st) {
    DepOut<FP> o;
    cudaError_t err = dep_scratch_begin<FP>(g, o, st);
    if (err != cudaSuccess) return err;
    err = launch_deposit_kernel<FP>(e, g, dc, o, device, st);
    if (err != cudaSuccess) {
        dep_scratch_free<FP>(o, st);
        return err;
    }
    return dep_scratch_end<FP>(g, o, Jx, Jy, Jz, st);
}

template cudaError_t launch_deposit<float>(const EnsView &, const GridArgs<float> &,
                                           const DepCoefs<float> &, void *, void *, void *, int,
                                           cudaStream_t);
template cudaError_t launch_deposit<double>(const EnsView &, const GridArgs<double> &,
                                            const DepCoefs<double> &, void *, void *, void *,
                                            int, cudaStream_t);

template cudaError_t sort_by_cell<float>(const EnsView &, const GridArgs<float> &, int,
                                         cudaStream_t);
template cudaError_t sort_by_cell<double>(const EnsView &, const GridArgs<double> &, int,
                                          cudaStream_t);

}  // namespace boris
