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
// (periodic), 12 FP = [E B](i) [E B](i+1): the CIC gather loads a cell's two
// x-nodes with 3 (fp32) / 6 (fp64) 128-bit loads, 12 per particle instead of 16.
// ---------------------------------------------------------------------------
template <typename FP>
__global__ void k_grid_pack(int64_t ncell, int nx, const FP *Ex, const FP *Ey, const FP *Ez,
                            const FP *Bx, const FP *By, const FP *Bz, FP *nodes) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ncell; i += stride) {
        const int64_t ix = i % nx;
        const int64_t i1 = i - ix + (ix + 1 == nx ? 0 : ix + 1);
        FP *r = nodes + kGridRecord * i;
        r[0] = Ex[i];  r[1] = Ey[i];  r[2] = Ez[i];
        r[3] = Bx[i];  r[4] = By[i];  r[5] = Bz[i];
        r[6] = Ex[i1]; r[7] = Ey[i1]; r[8] = Ez[i1];
        r[9] = Bx[i1]; r[10] = By[i1]; r[11] = Bz[i1];
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
template <typename FP, bool KEYS>
__global__ void __launch_bounds__(kRsThreads)
    k_rs_hist(EnsView e, const __grid_constant__ GridArgs<FP> g, uint32_t *keys, int64_t n,
              int shift, int bins, uint32_t *hist, int64_t nb) {
    constexpr int RB = sizeof(FP) == 4 ? BORIS_AOS_RECORD_BYTES_FP32 : BORIS_AOS_RECORD_BYTES_FP64;
    __shared__ uint32_t cnt[kRsMaxBins];
    for (int b = threadIdx.x; b < bins; b += kRsThreads) cnt[b] = 0;
    __syncthreads();
    const uint32_t mask = (uint32_t)bins - 1u;
    const int64_t t0 = (int64_t)blockIdx.x * kRsTile;
    const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
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
            } else {
                key = keys[i];
            }
            d = (int)((key >> shift) & mask);
        }
        // warp-aggregated: one shared atomic per distinct digit in the warp (sorted
        // input puts a whole warp in one bin, where per-lane atomics serialise)
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (d < bins && __popc(peers & lt) == 0) atomicAdd(&cnt[d], (uint32_t)__popc(peers));
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
    __shared__ uint32_t s[kScanThreads];
    const int64_t c0 = (int64_t)blockIdx.x * kScanChunk + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems], sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = (c0 + k < len) ? data[c0 + k] : 0u;
        sum += v[k];
    }
    s[threadIdx.x] = sum;
    __syncthreads();
    for (int off = 1; off < kScanThreads; off <<= 1) {  // Hillis-Steele inclusive
        const uint32_t add = threadIdx.x >= (unsigned)off ? s[threadIdx.x - off] : 0u;
        __syncthreads();
        s[threadIdx.x] += add;
        __syncthreads();
    }
    uint32_t run = s[threadIdx.x] - sum;  // exclusive prefix of this thread
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (c0 + k < len) data[c0 + k] = run;
        run += v[k];
    }
    if (threadIdx.x == kScanThreads - 1 && chunk_tot) chunk_tot[blockIdx.x] = s[threadIdx.x];
}

__global__ void k_scan_add(uint32_t *data, int64_t len, const uint32_t *chunk_off) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < len) data[i] += chunk_off[i / kScanChunk];
}

static cudaError_t exclusive_scan(uint32_t *data, int64_t len, cudaStream_t st) {
    const int64_t chunks = (len + kScanChunk - 1) / kScanChunk;
    if (chunks <= 1) {
        k_scan_chunks<<<1, kScanThreads, 0, st>>>(data, len, nullptr);
        return cudaGetLastError();
    }
    uint32_t *tot = nullptr;
    cudaError_t err = scratch_alloc((void **)&tot, (size_t)chunks * sizeof(uint32_t), st);
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
// are written straight from registers with 16 B vector stores.  Otherwise the
// records of a 256-particle tile are assembled in shared memory (thread t writes
// slots t*RS + a; RS = 9 is odd, so fp32 writes are conflict-free) and leave as
// contiguous 16 B vector stores: every written sector is written whole either way
// (scalar stores at a 36 B lane stride took 3x the time of the traffic).
constexpr int kPackTile = 256;

template <typename FP>
__global__ void __launch_bounds__(kPackTile)
    k_pack_soa_vec(const __grid_constant__ PermPlan p, int64_t n, FP *rec) {
    constexpr int V = 16 / sizeof(FP);  // FP per 16 B vector
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        FP v[8];
#pragma unroll
        for (int a = 0; a < 8; ++a)
            if (a < p.nf) v[a] = ((const FP *)p.arr[a])[i];
        uint4 *r = reinterpret_cast<uint4 *>(rec + i * p.rs);
#pragma unroll
        for (int k = 0; k < 8 / V; ++k)
            if (k * V < p.nf) {
                uint4 u;
                memcpy(&u, v + k * V, 16);
                r[k] = u;
            }
    }
}

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

// Four particles per thread (i = base + k*256 + tid): 4 x RS independent record
// loads in flight, every store warp-coalesced.
template <typename FP>
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
#pragma unroll
            for (int a = 0; a < 8; ++a)
                if (a < p.nf) v[k][a] = __ldg(r + a);
            if (p.type) t[k] = __ldg(reinterpret_cast<const W *>(r) + p.nf);
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

    for (int p = 0; p < passes && err == cudaSuccess; ++p) {
        const int shift = dbits * p;
        if (p == 0)
            k_rs_hist<FP, true><<<(unsigned)nb, kRsThreads, 0, st>>>(e, g, k0, n, shift, bins,
                                                                   hist, nb);
        else
            k_rs_hist<FP, false><<<(unsigned)nb, kRsThreads, 0, st>>>(e, g, k0, n, shift, bins,
                                                                    hist, nb);
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
        if (e.layout == BORIS_LAYOUT_SOA) {
            // pack records, then gather them through the permutation into the arrays
            const PermPlan plan = perm_plan(e.soa);
            FP *rec = nullptr;
            err = scratch_alloc((void **)&rec, (size_t)n * plan.rs * sizeof(FP), st);
            if (err == cudaSuccess) {
                const size_t smem = (size_t)kPackTile * plan.rs * sizeof(FP);
                if (!plan.type && plan.rs * sizeof(FP) % 16 == 0)
                    k_pack_soa_vec<FP><<<grid1d(n), kPackTile, 0, st>>>(plan, n, rec);
                else
                    k_pack_soa<FP><<<grid1d(n), kPackTile, smem, st>>>(plan, n, rec);
                err = cudaGetLastError();
                if (err == cudaSuccess) {
                    k_unpack_soa<FP><<<grid1d((n + 3) / 4), 256, 0, st>>>(plan, v0, n, rec);
                    err = cudaGetLastError();
                }
                scratch_free(rec, st);
            }
        } else {
            err = permute_array<RB>(e.aos, tmp, v0, n, st);
        }
    }
    scratch_free(buf, st);
    return err;
}

// ---------------------------------------------------------------------------
// Current deposition (reading c-dep): direct CIC deposition
// of q w v^{n+1/2} at r^{n+1/2} = r^{n+1} - (dt/2) v^{n+1/2}, divided by the cell
// volume, with hardware float/double atomics (red.global.add) into J.
// ---------------------------------------------------------------------------
// Warp-aggregated scatter: lanes holding the same node in CONTIGUOUS lanes (the
// common case for particles sorted by cell) are summed with a segmented shuffle
// scan and only each segment's last lane issues the atomics.  Equal nodes in
// non-contiguous lanes simply stay separate segments (still correct).

template <typename FP>
__device__ __forceinline__ void warp_scatter_add(uint32_t node, FP vx, FP vy, FP vz, FP *Jx,
                                                 FP *Jy, FP *Jz) {
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
    if ((lane == 31 || next != node) && node != kNoNode) {
        atomicAdd(Jx + node, vx);
        atomicAdd(Jy + node, vy);
        atomicAdd(Jz + node, vz);
    }
}

template <typename FP>
__global__ void __launch_bounds__(256)
    k_deposit(EnsView e, const __grid_constant__ GridArgs<FP> g,
              const __grid_constant__ DepCoefs<FP> dc, FP *Jx, FP *Jy, FP *Jz) {
    constexpr int RB = sizeof(FP) == 4 ? BORIS_AOS_RECORD_BYTES_FP32 : BORIS_AOS_RECORD_BYTES_FP64;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // whole blocks iterate together so every lane takes part in the warp shuffles
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < e.n; base += stride) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < e.n;
        FP x = FP(0), y = FP(0), z = FP(0), px = FP(0), py = FP(0), pz = FP(0), w = FP(0);
        int ty = 0;
        if (valid) {
            if (e.layout == BORIS_LAYOUT_SOA) {
                x = ((const FP *)e.soa.x)[i];
                y = ((const FP *)e.soa.y)[i];
                z = ((const FP *)e.soa.z)[i];
                px = ((const FP *)e.soa.px)[i];
                py = ((const FP *)e.soa.py)[i];
                pz = ((const FP *)e.soa.pz)[i];
                w = e.soa.w ? ((const FP *)e.soa.w)[i] : FP(1);
                if (e.soa.type) ty = e.soa.type[i];
            } else {
                const FP *r = (const FP *)((const unsigned char *)e.aos + i * RB);
                x = r[0]; y = r[1]; z = r[2];
                px = r[3]; py = r[4]; pz = r[5];
                w = r[6];
                ty = *(const int16_t *)(r + 8);
            }
        }
        const DepCoef<FP> t = dc.t[dc.n_types > 1 ? ty : 0];
        const FP ux = b_mul(px, t.S), uy = b_mul(py, t.S), uz = b_mul(pz, t.S);
        // v = p/(gamma m) = u/(S m gamma)
        const FP vf = b_mul(t.inv_Sm, b_rsqrt(b_fma(t.kappa2, b_norm2(ux, uy, uz), FP(1))));
        const FP vx = b_mul(ux, vf), vy = b_mul(uy, vf), vz = b_mul(uz, vf);
        // half-step position
        const FP xh = b_fma(-dc.half_dt, vx, x), yh = b_fma(-dc.half_dt, vy, y),
                 zh = b_fma(-dc.half_dt, vz, z);
        int ix[2], iy[2], iz[2];
        FP fx, fy, fz;
        grid_axis<FP>(xh, g.org[0], g.inv_h[0], g.nf[0], g.inv_nf[0], g.n[0], ix[0], ix[1], fx);
        grid_axis<FP>(yh, g.org[1], g.inv_h[1], g.nf[1], g.inv_nf[1], g.n[1], iy[0], iy[1], fy);
        grid_axis<FP>(zh, g.org[2], g.inv_h[2], g.nf[2], g.inv_nf[2], g.n[2], iz[0], iz[1], fz);
        const FP wx[2] = {b_add(FP(1), -fx), fx};
        const FP wy[2] = {b_add(FP(1), -fy), fy};
        const FP wz[2] = {b_add(FP(1), -fz), fz};
        const FP qw = b_mul(t.q_vol, w);
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const FP wyz = b_mul(qw, b_mul(wy[b], wz[c]));
                const uint32_t row =
                    ((uint32_t)iz[c] * (uint32_t)g.n[1] + (uint32_t)iy[b]) * (uint32_t)g.n[0];
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const FP s = b_mul(wx[a], wyz);
                    const uint32_t node = valid ? row + (uint32_t)ix[a] : kNoNode;
                    warp_scatter_add<FP>(node, b_mul(s, vx), b_mul(s, vy), b_mul(s, vz), Jx, Jy,
                                         Jz);
                }
            }
    }
}

// ---------------------------------------------------------------------------
// Run-accumulating deposition (SoA): each lane deposits K consecutive particles,
// keeping the 8 nodes x 3 components of its current cell in registers and
// issuing atomics only when the cell changes.  For particles sorted by cell
// (boris_ensemble_sort_by_cell) one flush covers a whole run.  Warp tiles are
// staged through shared memory with coalesced loads and a skewed layout
// (p -> p + p/K) so the per-lane sequential reads are bank-conflict free.
// ---------------------------------------------------------------------------
template <typename FP>
struct DepRuns {
    static constexpr int K = 8;          // particles per lane per tile
    static constexpr int WARPS = sizeof(FP) == 4 ? 4 : 2;  // <= 48 KB static smem
    static constexpr int TILE = 32 * K;  // particles per warp tile
    static constexpr int SK = TILE + TILE / K;
};

// fp32 with 16 B-aligned arrays: DIRECT (no shared-memory staging; each lane
// loads its K = 8 consecutive particles with two 128-bit loads per array, a
// warp's loads cover the tile contiguously).  fp64 or unaligned: staged tiles.
#ifndef BORIS_DEP_PREFETCH
#define BORIS_DEP_PREFETCH 0
#endif
#ifndef BORIS_DEP_DIRECT_MINB
#define BORIS_DEP_DIRECT_MINB (BORIS_DEP_PREFETCH ? 1 : 2)
#endif
template <typename FP, bool DIRECT>
__global__ void __launch_bounds__((DIRECT ? 8 : DepRuns<FP>::WARPS) * 32,
                                  DIRECT ? BORIS_DEP_DIRECT_MINB : 6)
    k_deposit_runs(EnsView e, const __grid_constant__ GridArgs<FP> g,
                   const __grid_constant__ DepCoefs<FP> dc, FP *Jx, FP *Jy, FP *Jz) {
    using R = DepRuns<FP>;
    constexpr int NW = DIRECT ? 8 : R::WARPS;
    __shared__ FP s[DIRECT ? 1 : R::WARPS][7][DIRECT ? 1 : R::SK];
    __shared__ int16_t s_ty[DIRECT ? 1 : R::WARPS][DIRECT ? 1 : R::SK];
    __shared__ typename DepositRun<FP>::MergeSmem s_merge[DIRECT && kTransposedMerge<FP> ? 8 : 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const FP *arr[7] = {(const FP *)e.soa.x, (const FP *)e.soa.y, (const FP *)e.soa.z,
                        (const FP *)e.soa.px, (const FP *)e.soa.py, (const FP *)e.soa.pz,
                        (const FP *)e.soa.w};
    const bool multi = dc.n_types > 1 && e.soa.type;
    const int64_t stride = (int64_t)gridDim.x * NW * R::TILE;
    FP rv[DIRECT ? 7 : 1][DIRECT ? R::K : 1];
    int16_t rty[DIRECT ? R::K : 1];
    // DIRECT: lane's K = 8 consecutive particles of the tile at `tb`, two 128-bit
    // loads per array (scalar loads in the ragged last tile).
    auto load_direct = [&](int64_t tb, FP (&dv)[DIRECT ? 7 : 1][DIRECT ? R::K : 1],
                           int16_t (&dty)[DIRECT ? R::K : 1]) {
        if constexpr (DIRECT) {
            static_assert(sizeof(FP) == 4 && R::K == 8, "direct staging: fp32, K = 8");
            const int64_t i0 = tb + lane * R::K;
            if (i0 + R::K <= e.n) {
#pragma unroll
                for (int a = 0; a < 7; ++a)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        float4 v = arr[a] ? __ldg(reinterpret_cast<const float4 *>(arr[a] + i0) + h)
                                          : make_float4(1.f, 1.f, 1.f, 1.f);
                        dv[a][4 * h] = v.x; dv[a][4 * h + 1] = v.y;
                        dv[a][4 * h + 2] = v.z; dv[a][4 * h + 3] = v.w;
                    }
                if (multi) {
                    const uint4 t4 = __ldg(reinterpret_cast<const uint4 *>(e.soa.type + i0));
                    const uint32_t tw[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
                    for (int j = 0; j < R::K; ++j)
                        dty[j] = (int16_t)(tw[j >> 1] >> (16 * (j & 1)));
                }
            } else {
#pragma unroll
                for (int j = 0; j < R::K; ++j) {
                    const int64_t i = i0 + j;
#pragma unroll
                    for (int a = 0; a < 7; ++a)
                        dv[a][j] = (i < e.n) ? (arr[a] ? arr[a][i] : FP(1)) : FP(0);
                    dty[j] = (multi && i < e.n) ? e.soa.type[i] : (int16_t)0;
                }
            }
        }
    };
#if BORIS_DEP_PREFETCH
    // software pipeline: the next tile's loads are in flight during this tile's
    // arithmetic, scan and atomics
    FP nv[DIRECT ? 7 : 1][DIRECT ? R::K : 1];
    int16_t nty[DIRECT ? R::K : 1];
    const int64_t first = ((int64_t)blockIdx.x * NW + warp) * R::TILE;
    if (DIRECT && first < e.n) load_direct(first, nv, nty);
#endif
    for (int64_t base = ((int64_t)blockIdx.x * NW + warp) * R::TILE; base < e.n;
         base += stride) {
        if constexpr (DIRECT) {
#if BORIS_DEP_PREFETCH
#pragma unroll
            for (int j = 0; j < R::K; ++j) {
#pragma unroll
                for (int a = 0; a < 7; ++a) rv[a][j] = nv[a][j];
                rty[j] = nty[j];
            }
            if (base + stride < e.n) load_direct(base + stride, nv, nty);
#else
            load_direct(base, rv, rty);
#endif
        } else {
            // coalesced warp loads into the skewed tile
#pragma unroll
            for (int r = 0; r < R::K; ++r) {
                const int p = r * 32 + lane;
                const int64_t i = base + p;
                const int sp = p + p / R::K;
#pragma unroll
                for (int a = 0; a < 7; ++a)
                    s[warp][a][sp] = (i < e.n) ? (arr[a] ? arr[a][i] : FP(1)) : FP(0);
                if (multi) s_ty[warp][sp] = (i < e.n) ? e.soa.type[i] : (int16_t)0;
            }
            __syncwarp();
        }
        DepositRun<FP> run;
        run.reset();
        constexpr int kUnrollJ = DIRECT ? R::K : 1;  // register arrays need constant indices
#pragma unroll kUnrollJ
        for (int j = 0; j < R::K; ++j) {
            const int p = lane * R::K + j;
            if (base + p >= e.n) break;
            const int sp = DIRECT ? 0 : p + p / R::K;
            const FP x = DIRECT ? rv[0][j] : s[warp][0][sp];
            const FP y = DIRECT ? rv[1][j] : s[warp][1][sp];
            const FP z = DIRECT ? rv[2][j] : s[warp][2][sp];
            const FP px = DIRECT ? rv[3][j] : s[warp][3][sp];
            const FP py = DIRECT ? rv[4][j] : s[warp][4][sp];
            const FP pz = DIRECT ? rv[5][j] : s[warp][5][sp];
            const FP w = DIRECT ? rv[6][j] : s[warp][6][sp];
            const DepCoef<FP> t = dc.t[multi ? (DIRECT ? rty[j] : s_ty[warp][sp]) : 0];
            run.add(g, t, dc.half_dt, x, y, z, px, py, pz, w, Jx, Jy, Jz);
        }
        // end of tile: merge lanes holding the same cell, one atomic per segment
        if constexpr (DIRECT && kTransposedMerge<FP>) {
            run.merge_flush(g, Jx, Jy, Jz, s_merge[warp], lane);
        } else {
            run.warp_merge(g, lane);
            run.flush(g, Jx, Jy, Jz);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Warp-run deposition (SoA, any alignment; deposit.cuh WarpRun): each warp owns a
// contiguous chunk of particles and walks it in rounds of 32 consecutive
// particles (lane l takes particle base + l: 4/8 B loads, warp-coalesced), PD
// rounds of loads in flight ahead of the arithmetic (register ring).  Sorted by
// cell, a round almost always lies in the warp's open cell: 24 FMA per particle,
// one warp reduction + one 24-lane atomic instruction per cell.
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
                   const __grid_constant__ DepCoefs<FP> dc, FP *Jx, FP *Jy, FP *Jz,
                   int64_t chunk) {
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
            run.round(g, part, i < end, Jx, Jy, Jz, sm[warp], lane);
        }
    }
    if (run.open) run.flush(g, Jx, Jy, Jz, sm[warp], lane);
}

template <typename FP>
__global__ void k_zero3(FP *a, FP *b, FP *c, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        a[i] = FP(0);
        b[i] = FP(0);
        c[i] = FP(0);
    }
}

// Zero J: one launch for the three arrays (three memsets cost ~3 launch gaps).
template <typename FP>
cudaError_t launch_zero3(void *Jx, void *Jy, void *Jz, int64_t n, cudaStream_t st) {
    const int64_t blocks = (n + 255) / 256;
    k_zero3<FP><<<(unsigned)(blocks < 4096 ? (blocks > 0 ? blocks : 1) : 4096), 256, 0, st>>>(
        (FP *)Jx, (FP *)Jy, (FP *)Jz, n);
    return cudaGetLastError();
}
template cudaError_t launch_zero3<float>(void *, void *, void *, int64_t, cudaStream_t);
template cudaError_t launch_zero3<double>(void *, void *, void *, int64_t, cudaStream_t);

template <typename FP>
cudaError_t launch_deposit(const EnsView &e, const GridArgs<FP> &g, const DepCoefs<FP> &dc,
                           void *Jx, void *Jy, void *Jz, int device, cudaStream_t st) {
    const int64_t ncell = (int64_t)g.n[0] * g.n[1] * g.n[2];
    cudaError_t err = launch_zero3<FP>(Jx, Jy, Jz, ncell, st);
    if (err != cudaSuccess || e.n == 0) return err;
    // fp32 with 16 B-aligned arrays: lane runs (k_deposit_runs DIRECT, 128-bit loads);
    // fp64 or unaligned: warp runs (k_deposit_warp).  Measured on 10^7 sorted
    // particles, 64^3 grid: fp32 11.0 (lane) vs 13.2 ps (warp), fp64 34.0 vs 22.5 ps.
    if constexpr (sizeof(FP) == 4) {
        auto al16 = [](const void *q) { return ((uintptr_t)q & 15u) == 0; };
        if (e.layout == BORIS_LAYOUT_SOA && al16(e.soa.x) && al16(e.soa.y) && al16(e.soa.z) &&
            al16(e.soa.px) && al16(e.soa.py) && al16(e.soa.pz) && al16(e.soa.w) &&
            al16(e.soa.type)) {
            using R = DepRuns<FP>;
            const int64_t tiles = (e.n + R::TILE - 1) / R::TILE;
            const int64_t blocks = (tiles + 7) / 8;
            const unsigned grid = (unsigned)stream_grid(blocks, 4, device);
            k_deposit_runs<FP, true><<<grid, 8 * 32, 0, st>>>(e, g, dc, (FP *)Jx, (FP *)Jy,
                                                               (FP *)Jz);
            return cudaGetLastError();
        }
    }
    if (e.layout == BORIS_LAYOUT_SOA) {
        // one contiguous chunk per warp, a multiple of 32 particles, sized so the
        // resident blocks cover the ensemble in one wave
        using D = DepWarp<FP>;
        const int64_t warps = (int64_t)sm_count(device) * D::MINB * D::WARPS;
        int64_t chunk = (e.n + warps - 1) / warps;
        chunk = (chunk + 31) / 32 * 32;
        const int64_t blocks = ((e.n + chunk - 1) / chunk + D::WARPS - 1) / D::WARPS;
        const bool multi = dc.n_types > 1 && e.soa.type;
        if (multi)
            k_deposit_warp<FP, true><<<(unsigned)blocks, D::WARPS * 32, 0, st>>>(
                e, g, dc, (FP *)Jx, (FP *)Jy, (FP *)Jz, chunk);
        else
            k_deposit_warp<FP, false><<<(unsigned)blocks, D::WARPS * 32, 0, st>>>(
                e, g, dc, (FP *)Jx, (FP *)Jy, (FP *)Jz, chunk);
        return cudaGetLastError();
    }
    const int64_t blocks = (e.n + 255) / 256;
    const unsigned grid = (unsigned)stream_grid(blocks, 8, device);
    k_deposit<FP><<<grid, 256, 0, st>>>(e, g, dc, (FP *)Jx, (FP *)Jy, (FP *)Jz);
    return cudaGetLastError();
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
