// Integer prefix passes: CSR row pointer and the active-function index.
//
//  tq_scan_indptr  <- the indptr of _Pattern / scipy CSR   src/assembly.py:154-166
//  tq_active_index <- active_functions + col_of            src/trimming.py:514-517,
//                                                          src/assembly.py:150-153
// Row pointer: one cooperative kernel (slab sums, grid barrier, rescan).  Active index: three-phase
// tiled scan (tile sums -> scan of tile sums -> tile rescan).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace tq {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kTile = kScanThreads * kScanItems;

struct ActiveIn {
    const int8_t* fc;
    __device__ int64_t operator()(int64_t i) const { return fc[i] != TQ_EXTERIOR ? 1 : 0; }
};

template <class In>
__global__ void k_tile_sums(In in, int64_t n, int64_t* tile_sums) {
    __shared__ int64_t red[kScanThreads / 32];
    int64_t base = (int64_t)blockIdx.x * kTile;
    int64_t s = 0;
    for (int k = threadIdx.x; k < kTile; k += kScanThreads) {
        int64_t i = base + k;
        if (i < n) s += in(i);
    }
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) t += red[w];
        tile_sums[blockIdx.x] = t;
    }
}

// exclusive scan of tile sums in one block; total -> tile_sums[ntiles]
__global__ void k_scan_tiles(int64_t* tile_sums, int64_t ntiles) {
    __shared__ int64_t carry;
    __shared__ int64_t wsum[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < ntiles; b0 += blockDim.x) {
        int64_t i = b0 + threadIdx.x;
        int64_t v = i < ntiles ? tile_sums[i] : 0;
        int64_t x = v;
        int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int off = 1; off < 32; off <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        if (w == 0) {
            int nw = blockDim.x >> 5;
            int64_t z = lane < nw ? wsum[lane] : 0;
            for (int off = 1; off < 32; off <<= 1) {
                int64_t y = __shfl_up_sync(0xffffffffu, z, off);
                if (lane >= off) z += y;
            }
            if (lane < nw) wsum[lane] = z;
        }
        __syncthreads();
        int64_t incl = x + (w > 0 ? wsum[w - 1] : 0) + carry;
        if (i < ntiles) tile_sums[i] = incl - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) tile_sums[ntiles] = carry;
}

// per-tile exclusive scan; Out(i, v, excl) consumes each element
template <class In, class Out>
__global__ void k_tile_apply(In in, int64_t n, const int64_t* tile_off, Out out) {
    __shared__ int64_t wsum[kScanThreads / 32];
    int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kScanItems;
    int64_t loc[kScanItems];
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t i = base + k;
        loc[k] = i < n ? in(i) : 0;
        s += loc[k];
    }
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t x = s;
    for (int off = 1; off < 32; off <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    int64_t woff = 0;
    for (int q = 0; q < w; ++q) woff += wsum[q];
    int64_t run = tile_off[blockIdx.x] + woff + x - s;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t i = base + k;
        if (i < n) out(i, loc[k], run);
        run += loc[k];
    }
}

struct ActiveOut {
    int32_t* col_of;
    int32_t* active;
    __device__ void operator()(int64_t i, int64_t v, int64_t excl) const {
        col_of[i] = v ? (int32_t)excl : -1;
        if (v) active[excl] = (int32_t)i;
    }
};

template <class In, class Out>
int scan_generic(In in, int64_t n, Out out, int64_t* total_h, cudaStream_t st) {
    int64_t ntiles = (n + kTile - 1) / kTile;
    if (ntiles == 0) ntiles = 1;
    int64_t* tiles = nullptr;
    TQ_CUDA(cudaMallocAsync(&tiles, (ntiles + 1) * sizeof(int64_t), st));
    k_tile_sums<<<(unsigned)ntiles, kScanThreads, 0, st>>>(in, n, tiles); ::tq::note_launch();
    k_scan_tiles<<<1, 1024, 0, st>>>(tiles, ntiles); ::tq::note_launch();
    k_tile_apply<<<(unsigned)ntiles, kScanThreads, 0, st>>>(in, n, tiles, out); ::tq::note_launch();
    TQ_LAUNCH_CHECK("scan");
    if (total_h) {
        TQ_CUDA(cudaMemcpyAsync(total_h, tiles + ntiles, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    }
    TQ_CUDA(cudaFreeAsync(tiles, st));
    if (total_h) TQ_CUDA(cudaStreamSynchronize(st));
    return TQ_OK;
}


// Row-pointer scan in one cooperative kernel: every block owns a contiguous
// slab of the counts (all blocks co-resident), sums it, meets the others at
// one grid barrier, takes its prefix from the block sums before it, and
// rescans its slab (second read served by L2) writing indptr with int4
// stores.  No look-back chain and no second launch.
constexpr int kCoopThreads = 512;

__device__ __forceinline__ int4 load4(const int32_t* p, int64_t i, int64_t hi, bool aligned) {
    if (aligned && i + 3 < hi) return __ldg(reinterpret_cast<const int4*>(p + i));
    int4 q = make_int4(0, 0, 0, 0);
    if (i < hi) q.x = p[i];
    if (i + 1 < hi) q.y = p[i + 1];
    if (i + 2 < hi) q.z = p[i + 2];
    if (i + 3 < hi) q.w = p[i + 3];
    return q;
}

// block-wide sum of one value per thread (result in every thread)
__device__ __forceinline__ long long block_sum(long long v, long long* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    long long t = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
    return t;
}

__global__ void __launch_bounds__(kCoopThreads) k_scan_coop(const int32_t* __restrict__ counts, int32_t n,
                                                           int32_t* __restrict__ indptr,
                                                           long long* __restrict__ blocksums, int32_t* ovf,
                                                           int64_t* total_out) {
    __shared__ long long red[kCoopThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t slab = (((int64_t)n + gridDim.x - 1) / gridDim.x + 3) / 4 * 4;
    const int64_t lo = min((int64_t)n, (int64_t)blockIdx.x * slab), hi = min((int64_t)n, lo + slab);
    const bool in_al = (reinterpret_cast<uintptr_t>(counts) & 15) == 0;
    const bool out_al = (reinterpret_cast<uintptr_t>(indptr) & 15) == 0;
    // phase 1: slab sum (kSeg int4 per thread in flight)
    constexpr int kSeg = 4, kRound = 4 * kCoopThreads * kSeg;
    long long s = 0;
    for (int64_t base = lo; base < hi; base += kRound) {
        int4 q[kSeg];
#pragma unroll
        for (int j = 0; j < kSeg; ++j) q[j] = load4(counts, base + 4 * (j * kCoopThreads + threadIdx.x), hi, in_al);
#pragma unroll
        for (int j = 0; j < kSeg; ++j) s += (long long)q[j].x + q[j].y + q[j].z + q[j].w;
    }
    const long long mine = block_sum(s, red);
    if (threadIdx.x == 0) blocksums[blockIdx.x] = mine;
    cg::this_grid().sync();
    // phase 2: prefix of this slab
    long long p = 0;
    for (int k = threadIdx.x; k < (int)blockIdx.x; k += kCoopThreads) p += blocksums[k];
    long long carry = block_sum(p, red);
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        const long long tot = carry + mine;
        if (tot > 0x7fffffffLL) *ovf = 1;
        indptr[n] = (int32_t)tot;
        *total_out = tot;
    }
    // phase 3: rescan, kSeg warp-striped segments per round scanned together
    __shared__ long long wseg[kSeg][kCoopThreads / 32];
    bool over = false;
    for (int64_t base = lo; base < hi; base += kRound) {
        int4 q[kSeg];
        long long t[kSeg], x[kSeg];
#pragma unroll
        for (int j = 0; j < kSeg; ++j) {
            q[j] = load4(counts, base + 4 * (j * kCoopThreads + threadIdx.x), hi, in_al);
            t[j] = (long long)q[j].x + q[j].y + q[j].z + q[j].w;
            x[j] = t[j];
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
            for (int j = 0; j < kSeg; ++j) {
                const long long y = __shfl_up_sync(0xffffffffu, x[j], off);
                if (lane >= off) x[j] += y;
            }
        }
        __syncthreads();
        if (lane == 31) {
#pragma unroll
            for (int j = 0; j < kSeg; ++j) wseg[j][w] = x[j];
        }
        __syncthreads();
        long long segbase = carry;
#pragma unroll
        for (int j = 0; j < kSeg; ++j) {
            long long woff = 0, tot = 0;
            for (int k = 0; k < kCoopThreads / 32; ++k) {
                const long long z = wseg[j][k];
                woff += k < w ? z : 0;
                tot += z;
            }
            const int64_t i = base + 4 * (j * kCoopThreads + threadIdx.x);
            const long long e0 = segbase + woff + (x[j] - t[j]), e1 = e0 + q[j].x, e2 = e1 + q[j].y, e3 = e2 + q[j].z;
            over |= i < hi && e3 > 0x7fffffffLL;
            if (out_al && i + 3 < hi) {
                *reinterpret_cast<int4*>(indptr + i) = make_int4((int)e0, (int)e1, (int)e2, (int)e3);
            } else {
                if (i < hi) indptr[i] = (int32_t)e0;
                if (i + 1 < hi) indptr[i + 1] = (int32_t)e1;
                if (i + 2 < hi) indptr[i + 2] = (int32_t)e2;
                if (i + 3 < hi) indptr[i + 3] = (int32_t)e3;
            }
            segbase += tot;
        }
        carry = segbase;
    }
    if (over) atomicOr(ovf, 1);
}

// Tile mode: exclusive scan of the per-32-row tile sums (ceil(nrows/32)
// values, written by the count passes just before and L2-resident).  Block b
// owns 1024 tiles and reduces every tile sum before its range itself (int4
// loads, all in flight; at most ~0.4 MB of L2 reads per block), then scans its
// own range: no inter-block flags, barrier or workspace reset.  Bases go to
// the second half of the buffer (the sums stay readable by the other blocks).
constexpr int kTileScanThreads = 1024;

// MODE 0: every tile -> bases, total, overflow flag (and the check against
// the nnz the early scan was given).  MODE 1 (grid 2G): blocks [0, G) the
// head tiles (prefix sums), blocks [G, 2G) the tail tiles (nnz - suffix
// sums), both into the early bases.
__device__ __forceinline__ long long sum_range(const int32_t* __restrict__ sums, int lo, int hi) {
    long long acc = 0;
    if (lo < hi && (lo & 3) == 0) {          // vector loads from an aligned start
        const int4* s4 = reinterpret_cast<const int4*>(sums + lo);
        const int n4 = (hi - lo) >> 2;
        constexpr int U = 8;
        for (int q0 = threadIdx.x; q0 < n4; q0 += U * kTileScanThreads) {
            int4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = q0 + u * kTileScanThreads;
                v[u] = q < n4 ? __ldg(s4 + q) : make_int4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) acc += (long long)v[u].x + v[u].y + v[u].z + v[u].w;
        }
        lo += n4 << 2;
    }
    constexpr int U = 8;
    for (int k0 = lo + threadIdx.x; k0 < hi; k0 += U * kTileScanThreads) {
        int v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = k0 + u * kTileScanThreads;
            v[u] = k < hi ? __ldg(sums + k) : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    return acc;
}

template <int MODE>
__global__ void __launch_bounds__(kTileScanThreads) k_scan_tiles(tq_rowctx c, int32_t* __restrict__ indptr_last,
                                                                long long nnz, int with_tail) {
    __shared__ long long red[32];
    __shared__ long long wtot[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nr = c.row_end - c.row_begin, NT = TQ_TILE_NT(nr);
    const int32_t* __restrict__ sums = c.tiles;
    int32_t* ctl = c.tiles + TQ_TILE_CTL(nr);
    const int G = (NT + kTileScanThreads - 1) / kTileScanThreads;
    const bool tail = MODE == 1 && (int)blockIdx.x >= G;
    int lo, hi;                                  // this launch's tile range
    if (MODE == 0) { lo = 0; hi = NT; }
    else if (!tail) { lo = 0; hi = head_tiles(c); }
    else { lo = with_tail ? max(tail_first_raw(c), head_tiles(c)) : NT; hi = NT; }
    const int t0 = lo + (tail ? (int)blockIdx.x - G : (int)blockIdx.x) * kTileScanThreads;
    if (t0 >= hi) return;
    // head / full: the sum of every tile before the block; tail: after it
    long long outside = tail ? sum_range(sums, t0 + kTileScanThreads, hi) : sum_range(sums, 0, t0);
    const int i = t0 + threadIdx.x;
    const int v = i < hi ? __ldg(sums + i) : 0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) outside += __shfl_xor_sync(0xffffffffu, outside, off);
    long long x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) wtot[w] = x;
    if (lane == 0) red[w] = outside;
    __syncthreads();
    long long out = 0, woff = 0, btot = 0;
    for (int k = 0; k < 32; ++k) {
        out += red[k];
        woff += k < w ? wtot[k] : 0;
        btot += wtot[k];
    }
    const long long excl = woff + x - v;                 // within the block
    int32_t* __restrict__ bases = c.tiles + (MODE == 0 ? TQ_TILE_PAD(nr) : TQ_TILE_EARLY(nr));
    if (i < hi) bases[i] = (int32_t)(tail ? nnz - (out + btot - excl) : out + excl);
    if (MODE == 0 && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        const long long total = out + btot;
        *indptr_last = (int32_t)total;
        bases[NT] = (int32_t)total;
        bases[NT + 1] = total > 0x7fffffffLL ? 1 : 0;   // overflow flag
        if (ctl[6] && total != (long long)ctl[5]) ctl[4] = 1;   // early tail bases assumed another nnz
    }
    if (MODE == 1 && blockIdx.x == 0 && threadIdx.x == 0) {
        if (nnz >= 0) {                                // the count the caller expects
            ctl[5] = (int32_t)nnz;
            ctl[6] = 1;
        }
        ctl[7] = with_tail;                            // the tail tiles are early
    }
}

}  // namespace tq

using namespace tq;

extern "C" int tq_scan_tiles(tq_rowctx c, int32_t* indptr, int64_t* nnz_h, void* stream) {
    cudaStream_t st = S(stream);
    const int nrows = c.row_end - c.row_begin;
    if (!c.tiles || !c.counts) { set_error("tq_scan_tiles needs the context's counts and tiles"); return TQ_EINVAL; }
    if (nrows <= 0) {
        TQ_CUDA(cudaMemsetAsync(indptr, 0, sizeof(int32_t), st));
        if (nnz_h) *nnz_h = 0;
        return TQ_OK;
    }
    const int ntiles = (nrows + 31) / 32;
    int32_t* bases = tq_tile_bases(c.tiles, nrows);
    const int grid = (ntiles + kTileScanThreads - 1) / kTileScanThreads;
    k_scan_tiles<0><<<grid, kTileScanThreads, 0, st>>>(c, indptr + nrows, -1, 0); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_scan_tiles");
    if (nnz_h) {
        int32_t h[2] = {0, 0};
        TQ_CUDA(cudaMemcpyAsync(h, bases + ntiles, sizeof(h), cudaMemcpyDeviceToHost, st));
        TQ_CUDA(cudaStreamSynchronize(st));
        if (h[1]) { set_error("nnz does not fit int32 CSR indices"); return TQ_EOVERFLOW; }
        *nnz_h = h[0];
    }
    return TQ_OK;
}


static int coop_grid() {
    static int g[64] = {};
    int d = 0;
    cudaGetDevice(&d);
    if (!g[d]) {
        int per_sm = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_scan_coop, kCoopThreads, 0);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
        g[d] = std::max(per_sm, 1) * std::max(sms, 1);
    }
    return g[d];
}

extern "C" int64_t tq_scan_workspace_bytes(int32_t nrows) {
    (void)nrows;
    return (int64_t)(coop_grid() + 2) * (int64_t)sizeof(int64_t);
}

// `ws`: caller scratch of tq_scan_workspace_bytes(nrows) bytes.
// nnz_h == NULL: no host read-back (stream-capture safe; the caller knows nnz)
extern "C" int tq_scan_indptr_ws(const int32_t* counts, int32_t nrows, int32_t* indptr, void* ws_v,
                                 int64_t* nnz_h, void* stream) {
    cudaStream_t st = S(stream);
    // workspace: [total i64][ovf i32, pad][block sums i64 x grid]
    int64_t* ws = static_cast<int64_t*>(ws_v);
    int32_t* ovf = reinterpret_cast<int32_t*>(ws + 1);
    long long* blocksums = reinterpret_cast<long long*>(ws + 2);
    TQ_CUDA(cudaMemsetAsync(ws, 0, 2 * sizeof(int64_t), st));
    if (nrows > 0) {
        // blocks: co-resident (cooperative launch), >= ~4096 counts each
        const int grid = (int)std::min<int64_t>(coop_grid(), std::max<int64_t>((nrows + 4095) / 4096, 1));
        const int32_t* a0 = counts;
        int32_t a1 = nrows;
        int32_t* a2 = indptr;
        long long* a3 = blocksums;
        int32_t* a4 = ovf;
        int64_t* a5 = ws;
        void* args[] = {&a0, &a1, &a2, &a3, &a4, &a5};
        TQ_CUDA(cudaLaunchCooperativeKernel((const void*)k_scan_coop, grid, kCoopThreads, args, 0, st));
        ::tq::note_launch();
    } else {
        TQ_CUDA(cudaMemsetAsync(indptr, 0, sizeof(int32_t), st));
    }
    TQ_LAUNCH_CHECK("scan");
    if (nnz_h) {
        int64_t total = 0;
        int32_t hovf = 0;
        TQ_CUDA(cudaMemcpyAsync(&total, ws, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        TQ_CUDA(cudaMemcpyAsync(&hovf, ovf, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        TQ_CUDA(cudaStreamSynchronize(st));
        if (hovf || total > 0x7fffffffLL) {
            set_error("nnz %lld does not fit int32 CSR indices", (long long)total);
            return TQ_EOVERFLOW;
        }
        *nnz_h = total;
    }
    return TQ_OK;
}

// as tq_scan_indptr_ws with a stream-ordered workspace of its own
extern "C" int tq_scan_indptr(const int32_t* counts, int32_t nrows, int32_t* indptr, int64_t* nnz_h,
                              void* stream) {
    cudaStream_t st = S(stream);
    void* ws = nullptr;
    TQ_CUDA(cudaMallocAsync(&ws, tq_scan_workspace_bytes(nrows), st));
    const int rc = tq_scan_indptr_ws(counts, nrows, indptr, ws, nnz_h, stream);
    TQ_CUDA(cudaFreeAsync(ws, st));
    return rc;
}

extern "C" int tq_active_index(const int8_t* func_class, int64_t nfun, int32_t* col_of, int32_t* active,
                               int32_t* K_h, void* stream) {
    int64_t total = 0;
    int rc = scan_generic(ActiveIn{func_class}, nfun, ActiveOut{col_of, active}, &total, S(stream));
    if (rc) return rc;
    *K_h = (int32_t)total;
    return TQ_OK;
}

__global__ void k_tiles_expect(int32_t* __restrict__ ctl, int32_t nnz) {
    ctl[5] = nnz;
    ctl[6] = 1;
}

// The nnz a captured pass sized its output with: the next tq_scan_tiles
// compares its total against it and sets TQ_TILE_CTL + 4 on a mismatch, and
// the tile-mode fill kernels then write nothing (a replay whose counts moved
// must not write past the captured buffers; GraphFormation.check raises).
extern "C" int tq_tiles_expect(tq_rowctx c, int64_t nnz, void* stream) {
    const int nrows = c.row_end - c.row_begin;
    if (!c.tiles) { set_error("tq_tiles_expect needs the context's tiles"); return TQ_EINVAL; }
    if (nnz < 0 || nnz > 0x7fffffffLL) { set_error("nnz %lld out of range", (long long)nnz); return TQ_EINVAL; }
    if (nrows <= 0) return TQ_OK;
    k_tiles_expect<<<1, 1, 0, S(stream)>>>(c.tiles + TQ_TILE_CTL(nrows), (int32_t)nnz); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_tiles_expect");
    return TQ_OK;
}

extern "C" int tq_scan_tiles_early(tq_rowctx c, int64_t nnz, int32_t tail, void* stream) {
    const int nrows = c.row_end - c.row_begin;
    if (!c.tiles || !c.counts) { set_error("tq_scan_tiles_early needs the context's counts and tiles"); return TQ_EINVAL; }
    if (nnz > 0x7fffffffLL || (tail && nnz < 0)) { set_error("nnz %lld out of range", (long long)nnz); return TQ_EINVAL; }
    if (nrows <= 0) return TQ_OK;
    const int G = (TQ_TILE_NT(nrows) + kTileScanThreads - 1) / kTileScanThreads;
    k_scan_tiles<1><<<2 * G, kTileScanThreads, 0, S(stream)>>>(c, nullptr, nnz, tail ? 1 : 0); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_scan_tiles_early");
    return TQ_OK;
}
