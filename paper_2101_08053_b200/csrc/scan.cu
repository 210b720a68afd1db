// Integer prefix passes: CSR row pointer and the active-function index.
//
//  tq_scan_indptr  <- the indptr of _Pattern / scipy CSR   src/assembly.py:154-166
//  tq_active_index <- active_functions + col_of            src/trimming.py:514-517,
//                                                          src/assembly.py:150-153
// Three-phase tiled scan (tile sums -> scan of tile sums -> tile rescan).
#include "common.cuh"

namespace tq {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kTile = kScanThreads * kScanItems;

struct CountsIn {
    const int32_t* v;
    __device__ int64_t operator()(int64_t i) const { return v[i]; }
};
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

struct IndptrOut {
    int32_t* indptr;
    int32_t* overflow;
    __device__ void operator()(int64_t i, int64_t v, int64_t excl) const {
        if (excl > 0x7fffffffLL) atomicOr(overflow, 1);
        indptr[i] = (int32_t)excl;
    }
};
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

__global__ void k_set_last(int32_t* indptr, int64_t n, const int64_t* total) {
    indptr[n] = (int32_t)(*total);
}

}  // namespace tq

using namespace tq;

__global__ void k_scan_finish(int32_t* indptr, int32_t nrows, const int64_t* total, int32_t* ovf) {
    if (threadIdx.x == 0) {
        int64_t t = *total;
        if (t > 0x7fffffffLL) *ovf = 1;
        indptr[nrows] = (int32_t)t;
    }
}

// nnz_h == NULL: no host read-back (stream-capture safe; the caller knows nnz)
extern "C" int tq_scan_indptr(const int32_t* counts, int32_t nrows, int32_t* indptr, int64_t* nnz_h,
                              void* stream) {
    cudaStream_t st = S(stream);
    int64_t ntiles = (nrows + kTile - 1) / kTile;
    if (ntiles == 0) ntiles = 1;
    int64_t* tiles = nullptr;
    TQ_CUDA(cudaMallocAsync(&tiles, (ntiles + 2) * sizeof(int64_t), st));
    int32_t* ovf = reinterpret_cast<int32_t*>(tiles + ntiles + 1);
    TQ_CUDA(cudaMemsetAsync(ovf, 0, sizeof(int32_t), st));
    CountsIn in{counts};
    k_tile_sums<<<(unsigned)ntiles, kScanThreads, 0, st>>>(in, nrows, tiles); ::tq::note_launch();
    k_scan_tiles<<<1, 1024, 0, st>>>(tiles, ntiles); ::tq::note_launch();
    k_tile_apply<<<(unsigned)ntiles, kScanThreads, 0, st>>>(in, nrows, tiles, IndptrOut{indptr, ovf}); ::tq::note_launch();
    k_scan_finish<<<1, 32, 0, st>>>(indptr, nrows, tiles + ntiles, ovf); ::tq::note_launch();
    TQ_LAUNCH_CHECK("scan");
    int64_t total = 0;
    int32_t hovf = 0;
    if (nnz_h) {
        TQ_CUDA(cudaMemcpyAsync(&total, tiles + ntiles, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        TQ_CUDA(cudaMemcpyAsync(&hovf, ovf, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    }
    TQ_CUDA(cudaFreeAsync(tiles, st));
    if (nnz_h) {
        TQ_CUDA(cudaStreamSynchronize(st));
        if (hovf || total > 0x7fffffffLL) {
            set_error("nnz %lld does not fit int32 CSR indices", (long long)total);
            return TQ_EOVERFLOW;
        }
        *nnz_h = total;
    }
    return TQ_OK;
}

extern "C" int tq_active_index(const int8_t* func_class, int64_t nfun, int32_t* col_of, int32_t* active,
                               int32_t* K_h, void* stream) {
    int64_t total = 0;
    int rc = scan_generic(ActiveIn{func_class}, nfun, ActiveOut{col_of, active}, &total, S(stream));
    if (rc) return rc;
    *K_h = (int32_t)total;
    return TQ_OK;
}
