// Subsystem (6): the SPD solve of the L2 projection on the device CSR.
//
//  tq_csr_diag   <- A.diagonal()                          src/projection.py:159
//  tq_spmv       <- As @ y, A @ x (scaled / unscaled)      src/projection.py:160-161,196-201
//  tq_cg_scaled  <- spla.cg(As, r, rtol, atol=0, maxiter)  src/projection.py:180-186
//
// The reference solves the Jacobi-scaled system As = S A S (S = diag(A)^-1/2)
// with unpreconditioned conjugate gradients above DIRECT_LIMIT rows and
// refines iteratively.  Here the CSR formed on the GPU stays in HBM and the
// whole CG run is ONE cooperative kernel: a grid-stride warp-per-row SpMV,
// elementwise updates, and three grid barriers per iteration; every dot
// product is reduced to per-block partials that each block then sums in
// block order, so the scalars (and the iteration count) are identical on
// every block and from run to run.  The iteration follows scipy's cg
// exactly: test ||r|| < atol first, p = r on the first spin, p = r + beta p
// after, alpha = rho / (p . A p).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace tq {

constexpr int kCgThreads = 256;

// sum over the block (result valid in every thread)
__device__ __forceinline__ double cg_block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int k = 0; k < kCgThreads / 32; ++k) t += red[k];
    return t;
}

// deterministic grid sum of per-block partials (every block, block order)
__device__ __forceinline__ double cg_grid_total(const double* part, double* red) {
    double v = 0.0;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += kCgThreads) v += part[k];
    return cg_block_sum(v, red);
}

// row i of y = A (sr .* x) on a half-warp (hl = lane within the half, 0..15):
// rounds of 128 entries, all index/value loads issued before the dependent
// gathers; a warp carries two rows, so more bytes are in flight per warp.
// Returns the row value in every lane of the half.
__device__ __forceinline__ double spmv_row_half(const int32_t* __restrict__ indptr,
                                                const int32_t* __restrict__ indices,
                                                const double* __restrict__ data, const double* __restrict__ sr,
                                                const double* x, int i, int hl, bool valid) {
    double acc = 0.0;
    const int a = valid ? indptr[i] : 0, b = valid ? indptr[i + 1] : 0;
    for (int k0 = a; k0 < b; k0 += 128) {
        int j[8];
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = k0 + 16 * u + hl;
            j[u] = k < b ? __ldcs(indices + k) : -1;   // the matrix streams once per product
            v[u] = k < b ? __ldcs(data + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (j[u] >= 0) acc += v[u] * (sr ? sr[j[u]] * x[j[u]] : x[j[u]]);
    }
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    return acc;
}

__global__ void k_csr_diag(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                           const double* __restrict__ data, int n, double* __restrict__ diag) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int lo = indptr[i], hi = indptr[i + 1];     // sorted columns: binary search for i
        double d = 0.0;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const int c = indices[mid];
            if (c == i) { d = data[mid]; break; }
            if (c < i) lo = mid + 1; else hi = mid;
        }
        diag[i] = d;
    }
}

__global__ void k_spmv(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                       const double* __restrict__ data, int n, const double* __restrict__ sl,
                       const double* __restrict__ sr, const double* __restrict__ x, double* __restrict__ y) {
    const int lane = threadIdx.x & 31, hl = lane & 15;
    const int halves = (gridDim.x * blockDim.x) >> 4;
    // uniform trip count per warp (the shuffles need all 32 lanes)
    const int h0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 4;
    for (int base = h0 & ~1; base < n; base += halves) {
        const int i = base + ((lane >> 4) & 1);
        const bool valid = i < n;
        const double v = spmv_row_half(indptr, indices, data, sr, x, i, hl, valid);
        if (valid && hl == 0) y[i] = sl ? sl[i] * v : v;
    }
}

struct CgState {
    double* x;
    double* r;
    double* p;
    double* q;
    double* sp;       // s .* p (the SpMV gathers one vector)
    double* part_a;   // [grid]
    double* part_b;   // [grid]
    int32_t* iters;   // out: iterations run (== maxiter: not converged)
    double* rnorm;    // out: final ||r||
};

__global__ void __launch_bounds__(kCgThreads) k_cg_scaled(const int32_t* __restrict__ indptr,
                                                         const int32_t* __restrict__ indices,
                                                         const double* __restrict__ data, int n,
                                                         const double* __restrict__ s,
                                                         const double* __restrict__ bvec, double rtol,
                                                         int maxiter, CgState st) {
    __shared__ double red[kCgThreads / 32];
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nthreads = gridDim.x * blockDim.x;
    const int warp = tid >> 5, nwarps = nthreads >> 5;
    // x = 0, r = b, rho = r . r
    double loc = 0.0;
    for (int i = tid; i < n; i += nthreads) {
        const double bi = bvec[i];
        st.x[i] = 0.0;
        st.r[i] = bi;
        loc += bi * bi;
    }
    double v = cg_block_sum(loc, red);
    if (threadIdx.x == 0) st.part_b[blockIdx.x] = v;
    grid.sync();
    double rr = cg_grid_total(st.part_b, red);
    const double atol = rtol * sqrt(rr);         // scipy: atol = max(atol=0, rtol * ||b||)
    double rho_prev = 1.0;
    int it = 0;
    for (; it < maxiter; ++it) {
        if (rr == 0.0 || sqrt(rr) < atol) break;   // same value on every block (b = 0: x = 0, as scipy)
        const double rho = rr;
        const double beta = it > 0 ? rho / rho_prev : 0.0;
        for (int i = tid; i < n; i += nthreads) {
            const double pi = it > 0 ? st.r[i] + beta * st.p[i] : st.r[i];
            st.p[i] = pi;
            st.sp[i] = s[i] * pi;
        }
        grid.sync();
        // q = As p = s .* (A (s .* p)), p . q
        loc = 0.0;
        for (int base = 2 * warp; base < n; base += 2 * nwarps) {
            const int i = base + (lane >> 4);
            const bool valid = i < n;
            const double vi = spmv_row_half(indptr, indices, data, nullptr, st.sp, i, lane & 15, valid);
            if (valid && (lane & 15) == 0) {
                const double qi = s[i] * vi;
                st.q[i] = qi;
                loc += st.p[i] * qi;
            }
        }
        v = cg_block_sum(loc, red);
        if (threadIdx.x == 0) st.part_a[blockIdx.x] = v;
        grid.sync();
        const double pq = cg_grid_total(st.part_a, red);
        const double alpha = rho / pq;
        loc = 0.0;
        for (int i = tid; i < n; i += nthreads) {
            st.x[i] += alpha * st.p[i];
            const double ri = st.r[i] - alpha * st.q[i];
            st.r[i] = ri;
            loc += ri * ri;
        }
        rho_prev = rho;
        v = cg_block_sum(loc, red);
        if (threadIdx.x == 0) st.part_b[blockIdx.x] = v;
        grid.sync();
        rr = cg_grid_total(st.part_b, red);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *st.iters = it;
        *st.rnorm = sqrt(rr);
    }
}

}  // namespace tq

using namespace tq;

extern "C" int tq_csr_diag(const int32_t* indptr, const int32_t* indices, const double* data, int32_t n,
                           double* diag, void* stream) {
    if (n <= 0) return TQ_OK;
    k_csr_diag<<<grid_for(n, 256), 256, 0, S(stream)>>>(indptr, indices, data, n, diag); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_csr_diag");
    return TQ_OK;
}

extern "C" int tq_spmv(const int32_t* indptr, const int32_t* indices, const double* data, int32_t n,
                       const double* sl, const double* sr, const double* x, double* y, void* stream) {
    if (n <= 0) return TQ_OK;
    const int grid = (int)std::min<int64_t>(((int64_t)n * 32 + 255) / 256, (int64_t)kSms * 16);
    k_spmv<<<grid, 256, 0, S(stream)>>>(indptr, indices, data, n, sl, sr, x, y); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_spmv");
    return TQ_OK;
}

static int cg_grid() {
    static int g[64] = {};
    int d = 0;
    cudaGetDevice(&d);
    if (!g[d]) {
        int per_sm = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg_scaled, kCgThreads, 0);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
        g[d] = std::max(per_sm, 1) * std::max(sms, 1);
    }
    return g[d];
}

extern "C" int64_t tq_cg_workspace_bytes(int32_t n) {
    return (int64_t)sizeof(double) * (4 * (int64_t)std::max(n, 1) + 2 * (int64_t)cg_grid() + 2);
}

extern "C" int tq_cg_scaled(const int32_t* indptr, const int32_t* indices, const double* data, int32_t n,
                            const double* s, const double* b, double* x, double rtol, int32_t maxiter,
                            void* work, int32_t* iters_dev, double* rnorm_dev, void* stream) {
    if (n <= 0) return TQ_OK;
    if (!(rtol > 0.0) || maxiter < 0) { set_error("invalid CG tolerance or iteration limit"); return TQ_EINVAL; }
    // blocks: co-resident (cooperative launch), about a warp per 8 rows at least
    const int grid = (int)std::min<int64_t>(cg_grid(), std::max<int64_t>(((int64_t)n * 4 + kCgThreads - 1) / kCgThreads, 1));
    double* w = static_cast<double*>(work);
    const int64_t nn = std::max(n, 1);
    CgState st{x, w, w + nn, w + 2 * nn, w + 3 * nn, w + 4 * nn, w + 4 * nn + cg_grid(), iters_dev, rnorm_dev};
    const int32_t* a0 = indptr;
    const int32_t* a1 = indices;
    const double* a2 = data;
    int32_t a3 = n;
    const double* a4 = s;
    const double* a5 = b;
    double a6 = rtol;
    int32_t a7 = maxiter;
    void* args[] = {&a0, &a1, &a2, &a3, &a4, &a5, &a6, &a7, &st};
    TQ_CUDA(cudaLaunchCooperativeKernel((const void*)k_cg_scaled, grid, kCgThreads, args, 0, S(stream)));
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_cg_scaled");
    return TQ_OK;
}
