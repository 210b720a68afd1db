// Shared helpers for the trimquad_b200 native library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/trimquad_b200.h"

namespace tq {

void set_error(const char* fmt, ...);
void note_launch();
int check_cuda(cudaError_t e, const char* what);

#define TQ_CUDA(call)                                              \
    do {                                                           \
        cudaError_t _e = (call);                                   \
        if (_e != cudaSuccess) return ::tq::check_cuda(_e, #call); \
    } while (0)

#define TQ_LAUNCH_CHECK(name)                                        \
    do {                                                             \
        cudaError_t _e = cudaGetLastError();                         \
        if (_e != cudaSuccess) return ::tq::check_cuda(_e, name);    \
    } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kMaxP = 10;          // largest supported degree
constexpr int kSms = 148;          // B200 SM count (grid sizing)

// device status word bits (accumulated with atomicOr by kernels)
constexpr int kStatusDomain = 1;   // coordinate outside the knot domain
constexpr int kStatusTrim = 2;     // unsupported trimming configuration
constexpr int kStatusOverflow = 4;

// searchsorted(a, x, side="right") on a sorted device array
__host__ __device__ inline int upper_bound_d(const double* a, int n, double x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// searchsorted(a, x, side="right") on a sorted int array
__host__ __device__ inline int upper_bound_d_int(const int32_t* a, int n, int x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// searchsorted(a, x, side="left")
__host__ __device__ inline int lower_bound_d(const double* a, int n, double x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// knot span of u (src/splines.py:114-122): searchsorted right - 1, clipped
__host__ __device__ inline int find_span(const double* knots, int nknots, int p, int n, double u) {
    int s = upper_bound_d(knots, nknots, u) - 1;
    if (s < p) s = p;
    if (s > n - 1) s = n - 1;
    return s;
}

// Cox-de Boor triangle (NURBS book A2.2) -- the p+1 non-zero values at u on
// span `span`; same operation order as src/splines.py:256-268.
template <int P>
__host__ __device__ inline void basis_funs(const double* kn, int span, double u, double* N) {
    double left[P + 1], right[P + 1];
    N[0] = 1.0;
#pragma unroll
    for (int j = 1; j <= P; ++j) {
        left[j - 1] = u - kn[span + 1 - j];
        right[j - 1] = kn[span + j] - u;
        double saved = 0.0;
#pragma unroll
        for (int r = 0; r < j; ++r) {
            double temp = N[r] / (right[r] + left[j - r - 1]);
            N[r] = saved + right[r] * temp;
            saved = left[j - r - 1] * temp;
        }
        N[j] = saved;
    }
}

// runtime-degree version (p <= kMaxP)
__host__ __device__ inline void basis_funs_rt(const double* kn, int p, int span, double u, double* N) {
    double left[kMaxP + 1], right[kMaxP + 1];
    N[0] = 1.0;
    for (int j = 1; j <= p; ++j) {
        left[j - 1] = u - kn[span + 1 - j];
        right[j - 1] = kn[span + j] - u;
        double saved = 0.0;
        for (int r = 0; r < j; ++r) {
            double temp = N[r] / (right[r] + left[j - r - 1]);
            N[r] = saved + right[r] * temp;
            saved = left[j - r - 1] * temp;
        }
        N[j] = saved;
    }
}

// values + first derivatives on span (derivative via degree p-1 values)
__host__ __device__ inline void basis_funs_ders_rt(const double* kn, int p, int span, double u,
                                                   double* N, double* D) {
    basis_funs_rt(kn, p, span, u, N);
    if (p == 0) { D[0] = 0.0; return; }
    double Nl[kMaxP + 1];
    basis_funs_rt(kn, p - 1, span, u, Nl);  // B_{span-p+1 .. span, p-1}
    for (int k = 0; k <= p; ++k) {
        int i = span - p + k;
        double acc = 0.0;
        if (k >= 1) {
            double den = kn[i + p] - kn[i];
            if (den > 0.0) acc += (double)p / den * Nl[k - 1];
        }
        if (k <= p - 1) {
            double den = kn[i + p + 1] - kn[i + 1];
            if (den > 0.0) acc -= (double)p / den * Nl[k];
        }
        D[k] = acc;
    }
}

// compile-time-degree values + first derivatives (the runtime-degree
// basis_funs_ders_rt above is miscompiled for sm_100a at -O3 in some inlining
// contexts -- wrong derivatives, measured with CUDA 12.9 in k_geo_lines --
// so new kernels dispatch on the degree and use this one)
template <int P>
__host__ __device__ inline void basis_funs_ders(const double* kn, int span, double u, double* N, double* D) {
    basis_funs<P>(kn, span, u, N);
    if (P == 0) { D[0] = 0.0; return; }
    double Nl[P + 1];
    basis_funs<(P > 0 ? P - 1 : 0)>(kn, span, u, Nl);
#pragma unroll
    for (int k = 0; k <= P; ++k) {
        const int i = span - P + k;
        double acc = 0.0;
        if (k >= 1) {
            const double den = kn[i + P] - kn[i];
            if (den > 0.0) acc += (double)P / den * Nl[k - 1];
        }
        if (k <= P - 1) {
            const double den = kn[i + P + 1] - kn[i + 1];
            if (den > 0.0) acc -= (double)P / den * Nl[k];
        }
        D[k] = acc;
    }
}

// tile mode: number of head tiles (those before the tile holding the first
// list-A row; all tiles when list A is empty), from count pass 1's control word
__device__ __forceinline__ int head_tiles(const tq_rowctx& c) {
    const int n = c.row_end - c.row_begin;
    const int enc = c.tiles[TQ_TILE_CTL(n)];
    if (enc == 0) return TQ_TILE_NT(n);
    return ((0x7fffffff - enc) - c.row_begin) >> 5;
}

// first tail tile (after the tile holding the last list-A row; NT: no tail)
__device__ __forceinline__ int tail_first_raw(const tq_rowctx& c) {
    const int n = c.row_end - c.row_begin;
    const int last1 = c.tiles[TQ_TILE_CTL(n) + 1];
    if (last1 == 0) return TQ_TILE_NT(n);
    return ((last1 - 1 - c.row_begin) >> 5) + 1;
}

// ... when the early scan gave the tail tiles bases (control word 7), else NT
__device__ __forceinline__ int tail_first(const tq_rowctx& c) {
    const int n = c.row_end - c.row_begin;
    return c.tiles[TQ_TILE_CTL(n) + 7] ? tail_first_raw(c) : TQ_TILE_NT(n);
}

inline int grid_for(int64_t work, int per_block) {
    int64_t g = (work + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > (int64_t)kSms * 64) g = kSms * 64;
    return (int)g;
}

}  // namespace tq
