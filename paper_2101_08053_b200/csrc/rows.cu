// Subsystem (4): sum-factorized row assembly written straight into CSR.
//
//  tq_wq_products <- the direction-wise contraction of sum_factor_row
//                    (src/assembly.py:245-252) for a coefficient-free direction
//  tq_row_counts / tq_fill_rows
//                 <- _interior_rows_batched + _Run.finish
//                    (src/assembly.py:409-449, 400-404): symmetrisation
//                    0.5*(M + M^T), exact-zero drop and sorted columns, fused
//                    into the row writer.
//
// Raw (unsymmetrised) row values come from one of two sources:
//   slot[i] <  0 : separable row, M_ij = a1[i1][j1] * a2[i2][j2]
//                  (interior test function, c == 1: the sum-factor contraction
//                  with a unit coefficient grid factorizes exactly);
//   slot[i] >= 0 : raw block raw[slot][(j1-i1+p1)*(2p2+1) + (j2-i2+p2)]
//                  written by the cut-row / general-coefficient kernels.
// The kept pattern is decided by value, (M_ij + M_ji) != 0, exactly the
// scipy CSR-add zero drop of the reference.
#include "common.cuh"

namespace tq {

__global__ void k_wq_products(tq_space1d s, tq_layout lay, const int32_t* __restrict__ first,
                              const double* __restrict__ vals, tq_rules rules, double* __restrict__ a) {
    const int p = s.p, W = 2 * p + 1;
    int64_t total = (int64_t)s.n * W;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int i = (int)(t / W), o = (int)(t % W);
        int j = i - p + o;
        double acc = 0.0;
        int k0 = rules.k0[i];
        if (k0 >= 0 && j >= s.ov_lo[i] && j <= s.ov_hi[i]) {
            int64_t w0 = rules.wptr[i], w1 = rules.wptr[i + 1];
            for (int64_t q = 0; q < w1 - w0; ++q) {
                int k = k0 + (int)q;
                int r = j - first[k];
                if (r >= 0 && r <= p) acc += rules.w[w0 + q] * vals[(int64_t)k * (p + 1) + r];
            }
        }
        a[t] = acc;
    }
}

struct RowGeom {
    int i1, i2, s_i, j1lo, j2lo, t1, t2;
};

__device__ inline RowGeom row_geom(const tq_rowctx& c, int r) {
    RowGeom g;
    int idx = c.active[r];
    g.i1 = idx / c.n2;
    g.i2 = idx - g.i1 * c.n2;
    g.s_i = c.slot[idx];
    g.j1lo = c.ov_lo1[g.i1];
    g.j2lo = c.ov_lo2[g.i2];
    g.t1 = c.ov_hi1[g.i1] - g.j1lo + 1;
    g.t2 = c.ov_hi2[g.i2] - g.j2lo + 1;
    return g;
}

// unsymmetrised value of row (i1,i2) at column (j1,j2)
__device__ __forceinline__ double raw_value(const tq_rowctx& c, int i1, int i2, int s_i, int j1, int j2) {
    const int W1 = 2 * c.p1 + 1, W2 = 2 * c.p2 + 1;
    const int o1 = j1 - i1 + c.p1, o2 = j2 - i2 + c.p2;
    if (s_i < 0) return __ldg(c.a1 + (int64_t)i1 * W1 + o1) * __ldg(c.a2 + (int64_t)i2 * W2 + o2);
    return __ldg(c.raw + (int64_t)s_i * (W1 * W2) + o1 * W2 + o2);
}

// symmetrised sum M_ij + M_ji for column j; returns col index or -1
__device__ __forceinline__ int entry(const tq_rowctx& c, const RowGeom& g, int e, double& v) {
    int q1 = e / g.t2;
    int j1 = g.j1lo + q1, j2 = g.j2lo + (e - q1 * g.t2);
    int jidx = j1 * c.n2 + j2;
    int col = __ldg(c.col_of + jidx);
    if (col < 0) return -1;
    int s_j = __ldg(c.slot + jidx);
    v = raw_value(c, g.i1, g.i2, g.s_i, j1, j2) + raw_value(c, j1, j2, s_j, g.i1, g.i2);
    return v != 0.0 ? col : -1;
}

constexpr int kTileRows = 64;

// counts: one thread per row for the deep test, the warp for the rest
__global__ void k_row_counts(tq_rowctx c, int32_t* __restrict__ counts) {
    __shared__ int todo[kTileRows];
    __shared__ int ntodo;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int R0 = c.row_begin + blockIdx.x * kTileRows; R0 < c.row_end; R0 += gridDim.x * kTileRows) {
        if (threadIdx.x == 0) ntodo = 0;
        __syncthreads();
        if (threadIdx.x < kTileRows) {
            int r = R0 + threadIdx.x;
            if (r < c.row_end) {
                int idx = c.active[r];
                if (c.deep && c.deep[idx]) {
                    int i1 = idx / c.n2, i2 = idx - (idx / c.n2) * c.n2;
                    counts[r - c.row_begin] = (c.ov_hi1[i1] - c.ov_lo1[i1] + 1) * (c.ov_hi2[i2] - c.ov_lo2[i2] + 1);
                } else {
                    todo[atomicAdd(&ntodo, 1)] = r;
                }
            }
        }
        __syncthreads();
        for (int q = warp; q < ntodo; q += nwarps) {
            int r = todo[q];
            RowGeom g = row_geom(c, r);
            int n = g.t1 * g.t2, cnt = 0;
            for (int e0 = 0; e0 < n; e0 += 32) {
                int e = e0 + lane;
                double v;
                bool keep = e < n && entry(c, g, e, v) >= 0;
                cnt += __popc(__ballot_sync(0xffffffffu, keep));
            }
            if (lane == 0) counts[r - c.row_begin] = cnt;
        }
        __syncthreads();
    }
}

// Tile fill: a block stages kTileRows rows -- metadata (phase 1) and, for
// deep rows, the 5(2P+1) direction factors and column bases (phase 2) -- in
// shared memory, then each warp emits whole CSR rows from shared memory with
// coalesced stores (phase 3).  Two dependent-load rounds per tile instead of
// three per row.
template <int P>
__global__ void __launch_bounds__(256) k_fill_tiles(tq_rowctx c, const int32_t* __restrict__ indptr,
                                                     int32_t* __restrict__ indices, double* __restrict__ data) {
    constexpr int W = 2 * P + 1;
    constexpr int kTileRows = P <= 6 ? 64 : 32;
    __shared__ int s_idx[kTileRows], s_pos[kTileRows], s_geo[kTileRows][4];  // j1lo j2lo t1 t2
    __shared__ unsigned char s_deep[kTileRows];
    __shared__ double s_f[kTileRows][4][W];   // A1 A1T A2 A2T
    __shared__ int s_cb[kTileRows][W];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    for (int R0 = c.row_begin + blockIdx.x * kTileRows; R0 < c.row_end; R0 += gridDim.x * kTileRows) {
        const int nr = min(kTileRows, c.row_end - R0);
        if (threadIdx.x < nr) {
            int t = threadIdx.x, r = R0 + t;
            int idx = __ldg(c.active + r);
            int i1 = idx / c.n2, i2 = idx - i1 * c.n2;
            s_idx[t] = idx;
            s_pos[t] = __ldg(indptr + (r - c.row_begin));
            s_deep[t] = c.deep ? __ldg(c.deep + idx) : 0;
            s_geo[t][0] = __ldg(c.ov_lo1 + i1);
            s_geo[t][1] = __ldg(c.ov_lo2 + i2);
            s_geo[t][2] = __ldg(c.ov_hi1 + i1) - s_geo[t][0] + 1;
            s_geo[t][3] = __ldg(c.ov_hi2 + i2) - s_geo[t][1] + 1;
        }
        __syncthreads();
        // phase 2: factors of deep rows, (row, lane-slot) spread over the block
        for (int q = threadIdx.x; q < nr * W; q += blockDim.x) {
            int t = q / W, o = q - t * W;
            if (!s_deep[t]) continue;
            int idx = s_idx[t];
            int i1 = idx / c.n2, i2 = idx - i1 * c.n2;
            int j1 = i1 - P + o, j2 = i2 - P + o;
            double A1 = 0.0, A1T = 0.0, A2 = 0.0, A2T = 0.0;
            int cb = 0;
            if (j1 >= s_geo[t][0] && j1 < s_geo[t][0] + s_geo[t][2]) {
                A1 = __ldg(c.a1 + (int64_t)i1 * W + o);
                A1T = __ldg(c.a1 + (int64_t)j1 * W + (2 * P - o));
                cb = __ldg(c.col_of + (int64_t)j1 * c.n2 + s_geo[t][1]);
            }
            if (j2 >= s_geo[t][1] && j2 < s_geo[t][1] + s_geo[t][3]) {
                A2 = __ldg(c.a2 + (int64_t)i2 * W + o);
                A2T = __ldg(c.a2 + (int64_t)j2 * W + (2 * P - o));
            }
            s_f[t][0][o] = A1; s_f[t][1][o] = A1T; s_f[t][2][o] = A2; s_f[t][3][o] = A2T;
            s_cb[t][o] = cb;
        }
        __syncthreads();
        // phase 3a: uniform tile (all rows deep with full windows) -> the tile
        // is one contiguous CSR span of nr*W*W entries: flat emit with
        // 16-byte vector stores (int4 indices, 2 x double2 values per quad)
        __shared__ int s_uniform;
        if (threadIdx.x == 0) {
            int u = 1;
            for (int t = 0; t < nr; ++t)
                u &= (s_deep[t] && s_geo[t][2] == W && s_geo[t][3] == W) ? 1 : 0;
            s_uniform = u;
        }
        __syncthreads();
        if (s_uniform) {
            constexpr int WW = W * W;
            const int n = nr * WW;
            const int pos0 = s_pos[0];
            const int head = (4 - (pos0 & 3)) & 3;
            auto coord = [&](int e, int& t, int& q1, int& q2) {
                t = e / WW;
                int rem = e - t * WW;
                q1 = rem / W;
                q2 = rem - q1 * W;
            };
            auto value = [&](int t, int q1, int q2) {
                return 0.5 * (s_f[t][0][q1] * s_f[t][2][q2] + s_f[t][1][q1] * s_f[t][3][q2]);
            };
            // ragged head and tail, scalar
            const int nq = (n - head) >> 2;
            const int tail0 = head + 4 * nq;
            for (int e = threadIdx.x; e < head + (n - tail0); e += blockDim.x) {
                int ee = e < head ? e : tail0 + (e - head);
                if (ee >= n) continue;
                int t, q1, q2;
                coord(ee, t, q1, q2);
                indices[pos0 + ee] = s_cb[t][q1] + q2;
                data[pos0 + ee] = value(t, q1, q2);
            }
            int4* idx4 = reinterpret_cast<int4*>(indices + pos0 + head);
            double2* dat2 = reinterpret_cast<double2*>(data + pos0 + head);
            for (int k = threadIdx.x; k < nq; k += blockDim.x) {
                int e = head + 4 * k;
                int t, q1, q2;
                coord(e, t, q1, q2);
                int c[4];
                double v[4];
#pragma unroll
                for (int z = 0; z < 4; ++z) {
                    c[z] = s_cb[t][q1] + q2;
                    v[z] = value(t, q1, q2);
                    if (++q2 == W) { q2 = 0; if (++q1 == W) { q1 = 0; ++t; } }
                }
                idx4[k] = make_int4(c[0], c[1], c[2], c[3]);
                dat2[2 * k] = make_double2(v[0], v[1]);
                dat2[2 * k + 1] = make_double2(v[2], v[3]);
            }
            __syncthreads();
            continue;
        }
        // phase 3: emit
        for (int t = warp; t < nr; t += nwarps) {
            int pos = s_pos[t];
            int j1lo = s_geo[t][0], j2lo = s_geo[t][1], t1 = s_geo[t][2], t2 = s_geo[t][3];
            int n = t1 * t2;
            if (s_deep[t]) {
                int idx = s_idx[t];
                int i1 = idx / c.n2, i2 = idx - i1 * c.n2;
                int off1 = j1lo - (i1 - P), off2 = j2lo - (i2 - P);
                for (int e = lane; e < n; e += 32) {
                    int q1 = (t2 == W) ? e / W : e / t2;
                    int q2 = e - q1 * t2;
                    int o1 = off1 + q1, o2 = off2 + q2;
                    double v = s_f[t][0][o1] * s_f[t][2][o2] + s_f[t][1][o1] * s_f[t][3][o2];
                    indices[pos + e] = s_cb[t][o1] + q2;
                    data[pos + e] = 0.5 * v;
                }
            } else {
                RowGeom g = row_geom(c, R0 + t);
                for (int e0 = 0; e0 < n; e0 += 32) {
                    int e = e0 + lane;
                    double v = 0.0;
                    int col = e < n ? entry(c, g, e, v) : -1;
                    unsigned m = __ballot_sync(0xffffffffu, col >= 0);
                    if (col >= 0) {
                        int at = pos + __popc(m & lt);
                        indices[at] = col;
                        data[at] = 0.5 * v;
                    }
                    pos += __popc(m);
                }
            }
        }
        __syncthreads();
    }
}

// generic fill (unequal degrees or no separable factors)
__global__ void k_fill_rows(tq_rowctx c, const int32_t* __restrict__ indptr, int32_t* __restrict__ indices,
                            double* __restrict__ data) {
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    for (int r = c.row_begin + blockIdx.x * wpb + (threadIdx.x >> 5); r < c.row_end; r += gridDim.x * wpb) {
        RowGeom g = row_geom(c, r);
        int pos = indptr[r - c.row_begin];
        int n = g.t1 * g.t2;
        for (int e0 = 0; e0 < n; e0 += 32) {
            int e = e0 + lane;
            double v = 0.0;
            int col = e < n ? entry(c, g, e, v) : -1;
            unsigned m = __ballot_sync(0xffffffffu, col >= 0);
            if (col >= 0) {
                int at = pos + __popc(m & lt);
                indices[at] = col;
                data[at] = 0.5 * v;
            }
            pos += __popc(m);
        }
    }
}

// 1-D positivity of a direction's factors over each window
__global__ void k_pos(const double* __restrict__ a, int n, int p, const int32_t* __restrict__ ov_lo,
                      const int32_t* __restrict__ ov_hi, int8_t* __restrict__ pos) {
    const int W = 2 * p + 1;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        bool ok = true;
        for (int j = ov_lo[i]; j <= ov_hi[i]; ++j)
            ok = ok && a[(int64_t)i * W + (j - i + p)] > 0.0 && a[(int64_t)j * W + (i - j + p)] > 0.0;
        pos[i] = ok;
    }
}

__global__ void k_deep_init(tq_rowctx c, const int8_t* __restrict__ fc, const int8_t* __restrict__ pos1,
                            const int8_t* __restrict__ pos2, int8_t* __restrict__ deep) {
    int64_t total = (int64_t)c.n1 * c.n2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int i1 = (int)(t / c.n2), i2 = (int)(t - (int64_t)i1 * c.n2);
        deep[t] = (fc[t] == TQ_INTERIOR && c.slot[t] < 0 && pos1[i1] && pos2[i2]) ? 1 : 0;
    }
}

// a raw row j spoils the fast path of every row i with j in window(i), i.e.
// every i in window(j) (the overlap relation is symmetric)
__global__ void k_deep_clear(tq_rowctx c, const int32_t* __restrict__ raw_rows, int nraw, int8_t* deep) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nraw; r += gridDim.x * blockDim.x) {
        int idx = raw_rows[r];
        int j1 = idx / c.n2, j2 = idx - j1 * c.n2;
        for (int i1 = c.ov_lo1[j1]; i1 <= c.ov_hi1[j1]; ++i1)
            for (int i2 = c.ov_lo2[j2]; i2 <= c.ov_hi2[j2]; ++i2) deep[(int64_t)i1 * c.n2 + i2] = 0;
    }
}

}  // namespace tq

using namespace tq;

extern "C" int tq_wq_products(tq_space1d s, tq_layout lay, const int32_t* first, const double* vals,
                              tq_rules rules, double* a, void* stream) {
    int64_t total = (int64_t)s.n * (2 * s.p + 1);
    if (total == 0) return TQ_OK;
    k_wq_products<<<grid_for(total, 128), 128, 0, S(stream)>>>(s, lay, first, vals, rules, a); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_wq_products");
    return TQ_OK;
}

extern "C" int tq_row_counts(tq_rowctx c, int32_t* counts, void* stream) {
    int nrows = c.row_end - c.row_begin;
    if (nrows <= 0) return TQ_OK;
    int grid = (int)std::min<int64_t>((nrows + kTileRows - 1) / kTileRows, (int64_t)kSms * 16);
    k_row_counts<<<grid, 256, 0, S(stream)>>>(c, counts); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_row_counts");
    return TQ_OK;
}

extern "C" int tq_fill_rows(tq_rowctx c, const int32_t* indptr, int32_t* indices, double* data,
                            void* stream) {
    int nrows = c.row_end - c.row_begin;
    if (nrows <= 0) return TQ_OK;
    int P = (c.p1 == c.p2 && c.a1 && c.deep) ? c.p1 : 0;
    int tr = P <= 6 ? 64 : 32;
    auto wave = [&](const void* fn) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0);
        int64_t full = (int64_t)kSms * std::max(per_sm, 1);
        return (int)std::min<int64_t>((nrows + tr - 1) / tr, full);
    };
    switch (P) {
#define CASE(Q) case Q: k_fill_tiles<Q><<<wave((const void*)k_fill_tiles<Q>), 256, 0, S(stream)>>>(c, indptr, indices, data); ::tq::note_launch(); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
        default: {
            int grid = (int)std::min<int64_t>((nrows + 7) / 8, (int64_t)kSms * 32);
            k_fill_rows<<<grid, 256, 0, S(stream)>>>(c, indptr, indices, data); ::tq::note_launch();
        }
    }
    TQ_LAUNCH_CHECK("k_fill_rows");
    return TQ_OK;
}

extern "C" int tq_deep_flags(tq_rowctx c, const int8_t* func_class, const int32_t* raw_rows, int32_t nraw,
                             int8_t* deep, void* stream) {
    int64_t nf = (int64_t)c.n1 * c.n2;
    if (!c.a1 || !c.a2) {
        TQ_CUDA(cudaMemsetAsync(deep, 0, nf, S(stream)));
        return TQ_OK;
    }
    int8_t* pos = nullptr;
    TQ_CUDA(cudaMallocAsync(&pos, c.n1 + c.n2, S(stream)));
    k_pos<<<grid_for(c.n1, 128), 128, 0, S(stream)>>>(c.a1, c.n1, c.p1, c.ov_lo1, c.ov_hi1, pos); ::tq::note_launch();
    k_pos<<<grid_for(c.n2, 128), 128, 0, S(stream)>>>(c.a2, c.n2, c.p2, c.ov_lo2, c.ov_hi2, pos + c.n1); ::tq::note_launch();
    k_deep_init<<<grid_for(nf, 256), 256, 0, S(stream)>>>(c, func_class, pos, pos + c.n1, deep); ::tq::note_launch();
    if (nraw > 0) k_deep_clear<<<grid_for(nraw, 128), 128, 0, S(stream)>>>(c, raw_rows, nraw, deep); ::tq::note_launch();
    TQ_LAUNCH_CHECK("deep flags");
    TQ_CUDA(cudaFreeAsync(pos, S(stream)));
    return TQ_OK;
}
