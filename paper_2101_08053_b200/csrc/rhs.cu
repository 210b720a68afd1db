// L2 projection: right-hand side and error reduction on the GPU.
//
//  tq_rhs      <- assemble_rhs  src/projection.py:101-145
//     b_i = sum over interior elements of (p+2)^2-point Gauss f c w B_i
//           + sum over cut-cell points of f c w B_i.
//     Sum factorized: T[(e1,g1)][i2] = sum_{e2 in supp i2, (e1,e2) interior}
//     sum_g2 F w V2 (stage 1), b_i = sum_{e1 in supp i1} sum_g1 V1 T (stage 2);
//     cut rows then gather their cut-cell points.  Row-gather, no atomics.
//  tq_l2_parts <- l2_error      src/projection.py:221-260
//     (num, den) partial sums per block, reduced in a fixed order.
#include "common.cuh"

namespace tq {

// f(x, y) of a device target: sum_k coef_k phi(ax x + bx) psi(ay y + by)
__device__ inline double phi(int kind, double t) {
    switch (kind) {
        case 1: return sin(t);
        case 2: return cos(t);
        case 3: return exp(t);
        default: return 1.0;
    }
}

__device__ inline double target_value(const tq_target& f, double x, double y) {
    double acc = 0.0;
    for (int k = 0; k < f.nterms; ++k) {
        const double* t = f.terms + 7 * k;
        acc += t[0] * phi((int)t[1], t[2] * x + t[3]) * phi((int)t[4], t[5] * y + t[6]);
    }
    return acc;
}

// f at Gauss point (r1, r2) = (x, y) of the tensor grid, per target kind
__device__ __forceinline__ double target_at(const tq_projctx& c, int64_t r1, int64_t r2, double x, double y) {
    const tq_target& f = c.target;
    if (f.kind == 0) return f.grid[r1 * f.ld + r2];
    if (f.kind == 2) {
        const int64_t n2 = (int64_t)c.nel2 * c.g2n, st = f.ld + n2;
        double acc = 0.0;
        for (int k = 0; k < f.nterms; ++k) acc += f.terms[7 * k] * f.grid[k * st + r1] * f.grid[k * st + f.ld + r2];
        return acc;
    }
    return target_value(f, x, y);
}

// kind-2 tables: the x and y factors of every term at the Gauss coordinates
__global__ void k_target_tables(tq_target f, const double* __restrict__ x1, int64_t n1,
                                const double* __restrict__ x2, int64_t n2, double* __restrict__ out) {
    const int64_t st = n1 + n2, total = (int64_t)f.nterms * st;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(t / st);
        const int64_t i = t - k * st;
        const double* tm = f.terms + 7 * k;
        out[t] = i < n1 ? phi((int)tm[1], tm[2] * x1[i] + tm[3]) : phi((int)tm[4], tm[5] * x2[i - n1] + tm[6]);
    }
}

// stage 1: one block per (point row r1, chunk of i2 functions)
constexpr int kChunk = 128;

__global__ void k_rhs_stage1(tq_projctx c, double* __restrict__ T) {
    extern __shared__ double sF[];
    const int g = c.g1n, g2n = c.g2n, q2 = c.p2 + 1;
    const int nchunks = (c.n2 + kChunk - 1) / kChunk;
    for (int64_t blk = blockIdx.x; blk < (int64_t)c.nel1 * g * nchunks; blk += gridDim.x) {
        const int r1 = (int)(blk / nchunks), ch = (int)(blk % nchunks);
        const int e1 = r1 / g;
        const int I0 = ch * kChunk, I1 = min(I0 + kChunk, c.n2) - 1;
        const int ea = c.el_first2[I0], eb = c.el_last2[I1];
        const double x = c.x1[r1], w1 = c.w1[r1];
        const int npts = (eb - ea + 1) * g2n;
        __syncthreads();
        for (int q = threadIdx.x; q < npts; q += blockDim.x) {
            int e2 = ea + q / g2n, g2 = q - (q / g2n) * g2n;
            double v = 0.0;
            if (c.elem_class[(int64_t)e1 * c.nel2 + e2] == TQ_INTERIOR) {
                int64_t p2 = (int64_t)e2 * g2n + g2;
                double y = c.x2[p2];
                double f = target_at(c, r1, p2, x, y);
                double cc = c.cgrid ? c.cgrid[(int64_t)r1 * c.cld + p2] : 1.0;
                v = f * cc * (w1 * c.w2[p2]);
            }
            sF[q] = v;
        }
        __syncthreads();
        for (int i2 = I0 + threadIdx.x; i2 <= I1; i2 += blockDim.x) {
            double acc = 0.0;
            for (int e2 = c.el_first2[i2]; e2 <= c.el_last2[i2]; ++e2) {
                int a2 = i2 - (c.espan2[e2] - c.p2);
                const double* V = c.v2 + (int64_t)e2 * g2n * q2;
                const double* F = sF + (e2 - ea) * g2n;
                for (int g2 = 0; g2 < g2n; ++g2) acc += F[g2] * V[g2 * q2 + a2];
            }
            T[(int64_t)r1 * c.n2 + i2] = acc;
        }
    }
}

// stage 2: one thread per active row
__global__ void k_rhs_stage2(tq_projctx c, const double* __restrict__ T, double* __restrict__ b) {
    const int g = c.g1n, q1 = c.p1 + 1;
    for (int r = c.row_begin + blockIdx.x * blockDim.x + threadIdx.x; r < c.row_end; r += gridDim.x * blockDim.x) {
        int idx = c.active[r];
        int i1 = idx / c.n2, i2 = idx - (idx / c.n2) * c.n2;
        double acc = 0.0;
        for (int e1 = c.el_first1[i1]; e1 <= c.el_last1[i1]; ++e1) {
            int a1 = i1 - (c.espan1[e1] - c.p1);
            const double* V = c.v1 + (int64_t)e1 * g * q1;
            for (int g1 = 0; g1 < g; ++g1) acc += V[g1 * q1 + a1] * T[((int64_t)e1 * g + g1) * c.n2 + i2];
        }
        b[r - c.row_begin] = acc;
    }
}

// cut-cell points of the cut rows: b_i += sum f c w B_i (warp per row)
__global__ void k_rhs_cut(tq_projctx c, const int32_t* __restrict__ rows, int nrows, double* __restrict__ b) {
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int q1 = c.p1 + 1, q2 = c.p2 + 1;
    for (int k = blockIdx.x * wpb + (threadIdx.x >> 5); k < nrows; k += gridDim.x * wpb) {
        int r = rows[k];
        int idx = c.active[r];
        int i1 = idx / c.n2, i2 = idx - (idx / c.n2) * c.n2;
        int ea1 = max(c.el_first1[i1] - 1, 0), eb1 = min(c.el_last1[i1] + 1, c.nel1 - 1);
        int ea2 = max(c.el_first2[i2] - 1, 0), eb2 = min(c.el_last2[i2] + 1, c.nel2 - 1);
        double acc = 0.0;
        for (int e1 = ea1; e1 <= eb1; ++e1)
            for (int e2 = ea2; e2 <= eb2; ++e2) {
                int id = c.cutidx[(int64_t)e1 * c.nel2 + e2];
                if (id < 0) continue;
                for (int64_t pt = c.cut_ptr[id] + lane; pt < c.cut_ptr[id + 1]; pt += 32) {
                    int a1 = i1 - c.cfirst1[pt], a2 = i2 - c.cfirst2[pt];
                    if (a1 < 0 || a1 > c.p1 || a2 < 0 || a2 > c.p2) continue;
                    acc += c.cut_fcw[pt] * (c.cvals1[pt * q1 + a1] * c.cvals2[pt * q2 + a2]);
                }
            }
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) b[r - c.row_begin] += acc;
    }
}

// per-point target values f(P) (device target) times weight
__global__ void k_target_points(tq_target f, const double* P, const double* w, int64_t n, double* out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = target_value(f, P[2 * t], P[2 * t + 1]) * (w ? w[t] : 1.0);
}

// L2 error parts over interior elements [e_begin, e_end) (row-major element
// index) and cut points: block partials (num, den) -> parts[2*block]
__global__ void k_l2_elements(tq_projctx c, const double* __restrict__ C, int64_t e_begin, int64_t e_end,
                              double* __restrict__ parts) {
    __shared__ double red[2][32];
    const int g1n = c.g1n, g2n = c.g2n, q1 = c.p1 + 1, q2 = c.p2 + 1;
    double num = 0.0, den = 0.0;
    for (int64_t t = e_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < e_end;
         t += (int64_t)gridDim.x * blockDim.x) {
        int e1 = (int)(t / c.nel2), e2 = (int)(t - (t / c.nel2) * c.nel2);
        if (c.elem_class[t] != TQ_INTERIOR) continue;
        int f1 = c.espan1[e1] - c.p1, f2 = c.espan2[e2] - c.p2;
        const double* V1 = c.v1 + (int64_t)e1 * g1n * q1;
        const double* V2 = c.v2 + (int64_t)e2 * g2n * q2;
        for (int g1 = 0; g1 < g1n; ++g1) {
            double x = c.x1[(int64_t)e1 * g1n + g1], w1 = c.w1[(int64_t)e1 * g1n + g1];
            for (int g2 = 0; g2 < g2n; ++g2) {
                double y = c.x2[(int64_t)e2 * g2n + g2], w2 = c.w2[(int64_t)e2 * g2n + g2];
                double uh = 0.0;
                for (int a1 = 0; a1 < q1; ++a1) {
                    double s = 0.0;
                    const double* Crow = C + (int64_t)(f1 + a1) * c.n2 + f2;
                    for (int a2 = 0; a2 < q2; ++a2) s += Crow[a2] * V2[g2 * q2 + a2];
                    uh += V1[g1 * q1 + a1] * s;
                }
                int64_t pr = (int64_t)e1 * g1n + g1, pc = (int64_t)e2 * g2n + g2;
                double f = target_at(c, pr, pc, x, y);
                double w = w1 * w2;
                num += w * (uh - f) * (uh - f);
                den += w * f * f;
            }
        }
    }
    for (int off = 16; off > 0; off >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, off);
        den += __shfl_xor_sync(0xffffffffu, den, off);
    }
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { red[0][w] = num; red[1][w] = den; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, d = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { a += red[0][k]; d += red[1][k]; }
        parts[2 * blockIdx.x] = a;
        parts[2 * blockIdx.x + 1] = d;
    }
}

// The same sums for p1 == p2 == P: a block takes 128 consecutive elements
// (row-major), stages their direction-2 tables (values, points, weights and,
// for a kind-2 target, the y factors) in shared memory with coalesced loads,
// and a thread sums one element: per g2 the contraction S[a1] = sum_a2 C V2
// of its coefficient block (registers), then u_h = sum_a1 V1 S per g1 --
// the terms of k_l2_elements (u_h, f, w exactly as there; the partial sums
// in another order).
constexpr int kL2Chunk = 64;
// per-element staging stride (doubles): odd, so the 32 threads' rows fall on
// distinct bank pairs (an even stride of 56 at P = 4 put every lane of a
// half-warp on the same two banks: 16-way conflicts on every table read)
__host__ __device__ constexpr int l2_stride(int P) { return ((P + 3) * (P + 1) + 3 * (P + 3)) | 1; }

template <int P>
__global__ void __launch_bounds__(kL2Chunk, 8) k_l2_elements_s(tq_projctx c, const double* __restrict__ C,
                                                                int64_t e_begin, int64_t e_end,
                                                                double* __restrict__ parts) {
    extern __shared__ double sm[];
    __shared__ double red[2][kL2Chunk / 32];
    constexpr int Q = P + 1, G = P + 3, ST = l2_stride(P);      // per element: V2, y, w2, psi (one term)
    constexpr int R1 = G * Q + 3 * G;                            // per element row: V1, x, w1, phi
    const bool sep = c.target.kind == 2 && c.target.nterms == 1;
    double* rows = sm + kL2Chunk * ST;                           // the chunk's (at most two) element rows
    double num = 0.0, den = 0.0;
    for (int64_t t0 = e_begin + (int64_t)blockIdx.x * kL2Chunk; t0 < e_end; t0 += (int64_t)gridDim.x * kL2Chunk) {
        const int nin = (int)(e_end - t0 < kL2Chunk ? e_end - t0 : kL2Chunk);
        const int e1a = (int)(t0 / c.nel2), e2a = (int)(t0 - (int64_t)e1a * c.nel2);
        __syncthreads();
        // stage the chunk's direction-2 tables (slot j: element t0 + j) and its rows' direction-1 tables
        for (int q = threadIdx.x; q < nin * (G * Q); q += kL2Chunk) {
            const int j = q / (G * Q), k = q - j * (G * Q);
            int e2 = e2a + j;
            if (e2 >= c.nel2) e2 -= c.nel2;
            sm[j * ST + k] = c.v2[(int64_t)e2 * G * Q + k];
        }
        for (int q = threadIdx.x; q < nin * G; q += kL2Chunk) {
            const int j = q / G, g = q - j * G;
            int e2 = e2a + j;
            if (e2 >= c.nel2) e2 -= c.nel2;
            const int64_t pc = (int64_t)e2 * G + g;
            double* o = sm + j * ST + G * Q;
            o[g] = c.x2[pc];
            o[G + g] = c.w2[pc];
            o[2 * G + g] = sep ? c.target.grid[c.target.ld + pc] : 0.0;
        }
        for (int q = threadIdx.x; q < 2 * R1; q += kL2Chunk) {
            const int rr = q / R1, k = q - rr * R1;
            const int e1 = e1a + rr;
            if (e1 >= c.nel1) continue;
            double v;
            if (k < G * Q) v = c.v1[(int64_t)e1 * G * Q + k];
            else if (k < G * Q + G) v = c.x1[(int64_t)e1 * G + (k - G * Q)];
            else if (k < G * Q + 2 * G) v = c.w1[(int64_t)e1 * G + (k - G * Q - G)];
            else v = sep ? c.target.grid[(int64_t)e1 * G + (k - G * Q - 2 * G)] : 0.0;
            rows[rr * R1 + k] = v;
        }
        __syncthreads();
        const int j = threadIdx.x;
        if (j >= nin) continue;
        const int64_t t = t0 + j;
        if (c.elem_class[t] != TQ_INTERIOR) continue;
        const int e1 = (int)(t / c.nel2), e2 = (int)(t - (t / c.nel2) * c.nel2);
        const int f1 = c.espan1[e1] - P, f2 = c.espan2[e2] - P;
        const double* r1 = rows + (e1 - e1a) * R1;
        const double* s2 = sm + j * ST;
        double cb[Q][Q];
#pragma unroll
        for (int a1 = 0; a1 < Q; ++a1)
#pragma unroll
            for (int a2 = 0; a2 < Q; ++a2) cb[a1][a2] = C[(int64_t)(f1 + a1) * c.n2 + f2 + a2];
        const double tk = sep ? c.target.terms[0] : 0.0;
#pragma unroll 1
        for (int g2 = 0; g2 < G; ++g2) {
            double S[Q];
#pragma unroll
            for (int a1 = 0; a1 < Q; ++a1) {
                double sa = 0.0;
#pragma unroll
                for (int a2 = 0; a2 < Q; ++a2) sa += cb[a1][a2] * s2[g2 * Q + a2];
                S[a1] = sa;
            }
            const double y = s2[G * Q + g2], w2 = s2[G * Q + G + g2], psi = s2[G * Q + 2 * G + g2];
            const int64_t pc = (int64_t)e2 * G + g2;
#pragma unroll
            for (int g1 = 0; g1 < G; ++g1) {
                double uh = 0.0;
#pragma unroll
                for (int a1 = 0; a1 < Q; ++a1) uh += r1[g1 * Q + a1] * S[a1];
                double f;
                if (sep) {
                    double acc = 0.0;
                    acc += tk * r1[G * Q + 2 * G + g1] * psi;
                    f = acc;
                } else {
                    f = target_at(c, (int64_t)e1 * G + g1, pc, r1[G * Q + g1], y);
                }
                const double w = r1[G * Q + G + g1] * w2;
                num += w * (uh - f) * (uh - f);
                den += w * f * f;
            }
        }
    }
    for (int off = 16; off > 0; off >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, off);
        den += __shfl_xor_sync(0xffffffffu, den, off);
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { red[0][w] = num; red[1][w] = den; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, d = 0.0;
        for (int k = 0; k < kL2Chunk / 32; ++k) { a += red[0][k]; d += red[1][k]; }
        parts[2 * blockIdx.x] = a;
        parts[2 * blockIdx.x + 1] = d;
    }
}

// Tiled form of k_l2_elements_s: a block takes a tile of kL2Rows element rows
// x kL2Chunk element columns, stages the columns' direction-2 tables ONCE for
// the tile's rows (k_l2_elements_s re-staged them for every row: the staging
// loads, not the sums, set its time), the rows' direction-1 tables and the
// tile's coefficient window, and two threads walk each column down the
// tile's rows (alternate rows; 224 registers, two blocks per SM: measured
// best against 168 / 128-register bounds).  Per element the terms and
// their order are those of k_l2_elements_s; only the order of the partial
// sums over elements changes.
constexpr int kL2Rows = 16, kL2Threads = 2 * kL2Chunk;
#ifndef TQ_L2_MINB
#define TQ_L2_MINB 2
#endif

template <int P>
__global__ void __launch_bounds__(kL2Threads, TQ_L2_MINB) k_l2_tiles(tq_projctx c, const double* __restrict__ C,
                                                         int64_t e_begin, int64_t e_end, double* __restrict__ parts) {
    extern __shared__ double sm[];
    __shared__ double red[2][kL2Threads / 32];
    constexpr int Q = P + 1, G = P + 3, ST = l2_stride(P);
    constexpr int R1 = G * Q + 3 * G;                            // per element row: V1, x, w1, phi
    const bool sep = c.target.kind == 2 && c.target.nterms == 1;
    double* rows = sm + kL2Chunk * ST;                           // [kL2Rows][R1]
    // the tile's coefficient window: rows f1(e1a) .. f1(last) + P, columns
    // f2(e2a) .. f2(last) + P (staged when it fits; else read from C)
    constexpr int CR = kL2Rows + P, CC = kL2Chunk + P, LDC = CC | 1;
    double* cs = rows + kL2Rows * R1;                            // [CR][LDC]
    double num = 0.0, den = 0.0;
    const int r_first = (int)(e_begin / c.nel2), r_last = (int)((e_end - 1) / c.nel2);
    const int nrt = (r_last - r_first + kL2Rows) / kL2Rows, nct = (c.nel2 + kL2Chunk - 1) / kL2Chunk;
    const int64_t ntiles = (int64_t)nrt * nct;
    const double tk = sep ? c.target.terms[0] : 0.0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int rt = (int)(tile / nct), ct = (int)(tile - (int64_t)rt * nct);
        const int e1a = r_first + rt * kL2Rows, e2a = ct * kL2Chunk;
        const int nr = min(kL2Rows, r_last + 1 - e1a), ncol = min(kL2Chunk, c.nel2 - e2a);
        __syncthreads();
        for (int q = threadIdx.x; q < ncol * (G * Q); q += kL2Threads) {
            const int j = q / (G * Q), k = q - j * (G * Q);
            sm[j * ST + k] = c.v2[(int64_t)(e2a + j) * G * Q + k];
        }
        for (int q = threadIdx.x; q < ncol * G; q += kL2Threads) {
            const int j = q / G, g = q - j * G;
            const int64_t pc = (int64_t)(e2a + j) * G + g;
            double* o = sm + j * ST + G * Q;
            o[g] = c.x2[pc];
            o[G + g] = c.w2[pc];
            o[2 * G + g] = sep ? c.target.grid[c.target.ld + pc] : 0.0;
        }
        for (int q = threadIdx.x; q < nr * R1; q += kL2Threads) {
            const int rr = q / R1, k = q - rr * R1;
            const int e1 = e1a + rr;
            double v;
            if (k < G * Q) v = c.v1[(int64_t)e1 * G * Q + k];
            else if (k < G * Q + G) v = c.x1[(int64_t)e1 * G + (k - G * Q)];
            else if (k < G * Q + 2 * G) v = c.w1[(int64_t)e1 * G + (k - G * Q - G)];
            else v = sep ? c.target.grid[(int64_t)e1 * G + (k - G * Q - 2 * G)] : 0.0;
            rows[rr * R1 + k] = v;
        }
        const int r0 = c.espan1[e1a] - P, rn = c.espan1[e1a + nr - 1] + 1 - r0;
        const int c0 = c.espan2[e2a] - P, cn = c.espan2[e2a + ncol - 1] + 1 - c0;
        const bool staged = rn <= CR && cn <= CC;                   // (uniform across the block)
        if (staged)
            for (int q = threadIdx.x; q < rn * cn; q += kL2Threads) {
                const int rr = q / cn, cc = q - rr * cn;
                cs[rr * LDC + cc] = C[(int64_t)(r0 + rr) * c.n2 + c0 + cc];
            }
        __syncthreads();
        // two threads per column, alternate rows
        const int j = threadIdx.x % kL2Chunk, h = threadIdx.x / kL2Chunk;
        if (j >= ncol) continue;
        const int e2 = e2a + j;
        const int f2 = c.espan2[e2] - P;
        const double* s2 = sm + j * ST;
        for (int rr = h; rr < nr; rr += kL2Threads / kL2Chunk) {
            const int e1 = e1a + rr;
            const int64_t t = (int64_t)e1 * c.nel2 + e2;
            if (t < e_begin || t >= e_end || c.elem_class[t] != TQ_INTERIOR) continue;
            const int f1 = c.espan1[e1] - P;
            const double* r1 = rows + rr * R1;
            double cb[Q][Q];
            if (staged) {
                const double* cw = cs + (f1 - r0) * LDC + (f2 - c0);
#pragma unroll
                for (int a1 = 0; a1 < Q; ++a1)
#pragma unroll
                    for (int a2 = 0; a2 < Q; ++a2) cb[a1][a2] = cw[a1 * LDC + a2];
            } else {
#pragma unroll
                for (int a1 = 0; a1 < Q; ++a1)
#pragma unroll
                    for (int a2 = 0; a2 < Q; ++a2) cb[a1][a2] = C[(int64_t)(f1 + a1) * c.n2 + f2 + a2];
            }
#pragma unroll 1
            for (int g2 = 0; g2 < G; ++g2) {
                double S[Q];
#pragma unroll
                for (int a1 = 0; a1 < Q; ++a1) {
                    double sa = 0.0;
#pragma unroll
                    for (int a2 = 0; a2 < Q; ++a2) sa += cb[a1][a2] * s2[g2 * Q + a2];
                    S[a1] = sa;
                }
                const double y = s2[G * Q + g2], w2 = s2[G * Q + G + g2], psi = s2[G * Q + 2 * G + g2];
                const int64_t pc = (int64_t)e2 * G + g2;
#pragma unroll
                for (int g1 = 0; g1 < G; ++g1) {
                    double uh = 0.0;
#pragma unroll
                    for (int a1 = 0; a1 < Q; ++a1) uh += r1[g1 * Q + a1] * S[a1];
                    double f;
                    if (sep) {
                        double acc = 0.0;
                        acc += tk * r1[G * Q + 2 * G + g1] * psi;
                        f = acc;
                    } else {
                        f = target_at(c, (int64_t)e1 * G + g1, pc, r1[G * Q + g1], y);
                    }
                    const double w = r1[G * Q + G + g1] * w2;
                    num += w * (uh - f) * (uh - f);
                    den += w * f * f;
                }
            }
        }
    }
    for (int off = 16; off > 0; off >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, off);
        den += __shfl_xor_sync(0xffffffffu, den, off);
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { red[0][w] = num; red[1][w] = den; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, d = 0.0;
        for (int k = 0; k < kL2Threads / 32; ++k) { a += red[0][k]; d += red[1][k]; }
        parts[2 * blockIdx.x] = a;
        parts[2 * blockIdx.x + 1] = d;
    }
}

// ---- separable fast path of the RHS (kind-2 target, c == 1) ---------------
// f = sum_k t_k phi_k(x) psi_k(y) and the Gauss rule is a tensor rule, so
//   b_i = sum_k sum_{e1, e2 interior} Q1_k[e1][a1] Q2_k[e2][a2],
//   Q1_k[e][a] = sum_g V1[e][g][a] (t_k phi_k(x_eg) w_eg),
//   Q2_k[e][a] = sum_g V2[e][g][a] (psi_k(y_eg) w_eg)
// (the same terms as the two-stage kernels, grouped per 1-D element); a row
// whose support is all interior is the product of two 1-D sums
// A_k[i] = sum_{e in supp i} Q_k[e][i - f(e)].

// Q tables: one thread per (term, direction, element, local function)
__global__ void k_rhs_q(tq_projctx c, double* __restrict__ Q1, double* __restrict__ Q2) {
    const tq_target& f = c.target;
    const int q1 = c.p1 + 1, q2 = c.p2 + 1;
    const int64_t n1tot = (int64_t)c.nel1 * q1, n2tot = (int64_t)c.nel2 * q2;
    const int64_t per = n1tot + n2tot, st = f.ld + (int64_t)c.nel2 * c.g2n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)f.nterms * per;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(t / per);
        const int64_t u = t - k * per;
        const double* tab = f.grid + k * st;
        double acc = 0.0;
        if (u < n1tot) {
            const int e = (int)(u / q1), a = (int)(u - (int64_t)e * q1);
            const double tk = f.terms[7 * k];
            for (int g = 0; g < c.g1n; ++g) {
                const int64_t pt = (int64_t)e * c.g1n + g;
                acc += c.v1[pt * q1 + a] * ((tk * tab[pt]) * c.w1[pt]);
            }
            Q1[(int64_t)k * n1tot + u] = acc;
        } else {
            const int64_t v = u - n1tot;
            const int e = (int)(v / q2), a = (int)(v - (int64_t)e * q2);
            for (int g = 0; g < c.g2n; ++g) {
                const int64_t pt = (int64_t)e * c.g2n + g;
                acc += c.v2[pt * q2 + a] * (tab[f.ld + pt] * c.w2[pt]);
            }
            Q2[(int64_t)k * n2tot + v] = acc;
        }
    }
}

// 1-D support sums A_k[i] per direction: thread per (term, direction, function)
__global__ void k_rhs_a(tq_projctx c, const double* __restrict__ Q1, const double* __restrict__ Q2,
                        double* __restrict__ A1, double* __restrict__ A2) {
    const int q1 = c.p1 + 1, q2 = c.p2 + 1;
    const int64_t per = (int64_t)c.n1 + c.n2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)c.target.nterms * per;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(t / per);
        const int64_t u = t - k * per;
        double acc = 0.0;
        if (u < c.n1) {
            const int i = (int)u;
            const double* Q = Q1 + (int64_t)k * c.nel1 * q1;
            for (int e = c.el_first1[i]; e <= c.el_last1[i]; ++e) acc += Q[(int64_t)e * q1 + (i - (c.espan1[e] - c.p1))];
            A1[(int64_t)k * c.n1 + i] = acc;
        } else {
            const int i = (int)(u - c.n1);
            const double* Q = Q2 + (int64_t)k * c.nel2 * q2;
            for (int e = c.el_first2[i]; e <= c.el_last2[i]; ++e) acc += Q[(int64_t)e * q2 + (i - (c.espan2[e] - c.p2))];
            A2[(int64_t)k * c.n2 + i] = acc;
        }
    }
}

// rows: product of the 1-D sums when the support is all interior, else the
// masked element double sum
__global__ void k_rhs_sep_rows(tq_projctx c, const int8_t* __restrict__ fclass, const double* __restrict__ Q1,
                               const double* __restrict__ Q2, const double* __restrict__ A1,
                               const double* __restrict__ A2, double* __restrict__ b) {
    const int q1 = c.p1 + 1, q2 = c.p2 + 1;
    for (int r = c.row_begin + blockIdx.x * blockDim.x + threadIdx.x; r < c.row_end; r += gridDim.x * blockDim.x) {
        const int idx = c.active[r];
        const int i1 = idx / c.n2, i2 = idx - (idx / c.n2) * c.n2;
        double acc = 0.0;
        if (fclass[idx] == TQ_INTERIOR) {
            for (int k = 0; k < c.target.nterms; ++k) acc += A1[(int64_t)k * c.n1 + i1] * A2[(int64_t)k * c.n2 + i2];
        } else {
            for (int k = 0; k < c.target.nterms; ++k) {
                const double* Qa = Q1 + (int64_t)k * c.nel1 * q1;
                const double* Qb = Q2 + (int64_t)k * c.nel2 * q2;
                for (int e1 = c.el_first1[i1]; e1 <= c.el_last1[i1]; ++e1) {
                    const double v1 = Qa[(int64_t)e1 * q1 + (i1 - (c.espan1[e1] - c.p1))];
                    double s = 0.0;
                    for (int e2 = c.el_first2[i2]; e2 <= c.el_last2[i2]; ++e2)
                        if (c.elem_class[(int64_t)e1 * c.nel2 + e2] == TQ_INTERIOR)
                            s += Qb[(int64_t)e2 * q2 + (i2 - (c.espan2[e2] - c.p2))];
                    acc += v1 * s;
                }
            }
        }
        b[r - c.row_begin] = acc;
    }
}

__global__ void k_l2_cut(tq_projctx c, const double* __restrict__ C, int64_t p_begin, int64_t p_end,
                         const double* __restrict__ fpts, double* __restrict__ parts) {
    __shared__ double red[2][32];
    const int q1 = c.p1 + 1, q2 = c.p2 + 1;
    double num = 0.0, den = 0.0;
    for (int64_t pt = p_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pt < p_end;
         pt += (int64_t)gridDim.x * blockDim.x) {
        int f1 = c.cfirst1[pt], f2 = c.cfirst2[pt];
        double uh = 0.0;
        for (int a1 = 0; a1 < q1; ++a1) {
            double s = 0.0;
            for (int a2 = 0; a2 < q2; ++a2) s += C[(int64_t)(f1 + a1) * c.n2 + f2 + a2] * c.cvals2[pt * q2 + a2];
            uh += c.cvals1[pt * q1 + a1] * s;
        }
        double f = fpts[pt], w = c.cut_w[pt];
        num += w * (uh - f) * (uh - f);
        den += w * f * f;
    }
    for (int off = 16; off > 0; off >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, off);
        den += __shfl_xor_sync(0xffffffffu, den, off);
    }
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { red[0][w] = num; red[1][w] = den; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, d = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { a += red[0][k]; d += red[1][k]; }
        parts[2 * blockIdx.x] = a;
        parts[2 * blockIdx.x + 1] = d;
    }
}

// fixed-order reduction of the block partials (one warp: lane l sums parts
// l, l+32, ...; then a fixed shuffle tree) -- deterministic run to run
__global__ void k_reduce_parts(const double* parts, int n, double* out) {
    if (blockIdx.x != 0 || threadIdx.x >= 32) return;
    double a = 0.0, d = 0.0;
    for (int k = threadIdx.x; k < n; k += 32) { a += parts[2 * k]; d += parts[2 * k + 1]; }
    for (int off = 16; off > 0; off >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, off);
        d += __shfl_xor_sync(0xffffffffu, d, off);
    }
    if (threadIdx.x == 0) {
        out[0] += a;
        out[1] += d;
    }
}

}  // namespace tq

using namespace tq;

extern "C" int tq_rhs(tq_projctx c, double* T, const int32_t* cut_rows, int32_t ncut, double* b, void* stream) {
    cudaStream_t st = S(stream);
    int nchunks = (c.n2 + kChunk - 1) / kChunk;
    int64_t nblk = (int64_t)c.nel1 * c.g1n * nchunks;
    // widest chunk: elements spanned by kChunk consecutive functions + p
    size_t shm = sizeof(double) * (size_t)(kChunk + 2 * c.p2 + 2) * c.g2n;
    TQ_CUDA(cudaFuncSetAttribute(k_rhs_stage1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    k_rhs_stage1<<<(int)std::min<int64_t>(nblk, (int64_t)kSms * 32), kChunk, shm, st>>>(c, T); ::tq::note_launch();
    int nrows = c.row_end - c.row_begin;
    if (nrows > 0) k_rhs_stage2<<<grid_for(nrows, 256), 256, 0, st>>>(c, T, b); ::tq::note_launch();
    if (ncut > 0 && c.cut_ptr) k_rhs_cut<<<grid_for(ncut, 4), 128, 0, st>>>(c, cut_rows, ncut, b); ::tq::note_launch();
    TQ_LAUNCH_CHECK("tq_rhs");
    return TQ_OK;
}

extern "C" int tq_target_points(tq_target f, const double* P, const double* w, int64_t n, double* out,
                                void* stream) {
    if (n == 0) return TQ_OK;
    k_target_points<<<grid_for(n, 256), 256, 0, S(stream)>>>(f, P, w, n, out); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_target_points");
    return TQ_OK;
}

extern "C" int tq_l2_parts(tq_projctx c, const double* C, int64_t e_begin, int64_t e_end, int64_t p_begin,
                           int64_t p_end, const double* fpts, double* num_den, void* stream) {
    cudaStream_t st = S(stream);
    const int nb = kSms * 4, nbe = kSms * 8;
    double* parts = nullptr;
    TQ_CUDA(cudaMallocAsync(&parts, sizeof(double) * 2 * nbe, st));
    TQ_CUDA(cudaMemsetAsync(num_den, 0, 2 * sizeof(double), st));
    if (e_end > e_begin) {
        // (a chunk spans at most two element rows when nel2 >= kL2Chunk)
        const bool tq_t = c.p1 == c.p2 && c.g1n == c.p1 + 3 && c.g2n == c.p2 + 3 && c.p1 >= 1 && c.p1 <= 5 &&
                          c.nel2 >= kL2Chunk;
        if (tq_t) {
            static const bool tiled = !(getenv("TQ_L2_ROWS") && atoi(getenv("TQ_L2_ROWS")) == 1);   // A/B knob
            const size_t shm = tiled ? sizeof(double) * (kL2Chunk * l2_stride(c.p1) + kL2Rows * l2_stride(c.p1) +
                                                         (kL2Rows + c.p1) * ((kL2Chunk + c.p1) | 1))
                                     : sizeof(double) * (kL2Chunk + 2) * l2_stride(c.p1);
            switch (c.p1) {
#define CASE(P) case P: \
                if (tiled) { \
                    TQ_CUDA(cudaFuncSetAttribute(k_l2_tiles<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm)); \
                    k_l2_tiles<P><<<nbe, kL2Threads, shm, st>>>(c, C, e_begin, e_end, parts); \
                } else { \
                    TQ_CUDA(cudaFuncSetAttribute(k_l2_elements_s<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm)); \
                    k_l2_elements_s<P><<<nbe, kL2Chunk, shm, st>>>(c, C, e_begin, e_end, parts); \
                } break;
                CASE(1) CASE(2) CASE(3) CASE(4) CASE(5)
#undef CASE
            }
        } else {
            k_l2_elements<<<nb, 256, 0, st>>>(c, C, e_begin, e_end, parts);
        }
        ::tq::note_launch();
        k_reduce_parts<<<1, 32, 0, st>>>(parts, tq_t ? nbe : nb, num_den); ::tq::note_launch();
    }
    if (p_end > p_begin && c.cut_ptr) {
        k_l2_cut<<<nb, 256, 0, st>>>(c, C, p_begin, p_end, fpts, parts); ::tq::note_launch();
        k_reduce_parts<<<1, 32, 0, st>>>(parts, nb, num_den); ::tq::note_launch();
    }
    TQ_LAUNCH_CHECK("tq_l2_parts");
    TQ_CUDA(cudaFreeAsync(parts, st));
    return TQ_OK;
}

extern "C" int tq_target_tables(tq_target f, const double* x1, int64_t n1, const double* x2, int64_t n2, double* out,
                                void* stream) {
    const int64_t total = (int64_t)f.nterms * (n1 + n2);
    if (total == 0) return TQ_OK;
    if (f.kind != 1) { set_error("tq_target_tables: a kind-1 (separable) target"); return TQ_EINVAL; }
    k_target_tables<<<grid_for(total, 256), 256, 0, S(stream)>>>(f, x1, n1, x2, n2, out); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_target_tables");
    return TQ_OK;
}

extern "C" int tq_rhs_separable(tq_projctx c, const int8_t* func_class, double* work, const int32_t* cut_rows,
                                int32_t ncut, double* b, void* stream) {
    if (c.target.kind != 2 || c.cgrid) { set_error("tq_rhs_separable: a kind-2 target and c == 1"); return TQ_EINVAL; }
    cudaStream_t st = S(stream);
    const int nt = c.target.nterms;
    double* Q1 = work;
    double* Q2 = Q1 + (int64_t)nt * c.nel1 * (c.p1 + 1);
    double* A1 = Q2 + (int64_t)nt * c.nel2 * (c.p2 + 1);
    double* A2 = A1 + (int64_t)nt * c.n1;
    const int64_t nq = (int64_t)nt * ((int64_t)c.nel1 * (c.p1 + 1) + (int64_t)c.nel2 * (c.p2 + 1));
    k_rhs_q<<<grid_for(nq, 256), 256, 0, st>>>(c, Q1, Q2); ::tq::note_launch();
    k_rhs_a<<<grid_for((int64_t)nt * (c.n1 + c.n2), 256), 256, 0, st>>>(c, Q1, Q2, A1, A2); ::tq::note_launch();
    const int nrows = c.row_end - c.row_begin;
    if (nrows > 0) k_rhs_sep_rows<<<grid_for(nrows, 256), 256, 0, st>>>(c, func_class, Q1, Q2, A1, A2, b);
    ::tq::note_launch();
    if (ncut > 0 && c.cut_ptr) k_rhs_cut<<<grid_for(ncut, 4), 128, 0, st>>>(c, cut_rows, ncut, b); ::tq::note_launch();
    TQ_LAUNCH_CHECK("tq_rhs_separable");
    return TQ_OK;
}

extern "C" int64_t tq_rhs_separable_work(tq_projctx c) {
    const int64_t nt = c.target.nterms;
    return nt * ((int64_t)c.nel1 * (c.p1 + 1) + (int64_t)c.nel2 * (c.p2 + 1) + c.n1 + c.n2);
}
