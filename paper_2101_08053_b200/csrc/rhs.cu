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
                double f = c.target.kind == 0 ? c.target.grid[(int64_t)r1 * c.target.ld + p2]
                                              : target_value(c.target, x, y);
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
                double f = c.target.kind == 0 ? c.target.grid[pr * c.target.ld + pc] : target_value(c.target, x, y);
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

__global__ void k_reduce_parts(const double* parts, int n, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double a = 0.0, d = 0.0;
        for (int k = 0; k < n; ++k) { a += parts[2 * k]; d += parts[2 * k + 1]; }
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
    const int nb = kSms * 4;
    double* parts = nullptr;
    TQ_CUDA(cudaMallocAsync(&parts, sizeof(double) * 2 * nb, st));
    TQ_CUDA(cudaMemsetAsync(num_den, 0, 2 * sizeof(double), st));
    if (e_end > e_begin) {
        k_l2_elements<<<nb, 256, 0, st>>>(c, C, e_begin, e_end, parts); ::tq::note_launch();
        k_reduce_parts<<<1, 32, 0, st>>>(parts, nb, num_den); ::tq::note_launch();
    }
    if (p_end > p_begin && c.cut_ptr) {
        k_l2_cut<<<nb, 256, 0, st>>>(c, C, p_begin, p_end, fpts, parts); ::tq::note_launch();
        k_reduce_parts<<<1, 32, 0, st>>>(parts, nb, num_den); ::tq::note_launch();
    }
    TQ_LAUNCH_CHECK("tq_l2_parts");
    TQ_CUDA(cudaFreeAsync(parts, st));
    return TQ_OK;
}
