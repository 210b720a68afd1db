// Subsystem (1): weighted-quadrature weights as batched small FP64 solves.
//
//  tq_wq_solve     <- _solve_rows + _qr_basic_solve   src/quadrature.py:263-303
//  tq_dwq_combine  <- build_dwq step 4 (w = S^T w~)   src/quadrature.py:434-444
//
// One warp per moment system A w = b (A: t trials x m points, t <= 2p+1).
// Householder QR with column pivoting (largest remaining column norm, first
// index on ties, norms recomputed exactly at every step), rank by
// |R_kk| > max(t,m) eps |R_00|, back substitution on the leading rank block:
// the *basic* least-squares solution the reference obtains from LAPACK
// dgeqp3.  Pivot ties may resolve differently from LAPACK's downdated norms
// (SURVEY F6); any exact solution reproduces the moments, which is what the
// residual check below certifies.
#include "common.cuh"

namespace tq {

__device__ inline void warp_argmax(double& v, int& idx) {
    for (int off = 16; off > 0; off >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, v, off);
        int oi = __shfl_xor_sync(0xffffffffu, idx, off);
        if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
    }
}

__device__ inline double warp_sum(double v) {
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

__device__ inline double warp_max(double v) {
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    return v;
}

// colloc value B_j(x_k) from the banded basis table
__device__ inline double colloc(const int32_t* first, const double* vals, int p, int k, int j) {
    int r = j - first[k];
    return (r >= 0 && r <= p) ? vals[(int64_t)k * (p + 1) + r] : 0.0;
}

__global__ void k_wq_solve(tq_space1d s, tq_layout lay, const int32_t* __restrict__ first,
                           const double* __restrict__ vals, const double* __restrict__ mom,
                           const int32_t* __restrict__ rows, int nrows, int tmax, int mmax,
                           const int64_t* __restrict__ wptr, int32_t* __restrict__ k0out,
                           double* __restrict__ wout, int32_t* __restrict__ fail, double* __restrict__ prod) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int per = 2 * tmax * mmax + tmax + 2 * mmax;  // A, A0, b, w + perm (as double slots)
    double* A = smem + (size_t)wib * per;           // column-major, ld = t
    double* A0 = A + tmax * mmax;                   // untouched copy for the residual check
    double* b = A0 + tmax * mmax;
    double* w = b + tmax;
    int* perm = reinterpret_cast<int*>(w + mmax);
    const int p = s.p, W = 2 * p + 1;

    for (int r = blockIdx.x * wpb + wib; r < nrows; r += gridDim.x * wpb) {
        const int i = rows[r];
        const int e0 = s.el_first[i], e1 = s.el_last[i];
        const int k0 = lay.offsets[e0], k1 = lay.offsets[e1 + 1];
        const int m = k1 - k0;
        const int j0 = s.ov_lo[i], t = s.ov_hi[i] - j0 + 1;
        if (m > mmax || t > tmax || wptr[i + 1] - wptr[i] != m) {
            if (lane == 0) fail[r] = 2;   // bounds violation: reported through the fail flags
            continue;
        }
        // load A (t x m) and b
        for (int q = lane; q < t * m; q += 32) {
            int c = q / t, rr = q % t;
            const double a = colloc(first, vals, p, k0 + c, j0 + rr);
            A[c * t + rr] = a;
            A0[c * t + rr] = a;
        }
        for (int rr = lane; rr < t; rr += 32) b[rr] = mom[(int64_t)i * W + (j0 + rr - i + p)];
        for (int c = lane; c < m; c += 32) perm[c] = c;
        __syncwarp();

        const int kmax = t < m ? t : m;
        double r00 = 0.0;
        int rank = 0;
        for (int k = 0; k < kmax; ++k) {
            // pivot: largest norm of A[k:t, c], c >= k
            double best = -1.0;
            int bi = 0x7fffffff;
            for (int c = k + lane; c < m; c += 32) {
                double ss = 0.0;
                for (int rr = k; rr < t; ++rr) { double a = A[c * t + rr]; ss += a * a; }
                double nv = sqrt(ss);
                if (nv > best || (nv == best && c < bi)) { best = nv; bi = c; }
            }
            warp_argmax(best, bi);
            if (bi != k) {
                for (int rr = lane; rr < t; rr += 32) {
                    double tmp = A[k * t + rr]; A[k * t + rr] = A[bi * t + rr]; A[bi * t + rr] = tmp;
                }
                if (lane == 0) { int tp = perm[k]; perm[k] = perm[bi]; perm[bi] = tp; }
            }
            __syncwarp();
            // Householder reflector of x = A[k:t, k] (dlarfg convention)
            double alpha = A[k * t + k];
            double xs = 0.0;
            for (int rr = k + 1 + lane; rr < t; rr += 32) { double a = A[k * t + rr]; xs += a * a; }
            xs = warp_sum(xs);
            double xnorm = sqrt(xs);
            double beta = alpha, tau = 0.0, scal = 0.0;
            if (xnorm != 0.0) {
                beta = -copysign(hypot(alpha, xnorm), alpha);
                tau = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
            __syncwarp();
            for (int rr = k + 1 + lane; rr < t; rr += 32) A[k * t + rr] *= scal;  // v (v0 = 1)
            __syncwarp();
            if (lane == 0) A[k * t + k] = beta;
            // apply H = I - tau v v^T to the remaining columns and to b
            if (tau != 0.0) {
                for (int c = k + 1 + lane; c <= m; c += 32) {
                    double* col = (c < m) ? (A + c * t) : b;
                    double dot = col[k];
                    for (int rr = k + 1; rr < t; ++rr) dot += A[k * t + rr] * col[rr];
                    dot *= tau;
                    col[k] -= dot;
                    for (int rr = k + 1; rr < t; ++rr) col[rr] -= dot * A[k * t + rr];
                }
            }
            __syncwarp();
            if (k == 0) r00 = fabs(beta);
        }
        // rank (src/quadrature.py:271-273)
        {
            const double thr = (double)(t > m ? t : m) * 2.220446049250313e-16 * r00;
            for (int k = 0; k < kmax; ++k)
                if (fabs(A[k * t + k]) > thr) ++rank;
        }
        // back substitution on the leading rank block, scatter to pivots
        for (int c = lane; c < m; c += 32) w[c] = 0.0;
        __syncwarp();
        if (lane == 0) {
            double z[2 * kMaxP + 2];
            for (int k = rank - 1; k >= 0; --k) {
                double acc = b[k];
                for (int c = k + 1; c < rank; ++c) acc -= A[c * t + k] * z[c];
                z[k] = acc / A[k * t + k];
            }
            for (int k = 0; k < rank; ++k) w[perm[k]] = z[k];
        }
        __syncwarp();
        // residual with the original system (src/quadrature.py:299-301).
        // (A w)[j] = sum_k w_k B_j(x_k) is also the direction product of
        // sum_factor_row (src/assembly.py:245-252): written out when asked
        // (same terms, same order as tq_wq_products -> bit-identical)
        double rmax = 0.0, bmax = 0.0;
        if (prod)
            for (int o = lane; o < W; o += 32) {
                const int j = i - p + o;
                if (j < j0 || j >= j0 + t) prod[(int64_t)i * W + o] = 0.0;
            }
        for (int rr = lane; rr < t; rr += 32) {
            double acc = 0.0;
            for (int c = 0; c < m; ++c) acc += A0[c * t + rr] * w[c];
            if (prod) prod[(int64_t)i * W + (j0 + rr - i + p)] = acc;
            double bb = mom[(int64_t)i * W + (j0 + rr - i + p)];
            rmax = fmax(rmax, fabs(acc - bb));
            bmax = fmax(bmax, fabs(bb));
        }
        rmax = warp_max(rmax);
        bmax = warp_max(bmax);
        double* dst = wout + wptr[i];
        for (int c = lane; c < m; c += 32) dst[c] = w[c];
        if (lane == 0) {
            k0out[i] = k0;
            fail[r] = (rmax > 1e-12 * fmax(bmax, 1e-300)) ? 1 : 0;
        }
        __syncwarp();
    }
}

// warp per wanted row, lane per output weight: each lane accumulates its
// weight over the S entries of the row in entry order (the same additions,
// in the same order, as a serial dst[q] += s_ij w~ loop -- bit-identical),
// in a register instead of through memory.
__global__ void k_dwq_combine(const int32_t* __restrict__ rows, int nrows, const int32_t* __restrict__ colptr,
                              const int32_t* __restrict__ rowidx, const double* __restrict__ sval,
                              tq_rules fine, tq_rules out) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int r = warp; r < nrows; r += nwarps) {
        const int j = rows[r];
        const int64_t o0 = out.wptr[j];
        const int len = (int)(out.wptr[j + 1] - o0), k0 = out.k0[j];
        const int c0 = colptr[j], nent = colptr[j + 1] - c0;
        double* dst = const_cast<double*>(out.w) + o0;
        for (int q0 = 0; q0 < len; q0 += 32) {
            const int q = q0 + lane;
            double acc = 0.0;
            for (int e0 = 0; e0 < nent; e0 += 32) {
                // the row's S entries and their fine rows, one per lane
                int fi = 0, fk0 = 0, flen = 0;
                int64_t f0 = 0;
                double sij = 0.0;
                if (e0 + lane < nent) {
                    fi = rowidx[c0 + e0 + lane];
                    sij = sval[c0 + e0 + lane];
                    fk0 = fine.k0[fi];
                    f0 = fine.wptr[fi];
                    flen = (int)(fine.wptr[fi + 1] - f0);
                }
                const int ne = min(32, nent - e0);
                for (int e = 0; e < ne; ++e) {
                    const double s_e = __shfl_sync(0xffffffffu, sij, e);
                    const int off = __shfl_sync(0xffffffffu, fk0, e) - k0;
                    const int fl = __shfl_sync(0xffffffffu, flen, e);
                    const int64_t fb = __shfl_sync(0xffffffffu, f0, e);
                    const int kk = q - off;
                    if (q < len && kk >= 0 && kk < fl) acc += s_e * fine.w[fb + kk];
                }
            }
            if (q < len) dst[q] = acc;
        }
    }
}

}  // namespace tq

using namespace tq;

extern "C" int tq_wq_solve(tq_space1d s, tq_layout lay, const int32_t* first, const double* vals,
                           const double* mom, const int32_t* rows, int32_t nrows, int32_t tmax,
                           int32_t mmax, int64_t* wptr, int32_t* k0, double* w, int32_t* fail,
                           double* products, void* stream) {
    if (nrows == 0) return TQ_OK;
    if (tmax > 2 * kMaxP + 1) { set_error("too many trials per system (%d)", tmax); return TQ_EINVAL; }
    const int wpb = 4;
    size_t per = 2 * (size_t)tmax * mmax + tmax + 2 * mmax;
    size_t shm = per * sizeof(double) * wpb;
    if (shm > 200 * 1024) { set_error("moment system too large (t=%d, m=%d)", tmax, mmax); return TQ_EINVAL; }
    TQ_CUDA(cudaFuncSetAttribute(k_wq_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    int grid = (nrows + wpb - 1) / wpb;
    k_wq_solve<<<grid, 32 * wpb, shm, S(stream)>>>(s, lay, first, vals, mom, rows, nrows, tmax, mmax,
                                                   wptr, k0, w, fail, products); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_wq_solve");
    return TQ_OK;
}

extern "C" int tq_dwq_combine(const int32_t* rows, int32_t nrows, const int32_t* s_colptr,
                              const int32_t* s_rowidx, const double* s_val, tq_rules fine,
                              tq_rules out_rules, void* stream) {
    if (nrows == 0) return TQ_OK;
    k_dwq_combine<<<grid_for((int64_t)nrows * 32, 128), 128, 0, S(stream)>>>(rows, nrows, s_colptr, s_rowidx,
                                                                              s_val, fine, out_rules);
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_dwq_combine");
    return TQ_OK;
}
