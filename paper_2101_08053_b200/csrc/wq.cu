// Subsystem (1): weighted-quadrature weights as batched small FP64 solves.
//
//  tq_wq_solve     <- _solve_rows + _qr_basic_solve   src/quadrature.py:263-303
//  tq_dwq_combine  <- build_dwq step 4 (w = S^T w~)   src/quadrature.py:434-444
//
// One warp per moment system A w = b (A: t trials x m points, t <= 2p+1).
// Householder QR with column pivoting exactly as LAPACK dgeqp3/dlaqp2 pivots
// (see below: same pivot sequence, SURVEY F6 closed), rank by
// |R_kk| > max(t,m) eps |R_00|, back substitution on the leading rank block:
// the *basic* least-squares solution the reference obtains from
// scipy.linalg.qr.  The residual check certifies every row.
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

// ---- LAPACK dgeqp3 / dlaqp2 pivoting, reproduced --------------------------
// The reference solves every moment system with scipy.linalg.qr(pivoting=True)
// = LAPACK dgeqp3, which for min(t, m) < 32 runs the unblocked dlaqp2 over
// OpenBLAS kernels.  Its pivot choices (ties of mirrored columns included)
// follow from (scripts/probes/lapack_pivot_emul.py: 1977/1977 systems, p = 1..8):
//   * column norms correctly rounded (dnrm2): squares summed in
//     double-double, then a correctly rounded square root;
//   * idamax: first maximum of the partial norms vn1;
//   * partial-norm downdating vn1 *= sqrt(1 - (|r_kj|/vn1)^2) with the
//     tol3z = sqrt(eps) recomputation rule;
//   * dlarfg with dlapy2 = w sqrt(1 + (z/w)^2) and x *= 1/(alpha - beta);
//   * dlarf trimmed to the last non-zero of v (lastv) and the last non-zero
//     column (lastc); w = C^T v as OpenBLAS dgemv_t does it -- four FMA lane
//     accumulators over rows r < m - m%4, reduced (p0 + p2) + (p1 + p3), the
//     m%4 leftover rows as a plain product-sum added last (m < 4: the scalar
//     path, fma(a0, x0, a1 x1) then FMAs) -- and the rank-1
//     update C += v (-tau w_j) with one FMA per entry (dger).
// This file is compiled with -fmad=false: every fused operation above is an
// explicit __fma_rn, every other one is a separate IEEE operation.
constexpr double kTol3z = 1.4901161193847656e-08;   // sqrt(DLAMCH('Epsilon'))

// correctly rounded sqrt(sum x_r^2), r < n, stride 1
__device__ inline double cr_norm(const double* x, int n) {
    double hi = 0.0, lo = 0.0;
    for (int r = 0; r < n; ++r) {
        const double v = x[r];
        const double p = v * v;
        const double pe = __fma_rn(v, v, -p);
        const double s = hi + p;
        const double bb = s - hi;
        const double err = (hi - (s - bb)) + (p - bb);
        hi = s;
        lo = lo + err + pe;
    }
    const double s = hi + lo;
    lo = lo - (s - hi);
    hi = s;
    if (!(hi > 0.0)) return 0.0;
    double r = sqrt(hi);
    const double e = __fma_rn(-r, r, hi) + lo;
    const double up = nextafter(r, INFINITY), u = up - r;
    if (e - r * u > 0.25 * u * u) return up;
    const double dn = nextafter(r, 0.0), d = r - dn;
    if (-e - r * d > -0.25 * d * d) return dn;
    return r;
}

__device__ inline double dlapy2(double x, double y) {
    const double xa = fabs(x), ya = fabs(y);
    const double w = fmax(xa, ya), z = fmin(xa, ya);
    if (z == 0.0) return w;
    const double q = z / w;
    return w * sqrt(1.0 + q * q);
}

// OpenBLAS dgemv_t's dot of one column with v over rows [0, m).  Fewer than
// four rows take the kernel's scalar path: fma(a0, x0, a1 x1), then one FMA
// per further row.
__device__ inline double gemv_dot(const double* col, const double* v, int m) {
    if (m < 4) {
        if (m <= 0) return 0.0;
        if (m == 1) return col[0] * v[0];
        double tl = __fma_rn(col[0], v[0], col[1] * v[1]);
        if (m == 3) tl = __fma_rn(col[2], v[2], tl);
        return tl;
    }
    const int m1 = m - (m & 3);
    double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
    for (int r = 0; r < m1; r += 4) {
        p0 = __fma_rn(col[r], v[r], p0);
        p1 = __fma_rn(col[r + 1], v[r + 1], p1);
        p2 = __fma_rn(col[r + 2], v[r + 2], p2);
        p3 = __fma_rn(col[r + 3], v[r + 3], p3);
    }
    double y = 0.0 + ((p0 + p2) + (p1 + p3));
    if (m1 < m) {
        double tl = col[m1] * v[m1];
        for (int r = m1 + 1; r < m; ++r) tl = tl + col[r] * v[r];
        y = y + tl;
    }
    return y;
}

__global__ void k_wq_solve(tq_space1d s, tq_layout lay, const int32_t* __restrict__ first,
                           const double* __restrict__ vals, const double* __restrict__ mom,
                           const int32_t* __restrict__ rows, int nrows, int tmax, int mmax,
                           const int64_t* __restrict__ wptr, int32_t* __restrict__ k0out,
                           double* __restrict__ wout, int32_t* __restrict__ fail, double* __restrict__ prod) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int per = 2 * tmax * mmax + 2 * tmax + 4 * mmax;  // A, A0, b, v, w, vn1, vn2 + perm
    double* A = smem + (size_t)wib * per;           // column-major, ld = t
    double* A0 = A + tmax * mmax;                   // untouched copy for the residual check
    double* b = A0 + tmax * mmax;
    double* vh = b + tmax;                          // the current reflector (v0 = 1)
    double* w = vh + tmax;
    double* vn1 = w + mmax;
    double* vn2 = vn1 + mmax;
    int* perm = reinterpret_cast<int*>(vn2 + mmax);
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
        for (int c = lane; c < m; c += 32) { const double nv = cr_norm(A + c * t, t); vn1[c] = nv; vn2[c] = nv; }
        __syncwarp();

        const int kmax = t < m ? t : m;
        double r00 = 0.0;
        int rank = 0;
        for (int k = 0; k < kmax; ++k) {
            // pivot: idamax over vn1[k..m) (first maximum)
            double best = -1.0;
            int bi = 0x7fffffff;
            for (int c = k + lane; c < m; c += 32) {
                const double nv = vn1[c];
                if (nv > best || (nv == best && c < bi)) { best = nv; bi = c; }
            }
            warp_argmax(best, bi);
            if (bi != k) {
                for (int rr = lane; rr < t; rr += 32) {
                    double tmp = A[k * t + rr]; A[k * t + rr] = A[bi * t + rr]; A[bi * t + rr] = tmp;
                }
                if (lane == 0) {
                    int tp = perm[k]; perm[k] = perm[bi]; perm[bi] = tp;
                    vn1[bi] = vn1[k];
                    vn2[bi] = vn2[k];
                }
            }
            __syncwarp();
            // dlarfg on x = A[k:t, k]
            double beta = A[k * t + k], tau = 0.0;
            int lastv = 0;
            if (lane == 0) {
                const double alpha = beta;
                const double xnorm = k + 1 < t ? cr_norm(A + k * t + k + 1, t - k - 1) : 0.0;
                if (xnorm != 0.0) {
                    beta = -copysign(dlapy2(alpha, xnorm), alpha);
                    tau = (beta - alpha) / beta;
                    const double scal = 1.0 / (alpha - beta);
                    for (int rr = k + 1; rr < t; ++rr) A[k * t + rr] = A[k * t + rr] * scal;
                    A[k * t + k] = beta;
                }
                // the reflector v = (1, A[k+1:t, k]) trimmed to its last non-zero (dlarf lastv)
                vh[0] = 1.0;
                lastv = 1;
                for (int rr = k + 1; rr < t; ++rr) {
                    vh[rr - k] = A[k * t + rr];
                    if (vh[rr - k] != 0.0) lastv = rr - k + 1;
                }
            }
            beta = __shfl_sync(0xffffffffu, beta, 0);
            tau = __shfl_sync(0xffffffffu, tau, 0);
            lastv = __shfl_sync(0xffffffffu, lastv, 0);
            __syncwarp();
            // dlarf: H = I - tau v v^T on columns k+1.. (trailing zero columns
            // of C(1:lastv, :) are untouched either way) and on b
            if (tau != 0.0) {
                for (int c = k + 1 + lane; c <= m; c += 32) {
                    double* col = (c < m ? A + c * t : b) + k;
                    const double temp = -tau * gemv_dot(col, vh, lastv);
                    for (int rr = 0; rr < lastv; ++rr) col[rr] = __fma_rn(vh[rr], temp, col[rr]);
                }
            }
            __syncwarp();
            // partial column norms (dlaqp2)
            for (int c = k + 1 + lane; c < m; c += 32) {
                if (vn1[c] != 0.0) {
                    const double q = fabs(A[c * t + k]) / vn1[c];
                    double temp = 1.0 - q * q;
                    temp = temp > 0.0 ? temp : 0.0;
                    const double rt = vn1[c] / vn2[c];
                    const double temp2 = temp * (rt * rt);
                    if (temp2 <= kTol3z) {
                        const double nv = k + 1 < t ? cr_norm(A + c * t + k + 1, t - k - 1) : 0.0;
                        vn1[c] = nv;
                        vn2[c] = nv;
                    } else {
                        vn1[c] = vn1[c] * sqrt(temp);
                    }
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
        // (same terms, same fused order as tq_wq_products -> bit-identical)
        double rmax = 0.0, bmax = 0.0;
        if (prod)
            for (int o = lane; o < W; o += 32) {
                const int j = i - p + o;
                if (j < j0 || j >= j0 + t) prod[(int64_t)i * W + o] = 0.0;
            }
        for (int rr = lane; rr < t; rr += 32) {
            double acc = 0.0;
            for (int c = 0; c < m; ++c) acc = __fma_rn(A0[c * t + rr], w[c], acc);
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
    size_t per = 2 * (size_t)tmax * mmax + 2 * (size_t)tmax + 4 * (size_t)mmax;
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
