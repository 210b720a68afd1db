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

// A group of G lanes (G = 32: a warp; 16: a half-warp) working on one system.
template <int G>
struct Grp {
    unsigned mask;
    int lane;
    __device__ Grp() {
        const int l = threadIdx.x & 31;
        lane = l & (G - 1);
        mask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (l & ~(G - 1)));
    }
    __device__ void sync() const { __syncwarp(mask); }
    __device__ void argmax(double& v, int& idx) const {
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
            const double ov = __shfl_xor_sync(mask, v, off, G);
            const int oi = __shfl_xor_sync(mask, idx, off, G);
            if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
        }
    }
    __device__ double dmax(double v) const {
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(mask, v, off, G));
        return v;
    }
    __device__ int imax(int v) const {
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) v = max(v, __shfl_xor_sync(mask, v, off, G));
        return v;
    }
};

// cr_norm / gemv_dot with the loop bounded at compile time (NB >= n), same
// operation order
template <int NB>
__device__ inline double cr_norm_b(const double* x, int n) {
    double hi = 0.0, lo = 0.0;
#pragma unroll
    for (int r = 0; r < NB; ++r) {
        if (r < n) {
            const double v = x[r];
            const double p = v * v;
            const double pe = __fma_rn(v, v, -p);
            const double s = hi + p;
            const double bb = s - hi;
            const double err = (hi - (s - bb)) + (p - bb);
            hi = s;
            lo = lo + err + pe;
        }
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

template <int NB>
__device__ inline double gemv_dot_b(const double* col, const double* v, int m) {
    if (m < 4) {
        if (m <= 0) return 0.0;
        if (m == 1) return col[0] * v[0];
        double tl = __fma_rn(col[0], v[0], col[1] * v[1]);
        if (m == 3) tl = __fma_rn(col[2], v[2], tl);
        return tl;
    }
    const int m1 = m - (m & 3);
    double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
    for (int r = 0; r + 3 < NB; r += 4) {
        if (r < m1) {
            p0 = __fma_rn(col[r], v[r], p0);
            p1 = __fma_rn(col[r + 1], v[r + 1], p1);
            p2 = __fma_rn(col[r + 2], v[r + 2], p2);
            p3 = __fma_rn(col[r + 3], v[r + 3], p3);
        }
    }
    double y = 0.0 + ((p0 + p2) + (p1 + p3));
    if (m1 < m) {
        double tl = col[m1] * v[m1];
        for (int r = m1 + 1; r < m; ++r) tl = tl + col[r] * v[r];
        y = y + tl;
    }
    return y;
}

// Per-warp shared workspace of one moment system.
struct FitWs {
    double *A, *A0, *b, *vh, *w, *vn1, *vn2;
    int* perm;
    __device__ FitWs(double* base, int tmax, int mmax) {
        A = base;                      // column-major, ld = t
        A0 = A + tmax * mmax;          // untouched copy for the residual check
        b = A0 + tmax * mmax;
        vh = b + tmax;                 // the current reflector (v0 = 1)
        w = vh + tmax;
        vn1 = w + mmax;
        vn2 = vn1 + mmax;
        perm = reinterpret_cast<int*>(vn2 + mmax);
    }
    __host__ __device__ static int doubles(int tmax, int mmax) { return 2 * tmax * mmax + 2 * tmax + 4 * mmax; }
};

// The basic solution of A w = b (A: t x m in ws.A / ws.A0, b in ws.b): LAPACK
// dgeqp3 pivoting (above), rank rule, back substitution in reference-BLAS
// dtrsv order (column sweep: z_k = b_k / R_kk, then b_i -= z_k R_ik, i < k);
// w in ws.w.  G lanes per system; TM >= t bounds the unrolled loops.
template <int G, int TM>
__device__ void qr_basic(FitWs& ws, int t, int m, const Grp<G>& g) {
    double* A = ws.A;
    double* b = ws.b;
    double* vh = ws.vh;
    double* vn1 = ws.vn1;
    double* vn2 = ws.vn2;
    int* perm = ws.perm;
    const int lane = g.lane;
    for (int c = lane; c < m; c += G) {
        perm[c] = c;
        const double nv = cr_norm_b<TM>(A + c * t, t);
        vn1[c] = nv;
        vn2[c] = nv;
    }
    g.sync();
    const int kmax = t < m ? t : m;
    double r00 = 0.0;
    for (int k = 0; k < kmax; ++k) {
        // pivot: idamax over vn1[k..m) (first maximum)
        double best = -1.0;
        int bi = 0x7fffffff;
        for (int c = k + lane; c < m; c += G) {
            const double nv = vn1[c];
            if (nv > best || (nv == best && c < bi)) { best = nv; bi = c; }
        }
        g.argmax(best, bi);
        if (bi != k) {
            for (int rr = lane; rr < t; rr += G) {
                double tmp = A[k * t + rr]; A[k * t + rr] = A[bi * t + rr]; A[bi * t + rr] = tmp;
            }
            if (lane == 0) {
                int tp = perm[k]; perm[k] = perm[bi]; perm[bi] = tp;
                vn1[bi] = vn1[k];
                vn2[bi] = vn2[k];
            }
        }
        g.sync();
        // dlarfg on x = A[k:t, k]: every lane computes it (identical values)
        const double alpha = A[k * t + k];
        const double xnorm = k + 1 < t ? cr_norm_b<TM>(A + k * t + k + 1, t - k - 1) : 0.0;
        double beta = alpha, tau = 0.0, scal = 1.0;
        if (xnorm != 0.0) {
            beta = -copysign(dlapy2(alpha, xnorm), alpha);
            tau = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        g.sync();
        // scaled reflector v = (1, x * scal), trimmed to its last non-zero (dlarf lastv)
        int lastv = 1;
        for (int rr = k + 1 + lane; rr < t; rr += G) {
            double x = A[k * t + rr];
            if (xnorm != 0.0) { x = x * scal; A[k * t + rr] = x; }
            vh[rr - k] = x;
            if (x != 0.0) lastv = rr - k + 1;
        }
        lastv = g.imax(lastv);
        if (lane == 0) {
            vh[0] = 1.0;
            if (xnorm != 0.0) A[k * t + k] = beta;
        }
        g.sync();
        // dlarf: H = I - tau v v^T on columns k+1.. and on b
        if (tau != 0.0) {
            for (int c = k + 1 + lane; c <= m; c += G) {
                double* col = (c < m ? A + c * t : b) + k;
                const double temp = -tau * gemv_dot_b<TM>(col, vh, lastv);
#pragma unroll
                for (int rr = 0; rr < TM; ++rr)
                    if (rr < lastv) col[rr] = __fma_rn(vh[rr], temp, col[rr]);
            }
        }
        g.sync();
        // partial column norms (dlaqp2)
        for (int c = k + 1 + lane; c < m; c += G) {
            if (vn1[c] != 0.0) {
                const double q = fabs(A[c * t + k]) / vn1[c];
                double temp = 1.0 - q * q;
                temp = temp > 0.0 ? temp : 0.0;
                const double rt = vn1[c] / vn2[c];
                const double temp2 = temp * (rt * rt);
                if (temp2 <= kTol3z) {
                    const double nv = k + 1 < t ? cr_norm_b<TM>(A + c * t + k + 1, t - k - 1) : 0.0;
                    vn1[c] = nv;
                    vn2[c] = nv;
                } else {
                    vn1[c] = vn1[c] * sqrt(temp);
                }
            }
        }
        g.sync();
        if (k == 0) r00 = fabs(beta);
    }
    // rank (src/quadrature.py:271-273)
    int rank = 0;
    {
        const double thr = (double)(t > m ? t : m) * 2.220446049250313e-16 * r00;
        for (int k = 0; k < kmax; ++k)
            if (fabs(A[k * t + k]) > thr) ++rank;
    }
    for (int c = lane; c < m; c += G) ws.w[c] = 0.0;
    g.sync();
    // back substitution, column sweep over the leading rank block
    for (int k = rank - 1; k >= 0; --k) {
        const double zk = b[k] / A[k * t + k];
        g.sync();
        for (int rr = lane; rr < k; rr += G) b[rr] = b[rr] - zk * A[k * t + rr];
        if (lane == 0) ws.w[perm[k]] = zk;
        g.sync();
    }
}

// Residual with the original system (src/quadrature.py:299-301) against the
// moments `bm` (t values) and the outputs.  (A w)[j] = sum_k w_k B_j(x_k) is
// also the direction product of sum_factor_row (src/assembly.py:245-252):
// written out when asked (same terms, same fused order as tq_wq_products ->
// bit-identical).
template <int G>
__device__ void fit_outputs(FitWs& ws, int t, int m, int i, int p, int j0, int k0, const double* bm,
                            double* wdst, int32_t* k0out, int32_t* failr, double* prod, const Grp<G>& g) {
    const int W = 2 * p + 1;
    const int lane = g.lane;
    double rmax = 0.0, bmax = 0.0;
    if (prod)
        for (int o = lane; o < W; o += G) {
            const int j = i - p + o;
            if (j < j0 || j >= j0 + t) prod[(int64_t)i * W + o] = 0.0;
        }
    for (int rr = lane; rr < t; rr += G) {
        double acc = 0.0;
        for (int c = 0; c < m; ++c) acc = __fma_rn(ws.A0[c * t + rr], ws.w[c], acc);
        if (prod) prod[(int64_t)i * W + (j0 + rr - i + p)] = acc;
        const double bb = bm[rr];
        rmax = fmax(rmax, fabs(acc - bb));
        bmax = fmax(bmax, fabs(bb));
    }
    rmax = g.dmax(rmax);
    bmax = g.dmax(bmax);
    for (int c = lane; c < m; c += G) wdst[c] = ws.w[c];
    if (lane == 0) {
        k0out[i] = k0;
        *failr = (rmax > 1e-12 * fmax(bmax, 1e-300)) ? 1 : 0;
    }
    g.sync();
}

__global__ void k_wq_solve(tq_space1d s, tq_layout lay, const int32_t* __restrict__ first,
                           const double* __restrict__ vals, const double* __restrict__ mom,
                           const int32_t* __restrict__ rows, int nrows, int tmax, int mmax,
                           const int64_t* __restrict__ wptr, int32_t* __restrict__ k0out,
                           double* __restrict__ wout, int32_t* __restrict__ fail, double* __restrict__ prod) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    FitWs ws(smem + (size_t)wib * FitWs::doubles(tmax, mmax), tmax, mmax);
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
            ws.A[c * t + rr] = a;
            ws.A0[c * t + rr] = a;
        }
        for (int rr = lane; rr < t; rr += 32) ws.b[rr] = mom[(int64_t)i * W + (j0 + rr - i + p)];
        __syncwarp();
        const Grp<32> g;
        qr_basic<32, 2 * kMaxP + 1>(ws, t, m, g);
        fit_outputs<32>(ws, t, m, i, p, j0, k0, mom + (int64_t)i * W + (j0 - i + p), wout + wptr[i], k0out,
                        fail + r, prod, g);
    }
}

// ---- fused, batched fits ----------------------------------------------------
// Every moment system of several rule sets in one launch, warp per (set,
// row).  Each warp forms its own system: the exact moments b_j = int B_i B_j
// over the (p+1)-point element Gauss rule of i's support (the tq_moments_1d_g
// arithmetic: per element a Gauss sum, elements in order) and the
// collocation block A = B_j(x_k) at the layout points of i's support
// (Cox-de Boor on the element's span, the reference's operation order) --
// then solves and writes as k_wq_solve.  One launch replaces the
// basis-table / Gauss-table / moments / solve chain of every rule set.
__device__ __host__ inline int fit_ws_doubles(int tmax, int mmax, int pmax) {
    return FitWs::doubles(tmax, mmax) + (pmax + 1) * (pmax + 1) * (pmax + 2) + tmax;
}

// G lanes per system, degree P at compile time (the Cox-de Boor triangle,
// the Gauss sums and the QR's row loops unroll; no local-memory arrays).
template <int P, int G>
__global__ void __launch_bounds__(128) k_wq_fit(tq_fitbatch B, int tmax, int mmax) {
    constexpr int TM = 2 * P + 1, NG = P + 1;
    extern __shared__ double smem[];
    const Grp<G> g;
    const int lane = g.lane;
    const int gib = threadIdx.x / G, gpb = blockDim.x / G;
    double* base = smem + (size_t)gib * fit_ws_doubles(tmax, mmax, P);
    FitWs ws(base, tmax, mmax);
    double* gt = base + FitWs::doubles(tmax, mmax);          // Gauss table of the support: [e][g][0..p, w]
    double* bm = gt + (P + 1) * (P + 1) * (P + 2);           // the moments b (t values)
    const int total = B.start[B.nsets];
    for (int item = blockIdx.x * gpb + gib; item < total; item += gridDim.x * gpb) {
        int sidx = 0;
        while (item >= B.start[sidx + 1]) ++sidx;
        const tq_fitset& F = B.set[sidx];
        const tq_space1d& s = F.s;
        const int r = item - B.start[sidx];
        const int i = F.rows[r];
        const int e0 = s.el_first[i], e1 = s.el_last[i];
        const int k0 = F.lay.offsets[e0], k1 = F.lay.offsets[e1 + 1];
        const int m = k1 - k0;
        const int j0 = s.ov_lo[i], t = s.ov_hi[i] - j0 + 1;
        if (m > mmax || t > tmax || t > TM || F.wptr[i + 1] - F.wptr[i] != m) {
            if (lane == 0) F.fail[r] = 2;
            continue;
        }
        const int ne = e1 - e0 + 1;
        // (1) Gauss table of the support elements: lane per (element, point)
        for (int q = lane; q < ne * NG; q += G) {
            const int le = q / NG, gq = q - le * NG;
            const int e = e0 + le;
            const double a = s.bp[e], bb = s.bp[e + 1];
            const double mid = 0.5 * (a + bb), half = 0.5 * (bb - a);
            double N[P + 1];
            basis_funs<P>(s.knots, s.espan[e], mid + half * B.gx[gq], N);
            double* o = gt + (size_t)q * (P + 2);
#pragma unroll
            for (int k = 0; k <= P; ++k) o[k] = N[k];
            o[P + 1] = half * B.gw[gq];
        }
        // (2) the collocation block: lane per layout point of the support
        for (int c = lane; c < m; c += G) {
            const int kk = k0 + c;
            int e = e0;
            while (F.lay.offsets[e + 1] <= kk) ++e;
            const int span = s.espan[e];
            double N[P + 1];
            basis_funs<P>(s.knots, span, F.lay.pts[kk], N);
            const int off0 = j0 - (span - P);
#pragma unroll
            for (int rr = 0; rr < TM; ++rr) {
                if (rr < t) {
                    const int off = off0 + rr;
                    double a = 0.0;
#pragma unroll
                    for (int q = 0; q <= P; ++q) a = off == q ? N[q] : a;
                    ws.A[c * t + rr] = a;
                    ws.A0[c * t + rr] = a;
                }
            }
        }
        g.sync();
        // (3) moments b_j, j = j0 + rr: per element the Gauss sum, elements in
        //     order (k_moments: acc += sum_g v_i v_j w over the shared support)
        for (int rr = lane; rr < t; rr += G) {
            const int j = j0 + rr;
            const int ea = max(e0, s.el_first[j]), eb = min(e1, s.el_last[j]);
            double acc = 0.0;
            for (int e = ea; e <= eb; ++e) {
                const int f = s.espan[e] - P;
                const double* row = gt + (size_t)(e - e0) * NG * (P + 2);
                double part = 0.0;
#pragma unroll
                for (int gq = 0; gq < NG; ++gq) {
                    const double* v = row + gq * (P + 2);
                    part = part + v[i - f] * v[j - f] * v[P + 1];
                }
                acc += part;
            }
            bm[rr] = acc;
            ws.b[rr] = acc;
        }
        g.sync();
        qr_basic<G, TM>(ws, t, m, g);
        fit_outputs<G>(ws, t, m, i, P, j0, k0, bm, F.w + F.wptr[i], F.k0, F.fail + r, F.products, g);
    }
}

__device__ inline void combine_row(int j, int lane, const int32_t* __restrict__ colptr,
                                   const int32_t* __restrict__ rowidx, const double* __restrict__ sval,
                                   const tq_rules& fine, const tq_rules& out) {
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
                // dst[q] += s_ij w~: a product and a sum, as numpy does it
                if (q < len && kk >= 0 && kk < fl) acc = acc + s_e * fine.w[fb + kk];
            }
        }
        if (q < len) dst[q] = acc;
    }
}

// warp per wanted row, lane per output weight: each lane accumulates its
// weight over the S entries of the row in entry order (the same additions,
// in the same order, as the reference's serial w += s_ij w~ loop,
// src/quadrature.py:435-444 -- bit-identical), in a register.
__global__ void k_dwq_combine(const int32_t* __restrict__ rows, int nrows, const int32_t* __restrict__ colptr,
                              const int32_t* __restrict__ rowidx, const double* __restrict__ sval,
                              tq_rules fine, tq_rules out) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int r = warp; r < nrows; r += nwarps) combine_row(rows[r], lane, colptr, rowidx, sval, fine, out);
}

// every DWQ set's combination in one launch: warp per (set, wanted row),
// the arithmetic of k_dwq_combine
__global__ void k_dwq_combine_sets(tq_combinebatch B) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    const int total = B.start[B.nsets];
    for (int item = warp; item < total; item += nwarps) {
        int sidx = 0;
        while (item >= B.start[sidx + 1]) ++sidx;
        const tq_combineset& C = B.set[sidx];
        const int j = C.rows[item - B.start[sidx]];
        combine_row(j, lane, C.colptr, C.rowidx, C.sval, C.fine, C.out);
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
    size_t per = FitWs::doubles(tmax, mmax);
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

template <int P, int G>
static int launch_fit(const tq_fitbatch& B, int total, int tmax, int mmax, cudaStream_t st) {
    const int gpb = 128 / G;
    const size_t shm = (size_t)fit_ws_doubles(tmax, mmax, P) * sizeof(double) * gpb;
    if (shm > 220 * 1024) { set_error("moment system too large (t=%d, m=%d)", tmax, mmax); return TQ_EINVAL; }
    static int set_for = -1;      // the attribute is per-device state
    int dev = 0;
    cudaGetDevice(&dev);
    if (set_for != dev) {
        TQ_CUDA(cudaFuncSetAttribute(k_wq_fit<P, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        set_for = dev;
    }
    const int grid = (total + gpb - 1) / gpb;
    k_wq_fit<P, G><<<grid, 128, shm, st>>>(B, tmax, mmax); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_wq_fit");
    return TQ_OK;
}

template <int P>
static int launch_fit_p(const tq_fitbatch& B, int total, int tmax, int mmax, cudaStream_t st) {
    // half a warp per system while the columns (points) fit in 16 lanes
    return mmax <= 16 ? launch_fit<P, 16>(B, total, tmax, mmax, st) : launch_fit<P, 32>(B, total, tmax, mmax, st);
}

extern "C" int tq_wq_fit_sets(const tq_fitbatch* batch_h, int32_t tmax, int32_t mmax, void* stream) {
    tq_fitbatch B = *batch_h;
    if (B.nsets < 0 || B.nsets > TQ_FIT_MAX_SETS) { set_error("tq_wq_fit_sets: %d sets", B.nsets); return TQ_EINVAL; }
    B.start[0] = 0;
    int p = -1;
    for (int k = 0; k < B.nsets; ++k) {
        if (k && B.set[k].s.p != p) { set_error("tq_wq_fit_sets: sets of one degree only"); return TQ_EINVAL; }
        p = B.set[k].s.p;
        B.start[k + 1] = B.start[k] + B.set[k].nrows;
    }
    const int total = B.start[B.nsets];
    if (total == 0) return TQ_OK;
    if (tmax > 2 * p + 1) { set_error("too many trials per system (%d)", tmax); return TQ_EINVAL; }
    cudaStream_t st = S(stream);
    switch (p) {
#define CASE(P) case P: return launch_fit_p<P>(B, total, tmax, mmax, st);
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
        default:
            set_error("tq_wq_fit_sets: degree %d unsupported (1..%d)", p, kMaxP);
            return TQ_EINVAL;
    }
}

extern "C" int tq_dwq_combine_sets(const tq_combinebatch* batch_h, void* stream) {
    tq_combinebatch B = *batch_h;
    if (B.nsets < 0 || B.nsets > TQ_FIT_MAX_SETS) { set_error("tq_dwq_combine_sets: %d sets", B.nsets); return TQ_EINVAL; }
    B.start[0] = 0;
    for (int k = 0; k < B.nsets; ++k) B.start[k + 1] = B.start[k] + B.set[k].nrows;
    const int total = B.start[B.nsets];
    if (total == 0) return TQ_OK;
    k_dwq_combine_sets<<<grid_for((int64_t)total * 32, 128), 128, 0, S(stream)>>>(B); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_dwq_combine_sets");
    return TQ_OK;
}
