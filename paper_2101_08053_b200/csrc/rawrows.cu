// Subsystems (3)+(4): rows that are not separable -- cut rows (hybrid Gauss,
// DWQ box + Gauss residual, naive masked WQ), rows with a coefficient c != 1,
// and every row of the element-Gauss `reference` strategy.  Each row gets a
// dense local block raw[r][(j1-i1+p1)*(2p2+1) + (j2-i2+p2)] (unsymmetrised
// M_ij), consumed by the fused symmetrise/compact/CSR writer in rows.cu.
//
//  tq_raw_regular   <- sum_factor_row (src/assembly.py:218-252),
//                      _Run.element_block (:310-332), _gauss_rows_by_element
//                      (:623-643), _cut_regular_rows (:553-610), reference
//                      strategy element loop (:522-528)
//  tq_raw_cutcells  <- _Run.add_cut_blocks (:369-398)
//  tq_coeff_grid / tq_coeff_points <- CoefficientField.grid / .at (:54-85)
//                      for a B-spline geometry map (c = det J)
//
// One warp per row; the row block, the two weighted collocation slices and
// the inner contraction live in shared memory.
#include <limits.h>
#include <stdlib.h>

#include "common.cuh"

namespace tq {

struct RowDesc {
    int fidx, mode, set1, set2, a1, b1, a2, b2;
};

// The raw block of descriptor row r: row-major (raw + r W1 W2, stride 1) or,
// in the planes layout, entry q at raw[q * raw_ld + store[r]].
struct RawRow {
    double* p;
    int64_t s;
    __device__ __forceinline__ double& operator[](int q) const { return p[q * s]; }
};

__device__ __forceinline__ RawRow raw_row(const tq_rawctx& c, int r) {
    if (c.raw_ld) return RawRow{c.raw + c.store[r], c.raw_ld};
    return RawRow{c.raw + (int64_t)r * ((2 * c.p1 + 1) * (2 * c.p2 + 1)), 1};
}

__device__ inline double colloc_at(const tq_ruleset& s, int p, int k, int j) {
    int r = j - s.first[k];
    return (r >= 0 && r <= p) ? s.vals[(int64_t)k * (p + 1) + r] : 0.0;
}

// element of layout point k
__device__ inline int elem_of_point(const tq_layout& lay, int k) {
    return upper_bound_d_int(lay.offsets, lay.nel + 1, k) - 1;
}

// Gauss element-block entry (test local a, trial local b) of element (e1,e2)
__device__ inline double gauss_entry(const tq_rawctx& c, int e1, int e2, int a1, int a2, int b1, int b2) {
    const int q1 = c.p1 + 1, q2 = c.p2 + 1;
    if (!c.cg) {
        // c == 1: the element block is the product of two 1-D element masses
        return c.em1[((int64_t)e1 * q1 + a1) * q1 + b1] * c.em2[((int64_t)e2 * q2 + a2) * q2 + b2];
    }
    const int64_t ld = (int64_t)c.nel2 * c.ng2;
    double acc = 0.0;
    for (int g1 = 0; g1 < c.ng1; ++g1) {
        const double* v1 = c.ev1 + ((int64_t)e1 * c.ng1 + g1) * q1;
        double f1 = v1[a1] * v1[b1];
        double w1 = c.ew1[(int64_t)e1 * c.ng1 + g1];
        const double* cgr = c.cg + ((int64_t)e1 * c.ng1 + g1) * ld + (int64_t)e2 * c.ng2;
        double part = 0.0;
        for (int g2 = 0; g2 < c.ng2; ++g2) {
            const double* v2 = c.ev2 + ((int64_t)e2 * c.ng2 + g2) * q2;
            double cw = cgr[g2] * (w1 * c.ew2[(int64_t)e2 * c.ng2 + g2]);
            part += (v2[a2] * v2[b2]) * cw;
        }
        acc += f1 * part;
    }
    return acc;
}

// element 1-D masses em[e][a][b] = sum_g w_g V[g][a] V[g][b] (c == 1 Gauss blocks)
__global__ void k_elem_mass(const double* __restrict__ ev, const double* __restrict__ ew, int nel, int ng, int p,
                            double* __restrict__ em) {
    const int q = p + 1;
    const int64_t total = (int64_t)nel * q * q;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int e = (int)(t / (q * q)), r = (int)(t - (int64_t)e * q * q), a = r / q, b = r - (r / q) * q;
        double m = 0.0;
        for (int g = 0; g < ng; ++g) {
            const double* v = ev + ((int64_t)e * ng + g) * q;
            m += (v[a] * v[b]) * ew[(int64_t)e * ng + g];
        }
        em[t] = m;
    }
}

// PARTS: 1 = element-Gauss part only (writes the row block; needs no WQ
// rules), 2 = sum-factorization part only (adds onto the stored block),
// 3 = both.  Split or fused, each entry sees the same additions in the same
// order, so the results are bit-identical.
// doubles per warp for the staged element window (em slices, spans, flags)
__host__ __device__ inline int regular_window_slots(int p1, int p2) {
    const int q1 = p1 + 1, q2 = p2 + 1;
    return q1 * q1 + q2 * q2 + (q1 + q2 + q1 * q2 + 1) / 2 + 1;
}

template <int PARTS>
__global__ void k_raw_regular(tq_rawctx c, int r0, int r1) {
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int W1 = 2 * c.p1 + 1, W2 = 2 * c.p2 + 1, T = W1 * W2;
    const int ni = c.nmax1 > c.p1 + 1 ? c.nmax1 : c.p1 + 1;    // inner rows (sum factorization / Gauss stage 1)
    // c != 1: the row's coefficient window is staged too (regular_smem_per_warp)
    const int per = T + c.nmax1 * W1 + c.nmax2 * W2 + W2 * ni + W1 + W2 + regular_window_slots(c.p1, c.p2) +
                    (c.grids ? c.nmax1 * c.nmax2 : 0);
    double* blk = sm + (size_t)wib * per;
    double* B1 = blk + T;
    double* B2 = B1 + c.nmax1 * W1;
    double* inner = B2 + c.nmax2 * W2;
    double* S1 = inner + W2 * ni;
    double* S2 = S1 + W1;
    const int q1 = c.p1 + 1, q2 = c.p2 + 1;
    // element window of the c == 1 Gauss stage
    double* E1 = S2 + W2;
    double* E2 = E1 + q1 * q1;
    int* F1 = reinterpret_cast<int*>(E2 + q2 * q2);
    int* F2 = F1 + q1;
    int* MK = F2 + q2;
    double* GS = S2 + W2 + regular_window_slots(c.p1, c.p2);    // n1 x n2 coefficient window (c != 1)

    for (int r = r0 + blockIdx.x * wpb + wib; r < r1; r += gridDim.x * wpb) {
        RowDesc d = reinterpret_cast<const RowDesc*>(c.desc)[r];
        const int i1 = d.fidx / c.n2, i2 = d.fidx - (d.fidx / c.n2) * c.n2;
        if (PARTS == 2 && d.mode == TQ_ROW_GAUSS) continue;     // nothing to add
        if (PARTS == 2) {
            const RawRow src = raw_row(c, r);
            for (int q = lane; q < T; q += 32) blk[q] = src[q];
        } else {
            for (int q = lane; q < T; q += 32) blk[q] = 0.0;
        }
        __syncwarp();
        // -- element Gauss over interior support elements (GAUSS, BOX residual)
        if ((PARTS & 1) && (d.mode == TQ_ROW_GAUSS || d.mode == TQ_ROW_BOX) && !c.cg) {
            // c == 1: every element block is em1 (x) em2, so the row's block
            // is a two-stage contraction over its (p1+1) x (p2+1) element grid:
            //   inner[k1][o2] = sum_e2 [interior, outside box] em2[e2][a2][b2(o2)]
            //   blk[o1][o2]   = sum_k1 em1[e1][a1][b1(o1)] inner[k1][o2]
            // (dependency chains of <= p+1 terms instead of a warp-serial
            // loop over the elements; same terms, grouped by e1)
            // The row's element window (spans, interior flags, em slices) is
            // staged first with independent loads; both stages then read
            // shared memory only.
            const int ef1 = c.el_first1[i1], ne1 = c.el_last1[i1] - ef1 + 1;
            const int ef2 = c.el_first2[i2], ne2 = c.el_last2[i2] - ef2 + 1;
            const bool box = d.mode == TQ_ROW_BOX && d.a1 >= 0;
            for (int l = lane; l < ne1 * q1; l += 32) {
                const int k1 = l / q1, b1 = l - k1 * q1, e1 = ef1 + k1;
                const int f1 = c.espan1[e1] - c.p1;
                if (b1 == 0) F1[k1] = f1;
                E1[l] = c.em1[((int64_t)e1 * q1 + (i1 - f1)) * q1 + b1];
            }
            for (int l = lane; l < ne2 * q2; l += 32) {
                const int k2 = l / q2, b2 = l - k2 * q2, e2 = ef2 + k2;
                const int f2 = c.espan2[e2] - c.p2;
                if (b2 == 0) F2[k2] = f2;
                E2[l] = c.em2[((int64_t)e2 * q2 + (i2 - f2)) * q2 + b2];
            }
            for (int l = lane; l < ne1 * ne2; l += 32) {
                const int k1 = l / ne2, e1 = ef1 + k1, e2 = ef2 + (l - k1 * ne2);
                bool ok = c.elem_class[(int64_t)e1 * c.nel2 + e2] == TQ_INTERIOR;
                if (box && e1 >= d.a1 && e1 <= d.b1 && e2 >= d.a2 && e2 <= d.b2) ok = false;
                MK[l] = ok ? 1 : 0;
            }
            __syncwarp();
            for (int t = lane; t < ne1 * W2; t += 32) {
                const int k1 = t / W2, o2 = t - (t / W2) * W2;
                const int j2 = i2 - c.p2 + o2;
                double acc = 0.0;
                if (j2 >= 0 && j2 < c.n2) {
                    for (int k2 = 0; k2 < ne2; ++k2) {
                        if (!MK[k1 * ne2 + k2]) continue;
                        const int b2 = j2 - F2[k2];
                        if (b2 < 0 || b2 > c.p2) continue;
                        acc += E2[k2 * q2 + b2];
                    }
                }
                inner[t] = acc;
            }
            __syncwarp();
            for (int q = lane; q < T; q += 32) {
                const int o1 = q / W2, o2 = q - (q / W2) * W2;
                const int j1 = i1 - c.p1 + o1;
                double acc = 0.0;
                if (j1 >= 0 && j1 < c.n1) {
                    for (int k1 = 0; k1 < ne1; ++k1) {
                        const int b1 = j1 - F1[k1];
                        if (b1 < 0 || b1 > c.p1) continue;
                        acc += E1[k1 * q1 + b1] * inner[k1 * W2 + o2];
                    }
                }
                blk[q] += acc;
            }
            __syncwarp();
        } else if ((PARTS & 1) && (d.mode == TQ_ROW_GAUSS || d.mode == TQ_ROW_BOX)) {
            for (int e1 = c.el_first1[i1]; e1 <= c.el_last1[i1]; ++e1) {
                for (int e2 = c.el_first2[i2]; e2 <= c.el_last2[i2]; ++e2) {
                    if (c.elem_class[(int64_t)e1 * c.nel2 + e2] != TQ_INTERIOR) continue;
                    if (d.mode == TQ_ROW_BOX && d.a1 >= 0 && e1 >= d.a1 && e1 <= d.b1 && e2 >= d.a2 && e2 <= d.b2)
                        continue;
                    const int f1 = c.espan1[e1] - c.p1, f2 = c.espan2[e2] - c.p2;
                    const int a1 = i1 - f1, a2 = i2 - f2;
                    for (int q = lane; q < q1 * q2; q += 32) {
                        int b1 = q / q2, b2 = q - (q / q2) * q2;
                        double v = gauss_entry(c, e1, e2, a1, a2, b1, b2);
                        blk[(f1 + b1 - i1 + c.p1) * W2 + (f2 + b2 - i2 + c.p2)] += v;
                    }
                    __syncwarp();
                }
            }
        }
        // -- sum factorization (BOX, MASK)
        if ((PARTS & 2) && (d.mode == TQ_ROW_BOX || d.mode == TQ_ROW_MASK)) {
            const tq_ruleset s1 = c.sets1[d.set1];
            const tq_ruleset s2 = c.sets2[d.set2];
            const int k01 = s1.rules.k0[i1], k02 = s2.rules.k0[i2];
            const int len1 = (int)(s1.rules.wptr[i1 + 1] - s1.rules.wptr[i1]);
            const int len2 = (int)(s2.rules.wptr[i2 + 1] - s2.rules.wptr[i2]);
            int lo1 = k01, hi1 = k01 + len1, lo2 = k02, hi2 = k02 + len2;
            if (d.mode == TQ_ROW_BOX && d.a1 >= 0) {
                lo1 = max(lo1, s1.lay.offsets[d.a1]);
                hi1 = min(hi1, s1.lay.offsets[d.b1 + 1]);
                lo2 = max(lo2, s2.lay.offsets[d.a2]);
                hi2 = min(hi2, s2.lay.offsets[d.b2 + 1]);
            }
            const int n1 = hi1 - lo1, n2 = hi2 - lo2;
            if (k01 >= 0 && k02 >= 0 && n1 > 0 && n2 > 0) {
                const double* w1 = s1.rules.w + s1.rules.wptr[i1] + (lo1 - k01);
                const double* w2 = s2.rules.w + s2.rules.wptr[i2] + (lo2 - k02);
                const int jl1 = c.ov_lo1[i1], jh1 = c.ov_hi1[i1], jl2 = c.ov_lo2[i2], jh2 = c.ov_hi2[i2];
                for (int q = lane; q < n1 * W1; q += 32) {
                    int k = q / W1, o = q - (q / W1) * W1;
                    int j = i1 - c.p1 + o;
                    B1[q] = (j >= jl1 && j <= jh1) ? colloc_at(s1, c.p1, lo1 + k, j) * w1[k] : 0.0;
                }
                for (int q = lane; q < n2 * W2; q += 32) {
                    int k = q / W2, o = q - (q / W2) * W2;
                    int j = i2 - c.p2 + o;
                    B2[q] = (j >= jl2 && j <= jh2) ? colloc_at(s2, c.p2, lo2 + k, j) * w2[k] : 0.0;
                }
                __syncwarp();
                const double* G = c.grids ? c.grids[d.set1 * c.nsets2 + d.set2] : nullptr;
                if (!G && d.mode == TQ_ROW_BOX) {
                    // c == 1: the contraction factorizes into two 1-D sums
                    for (int o = lane; o < W1; o += 32) {
                        double acc = 0.0;
                        for (int k = 0; k < n1; ++k) acc += B1[k * W1 + o];
                        S1[o] = acc;
                    }
                    for (int o = lane; o < W2; o += 32) {
                        double acc = 0.0;
                        for (int k = 0; k < n2; ++k) acc += B2[k * W2 + o];
                        S2[o] = acc;
                    }
                    __syncwarp();
                    for (int q = lane; q < T; q += 32) {
                        int o1 = q / W2, o2 = q - (q / W2) * W2;
                        blk[q] += S1[o1] * S2[o2];
                    }
                } else if (G) {
                    // inner[o2][k1] = sum_k2 B2[k2][o2] G[k1][k2] (mask), with the
                    // row's n1 x n2 window of G (and the mask) staged first:
                    // one coalesced run per k1 instead of a global load per term
                    const int ld = s2.lay.npts;
                    for (int q = lane; q < n1 * n2; q += 32) {
                        const int k1 = q / n2, k2 = q - k1 * n2;
                        double g = G[(int64_t)(lo1 + k1) * ld + (lo2 + k2)];
                        if (d.mode == TQ_ROW_MASK) {
                            const int e1p = elem_of_point(s1.lay, lo1 + k1), e2p = elem_of_point(s2.lay, lo2 + k2);
                            if (c.elem_class[(int64_t)e1p * c.nel2 + e2p] != TQ_INTERIOR) g = 0.0;
                        }
                        GS[q] = g;
                    }
                    __syncwarp();
                    for (int q = lane; q < W2 * n1; q += 32) {
                        const int o2 = q / n1, k1 = q - (q / n1) * n1;
                        const double* gr = GS + k1 * n2;
                        double acc = 0.0;
                        for (int k2 = 0; k2 < n2; ++k2) acc += B2[k2 * W2 + o2] * gr[k2];
                        inner[o2 * n1 + k1] = acc;
                    }
                    __syncwarp();
                    for (int q = lane; q < T; q += 32) {
                        int o1 = q / W2, o2 = q - (q / W2) * W2;
                        double acc = 0.0;
                        for (int k1 = 0; k1 < n1; ++k1) acc += B1[k1 * W1 + o1] * inner[o2 * n1 + k1];
                        blk[q] += acc;
                    }
                } else {
                    // inner[o2][k1] = sum_k2 B2[k2][o2] G[k1][k2] (mask)
                    const int ld = s2.lay.npts;
                    for (int q = lane; q < W2 * n1; q += 32) {
                        int o2 = q / n1, k1 = q - (q / n1) * n1;
                        int e1p = d.mode == TQ_ROW_MASK ? elem_of_point(s1.lay, lo1 + k1) : 0;
                        double acc = 0.0;
                        for (int k2 = 0; k2 < n2; ++k2) {
                            double g = G ? G[(int64_t)(lo1 + k1) * ld + (lo2 + k2)] : 1.0;
                            if (d.mode == TQ_ROW_MASK) {
                                int e2p = elem_of_point(s2.lay, lo2 + k2);
                                if (c.elem_class[(int64_t)e1p * c.nel2 + e2p] != TQ_INTERIOR) g = 0.0;
                            }
                            acc += B2[k2 * W2 + o2] * g;
                        }
                        inner[o2 * n1 + k1] = acc;
                    }
                    __syncwarp();
                    for (int q = lane; q < T; q += 32) {
                        int o1 = q / W2, o2 = q - (q / W2) * W2;
                        double acc = 0.0;
                        for (int k1 = 0; k1 < n1; ++k1) acc += B1[k1 * W1 + o1] * inner[o2 * n1 + k1];
                        blk[q] += acc;
                    }
                }
                __syncwarp();
            }
        }
        const RawRow dst = raw_row(c, r);
        for (int q = lane; q < T; q += 32) dst[q] = blk[q];
        __syncwarp();
    }
}

// The c != 1 element-Gauss part (PARTS == 1 with a coefficient grid): one
// warp per row, sum factorization over the row's (p1+1) x (p2+1) support
// elements instead of a (p+1)^2-point loop per block entry.  For each
// support column e1 (skipped when none of its elements is interior and
// outside the box):
//   inner[g1][o2] = sum_{e2 ok} sum_g2 c(e1,g1,e2,g2) w2 V2(e2,g2,a2) V2(e2,g2,b2)
//   blk[o1][o2]  += sum_g1 w1 V1(e1,g1,a1) V1(e1,g1,b1) inner[g1][o2]
// (o2 = j2 - i2 + p2, j2 = f2(e2) + b2; o1 likewise): ~(p+1)^4 (2 + (2p+1)/(p+1))
// FMA per column instead of (p+1)^6.  The row's element window (spans,
// flags, direction-2 values) is staged once, the column's c slice (one
// contiguous run per g1) and direction-1 products per column; every stage
// reads shared memory only.  MASK rows get an all-zero block, like the
// generic kernel.  Same terms as _Run.element_block (src/assembly.py:310-332)
// summed in a different order (not bit-identical to the generic kernel).
__host__ __device__ inline int gauss_coef_slots(int p1, int p2, int ng1, int ng2) {
    const int q1 = p1 + 1, q2 = p2 + 1, W1 = 2 * p1 + 1, W2 = 2 * p2 + 1;
    return W1 * W2                       // blk
           + q2 * ng2 * q2               // V2 window
           + q2 * ng2                    // w2 V2(a2)
           + ng1 * q2 * ng2              // c slice x w2 V2(a2), one column
           + ng1 * W2                    // inner
           + ng1 * q1                    // w1 V1(a1) V1(b1)
           + (q1 + q2 + q1 * q2 + 1) / 2 + 1;   // spans and flags (ints)
}

// A BOX row whose box is its whole support (the interior rows of the c != 1
// BOX plan) has no element-Gauss part: the Gauss kernel leaves its block
// untouched and the sum-factorization kernel writes it (0 + x == x: the
// same values as zero-then-add).
__device__ __forceinline__ bool full_box_row(const tq_rawctx& c, const RowDesc& d, int i1, int i2) {
    return d.mode == TQ_ROW_BOX && d.a1 == c.el_first1[i1] && d.b1 == c.el_last1[i1] && d.a2 == c.el_first2[i2] &&
           d.b2 == c.el_last2[i2];
}

template <int NT, int P>
__global__ void __launch_bounds__(NT) k_raw_gauss_coef(tq_rawctx c, int r0, int r1) {
    // one block of NT threads per row (the row's windows are shared by the
    // whole block: NT/32 times the parallelism of a warp per row for the
    // same shared memory).  P > 0: p1 == p2 == P and P + 1 Gauss points per
    // element at compile time (constant divisors in the index arithmetic).
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    const int p1 = P ? P : c.p1, p2 = P ? P : c.p2, q1 = p1 + 1, q2 = p2 + 1, W2 = 2 * p2 + 1,
              T = (2 * p1 + 1) * W2;
    const int ng1 = P ? P + 1 : c.ng1, ng2 = P ? P + 1 : c.ng2;
    double* blk = sm;
    double* V2 = blk + T;                   // [k2][g2][b2]
    double* A2 = V2 + q2 * ng2 * q2;        // [k2][g2]
    double* CV = A2 + q2 * ng2;             // [g1][k2][g2]
    double* inner = CV + ng1 * q2 * ng2;    // [g1][o2]
    double* P1 = inner + ng1 * W2;          // [g1][b1]
    int* F1 = reinterpret_cast<int*>(P1 + ng1 * q1);
    int* F2 = F1 + q1;
    int* MK = F2 + q2;
    const int64_t ld = (int64_t)c.nel2 * ng2;
    for (int r = r0 + blockIdx.x; r < r1; r += gridDim.x) {
        const RowDesc d = reinterpret_cast<const RowDesc*>(c.desc)[r];
        const RawRow dst = raw_row(c, r);
        bool work = d.mode == TQ_ROW_GAUSS || d.mode == TQ_ROW_BOX;
        const int i1 = d.fidx / c.n2, i2 = d.fidx - (d.fidx / c.n2) * c.n2;
        if (full_box_row(c, d, i1, i2)) continue;        // uniform: written by k_raw_sf_coef
        const int ef1 = c.el_first1[i1], ne1 = c.el_last1[i1] - ef1 + 1;
        const int ef2 = c.el_first2[i2], ne2 = c.el_last2[i2] - ef2 + 1;
        bool mine = false;
        if (work) {
            const bool box = d.mode == TQ_ROW_BOX && d.a1 >= 0;
            for (int k = tid; k < ne1; k += NT) F1[k] = c.espan1[ef1 + k] - p1;
            for (int k = tid; k < ne2; k += NT) F2[k] = c.espan2[ef2 + k] - p2;
            for (int l = tid; l < ne1 * ne2; l += NT) {
                const int k1 = l / ne2, e1 = ef1 + k1, e2 = ef2 + (l - k1 * ne2);
                bool ok = c.elem_class[(int64_t)e1 * c.nel2 + e2] == TQ_INTERIOR;
                if (box && e1 >= d.a1 && e1 <= d.b1 && e2 >= d.a2 && e2 <= d.b2) ok = false;
                MK[l] = ok ? 1 : 0;
                mine = mine || ok;
            }
        }
        // rows whose box covers every interior support element (all the
        // interior rows of the c != 1 BOX plan) have no Gauss part
        if (!__syncthreads_or(mine)) {
            for (int q = tid; q < T; q += NT) dst[q] = 0.0;
            continue;
        }
        for (int q = tid; q < T; q += NT) blk[q] = 0.0;
        // direction-2 window: the elements are consecutive, so their value
        // tables are one contiguous run
        const double* v2src = c.ev2 + (int64_t)ef2 * ng2 * q2;
        for (int l = tid; l < ne2 * ng2 * q2; l += NT) V2[l] = v2src[l];
        __syncthreads();
        for (int l = tid; l < ne2 * ng2; l += NT) {
            const int k2 = l / ng2;
            A2[l] = c.ew2[(int64_t)ef2 * ng2 + l] * V2[l * q2 + (i2 - F2[k2])];
        }
        __syncthreads();
        for (int k1 = 0; k1 < ne1; ++k1) {
            bool any = false;
            for (int k2 = 0; k2 < ne2; ++k2) any = any || MK[k1 * ne2 + k2];
            if (!any) continue;                 // uniform across the block
            const int e1 = ef1 + k1, a1 = i1 - F1[k1];
            for (int l = tid; l < ng1 * ne2 * ng2; l += NT) {
                const int g1 = l / (ne2 * ng2), m = l - g1 * (ne2 * ng2);
                CV[l] = c.cg[((int64_t)e1 * ng1 + g1) * ld + (int64_t)ef2 * ng2 + m] * A2[m];
            }
            for (int l = tid; l < ng1 * q1; l += NT) {
                const int g1 = l / q1, b1 = l - g1 * q1;
                const double* v = c.ev1 + ((int64_t)e1 * ng1 + g1) * q1;
                P1[l] = (c.ew1[(int64_t)e1 * ng1 + g1] * v[a1]) * v[b1];
            }
            __syncthreads();
            for (int t = tid; t < ng1 * W2; t += NT) {
                const int g1 = t / W2, o2 = t - g1 * W2;
                const int j2 = i2 - p2 + o2;
                double acc = 0.0;
                for (int k2 = 0; k2 < ne2; ++k2) {
                    const int b2 = j2 - F2[k2];
                    if (b2 < 0 || b2 > p2 || !MK[k1 * ne2 + k2]) continue;
                    const double* cv = CV + (g1 * ne2 + k2) * ng2;
                    const double* v2 = V2 + k2 * ng2 * q2 + b2;
                    for (int g2 = 0; g2 < ng2; ++g2) acc += cv[g2] * v2[g2 * q2];
                }
                inner[t] = acc;
            }
            __syncthreads();
            for (int t = tid; t < q1 * W2; t += NT) {
                const int b1 = t / W2, o2 = t - b1 * W2;
                double acc = 0.0;
                for (int g1 = 0; g1 < ng1; ++g1) acc += P1[g1 * q1 + b1] * inner[g1 * W2 + o2];
                blk[(F1[k1] + b1 - i1 + p1) * W2 + o2] += acc;
            }
            __syncthreads();
        }
        for (int q = tid; q < T; q += NT) dst[q] = blk[q];
        __syncthreads();
    }
}

// The c != 1 sum-factorization part (PARTS == 2 with coefficient grids): one
// block of NT threads per row; the weighted collocation slices and the row's
// n1 x n2 coefficient window (masked for MASK rows) are staged in shared
// memory, then inner[o2][k1] = sum_k2 B2[k2][o2] G[k1][k2] and
// M[o1][o2] += sum_k1 B1[k1][o1] inner[o2][k1] -- the additions of the
// warp-per-row kernel in the same order (sum_factor_row, src/assembly.py:218-252).
// (the coefficient window and inner have odd row strides: the column
// accesses of the two contractions are bank-conflict free)
constexpr int kSfOB = 4;      // outputs per thread along the window in the c != 1 contractions

__host__ __device__ inline int sf_coef_slots(const tq_rawctx& c) {
    const int W1 = 2 * c.p1 + 1, W2 = 2 * c.p2 + 1;
    return c.nmax1 * W1 + c.nmax2 * W2 + c.nmax1 * (c.nmax2 | 1) + W2 * (c.nmax1 | 1);
}

// P > 0: p1 == p2 == P at compile time (window sizes constant: the index
// arithmetic of every stage divides by constants); P == 0: runtime degrees.
template <int NT, int P>
__global__ void __launch_bounds__(NT) k_raw_sf_coef(tq_rawctx c, int r0, int r1) {
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    const int W1 = P ? 2 * P + 1 : 2 * c.p1 + 1, W2 = P ? 2 * P + 1 : 2 * c.p2 + 1, T = W1 * W2;
    const int p1 = P ? P : c.p1, p2 = P ? P : c.p2;
    // outputs per thread along the window: a third of it (P > 0), else kSfOB
    constexpr int OB = P ? (2 * P + 3) / 3 : kSfOB;
    double* B1 = sm;
    double* B2 = B1 + c.nmax1 * W1;
    double* GS = B2 + c.nmax2 * W2;
    double* inner = GS + c.nmax1 * (c.nmax2 | 1);
    for (int r = r0 + blockIdx.x; r < r1; r += gridDim.x) {
        const RowDesc d = reinterpret_cast<const RowDesc*>(c.desc)[r];
        if (d.mode != TQ_ROW_BOX && d.mode != TQ_ROW_MASK) continue;     // uniform: nothing to add
        const int i1 = d.fidx / c.n2, i2 = d.fidx - (d.fidx / c.n2) * c.n2;
        const tq_ruleset s1 = c.sets1[d.set1];
        const tq_ruleset s2 = c.sets2[d.set2];
        const int k01 = s1.rules.k0[i1], k02 = s2.rules.k0[i2];
        const int len1 = (int)(s1.rules.wptr[i1 + 1] - s1.rules.wptr[i1]);
        const int len2 = (int)(s2.rules.wptr[i2 + 1] - s2.rules.wptr[i2]);
        int lo1 = k01, hi1 = k01 + len1, lo2 = k02, hi2 = k02 + len2;
        if (d.mode == TQ_ROW_BOX && d.a1 >= 0) {
            lo1 = max(lo1, s1.lay.offsets[d.a1]);
            hi1 = min(hi1, s1.lay.offsets[d.b1 + 1]);
            lo2 = max(lo2, s2.lay.offsets[d.a2]);
            hi2 = min(hi2, s2.lay.offsets[d.b2 + 1]);
        }
        const int n1 = hi1 - lo1, n2 = hi2 - lo2;
        const int ldg = n2 | 1, ldi = n1 | 1;            // odd strides
        const bool write = full_box_row(c, d, i1, i2);
        if (!(k01 >= 0 && k02 >= 0 && n1 > 0 && n2 > 0)) {       // uniform
            if (write)
                for (int q = tid; q < T; q += NT) raw_row(c, r)[q] = 0.0;
            continue;
        }
        const double* w1 = s1.rules.w + s1.rules.wptr[i1] + (lo1 - k01);
        const double* w2 = s2.rules.w + s2.rules.wptr[i2] + (lo2 - k02);
        const int jl1 = c.ov_lo1[i1], jh1 = c.ov_hi1[i1], jl2 = c.ov_lo2[i2], jh2 = c.ov_hi2[i2];
        for (int q = tid; q < n1 * W1; q += NT) {
            const int k = q / W1, o = q - (q / W1) * W1;
            const int j = i1 - p1 + o;
            B1[q] = (j >= jl1 && j <= jh1) ? colloc_at(s1, p1, lo1 + k, j) * w1[k] : 0.0;
        }
        for (int q = tid; q < n2 * W2; q += NT) {
            const int k = q / W2, o = q - (q / W2) * W2;
            const int j = i2 - p2 + o;
            B2[q] = (j >= jl2 && j <= jh2) ? colloc_at(s2, p2, lo2 + k, j) * w2[k] : 0.0;
        }
        const double* G = c.grids[d.set1 * c.nsets2 + d.set2];
        const int ld = s2.lay.npts;
        for (int q = tid; q < n1 * n2; q += NT) {
            const int k1 = q / n2, k2 = q - k1 * n2;
            double g = G[(int64_t)(lo1 + k1) * ld + (lo2 + k2)];
            if (d.mode == TQ_ROW_MASK) {
                const int e1p = elem_of_point(s1.lay, lo1 + k1), e2p = elem_of_point(s2.lay, lo2 + k2);
                if (c.elem_class[(int64_t)e1p * c.nel2 + e2p] != TQ_INTERIOR) g = 0.0;
            }
            GS[k1 * ldg + k2] = g;
        }
        __syncthreads();
        // stage 1: a thread owns one k1 and OB consecutive o2 (lanes run
        // over k1: the column reads of G are conflict-free, the B2 reads
        // broadcast; one G load feeds OB FMAs)
        {
            int KT = 32;                               // power of two >= n1
            while (KT < n1) KT *= 2;
            const int ng = (W2 + OB - 1) / OB;
            for (int q = tid; q < KT * ng; q += NT) {
                const int k1 = q & (KT - 1), og = q / KT;
                if (k1 >= n1) continue;
                const int o0 = og * OB;
                const double* gr = GS + k1 * ldg;
                double acc[OB];
#pragma unroll
                for (int z = 0; z < OB; ++z) acc[z] = 0.0;
                for (int k2 = 0; k2 < n2; ++k2) {
                    const double g = gr[k2];
                    const double* b2 = B2 + k2 * W2 + o0;
#pragma unroll
                    for (int z = 0; z < OB; ++z)
                        if (o0 + z < W2) acc[z] += b2[z] * g;
                }
#pragma unroll
                for (int z = 0; z < OB; ++z)
                    if (o0 + z < W2) inner[(o0 + z) * ldi + k1] = acc[z];
            }
        }
        __syncthreads();
        // stage 2: a thread owns one o2 and OB consecutive o1 (one inner
        // load feeds OB FMAs; the B1 reads broadcast)
        const RawRow dst = raw_row(c, r);
        {
            const int ng = (W1 + OB - 1) / OB;
            for (int q = tid; q < W2 * ng; q += NT) {
                const int og = q / W2, o2 = q - og * W2, o0 = og * OB;
                const double* in = inner + o2 * ldi;
                double acc[OB];
#pragma unroll
                for (int z = 0; z < OB; ++z) acc[z] = 0.0;
                for (int k1 = 0; k1 < n1; ++k1) {
                    const double v = in[k1];
                    const double* b1 = B1 + k1 * W1 + o0;
#pragma unroll
                    for (int z = 0; z < OB; ++z)
                        if (o0 + z < W1) acc[z] += b1[z] * v;
                }
#pragma unroll
                for (int z = 0; z < OB; ++z) {
                    if (o0 + z >= W1) break;
                    const int qq = (o0 + z) * W2 + o2;
                    if (write) dst[qq] = acc[z];
                    else dst[qq] += acc[z];
                }
            }
        }
        __syncthreads();
    }
}

// Element blocks of the cut elements: one warp per (cut element, span key)
// group, G[A][B] = sum_pts (c w) B_A B_B with A = (a1, a2), B = (b1, b2)
// local indices -- the B2d^T (cw B2d) of src/assembly.py:384-387.  A group
// holds ~q^2 points and Q^2 entries, so the work is tiny and latency-bound:
// lane l owns the (a1, b1) pair l (+32, ...) and keeps the Q2 x Q2 (a2, b2)
// accumulators in registers; points are staged 32 at a time in warp-private
// shared memory (one lane gathers one point through the group permutation).
template <int Q2>
__global__ void k_cut_blocks(tq_rawctx c) {
    extern __shared__ double sm[];
    const int q1 = c.p1 + 1, Q = q1 * Q2, st = q1 + Q2 + 1;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    double* sp = sm + wib * 32 * st;
    for (int g = blockIdx.x * wpb + wib; g < c.ngroups; g += gridDim.x * wpb) {
        const int64_t p0 = c.grp_pts[g], pe = c.grp_pts[g + 1];
        for (int pr0 = 0; pr0 < q1 * q1; pr0 += 32) {
            const int pr = pr0 + lane;
            const bool act = pr < q1 * q1;
            const int a1 = act ? pr / q1 : 0, b1 = act ? pr - (pr / q1) * q1 : 0;
            double acc[Q2 * Q2];
#pragma unroll
            for (int z = 0; z < Q2 * Q2; ++z) acc[z] = 0.0;
            for (int64_t base = p0; base < pe; base += 32) {
                const int np = (int)(pe - base < 32 ? pe - base : 32);
                __syncwarp();
                if (lane < np) {
                    const int64_t pt = c.grp_perm[base + lane];
                    double* d = sp + lane * st;
                    for (int o = 0; o < q1; ++o) d[o] = c.cvals1[pt * q1 + o];
#pragma unroll
                    for (int o = 0; o < Q2; ++o) d[q1 + o] = c.cvals2[pt * Q2 + o];
                    d[q1 + Q2] = c.cut_cw[pt];
                }
                __syncwarp();
                if (act) {
                    for (int k = 0; k < np; ++k) {
                        const double* d = sp + k * st;
                        const double s = (d[q1 + Q2] * d[a1]) * d[b1];
                        double v2[Q2];
#pragma unroll
                        for (int o = 0; o < Q2; ++o) v2[o] = d[q1 + o];
#pragma unroll
                        for (int a2 = 0; a2 < Q2; ++a2) {
                            const double u = s * v2[a2];
#pragma unroll
                            for (int b2 = 0; b2 < Q2; ++b2) acc[a2 * Q2 + b2] = fma(u, v2[b2], acc[a2 * Q2 + b2]);
                        }
                    }
                }
            }
            if (act) {
                double* out = c.grp_blocks + (int64_t)g * Q * Q;
#pragma unroll
                for (int a2 = 0; a2 < Q2; ++a2)
#pragma unroll
                    for (int b2 = 0; b2 < Q2; ++b2) out[(a1 * Q2 + a2) * Q + b1 * Q2 + b2] = acc[a2 * Q2 + b2];
            }
        }
    }
}

// The same element blocks with one block of kCbThreads per group (large
// degrees: q^2 (a1, b1) pairs x Q2^2 accumulators no longer fit a warp):
// a thread owns one (a1, b1) pair and kCbA2 consecutive a2 -- kCbA2 x Q2
// accumulators -- and the group's points are staged kCbChunk at a time for
// the whole block.  Per output the additions are those of k_cut_blocks in
// the same order (bit-identical).
constexpr int kCbThreads = 256, kCbChunk = 256, kCbA2 = 3;

template <int Q2>
__global__ void __launch_bounds__(kCbThreads) k_cut_blocks_wide(tq_rawctx c) {
    extern __shared__ double sm[];
    constexpr int S = (Q2 + kCbA2 - 1) / kCbA2;          // a2 subsets per (a1, b1)
    const int q1 = c.p1 + 1, Q = q1 * Q2, st = q1 + Q2 + 1;
    const int ntask = q1 * q1 * S;
    for (int g = blockIdx.x; g < c.ngroups; g += gridDim.x) {
        const int64_t p0 = c.grp_pts[g], pe = c.grp_pts[g + 1];
        for (int t0 = 0; t0 < ntask; t0 += kCbThreads) {      // one pass when q1^2 S <= kCbThreads
            const int t = t0 + threadIdx.x;
            const bool act = t < ntask;
            const int pr = act ? t / S : 0, sub = act ? t - (t / S) * S : 0;
            const int a1 = pr / q1, b1 = pr - (pr / q1) * q1, a20 = sub * kCbA2;
            double acc[kCbA2 * Q2];
#pragma unroll
            for (int z = 0; z < kCbA2 * Q2; ++z) acc[z] = 0.0;
            for (int64_t base = p0; base < pe; base += kCbChunk) {
                const int np = (int)(pe - base < kCbChunk ? pe - base : kCbChunk);
                __syncthreads();
                // a thread stages whole points: one permutation lookup, then
                // q1 + Q2 + 1 independent loads
                for (int k = threadIdx.x; k < np; k += kCbThreads) {
                    const int64_t pt = c.grp_perm[base + k];
                    double* d = sm + k * st;
                    for (int o = 0; o < q1; ++o) d[o] = c.cvals1[pt * q1 + o];
#pragma unroll
                    for (int o = 0; o < Q2; ++o) d[q1 + o] = c.cvals2[pt * Q2 + o];
                    d[q1 + Q2] = c.cut_cw[pt];
                }
                __syncthreads();
                if (act) {
                    for (int k = 0; k < np; ++k) {
                        const double* d = sm + k * st;
                        const double s = (d[q1 + Q2] * d[a1]) * d[b1];
                        double v2[Q2];
#pragma unroll
                        for (int o = 0; o < Q2; ++o) v2[o] = d[q1 + o];
#pragma unroll
                        for (int z = 0; z < kCbA2; ++z) {
                            if (a20 + z >= Q2) break;
                            const double u = s * d[q1 + a20 + z];     // (no runtime index into v2: registers)
#pragma unroll
                            for (int b2 = 0; b2 < Q2; ++b2) acc[z * Q2 + b2] = fma(u, v2[b2], acc[z * Q2 + b2]);
                        }
                    }
                }
            }
            if (act) {
                double* out = c.grp_blocks + (int64_t)g * Q * Q;
#pragma unroll
                for (int z = 0; z < kCbA2; ++z) {
                    if (a20 + z >= Q2) break;
#pragma unroll
                    for (int b2 = 0; b2 < Q2; ++b2) out[(a1 * Q2 + a20 + z) * Q + b1 * Q2 + b2] = acc[z * Q2 + b2];
                }
            }
        }
    }
}

// Row gather of the element blocks into the raw rows (warp per row).
// (planes layout: the row's contributions are summed in a warp-private
// shared block first and added to its strided planes once)
__global__ void k_raw_cutcells(tq_rawctx c, int r0, int r1) {
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int W2 = 2 * c.p2 + 1, T = (2 * c.p1 + 1) * W2;
    const int q1 = c.p1 + 1, q2 = c.p2 + 1, Q = q1 * q2;
    double* acc = sm + (threadIdx.x >> 5) * T;
    for (int r = r0 + blockIdx.x * wpb + (threadIdx.x >> 5); r < r1; r += gridDim.x * wpb) {
        RowDesc d = reinterpret_cast<const RowDesc*>(c.desc)[r];
        const int i1 = d.fidx / c.n2, i2 = d.fidx - (d.fidx / c.n2) * c.n2;
        const int ea1 = max(c.el_first1[i1] - 1, 0), eb1 = min(c.el_last1[i1] + 1, c.nel1 - 1);
        const int ea2 = max(c.el_first2[i2] - 1, 0), eb2 = min(c.el_last2[i2] + 1, c.nel2 - 1);
        const int w2 = eb2 - ea2 + 1, nh = (eb1 - ea1 + 1) * w2;
        const RawRow dst = c.raw_ld ? RawRow{acc, 1} : raw_row(c, r);
        bool touched = false;
        if (c.raw_ld) {
            for (int q = lane; q < T; q += 32) acc[q] = 0.0;
            __syncwarp();
        }
        for (int h0 = 0; h0 < nh; h0 += 32) {
            int h = h0 + lane;
            int id = -1;
            if (h < nh) id = c.cutidx[(int64_t)(ea1 + h / w2) * c.nel2 + (ea2 + h % w2)];
            unsigned m = __ballot_sync(0xffffffffu, id >= 0);
            while (m) {
                int src = __ffs(m) - 1;
                m &= m - 1;
                int cid = __shfl_sync(0xffffffffu, id, src);
                for (int g = c.grp_ptr[cid]; g < c.grp_ptr[cid + 1]; ++g) {
                    const int f1 = c.grp_key[2 * g], f2 = c.grp_key[2 * g + 1];
                    const int a1 = i1 - f1, a2 = i2 - f2;
                    if (a1 < 0 || a1 > c.p1 || a2 < 0 || a2 > c.p2) continue;
                    touched = true;
                    const double* G = c.grp_blocks + ((int64_t)g * Q + (a1 * q2 + a2)) * Q;
                    for (int B = lane; B < Q; B += 32) {
                        int b1 = B / q2, b2 = B - (B / q2) * q2;
                        dst[(f1 + b1 - i1 + c.p1) * W2 + (f2 + b2 - i2 + c.p2)] += G[B];
                    }
                }
            }
        }
        if (c.raw_ld && touched) {      // warp-uniform
            __syncwarp();
            const RawRow out = raw_row(c, r);
            for (int q = lane; q < T; q += 32) out[q] += acc[q];
        }
        __syncwarp();
    }
}

// Per raw row, the span-key groups k_raw_cutcells adds (cut elements of the
// row's support window in window order, their groups in order, key within
// the row's reach): geometry of the plan, built once per configuration
// (COUNT: the counts; else the (group, key1, key2) triplets at off[r - r0]).
template <bool COUNT>
__global__ void k_row_groups(tq_rawctx c, int r0, int r1, const int32_t* __restrict__ off, int32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int r = r0 + warp; r < r1; r += nw) {
        RowDesc d = reinterpret_cast<const RowDesc*>(c.desc)[r];
        const int i1 = d.fidx / c.n2, i2 = d.fidx - (d.fidx / c.n2) * c.n2;
        const int ea1 = max(c.el_first1[i1] - 1, 0), eb1 = min(c.el_last1[i1] + 1, c.nel1 - 1);
        const int ea2 = max(c.el_first2[i2] - 1, 0), eb2 = min(c.el_last2[i2] + 1, c.nel2 - 1);
        const int w2 = eb2 - ea2 + 1, nh = (eb1 - ea1 + 1) * w2;
        int n = 0;
        int32_t* o = COUNT ? nullptr : out + 3 * (int64_t)off[r - r0];
        for (int h0 = 0; h0 < nh; h0 += 32) {
            const int h = h0 + lane;
            const int id = h < nh ? c.cutidx[(int64_t)(ea1 + h / w2) * c.nel2 + (ea2 + h % w2)] : -1;
            unsigned m = __ballot_sync(0xffffffffu, id >= 0);
            while (m) {
                const int src = __ffs(m) - 1;
                m &= m - 1;
                const int cid = __shfl_sync(0xffffffffu, id, src);
                const int gb = c.grp_ptr[cid], ge = c.grp_ptr[cid + 1];
                for (int g0 = gb; g0 < ge; g0 += 32) {       // lanes over the element's groups
                    const int g = g0 + lane;
                    bool ok = false;
                    int f1 = 0, f2 = 0;
                    if (g < ge) {
                        f1 = c.grp_key[2 * g];
                        f2 = c.grp_key[2 * g + 1];
                        const int a1 = i1 - f1, a2 = i2 - f2;
                        ok = a1 >= 0 && a1 <= c.p1 && a2 >= 0 && a2 <= c.p2;
                    }
                    const unsigned vm = __ballot_sync(0xffffffffu, ok);
                    if (!COUNT && ok) {
                        const int at = n + __popc(vm & ((1u << lane) - 1u));
                        o[3 * at] = g;
                        o[3 * at + 1] = f1;
                        o[3 * at + 2] = f2;
                    }
                    n += __popc(vm);
                }
            }
        }
        if (COUNT && lane == 0) out[r - r0] = n;
    }
}

// k_raw_cutcells over the per-row group lists (k_row_groups): the group
// row slices of a batch of kCcBatch groups are loaded together, then added
// in list order into a shared copy of the row (row-major raw rows: loaded
// first, so the result is bit-identical to k_raw_cutcells; planes: summed
// from zero and added, as there).  A few dependent load rounds per row
// instead of the element-window scan and two global round trips per group.
constexpr int kCcBatch = 8;

__global__ void k_raw_cutcells_list(tq_rawctx c, int r0, int r1, const int32_t* __restrict__ rg_ptr,
                                    const int32_t* __restrict__ rg) {
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5, wib = threadIdx.x >> 5;
    const int W2 = 2 * c.p2 + 1, T = (2 * c.p1 + 1) * W2;
    const int q2 = c.p2 + 1, Q = (c.p1 + 1) * q2;
    double* acc = sm + wib * T;
    const int lb1 = lane / q2, lb2 = lane - (lane / q2) * q2;
    for (int r = r0 + blockIdx.x * wpb + wib; r < r1; r += gridDim.x * wpb) {
        const int gb = __ldg(rg_ptr + (r - r0)), ge = __ldg(rg_ptr + (r - r0) + 1);
        if (ge == gb) continue;
        RowDesc d = reinterpret_cast<const RowDesc*>(c.desc)[r];
        const int i1 = d.fidx / c.n2, i2 = d.fidx - (d.fidx / c.n2) * c.n2;
        const RawRow out = raw_row(c, r);
        for (int q = lane; q < T; q += 32) acc[q] = c.raw_ld ? 0.0 : out[q];
        __syncwarp();
        for (int k0 = gb; k0 < ge; k0 += kCcBatch) {
            double v[kCcBatch];
            int at[kCcBatch];
#pragma unroll
            for (int u = 0; u < kCcBatch; ++u) {
                const int k = k0 + u;
                at[u] = -1;
                v[u] = 0.0;
                if (k < ge && lane < Q) {
                    const int g = __ldg(rg + 3 * k), f1 = __ldg(rg + 3 * k + 1), f2 = __ldg(rg + 3 * k + 2);
                    const int a1 = i1 - f1, a2 = i2 - f2;
                    v[u] = __ldg(c.grp_blocks + ((int64_t)g * Q + (a1 * q2 + a2)) * Q + lane);
                    at[u] = (f1 + lb1 - i1 + c.p1) * W2 + (f2 + lb2 - i2 + c.p2);
                }
            }
#pragma unroll
            for (int u = 0; u < kCcBatch; ++u) {
                if (at[u] >= 0) acc[at[u]] += v[u];
                __syncwarp();
            }
        }
        __syncwarp();
        if (c.raw_ld) {
            for (int q = lane; q < T; q += 32) out[q] += acc[q];
        } else {
            for (int q = lane; q < T; q += 32) out[q] = acc[q];
        }
        __syncwarp();
    }
}

__device__ inline double detj(const tq_coeff& g, double u, double v) {
    double N1[kMaxP + 1], D1[kMaxP + 1], N2[kMaxP + 1], D2[kMaxP + 1];
    const int nk = g.n + g.p + 1;
    int s1 = find_span(g.knots, nk, g.p, g.n, u), s2 = find_span(g.knots, nk, g.p, g.n, v);
    basis_funs_ders_rt(g.knots, g.p, s1, u, N1, D1);
    basis_funs_ders_rt(g.knots, g.p, s2, v, N2, D2);
    double xu = 0, xv = 0, yu = 0, yv = 0;
    for (int a = 0; a <= g.p; ++a)
        for (int b = 0; b <= g.p; ++b) {
            int64_t idx = (int64_t)(s1 - g.p + a) * g.n + (s2 - g.p + b);
            double X = g.X[idx], Y = g.Y[idx];
            xu += D1[a] * N2[b] * X;
            xv += N1[a] * D2[b] * X;
            yu += D1[a] * N2[b] * Y;
            yv += N1[a] * D2[b] * Y;
        }
    return xu * yv - xv * yu;
}

__global__ void k_coeff_grid(tq_coeff g, const double* x1, int n1, const double* x2, int n2, double* out) {
    int64_t total = (int64_t)n1 * n2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int a = (int)(t / n2), b = (int)(t - (int64_t)a * n2);
        out[t] = detj(g, x1[a], x2[b]);
    }
}

// Tensor grids: a block covers kCgA x kCgB grid points.  The spans and
// basis values (and derivatives) of its grid lines are computed once into
// shared memory; then the control net is contracted along direction 2 for
// every b-line of the tile (XB[i][b] = sum_j N_j(x2_b) X[i][j], and with the
// derivatives), and each point is a (p+1)-term contraction per partial
// derivative: 4 (p+1) multiply-adds instead of 4 (p+1)^2.  (Same terms as
// detj, summed in a different order.)  Tiles whose a-lines touch more than
// kCgR control rows fall back to the per-point contraction.
constexpr int kCgA = 32, kCgB = 64, kCgR = 12;

__global__ void __launch_bounds__(256) k_coeff_grid_tiled(tq_coeff g, const double* __restrict__ x1, int n1,
                                                          const double* __restrict__ x2, int n2,
                                                          double* __restrict__ out) {
    constexpr int P1 = kMaxP + 1;
    __shared__ double Na[kCgA][P1], Da[kCgA][P1], Nb[kCgB][P1], Db[kCgB][P1];
    __shared__ double XB[kCgR][kCgB], XDB[kCgR][kCgB], YB[kCgR][kCgB], YDB[kCgR][kCgB];
    __shared__ int sa[kCgA], sb[kCgB];
    __shared__ int rng[2];
    const int a0 = blockIdx.y * kCgA, b0 = blockIdx.x * kCgB;
    const int nk = g.n + g.p + 1;
    if (threadIdx.x == 0) {
        rng[0] = INT_MAX;
        rng[1] = INT_MIN;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < kCgA + kCgB; t += blockDim.x) {
        const bool isa = t < kCgA;
        const int l = isa ? t : t - kCgA;
        const int gi = (isa ? a0 : b0) + l;
        if (gi >= (isa ? n1 : n2)) continue;
        const double u = isa ? x1[gi] : x2[gi];
        const int sp = find_span(g.knots, nk, g.p, g.n, u);
        double N[P1], D[P1];
        basis_funs_ders_rt(g.knots, g.p, sp, u, N, D);
        double* No = isa ? Na[l] : Nb[l];
        double* Do = isa ? Da[l] : Db[l];
        for (int k = 0; k <= g.p; ++k) {
            No[k] = N[k];
            Do[k] = D[k];
        }
        (isa ? sa : sb)[l] = sp;
        if (isa) {
            atomicMin(&rng[0], sp - g.p);
            atomicMax(&rng[1], sp);
        }
    }
    __syncthreads();
    const int i0 = rng[0], R = rng[1] - rng[0] + 1;
    const int nbl = min(kCgB, n2 - b0), nal = min(kCgA, n1 - a0);
    if (R <= kCgR) {
        for (int t = threadIdx.x; t < R * nbl; t += blockDim.x) {
            const int ii = t / nbl, bl = t - ii * nbl;
            const double* Xr = g.X + (int64_t)(i0 + ii) * g.n + (sb[bl] - g.p);
            const double* Yr = g.Y + (int64_t)(i0 + ii) * g.n + (sb[bl] - g.p);
            double xb = 0, xdb = 0, yb = 0, ydb = 0;
            for (int j = 0; j <= g.p; ++j) {
                const double X = __ldg(Xr + j), Y = __ldg(Yr + j);
                xb += Nb[bl][j] * X;
                xdb += Db[bl][j] * X;
                yb += Nb[bl][j] * Y;
                ydb += Db[bl][j] * Y;
            }
            XB[ii][bl] = xb;
            XDB[ii][bl] = xdb;
            YB[ii][bl] = yb;
            YDB[ii][bl] = ydb;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < nal * nbl; t += blockDim.x) {
            const int al = t / nbl, bl = t - al * nbl;
            const int r0 = sa[al] - g.p - i0;
            double xu = 0, xv = 0, yu = 0, yv = 0;
            for (int i = 0; i <= g.p; ++i) {
                xu += Da[al][i] * XB[r0 + i][bl];
                xv += Na[al][i] * XDB[r0 + i][bl];
                yu += Da[al][i] * YB[r0 + i][bl];
                yv += Na[al][i] * YDB[r0 + i][bl];
            }
            out[(int64_t)(a0 + al) * n2 + b0 + bl] = xu * yv - xv * yu;
        }
        return;
    }
    for (int t = threadIdx.x; t < nal * nbl; t += blockDim.x) {      // wide tile: per point
        const int al = t / nbl, bl = t - al * nbl;
        const int s1 = sa[al], s2 = sb[bl];
        double xu = 0, xv = 0, yu = 0, yv = 0;
        for (int i = 0; i <= g.p; ++i)
            for (int j = 0; j <= g.p; ++j) {
                const int64_t idx = (int64_t)(s1 - g.p + i) * g.n + (s2 - g.p + j);
                const double X = __ldg(g.X + idx), Y = __ldg(g.Y + idx);
                xu += Da[al][i] * Nb[bl][j] * X;
                xv += Na[al][i] * Db[bl][j] * X;
                yu += Da[al][i] * Nb[bl][j] * Y;
                yv += Na[al][i] * Db[bl][j] * Y;
            }
        out[(int64_t)(a0 + al) * n2 + b0 + bl] = xu * yv - xv * yu;
    }
}

__global__ void k_coeff_points(tq_coeff g, const double* P, int64_t n, const double* w, double* out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        double v = detj(g, P[2 * t], P[2 * t + 1]);
        out[t] = w ? v * w[t] : v;
    }
}


// The c == 1 element-Gauss part (PARTS == 1) for p1 == p2 == P: the same
// window staging, terms and summation order as the generic kernel, with
// compile-time extents (constant divisions, unrolled predicated element
// loops) -- the generic version is integer/branch bound.  Rows of other
// modes get a zero block.
template <int P>
__global__ void __launch_bounds__(256) k_raw_gauss_sep(tq_rawctx c, int r0, int r1) {
    constexpr int Q = P + 1, W = 2 * P + 1, T = W * W, WPB = 8;
    __shared__ double sE1[WPB][Q * Q], sE2[WPB][Q * Q], sIn[WPB][Q * W];
    __shared__ int sF1[WPB][Q], sF2[WPB][Q], sMK[WPB][Q * Q];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* E1 = sE1[wib];
    double* E2 = sE2[wib];
    double* inner = sIn[wib];
    int* F1 = sF1[wib];
    int* F2 = sF2[wib];
    int* MK = sMK[wib];
    for (int r = r0 + blockIdx.x * WPB + wib; r < r1; r += gridDim.x * WPB) {
        const RowDesc d = reinterpret_cast<const RowDesc*>(c.desc)[r];
        const int i1 = d.fidx / c.n2, i2 = d.fidx - i1 * c.n2;
        const RawRow dst = raw_row(c, r);
        if (d.mode != TQ_ROW_GAUSS && d.mode != TQ_ROW_BOX) {
            for (int q = lane; q < T; q += 32) dst[q] = 0.0;
            continue;
        }
        const int ef1 = c.el_first1[i1], ne1 = c.el_last1[i1] - ef1 + 1;
        const int ef2 = c.el_first2[i2], ne2 = c.el_last2[i2] - ef2 + 1;
        const bool box = d.mode == TQ_ROW_BOX && d.a1 >= 0;
        for (int l = lane; l < Q * Q; l += 32) {
            const int k = l / Q, b = l - k * Q;
            if (k < ne1) {
                const int e1 = ef1 + k, f1 = c.espan1[e1] - P;
                if (b == 0) F1[k] = f1;
                E1[l] = c.em1[((int64_t)e1 * Q + (i1 - f1)) * Q + b];
            }
            if (k < ne2) {
                const int e2 = ef2 + k, f2 = c.espan2[e2] - P;
                if (b == 0) F2[k] = f2;
                E2[l] = c.em2[((int64_t)e2 * Q + (i2 - f2)) * Q + b];
            }
            // interior flag of element (ef1 + k, ef2 + b), outside the box
            bool ok = false;
            if (k < ne1 && b < ne2) {
                const int e1 = ef1 + k, e2 = ef2 + b;
                ok = c.elem_class[(int64_t)e1 * c.nel2 + e2] == TQ_INTERIOR;
                if (box && e1 >= d.a1 && e1 <= d.b1 && e2 >= d.a2 && e2 <= d.b2) ok = false;
            }
            MK[l] = ok ? 1 : 0;
        }
        __syncwarp();
        for (int t = lane; t < Q * W; t += 32) {
            const int k1 = t / W, o2 = t - k1 * W;
            const int j2 = i2 - P + o2;
            double acc = 0.0;
            if (k1 < ne1 && j2 >= 0 && j2 < c.n2) {
#pragma unroll
                for (int k2 = 0; k2 < Q; ++k2) {
                    if (k2 >= ne2 || !MK[k1 * Q + k2]) continue;
                    const int b2 = j2 - F2[k2];
                    if (b2 < 0 || b2 > P) continue;
                    acc += E2[k2 * Q + b2];
                }
            }
            inner[t] = acc;
        }
        __syncwarp();
        for (int q = lane; q < T; q += 32) {
            const int o1 = q / W, o2 = q - o1 * W;
            const int j1 = i1 - P + o1;
            double acc = 0.0;
            if (j1 >= 0 && j1 < c.n1) {
#pragma unroll
                for (int k1 = 0; k1 < Q; ++k1) {
                    if (k1 >= ne1) continue;
                    const int b1 = j1 - F1[k1];
                    if (b1 < 0 || b1 > P) continue;
                    acc += E1[k1 * Q + b1] * inner[k1 * W + o2];
                }
            }
            dst[q] = 0.0 + acc;          // the generic kernel's zeroed block plus the sum
        }
        __syncwarp();
    }
}

}  // namespace tq

using namespace tq;

static size_t regular_smem_per_warp(const tq_rawctx& c) {
    const int W1 = 2 * c.p1 + 1, W2 = 2 * c.p2 + 1;
    const int ni = std::max(c.nmax1, c.p1 + 1);
    return sizeof(double) * ((size_t)W1 * W2 + (size_t)c.nmax1 * W1 + (size_t)c.nmax2 * W2 + (size_t)W2 * ni + W1 + W2 +
                             regular_window_slots(c.p1, c.p2) + (c.grids ? (size_t)c.nmax1 * c.nmax2 : 0));
}

template <int PARTS>
static int raw_regular_launch(const tq_rawctx& c, int32_t r0, int32_t r1, void* stream) {
    if (r1 <= r0) return TQ_OK;
    int wpb = 4;
    size_t shm = regular_smem_per_warp(c) * wpb;
    while (shm > 200 * 1024 && wpb > 1) { wpb /= 2; shm = regular_smem_per_warp(c) * wpb; }
    if (shm > 200 * 1024) { set_error("raw-row workspace too large"); return TQ_EINVAL; }
    TQ_CUDA(cudaFuncSetAttribute(k_raw_regular<PARTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    int grid = (int)std::min<int64_t>((r1 - r0 + wpb - 1) / wpb, (int64_t)kSms * 32);
    k_raw_regular<PARTS><<<grid, 32 * wpb, shm, S(stream)>>>(c, r0, r1); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_raw_regular");
    return TQ_OK;
}

constexpr int kCoefRowThreads = 128;     // threads per row of the c != 1 raw-row kernels

template <int P>
static int raw_gauss_coef_launch_p(const tq_rawctx& c, int32_t r0, int32_t r1, void* stream) {
    const size_t shm = sizeof(double) * gauss_coef_slots(c.p1, c.p2, c.ng1, c.ng2);
    if (shm > 200 * 1024) { set_error("raw-row workspace too large"); return TQ_EINVAL; }
    TQ_CUDA(cudaFuncSetAttribute(k_raw_gauss_coef<kCoefRowThreads, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)shm));
    const int grid = (int)std::min<int64_t>(r1 - r0, (int64_t)kSms * 32);
    k_raw_gauss_coef<kCoefRowThreads, P><<<grid, kCoefRowThreads, shm, S(stream)>>>(c, r0, r1); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_raw_gauss_coef");
    return TQ_OK;
}

static int raw_gauss_coef_launch(const tq_rawctx& c, int32_t r0, int32_t r1, void* stream) {
    if (r1 <= r0) return TQ_OK;
    if (c.p1 == c.p2 && c.ng1 == c.p1 + 1 && c.ng2 == c.p2 + 1) {
        switch (c.p1) {
#define TQ_GCP(Q) case Q: return raw_gauss_coef_launch_p<Q>(c, r0, r1, stream);
            TQ_GCP(1) TQ_GCP(2) TQ_GCP(3) TQ_GCP(4) TQ_GCP(5) TQ_GCP(6) TQ_GCP(7) TQ_GCP(8)
#undef TQ_GCP
            default: break;
        }
    }
    return raw_gauss_coef_launch_p<0>(c, r0, r1, stream);
}

template <int NT, int P>
static int raw_sf_coef_launch_p(const tq_rawctx& c, int32_t r0, int32_t r1, void* stream) {
    const size_t shm = sizeof(double) * sf_coef_slots(c);
    if (shm > 200 * 1024) { set_error("raw-row workspace too large"); return TQ_EINVAL; }
    TQ_CUDA(cudaFuncSetAttribute(k_raw_sf_coef<NT, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    const int grid = (int)std::min<int64_t>(r1 - r0, (int64_t)kSms * 32);
    k_raw_sf_coef<NT, P><<<grid, NT, shm, S(stream)>>>(c, r0, r1); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_raw_sf_coef");
    return TQ_OK;
}

template <int NT>
static int raw_sf_coef_launch_nt(const tq_rawctx& c, int32_t r0, int32_t r1, void* stream) {
    if (c.p1 == c.p2) {
        switch (c.p1) {
#define TQ_SFP(Q) case Q: return raw_sf_coef_launch_p<NT, Q>(c, r0, r1, stream);
            TQ_SFP(1) TQ_SFP(2) TQ_SFP(3) TQ_SFP(4) TQ_SFP(5) TQ_SFP(6) TQ_SFP(7) TQ_SFP(8)
#undef TQ_SFP
            default: break;
        }
    }
    return raw_sf_coef_launch_p<NT, 0>(c, r0, r1, stream);
}

static int raw_sf_coef_launch(const tq_rawctx& c, int32_t r0, int32_t r1, void* stream) {
    if (r1 <= r0) return TQ_OK;
    static const int nt = getenv("TQ_SF_ROW_THREADS") ? atoi(getenv("TQ_SF_ROW_THREADS")) : kCoefRowThreads;
    if (nt == 64) return raw_sf_coef_launch_nt<64>(c, r0, r1, stream);
    if (nt == 256) return raw_sf_coef_launch_nt<256>(c, r0, r1, stream);
    return raw_sf_coef_launch_nt<kCoefRowThreads>(c, r0, r1, stream);
}

extern "C" int tq_raw_regular(tq_rawctx c, int32_t r0, int32_t r1, void* stream) {
    if (c.cg) {     // c != 1: the sum-factorized element-Gauss kernel, then the WQ part onto it
        int rc = raw_gauss_coef_launch(c, r0, r1, stream);
        if (rc) return rc;
        return c.grids ? raw_sf_coef_launch(c, r0, r1, stream) : raw_regular_launch<2>(c, r0, r1, stream);
    }
    return raw_regular_launch<3>(c, r0, r1, stream);
}

extern "C" int tq_raw_gauss(tq_rawctx c, int32_t r0, int32_t r1, void* stream) {
    static const bool generic = getenv("TQ_RAW_GAUSS_GENERIC") != nullptr;   // A/B and the parity test
    if (r1 > r0 && !generic && !c.cg && c.p1 == c.p2 && c.p1 >= 1 && c.p1 <= 8) {
        const int grid = (int)std::min<int64_t>((r1 - r0 + 7) / 8, (int64_t)kSms * 16);
        switch (c.p1) {
#define CASE(Q) case Q: k_raw_gauss_sep<Q><<<grid, 256, 0, S(stream)>>>(c, r0, r1); break;
            CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
        }
        ::tq::note_launch();
        TQ_LAUNCH_CHECK("k_raw_gauss_sep");
        return TQ_OK;
    }
    if (c.cg) return raw_gauss_coef_launch(c, r0, r1, stream);
    return raw_regular_launch<1>(c, r0, r1, stream);
}

extern "C" int tq_raw_sumfactor(tq_rawctx c, int32_t r0, int32_t r1, void* stream) {
    if (c.grids) return raw_sf_coef_launch(c, r0, r1, stream);
    return raw_regular_launch<2>(c, r0, r1, stream);
}

extern "C" int tq_elem_mass(const double* ev, const double* ew, int32_t nel, int32_t ng, int32_t p, double* em,
                            void* stream) {
    if ((int64_t)nel * (p + 1) * (p + 1) == 0) return TQ_OK;
    k_elem_mass<<<grid_for((int64_t)nel * (p + 1) * (p + 1), 128), 128, 0, S(stream)>>>(ev, ew, nel, ng, p, em); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_elem_mass");
    return TQ_OK;
}

// q2 from which the cut-element blocks use a block per group (env
// TQ_CUT_BLOCKS_WIDE_FROM overrides: the A/B knob and the parity test)
static const int kCutBlocksWideFrom = getenv("TQ_CUT_BLOCKS_WIDE_FROM") ? atoi(getenv("TQ_CUT_BLOCKS_WIDE_FROM")) : 7;

extern "C" int tq_cut_blocks(tq_rawctx c, void* stream) {
    if (c.ngroups <= 0) return TQ_OK;
    if (c.p1 < 1 || c.p1 > kMaxP || c.p2 < 1 || c.p2 > kMaxP) { set_error("degree out of range"); return TQ_EINVAL; }
    if (c.p2 + 1 >= kCutBlocksWideFrom) {       // large degrees: a block per group
        const size_t shm = sizeof(double) * kCbChunk * (c.p1 + c.p2 + 3);
        const int grid = (int)std::min<int64_t>(c.ngroups, (int64_t)kSms * 64);
        switch (c.p2 + 1) {
#define TQ_CBW(Q2) case Q2: k_cut_blocks_wide<Q2><<<grid, kCbThreads, shm, S(stream)>>>(c); break;
            TQ_CBW(5) TQ_CBW(6) TQ_CBW(7) TQ_CBW(8) TQ_CBW(9) TQ_CBW(10) TQ_CBW(11)
#undef TQ_CBW
            default: set_error("degree out of range"); return TQ_EINVAL;
        }
        ::tq::note_launch();
        TQ_LAUNCH_CHECK("k_cut_blocks_wide");
        return TQ_OK;
    }
    constexpr int wpb = 4;
    const size_t shm = sizeof(double) * wpb * 32 * (c.p1 + c.p2 + 3);
    const int grid = (int)std::min<int64_t>((c.ngroups + wpb - 1) / wpb, (int64_t)kSms * 64);
    switch (c.p2 + 1) {
#define TQ_CB(Q2) case Q2: k_cut_blocks<Q2><<<grid, 32 * wpb, shm, S(stream)>>>(c); break;
        TQ_CB(2) TQ_CB(3) TQ_CB(4) TQ_CB(5) TQ_CB(6) TQ_CB(7) TQ_CB(8) TQ_CB(9) TQ_CB(10) TQ_CB(11)
#undef TQ_CB
    }
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_cut_blocks");
    return TQ_OK;
}

extern "C" int tq_raw_cutcells(tq_rawctx c, int32_t r0, int32_t r1, void* stream);

// per-row group lists of rows [r0, r1) (geometry): counts (r1 - r0 ints),
// then, with off = their exclusive prefix (r1 - r0 ints), the triplets
// (3 * total ints: group, key1, key2)
extern "C" int tq_row_groups(tq_rawctx c, int32_t r0, int32_t r1, const int32_t* off, int32_t* out, void* stream) {
    if (r1 <= r0) return TQ_OK;
    if (!c.cut_ptr || c.ngroups <= 0) { set_error("tq_row_groups needs the cut-element tables"); return TQ_EINVAL; }
    const int grid = (int)std::min<int64_t>((r1 - r0 + 7) / 8, (int64_t)kSms * 16);
    if (off) k_row_groups<false><<<grid, 256, 0, S(stream)>>>(c, r0, r1, off, out);
    else k_row_groups<true><<<grid, 256, 0, S(stream)>>>(c, r0, r1, nullptr, out);
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_row_groups");
    return TQ_OK;
}

// tq_raw_cutcells with the rows' group lists of tq_row_groups (rg_ptr:
// r1 - r0 + 1 offsets, rg: triplets)
extern "C" int tq_raw_cutcells_list(tq_rawctx c, int32_t r0, int32_t r1, const int32_t* rg_ptr, const int32_t* rg,
                                    void* stream) {
    if (r1 <= r0 || !c.cut_ptr || c.ngroups <= 0) return TQ_OK;
    if ((c.p1 + 1) * (c.p2 + 1) > 32) return tq_raw_cutcells(c, r0, r1, stream);     // a lane per slice entry
    const int grid = (int)std::min<int64_t>((r1 - r0 + 7) / 8, (int64_t)kSms * 16);
    const size_t shm = sizeof(double) * 8 * (2 * c.p1 + 1) * (2 * c.p2 + 1);
    k_raw_cutcells_list<<<grid, 256, shm, S(stream)>>>(c, r0, r1, rg_ptr, rg);
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_raw_cutcells_list");
    return TQ_OK;
}

extern "C" int tq_raw_cutcells(tq_rawctx c, int32_t r0, int32_t r1, void* stream) {
    if (r1 <= r0 || !c.cut_ptr || c.ngroups <= 0) return TQ_OK;
    int grid = (int)std::min<int64_t>((r1 - r0 + 7) / 8, (int64_t)kSms * 16);
    const size_t shm = c.raw_ld ? sizeof(double) * 8 * (2 * c.p1 + 1) * (2 * c.p2 + 1) : 0;
    k_raw_cutcells<<<grid, 256, shm, S(stream)>>>(c, r0, r1); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_raw_cutcells");
    return TQ_OK;
}

extern "C" int tq_coeff_grid(tq_coeff g, const double* x1, int32_t n1, const double* x2, int32_t n2, double* out,
                             void* stream) {
    if ((int64_t)n1 * n2 == 0) return TQ_OK;
    if (g.kind != TQ_COEFF_GEOMETRY || g.p > kMaxP) { set_error("unsupported coefficient field"); return TQ_EINVAL; }
    static const bool pointwise = getenv("TQ_COEFF_POINTWISE") != nullptr;    // A/B and the parity test
    if (pointwise) {
        k_coeff_grid<<<grid_for((int64_t)n1 * n2, 128), 128, 0, S(stream)>>>(g, x1, n1, x2, n2, out);
    } else {
        const dim3 grid((n2 + kCgB - 1) / kCgB, (n1 + kCgA - 1) / kCgA);
        k_coeff_grid_tiled<<<grid, 256, 0, S(stream)>>>(g, x1, n1, x2, n2, out);
    }
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_coeff_grid");
    return TQ_OK;
}

extern "C" int tq_coeff_points(tq_coeff g, const double* pts, int64_t n, const double* w, double* out,
                               void* stream) {
    if (n == 0) return TQ_OK;
    if (g.kind != TQ_COEFF_GEOMETRY || g.p > kMaxP) { set_error("unsupported coefficient field"); return TQ_EINVAL; }
    k_coeff_points<<<grid_for(n, 128), 128, 0, S(stream)>>>(g, pts, n, w, out); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_coeff_points");
    return TQ_OK;
}
