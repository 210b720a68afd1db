// Cut rows of the c != 1 all-raw path, element-centric.  A cut row's
// non-WQ part is a sum of element blocks: the element-Gauss blocks of the
// interior elements of its support outside its box (_Run.element_block,
// src/assembly.py:310-332) and the span-key group blocks of the nearby cut
// elements (_Run.add_cut_blocks, src/assembly.py:369-398).  Each block
//   E[(a1,a2)][(b1,b2)] = sum_pts cw v1[a1] v1[b1] v2[a2] v2[b2]
// is symmetric in (a1,b1) and in (a2,b2) separately, so it is formed once
// per element in "pair" form E[s(a1,b1)][s(a2,b2)] (q(q+1)/2 pairs per
// direction, 2025 values at p = 8 instead of 6561) by small GEMM-shaped
// contractions:
//   tq_gauss_pairs: tensor Gauss grids, sum-factorised over the points
//                   (T[g1][s2] = sum_g2 c w v2 v2, E = sum_g1 v1 v1 T);
//   tq_cut_pairs:   scattered cut-cell points, E = P1^T P2 with
//                   P1[k][s1] = cw v1 v1, P2[k][s2] = v2 v2 (register tiles);
// and tq_cut_rows_gather sums, per cut row, the row slices of the blocks it
// reads into a shared row block and writes the row's planes once (the WQ
// sum-factorization part of BOX / MASK rows is added afterwards).
#include "common.cuh"

namespace tq {

struct RowDescC {
    int fidx, mode, set1, set2, a1, b1, a2, b2;
};

template <int Q>
struct Pairs {
    static constexpr int NP = Q * (Q + 1) / 2;
    // pair index of (a, b), a <= b
    __host__ __device__ static constexpr int of(int a, int b) { return a * Q - (a * (a - 1)) / 2 + (b - a); }
};

// (a, b) of every pair, in shared memory
template <int Q>
__device__ __forceinline__ void pair_tables(int* pa, int* pb) {
    for (int a = threadIdx.x; a < Q; a += blockDim.x)
        for (int b = a; b < Q; ++b) {
            pa[Pairs<Q>::of(a, b)] = a;
            pb[Pairs<Q>::of(a, b)] = b;
        }
}

// ---------------------------------------------------------------------------
// Element-Gauss blocks of the listed interior elements (q = ng = p + 1).
// cgp: c at the elements' Gauss grids, [slot][g1][g2].
// ---------------------------------------------------------------------------
template <int Q>
__global__ void __launch_bounds__(128) k_gauss_pairs(tq_rawctx c, const int32_t* __restrict__ gel, int nslot,
                                                     const double* __restrict__ cgp, double* __restrict__ E) {
    constexpr int NP = Pairs<Q>::NP;
    __shared__ double V1[Q][Q], V2[Q][Q], Wc[Q][Q + 1], PV1[Q][NP], PV2[Q][NP], T[Q][NP];
    __shared__ int pa[NP], pb[NP];
    pair_tables<Q>(pa, pb);
    for (int slot = blockIdx.x; slot < nslot; slot += gridDim.x) {
        const int e1 = gel[2 * slot], e2 = gel[2 * slot + 1];
        __syncthreads();
        for (int t = threadIdx.x; t < Q * Q; t += blockDim.x) {
            const int g = t / Q, a = t - g * Q;
            V1[g][a] = c.ev1[((int64_t)e1 * Q + g) * Q + a];
            V2[g][a] = c.ev2[((int64_t)e2 * Q + g) * Q + a];
            // the weights of gauss_entry: c (w1 w2)
            Wc[g][a] = cgp[((int64_t)slot * Q + g) * Q + a] * (c.ew1[(int64_t)e1 * Q + g] * c.ew2[(int64_t)e2 * Q + a]);
        }
        __syncthreads();
        for (int t = threadIdx.x; t < Q * NP; t += blockDim.x) {
            const int g = t / NP, s = t - g * NP;
            PV1[g][s] = V1[g][pa[s]] * V1[g][pb[s]];
            PV2[g][s] = V2[g][pa[s]] * V2[g][pb[s]];
        }
        __syncthreads();
        for (int t = threadIdx.x; t < Q * NP; t += blockDim.x) {
            const int g1 = t / NP, s2 = t - g1 * NP;
            double acc = 0.0;
#pragma unroll
            for (int g2 = 0; g2 < Q; ++g2) acc += PV2[g2][s2] * Wc[g1][g2];
            T[g1][s2] = acc;
        }
        __syncthreads();
        double* out = E + (int64_t)slot * NP * NP;
        for (int t = threadIdx.x; t < NP * NP; t += blockDim.x) {
            const int s1 = t / NP, s2 = t - s1 * NP;
            double acc = 0.0;
#pragma unroll
            for (int g1 = 0; g1 < Q; ++g1) acc += PV1[g1][s1] * T[g1][s2];
            out[t] = acc;
        }
    }
}

// ---------------------------------------------------------------------------
// Span-key group blocks of the cut elements: one block of 128 threads per
// group; points staged KC at a time (v1, v2, cw through the group
// permutation), their pair products P1 / P2 formed in shared memory, then a
// thread accumulates a TA x TB tile of E = P1^T P2.
// ---------------------------------------------------------------------------
constexpr int kCpThreads = 128, kCpChunk = 32;

template <int Q>
__global__ void __launch_bounds__(kCpThreads) k_cut_pairs(tq_rawctx c, double* __restrict__ E) {
    constexpr int NP = Pairs<Q>::NP, TA = (NP + 7) / 8, TB = (NP + 15) / 16, NA = 8 * TA, NB = 16 * TB;
    constexpr int ST = 2 * Q + 1;
    __shared__ double S[kCpChunk][ST];
    __shared__ double P1[kCpChunk][NA], P2[kCpChunk][NB];
    __shared__ int pa[NP], pb[NP];
    pair_tables<Q>(pa, pb);
    const int tid = threadIdx.x, ta = tid / 16, tb = tid - (tid / 16) * 16;
    for (int g = blockIdx.x; g < c.ngroups; g += gridDim.x) {
        const int64_t p0 = c.grp_pts[g], pe = c.grp_pts[g + 1];
        double acc[TA][TB];
#pragma unroll
        for (int i = 0; i < TA; ++i)
#pragma unroll
            for (int j = 0; j < TB; ++j) acc[i][j] = 0.0;
        for (int64_t base = p0; base < pe; base += kCpChunk) {
            const int np = (int)(pe - base < kCpChunk ? pe - base : kCpChunk);
            __syncthreads();
            for (int k = tid; k < np; k += kCpThreads) {
                const int64_t pt = c.grp_perm[base + k];
#pragma unroll
                for (int o = 0; o < Q; ++o) {
                    S[k][o] = c.cvals1[pt * Q + o];
                    S[k][Q + o] = c.cvals2[pt * Q + o];
                }
                S[k][2 * Q] = c.cut_cw[pt];
            }
            __syncthreads();
            for (int t = tid; t < kCpChunk * NA; t += kCpThreads) {
                const int k = t / NA, s = t - k * NA;
                P1[k][s] = (k < np && s < NP) ? (S[k][2 * Q] * S[k][pa[s]]) * S[k][pb[s]] : 0.0;
            }
            for (int t = tid; t < kCpChunk * NB; t += kCpThreads) {
                const int k = t / NB, s = t - k * NB;
                P2[k][s] = (k < np && s < NP) ? S[k][Q + pa[s]] * S[k][Q + pb[s]] : 0.0;
            }
            __syncthreads();
            for (int k = 0; k < np; ++k) {
                double x[TA], y[TB];
#pragma unroll
                for (int i = 0; i < TA; ++i) x[i] = P1[k][ta * TA + i];
#pragma unroll
                for (int j = 0; j < TB; ++j) y[j] = P2[k][tb * TB + j];
#pragma unroll
                for (int i = 0; i < TA; ++i)
#pragma unroll
                    for (int j = 0; j < TB; ++j) acc[i][j] = fma(x[i], y[j], acc[i][j]);
            }
        }
        double* out = E + (int64_t)g * NP * NP;
#pragma unroll
        for (int i = 0; i < TA; ++i)
#pragma unroll
            for (int j = 0; j < TB; ++j) {
                const int s1 = ta * TA + i, s2 = tb * TB + j;
                if (s1 < NP && s2 < NP) out[s1 * NP + s2] = acc[i][j];
            }
    }
}

// ---------------------------------------------------------------------------
// Per cut row (descriptor rows [r0, r1), warp per row): the Gauss part (GAUSS
// and BOX rows: interior support elements outside the box) and the cut-cell
// part (span-key groups of the cut elements within one element of the
// support), summed in a warp-private shared row block in a fixed order,
// then written to the row's planes.  gslot: element -> Gauss block slot.
// ---------------------------------------------------------------------------
template <int P>
__global__ void __launch_bounds__(256) k_cut_rows_gather(tq_rawctx c, int r0, int r1, const int32_t* __restrict__ gslot,
                                                         const double* __restrict__ Eg, const double* __restrict__ Ec,
                                                         int* __restrict__ status) {
    constexpr int Q = P + 1, W = 2 * P + 1, T = W * W, NP = Pairs<Q>::NP, QQ = Q * Q;
    constexpr int WPB = 8;
    __shared__ double acc_s[WPB][T];
    __shared__ int pidx[Q][Q];
    for (int t = threadIdx.x; t < QQ; t += blockDim.x) {
        const int a = t / Q, b = t - (t / Q) * Q;
        pidx[a][b] = a <= b ? Pairs<Q>::of(a, b) : Pairs<Q>::of(b, a);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* acc = acc_s[wib];
    for (int r = r0 + blockIdx.x * WPB + wib; r < r1; r += gridDim.x * WPB) {
        const RowDescC d = reinterpret_cast<const RowDescC*>(c.desc)[r];
        const int i1 = d.fidx / c.n2, i2 = d.fidx - (d.fidx / c.n2) * c.n2;
        for (int q = lane; q < T; q += 32) acc[q] = 0.0;
        __syncwarp();
        if (d.mode == TQ_ROW_GAUSS || d.mode == TQ_ROW_BOX) {
            const bool box = d.mode == TQ_ROW_BOX && d.a1 >= 0;
            for (int e1 = c.el_first1[i1]; e1 <= c.el_last1[i1]; ++e1) {
                const int f1 = c.espan1[e1] - P, a1 = i1 - f1;
                for (int e2 = c.el_first2[i2]; e2 <= c.el_last2[i2]; ++e2) {
                    const int64_t e = (int64_t)e1 * c.nel2 + e2;
                    if (c.elem_class[e] != TQ_INTERIOR) continue;
                    if (box && e1 >= d.a1 && e1 <= d.b1 && e2 >= d.a2 && e2 <= d.b2) continue;
                    const int slot = gslot[e];
                    if (slot < 0) {       // the element list missed an element: flagged, never silent
                        if (lane == 0) atomicOr(status, 4);
                        continue;
                    }
                    const int f2 = c.espan2[e2] - P, a2 = i2 - f2;
                    const double* Es = Eg + (int64_t)slot * NP * NP;
                    for (int B = lane; B < QQ; B += 32) {
                        const int b1 = B / Q, b2 = B - (B / Q) * Q;
                        acc[(f1 + b1 - i1 + P) * W + (f2 + b2 - i2 + P)] +=
                            __ldg(Es + pidx[a1][b1] * NP + pidx[a2][b2]);
                    }
                    __syncwarp();
                }
            }
        }
        if (Ec && c.cut_ptr) {
            const int ea1 = max(c.el_first1[i1] - 1, 0), eb1 = min(c.el_last1[i1] + 1, c.nel1 - 1);
            const int ea2 = max(c.el_first2[i2] - 1, 0), eb2 = min(c.el_last2[i2] + 1, c.nel2 - 1);
            const int w2 = eb2 - ea2 + 1, nh = (eb1 - ea1 + 1) * w2;
            for (int h0 = 0; h0 < nh; h0 += 32) {
                const int h = h0 + lane;
                int id = -1;
                if (h < nh) id = c.cutidx[(int64_t)(ea1 + h / w2) * c.nel2 + (ea2 + h % w2)];
                unsigned m = __ballot_sync(0xffffffffu, id >= 0);
                while (m) {
                    const int src = __ffs(m) - 1;
                    m &= m - 1;
                    const int cid = __shfl_sync(0xffffffffu, id, src);
                    for (int g = c.grp_ptr[cid]; g < c.grp_ptr[cid + 1]; ++g) {
                        const int f1 = c.grp_key[2 * g], f2 = c.grp_key[2 * g + 1];
                        const int a1 = i1 - f1, a2 = i2 - f2;
                        if (a1 < 0 || a1 > P || a2 < 0 || a2 > P) continue;
                        const double* Es = Ec + (int64_t)g * NP * NP;
                        for (int B = lane; B < QQ; B += 32) {
                            const int b1 = B / Q, b2 = B - (B / Q) * Q;
                            acc[(f1 + b1 - i1 + P) * W + (f2 + b2 - i2 + P)] +=
                                __ldg(Es + pidx[a1][b1] * NP + pidx[a2][b2]);
                        }
                        __syncwarp();
                    }
                }
            }
        }
        __syncwarp();
        double* dst = c.raw + c.store[r];
        for (int q = lane; q < T; q += 32) dst[(int64_t)q * c.raw_ld] = acc[q];
        __syncwarp();
    }
}

}  // namespace tq

using namespace tq;

extern "C" int64_t tq_pair_block_doubles(int32_t p) {
    const int64_t np = (int64_t)(p + 1) * (p + 2) / 2;
    return np * np;
}

// Element-Gauss blocks in pair form of the listed elements (gel: nslot x 2
// element indices; cgp: c at their (p+1)^2 Gauss points, [slot][g1][g2];
// E: nslot x tq_pair_block_doubles(p)).  Needs p1 == p2 and ng = p + 1.
extern "C" int tq_gauss_pairs(tq_rawctx c, const int32_t* gel, int32_t nslot, const double* cgp, double* E,
                              void* stream) {
    if (nslot <= 0) return TQ_OK;
    if (c.p1 != c.p2 || c.ng1 != c.p1 + 1 || c.ng2 != c.p2 + 1) { set_error("tq_gauss_pairs needs p1 == p2 and p + 1 Gauss points"); return TQ_EINVAL; }
    const int grid = std::min(nslot, kSms * 16);
    switch (c.p1 + 1) {
#define CASE(Q) case Q: k_gauss_pairs<Q><<<grid, 128, 0, S(stream)>>>(c, gel, nslot, cgp, E); break;
        CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11)
#undef CASE
        default: set_error("degree out of range"); return TQ_EINVAL;
    }
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_gauss_pairs");
    return TQ_OK;
}

// Span-key group blocks in pair form (E: ngroups x tq_pair_block_doubles(p)).
extern "C" int tq_cut_pairs(tq_rawctx c, double* E, void* stream) {
    if (c.ngroups <= 0) return TQ_OK;
    if (c.p1 != c.p2) { set_error("tq_cut_pairs needs p1 == p2"); return TQ_EINVAL; }
    const int grid = std::min(c.ngroups, kSms * 16);
    switch (c.p1 + 1) {
#define CASE(Q) case Q: k_cut_pairs<Q><<<grid, kCpThreads, 0, S(stream)>>>(c, E); break;
        CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11)
#undef CASE
        default: set_error("degree out of range"); return TQ_EINVAL;
    }
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_cut_pairs");
    return TQ_OK;
}

// Rows [r0, r1) (the cut rows, planes layout): Gauss + cut-cell parts from
// the pair blocks (Eg / gslot: tq_gauss_pairs, Ec: tq_cut_pairs or NULL),
// written to the planes.  status |= 4 when a needed Gauss block is missing.
extern "C" int tq_cut_rows_gather(tq_rawctx c, int32_t r0, int32_t r1, const int32_t* gslot, const double* Eg,
                                  const double* Ec, int32_t* status, void* stream) {
    if (r1 <= r0) return TQ_OK;
    if (!c.raw_ld || !c.store || c.p1 != c.p2) { set_error("tq_cut_rows_gather needs the planes layout and p1 == p2"); return TQ_EINVAL; }
    const int grid = (int)std::min<int64_t>((r1 - r0 + 7) / 8, (int64_t)kSms * 8);
    switch (c.p1) {
#define CASE(Q) case Q: k_cut_rows_gather<Q><<<grid, 256, 0, S(stream)>>>(c, r0, r1, gslot, Eg, Ec, status); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
        default: set_error("degree out of range"); return TQ_EINVAL;
    }
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_cut_rows_gather");
    return TQ_OK;
}
