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
#include <limits.h>

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

// FP64 tensor-core product of two fragments: C (8 x 8) += A (8 x 4) B (4 x 8)
// with lane l holding A[l/4][l%4], B[l%4][l/4], C[l/4][2(l%4) .. +1]
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

#ifndef TQ_CP_DMMA
#define TQ_CP_DMMA 1
#endif

// pair-product operand stride: >= the padded width, = 4 (mod 16) doubles, so
// a fragment load (4 rows x 8 columns) hits distinct banks per half-warp
__host__ __device__ constexpr int cp_lda(int npad) { return npad + ((4 - npad % 16) + 16) % 16; }

// ---------------------------------------------------------------------------
// Element-Gauss blocks of the listed interior elements (q = ng = p + 1).
// c at the element's Gauss grid: det J of the geometry map computed here
// from per-line basis tables (geo.kind == TQ_COEFF_GEOMETRY; the element's
// points are X1[e1 q + g] x X2[e2 q + g]), else read from cgp[slot][g1][g2].
// E = PV1^T T is a (NP x q) (q x NP) product: a thread owns a 3 x 6 tile.
// ---------------------------------------------------------------------------
constexpr int kGpThreads = 128;
// element-Gauss and cut pair blocks: 8 resident blocks per SM (64
// registers; 128 / 80 with no bound): config 4 p = 8 step 0.522 -> 0.506 ms
// (the pair kernels overlap the fits and strips better)
#ifndef TQ_GP_MINB
#define TQ_GP_MINB 8
#endif
#ifndef TQ_CP_MINB
#define TQ_CP_MINB 8
#endif

// geometry-map line tables at points u: span, then N[0..p], D[0..p]
template <int PG>
__global__ void k_geo_lines(tq_coeff geo, const double* __restrict__ u, int n, int32_t* __restrict__ span,
                            double* __restrict__ nd) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const double x = u[t];
    const int sp = find_span(geo.knots, geo.n + PG + 1, PG, geo.n, x);
    double N[PG + 1], D[PG + 1];
    basis_funs_ders<PG>(geo.knots, sp, x, N, D);
    span[t] = sp;
#pragma unroll
    for (int k = 0; k <= PG; ++k) {
        nd[(int64_t)t * 2 * (PG + 1) + k] = N[k];
        nd[(int64_t)t * 2 * (PG + 1) + PG + 1 + k] = D[k];
    }
}

template <int Q>
__global__ void __launch_bounds__(kGpThreads, TQ_GP_MINB) k_gauss_pairs(tq_rawctx c, tq_coeff geo, const double* __restrict__ X1,
                                                            const double* __restrict__ X2,
                                                            const int32_t* __restrict__ gel, int nslot,
                                                            const double* __restrict__ cgp, double* __restrict__ E,
                                                            const int32_t* __restrict__ lsp1,
                                                            const double* __restrict__ lnd1,
                                                            const int32_t* __restrict__ lsp2,
                                                            const double* __restrict__ lnd2) {
    // E = PV1^T T on the FP64 tensor cores (mma.sync m8n8k4): NP x NP in
    // 8 x 8 tiles (2 x 2 warps, TR x TR tiles each), K = Q Gauss points
    // padded to a multiple of 4 with zero rows
    constexpr int NP = Pairs<Q>::NP, NT8 = (NP + 7) / 8, NPAD = 8 * NT8, LDA = cp_lda(NPAD), TR = (NT8 + 1) / 2;
    constexpr int KP = (Q + 3) & ~3;
    constexpr int NA = NPAD, NB = NPAD;
    constexpr int PG = kMaxP + 1;
    __shared__ double V1[Q][Q], V2[Q][Q], Wc[Q][Q + 1];
    __shared__ __align__(16) double PV1[KP][LDA], T[KP][LDA];
    __shared__ double Na[Q][PG], Da[Q][PG], Nb[Q][PG], Db[Q][PG];
    __shared__ double XB[PG][Q], XDB[PG][Q], YB[PG][Q], YDB[PG][Q];
    __shared__ int sa[Q], sb[Q], pa[NP], pb[NP];
    constexpr int KN = 128;                    // geometry knots kept in shared memory (when they fit)
    __shared__ double kn_s[KN], XW[PG][PG], YW[PG][PG];
    pair_tables<Q>(pa, pb);
    const int tid = threadIdx.x;
    for (int t = tid; t < (KP - Q) * LDA; t += blockDim.x) {      // the K padding rows stay zero
        PV1[Q + t / LDA][t % LDA] = 0.0;
        T[Q + t / LDA][t % LDA] = 0.0;
    }
    const bool inline_c = geo.kind == TQ_COEFF_GEOMETRY;
    const int nk = geo.n + geo.p + 1;
    const double* knots = geo.knots;
    if (inline_c && nk <= KN) {
        for (int t = tid; t < nk; t += blockDim.x) kn_s[t] = geo.knots[t];
        knots = kn_s;
    }
    __syncthreads();
    for (int slot = blockIdx.x; slot < nslot; slot += gridDim.x) {
        const int e1 = gel[2 * slot], e2 = gel[2 * slot + 1];
        __syncthreads();
        for (int t = tid; t < Q * Q; t += blockDim.x) {
            const int g = t / Q, a = t - g * Q;
            V1[g][a] = c.ev1[((int64_t)e1 * Q + g) * Q + a];
            V2[g][a] = c.ev2[((int64_t)e2 * Q + g) * Q + a];
        }
        if (inline_c && lsp1) {              // precomputed line tables (tq_geo_lines)
            const int pg1 = geo.p + 1;
            for (int t = tid; t < 2 * Q * pg1; t += blockDim.x) {
                const bool d1 = t < Q * pg1;
                const int u = d1 ? t : t - Q * pg1, g = u / pg1, k = u - (u / pg1) * pg1;
                const int64_t pt = (int64_t)(d1 ? e1 : e2) * Q + g;
                const double* nd = (d1 ? lnd1 : lnd2) + pt * 2 * pg1;
                (d1 ? Na : Nb)[g][k] = nd[k];
                (d1 ? Da : Db)[g][k] = nd[pg1 + k];
                if (k == 0) (d1 ? sa : sb)[g] = (d1 ? lsp1 : lsp2)[pt];
            }
        } else if (inline_c && tid < 2 * Q) {       // line tables of the geometry map
            const bool d1 = tid < Q;
            const int g = d1 ? tid : tid - Q;
            const double u = d1 ? X1[(int64_t)e1 * Q + g] : X2[(int64_t)e2 * Q + g];
            const int sp = find_span(knots, nk, geo.p, geo.n, u);
            double N[PG], D[PG];
            basis_funs_ders_rt(knots, geo.p, sp, u, N, D);
            for (int k = 0; k <= geo.p; ++k) {
                (d1 ? Na : Nb)[g][k] = N[k];
                (d1 ? Da : Db)[g][k] = D[k];
            }
            (d1 ? sa : sb)[g] = sp;
        }
        __syncthreads();
        // one geometry span per direction over the element (the usual case:
        // the analysis mesh refines the geometry's): the control net is
        // contracted along direction 2 first, as in k_coeff_grid_tiled
        bool tensor = false;
        if (inline_c) {
            tensor = true;
            for (int g = 1; g < Q; ++g) tensor = tensor && sa[g] == sa[0] && sb[g] == sb[0];
        }
        if (tensor) {
            const int pg = geo.p;
            for (int t = tid; t < (pg + 1) * (pg + 1); t += blockDim.x) {      // the control window
                const int a = t / (pg + 1), b = t - (t / (pg + 1)) * (pg + 1);
                const int64_t idx = (int64_t)(sa[0] - pg + a) * geo.n + (sb[0] - pg + b);
                XW[a][b] = __ldg(geo.X + idx);
                YW[a][b] = __ldg(geo.Y + idx);
            }
            __syncthreads();
            for (int t = tid; t < (pg + 1) * Q; t += blockDim.x) {
                const int a = t / Q, g2 = t - (t / Q) * Q;
                double xb = 0, xdb = 0, yb = 0, ydb = 0;
                for (int b = 0; b <= pg; ++b) {
                    const double Xc = XW[a][b], Yc = YW[a][b];
                    xb += Nb[g2][b] * Xc;
                    xdb += Db[g2][b] * Xc;
                    yb += Nb[g2][b] * Yc;
                    ydb += Db[g2][b] * Yc;
                }
                XB[a][g2] = xb;
                XDB[a][g2] = xdb;
                YB[a][g2] = yb;
                YDB[a][g2] = ydb;
            }
            __syncthreads();
        }
        for (int t = tid; t < Q * Q; t += blockDim.x) {
            const int g1 = t / Q, g2 = t - g1 * Q;
            double cv;
            if (tensor) {
                double xu = 0, xv = 0, yu = 0, yv = 0;
                for (int a = 0; a <= geo.p; ++a) {
                    xu += Da[g1][a] * XB[a][g2];
                    xv += Na[g1][a] * XDB[a][g2];
                    yu += Da[g1][a] * YB[a][g2];
                    yv += Na[g1][a] * YDB[a][g2];
                }
                cv = xu * yv - xv * yu;
            } else if (inline_c) {      // detj (rawrows.cu): the same terms in the same order
                double xu = 0, xv = 0, yu = 0, yv = 0;
                for (int a = 0; a <= geo.p; ++a)
                    for (int b = 0; b <= geo.p; ++b) {
                        const int64_t idx = (int64_t)(sa[g1] - geo.p + a) * geo.n + (sb[g2] - geo.p + b);
                        const double Xc = __ldg(geo.X + idx), Yc = __ldg(geo.Y + idx);
                        xu += Da[g1][a] * Nb[g2][b] * Xc;
                        xv += Na[g1][a] * Db[g2][b] * Xc;
                        yu += Da[g1][a] * Nb[g2][b] * Yc;
                        yv += Na[g1][a] * Db[g2][b] * Yc;
                    }
                cv = xu * yv - xv * yu;
            } else {
                cv = cgp[((int64_t)slot * Q + g1) * Q + g2];
            }
            // the weights of gauss_entry: c (w1 w2)
            Wc[g1][g2] = cv * (c.ew1[(int64_t)e1 * Q + g1] * c.ew2[(int64_t)e2 * Q + g2]);
        }
        __syncthreads();
        for (int t = tid; t < Q * NA; t += blockDim.x) {
            const int g = t / NA, s = t - g * NA;
            PV1[g][s] = s < NP ? V1[g][pa[s]] * V1[g][pb[s]] : 0.0;
        }
        for (int t = tid; t < Q * NB; t += blockDim.x) {
            const int g1 = t / NB, s2 = t - g1 * NB;
            double acc = 0.0;
            if (s2 < NP) {
                const int a2 = pa[s2], b2 = pb[s2];
#pragma unroll
                for (int g2 = 0; g2 < Q; ++g2) acc += (V2[g2][a2] * V2[g2][b2]) * Wc[g1][g2];
            }
            T[g1][s2] = acc;
        }
        __syncthreads();
        {
            const int lane = tid & 31, warp = tid >> 5, wr = warp >> 1, wc = warp & 1, fr = lane >> 2, fk = lane & 3;
            double acc[TR][TR][2];
#pragma unroll
            for (int i = 0; i < TR; ++i)
#pragma unroll
                for (int j = 0; j < TR; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
            for (int k0 = 0; k0 < KP; k0 += 4) {
                double af[TR], bf[TR];
#pragma unroll
                for (int i = 0; i < TR; ++i) {
                    const int tr = wr * TR + i, tc = wc * TR + i;
                    af[i] = tr < NT8 ? PV1[k0 + fk][tr * 8 + fr] : 0.0;
                    bf[i] = tc < NT8 ? T[k0 + fk][tc * 8 + fr] : 0.0;
                }
#pragma unroll
                for (int i = 0; i < TR; ++i)
#pragma unroll
                    for (int j = 0; j < TR; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
            double* out = E + (int64_t)slot * NP * NP;
#pragma unroll
            for (int i = 0; i < TR; ++i)
#pragma unroll
                for (int j = 0; j < TR; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int s1 = (wr * TR + i) * 8 + fr, s2 = (wc * TR + j) * 8 + 2 * fk + h;
                        if (s1 < NP && s2 < NP) out[s1 * NP + s2] = acc[i][j][h];
                    }
        }
    }
}

// ---------------------------------------------------------------------------
// Span-key group blocks of the cut elements, by pieces of at most kCpPiece
// points (a group's pieces are summed in order by k_cut_pairs_reduce: the
// largest groups no longer set the kernel's length).  One block of 128
// threads per piece; points staged kCpChunk at a time (v1, v2, cw through the
// group permutation), their pair products P1 / P2 formed in shared memory,
// then a thread accumulates a TA x TB tile of P1^T P2.
// pieces: npieces x 2 int64 (group, first point); piece end = min(first +
// kCpPiece, the group's end).
// ---------------------------------------------------------------------------
constexpr int kCpThreads = 128, kCpChunk = 32, kCpPiece = 128;

template <int Q>
__global__ void __launch_bounds__(kCpThreads, TQ_CP_MINB) k_cut_pairs(tq_rawctx c, const int64_t* __restrict__ pieces,
                                                          int npieces, double* __restrict__ Epart,
                                                          const int32_t* __restrict__ gpiece, double* __restrict__ E) {
    constexpr int NP = Pairs<Q>::NP, ST = 2 * Q + 1;
    if constexpr (TQ_CP_DMMA && Q <= 10) {      // (Q = 11: the padded operands exceed the static stage)
    // E = P1^T P2 on the FP64 tensor cores (mma.sync m8n8k4): the NP x NP
    // block in 8 x 8 tiles, a 2 x 2 grid of warps each owning TR x TR tiles;
    // per 4 points a warp loads TR A and TR B fragments for TR^2 MMAs
    constexpr int NT8 = (NP + 7) / 8, NPAD = 8 * NT8, LDA = cp_lda(NPAD), TR = (NT8 + 1) / 2;
    __shared__ double S[kCpChunk][ST];
    __shared__ __align__(16) double P1[kCpChunk][LDA], P2[kCpChunk][LDA];
    __shared__ int pa[NP], pb[NP];
    pair_tables<Q>(pa, pb);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wr = warp >> 1, wc = warp & 1, fr = lane >> 2, fk = lane & 3;
    for (int pc = blockIdx.x; pc < npieces; pc += gridDim.x) {
        const int g = (int)pieces[2 * pc];
        const int64_t p0 = pieces[2 * pc + 1], pe = min(p0 + kCpPiece, (int64_t)c.grp_pts[g + 1]);
        double acc[TR][TR][2];
#pragma unroll
        for (int i = 0; i < TR; ++i)
#pragma unroll
            for (int j = 0; j < TR; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int64_t base = p0; base < pe; base += kCpChunk) {
            const int np = (int)(pe - base < kCpChunk ? pe - base : kCpChunk);
            __syncthreads();
            for (int t = tid; t < np * ST; t += kCpThreads) {
                const int k = t / ST, o = t - k * ST;
                const int64_t pt = c.grp_perm[base + k];
                S[k][o] = o < Q ? c.cvals1[pt * Q + o] : (o < 2 * Q ? c.cvals2[pt * Q + (o - Q)] : c.cut_cw[pt]);
            }
            __syncthreads();
            for (int t = tid; t < kCpChunk * NPAD; t += kCpThreads) {
                const int k = t / NPAD, s = t - k * NPAD;
                const bool ok = k < np && s < NP;
                P1[k][s] = ok ? (S[k][2 * Q] * S[k][pa[s]]) * S[k][pb[s]] : 0.0;
                P2[k][s] = ok ? S[k][Q + pa[s]] * S[k][Q + pb[s]] : 0.0;
            }
            __syncthreads();
            for (int k0 = 0; k0 < np; k0 += 4) {
                double af[TR], bf[TR];
#pragma unroll
                for (int i = 0; i < TR; ++i) {
                    const int tr = wr * TR + i, tc = wc * TR + i;
                    af[i] = tr < NT8 ? P1[k0 + fk][tr * 8 + fr] : 0.0;
                    bf[i] = tc < NT8 ? P2[k0 + fk][tc * 8 + fr] : 0.0;
                }
#pragma unroll
                for (int i = 0; i < TR; ++i)
#pragma unroll
                    for (int j = 0; j < TR; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
        }
        // a group of one piece writes its block directly (the reduce skips it)
        double* out = gpiece[g + 1] - gpiece[g] == 1 ? E + (int64_t)g * NP * NP : Epart + (int64_t)pc * NP * NP;
#pragma unroll
        for (int i = 0; i < TR; ++i)
#pragma unroll
            for (int j = 0; j < TR; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int s1 = (wr * TR + i) * 8 + fr, s2 = (wc * TR + j) * 8 + 2 * fk + h;
                    if (s1 < NP && s2 < NP) out[s1 * NP + s2] = acc[i][j][h];
                }
    }
    } else {
    constexpr int TA = (NP + 7) / 8, TB = (NP + 15) / 16, NA = 8 * TA, NB = 16 * TB;
    __shared__ double S[kCpChunk][ST];
    __shared__ double P1[kCpChunk][NA], P2[kCpChunk][NB];
    __shared__ int pa[NP], pb[NP];
    pair_tables<Q>(pa, pb);
    const int tid = threadIdx.x, ta = tid / 16, tb = tid - (tid / 16) * 16;
    for (int pc = blockIdx.x; pc < npieces; pc += gridDim.x) {
        const int g = (int)pieces[2 * pc];
        const int64_t p0 = pieces[2 * pc + 1], pe = min(p0 + kCpPiece, (int64_t)c.grp_pts[g + 1]);
        double acc[TA][TB];
#pragma unroll
        for (int i = 0; i < TA; ++i)
#pragma unroll
            for (int j = 0; j < TB; ++j) acc[i][j] = 0.0;
        for (int64_t base = p0; base < pe; base += kCpChunk) {
            const int np = (int)(pe - base < kCpChunk ? pe - base : kCpChunk);
            __syncthreads();
            for (int t = tid; t < np * ST; t += kCpThreads) {
                const int k = t / ST, o = t - k * ST;
                const int64_t pt = c.grp_perm[base + k];
                S[k][o] = o < Q ? c.cvals1[pt * Q + o] : (o < 2 * Q ? c.cvals2[pt * Q + (o - Q)] : c.cut_cw[pt]);
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
        double* out = gpiece[g + 1] - gpiece[g] == 1 ? E + (int64_t)g * NP * NP : Epart + (int64_t)pc * NP * NP;
#pragma unroll
        for (int i = 0; i < TA; ++i)
#pragma unroll
            for (int j = 0; j < TB; ++j) {
                const int s1 = ta * TA + i, s2 = tb * TB + j;
                if (s1 < NP && s2 < NP) out[s1 * NP + s2] = acc[i][j];
            }
    }
    }
}

// E[g] = sum of its pieces in order (gpiece: ngroups + 1 piece offsets), groups of two or more pieces
__global__ void k_cut_pairs_reduce(const int32_t* __restrict__ gpiece, int ngroups, int npp,
                                   const double* __restrict__ Epart, double* __restrict__ E) {
    const int64_t total = (int64_t)ngroups * npp;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int g = (int)(t / npp), e = (int)(t - (int64_t)g * npp);
        if (gpiece[g + 1] - gpiece[g] == 1) continue;       // written by k_cut_pairs
        double acc = 0.0;
        for (int pc = gpiece[g]; pc < gpiece[g + 1]; ++pc) acc += Epart[(int64_t)pc * npp + e];
        E[t] = acc;
    }
}

// ---------------------------------------------------------------------------
// Per cut row (descriptor rows [r0, r1)): a block per row, a thread per
// window entry o = (o1, o2), j = (i1 - p + o1, i2 - p + o2).  The row's
// support elements (slot of their Gauss block, -1 when excluded: not
// interior, inside the box, or MASK rows) are staged with, per window line,
// the range of support elements whose span covers j (the spans increase
// along the support, so it is one range); the row's span-key groups come as
// a list (rg_ptr / rg: group, key1, key2; geometry, built once per plan).
// Every thread sums its entry's terms -- Gauss elements in (e1, e2) order,
// then the groups in list order -- in registers, and writes the row's plane
// entry.  gslot: element -> Gauss block slot.
// ---------------------------------------------------------------------------
template <int P>
__global__ void __launch_bounds__(32 * (((2 * P + 1) * (2 * P + 1) + 31) / 32))
k_cut_rows_gather(tq_rawctx c, int r0, int r1, const int32_t* __restrict__ gslot, const double* __restrict__ Eg,
                  const double* __restrict__ Ec, const int32_t* __restrict__ rg_ptr, const int32_t* __restrict__ rg,
                  int* __restrict__ status) {
    constexpr int Q = P + 1, W = 2 * P + 1, T = W * W, NP = Pairs<Q>::NP;
    __shared__ int S[Q][Q], F1[Q], F2[Q], pidx[Q][Q], K1[W][2], OFF1[W][Q], OFF2[W][Q];
    const int tid = threadIdx.x;
    for (int t = tid; t < Q * Q; t += blockDim.x) {
        const int a = t / Q, b = t - (t / Q) * Q;
        pidx[a][b] = a <= b ? Pairs<Q>::of(a, b) : Pairs<Q>::of(b, a);
    }
    const int o1 = tid / W, o2 = tid - (tid / W) * W;
    for (int r = r0 + blockIdx.x; r < r1; r += gridDim.x) {
        const RowDescC d = reinterpret_cast<const RowDescC*>(c.desc)[r];
        const int i1 = d.fidx / c.n2, i2 = d.fidx - (d.fidx / c.n2) * c.n2;
        const int ef1 = c.el_first1[i1], ef2 = c.el_first2[i2];
        const int ne1 = c.el_last1[i1] - ef1 + 1, ne2 = c.el_last2[i2] - ef2 + 1;
        const bool gauss = d.mode == TQ_ROW_GAUSS || d.mode == TQ_ROW_BOX;
        const bool box = d.mode == TQ_ROW_BOX && d.a1 >= 0;
        __syncthreads();
        for (int t = tid; t < Q * Q; t += blockDim.x) {
            const int k1 = t / Q, k2 = t - (t / Q) * Q;
            int sl = -1;
            if (gauss && k1 < ne1 && k2 < ne2) {
                const int e1 = ef1 + k1, e2 = ef2 + k2;
                const int64_t e = (int64_t)e1 * c.nel2 + e2;
                const bool inbox = box && e1 >= d.a1 && e1 <= d.b1 && e2 >= d.a2 && e2 <= d.b2;
                const int gs = gslot[e];
                const bool inner = c.elem_class[e] == TQ_INTERIOR;
                if (inner && !inbox) {
                    sl = gs;
                    if (sl < 0) atomicOr(status, 4);      // the element list missed it: flagged
                }
            }
            S[k1][k2] = sl < 0 ? -1 : sl * (NP * NP);      // block offset (or -1)
            if (k2 == 0) F1[k1] = k1 < ne1 ? c.espan1[ef1 + k1] - P : INT_MAX / 2;
            if (k1 == 0) F2[k2] = k2 < ne2 ? c.espan2[ef2 + k2] - P : INT_MAX / 2;
        }
        __syncthreads();
        // per window line o and support element k: the pair offset of
        // (a, b) = (i - F(k), j - F(k)) when F(k) covers j (else -1), and the
        // range of such k for direction 1
        for (int t = tid; t < 2 * W * Q; t += blockDim.x) {
            const bool d1 = t < W * Q;
            const int u = d1 ? t : t - W * Q, o = u / Q, k = u - (u / Q) * Q;
            const int i = d1 ? i1 : i2, j = i - P + o, F = (d1 ? F1 : F2)[k];
            const bool ok = k < (d1 ? ne1 : ne2) && F >= j - P && F <= j;
            (d1 ? OFF1 : OFF2)[o][k] = ok ? pidx[i - F][j - F] * (d1 ? NP : 1) : -1;
        }
        if (tid < W) {
            int lo = 0, hi = -1;
            const int j = i1 - P + tid;
            for (int k = 0; k < ne1; ++k)
                if (F1[k] >= j - P && F1[k] <= j) {
                    if (hi < lo) lo = k;
                    hi = k;
                }
            K1[tid][0] = lo;
            K1[tid][1] = hi;
        }
        __syncthreads();
        if (tid < T) {
            const int j1 = i1 - P + o1, j2 = i2 - P + o2;
            const int lo1 = K1[o1][0], hi1 = K1[o1][1];
            int off2[Q];
#pragma unroll
            for (int k2 = 0; k2 < Q; ++k2) off2[k2] = OFF2[o2][k2];
            double acc = 0.0;
            // a window line's terms are loaded together (Q predicated loads in
            // flight), then added in order
            for (int k1 = lo1; k1 <= hi1; ++k1) {
                const int pr1 = OFF1[o1][k1];
                double v[Q];
                bool ok[Q];
#pragma unroll
                for (int k2 = 0; k2 < Q; ++k2) {
                    const int sl = S[k1][k2];
                    ok[k2] = sl >= 0 && off2[k2] >= 0;
                    v[k2] = ok[k2] ? __ldg(Eg + (sl + pr1 + off2[k2])) : 0.0;
                }
#pragma unroll
                for (int k2 = 0; k2 < Q; ++k2)
                    if (ok[k2]) acc += v[k2];
            }
            if (Ec) {
                const int gb = rg_ptr[r - r0], ge = rg_ptr[r - r0 + 1];
                constexpr int GU = 8;
                for (int k0 = gb; k0 < ge; k0 += GU) {
                    double v[GU];
                    bool ok[GU];
#pragma unroll
                    for (int u = 0; u < GU; ++u) {
                        const int k = k0 + u;
                        ok[u] = false;
                        v[u] = 0.0;
                        if (k < ge) {
                            const int g = __ldg(rg + 3 * k), f1 = __ldg(rg + 3 * k + 1), f2 = __ldg(rg + 3 * k + 2);
                            const int b1 = j1 - f1, b2 = j2 - f2;
                            ok[u] = b1 >= 0 && b1 <= P && b2 >= 0 && b2 <= P;
                            if (ok[u])
                                v[u] = __ldg(Ec + (int64_t)g * (NP * NP) + pidx[i1 - f1][b1] * NP + pidx[i2 - f2][b2]);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < GU; ++u)
                        if (ok[u]) acc += v[u];
                }
            }
            c.raw[(int64_t)tid * c.raw_ld + c.store[r]] = acc;
        }
    }
}

// Element-major form of the same gather.  The row block is accumulated in
// shared memory; element e with first functions (F1, F2) adds
// E_e[pair(i1 - F1, b1)][pair(i2 - F2, b2)] to entry (F1 + b1 - i1 + P,
// F2 + b2 - i2 + P).  Entry line o1 belongs to warp o1 mod NWG, so every
// entry is updated by one warp only; within a warp the lanes cover (b1, b2)
// pairs of one element at a time (distinct entries) and the elements are
// walked in the entry-major kernel's order -- Gauss elements (k1, k2)
// ascending, then the row's groups in list order -- with a warp barrier
// between elements.  Every entry receives the same additions in the same
// order as in k_cut_rows_gather (bit-identical), at one load per element and
// lane instead of a predicated Q x Q sweep per entry.
template <int P>
struct GatherEm {
    static constexpr int Q = P + 1, MB = 32 / Q, NWG = (Q + MB - 1) / MB;
};

template <int P>
__global__ void __launch_bounds__(32 * GatherEm<P>::NWG)
k_cut_rows_gather_em(tq_rawctx c, int r0, int r1, const int32_t* __restrict__ gslot, const double* __restrict__ Eg,
                     const double* __restrict__ Ec, const int32_t* __restrict__ rg_ptr, const int32_t* __restrict__ rg,
                     int* __restrict__ status) {
    constexpr int Q = P + 1, W = 2 * P + 1, T = W * W, NP = Pairs<Q>::NP, QQ = Q * Q, GB = 8;
    constexpr int MB = GatherEm<P>::MB, NWG = GatherEm<P>::NWG, NT = 32 * NWG;
    __shared__ double acc[T];
    __shared__ int S[QQ], F1[Q], F2[Q], pidx[Q][Q];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int t = tid; t < QQ; t += NT) {
        const int a = t / Q, b = t - (t / Q) * Q;
        pidx[a][b] = a <= b ? Pairs<Q>::of(a, b) : Pairs<Q>::of(b, a);
    }
    const bool lact = lane < MB * Q;
    const int b2 = lane % Q, m = lane / Q;
    for (int r = r0 + blockIdx.x; r < r1; r += gridDim.x) {
        const RowDescC d = reinterpret_cast<const RowDescC*>(c.desc)[r];
        const int i1 = d.fidx / c.n2, i2 = d.fidx - (d.fidx / c.n2) * c.n2;
        const int ef1 = c.el_first1[i1], ef2 = c.el_first2[i2];
        const int ne1 = c.el_last1[i1] - ef1 + 1, ne2 = c.el_last2[i2] - ef2 + 1;
        const bool gauss = d.mode == TQ_ROW_GAUSS || d.mode == TQ_ROW_BOX;
        const bool box = d.mode == TQ_ROW_BOX && d.a1 >= 0;
        __syncthreads();          // the previous row's block is written out
        for (int t = tid; t < T; t += NT) acc[t] = 0.0;
        for (int t = tid; t < QQ; t += NT) {
            const int k1 = t / Q, k2 = t - (t / Q) * Q;
            int sl = -1;
            if (gauss && k1 < ne1 && k2 < ne2) {
                const int e1 = ef1 + k1, e2 = ef2 + k2;
                const int64_t e = (int64_t)e1 * c.nel2 + e2;
                const bool inbox = box && e1 >= d.a1 && e1 <= d.b1 && e2 >= d.a2 && e2 <= d.b2;
                if (c.elem_class[e] == TQ_INTERIOR && !inbox) {
                    sl = gslot[e];
                    if (sl < 0) atomicOr(status, 4);      // the element list missed it: flagged
                }
            }
            S[t] = sl;
            if (k2 == 0) F1[k1] = k1 < ne1 ? c.espan1[ef1 + k1] - P : 0;
            if (k1 == 0) F2[k2] = k2 < ne2 ? c.espan2[ef2 + k2] - P : 0;
        }
        __syncthreads();
        // lane -> b1 of this warp's entry lines for an element starting at f1
        auto lane_b1 = [&](int f1) {
            const int base = f1 - i1 + P;                     // o1 of b1 = 0
            const int start = ((warp - base) % NWG + NWG) % NWG;
            return start + NWG * m;
        };
        // per-lane direction-2 parts of the support columns k2 (fixed over k1)
        int A2[Q], O2[Q];
#pragma unroll
        for (int k2 = 0; k2 < Q; ++k2) {
            const int f2 = F2[k2];
            const bool ok2 = k2 < ne2;
            A2[k2] = ok2 ? pidx[i2 - f2][b2] : 0;
            O2[k2] = f2 + b2 - i2 + P;
        }
        // Gauss elements, (k1, k2) ascending: one support line k1 per batch
        for (int k1 = 0; k1 < ne1; ++k1) {
            const int f1 = F1[k1], b1 = lane_b1(f1);
            const bool ok1 = lact && b1 < Q;
            const int A1 = ok1 ? pidx[i1 - f1][b1] * NP : 0;
            const int o1w = (f1 + b1 - i1 + P) * W;
            double v[Q];
            int sl[Q];
#pragma unroll
            for (int k2 = 0; k2 < Q; ++k2) {
                sl[k2] = S[k1 * Q + k2];
                v[k2] = (ok1 && sl[k2] >= 0) ? __ldg(Eg + ((int64_t)sl[k2] * (NP * NP) + A1 + A2[k2])) : 0.0;
            }
#pragma unroll
            for (int k2 = 0; k2 < Q; ++k2) {
                if (ok1 && sl[k2] >= 0) acc[o1w + O2[k2]] += v[k2];
                __syncwarp();
            }
        }
        // span-key groups of the row, list order
        if (Ec) {
            const int gb = rg_ptr[r - r0], ge = rg_ptr[r - r0 + 1];
            for (int k0 = gb; k0 < ge; k0 += GB) {
                double v[GB];
                int at[GB];
#pragma unroll
                for (int u = 0; u < GB; ++u) {
                    const int k = k0 + u;
                    v[u] = 0.0;
                    at[u] = -1;
                    if (k < ge) {
                        const int g = __ldg(rg + 3 * k), f1 = __ldg(rg + 3 * k + 1), f2 = __ldg(rg + 3 * k + 2);
                        const int b1 = lane_b1(f1);
                        if (lact && b1 < Q) {
                            v[u] = __ldg(Ec + ((int64_t)g * (NP * NP) + pidx[i1 - f1][b1] * NP + pidx[i2 - f2][b2]));
                            at[u] = (f1 + b1 - i1 + P) * W + (f2 + b2 - i2 + P);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < GB; ++u) {
                    if (at[u] >= 0) acc[at[u]] += v[u];
                    __syncwarp();
                }
            }
        }
        __syncthreads();
        const int64_t st = c.store[r];
        for (int t = tid; t < T; t += NT) c.raw[(int64_t)t * c.raw_ld + st] = acc[t];
    }
}

}  // namespace tq

using namespace tq;

extern "C" int64_t tq_pair_block_doubles(int32_t p) {
    const int64_t np = (int64_t)(p + 1) * (p + 2) / 2;
    return np * np;
}

// Element-Gauss blocks in pair form of the listed elements (gel: nslot x 2
// element indices; E: nslot x tq_pair_block_doubles(p)).  c: det J computed
// in the kernel when geo.kind == TQ_COEFF_GEOMETRY (X1 / X2: the element
// Gauss points per direction, nel x (p+1)), else cgp = c at the elements'
// (p+1)^2 Gauss points, [slot][g1][g2].  Needs p1 == p2 and ng = p + 1.
// geometry line tables of the element Gauss points for tq_gauss_pairs
// (n points u: span n int32, nd n x 2 (p_geo + 1) doubles)
extern "C" int tq_geo_lines(tq_coeff geo, const double* u, int32_t n, int32_t* span, double* nd, void* stream) {
    if (n <= 0) return TQ_OK;
    if (geo.kind != TQ_COEFF_GEOMETRY || geo.p > kMaxP) { set_error("tq_geo_lines needs a geometry map"); return TQ_EINVAL; }
    switch (geo.p) {
#define CASE(Q) case Q: k_geo_lines<Q><<<(n + 127) / 128, 128, 0, S(stream)>>>(geo, u, n, span, nd); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
        default: set_error("geometry degree out of range"); return TQ_EINVAL;
    }
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_geo_lines");
    return TQ_OK;
}

extern "C" int tq_gauss_pairs(tq_rawctx c, tq_coeff geo, const double* X1, const double* X2, const int32_t* gel,
                              int32_t nslot, const double* cgp, double* E, const int32_t* lsp1, const double* lnd1,
                              const int32_t* lsp2, const double* lnd2, void* stream) {
    if (nslot <= 0) return TQ_OK;
    if (c.p1 != c.p2 || c.ng1 != c.p1 + 1 || c.ng2 != c.p2 + 1) { set_error("tq_gauss_pairs needs p1 == p2 and p + 1 Gauss points"); return TQ_EINVAL; }
    if (geo.kind == TQ_COEFF_GEOMETRY ? (geo.p > kMaxP || !X1 || !X2) : !cgp) { set_error("tq_gauss_pairs: no coefficient"); return TQ_EINVAL; }
    const int grid = std::min(nslot, kSms * 16);
    switch (c.p1 + 1) {
#define CASE(Q) case Q: k_gauss_pairs<Q><<<grid, kGpThreads, 0, S(stream)>>>(c, geo, X1, X2, gel, nslot, cgp, E, \
            lsp1, lnd1, lsp2, lnd2); break;
        CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9)
#undef CASE
        default: set_error("degree out of range for the pair blocks"); return TQ_EINVAL;
    }
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_gauss_pairs");
    return TQ_OK;
}

extern "C" int32_t tq_cut_pair_piece(void) { return kCpPiece; }

// Span-key group blocks in pair form (E: ngroups x tq_pair_block_doubles(p)),
// by pieces of at most tq_cut_pair_piece() points: pieces npieces x 2 int64
// (group, first point), gpiece ngroups + 1 piece offsets per group, Epart
// npieces x tq_pair_block_doubles(p) scratch.
extern "C" int tq_cut_pairs(tq_rawctx c, const int64_t* pieces, int32_t npieces, const int32_t* gpiece, double* Epart,
                            double* E, void* stream) {
    if (c.ngroups <= 0) return TQ_OK;
    if (c.p1 != c.p2) { set_error("tq_cut_pairs needs p1 == p2"); return TQ_EINVAL; }
    const int grid = std::min(npieces, kSms * 16);
    switch (c.p1 + 1) {
#define CASE(Q) case Q: k_cut_pairs<Q><<<grid, kCpThreads, 0, S(stream)>>>(c, pieces, npieces, Epart, gpiece, E); break;
        CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11)
#undef CASE
        default: set_error("degree out of range"); return TQ_EINVAL;
    }
    ::tq::note_launch();
    const int npp = (int)tq_pair_block_doubles(c.p1);
    k_cut_pairs_reduce<<<grid_for((int64_t)c.ngroups * npp, 256), 256, 0, S(stream)>>>(gpiece, c.ngroups, npp, Epart, E);
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_cut_pairs");
    return TQ_OK;
}

// Rows [r0, r1) (the cut rows, planes layout): Gauss + cut-cell parts from
// the pair blocks (Eg / gslot: tq_gauss_pairs, Ec: tq_cut_pairs or NULL),
// written to the planes (rg_ptr: r1 - r0 + 1 offsets into rg = the rows'
// span-key groups, 3 ints each: group, key1, key2).  status |= 4 when a
// needed Gauss block is missing.
extern "C" int tq_cut_rows_gather(tq_rawctx c, int32_t r0, int32_t r1, const int32_t* gslot, const double* Eg,
                                  const double* Ec, const int32_t* rg_ptr, const int32_t* rg, int32_t* status,
                                  void* stream) {
    if (r1 <= r0) return TQ_OK;
    if (!c.raw_ld || !c.store || c.p1 != c.p2) { set_error("tq_cut_rows_gather needs the planes layout and p1 == p2"); return TQ_EINVAL; }
    // element-major (default; 127 -> 91 us at config 4 p = 8, bit-identical)
    // or the entry-major kernel (TQ_GATHER_EM=0: A/B and the equality test)
    static int em = -1;
    if (em < 0) {
        const char* e = getenv("TQ_GATHER_EM");
        em = e ? atoi(e) : 1;
    }
    const int grid = (int)std::min<int64_t>(r1 - r0, (int64_t)kSms * (em ? 32 : 16));
    switch (c.p1) {
#define CASE(Q) case Q: \
        if (em) k_cut_rows_gather_em<Q><<<grid, 32 * GatherEm<Q>::NWG, 0, S(stream)>>>(c, r0, r1, gslot, Eg, Ec, rg_ptr, \
                                                                                      rg, status); \
        else k_cut_rows_gather<Q><<<grid, 32 * (((2 * Q + 1) * (2 * Q + 1) + 31) / 32), 0, S(stream)>>>( \
            c, r0, r1, gslot, Eg, Ec, rg_ptr, rg, status); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
        default: set_error("degree out of range"); return TQ_EINVAL;
    }
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_cut_rows_gather");
    return TQ_OK;
}
