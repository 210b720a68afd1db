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
#include <stdlib.h>

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

// tile mode: offset of row r = its tile base + the counts of the rows before
// it in the tile (warp-collective; every lane gets the value)
__device__ __forceinline__ int tile_offset(const tq_rowctx& c, int r, int lane) {
    const int rel = r - c.row_begin;
    const int cnt = lane < (rel & 31) ? __ldg(c.counts + ((rel & ~31) + lane)) : 0;
    return __ldg((c.tiles + TQ_TILE_PAD(c.row_end - c.row_begin)) + (rel >> 5)) + __reduce_add_sync(0xffffffffu, cnt);
}

// floor(x / n) for 0 <= x < 2^24 and n >= 1: float reciprocal, one
// correction step (exact: the float estimate is off by at most one)
__device__ __forceinline__ int fdiv24(int x, int n, float inv) {
    int q = __float2int_rz(__int2float_rn(x) * inv);
    const int r = x - q * n;
    q += (r >= n) - (r < 0);
    return q;
}

// i1 = idx / n2 for a function index (float path when n1 * n2 < 2^24)
__device__ __forceinline__ int row_of(const tq_rowctx& c, int idx) {
    return c.n1 * c.n2 < (1 << 24) ? fdiv24(idx, c.n2, __frcp_rn((float)c.n2)) : idx / c.n2;
}

// q1 = e / t2 for a window entry (e < 2^24)
__device__ __forceinline__ int win_div(int e, int t2, float inv_t2) { return fdiv24(e, t2, inv_t2); }

struct RowGeom {
    int i1, i2, s_i, j1lo, j2lo, t1, t2;
};

__device__ inline RowGeom row_geom(const tq_rowctx& c, int r) {
    RowGeom g;
    int idx = c.active[r];
    g.i1 = row_of(c, idx);
    g.i2 = idx - g.i1 * c.n2;
    g.s_i = c.slot[idx];
    g.j1lo = c.ov_lo1[g.i1];
    g.j2lo = c.ov_lo2[g.i2];
    g.t1 = c.ov_hi1[g.i1] - g.j1lo + 1;
    g.t2 = c.ov_hi2[g.i2] - g.j2lo + 1;
    return g;
}

// an interior separable row on positive factor lines: every window entry has
// a positive partner sum (tq_rowctx.fclass / pos), counted geometrically
__device__ __forceinline__ bool near_row(const tq_rowctx& c, const RowGeom& g) {
    return c.fclass && c.pos && c.tiles && g.s_i < 0 && __ldg(c.fclass + ((int64_t)g.i1 * c.n2 + g.i2)) == TQ_INTERIOR &&
           __ldg(c.pos + g.i1) && __ldg(c.pos + c.n1 + g.i2);
}

// unsymmetrised value of row (i1,i2) at column (j1,j2).  Every symmetrised
// entry is formed as round(round(M_ij) + round(M_ji)) -- explicitly rounded
// products and sum, never contracted into an FMA -- so M_ij and M_ji are
// the same double (the reference's 0.5 (M + M^T) is exactly symmetric).
__device__ __forceinline__ double raw_value(const tq_rowctx& c, int i1, int i2, int s_i, int j1, int j2) {
    const int W1 = 2 * c.p1 + 1, W2 = 2 * c.p2 + 1;
    const int o1 = j1 - i1 + c.p1, o2 = j2 - i2 + c.p2;
    if (s_i < 0) return __dmul_rn(__ldg(c.a1 + (int64_t)i1 * W1 + o1), __ldg(c.a2 + (int64_t)i2 * W2 + o2));
    if (c.raw_ld) return __ldg(c.raw + (int64_t)(o1 * W2 + o2) * c.raw_ld + s_i);
    return __ldg(c.raw + (int64_t)s_i * (W1 * W2) + o1 * W2 + o2);
}

// symmetrised sum M_ij + M_ji for column j; returns col index or -1
__device__ __forceinline__ int entry(const tq_rowctx& c, const RowGeom& g, int e, double& v) {
    int q1 = win_div(e, g.t2, __frcp_rn((float)g.t2));
    int j1 = g.j1lo + q1, j2 = g.j2lo + (e - q1 * g.t2);
    int jidx = j1 * c.n2 + j2;
    int col = __ldg(c.col_of + jidx);
    if (col < 0) return -1;
    int s_j = __ldg(c.slot + jidx);
    v = __dadd_rn(raw_value(c, g.i1, g.i2, g.s_i, j1, j2), raw_value(c, j1, j2, s_j, g.i1, g.i2));
    return v != 0.0 ? col : -1;
}

// U chunks of 32 entries of row g at once (lane's entries e0 + 32u + lane):
// col_of, slot and the row's own raw value depend only on the column, so they
// are issued together; only the partner's raw value waits for slot[j] -- two
// dependent load levels per 32U entries instead of three per 32.  col[u] =
// kept column or -1, v[u] = M_ij + M_ji (same expression as entry()).
template <int U>
__device__ __forceinline__ void entries_batch(const tq_rowctx& c, const RowGeom& g, int e0, int lane, int n,
                                              int* col, double* v) {
    int cl[U], sj[U], j1[U], j2[U];
    double vi[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int e = e0 + 32 * u + lane;
        const bool valid = e < n;
        const int ee = valid ? e : 0;
        const int q1 = win_div(ee, g.t2, __frcp_rn((float)g.t2));
        j1[u] = g.j1lo + q1;
        j2[u] = g.j2lo + (ee - q1 * g.t2);
        const int jidx = j1[u] * c.n2 + j2[u];
        cl[u] = valid ? __ldg(c.col_of + jidx) : -1;
        sj[u] = valid ? __ldg(c.slot + jidx) : -1;
        vi[u] = valid ? raw_value(c, g.i1, g.i2, g.s_i, j1[u], j2[u]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        col[u] = -1;
        v[u] = 0.0;
        if (cl[u] >= 0) {
            const double w = __dadd_rn(vi[u], raw_value(c, j1[u], j2[u], sj[u], g.i1, g.i2));
            v[u] = w;
            col[u] = w != 0.0 ? cl[u] : -1;
        }
    }
}

// Counts, pass 1 (thread per row, no raw values needed): deep rows are
// counted arithmetically and flagged fast when their window is full; other
// rows are appended to list A (counted by pass 2), deep rows with a partial
// window to list B (both lists feed the row-parallel fill).
// GEO: deep = geo[idx] && pos[i1] && pos[n1 + i2] from the geometric flags
// and the per-line factor positivity (no deep array is formed); otherwise
// c.deep holds complete deep flags.
// SPEC (with GEO): every line's factors assumed positive (pos not read) --
// the speculative pass launched before the factors exist; tq_row_counts_verify
// redoes the pass (guard != 0) only when some line is not positive.
template <bool GEO, bool SPEC = false>
__global__ void k_row_counts_deep(tq_rowctx c, const int8_t* __restrict__ geo, const int8_t* __restrict__ pos,
                                  int32_t* __restrict__ counts,
                                  int* __restrict__ list, int* __restrict__ nlist, int* __restrict__ listb,
                                  int* __restrict__ nlistb, const int* __restrict__ guard = nullptr) {
    if (guard && *guard == 0) return;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    // grid-stride loop with a warp-uniform trip count (the appends are warp-aggregated)
    const int n = c.row_end - c.row_begin, stride = gridDim.x * blockDim.x;
    for (int base = blockIdx.x * blockDim.x; base < n; base += stride) {
        const int r = c.row_begin + base + threadIdx.x;
        bool to_a = false, to_b = false;
        int mycount = 0;      // list-A rows: added by pass 2
        if (r < c.row_end) {
            const int idx = __ldg(c.active + r);
            const int i1 = row_of(c, idx), i2 = idx - i1 * c.n2;
            bool deep;
            if (GEO && SPEC) deep = __ldg(geo + idx);
            else if (GEO) deep = __ldg(geo + idx) && __ldg(pos + i1) && __ldg(pos + c.n1 + i2);
            else deep = c.deep && __ldg(c.deep + idx);
            if (deep) {
                const int t1 = __ldg(c.ov_hi1 + i1) - __ldg(c.ov_lo1 + i1) + 1;
                const int t2 = __ldg(c.ov_hi2 + i2) - __ldg(c.ov_lo2 + i2) + 1;
                counts[r - c.row_begin] = t1 * t2;
                mycount = t1 * t2;
                const bool full = t1 == 2 * c.p1 + 1 && t2 == 2 * c.p2 + 1;
                if (c.rowfast) c.rowfast[r - c.row_begin] = full ? 1 : 0;
                to_b = !(full && c.rowfast);
            } else {
                if (c.rowfast) c.rowfast[r - c.row_begin] = 0;
                to_a = true;
            }
        }
        const unsigned ma = __ballot_sync(0xffffffffu, to_a), mb = __ballot_sync(0xffffffffu, to_b);
        int ba = 0, bb = 0;
        if (lane == 0) {
            if (ma) ba = atomicAdd(nlist, __popc(ma));
            if (mb) bb = atomicAdd(nlistb, __popc(mb));
        }
        ba = __shfl_sync(0xffffffffu, ba, 0);
        bb = __shfl_sync(0xffffffffu, bb, 0);
        if (to_a) list[ba + __popc(ma & lt)] = r;
        if (to_b) listb[bb + __popc(mb & lt)] = r;
        if (c.tiles) {          // warp = one 32-row tile (base is a multiple of the block size)
            const int tsum = __reduce_add_sync(0xffffffffu, mycount);
            const int t = (base + threadIdx.x) >> 5;
            if (lane == 0 && (t << 5) < n) c.tiles[t] = tsum;
            // first list-A row (encoded INT_MAX - row: the largest code wins)
            const unsigned enc = __reduce_max_sync(0xffffffffu, to_a ? (unsigned)(0x7fffffff - r) : 0u);
            if (lane == 0 && enc) atomicMax(reinterpret_cast<unsigned*>(c.tiles + TQ_TILE_CTL(n)), enc);
            // last list-A row + 1
            const unsigned last1 = __reduce_max_sync(0xffffffffu, to_a ? (unsigned)(r + 1) : 0u);
            if (lane == 0 && last1) atomicMax(reinterpret_cast<unsigned*>(c.tiles + TQ_TILE_CTL(n) + 1), last1);
        }
    }
}

// The entries of R rows at once, 3 chunks of 32 per row (rows of <= 96
// entries): the column-only loads of all 3R chunks are issued together, then
// the partners' raw values -- two dependent load levels for R rows.
template <int R>
__device__ __forceinline__ void entries_rows(const tq_rowctx& c, const RowGeom* g, const bool* ok, int lane,
                                             int* col, double* v) {
    constexpr int U = 3 * R;
    int cl[U], sj[U], j1[U], j2[U];
    double vi[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const RowGeom& G = g[u / 3];
        const int n = G.t1 * G.t2;
        const int e = 32 * (u % 3) + lane;
        const bool valid = ok[u / 3] && e < n;
        const int ee = valid ? e : 0;
        const int q1 = win_div(ee, G.t2, __frcp_rn((float)G.t2));
        j1[u] = G.j1lo + q1;
        j2[u] = G.j2lo + (ee - q1 * G.t2);
        const int jidx = j1[u] * c.n2 + j2[u];
        cl[u] = valid ? __ldg(c.col_of + jidx) : -1;
        sj[u] = valid ? __ldg(c.slot + jidx) : -1;
        vi[u] = valid ? raw_value(c, G.i1, G.i2, G.s_i, j1[u], j2[u]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const RowGeom& G = g[u / 3];
        col[u] = -1;
        v[u] = 0.0;
        if (cl[u] >= 0) {
            const double w = __dadd_rn(vi[u], raw_value(c, j1[u], j2[u], sj[u], G.i1, G.i2));
            v[u] = w;
            col[u] = w != 0.0 ? cl[u] : -1;
        }
    }
}

// Counts, pass 2 (warp per kRowsPass2 listed rows): value-based symmetric
// zero test.  The rows' geometry and entry loads are issued together (the
// pass is a chain of dependent loads per row); rows of more than 96 entries
// (p > 4) go one at a time.
constexpr int kRowsPass2 = 2;

// Row geometry of the listed rows, one coalesced 32-byte record each
// (k_list_geometry, launched right after count pass 1, off the critical
// path): count pass 2 then starts from one load per row instead of the
// list -> active -> slot / overlap chain.  near: near_row(), counted
// geometrically.
struct alignas(16) ListRec {
    int r, i1, i2, s_i, j1lo, j2lo, t1, t2n;      // t2n = t2 | near << 16
};

__global__ void k_list_geometry(tq_rowctx c, const int* __restrict__ list, const int* __restrict__ nlist,
                                ListRec* __restrict__ rec) {
    const int n = *nlist;
    for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
        const int r = list[u];
        const RowGeom g = row_geom(c, r);
        ListRec x;
        x.r = r;
        x.i1 = g.i1;
        x.i2 = g.i2;
        x.s_i = g.s_i;
        x.j1lo = g.j1lo;
        x.j2lo = g.j2lo;
        x.t1 = g.t1;
        x.t2n = g.t2 | (near_row(c, g) ? 1 << 16 : 0);
        rec[u] = x;
    }
}

__global__ void k_row_counts_list(tq_rowctx c, int32_t* __restrict__ counts, const int* __restrict__ list,
                                  const int* __restrict__ nlist, const ListRec* __restrict__ recs = nullptr) {
    constexpr int R = kRowsPass2;
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const int n_rows = *nlist;
    for (int q0 = warp * R; q0 < n_rows; q0 += nw * R) {
        int r[R], cnt[R];
        bool ok[R];
        RowGeom g[R];
        bool small = true;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            ok[k] = q0 + k < n_rows;
            bool near;
            if (recs) {           // the row's geometry in one record
                const ListRec x = recs[ok[k] ? q0 + k : q0];
                r[k] = x.r;
                g[k].i1 = x.i1;
                g[k].i2 = x.i2;
                g[k].s_i = x.s_i;
                g[k].j1lo = x.j1lo;
                g[k].j2lo = x.j2lo;
                g[k].t1 = x.t1;
                g[k].t2 = x.t2n & 0xffff;
                near = (x.t2n >> 16) != 0;
            } else {
                r[k] = ok[k] ? list[q0 + k] : list[q0];
                g[k] = row_geom(c, r[k]);
                near = near_row(c, g[k]);
            }
            small = small && g[k].t1 * g[k].t2 <= 96;
            cnt[k] = 0;
            if (ok[k] && near) {      // counted geometrically, no entry loads
                cnt[k] = g[k].t1 * g[k].t2;
                ok[k] = false;
            }
        }
        bool any = false;
#pragma unroll
        for (int k = 0; k < R; ++k) any = any || ok[k];
        if (small && any) {
            int col[3 * R];
            double v[3 * R];
            entries_rows<R>(c, g, ok, lane, col, v);
#pragma unroll
            for (int u = 0; u < 3 * R; ++u) cnt[u / 3] += __popc(__ballot_sync(0xffffffffu, col[u] >= 0));
        } else if (!small) {
            for (int k = 0; k < R; ++k) {
                if (!ok[k]) continue;
                const int n = g[k].t1 * g[k].t2;
                for (int e0 = 0; e0 < n; e0 += 96) {
                    int col[3];
                    double v[3];
                    entries_batch<3>(c, g[k], e0, lane, n, col, v);
#pragma unroll
                    for (int u = 0; u < 3; ++u) cnt[k] += __popc(__ballot_sync(0xffffffffu, col[u] >= 0));
                }
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < R; ++k) {
                if (q0 + k >= n_rows) continue;
                counts[r[k] - c.row_begin] = cnt[k];
                if (c.tiles) atomicAdd(c.tiles + ((r[k] - c.row_begin) >> 5), cnt[k]);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Fill kernel (separable path).  Work unit: a warp tile of 32 consecutive
// active rows, assigned statically; the next tile's per-row words (active id,
// CSR offset, fast flag from the count pass) are prefetched while the
// current tile is processed.
//
//  regular tile -- 32 deep full-window rows on one i1-line with consecutive
//    i2 (94% of the tiles at config 5): the direction-1 factors and column
//    bases are shared by the whole tile and the direction-2 factors form one
//    contiguous band, so a single round of coalesced loads feeds 32 rows.
//    Rows are built in shared memory, kChunk rows at a time, lane -> (q1, q2)
//    with q2 = lane % W fixed, and written to HBM by TMA bulk copies
//    (cp.async.bulk.global.shared::cta), one staging buffer per warp (more resident warps beat double buffering); the
//    16-byte-unaligned ends go through plain stores.
//  irregular tile -- recorded in a list and processed by k_fill_irregular,
//    one warp per row over the whole GPU (these tiles cluster along the
//    trimming curve; row-parallel processing keeps them off the critical path).
// ---------------------------------------------------------------------------
constexpr int kWarpRows = 32;
#ifndef TQ_FILL_SPLIT_TAIL
#define TQ_FILL_SPLIT_TAIL 1
#endif
constexpr bool kFillSplitTail = TQ_FILL_SPLIT_TAIL != 0;   // the last wave of tiles in 16-row halves
#ifndef TQ_FILL_STAGES
#define TQ_FILL_STAGES 1     // one staging buffer per warp: more resident warps beat double buffering (measured)
#endif

#ifndef TQ_FILL_ENTRIES
#define TQ_FILL_ENTRIES 891
#endif
template <int P>
constexpr int fill_chunk() {   // rows per bulk copy: ~10.7 KB of staged entries (11 rows at P = 4, measured best)
    return TQ_FILL_ENTRIES / ((2 * P + 1) * (2 * P + 1)) < 1 ? 1 : (TQ_FILL_ENTRIES / ((2 * P + 1) * (2 * P + 1)) > 32 ? 32 : TQ_FILL_ENTRIES / ((2 * P + 1) * (2 * P + 1)));
}

template <int P>
struct alignas(16) FillStage {
    static constexpr int WW = (2 * P + 1) * (2 * P + 1);
    double d[fill_chunk<P>() * WW + 2];
    alignas(16) int x[fill_chunk<P>() * WW + 4];
};

template <int P>
constexpr int fill_stages() { return TQ_FILL_STAGES; }

template <int P>
struct alignas(16) RegularSlice {
    static constexpr int W = 2 * P + 1;
    FillStage<P> stage[fill_stages<P>()];
    double band[(32 + 2 * P) * W];
};

template <int P>
constexpr size_t fill_slice_bytes() { return (sizeof(RegularSlice<P>) + 15) / 16 * 16; }

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(gdst), "r"((unsigned)__cvta_generic_to_shared(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Emit a run of L (<= 32) consecutive fast rows (i1, i20 .. i20+L-1), CSR
// start pos0 (rows have exactly (2P+1)^2 entries, so the run is one span).
template <int P>
__device__ __forceinline__ void emit_run(const tq_rowctx& c, RegularSlice<P>& S, int lane, int i1, int i20, int L,
                                         int pos0, int& nbulk, int32_t* __restrict__ indices,
                                         double* __restrict__ data) {
    constexpr int W = 2 * P + 1, WW = W * W, R = 32 / W, CH = fill_chunk<P>(), M = (W + R - 1) / R;
    __syncwarp();
    const bool act = lane < R * W;
    const int q2 = lane % W, r0 = lane / W;
    // direction-1 factors and column bases of this lane's q1 = m R + r0 (fixed for the run)
    double rl1[M], rl1t[M];
    int rcb[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int q1 = m * R + r0, j1 = i1 - P + q1;
        const bool ok = act && q1 < W;
        rl1[m] = ok ? __ldg(c.a1 + (int64_t)i1 * W + q1) : 0.0;
        rl1t[m] = ok ? __ldg(c.a1 + (int64_t)j1 * W + (2 * P - q1)) : 0.0;
        rcb[m] = ok ? __ldg(c.col_of + (int64_t)j1 * c.n2 + (i20 - P)) : 0;
    }
    const double* bsrc = c.a2 + (int64_t)(i20 - P) * W;
    for (int q = lane; q < (L + 2 * P) * W; q += 32) S.band[q] = __ldg(bsrc + q);
    __syncwarp();
    for (int k = 0; k * CH < L; ++k) {
        const int rows = min(CH, L - k * CH);
        const int n = rows * WW;
        constexpr int NS = fill_stages<P>();
        FillStage<P>& st = S.stage[nbulk % NS];
        if (lane == 0 && nbulk >= NS) bulk_wait_read<NS - 1>();   // last reader of this buffer is done
        __syncwarp();
        const int pos = pos0 + k * CH * WW;
        const int offd = pos & 1, offx = pos & 3;
        for (int tt = 0; tt < rows; ++tt) {
            const int t = k * CH + tt;
            const double a2 = S.band[(t + P) * W + q2], a2t = S.band[(t + q2) * W + (2 * P - q2)];
#pragma unroll
            for (int m = 0; m < M; ++m) {
                const int q1 = m * R + r0;
                if (act && q1 < W) {
                    const int e = tt * WW + q1 * W + q2;
                    st.x[offx + e] = rcb[m] + t + q2;
                    st.d[offd + e] = 0.5 * __dadd_rn(__dmul_rn(rl1[m], a2), __dmul_rn(rl1t[m], a2t));
                }
            }
        }
        fence_async_shared();
        __syncwarp();
        const int sd = (pos + 1) & ~1, ed = (pos + n) & ~1;
        const int sx = (pos + 3) & ~3, ex = (pos + n) & ~3;
        if (lane == 0) {
            if (ed > sd) bulk_store(data + sd, st.d + (sd - (pos & ~1)), (unsigned)(ed - sd) * 8u);
            if (ex > sx) bulk_store(indices + sx, st.x + (sx - (pos & ~3)), (unsigned)(ex - sx) * 4u);
            bulk_commit();
        }
        ++nbulk;
        if (lane == 1 && sd > pos) data[pos] = st.d[offd];
        if (lane == 2 && ed < pos + n && ed >= sd) data[pos + n - 1] = st.d[offd + n - 1];
        if (lane >= 3 && lane < 3 + min(sx - pos, n)) indices[pos + lane - 3] = st.x[offx + lane - 3];
        if (lane >= 8 && ex >= sx && lane < 8 + (pos + n - ex)) indices[ex + lane - 8] = st.x[offx + (ex - pos) + lane - 8];
    }
}

template <int P>
__global__ void __launch_bounds__(256) k_fill_tiles(tq_rowctx c, int32_t* __restrict__ indptr,
                                                     int32_t* __restrict__ indices, double* __restrict__ data,
                                                     int* __restrict__ irr_rows, int* __restrict__ irr_count,
                                                     int part) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    RegularSlice<P>& S = *reinterpret_cast<RegularSlice<P>*>(smraw + fill_slice_bytes<P>() * wib);
    const unsigned lt = (1u << lane) - 1u;
    const int nwarps = gridDim.x * wpb;
    int nbulk = 0;
    // tile mode: the per-row word is the count, the offset comes from the
    // tile base + an exclusive warp scan (and is written to indptr here).
    // Tiles are numbered within the part (part 1: head then tail tiles,
    // part 2: the tiles in between) and assigned dynamically from a counter
    // per part -- warps that start late, beside other kernels, just take
    // fewer tiles; the next tile is claimed one ahead for the prefetch.
    // Without tile mode: all tiles, static stride.
    const bool tm = c.tiles != nullptr;
    const int nr = c.row_end - c.row_begin, NT = (nr + kWarpRows - 1) / kWarpRows;
    // the scan found another nnz than the captured pass sized the output
    // with (tq_tiles_expect): write nothing
    if (tm && part != 1 && c.tiles[TQ_TILE_CTL(nr) + 4]) return;
    const int32_t* tbase = tm ? (c.tiles + TQ_TILE_PAD(nr)) : nullptr;
    int tA = NT, tB = NT;
    if (tm && part) {
        tA = head_tiles(c);
        tB = max(tail_first(c), tA);
        if (part == 1) tbase = c.tiles + TQ_TILE_EARLY(nr);
    }
    const int ntp = part == 1 ? tA + (NT - tB) : part == 2 ? tB - tA : NT;   // tiles in this part
    int* ctr = tm ? c.tiles + TQ_TILE_CTL(nr) + (part == 1 ? 3 : 2) : nullptr;
    // work units: the part's tiles, the last `ks` of them split into two
    // 16-row halves (dynamic claims only: the final wave of 26-us tiles
    // would otherwise leave most warps idle at the end of the fill)
    const int ks = ctr ? min(ntp, kFillSplitTail ? nwarps : 0) : 0;
    const int nunits = ntp + ks;
    auto unit_tile = [&](int u) -> int { return u < ntp - ks ? u : ntp - ks + ((u - (ntp - ks)) >> 1); };
    auto unit_half = [&](int u) -> int { return u < ntp - ks ? -1 : ((u - (ntp - ks)) & 1); };
    auto tile_row = [&](int u) -> int {       // unit -> first row of its tile (row_end: done)
        if (u >= nunits) return c.row_end;
        const int t = unit_tile(u);
        const int tile = part == 1 ? (t < tA ? t : tB + (t - tA)) : part == 2 ? tA + t : t;
        return c.row_begin + kWarpRows * tile;
    };
    int tcur = blockIdx.x * wpb + wib;
    if (ctr) {
        int t = 0;
        if (lane == 0) t = atomicAdd(ctr, 1);
        tcur = __shfl_sync(0xffffffffu, t, 0);
    }
    const int rhi = c.row_end;
    int R0 = tile_row(tcur);
    int n_idx = 0, n_pos = 0, n_fast = 0, n_tb = 0;
    if (R0 + lane < rhi) {
        n_idx = __ldg(c.active + R0 + lane);
        n_pos = __ldg((tm ? c.counts : indptr) + (R0 + lane - c.row_begin));
        n_fast = c.rowfast ? __ldg(c.rowfast + (R0 + lane - c.row_begin)) : 0;
    }
    if (tm && R0 < rhi) n_tb = __ldg(tbase + ((R0 - c.row_begin) >> 5));
    for (int R1; R0 < rhi; R0 = R1) {
        // a half-tile unit processes its 16 lanes' rows (the offsets still
        // come from the whole tile's counts)
        const int half = unit_half(tcur);
        const bool valid = R0 + lane < rhi && (half < 0 || (lane >> 4) == half);
        int my_pos = n_pos;
        const int my_idx = n_idx, my_fast = valid ? n_fast : 0;
        if (tm) {
            int x = my_pos;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, off);
                if (lane >= off) x += y;
            }
            my_pos = n_tb + x - my_pos;
            if (valid) indptr[R0 + lane - c.row_begin] = my_pos;
        }
        if (ctr) {
            int t = 0;
            if (lane == 0) t = atomicAdd(ctr, 1);
            tcur = __shfl_sync(0xffffffffu, t, 0);
        } else {
            tcur += nwarps;
        }
        R1 = tile_row(tcur);
        if (R1 + lane < rhi) {
            n_idx = __ldg(c.active + R1 + lane);
            n_pos = __ldg((tm ? c.counts : indptr) + (R1 + lane - c.row_begin));
            n_fast = c.rowfast ? __ldg(c.rowfast + (R1 + lane - c.row_begin)) : 0;
        }
        if (tm && R1 < rhi) n_tb = __ldg(tbase + ((R1 - c.row_begin) >> 5));
        // rows that are not fast go to the row-parallel irregular kernel
        // (listed here unless the count pass already listed them)
        const unsigned slow = irr_rows ? __ballot_sync(0xffffffffu, valid && !my_fast) : 0u;
        if (slow) {
            int base = 0;
            if (lane == 0) base = atomicAdd(irr_count, __popc(slow));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (valid && !my_fast) irr_rows[base + __popc(slow & lt)] = R0 + lane;
        }
        // runs of consecutive fast rows on one i1-line: start where the
        // previous lane is not fast, not consecutive, or on another line
        const int prev_idx = __shfl_up_sync(0xffffffffu, my_idx, 1);
        const int prev_fast = __shfl_up_sync(0xffffffffu, my_fast, 1);
        const bool start = my_fast && (lane == 0 || !prev_fast || my_idx != prev_idx + 1 ||
                                       my_idx / c.n2 != prev_idx / c.n2);
        unsigned starts = __ballot_sync(0xffffffffu, start);
        const unsigned fastm = __ballot_sync(0xffffffffu, my_fast != 0);
        while (starts) {
            const int s0 = __ffs(starts) - 1;
            starts &= starts - 1;
            // run length: consecutive fast lanes from s0 until the next start or a slow lane
            const unsigned after = (fastm >> s0);
            const unsigned stop_mask = (~after) | ((starts >> s0) & ~1u);
            const int L = stop_mask ? __ffs(stop_mask) - 1 : 32 - s0;
            const int idx0 = __shfl_sync(0xffffffffu, my_idx, s0);
            const int pos0 = __shfl_sync(0xffffffffu, my_pos, s0);
            const int i1 = idx0 / c.n2;
            emit_run<P>(c, S, lane, i1, idx0 - i1 * c.n2, L, pos0, nbulk, indices, data);
        }
    }
    if (lane == 0) bulk_wait_all();
}

// Listed rows (list A then list B), one warp per row over the whole GPU: deep
// rows from their direction factors (lanes 0..2P hold A1, A1T, column base,
// A2, A2T; entries built by shuffles), other rows through the value-based
// symmetrise/compact path.
template <int P>
__global__ void __launch_bounds__(256) k_fill_irregular(tq_rowctx c, const int32_t* __restrict__ indptr,
                                                         int32_t* __restrict__ indices, double* __restrict__ data,
                                                         const int* __restrict__ irr_rows,
                                                         const int* __restrict__ irr_count,
                                                         const int* __restrict__ irr_rows_b,
                                                         const int* __restrict__ irr_count_b) {
    constexpr int W = 2 * P + 1;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    if (c.tiles && c.tiles[TQ_TILE_CTL(c.row_end - c.row_begin) + 4]) return;     // see k_fill_tiles
    const int na = *irr_count, nrows = na + (irr_count_b ? *irr_count_b : 0);
    for (int u = warp; u < nrows; u += nw) {
        const int r = u < na ? irr_rows[u] : irr_rows_b[u - na];
        RowGeom g = row_geom(c, r);
        int pos = c.tiles ? tile_offset(c, r, lane) : __ldg(indptr + (r - c.row_begin));
        const int n = g.t1 * g.t2;
        // deep rows: list B when the count pass gave the lists, else the flags
        const bool deep_row = irr_rows_b ? u >= na : c.deep[c.active[r]] != 0;
        if (deep_row) {
            double A1 = 0.0, A1T = 0.0, A2 = 0.0, A2T = 0.0;
            int CB = 0;
            if (lane < W) {
                const int j1 = g.i1 - P + lane, j2 = g.i2 - P + lane;
                if (j1 >= g.j1lo && j1 < g.j1lo + g.t1) {
                    A1 = __ldg(c.a1 + (int64_t)g.i1 * W + lane);
                    A1T = __ldg(c.a1 + (int64_t)j1 * W + (2 * P - lane));
                    CB = __ldg(c.col_of + (int64_t)j1 * c.n2 + g.j2lo);
                }
                if (j2 >= g.j2lo && j2 < g.j2lo + g.t2) {
                    A2 = __ldg(c.a2 + (int64_t)g.i2 * W + lane);
                    A2T = __ldg(c.a2 + (int64_t)j2 * W + (2 * P - lane));
                }
            }
            const int off1 = g.j1lo - (g.i1 - P), off2 = g.j2lo - (g.i2 - P);
            for (int e0 = 0; e0 < n; e0 += 32) {
                const int e = e0 + lane;
                const int ee = e < n ? e : n - 1;
                const int q1 = win_div(ee, g.t2, __frcp_rn((float)g.t2)), q2 = ee - q1 * g.t2;
                const int o1 = off1 + q1, o2 = off2 + q2;
                const double a1 = __shfl_sync(0xffffffffu, A1, o1), a1t = __shfl_sync(0xffffffffu, A1T, o1);
                const double a2 = __shfl_sync(0xffffffffu, A2, o2), a2t = __shfl_sync(0xffffffffu, A2T, o2);
                const int cb = __shfl_sync(0xffffffffu, CB, o1);
                if (e < n) {
                    indices[pos + e] = cb + q2;
                    data[pos + e] = 0.5 * __dadd_rn(__dmul_rn(a1, a2), __dmul_rn(a1t, a2t));
                }
            }
        } else {
            const int pos0 = pos;
            for (int e0 = 0; e0 < n; e0 += 96) {
                int col[3];
                double v[3];
                entries_batch<3>(c, g, e0, lane, n, col, v);
#pragma unroll
                for (int u = 0; u < 3; ++u) {       // entries stay in column order
                    const unsigned m = __ballot_sync(0xffffffffu, col[u] >= 0);
                    if (col[u] >= 0) {
                        const int at = pos + __popc(m & lt);
                        indices[at] = col[u];
                        data[at] = 0.5 * v[u];
                    }
                    pos += __popc(m);
                }
            }
            // a geometrically counted row (near_row) must keep its whole window
            if (lane == 0 && pos - pos0 != n && c.tiles && near_row(c, g))
                atomicOr(c.tiles + TQ_TILE_CTL(c.row_end - c.row_begin) + 8, 1);
        }
    }
}

// generic fill (unequal degrees or no separable factors)
__global__ void k_fill_rows(tq_rowctx c, int32_t* __restrict__ indptr, int32_t* __restrict__ indices,
                            double* __restrict__ data) {
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    for (int r = c.row_begin + blockIdx.x * wpb + (threadIdx.x >> 5); r < c.row_end; r += gridDim.x * wpb) {
        RowGeom g = row_geom(c, r);
        int pos;
        if (c.tiles) {
            pos = tile_offset(c, r, lane);
            if (lane == 0) indptr[r - c.row_begin] = pos;
        } else {
            pos = indptr[r - c.row_begin];
        }
        int n = g.t1 * g.t2;
        const int pos0 = pos;
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
        if (lane == 0 && pos - pos0 != n && c.tiles && near_row(c, g))      // see k_fill_irregular
            atomicOr(c.tiles + TQ_TILE_CTL(c.row_end - c.row_begin) + 8, 1);
    }
}

// both directions in one launch: threads [0, n1) direction 1, [n1, n1+n2) direction 2
// per-line factor positivity; `bad` (optional) counts the non-positive lines
__global__ void k_pos2(tq_rowctx c, int8_t* __restrict__ pos, int* __restrict__ bad = nullptr) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = true;
    if (t < c.n1) {
        for (int j = c.ov_lo1[t]; j <= c.ov_hi1[t]; ++j)
            ok = ok && c.a1[(int64_t)t * (2 * c.p1 + 1) + (j - t + c.p1)] > 0.0 &&
                 c.a1[(int64_t)j * (2 * c.p1 + 1) + (t - j + c.p1)] > 0.0;
        pos[t] = ok;
    } else if (t < c.n1 + c.n2) {
        const int i = t - c.n1;
        for (int j = c.ov_lo2[i]; j <= c.ov_hi2[i]; ++j)
            ok = ok && c.a2[(int64_t)i * (2 * c.p2 + 1) + (j - i + c.p2)] > 0.0 &&
                 c.a2[(int64_t)j * (2 * c.p2 + 1) + (i - j + c.p2)] > 0.0;
        pos[t] = ok;
    }
    if (bad && !ok) atomicAdd(bad, 1);
}

// the cached count pass: the line positivity of this pass against the one
// the cached pass was made with; flags[0] = changed, flags[1] = dirty (the
// cache arrays hold a redo's results), flags[2] = redo guard
__global__ void k_pos2_cmp(tq_rowctx c, int8_t* __restrict__ pos, const int8_t* __restrict__ pos_cached,
                           int* __restrict__ flags) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = true;
    if (t < c.n1) {
        for (int j = c.ov_lo1[t]; j <= c.ov_hi1[t]; ++j)
            ok = ok && c.a1[(int64_t)t * (2 * c.p1 + 1) + (j - t + c.p1)] > 0.0 &&
                 c.a1[(int64_t)j * (2 * c.p1 + 1) + (t - j + c.p1)] > 0.0;
    } else if (t < c.n1 + c.n2) {
        const int i = t - c.n1;
        for (int j = c.ov_lo2[i]; j <= c.ov_hi2[i]; ++j)
            ok = ok && c.a2[(int64_t)i * (2 * c.p2 + 1) + (j - i + c.p2)] > 0.0 &&
                 c.a2[(int64_t)j * (2 * c.p2 + 1) + (i - j + c.p2)] > 0.0;
    }
    if (t < c.n1 + c.n2) {
        pos[t] = ok;
        if ((int8_t)ok != pos_cached[t]) atomicOr(flags, 1);
    }
}

__global__ void k_copy_i32(int32_t* __restrict__ dst, const int32_t* __restrict__ src, int64_t n) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        dst[t] = src[t];
}

__global__ void k_counts_cached_guard(int* __restrict__ flags, int32_t* __restrict__ work,
                                      int32_t* __restrict__ ctl) {
    const int redo = flags[0] | flags[1];
    flags[2] = redo;
    flags[1] = flags[0];        // after a redo the arrays hold this pass's results
    if (redo) {
        work[0] = 0;
        work[1] = 0;
        if (ctl) {
            ctl[0] = 0;
            ctl[1] = 0;
        }
    }
}

// before the redo of a speculative pass (only when some line is not
// positive): the list counters and the first/last list-A words start over
__global__ void k_counts_reset_if_bad(const int* __restrict__ bad, int32_t* __restrict__ work,
                                      int32_t* __restrict__ ctl) {
    if (*bad == 0) return;
    work[0] = 0;
    work[1] = 0;
    if (ctl) {
        ctl[0] = 0;
        ctl[1] = 0;
    }
}

// geometric part of the deep flag: interior, not raw (separable)
__global__ void k_deep_init(tq_rowctx c, const int8_t* __restrict__ fc, int8_t* __restrict__ geo) {
    int64_t total = (int64_t)c.n1 * c.n2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x)
        geo[t] = (fc[t] == TQ_INTERIOR && c.slot[t] < 0) ? 1 : 0;
}

// deep = geometric flag && positive factors in both directions (row i1 per blockIdx.y)
__global__ void k_deep_apply(tq_rowctx c, const int8_t* __restrict__ geo, const int8_t* __restrict__ pos,
                             int8_t* __restrict__ deep) {
    const int i1 = blockIdx.y;
    // only the lines of the context's row block are read (counts, fill)
    if (c.row_end > c.row_begin &&
        (i1 < c.active[c.row_begin] / c.n2 || i1 > c.active[c.row_end - 1] / c.n2)) return;
    const bool p1 = pos[i1];
    const int64_t base = (int64_t)i1 * c.n2;
    for (int i2 = blockIdx.x * blockDim.x + threadIdx.x; i2 < c.n2; i2 += gridDim.x * blockDim.x)
        deep[base + i2] = (p1 && geo[base + i2] && pos[c.n1 + i2]) ? 1 : 0;
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

// pass 1 only needs the deep flags; pass 2 needs the raw rows.  `work`:
// caller scratch of 2 (row_end - row_begin) + 2 ints: [0] = |A|, [1] = |B|,
// list A at work + 2, list B at work + 2 + nrows.
extern "C" int tq_row_counts_deep(tq_rowctx c, int32_t* counts, int32_t* work, void* stream) {
    int nrows = c.row_end - c.row_begin;
    TQ_CUDA(cudaMemsetAsync(work, 0, 2 * sizeof(int32_t), S(stream)));
    if (c.tiles && nrows > 0) TQ_CUDA(cudaMemsetAsync(c.tiles + TQ_TILE_CTL(nrows), 0, 9 * sizeof(int32_t), S(stream)));
    if (nrows <= 0) return TQ_OK;
    k_row_counts_deep<false><<<grid_for(nrows, 256), 256, 0, S(stream)>>>(c, nullptr, nullptr, counts, work + 2, work,
                                                                           work + 2 + nrows, work + 1); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_row_counts_deep");
    return TQ_OK;
}

// as tq_row_counts_deep, from the geometric deep flags of tq_deep_geometry
// and the per-line factor positivity (k_pos2 of a1, a2; c.deep is not read).
// `pos`: caller scratch of n1 + n2 bytes.
extern "C" int tq_row_counts_geo(tq_rowctx c, const int8_t* geo, int8_t* pos, int32_t* counts, int32_t* work,
                                 void* stream) {
    int nrows = c.row_end - c.row_begin;
    TQ_CUDA(cudaMemsetAsync(work, 0, 2 * sizeof(int32_t), S(stream)));
    if (nrows <= 0) return TQ_OK;
    if (!c.a1 || !c.a2) { set_error("tq_row_counts_geo needs the separable factors"); return TQ_EINVAL; }
    if (c.tiles) TQ_CUDA(cudaMemsetAsync(c.tiles + TQ_TILE_CTL(nrows), 0, 9 * sizeof(int32_t), S(stream)));
    k_pos2<<<grid_for(c.n1 + c.n2, 128), 128, 0, S(stream)>>>(c, pos); ::tq::note_launch();
    k_row_counts_deep<true><<<grid_for(nrows, 256), 256, 0, S(stream)>>>(c, geo, pos, counts, work + 2, work,
                                                                          work + 2 + nrows, work + 1); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_row_counts_geo");
    return TQ_OK;
}

// Speculative count pass 1: tq_row_counts_geo with every line's factors
// assumed positive, launched from the cached geometric flags before the fits
// (it needs no factor).  tq_row_counts_verify, after the factors, computes the
// positivity and redoes the pass only if some line is not positive (device-
// side guard: no host decision, graph-capturable).  `bad`: 1 int of scratch.
extern "C" int tq_row_counts_spec(tq_rowctx c, const int8_t* geo, int32_t* counts, int32_t* work, void* stream) {
    int nrows = c.row_end - c.row_begin;
    TQ_CUDA(cudaMemsetAsync(work, 0, 2 * sizeof(int32_t), S(stream)));
    if (nrows <= 0) return TQ_OK;
    if (c.tiles) TQ_CUDA(cudaMemsetAsync(c.tiles + TQ_TILE_CTL(nrows), 0, 9 * sizeof(int32_t), S(stream)));
    k_row_counts_deep<true, true><<<grid_for(nrows, 256), 256, 0, S(stream)>>>(c, geo, nullptr, counts, work + 2,
                                                                                work, work + 2 + nrows, work + 1);
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_row_counts_spec");
    return TQ_OK;
}

extern "C" int tq_row_counts_verify(tq_rowctx c, const int8_t* geo, int8_t* pos, int32_t* bad, int32_t* counts,
                                    int32_t* work, void* stream) {
    int nrows = c.row_end - c.row_begin;
    if (nrows <= 0) return TQ_OK;
    if (!c.a1 || !c.a2) { set_error("tq_row_counts_verify needs the separable factors"); return TQ_EINVAL; }
    TQ_CUDA(cudaMemsetAsync(bad, 0, sizeof(int32_t), S(stream)));
    k_pos2<<<grid_for(c.n1 + c.n2, 128), 128, 0, S(stream)>>>(c, pos, bad); ::tq::note_launch();
    k_counts_reset_if_bad<<<1, 1, 0, S(stream)>>>(bad, work, c.tiles ? c.tiles + TQ_TILE_CTL(nrows) : nullptr);
    ::tq::note_launch();
    k_row_counts_deep<true><<<grid_for(nrows, 256), 256, 0, S(stream)>>>(c, geo, pos, counts, work + 2, work,
                                                                          work + 2 + nrows, work + 1, bad);
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_row_counts_verify");
    return TQ_OK;
}

extern "C" int tq_row_counts_cached(tq_rowctx c, const int8_t* geo, int8_t* pos, const int8_t* pos_cached,
                                    int32_t* flags, int32_t* counts, int32_t* work, const int32_t* tiles0,
                                    void* stream) {
    int nrows = c.row_end - c.row_begin;
    if (nrows <= 0) return TQ_OK;
    if (!c.a1 || !c.a2 || !c.tiles) { set_error("tq_row_counts_cached needs the separable factors and tiles"); return TQ_EINVAL; }
    cudaStream_t st = S(stream);
    // (a kernel copy: a device-to-device memcpy node in a captured graph
    // goes to a copy engine and sits on the pass's critical path)
    const int64_t nt = TQ_TILE_INTS(nrows);
    k_copy_i32<<<grid_for(nt, 256), 256, 0, st>>>(c.tiles, tiles0, nt); ::tq::note_launch();
    TQ_CUDA(cudaMemsetAsync(flags, 0, sizeof(int32_t), st));
    k_pos2_cmp<<<grid_for(c.n1 + c.n2, 128), 128, 0, st>>>(c, pos, pos_cached, flags); ::tq::note_launch();
    k_counts_cached_guard<<<1, 1, 0, st>>>(flags, work, c.tiles + TQ_TILE_CTL(nrows)); ::tq::note_launch();
    // guarded redo (a no-op unless the positivity changed): a capped grid
    k_row_counts_deep<true><<<std::min(grid_for(nrows, 256), kSms * 8), 256, 0, st>>>(c, geo, pos, counts, work + 2,
                                                                                      work, work + 2 + nrows,
                                                                                      work + 1, flags + 2);
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("tq_row_counts_cached");
    return TQ_OK;
}

extern "C" int tq_row_counts_rest(tq_rowctx c, int32_t* counts, const int32_t* work, void* stream) {
    if (c.row_end <= c.row_begin) return TQ_OK;
    k_row_counts_list<<<kSms * 16, 256, 0, S(stream)>>>(c, counts, work + 2, work); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_row_counts_list");
    return TQ_OK;
}

extern "C" int64_t tq_list_record_bytes(void) { return (int64_t)sizeof(ListRec); }

// the geometry records of list A (work: the count passes' lists; rec:
// (row_end - row_begin) * tq_list_record_bytes() bytes)
extern "C" int tq_list_geometry(tq_rowctx c, const int32_t* work, void* rec, void* stream) {
    if (c.row_end <= c.row_begin) return TQ_OK;
    k_list_geometry<<<kSms * 8, 256, 0, S(stream)>>>(c, work + 2, work, static_cast<ListRec*>(rec));
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_list_geometry");
    return TQ_OK;
}

// tq_row_counts_rest from the records of tq_list_geometry
extern "C" int tq_row_counts_rest_rec(tq_rowctx c, int32_t* counts, const int32_t* work, const void* rec,
                                      void* stream) {
    if (c.row_end <= c.row_begin) return TQ_OK;
    k_row_counts_list<<<kSms * 16, 256, 0, S(stream)>>>(c, counts, work + 2, work,
                                                        static_cast<const ListRec*>(rec));
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_row_counts_list");
    return TQ_OK;
}

extern "C" int tq_row_counts(tq_rowctx c, int32_t* counts, void* stream) {
    int nrows = c.row_end - c.row_begin;
    if (nrows <= 0) return TQ_OK;
    int32_t* work = nullptr;
    TQ_CUDA(cudaMallocAsync(&work, sizeof(int32_t) * (2 * (int64_t)nrows + 2), S(stream)));
    int rc = tq_row_counts_deep(c, counts, work, stream);
    if (!rc) rc = tq_row_counts_rest(c, counts, work, stream);
    TQ_CUDA(cudaFreeAsync(work, S(stream)));
    return rc;
}

extern "C" int tq_fill_rows(tq_rowctx c, const int32_t* indptr, int32_t* indices, double* data,
                            void* stream) {
    int nrows = c.row_end - c.row_begin;
    if (nrows <= 0) return TQ_OK;
    if (c.tiles) { set_error("tq_fill_rows reads a complete indptr (tile mode: tq_fill_fast + tq_fill_listed)"); return TQ_EINVAL; }
    int32_t* ip = const_cast<int32_t*>(indptr);   // read only here
    int P = (c.p1 == c.p2 && c.a1 && c.deep) ? c.p1 : 0;
    int* irr = nullptr;   // [0] = count, [1..] = rows for the irregular kernel
    cudaStream_t st = S(stream);
    auto launch = [&](auto kern, auto kirr, size_t per_warp) -> int {
        // launch configuration cached per kernel instance (host calls kept
        // off the per-pass path)
        // (per device: the shared-memory attribute is per-device state)
        static int cached_wpb[kMaxP + 1][16] = {}, cached_per_sm[kMaxP + 1][16] = {};
        int dev = 0;
        TQ_CUDA(cudaGetDevice(&dev));
        int wpb = cached_wpb[P][dev & 15];
        int per_sm = cached_per_sm[P][dev & 15];
        if (!wpb) {
            wpb = 8;
            while (per_warp * wpb > 160 * 1024 && wpb > 1) wpb /= 2;
            TQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(per_warp * wpb)));
            TQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * wpb, per_warp * wpb));
            cached_wpb[P][dev & 15] = wpb;
            cached_per_sm[P][dev & 15] = per_sm;
        }
        const size_t shm = per_warp * wpb;
        const int64_t full = (int64_t)kSms * std::max(per_sm, 1);
        const int grid = (int)std::min<int64_t>((nrows + wpb * kWarpRows - 1) / (wpb * kWarpRows), full);
        TQ_CUDA(cudaMallocAsync(&irr, sizeof(int) * (nrows + 1), st));
        TQ_CUDA(cudaMemsetAsync(irr, 0, sizeof(int), st));
        kern<<<grid, 32 * wpb, shm, st>>>(c, ip, indices, data, irr + 1, irr, 0); ::tq::note_launch();
        kirr<<<kSms * 8, 256, 0, st>>>(c, ip, indices, data, irr + 1, irr, nullptr, nullptr); ::tq::note_launch();
        TQ_CUDA(cudaFreeAsync(irr, st));
        return TQ_OK;
    };
    int rc = TQ_OK;
    switch (P) {
#define CASE(Q) case Q: rc = launch(k_fill_tiles<Q>, k_fill_irregular<Q>, fill_slice_bytes<Q>()); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
        default: {
            int grid = (int)std::min<int64_t>((nrows + 7) / 8, (int64_t)kSms * 32);
            k_fill_rows<<<grid, 256, 0, S(stream)>>>(c, ip, indices, data); ::tq::note_launch();
        }
    }
    if (rc) return rc;
    TQ_LAUNCH_CHECK("k_fill_rows");
    return TQ_OK;
}

// Split fill (used with the lists of tq_row_counts_deep): runs of fast rows
// by warp tiles, and the listed rows by the row-parallel kernel; the two
// write disjoint rows and may run concurrently on different streams.
template <int P>
static int fill_fast_launch(const tq_rowctx& c, int32_t* indptr, int32_t* indices, double* data,
                            cudaStream_t st, int part = 0, int blocks_per_sm = 0) {
    // cached per device (the shared-memory attribute is per-device state)
    static int cached_wpb_d[16] = {}, cached_per_sm_d[16] = {};
    int dev = 0;
    TQ_CUDA(cudaGetDevice(&dev));
    int& cached_wpb = cached_wpb_d[dev & 15];
    int& cached_per_sm = cached_per_sm_d[dev & 15];
    const size_t per_warp = fill_slice_bytes<P>();
    if (!cached_wpb) {
        // warps per block maximising resident warps per SM (shared memory bound)
        int smem_max = 0;
        TQ_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        TQ_CUDA(cudaFuncSetAttribute(k_fill_tiles<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
        int best_w = 0;
        for (int wpb = 1; wpb <= 8; ++wpb) {
            if (per_warp * wpb > (size_t)smem_max) break;
            int per_sm = 0;
            TQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fill_tiles<P>, 32 * wpb, per_warp * wpb));
            if (per_sm * wpb > best_w || (per_sm * wpb == best_w && wpb > cached_wpb)) {
                best_w = per_sm * wpb;
                cached_wpb = wpb;
                cached_per_sm = per_sm;
            }
        }
        if (!cached_wpb) { set_error("fill staging does not fit in shared memory"); return TQ_EINVAL; }
    }
    const int wpb = cached_wpb, nrows = c.row_end - c.row_begin;
    int per_sm = std::max(cached_per_sm, 1);
    if (blocks_per_sm > 0) per_sm = std::min(per_sm, blocks_per_sm);
    const int64_t full = (int64_t)kSms * per_sm;
    const int grid = (int)std::min<int64_t>((nrows + wpb * kWarpRows - 1) / (wpb * kWarpRows), full);
    k_fill_tiles<P><<<grid, 32 * wpb, per_warp * wpb, st>>>(c, indptr, indices, data, nullptr, nullptr, part);
    ::tq::note_launch();
    return TQ_OK;
}

static int fill_P(const tq_rowctx& c) { return (c.p1 == c.p2 && c.a1 && c.deep) ? c.p1 : 0; }

extern "C" int tq_fill_fast(tq_rowctx c, int32_t* indptr, int32_t* indices, double* data, void* stream) {
    const int nrows = c.row_end - c.row_begin;
    if (nrows <= 0) return TQ_OK;
    int rc = TQ_OK;
    switch (fill_P(c)) {
#define CASE(Q) case Q: rc = fill_fast_launch<Q>(c, indptr, indices, data, S(stream)); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
        default: {   // no separable factors: every row through the generic fill
            int grid = (int)std::min<int64_t>((nrows + 7) / 8, (int64_t)kSms * 32);
            k_fill_rows<<<grid, 256, 0, S(stream)>>>(c, indptr, indices, data); ::tq::note_launch();
        }
    }
    if (rc) return rc;
    TQ_LAUNCH_CHECK("tq_fill_fast");
    return TQ_OK;
}

extern "C" int tq_fill_fast_part(tq_rowctx c, int32_t* indptr, int32_t* indices, double* data, int32_t part,
                                 int32_t blocks_per_sm, void* stream) {
    const int nrows = c.row_end - c.row_begin;
    if (nrows <= 0) return TQ_OK;
    if (part < 0 || part > 2 || (part && !c.tiles)) { set_error("fill part %d needs tile mode", part); return TQ_EINVAL; }
    const int P = fill_P(c);
    if (P == 0) {            // generic fill: every row in part 0 / 2
        if (part == 1) return TQ_OK;
        return tq_fill_fast(c, indptr, indices, data, stream);
    }
    int rc = TQ_OK;
    switch (P) {
#define CASE(Q) case Q: rc = fill_fast_launch<Q>(c, indptr, indices, data, S(stream), part, blocks_per_sm); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
    }
    if (rc) return rc;
    TQ_LAUNCH_CHECK("tq_fill_fast_part");
    return TQ_OK;
}

extern "C" int tq_fill_listed(tq_rowctx c, const int32_t* indptr, int32_t* indices, double* data,
                              const int32_t* work, void* stream) {
    const int nrows = c.row_end - c.row_begin;
    if (nrows <= 0) return TQ_OK;
    switch (fill_P(c)) {
#define CASE(Q) case Q: k_fill_irregular<Q><<<kSms * 8, 256, 0, S(stream)>>>(c, indptr, indices, data, work + 2, \
            work, work + 2 + nrows, work + 1); ::tq::note_launch(); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
        default: return TQ_OK;   // tq_fill_fast covered every row
    }
    TQ_LAUNCH_CHECK("tq_fill_listed");
    return TQ_OK;
}

// geometric part (cacheable per row plan): interior && not raw && no raw row in the window
extern "C" int tq_deep_geometry(tq_rowctx c, const int8_t* func_class, const int32_t* raw_rows, int32_t nraw,
                                int8_t* geo, void* stream) {
    int64_t nf = (int64_t)c.n1 * c.n2;
    if (nf == 0) return TQ_OK;
    k_deep_init<<<grid_for(nf, 256), 256, 0, S(stream)>>>(c, func_class, geo); ::tq::note_launch();
    if (nraw > 0) { k_deep_clear<<<grid_for(nraw, 128), 128, 0, S(stream)>>>(c, raw_rows, nraw, geo); ::tq::note_launch(); }
    TQ_LAUNCH_CHECK("deep geometry");
    return TQ_OK;
}

// per pass: deep = geo && positive direction factors (a1, a2 of the context)
extern "C" int tq_deep_apply(tq_rowctx c, const int8_t* geo, int8_t* deep, void* stream) {
    int64_t nf = (int64_t)c.n1 * c.n2;
    if (nf == 0) return TQ_OK;
    if (!c.a1 || !c.a2) {
        TQ_CUDA(cudaMemsetAsync(deep, 0, nf, S(stream)));
        return TQ_OK;
    }
    int8_t* pos = nullptr;
    TQ_CUDA(cudaMallocAsync(&pos, c.n1 + c.n2, S(stream)));
    k_pos2<<<grid_for(c.n1 + c.n2, 128), 128, 0, S(stream)>>>(c, pos); ::tq::note_launch();
    dim3 grid((unsigned)std::min<int64_t>((c.n2 + 255) / 256, 4), (unsigned)c.n1);
    k_deep_apply<<<grid, 256, 0, S(stream)>>>(c, geo, pos, deep); ::tq::note_launch();
    TQ_LAUNCH_CHECK("deep apply");
    TQ_CUDA(cudaFreeAsync(pos, S(stream)));
    return TQ_OK;
}

extern "C" int tq_deep_flags(tq_rowctx c, const int8_t* func_class, const int32_t* raw_rows, int32_t nraw,
                             int8_t* deep, void* stream) {
    if (!c.a1 || !c.a2) return tq_deep_apply(c, nullptr, deep, stream);
    int rc = tq_deep_geometry(c, func_class, raw_rows, nraw, deep, stream);   // in place: geo -> deep
    return rc ? rc : tq_deep_apply(c, deep, deep, stream);
}
