// The all-raw formation path (c != 1, or the element-Gauss `reference`
// strategy): every active row is a raw row, stored in the planes layout
// raw[o * ld + s] -- window entry o = (j1 - i1 + p1)(2p2 + 1) + (j2 - i2 + p2)
// of the row with storage index s = active index - raw_base.  The planes of
// consecutive rows are contiguous, so both kernels here move whole 128-byte
// lines per warp instruction.
//
//  tq_sf_strips  <- sum_factor_row (src/assembly.py:218-252) for the interior
//                   rows of the c != 1 BOX plan (_interior_rows_batched,
//                   src/assembly.py:409-449): rows of one direction-1 line
//                   with consecutive i2 form a strip that shares the
//                   direction-1 contraction of the coefficient grid.
//  tq_planes_csr <- _Run.finish (src/assembly.py:400-404): 0.5 (M + M^T),
//                   exact-zero drop and sorted columns, in ONE pass (tile
//                   counts published with a decoupled look-back scan).
#include <limits.h>

#include "common.cuh"

namespace tq {

__device__ __forceinline__ double colloc_val(const tq_ruleset& s, int p, int k, int j) {
    const int r = j - s.first[k];
    return (r >= 0 && r <= p) ? s.vals[(int64_t)k * (p + 1) + r] : 0.0;
}

// ---------------------------------------------------------------------------
// Weighted collocation tables of the standard rules, once per pass:
// BW_d[i][k][o] = colloc_d(k0_d(i) + k, i - p + o) w_d(i)[k] for k < the row's
// length and j = i - p + o in the overlap range of i, else 0; i < n_d,
// k < nmax_d, o < WP (the strips' padded window).  *status |= 2 when a rule
// row is longer than nmax_d.
// ---------------------------------------------------------------------------
__host__ __device__ inline int bw_wp(int p) { return 3 * ((2 * p + 3) / 3); }
// doubles per table row (one test function): even, so rows start 16-byte aligned
__host__ __device__ inline int bw_row(int p, int nmax) { return (nmax * bw_wp(p) + 1) & ~1; }

__global__ void k_bw_tables(tq_rawctx c, double* __restrict__ bw1, double* __restrict__ bw2,
                            int* __restrict__ status) {
    const int WP = bw_wp(c.p1), R1 = bw_row(c.p1, c.nmax1), R2 = bw_row(c.p2, c.nmax2);
    const int64_t t1 = (int64_t)c.n1 * R1, total = t1 + (int64_t)c.n2 * R2;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const bool d1 = q < t1;
        const int64_t e = d1 ? q : q - t1;
        const int nmax = d1 ? c.nmax1 : c.nmax2, p = d1 ? c.p1 : c.p2, RS = d1 ? R1 : R2;
        const tq_ruleset& R = d1 ? c.sets1[0] : c.sets2[0];
        const int i = (int)(e / RS), rem = (int)(e - (int64_t)i * RS);
        const int k = rem / WP, o = rem - k * WP, j = i - p + o;
        const int k0 = R.rules.k0[i];
        const int len = k0 >= 0 ? (int)(R.rules.wptr[i + 1] - R.rules.wptr[i]) : 0;
        if (rem == 0 && len > nmax) atomicOr(status, 2);
        double v = 0.0;
        if (k < len && k < nmax && o <= 2 * p && j >= (d1 ? c.ov_lo1 : c.ov_lo2)[i] &&
            j <= (d1 ? c.ov_hi1 : c.ov_hi2)[i])
            v = colloc_val(R, p, k0 + k, j) * R.rules.w[R.rules.wptr[i] + k];
        (d1 ? bw1 : bw2)[e] = v;
    }
}

// ---------------------------------------------------------------------------
// Strips.  One strip = up to TS rows (i1, i20 + t) of the c != 1 BOX plan
// whose box is their whole support (standard rules in both directions).
// With B_d = the BW tables above and the coefficient grid G on the WQ points:
//   stage A (shared by the strip):  X[u][o1] = sum_k1 B1[k1][o1] G[k1][u0 + u]
//            over the union u of the rows' direction-2 point windows;
//   stage B (per row t):            M_t[o1][o2] = sum_kk X[k0_t - u0 + kk][o1] B2_t[kk][o2].
// The same products as sum_factor_row with the direction-1 contraction done
// first (one stage-A pass per strip instead of one direction-2 pass per row:
// about half the multiply-adds of the row-by-row form).  A thread of stage B
// owns a BA x BA register tile of one row's block (a 3 x 3 grid of tiles per
// row); lanes run over the strip's rows, so every store is a run of 16
// consecutive storage slots of one plane.
// strips: nstrips x (2 + TS) ints: i1, i20, storage index of row t (or -1).
// ---------------------------------------------------------------------------
constexpr int kStripRows = 16;

// shared row stride of the B2 stage: an odd number of 16-byte units (the
// rows' 16 lanes spread over the banks; rows stay 16-byte aligned)
__host__ __device__ inline int strip_b2_stride(int p, int n2m) {
    const int m = (n2m * bw_wp(p) + 1) / 2;
    return 2 * (m | 1);
}

// row stride of the coefficient stage: even (16-byte aligned rows) with a
// slot of slack for an odd first column
__host__ __device__ inline int strip_gs_stride(int nu_max) { return (nu_max + 3) & ~1; }

// shared stage offsets (doubles): two buffers of B1 | GS (stage A's operands,
// prefetched one strip ahead), ONE B2 stage (refilled while stage A of the
// next strip runs), then X; the 16-byte copy targets start at even offsets
struct StripSmem {
    int gs, abuf, b2, x, total;
    // b2cap > 0: the B2 stage holds the rows packed (each row its own odd
    // number of 16-byte units, strip_b2_stride of its length), b2cap doubles
    __host__ __device__ StripSmem(int p, int n1m, int n2m, int nu_max, int ts, int b2cap = 0) {
        const int WP = bw_wp(p), WPI = WP | 1;
        gs = (n1m * WP + 1) & ~1;
        abuf = gs + n1m * strip_gs_stride(nu_max);
        b2 = 2 * abuf;
        x = b2 + (b2cap > 0 ? b2cap : ts * strip_b2_stride(p, n2m));
        total = x + nu_max * WPI;
    }
};

__host__ __device__ inline size_t strip_smem_doubles(int p, int n1m, int n2m, int nu_max, int ts, int b2cap = 0) {
    return (size_t)StripSmem(p, n1m, n2m, nu_max, ts, b2cap).total;
}

__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(sdst)),
                 "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(sdst)),
                 "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void fence_proxy_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// one-dimensional TMA bulk copies into shared memory, completing on an mbarrier
__device__ __forceinline__ unsigned sptr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sptr(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
    unsigned done;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(sptr(b)), "r"(phase) : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sptr(sdst)), "l"(gsrc), "r"(bytes), "r"(sptr(b)) : "memory");
}

// mbarrier arrive (no transaction bytes)
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sptr(b)) : "memory");
}
// named barrier of the consumer warps
__device__ __forceinline__ void consumers_sync(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }

template <int TS>
struct StripHdr {
    int k0[TS], n2[TS], st[TS], off2[TS];     // off2: B2 row offset in 16-byte units
    int i1, i20, u0, nu, k01, n1, sh, pad;
};

// Warp-specialised: warp CW (the producer) reads strip s + G's header and
// stages its stage-A operands (TMA bulk copies of the B1 table row and the
// coefficient rows) into the free A buffer while the consumer warps
// 0..CW-1 compute strip s; the B2 rows of a strip go to the single B2 stage
// as soon as the consumers are done with the previous strip's stage B, so
// they arrive while stage A of the strip runs (one B2 stage instead of two:
// the long-rule classes fit two blocks per SM).  full_a[b] / empty_a[b]
// hand the A buffers over, full_b / empty_b the B2 stage.  n1m, n2m: the
// rule-row capacity of the stage (the strips of one launch have shorter
// rows than the tables' stride c.nmax1/2 when the boundary strips go to a
// second launch).
template <int P, int TS>
__global__ void __launch_bounds__(32 * ((TS * 9 + 31) / 32) + 32) k_sf_strips(
    tq_rawctx c, const int32_t* __restrict__ strips, int nstrips, int n1m, int n2m, int nu_max, int b2cap,
    const double* __restrict__ bw1, const double* __restrict__ bw2, int* __restrict__ status) {
    constexpr int W = 2 * P + 1, BA = (W + 2) / 3, WP = 3 * BA, WPI = WP | 1, NB = TS * 9;
    constexpr int CW = (NB + 31) / 32, NC = 32 * CW;      // consumer warps / threads
    extern __shared__ __align__(128) double sm[];       // 16-byte aligned bulk-copy targets
    const StripSmem L(P, n1m, n2m, nu_max, TS, b2cap);
    const int SB = strip_b2_stride(P, n2m), GL = strip_gs_stride(nu_max);
    double* X = sm + L.x;                 // [nu][WPI]
    double* B2 = sm + L.b2;               // [TS][SB]
    __shared__ StripHdr<TS> H[2];
    __shared__ __align__(8) uint64_t full_a[2], empty_a[2], full_b, empty_b;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const tq_ruleset R1 = c.sets1[0], R2 = c.sets2[0];
    const double* __restrict__ G = c.grids[0];
    const int ldG = R2.lay.npts;
    if (tid == 0) {
        mbar_init(&full_a[0], 1);
        mbar_init(&full_a[1], 1);
        mbar_init(&empty_a[0], 1);
        mbar_init(&empty_a[1], 1);
        mbar_init(&full_b, 1);
        mbar_init(&empty_b, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == CW) {
        // ---------------- producer
        const bool bulk = (ldG & 1) == 0;     // coefficient rows 16-byte aligned
        for (int it = 0, s = blockIdx.x; s < nstrips; s += gridDim.x, ++it) {
            const int b = it & 1;
            if (it >= 2) mbar_wait(&empty_a[b], ((it >> 1) & 1) ^ 1);
            StripHdr<TS>& h = H[b];
            const int32_t* st = strips + (int64_t)s * (2 + TS);
            const int i1 = st[0], i20 = st[1];
            int k0 = -1, n2 = 0, sidx = -1;
            if (lane < TS) {
                sidx = st[2 + lane];
                if (sidx >= 0) {
                    const int i2 = i20 + lane;
                    k0 = R2.rules.k0[i2];
                    n2 = k0 >= 0 ? (int)(R2.rules.wptr[i2 + 1] - R2.rules.wptr[i2]) : 0;
                }
                h.k0[lane] = k0;
                h.n2[lane] = n2;
                h.st[lane] = sidx;
            }
            // B2 stage offsets: packed rows (b2cap > 0) or a fixed stride
            const int alloc = lane < TS ? (b2cap > 0 ? (n2 > 0 ? strip_b2_stride(P, n2) : 0) : SB) : 0;
            int incl = alloc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane < TS) h.off2[lane] = (incl - alloc) >> 1;     // allocations are even
            int lo = n2 > 0 ? k0 : INT_MAX, hi = n2 > 0 ? k0 + n2 : INT_MIN, bad = n2 > n2m;
            lo = __reduce_min_sync(0xffffffffu, lo);
            hi = __reduce_max_sync(0xffffffffu, hi);
            bad = __reduce_or_sync(0xffffffffu, bad);
            if (b2cap > 0 && __shfl_sync(0xffffffffu, incl, 31) > b2cap) bad = 1;
            const int k01 = R1.rules.k0[i1];
            int n1 = k01 >= 0 ? (int)(R1.rules.wptr[i1 + 1] - R1.rules.wptr[i1]) : 0;
            int nu = hi > lo ? hi - lo : 0;
            if (nu > nu_max || n1 > n1m || bad) {      // workspace bound broken: flagged, never silent
                if (lane == 0) atomicOr(status, 1);
                nu = 0;
            }
            if (nu == 0) n1 = 0;
            const int sh = bulk ? (lo & 1) : 0;
            double* B1 = sm + b * L.abuf;
            double* GS = B1 + L.gs;
            if (n1 > 0 && !bulk) {        // odd grid stride: the coefficient rows through registers
                for (int k = 0; k < n1; ++k)
                    for (int u = lane; u < nu; u += 32) GS[k * GL + u] = __ldg(G + (int64_t)(k01 + k) * ldG + lo + u);
                __threadfence_block();
            }
            __syncwarp();
            if (lane == 0) {
                h.i1 = i1;
                h.i20 = i20;
                h.u0 = lo;
                h.nu = nu;
                h.k01 = k01;
                h.n1 = n1;
                h.sh = sh;
                if (n1 > 0) {
                    const unsigned b1b = 8u * ((n1 * WP + 1) & ~1);
                    const int ua = lo & ~1, gl = (sh + nu + 1) & ~1;
                    fence_proxy_async_shared();       // the buffer's earlier reads precede these writes
                    mbar_expect_tx(&full_a[b], b1b + (bulk ? 8u * n1 * gl : 0u));
                    bulk_g2s(B1, bw1 + (int64_t)i1 * bw_row(P, c.nmax1), b1b, &full_a[b]);
                    if (bulk)
                        for (int k = 0; k < n1; ++k)
                            bulk_g2s(GS + k * GL, G + (int64_t)(k01 + k) * ldG + ua, 8u * gl, &full_a[b]);
                } else {
                    mbar_arrive(&full_a[b]);
                }
                // the B2 rows once the previous strip's stage B is done
                if (it >= 1) mbar_wait(&empty_b, (it - 1) & 1);
                if (n1 > 0) {
                    const int nrow = min(TS, c.n2 - i20), R2s = bw_row(P, c.nmax2);
                    // the rows' own lengths (packed) or the class capacity
                    unsigned tot = 0;
                    for (int t = 0; t < nrow; ++t)
                        tot += b2cap > 0 ? 8u * ((h.n2[t] * WP + 1) & ~1) : 8u * ((n2m * WP + 1) & ~1);
                    fence_proxy_async_shared();
                    mbar_expect_tx(&full_b, tot);
                    for (int t = 0; t < nrow; ++t) {
                        const unsigned bt = b2cap > 0 ? 8u * ((h.n2[t] * WP + 1) & ~1) : 8u * ((n2m * WP + 1) & ~1);
                        if (bt) bulk_g2s(B2 + 2 * h.off2[t], bw2 + (int64_t)(i20 + t) * R2s, bt, &full_b);
                    }
                    if (!tot) mbar_arrive(&full_b);
                } else {
                    mbar_arrive(&full_b);
                }
            }
            __syncwarp();
        }
        return;
    }
    // ---------------- consumers
    for (int it = 0, s = blockIdx.x; s < nstrips; s += gridDim.x, ++it) {
        const int b = it & 1;
        mbar_wait(&full_a[b], (it >> 1) & 1);
        const StripHdr<TS>& h = H[b];
        const double* B1 = sm + b * L.abuf;
        const double* GS = B1 + L.gs;
        const int u0 = h.u0, nu = h.nu, n1 = h.n1, sh = h.sh;
        // stage A: lanes run over u (conflict-free column reads of GS; the B1
        // reads broadcast)
        for (int q = tid; q < 3 * nu; q += NC) {
            const int ob = q / nu, u = q - ob * nu;
            double acc[BA];
#pragma unroll
            for (int i = 0; i < BA; ++i) acc[i] = 0.0;
            for (int k1 = 0; k1 < n1; ++k1) {
                const double g = GS[k1 * GL + sh + u];
                const double* bb = B1 + k1 * WP + ob * BA;
#pragma unroll
                for (int i = 0; i < BA; ++i) acc[i] = fma(bb[i], g, acc[i]);
            }
#pragma unroll
            for (int i = 0; i < BA; ++i) X[u * WPI + ob * BA + i] = acc[i];
        }
        consumers_sync(NC);
        mbar_wait(&full_b, it & 1);
        // stage B: thread (t = lane row, a, b) owns rows a*BA.., columns b*BA.. of row t
        if (tid < NB) {
            const int t = tid % TS, ab = tid / TS, a = ab / 3, bq = ab - a * 3;
            const int n2 = n1 > 0 ? h.n2[t] : 0, sidx = h.st[t];
            double acc[BA][BA];
#pragma unroll
            for (int i = 0; i < BA; ++i)
#pragma unroll
                for (int j = 0; j < BA; ++j) acc[i][j] = 0.0;
            const double* x = X + (n2 > 0 ? h.k0[t] - u0 : 0) * WPI + a * BA;
            const double* y = B2 + 2 * h.off2[t] + bq * BA;      // 16-byte aligned: vector loads
            for (int kk = 0; kk < n2; ++kk) {
                double xv[BA], yv[BA];
#pragma unroll
                for (int i = 0; i < BA; ++i) {
                    xv[i] = x[kk * WPI + i];
                    yv[i] = y[kk * WP + i];
                }
#pragma unroll
                for (int i = 0; i < BA; ++i)
#pragma unroll
                    for (int j = 0; j < BA; ++j) acc[i][j] = fma(xv[i], yv[j], acc[i][j]);
            }
            if (sidx >= 0) {
                double* dst = c.raw + sidx;
#pragma unroll
                for (int i = 0; i < BA; ++i)
#pragma unroll
                    for (int j = 0; j < BA; ++j) {
                        const int o1 = a * BA + i, o2 = bq * BA + j;
                        if (o1 < W && o2 < W) dst[(int64_t)(o1 * W + o2) * c.raw_ld] = acc[i][j];
                    }
            }
        }
        consumers_sync(NC);          // X, the B2 stage and A buffer b are free
        if (tid == 0) {
            mbar_arrive(&empty_b);
            mbar_arrive(&empty_a[b]);
        }
    }
}

// ---------------------------------------------------------------------------
// Symmetrise / zero-drop / CSR in one pass over the planes.  A block takes
// 16-row tiles in ticket order.  Phase 1: half-warp lane = row, half-warp h
// of warp w = window lines o1 = 2w + h, 2w + h + 16, ..: M_ij + M_ji from two coalesced plane reads (the row's
// own plane o and the partner's mirrored plane T-1-o), kept columns into a
// [row][entry] shared stage.  Phase 2: per-row counts, the tile total
// published and the tile's offset found by a decoupled look-back over the
// earlier tiles' words (flag 1 = aggregate, 2 = inclusive prefix).  Phase 3:
// warp per row, ballot-compacted contiguous stores of the kept entries.
// ctl: [0] tile ticket, [1] nnz, [2] flags (1 = nnz differs from `expect`,
// 2 = capacity exceeded; nothing past `cap` is written).
// ---------------------------------------------------------------------------
constexpr int kPlThreadsPerRow = 16;      // block = 16 threads per tile row (256 at 16 rows, 128 at 8)

// the look-back words carry flag and value in one 64-bit word, so relaxed
// single-copy-atomic accesses suffice (no other data is published with them;
// an acquire load would invalidate L1 on every spin)
__device__ __forceinline__ void lb_store(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long lb_pack(unsigned flag, unsigned v) {
    return ((unsigned long long)flag << 32) | v;
}

__device__ __forceinline__ int pl_row_of(const tq_rowctx& c, int idx) { return idx / c.n2; }

template <int P, int kPlTile>
__global__ void __launch_bounds__(kPlThreadsPerRow * kPlTile, 64 / kPlTile) k_planes_csr(tq_rowctx c, int32_t raw_base, int32_t* __restrict__ indptr,
                                                            int32_t* __restrict__ indices, double* __restrict__ data,
                                                            int64_t cap, unsigned long long* __restrict__ state,
                                                            int32_t* __restrict__ ctl, int64_t expect) {
    constexpr int W = 2 * P + 1, T = W * W, kPlThreads = kPlThreadsPerRow * kPlTile, NW = kPlThreads / 32;
    extern __shared__ double sm[];
    double* sv = sm;                                            // [kPlTile][T]
    int* sc = reinterpret_cast<int*>(sv + kPlTile * T);        // [kPlTile][T]
    __shared__ int s_tile, s_off[kPlTile], s_cnt[kPlTile];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int n = c.row_end - c.row_begin, nt = (n + kPlTile - 1) / kPlTile;
    const double* __restrict__ raw = c.raw;
    const int64_t ld = c.raw_ld;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(ctl, 1);
        __syncthreads();
        const int tile = s_tile;
        if (tile >= nt) break;
        // ---- phase 1
        {
            const int tr = lane & (kPlTile - 1), half = lane / kPlTile;
            const int r = c.row_begin + tile * kPlTile + tr;
            const bool have = r < c.row_end;
            int i1 = 0, i2 = 0, jl1 = 1, jh1 = 0, jl2 = 1, jh2 = 0;
            if (have) {
                const int idx = __ldg(c.active + r);
                i1 = pl_row_of(c, idx);
                i2 = idx - i1 * c.n2;
                jl1 = __ldg(c.ov_lo1 + i1);
                jh1 = __ldg(c.ov_hi1 + i1);
                jl2 = __ldg(c.ov_lo2 + i2);
                jh2 = __ldg(c.ov_hi2 + i2);
            }
            const int si = r - raw_base;
            // entries o = hw, hw + 16, .. of the row (hw = the half-warp's
            // index): every half-warp gets ceil(T / 16) entries, loaded in
            // chunks of CH (column loads, then the partners' values)
            constexpr int SUB = 32 / kPlTile, NH = SUB * NW, PER = (T + NH - 1) / NH;
            constexpr int NCH = (PER + 7) / 8, CH = (PER + NCH - 1) / NCH;
            const int hw = SUB * warp + half;
            // window-offset bounds of this row (j in the overlap range)
            const int o1lo = jl1 - i1 + P, o1hi = jh1 - i1 + P, o2lo = jl2 - i2 + P, o2hi = jh2 - i2 + P;
            const int* colbase = c.col_of + ((int64_t)(i1 - P) * c.n2 + (i2 - P));
            const double* own = raw + si;
            const double* part = raw + (int64_t)(T - 1) * ld - raw_base;
#pragma unroll
            for (int k0 = 0; k0 < PER; k0 += CH) {
                int col[CH];
                double vi[CH];
#pragma unroll
                for (int k = 0; k < CH; ++k) {
                    const int o = hw + (k0 + k) * NH;
                    const int o1 = o / W, o2 = o - o1 * W;
                    const bool ok = k0 + k < PER && o < T && have && o1 >= o1lo && o1 <= o1hi && o2 >= o2lo &&
                                    o2 <= o2hi;
                    col[k] = ok ? __ldg(colbase + o1 * c.n2 + o2) : -1;
                    vi[k] = ok ? __ldg(own + (int64_t)o * ld) : 0.0;
                }
#pragma unroll
                for (int k = 0; k < CH; ++k) {
                    const int o = hw + (k0 + k) * NH;
                    int cl = col[k];
                    double v = 0.0;
                    if (cl >= 0) {
                        v = __dadd_rn(vi[k], __ldg(part - (int64_t)o * ld + cl));
                        if (v == 0.0) cl = -1;
                    }
                    if (k0 + k < PER && o < T) {
                        sv[tr * T + o] = 0.5 * v;
                        sc[tr * T + o] = cl;
                    }
                }
            }
        }
        __syncthreads();
        // ---- phase 2
        for (int t = warp; t < kPlTile; t += NW) {
            int cnt = 0;
            for (int o = lane; o < T; o += 32) cnt += sc[t * T + o] >= 0;
            cnt = __reduce_add_sync(0xffffffffu, cnt);
            if (lane == 0) s_cnt[t] = cnt;
        }
        __syncthreads();
        if (warp == 0) {
            const int cnt = lane < kPlTile ? s_cnt[lane] : 0;
            int incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += y;
            }
            const int agg = __shfl_sync(0xffffffffu, incl, 31);
            if (lane == 0) lb_store(state + tile, lb_pack(tile == 0 ? 2u : 1u, (unsigned)agg));
            int excl = 0;
            if (tile > 0) {
                for (int j = tile - 1;; j -= 32) {
                    const int jj = j - lane;
                    unsigned long long w = lb_pack(2u, 0u);
                    if (jj >= 0) {
                        do {
                            w = lb_load(state + jj);
                        } while ((w >> 32) == 0);
                    }
                    const unsigned inc = __ballot_sync(0xffffffffu, (w >> 32) == 2);
                    const int first = inc ? __ffs(inc) - 1 : 31;
                    excl += __reduce_add_sync(0xffffffffu, lane <= first ? (int)(w & 0xffffffffu) : 0);
                    if (inc) break;
                }
                if (lane == 0) lb_store(state + tile, lb_pack(2u, (unsigned)(excl + agg)));
            }
            if (lane < kPlTile) s_off[lane] = excl + incl - cnt;
            if (tile == nt - 1 && lane == 0) {
                const int total = excl + agg;
                ctl[1] = total;
                indptr[n] = total;
                int fl = 0;
                if (expect >= 0 && total != expect) fl |= 1;
                if (total > cap) fl |= 2;
                if (fl) atomicOr(ctl + 2, fl);
            }
        }
        __syncthreads();
        // ---- phase 3
        for (int t = warp; t < kPlTile; t += NW) {
            const int rr = c.row_begin + tile * kPlTile + t;
            if (rr >= c.row_end) break;
            int pos = s_off[t];
            if (lane == 0) indptr[rr - c.row_begin] = pos;
            for (int o0 = 0; o0 < T; o0 += 32) {
                const int o = o0 + lane;
                const int cl = o < T ? sc[t * T + o] : -1;
                const unsigned m = __ballot_sync(0xffffffffu, cl >= 0);
                if (cl >= 0) {
                    const int at = pos + __popc(m & lt);
                    if (at < cap) {
                        indices[at] = cl;
                        data[at] = sv[t * T + o];
                    }
                }
                pos += __popc(m);
            }
        }
        __syncthreads();
    }
}

}  // namespace tq

using namespace tq;

template <int P, int TS>
static int sf_strips_launch(const tq_rawctx& c, const int32_t* strips, int32_t nstrips, int32_t n1m, int32_t n2m,
                            int32_t nu_max, int32_t b2cap, const double* bw1, const double* bw2, int32_t* status,
                            cudaStream_t st) {
    const size_t shm = sizeof(double) * strip_smem_doubles(P, n1m, n2m, nu_max, TS, b2cap);
    if (shm > 220 * 1024) { set_error("strip workspace too large (%zu bytes)", shm); return TQ_EINVAL; }
    auto kern = k_sf_strips<P, TS>;
    constexpr int NT = 32 * ((TS * 9 + 31) / 32) + 32;
    TQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    int per_sm = 0;
    TQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, shm));
    // at least two strips per block (the producer runs one strip ahead)
    const int grid = (int)std::min<int64_t>((nstrips + 1) / 2, (int64_t)kSms * std::max(per_sm, 1));
    kern<<<grid, NT, shm, st>>>(c, strips, nstrips, n1m, n2m, nu_max, b2cap, bw1, bw2, status);
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_sf_strips");
    return TQ_OK;
}

template <int P, int TS>
static int sf_strips_occupancy(int32_t n1m, int32_t n2m, int32_t nu_max, int32_t b2cap) {
    const size_t shm = sizeof(double) * strip_smem_doubles(P, n1m, n2m, nu_max, TS, b2cap);
    if (shm > 220 * 1024) return 0;
    auto kern = k_sf_strips<P, TS>;
    constexpr int NT = 32 * ((TS * 9 + 31) / 32) + 32;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm) != cudaSuccess) return -1;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, shm) != cudaSuccess) return -1;
    return per_sm;
}

// resident tq_sf_strips blocks per SM of a launch class (the host groups
// strips into launches by it); < 0 on a CUDA error
extern "C" int32_t tq_sf_strips_occupancy(int32_t p, int32_t rows, int32_t n1m, int32_t n2m, int32_t nu_max,
                                          int32_t b2cap) {
    switch (p) {
#define CASE(Q) case Q: return rows == 8 ? sf_strips_occupancy<Q, 8>(n1m, n2m, nu_max, b2cap) \
                                          : sf_strips_occupancy<Q, kStripRows>(n1m, n2m, nu_max, b2cap);
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
    }
    return -1;
}

extern "C" int64_t tq_bw_table_doubles(tq_rawctx c) {
    return (int64_t)c.n1 * bw_row(c.p1, c.nmax1) + (int64_t)c.n2 * bw_row(c.p2, c.nmax2);
}

// the weighted collocation tables of the standard rules (bw: tq_bw_table_doubles)
extern "C" int tq_bw_tables(tq_rawctx c, double* bw, int32_t* status, void* stream) {
    if (!c.sets1 || !c.sets2 || c.p1 != c.p2) { set_error("tq_bw_tables needs rule sets and p1 == p2"); return TQ_EINVAL; }
    const int64_t nb = tq_bw_table_doubles(c);
    if (nb <= 0) return TQ_OK;
    k_bw_tables<<<grid_for(nb, 256), 256, 0, S(stream)>>>(c, bw, bw + (int64_t)c.n1 * bw_row(c.p1, c.nmax1), status);
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_bw_tables");
    return TQ_OK;
}

extern "C" int tq_sf_strips(tq_rawctx c, int32_t rows, const int32_t* strips, int32_t nstrips, int32_t n1m,
                            int32_t n2m, int32_t nu_max, int32_t b2cap, const double* bw, int32_t* status,
                            void* stream) {
    if (rows != kStripRows && rows != 8) { set_error("strips of %d rows (16 or 8)", rows); return TQ_EINVAL; }
    if (nstrips <= 0) return TQ_OK;
    if (!c.grids || !c.raw_ld || c.p1 != c.p2) { set_error("tq_sf_strips needs coefficient grids, planes and p1 == p2"); return TQ_EINVAL; }
    if (c.p1 < 1 || c.p1 > kMaxP) { set_error("degree out of range"); return TQ_EINVAL; }
    if (n1m > c.nmax1 || n2m > c.nmax2) { set_error("strip capacity above the tables' stride"); return TQ_EINVAL; }
    const double* bw1 = bw;
    const double* bw2 = bw + (int64_t)c.n1 * bw_row(c.p1, c.nmax1);
    switch (c.p1) {
#define CASE(Q) case Q: return rows == 8 ? sf_strips_launch<Q, 8>(c, strips, nstrips, n1m, n2m, nu_max, b2cap, bw1, \
                                                                      bw2, status, S(stream)) \
                                          : sf_strips_launch<Q, kStripRows>(c, strips, nstrips, n1m, n2m, nu_max, \
                                                                            b2cap, bw1, bw2, status, S(stream));
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
    }
    return TQ_EINVAL;
}

extern "C" int64_t tq_planes_state_bytes(int32_t nrows) {
    return (int64_t)sizeof(unsigned long long) * ((nrows + 7) / 8 + 1);      // the smallest tile (8 rows)
}

template <int P, int kPlTile>
static int planes_csr_launch(const tq_rowctx& c, int32_t raw_base, int32_t* indptr, int32_t* indices, double* data,
                             int64_t cap, void* state, int32_t* ctl, int64_t expect, cudaStream_t st) {
    constexpr int T = (2 * P + 1) * (2 * P + 1);
    const size_t shm = (size_t)kPlTile * T * (sizeof(double) + sizeof(int));
    constexpr int kPlThreads = kPlThreadsPerRow * kPlTile;
    auto kern = k_planes_csr<P, kPlTile>;
    static int per_sm_cache[kMaxP + 1][16] = {};
    int dev = 0;
    TQ_CUDA(cudaGetDevice(&dev));
    int& per_sm = per_sm_cache[P][dev & 15];
    if (!per_sm) {
        TQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
        TQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPlThreads, shm));
        if (per_sm < 1) { set_error("planes stage does not fit in shared memory"); return TQ_EINVAL; }
    }
    const int nrows = c.row_end - c.row_begin, nt = (nrows + kPlTile - 1) / kPlTile;
    TQ_CUDA(cudaMemsetAsync(state, 0, (size_t)tq_planes_state_bytes(nrows), st));
    TQ_CUDA(cudaMemsetAsync(ctl, 0, 3 * sizeof(int32_t), st));
    const int grid = std::min(nt, kSms * per_sm);
    kern<<<grid, kPlThreads, shm, st>>>(c, raw_base, indptr, indices, data, cap,
                                        reinterpret_cast<unsigned long long*>(state), ctl, expect);
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_planes_csr");
    return TQ_OK;
}

// CSR rows [row_begin, row_end) of an all-raw formation from its planes
// (c.raw, c.raw_ld; storage index = active row - raw_base).  indptr:
// nrows + 1; indices/data: `cap` entries (>= nnz; the window total is
// always enough); state: tq_planes_state_bytes(nrows) bytes of scratch;
// ctl: 3 ints (ctl[1] = nnz, ctl[2] = flags, see k_planes_csr); expect: the
// nnz a replayed pass must reproduce (-1: none).  nnz_h (optional) reads
// ctl[1] back (synchronising the stream).
extern "C" int tq_planes_csr(tq_rowctx c, int32_t raw_base, int32_t* indptr, int32_t* indices, double* data,
                             int64_t cap, void* state, int32_t* ctl, int64_t expect, int64_t* nnz_h, void* stream) {
    const int nrows = c.row_end - c.row_begin;
    cudaStream_t st = S(stream);
    if (nrows <= 0) {
        TQ_CUDA(cudaMemsetAsync(indptr, 0, sizeof(int32_t), st));
        if (nnz_h) *nnz_h = 0;
        return TQ_OK;
    }
    if (!c.raw_ld || c.p1 != c.p2) { set_error("tq_planes_csr needs the planes layout and p1 == p2"); return TQ_EINVAL; }
    int rc = TQ_EINVAL;
    // rows per tile: 16 (default) or 8 (TQ_PL_TILE=8: half the stage, twice the resident blocks)
    static const bool tile8 = [] { const char* e = getenv("TQ_PL_TILE"); return e && atoi(e) == 8; }();
    switch (c.p1) {
#define CASE(Q) case Q: rc = tile8 ? planes_csr_launch<Q, 8>(c, raw_base, indptr, indices, data, cap, state, ctl, expect, st) \
                           : planes_csr_launch<Q, 16>(c, raw_base, indptr, indices, data, cap, state, ctl, expect, st); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
        default: set_error("degree out of range"); return TQ_EINVAL;
    }
    if (rc) return rc;
    if (nnz_h) {
        int32_t h[3];
        TQ_CUDA(cudaMemcpyAsync(h, ctl, sizeof(h), cudaMemcpyDeviceToHost, st));
        TQ_CUDA(cudaStreamSynchronize(st));
        if (h[2] & 2) { set_error("planes CSR: nnz %d exceeds the capacity %lld", h[1], (long long)cap); return TQ_EOVERFLOW; }
        *nnz_h = h[1];
    }
    return TQ_OK;
}
