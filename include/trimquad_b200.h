/*
 * trimquad_b200 -- C ABI of the B200-native formation path of arXiv 2101.08053
 * (weighted-quadrature row assembly of trimmed bivariate B-spline mass
 * matrices and the L2-projection right-hand side).
 *
 * Conventions
 *   - every entry point returns 0 on success or a TQ_E* status; the message of
 *     the last failure on the calling thread is in tq_last_error();
 *   - every array argument is a caller-owned DEVICE pointer unless its name
 *     ends in _h (host pointer); sizes are element counts;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *   - no hidden global device state: all buffers belong to the caller.
 *
 * Each entry point names the reference interface it replaces
 * (src/ = /root/reference/pkg/src/trimquad/).
 */
#ifndef TRIMQUAD_B200_H
#define TRIMQUAD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> Python exceptions (paper_2101_08053_b200/_lib.py) */
#define TQ_OK 0
#define TQ_EINVAL 1        /* ValueError                    */
#define TQ_ERULE 2         /* RuleConstructionError          */
#define TQ_ETRIM 3         /* TrimmingConfigurationError     */
#define TQ_EPATTERN 4      /* RuntimeError (pattern miss)    */
#define TQ_ECUDA 5         /* RuntimeError (CUDA failure)    */
#define TQ_EOVERFLOW 6     /* OverflowError (nnz >= 2^31)    */

/* element / function classes (src/trimming.py:53-56) */
#define TQ_INTERIOR 0
#define TQ_CUT 1
#define TQ_EXTERIOR 2

/* one univariate B-spline space (src/splines.py:32-232); device arrays */
typedef struct {
    const double* knots;     /* nknots = n + p + 1 */
    const double* bp;        /* nel + 1 breakpoints */
    const int32_t* espan;    /* nel: knot span of each element */
    const int32_t* el_first; /* n: first support element */
    const int32_t* el_last;  /* n: last support element */
    const int32_t* ov_lo;    /* n: first overlapping trial */
    const int32_t* ov_hi;    /* n: last overlapping trial */
    int32_t nknots, p, n, nel;
} tq_space1d;

/* a point layout (src/quadrature.py:74-121); device arrays */
typedef struct {
    const double* pts;       /* npts, sorted, strictly interior to elements */
    const int32_t* offsets;  /* nel + 1 */
    int32_t npts, nel;
} tq_layout;

/* a weighted rule set (src/quadrature.py:201-260): row i holds weights
 * w[wptr[i] .. wptr[i+1]) on layout points k0[i] ..; k0[i] < 0: no rule */
typedef struct {
    const int64_t* wptr;     /* n + 1 */
    const int32_t* k0;       /* n */
    const double* w;
} tq_rules;

/* trimming curve descriptor (src/trimming.py:69-351 + harness curves) */
#define TQ_CURVE_LINE 1           /* data: p0x p0y p1x p1y                    */
#define TQ_CURVE_ARC 2            /* data: cx cy r theta0 theta1              */
#define TQ_CURVE_CLOSED_CIRCLE 3  /* data: cx cy r ccw(0/1) seam              */
#define TQ_CURVE_BEZIER 4         /* data: 4 ctrl (x,y) + 3 anchors (x,y)     */
#define TQ_CURVE_BSPLINE 5        /* data: shift, ccw(0/1), m ctrl (x,y)      */
/* tq_curve_eval operations (src/trimming.py:69-95) */
#define TQ_CURVE_OP_EVALUATE 0         /* in: n parameters t   out: n (x,y)  */
#define TQ_CURVE_OP_DERIVATIVE 1       /* in: n parameters t   out: n (dx,dy)*/
#define TQ_CURVE_OP_SIGNED_DISTANCE 2  /* in: n points (x,y)   out: n        */
#define TQ_CURVE_OP_IS_INSIDE 3        /* in: n points (x,y)   out: n 0/1    */
typedef struct {
    int32_t kind;
    int32_t m;               /* control points (BSPLINE), else 0 */
    const double* data;      /* host or device pointer per entry point */
} tq_curve;

/* coefficient field c(u1,u2) (src/assembly.py:54-85) */
#define TQ_COEFF_IDENTITY 0
#define TQ_COEFF_GEOMETRY 1  /* det J of a B-spline map; data below           */
typedef struct {
    int32_t kind;
    int32_t p, n;            /* geometry spline degree and #functions/dir     */
    const double* knots;     /* device: n + p + 1 (same in both directions)   */
    const double* X;         /* device: n*n control x, row-major (i1, i2)     */
    const double* Y;         /* device: n*n control y                         */
} tq_coeff;

int tq_version(void);
/* keep freed cudaMallocAsync memory in the device's default pool (release
 * threshold = max) so scratch allocations of later calls re-map nothing */
int tq_pool_keep(int32_t device);
/* a captured graph (cudaGraph_t) instantiated with per-node priorities
 * (use_node_priority != 0: each kernel node runs at the priority of the
 * stream it was captured on), launched, destroyed; node priority census
 * (hist[k] = kernel nodes of priority -k, k < 8) */
int tq_graph_instantiate(void* graph, int32_t use_node_priority, void** exec);
int tq_graph_launch(void* exec, void* stream);
int tq_graph_exec_destroy(void* exec);
int tq_graph_node_priorities(void* graph, int32_t* hist, int32_t* nkernels);
/* graph nodes by cudaGraphNodeType (counts[0..11]) */
int tq_graph_node_types(void* graph, int32_t* counts);
const char* tq_last_error(void);
int tq_device_sync(void* stream);
/* kernels launched by the library since it was loaded (host counter) */
long long tq_launch_count(void);
/* timeline probe: stamps[slot] = device global timer (ns), in stream order
   (diagnostic; not counted as a launch) */
int tq_debug_stamp(unsigned long long* stamps, int32_t slot, void* stream);

/* ---- subsystem (1): basis, moments, weights ------------------------------ */

/* Cox-de Boor at n points: first function index and p+1 values (and first
 * derivatives if ders != NULL).  Replaces Basis1D.eval_nonzero_batch
 * (src/splines.py:245-269). */
int tq_basis_eval(tq_space1d s, const double* u, int64_t n, int32_t* first,
                  double* vals, double* ders, int32_t* status, void* stream);

/* several Cox-de Boor evaluations (one degree) in one launch; the batch is
 * passed by value (kernel parameter, capturable).  Each task as
 * tq_basis_eval without derivatives or domain status (points in the domain
 * by construction).  `block_start` / `stage_bytes` are filled in by the call. */
#define TQ_EVAL_MAX_TASKS 16
typedef struct {
    tq_space1d s;
    const double* u;
    int64_t n;
    int32_t* first;
    double* vals;
} tq_evaltask;
typedef struct {
    tq_evaltask task[TQ_EVAL_MAX_TASKS];
    int32_t ntasks;
    int32_t block_start[TQ_EVAL_MAX_TASKS + 1];
    int32_t stage_bytes;
} tq_evalbatch;
int tq_basis_eval_multi(const tq_evalbatch* batch_h, void* stream);

/* exact banded 1-D mass matrix mom[i*(2p+1) + (j-i+p)] with (p+1)-point
 * Gauss per element.  Replaces mass_matrix_1d (src/quadrature.py:160-188). */
int tq_moments_1d_g(tq_space1d s, const double* gx, const double* gw, int32_t ng,
                    double* mom, void* stream);

/* dense n_test x n_trial exact mass matrix between two spaces on the same
 * breakpoints, max(p_test, p_trial)+1 Gauss points per element (gx/gw: the
 * device rule on [-1,1]).  Replaces mass_matrix_1d(basis, trial_basis)
 * (src/quadrature.py:160-188). */
int tq_mass_1d_mixed(tq_space1d test, tq_space1d trial, const double* gx, const double* gw,
                     int32_t ng, double* M, void* stream);

/* batched moment fits, one pivoted-QR basic solve per listed test row, on
 * layout `lay` with basis values (first, vals) at its points.  Writes
 * rules.w (at wptr offsets), rules.k0, and fail[r] = 1 where the residual
 * exceeds 1e-12 max|b|.  Replaces _solve_rows/_qr_basic_solve
 * (src/quadrature.py:263-303).  `products` (nullable, n x (2p+1)): the
 * direction products a[i][j-i+p] = sum_k w_i[k] B_j(x_k) of the solved rows,
 * bit-identical to tq_wq_products on the same rules. */
int tq_wq_solve(tq_space1d s, tq_layout lay, const int32_t* first, const double* vals,
                const double* mom, const int32_t* rows, int32_t nrows,
                int32_t tmax, int32_t mmax, int64_t* wptr, int32_t* k0, double* w,
                int32_t* fail, double* products, void* stream);

/* Fused, batched moment fits: every listed row of up to TQ_FIT_MAX_SETS rule
 * sets in ONE launch, warp per system, each warp forming its own exact
 * moments and collocation block and solving as tq_wq_solve (same pivots,
 * same outputs).  Replaces, per set, the tq_basis_eval -> tq_moments_1d_g ->
 * tq_wq_solve chain (src/quadrature.py:281-303 for every set the assembly
 * builds, src/assembly.py:454-489).  The batch is passed by value (a kernel
 * parameter: no upload, capturable); gx/gw: the (p+1)-point Gauss rule on
 * [-1,1] of the (common) degree.  `start` is filled in by the call. */
#define TQ_FIT_MAX_SETS 16
typedef struct {
    tq_space1d s;            /* basis of the set (refined basis for DWQ fits) */
    tq_layout lay;           /* its point layout                               */
    const int32_t* rows;     /* rows to fit                                    */
    int32_t nrows;
    const int64_t* wptr;     /* n + 1 weight offsets                           */
    int32_t* k0;             /* out: first point of each fitted row            */
    double* w;               /* out: weights at wptr                           */
    int32_t* fail;           /* out: per listed row, residual flag             */
    double* products;        /* out, nullable: n x (2p+1) direction products   */
} tq_fitset;
typedef struct {
    tq_fitset set[TQ_FIT_MAX_SETS];
    int32_t nsets;
    int32_t start[TQ_FIT_MAX_SETS + 1];
    const double* gx;
    const double* gw;
} tq_fitbatch;
int tq_wq_fit_sets(const tq_fitbatch* batch_h, int32_t tmax, int32_t mmax, void* stream);

/* every DWQ set's w = S^T w~ (tq_dwq_combine) in one launch; by value */
typedef struct {
    const int32_t* rows;     /* wanted original rows */
    int32_t nrows;
    const int32_t* colptr;   /* S in CSC */
    const int32_t* rowidx;
    const double* sval;
    tq_rules fine;           /* the refined fits */
    tq_rules out;            /* the set's rules (w written) */
} tq_combineset;
typedef struct {
    tq_combineset set[TQ_FIT_MAX_SETS];
    int32_t nsets;
    int32_t start[TQ_FIT_MAX_SETS + 1];
} tq_combinebatch;
int tq_dwq_combine_sets(const tq_combinebatch* batch_h, void* stream);

/* DWQ combination w_j = sum_i S_ij w~_i over augmented points (S in CSC,
 * device).  Replaces build_dwq step 4 (src/quadrature.py:434-444). */
int tq_dwq_combine(const int32_t* rows, int32_t nrows, const int32_t* s_colptr,
                   const int32_t* s_rowidx, const double* s_val,
                   tq_rules fine, tq_rules out_rules, void* stream);

/* ---- subsystem (2): classification --------------------------------------- */

/* element classes nel1 x nel2 (int8, row-major).  Replaces classify_elements
 * (src/trimming.py:607-733).  `curves` data pointers are DEVICE pointers. */
int tq_classify_elements(const tq_curve* curves_h, int32_t ncurves,
                         tq_space1d s1, tq_space1d s2, int8_t* elem_class,
                         int32_t* status, void* stream);

/* function classes n1 x n2 and discontinuity-face flags per direction.
 * Replaces TrimConfiguration.__init__ (src/trimming.py:441-484). */
int tq_function_classes(tq_space1d s1, tq_space1d s2, const int8_t* elem_class,
                        int8_t* func_class, int32_t* face1, int32_t* face2, void* stream);

/* active compact index col_of (n1*n2, -1 = exterior), active list and K
 * (host out).  Replaces active_functions + _Pattern.col_of
 * (src/trimming.py:514-517, src/assembly.py:148-153). */
int tq_active_index(const int8_t* func_class, int64_t nfun, int32_t* col_of,
                    int32_t* active, int32_t* K_h, void* stream);

/* DWQ routing of each cut row (src/trimming.py:545-586): route[r*8 + ...] =
 * {eligible, iu1, iu2, a1, b1, a2, b2, 0}; iu = index into the udisc arrays
 * or -1; a1 = -1 when no all-interior box exists. */
int tq_dwq_route(tq_space1d s1, tq_space1d s2, const int8_t* elem_class,
                 const double* udisc1, int32_t nu1, const double* udisc2, int32_t nu2,
                 const int32_t* cut_rows, int32_t ncut, int32_t* route, void* stream);

/* ---- subsystems (3)+(4): rows ------------------------------------------- */

/* banded WQ product table a[i*(2p+1) + (j-i+p)] = sum_k w_i[k] B_j(x_k) --
 * the direction-wise contraction of sum_factor_row (src/assembly.py:245-252)
 * for a coefficient-free direction. */
int tq_wq_products(tq_space1d s, tq_layout lay, const int32_t* first, const double* vals,
                   tq_rules rules, double* a, void* stream);

/* per-row kept-entry counts of the symmetrised pattern and the final CSR
 * fill (src/assembly.py:400-404 fused with the row assembly
 * src/assembly.py:409-449).  See DESIGN.md "rows". */
typedef struct {
    int32_t n1, n2, p1, p2;
    const int32_t* ov_lo1; const int32_t* ov_hi1;
    const int32_t* ov_lo2; const int32_t* ov_hi2;
    const int32_t* col_of;       /* n1*n2 */
    const int32_t* active;       /* K: i1*n2 + i2 */
    const int32_t* slot;         /* n1*n2: raw-block slot or -1 (separable) */
    const double* a1;            /* n1*(2p1+1) */
    const double* a2;            /* n2*(2p2+1) */
    const double* raw;           /* nslots * (2p1+1)*(2p2+1) */
    const int8_t* deep;          /* n1*n2: 1 = separable row whose window holds
                                    only separable rows with positive factors */
    int8_t* rowfast;             /* per active row (written by tq_row_counts):
                                    deep with full (2p+1)^2 windows */
    int32_t row_begin, row_end;  /* active rows [begin, end) */
    /* optional (NULL: the fill reads a complete indptr): per-row counts and
       per-32-row tile sums.  The count passes write the tile sums,
       tq_scan_tiles turns them into tile bases in place, and the fill kernels
       then derive each row's offset from its tile base and the counts before
       it in the tile, writing indptr[0 .. nrows) themselves. */
    const int32_t* counts;
    int32_t* tiles;              /* TQ_TILE_INTS(nrows) ints: the sums, then
                                    the bases (tq_tile_bases) */
    int64_t raw_ld;              /* 0: raw blocks row-major (slot * W + o);
                                    > 0: planes, entry o of slot s at
                                    raw[o * raw_ld + s] (tq_planes_csr) */
    /* optional (NULL: off): function classes (n1*n2) and the per-line factor
       positivity of this pass (n1 + n2, k_pos2).  An interior separable row
       whose two lines are positive has only positive partner sums M_ij + M_ji
       (its own products are positive, and every partner's value is the
       integral of B_i B_j over part of supp(i), which is visible): the value
       count of tq_row_counts_rest counts it geometrically, and the fill
       verifies it -- a dropped entry in such a row sets TQ_TILE_CTL + 8. */
    const int8_t* fclass;
    const int8_t* pos;
} tq_rowctx;

/* tile-mode buffer layout (ints): the tile sums (padded to a multiple of 4
   for vector loads) | the tile bases, the total, an overflow flag | the early
   bases (head tiles before the first list-A row and tail tiles after the last
   one: final after count pass 1, the tail ones given nnz) | eight control
   words: first list-A row (encoded INT_MAX - row, 0 = none), last list-A row
   + 1 (0 = none), the fill's tile counters; zeroed by the count pass */
#define TQ_TILE_NT(nrows) (((nrows) + 31) / 32)
#define TQ_TILE_PAD(nrows) ((TQ_TILE_NT(nrows) + 3) / 4 * 4)
#define TQ_TILE_EARLY(nrows) (TQ_TILE_PAD(nrows) + TQ_TILE_NT(nrows) + 2)
#define TQ_TILE_CTL(nrows) (TQ_TILE_EARLY(nrows) + TQ_TILE_NT(nrows))
#define TQ_TILE_INTS(nrows) (TQ_TILE_CTL(nrows) + 9)
static inline int32_t* tq_tile_bases(int32_t* tiles, int32_t nrows) { return tiles + TQ_TILE_PAD(nrows); }

/* deep-row flags: deep[i] = separable(i) && no raw row in window(i) &&
 * positive direction factors (the fill then needs no per-entry gathers) */
int tq_deep_flags(tq_rowctx c, const int8_t* func_class, const int32_t* raw_rows,
                  int32_t nraw, int8_t* deep, void* stream);
/* tq_deep_flags in two parts: the geometric flag (interior, not raw, no raw
 * row in the window; depends only on the row plan, so callers may keep it)
 * and the per-pass positivity of the direction factors a1, a2 */
int tq_deep_geometry(tq_rowctx c, const int8_t* func_class, const int32_t* raw_rows,
                     int32_t nraw, int8_t* geo, void* stream);
/* tq_deep_apply writes the flags of the direction-1 lines spanned by the
 * context's rows [row_begin, row_end) (the only ones the counts and the fill
 * of that row block read); flags on other lines are left unchanged */
int tq_deep_apply(tq_rowctx c, const int8_t* geo, int8_t* deep, void* stream);

int tq_row_counts(tq_rowctx c, int32_t* counts, void* stream);
/* the two passes of tq_row_counts, separately launchable so the deep pass can
 * overlap the raw-row kernels.  `work` = caller scratch of 2*nrows + 2 ints:
 * work[0] = |A|, work[1] = |B|, list A (rows needing the value-based count)
 * at work + 2, list B (deep rows with a partial window) at work + 2 + nrows */
int tq_row_counts_deep(tq_rowctx c, int32_t* counts, int32_t* work, void* stream);
int tq_row_counts_rest(tq_rowctx c, int32_t* counts, const int32_t* work, void* stream);
/* count pass 2 split: the listed rows' geometry records (one 32-byte record
 * per list-A row, rec: (row_end - row_begin) * tq_list_record_bytes()),
 * then the value-based counts from them (the same counts as
 * tq_row_counts_rest) */
int64_t tq_list_record_bytes(void);
int tq_list_geometry(tq_rowctx c, const int32_t* work, void* rec, void* stream);
int tq_row_counts_rest_rec(tq_rowctx c, int32_t* counts, const int32_t* work, const void* rec, void* stream);
/* tq_row_counts_deep from the geometric flags of tq_deep_geometry and the
 * per-line factor positivity (computed here into `pos`, n1 + n2 bytes of
 * caller scratch); c.deep is not read.  The lists then carry the deep /
 * not-deep split that tq_fill_listed uses, so no deep array is formed. */
int tq_row_counts_geo(tq_rowctx c, const int8_t* geo, int8_t* pos, int32_t* counts, int32_t* work,
                      void* stream);
/* count pass 1 from a cache: the arrays of an earlier tq_row_counts_geo on
 * the same row plan (counts, rowfast, work lists, and `tiles0` = its tile
 * buffer right after the pass) are reused; this call restores c.tiles from
 * tiles0, recomputes the line positivity into `pos`, and redoes the pass on
 * the device (into the same arrays) only when the positivity differs from
 * `pos_cached` or an earlier redo left them dirty.  `flags`: 3 ints, the
 * dirty word (flags[1]) zero-initialised once by the caller and kept. */
int tq_row_counts_cached(tq_rowctx c, const int8_t* geo, int8_t* pos, const int8_t* pos_cached,
                         int32_t* flags, int32_t* counts, int32_t* work, const int32_t* tiles0, void* stream);
/* speculative count pass 1 (tq_row_counts_geo with every line's factors
 * assumed positive; needs no factor, so it can run before the fits) and its
 * check: tq_row_counts_verify computes the positivity (pos: n1+n2 bytes,
 * bad: 1 int scratch) and, only if some line is not positive, redoes the
 * pass exactly as tq_row_counts_geo (device-side guard). */
int tq_row_counts_spec(tq_rowctx c, const int8_t* geo, int32_t* counts, int32_t* work, void* stream);
int tq_row_counts_verify(tq_rowctx c, const int8_t* geo, int8_t* pos, int32_t* bad, int32_t* counts,
                         int32_t* work, void* stream);
int tq_scan_indptr(const int32_t* counts, int32_t nrows, int32_t* indptr,
                   int64_t* nnz_h, void* stream);
/* the same with caller scratch of tq_scan_workspace_bytes(nrows) bytes */
int64_t tq_scan_workspace_bytes(int32_t nrows);
int tq_scan_indptr_ws(const int32_t* counts, int32_t nrows, int32_t* indptr, void* ws,
                      int64_t* nnz_h, void* stream);
/* tile mode (c.counts, c.tiles set, after the count passes): exclusive scan
 * of the tile sums -> tile bases (second half of c.tiles); indptr[nrows] = nnz.  nnz_h: as
 * tq_scan_indptr.  The fill kernels then write indptr[0 .. nrows). */
int tq_scan_tiles(tq_rowctx c, int32_t* indptr, int64_t* nnz_h, void* stream);
/* the nnz a captured (replayed) pass sized its output with: the following
 * tq_scan_tiles compares its total against it; a mismatch sets the flag word
 * TQ_TILE_CTL + 4 and the tile-mode fills (tq_fill_fast(_part),
 * tq_fill_listed) then write nothing. */
int tq_tiles_expect(tq_rowctx c, int64_t nnz, void* stream);
int tq_fill_rows(tq_rowctx c, const int32_t* indptr, int32_t* indices, double* data,
                 void* stream);
/* tq_fill_rows split in two after tq_row_counts_deep/_rest: tq_fill_fast
 * writes the fast rows (every row when the context has no separable
 * factors), tq_fill_listed the rows of lists A and B in `work`.  They write
 * disjoint rows and may run concurrently on two streams.  In tile mode
 * tq_fill_fast also writes indptr[0 .. nrows) (every row's offset). */
int tq_fill_fast(tq_rowctx c, int32_t* indptr, int32_t* indices, double* data, void* stream);
/* tile mode, split around the listed rows: part 1 = the early tiles (before
 * the tile holding the first list-A row and after the one holding the last;
 * after count pass 1 and tq_scan_tiles_early, may run concurrently with the
 * raw rows and count pass 2), part 2 = the tiles in between (after
 * tq_scan_tiles); part 0 = all.  blocks_per_sm > 0 caps the grid (a part
 * running beside other kernels). */
int tq_fill_fast_part(tq_rowctx c, int32_t* indptr, int32_t* indices, double* data, int32_t part,
                      int32_t blocks_per_sm, void* stream);
/* early bases after count pass 1: head tiles by prefix sums and, with
 * tail != 0, the tail tiles as nnz - suffix sums.  nnz (>= 0) is the count
 * known in advance (a captured pass, which sized the output with it):
 * tq_scan_tiles later checks the total against it, a mismatch sets the flag
 * word TQ_TILE_CTL + 4.  nnz < 0: unknown (head only, no check). */
int tq_scan_tiles_early(tq_rowctx c, int64_t nnz, int32_t tail, void* stream);
int tq_fill_listed(tq_rowctx c, const int32_t* indptr, int32_t* indices, double* data,
                   const int32_t* work, void* stream);


/* ---- raw (non-separable) rows ------------------------------------------ */

/* a rule set with its basis table at the layout points */
typedef struct {
    tq_rules rules;
    tq_layout lay;
    const int32_t* first;    /* npts */
    const double* vals;      /* npts x (p+1) */
} tq_ruleset;

#define TQ_ROW_GAUSS 0   /* element Gauss over the interior support elements */
#define TQ_ROW_BOX 1     /* sum factorization over a point box + Gauss residual */
#define TQ_ROW_MASK 2    /* naive WQ: sum factorization masked to interior elements */

/* Everything the raw-row kernels read; all device pointers. */
typedef struct {
    int32_t n1, n2, p1, p2, nel1, nel2;
    const int32_t* el_first1; const int32_t* el_last1;
    const int32_t* el_first2; const int32_t* el_last2;
    const int32_t* ov_lo1; const int32_t* ov_hi1;
    const int32_t* ov_lo2; const int32_t* ov_hi2;
    const int32_t* espan1; const int32_t* espan2;
    const int8_t* elem_class;        /* nel1*nel2 */
    int32_t ng1, ng2;                /* element Gauss points per direction (p+1) */
    const double* ew1; const double* ev1;   /* nel*ng weights; nel*ng*(p+1) values */
    const double* ew2; const double* ev2;
    const double* em1; const double* em2;   /* nel*(p+1)^2 element 1-D masses (c == 1) */
    const double* cg;                /* c at element Gauss points, (nel1*ng1) x (nel2*ng2); NULL: c == 1 */
    const tq_ruleset* sets1; const tq_ruleset* sets2;
    int32_t nsets1, nsets2;
    const double* const* grids;      /* nsets1*nsets2 coefficient grids; NULL table: c == 1 */
    const int32_t* cutidx;           /* nel1*nel2 -> cut element id, -1 */
    const int64_t* cut_ptr;          /* ncut + 1 */
    const double* cut_cw;            /* c * w per cut point */
    const int32_t* cfirst1; const double* cvals1;
    const int32_t* cfirst2; const double* cvals2;
    const int32_t* grp_ptr;          /* ncut + 1: span-key groups of each cut element */
    const int32_t* grp_key;          /* ngroups x 2: (first1, first2) of the group */
    const int64_t* grp_pts;          /* ngroups + 1: ranges into grp_perm */
    const int64_t* grp_perm;         /* cut points ordered by (element, key) */
    double* grp_blocks;              /* ngroups x ((p1+1)(p2+1))^2 element blocks */
    int32_t ngroups;
    const int32_t* desc;             /* nraw x 8: fidx, mode, set1, set2, a1, b1, a2, b2 */
    int32_t nraw;
    int32_t nmax1, nmax2;            /* max points of one rule row per direction */
    double* raw;                     /* nraw x (2p1+1)(2p2+1), or planes (raw_ld) */
    /* planes layout (raw_ld > 0): entry q of descriptor row r is stored at
       raw[q * raw_ld + store[r]]; the storage index of a row is its active
       index minus the block's first one, so the planes of consecutive rows
       are contiguous (coalesced symmetrisation, tq_planes_csr) */
    const int32_t* store;
    int64_t raw_ld;
} tq_rawctx;

/* regular-support part of raw rows [r0, r1) (overwrites their blocks).
 * Replaces sum_factor_row / _gauss_rows_by_element / _cut_regular_rows /
 * the element loop of the reference strategy (src/assembly.py:218-252,
 * 522-528, 553-648). */
int tq_raw_regular(tq_rawctx c, int32_t r0, int32_t r1, void* stream);
/* tq_raw_regular in two launches: the element-Gauss part (writes the row
 * blocks; element tables only, no WQ rules) and the sum-factorization part
 * (adds onto them).  Bit-identical to the fused call. */
int tq_raw_gauss(tq_rawctx c, int32_t r0, int32_t r1, void* stream);
int tq_raw_sumfactor(tq_rawctx c, int32_t r0, int32_t r1, void* stream);

/* cut-element part of raw rows [r0, r1) (accumulates): element blocks
 * B^T diag(c w) B per (cut element, span key) group, then a row gather.
 * Replaces _Run.add_cut_blocks (src/assembly.py:369-398). */
int tq_cut_blocks(tq_rawctx c, void* stream);
/* element 1-D masses em[e][a][b] = sum_g w V_a V_b from element Gauss tables
 * (ev: nel*ng*(p+1), ew: nel*ng) -- the c == 1 factors of _Run.element_block
 * (src/assembly.py:310-332) */
int tq_elem_mass(const double* ev, const double* ew, int32_t nel, int32_t ng, int32_t p, double* em,
                 void* stream);
int tq_raw_cutcells(tq_rawctx c, int32_t r0, int32_t r1, void* stream);
/* per-row span-key group lists of raw rows [r0, r1) (geometry of the plan):
 * off == NULL: out = the counts (r1 - r0 ints); else out = the triplets
 * (group, key1, key2) at 3 * off[r - r0] (off: exclusive prefix of the
 * counts) -- in tq_raw_cutcells's order */
int tq_row_groups(tq_rawctx c, int32_t r0, int32_t r1, const int32_t* off, int32_t* out, void* stream);
/* tq_raw_cutcells over those lists (rg_ptr: r1 - r0 + 1 offsets); the same
 * additions in the same order */
int tq_raw_cutcells_list(tq_rawctx c, int32_t r0, int32_t r1, const int32_t* rg_ptr, const int32_t* rg,
                         void* stream);

/* ---- the all-raw path in the planes layout (c.raw_ld > 0) --------------- */

/* interior rows of the c != 1 BOX plan (box = whole support, standard rules)
 * by strips of up to `rows` (16 or 8) rows (i1, i20 + t): strips = nstrips x
 * (2 + rows) ints (i1, i20, storage index of row t or -1); nu_max bounds the union of a
 * strip's direction-2 point windows and n1m / n2m its rule rows (shared-
 * memory sizing, <= the context's nmax); b2cap > 0: the strip's direction-2
 * table rows are staged packed, each row sized by its own rule length, in
 * b2cap doubles (the largest sum over the strips of the launch of
 * 2 * (((len * wp + 1) / 2) | 1), wp = 3 * ((2p + 3) / 3)); b2cap = 0: rows
 * of n2m each; bw: the tables of tq_bw_tables; a strip that breaks a bound
 * sets *status |= 1 and writes zero blocks.  Replaces sum_factor_row over
 * _interior_rows_batched (src/assembly.py:218-252, 409-449); writes the
 * rows' planes. */
int tq_sf_strips(tq_rawctx c, int32_t rows, const int32_t* strips, int32_t nstrips, int32_t n1m, int32_t n2m,
                 int32_t nu_max, int32_t b2cap, const double* bw, int32_t* status, void* stream);
/* resident tq_sf_strips blocks per SM for a launch of that shape (0: the
 * stage does not fit; < 0: CUDA error) -- the host merges strip classes into
 * one launch when that does not lower the occupancy */
int32_t tq_sf_strips_occupancy(int32_t p, int32_t rows, int32_t n1m, int32_t n2m, int32_t nu_max, int32_t b2cap);
/* the weighted collocation tables of the standard rules tq_sf_strips reads
 * (bw: n_d x nmax_d x the padded window, both directions; size in doubles
 * from tq_bw_table_doubles); *status |= 2 when a rule row is longer than
 * the context's nmax */
int64_t tq_bw_table_doubles(tq_rawctx c);
int tq_bw_tables(tq_rawctx c, double* bw, int32_t* status, void* stream);
/* symmetrise / zero-drop / CSR of rows [row_begin, row_end) in one pass
 * (_Run.finish, src/assembly.py:400-404) from the planes (c.raw, c.raw_ld;
 * storage index = active row - raw_base): indptr nrows + 1, indices/data
 * `cap` entries, state tq_planes_state_bytes(nrows) bytes of scratch, ctl 3
 * ints ([1] nnz, [2] flags: 1 = nnz != expect (expect >= 0), 2 = nnz > cap).
 * nnz_h (optional) reads nnz back, synchronising the stream. */
/* cut rows of the c != 1 planes path, element-centric: element-Gauss blocks
 * of the listed interior elements (gel: nslot x 2; cgp: c at their (p+1)^2
 * Gauss points) and span-key group blocks of the cut elements, both in pair
 * form (q(q+1)/2 x q(q+1)/2 per block: E[(a1,a2)][(b1,b2)] is symmetric in
 * (a1,b1) and (a2,b2)); then per cut row the sum of the row slices it reads,
 * written to its planes (gslot: element -> Gauss slot; rg_ptr / rg: the
 * rows' span-key groups, 3 ints each = group, key1, key2; status |= 4 when
 * a needed element block is missing).  c of the Gauss blocks: det J computed in the kernel for a
 * geometry map (X1/X2: element Gauss points), else cgp at their points.  Replaces _Run.element_block and
 * _Run.add_cut_blocks (src/assembly.py:310-332, 369-398). */
int64_t tq_pair_block_doubles(int32_t p);
int tq_gauss_pairs(tq_rawctx c, tq_coeff geo, const double* X1, const double* X2, const int32_t* gel,
                   int32_t nslot, const double* cgp, double* E, const int32_t* lsp1, const double* lnd1,
                   const int32_t* lsp2, const double* lnd2, void* stream);
/* geometry-map line tables (span; N[0..p], D[0..p]) at n points, read by
 * tq_gauss_pairs for the element Gauss points (NULL tables: computed inline) */
int tq_geo_lines(tq_coeff geo, const double* u, int32_t n, int32_t* span, double* nd, void* stream);
/* the group blocks by pieces of at most tq_cut_pair_piece() points (pieces:
 * npieces x 2 int64 = group, first point; gpiece: ngroups + 1 offsets;
 * Epart: npieces blocks of scratch), summed per group in piece order */
int32_t tq_cut_pair_piece(void);
int tq_cut_pairs(tq_rawctx c, const int64_t* pieces, int32_t npieces, const int32_t* gpiece, double* Epart,
                 double* E, void* stream);
int tq_cut_rows_gather(tq_rawctx c, int32_t r0, int32_t r1, const int32_t* gslot, const double* Eg,
                       const double* Ec, const int32_t* rg_ptr, const int32_t* rg, int32_t* status,
                       void* stream);
int64_t tq_planes_state_bytes(int32_t nrows);
int tq_planes_csr(tq_rowctx c, int32_t raw_base, int32_t* indptr, int32_t* indices, double* data,
                  int64_t cap, void* state, int32_t* ctl, int64_t expect, int64_t* nnz_h, void* stream);

/* coefficient c = det J of a B-spline geometry map on a tensor grid / at
 * points (the reference takes a host callable, src/assembly.py:54-85) */
int tq_coeff_grid(tq_coeff g, const double* x1, int32_t n1, const double* x2, int32_t n2,
                  double* out, void* stream);
int tq_coeff_points(tq_coeff g, const double* pts, int64_t n, const double* w, double* out,
                    void* stream);

/* ---- host-native cut-cell quadrature (geometry input of subsystem 3) ------ */

/* Decompose every listed cut element (cut_el_h: ncut x 2 element indices,
 * row-major order) against the curves (HOST data pointers) and place
 * (q+1)^2 Gauss points per sub-cell.  tabs_h: q+1 Lobatto nodes on [0,1],
 * q+1 Gauss nodes and weights on [0,1], the (q+1)x(q+1) Lagrange values and
 * derivatives at the Gauss nodes.  Returns an opaque handle (NULL on failure,
 * status in *status_h).  Replaces cut_cell_quadrature / decompose_cut_element
 * (src/trimming.py:938-1111) with the closed-curve seam routing of SURVEY F3. */
void* tq_cutcell_build(const tq_curve* curves_h, int32_t ncurves, const double* bp1_h, int32_t nel1,
                       const double* bp2_h, int32_t nel2, const int32_t* cut_el_h, int32_t ncut,
                       int32_t q, const double* tabs_h, int32_t* status_h);
int64_t tq_cutcell_npoints(void* handle);
/* ptr_h: ncut+1 point offsets; pts_h: npoints x 2; w_h: npoints; ncells_h: ncut */
int tq_cutcell_copy(void* handle, int64_t* ptr_h, double* pts_h, double* w_h, int32_t* ncells_h);
void tq_cutcell_free(void* handle);
/* the same decomposition on the device, one thread per cut element, in two
 * calls.  Count pass (pts == NULL): ptr[z+1] = points of element z (ptr[0]
 * caller-zeroed), ncells[z] = sub-cells, status[z] = 0 ok / 1 max split
 * depth / 2 folded / 3 not crossed by exactly one curve / 4 capacity.  The
 * caller turns ptr into offsets (inclusive scan of ptr[1..]) and calls again
 * with pts (2 per point) and w to write.  bp1/bp2 breakpoints, cut_el
 * (ncut x 2 int32, row-major element order) and the outputs are device
 * arrays; curves and tabs (as for tq_cutcell_build) are host arrays (staged
 * before the call returns).  The three device entry points are asynchronous
 * on `stream`: the outputs are valid in stream order, not on return. */
int tq_cutcell_device(const tq_curve* curves_h, int32_t ncurves, const double* bp1, const double* bp2,
                      const int32_t* cut_el, int32_t ncut, int32_t q, const double* tabs_h, int64_t* ptr,
                      double* pts, double* w, int32_t* ncells, int32_t* status, void* stream);
/* single-decomposition schedule.  Slot pass: element z writes up to `cap`
 * points into slot_pts[2*cap*z ..] / slot_w[cap*z ..] and, as the count
 * pass above, ptr[z+1], ncells[z] and status[z] (its full count, also when
 * it exceeds cap).  The caller scans ptr, then the pack call copies every
 * slot within capacity to its offsets and, when any_overflow != 0,
 * decomposes again (write mode) the elements whose count exceeds cap. */
int tq_cutcell_device_slots(const tq_curve* curves_h, int32_t ncurves, const double* bp1, const double* bp2,
                            const int32_t* cut_el, int32_t ncut, int32_t q, const double* tabs_h, int64_t cap,
                            double* slot_pts, double* slot_w, int64_t* ptr, int32_t* ncells, int32_t* status,
                            void* stream);
int tq_cutcell_device_pack(const tq_curve* curves_h, int32_t ncurves, const double* bp1, const double* bp2,
                           const int32_t* cut_el, int32_t ncut, int32_t q, const double* tabs_h, int64_t cap,
                           const double* slot_pts, const double* slot_w, const int64_t* ptr, double* pts,
                           double* w, int32_t any_overflow, void* stream);

/* ---- L2 projection: RHS and error ---------------------------------------- */

/* target f(x, y): kind 0 = values on the Gauss tensor grid (grid[r1*ld + r2]);
 * kind 1 = sum_k terms[7k] * phi(terms[7k+1], terms[7k+2] x + terms[7k+3])
 *                        * phi(terms[7k+4], terms[7k+5] y + terms[7k+6]),
 * phi kinds 0 = 1, 1 = sin, 2 = cos, 3 = exp (evaluated in-kernel);
 * kind 2 = kind 1 with its factors tabulated per Gauss coordinate
 * (tq_target_tables): grid[k*(ld + n2) + r1] = phi_k(x_r1), grid[k*(ld + n2)
 * + ld + r2] = psi_k(y_r2), ld = nel1*g1n -- the same values, evaluated once
 * per coordinate instead of once per tensor point */
typedef struct {
    int32_t kind, nterms;
    const double* terms;
    const double* grid;
    int64_t ld;
} tq_target;

typedef struct {
    int32_t n1, n2, p1, p2, nel1, nel2;
    const int32_t* el_first1; const int32_t* el_last1;
    const int32_t* el_first2; const int32_t* el_last2;
    const int32_t* espan1; const int32_t* espan2;
    const int8_t* elem_class;
    int32_t g1n, g2n;                /* Gauss points per element (p+2 RHS, p+3 error) */
    const double* x1; const double* w1; const double* v1;   /* nel*g, nel*g, nel*g*(p+1) */
    const double* x2; const double* w2; const double* v2;
    const double* cgrid; int64_t cld;   /* c on the Gauss tensor grid, NULL: c == 1 */
    tq_target target;
    const int32_t* active;
    int32_t row_begin, row_end;
    const int32_t* cutidx; const int64_t* cut_ptr;
    const double* cut_fcw;           /* f c w per cut point (RHS) */
    const double* cut_w;             /* w per cut point (error) */
    const int32_t* cfirst1; const double* cvals1;
    const int32_t* cfirst2; const double* cvals2;
} tq_projctx;

/* b over active rows [row_begin, row_end) (T: scratch (nel1*g1n) x n2). */
int tq_rhs(tq_projctx c, double* T, const int32_t* cut_rows, int32_t ncut, double* b, void* stream);
int tq_target_points(tq_target f, const double* P, const double* w, int64_t n, double* out, void* stream);
/* the RHS for a kind-2 (tabulated separable) target with c == 1: per
 * direction the element integrals Q_k[e][a] of each factor, their support
 * sums A_k[i], then b_i = sum_k A1_k[i1] A2_k[i2] for all-interior supports
 * and the interior-masked element double sum otherwise, plus the cut-cell
 * points (replaces tq_rhs's two tensor stages for this case).
 * `work`: tq_rhs_separable_work(c) doubles. */
int tq_rhs_separable(tq_projctx c, const int8_t* func_class, double* work, const int32_t* cut_rows,
                     int32_t ncut, double* b, void* stream);
int64_t tq_rhs_separable_work(tq_projctx c);
/* the kind-2 tables of a kind-1 target at the Gauss coordinates x1 (n1) and
 * x2 (n2): out[k*(n1+n2) + i] (see tq_target) */
int tq_target_tables(tq_target f, const double* x1, int64_t n1, const double* x2, int64_t n2, double* out,
                     void* stream);
/* (num, den) of the relative L2 error over interior elements [e_begin, e_end)
 * (row-major ids) and cut points [p_begin, p_end); C is the n1 x n2
 * coefficient grid (zeros off the active set). */
int tq_l2_parts(tq_projctx c, const double* C, int64_t e_begin, int64_t e_end, int64_t p_begin,
                int64_t p_end, const double* fpts, double* num_den, void* stream);

/* ---- subsystem (6): SPD solve of the projection (device CSR) ------------ */

/* diag[i] = A_ii of a CSR with sorted columns (A.diagonal(),
 * src/projection.py:159) */
int tq_csr_diag(const int32_t* indptr, const int32_t* indices, const double* data, int32_t n,
                double* diag, void* stream);
/* y = diag(sl) A diag(sr) x; sl / sr may be NULL (identity).  As @ y and
 * A @ x of src/projection.py:196-201 */
int tq_spmv(const int32_t* indptr, const int32_t* indices, const double* data, int32_t n,
            const double* sl, const double* sr, const double* x, double* y, void* stream);
/* conjugate gradients on As = diag(s) A diag(s) from x0 = 0, scipy's cg
 * iteration (src/projection.py:180-186: rtol, atol = 0, maxiter): one
 * cooperative kernel.  `work`: tq_cg_workspace_bytes(n) bytes.  iters_dev
 * receives the iterations run (== maxiter: not converged), rnorm_dev the
 * final ||r|| (device scalars, no host sync). */
int64_t tq_cg_workspace_bytes(int32_t n);
int tq_cg_scaled(const int32_t* indptr, const int32_t* indices, const double* data, int32_t n,
                 const double* s, const double* b, double* x, double rtol, int32_t maxiter,
                 void* work, int32_t* iters_dev, double* rnorm_dev, void* stream);

/* ---- public lower-level API of the drop-in ------------------------------- */

/* The trimming-curve predicate interface on the device, one curve (data:
 * HOST pointer), `in`/`out` device arrays per TQ_CURVE_OP_*.  Replaces
 * TrimmingCurve.evaluate / derivative / signed_distance / is_inside
 * (src/trimming.py:69-95, per-curve :98-351). */
int tq_curve_eval(const tq_curve* curve_h, int32_t op, const double* in, int64_t n, double* out,
                  void* stream);

/* Hits (t, cross coordinate) of one curve with the grid line {axis = level}
 * (axis 0: vertical u1 = level), as the classifier sees them (tangential
 * touches dropped, duplicates merged, sorted by cross coordinate).  Device
 * outputs: ht/hc (first min(count, cap) hits), count[0] = hits found,
 * count[1] = overflow flag.  Replaces TrimmingCurve.intersect_line
 * (src/trimming.py:86-93, per-curve :124-134, :181-201, :324-351). */
int tq_curve_intersect_line(const tq_curve* curve_h, int32_t axis, double level, int32_t cap,
                            double* ht, double* hc, int32_t* count, void* stream);

/* Batched sum factorisation of caller-supplied rows (device arrays): per
 * row r, dims[4r..] = (n1, n2, t1, t2) and offs[7r..] = offsets into `data`
 * of C1 (n1 x t1), w1 (n1), C2 (n2 x t2), w2 (n2), G (n1 x n2), mask
 * (n1 x n2, < 0: none) and into `scratch` of a t2 x n1 work area; the
 * t1 x t2 block goes to out + out_off[r].  Replaces sum_factor_row
 * (src/assembly.py:218-252). */
int tq_sum_factor_rows(int32_t nrows, const int32_t* dims, const int64_t* offs, const int64_t* out_off,
                       const double* data, double* scratch, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TRIMQUAD_B200_H */
