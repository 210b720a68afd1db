// Subsystem (1): univariate basis evaluation and exact 1-D moments.
//
//  tq_basis_eval  <- Basis1D.eval_nonzero_batch   src/splines.py:245-269
//  tq_moments_1d  <- mass_matrix_1d              src/quadrature.py:160-188
//  tq_mass_1d_mixed <- mass_matrix_1d(basis, trial_basis)  (same lines)
#include <algorithm>

#include "common.cuh"

namespace tq {

// The knot vector is staged in shared memory when it fits (the span search
// is a chain of dependent loads: from shared memory instead of L2).
template <int P>
__global__ void k_basis_eval(tq_space1d s, const double* __restrict__ u, int64_t n,
                             int32_t* __restrict__ first, double* __restrict__ vals,
                             double* __restrict__ ders, int32_t* status, int staged) {
    extern __shared__ double skn[];
    const double* kn = s.knots;
    if (staged) {
        // all loads in flight before the stores (not one latency per knot)
        constexpr int U = 8;
        for (int k0 = threadIdx.x; k0 < s.nknots; k0 += U * blockDim.x) {
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = k0 + u * blockDim.x;
                v[u] = k < s.nknots ? __ldg(s.knots + k) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = k0 + u * blockDim.x;
                if (k < s.nknots) skn[k] = v[u];
            }
        }
        __syncthreads();
        kn = skn;
    }
    const double lo = kn[0], hi = kn[s.nknots - 1];
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        double x = u[t];
        if (!(x >= lo && x <= hi)) {
            if (status) atomicOr(status, kStatusDomain);
            x = x < lo ? lo : hi;
        }
        int span = find_span(kn, s.nknots, P, s.n, x);
        double N[P + 1];
        if (ders) {
            double D[kMaxP + 1];
            double Nr[kMaxP + 1];
            basis_funs_ders_rt(kn, P, span, x, Nr, D);
#pragma unroll
            for (int k = 0; k <= P; ++k) { N[k] = Nr[k]; ders[t * (P + 1) + k] = D[k]; }
        } else {
            basis_funs<P>(kn, span, x, N);
        }
        first[t] = span - P;
#pragma unroll
        for (int k = 0; k <= P; ++k) vals[t * (P + 1) + k] = N[k];
    }
}

// Several evaluations in one launch: the blocks are split among the tasks
// by their block counts, each block stages its task's knots and runs the
// k_basis_eval loop on its share of the task's points.
template <int P>
__global__ void k_basis_eval_multi(tq_evalbatch B) {
    extern __shared__ double skn[];
    int k = 0;
    while ((int)blockIdx.x >= B.block_start[k + 1]) ++k;
    const tq_evaltask& T = B.task[k];
    const tq_space1d& s = T.s;
    const double* kn = s.knots;
    const bool staged = (size_t)s.nknots * sizeof(double) <= (size_t)B.stage_bytes;
    if (staged) {
        for (int q = threadIdx.x; q < s.nknots; q += blockDim.x) skn[q] = __ldg(s.knots + q);
        __syncthreads();
        kn = skn;
    }
    const int nb = B.block_start[k + 1] - B.block_start[k];
    const int b = blockIdx.x - B.block_start[k];
    for (int64_t t = b * (int64_t)blockDim.x + threadIdx.x; t < T.n; t += (int64_t)nb * blockDim.x) {
        const double x = T.u[t];
        const int span = find_span(kn, s.nknots, P, s.n, x);
        double N[P + 1];
        basis_funs<P>(kn, span, x, N);
        T.first[t] = span - P;
#pragma unroll
        for (int q = 0; q <= P; ++q) T.vals[t * (P + 1) + q] = N[q];
    }
}

// Basis values and weights at the (p+1)-point element Gauss points:
// tab[(e*ng + g)*(p+2) + k] = B_{span(e)-p+k}(x_eg) for k <= p, and the
// mapped weight in slot p+1.
__global__ void k_gauss_table(tq_space1d s, const double* __restrict__ gx, const double* __restrict__ gw,
                              int ng, double* __restrict__ tab) {
    const int p = s.p;
    const int total = s.nel * ng;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int e = t / ng, g = t - e * ng;
        const double a = s.bp[e], b = s.bp[e + 1];
        const double mid = 0.5 * (a + b), half = 0.5 * (b - a);
        double N[kMaxP + 1];
        basis_funs_rt(s.knots, p, s.espan[e], mid + half * gx[g], N);
        double* out = tab + (int64_t)t * (p + 2);
        for (int k = 0; k <= p; ++k) out[k] = N[k];
        out[p + 1] = half * gw[g];
    }
}

// Banded exact 1-D mass matrix: thread per (i, o), j = i - p + o; element
// loop over the shared support in element order (the order np.add.at
// accumulates element blocks in the reference), values from the table.
__global__ void k_moments(tq_space1d s, const double* __restrict__ tab, int ng, double* __restrict__ mom) {
    const int p = s.p, W = 2 * p + 1;
    int64_t total = (int64_t)s.n * W;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int i = (int)(t / W), o = (int)(t % W);
        int j = i - p + o;
        double acc = 0.0;
        if (j >= 0 && j < s.n && j >= s.ov_lo[i] && j <= s.ov_hi[i]) {
            int ea = max(s.el_first[i], s.el_first[j]);
            int eb = min(s.el_last[i], s.el_last[j]);
            for (int e = ea; e <= eb; ++e) {
                const int f = s.espan[e] - p;
                const double* row = tab + (int64_t)e * ng * (p + 2);
                double part = 0.0;
                for (int g = 0; g < ng; ++g) {
                    const double* v = row + g * (p + 2);
                    part += v[i - f] * v[j - f] * v[p + 1];
                }
                acc += part;
            }
        }
        mom[t] = acc;
    }
}

// Dense exact mass matrix between a test and a trial space on the same
// breakpoints (mass_matrix_1d(basis, trial_basis), src/quadrature.py:160-188):
// thread per (i, j); element loop over the test support in element order
// (np.add.at accumulates the element blocks in that order), Gauss sum per
// element first.  The trial span of an element is the one of its first
// Gauss point, as in the reference (fj.reshape(nel, g)[:, 0]).
__global__ void k_mass_mixed(tq_space1d s, tq_space1d t, const double* __restrict__ gx,
                             const double* __restrict__ gw, int ng, double* __restrict__ M) {
    const int64_t total = (int64_t)s.n * t.n;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx / t.n), j = (int)(idx - (int64_t)(idx / t.n) * t.n);
        double acc = 0.0;
        for (int e = s.el_first[i]; e <= s.el_last[i]; ++e) {
            const double a = s.bp[e], b = s.bp[e + 1];
            const double mid = 0.5 * (a + b), half = 0.5 * (b - a);
            const int fi = s.espan[e] - s.p;
            const int tspan = find_span(t.knots, t.nknots, t.p, t.n, mid + half * gx[0]);
            const int fj = tspan - t.p;
            if (j < fj || j > fj + t.p) continue;
            double part = 0.0;
            for (int g = 0; g < ng; ++g) {
                const double x = mid + half * gx[g];
                double Ni[kMaxP + 1], Nj[kMaxP + 1];
                basis_funs_rt(s.knots, s.p, s.espan[e], x, Ni);
                basis_funs_rt(t.knots, t.p, tspan, x, Nj);
                part += Ni[i - fi] * Nj[j - fj] * (half * gw[g]);
            }
            acc += part;
        }
        M[idx] = acc;
    }
}

}  // namespace tq

using namespace tq;

extern "C" int tq_mass_1d_mixed(tq_space1d test, tq_space1d trial, const double* gx, const double* gw,
                                int32_t ng, double* M, void* stream) {
    if (test.p > kMaxP || trial.p > kMaxP) { set_error("degree unsupported (max %d)", kMaxP); return TQ_EINVAL; }
    if (test.nel != trial.nel) {
        set_error("test and trial spaces must share the breakpoints (%d vs %d elements)", test.nel, trial.nel);
        return TQ_EINVAL;
    }
    const int64_t total = (int64_t)test.n * trial.n;
    if (total == 0) return TQ_OK;
    k_mass_mixed<<<grid_for(total, 128), 128, 0, S(stream)>>>(test, trial, gx, gw, ng, M); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_mass_mixed");
    return TQ_OK;
}

extern "C" int tq_basis_eval(tq_space1d s, const double* u, int64_t n, int32_t* first,
                             double* vals, double* ders, int32_t* status, void* stream) {
    if (n == 0) return TQ_OK;
    if (s.p < 0 || s.p > kMaxP) { set_error("degree %d unsupported (max %d)", s.p, kMaxP); return TQ_EINVAL; }
    int grid = grid_for(n, 256);
    const size_t kbytes = sizeof(double) * (size_t)s.nknots;
    const int staged = kbytes <= 32 * 1024;
    const size_t shm = staged ? kbytes : 0;
    switch (s.p) {
#define CASE(P) case P: k_basis_eval<P><<<grid, 256, shm, S(stream)>>>(s, u, n, first, vals, ders, status, staged); ::tq::note_launch(); break;
        CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
    }
    TQ_LAUNCH_CHECK("k_basis_eval");
    return TQ_OK;
}

extern "C" int tq_basis_eval_multi(const tq_evalbatch* batch_h, void* stream) {
    tq_evalbatch B = *batch_h;
    if (B.ntasks <= 0) return TQ_OK;
    if (B.ntasks > TQ_EVAL_MAX_TASKS) { set_error("tq_basis_eval_multi: %d tasks", B.ntasks); return TQ_EINVAL; }
    const int p = B.task[0].s.p;
    size_t stage = 0;
    B.block_start[0] = 0;
    for (int k = 0; k < B.ntasks; ++k) {
        if (B.task[k].s.p != p) { set_error("tq_basis_eval_multi: tasks of one degree only"); return TQ_EINVAL; }
        const int64_t nb = std::max<int64_t>(1, std::min<int64_t>((B.task[k].n + 255) / 256, 4 * 148));
        B.block_start[k + 1] = B.block_start[k] + (int)nb;
        stage = std::max(stage, (size_t)B.task[k].s.nknots * sizeof(double));
    }
    if (p < 0 || p > kMaxP) { set_error("degree %d unsupported", p); return TQ_EINVAL; }
    // a block evaluates ~256 points (one per thread): staging the knots pays
    // only while they are few; large knot vectors are read through L1 (the
    // staging of 2053 knots per block dominated the launch at config 5)
    static const size_t stage_max = getenv("TQ_BASIS_STAGE_MAX") ? (size_t)atol(getenv("TQ_BASIS_STAGE_MAX"))
                                                                  : 512 * sizeof(double);
    if (stage > stage_max) stage = 0;
    B.stage_bytes = (int32_t)stage;
    const int grid = B.block_start[B.ntasks];
    switch (p) {
#define CASE(P) case P: k_basis_eval_multi<P><<<grid, 256, stage, S(stream)>>>(B); ::tq::note_launch(); break;
        CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
    }
    TQ_LAUNCH_CHECK("k_basis_eval_multi");
    return TQ_OK;
}

extern "C" int tq_moments_1d_g(tq_space1d s, const double* gx, const double* gw, int32_t ng,
                               double* mom, void* stream) {
    if (s.p > kMaxP) { set_error("degree %d unsupported", s.p); return TQ_EINVAL; }
    double* tab = nullptr;
    TQ_CUDA(cudaMallocAsync(&tab, sizeof(double) * (size_t)s.nel * ng * (s.p + 2), S(stream)));
    k_gauss_table<<<grid_for((int64_t)s.nel * ng, 128), 128, 0, S(stream)>>>(s, gx, gw, ng, tab); ::tq::note_launch();
    int64_t total = (int64_t)s.n * (2 * s.p + 1);
    k_moments<<<grid_for(total, 128), 128, 0, S(stream)>>>(s, tab, ng, mom); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_moments");
    TQ_CUDA(cudaFreeAsync(tab, S(stream)));
    return TQ_OK;
}
