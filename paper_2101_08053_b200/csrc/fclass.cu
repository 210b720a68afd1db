// Subsystem (2), integer part: function classes and discontinuity faces.
//
//  tq_function_classes <- TrimConfiguration.__init__  src/trimming.py:441-484
//    func class: CUT if any cut element in the support or the support mixes
//    interior and non-interior elements; INTERIOR if all interior; else
//    EXTERIOR.  face flags: a breakpoint separating a (CUT, INTERIOR) pair.
#include "common.cuh"

namespace tq {

__global__ void k_func_class(tq_space1d s1, tq_space1d s2, const int8_t* __restrict__ ec,
                             int8_t* __restrict__ fc) {
    int64_t total = (int64_t)s1.n * s2.n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int i1 = (int)(t / s2.n), i2 = (int)(t % s2.n);
        int a1 = s1.el_first[i1], b1 = s1.el_last[i1];
        int a2 = s2.el_first[i2], b2 = s2.el_last[i2];
        int n_int = 0, n_cut = 0;
        for (int e1 = a1; e1 <= b1; ++e1)
            for (int e2 = a2; e2 <= b2; ++e2) {
                int8_t c = ec[(int64_t)e1 * s2.nel + e2];
                n_int += (c == TQ_INTERIOR);
                n_cut += (c == TQ_CUT);
            }
        int total_el = (b1 - a1 + 1) * (b2 - a2 + 1);
        int8_t cls = TQ_EXTERIOR;
        if (n_cut > 0 || (n_int > 0 && n_int < total_el)) cls = TQ_CUT;
        else if (n_int == total_el) cls = TQ_INTERIOR;
        fc[t] = cls;
    }
}

__device__ inline bool mixed_pair(int8_t a, int8_t b) {
    return (a == TQ_CUT && b == TQ_INTERIOR) || (a == TQ_INTERIOR && b == TQ_CUT);
}

__global__ void k_faces(int nel1, int nel2, const int8_t* __restrict__ ec, int32_t* face1, int32_t* face2) {
    int64_t total = (int64_t)nel1 * nel2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int e1 = (int)(t / nel2), e2 = (int)(t % nel2);
        int8_t c = ec[t];
        if (e1 + 1 < nel1 && mixed_pair(c, ec[t + nel2])) face1[e1] = 1;
        if (e2 + 1 < nel2 && mixed_pair(c, ec[t + 1])) face2[e2] = 1;
    }
}

// DWQ routing of one cut row (src/trimming.py:545-586)
__device__ inline bool all_interior(const int8_t* ec, int nel2, int a1, int b1, int a2, int b2) {
    if (b1 < a1 || b2 < a2) return false;
    for (int e1 = a1; e1 <= b1; ++e1)
        for (int e2 = a2; e2 <= b2; ++e2)
            if (ec[(int64_t)e1 * nel2 + e2] != TQ_INTERIOR) return false;
    return true;
}

__device__ inline int nearest_bp(const double* bp, int nb, double u) {
    int best = 0;
    double bd = fabs(bp[0] - u);
    for (int k = 1; k < nb; ++k) {
        double d = fabs(bp[k] - u);
        if (d < bd) { bd = d; best = k; }
    }
    return best;
}

__global__ void k_dwq_route(tq_space1d s1, tq_space1d s2, const int8_t* __restrict__ ec,
                            const double* __restrict__ u1, int nu1, const double* __restrict__ u2, int nu2,
                            const int32_t* __restrict__ rows, int nrows, int32_t* __restrict__ route) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
        int idx = rows[r];
        int i1 = idx / s2.n, i2 = idx - (idx / s2.n) * s2.n;
        int a1 = s1.el_first[i1], e1 = s1.el_last[i1], a2 = s2.el_first[i2], e2 = s2.el_last[i2];
        double lo1 = s1.knots[i1], hi1 = s1.knots[i1 + s1.p + 1];
        double lo2 = s2.knots[i2], hi2 = s2.knots[i2 + s2.p + 1];
        int c1 = -1, n1 = 0, c2 = -1, n2 = 0;
        for (int k = 0; k < nu1; ++k)
            if (lo1 + 1e-12 < u1[k] && u1[k] < hi1 - 1e-12) { if (n1 == 0) c1 = k; ++n1; }
        for (int k = 0; k < nu2; ++k)
            if (lo2 + 1e-12 < u2[k] && u2[k] < hi2 - 1e-12) { if (n2 == 0) c2 = k; ++n2; }
        int32_t* out = route + 8 * (int64_t)r;
        for (int q = 0; q < 8; ++q) out[q] = -1;
        if (n1 > 1 || n2 > 1) { out[0] = 0; continue; }
        // options per direction: (lo, hi, used-u index)
        int o1lo[2], o1hi[2], o1u[2], no1 = 0, o2lo[2], o2hi[2], o2u[2], no2 = 0;
        if (c1 < 0) { o1lo[0] = a1; o1hi[0] = e1; o1u[0] = -1; no1 = 1; }
        else {
            int k = nearest_bp(s1.bp, s1.nel + 1, u1[c1]);
            if (k - 1 >= a1) { o1lo[no1] = a1; o1hi[no1] = k - 1; o1u[no1] = c1; ++no1; }
            if (k <= e1) { o1lo[no1] = k; o1hi[no1] = e1; o1u[no1] = c1; ++no1; }
        }
        if (c2 < 0) { o2lo[0] = a2; o2hi[0] = e2; o2u[0] = -1; no2 = 1; }
        else {
            int k = nearest_bp(s2.bp, s2.nel + 1, u2[c2]);
            if (k - 1 >= a2) { o2lo[no2] = a2; o2hi[no2] = k - 1; o2u[no2] = c2; ++no2; }
            if (k <= e2) { o2lo[no2] = k; o2hi[no2] = e2; o2u[no2] = c2; ++no2; }
        }
        int best = -1, bcnt = 0;
        for (int x = 0; x < no1; ++x)
            for (int y = 0; y < no2; ++y) {
                if (!all_interior(ec, s2.nel, o1lo[x], o1hi[x], o2lo[y], o2hi[y])) continue;
                int cnt = (o1hi[x] - o1lo[x] + 1) * (o2hi[y] - o2lo[y] + 1);
                if (best < 0 || cnt > bcnt) { best = x * 2 + y; bcnt = cnt; }
            }
        out[0] = 1;
        if (best >= 0) {
            int x = best / 2, y = best % 2;
            out[1] = o1u[x]; out[2] = o2u[y];
            out[3] = o1lo[x]; out[4] = o1hi[x]; out[5] = o2lo[y]; out[6] = o2hi[y];
        }
    }
}

}  // namespace tq

using namespace tq;

extern "C" int tq_dwq_route(tq_space1d s1, tq_space1d s2, const int8_t* elem_class, const double* udisc1,
                            int32_t nu1, const double* udisc2, int32_t nu2, const int32_t* cut_rows,
                            int32_t ncut, int32_t* route, void* stream) {
    if (ncut == 0) return TQ_OK;
    k_dwq_route<<<grid_for(ncut, 128), 128, 0, S(stream)>>>(s1, s2, elem_class, udisc1, nu1, udisc2, nu2,
                                                            cut_rows, ncut, route); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_dwq_route");
    return TQ_OK;
}

extern "C" int tq_function_classes(tq_space1d s1, tq_space1d s2, const int8_t* elem_class,
                                   int8_t* func_class, int32_t* face1, int32_t* face2, void* stream) {
    int64_t nf = (int64_t)s1.n * s2.n;
    k_func_class<<<grid_for(nf, 256), 256, 0, S(stream)>>>(s1, s2, elem_class, func_class); ::tq::note_launch();
    int64_t ne = (int64_t)s1.nel * s2.nel;
    k_faces<<<grid_for(ne, 256), 256, 0, S(stream)>>>(s1.nel, s2.nel, elem_class, face1, face2); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_func_class/k_faces");
    return TQ_OK;
}
