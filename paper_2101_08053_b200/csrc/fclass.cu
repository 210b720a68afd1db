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

}  // namespace tq

using namespace tq;

extern "C" int tq_function_classes(tq_space1d s1, tq_space1d s2, const int8_t* elem_class,
                                   int8_t* func_class, int32_t* face1, int32_t* face2, void* stream) {
    int64_t nf = (int64_t)s1.n * s2.n;
    k_func_class<<<grid_for(nf, 256), 256, 0, S(stream)>>>(s1, s2, elem_class, func_class);
    int64_t ne = (int64_t)s1.nel * s2.nel;
    k_faces<<<grid_for(ne, 256), 256, 0, S(stream)>>>(s1.nel, s2.nel, elem_class, face1, face2);
    TQ_LAUNCH_CHECK("k_func_class/k_faces");
    return TQ_OK;
}
