// Public predicate entry points of the drop-in: the trimming-curve interface
// (src/trimming.py:69-95 -- evaluate, derivative, signed_distance, is_inside,
// intersect_line) evaluated on the device with the same predicates the
// classifier and the cut-cell decomposition use (curves.cuh; compiled with
// -fmad=false like them, so a point the classifier called inside is inside
// here too).
//
//  tq_curve_eval            <- TrimmingCurve.evaluate / derivative /
//                              signed_distance / is_inside
//  tq_curve_intersect_line  <- TrimmingCurve.intersect_line
#include <vector>

#include "common.cuh"
#include "curve_compile.h"

namespace tq {

__global__ void k_curve_eval(const CurveC* __restrict__ cv, int op, const double* __restrict__ in, int64_t n,
                             double* __restrict__ out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const CurveC& c = cv[0];
        switch (op) {
            case TQ_CURVE_OP_EVALUATE: {
                double x, y;
                curve_eval(c, in[t], x, y);
                out[2 * t] = x;
                out[2 * t + 1] = y;
                break;
            }
            case TQ_CURVE_OP_DERIVATIVE: {
                double dx, dy;
                curve_deriv(c, in[t], dx, dy);
                out[2 * t] = dx;
                out[2 * t + 1] = dy;
                break;
            }
            case TQ_CURVE_OP_SIGNED_DISTANCE:
                out[t] = curve_signed_distance(c, in[2 * t], in[2 * t + 1]);
                break;
            default:
                out[t] = curve_is_inside(c, in[2 * t], in[2 * t + 1]) ? 1.0 : 0.0;
        }
    }
}

__global__ void k_curve_intersect(const CurveC* __restrict__ cv, int axis, double level, int cap,
                                  double* __restrict__ ht, double* __restrict__ hc, int32_t* __restrict__ count) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    double bt[kMaxHits], bc[kMaxHits];
    int ovf = 0;
    int n = curve_intersect_line(cv[0], axis, level, bt, bc, kMaxHits, &ovf);
    int m = n < cap ? n : cap;
    for (int k = 0; k < m; ++k) { ht[k] = bt[k]; hc[k] = bc[k]; }
    count[0] = n;
    count[1] = ovf;
}

// compiled curve tables on the device (freed stream-ordered after use)
struct DevCurve {
    CurveC* cv = nullptr;
    double* buf = nullptr;
};

inline int upload_curve(const tq_curve* curve_h, cudaStream_t st, DevCurve& d) {
    std::vector<CurveC> cv;
    std::vector<double> buf;
    if (!compile_curves(curve_h, 1, cv, buf)) {
        set_error("unsupported trimming curve kind on the device path");
        return TQ_EINVAL;
    }
    size_t nb = std::max<size_t>(buf.size(), 1);
    TQ_CUDA(cudaMallocAsync(&d.buf, nb * sizeof(double), st));
    TQ_CUDA(cudaMallocAsync(&d.cv, sizeof(CurveC), st));
    if (!buf.empty())
        TQ_CUDA(cudaMemcpyAsync(d.buf, buf.data(), buf.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    cv[0].buf = d.buf;
    TQ_CUDA(cudaMemcpyAsync(d.cv, cv.data(), sizeof(CurveC), cudaMemcpyHostToDevice, st));
    return TQ_OK;
}

inline void free_curve(DevCurve& d, cudaStream_t st) {
    cudaFreeAsync(d.cv, st);
    cudaFreeAsync(d.buf, st);
}

}  // namespace tq

using namespace tq;

extern "C" int tq_curve_eval(const tq_curve* curve_h, int32_t op, const double* in, int64_t n, double* out,
                             void* stream) {
    if (op < TQ_CURVE_OP_EVALUATE || op > TQ_CURVE_OP_IS_INSIDE) {
        set_error("tq_curve_eval: unknown op");
        return TQ_EINVAL;
    }
    if (n <= 0) return TQ_OK;
    cudaStream_t st = S(stream);
    DevCurve d;
    int rc = upload_curve(curve_h, st, d);
    if (rc != TQ_OK) return rc;
    k_curve_eval<<<grid_for(n, 128), 128, 0, st>>>(d.cv, op, in, n, out); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_curve_eval");
    free_curve(d, st);
    return TQ_OK;
}

extern "C" int tq_curve_intersect_line(const tq_curve* curve_h, int32_t axis, double level, int32_t cap,
                                       double* ht, double* hc, int32_t* count, void* stream) {
    if (axis != 0 && axis != 1) {
        set_error("tq_curve_intersect_line: axis must be 0 ('v') or 1 ('h')");
        return TQ_EINVAL;
    }
    cudaStream_t st = S(stream);
    DevCurve d;
    int rc = upload_curve(curve_h, st, d);
    if (rc != TQ_OK) return rc;
    k_curve_intersect<<<1, 32, 0, st>>>(d.cv, axis, level, cap, ht, hc, count); ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_curve_intersect");
    free_curve(d, st);
    return TQ_OK;
}
