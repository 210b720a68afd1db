// Subsystem (2): trimming-curve / knot-span intersection and element
// classification as an integer pass (compiled with -fmad=false).
//
//  tq_classify_elements <- classify_elements  src/trimming.py:607-733
//    k_nodes    node in/on flags               :625-635
//    k_lines    grid-line sweeps               :644-666
//    k_elements corner/crossing/sampling rule  :667-708
//    k_guard    floating-curve check           :710-731
#include <vector>

#include "common.cuh"
#include "curve_compile.h"

namespace tq {

constexpr int kLineCap = 32;   // accepted hits per (curve, grid line)
constexpr int kStatusHits = 8;

__global__ void k_nodes(const CurveC* __restrict__ cv, int nc, tq_space1d s1, tq_space1d s2,
                        uint8_t* __restrict__ flags) {
    const int N2 = s2.nel + 1;
    int64_t total = (int64_t)(s1.nel + 1) * N2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int i = (int)(t / N2), j = (int)(t - (int64_t)i * N2);
        double x = s1.bp[i], y = s2.bp[j];
        bool in = true, on = false;
        for (int c = 0; c < nc; ++c) {
            double sd = curve_signed_distance(cv[c], x, y);
            on = on || fabs(sd) <= kOnCurveTol;
            in = in && sd >= -kOnCurveTol;
        }
        flags[t] = (in ? 1 : 0) | (on ? 2 : 0);
    }
}

// one thread per (curve, grid line); accepted hits stored with their cell
__global__ void k_lines(const CurveC* __restrict__ cv, int nc, tq_space1d s1, tq_space1d s2,
                        double* __restrict__ hcoord, int32_t* __restrict__ hcell, int32_t* __restrict__ hcount,
                        int32_t* status) {
    const int L = (s1.nel + 1) + (s2.nel + 1);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nc * L; t += gridDim.x * blockDim.x) {
        int c = t / L, l = t - c * L;
        int axis = l <= s1.nel ? 0 : 1;
        double level = axis == 0 ? s1.bp[l] : s2.bp[l - (s1.nel + 1)];
        const double* obp = axis == 0 ? s2.bp : s1.bp;
        int onel = axis == 0 ? s2.nel : s1.nel;
        double ht[kMaxHits], hc[kMaxHits];
        int ovf = 0;
        int nh = curve_intersect_line(cv[c], axis, level, ht, hc, kMaxHits, &ovf);
        int acc = 0;
        for (int q = 0; q < nh; ++q) {
            if (curve_is_tangential(cv[c], ht[q], axis)) continue;
            double y = hc[q];
            int j = lower_bound_d(obp, onel + 1, y) - 1;   // searchsorted(side=left) - 1
            bool touch = false;
            if (j >= 0 && fabs(obp[j] - y) <= kOnCurveTol) touch = true;
            if (j + 1 <= onel && fabs(obp[j + 1] - y) <= kOnCurveTol) touch = true;
            if (j + 2 <= onel && fabs(obp[j + 2] - y) <= kOnCurveTol) touch = true;
            if (touch) continue;
            if (j >= 0 && j < onel) {
                if (acc < kLineCap) {
                    hcoord[(int64_t)t * kLineCap + acc] = y;
                    hcell[(int64_t)t * kLineCap + acc] = j;
                    ++acc;
                } else {
                    ovf = 1;
                }
            }
        }
        hcount[t] = acc;
        if (ovf) atomicOr(status, kStatusHits);
    }
}

struct Dedup {
    bool have = false, two = false;
    double x0 = 0.0, y0 = 0.0, snap = 0.0;
    __device__ void add(double x, double y) {
        if (two) return;
        if (!have) { have = true; x0 = x; y0 = y; return; }
        if (fmax(fabs(x - x0), fabs(y - y0)) > snap) two = true;
    }
};

__global__ void k_elements(const CurveC* __restrict__ cv, int nc, tq_space1d s1, tq_space1d s2,
                           const uint8_t* __restrict__ flags, const double* __restrict__ hcoord,
                           const int32_t* __restrict__ hcell, const int32_t* __restrict__ hcount,
                           int8_t* __restrict__ ec) {
    const int N2 = s2.nel + 1;
    const int L = (s1.nel + 1) + (s2.nel + 1);
    int64_t total = (int64_t)s1.nel * s2.nel;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int e1 = (int)(t / s2.nel), e2 = (int)(t - (int64_t)e1 * s2.nel);
        uint8_t f00 = flags[(int64_t)e1 * N2 + e2], f01 = flags[(int64_t)e1 * N2 + e2 + 1];
        uint8_t f10 = flags[(int64_t)(e1 + 1) * N2 + e2], f11 = flags[(int64_t)(e1 + 1) * N2 + e2 + 1];
        int n_in = (f00 & 1) + (f01 & 1) + (f10 & 1) + (f11 & 1);
        bool mixed = n_in > 0 && n_in < 4;
        double x0 = s1.bp[e1], x1 = s1.bp[e1 + 1], y0 = s2.bp[e2], y1 = s2.bp[e2 + 1];
        double hx = x1 - x0, hy = y1 - y0;
        Dedup dd;
        dd.snap = 1e-10 * fmax(hx, hy);
        int npts = 0;
        for (int c = 0; c < nc; ++c) {
            // vertical lines e1 then e1+1, horizontal lines e2 then e2+1
            for (int side = 0; side < 4; ++side) {
                int l = side == 0 ? e1 : side == 1 ? e1 + 1 : (s1.nel + 1) + e2 + (side - 2);
                int want = side < 2 ? e2 : e1;
                int64_t base = ((int64_t)c * L + l) * kLineCap;
                int cnt = hcount[(int64_t)c * L + l];
                for (int q = 0; q < cnt; ++q) {
                    if (hcell[base + q] != want) continue;
                    double v = hcoord[base + q];
                    double px = side == 0 ? x0 : side == 1 ? x1 : v;
                    double py = side < 2 ? v : (side == 2 ? y0 : y1);
                    dd.add(px, py);
                    ++npts;
                }
            }
        }
        // nodes on a curve, row-major node order
        if (f00 & 2) { dd.add(x0, y0); ++npts; }
        if (f01 & 2) { dd.add(x0, y1); ++npts; }
        if (f10 & 2) { dd.add(x1, y0); ++npts; }
        if (f11 & 2) { dd.add(x1, y1); ++npts; }
        int8_t cls;
        if (!mixed && npts == 0) {
            cls = n_in == 4 ? TQ_INTERIOR : TQ_EXTERIOR;
        } else if (dd.two) {
            cls = TQ_CUT;
        } else {
            const double fx[5] = {0.5, 0.25, 0.75, 0.25, 0.75};
            const double fy[5] = {0.5, 0.25, 0.25, 0.75, 0.75};
            int nin = 0;
            for (int k = 0; k < 5; ++k) {
                double sx = x0 + hx * fx[k], sy = y0 + hy * fy[k];
                bool ok = true;
                for (int c = 0; c < nc; ++c) ok = ok && curve_is_inside(cv[c], sx, sy);
                nin += ok;
            }
            cls = nin == 5 ? TQ_INTERIOR : (nin == 0 ? TQ_EXTERIOR : TQ_CUT);
        }
        ec[t] = cls;
    }
}

__global__ void k_guard(const CurveC* __restrict__ cv, int nc, tq_space1d s1, tq_space1d s2,
                        const int8_t* __restrict__ ec, int32_t* status) {
    const int S = 511;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nc * S; t += gridDim.x * blockDim.x) {
        int c = t / S, k = t - c * S;
        double tt = (k + 1) / 512.0;   // np.linspace(0, 1, 513)[1:-1]
        double x, y;
        curve_eval(cv[c], tt, x, y);
        int e1 = upper_bound_d(s1.bp, s1.nel + 1, x) - 1;
        int e2 = upper_bound_d(s2.bp, s2.nel + 1, y) - 1;
        e1 = e1 < 0 ? 0 : (e1 > s1.nel - 1 ? s1.nel - 1 : e1);
        e2 = e2 < 0 ? 0 : (e2 > s2.nel - 1 ? s2.nel - 1 : e2);
        if (ec[(int64_t)e1 * s2.nel + e2] == TQ_CUT) continue;
        double x0 = s1.bp[e1], x1 = s1.bp[e1 + 1], y0 = s2.bp[e2], y1 = s2.bp[e2 + 1];
        double mg = 1e-9 * fmax(x1 - x0, y1 - y0);
        if (x0 + mg < x && x < x1 - mg && y0 + mg < y && y < y1 - mg) atomicOr(status, kStatusTrim);
    }
}

}  // namespace tq

using namespace tq;

extern "C" int tq_classify_elements(const tq_curve* curves_h, int32_t ncurves, tq_space1d s1, tq_space1d s2,
                                    int8_t* elem_class, int32_t* status, void* stream) {
    cudaStream_t st = S(stream);
    std::vector<CurveC> cv;
    std::vector<double> buf;
    if (!compile_curves(curves_h, ncurves, cv, buf)) {
        set_error("unsupported trimming curve kind on the device path");
        return TQ_EINVAL;
    }
    double* dbuf = nullptr;
    CurveC* dcv = nullptr;
    size_t nb = std::max<size_t>(buf.size(), 1);
    TQ_CUDA(cudaMallocAsync(&dbuf, nb * sizeof(double), st));
    TQ_CUDA(cudaMallocAsync(&dcv, cv.size() * sizeof(CurveC), st));
    if (!buf.empty())
        TQ_CUDA(cudaMemcpyAsync(dbuf, buf.data(), buf.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    for (auto& c : cv) c.buf = dbuf;
    TQ_CUDA(cudaMemcpyAsync(dcv, cv.data(), cv.size() * sizeof(CurveC), cudaMemcpyHostToDevice, st));

    const int64_t nn = (int64_t)(s1.nel + 1) * (s2.nel + 1);
    const int L = (s1.nel + 1) + (s2.nel + 1);
    uint8_t* flags = nullptr;
    double* hcoord = nullptr;
    int32_t *hcell = nullptr, *hcount = nullptr;
    TQ_CUDA(cudaMallocAsync(&flags, nn, st));
    TQ_CUDA(cudaMallocAsync(&hcoord, (size_t)ncurves * L * kLineCap * sizeof(double), st));
    TQ_CUDA(cudaMallocAsync(&hcell, (size_t)ncurves * L * kLineCap * sizeof(int32_t), st));
    TQ_CUDA(cudaMallocAsync(&hcount, (size_t)ncurves * L * sizeof(int32_t), st));
    k_nodes<<<grid_for(nn, 128), 128, 0, st>>>(dcv, ncurves, s1, s2, flags); ::tq::note_launch();
    k_lines<<<grid_for((int64_t)ncurves * L, 64), 64, 0, st>>>(dcv, ncurves, s1, s2, hcoord, hcell, hcount,
                                                               status); ::tq::note_launch();
    int64_t ne = (int64_t)s1.nel * s2.nel;
    k_elements<<<grid_for(ne, 128), 128, 0, st>>>(dcv, ncurves, s1, s2, flags, hcoord, hcell, hcount,
                                                  elem_class); ::tq::note_launch();
    k_guard<<<grid_for((int64_t)ncurves * 511, 128), 128, 0, st>>>(dcv, ncurves, s1, s2, elem_class, status); ::tq::note_launch();
    TQ_LAUNCH_CHECK("classify");
    cudaFreeAsync(flags, st);
    cudaFreeAsync(hcoord, st);
    cudaFreeAsync(hcell, st);
    cudaFreeAsync(hcount, st);
    cudaFreeAsync(dbuf, st);
    cudaFreeAsync(dcv, st);
    int32_t hst = 0;
    TQ_CUDA(cudaMemcpyAsync(&hst, status, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    TQ_CUDA(cudaStreamSynchronize(st));
    if (hst & kStatusHits) { set_error("too many curve crossings on one grid line"); return TQ_ETRIM; }
    if (hst & kStatusTrim) {
        set_error("curve passes through an element without crossing its boundary; configuration not supported");
        return TQ_ETRIM;
    }
    return TQ_OK;
}
