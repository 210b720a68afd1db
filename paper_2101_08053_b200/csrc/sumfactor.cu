// tq_sum_factor_rows <- sum_factor_row (src/assembly.py:218-252), batched:
// the public per-row sum factorisation with caller-supplied collocation
// slices, weight rows and coefficient window (the formation pipeline itself
// uses the fused raw-row kernels of rawrows.cu; this entry point serves the
// reference's lower-level API and its tests).
//
// Row r (dims[4r..4r+3] = n1, n2, t1, t2; offs[7r..7r+6] into `data` / `out`
// / `scratch`):
//   B1 = C1 (n1 x t1) * w1[:, None]          C1 at offs[0], w1 at offs[1]
//   B2 = C2 (n2 x t2) * w2[:, None]          C2 at offs[2], w2 at offs[3]
//   G  = grid window (n1 x n2) [* mask]      G  at offs[4], mask at offs[5] (< 0: none)
//   inner = B2^T G^T   (t2 x n1)             scratch at offs[6]
//   block = B1^T inner^T  (t1 x t2)          out at the row's prefix t1*t2
// One block per row; the two contractions are separated by a block barrier.
#include "common.cuh"

namespace tq {

__global__ void k_sum_factor_rows(int32_t nrows, const int32_t* __restrict__ dims, const int64_t* __restrict__ offs,
                                  const int64_t* __restrict__ out_off, const double* __restrict__ data,
                                  double* __restrict__ scratch, double* __restrict__ out) {
    for (int r = blockIdx.x; r < nrows; r += gridDim.x) {
        const int n1 = dims[4 * r], n2 = dims[4 * r + 1], t1 = dims[4 * r + 2], t2 = dims[4 * r + 3];
        const int64_t* o = offs + 7 * (int64_t)r;
        const double* C1 = data + o[0];
        const double* w1 = data + o[1];
        const double* C2 = data + o[2];
        const double* w2 = data + o[3];
        const double* G = data + o[4];
        const double* mask = o[5] >= 0 ? data + o[5] : nullptr;
        double* inner = scratch + o[6];
        double* blk = out + out_off[r];
        // inner[o2][k1] = sum_k2 (C2[k2][o2] w2[k2]) * (G[k1][k2] mask[k1][k2])
        for (int idx = threadIdx.x; idx < t2 * n1; idx += blockDim.x) {
            const int o2 = idx / n1, k1 = idx - o2 * n1;
            double s = 0.0;
            for (int k2 = 0; k2 < n2; ++k2) {
                double g = G[(int64_t)k1 * n2 + k2];
                if (mask) g = g * mask[(int64_t)k1 * n2 + k2];
                s += (C2[(int64_t)k2 * t2 + o2] * w2[k2]) * g;
            }
            inner[idx] = s;
        }
        __syncthreads();
        // block[o1][o2] = sum_k1 (C1[k1][o1] w1[k1]) * inner[o2][k1]
        for (int idx = threadIdx.x; idx < t1 * t2; idx += blockDim.x) {
            const int o1 = idx / t2, o2 = idx - o1 * t2;
            double s = 0.0;
            for (int k1 = 0; k1 < n1; ++k1) s += (C1[(int64_t)k1 * t1 + o1] * w1[k1]) * inner[(int64_t)o2 * n1 + k1];
            blk[idx] = s;
        }
        __syncthreads();
    }
}

}  // namespace tq

using namespace tq;

extern "C" int tq_sum_factor_rows(int32_t nrows, const int32_t* dims, const int64_t* offs, const int64_t* out_off,
                                  const double* data, double* scratch, double* out, void* stream) {
    if (nrows <= 0) return TQ_OK;
    const int blocks = nrows < 4 * 148 ? nrows : 4 * 148;
    k_sum_factor_rows<<<blocks, 128, 0, S(stream)>>>(nrows, dims, offs, out_off, data, scratch, out);
    ::tq::note_launch();
    TQ_LAUNCH_CHECK("k_sum_factor_rows");
    return TQ_OK;
}
