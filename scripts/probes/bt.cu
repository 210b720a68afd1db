#include <cstdio>
#include "../../paper_2101_08053_b200/csrc/common.cuh"
namespace tq { void set_error(const char*, ...) {} void note_launch() {} int check_cuda(cudaError_t, const char*) { return 0; } }
__global__ void k(const double* kn, double u, double* out, int p, int n) {
  double N[11], D[11];
  int sp = tq::find_span(kn, n + p + 1, p, n, u);
  tq::basis_funs_ders_rt(kn, p, sp, u, N, D);
  for (int i = 0; i < 4; ++i) { out[i] = N[i]; out[4 + i] = D[i]; }
  out[8] = sp;
}
int main() {
  double h[15] = {0,0,0,0,0.125,0.25,0.375,0.5,0.625,0.75,0.875,1,1,1,1};
  double *kn, *out; cudaMalloc(&kn, 15*8); cudaMalloc(&out, 9*8);
  cudaMemcpy(kn, h, 15*8, cudaMemcpyHostToDevice);
  k<<<1,1>>>(kn, 0.0014465, out, 3, 11);
  double o[9]; cudaMemcpy(o, out, 72, cudaMemcpyDeviceToHost);
  printf("dev span %g N %g %g %g %g D %g %g %g %g\n", o[8], o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7]);
}
