// Phase timing of the CholeskyQR2 factorization kernel (csrc/cholqr.cu):
// build variants with -DCHOL_EXP_{NOTRAIL,NODIAG,NOBLKROW,NONEXT} (see
// tools/chol_probe.sh); each prints the mean chol_inv time for l = argv[1].
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
namespace rlra {
#ifdef CHOL_TRACE
void chol_set_trace(unsigned long long* p);
#endif
int chol_inv(double* g, int64_t ldg, int64_t l, double* x, int64_t ldx, int* flag, double cond_limit,
             cudaStream_t st);
}
int main(int argc, char** argv) {
  const int l = argc > 1 ? atoi(argv[1]) : 220, reps = 50;
  std::vector<double> x((size_t)l * l), g((size_t)l * l, 0.0);
  srand(3);
  for (auto& v : x) v = rand() / (double)RAND_MAX - 0.5;
  for (int i = 0; i < l; i++)
    for (int j = 0; j < l; j++) {
      double s = (i == j) ? l : 0.0;
      for (int k = 0; k < l; k++) s += x[k + (size_t)i * l] * x[k + (size_t)j * l];
      g[i + (size_t)j * l] = s;
    }
  double *dg, *dx;
  int* flag;
  cudaMalloc(&dg, (size_t)reps * l * l * 8);
  cudaMalloc(&dx, (size_t)l * l * 8);
  cudaMalloc(&flag, 4);
  cudaMemset(flag, 0, 4);
  for (int r = 0; r < reps; r++) cudaMemcpy(dg + (size_t)r * l * l, g.data(), (size_t)l * l * 8, cudaMemcpyHostToDevice);
  rlra::chol_inv(dg, l, l, dx, l, flag, 1e12, 0);
  cudaDeviceSynchronize();
  for (int r = 0; r < reps; r++) cudaMemcpy(dg + (size_t)r * l * l, g.data(), (size_t)l * l * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; r++) rlra::chol_inv(dg + (size_t)r * l * l, l, l, dx, l, flag, 1e12, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int hf;
  cudaMemcpy(&hf, flag, 4, cudaMemcpyDeviceToHost);
  // R^T R against G on the first copy (meaningful for the ungated build only)
  std::vector<double> rp((size_t)l * (l + 1) / 2);
  cudaMemcpy(rp.data(), dg, rp.size() * 8, cudaMemcpyDeviceToHost);
  double err = 0, nrm = 0;
  for (int i = 0; i < l; i++)
    for (int j = i; j < l; j++) {
      double s = 0;
      for (int k = 0; k <= i; k++) s += rp[(size_t)i * (i + 1) / 2 + k] * rp[(size_t)j * (j + 1) / 2 + k];
      const double d = s - g[i + (size_t)j * l];
      err += d * d;
      nrm += g[i + (size_t)j * l] * g[i + (size_t)j * l];
    }
#ifdef CHOL_TRACE
  {
    unsigned long long* tr;
    cudaMalloc(&tr, 20 * 8 * 8);
    cudaMemset(tr, 0, 20 * 8 * 8);
    rlra::chol_set_trace(tr);
    cudaMemcpy(dg, g.data(), (size_t)l * l * 8, cudaMemcpyHostToDevice);
    rlra::chol_inv(dg, l, l, dx, l, flag, 1e12, 0);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(160);
    cudaMemcpy(h.data(), tr, 160 * 8, cudaMemcpyDeviceToHost);
    const unsigned long long t0 = h[0];
    printf("it: top  blkrow(w0) blkrow(w1) sync2 next diag trail(w1) trail(w15)   [ns from it=-1 top]\n");
    for (int r = 0; r < 20; r++) {
      if (!h[r * 8]) break;
      printf("%3d:", r - 1);
      for (int c = 0; c < 8; c++) printf(" %7lld", h[r * 8 + c] ? (long long)(h[r * 8 + c] - t0) : -1ll);
      printf("\n");
    }
    rlra::chol_set_trace(nullptr);
  }
#endif
  printf("l=%d chol_inv %.1f us flag=%d relerr=%.2e (%s)\n", l, ms * 1e3 / reps, hf, std::sqrt(err / nrm),
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
