// Timeline of one cluster GEPP panel (globaltimer stamps per CTA and step).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
namespace rlra {
extern unsigned long long* g_lu_trace;
int getrf(double* a, int64_t lda, int64_t m, int64_t n, int64_t* piv, int64_t* nonzero_diag_dev,
          int* zflag_out, void* ws, size_t ws_bytes, cudaStream_t st);
size_t getrf_workspace_bytes(int64_t m, int64_t n);
int fill_iota(int64_t* p, int64_t m, cudaStream_t st);
}
int main(int argc, char** argv) {
  int64_t m = argc > 1 ? atoll(argv[1]) : 10000, n = argc > 2 ? atoll(argv[2]) : 32;
  std::vector<double> h(m * n);
  srand(1);
  for (auto& x : h) x = rand() / (double)RAND_MAX - 0.5;
  double* a; int64_t* piv; void* ws; unsigned long long* tr;
  size_t wb = rlra::getrf_workspace_bytes(m, n);
  cudaMalloc(&a, m * n * 8); cudaMalloc(&piv, m * 8); cudaMalloc(&ws, wb); cudaMalloc(&tr, 16 * 128 * 8);
  for (int rep = 0; rep < 3; rep++) {
    cudaMemcpy(a, h.data(), m * n * 8, cudaMemcpyHostToDevice);
    cudaMemset(tr, 0, 16 * 128 * 8);
    rlra::g_lu_trace = tr;
    rlra::fill_iota(piv, m, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    int rc = rlra::getrf(a, m, m, n, piv, nullptr, nullptr, ws, wb, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("rep %d rc %d getrf %ld x %ld: %.1f us (%s)\n", rep, rc, (long)m, (long)n, ms * 1e3,
           cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<unsigned long long> t(16 * 128);
  cudaMemcpy(t.data(), tr, t.size() * 8, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < 16; b++) if (t[b * 128] && t[b * 128] < t0) t0 = t[b * 128];
  auto T = [&](int b, int s) { return t[b * 128 + s] ? (t[b * 128 + s] - t0) / 1e3 : -1.0; };
  for (int b : {0, 15}) {
    printf("CTA %d: start %.2f before-sync %.2f after-sync %.2f end %.2f exit %.2f\n", b, T(b, 0), T(b, 1), T(b, 2),
           T(b, 126), T(b, 127));
    for (int jj = 0; jj < 6; jj++)
      printf("  step %d: pre %.2f got %.2f synced %.2f lookahead %.2f argmax %.2f pushed %.2f\n", jj, T(b, 8 + 8 * jj),
             T(b, 8 + 8 * jj + 1), T(b, 8 + 8 * jj + 2), T(b, 8 + 8 * jj + 3), T(b, 8 + 8 * jj + 4), T(b, 8 + 8 * jj + 5));
  }
  return 0;
}
