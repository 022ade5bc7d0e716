// Timeline of the one-launch cluster GEPP (csrc/getrf_full.cu): globaltimer
// stamps per panel on CTA 0 (build with -DRLRA_LU_TRACE; see tools/build_traces.sh).
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
  int64_t m = argc > 1 ? atoll(argv[1]) : 20000, n = argc > 2 ? atoll(argv[2]) : 220;
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
  unsigned long long t0 = t[0];
  auto T = [&](int s) { return t[s] ? (t[s] - t0) / 1e3 : -1.0; };
  printf("panel: start | steps done | sync1 | sync2 | U12 | trailing   (us from panel 0 start, CTA 0)\n");
  for (int p = 0; p * 6 + 5 < 64 && p < 10 && t[p * 6]; p++)
    printf("  %2d: %8.2f %8.2f %8.2f %8.2f %8.2f %8.2f   steps %.2f  inter %.2f\n", p, T(6 * p), T(6 * p + 1),
           T(6 * p + 2), T(6 * p + 3), T(6 * p + 4), T(6 * p + 5), T(6 * p + 1) - T(6 * p),
           (t[6 * p + 5] ? T(6 * p + 5) : T(6 * p + 2)) - T(6 * p + 1));
  printf("steps of panel 0 (CTA 0 / 15, tid 0): pre-wait got mult pre-bar post-red staged(w0) pushed bulk\n");
  for (int b : {0, 15})
    for (int jj = 0; jj < 8; jj++) {
      auto S = [&](int i) { unsigned long long v = t[b * 128 + 64 + 8 * jj + i]; return v ? (v - t0) / 1e3 : -1.0; };
      printf("  cta %2d step %2d: %7.2f %7.2f %7.2f %7.2f %7.2f %7.2f %7.2f %7.2f\n", b, jj, S(0), S(1), S(2), S(3),
             S(4), S(5), S(6), S(7));
    }
  return 0;
}
