// FP64 pipe micro-benchmark for B200 (sm_100a): DMMA shapes vs DFMA vs DMUL+DADD,
// plus a cooperative grid-barrier latency probe.  Used to pick the roofline
// denominator and the GEMM instruction.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_mma884(double* out, int iters) {
  double c[8][2];
  for (int i = 0; i < 8; i++) c[i][0] = c[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_mma16816(double* out, int iters) {
  double c[4][4];
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) c[i][j] = 0.0;
  double a[8], b[4];
  for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; i++) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) s += c[i][j];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_mma1684(double* out, int iters) {
  double c[8][4];
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) c[i][j] = 0.0;
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) s += c[i][j];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_dfma(double* out, int iters) {
  double c[16];
  for (int i = 0; i < 16; i++) c[i] = i;
  double a = 1.0 - threadIdx.x * 1e-9, b = 1e-9 * threadIdx.x;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) c[i] = fma(c[i], a, b);
  }
  double s = 0; for (int i = 0; i < 16; i++) s += c[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_dmuladd(double* out, int iters) {
  double c[16];
  for (int i = 0; i < 16; i++) c[i] = i;
  double a = 1.0 - threadIdx.x * 1e-9, b = 1e-9 * threadIdx.x;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) c[i] = __dsub_rn(c[i], __dmul_rn(b, a));
  }
  double s = 0; for (int i = 0; i < 16; i++) s += c[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_gridsync(int* out, int iters) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; i++) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}

__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <typename F>
float timeit(F f, int reps) {
  cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(s);
  for (int i = 0; i < reps; i++) f();
  cudaEventRecord(e); cudaEventSynchronize(e);
  float ms; cudaEventElapsedTime(&ms, s, e);
  return ms / reps;
}

int main() {
  double* out; CK(cudaMalloc(&out, 64));
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", nsm, clk);
  int iters = 4096;
  for (int bpsm = 1; bpsm <= 4; bpsm *= 2)
    for (int threads = 128; threads <= 512; threads *= 2) {
      int grid = nsm * bpsm;
      float ms = timeit([&] { k_mma884<<<grid, threads>>>(out, iters); }, 5);
      double fl = 2.0 * 8 * 8 * 4 * 8.0 * iters * (threads / 32) * grid;
      printf("mma m8n8k4   grid %4d thr %3d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, fl / ms / 1e9);
      ms = timeit([&] { k_mma1684<<<grid, threads>>>(out, iters); }, 5);
      fl = 2.0 * 16 * 8 * 4 * 8.0 * iters * (threads / 32) * grid;
      printf("mma m16n8k4  grid %4d thr %3d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, fl / ms / 1e9);
      ms = timeit([&] { k_mma16816<<<grid, threads>>>(out, iters / 4); }, 5);
      fl = 2.0 * 16 * 8 * 16 * 4.0 * (iters / 4) * (threads / 32) * grid;
      printf("mma m16n8k16 grid %4d thr %3d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, fl / ms / 1e9);
      ms = timeit([&] { k_dfma<<<grid, threads>>>(out, iters); }, 5);
      fl = 2.0 * 16 * iters * (double)threads * grid;
      printf("dfma         grid %4d thr %3d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, fl / ms / 1e9);
      ms = timeit([&] { k_dmuladd<<<grid, threads>>>(out, iters); }, 5);
      fl = 2.0 * 16 * iters * (double)threads * grid;
      printf("dmul+dsub    grid %4d thr %3d: %.3f ms  %.2f TFLOP/s (2 flop per mul+sub)\n", grid, threads, ms, fl / ms / 1e9);
    }
  // sustained: long DMMA loop (~2 s)
  {
    int grid = nsm * 2, threads = 256;
    float ms = timeit([&] { k_mma16816<<<grid, threads>>>(out, 262144); }, 3);
    double fl = 2.0 * 16 * 8 * 16 * 4.0 * 262144 * (threads / 32) * grid;
    printf("SUSTAINED mma m16n8k16 grid %d thr %d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, fl / ms / 1e9);
    ms = timeit([&] { k_dfma<<<grid, threads>>>(out, 262144 * 8); }, 3);
    fl = 2.0 * 16 * 262144.0 * 8 * threads * grid;
    printf("SUSTAINED dfma grid %d thr %d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, fl / ms / 1e9);
  }
  // grid sync latency
  {
    int* iout; CK(cudaMalloc(&iout, 64));
    for (int threads = 128; threads <= 512; threads *= 2) {
      int grid = nsm; int it = 2000;
      void* args[] = {&iout, &it};
      float ms = timeit([&] { cudaLaunchCooperativeKernel((void*)k_gridsync, grid, threads, args, 0, 0); }, 3);
      printf("grid.sync grid %d thr %d: %.3f us per sync\n", grid, threads, ms * 1e3 / it);
    }
    CK(cudaGetLastError());
  }
  // HBM copy of doubles
  {
    size_t n = (size_t)1 << 28; // 2 GiB per buffer of double2? n double2 = 4 GiB; use 1<<27
    n = (size_t)1 << 27;
    double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
    cudaMemset(a, 0, n * 16);
    float ms = timeit([&] { k_copy<<<nsm * 8, 512>>>(a, b, n); }, 10);
    printf("copy %.1f GB: %.3f ms  %.1f GB/s (read+write)\n", n * 32 / 1e9, ms, n * 32.0 / ms / 1e6);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
