// K6: triangular solves of the single-pass tail and the pseudoinverse check.
//   X = R^{-T} B  (R upper l x l): kernels.pinv_transpose_apply
//   (rlra/kernels.py:92-96, SciPy solve_triangular(trans='T')), blocked: a DMMA
//   GEMM update per 32-row block, then forward substitution on the diagonal block.
//   min_i |R_ii| for pinv_factor's rank test (rlra/kernels.py:75-79).
#include "common.cuh"

namespace rlra {

int gemm(bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
         void* ws, size_t ws_bytes, cudaStream_t st);

constexpr int TRSM_NB = 32;

// Solve R_bb^T X_b = X_b in place, R_bb the nb x nb diagonal block at (i0, i0).
__global__ void trsm_rt_diag_kernel(const double* __restrict__ r, int64_t ldr, int64_t i0, int nb,
                                    double* x, int64_t ldx, int64_t ncols) {
  __shared__ double R[TRSM_NB][TRSM_NB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    int a = e % nb, b = e / nb;
    R[a][b] = r[cm(i0 + a, i0 + b, ldr)];
  }
  __syncthreads();
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncols;
       c += (int64_t)gridDim.x * blockDim.x) {
    double v[TRSM_NB];
    double* col = x + cm(i0, c, ldx);
#pragma unroll
    for (int s = 0; s < TRSM_NB; s++) v[s] = s < nb ? col[s] : 0.0;
#pragma unroll
    for (int s = 0; s < TRSM_NB; s++) {
      if (s >= nb) break;
      double acc = v[s];
#pragma unroll
      for (int t = 0; t < TRSM_NB; t++)
        if (t < s) acc -= R[t][s] * v[t];
      v[s] = acc / R[s][s];
    }
#pragma unroll
    for (int s = 0; s < TRSM_NB; s++)
      if (s < nb) col[s] = v[s];
  }
}

// X (l x ncols, in place over B) = R^{-T} B, R upper triangular l x l.
int trsm_rt(const double* r, int64_t ldr, int64_t l, double* x, int64_t ldx, int64_t ncols,
            void* ws, size_t ws_bytes, cudaStream_t st) {
  if (l <= 0 || ncols <= 0) return 0;
  for (int64_t i0 = 0; i0 < l; i0 += TRSM_NB) {
    const int nb = (int)std::min<int64_t>(TRSM_NB, l - i0);
    if (i0 > 0) {
      // X_b -= R(0:i0, b)^T X(0:i0, :)
      if (gemm(true, false, nb, ncols, i0, -1.0, r + cm(0, i0, ldr), ldr, x, ldx, 1.0,
               x + cm(i0, 0, ldx), ldx, ws, ws_bytes, st))
        return -1;
    }
    int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(ncols, 64), 1024));
    trsm_rt_diag_kernel<<<blocks, 64, 0, st>>>(r, ldr, i0, nb, x, ldx, ncols);
    RLRA_LAUNCHED();
  }
  return 0;
}

// Solve R_bb X_b = X_b in place (backward substitution), R_bb the nb x nb
// diagonal block at (i0, i0) of the upper-triangular R.
__global__ void trsm_un_diag_kernel(const double* __restrict__ r, int64_t ldr, int64_t i0, int nb,
                                    double* x, int64_t ldx, int64_t ncols) {
  __shared__ double R[TRSM_NB][TRSM_NB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    int a = e % nb, b = e / nb;
    R[a][b] = r[cm(i0 + a, i0 + b, ldr)];
  }
  __syncthreads();
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncols;
       c += (int64_t)gridDim.x * blockDim.x) {
    double v[TRSM_NB];
    double* col = x + cm(i0, c, ldx);
#pragma unroll
    for (int s = 0; s < TRSM_NB; s++) v[s] = s < nb ? col[s] : 0.0;
#pragma unroll
    for (int s = TRSM_NB - 1; s >= 0; s--) {
      if (s >= nb) continue;
      double acc = v[s];
#pragma unroll
      for (int t = 0; t < TRSM_NB; t++)
        if (t > s && t < nb) acc -= R[s][t] * v[t];
      v[s] = acc / R[s][s];
    }
#pragma unroll
    for (int s = 0; s < TRSM_NB; s++)
      if (s < nb) col[s] = v[s];
  }
}

// X (l x ncols, in place over B) = R^{-1} B, R upper triangular l x l
// (SciPy solve_triangular(R, B, lower=False), rlra/fixedrank.py:113); blocks
// from the bottom: X_b -= R(b, below) X(below, :) on the DMMA pipe, then the
// diagonal block.
int trsm_un(const double* r, int64_t ldr, int64_t l, double* x, int64_t ldx, int64_t ncols,
            void* ws, size_t ws_bytes, cudaStream_t st) {
  if (l <= 0 || ncols <= 0) return 0;
  const int64_t nblk = ceil_div(l, TRSM_NB);
  for (int64_t b = nblk - 1; b >= 0; b--) {
    const int64_t i0 = b * TRSM_NB;
    const int nb = (int)std::min<int64_t>(TRSM_NB, l - i0);
    const int64_t i1 = i0 + nb;
    if (i1 < l) {
      if (gemm(false, false, nb, ncols, l - i1, -1.0, r + cm(i0, i1, ldr), ldr, x + cm(i1, 0, ldx), ldx, 1.0,
               x + cm(i0, 0, ldx), ldx, ws, ws_bytes, st))
        return -1;
    }
    int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(ncols, 64), 1024));
    trsm_un_diag_kernel<<<blocks, 64, 0, st>>>(r, ldr, i0, nb, x, ldx, ncols);
    RLRA_LAUNCHED();
  }
  return 0;
}

__global__ void diag_absmin_kernel(const double* a, int64_t lda, int64_t r, double* out) {
  __shared__ double s[32];
  double mn = INFINITY;
  for (int64_t i = threadIdx.x; i < r; i += blockDim.x) mn = fmin(mn, fabs(a[cm(i, i, lda)]));
#pragma unroll
  for (int off = 16; off; off >>= 1) mn = fmin(mn, __shfl_down_sync(0xffffffffu, mn, off));
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) m = fmin(m, s[w]);
    *out = m;
  }
}

int diag_absmin(const double* a, int64_t lda, int64_t r, double* out_dev, cudaStream_t st) {
  diag_absmin_kernel<<<1, 256, 0, st>>>(a, lda, r, out_dev);
  RLRA_LAUNCHED();
  return 0;
}

}  // namespace rlra
