// Bandwidth-bound helpers on the hot path:
//   * W = P^T L, the row-unpermuted unit-lower factor of an interior GEPP
//     (rlra/rangefinder.py:73-77 -> rlra/core.py:103-109), as a gather through
//     the inverse permutation so the HBM writes stay coalesced;
//   * unit-L / upper-U extraction of a packed LU (rlra/kernels.py:51-53);
//   * compensated (double-double), deterministic sums of squares: ||A||_F^2
//     (rlra/accessors.py:33-34 used at rlra/fixedprec.py:72) and per-column
//     energies of G (rlra/fixedprec.py:75-80, :105-107);
//   * transpose (U = L2^T, rlra/fixedrank.py:146).
#include "common.cuh"

namespace rlra {

// ---------------------------------------------------------------- double-double
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}
__device__ __forceinline__ DD dd_add(DD x, DD y) {
  DD s = two_sum(x.hi, y.hi);
  double lo = s.lo + x.lo + y.lo;
  return two_sum(s.hi, lo);
}
__device__ __forceinline__ DD dd_add_sq(DD acc, double x) {
  double p = x * x;
  double e = fma(x, x, -p);  // exact square = p + e
  DD s = two_sum(acc.hi, p);
  double lo = s.lo + acc.lo + e;
  return two_sum(s.hi, lo);
}
__device__ DD dd_warp_reduce(DD v) {
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    DD o{__shfl_down_sync(0xffffffffu, v.hi, off), __shfl_down_sync(0xffffffffu, v.lo, off)};
    v = dd_add(v, o);
  }
  return v;
}
// block reduce with a fixed tree (deterministic); result valid in thread 0
__device__ DD dd_block_reduce(DD v) {
  __shared__ double s_hi[32], s_lo[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = dd_warp_reduce(v);
  __syncthreads();
  if (lane == 0) { s_hi[warp] = v.hi; s_lo[warp] = v.lo; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    DD w = lane < nw ? DD{s_hi[lane], s_lo[lane]} : DD{0.0, 0.0};
    v = dd_warp_reduce(w);
  }
  return v;
}

// ---------------------------------------------------------------- ||A||_F^2
__global__ void sumsq_partial_kernel(const double* __restrict__ a, int64_t lda, int64_t m,
                                     int64_t n, int64_t cols_per_block, double* partial) {
  const int64_t c0 = blockIdx.x * cols_per_block;
  const int64_t c1 = min(n, c0 + cols_per_block);
  DD acc{0.0, 0.0};
  for (int64_t c = c0; c < c1; c++) {
    const double* col = a + cm(0, c, lda);
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) acc = dd_add_sq(acc, __ldg(col + i));
  }
  acc = dd_block_reduce(acc);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = acc.hi;
    partial[2 * blockIdx.x + 1] = acc.lo;
  }
}
__global__ void dd_finish_kernel(const double* partial, int nparts, double* out) {
  DD acc{0.0, 0.0};
  for (int q = threadIdx.x; q < nparts; q += blockDim.x)
    acc = dd_add(acc, DD{partial[2 * q], partial[2 * q + 1]});
  acc = dd_block_reduce(acc);
  if (threadIdx.x == 0) *out = acc.hi + acc.lo;
}

size_t sumsq_workspace_bytes(int64_t, int64_t n) {
  int64_t parts = std::min<int64_t>(n, (int64_t)device_info().sm_count * 8);
  return (size_t)(parts > 0 ? parts : 1) * 2 * sizeof(double);
}

int sumsq(const double* a, int64_t lda, int64_t m, int64_t n, double* out_dev, void* ws,
          size_t ws_bytes, cudaStream_t st) {
  if (m <= 0 || n <= 0) {
    RLRA_CHECK_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double), st));
    return 0;
  }
  int64_t parts = std::min<int64_t>(n, (int64_t)device_info().sm_count * 8);
  int64_t cpb = ceil_div(n, parts);
  parts = ceil_div(n, cpb);
  RLRA_REQUIRE(ws_bytes >= (size_t)parts * 2 * sizeof(double), "sumsq: workspace too small");
  double* partial = static_cast<double*>(ws);
  sumsq_partial_kernel<<<(unsigned)parts, 512, 0, st>>>(a, lda, m, n, cpb, partial);
  RLRA_LAUNCHED();
  dd_finish_kernel<<<1, 1024, 0, st>>>(partial, (int)parts, out_dev);
  RLRA_LAUNCHED();
  return 0;
}

// ---------------------------------------------------------------- K9 validation residual
// ||A[p, :][:, q] - L U||_F^2 over one block of w columns of L U (rlra/
// fixedrank.py:149-155 with rlra/core.py:56-65, without materialising the
// m x n reconstruction): CTA j takes column j of the block, reads A's column
// q_blk[j] gathered through p (the column, <= 2 MB, stays in L2) and the
// block's column j contiguously; compensated sums, one partial per column.
__global__ void resid_sumsq_kernel(const double* __restrict__ a, int64_t lda, int64_t m,
                                   const int64_t* __restrict__ p, const int64_t* __restrict__ qb,
                                   const double* __restrict__ lu, int64_t ldlu, double* partial) {
  const int64_t j = blockIdx.x;
  const double* acol = a + cm(0, __ldg(qb + j), lda);
  const double* lcol = lu + cm(0, j, ldlu);
  DD acc{0.0, 0.0};
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) acc = dd_add_sq(acc, __ldg(acol + __ldg(p + i)) - lcol[i]);
  acc = dd_block_reduce(acc);
  if (threadIdx.x == 0) {
    partial[2 * j] = acc.hi;
    partial[2 * j + 1] = acc.lo;
  }
}

int resid_sumsq_block(const double* a, int64_t lda, int64_t m, const int64_t* p, const int64_t* qb, int64_t w,
                      const double* lu, int64_t ldlu, double* partial, cudaStream_t st) {
  if (w <= 0) return 0;
  RLRA_REQUIRE(w <= 2147483647 && m >= 1, "resid_sumsq_block: bad shape");
  resid_sumsq_kernel<<<(unsigned)w, 512, 0, st>>>(a, lda, m, p, qb, lu, ldlu, partial);
  RLRA_LAUNCHED();
  return 0;
}

int dd_finish(const double* partial, int64_t nparts, double* out_dev, cudaStream_t st) {
  RLRA_REQUIRE(nparts >= 1 && nparts <= 2147483647, "dd_finish: bad count");
  dd_finish_kernel<<<1, 1024, 0, st>>>(partial, (int)nparts, out_dev);
  RLRA_LAUNCHED();
  return 0;
}

// ---------------------------------------------------------------- sparse products
static int grid_for(int64_t total);

// Y (rows x l, column-major) = S X for S in CSR (rowptr/colidx/vals) and X
// column-major -- SparseAccessor.matmul / rmatmul (rlra/accessors.py:40-64)
// with the CSR of A for A X and the CSR of A^T (= CSC of A) for A^T X.  One
// thread per (row, column of X): consecutive threads take consecutive rows
// (coalesced Y), the row's nonzeros are read in ascending order (fixed
// summation order, deterministic).
__global__ void spmm_csr_kernel(const int64_t* __restrict__ rowptr, const int64_t* __restrict__ colidx,
                                const double* __restrict__ vals, int64_t rows, const double* __restrict__ x,
                                int64_t ldx, int64_t l, double* __restrict__ y, int64_t ldy) {
  const int64_t total = rows * l;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % rows, c = e / rows;
    const double* xc = x + c * ldx;
    double acc = 0.0;
    const int64_t k1 = __ldg(rowptr + r + 1);
    for (int64_t k = __ldg(rowptr + r); k < k1; k++) acc = fma(__ldg(vals + k), __ldg(xc + __ldg(colidx + k)), acc);
    y[r + c * ldy] = acc;
  }
}

int spmm_csr(const int64_t* rowptr, const int64_t* colidx, const double* vals, int64_t rows, const double* x,
             int64_t ldx, int64_t l, double* y, int64_t ldy, cudaStream_t st) {
  if (rows <= 0 || l <= 0) return 0;
  spmm_csr_kernel<<<grid_for(rows * l), 256, 0, st>>>(rowptr, colidx, vals, rows, x, ldx, l, y, ldy);
  RLRA_LAUNCHED();
  return 0;
}

// ---------------------------------------------------------------- column energies
__global__ void colsumsq_kernel(const double* __restrict__ a, int64_t lda, int64_t m, int64_t n,
                                double* out) {
  for (int64_t c = blockIdx.x; c < n; c += gridDim.x) {
    const double* col = a + cm(0, c, lda);
    DD acc{0.0, 0.0};
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) acc = dd_add_sq(acc, __ldg(col + i));
    acc = dd_block_reduce(acc);
    if (threadIdx.x == 0) out[c] = acc.hi + acc.lo;
  }
}

int colsumsq(const double* a, int64_t lda, int64_t m, int64_t n, double* out_dev, cudaStream_t st) {
  if (n <= 0) return 0;
  int blocks = (int)std::min<int64_t>(n, 65535);
  colsumsq_kernel<<<blocks, 256, 0, st>>>(a, lda, m, n, out_dev);
  RLRA_LAUNCHED();
  return 0;
}

// ---------------------------------------------------------------- permutations / extraction
__global__ void inv_perm_kernel(const int64_t* __restrict__ p, int64_t m, int64_t* __restrict__ pinv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    pinv[p[i]] = i;
}

// W[r, c] = L(pinv[r], c) with L the unit-lower factor of the packed LU.
__global__ void lu_basis_kernel(const double* __restrict__ lu, int64_t ldlu, int64_t m, int64_t k,
                                const int64_t* __restrict__ pinv, double* __restrict__ w,
                                int64_t ldw) {
  const int64_t total = m * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % m, c = e / m;
    const int64_t i = __ldg(pinv + r);
    double v = c < i ? __ldg(lu + cm(i, c, ldlu)) : (c == i ? 1.0 : 0.0);
    w[cm(r, c, ldw)] = v;
  }
}

// out[r, c] = x[pinv[r], c], i.e. out[p[i], :] = x[i, :] (rlra/core.py:103-109).
__global__ void row_gather_kernel(const double* __restrict__ x, int64_t ldx, int64_t m, int64_t n,
                                  const int64_t* __restrict__ pinv, double* __restrict__ out, int64_t ldo) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % m, c = e / m;
    out[cm(r, c, ldo)] = __ldg(x + cm(__ldg(pinv + r), c, ldx));
  }
}

__global__ void extract_l_kernel(const double* __restrict__ lu, int64_t ldlu, int64_t m, int64_t k,
                                 double* __restrict__ l, int64_t ldl) {
  const int64_t total = m * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, c = e / m;
    l[cm(i, c, ldl)] = c < i ? lu[cm(i, c, ldlu)] : (c == i ? 1.0 : 0.0);
  }
}

__global__ void extract_u_kernel(const double* __restrict__ lu, int64_t ldlu, int64_t k, int64_t n,
                                 double* __restrict__ u, int64_t ldu) {
  const int64_t total = k * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % k, c = e / k;
    u[cm(i, c, ldu)] = i <= c ? lu[cm(i, c, ldlu)] : 0.0;
  }
}

// out (n x m) = in^T (in m x n), 32x32 smem tiles
__global__ void transpose_kernel(const double* __restrict__ in, int64_t ldi, int64_t m, int64_t n,
                                 double* __restrict__ out, int64_t ldo) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    int64_t r = r0 + threadIdx.x, c = c0 + k;
    if (r < m && c < n) tile[k][threadIdx.x] = in[cm(r, c, ldi)];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    int64_t r = c0 + threadIdx.x, c = r0 + k;  // out(r, c) = in(c, r)
    if (r < n && c < m) out[cm(r, c, ldo)] = tile[threadIdx.x][k];
  }
}

static int grid_for(int64_t total) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), (int64_t)device_info().sm_count * 16));
}

int inv_perm(const int64_t* p, int64_t m, int64_t* pinv, cudaStream_t st) {
  if (m <= 0) return 0;
  inv_perm_kernel<<<grid_for(m), 256, 0, st>>>(p, m, pinv);
  RLRA_LAUNCHED();
  return 0;
}

int lu_basis(const double* lu, int64_t ldlu, int64_t m, int64_t k, const int64_t* piv,
             int64_t* pinv_ws, double* w, int64_t ldw, cudaStream_t st) {
  if (m <= 0 || k <= 0) return 0;
  if (inv_perm(piv, m, pinv_ws, st)) return -1;
  lu_basis_kernel<<<grid_for(m * k), 256, 0, st>>>(lu, ldlu, m, k, pinv_ws, w, ldw);
  RLRA_LAUNCHED();
  return 0;
}

int apply_inv_row_perm(const int64_t* p, int64_t m, int64_t n, const double* x, int64_t ldx, int64_t* pinv_ws,
                       double* out, int64_t ldo, cudaStream_t st) {
  if (m <= 0 || n <= 0) return 0;
  if (inv_perm(p, m, pinv_ws, st)) return -1;
  row_gather_kernel<<<grid_for(m * n), 256, 0, st>>>(x, ldx, m, n, pinv_ws, out, ldo);
  RLRA_LAUNCHED();
  return 0;
}

int extract_l(const double* lu, int64_t ldlu, int64_t m, int64_t k, double* l, int64_t ldl,
              cudaStream_t st) {
  if (m <= 0 || k <= 0) return 0;
  extract_l_kernel<<<grid_for(m * k), 256, 0, st>>>(lu, ldlu, m, k, l, ldl);
  RLRA_LAUNCHED();
  return 0;
}

int extract_u(const double* lu, int64_t ldlu, int64_t k, int64_t n, double* u, int64_t ldu,
              cudaStream_t st) {
  if (k <= 0 || n <= 0) return 0;
  extract_u_kernel<<<grid_for(k * n), 256, 0, st>>>(lu, ldlu, k, n, u, ldu);
  RLRA_LAUNCHED();
  return 0;
}

int transpose(const double* in, int64_t ldi, int64_t m, int64_t n, double* out, int64_t ldo,
              cudaStream_t st) {
  if (m <= 0 || n <= 0) return 0;
  dim3 grid((unsigned)ceil_div(m, 32), (unsigned)ceil_div(n, 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(in, ldi, m, n, out, ldo);
  RLRA_LAUNCHED();
  return 0;
}

}  // namespace rlra
