// K3: partial-pivot LU (GEPP) of tall-skinny sketches, BIT-EXACT with the
// reference kernel rlra/_lu_cython.pyx:14-55 (and its twin rlra/_lu_numpy.py).
//
// Blocked right-looking LU, panel width NB = 32.  Bit-exactness holds because
// every matrix element receives exactly the reference's sequence of roundings:
//   * within the panel the column steps run in order, one grid barrier each;
//   * the trailing update subtracts the panel's rank-1 terms in ascending
//     step order, each as DMUL then DSUB (no FMA, like -ffp-contract=off);
//   * U12 is produced by forward substitution in the same ascending order;
//   * multipliers are IEEE divisions by the pivot (not reciprocal multiplies);
//   * zero-pivot steps (amax <= 1e-14 * colmax, colmax over the WHOLE column)
//     zero their L column and are skipped by every later update, exactly as the
//     reference's `continue` skips its update loop;
//   * pivot = first maximum (smallest row index among equal |values|).
// Row swaps are full-row (the reference swaps all n columns, :40-48); columns
// outside the panel are permuted after the panel by a gather/scatter kernel.
#include "common.cuh"

namespace rlra {

constexpr int LU_NB = 32;
constexpr double ZERO_PIVOT_RTOL = 1e-14;  // rlra/_lu_cython.pyx:11
constexpr int PANEL_THREADS = 256;

struct LuWork {
  double* cand_val;    // [2][G]   local first-max |a| over own rows >= j (-1 if none)
  int64_t* cand_idx;   // [2][G]
  double* cand_cmax;   // [2][G]   local max |a| over own rows in [j0, j)
  double* cand_row;    // [2][G][NB] panel row of the local argmax
  double* diag_row;    // [2][NB]  current panel row j
  double* above;       // [G][NB]  max |a| over rows < j0, per panel column
  unsigned* bar;       // grid barrier (2 words)
  int64_t* ipiv;       // [r] pivot row chosen at step j (== j when no swap)
  int* zflag;          // [r] 1 when step j was a zero pivot
  int64_t* perm_rows;  // [2*NB] rows touched by the panel's swaps
  int64_t* perm_src;   // [2*NB] source row of each touched row after the swaps
  int* perm_cnt;       // [1]
  int64_t* count;      // [1] nonzero diagonal count
};

struct PanelArgs {
  double* a;
  int64_t lda, m, n, j0;
  int nb;
  int64_t rows_per_cta;   // active rows [j0, m) split in contiguous chunks
  int64_t above_per_cta;  // rows [0, j0) split in contiguous chunks
  int64_t* piv;
  LuWork w;
};

// strict-greater first-max merge: (v,i) replaces best when v > best or (v == best && i < besti)
__device__ __forceinline__ bool better(double v, int64_t i, double bv, int64_t bi) {
  return v > bv || (v == bv && i < bi);
}

// Block-wide reduction of (value, index) with first-max semantics; also max of cmax.
__device__ void block_argmax(double& v, int64_t& idx, double& cmax, double* s_v, int64_t* s_i,
                             double* s_c) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    double ov = __shfl_down_sync(0xffffffffu, v, off);
    long long oi = __shfl_down_sync(0xffffffffu, (long long)idx, off);
    double oc = __shfl_down_sync(0xffffffffu, cmax, off);
    if (better(ov, oi, v, idx)) { v = ov; idx = oi; }
    if (oc > cmax) cmax = oc;
  }
  if (lane == 0) { s_v[warp] = v; s_i[warp] = idx; s_c[warp] = cmax; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    v = lane < nw ? s_v[lane] : -1.0;
    idx = lane < nw ? s_i[lane] : INT64_MAX;
    cmax = lane < nw ? s_c[lane] : -1.0;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      double ov = __shfl_down_sync(0xffffffffu, v, off);
      long long oi = __shfl_down_sync(0xffffffffu, (long long)idx, off);
      double oc = __shfl_down_sync(0xffffffffu, cmax, off);
      if (better(ov, oi, v, idx)) { v = ov; idx = oi; }
      if (oc > cmax) cmax = oc;
    }
  }
  __syncthreads();
}

// Local candidate search for panel column c (step row j) over this CTA's rows,
// then publish into buffer `par`.
__device__ void publish_candidates(const PanelArgs& p, int c, int64_t j, int par, int64_t rb,
                                   int64_t re, double* s_v, int64_t* s_i, double* s_c,
                                   int64_t* s_best) {
  const int G = gridDim.x, b = blockIdx.x;
  const double* col = p.a + cm(0, p.j0 + c, p.lda);
  double v = -1.0, cmax = -1.0;
  int64_t idx = INT64_MAX;
  for (int64_t i = rb + threadIdx.x; i < re; i += blockDim.x) {
    double x = fabs(col[i]);
    if (i >= j) {
      if (better(x, i, v, idx)) { v = x; idx = i; }
    } else if (x > cmax) {
      cmax = x;  // rows in [j0, j): already pivoted, part of colmax
    }
  }
  block_argmax(v, idx, cmax, s_v, s_i, s_c);
  if (threadIdx.x == 0) {
    __stcg(p.w.cand_val + par * G + b, v);
    __stcg(p.w.cand_idx + par * G + b, idx);
    __stcg(p.w.cand_cmax + par * G + b, cmax);
    *s_best = (v >= 0.0) ? idx : -1;
  }
  __syncthreads();
  const int64_t best = *s_best;
  if (best >= 0 && threadIdx.x < p.nb)
    __stcg(p.w.cand_row + ((int64_t)par * G + b) * LU_NB + threadIdx.x,
           p.a[cm(best, p.j0 + threadIdx.x, p.lda)]);
  if (j >= rb && j < re && threadIdx.x < p.nb)
    __stcg(p.w.diag_row + par * LU_NB + threadIdx.x, p.a[cm(j, p.j0 + threadIdx.x, p.lda)]);
}

__global__ void __launch_bounds__(PANEL_THREADS)
lu_panel_kernel(PanelArgs p) {
  __shared__ double s_v[32], s_c[32];
  __shared__ int64_t s_i[32];
  __shared__ int64_t s_best;
  __shared__ double s_above[LU_NB];
  __shared__ double s_u[LU_NB];
  __shared__ int64_t s_prow;
  __shared__ int s_zero, s_winner;

  const int G = gridDim.x, b = blockIdx.x;
  const int nb = p.nb;
  const int64_t rb = min(p.m, p.j0 + (int64_t)b * p.rows_per_cta);
  const int64_t re = min(p.m, rb + p.rows_per_cta);

  // ---- prologue: colmax contribution of rows < j0 (final U rows), per panel column
  {
    const int64_t ab = min(p.j0, (int64_t)b * p.above_per_cta);
    const int64_t ae = min(p.j0, ab + p.above_per_cta);
    for (int c = 0; c < nb; c++) {
      const double* col = p.a + cm(0, p.j0 + c, p.lda);
      double cmax = -1.0, v = -1.0;
      int64_t idx = INT64_MAX;
      for (int64_t i = ab + threadIdx.x; i < ae; i += blockDim.x) {
        double x = fabs(col[i]);
        if (x > cmax) cmax = x;
      }
      block_argmax(v, idx, cmax, s_v, s_i, s_c);
      if (threadIdx.x == 0) __stcg(p.w.above + (int64_t)b * LU_NB + c, cmax);
    }
  }
  publish_candidates(p, 0, p.j0, 0, rb, re, s_v, s_i, s_c, &s_best);

  for (int jj = 0; jj < nb; jj++) {
    const int64_t j = p.j0 + jj;
    const int par = jj & 1;
    grid_barrier(p.w.bar, G);
    if (jj == 0) {
      // reduce the rows-above maxima once per panel
      if (threadIdx.x < nb) {
        double mx = -1.0;
        for (int q = 0; q < G; q++) {
          double x = __ldcg(p.w.above + (int64_t)q * LU_NB + threadIdx.x);
          if (x > mx) mx = x;
        }
        s_above[threadIdx.x] = mx;
      }
      __syncthreads();
    }
    // ---- global pivot decision (every CTA redundantly, same order -> same answer)
    if (threadIdx.x < 32) {
      double v = -1.0, cmax = -1.0;
      int64_t idx = INT64_MAX;
      int who = -1;
      for (int q = threadIdx.x; q < G; q += 32) {
        double qv = __ldcg(p.w.cand_val + par * G + q);
        int64_t qi = __ldcg(p.w.cand_idx + par * G + q);
        double qc = __ldcg(p.w.cand_cmax + par * G + q);
        if (qv >= 0.0 && better(qv, qi, v, idx)) { v = qv; idx = qi; who = q; }
        if (qc > cmax) cmax = qc;
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        double ov = __shfl_down_sync(0xffffffffu, v, off);
        long long oi = __shfl_down_sync(0xffffffffu, (long long)idx, off);
        int ow = __shfl_down_sync(0xffffffffu, who, off);
        double oc = __shfl_down_sync(0xffffffffu, cmax, off);
        if (ow >= 0 && better(ov, oi, v, idx)) { v = ov; idx = oi; who = ow; }
        if (oc > cmax) cmax = oc;
      }
      if (threadIdx.x == 0) {
        // reference: amax = first max over rows >= j (or -1), colmax = amax then
        // max over rows < j with strict '>' (rlra/_lu_cython.pyx:23-35)
        double amax = v;  // -1 when every candidate is NaN / absent
        double colmax = amax;
        double ab = s_above[jj];
        if (ab > colmax) colmax = ab;
        if (cmax > colmax) colmax = cmax;
        int zero = (amax <= ZERO_PIVOT_RTOL * colmax) ? 1 : 0;
        s_zero = zero;
        s_prow = zero ? j : idx;
        s_winner = who;
        if (b == 0) {
          p.w.zflag[j] = zero;
          p.w.ipiv[j] = zero ? j : idx;
        }
      }
    }
    __syncthreads();
    const int zero = s_zero;
    const int64_t prow = s_prow;
    if (zero) {
      // zero the L column below the diagonal; no swap, no update (:36-39)
      double* col = p.a + cm(0, j, p.lda);
      for (int64_t i = max(rb, j + 1) + threadIdx.x; i < re; i += blockDim.x) col[i] = 0.0;
    } else {
      if (threadIdx.x < nb)
        s_u[threadIdx.x] = __ldcg(p.w.cand_row + ((int64_t)par * G + s_winner) * LU_NB + threadIdx.x);
      __syncthreads();
      if (prow != j) {
        if (j >= rb && j < re && threadIdx.x < nb)
          p.a[cm(j, p.j0 + threadIdx.x, p.lda)] = s_u[threadIdx.x];
        if (prow >= rb && prow < re && threadIdx.x < nb)
          p.a[cm(prow, p.j0 + threadIdx.x, p.lda)] = __ldcg(p.w.diag_row + par * LU_NB + threadIdx.x);
        if (b == 0 && threadIdx.x == 0) {
          int64_t t = p.piv[j];
          p.piv[j] = p.piv[prow];
          p.piv[prow] = t;
        }
      }
      __syncthreads();
      const double ujj = s_u[jj];
      for (int64_t i = max(rb, j + 1) + threadIdx.x; i < re; i += blockDim.x) {
        double l = p.a[cm(i, j, p.lda)] / ujj;  // IEEE division (:49-51)
        p.a[cm(i, j, p.lda)] = l;
        for (int c = jj + 1; c < nb; c++) {
          double* e = p.a + cm(i, p.j0 + c, p.lda);
          *e = sub_mul_nofma(*e, l, s_u[c]);  // (:52-55)
        }
      }
    }
    __syncthreads();
    if (jj + 1 < nb) publish_candidates(p, jj + 1, j + 1, par ^ 1, rb, re, s_v, s_i, s_c, &s_best);
  }

  // ---- net row permutation of this panel for the columns outside it (CTA 0)
  if (b == 0 && threadIdx.x == 0) {
    int cnt = 0;
    int64_t* rows = p.w.perm_rows;
    int64_t* src = p.w.perm_src;
    auto find = [&](int64_t r) {
      for (int k = 0; k < cnt; k++)
        if (rows[k] == r) return k;
      rows[cnt] = r;
      src[cnt] = r;
      return cnt++;
    };
    for (int jj = 0; jj < nb; jj++) {
      int64_t j = p.j0 + jj, pr = p.w.ipiv[j];
      if (pr == j) continue;
      int ka = find(j), kb = find(pr);
      int64_t t = src[ka];
      src[ka] = src[kb];
      src[kb] = t;
    }
    *p.w.perm_cnt = cnt;
  }
}

// Apply the panel's net row permutation to columns [0, j0) and [j0+nb, n).
// One warp per column: gather every touched row, then scatter.
__global__ void lu_laswp_kernel(double* a, int64_t lda, int64_t n, int64_t j0, int nb,
                                const int64_t* rows, const int64_t* src, const int* cnt_p) {
  const int cnt = *cnt_p;
  if (cnt == 0) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ncols = n - nb;
  for (int64_t w = warp; w < ncols; w += nwarps) {
    const int64_t c = w < j0 ? w : w + nb;
    double* col = a + cm(0, c, lda);
    double v0 = 0.0, v1 = 0.0;
    if (lane < cnt) v0 = col[src[lane]];
    if (lane + 32 < cnt) v1 = col[src[lane + 32]];
    __syncwarp();
    if (lane < cnt) col[rows[lane]] = v0;
    if (lane + 32 < cnt) col[rows[lane + 32]] = v1;
  }
}

// U12 = L11^{-1} A12 by forward substitution in ascending step order, one thread
// per column; zero-pivot steps are skipped (the reference never applies them).
__global__ void lu_trsm_kernel(double* a, int64_t lda, int64_t j0, int nb, int64_t c0, int64_t n,
                               const int* zflag) {
  __shared__ double L[LU_NB][LU_NB + 1];
  __shared__ int z[LU_NB];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    int r = e % nb, c = e / nb;
    L[r][c] = a[cm(j0 + r, j0 + c, lda)];
  }
  if (threadIdx.x < nb) z[threadIdx.x] = zflag[j0 + threadIdx.x];
  __syncthreads();
  for (int64_t c = c0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    double x[LU_NB];
    double* col = a + cm(j0, c, lda);
#pragma unroll
    for (int s = 0; s < LU_NB; s++) x[s] = s < nb ? col[s] : 0.0;
#pragma unroll
    for (int t = 0; t < LU_NB; t++) {
      if (t >= nb || z[t]) continue;
#pragma unroll
      for (int s = t + 1; s < LU_NB; s++)
        if (s < nb) x[s] = sub_mul_nofma(x[s], L[s][t], x[t]);
    }
#pragma unroll
    for (int s = 1; s < LU_NB; s++)
      if (s < nb) col[s] = x[s];
  }
}

// A22 -= L21 * U12 with the panel's steps applied in ascending order, DMUL+DSUB.
constexpr int UPD_TM = 64, UPD_TN = 64;
__global__ void __launch_bounds__(256)
lu_update_kernel(double* a, int64_t lda, int64_t j0, int nb, int64_t r0, int64_t m, int64_t c0,
                 int64_t n, const int* zflag) {
  __shared__ double Ls[LU_NB][UPD_TM];
  __shared__ double Us[LU_NB][UPD_TN + 1];
  __shared__ int z[LU_NB];
  const int64_t rt = r0 + (int64_t)blockIdx.x * UPD_TM;
  const int64_t ct = c0 + (int64_t)blockIdx.y * UPD_TN;
  for (int e = threadIdx.x; e < nb * UPD_TM; e += blockDim.x) {
    int r = e % UPD_TM, t = e / UPD_TM;
    int64_t gr = rt + r;
    Ls[t][r] = gr < m ? a[cm(gr, j0 + t, lda)] : 0.0;
  }
  for (int e = threadIdx.x; e < nb * UPD_TN; e += blockDim.x) {
    int t = e % nb, c = e / nb;
    int64_t gc = ct + c;
    Us[t][c] = gc < n ? a[cm(j0 + t, gc, lda)] : 0.0;
  }
  if (threadIdx.x < nb) z[threadIdx.x] = zflag[j0 + threadIdx.x];
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int ii = 0; ii < 4; ii++)
#pragma unroll
    for (int jj = 0; jj < 4; jj++) {
      int64_t gr = rt + tx + 16 * ii, gc = ct + ty + 16 * jj;
      acc[ii][jj] = (gr < m && gc < n) ? a[cm(gr, gc, lda)] : 0.0;
    }
  for (int t = 0; t < nb; t++) {
    if (z[t]) continue;
    double l[4], u[4];
#pragma unroll
    for (int ii = 0; ii < 4; ii++) l[ii] = Ls[t][tx + 16 * ii];
#pragma unroll
    for (int jj = 0; jj < 4; jj++) u[jj] = Us[t][ty + 16 * jj];
#pragma unroll
    for (int ii = 0; ii < 4; ii++)
#pragma unroll
      for (int jj = 0; jj < 4; jj++) acc[ii][jj] = sub_mul_nofma(acc[ii][jj], l[ii], u[jj]);
  }
#pragma unroll
  for (int ii = 0; ii < 4; ii++)
#pragma unroll
    for (int jj = 0; jj < 4; jj++) {
      int64_t gr = rt + tx + 16 * ii, gc = ct + ty + 16 * jj;
      if (gr < m && gc < n) a[cm(gr, gc, lda)] = acc[ii][jj];
    }
}

__global__ void iota_kernel(int64_t* p, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = i;
}

__global__ void count_nonzero_diag_kernel(const double* a, int64_t lda, int64_t r, int64_t* out) {
  __shared__ int64_t s[32];
  int64_t cnt = 0;
  for (int64_t i = threadIdx.x; i < r; i += blockDim.x) cnt += (a[cm(i, i, lda)] != 0.0);
#pragma unroll
  for (int off = 16; off; off >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, off);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) tot += s[w];
    *out = tot;
  }
}

// ------------------------------------------------------------------ host side
static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct LuLayout {
  size_t off[13];
  size_t total;
};

static LuLayout lu_layout(int64_t r, int G) {
  LuLayout L{};
  size_t o = 0;
  auto take = [&](int k, size_t bytes) { L.off[k] = o; o += align_up(bytes); };
  take(0, 2 * G * sizeof(double));
  take(1, 2 * G * sizeof(int64_t));
  take(2, 2 * G * sizeof(double));
  take(3, 2 * (size_t)G * LU_NB * sizeof(double));
  take(4, 2 * LU_NB * sizeof(double));
  take(5, (size_t)G * LU_NB * sizeof(double));
  take(6, 2 * sizeof(unsigned));
  take(7, (size_t)(r > 0 ? r : 1) * sizeof(int64_t));
  take(8, (size_t)(r > 0 ? r : 1) * sizeof(int));
  take(9, 2 * LU_NB * sizeof(int64_t));
  take(10, 2 * LU_NB * sizeof(int64_t));
  take(11, sizeof(int));
  take(12, sizeof(int64_t));
  L.total = o;
  return L;
}

size_t getrf_workspace_bytes(int64_t m, int64_t n) {
  int64_t r = m < n ? m : n;
  return lu_layout(r, device_info().sm_count).total;
}

static LuWork lu_work(void* ws, int64_t r, int G) {
  LuLayout L = lu_layout(r, G);
  char* base = static_cast<char*>(ws);
  LuWork w;
  w.cand_val = reinterpret_cast<double*>(base + L.off[0]);
  w.cand_idx = reinterpret_cast<int64_t*>(base + L.off[1]);
  w.cand_cmax = reinterpret_cast<double*>(base + L.off[2]);
  w.cand_row = reinterpret_cast<double*>(base + L.off[3]);
  w.diag_row = reinterpret_cast<double*>(base + L.off[4]);
  w.above = reinterpret_cast<double*>(base + L.off[5]);
  w.bar = reinterpret_cast<unsigned*>(base + L.off[6]);
  w.ipiv = reinterpret_cast<int64_t*>(base + L.off[7]);
  w.zflag = reinterpret_cast<int*>(base + L.off[8]);
  w.perm_rows = reinterpret_cast<int64_t*>(base + L.off[9]);
  w.perm_src = reinterpret_cast<int64_t*>(base + L.off[10]);
  w.perm_cnt = reinterpret_cast<int*>(base + L.off[11]);
  w.count = reinterpret_cast<int64_t*>(base + L.off[12]);
  return w;
}

int count_nonzero_diag(const double* a, int64_t lda, int64_t r, int64_t* out_dev, cudaStream_t st) {
  count_nonzero_diag_kernel<<<1, 256, 0, st>>>(a, lda, r, out_dev);
  RLRA_CHECK_CUDA(cudaGetLastError());
  return 0;
}

int fill_iota(int64_t* p, int64_t m, cudaStream_t st) {
  if (m <= 0) return 0;
  int blocks = (int)std::min<int64_t>(ceil_div(m, 256), 4096);
  iota_kernel<<<blocks, 256, 0, st>>>(p, m);
  RLRA_CHECK_CUDA(cudaGetLastError());
  return 0;
}

// Packed in-place GEPP: on return `a` holds unit-L multipliers below the
// diagonal and U on/above it, `piv` (caller-preloaded, typically 0..m-1) is
// permuted like the reference's piv (rlra/_lu_cython.pyx:14, rlra/kernels.py:48),
// and *nonzero_diag_dev (device int64) receives count_nonzero(diag(U)).
int getrf(double* a, int64_t lda, int64_t m, int64_t n, int64_t* piv, int64_t* nonzero_diag_dev,
          int* zflag_out, void* ws, size_t ws_bytes, cudaStream_t st) {
  RLRA_REQUIRE(m >= 0 && n >= 0, "getrf: negative dimension");
  RLRA_REQUIRE(lda >= (m > 0 ? m : 1), "getrf: lda < m");
  const int64_t r = m < n ? m : n;
  const int sms = device_info().sm_count;
  LuLayout L = lu_layout(r, sms);
  RLRA_REQUIRE(ws != nullptr && ws_bytes >= L.total, "getrf: workspace too small (%zu < %zu)",
               ws_bytes, L.total);
  LuWork w = lu_work(ws, r, sms);
  RLRA_CHECK_CUDA(cudaMemsetAsync(w.bar, 0, 2 * sizeof(unsigned), st));
  for (int64_t j0 = 0; j0 < r; j0 += LU_NB) {
    const int nb = (int)std::min<int64_t>(LU_NB, r - j0);
    const int64_t active = m - j0;
    // enough rows per CTA to amortise the barrier; at most one CTA per SM
    int G = (int)std::min<int64_t>(sms, std::max<int64_t>(1, ceil_div(active, 128)));
    PanelArgs pa;
    pa.a = a; pa.lda = lda; pa.m = m; pa.n = n; pa.j0 = j0; pa.nb = nb;
    pa.rows_per_cta = ceil_div(active, G);
    pa.above_per_cta = std::max<int64_t>(1, ceil_div(j0, G));
    pa.piv = piv;
    pa.w = w;
    void* args[] = {&pa};
    RLRA_CHECK_CUDA(cudaLaunchCooperativeKernel((void*)lu_panel_kernel, dim3(G), dim3(PANEL_THREADS),
                                                args, 0, st));
    if (n > nb) {
      int64_t ncols = n - nb;
      int blocks = (int)std::min<int64_t>(ceil_div(ncols * 32, 256), 2048);
      lu_laswp_kernel<<<blocks, 256, 0, st>>>(a, lda, n, j0, nb, w.perm_rows, w.perm_src, w.perm_cnt);
      RLRA_CHECK_CUDA(cudaGetLastError());
    }
    const int64_t c0 = j0 + nb;
    if (c0 < n) {
      int blocks = (int)std::min<int64_t>(ceil_div(n - c0, 128), 1024);
      lu_trsm_kernel<<<blocks, 128, 0, st>>>(a, lda, j0, nb, c0, n, w.zflag);
      RLRA_CHECK_CUDA(cudaGetLastError());
      if (c0 < m) {
        dim3 grid((unsigned)ceil_div(m - c0, UPD_TM), (unsigned)ceil_div(n - c0, UPD_TN));
        lu_update_kernel<<<grid, 256, 0, st>>>(a, lda, j0, nb, c0, m, c0, n, w.zflag);
        RLRA_CHECK_CUDA(cudaGetLastError());
      }
    }
  }
  if (nonzero_diag_dev) {
    count_nonzero_diag_kernel<<<1, 256, 0, st>>>(a, lda, r, nonzero_diag_dev);
    RLRA_CHECK_CUDA(cudaGetLastError());
  }
  if (zflag_out && r > 0)
    RLRA_CHECK_CUDA(cudaMemcpyAsync(zflag_out, w.zflag, r * sizeof(int), cudaMemcpyDeviceToDevice, st));
  return 0;
}

}  // namespace rlra
