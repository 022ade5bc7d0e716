// K4: Householder QR with explicit thin Q, replacing the reference's
// kernels.eqr -> np.linalg.qr(mode="reduced") (LAPACK dgeqrf + dorgqr,
// rlra/kernels.py:57-61) used by rangefinder._qr_basis (rlra/rangefinder.py:67-70)
// and kernels.pinv_factor (rlra/kernels.py:64-79).
//
// Blocked right-looking Householder (panel width QR_NB = 32), LAPACK dlarfg sign
// convention (beta = -sign(alpha) * ||x||, tau = (beta - alpha) / beta, v(1) = 1),
// so R's diagonal signs and Q's column signs follow NumPy's.  CholeskyQR2 is not
// used: the final-QR inputs reach cond 6.7e8.
//   panel:    cooperative kernel, one grid barrier per column; each barrier
//             reduces the column norm AND the dot products with the remaining
//             panel columns in one deterministic fixed-order pass;
//   T factor: Gram V^T V via the DMMA GEMM, then dlarft on one CTA;
//   trailing: C -= V T^T (V^T C) as three DMMA GEMMs;
//   orgqr:    Q = B_0 ... B_{P-1} [I; 0] accumulated backwards, GEMMs again.
#include "common.cuh"

namespace rlra {

int gemm(bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
         void* ws, size_t ws_bytes, cudaStream_t st);
size_t gemm_workspace_bytes(int64_t M, int64_t N, int64_t K);

constexpr int QR_NB = 32;
constexpr int QR_THREADS = 256;

struct QrPanelArgs {
  double* a;
  int64_t lda, m, j0;
  int nb;
  int64_t rows_per_cta;
  double* part;      // [2][G][QR_NB + 1] partial sums: [0] = sum x_i^2, [1+c] = sum x_i a_ic
  double* diag;      // [2][QR_NB] row j of the panel
  double* tau;       // [n]
  unsigned* bar;
};

__global__ void __launch_bounds__(QR_THREADS) qr_panel_kernel(QrPanelArgs p) {
  __shared__ double s_red[QR_THREADS / 32][QR_NB + 1];
  __shared__ double s_w[QR_NB + 1];
  __shared__ double s_row[QR_NB];
  __shared__ double s_scal, s_tau, s_beta;
  const int G = gridDim.x, b = blockIdx.x;
  const int nb = p.nb;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t rb = min(p.m, p.j0 + (int64_t)b * p.rows_per_cta);
  const int64_t re = min(p.m, rb + p.rows_per_cta);

  for (int jj = 0; jj < nb; jj++) {
    const int64_t j = p.j0 + jj;
    const int par = jj & 1;
    // ---- partial sums over own rows i > j: x.x and x.a_c for c > jj
    {
      double acc[QR_NB + 1];
#pragma unroll
      for (int c = 0; c <= QR_NB; c++) acc[c] = 0.0;
      const double* colj = p.a + cm(0, j, p.lda);
      for (int64_t i = max(rb, j + 1) + threadIdx.x; i < re; i += blockDim.x) {
        double x = colj[i];
        acc[0] += x * x;
#pragma unroll
        for (int c = 1; c < QR_NB; c++)
          if (c > jj && c < nb) acc[c + 1] += x * p.a[cm(i, p.j0 + c, p.lda)];
      }
      // fixed-order tree: warp shuffles then warps in index order
#pragma unroll
      for (int c = 0; c <= QR_NB; c++) {
        double v = acc[c];
#pragma unroll
        for (int off = 16; off; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
        if (lane == 0) s_red[warp][c] = v;
      }
      __syncthreads();
      if (threadIdx.x <= QR_NB) {
        double v = 0.0;
        for (int w = 0; w < QR_THREADS / 32; w++) v += s_red[w][threadIdx.x];
        __stcg(p.part + ((int64_t)par * G + b) * (QR_NB + 1) + threadIdx.x, v);
      }
      if (j >= rb && j < re && threadIdx.x < nb)
        __stcg(p.diag + par * QR_NB + threadIdx.x, p.a[cm(j, p.j0 + threadIdx.x, p.lda)]);
    }
    grid_barrier(p.bar, G);
    // ---- every CTA reduces the partials in the same fixed order
    if (threadIdx.x <= QR_NB) {
      double v = 0.0;
      for (int q = 0; q < G; q++) v += __ldcg(p.part + ((int64_t)par * G + q) * (QR_NB + 1) + threadIdx.x);
      s_w[threadIdx.x] = v;
    }
    if (threadIdx.x < nb) s_row[threadIdx.x] = __ldcg(p.diag + par * QR_NB + threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0) {
      // dlarfg: alpha = a(j,j), xnorm = ||a(j+1:m, j)||
      const double alpha = s_row[jj];
      const double xnorm = sqrt(s_w[0]);
      if (xnorm == 0.0) {
        s_tau = 0.0;
        s_beta = alpha;
        s_scal = 0.0;
      } else {
        const double beta = -copysign(hypot(alpha, xnorm), alpha);
        s_tau = (beta - alpha) / beta;
        s_scal = 1.0 / (alpha - beta);
        s_beta = beta;
      }
      if (b == 0) p.tau[j] = s_tau;
    }
    __syncthreads();
    const double tau = s_tau, scal = s_scal;
    if (tau != 0.0) {
      // w_c = v^T a_c = a(j,c) + scal * sum_{i>j} x_i a_ic ; then a_c -= tau * w_c * v
      if (threadIdx.x < nb && threadIdx.x > jj)
        s_w[threadIdx.x + 1] = tau * (s_row[threadIdx.x] + scal * s_w[threadIdx.x + 1]);
      __syncthreads();
      for (int64_t i = max(rb, j + 1) + threadIdx.x; i < re; i += blockDim.x) {
        double vi = p.a[cm(i, j, p.lda)] * scal;
        p.a[cm(i, j, p.lda)] = vi;
        for (int c = jj + 1; c < nb; c++) {
          double* e = p.a + cm(i, p.j0 + c, p.lda);
          *e = *e - s_w[c + 1] * vi;
        }
      }
      if (j >= rb && j < re) {
        if (threadIdx.x < nb && threadIdx.x > jj)
          p.a[cm(j, p.j0 + threadIdx.x, p.lda)] = s_row[threadIdx.x] - s_w[threadIdx.x + 1];
        if (threadIdx.x == 0) p.a[cm(j, j, p.lda)] = s_beta;
      }
    }
    __syncthreads();
  }
}

// Explicit V (rows j0..m-1 of the panel, unit diagonal, zeros above) for the GEMMs.
__global__ void qr_make_v_kernel(const double* __restrict__ a, int64_t lda, int64_t j0, int64_t rows,
                                 int nb, double* __restrict__ v, int64_t ldv) {
  const int64_t total = rows * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % rows;
    const int c = (int)(e / rows);
    double x = r > c ? a[cm(j0 + r, j0 + c, lda)] : (r == c ? 1.0 : 0.0);
    v[cm(r, c, ldv)] = x;
  }
}

// dlarft (forward, columnwise) from the Gram matrix S = V^T V:
// T(i,i) = tau_i ; T(0:i, i) = -tau_i * T(0:i,0:i) * S(0:i, i)
__global__ void qr_larft_kernel(const double* __restrict__ gram, int nb, const double* __restrict__ tau,
                                double* __restrict__ T) {
  __shared__ double Ts[QR_NB][QR_NB + 1];
  __shared__ double y[QR_NB];
  const int t = threadIdx.x;
  for (int e = t; e < QR_NB * QR_NB; e += blockDim.x) Ts[e % QR_NB][e / QR_NB] = 0.0;
  __syncthreads();
  for (int i = 0; i < nb; i++) {
    const double ti = tau[i];
    if (t < i) y[t] = -ti * gram[t + i * nb];
    __syncthreads();
    if (t < i) {
      double s = 0.0;
      for (int k = t; k < i; k++) s += Ts[t][k] * y[k];
      Ts[t][i] = s;
    }
    if (t == 0) Ts[i][i] = ti;
    __syncthreads();
  }
  for (int e = t; e < nb * nb; e += blockDim.x) T[e] = Ts[e % nb][e / nb];
}

__global__ void set_identity_kernel(double* q, int64_t ldq, int64_t m, int64_t n) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % m, c = e / m;
    q[cm(r, c, ldq)] = (r == c) ? 1.0 : 0.0;
  }
}

// ------------------------------------------------------------------ host side
static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct QrLayout {
  size_t part, diag, bar, vbuf, gram, tblocks, wbuf, w2buf, gemm_ws, total;
};

static QrLayout qr_layout(int64_t m, int64_t n, int G) {
  QrLayout L{};
  size_t o = 0;
  auto take = [&](size_t& off, size_t bytes) { off = o; o += al(bytes); };
  const int64_t npan = ceil_div(n, QR_NB);
  take(L.part, 2 * (size_t)G * (QR_NB + 1) * sizeof(double));
  take(L.diag, 2 * QR_NB * sizeof(double));
  take(L.bar, 2 * sizeof(unsigned));
  take(L.vbuf, (size_t)m * QR_NB * sizeof(double));
  take(L.gram, QR_NB * QR_NB * sizeof(double));
  take(L.tblocks, (size_t)npan * QR_NB * QR_NB * sizeof(double));
  take(L.wbuf, (size_t)QR_NB * n * sizeof(double));
  take(L.w2buf, (size_t)QR_NB * n * sizeof(double));
  // split-K partials of the skinny (QR_NB-row) GEMMs: at most 16 splits
  size_t g = (size_t)16 * QR_NB * std::max<int64_t>(n, QR_NB) * sizeof(double);
  g = std::max(g, gemm_workspace_bytes(m, n, QR_NB));
  take(L.gemm_ws, g);
  L.total = o;
  return L;
}

size_t geqrf_workspace_bytes(int64_t m, int64_t n) {
  return qr_layout(m, n, device_info().sm_count).total;
}

static int grid_for_q(int64_t total) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), (int64_t)device_info().sm_count * 16));
}

// Factor a (m x n, m >= n) in place: R on/above the diagonal, Householder
// vectors below it; tau[n]; the per-panel T factors stay in the workspace for
// orgqr (call orgqr with the SAME workspace, untouched in between).
int geqrf(double* a, int64_t lda, int64_t m, int64_t n, double* tau, void* ws, size_t ws_bytes,
          cudaStream_t st) {
  RLRA_REQUIRE(m >= n && n >= 0, "geqrf: need m >= n >= 0 (got %lld x %lld)", (long long)m, (long long)n);
  if (n == 0) return 0;
  const int sms = device_info().sm_count;
  QrLayout L = qr_layout(m, n, sms);
  RLRA_REQUIRE(ws && ws_bytes >= L.total, "geqrf: workspace too small (%zu < %zu)", ws_bytes, L.total);
  char* base = static_cast<char*>(ws);
  unsigned* bar = reinterpret_cast<unsigned*>(base + L.bar);
  double* vbuf = reinterpret_cast<double*>(base + L.vbuf);
  double* gram = reinterpret_cast<double*>(base + L.gram);
  double* tbl = reinterpret_cast<double*>(base + L.tblocks);
  double* wbuf = reinterpret_cast<double*>(base + L.wbuf);
  double* w2buf = reinterpret_cast<double*>(base + L.w2buf);
  void* gws = base + L.gemm_ws;
  const size_t gws_bytes = L.total - L.gemm_ws;
  RLRA_CHECK_CUDA(cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), st));
  for (int64_t j0 = 0, pidx = 0; j0 < n; j0 += QR_NB, pidx++) {
    const int nb = (int)std::min<int64_t>(QR_NB, n - j0);
    const int64_t rows = m - j0;
    int G = (int)std::min<int64_t>(sms, std::max<int64_t>(1, ceil_div(rows, 128)));
    QrPanelArgs pa{a, lda, m, j0, nb, ceil_div(rows, G),
                   reinterpret_cast<double*>(base + L.part), reinterpret_cast<double*>(base + L.diag),
                   tau, bar};
    void* args[] = {&pa};
    RLRA_CHECK_CUDA(cudaLaunchCooperativeKernel((void*)qr_panel_kernel, dim3(G), dim3(QR_THREADS), args, 0, st));
    // explicit V and the T factor of this panel
    qr_make_v_kernel<<<grid_for_q(rows * nb), 256, 0, st>>>(a, lda, j0, rows, nb, vbuf, rows);
    RLRA_CHECK_CUDA(cudaGetLastError());
    if (gemm(true, false, nb, nb, rows, 1.0, vbuf, rows, vbuf, rows, 0.0, gram, nb, gws, gws_bytes, st)) return -1;
    double* T = tbl + pidx * QR_NB * QR_NB;
    qr_larft_kernel<<<1, 32, 0, st>>>(gram, nb, tau + j0, T);
    RLRA_CHECK_CUDA(cudaGetLastError());
    // trailing update C = (I - V T^T V^T) C on columns [j0+nb, n)
    const int64_t nc = n - j0 - nb;
    if (nc > 0) {
      double* C = a + cm(j0, j0 + nb, lda);
      if (gemm(true, false, nb, nc, rows, 1.0, vbuf, rows, C, lda, 0.0, wbuf, nb, gws, gws_bytes, st)) return -1;
      if (gemm(true, false, nb, nc, nb, 1.0, T, nb, wbuf, nb, 0.0, w2buf, nb, gws, gws_bytes, st)) return -1;
      if (gemm(false, false, rows, nc, nb, -1.0, vbuf, rows, w2buf, nb, 1.0, C, lda, gws, gws_bytes, st)) return -1;
    }
  }
  return 0;
}

// Q (m x n, ldq) = H_0 ... H_{n-1} [I; 0] from geqrf's output and workspace.
int orgqr(const double* a, int64_t lda, int64_t m, int64_t n, double* q, int64_t ldq, void* ws,
          size_t ws_bytes, cudaStream_t st) {
  RLRA_REQUIRE(m >= n && n >= 0, "orgqr: need m >= n >= 0");
  if (n == 0) return 0;
  const int sms = device_info().sm_count;
  QrLayout L = qr_layout(m, n, sms);
  RLRA_REQUIRE(ws && ws_bytes >= L.total, "orgqr: workspace too small");
  char* base = static_cast<char*>(ws);
  double* vbuf = reinterpret_cast<double*>(base + L.vbuf);
  double* tbl = reinterpret_cast<double*>(base + L.tblocks);
  double* wbuf = reinterpret_cast<double*>(base + L.wbuf);
  double* w2buf = reinterpret_cast<double*>(base + L.w2buf);
  void* gws = base + L.gemm_ws;
  const size_t gws_bytes = L.total - L.gemm_ws;
  set_identity_kernel<<<grid_for_q(m * n), 256, 0, st>>>(q, ldq, m, n);
  RLRA_CHECK_CUDA(cudaGetLastError());
  const int64_t npan = ceil_div(n, QR_NB);
  for (int64_t pidx = npan - 1; pidx >= 0; pidx--) {
    const int64_t j0 = pidx * QR_NB;
    const int nb = (int)std::min<int64_t>(QR_NB, n - j0);
    const int64_t rows = m - j0;
    const int64_t nc = n - j0;
    qr_make_v_kernel<<<grid_for_q(rows * nb), 256, 0, st>>>(a, lda, j0, rows, nb, vbuf, rows);
    RLRA_CHECK_CUDA(cudaGetLastError());
    const double* T = tbl + pidx * QR_NB * QR_NB;
    double* Qs = q + cm(j0, j0, ldq);
    // Qs = (I - V T V^T) Qs
    if (gemm(true, false, nb, nc, rows, 1.0, vbuf, rows, Qs, ldq, 0.0, wbuf, nb, gws, gws_bytes, st)) return -1;
    if (gemm(false, false, nb, nc, nb, 1.0, T, nb, wbuf, nb, 0.0, w2buf, nb, gws, gws_bytes, st)) return -1;
    if (gemm(false, false, rows, nc, nb, -1.0, vbuf, rows, w2buf, nb, 1.0, Qs, ldq, gws, gws_bytes, st)) return -1;
  }
  return 0;
}

}  // namespace rlra
