// K4: Householder QR with explicit thin Q, replacing the reference's
// kernels.eqr -> np.linalg.qr(mode="reduced") (LAPACK dgeqrf + dorgqr,
// rlra/kernels.py:57-61) used by rangefinder._qr_basis (rlra/rangefinder.py:67-70)
// and kernels.pinv_factor (rlra/kernels.py:64-79).
//
// Blocked right-looking Householder (panel width QR_NB = 32, two-level: outer
// blocks of QR_NBO = 128 columns carry the trailing update), LAPACK dlarfg sign
// convention (beta = -sign(alpha) * ||x||, tau = (beta - alpha) / beta, v(1) = 1),
// so R's diagonal signs and Q's column signs follow NumPy's.  CholeskyQR2 is not
// used: the final-QR inputs reach cond 6.7e8.
//   panel:    cooperative kernel, one grid barrier per column; each barrier
//             reduces the column norm AND the dot products with the remaining
//             panel columns in one deterministic fixed-order pass;
//   T factor: Gram V^T V via the DMMA GEMM, then dlarft on one CTA;
//   trailing: C -= V T^T (V^T C) as three DMMA GEMMs;
//   orgqr:    Q = B_0 ... B_{P-1} [I; 0] accumulated backwards, GEMMs again.
#include <cooperative_groups.h>

#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"

namespace rlra {

int gemm(bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
         void* ws, size_t ws_bytes, cudaStream_t st);
size_t gemm_workspace_bytes(int64_t M, int64_t N, int64_t K);

constexpr int QR_NB = 32;

struct QrPanelArgs {
  double* a;
  int64_t lda, m, j0;
  int nb;
  int64_t rows_per_cta;
  double* part;      // [2][G][QR_NB + 1] partial sums: [0] = sum x_i^2, [1+c] = sum x_i a_ic
  double* diag;      // [2][QR_NB] row j of the panel
  double* tau;       // [n]
  unsigned* bar;
  unsigned bar_base;  // monotonic grid-barrier counter at kernel entry
  double* recg;       // cluster panel: global staging of the multicast records
};

// Householder panel with the CTA's panel rows resident in SHARED MEMORY
// (column-major s_a[c * R + r]).  Per column: the norm of x = a(j+1:, j) and the
// dot products x . a_c (c > jj) are computed warp-per-value in a fixed order,
// published, one grid barrier, a fixed-order cross-CTA sum (deterministic),
// dlarfg on every CTA redundantly, and the rank-1 update of the own rows.
template <int THREADS>
__global__ void __launch_bounds__(THREADS, 1) qr_panel_smem_kernel(QrPanelArgs p) {
  constexpr int NV = QR_NB + 1;
  constexpr int NW = THREADS / 32;
  constexpr int CH = THREADS / NV;  // chunks of the cross-CTA sum
  extern __shared__ __align__(16) double s_a[];
  __shared__ double s_chunk[CH][NV];
  __shared__ double s_w[NV];
  __shared__ double s_row[QR_NB];
  __shared__ double s_scal, s_tau, s_beta;
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int nb = p.nb;
  const int64_t R = p.rows_per_cta;
  const int64_t rb = min(p.m, p.j0 + (int64_t)b * R);
  const int64_t re = min(p.m, rb + R);
  const int nr = (int)(re - rb);

  for (int c = 0; c < nb; c++)
    for (int r = tid; r < nr; r += THREADS) s_a[c * R + r] = p.a[cm(rb + r, p.j0 + c, p.lda)];
  __syncthreads();

  for (int jj = 0; jj < nb; jj++) {
    const int64_t j = p.j0 + jj;
    const int par = jj & 1;
    const int r0 = (int)max((int64_t)0, j + 1 - rb);  // local rows strictly below row j
    const double* x = s_a + jj * R;
    // value q: q == 0 -> ||x||^2, q >= 1 -> x . a_{jj+q}
    const int cnt = nb - jj;
    for (int q = warp; q < cnt; q += NW) {
      const double* y = s_a + (q == 0 ? jj : jj + q) * R;
      double acc = 0.0;
      for (int r = r0 + lane; r < nr; r += 32) acc += x[r] * y[r];
#pragma unroll
      for (int off = 16; off; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
      if (lane == 0) __stcg(p.part + ((int64_t)par * G + b) * NV + (q == 0 ? 0 : jj + q + 1), acc);
    }
    if (j >= rb && j < re && tid < nb) __stcg(p.diag + par * QR_NB + tid, s_a[tid * R + (j - rb)]);
    grid_barrier_mono(p.bar, p.bar_base + (unsigned)G * (jj + 1));
    // ---- fixed-order cross-CTA reduction: CH chunks of CTAs, then chunks in order
    if (tid < CH * NV) {
      const int c = tid % NV, ch = tid / NV;
      if (c == 0 || (c >= jj + 2 && c <= nb)) {
        const int q0 = (int)(((int64_t)G * ch) / CH), q1 = (int)(((int64_t)G * (ch + 1)) / CH);
        double v = 0.0;
        for (int q = q0; q < q1; q++) v += __ldcg(p.part + ((int64_t)par * G + q) * NV + c);
        s_chunk[ch][c] = v;
      }
    }
    if (tid < nb) s_row[tid] = __ldcg(p.diag + par * QR_NB + tid);
    __syncthreads();
    if (tid < NV && (tid == 0 || (tid >= jj + 2 && tid <= nb))) {
      double v = 0.0;
      for (int ch = 0; ch < CH; ch++) v += s_chunk[ch][tid];
      s_w[tid] = v;
    }
    __syncthreads();
    if (tid == 0) {
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
      // w_c = tau * v^T a_c = tau * (a(j,c) + scal * x . a_c) ; a_c -= w_c v
      if (tid < nb && tid > jj) s_w[tid + 1] = tau * (s_row[tid] + scal * s_w[tid + 1]);
      __syncthreads();
      double* xc = s_a + jj * R;
      for (int r = r0 + tid; r < nr; r += THREADS) {
        const double vi = xc[r] * scal;
        xc[r] = vi;
        for (int c = jj + 1; c < nb; c++) s_a[c * R + r] -= s_w[c + 1] * vi;
      }
      if (j >= rb && j < re && tid < nb) {
        if (tid > jj) s_a[tid * R + (j - rb)] = s_row[tid] - s_w[tid + 1];
        if (tid == jj) s_a[tid * R + (j - rb)] = s_beta;
      }
    }
    __syncthreads();
  }
  for (int c = 0; c < nb; c++)
    for (int r = tid; r < nr; r += THREADS) p.a[cm(rb + r, p.j0 + c, p.lda)] = s_a[c * R + r];
}

static constexpr int QR_PANEL_SMEM_BYTES = 200 * 1024;

// Cluster-resident Householder panel (<= 16 CTAs on one GPC, rows in shared
// memory).  Per column each CTA computes its partial ||x||^2 and x . a_c
// (c > jj) in a fixed order, stages them (plus row j when it owns it) in a
// global slot and multicasts them with ONE bulk copy into every peer's shared
// memory (completing on the peers' mbarriers); every CTA then sums the CS
// partials in rank order -- identical, deterministic sums everywhere -- and
// applies dlarfg and the rank-1 update to its rows.
template <int PW, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) qr_panel_cluster_kernel(QrPanelArgs p) {
  namespace cg = cooperative_groups;
  constexpr int MAXCS = 16;
  constexpr int RECQ = 2 + PW;  // {sum x^2, 0, sum x a_c (c < PW)}
  constexpr int NW = THREADS / 32;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double s_a[];
  __shared__ __align__(16) double recv[2][MAXCS][RECQ];
  __shared__ __align__(16) double recv_row[2][PW];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ __align__(8) uint64_t ldbar;
  __shared__ double s_part[RECQ];
  __shared__ double s_w[PW + 1];
  __shared__ double s_scal, s_tau, s_beta;

  const int CS = (int)cluster.num_blocks(), b = (int)cluster.block_rank(), tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int nb = p.nb;
  const int64_t R = p.rows_per_cta;
  const int Ri = (int)R;
  const int64_t rb = min(p.m, p.j0 + (int64_t)b * R);
  const int64_t re = min(p.m, rb + R);
  const int nr = (int)(re - rb);
  const unsigned tx_bytes = CS * RECQ * 8u + PW * 8u;

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&ldbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const bool bulk_ok = ((R & 1) == 0) && ((p.lda & 1) == 0) && ((rb & 1) == 0);
  const int nr_bulk = bulk_ok ? (nr & ~1) : 0;
  if (nr_bulk > 0 && tid == 0) {
    mbar_arrive_expect_tx(&ldbar, (unsigned)(nb * nr_bulk * 8));
    for (int c = 0; c < nb; c++)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              smem_u32(s_a + c * Ri)),
          "l"(p.a + cm(rb, p.j0 + c, p.lda)), "r"((unsigned)(nr_bulk * 8)), "r"(smem_u32(&ldbar))
          : "memory");
  }
  for (int c = 0; c < nb; c++)
    for (int r = nr_bulk + tid; r < nr; r += THREADS) s_a[c * Ri + r] = p.a[cm(rb + r, p.j0 + c, p.lda)];
  if (nr_bulk > 0) mbar_wait_parity(&ldbar, 0);
  if (tid == 0) {
    mbar_arrive_expect_tx(&mbar[0], tx_bytes);
    mbar_arrive_expect_tx(&mbar[1], tx_bytes);
  }
  cluster.sync();  // mbarrier inits visible cluster-wide
  unsigned phase_bits = 0u;

  for (int jj = 0; jj < nb; jj++) {
    const int64_t j = p.j0 + jj;
    const int par = jj & 1;
    const int r0 = (int)max((int64_t)0, j + 1 - rb);  // local rows strictly below row j
    const double* x = s_a + jj * Ri;
    // ---- partial sums, one warp per value (fixed order: lane-strided rows, xor tree)
    const int cnt = nb - jj;  // value q: 0 -> ||x||^2, q >= 1 -> x . a_{jj+q}
    for (int q = warp; q < cnt; q += NW) {
      const double* y = s_a + (q == 0 ? jj : jj + q) * Ri;
      double acc = 0.0;
      for (int r = r0 + lane; r < nr; r += 32) acc += x[r] * y[r];
#pragma unroll
      for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) s_part[q == 0 ? 0 : 2 + jj + q] = acc;
    }
    __syncthreads();
    if (warp == 0) {
      // stage {sum x^2, 0, dots} (+ row j when this CTA owns it), multicast to all
      double* slot = p.recg + ((int64_t)par * MAXCS + b) * RECQ;
      double* rslot = p.recg + 2 * MAXCS * RECQ + par * PW;
      for (int e = lane; e < RECQ; e += 32) {
        double v = 0.0;
        if (e == 0) v = s_part[0];
        else if (e >= 2 + jj + 1 && e < 2 + nb) v = s_part[e];
        slot[e] = v;
      }
      const bool own_j = (j >= rb && j < re);
      if (own_j && lane < PW) rslot[lane] = lane < nb ? s_a[lane * Ri + (int)(j - rb)] : 0.0;
      asm volatile("fence.proxy.async.global;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const unsigned short mask = (unsigned short)((1u << CS) - 1u);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;\n" ::"r"(
                smem_u32(&recv[par][b][0])),
            "l"(slot), "r"((unsigned)(RECQ * 8)), "r"(smem_u32(&mbar[par])), "h"(mask)
            : "memory");
        if (own_j)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;\n" ::"r"(
                  smem_u32(&recv_row[par][0])),
              "l"(rslot), "r"((unsigned)(PW * 8)), "r"(smem_u32(&mbar[par])), "h"(mask)
              : "memory");
      }
      mbar_wait_parity(&mbar[par], (phase_bits >> par) & 1u);
      // fixed-order sums over the CS partials -> identical in every CTA
      if (lane < RECQ && (lane == 0 || (lane >= 2 + jj + 1 && lane < 2 + nb))) {
        double v = 0.0;
        for (int q = 0; q < CS; q++) v += recv[par][q][lane];
        if (lane == 0) s_w[0] = v;
        else s_w[lane - 1] = v;  // s_w[1 + c] = x . a_c
      }
      if (lane + 32 < RECQ && lane + 32 < 2 + nb) {
        double v = 0.0;
        for (int q = 0; q < CS; q++) v += recv[par][q][lane + 32];
        s_w[lane + 31] = v;
      }
      __syncwarp();
      if (lane == 0) {
        // dlarfg: alpha = a(j,j), xnorm = ||a(j+1:m, j)||
        const double alpha = recv_row[par][jj];
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
      __syncwarp();
      if (lane < nb && lane > jj && s_tau != 0.0)
        s_w[lane + 1] = s_tau * (recv_row[par][lane] + s_scal * s_w[lane + 1]);
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&mbar[par], tx_bytes);  // re-arm for step jj + 2
      phase_bits ^= 1u << par;
    }
    __syncthreads();
    const double tau = s_tau, scal = s_scal;
    if (tau != 0.0) {
      double* xc = s_a + jj * Ri;
      for (int r = r0 + tid; r < nr; r += THREADS) {
        const double vi = xc[r] * scal;
        xc[r] = vi;
        for (int c = jj + 1; c < nb; c++) s_a[c * Ri + r] -= s_w[c + 1] * vi;
      }
      if (j >= rb && j < re && tid < nb) {
        if (tid > jj) s_a[tid * Ri + (int)(j - rb)] = recv_row[par][tid] - s_w[tid + 1];
        if (tid == jj) s_a[tid * Ri + (int)(j - rb)] = s_beta;
      }
    }
    __syncthreads();
  }
  if (nr_bulk > 0) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid < nb) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                       p.a + cm(rb, p.j0 + tid, p.lda)),
                   "r"(smem_u32(s_a + tid * Ri)), "r"((unsigned)(nr_bulk * 8))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  }
  for (int c = 0; c < nb; c++)
    for (int r = nr_bulk + tid; r < nr; r += THREADS) p.a[cm(rb + r, p.j0 + c, p.lda)] = s_a[c * Ri + r];
  if (nr_bulk > 0 && tid < nb) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
  cluster.sync();
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
// The block stages S and tau in shared memory; warp 0 runs the recurrence.
__global__ void qr_larft_kernel(const double* __restrict__ gram, int nb, const double* __restrict__ tau,
                                double* __restrict__ T) {
  __shared__ double Ss[QR_NB][QR_NB + 1];
  __shared__ double Ts[QR_NB][QR_NB + 1];
  __shared__ double ts[QR_NB], y[QR_NB];
  for (int e = threadIdx.x; e < QR_NB * QR_NB; e += blockDim.x) {
    const int r = e % QR_NB, c = e / QR_NB;
    Ss[r][c] = (r < nb && c < nb) ? gram[r + c * nb] : 0.0;
    Ts[r][c] = 0.0;
  }
  if (threadIdx.x < nb) ts[threadIdx.x] = tau[threadIdx.x];
  __syncthreads();
  if (threadIdx.x < 32) {
    const int t = threadIdx.x;
    for (int i = 0; i < nb; i++) {
      const double ti = ts[i];
      if (t < i) y[t] = -ti * Ss[t][i];
      __syncwarp();
      if (t < i) {
        double acc = 0.0;
        for (int k = t; k < i; k++) acc += Ts[t][k] * y[k];
        Ts[t][i] = acc;
      }
      if (t == 0) Ts[i][i] = ti;
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) T[e] = Ts[e % nb][e / nb];
}

// dlarft for an outer block of nbo <= QR_NBO columns: the same recurrence with
// T in shared memory (dynamic) and S read from global memory; one CTA, thread
// t owns row t of T.
constexpr int QR_NBO = 128;
__global__ void __launch_bounds__(QR_NBO) qr_larft_big_kernel(const double* __restrict__ gram, int nb,
                                                             const double* __restrict__ tau,
                                                             double* __restrict__ T) {
  extern __shared__ double Tsb[];  // [QR_NBO][QR_NBO + 1], row t at t * (QR_NBO + 1)
  __shared__ double y[QR_NBO];
  const int t = threadIdx.x;
  constexpr int LD = QR_NBO + 1;
  for (int c = 0; c < nb; c++) Tsb[t * LD + c] = 0.0;
  __syncthreads();
  for (int i = 0; i < nb; i++) {
    const double ti = tau[i];
    if (t < i) y[t] = -ti * gram[t + (int64_t)i * nb];
    __syncthreads();
    if (t < i) {
      double acc = 0.0;
      for (int k = t; k < i; k++) acc += Tsb[t * LD + k] * y[k];
      Tsb[t * LD + i] = acc;
    }
    if (t == i) Tsb[t * LD + i] = ti;
    __syncthreads();
  }
  if (t < nb)
    for (int c = 0; c < nb; c++) T[t + (int64_t)c * nb] = Tsb[t * LD + c];
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

// Panel width for m rows (geqrf and orgqr must agree): 32 while a 32-column
// panel of every row fits in one CTA's shared memory per SM, else 16 or 8.
static int64_t qr_rows_cap(int pw) { return (int64_t)(QR_PANEL_SMEM_BYTES / (pw * 8)); }
static int qr_pw(int64_t m, int sms) {
  if (m <= sms * qr_rows_cap(32)) return 32;
  if (m <= sms * qr_rows_cap(16)) return 16;
  return 8;
}

struct QrLayout {
  size_t part, diag, bar, recg, gramp, vbuf, gram, tblocks, tbig, wbuf, w2buf, gemm_ws, total;
};

static QrLayout qr_layout(int64_t m, int64_t n, int G) {
  QrLayout L{};
  size_t o = 0;
  auto take = [&](size_t& off, size_t bytes) { off = o; o += al(bytes); };
  const int64_t npan = ceil_div(n, 8);  // smallest panel width is 8
  take(L.part, 2 * (size_t)G * (QR_NB + 1) * sizeof(double));
  take(L.diag, 2 * QR_NB * sizeof(double));
  take(L.bar, 2 * sizeof(unsigned));
  take(L.recg, (size_t)(2 * 16 * (2 + QR_NB) + 2 * QR_NB) * sizeof(double));
  take(L.gramp, (size_t)16 * QR_NB * QR_NB * sizeof(double));
  take(L.vbuf, (size_t)m * QR_NBO * sizeof(double));
  take(L.gram, QR_NBO * QR_NBO * sizeof(double));
  take(L.tblocks, (size_t)npan * QR_NB * QR_NB * sizeof(double));
  take(L.tbig, (size_t)ceil_div(n, QR_NBO) * QR_NBO * QR_NBO * sizeof(double));
  take(L.wbuf, (size_t)QR_NBO * n * sizeof(double));
  take(L.w2buf, (size_t)QR_NBO * n * sizeof(double));
  // split-K partials of the skinny GEMMs: at most 32 splits
  size_t g = (size_t)32 * QR_NBO * std::max<int64_t>(n, QR_NBO) * sizeof(double);
  g = std::max(g, gemm_workspace_bytes(m, n, QR_NBO));
  take(L.gemm_ws, g);
  L.total = o;
  return L;
}

size_t geqrf_workspace_bytes(int64_t m, int64_t n) {
  return qr_layout(m, n, device_info().sm_count).total;
}

// Largest cluster (<= 16) that co-schedules one 512-thread CTA with the full
// panel shared memory per SM; 1 when clusters are unavailable.
static int qr_max_cluster() {
  static int cached[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  if (cached[dev & 63]) return cached[dev & 63];
  int best = 1;
  const void* kern = (const void*)qr_panel_cluster_kernel<16, 512>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, QR_PANEL_SMEM_BYTES) ==
          cudaSuccess &&
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
    for (int cs = 16; cs >= 2; cs /= 2) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = QR_PANEL_SMEM_BYTES;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) == cudaSuccess && ncl > 0) {
        best = cs;
        break;
      }
    }
  }
  cudaGetLastError();
  cached[dev & 63] = best;
  return best;
}

static int qr_prepare_kernel(const void* kern) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  RLRA_CHECK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({dev, kern})) return 0;
  RLRA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, QR_PANEL_SMEM_BYTES));
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaGetLastError();
  done.insert({dev, kern});
  return 0;
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
  double* tbig = reinterpret_cast<double*>(base + L.tbig);
  double* wbuf = reinterpret_cast<double*>(base + L.wbuf);
  double* w2buf = reinterpret_cast<double*>(base + L.w2buf);
  void* gws = base + L.gemm_ws;
  const size_t gws_bytes = L.total - L.gemm_ws;
  RLRA_CHECK_CUDA(cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), st));
  {
    static std::once_flag once;
    static cudaError_t e = cudaSuccess;
    std::call_once(once, [] {
      e = cudaFuncSetAttribute(qr_larft_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)((size_t)QR_NBO * (QR_NBO + 1) * sizeof(double)));
    });
    RLRA_CHECK_CUDA(e);
  }
  // Panel: one thread-block cluster (DSMEM multicast exchange) while the rows
  // fit 16 CTAs' shared memory, else one CTA per SM with a grid barrier.
  const int cmax = qr_max_cluster();
  const bool use_cluster = cmax > 1 && m <= cmax * qr_rows_cap(16);
  const int pw = use_cluster ? (m <= cmax * qr_rows_cap(32) ? 32 : 16) : qr_pw(m, sms);
  RLRA_REQUIRE(m <= sms * qr_rows_cap(8), "geqrf: m = %lld exceeds the panel capacity", (long long)m);
  const void* kern = use_cluster ? (pw == 32 ? (const void*)qr_panel_cluster_kernel<32, 512>
                                             : (const void*)qr_panel_cluster_kernel<16, 512>)
                                 : (const void*)qr_panel_smem_kernel<256>;
  if (qr_prepare_kernel(kern)) return -1;
  unsigned bar_base = 0;
  for (int64_t j0 = 0, pidx = 0; j0 < n; j0 += pw, pidx++) {
    const int nb = (int)std::min<int64_t>(pw, n - j0);
    const int64_t rows = m - j0;
    const int limit = use_cluster ? cmax : sms;
    const int64_t target = std::min<int64_t>(qr_rows_cap(pw), use_cluster ? 512 : 256);
    int G = (int)std::min<int64_t>(limit, ceil_div(rows, target));
    G = (int)std::max<int64_t>(G, ceil_div(rows, qr_rows_cap(pw)));
    int64_t R = ceil_div(rows, G);
    R += R & 1;  // even: 16-byte aligned bulk copies of the panel columns
    double* T = tbl + pidx * QR_NB * QR_NB;
    QrPanelArgs pa{a, lda, m, j0, nb, R,
                   reinterpret_cast<double*>(base + L.part), reinterpret_cast<double*>(base + L.diag),
                   tau, bar, bar_base, reinterpret_cast<double*>(base + L.recg)};
    const size_t smem = (size_t)pa.rows_per_cta * nb * sizeof(double);
    void* args[] = {&pa};
    if (use_cluster) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = G;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      RLRA_CHECK_CUDA(cudaLaunchKernelExC(&cfg, kern, args));
    } else {
      RLRA_CHECK_CUDA(cudaLaunchCooperativeKernel(kern, dim3(G), dim3(256), args, smem, st));
      bar_base += (unsigned)G * nb;
    }
    note_launch();
    // explicit V and the T factor of this panel (Gram on the DMMA GEMM + dlarft)
    qr_make_v_kernel<<<grid_for_q(rows * nb), 256, 0, st>>>(a, lda, j0, rows, nb, vbuf, rows);
    RLRA_LAUNCHED();
    if (gemm(true, false, nb, nb, rows, 1.0, vbuf, rows, vbuf, rows, 0.0, gram, nb, gws, gws_bytes, st)) return -1;
    qr_larft_kernel<<<1, 256, 0, st>>>(gram, nb, tau + j0, T);
    RLRA_LAUNCHED();
    // two-level blocking: the panel's update C = (I - V T^T V^T) C reaches the
    // columns of its outer block of QR_NBO only; a completed outer block is
    // applied to everything right of it at once with its own block reflector
    // (V_b, T_b: GEMMs with a 128-deep inner dimension instead of 16)
    const int64_t ob0 = (j0 / QR_NBO) * QR_NBO, oend = std::min<int64_t>(n, ob0 + QR_NBO);
    const int64_t nc = oend - j0 - nb;
    if (nc > 0) {
      double* C = a + cm(j0, j0 + nb, lda);
      if (gemm(true, false, nb, nc, rows, 1.0, vbuf, rows, C, lda, 0.0, wbuf, nb, gws, gws_bytes, st)) return -1;
      if (gemm(true, false, nb, nc, nb, 1.0, T, nb, wbuf, nb, 0.0, w2buf, nb, gws, gws_bytes, st)) return -1;
      if (gemm(false, false, rows, nc, nb, -1.0, vbuf, rows, w2buf, nb, 1.0, C, lda, gws, gws_bytes, st)) return -1;
    }
    if (j0 + nb == oend) {  // outer block complete: V_b, T_b (kept for orgqr), update the rest
      const int64_t rb = m - ob0;
      const int nbo = (int)(oend - ob0);
      double* Tb = tbig + (ob0 / QR_NBO) * QR_NBO * QR_NBO;
      qr_make_v_kernel<<<grid_for_q(rb * nbo), 256, 0, st>>>(a, lda, ob0, rb, nbo, vbuf, rb);
      RLRA_LAUNCHED();
      if (gemm(true, false, nbo, nbo, rb, 1.0, vbuf, rb, vbuf, rb, 0.0, gram, nbo, gws, gws_bytes, st)) return -1;
      qr_larft_big_kernel<<<1, QR_NBO, (size_t)QR_NBO * (QR_NBO + 1) * sizeof(double), st>>>(gram, nbo, tau + ob0,
                                                                                           Tb);
      RLRA_LAUNCHED();
      const int64_t ncb = n - oend;
      if (ncb > 0) {
        double* C = a + cm(ob0, oend, lda);
        if (gemm(true, false, nbo, ncb, rb, 1.0, vbuf, rb, C, lda, 0.0, wbuf, nbo, gws, gws_bytes, st)) return -1;
        if (gemm(true, false, nbo, ncb, nbo, 1.0, Tb, nbo, wbuf, nbo, 0.0, w2buf, nbo, gws, gws_bytes, st))
          return -1;
        if (gemm(false, false, rb, ncb, nbo, -1.0, vbuf, rb, w2buf, nbo, 1.0, C, lda, gws, gws_bytes, st))
          return -1;
      }
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
  double* wbuf = reinterpret_cast<double*>(base + L.wbuf);
  double* w2buf = reinterpret_cast<double*>(base + L.w2buf);
  void* gws = base + L.gemm_ws;
  const size_t gws_bytes = L.total - L.gemm_ws;
  set_identity_kernel<<<grid_for_q(m * n), 256, 0, st>>>(q, ldq, m, n);
  RLRA_LAUNCHED();
  double* tbig = reinterpret_cast<double*>(base + L.tbig);
  // outer blocks (V_b, T_b from geqrf), last to first
  for (int64_t ob = ceil_div(n, QR_NBO) - 1; ob >= 0; ob--) {
    const int64_t ob0 = ob * QR_NBO;
    const int nbo = (int)std::min<int64_t>(QR_NBO, n - ob0);
    const int64_t rows = m - ob0;
    const int64_t nc = n - ob0;
    qr_make_v_kernel<<<grid_for_q(rows * nbo), 256, 0, st>>>(a, lda, ob0, rows, nbo, vbuf, rows);
    RLRA_LAUNCHED();
    const double* Tb = tbig + ob * QR_NBO * QR_NBO;
    double* Qs = q + cm(ob0, ob0, ldq);
    // Qs = (I - V T V^T) Qs
    if (gemm(true, false, nbo, nc, rows, 1.0, vbuf, rows, Qs, ldq, 0.0, wbuf, nbo, gws, gws_bytes, st)) return -1;
    if (gemm(false, false, nbo, nc, nbo, 1.0, Tb, nbo, wbuf, nbo, 0.0, w2buf, nbo, gws, gws_bytes, st)) return -1;
    if (gemm(false, false, rows, nc, nbo, -1.0, vbuf, rows, w2buf, nbo, 1.0, Qs, ldq, gws, gws_bytes, st))
      return -1;
  }
  return 0;
}

}  // namespace rlra
