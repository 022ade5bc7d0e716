// Small dense SVD for the randomized-SVD baseline (rlra/fixedrank.py:49-76,
// np.linalg.svd of the l x n projection B = Q^T A).  The driver reduces B to
// its l x l triangular factor on device (Householder QR of B^T, K4) and this
// file factors that square matrix by ONE-SIDED (Hestenes) JACOBI:
//   X V = W with mutually orthogonal columns, s_j = ||W_j||, U_j = W_j / s_j,
// so X = U diag(s) V^T.  One-sided Jacobi computes singular values to high
// relative accuracy (at least LAPACK gesdd's), which is what the reference's
// S is compared against.
//
// Parallel ordering: round-robin tournament over the (even-padded) columns,
// l_pad/2 disjoint pairs per round, one warp per pair; a cooperative grid of
// CTAs shares the rounds, separated by a monotonic grid barrier.  X and V live
// in global memory (l <= 1024: <= 8 MB each, L2-resident).  A sweep whose
// rotations were all below tol * sqrt(alpha beta) ends the iteration.
// The second kernel forms s, U and sorts the triplets by nonincreasing s
// (ties by index) -- the reference's LAPACK ordering.
#include "common.cuh"

namespace rlra {

namespace svdj {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxL = 1024;
constexpr int kMaxSweeps = 60;

struct State {
  unsigned bar;                    // monotonic grid barrier counter
  unsigned rotated[kMaxSweeps];    // sweep s applied a significant rotation
  int sweeps;                      // sweeps executed
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// round r of the circle method over N (even) players: pair i
__device__ __forceinline__ void tournament_pair(int N, int r, int i, int& a, int& b) {
  if (i == 0) {
    a = r;
    b = N - 1;
  } else {
    a = (r + i) % (N - 1);
    b = (r - i + (N - 1)) % (N - 1);
  }
  if (a > b) {
    const int t = a;
    a = b;
    b = t;
  }
}

__global__ void __launch_bounds__(kThreads) jacobi_kernel(const double* __restrict__ a, int64_t lda, int m, int l,
                                                          double* __restrict__ x, double* __restrict__ v,
                                                          State* st, double tol) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int nw = gridDim.x * kWarps;
  const int N = l + (l & 1);
  // X = A (column-major, ld = m), V = I (ld = l)
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < (int64_t)m * l; e += (int64_t)gridDim.x * kThreads)
    x[e] = a[(e % m) + (e / m) * lda];
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < (int64_t)l * l; e += (int64_t)gridDim.x * kThreads)
    v[e] = (e % l == e / l) ? 1.0 : 0.0;
  unsigned nbar = 1;
  __threadfence();
  grid_barrier_mono(&st->bar, nbar * gridDim.x);
  int sweep = 0;
  for (; sweep < kMaxSweeps; ++sweep) {
    for (int r = 0; r < N - 1; ++r) {
      for (int i = gw; i < N / 2; i += nw) {
        int p, q;
        tournament_pair(N, r, i, p, q);
        if (q >= l) continue;  // dummy column of an odd l
        double* xp = x + (int64_t)p * m;
        double* xq = x + (int64_t)q * m;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int k = lane; k < m; k += 32) {
          const double u = xp[k], w = xq[k];
          al = fma(u, u, al);
          be = fma(w, w, be);
          ga = fma(u, w, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (ga == 0.0 || fabs(ga) <= tol * sqrt(al) * sqrt(be)) continue;
        if (lane == 0) st->rotated[sweep] = 1u;
        // rotation annihilating the (p, q) inner product (Rutishauser's form)
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        const double c = 1.0 / sqrt(fma(t, t, 1.0)), s = c * t;
        for (int k = lane; k < m; k += 32) {
          const double u = xp[k], w = xq[k];
          xp[k] = c * u - s * w;
          xq[k] = s * u + c * w;
        }
        double* vp = v + (int64_t)p * l;
        double* vq = v + (int64_t)q * l;
        for (int k = lane; k < l; k += 32) {
          const double u = vp[k], w = vq[k];
          vp[k] = c * u - s * w;
          vq[k] = s * u + c * w;
        }
      }
      __threadfence();
      ++nbar;
      grid_barrier_mono(&st->bar, nbar * gridDim.x);
    }
    if (*(volatile unsigned*)&st->rotated[sweep] == 0u) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) st->sweeps = sweep + 1;
}

// s_j = ||W_j||, U_j = W_j / s_j; triplets sorted by nonincreasing s.
__global__ void __launch_bounds__(kThreads) finish_kernel(const double* __restrict__ x, int m, int l,
                                                          const double* __restrict__ v, double* __restrict__ u,
                                                          int64_t ldu, double* __restrict__ s,
                                                          double* __restrict__ vo, int64_t ldv) {
  __shared__ double sn[kMaxL];
  __shared__ int rank[kMaxL];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < l; j += kWarps) {
    double acc = 0.0;
    for (int k = lane; k < m; k += 32) acc = fma(x[(int64_t)j * m + k], x[(int64_t)j * m + k], acc);
    acc = warp_sum(acc);
    if (lane == 0) sn[j] = sqrt(acc);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < l; j += kThreads) {
    int rk = 0;
    const double sj = sn[j];
    for (int i = 0; i < l; ++i) rk += (sn[i] > sj || (sn[i] == sj && i < j)) ? 1 : 0;
    rank[j] = rk;
  }
  __syncthreads();
  for (int j = warp; j < l; j += kWarps) {
    const int d = rank[j];
    const double sj = sn[j];
    const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    for (int k = lane; k < m; k += 32) u[(int64_t)d * ldu + k] = x[(int64_t)j * m + k] * inv;
    for (int k = lane; k < l; k += 32) vo[(int64_t)d * ldv + k] = v[(int64_t)j * l + k];
    if (lane == 0) s[d] = sj;
  }
}

}  // namespace svdj

int svd_jacobi_max_l() { return svdj::kMaxL; }

size_t svd_jacobi_workspace(int64_t m, int64_t l) {
  if (m < 1 || l < 1) return 0;
  return 1024 + (size_t)(m * l + l * l) * sizeof(double);
}

int svd_jacobi(const double* a, int64_t lda, int64_t m, int64_t l, double* u, int64_t ldu, double* s, double* v,
               int64_t ldv, int* sweeps_out, void* ws, size_t ws_bytes, cudaStream_t st) {
  RLRA_REQUIRE(l >= 1 && l <= svdj::kMaxL && m >= l && m <= (1 << 20), "svd_jacobi: need 1 <= l <= %d, l <= m",
               svdj::kMaxL);
  RLRA_REQUIRE(lda >= m && ldu >= m && ldv >= l, "svd_jacobi: bad leading dimensions");
  RLRA_REQUIRE(ws && ws_bytes >= svd_jacobi_workspace(m, l), "svd_jacobi: workspace too small");
  uint8_t* base = static_cast<uint8_t*>(ws);
  svdj::State* state = reinterpret_cast<svdj::State*>(base);
  double* x = reinterpret_cast<double*>(base + 1024);
  double* vv = x + m * l;
  RLRA_CHECK_CUDA(cudaMemsetAsync(state, 0, sizeof(svdj::State), st));
  const int pairs = (int)((l + 1) / 2);
  int dev = 0, per_sm = 0;
  RLRA_CHECK_CUDA(cudaGetDevice(&dev));
  RLRA_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, svdj::jacobi_kernel, svdj::kThreads, 0));
  int grid = (int)std::min<int64_t>(ceil_div(pairs, svdj::kWarps), (int64_t)device_info().sm_count * per_sm);
  grid = grid < 1 ? 1 : grid;
  const double tol = 4.0 * 2.220446049250313e-16;
  int mi = (int)m, li = (int)l;
  void* args[] = {(void*)&a, (void*)&lda, (void*)&mi, (void*)&li, (void*)&x, (void*)&vv, (void*)&state,
                  (void*)&tol};
  RLRA_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)svdj::jacobi_kernel, dim3(grid), dim3(svdj::kThreads),
                                              args, 0, st));
  RLRA_LAUNCHED();
  svdj::finish_kernel<<<1, svdj::kThreads, 0, st>>>(x, mi, li, vv, u, ldu, s, v, ldv);
  RLRA_LAUNCHED();
  if (sweeps_out)
    RLRA_CHECK_CUDA(cudaMemcpyAsync(sweeps_out, &state->sweeps, sizeof(int), cudaMemcpyDeviceToDevice, st));
  return 0;
}

}  // namespace rlra
