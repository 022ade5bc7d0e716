// K4 fast path: the final basis of powerlu by CholeskyQR2 instead of Householder.
// The Householder panels of K4 are latency bound (one cluster exchange per
// column); CholeskyQR2 turns the whole QR of the n x l sketch Z into four
// tall GEMMs on the FP64 tensor pipe plus two l x l factorizations:
//   G1 = Z^T Z,  R1 = chol(G1),  Q1 = Z R1^{-1}
//   G2 = Q1^T Q1, R2 = chol(G2), Q = Q1 R2^{-1}
// (Fukaya et al.; orthogonal to working precision for cond(Z) < ~u^{-1/2}).
// Q spans range(Z) like LAPACK's Householder Q (rlra/kernels.py:57-61); the
// columns may differ in sign, which leaves every powerlu output (p, q, L, U)
// unchanged -- flipping column j of V_k flips column j of G = A V_k and of
// U1, and B = V_k U1^T is sign-invariant.  Structural rank collapse (an exactly
// dependent sketch column, rlra/rangefinder.py:55-64) and ill-conditioned
// sketches make the Cholesky fail or exceed the condition bound; the kernel
// then raises a device flag and the driver redoes the call on the Householder
// path, so exceptions and results keep the reference semantics.
//
// chol_kernel: one CTA, the l x l matrix packed (upper triangle) in shared
// memory, blocked right-looking Cholesky G = R^T R; R (packed) replaces G.
// inv_upper_kernel: X = R^{-1}, one warp per column, ceil(l/16) CTAs.
#include <algorithm>

#include "common.cuh"

namespace rlra {

constexpr int CHOL_THREADS = 512;

__host__ __device__ __forceinline__ int pk(int i, int j) { return j * (j + 1) / 2 + i; }  // i <= j

// global -> shared staging with every element in flight at once (LDGSTS): the
// plain load/store loops waited one global latency per handful of elements
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Blocked (CHOL_NB = 16) right-looking Cholesky in shared memory, one CTA:
//   diagonal block by warp 0 in registers (shuffles), the block row by a
//   forward substitution per column (one thread each), the NEXT diagonal block
//   updated first by warps 0-3 (named barrier 1, 128 threads) so that warp 0
//   can start on it while the rest of the trailing triangle gets its rank-16
//   update in 2-D super-tiles of 4 x 4 register tiles.
// Then X = R^{-1} column by column (one warp each, back substitution, R read
// only), written straight to global memory.
constexpr int CHOL_NB = 16;

#ifdef CHOL_TRACE  // tools/chol_probe.cu: globaltimer stamps [iteration][8]
__device__ unsigned long long* g_chol_trace;
void chol_set_trace(unsigned long long* p) { cudaMemcpyToSymbol(g_chol_trace, &p, sizeof(p)); }
#define CTRACE(slot)                                                                           \
  do {                                                                                         \
    unsigned long long t_;                                                                     \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                     \
    if (g_chol_trace && it + 1 < 20) g_chol_trace[(it + 1) * 8 + (slot)] = t_;                 \
  } while (0)
#else
#define CTRACE(slot) \
  do {               \
  } while (0)
#endif
constexpr int CHOL_MAXL = 256;

__global__ void __launch_bounds__(CHOL_THREADS, 1)
    chol_kernel(double* __restrict__ g, int64_t ldg, int l, int* __restrict__ flag, double cond_limit) {
  extern __shared__ double P[];
  double* dinv = P + (size_t)l * (l + 1) / 2;  // 1 / R_ii
  __shared__ double Xkk[CHOL_NB][CHOL_NB + 1];  // current diagonal block R_kk (row-major)
  __shared__ int s_bad;
  __shared__ double s_rmin, s_rmax;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = CHOL_THREADS / 32;
  for (int j = warp; j < l; j += NW)
    for (int i = lane; i <= j; i += 32) cp_async8(&P[pk(i, j)], &g[i + (int64_t)j * ldg]);
  cp_async_wait_all();
  if (tid == 0) {
    s_bad = 0;
    s_rmin = INFINITY;
    s_rmax = 0.0;
  }
  __syncthreads();
  // (1) factor the diagonal block at k0 (warp 0): lane c holds column k0 + c
  auto diag = [&](const int k0, const int b) {
      double gg[CHOL_NB];
#pragma unroll
      for (int i = 0; i < CHOL_NB; i++) gg[i] = (lane < b && i <= lane) ? P[pk(k0 + i, k0 + lane)] : 0.0;
      bool bad = false;
      double rmin = INFINITY, rmax = 0.0;
#pragma unroll
      for (int s2 = 0; s2 < CHOL_NB; s2++) {
        if (s2 < b) {
          const double d = __shfl_sync(0xffffffffu, gg[s2], s2);
          if (!(d > 0.0 && d < INFINITY)) bad = true;
          const double ir = rsqrt(d), r = d * ir;
          rmin = fmin(rmin, r);
          rmax = fmax(rmax, r);
          if (lane == s2) gg[s2] = r;
          else if (lane > s2) gg[s2] *= ir;
#pragma unroll
          for (int i = s2 + 1; i < CHOL_NB; i++) {
            const double rsi = __shfl_sync(0xffffffffu, gg[s2], i);
            if (lane >= i && i < b) gg[i] = fma(-rsi, gg[s2], gg[i]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < CHOL_NB; i++)
        if (lane < b && i <= lane) P[pk(k0 + i, k0 + lane)] = gg[i];
      double dl = 1.0;
#pragma unroll
      for (int i = 0; i < CHOL_NB; i++)
        if (i == lane) dl = gg[i];
      if (lane < b) dinv[k0 + lane] = 1.0 / dl;
      // R_kk staged row-major for the block-row substitution (zero outside
      // the b x b triangle)
#pragma unroll
      for (int i = 0; i < CHOL_NB; i++)
        if (lane < CHOL_NB) Xkk[i][lane] = (i <= lane && lane < b) ? gg[i] : 0.0;
      if (lane == 0) {
        if (bad) s_bad = 1;
        s_rmin = fmin(s_rmin, rmin);
        s_rmax = fmax(s_rmax, rmax);
      }
  };
  // iteration it applies block it (k0 = it * NB) and factors block it + 1;
  // it = -1 only factors block 0 -- ONE inlined copy of diag() (code size:
  // the unrolled register factorization is the bulk of the kernel's SASS)
  for (int it = -1;; it++) {
    const int k0 = it * CHOL_NB;
    const int b = it < 0 ? 0 : min(CHOL_NB, l - k0);
    if (tid == 0) CTRACE(0);
    if (s_bad) break;
    const int c0 = it < 0 ? 0 : k0 + b, m = l - c0;
    if (m <= 0) break;
    // ---- (2) block row: R(k0.., j) = R_kk^{-T} G(k0.., j), one thread per
    // column: forward substitution with the column's 16 entries in registers
    // (R_kk reads are warp broadcasts; no inverse of R_kk on the warp-0 chain)
#ifdef CHOL_EXP_NOBLKROW
    for (int jj = tid; false; jj += CHOL_THREADS) {
#else
    for (int jj = tid; it >= 0 && jj < m; jj += CHOL_THREADS) {
#endif
      const int j = c0 + jj, cj = j * (j + 1) / 2 + k0;
      double x[CHOL_NB];
#pragma unroll
      for (int u = 0; u < CHOL_NB; u++) x[u] = (u < b) ? P[cj + u] : 0.0;
#pragma unroll
      for (int s2 = 0; s2 < CHOL_NB; s2++) {
        x[s2] *= (s2 < b) ? dinv[k0 + s2] : 1.0;
#pragma unroll
        for (int u = s2 + 1; u < CHOL_NB; u++) x[u] = fma(-Xkk[s2][u], x[s2], x[u]);
        asm volatile("" ::: "memory");  // keep the R_kk row loads per step (no hoisting / spills)
      }
#pragma unroll
      for (int u = 0; u < CHOL_NB; u++)
        if (u < b) P[cj + u] = x[u];
    }
    if (tid == 0) CTRACE(1);
    if (tid == 32) CTRACE(5);
    __syncthreads();
    if (tid == 0) CTRACE(2);
    // ---- (3) trailing triangle -= R(k0.., :)^T R(k0.., :).  Look-ahead: warps
    // 0..3 update the NEXT diagonal block (bar.sync 1, 128), warp 0 then factors
    // it while the other warps update the rest of the triangle in 4 x 4 tiles.
    const int bn = min(CHOL_NB, m);
    if (warp < 4) {
      // the next diagonal block's update, one entry per thread of warps 0..3
#ifdef CHOL_EXP_NONEXT
      const int ne = 0;
#else
      const int ne = it < 0 ? 0 : bn * (bn + 1) / 2;
#endif
      for (int e = tid; e < ne; e += 128) {
        int jj = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
        while (jj * (jj + 1) / 2 > e) --jj;
        while ((jj + 1) * (jj + 2) / 2 <= e) ++jj;
        const int i = c0 + (e - jj * (jj + 1) / 2), j = c0 + jj;
        const int bi = i * (i + 1) / 2 + k0, bj = j * (j + 1) / 2 + k0;
        double acc = 0.0;
#pragma unroll
        for (int s2 = 0; s2 < CHOL_NB; s2++)
          if (s2 < b) acc = fma(P[bi + s2], P[bj + s2], acc);
        P[pk(i, j)] -= acc;
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
    }
    if (warp == 0) {
      if (lane == 0) CTRACE(3);
#ifdef CHOL_EXP_NODIAG
      if (it < 0)
#endif
      diag(c0, bn);
      if (lane == 0) CTRACE(4);
    } else {
#ifdef CHOL_EXP_NOTRAIL
      const int mt = 0;
#else
      const int mt = it < 0 ? 0 : (m + 3) >> 2;
#endif
      // 4 x 4 register tiles, grouped per warp into 4 (ta) x 8 (tb) super-tiles:
      // a block-row load touches 4 (ra) or 8 (rb) distinct addresses per warp
      // instead of 32 scattered columns (the former 1-D tile order ran the
      // trailing update at ~5-way shared-memory bank conflicts)
      const int nsa = (mt + 3) >> 2, nsb = (mt + 7) >> 3;
      const int lim = c0 + bn;  // entries with i, j < lim belong to warps 0..3
      for (int st = warp - 1; st < nsa * nsb; st += NW - 1) {
        const int sa = st % nsa, sb = st / nsa;
        if (4 * sa > 8 * sb + 7) continue;  // whole super-tile below the diagonal
        const int ta = 4 * sa + (lane & 3), tb = 8 * sb + (lane >> 2);
        if (ta > tb || tb >= mt) continue;
        const int ja = c0 + 4 * ta, jb = c0 + 4 * tb;
        if (jb + 3 < lim) continue;  // whole tile inside the next diagonal block
        double acc[4][4];
#pragma unroll
        for (int q = 0; q < 4; q++)
#pragma unroll
          for (int w = 0; w < 4; w++) acc[q][w] = 0.0;
        // packed column c holds rows 0..c contiguously: the block row's entries
        // (k0 + s2, c) sit at c(c+1)/2 + k0 + s2 (columns past l are clamped:
        // their products are never stored)
        int ba[4], bb[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int ca = min(ja + q, l - 1), cb = min(jb + q, l - 1);
          ba[q] = ca * (ca + 1) / 2 + k0;
          bb[q] = cb * (cb + 1) / 2 + k0;
        }
#pragma unroll 4
        for (int s2 = 0; s2 < b; s2++) {
          double ra[4], rb[4];
#pragma unroll
          for (int q = 0; q < 4; q++) {
            ra[q] = P[ba[q] + s2];
            rb[q] = P[bb[q] + s2];
          }
#pragma unroll
          for (int q = 0; q < 4; q++)
#pragma unroll
            for (int w = 0; w < 4; w++) acc[q][w] = fma(ra[q], rb[w], acc[q][w]);
        }
#pragma unroll
        for (int q = 0; q < 4; q++)
#pragma unroll
          for (int w = 0; w < 4; w++) {
            const int i = ja + q, j = jb + w;
            if (i <= j && j < l && !(j < lim)) P[pk(i, j)] -= acc[q][w];
          }
      }
    }
    if (tid == 32) CTRACE(6);
    if (tid == CHOL_THREADS - 1) CTRACE(7);
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0 && !s_bad && !(s_rmax <= cond_limit * s_rmin)) s_bad = 1;
  __syncthreads();
  if (s_bad) {
    if (tid == 0) atomicExch(flag, 1);
    return;
  }
  // R (packed upper) over the consumed G: rows of the inverse kernel's input
  const int np = l * (l + 1) / 2;
  for (int e = tid; e < np; e += CHOL_THREADS) g[e] = P[e];
}

// X = R^{-1}: warp per column, back substitution (x_t = acc_t / R_tt, then
// acc_i -= R_it x_t for i < t), R packed in shared memory; ceil(l/16) CTAs.
constexpr int INV_COLS = 16;

__global__ void __launch_bounds__(INV_COLS * 32, 1)
    inv_upper_kernel(const double* __restrict__ rp, int l, double* __restrict__ x, int64_t ldx,
                     const int* __restrict__ flag) {
  extern __shared__ double P[];
  double* dinv = P + (size_t)l * (l + 1) / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j = blockIdx.x * INV_COLS + warp;
  if (*flag) {  // the Cholesky declined: zero output (the caller falls back)
    if (j < l)
      for (int i = lane; i < l; i += 32) x[i + (int64_t)j * ldx] = 0.0;
    return;
  }
  const int np = l * (l + 1) / 2;
  for (int e = tid; e < np; e += blockDim.x) cp_async8(&P[e], &rp[e]);
  cp_async_wait_all();
  __syncthreads();
  for (int t = tid; t < l; t += blockDim.x) dinv[t] = 1.0 / P[pk(t, t)];
  __syncthreads();
  if (j >= l) return;
  double a[CHOL_MAXL / 32];
#pragma unroll
  for (int q = 0; q < CHOL_MAXL / 32; q++) a[q] = (lane + 32 * q == j) ? 1.0 : 0.0;
#pragma unroll
  for (int q = CHOL_MAXL / 32 - 1; q >= 0; q--) {
    if (32 * q > j) continue;
    const int thi = min(j, 32 * q + 31);
    for (int t = thi; t >= 32 * q; --t) {
      const double xt = __shfl_sync(0xffffffffu, a[q], t & 31) * dinv[t];
      if (lane == (t & 31)) a[q] = xt;
      const int ct = t * (t + 1) / 2;
#pragma unroll
      for (int q2 = 0; q2 <= q; q2++) {
        const int i = lane + 32 * q2;
        if (i < t) a[q2] = fma(-P[ct + i], xt, a[q2]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < CHOL_MAXL / 32; q++) {
    const int i = lane + 32 * q;
    if (i < l) x[i + (int64_t)j * ldx] = (i <= j) ? a[q] : 0.0;
  }
}

// Shifted CholeskyQR (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa 2020):
// G + s I with s = c * trace(G) (trace(Z^T Z) = ||Z||_F^2 >= ||Z||_2^2), so
// the Cholesky of the first step of sCholQR3 succeeds for cond(Z) up to ~u^-1.
// One CTA: fixed-order trace reduction, then the diagonal update.
__global__ void __launch_bounds__(256) shift_diag_kernel(double* __restrict__ g, int64_t ldg, int l, double c) {
  __shared__ double red[8];
  double t = 0.0;
  for (int i = threadIdx.x; i < l; i += 256) t += g[i + (int64_t)i * ldg];
#pragma unroll
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  double tr = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) tr += red[w];
  const double s = c * tr;
  for (int i = threadIdx.x; i < l; i += 256) g[i + (int64_t)i * ldg] += s;
}

// flag := 1 when max_i |d_ii| > cond_limit * min_i |d_ii| (or a zero / NaN
// diagonal): the condition bound of a blocked Cholesky across its blocks (the
// one-CTA kernel checks it inside a block).
__global__ void __launch_bounds__(256) diag_ratio_flag_kernel(const double* __restrict__ d, int64_t ldd, int l,
                                                              double cond_limit, int* __restrict__ flag) {
  __shared__ double rmax[8], rmin[8];
  double mx = 0.0, mn = __longlong_as_double(0x7FF0000000000000ll);
  bool bad = false;
  for (int i = threadIdx.x; i < l; i += 256) {
    const double v = fabs(d[i + (int64_t)i * ldd]);
    bad |= !(v > 0.0) || !(v <= 1.7976931348623157e308);
    mx = fmax(mx, v);
    mn = fmin(mn, v);
  }
  bad = __syncthreads_or(bad);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  if ((threadIdx.x & 31) == 0) {
    rmax[threadIdx.x >> 5] = mx;
    rmin[threadIdx.x >> 5] = mn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < 8; ++w) {
      mx = fmax(mx, rmax[w]);
      mn = fmin(mn, rmin[w]);
    }
    if (bad || !(mx <= cond_limit * mn)) atomicExch(flag, 1);
  }
}

// flag := 1 when max_ij |g_ij - delta_ij| > tol (or non-finite): the Gram of
// CholeskyQR's first Q deviates from I by ~u cond(Z)^2, so this declines
// sketches beyond ~u^-1/2 whatever their R diagonal ratio says.
__global__ void __launch_bounds__(256) gram_identity_flag_kernel(const double* __restrict__ g, int64_t ldg, int l,
                                                                 double tol, int* __restrict__ flag) {
  bool bad = false;
  const int64_t total = (int64_t)l * l;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total; e += (int64_t)gridDim.x * 256) {
    const int i = (int)(e % l), j = (int)(e / l);
    const double d = fabs(g[i + (int64_t)j * ldg] - (i == j ? 1.0 : 0.0));
    bad |= !(d <= tol);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

int gram_identity_flag(const double* g, int64_t ldg, int64_t l, double tol, int* flag, cudaStream_t st) {
  RLRA_REQUIRE(l >= 1 && ldg >= l && flag, "gram_identity_flag: bad arguments");
  const int64_t blocks = std::min<int64_t>(ceil_div(l * l, 256), 148);
  gram_identity_flag_kernel<<<(unsigned)blocks, 256, 0, st>>>(g, ldg, (int)l, tol, flag);
  RLRA_LAUNCHED();
  return 0;
}

int chol_shift_diag(double* g, int64_t ldg, int64_t l, double c, cudaStream_t st) {
  RLRA_REQUIRE(l >= 1 && ldg >= l, "chol_shift_diag: bad shape");
  shift_diag_kernel<<<1, 256, 0, st>>>(g, ldg, (int)l, c);
  RLRA_LAUNCHED();
  return 0;
}

int diag_ratio_flag(const double* d, int64_t ldd, int64_t l, double cond_limit, int* flag, cudaStream_t st) {
  RLRA_REQUIRE(l >= 1 && ldd >= l && flag, "diag_ratio_flag: bad arguments");
  diag_ratio_flag_kernel<<<1, 256, 0, st>>>(d, ldd, (int)l, cond_limit, flag);
  RLRA_LAUNCHED();
  return 0;
}

int chol_inv_max_l() {
  const int smem = device_info().max_smem_optin > 0 ? device_info().max_smem_optin : 227 * 1024;
  int l = 1;
  while (l + 1 <= CHOL_MAXL && (size_t)(l + 1) * (l + 2) / 2 * 8 + (size_t)(l + 1) * 8 + 10 * 1024 <= (size_t)smem) ++l;
  return l;
}

int chol_inv(double* g, int64_t ldg, int64_t l, double* x, int64_t ldx, int* flag, double cond_limit,
             cudaStream_t st) {
  RLRA_REQUIRE(l >= 1 && l <= chol_inv_max_l(), "chol_inv: l = %lld outside [1, %d]", (long long)l,
               chol_inv_max_l());
  RLRA_REQUIRE(ldg >= l && ldx >= l, "chol_inv: bad leading dimension");
  const size_t smem = (size_t)l * (l + 1) / 2 * 8 + (size_t)l * 8;
  static int configured = -1;
  int dev = 0;
  RLRA_CHECK_CUDA(cudaGetDevice(&dev));
  if (configured != dev) {
    RLRA_CHECK_CUDA(cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         device_info().max_smem_optin - 9 * 1024));
    RLRA_CHECK_CUDA(cudaFuncSetAttribute(inv_upper_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         device_info().max_smem_optin - 9 * 1024));
    configured = dev;
  }
  chol_kernel<<<1, CHOL_THREADS, smem, st>>>(g, ldg, (int)l, flag, cond_limit);
  RLRA_LAUNCHED();
  inv_upper_kernel<<<(unsigned)ceil_div(l, INV_COLS), INV_COLS * 32, smem, st>>>(g, (int)l, x, ldx, flag);
  RLRA_LAUNCHED();
  return 0;
}

}  // namespace rlra
