// K1/K2/K5: FP64 GEMM on the DMMA tensor pipe (mma.sync m8n8k4 f64 -> SASS
// DMMA.8x8x4; sm_100a has no tcgen05 kind::f64).
//
//   C (M x N, column-major, ldc) = alpha * op(A) * op(B) + beta * C
//   op(A) = A (M x K, col-major, M contiguous)      when !TA   -- Y = A W   (pass NN)
//         = A^T with A K x M col-major (K contiguous) when TA   -- Z = A^T W (pass TN)
//   op(B) = B (K x N, col-major, K contiguous)      when !TB
//         = B^T with B N x K col-major (N contiguous) when TB   -- V U1^T, L1 U2^T
//
// Replaces the reference's DenseAccessor.matmul / rmatmul (rlra/accessors.py:27-31,
// NumPy -> OpenBLAS dgemm) and the assembly products of
// rlra/fixedrank.py:145-146 / rlra/kernels.py:96.
//
// Design: CTA tile BM x BN x 16, 8 warps, warp tile (WM*8) x (WN*8) of register
// accumulators, a STAGES-deep cp.async ring (LDGSTS) in shared memory padded so
// every 64-bit fragment load is bank-conflict free, and a deterministic split-K
// (partials to workspace, fixed-order reduction) chosen on the host so the
// tile count fills whole waves of the 148 SMs.  No atomics: results are
// bitwise reproducible run to run.
#include "common.cuh"

namespace rlra {

struct GemmArgs {
  int64_t M, N, K;
  const double* A; int64_t lda;
  const double* B; int64_t ldb;
  double* C; int64_t ldc;
  double alpha, beta;
  int64_t ktiles_per_split;  // in units of BK
  int splits;
  double* partial;           // splits x M x N (ld = M) when splits > 1
};

__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int WARPS_M, int WARPS_N, int WM, int WN, int STAGES, bool TA, bool TB, int VEC>
struct GemmCfg {
  static constexpr int BM = WARPS_M * WM * 8;
  static constexpr int BN = WARPS_N * WN * 8;
  static constexpr int BK = 16;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  // smem strides (doubles); every stride == 4 (mod 16) => conflict-free LDS.64
  static constexpr int A_LD = TA ? (BK + 4) : (BM + 4);
  static constexpr int A_ROWS = TA ? BM : BK;
  static constexpr int B_LD = TB ? (BN + 4) : (BK + 4);
  static constexpr int B_ROWS = TB ? BK : BN;
  static constexpr int A_STAGE = A_LD * A_ROWS;
  static constexpr int B_STAGE = B_LD * B_ROWS;
  static constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * 8;
  static_assert(A_LD % 16 == 4 && B_LD % 16 == 4, "padding must keep fragment loads conflict-free");
};

template <int WARPS_M, int WARPS_N, int WM, int WN, int STAGES, bool TA, bool TB, int VEC>
__global__ void __launch_bounds__(WARPS_M * WARPS_N * 32, 1)
dgemm_dmma_kernel(GemmArgs p) {
  using Cfg = GemmCfg<WARPS_M, WARPS_N, WM, WN, STAGES, TA, TB, VEC>;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, THREADS = Cfg::THREADS;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::A_STAGE;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int warp_m = warp % WARPS_M, warp_n = warp / WARPS_M;
  const int64_t n0 = (int64_t)blockIdx.x * BN;
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int split = blockIdx.z;
  const int64_t ktiles_total = ceil_div(p.K, BK);
  const int64_t kt_begin = (int64_t)split * p.ktiles_per_split;
  const int64_t kt_end = min(ktiles_total, kt_begin + p.ktiles_per_split);
  const int64_t nkt = kt_end > kt_begin ? kt_end - kt_begin : 0;

  auto load_stage = [&](int slot, int64_t kt) {
    const int64_t k0 = kt * BK;
    double* as = As + slot * Cfg::A_STAGE;
    double* bs = Bs + slot * Cfg::B_STAGE;
    // ---- A tile
    if (!TA) {  // smem [k][m], m contiguous in global
      constexpr int CH = BM / VEC;  // chunks per k-row
      for (int c = tid; c < BK * CH; c += THREADS) {
        int kk = c / CH, mm = (c % CH) * VEC;
        int64_t gm = m0 + mm, gk = k0 + kk;
        bool ok = gm < p.M && gk < p.K;
        const double* src = ok ? p.A + cm(gm, gk, p.lda) : p.A;
        if (VEC == 2) cp_async_16(as + kk * Cfg::A_LD + mm, src, ok);
        else cp_async_8(as + kk * Cfg::A_LD + mm, src, ok);
      }
    } else {  // smem [m][k], k contiguous in global
      constexpr int CH = BK / VEC;
      for (int c = tid; c < BM * CH; c += THREADS) {
        int mm = c / CH, kk = (c % CH) * VEC;
        int64_t gm = m0 + mm, gk = k0 + kk;
        bool ok = gm < p.M && gk < p.K;
        const double* src = ok ? p.A + cm(gk, gm, p.lda) : p.A;
        if (VEC == 2) cp_async_16(as + mm * Cfg::A_LD + kk, src, ok);
        else cp_async_8(as + mm * Cfg::A_LD + kk, src, ok);
      }
    }
    // ---- B tile
    if (!TB) {  // smem [n][k], k contiguous in global
      constexpr int CH = BK / VEC;
      for (int c = tid; c < BN * CH; c += THREADS) {
        int nn = c / CH, kk = (c % CH) * VEC;
        int64_t gn = n0 + nn, gk = k0 + kk;
        bool ok = gn < p.N && gk < p.K;
        const double* src = ok ? p.B + cm(gk, gn, p.ldb) : p.B;
        if (VEC == 2) cp_async_16(bs + nn * Cfg::B_LD + kk, src, ok);
        else cp_async_8(bs + nn * Cfg::B_LD + kk, src, ok);
      }
    } else {  // smem [k][n], n contiguous in global
      constexpr int CH = BN / VEC;
      for (int c = tid; c < BK * CH; c += THREADS) {
        int kk = c / CH, nn = (c % CH) * VEC;
        int64_t gn = n0 + nn, gk = k0 + kk;
        bool ok = gn < p.N && gk < p.K;
        const double* src = ok ? p.B + cm(gn, gk, p.ldb) : p.B;
        if (VEC == 2) cp_async_16(bs + kk * Cfg::B_LD + nn, src, ok);
        else cp_async_8(bs + kk * Cfg::B_LD + nn, src, ok);
      }
    }
  };

  double acc[WM][WN][2];
#pragma unroll
  for (int i = 0; i < WM; i++)
#pragma unroll
    for (int j = 0; j < WN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; s++) {
    if (s < nkt) load_stage(s, kt_begin + s);
    cp_async_commit();
  }

  const int wm0 = warp_m * WM * 8;
  const int wn0 = warp_n * WN * 8;
  for (int64_t it = 0; it < nkt; it++) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int64_t nxt = it + STAGES - 1;
      if (nxt < nkt) load_stage((int)(nxt % STAGES), kt_begin + nxt);
      cp_async_commit();
    }
    const int slot = (int)(it % STAGES);
    const double* as = As + slot * Cfg::A_STAGE;
    const double* bs = Bs + slot * Cfg::B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[WM], bf[WN];
#pragma unroll
      for (int i = 0; i < WM; i++) {
        int mm = wm0 + i * 8 + g, k = kk + t;
        af[i] = TA ? as[mm * Cfg::A_LD + k] : as[k * Cfg::A_LD + mm];
      }
#pragma unroll
      for (int j = 0; j < WN; j++) {
        int nn = wn0 + j * 8 + g, k = kk + t;
        bf[j] = TB ? bs[k * Cfg::B_LD + nn] : bs[nn * Cfg::B_LD + k];
      }
#pragma unroll
      for (int i = 0; i < WM; i++)
#pragma unroll
        for (int j = 0; j < WN; j++) dmma_884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // ---- epilogue
#pragma unroll
  for (int i = 0; i < WM; i++) {
    int64_t gm = m0 + wm0 + i * 8 + g;
    if (gm >= p.M) continue;
#pragma unroll
    for (int j = 0; j < WN; j++) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        int64_t gn = n0 + wn0 + j * 8 + 2 * t + h;
        if (gn >= p.N) continue;
        double v = acc[i][j][h];
        if (p.splits > 1) {
          p.partial[(int64_t)split * p.M * p.N + gm + gn * p.M] = v;
        } else {
          double* c = p.C + cm(gm, gn, p.ldc);
          *c = (p.beta == 0.0) ? p.alpha * v : p.alpha * v + p.beta * *c;
        }
      }
    }
  }
}

// Fixed-order split-K reduction (deterministic), alpha/beta epilogue.
__global__ void splitk_reduce_kernel(const double* __restrict__ partial, int splits, int64_t M,
                                     int64_t N, double alpha, double beta, double* C, int64_t ldc) {
  const int64_t total = M * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = partial[e];
    for (int k = 1; k < splits; k++) s += partial[(int64_t)k * total + e];
    int64_t m = e % M, n = e / M;
    double* c = C + cm(m, n, ldc);
    *c = (beta == 0.0) ? alpha * s : alpha * s + beta * *c;
  }
}

// ------------------------------------------------------------------ host side
struct TileChoice {
  int bm, bn;
  int which;  // 0: 128x128, 1: 128x112, 2: 128x96, 3: 128x80
};

static TileChoice choose_tile(int64_t N) {
  const int bns[4] = {128, 112, 96, 80};
  TileChoice best{128, 128, 0};
  int64_t best_pad = -1;
  for (int w = 0; w < 4; w++) {
    int64_t padded = ceil_div(N, bns[w]) * bns[w];
    if (best_pad < 0 || padded < best_pad) {
      best_pad = padded;
      best = TileChoice{128, bns[w], w};
    }
  }
  return best;
}

struct SplitPlan {
  int splits;
  int64_t ktiles_per_split;
};

// Split-K plan from a simple time model (microseconds): waves x k-tiles per
// split x the DMMA time of one BM x BN x 16 k-tile (64 FMA/clk/SM at ~1.9 GHz),
// plus the fixed-order reduction (read s partials + write C at ~4 TB/s, and a
// launch).  Deterministic for a given shape and SM count.
static SplitPlan plan_splits(int64_t M, int64_t N, int bm, int bn, int64_t tiles, int64_t ktiles,
                             int slots) {
  const double t_ktile = (double)bm * bn * 16 / (64.0 * 1.9e3);
  SplitPlan best{1, ktiles};
  double best_t = 1e300;
  for (int s = 1; s <= 32; s++) {
    int64_t kps = ceil_div(ktiles, s);
    if (s > 1 && kps < 4) break;
    int64_t real_s = ceil_div(ktiles, kps);
    if (real_s != s) continue;
    double waves = (double)ceil_div(tiles * real_s, slots);
    double t = waves * kps * t_ktile;
    if (real_s > 1) t += 4.0 + (double)(real_s + 1) * M * N * 8 / 4e6;
    if (t < best_t * 0.98) {  // prefer fewer splits unless clearly faster
      best_t = t;
      best = SplitPlan{(int)real_s, kps};
    }
  }
  return best;
}

template <int WARPS_M, int WARPS_N, int WM, int WN, bool TA, bool TB, int VEC>
static int launch_cfg(GemmArgs& a, cudaStream_t st) {
  constexpr int STAGES = 4;
  using Cfg = GemmCfg<WARPS_M, WARPS_N, WM, WN, STAGES, TA, TB, VEC>;
  auto kern = dgemm_dmma_kernel<WARPS_M, WARPS_N, WM, WN, STAGES, TA, TB, VEC>;
  static unsigned attr_mask = 0;  // one bit per device ordinal
  int dev = 0;
  RLRA_CHECK_CUDA(cudaGetDevice(&dev));
  if (!(attr_mask & (1u << (dev & 31)))) {
    RLRA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::SMEM_BYTES));
    attr_mask |= 1u << (dev & 31);
  }
  dim3 grid((unsigned)ceil_div(a.N, Cfg::BN), (unsigned)ceil_div(a.M, Cfg::BM), (unsigned)a.splits);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(a);
  RLRA_LAUNCHED();
  return 0;
}

template <bool TA, bool TB, int VEC>
static int launch_tile(int which, GemmArgs& a, cudaStream_t st) {
  switch (which) {
    case 0: return launch_cfg<2, 4, 8, 4, TA, TB, VEC>(a, st);  // 128 x 128, warp 64x32
    case 1: return launch_cfg<4, 2, 4, 7, TA, TB, VEC>(a, st);  // 128 x 112, warp 32x56
    case 2: return launch_cfg<2, 4, 8, 3, TA, TB, VEC>(a, st);  // 128 x 96,  warp 64x24
    default: return launch_cfg<4, 2, 4, 5, TA, TB, VEC>(a, st); // 128 x 80,  warp 32x40
  }
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

bool tma_gemm_eligible(bool ta, bool tb, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                       const double* B, int64_t ldb);
size_t tma_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K);
int tma_gemm(bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
             const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* ws, size_t ws_bytes,
             cudaStream_t st);

int splitk_reduce(const double* partial, int splits, int64_t M, int64_t N, double alpha, double beta,
                  double* C, int64_t ldc, cudaStream_t st) {
  int64_t total = M * N;
  int blocks = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)device_info().sm_count * 8);
  splitk_reduce_kernel<<<blocks, 256, 0, st>>>(partial, splits, M, N, alpha, beta, C, ldc);
  RLRA_LAUNCHED();
  return 0;
}

// Upper bound over both mainloops (the TMA one needs aligned pointers, which a
// size query cannot see).
size_t gemm_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  const size_t tma = tma_gemm_workspace_bytes(M, N, K);
  TileChoice tc = choose_tile(N);
  int64_t tiles = ceil_div(M, tc.bm) * ceil_div(N, tc.bn);
  SplitPlan sp = plan_splits(M, N, tc.bm, tc.bn, tiles, ceil_div(K, 16), device_info().sm_count);
  const size_t legacy = sp.splits > 1 ? (size_t)sp.splits * M * N * sizeof(double) : 0;
  return std::max(tma, legacy);
}

int gemm(bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
         void* ws, size_t ws_bytes, cudaStream_t st) {
  RLRA_REQUIRE(M >= 0 && N >= 0 && K >= 0, "gemm: negative dimension");
  if (M == 0 || N == 0) return 0;
  RLRA_REQUIRE(ldc >= M, "gemm: ldc < M");
  if (tma_gemm_eligible(ta, tb, M, N, K, A, lda, B, ldb))
    return tma_gemm(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, ws_bytes, st);
  // K == 0 runs one split with no k-tiles: the epilogue writes alpha*0 + beta*C.
  TileChoice tc = choose_tile(N);
  int64_t tiles = ceil_div(M, tc.bm) * ceil_div(N, tc.bn);
  int64_t ktiles = ceil_div(K, 16);
  SplitPlan sp = K > 0 ? plan_splits(M, N, tc.bm, tc.bn, tiles, ktiles, device_info().sm_count)
                       : SplitPlan{1, 0};
  GemmArgs a{M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, sp.ktiles_per_split, sp.splits, nullptr};
  if (sp.splits > 1) {
    size_t need = (size_t)sp.splits * M * N * sizeof(double);
    RLRA_REQUIRE(ws != nullptr && ws_bytes >= need, "gemm: workspace too small (%zu < %zu)",
                 ws_bytes, need);
    a.partial = static_cast<double*>(ws);
  }
  // 16-byte vector loads need 16B-aligned bases, even leading dimensions and an
  // even extent along the contiguous dimension.
  bool vec = aligned16(A) && aligned16(B) && (lda % 2 == 0) && (ldb % 2 == 0) &&
             ((ta ? K : M) % 2 == 0) && ((tb ? N : K) % 2 == 0);
  int rc;
  if (!ta && !tb) rc = vec ? launch_tile<false, false, 2>(tc.which, a, st) : launch_tile<false, false, 1>(tc.which, a, st);
  else if (ta && !tb) rc = vec ? launch_tile<true, false, 2>(tc.which, a, st) : launch_tile<true, false, 1>(tc.which, a, st);
  else if (!ta && tb) rc = vec ? launch_tile<false, true, 2>(tc.which, a, st) : launch_tile<false, true, 1>(tc.which, a, st);
  else rc = vec ? launch_tile<true, true, 2>(tc.which, a, st) : launch_tile<true, true, 1>(tc.which, a, st);
  if (rc) return rc;
  if (sp.splits > 1) return splitk_reduce(a.partial, sp.splits, M, N, alpha, beta, C, ldc, st);
  return 0;
}

}  // namespace rlra
