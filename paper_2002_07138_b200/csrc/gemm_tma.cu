// K1/K2 pass GEMM, B200-native mainloop: TMA (cp.async.bulk.tensor) stages the A
// and B tiles into shared memory, mbarriers form a STAGES-deep full/empty ring,
// one producer warp issues the copies and 8 consumer warps only load fragments
// and issue DMMA (mma.sync m8n8k4 f64; sm_100a has no tcgen05 kind::f64).
//
// The tensor maps are 3-D views of the column-major operands that group 4
// consecutive elements of the contiguous dimension:
//   NN  A (M x K, m contiguous): dims {4 m, K, M/4}  box {4, 16, BM/4}
//       smem [m/4][k][m%4]   -> an m8n8k4 A fragment (8 m x 4 k) = 2 x 128 B rows
//   TN  A^T (K x M', k contig): dims {4 k, M', K/4}  box {4, BM, 4}
//       smem [k/4][m'][k%4]
//   B   (K x N, k contiguous):  dims {4 k, N, K/4}   box {4, BN, 4}
//       smem [k/4][n][k%4]
// so every fragment load of a half-warp reads 128 contiguous bytes (bank-
// conflict free without padding, which plain TMA boxes cannot add), and the
// hardware zero-fills the M / N / K tails.  Requirements (else the cp.async
// kernel in gemm.cu runs): 16-byte aligned bases, even leading dimensions,
// K % 4 == 0 and, for NN, M % 4 == 0.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"

namespace rlra {

struct TmaGemmArgs {
  int64_t M, N, K;
  double* C;
  int64_t ldc;
  double alpha, beta;
  int64_t ktiles_per_split;
  int splits;
  double* partial;
};

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init_cta(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra LAB_WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
          smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_addr(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int WARPS_M, int WARPS_N, int WM, int WN, int STAGES, bool TA, bool TB>
struct TmaCfg {
  static constexpr int BM = WARPS_M * WM * 8;
  static constexpr int BN = WARPS_N * WN * 8;
  static constexpr int BK = 16;
  static constexpr int CONSUMERS = WARPS_M * WARPS_N;
  static constexpr int THREADS = CONSUMERS * 32;
  static constexpr int A_STAGE = BM * BK;  // doubles
  static constexpr int B_STAGE = BN * BK;
  static constexpr int A_BYTES = A_STAGE * 8;
  static constexpr int B_BYTES = B_STAGE * 8;
  static constexpr int SMEM_BYTES = STAGES * (A_BYTES + B_BYTES) + 2 * STAGES * 8 + 1024;
};

template <int WARPS_M, int WARPS_N, int WM, int WN, int STAGES, bool TA, bool TB>
__global__ void __launch_bounds__(WARPS_M * WARPS_N * 32, 1)
dgemm_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                 TmaGemmArgs p) {
  using Cfg = TmaCfg<WARPS_M, WARPS_N, WM, WN, STAGES, TA, TB>;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte aligned stage buffers
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  double* As = reinterpret_cast<double*>(base);
  double* Bs = reinterpret_cast<double*>(base + STAGES * Cfg::A_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * (Cfg::A_BYTES + Cfg::B_BYTES));
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t n0 = (int64_t)blockIdx.x * BN;
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int split = blockIdx.z;
  const int64_t ktiles_total = ceil_div(p.K, BK);
  const int64_t kt_begin = (int64_t)split * p.ktiles_per_split;
  const int64_t kt_end = min(ktiles_total, kt_begin + p.ktiles_per_split);
  const int nkt = (int)(kt_end > kt_begin ? kt_end - kt_begin : 0);

  if (tid == 0) {
    for (int s = 0; s < STAGES; s++) {
      mbar_init_cta(&full[s], 1);
      mbar_init_cta(&empty[s], Cfg::CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // Producer: thread 0 (warp 0 also computes).  It fills the first STAGES slots,
  // then, after finishing k-tile it, refills the slot of k-tile it-1 (all warps
  // have usually released it by then) with k-tile it-1+STAGES.
  auto issue = [&](int it) {
    const int s = it % STAGES;
    mbar_expect_tx(&full[s], Cfg::A_BYTES + Cfg::B_BYTES);
    const int kg = (int)((kt_begin + it) * (BK / 4));  // k group index (units of 4)
    if (TA) tma_load_3d(As + s * Cfg::A_STAGE, &mapA, &full[s], 0, (int)m0, kg);
    else tma_load_3d(As + s * Cfg::A_STAGE, &mapA, &full[s], 0, kg * 4, (int)(m0 / 4));
    if (TB) tma_load_3d(Bs + s * Cfg::B_STAGE, &mapB, &full[s], 0, kg * 4, (int)(n0 / 4));
    else tma_load_3d(Bs + s * Cfg::B_STAGE, &mapB, &full[s], 0, (int)n0, kg);
  };
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
    for (int it = 0; it < STAGES && it < nkt; it++) issue(it);
  }

  // ---------------- consumer warps
  const int g = lane >> 2, t = lane & 3;
  const int warp_m = warp % WARPS_M, warp_n = warp / WARPS_M;
  const int wm0 = warp_m * WM * 8, wn0 = warp_n * WN * 8;
  double acc[WM][WN][2];
#pragma unroll
  for (int i = 0; i < WM; i++)
#pragma unroll
    for (int j = 0; j < WN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int it = 0; it < nkt; it++) {
    const int s = it % STAGES;
    mbar_wait(&full[s], (it / STAGES) & 1);
    const double* as = As + s * Cfg::A_STAGE;
    const double* bs = Bs + s * Cfg::B_STAGE;
#pragma unroll
    for (int kb = 0; kb < BK / 4; kb++) {
      double af[WM], bf[WN];
#pragma unroll
      for (int i = 0; i < WM; i++) {
        const int m = wm0 + i * 8 + g;
        af[i] = TA ? as[(kb * BM + m) * 4 + t] : as[((m >> 2) * BK + kb * 4 + t) * 4 + (m & 3)];
      }
#pragma unroll
      for (int j = 0; j < WN; j++) {
        const int n = wn0 + j * 8 + g;
        bf[j] = TB ? bs[((n >> 2) * BK + kb * 4 + t) * 4 + (n & 3)] : bs[(kb * BN + n) * 4 + t];
      }
#pragma unroll
      for (int i = 0; i < WM; i++)
#pragma unroll
        for (int j = 0; j < WN; j++) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_cta(&empty[s]);
    if (tid == 0 && it >= 1 && it - 1 + STAGES < nkt) {
      const int prev = it - 1;
      mbar_wait(&empty[prev % STAGES], (prev / STAGES) & 1);
      issue(prev + STAGES);
    }
  }

  // ---------------- epilogue
#pragma unroll
  for (int i = 0; i < WM; i++) {
    const int64_t gm = m0 + wm0 + i * 8 + g;
    if (gm >= p.M) continue;
#pragma unroll
    for (int j = 0; j < WN; j++) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int64_t gn = n0 + wn0 + j * 8 + 2 * t + h;
        if (gn >= p.N) continue;
        const double v = acc[i][j][h];
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

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

static bool encode3d(CUtensorMap* map, const double* ptr, uint64_t d0, uint64_t d1, uint64_t d2,
                     uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1,
                     uint32_t b2) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ptr), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

struct TmaTile {
  int bn, which;
};
static TmaTile tma_choose_tile(int64_t N) {
  const int bns[4] = {128, 112, 96, 80};
  TmaTile best{128, 0};
  int64_t best_pad = -1;
  for (int w = 0; w < 4; w++) {
    int64_t padded = ceil_div(N, bns[w]) * bns[w];
    if (best_pad < 0 || padded < best_pad) {
      best_pad = padded;
      best = TmaTile{bns[w], w};
    }
  }
  return best;
}

template <int WN, bool TA, bool TB>
static int tma_launch(const CUtensorMap& ma, const CUtensorMap& mb, TmaGemmArgs& a, cudaStream_t st) {
  constexpr int STAGES = 6;
  using Cfg = TmaCfg<4, 2, 4, WN, STAGES, TA, TB>;
  auto kern = dgemm_tma_kernel<4, 2, 4, WN, STAGES, TA, TB>;
  static unsigned mask = 0;
  int dev = 0;
  RLRA_CHECK_CUDA(cudaGetDevice(&dev));
  if (!(mask & (1u << (dev & 31)))) {
    RLRA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
    mask |= 1u << (dev & 31);
  }
  dim3 grid((unsigned)ceil_div(a.N, Cfg::BN), (unsigned)ceil_div(a.M, Cfg::BM), (unsigned)a.splits);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(ma, mb, a);
  RLRA_LAUNCHED();
  return 0;
}

struct SplitPlanT {
  int splits;
  int64_t kps;
};
// same time model as gemm.cu's planner
static SplitPlanT tma_plan(int64_t M, int64_t N, int bm, int bn, int64_t tiles, int64_t ktiles, int slots) {
  const double t_ktile = (double)bm * bn * 16 / (64.0 * 1.9e3);
  SplitPlanT best{1, ktiles};
  double best_t = 1e300;
  for (int s = 1; s <= 32; s++) {
    int64_t kps = ceil_div(ktiles, s);
    if (s > 1 && kps < 4) break;
    int64_t real_s = ceil_div(ktiles, kps);
    if (real_s != s) continue;
    double waves = (double)ceil_div(tiles * real_s, slots);
    double t = waves * kps * t_ktile;
    if (real_s > 1) t += 4.0 + (double)(real_s + 1) * M * N * 8 / 4e6;
    if (t < best_t * 0.98) {
      best_t = t;
      best = SplitPlanT{(int)real_s, kps};
    }
  }
  return best;
}

bool tma_gemm_eligible(bool ta, bool tb, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                       const double* B, int64_t ldb) {
  if (K <= 0 || M <= 0 || N <= 0) return false;
  if (tb && (N & 3)) return false;
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15)) return false;
  if ((lda & 1) || (ldb & 1) || (K & 3)) return false;
  if (!ta && (M & 3)) return false;
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return false;
  if (!get_encode()) return false;
  return true;
}

size_t tma_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  TmaTile tt = tma_choose_tile(N);
  int64_t tiles = ceil_div(M, 128) * ceil_div(N, tt.bn);
  SplitPlanT sp = tma_plan(M, N, 128, tt.bn, tiles, ceil_div(K, 16), device_info().sm_count);
  return sp.splits > 1 ? (size_t)sp.splits * M * N * sizeof(double) : 0;
}

int splitk_reduce(const double* partial, int splits, int64_t M, int64_t N, double alpha, double beta,
                  double* C, int64_t ldc, cudaStream_t st);

int tma_gemm(bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
             const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* ws, size_t ws_bytes,
             cudaStream_t st) {
  TmaTile tt = tma_choose_tile(N);
  const int BM = 128;
  CUtensorMap ma, mb;
  bool ok;
  if (ta)  // A^T: dims {4 k, M', K/4}, strides {lda*8, 32}
    ok = encode3d(&ma, A, 4, (uint64_t)M, (uint64_t)(K / 4), (uint64_t)lda * 8, 32, 4, BM, 4);
  else  // A: dims {4 m, K, M/4}, strides {lda*8, 32}
    ok = encode3d(&ma, A, 4, (uint64_t)K, (uint64_t)(M / 4), (uint64_t)lda * 8, 32, 4, 16, BM / 4);
  if (tb)  // B^T with B N x K (n contiguous): dims {4 n, K, N/4}
    ok = ok && encode3d(&mb, B, 4, (uint64_t)K, (uint64_t)(N / 4), (uint64_t)ldb * 8, 32, 4, 16, tt.bn / 4);
  else  // B (K x N, k contiguous): dims {4 k, N, K/4}
    ok = ok && encode3d(&mb, B, 4, (uint64_t)N, (uint64_t)(K / 4), (uint64_t)ldb * 8, 32, 4, tt.bn, 4);
  RLRA_REQUIRE(ok, "tma_gemm: cuTensorMapEncodeTiled failed");
  int64_t tiles = ceil_div(M, BM) * ceil_div(N, tt.bn);
  int64_t ktiles = ceil_div(K, 16);
  SplitPlanT sp = tma_plan(M, N, BM, tt.bn, tiles, ktiles, device_info().sm_count);
  TmaGemmArgs a{M, N, K, C, ldc, alpha, beta, sp.kps, sp.splits, nullptr};
  if (sp.splits > 1) {
    size_t need = (size_t)sp.splits * M * N * sizeof(double);
    RLRA_REQUIRE(ws != nullptr && ws_bytes >= need, "tma_gemm: workspace too small (%zu < %zu)", ws_bytes, need);
    a.partial = static_cast<double*>(ws);
  }
  int rc;
#define RLRA_TMA_CASE(WN)                                                             \
  rc = ta ? (tb ? tma_launch<WN, true, true>(ma, mb, a, st) : tma_launch<WN, true, false>(ma, mb, a, st)) \
          : (tb ? tma_launch<WN, false, true>(ma, mb, a, st) : tma_launch<WN, false, false>(ma, mb, a, st))
  switch (tt.which) {
    case 0: RLRA_TMA_CASE(8); break;
    case 1: RLRA_TMA_CASE(7); break;
    case 2: RLRA_TMA_CASE(6); break;
    default: RLRA_TMA_CASE(5); break;
  }
#undef RLRA_TMA_CASE
  if (rc) return rc;
  if (sp.splits > 1) return splitk_reduce(a.partial, sp.splits, M, N, alpha, beta, C, ldc, st);
  return 0;
}

}  // namespace rlra
