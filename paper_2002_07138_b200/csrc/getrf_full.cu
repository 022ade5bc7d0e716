// K3, one-launch variant: the whole GEPP of a tall sketch (m x n, n <= 256,
// m <= 16 * 256 * 6) by ONE 16-CTA thread-block cluster, bit-exact with the
// reference kernel rlra/_lu_cython.pyx:14-55 like the blocked path in getrf.cu.
//
// Why: the blocked path spends ~3 us per column step (two block barriers, a
// warp-0 decision broadcast, and a bulk update whose shared-memory traffic is
// ~1 byte per flop) and ~30 us per 16-column panel boundary in small
// swap / TRSM / update kernels.  Here
//   * the CTA's rows of the current 16-column panel live in REGISTERS
//     (thread t owns local rows t, t + 256, t + 512, ...), so the per-step updates
//     are pure FP64 ALU work with no shared-memory round trips;
//   * every warp takes the pivot decision redundantly from the multicast
//     records (no broadcast barrier); one block barrier per step (the argmax);
//   * the winning row's owner thread finishes its look-ahead and publishes the
//     record itself (global staging + one TMA multicast into every peer, which
//     completes on the peer's mbarrier, as in getrf.cu);
//   * between panels the cluster applies the row interchanges to the other
//     columns, forms U12 = L11^-1 A12 redundantly in every CTA (2 KB of L11,
//     no broadcast) and updates its own rows of the trailing columns with the
//     panel's multipliers straight from registers -- no kernel boundary at all.
// Operation order per element is the reference's: rank-1 terms in ascending
// step order, each DMUL then DSUB; multipliers by IEEE division; first-max
// pivot; zero-pivot rule against the whole-column max; zero-pivot steps
// skipped everywhere.
#include <cooperative_groups.h>

#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "common.cuh"

namespace rlra {
namespace lufull {

constexpr int W = 16;         // widest panel (8 when a thread holds 3 rows)
constexpr int T = 256;        // threads per CTA (8 warps: the per-step decision is replicated per warp)
constexpr int NW = T / 32;    // warps per CTA
constexpr int CS = 16;        // cluster size
constexpr int RECD = 2 + W;   // record: {|v|, row bits, row[W]} (<= 144 B)
constexpr int MAXRPT = 6;     // rows per thread
constexpr int MAXN = 256;     // widest sketch handled (trailing work runs on 16 SMs)
constexpr double ZTOL = 1e-14;  // rlra/_lu_cython.pyx:11
constexpr unsigned NONE = 0xffffffffu;

struct Args {
  double* a;
  int64_t lda, m, n;   // m >= n: factor all n columns
  int64_t* piv;        // int64[m], permuted like the reference's piv
  int64_t* ipiv;       // [n] pivot row of each step (== step when none / zero)
  int* zflag;          // [n] 1 for zero-pivot steps
  double* recg;        // [2][CS][RECD] records + [2][W] diagonal rows (multicast staging)
  int64_t R;           // rows per CTA
  unsigned long long* trace;  // RLRA_LU_TRACE builds: [CTA][128] globaltimer stamps
};

#ifdef RLRA_LU_TRACE
#define STEP_TRACE(jj, i)                                                                          \
  do {                                                                                              \
    if (threadIdx.x == 0 && x.p->trace && j0 == 0 && (jj) < 12) {                                   \
      unsigned long long t_;                                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                        \
      x.p->trace[(int64_t)x.b * 128 + 64 + 5 * (jj) + (i)] = t_;                                    \
    }                                                                                               \
  } while (0)
#define FULL_TRACE(slot)                                                                            \
  do {                                                                                              \
    if (threadIdx.x == 0 && p.trace && (slot) < 128) {                                              \
      unsigned long long t_;                                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                        \
      p.trace[(int64_t)x.b * 128 + (slot)] = t_;                                                    \
    }                                                                                               \
  } while (0)
#else
#define FULL_TRACE(slot) \
  do {                   \
  } while (0)
#define STEP_TRACE(jj, i) \
  do {                    \
  } while (0)
#endif

__device__ __forceinline__ double ieee_div(double x, double d, double rcp) {
  const double ax = fabs(x), ad = fabs(d);
  if (ax > 0x1p-960 && ax < 0x1p+960 && ad > 0x1p-960 && ad < 0x1p+960) {
    const double q0 = __dmul_rn(x, rcp);
    const double rem = fma(-d, q0, x);
    return fma(rem, rcp, q0);  // == RN(x / d) (Markstein)
  }
  return x / d;
}

// argmax key of |value|: non-negative doubles order like their bit patterns;
// NaN and "no row" map to 0 (they never beat a real row, and a maximum key of 0
// always ends in the zero-pivot branch, where the row index is irrelevant)
__device__ __forceinline__ unsigned long long vkey(double v) {
  return v >= 0.0 ? (unsigned long long)__double_as_longlong(v) : 0ull;
}

// warp-wide max of `key`, then the smallest `irel` holding it (first max)
__device__ __forceinline__ void warp_keymax(unsigned long long& key, unsigned& irel) {
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  const unsigned long long mk = ((unsigned long long)mh << 32) | ml;
  irel = __reduce_min_sync(0xffffffffu, key == mk ? irel : NONE);
  key = mk;
}

__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, unsigned parity) {
  const unsigned addr = smem_u32(bar);
  unsigned ok = 0;
  for (long long spin = 0;; ++spin) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) return;
    if (spin > (1ll << 28)) __trap();  // a lost record: fail loudly instead of hanging the GPU
  }
}

// 16 bytes from registers into a peer CTA's shared memory, completing on the
// peer's mbarrier (DSMEM store; no global staging, no proxy fence)
__device__ __forceinline__ void st_async2(unsigned raddr, double x0, double x1, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
               "d"(x0), "d"(x1), "r"(rbar)
               : "memory");
}

__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// compile-time loop: f(std::integral_constant<int, I>{}) for I in [B, E)
template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

struct Shared {
  __align__(16) double recv[2 * CS * RECD];  // every CTA's record, multicast in (by step parity)
  __align__(16) double recv_diag[2 * W];     // current diagonal row (pre-swap), multicast in
  double s_u[2 * W];                         // local copy of the step's pivot row (post-barrier readers)
  double l11[W][W + 1];
  unsigned long long wkey[NW];
  unsigned widx[NW];
  int64_t s_ipiv[W];
  int s_zf[W];
  int64_t prow_rows[2 * W], prow_src[2 * W];
  int pcnt;
  __align__(8) uint64_t mbar[2];
};

// Net row permutation of one panel's interchanges (j <-> ipiv[j], ascending),
// as (touched row, source row) pairs; one warp (every CTA computes its own copy).
__device__ int panel_perm(int64_t j0, int nb, const int64_t* ipiv, int64_t* rows, int64_t* src) {
  const int lane = threadIdx.x & 31;
  int cnt = 0;
  auto find = [&](int64_t r) -> int {
    const bool hit = lane < cnt && rows[lane] == r;
    const unsigned b = __ballot_sync(0xffffffffu, hit);
    if (b) return __ffs(b) - 1;
    if (lane == 0) {
      rows[cnt] = r;
      src[cnt] = r;
    }
    __syncwarp();
    return cnt++;
  };
  for (int q = 0; q < nb; q++) {
    const int64_t jq = j0 + q, pr = ipiv[q];
    if (pr == jq) continue;
    const int ka = find(jq), kb = find(pr);
    if (lane == 0) {
      const int64_t t = src[ka];
      src[ka] = src[kb];
      src[kb] = t;
    }
    __syncwarp();
  }
  return cnt;
}

// Shared-memory plan of one configuration (dynamic part).
template <int RPT, int W>
struct Plan {
  static constexpr int RS = T * RPT;                       // row slots per CTA (slot = k * T + tid)
  static constexpr int CB = RPT == 1 ? 8 : (RPT == 2 ? 4 : (RPT == 3 ? 3 : 2));  // trailing columns per chunk
  static constexpr int NCH = (RPT <= 2 || RPT >= 5) ? 3 : 2;                    // chunks in flight
  static size_t bytes(int64_t n) {
    return ((size_t)W * RS + (size_t)n * (1 + W) + (size_t)NCH * CB * RS) * sizeof(double);
  }
  static size_t max_bytes() { return bytes(MAXN); }
};

// Per-thread context of the cluster kernel.
struct Ctx {
  const Args* p;
  Shared* S;
  double* sL;      // [W][RS] retired panel columns of my row slots (L below, U on pivot rows)
  double* s_cmab;  // [n] max |a| over the rows above the current panel, per column
  double* s_u12;   // [W][n] U12 of the finished panel (column index relative)
  double* ring;    // [NCH][CB][RS] trailing-column staging
  int b, tid, lane, warp, nk;
  int64_t rb, re, g0;
};

template <int RPT, int W>
struct Panel {
  double a[RPT][W];  // register i = panel column jj + i at step jj (rotated each step)
  int lr[RPT];       // logical row held by my slot k (row interchanges only relabel)
};

// Record publication for the search column in register SC (logical row jn):
// local first max over my rows >= jn, warp max, the warp winner's owner (and
// row jn's holder) finish their look-ahead with step jj's terms when `fin`,
// one block barrier, CTA max (every warp); the warp holding the CTA winner
// stages the full panel row in shared memory and its lanes q < CS push it
// into peer q with DSMEM stores completing on the peer's mbarrier; the warp
// holding row jn pushes the diagonal row the same way.  Returns a bitmask of
// my slots already finished.
template <int RPT, int W, int SC>
__device__ __forceinline__ unsigned publish(const Ctx& x, Panel<RPT, W>& P, int jj, int nb, int jn, bool fin,
                                            const double* urow, unsigned par) {
  constexpr int RECD = 2 + W;
  constexpr int RS = Plan<RPT, W>::RS;
  Shared& S = *x.S;
  unsigned long long bk = 0ull;
  unsigned bi = NONE;
  int kb = -1;
#pragma unroll
  for (int k = 0; k < RPT; k++) {
    if (P.lr[k] >= jn) {
      const unsigned long long key = vkey(fabs(P.a[k][SC]));
      if (kb < 0 || key > bk || (key == bk && (unsigned)P.lr[k] < bi)) {
        bk = key;
        bi = (unsigned)P.lr[k];
        kb = k;
      }
    }
  }
  unsigned long long wk = bk;
  unsigned wi = bi;
  warp_keymax(wk, wi);
  if (x.lane == 0) {
    S.wkey[x.warp] = wk;
    S.widx[x.warp] = wi;
  }
  unsigned done = 0u;
  if (fin) {
#pragma unroll
    for (int k = 0; k < RPT; k++) {
      if ((k == kb && wi != NONE && bi == wi) || P.lr[k] == jn) {
        done |= 1u << k;
        const double l = P.a[k][0];
#pragma unroll
        for (int i = 2; i < W; i++)
          if (jj + i < nb) P.a[k][i] = sub_mul_nofma(P.a[k][i], l, urow[jj + i]);
      }
    }
  }
  __syncthreads();
  unsigned long long ck = x.lane < NW ? S.wkey[x.lane] : 0ull;
  unsigned ci = x.lane < NW ? S.widx[x.lane] : NONE;
  warp_keymax(ck, ci);
  const bool has = (ci != NONE);
  int kw = -1, kd = -1;  // my slot holding the CTA winner / row jn
#pragma unroll
  for (int k = 0; k < RPT; k++) {
    if (has && P.lr[k] == (int)ci) kw = k;
    if (P.lr[k] == jn) kd = k;
  }
  const unsigned bw = __ballot_sync(0xffffffffu, kw >= 0), bd = __ballot_sync(0xffffffffu, kd >= 0);
  const unsigned bar_l = smem_u32(&S.mbar[par]);
  // stage a row (registers -> its sL slot, columns >= jj) for the pushing lanes
  auto stage = [&](int kk) {
#pragma unroll
    for (int k = 0; k < RPT; k++)
      if (k == kk)
#pragma unroll
        for (int i = 0; i < W; i++)
          if (jj + i < W) x.sL[(size_t)(jj + i) * RS + k * T + x.tid] = P.a[k][i];
  };
  if (bw != 0u || (!has && x.warp == 0)) {  // this warp publishes the CTA record
    if (kw >= 0) stage(kw);
    __syncwarp();
    const int ol = bw ? __ffs(bw) - 1 : 0;
    const int ko = __shfl_sync(0xffffffffu, kw, ol);
    if (x.lane < CS) {
      const unsigned rdst = mapa_u32(smem_u32(S.recv + ((size_t)par * CS + x.b) * RECD), x.lane);
      const unsigned rbar = mapa_u32(bar_l, x.lane);
      const double v = has ? __longlong_as_double((long long)ck) : -1.0;
      const long long gi = has ? (long long)ci : (long long)INT64_MAX;
      st_async2(rdst, v, __longlong_as_double(gi), rbar);
      const int sl = ko * T + x.warp * 32 + ol;
#pragma unroll
      for (int c = 0; c < W; c += 2) {
        const double x0 = has ? x.sL[(size_t)c * RS + sl] : 0.0;
        const double x1 = has ? x.sL[(size_t)(c + 1) * RS + sl] : 0.0;
        st_async2(rdst + 8u * (2 + c), x0, x1, rbar);
      }
    }
  }
  if (bd != 0u) {  // this warp holds row jn: push the diagonal row
    if (kd >= 0 && kd != kw) stage(kd);
    __syncwarp();
    const int dl = __ffs(bd) - 1;
    const int kdd = __shfl_sync(0xffffffffu, kd, dl);
    if (x.lane < CS) {
      const unsigned rdst = mapa_u32(smem_u32(S.recv_diag + (size_t)par * W), x.lane);
      const unsigned rbar = mapa_u32(bar_l, x.lane);
      const int sl = kdd * T + x.warp * 32 + dl;
#pragma unroll
      for (int c = 0; c < W; c += 2)
        st_async2(rdst + 8u * c, x.sL[(size_t)c * RS + sl], x.sL[(size_t)(c + 1) * RS + sl], rbar);
    }
  }
  return done;
}

// Column step jj of the panel starting at j0 (pivot of logical row j = j0 + jj);
// on entry register 0 holds column jj of my rows, on exit the registers are
// rotated by one and column jj is retired to sL.
template <int RPT, int W>
__device__ __forceinline__ void step(const Ctx& x, Panel<RPT, W>& P, double& cm, unsigned& phase, int j0, int jj,
                                     int nb) {
  constexpr int RECD = 2 + W;
  constexpr int RS = Plan<RPT, W>::RS;
  Shared& S = *x.S;
  const int j = j0 + jj;
  const unsigned par = (unsigned)(j & 1);
  const unsigned tx_bytes = CS * RECD * 8u + W * 8u;
  STEP_TRACE(jj, 0);
  mbar_wait_bounded(&S.mbar[par], (phase >> par) & 1u);
  phase ^= 1u << par;
  STEP_TRACE(jj, 1);
  if (x.tid == 0) mbar_arrive_expect_tx(&S.mbar[par], tx_bytes);  // re-arm for step j + 2
  // decision, identical in every warp: first max over the CTA records (ties:
  // smallest logical row -- CTAs hold relabelled rows, so not the CTA rank)
  const double* rec = S.recv + (size_t)par * CS * RECD;
  unsigned long long rk = 0ull;
  unsigned ri = NONE;
  if (x.lane < CS) {
    rk = vkey(rec[x.lane * RECD]);
    const long long gi = __double_as_longlong(rec[x.lane * RECD + 1]);
    ri = (gi >= 0 && gi < (long long)NONE) ? (unsigned)gi : NONE;
  }
  const unsigned long long myk = rk;
  const unsigned myi = ri;
  warp_keymax(rk, ri);
  const unsigned wb = __ballot_sync(0xffffffffu, x.lane < CS && myk == rk && myi == ri);
  const unsigned rl = wb ? (unsigned)(__ffs(wb) - 1) : 0u;
  const double v = rk ? __longlong_as_double((long long)rk) : 0.0;
  const int idx = (int)ri;
  const double colmax = fmax(v, __shfl_sync(0xffffffffu, cm, jj));
  const bool zero = v <= ZTOL * colmax;  // rlra/_lu_cython.pyx:36-39
  const int prow = zero ? j : idx;
  const double* urow = zero ? S.recv_diag + (size_t)par * W : rec + (rl & 31u) * RECD + 2;
  if (x.lane > jj && x.lane < W) cm = fmax(cm, fabs(urow[x.lane]));  // row j joins the rows above
  if (x.tid < W) S.s_u[par * W + x.tid] = urow[x.tid];
  if (x.tid == 0) {
    S.s_ipiv[jj] = prow;
    S.s_zf[jj] = zero ? 1 : 0;
  }
  STEP_TRACE(jj, 2);
  // full-row interchange (:40-48): the rows' data stay where they are, their
  // logical labels swap (the write-back stores each slot at its logical row)
  unsigned below = 0u;
#pragma unroll
  for (int k = 0; k < RPT; k++) {
    if (!zero && prow != j) {
      if (P.lr[k] == prow) P.lr[k] = j;
      else if (P.lr[k] == j) P.lr[k] = prow;
    }
    if (P.lr[k] > j) below |= 1u << k;  // rows strictly below the diagonal
  }
  STEP_TRACE(jj, 3);
  // multipliers (IEEE division, :49-51) and the next column (:52-55)
  const double ujj = urow[jj];
  const double rcp = zero ? 0.0 : __drcp_rn(ujj);
  const double unx = urow[jj + 1 < W ? jj + 1 : jj];
#pragma unroll
  for (int k = 0; k < RPT; k++) {
    if ((below >> k) & 1u) {
      if (!zero) {
        const double l = ieee_div(P.a[k][0], ujj, rcp);
        P.a[k][0] = l;
        if (jj + 1 < W) P.a[k][1] = sub_mul_nofma(P.a[k][1], l, unx);
      } else {
        P.a[k][0] = 0.0;
      }
    }
  }
  STEP_TRACE(jj, 4);
  if (jj + 1 < nb) {
    const unsigned done = publish<RPT, W, 1>(x, P, jj, nb, j + 1, !zero, urow, par ^ 1u);
#ifndef LUF_EXP_NOBULK
    if (!zero) {  // bulk of step jj: columns jj+2.. of my other rows (overlaps the exchange)
#else
    if (false) {
#endif
      const double* su = S.s_u + par * W + jj;
      const unsigned bm = below & ~done;
#pragma unroll
      for (int i = 2; i < W; i++) {
        if (jj + i < nb) {
          const double uc = su[i];
#pragma unroll
          for (int k = 0; k < RPT; k++)
            if ((bm >> k) & 1u) P.a[k][i] = sub_mul_nofma(P.a[k][i], P.a[k][0], uc);
        }
      }
    }
  }
  // retire column jj, rotate
#pragma unroll
  for (int k = 0; k < RPT; k++) {
    x.sL[(size_t)jj * RS + k * T + x.tid] = P.a[k][0];
#pragma unroll
    for (int i = 0; i + 1 < W; i++) P.a[k][i] = P.a[k][i + 1];
    P.a[k][W - 1] = 0.0;
  }
}

template <int RPT, int W>
__global__ void __launch_bounds__(T, 1) lu_full_kernel(const Args p) {
  namespace cg = cooperative_groups;
  constexpr int RECD = 2 + W;
  using PL = Plan<RPT, W>;
  constexpr int RS = PL::RS, CB = PL::CB, NCH = PL::NCH;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ Shared S;
  extern __shared__ __align__(16) double dyn[];
  Ctx x;
  x.p = &p;
  x.S = &S;
  x.sL = dyn;
  x.s_cmab = x.sL + (size_t)W * RS;
  x.s_u12 = x.s_cmab + p.n;
  x.ring = x.s_u12 + (size_t)W * p.n;
  x.b = (int)cluster.block_rank();
  x.tid = threadIdx.x;
  x.lane = x.tid & 31;
  x.warp = x.tid >> 5;
  const int64_t m = p.m, n = p.n, lda = p.lda;
  x.rb = min(m, (int64_t)x.b * p.R);
  x.re = min(m, x.rb + p.R);
  x.g0 = x.rb + x.tid;
  const int nloc = (int)(x.re - x.rb);
  x.nk = 0;
#pragma unroll
  for (int k = 0; k < RPT; k++)
    if (x.tid + k * T < nloc) x.nk = k + 1;
  const int tid = x.tid, lane = x.lane, warp = x.warp, b = x.b;
  const unsigned tx_bytes = CS * RECD * 8u + W * 8u;

  if (tid == 0) {
    mbar_init(&S.mbar[0], 1);
    mbar_init(&S.mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    mbar_arrive_expect_tx(&S.mbar[0], tx_bytes);
    mbar_arrive_expect_tx(&S.mbar[1], tx_bytes);
  }
  for (int64_t c = tid; c < n; c += T) x.s_cmab[c] = -1.0;
  unsigned phase = 0u;  // bit q: parity of mbar[q]'s current phase
  Panel<RPT, W> P;
  cluster.sync();  // mbarriers initialised everywhere before the first DSMEM store

  for (int j0 = 0; j0 < (int)n; j0 += W) {
    const int nb = (int)min((int64_t)W, n - j0);
    // ---- panel prologue: my rows >= j0 of columns j0 .. j0+W-1 into registers
#pragma unroll
    for (int k = 0; k < RPT; k++) {
      const int64_t g = x.g0 + (int64_t)k * T;
      const bool act = k < x.nk && g >= j0;
      P.lr[k] = act ? (int)g : -1;
#pragma unroll
      for (int c = 0; c < W; c++) P.a[k][c] = (act && c < nb) ? p.a[g + (j0 + c) * lda] : 0.0;
    }
    double cm = (lane < nb) ? x.s_cmab[j0 + lane] : -1.0;  // lane c: colmax of panel column c so far
    const int pidx = j0 / W;
    FULL_TRACE(6 * pidx + 0);
    publish<RPT, W, 0>(x, P, 0, nb, j0, false, nullptr, (unsigned)(j0 & 1));
#pragma unroll 1
    for (int jj = 0; jj < nb; jj++) step<RPT, W>(x, P, cm, phase, j0, jj, nb);
    FULL_TRACE(6 * pidx + 1);

    // ---- panel epilogue: every slot's row to its LOGICAL row, interchanges elsewhere
#pragma unroll
    for (int k = 0; k < RPT; k++)
      if (P.lr[k] >= 0)
        for (int c = 0; c < nb; c++) p.a[P.lr[k] + (j0 + c) * lda] = x.sL[(size_t)c * RS + k * T + tid];
    __syncthreads();  // s_ipiv / s_zf complete
    if (warp == 0) {
      const int cnt = panel_perm(j0, nb, S.s_ipiv, S.prow_rows, S.prow_src);
      if (lane == 0) S.pcnt = cnt;
      if (b == 0) {
        if (lane < nb) {
          p.ipiv[j0 + lane] = S.s_ipiv[lane];
          p.zflag[j0 + lane] = S.s_zf[lane];
        }
        int64_t v0 = 0;  // the same net permutation on piv (:46-48)
        if (lane < cnt) v0 = p.piv[S.prow_src[lane]];
        __syncwarp();
        if (lane < cnt) p.piv[S.prow_rows[lane]] = v0;
      }
    }
    cluster.sync();  // (1) every panel row at its logical place; perm ready
    FULL_TRACE(6 * pidx + 2);
    const int cnt = S.pcnt;
    const int ce = j0 + nb;
    if (cnt > 0) {  // columns outside the panel: one warp per column, gather then scatter
      const int64_t nother = n - nb;
      for (int64_t q = b + (int64_t)CS * warp; q < nother; q += (int64_t)CS * NW) {
        const int64_t c = q < j0 ? q : q + nb;
        double* col = p.a + c * lda;
        const double v0 = lane < cnt ? col[S.prow_src[lane]] : 0.0;
        __syncwarp();
        if (lane < cnt) col[S.prow_rows[lane]] = v0;
      }
    }
    if (ce >= n) break;
    cluster.sync();  // (2) interchanges visible
    FULL_TRACE(6 * pidx + 3);
    // ---- U12 = L11^-1 A12 (every CTA, redundantly), forward substitution in
    // ascending step order, zero-pivot steps skipped; owners store their rows
    for (int e = tid; e < nb * nb; e += T) {
      const int r = e % nb, c = e / nb;
      S.l11[r][c] = p.a[(j0 + r) + (j0 + c) * lda];
    }
    unsigned zmask = 0u;
    for (int s2 = 0; s2 < nb; s2++)
      if (S.s_zf[s2]) zmask |= 1u << s2;
    __syncthreads();
    const int64_t ntr = n - ce;
    for (int64_t cr = tid; cr < ntr; cr += T) {  // one thread per column, U12 built in shared memory
      const double* col = p.a + (ce + cr) * lda + j0;
      double* uc = x.s_u12 + cr;
      double mx = x.s_cmab[ce + cr];
#pragma unroll 1
      for (int s2 = 0; s2 < nb; s2++) {
        double acc = col[s2];
#pragma unroll 4
        for (int t = 0; t < s2; t++)
          if (!((zmask >> t) & 1u)) acc = sub_mul_nofma(acc, S.l11[s2][t], uc[t * n]);
        uc[s2 * n] = acc;
        mx = fmax(mx, fabs(acc));
      }
      x.s_cmab[ce + cr] = mx;
    }
    __syncthreads();
    // CTAs owning rows j0 .. j0+nb-1 (all above the trailing rows) store U12
    for (int64_t e = tid; e < (int64_t)nb * ntr; e += T) {
      const int s2 = (int)(e % nb);
      const int64_t cr = e / nb, g = j0 + s2;
      if (g >= x.rb && g < x.re) p.a[g + (ce + cr) * lda] = x.s_u12[s2 * n + cr];
    }
    FULL_TRACE(6 * pidx + 4);
    // ---- trailing update of my logical rows >= ce: multipliers back into
    // registers, the rows of the trailing columns streamed through a private
    // cp.async ring (NCH chunks of CB columns), CB x RPT independent chains
    bool act[RPT];
#pragma unroll
    for (int k = 0; k < RPT; k++) {
      act[k] = P.lr[k] >= ce;
#pragma unroll
      for (int s2 = 0; s2 < W; s2++) P.a[k][s2] = (s2 < nb) ? x.sL[(size_t)s2 * RS + k * T + tid] : 0.0;
    }
    auto issue = [&](int64_t c0) {
      if (c0 < ntr) {
        double* slot = x.ring + (size_t)((c0 / CB) % NCH) * CB * RS + tid;
#pragma unroll
        for (int q = 0; q < CB; q++)
          if (c0 + q < ntr) {
            const double* src = p.a + (ce + c0 + q) * lda;
#pragma unroll
            for (int k = 0; k < RPT; k++)
              if (act[k]) cp_async8(slot + q * RS + k * T, src + P.lr[k]);
          }
      }
      cp_async_commit();
    };
#pragma unroll 1
    for (int q = 0; q < NCH - 1; q++) issue((int64_t)q * CB);
#pragma unroll 1
    for (int64_t c0 = 0; c0 < ntr; c0 += CB) {
      issue(c0 + (int64_t)(NCH - 1) * CB);
      cp_async_wait<NCH - 1>();
      const double* slot = x.ring + (size_t)((c0 / CB) % NCH) * CB * RS + tid;
      double y[CB][RPT];
#pragma unroll
      for (int q = 0; q < CB; q++)
#pragma unroll
        for (int k = 0; k < RPT; k++) y[q][k] = (act[k] && c0 + q < ntr) ? slot[q * RS + k * T] : 0.0;
#pragma unroll
      for (int s2 = 0; s2 < W; s2++) {
        if (s2 < nb && !((zmask >> s2) & 1u)) {
#pragma unroll
          for (int q = 0; q < CB; q++) {
            const double u = x.s_u12[s2 * n + min(c0 + q, ntr - 1)];
#pragma unroll
            for (int k = 0; k < RPT; k++) y[q][k] = sub_mul_nofma(y[q][k], P.a[k][s2], u);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < CB; q++)
        if (c0 + q < ntr) {
          double* dst = p.a + (ce + c0 + q) * lda;
#pragma unroll
          for (int k = 0; k < RPT; k++)
            if (act[k]) dst[P.lr[k]] = y[q][k];
        }
    }
    cp_async_wait<0>();
    // relabelled rows were updated by their holder CTA, not their owner: the
    // next panel's loads need every CTA's stores (also orders s_u12 reuse)
    cluster.sync();
    FULL_TRACE(6 * pidx + 5);
  }
  cluster.sync();  // nobody leaves while a peer may still address its shared memory
}

}  // namespace lufull

// Eligibility of the one-launch cluster GEPP (getrf.cu dispatches to it).
bool getrf_full_eligible(int64_t m, int64_t n, int cluster_max) {
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = getenv("RLRA_B200_LU_FULL");
    enabled = (e && e[0] == '1') ? 1 : 0;  // opt-in until it beats the blocked path
  }
  return enabled && cluster_max >= lufull::CS && n >= 1 && m >= n && n <= lufull::MAXN &&
         m >= (int64_t)lufull::CS * 32 && m <= (int64_t)lufull::CS * lufull::T * lufull::MAXRPT;
}

template <int RPT, int W>
static int launch_full(const lufull::Args& a, cudaStream_t st) {
  const void* kern = (const void*)lufull::lu_full_kernel<RPT, W>;
  using PL = lufull::Plan<RPT, W>;
  const size_t dyn = PL::bytes(a.n);
  static std::mutex mu;
  static bool done[64][lufull::MAXRPT + 1];
  int dev = 0;
  RLRA_CHECK_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!done[dev & 63][RPT]) {
      RLRA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      RLRA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PL::max_bytes()));
      done[dev & 63][RPT] = true;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(lufull::CS);
  cfg.blockDim = dim3(lufull::T);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = lufull::CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  lufull::Args args = a;
  void* kargs[] = {&args};
  RLRA_CHECK_CUDA(cudaLaunchKernelExC(&cfg, kern, kargs));
  note_launch();
  return 0;
}

extern unsigned long long* g_lu_trace;

int getrf_full(double* a, int64_t lda, int64_t m, int64_t n, int64_t* piv, int64_t* ipiv, int* zflag, double* recg,
               cudaStream_t st) {
  lufull::Args args;
  args.trace = g_lu_trace;
  args.a = a;
  args.lda = lda;
  args.m = m;
  args.n = n;
  args.piv = piv;
  args.ipiv = ipiv;
  args.zflag = zflag;
  args.recg = recg;
  args.R = ceil_div(m, lufull::CS);
  const int rpt = (int)ceil_div(args.R, lufull::T);
  RLRA_REQUIRE(rpt >= 1 && rpt <= lufull::MAXRPT, "getrf_full: m = %lld outside the register capacity",
               (long long)m);
  switch (rpt) {
    case 1: return launch_full<1, 16>(args, st);
    case 2: return launch_full<2, 16>(args, st);
    case 3: return launch_full<3, 16>(args, st);
    case 4: return launch_full<4, 16>(args, st);
    case 5: return launch_full<5, 8>(args, st);
    default: return launch_full<6, 8>(args, st);
  }
}

}  // namespace rlra
