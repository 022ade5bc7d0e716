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

// The file is compiled twice (csrc/Makefile): the primary build with 256
// threads per CTA (rows per thread up to 6: m <= 24576) and LUF_WIDE_CTA with
// 384 threads and at most 2 rows per thread (m <= 12288), measured 8 % faster
// there (fewer rows per thread on the column step's critical path); beyond 2
// rows per thread the 12 warps' instruction issue makes it slower than 256.
#ifdef LUF_WIDE_CTA
#define LUF_T 384
#define lufull lufull_wide
#define getrf_full getrf_full_wide
#endif

namespace rlra {
namespace lufull {

constexpr int W = 16;         // widest panel (8 when a thread holds 3 rows)
#ifndef LUF_T
#define LUF_T 256
#endif
constexpr int T = LUF_T;      // threads per CTA (8 warps: the per-step decision is replicated per warp)
constexpr int NW = T / 32;    // warps per CTA
constexpr int CS = 16;        // cluster size
constexpr int RECD = 2 + W;   // record: {|v|, row bits, row[W]} (<= 144 B)
constexpr int MAXRPT = 6;     // rows per thread
constexpr int MAXN = 1024;    // widest sketch handled (r02: 1024 -- C3 16384 x 1024 / 843; r01 capped it at 512)
constexpr double ZTOL = 1e-14;  // rlra/_lu_cython.pyx:11
constexpr unsigned NONE = 0xffffffffu;

struct Args {
  double* a;
  int64_t lda, m, n;   // m >= n: factor all n columns
  int64_t* piv;        // int64[m], permuted like the reference's piv
  int64_t* ipiv;       // [n] pivot row of each step (== step when none / zero)
  int* zflag;          // [n] 1 for zero-pivot steps
  double* recg;        // Handoff state (workspace, zeroed per launch)
  int64_t R;           // rows per CTA
  unsigned nhelpers;   // helper CTAs (grid = CS + nhelpers)
  unsigned long long* trace;  // RLRA_LU_TRACE builds: [CTA][128] globaltimer stamps
};

#ifdef RLRA_LU_TRACE
#define STEP_TRACE(jj, i)                                                                          \
  do {                                                                                              \
    if (threadIdx.x == 0 && x.p->trace && j0 == 0 && (jj) < 8) {                                    \
      unsigned long long t_;                                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                        \
      x.p->trace[(int64_t)x.b * 128 + 64 + 8 * (jj) + (i)] = t_;                                    \
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

// rare operands (zeros, values near the exponent range's ends): out of line, so
// that the column step's hot path stays short
__device__ __noinline__ double ieee_div_slow(double x, double d) { return x / d; }

__device__ __forceinline__ double ieee_div(double x, double d, double rcp) {
  const double ax = fabs(x), ad = fabs(d);
  if (ax > 0x1p-960 && ax < 0x1p+960 && ad > 0x1p-960 && ad < 0x1p+960) {
    const double q0 = __dmul_rn(x, rcp);
    const double rem = fma(-d, q0, x);
    return fma(rem, rcp, q0);  // == RN(x / d) (Markstein)
  }
  return ieee_div_slow(x, d);
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
  double s_u[2 * 2 * W];                     // local copy of the step's pivot row, zero beyond nb (post-barrier readers)
  __align__(16) double srow[2 * W], drow[2 * W];  // DSMEM push: staged record / diagonal rows (columns jj + i)
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

// Dynamic shared memory of the cooperative GEPP (same size for every CTA):
// panel CTAs: sL [W][T*RPT] + s_cmab [n] + s_u12 [W][W];
// helper CTAs: U12 of the far columns [W][n].
template <int RPT, int W>
struct Plan {
  static constexpr int RS = T * RPT;  // row slots per CTA (slot = k * T + tid)
  static size_t bytes(int64_t n) {
    const size_t panel = (size_t)W * RS + (size_t)n + (size_t)W * W;
    const size_t helper = (size_t)W * W + (size_t)W * n;
    return (panel > helper ? panel : helper) * sizeof(double);
  }
  static size_t max_bytes() { return bytes(MAXN); }
};

// Handoff state between the panel cluster and the helper clusters (global
// memory, zeroed per launch): counters, per-column max |U| over the rows
// above the current panel (as ordered bit patterns), each panel's net row
// permutation.
constexpr int MAXP = MAXN / 16;
struct Handoff {
  unsigned ready;            // panels whose L, U12 rows and permutation are published
  unsigned fardone[MAXP];    // helper CTAs done with panel b (interchanges + far update)
  unsigned u12done[MAXP];    // helper CTAs done with panel b's far U12 rows
  unsigned nextdone[MAXP];   // helper CTAs done with the next panel's columns (update by panel b)
  unsigned u12read[MAXP];    // helper CTAs (other than 0) done reading the next columns' rows j0..ce
  unsigned pad[(1 + 4 * MAXP + 127) / 128 * 128 - 1 - 4 * MAXP];  // counters on their own lines
  unsigned long long cmax[MAXN];
  int64_t prow[MAXP][2 * 16], psrc[MAXP][2 * 16];
  int pcnt[MAXP];
  // multicast staging: records in slots of 2 + 2 * 16 doubles, diagonal rows in slots of 2 * 16 -- the
  // holder stores its ROTATED registers at slot[jj + i] without a bound check (only 2 + 16 / 16 doubles are sent)
  __align__(16) double stage[2 * CS * (2 + 2 * 16) + 2 * 2 * 16];
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
#ifndef LUF_POLL_NS
#define LUF_POLL_NS 64
#endif
// one thread waits until *p >= target (acquire); bounded: a protocol error traps
__device__ __forceinline__ void wait_geq(const unsigned* p, unsigned target) {
  for (long long spin = 0; ld_acquire(p) < target; ++spin) {
    __nanosleep(LUF_POLL_NS);
    if (spin > (1ll << 26)) __trap();
  }
}

// Bytes every CTA receives for local step jr of a panel (its mbarrier's expected
// transaction count): CS records + one diagonal row.  The global-staging path
// always sends whole records; the DSMEM path only the columns >= (jr & ~1).
template <int W>
__device__ __forceinline__ unsigned step_tx_bytes(int jr) {
#ifdef LUF_PUSH_DSMEM
  const unsigned live = (unsigned)(W - (jr & ~1));
  return CS * (16u + 8u * live) + 8u * live;
#else
  (void)jr;
  return CS * (2u + W) * 8u + W * 8u;
#endif
}

// Per-thread context of the cluster kernel.
struct Ctx {
  const Args* p;
  Shared* S;
  double* sL;      // [W][RS] retired panel columns of my row slots (L below, U on pivot rows)
  double* s_cmab;  // [n] max |a| over the rows above the current panel, per column
  double* s_u12;   // [W][W] U12 of the next panel's columns
  double* gstage;  // global staging of this CTA's outgoing records (multicast source)
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
                                            const double* su, unsigned par) {
  [[maybe_unused]] const int j0 = SC == 0 ? 1 : jn - 1 - jj;  // for STEP_TRACE (panel 0 steps only)
  constexpr int RECD = 2 + W;
  [[maybe_unused]] constexpr int RS = Plan<RPT, W>::RS;
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
  if (SC) STEP_TRACE(jj, 3);
  __syncthreads();
  unsigned long long ck = x.lane < NW ? S.wkey[x.lane] : 0ull;
  unsigned ci = x.lane < NW ? S.widx[x.lane] : NONE;
  warp_keymax(ck, ci);
  if (SC) STEP_TRACE(jj, 4);
  const bool has = (ci != NONE);
  int kw = -1, kd = -1;  // my slot holding the CTA winner / row jn
#pragma unroll
  for (int k = 0; k < RPT; k++) {
    if (has && P.lr[k] == (int)ci) kw = k;
    if (P.lr[k] == jn) kd = k;
  }
  const unsigned bw = __ballot_sync(0xffffffffu, kw >= 0), bd = __ballot_sync(0xffffffffu, kd >= 0);
  const unsigned bar_l = smem_u32(&S.mbar[par]);
  // look-ahead of the two published rows only (CTA winner, row jn): step jj's
  // terms on their columns jj+2.. (warp-uniform branch: two warps at most).
  // The pivot row is read from this CTA's copy (su): after the barrier a peer
  // may already be multicasting step jj+2's records into recv[par].
  unsigned done = 0u;
  if (fin && (bw | bd) != 0u) {
#pragma unroll
    for (int k = 0; k < RPT; k++) {
      if (k == kw || k == kd) {
        done |= 1u << k;
        const double l = P.a[k][0];
#pragma unroll
        for (int i = 2; i < W; i++)
          P.a[k][i] = sub_mul_nofma(P.a[k][i], l, su[jj + i]);  // columns >= nb: padding, u = 0
      }
    }
  }
  // stage a row (registers -> its sL slot, columns >= jj) for the pushing lanes
#ifdef LUF_PUSH_DSMEM
  // The holder's warp stages the row's live columns (registers i <-> column jj + i) in a small
  // shared row buffer -- one unpredicated store per column after a warp-uniform slot switch --
  // and lanes q < CS push {|v|, row, columns >= c0} into peer q with DSMEM stores completing on
  // the peer's mbarrier; c0 = the first even column the receiving step reads (step_tx_bytes).
  const int c0 = (jj + SC) & ~1;
  auto stage = [&](unsigned bmask, int kk, double* row) {
    const int hl = __ffs(bmask) - 1;
    const int ko = __shfl_sync(0xffffffffu, kk, hl);
    static_for<0, RPT>([&](auto K) {
      if (ko == K.value && kk >= 0) {
#pragma unroll
        for (int i = 0; i < W; i++) row[jj + i] = P.a[K.value][i];
      }
    });
    __syncwarp();
  };
  if (bw != 0u || (!has && x.warp == 0)) {  // this warp publishes the CTA record
    if (bw != 0u) stage(bw, kw, S.srow);
    if (SC) STEP_TRACE(jj, 5);
    if (x.lane < CS) {
      const unsigned rdst = mapa_u32(smem_u32(S.recv + ((size_t)par * CS + x.b) * RECD), x.lane);
      const unsigned rbar = mapa_u32(bar_l, x.lane);
      const double v = has ? __longlong_as_double((long long)ck) : -1.0;
      const long long gi = has ? (long long)ci : (long long)INT64_MAX;
      st_async2(rdst, v, __longlong_as_double(gi), rbar);
      for (int c = c0; c < W; c += 2)
        st_async2(rdst + 8u * (2 + c), has ? S.srow[c] : 0.0, has ? S.srow[c + 1] : 0.0, rbar);
    }
  }
  if (bd != 0u) {  // this warp holds row jn: push the diagonal row
    stage(bd, kd, S.drow);
    if (x.lane < CS) {
      const unsigned rdst = mapa_u32(smem_u32(S.recv_diag + (size_t)par * W), x.lane);
      const unsigned rbar = mapa_u32(bar_l, x.lane);
      for (int c = c0; c < W; c += 2) st_async2(rdst + 8u * c, S.drow[c], S.drow[c + 1], rbar);
    }
  }
#else
  // the holder thread writes the row's live columns (>= jj: registers i <-> column jj + i) to a global
  // staging slot and multicasts it into every CTA with one bulk copy completing on each peer's
  // mbarrier.  Columns < jj of a record are never read (rows are relabelled, not moved: the L part
  // stays with its owner), so they are not staged.  The slot index of the holder's row is made
  // warp-uniform first: one unpredicated store per column instead of RPT predicated ones.
  constexpr int SLOT = 2 + 2 * W, DSLOT = 2 * W;
  auto emit = [&](unsigned bmask, int kk, double* slot) {
    const int hl = __ffs(bmask) - 1;
    const int ko = __shfl_sync(0xffffffffu, kk, hl);
    static_for<0, RPT>([&](auto K) {
      if (ko == K.value && kk >= 0) {
#pragma unroll
        for (int i = 0; i < W; i++) slot[jj + i] = P.a[K.value][i];
      }
    });
  };
  const unsigned short mask = (unsigned short)0xffffu;
  double* slot = x.gstage + ((size_t)par * CS + x.b) * SLOT;
  if (bw != 0u) emit(bw, kw, slot + 2);  // warp-uniform: the warp holding the CTA winner
  if (kw >= 0 || (!has && x.tid == 0)) {
    const double v = has ? __longlong_as_double((long long)ck) : -1.0;
    const long long gi = has ? (long long)ci : (long long)INT64_MAX;
    slot[0] = v;
    slot[1] = __longlong_as_double(gi);
    if (!has)
      for (int c = 0; c < W; c++) slot[2 + c] = 0.0;
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
        "%4;\n" ::"r"(smem_u32(S.recv + ((size_t)par * CS + x.b) * RECD)),
        "l"(slot), "r"((unsigned)(RECD * 8)), "r"(bar_l), "h"(mask)
        : "memory");
  }
  double* dslot = x.gstage + (size_t)2 * CS * SLOT + (size_t)par * DSLOT;
  if (bd != 0u) emit(bd, kd, dslot);  // warp-uniform: the warp holding row jn
  if (kd >= 0) {
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
        "%4;\n" ::"r"(smem_u32(S.recv_diag + (size_t)par * W)),
        "l"(dslot), "r"((unsigned)(W * 8)), "r"(bar_l), "h"(mask)
        : "memory");
  }
#endif
  if (SC) STEP_TRACE(jj, 6);
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
  // this barrier's next user is local step jj + 2, or step jj + 2 - nb (0 or 1) of the next panel
  const unsigned tx_bytes = step_tx_bytes<W>(jj + 2 < nb ? jj + 2 : 0);
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
  if (x.tid < 2 * W) S.s_u[par * 2 * W + x.tid] = x.tid < nb ? urow[x.tid] : 0.0;
  if (x.tid == 0) {
    S.s_ipiv[jj] = prow;
    S.s_zf[jj] = zero ? 1 : 0;
  }
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
#ifdef LUF_EXP_NULL
  if (jj < 0) {
#else
  {
#endif
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
  }
  STEP_TRACE(jj, 2);
  if (jj + 1 < nb) {
    const unsigned done = publish<RPT, W, 1>(x, P, jj, nb, j + 1, !zero, S.s_u + par * 2 * W, par ^ 1u);
#ifndef LUF_EXP_NOBULK
    if (!zero) {  // bulk of step jj: columns jj+2.. of my other rows (overlaps the exchange)
#else
    if (false) {
#endif
      const double* su = S.s_u + par * 2 * W + jj;  // zero beyond nb: padding columns stay inert
      const unsigned bm = below & ~done;
      double u[W];  // the pivot row once per thread, not once per row slot
#pragma unroll
      for (int i = 2; i < W; i++) u[i] = su[i];
#pragma unroll
      for (int k = 0; k < RPT; k++) {
        if ((bm >> k) & 1u) {
          const double l = P.a[k][0];
#pragma unroll
          for (int i = 2; i < W; i++) P.a[k][i] = sub_mul_nofma(P.a[k][i], l, u[i]);
        }
      }
    }
  }
  STEP_TRACE(jj, 7);
  // retire column jj, rotate
#pragma unroll
  for (int k = 0; k < RPT; k++) {
    x.sL[(size_t)jj * RS + k * T + x.tid] = P.a[k][0];
#pragma unroll
    for (int i = 0; i + 1 < W; i++) P.a[k][i] = P.a[k][i + 1];
    P.a[k][W - 1] = 0.0;
  }
}

// Cooperative launch: cluster 0 factors the panels (register-resident rows,
// see step / publish) and updates the NEXT panel's columns itself; clusters
// 1..NH (the helpers) apply each panel's interchanges to the other columns,
// form the far columns' U12 rows and update the far columns' rows below --
// in parallel with the panel cluster's next panel.  Ordering is by release /
// acquire counters in global memory; co-residency is guaranteed by the
// cooperative launch (a grid that does not fit fails to launch).
template <int RPT, int W>
__device__ void panel_role(const Args& p, Handoff* hs, double* dyn) {
  namespace cg = cooperative_groups;
  [[maybe_unused]] constexpr int RECD = 2 + W;
  constexpr int RS = Plan<RPT, W>::RS;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ Shared S;
  Ctx x;
  x.p = &p;
  x.S = &S;
  x.sL = dyn;
  x.s_cmab = x.sL + (size_t)W * RS;
  x.s_u12 = x.s_cmab + p.n;
  x.gstage = hs->stage;
  x.b = (int)cluster.block_rank();
  x.tid = threadIdx.x;
  x.lane = x.tid & 31;
  x.warp = x.tid >> 5;
  const int64_t m = p.m, n = p.n, lda = p.lda;
  const unsigned nhc = p.nhelpers;
  x.rb = min(m, (int64_t)x.b * p.R);
  x.re = min(m, x.rb + p.R);
  x.g0 = x.rb + x.tid;
  const int nloc = (int)(x.re - x.rb);
  x.nk = 0;
#pragma unroll
  for (int k = 0; k < RPT; k++)
    if (x.tid + k * T < nloc) x.nk = k + 1;
  const int tid = x.tid, lane = x.lane, warp = x.warp, b = x.b;
  const unsigned tx_bytes = step_tx_bytes<W>(0);  // steps 0 and 1 of panel 0 receive whole records

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
  // panel 0: plain loads
  {
    const int nb0 = (int)min((int64_t)W, n);
#pragma unroll
    for (int k = 0; k < RPT; k++) {
      const int64_t g = x.g0 + (int64_t)k * T;
      const bool act = k < x.nk;
      P.lr[k] = act ? (int)g : -1;
#pragma unroll
      for (int c = 0; c < W; c++) P.a[k][c] = (act && c < nb0) ? p.a[g + c * lda] : 0.0;
    }
  }
  cluster.sync();  // mbarriers initialised everywhere before the first DSMEM store

  for (int j0 = 0; j0 < (int)n; j0 += W) {
    const int nb = (int)min((int64_t)W, n - j0);
    const int pidx = j0 / W;
    double cm = (lane < nb) ? x.s_cmab[j0 + lane] : -1.0;  // lane c: colmax of panel column c so far
    FULL_TRACE(6 * pidx + 0);
    publish<RPT, W, 0>(x, P, 0, nb, j0, false, nullptr, (unsigned)(j0 & 1));
#pragma unroll 1
    for (int jj = 0; jj < nb; jj++) step<RPT, W>(x, P, cm, phase, j0, jj, nb);
    FULL_TRACE(6 * pidx + 1);

    // ---- epilogue: every slot's row to its LOGICAL row; pivots; permutation
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
        if (lane < cnt) {
          hs->prow[pidx][lane] = S.prow_rows[lane];
          hs->psrc[pidx][lane] = S.prow_src[lane];
        }
        if (lane == 0) hs->pcnt[pidx] = cnt;
        int64_t v0 = 0;  // the same net permutation on piv (:46-48)
        if (lane < cnt) v0 = p.piv[S.prow_src[lane]];
        __syncwarp();
        if (lane < cnt) p.piv[S.prow_rows[lane]] = v0;
      }
    }
    cluster.sync();  // (1) the whole panel at its logical rows, in global memory
    FULL_TRACE(6 * pidx + 2);
    const int ce = j0 + nb;
    const int nbn = ce < n ? (int)min((int64_t)W, n - ce) : 0;
    if (nbn > 0) {
      // the next panel's columns: helpers finished panel pidx-1's far update
      // of them; apply this panel's interchanges (one column per CTA)
      if (pidx >= 1) {
        if (tid == 0) wait_geq(&hs->fardone[pidx - 1], nhc);
        __syncthreads();
      }
      const int cnt = S.pcnt;
      if (b < nbn && warp == 0 && cnt > 0) {
        double* col = p.a + (int64_t)(ce + b) * lda;
        const double v0 = lane < cnt ? col[S.prow_src[lane]] : 0.0;
        __syncwarp();
        if (lane < cnt) col[S.prow_rows[lane]] = v0;
      }
      cluster.sync();  // (2) next columns interchanged
    }
    if (b == 0 && tid == 0) {
      __threadfence();
      st_release(&hs->ready, (unsigned)pidx + 1);  // helpers: next columns, far columns, L columns
    }
    FULL_TRACE(6 * pidx + 3);
    if (nbn == 0) break;
    // ---- next panel: the helpers form its U12 rows and update its rows below
    // (rank-nb with this panel's multipliers); load my physical rows >= ce
    if (tid == 0) wait_geq(&hs->nextdone[pidx], nhc);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < RPT; k++) {
      const int64_t g = x.g0 + (int64_t)k * T;
      const bool act = k < x.nk && g >= ce;
      P.lr[k] = act ? (int)g : -1;
#pragma unroll
      for (int c = 0; c < W; c++) P.a[k][c] = (act && c < nbn) ? p.a[g + (int64_t)(ce + c) * lda] : 0.0;
    }
    if (tid < nbn) {  // colmax of the next columns over the rows above: every U12 row so far
      const unsigned long long cb = hs->cmax[ce + tid];
      x.s_cmab[ce + tid] = cb ? __longlong_as_double((long long)cb) : -1.0;
    }
    __syncthreads();
    FULL_TRACE(6 * pidx + 5);
  }
  cluster.sync();  // nobody leaves while a peer may still address its shared memory
}

template <int W>
__device__ void helper_role(const Args& p, Handoff* hs, double* dyn) {
  __shared__ double l11[W][W + 1];
  __shared__ int64_t prw[2 * W], psr[2 * W];
  __shared__ int s_cnt;
  __shared__ unsigned s_zm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned h = blockIdx.x - CS, nhc = p.nhelpers;
  const int64_t m = p.m, n = p.n, lda = p.lda;
  double* u12 = dyn;              // [W][W] U12 of the next panel's columns
  double* u12f = dyn + W * W;     // [W][n - fs] U12 of the far columns
  const int np = (int)((n + W - 1) / W);
  for (int pidx = 0; pidx < np; pidx++) {
    const int j0 = pidx * W;
    const int nb = (int)min((int64_t)W, n - j0);
    const int ce = j0 + nb;
    const int nbn = ce < n ? (int)min((int64_t)W, n - ce) : 0;
    const int fs = ce + nbn;  // far columns [fs, n)
    const int nfar = (int)n - fs;
    if (tid == 0) {
      wait_geq(&hs->ready, (unsigned)pidx + 1);
      if (pidx >= 1) wait_geq(&hs->fardone[pidx - 1], nhc);
    }
    __syncthreads();
    const int cnt = hs->pcnt[pidx];
    if (tid < cnt) {
      prw[tid] = hs->prow[pidx][tid];
      psr[tid] = hs->psrc[pidx][tid];
    }
    if (warp == 0) {  // zero-pivot mask: one load per lane
      const unsigned z = __ballot_sync(0xffffffffu, lane < nb && p.zflag[j0 + lane] != 0);
      if (lane == 0) {
        s_zm = z;
        s_cnt = cnt;
      }
    }
    if (nfar > 0)
      for (int e = tid; e < nb * nb; e += T) {
        const int r = e % nb, c = e / nb;
        l11[r][c] = p.a[(j0 + r) + (int64_t)(j0 + c) * lda];
      }
    __syncthreads();
    const unsigned zm = s_zm;
    // ---- phase N: the next panel's columns [ce, fs) (already interchanged by
    // the panel cluster): U12 rows (every helper, half-warp per column), the
    // rank-nb update of my block of rows >= ce; helper 0 publishes U12 + colmax
    if (nbn > 0) {
      if (nfar <= 0)  // L11 not loaded above
        for (int e = tid; e < nb * nb; e += T) {
          const int r = e % nb, c = e / nb;
          l11[r][c] = p.a[(j0 + r) + (int64_t)(j0 + c) * lda];
        }
      __syncthreads();
      {
        const int cw = warp * 2 + (lane >> 4), l = lane & 15;
        double xv = 0.0;
        if (cw < nbn && l < nb) xv = p.a[(int64_t)(ce + cw) * lda + j0 + l];
        for (int t = 0; t + 1 < nb; t++) {
          const double xt = __shfl_sync(0xffffffffu, xv, t, 16);
          if (l > t && l < nb && !((zm >> t) & 1u)) xv = sub_mul_nofma(xv, l11[l][t], xt);
        }
        if (cw < nbn && l < nb) u12[(size_t)l * W + cw] = xv;
      }
      __syncthreads();
      // helper 0 overwrites rows j0..ce of the next columns with U12 only
      // after every other helper has read the (interchanged) originals
      if (h != 0 && tid == 0) red_release_add(&hs->u12read[pidx], 1u);
      const int64_t nrow = m - ce;
      const int64_t rbk = (nrow + nhc - 1) / nhc;
      const int64_t iend = min(m, ce + (int64_t)(h + 1) * rbk);
      for (int64_t i = ce + (int64_t)h * rbk + tid; i < iend; i += T) {
        double y[W];
#pragma unroll
        for (int c = 0; c < W; c++) y[c] = c < nbn ? p.a[i + (int64_t)(ce + c) * lda] : 0.0;
        double lv[W];  // all loads in flight before the update
#pragma unroll
        for (int s2 = 0; s2 < W; s2++) lv[s2] = s2 < nb ? p.a[i + (int64_t)(j0 + s2) * lda] : 0.0;
#pragma unroll
        for (int s2 = 0; s2 < W; s2++) {
          if (s2 >= nb || ((zm >> s2) & 1u)) continue;
          const double* us = u12 + (size_t)s2 * W;
#pragma unroll
          for (int c = 0; c < W; c++) y[c] = sub_mul_nofma(y[c], lv[s2], c < nbn ? us[c] : 0.0);
        }
#pragma unroll
        for (int c = 0; c < W; c++)
          if (c < nbn) p.a[i + (int64_t)(ce + c) * lda] = y[c];
      }
      if (h == 0) {
        if (tid == 0) wait_geq(&hs->u12read[pidx], nhc - 1);
        __syncthreads();
        for (int e = tid; e < nb * nbn; e += T) {
          const int s2 = e % nb, c = e / nb;
          p.a[(j0 + s2) + (int64_t)(ce + c) * lda] = u12[(size_t)s2 * W + c];
        }
        if (tid < nbn) {
          unsigned long long key = 0ull;
          for (int s2 = 0; s2 < nb; s2++) {
            const unsigned long long kk = vkey(fabs(u12[(size_t)s2 * W + tid]));
            key = kk > key ? kk : key;
          }
          if (key) atomicMax(&hs->cmax[ce + tid], key);
        }
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        red_release_add(&hs->nextdone[pidx], 1u);
      }
    }
    // ---- phase A: interchanges on columns [0, j0) and [fs, n); far U12 rows
    const int64_t na = (int64_t)j0 + nfar;
    for (int64_t q = (int64_t)h * (T / 32) + warp; q < na; q += (int64_t)nhc * (T / 32)) {
      const int64_t c = q < j0 ? q : fs + (q - j0);
      double* col = p.a + c * lda;
      if (cnt > 0) {
        const double v0 = lane < cnt ? col[psr[lane]] : 0.0;
        __syncwarp();
        if (lane < cnt) col[prw[lane]] = v0;
        __syncwarp();
      }
      if (c >= fs) {
        double xv = lane < nb ? col[j0 + lane] : 0.0;
        for (int t = 0; t + 1 < nb; t++) {
          const double xt = __shfl_sync(0xffffffffu, xv, t);
          if (lane > t && lane < nb && !((zm >> t) & 1u)) xv = sub_mul_nofma(xv, l11[lane < W ? lane : 0][t], xt);
        }
        if (lane < nb) col[j0 + lane] = xv;
        unsigned long long key = lane < nb ? vkey(fabs(xv)) : 0ull;
        unsigned dummy = 0u;
        warp_keymax(key, dummy);
        if (lane == 0 && key) atomicMax(&hs->cmax[c], key);
      }
    }
    __syncthreads();
    if (nfar <= 0) {
      if (tid == 0) red_release_add(&hs->fardone[pidx], 1u);
      continue;
    }
    if (tid == 0) {
      __threadfence();
      red_release_add(&hs->u12done[pidx], 1u);
      wait_geq(&hs->u12done[pidx], nhc);
    }
    __syncthreads();
    for (int e = tid; e < nb * nfar; e += T) {  // far U12 rows -> shared memory
      const int s2 = e % nb, c = e / nb;
      u12f[(size_t)s2 * nfar + c] = p.a[(j0 + s2) + (int64_t)(fs + c) * lda];
    }
    __syncthreads();
    // ---- phase B: my block of rows >= ce, all far columns (16-column batches)
    const int64_t nrow = m - ce;
    const int64_t rbk = (nrow + nhc - 1) / nhc;
    const int64_t iend = min(m, ce + (int64_t)(h + 1) * rbk);
    for (int64_t i = ce + (int64_t)h * rbk + tid; i < iend; i += T) {
      double lv[W];
#pragma unroll
      for (int s2 = 0; s2 < W; s2++) lv[s2] = s2 < nb ? p.a[i + (int64_t)(j0 + s2) * lda] : 0.0;
      constexpr int CBH = 16;
      for (int c0 = 0; c0 < nfar; c0 += CBH) {
        double y[CBH];
#pragma unroll
        for (int q = 0; q < CBH; q++) y[q] = (c0 + q < nfar) ? p.a[i + (int64_t)(fs + c0 + q) * lda] : 0.0;
#pragma unroll
        for (int s2 = 0; s2 < W; s2++) {
          if (s2 < nb && !((zm >> s2) & 1u)) {
            const double* us = u12f + (size_t)s2 * nfar + c0;
#pragma unroll
            for (int q = 0; q < CBH; q++) y[q] = sub_mul_nofma(y[q], lv[s2], (c0 + q < nfar) ? us[q] : 0.0);
          }
        }
#pragma unroll
        for (int q = 0; q < CBH; q++)
          if (c0 + q < nfar) p.a[i + (int64_t)(fs + c0 + q) * lda] = y[q];
      }
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      red_release_add(&hs->fardone[pidx], 1u);
    }
  }
}

template <int RPT, int W>
__global__ void __launch_bounds__(T, 1) lu_coop_kernel(const Args p) {
  extern __shared__ __align__(16) double dyn[];
  Handoff* hs = reinterpret_cast<Handoff*>(p.recg);
  if (blockIdx.x < (unsigned)CS) panel_role<RPT, W>(p, hs, dyn);
  else helper_role<W>(p, hs, dyn);
}

}  // namespace lufull

#ifndef LUF_WIDE_CTA
// Eligibility of the one-launch cluster GEPP (getrf.cu dispatches to it).
bool getrf_full_eligible(int64_t m, int64_t n, int cluster_max) {
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = getenv("RLRA_B200_LU_FULL");
    enabled = (e && e[0] == '0') ? 0 : 1;  // RLRA_B200_LU_FULL=0 selects the blocked path
    // Nsight Compute cannot replay cooperative cluster grids (the launch fails
    // inside the tool): under a CUDA injection library use the blocked path
    if (getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") || getenv("NV_TPS_LAUNCH_TOKEN")) enabled = 0;
  }
  // widths above 512 only while the far-column work stays small: beyond, the
  // blocked path's all-SM trailing update wins (profiles/r02_getrf_width.txt:
  // 4096 x 544 coop 2.12 vs blocked 2.30 ms; 16384 x 1024 coop 8.14 vs 6.25 ms)
  static int64_t wide_mn = -1;  // RLRA_B200_LU_FULL_WIDE_MN overrides the measured crossover (experiments)
  if (wide_mn < 0) {
    const char* e = getenv("RLRA_B200_LU_FULL_WIDE_MN");
    wide_mn = (e && atoll(e) > 0) ? atoll(e) : (int64_t)4500000;
  }
  const bool width_ok = n <= 512 || (n <= lufull::MAXN && m * n <= wide_mn);
  return enabled && cluster_max >= lufull::CS && n >= 1 && m >= n && width_ok &&
         m >= (int64_t)lufull::CS * 32 && m <= (int64_t)lufull::CS * lufull::T * lufull::MAXRPT;
}

size_t getrf_full_state_bytes() { return sizeof(lufull::Handoff); }

// rows the 384-thread build takes (2 rows per thread)
int64_t getrf_full_wide_rows() { return (int64_t)lufull::CS * 384 * 2; }
#endif

// Cooperative launch of the panel cluster + NH helper clusters (returns 1 when
// the device cannot hold a helper cluster next to the panel cluster: the
// caller then uses the blocked path).
template <int RPT, int W>
static int launch_full(lufull::Args a, cudaStream_t st) {
  const void* kern = (const void*)lufull::lu_coop_kernel<RPT, W>;
  using PL = lufull::Plan<RPT, W>;
  const size_t dyn = PL::bytes(a.n);
  static std::mutex mu;
  static int nclusters[64][lufull::MAXRPT + 1];
  int dev = 0;
  RLRA_CHECK_CUDA(cudaGetDevice(&dev));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(lufull::CS);
  cfg.blockDim = dim3(lufull::T);
  cfg.dynamicSmemBytes = PL::max_bytes();
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = lufull::CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!nclusters[dev & 63][RPT]) {
      RLRA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      RLRA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PL::max_bytes()));
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess) ncl = 0;
      cudaGetLastError();
      nclusters[dev & 63][RPT] = ncl > 0 ? ncl : -1;
    }
  }
  const int ncl = nclusters[dev & 63][RPT];
  if (ncl < 2) return 1;
  static int nh_cap = -1;  // helper clusters (RLRA_B200_LU_HELPERS overrides the default 6)
  if (nh_cap < 0) {
    const char* e = getenv("RLRA_B200_LU_HELPERS");
    nh_cap = (e && atoi(e) > 0) ? atoi(e) : 6;
  }
  const int nh = ncl - 1 < nh_cap ? ncl - 1 : nh_cap;
  a.nhelpers = (unsigned)(nh * lufull::CS);
  RLRA_CHECK_CUDA(cudaMemsetAsync(a.recg, 0, sizeof(lufull::Handoff), st));
  cfg.gridDim = dim3(lufull::CS * (1 + nh));
  cfg.dynamicSmemBytes = dyn;
  cfg.numAttrs = 2;
  void* kargs[] = {&a};
  const cudaError_t e = cudaLaunchKernelExC(&cfg, kern, kargs);
  if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorNotSupported || e == cudaErrorInvalidConfiguration ||
      e == cudaErrorNotPermitted) {
    // e.g. under a profiler that cannot replay cooperative cluster grids:
    // remember and let the caller take the blocked path
    cudaGetLastError();
    std::lock_guard<std::mutex> lock(mu);
    nclusters[dev & 63][RPT] = -1;
    return 1;
  }
  RLRA_CHECK_CUDA(e);
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
#ifdef LUF_WIDE_CTA
  RLRA_REQUIRE(rpt <= 2, "getrf_full_wide: m = %lld needs more than 2 rows per thread", (long long)m);
  return rpt == 1 ? launch_full<1, 16>(args, st) : launch_full<2, 16>(args, st);
#else
  switch (rpt) {
    case 1: return launch_full<1, 16>(args, st);
    case 2: return launch_full<2, 16>(args, st);
    case 3: return launch_full<3, 16>(args, st);
    case 4: return launch_full<4, 16>(args, st);
    case 5: return launch_full<5, 16>(args, st);
    default: return launch_full<6, 16>(args, st);
  }
#endif
}

}  // namespace rlra
