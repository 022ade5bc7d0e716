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
#include <cooperative_groups.h>

#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"

namespace rlra {

constexpr int LU_NB = 32;
constexpr double ZERO_PIVOT_RTOL = 1e-14;  // rlra/_lu_cython.pyx:11

struct LuWork {
  double* cand_val;    // [2][G]   local first-max |a| over own rows >= j (-1 if none)
  int64_t* cand_idx;   // [2][G]
  double* cand_cmax;   // [2][G]   local max |a| over own rows in [j0, j)
  double* cand_row;    // [2][G][LU_NB] panel row of the local argmax
  double* diag_row;    // [2][LU_NB]  current panel row j
  double* above;       // [G][LU_NB]  max |a| over rows < j0, per panel column
  unsigned* bar;       // grid barrier (2 words)
  int64_t* ipiv;       // [r] pivot row chosen at step j (== j when no swap)
  int* zflag;          // [r] 1 when step j was a zero pivot
  int64_t* perm_rows;  // [2*LU_NB] rows touched by the panel's swaps
  int64_t* perm_src;   // [2*LU_NB] source row of each touched row after the swaps
  int* perm_cnt;       // [1]
  int64_t* count;      // [1] nonzero diagonal count
  double* recg;        // cluster panel: [2][16][2+LU_NB] records + [2][LU_NB] diagonal rows (global staging for the multicast)
};

struct PanelArgs {
  double* a;
  int64_t lda, m, n, j0;
  int nb;
  int64_t rows_per_cta;   // active rows [j0, m) split in contiguous chunks
  int64_t above_per_cta;  // rows [0, j0) split in contiguous chunks
  int64_t* piv;
  LuWork w;
  unsigned bar_base;  // monotonic grid-barrier counter value at kernel entry
  unsigned long long* trace;  // RLRA_LU_TRACE builds only: [CTA][128] globaltimer stamps
};

// x / d correctly rounded (IEEE round-to-nearest, like C's `/`), given the
// correctly rounded reciprocal rcp = RN(1/d): Markstein's theorem -- q0 = RN(x*rcp),
// rem = x - d*q0 exactly (FMA), RN(q0 + rem*rcp) == RN(x/d) -- valid away from
// overflow / underflow; other operands take the hardware division path.
__device__ __noinline__ double ieee_div_slow_path(double x, double d) { return x / d; }  // rare: keep it out of the column step
__device__ __forceinline__ double ieee_div_by(double x, double d, double rcp) {
  const double ax = fabs(x), ad = fabs(d);
  if (ax > 0x1p-960 && ax < 0x1p+960 && ad > 0x1p-960 && ad < 0x1p+960) {
    const double q0 = __dmul_rn(x, rcp);
    const double rem = fma(-d, q0, x);
    return fma(rem, rcp, q0);
  }
  return ieee_div_slow_path(x, d);
}

// strict-greater first-max merge: (v,i) replaces best when v > best or (v == best && i < besti)
__device__ __forceinline__ bool better(double v, int64_t i, double bv, int64_t bi) {
  return v > bv || (v == bv && i < bi);
}

__device__ __forceinline__ void warp_argmax(double& v, int64_t& idx, double& cmax) {
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    double ov = __shfl_down_sync(0xffffffffu, v, off);
    long long oi = __shfl_down_sync(0xffffffffu, (long long)idx, off);
    double oc = __shfl_down_sync(0xffffffffu, cmax, off);
    if (better(ov, oi, v, idx)) { v = ov; idx = oi; }
    if (oc > cmax) cmax = oc;
  }
}

// Block-wide (value, index) first-max reduction + max of cmax; result broadcast
// to every thread through shared memory.
__device__ void block_argmax_bcast(double& v, int64_t& idx, double& cmax, double* s_v,
                                   int64_t* s_i, double* s_c) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_argmax(v, idx, cmax);
  if (lane == 0) { s_v[warp] = v; s_i[warp] = idx; s_c[warp] = cmax; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    v = lane < nw ? s_v[lane] : -1.0;
    idx = lane < nw ? s_i[lane] : INT64_MAX;
    cmax = lane < nw ? s_c[lane] : -1.0;
    warp_argmax(v, idx, cmax);
    if (lane == 0) { s_v[32] = v; s_i[32] = idx; s_c[32] = cmax; }
  }
  __syncthreads();
  v = s_v[32];
  idx = s_i[32];
  cmax = s_c[32];
  __syncthreads();
}

// Net row permutation of one panel's swap sequence (j <-> ipiv[j], j ascending),
// as (touched row, source row) pairs for the laswp gather/scatter.  Run by one
// warp with the lookups done lane-parallel in shared memory (<= 2*LU_NB rows).
__device__ int build_panel_perm(int64_t j0, int nb, const int64_t* s_ipiv, int64_t* s_rows,
                                int64_t* s_src, const LuWork& w) {
  const int lane = threadIdx.x & 31;
  int cnt = 0;
  auto find = [&](int64_t r) -> int {
    bool hit0 = lane < cnt && s_rows[lane] == r;
    bool hit1 = lane + 32 < cnt && s_rows[lane + 32] == r;
    unsigned b0 = __ballot_sync(0xffffffffu, hit0), b1 = __ballot_sync(0xffffffffu, hit1);
    if (b0) return __ffs(b0) - 1;
    if (b1) return 32 + __ffs(b1) - 1;
    if (lane == 0) { s_rows[cnt] = r; s_src[cnt] = r; }
    __syncwarp();
    return cnt++;
  };
  for (int q = 0; q < nb; q++) {
    const int64_t jq = j0 + q, pr = s_ipiv[q];
    if (pr == jq) continue;
    const int ka = find(jq), kb = find(pr);
    if (lane == 0) {
      int64_t t = s_src[ka];
      s_src[ka] = s_src[kb];
      s_src[kb] = t;
    }
    __syncwarp();
  }
  if (lane < cnt) { w.perm_rows[lane] = s_rows[lane]; w.perm_src[lane] = s_src[lane]; }
  if (lane + 32 < cnt) { w.perm_rows[lane + 32] = s_rows[lane + 32]; w.perm_src[lane + 32] = s_src[lane + 32]; }
  if (lane == 0) *w.perm_cnt = cnt;
  __syncwarp();
  return cnt;
}

// Panel factorization with the CTA's panel rows resident in SHARED MEMORY
// (column-major s_a[c * R + r], R = rows_per_cta), one grid barrier per column.
// Thread t handles local rows t, t + THREADS, ...; every inner loop has a
// runtime trip count (nb - jj), so no predicated full-width sweeps.
template <int PW, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) lu_panel_smem_kernel(PanelArgs p) {
  extern __shared__ __align__(16) double s_a[];
  __shared__ double s_v[33], s_c[33];
  __shared__ int64_t s_i[33];
  __shared__ double s_above[PW];
  __shared__ double s_u[PW];
  __shared__ double s_part[THREADS / 32][PW];
  __shared__ int64_t s_prow;
  __shared__ int s_zero, s_winner;
  __shared__ int64_t s_ipiv[PW], s_prow_rows[2 * PW], s_prow_src[2 * PW];

  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int nb = p.nb;
  const int64_t R = p.rows_per_cta;
  const int64_t rb = min(p.m, p.j0 + (int64_t)b * R);
  const int64_t re = min(p.m, rb + R);
  const int nr = (int)(re - rb);

  // ---- prologue 1: max |a| over rows < j0 (final U rows), per panel column
  {
    const int64_t ab = min(p.j0, (int64_t)b * p.above_per_cta);
    const int64_t ae = min(p.j0, ab + p.above_per_cta);
    double mx[PW];
#pragma unroll
    for (int c = 0; c < PW; c++) mx[c] = -1.0;
    for (int64_t i = ab + tid; i < ae; i += THREADS)
#pragma unroll
      for (int c = 0; c < PW; c++)
        if (c < nb) {
          double v = fabs(p.a[cm(i, p.j0 + c, p.lda)]);
          if (v > mx[c]) mx[c] = v;
        }
#pragma unroll
    for (int c = 0; c < PW; c++) {
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        double o = __shfl_down_sync(0xffffffffu, mx[c], off);
        if (o > mx[c]) mx[c] = o;
      }
      if ((tid & 31) == 0) s_part[tid >> 5][c] = mx[c];
    }
    __syncthreads();
    if (tid < nb) {
      double m2 = -1.0;
      for (int wv = 0; wv < THREADS / 32; wv++)
        if (s_part[wv][tid] > m2) m2 = s_part[wv][tid];
      __stcg(p.w.above + (int64_t)b * LU_NB + tid, m2);
    }
  }
  // ---- prologue 2: stage the panel rows in shared memory (coalesced)
  for (int c = 0; c < nb; c++)
    for (int r = tid; r < nr; r += THREADS) s_a[c * R + r] = p.a[cm(rb + r, p.j0 + c, p.lda)];
  __syncthreads();

  // local candidates of column c (step row j), published into buffer `par`
  auto publish = [&](int c, int64_t j, int par) {
    double v = -1.0, cmax = -1.0;
    int64_t idx = INT64_MAX;
    const double* col = s_a + c * R;
    for (int r = tid; r < nr; r += THREADS) {
      const int64_t i = rb + r;
      const double xv = fabs(col[r]);
      if (i >= j) {
        if (better(xv, i, v, idx)) { v = xv; idx = i; }
      } else if (xv > cmax) {
        cmax = xv;  // rows in [j0, j): pivoted rows, part of colmax
      }
    }
    block_argmax_bcast(v, idx, cmax, s_v, s_i, s_c);
    if (tid == 0) {
      __stcg(p.w.cand_val + par * G + b, v);
      __stcg(p.w.cand_idx + par * G + b, idx);
      __stcg(p.w.cand_cmax + par * G + b, cmax);
    }
    if (v >= 0.0 && tid < nb)
      __stcg(p.w.cand_row + ((int64_t)par * G + b) * LU_NB + tid, s_a[tid * R + (idx - rb)]);
    if (j >= rb && j < re && tid < nb)
      __stcg(p.w.diag_row + par * LU_NB + tid, s_a[tid * R + (j - rb)]);
  };

  publish(0, p.j0, 0);

  for (int jj = 0; jj < nb; jj++) {
    const int64_t j = p.j0 + jj;
    const int par = jj & 1;
    grid_barrier_mono(p.w.bar, p.bar_base + (unsigned)G * (jj + 1));
    if (jj == 0 && tid < nb) {
      double mx = -1.0;
      for (int q = 0; q < G; q++) {
        double v = __ldcg(p.w.above + (int64_t)q * LU_NB + tid);
        if (v > mx) mx = v;
      }
      s_above[tid] = mx;
    }
    // ---- global pivot decision: every CTA reduces the G candidates identically
    {
      double v = -1.0, cmax = -1.0;
      int64_t idx = INT64_MAX;
      if (tid < G) {
        double qv = __ldcg(p.w.cand_val + par * G + tid);
        if (qv >= 0.0) { v = qv; idx = __ldcg(p.w.cand_idx + par * G + tid); }
        cmax = __ldcg(p.w.cand_cmax + par * G + tid);
      }
      block_argmax_bcast(v, idx, cmax, s_v, s_i, s_c);
      if (tid == 0) {
        // reference: amax = first max over rows >= j (or -1); colmax = amax,
        // then max over rows < j with strict '>' (rlra/_lu_cython.pyx:23-35)
        double amax = v, colmax = amax;
        if (s_above[jj] > colmax) colmax = s_above[jj];
        if (cmax > colmax) colmax = cmax;
        const int zero = (amax <= ZERO_PIVOT_RTOL * colmax) ? 1 : 0;
        s_zero = zero;
        s_prow = zero ? j : idx;
        s_ipiv[jj] = zero ? j : idx;
        // owner CTA of the winning row (rows are split in contiguous chunks)
        s_winner = zero ? -1 : (int)((idx - p.j0) / R);
        if (b == 0) {
          p.w.zflag[j] = zero;
          p.w.ipiv[j] = zero ? j : idx;
          if (!zero && idx != j) {
            int64_t t = p.piv[j];
            p.piv[j] = p.piv[idx];
            p.piv[idx] = t;
          }
        }
      }
      __syncthreads();
    }
    const int zero = s_zero;
    const int64_t prow = s_prow;
    const int r0 = (int)max((int64_t)0, j + 1 - rb);  // first local row below the diagonal
    if (!zero) {
      if (tid < nb) {
        const double u = __ldcg(p.w.cand_row + ((int64_t)par * G + s_winner) * LU_NB + tid);
        s_u[tid] = u;
        // full-row swap inside the panel (:40-48)
        if (prow != j) {
          if (j >= rb && j < re) s_a[tid * R + (j - rb)] = u;
          if (prow >= rb && prow < re)
            s_a[tid * R + (prow - rb)] = __ldcg(p.w.diag_row + par * LU_NB + tid);
        }
      }
      __syncthreads();
      const double ujj = s_u[jj];
      double* colj = s_a + jj * R;
      // same thread->row mapping as publish(): each thread only touches its own
      // rows, so the fused candidate scan below needs no extra barrier
      for (int r = tid; r < nr; r += THREADS) {
        if (r < r0) continue;
        const double l = colj[r] / ujj;  // IEEE division (:49-51)
        colj[r] = l;
        for (int c = jj + 1; c < nb; c++) {
          double* e = s_a + c * R + r;
          *e = sub_mul_nofma(*e, l, s_u[c]);  // multiply then subtract (:52-55)
        }
      }
    } else {
      // zero pivot: zero the L column below the diagonal; no swap, no update (:36-39)
      for (int r = tid; r < nr; r += THREADS)
        if (r >= r0) s_a[jj * R + r] = 0.0;
    }
    if (jj + 1 < nb) publish(jj + 1, j + 1, par ^ 1);
  }

  // ---- write the panel back (coalesced)
  __syncthreads();
  for (int c = 0; c < nb; c++)
    for (int r = tid; r < nr; r += THREADS) p.a[cm(rb + r, p.j0 + c, p.lda)] = s_a[c * R + r];

  if (b == 0 && tid < 32) build_panel_perm(p.j0, nb, s_ipiv, s_prow_rows, s_prow_src, p.w);
}

// (value, index, cmax) first-max reduction over the whole block; every thread
// ends with the result.  Values are |a| >= 0 (or -1 for "no row"); the max is
// found with fmax shuffles (NaN never wins, like the reference's strict '>'),
// the smallest row index holding it with one redux.min, so ties keep the
// first maximum.  ONE __syncthreads; callers must separate consecutive uses of
// the staging arrays by another block barrier.  `base` is subtracted from the
// row indices so they fit the 32-bit redux.
__device__ __forceinline__ void block_argmax_all(double& v, int64_t& idx, double& cmax, double* s_v,
                                                 int64_t* s_i, double* s_c, int64_t base = 0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto warp_reduce = [&](double& vv, int64_t& ii, double& cc) {
    double vm = vv, cm2 = cc;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      vm = fmax(vm, __shfl_xor_sync(0xffffffffu, vm, off));
      cm2 = fmax(cm2, __shfl_xor_sync(0xffffffffu, cm2, off));
    }
    const unsigned key = (vv == vm && vm >= 0.0 && ii != INT64_MAX) ? (unsigned)(ii - base) : 0xffffffffu;
    const unsigned kmin = __reduce_min_sync(0xffffffffu, key);
    vv = vm;
    cc = cm2;
    ii = (kmin == 0xffffffffu) ? INT64_MAX : (int64_t)kmin + base;
  };
  warp_reduce(v, idx, cmax);
  if (lane == 0) { s_v[warp] = v; s_i[warp] = idx; s_c[warp] = cmax; }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  v = lane < nw ? s_v[lane] : -1.0;
  idx = lane < nw ? s_i[lane] : INT64_MAX;
  cmax = lane < nw ? s_c[lane] : -1.0;
  warp_reduce(v, idx, cmax);
}

// ---------------------------------------------------------------------------
// Cluster-resident panel (B200 thread-block cluster, up to 16 CTAs on one GPC).
// The panel rows live in the CTAs' shared memory.  Each column step, every CTA
// PUSHES its pivot candidate record (|value|, row, colmax, full panel row) into
// every peer's shared memory with a DSMEM bulk copy (cp.async.bulk, TMA engine)
// that completes on the peer's local mbarrier; the owner of the next diagonal
// row pushes that row the same way.  A CTA then only waits on its OWN
// mbarrier and decides from local data: no cluster-wide barrier, no
// MEMBAR.GPU, no remote loads on the critical path.  Records are double
// buffered by step parity; the wait for step s+1's records is what makes it
// safe to overwrite step s's slots (every peer has then finished reading).
template <int PW>
struct LuRec {
  double val, idx, cmax, pad;  // idx is an int64 stored bit-for-bit
  double row[PW];
};

template <int PW, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) lu_panel_cluster_kernel(PanelArgs p) {
  namespace cg = cooperative_groups;
  constexpr int MAXCS = 16;
  constexpr int RECD = 2 + PW;  // record doubles: {|value|, row index bits, row[PW]}
  static_assert(RECD % 2 == 0, "records are pushed as 16-byte pairs");
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double s_a[];
  __shared__ double s_v[32];
  __shared__ int64_t s_i[32];
  __shared__ double s_c[32];
  __shared__ __align__(16) double recv[2][MAXCS][RECD];  // pushed by every peer
  __shared__ __align__(16) double recv_diag[2][PW];      // current diagonal row (pre-swap)
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ __align__(8) uint64_t ldbar;
  __shared__ double c_above[PW];
  __shared__ double s_u[2][PW];   // pivot row of the step, double-buffered by parity
  __shared__ double s_rcp[2];
  __shared__ double s_part[THREADS / 32][PW];
  __shared__ int64_t s_prow[2];
  __shared__ int s_zero[2];
  __shared__ int64_t s_ipiv[PW], s_prow_rows[2 * PW], s_prow_src[2 * PW];
  __shared__ int s_zf[PW];

  const int CS = (int)cluster.num_blocks(), b = (int)cluster.block_rank(), tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
#ifdef RLRA_LU_TRACE
  auto trace = [&](int slot) {
    if (lane == 0 && warp == 0 && p.trace && slot < 128) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      p.trace[(int64_t)b * 128 + slot] = t;
    }
  };
#else
  auto trace = [&](int) {};
#endif
  trace(0);
  const int nb = p.nb;
  const int64_t R = p.rows_per_cta;
  const int64_t rb = min(p.m, p.j0 + (int64_t)b * R);
  const int64_t re = min(p.m, rb + R);
  const int nr = (int)(re - rb);
  const int Ri = (int)R;  // 32-bit shared-memory indexing
  const unsigned tx_bytes = CS * RECD * 8u + PW * 8u;

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&ldbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // ---- prologue 1: stage the panel rows -- one TMA bulk copy per column
  // (16-byte aligned when R, rb and lda are even; an odd last row is loaded directly)
  const bool bulk_ok = ((R & 1) == 0) && ((p.lda & 1) == 0) && ((rb & 1) == 0);
  const int nr_bulk = bulk_ok ? (nr & ~1) : 0;
  if (nr_bulk > 0 && tid == 0) {
    mbar_arrive_expect_tx(&ldbar, (unsigned)(nb * nr_bulk * 8));
    for (int c = 0; c < nb; c++)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              smem_u32(s_a + c * R)),
          "l"(p.a + cm(rb, p.j0 + c, p.lda)), "r"((unsigned)(nr_bulk * 8)), "r"(smem_u32(&ldbar))
          : "memory");
  }
  // ---- prologue 2 (overlaps the copies): max |a| over rows < j0 (final U rows)
  {
    const int64_t ab = min(p.j0, (int64_t)b * p.above_per_cta);
    const int64_t ae = min(p.j0, ab + p.above_per_cta);
    double mx[PW];
#pragma unroll
    for (int c = 0; c < PW; c++) mx[c] = -1.0;
    for (int64_t i = ab + tid; i < ae; i += THREADS)
#pragma unroll
      for (int c = 0; c < PW; c++)
        if (c < nb) {
          double v = fabs(p.a[cm(i, p.j0 + c, p.lda)]);
          if (v > mx[c]) mx[c] = v;
        }
#pragma unroll
    for (int c = 0; c < PW; c++) {
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        double o = __shfl_down_sync(0xffffffffu, mx[c], off);
        if (o > mx[c]) mx[c] = o;
      }
      if (lane == 0) s_part[warp][c] = mx[c];
    }
  }
  for (int c = 0; c < nb; c++)
    for (int r = nr_bulk + tid; r < nr; r += THREADS) s_a[c * R + r] = p.a[cm(rb + r, p.j0 + c, p.lda)];
  if (nr_bulk > 0) mbar_wait_parity(&ldbar, 0);
  __syncthreads();
  if (tid < PW) {
    double m2 = -1.0;
    for (int wv = 0; wv < THREADS / 32; wv++)
      if (s_part[wv][tid] > m2) m2 = s_part[wv][tid];
    c_above[tid] = m2;
  }
  if (tid == 0) {  // arm both phases' expected bytes
    mbar_arrive_expect_tx(&mbar[0], tx_bytes);
    mbar_arrive_expect_tx(&mbar[1], tx_bytes);
  }
  trace(1);
  cluster.sync();  // mbarrier inits + c_above visible cluster-wide (once per panel)
  trace(2);
  // warp 0, lane c: running colmax of column c = max(|a| over rows < j0,
  // |pivot row value| over this panel's earlier steps) -- the reference's
  // "whole column" colmax without a second reduction (rlra/_lu_cython.pyx:31-35)
  double colmax_mine = -1.0;
  if (warp == 0 && lane < nb)
    for (int q = 0; q < CS; q++) {
      double v = *cluster.map_shared_rank(&c_above[lane], q);
      if (v > colmax_mine) colmax_mine = v;
    }

  // Local first-max candidate of panel column c (rows >= j), then warp 0
  // finishes the look-ahead remainder (columns > c, multipliers in column c-1)
  // of the two rows that leave this CTA -- candidate row and next diagonal row
  // -- and pushes record + diagonal row into every peer with st.async, which
  // completes on the peer's mbarrier (no proxy fence, no source buffer).
  auto publish = [&](int c, int64_t j, int par, bool owe, int upar) {
    double v = -1.0, dummy = -1.0;
    int64_t idx = INT64_MAX;
    const double* col = s_a + c * R;
    for (int r = tid; r < nr; r += THREADS) {
      const int64_t i = rb + r;
      if (i >= j) {
        const double xv = fabs(col[r]);
        if (better(xv, i, v, idx)) { v = xv; idx = i; }
      }
    }
    block_argmax_all(v, idx, dummy, s_v, s_i, s_c, rb);
    if (c <= 12) trace(8 + 8 * (c - 1) + 4);
    const bool own_diag = (j >= rb && j < re);
    if (warp == 0) {
      const double* u = s_u[upar];
      if (owe) {
        const double* lcol = s_a + (c - 1) * R;
        if (lane > c && lane < nb) {
          if (v >= 0.0) {
            const int r = (int)(idx - rb);
            s_a[lane * R + r] = sub_mul_nofma(s_a[lane * R + r], lcol[r], u[lane]);
          }
          if (own_diag && j != idx) {
            const int r = (int)(j - rb);
            s_a[lane * R + r] = sub_mul_nofma(s_a[lane * R + r], lcol[r], u[lane]);
          }
        }
        __syncwarp();
      }
      // Record {v, idx, row[PW]} (and the next diagonal row) are staged in a
      // per-CTA global slot, then ONE multicast bulk copy (TMA engine) writes
      // them into every peer's shared memory at the same offset and completes
      // on every peer's mbarrier.  Slots are reused two steps later, after this
      // CTA has received the step's multicast (so the read is done).
      const int rr = (int)(idx - rb);
      double* slot = p.w.recg + ((int64_t)par * 16 + b) * RECD;
      double* dslot = p.w.recg + 2 * 16 * RECD + par * PW;
      for (int pr = lane; pr < RECD / 2; pr += 32) {
        double x0, x1;
        if (pr == 0) {
          x0 = v;
          x1 = __longlong_as_double((long long)idx);
        } else {
          const int c0 = 2 * pr - 2;
          x0 = (v >= 0.0 && c0 < nb) ? s_a[c0 * Ri + rr] : 0.0;
          x1 = (v >= 0.0 && c0 + 1 < nb) ? s_a[(c0 + 1) * Ri + rr] : 0.0;
        }
        reinterpret_cast<double2*>(slot)[pr] = make_double2(x0, x1);
      }
      if (own_diag && lane < PW / 2) {
        const int rj = (int)(j - rb);
        const double x0 = 2 * lane < nb ? s_a[(2 * lane) * Ri + rj] : 0.0;
        const double x1 = 2 * lane + 1 < nb ? s_a[(2 * lane + 1) * Ri + rj] : 0.0;
        reinterpret_cast<double2*>(dslot)[lane] = make_double2(x0, x1);
      }
      asm volatile("fence.proxy.async.global;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const unsigned short mask = (unsigned short)((1u << CS) - 1u);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;\n" ::"r"(
                smem_u32(&recv[par][b][0])),
            "l"(slot), "r"((unsigned)(RECD * 8)), "r"(smem_u32(&mbar[par])), "h"(mask)
            : "memory");
        if (own_diag)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;\n" ::"r"(
                  smem_u32(&recv_diag[par][0])),
              "l"(dslot), "r"((unsigned)(PW * 8)), "r"(smem_u32(&mbar[par])), "h"(mask)
              : "memory");
      }
    }
    if (c <= 12) trace(8 + 8 * (c - 1) + 5);
    return idx;  // the CTA's candidate row (or INT64_MAX)
  };

  publish(0, p.j0, 0, false, 0);
  unsigned phase_bits = 0u;  // bit k: phase parity of mbar[k]

  for (int jj = 0; jj < nb; jj++) {
    const int64_t j = p.j0 + jj;
    const int par = jj & 1;
    if (warp == 0) {
      if (jj < 12) trace(8 + 8 * jj + 0);
      mbar_wait_parity(&mbar[par], (phase_bits >> par) & 1u);
      if (jj < 12) trace(8 + 8 * jj + 1);
      // decide from the local copies of every peer's record
      // first max over the CTA records: ranks hold ascending row ranges and each
      // record is its CTA's first max, so the smallest lane among equal maxima wins
      double rv = -1.0;
      long long ri = INT64_MAX;
      if (lane < CS) {
        rv = recv[par][lane][0];
        ri = __double_as_longlong(recv[par][lane][1]);
      }
      double vm = rv;
#pragma unroll
      for (int o = 16; o; o >>= 1) vm = fmax(vm, __shfl_xor_sync(0xffffffffu, vm, o));
      const unsigned win = __reduce_min_sync(0xffffffffu, (rv == vm && rv >= 0.0) ? (unsigned)lane : 32u);
      const double v = (win < 32u) ? vm : -1.0;
      const int64_t idx = (int64_t)__shfl_sync(0xffffffffu, ri, (int)(win & 31u));
      // rlra/_lu_cython.pyx:23-39: first max, whole-column colmax, zero pivot
      double colmax = v;
      const double cm_j = __shfl_sync(0xffffffffu, colmax_mine, jj);
      if (cm_j > colmax) colmax = cm_j;
      const int zero = (v <= ZERO_PIVOT_RTOL * colmax) ? 1 : 0;
      const int64_t prow = zero ? j : idx;
      // pivot row (post-swap row j): the winner's record, or row j itself
      double u = 0.0;
      if (lane < nb) u = zero ? recv_diag[par][lane] : recv[par][win & 31u][2 + lane];
      if (lane < PW) s_u[par][lane] = u;
      if (lane > jj && lane < nb && fabs(u) > colmax_mine) colmax_mine = fabs(u);
      if (lane == 0) {
        s_zero[par] = zero;
        s_prow[par] = prow;
        s_ipiv[jj] = prow;
        s_zf[jj] = zero;
      }
      if (lane == jj) s_rcp[par] = zero ? 0.0 : __drcp_rn(u);
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&mbar[par], tx_bytes);  // re-arm for step jj + 2
      phase_bits ^= 1u << par;
    }
    // all warps: previous step's bulk update done; decision visible
    __syncthreads();
    if (jj < 12) trace(8 + 8 * jj + 2);
    const int zero = s_zero[par];
    const int64_t prow = s_prow[par];
    const double* u = s_u[par];
    const int64_t r0 = j + 1 - rb;  // first local row strictly below the diagonal
    const bool last = (jj + 1 >= nb);
    // full-row swap (:40-48), lane-parallel in the warps that own rows j / prow
    // (the owner thread then updates that row, so __syncwarp is enough)
    if (!zero && prow != j) {
      if (j >= rb && j < re && (((int)(j - rb) % THREADS) >> 5) == warp && lane < nb)
        s_a[lane * Ri + (int)(j - rb)] = u[lane];
      if (prow >= rb && prow < re && (((int)(prow - rb) % THREADS) >> 5) == warp && lane < nb)
        s_a[lane * Ri + (int)(prow - rb)] = recv_diag[par][lane];
      __syncwarp();
    }
    if (!zero) {
      // look-ahead: multipliers and the NEXT column only
      const double ujj = u[jj], rcp = s_rcp[par];
      const double unext = last ? 0.0 : u[jj + 1];
      double* colj = s_a + jj * Ri;
      double* coln = s_a + (jj + 1) * Ri;
      for (int r = tid; r < nr; r += THREADS) {
        if (r < r0) continue;
        const double l = ieee_div_by(colj[r], ujj, rcp);  // IEEE division (:49-51)
        colj[r] = l;
        if (!last) coln[r] = sub_mul_nofma(coln[r], l, unext);  // (:52-55), column jj+1
      }
    } else {
      // zero pivot: zero the L column below the diagonal; no swap, no update (:36-39)
      for (int r = tid; r < nr; r += THREADS)
        if (r >= r0) s_a[jj * R + r] = 0.0;
    }
    if (jj < 12) trace(8 + 8 * jj + 3);
    if (!last) {
      const int64_t cand = publish(jj + 1, j + 1, par ^ 1, !zero, par);
      if (!zero) {
        // bulk of the step's update (columns jj+2 ..) by warps 1.., overlapping
        // the exchange -- warp 0 goes straight to the next decision; the two
        // rows published above were finished by warp 0
        const double* colj = s_a + jj * Ri;
        if (warp > 0) {
          for (int r = tid - 32; r < nr; r += THREADS - 32) {
            if (r < r0) continue;
            const int64_t i = rb + r;
            if (i == cand || i == j + 1) continue;
            const double l = colj[r];
            int c = jj + 2;
            for (; c + 8 <= nb; c += 8) {  // 8 independent chains per batch (ILP)
              double vv[8];
#pragma unroll
              for (int q = 0; q < 8; q++) vv[q] = s_a[(c + q) * Ri + r];
#pragma unroll
              for (int q = 0; q < 8; q++) vv[q] = sub_mul_nofma(vv[q], l, u[c + q]);  // (:52-55)
#pragma unroll
              for (int q = 0; q < 8; q++) s_a[(c + q) * Ri + r] = vv[q];
            }
            for (; c < nb; c++) {
              double* e = s_a + c * Ri + r;
              *e = sub_mul_nofma(*e, l, u[c]);
            }
          }
        }
      }
    }
  }
  __syncthreads();
  // ---- write the panel back (bulk copies; an odd last row directly)
  if (nr_bulk > 0) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid < nb) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                       p.a + cm(rb, p.j0 + tid, p.lda)),
                   "r"(smem_u32(s_a + tid * R)), "r"((unsigned)(nr_bulk * 8))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  }
  for (int c = 0; c < nb; c++)
    for (int r = nr_bulk + tid; r < nr; r += THREADS) p.a[cm(rb + r, p.j0 + c, p.lda)] = s_a[c * R + r];
  if (b == 0 && warp == 1) {
    if (lane < nb) {
      p.w.ipiv[p.j0 + lane] = s_ipiv[lane];
      p.w.zflag[p.j0 + lane] = s_zf[lane];
    }
    const int cnt = build_panel_perm(p.j0, nb, s_ipiv, s_prow_rows, s_prow_src, p.w);
    // the same net permutation applied to piv (rlra/_lu_cython.pyx:46-48)
    int64_t v0 = 0, v1 = 0;
    if (lane < cnt) v0 = p.piv[s_prow_src[lane]];
    if (lane + 32 < cnt) v1 = p.piv[s_prow_src[lane + 32]];
    __syncwarp();
    if (lane < cnt) p.piv[s_prow_rows[lane]] = v0;
    if (lane + 32 < cnt) p.piv[s_prow_rows[lane + 32]] = v1;
  }
  if (nr_bulk > 0 && tid < nb) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
  trace(126);
  cluster.sync();  // no CTA leaves while a peer may still push into it
  trace(127);
}

static constexpr int LU_PANEL_SMEM_BYTES = 200 * 1024;
// the cooperative-grid panel kernels of width 8 / 16 (static smem <= 3.8 KB)
// may take 223 KB: 148 x 1784 rows of a 16-wide panel cover C5's 262144-row
// sketches (a 200 KB cap forced 8-wide panels there: twice the launches)
static constexpr int LU_PANEL_SMEM_BYTES_NARROW = 223 * 1024;
static int64_t grid_rows_cap(int pw) {
  return (int64_t)((pw == 32 ? LU_PANEL_SMEM_BYTES : LU_PANEL_SMEM_BYTES_NARROW) / (pw * 8));
}

// Apply the panel's net row permutation to columns [0, j0) and [j0+nb, n).
// One warp per column: gather every touched row, then scatter.
__global__ void lu_laswp_kernel(double* a, int64_t lda, int64_t n, int64_t j0, int nb,
                                const int64_t* rows, const int64_t* src, const int* cnt_p, int64_t c_lo = 0) {
  const int cnt = *cnt_p;
  if (cnt == 0) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ncols = n - c_lo - nb;  // columns [c_lo, n) except the panel [j0, j0 + nb)
  for (int64_t w = warp; w < ncols; w += nwarps) {
    const int64_t c = c_lo + w < j0 ? c_lo + w : c_lo + w + nb;
    double* col = a + cm(0, c, lda);
    double v0 = 0.0, v1 = 0.0;
    if (lane < cnt) v0 = col[src[lane]];
    if (lane + 32 < cnt) v1 = col[src[lane + 32]];
    __syncwarp();
    if (lane < cnt) col[rows[lane]] = v0;
    if (lane + 32 < cnt) col[rows[lane + 32]] = v1;
  }
}

// U12 = L11^{-1} A12 by forward substitution in ascending step order, one WARP
// per column (lane s holds row j0+s; step t broadcasts x[t]); zero-pivot steps
// are skipped (the reference never applies them).  Same operation order per
// element as the reference: bit-exact.
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
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t c = c0 + blockIdx.x * wpb + (threadIdx.x >> 5); c < n; c += (int64_t)gridDim.x * wpb) {
    double* col = a + cm(j0, c, lda);
    double x = lane < nb ? col[lane] : 0.0;
    for (int t = 0; t < nb - 1; t++) {
      const double xt = __shfl_sync(0xffffffffu, x, t);
      if (!z[t] && lane > t && lane < nb) x = sub_mul_nofma(x, L[lane][t], xt);
    }
    if (lane > 0 && lane < nb) col[lane] = x;
  }
}

// A22 -= L21 * U12 with the panel's steps applied in ascending order, DMUL+DSUB.
constexpr int UPD_TM = 64, UPD_TN = 64;
__global__ void __launch_bounds__(256, 4)
lu_update_kernel(double* a, int64_t lda, int64_t j0, int nb, int64_t r0, int64_t m, int64_t c0,
                 int64_t n, const int* zflag, const double* u = nullptr, int64_t ldu = 0) {
  if (u == nullptr) {  // U12 in the same matrix (rows j0 .. j0 + nb); else a separate (virtual-row) operand
    u = a;
    ldu = lda;
  }
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
    Us[t][c] = gc < n ? u[cm(j0 + t, gc, ldu)] : 0.0;
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
size_t getrf_full_state_bytes();  // getrf_full.cu
static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct LuLayout {
  size_t off[14];
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
  take(13, std::max((size_t)(2 * 16 * (2 + LU_NB) + 2 * LU_NB) * sizeof(double), getrf_full_state_bytes()));
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
  w.recg = reinterpret_cast<double*>(base + L.off[13]);
  return w;
}

int count_nonzero_diag(const double* a, int64_t lda, int64_t r, int64_t* out_dev, cudaStream_t st) {
  count_nonzero_diag_kernel<<<1, 256, 0, st>>>(a, lda, r, out_dev);
  RLRA_LAUNCHED();
  return 0;
}

int fill_iota(int64_t* p, int64_t m, cudaStream_t st) {
  if (m <= 0) return 0;
  int blocks = (int)std::min<int64_t>(ceil_div(m, 256), 4096);
  iota_kernel<<<blocks, 256, 0, st>>>(p, m);
  RLRA_LAUNCHED();
  return 0;
}

bool getrf_full_eligible(int64_t m, int64_t n, int cluster_max);
int getrf_full(double* a, int64_t lda, int64_t m, int64_t n, int64_t* piv, int64_t* ipiv, int* zflag, double* recg,
               cudaStream_t st);
int getrf_full_wide(double* a, int64_t lda, int64_t m, int64_t n, int64_t* piv, int64_t* ipiv, int* zflag, double* recg,
               cudaStream_t st);  // 384 threads per CTA, m <= getrf_full_wide_rows()
int64_t getrf_full_wide_rows();

unsigned long long* g_lu_trace = nullptr;  // set by rlra_b200_debug_lu_trace (tools only)
static unsigned long long* lu_trace_buffer() { return g_lu_trace; }

// Largest thread-block cluster (<= 16, non-portable above 8) that can hold one
// 512-thread CTA with the full panel shared memory per SM; 1 if none.
static int lu_max_cluster() {
  static int cached[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  if (cached[dev & 63]) return cached[dev & 63];
  int best = 1;
  const void* kern = (const void*)lu_panel_cluster_kernel<16, 512>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, LU_PANEL_SMEM_BYTES) ==
          cudaSuccess &&
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
    for (int cs = 16; cs >= 2; cs /= 2) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = LU_PANEL_SMEM_BYTES;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) == cudaSuccess && nclusters > 0) {
        best = cs;
        break;
      }
    }
  }
  cudaGetLastError();
  cached[dev & 63] = best;
  return best;
}

// Per-device auxiliary stream for the look-ahead trailing updates (NULL when
// disabled with RLRA_B200_LU_LOOKAHEAD=0).
static cudaStream_t lu_aux_stream() {
  static std::mutex mu;
  static cudaStream_t streams[64];
  static bool init[64];
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = getenv("RLRA_B200_LU_LOOKAHEAD");
    enabled = (e && e[0] == '0') ? 0 : 1;
  }
  if (!enabled) return nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!init[dev & 63]) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&streams[dev & 63], cudaStreamNonBlocking, lo) != cudaSuccess)
      streams[dev & 63] = nullptr;
    cudaGetLastError();
    init[dev & 63] = true;
  }
  return streams[dev & 63];
}

static int lu_prepare_kernel(const void* kern, int smem_bytes = LU_PANEL_SMEM_BYTES) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  RLRA_CHECK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({dev, kern})) return 0;
  RLRA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaGetLastError();
  done.insert({dev, kern});
  return 0;
}

// Packed in-place GEPP: on return `a` holds unit-L multipliers below the
// diagonal and U on/above it, `piv` (caller-preloaded, typically 0..m-1) is
// permuted like the reference's piv (rlra/_lu_cython.pyx:14, rlra/kernels.py:48),
// and *nonzero_diag_dev (device int64) receives count_nonzero(diag(U)).
// ------------------------------------------------------------------ distributed primitives
// The row-sharded exact GEPP (distributed.dist_getrf_) runs the blocked
// algorithm with every 32-column block's panel all-gathered: each rank factors
// the gathered m x 32 panel redundantly (identical pivots everywhere), U12
// comes from the block's 32 gathered rows, and each rank updates only its own
// rows.  Every element sees the reference's rounding sequence, exactly as in
// getrf(): the result is bit-identical to the one-GPU kernel.

__global__ void add_nonzero_diag_kernel(const double* a, int64_t lda, int64_t j0, int r, int64_t* out) {
  __shared__ int s[32];
  int cnt = 0;
  for (int i = threadIdx.x; i < r; i += blockDim.x) cnt += (a[cm(j0 + i, j0 + i, lda)] != 0.0);
#pragma unroll
  for (int off = 16; off; off >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, off);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) tot += s[w];
    *out += tot;
  }
}

// Factor the 32-column block [j0, j0 + nbo) of an m-row matrix in place: its
// panels, their interchanges restricted to the block's columns, the inner
// U12 / updates.  `a` is the VIRTUAL base (only columns [j0, j0 + nbo) are
// touched -- a gathered panel passed as panel - j0 * lda); rows < j0 are the
// rows above (they enter the zero-pivot column maxima only); piv (int64[m]) is
// permuted; zflag_out[j0 .. j0 + nbo) receives the zero-pivot flags,
// ipiv_out[j0 .. j0 + nbo) the pivot row of each step (the interchange
// sequence j <-> ipiv[j]) and *nonzero_out accumulates count_nonzero(diag(U)).  ws: a getrf
// workspace for (m, >= j0 + nbo) columns.
int getrf_block(double* a, int64_t lda, int64_t m, int64_t j0, int nbo, int64_t* piv, int* zflag_out,
                int64_t* ipiv_out, int64_t* nonzero_out, void* ws, size_t ws_bytes, cudaStream_t st) {
  RLRA_REQUIRE(m >= 1 && j0 >= 0 && nbo >= 1 && nbo <= LU_NB && j0 + nbo <= m && lda >= m,
               "getrf_block: bad block (m=%lld j0=%lld nbo=%d)", (long long)m, (long long)j0, nbo);
  const int sms = device_info().sm_count;
  LuLayout L = lu_layout(j0 + nbo, sms);
  RLRA_REQUIRE(ws != nullptr && ws_bytes >= L.total, "getrf_block: workspace too small (%zu < %zu)", ws_bytes,
               L.total);
  LuWork w = lu_work(ws, j0 + nbo, sms);
  RLRA_CHECK_CUDA(cudaMemsetAsync(w.bar, 0, 2 * sizeof(unsigned), st));
  auto rows_cap = [](int pw) { return (int64_t)(LU_PANEL_SMEM_BYTES / (pw * 8)); };
  const int cmax = lu_max_cluster();
  const bool use_cluster = cmax > 1 && m <= cmax * rows_cap(16);
  int pw;
  if (use_cluster) pw = (m <= cmax * rows_cap(32)) ? 32 : 16;
  else pw = (m <= sms * grid_rows_cap(32)) ? 32 : (m <= sms * grid_rows_cap(16) ? 16 : 8);
  RLRA_REQUIRE(m <= sms * grid_rows_cap(8), "getrf_block: m = %lld exceeds the panel capacity", (long long)m);
  const void* kern = use_cluster
      ? (pw == 32 ? (const void*)lu_panel_cluster_kernel<32, 512> : (const void*)lu_panel_cluster_kernel<16, 512>)
      : (pw == 32 ? (const void*)lu_panel_smem_kernel<32, 512>
                  : pw == 16 ? (const void*)lu_panel_smem_kernel<16, 512> : (const void*)lu_panel_smem_kernel<8, 512>);
  const int smem_cap = use_cluster || pw == 32 ? LU_PANEL_SMEM_BYTES : LU_PANEL_SMEM_BYTES_NARROW;
  auto cap = [&](int w_) { return use_cluster ? rows_cap(w_) : grid_rows_cap(w_); };
  if (lu_prepare_kernel(kern, smem_cap)) return -1;
  unsigned bar_base = 0;
  const int64_t ce = j0 + nbo;
  for (int64_t jp = j0; jp < ce; jp += pw) {
    const int nb = (int)std::min<int64_t>(pw, ce - jp);
    const int64_t active = m - jp;
    PanelArgs pa;
    pa.a = a; pa.lda = lda; pa.m = m; pa.n = ce; pa.j0 = jp; pa.nb = nb;
    pa.piv = piv;
    pa.w = w;
    pa.bar_base = bar_base;
    pa.trace = lu_trace_buffer();
    const int limit = use_cluster ? cmax : sms;
    const int64_t target = std::min<int64_t>(cap(pw), 512);
    int G = (int)std::min<int64_t>(limit, ceil_div(active, target));
    G = (int)std::max<int64_t>(G, ceil_div(active, cap(pw)));
    pa.rows_per_cta = ceil_div(active, G);
    pa.rows_per_cta += pa.rows_per_cta & 1;
    pa.above_per_cta = std::max<int64_t>(1, ceil_div(jp, G));
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
      RLRA_CHECK_CUDA(cudaLaunchCooperativeKernel(kern, dim3(G), dim3(512), args, smem, st));
      bar_base += (unsigned)G * nb;
    }
    note_launch();
    if (nbo > nb) {  // the panel's interchanges on the block's other columns only
      const int64_t ncols = nbo - nb;
      const int blocks = (int)std::min<int64_t>(ceil_div(ncols * 32, 256), 2048);
      lu_laswp_kernel<<<blocks, 256, 0, st>>>(a, lda, ce, jp, nb, w.perm_rows, w.perm_src, w.perm_cnt, j0);
      RLRA_LAUNCHED();
    }
    const int64_t c0 = jp + nb;
    if (c0 < ce) {
      lu_trsm_kernel<<<(unsigned)ceil_div(ce - c0, 4), 128, 0, st>>>(a, lda, jp, nb, c0, ce, w.zflag);
      RLRA_LAUNCHED();
      if (c0 < m) {
        dim3 grid((unsigned)ceil_div(m - c0, UPD_TM), (unsigned)ceil_div(ce - c0, UPD_TN));
        lu_update_kernel<<<grid, 256, 0, st>>>(a, lda, jp, nb, c0, m, c0, ce, w.zflag);
        RLRA_LAUNCHED();
      }
    }
  }
  if (zflag_out)
    RLRA_CHECK_CUDA(cudaMemcpyAsync(zflag_out + j0, w.zflag + j0, nbo * sizeof(int), cudaMemcpyDeviceToDevice, st));
  if (ipiv_out)  // pivot row chosen at each step (== j without a swap): the block's interchange sequence
    RLRA_CHECK_CUDA(cudaMemcpyAsync(ipiv_out + j0, w.ipiv + j0, nbo * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  if (nonzero_out) {
    add_nonzero_diag_kernel<<<1, 256, 0, st>>>(a, lda, j0, nbo, nonzero_out);
    RLRA_LAUNCHED();
  }
  return 0;
}

// U12 = L11^{-1} A12 (bit-exact forward substitution) on rows [j0, j0 + nb) of
// a virtual-row operand (the block's gathered rows passed as rows - j0).
int lu_trsm_rows(double* a, int64_t lda, int64_t j0, int nb, int64_t c0, int64_t c1, const int* zflag,
                 cudaStream_t st) {
  RLRA_REQUIRE(nb >= 1 && nb <= LU_NB && c1 >= c0, "lu_trsm_rows: bad arguments");
  if (c1 == c0) return 0;
  const int blocks = (int)std::min<int64_t>(ceil_div(c1 - c0, 4), 4096);
  lu_trsm_kernel<<<blocks, 128, 0, st>>>(a, lda, j0, nb, c0, c1, zflag);
  RLRA_LAUNCHED();
  return 0;
}

// A(r0:m, c0:c1) -= L(r0:m, j0:j0+nb) U(j0:j0+nb, c0:c1), L in `a`, U in `u`
// (virtual rows), bit-exact (rank-1 terms ascending, DMUL then DSUB).
int lu_update_split(double* a, int64_t lda, const double* u, int64_t ldu, int64_t j0, int nb, int64_t r0, int64_t m,
                    int64_t c0, int64_t c1, const int* zflag, cudaStream_t st) {
  RLRA_REQUIRE(nb >= 1 && nb <= LU_NB, "lu_update_split: bad nb");
  if (r0 >= m || c1 <= c0) return 0;
  dim3 grid((unsigned)ceil_div(m - r0, UPD_TM), (unsigned)ceil_div(c1 - c0, UPD_TN));
  lu_update_kernel<<<grid, 256, 0, st>>>(a, lda, j0, nb, r0, m, c0, c1, zflag, u, ldu);
  RLRA_LAUNCHED();
  return 0;
}

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
  // Panel placement.  Up to 16 x rows_cap rows: one thread-block cluster (DSMEM
  // + hardware cluster barrier).  Beyond: one CTA per SM with a global-memory
  // grid barrier.  Panel width 32 when every active row of a 32-wide panel fits
  // in shared memory, else 16 / 8 inner panels inside 32-wide outer blocks
  // (same rounding sequence per element: still bit-exact).
  auto rows_cap = [](int pw) { return (int64_t)(LU_PANEL_SMEM_BYTES / (pw * 8)); };
  const int cmax = lu_max_cluster();
  if (getrf_full_eligible(m, n, cmax)) {
    // narrow sketch: the whole factorization in one cooperative launch (getrf_full.cu)
    const int rc = m <= getrf_full_wide_rows() ? getrf_full_wide(a, lda, m, n, piv, w.ipiv, w.zflag, w.recg, st)
                                               : getrf_full(a, lda, m, n, piv, w.ipiv, w.zflag, w.recg, st);
    if (rc < 0) return -1;
    if (rc == 0) {
      if (nonzero_diag_dev) {
        count_nonzero_diag_kernel<<<1, 256, 0, st>>>(a, lda, r, nonzero_diag_dev);
        RLRA_LAUNCHED();
      }
      if (zflag_out && r > 0)
        RLRA_CHECK_CUDA(cudaMemcpyAsync(zflag_out, w.zflag, r * sizeof(int), cudaMemcpyDeviceToDevice, st));
      return 0;
    }
    // rc == 1: no room for helper clusters next to the panel cluster -> blocked path
  }
  const bool use_cluster = cmax > 1 && m <= cmax * rows_cap(16);
  int pw;
  if (use_cluster) pw = (m <= cmax * rows_cap(32)) ? 32 : 16;
  else pw = (m <= sms * grid_rows_cap(32)) ? 32 : (m <= sms * grid_rows_cap(16) ? 16 : 8);
  RLRA_REQUIRE(m <= sms * grid_rows_cap(8), "getrf: m = %lld exceeds the panel capacity", (long long)m);
  const void* kern = use_cluster
      ? (pw == 32 ? (const void*)lu_panel_cluster_kernel<32, 512> : (const void*)lu_panel_cluster_kernel<16, 512>)
      : (pw == 32 ? (const void*)lu_panel_smem_kernel<32, 512>
                  : pw == 16 ? (const void*)lu_panel_smem_kernel<16, 512> : (const void*)lu_panel_smem_kernel<8, 512>);
  const int smem_cap = use_cluster || pw == 32 ? LU_PANEL_SMEM_BYTES : LU_PANEL_SMEM_BYTES_NARROW;
  auto cap = [&](int w_) { return use_cluster ? rows_cap(w_) : grid_rows_cap(w_); };
  if (lu_prepare_kernel(kern, smem_cap)) return -1;
  unsigned bar_base = 0;
  // Look-ahead: after block b's panels, only the NEXT block's columns get the
  // trailing update on `st` (narrow); the rest (wide) runs on an auxiliary
  // stream while block b+1's panel factorization -- a 16-SM cluster -- runs on
  // `st`, joined before b+1's first row interchange touches those columns.
  // Every element still receives its rank-1 terms in ascending step order.
  cudaStream_t aux = lu_aux_stream();
  cudaEvent_t ev_narrow = nullptr, ev_wide = nullptr;
  if (aux) {
    RLRA_CHECK_CUDA(cudaEventCreateWithFlags(&ev_narrow, cudaEventDisableTiming));
    RLRA_CHECK_CUDA(cudaEventCreateWithFlags(&ev_wide, cudaEventDisableTiming));
  }
  struct Wide {
    bool pending = false, submitted = false;
    int64_t jo = 0, c0 = 0, ce = 0;
    int nbo = 0;
  } wide;
  auto trailing = [&](int64_t jo_, int nbo_, int64_t ce_, int64_t c0_, int64_t c1_, cudaStream_t s_) -> int {
    int blocks = (int)std::min<int64_t>(ceil_div(c1_ - c0_, 4), 4096);
    lu_trsm_kernel<<<blocks, 128, 0, s_>>>(a, lda, jo_, nbo_, c0_, c1_, w.zflag);
    RLRA_LAUNCHED();
    if (ce_ < m) {
      dim3 grid((unsigned)ceil_div(m - ce_, UPD_TM), (unsigned)ceil_div(c1_ - c0_, UPD_TN));
      lu_update_kernel<<<grid, 256, 0, s_>>>(a, lda, jo_, nbo_, ce_, m, c0_, c1_, w.zflag);
      RLRA_LAUNCHED();
    }
    return 0;
  };
  auto submit_wide = [&]() -> int {
    if (!wide.pending || wide.submitted) return 0;
    RLRA_CHECK_CUDA(cudaStreamWaitEvent(aux, ev_narrow, 0));
    if (trailing(wide.jo, wide.nbo, wide.ce, wide.c0, n, aux)) return -1;
    RLRA_CHECK_CUDA(cudaEventRecord(ev_wide, aux));
    wide.submitted = true;
    return 0;
  };
  auto join_wide = [&]() -> int {
    if (!wide.pending) return 0;
    if (submit_wide()) return -1;
    RLRA_CHECK_CUDA(cudaStreamWaitEvent(st, ev_wide, 0));
    wide.pending = wide.submitted = false;
    return 0;
  };
  for (int64_t jo = 0; jo < r; jo += LU_NB) {
    const int nbo = (int)std::min<int64_t>(LU_NB, r - jo);
    const int64_t ce = jo + nbo;
    for (int64_t j0 = jo; j0 < ce; j0 += pw) {
      const int nb = (int)std::min<int64_t>(pw, ce - j0);
      const int64_t active = m - j0;
      PanelArgs pa;
      pa.a = a; pa.lda = lda; pa.m = m; pa.n = n; pa.j0 = j0; pa.nb = nb;
      pa.piv = piv;
      pa.w = w;
      pa.bar_base = bar_base;
      pa.trace = lu_trace_buffer();
      const int limit = use_cluster ? cmax : sms;
      // about one row per thread, never more rows than shared memory holds
      const int64_t target = std::min<int64_t>(cap(pw), 512);
      int G = (int)std::min<int64_t>(limit, ceil_div(active, target));
      G = (int)std::max<int64_t>(G, ceil_div(active, cap(pw)));
      pa.rows_per_cta = ceil_div(active, G);
      pa.rows_per_cta += pa.rows_per_cta & 1;  // even: 16-byte aligned bulk copies of panel columns
      pa.above_per_cta = std::max<int64_t>(1, ceil_div(j0, G));
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
        RLRA_CHECK_CUDA(cudaLaunchCooperativeKernel(kern, dim3(G), dim3(512), args, smem, st));
        bar_base += (unsigned)G * nb;
      }
      note_launch();
      // the previous block's wide update overlaps this panel; join before the
      // interchanges reach its columns
      if (join_wide()) return -1;
      if (n > nb) {
        int64_t ncols = n - nb;
        int blocks = (int)std::min<int64_t>(ceil_div(ncols * 32, 256), 2048);
        lu_laswp_kernel<<<blocks, 256, 0, st>>>(a, lda, n, j0, nb, w.perm_rows, w.perm_src, w.perm_cnt);
        RLRA_LAUNCHED();
      }
      const int64_t c0 = j0 + nb;
      if (c0 < ce) {  // inner update, restricted to the outer block's columns
        lu_trsm_kernel<<<(unsigned)ceil_div(ce - c0, 4), 128, 0, st>>>(a, lda, j0, nb, c0, ce, w.zflag);
        RLRA_LAUNCHED();
        if (c0 < m) {
          dim3 grid((unsigned)ceil_div(m - c0, UPD_TM), (unsigned)ceil_div(ce - c0, UPD_TN));
          lu_update_kernel<<<grid, 256, 0, st>>>(a, lda, j0, nb, c0, m, c0, ce, w.zflag);
          RLRA_LAUNCHED();
        }
      }
    }
    if (ce < n) {  // outer trailing update with the whole 32-column block
      const int64_t ce2 = aux ? std::min<int64_t>(n, ce + LU_NB) : n;
      if (trailing(jo, nbo, ce, ce, ce2, st)) return -1;  // narrow: the next block's columns
      if (ce2 < n) {                                      // wide: deferred past the next panel launch
        RLRA_CHECK_CUDA(cudaEventRecord(ev_narrow, st));
        wide.pending = true;
        wide.submitted = false;
        wide.jo = jo;
        wide.nbo = nbo;
        wide.ce = ce;
        wide.c0 = ce2;
      }
    }
  }
  if (join_wide()) return -1;
  if (ev_narrow) cudaEventDestroy(ev_narrow);
  if (ev_wide) cudaEventDestroy(ev_wide);
  if (nonzero_diag_dev) {
    count_nonzero_diag_kernel<<<1, 256, 0, st>>>(a, lda, r, nonzero_diag_dev);
    RLRA_LAUNCHED();
  }
  if (zflag_out && r > 0)
    RLRA_CHECK_CUDA(cudaMemcpyAsync(zflag_out, w.zflag, r * sizeof(int), cudaMemcpyDeviceToDevice, st));
  return 0;
}

}  // namespace rlra
