// K1/K2 pass GEMMs as FP64 emulation on the int8 tensor cores (Ozaki scheme
// II: integer scaling + Chinese remaindering), the B200-first replacement of
// the DMMA pass for the two big products of every PowerLU pass
//   NN  C (m x l) = A   B      (rlra/accessors.py:27-28, A.matmul)
//   TN  C (n x l) = A^T B      (rlra/accessors.py:30-31, A.rmatmul)
// B200 runs FP64 at ~37 TFLOP/s (DMMA) but int8 MMA at ~4.5 POPS, so the
// product is computed exactly in integers:
//   1. A'' = rint(2^eA A) with one power-of-two scale such that every row and
//      column 2-norm of A'' is < 2^PA; B'' = rint(2^eB[j] B[:, j]) per column,
//      ||B''_j|| < 2^PB.  By Cauchy-Schwarz |(A''B'')_ij| < 2^(PA+PB) < M/2.
//   2. For NMOD pairwise-coprime moduli m_l <= 249 (M = prod m_l ~ 2^109.5 for
//      14) the residues A''_l = A'' mod m_l, B''_l in [-127, 127] are int8 and
//      C_l = A''_l B''_l is EXACT in the int32 accumulators (K <= 133144).
//   3. t_l = C_l mod m_l (uint8), and A''B'' = CRT(t_1..t_NMOD) in (-M/2, M/2)
//      is reconstructed exactly in 128-bit integers, rounded once to double
//      and unscaled by 2^-(eA+eB[j]).
// The only roundings are the scaling steps and the final conversion: with
// N_A = max over all row AND column 2-norms of A (one scale for both
// orientations), for C = A B
//   |C_ij - (AB)_ij| <= 2^-PA sqrt(K) N_A ||B_j|| + 2^-PB sqrt(K) ||A_i|| ||B_j||
//                       + 2^-52 ||A_i|| ||B_j||
// (K = contraction length; A_i the i-th row of op(A)).  This is NORMWISE in
// N_A, not per row: a row i with ||A_i|| << N_A gets a larger relative error
// than DGEMM would give it.  The dynamic-range guard (oz_guard below,
// rlra_b200_oz_guard) therefore admits an orientation only when
//   rho = N_A / min_i ||A_i|| <= T(K) = 2 (K - 2) / sqrt(K) - 2
// (min over the non-zero rows of op(A)), which makes the bound above at most
// K u ||A_i|| ||B_j||, u = 2^-53 -- the classical DGEMM bound (every inner
// product of length K in floating point).  Inputs that fail it (graded rows /
// columns, non-finite or out-of-range entries) take the FP64 DMMA GEMM
// instead (ops.OzPrep / ops.OzBlocked route them).  Results are exact
// functions of the inputs (tiling- and order-independent, so bitwise
// deterministic).
//
// Data layout.  The residues of A are written once per PowerLU call into
// 128 x 128-byte tiles (16 KB), tile (jb, ib) holding A''[ib*128 .. +128,
// jb*128 .. +128] with the ROW index i contiguous: row r = column j, byte c =
// row i, in the 128-byte-swizzled image the tensor core reads (16-byte chunk
// c/16 stored at chunk (c/16) ^ (r % 8)).  The TN product reads a tile as a
// K-major operand (K = i), the NN product reads the SAME bytes as an MN-major
// operand (M = i, K = j), so one residue set serves both orientations.  Tiles
// are plain contiguous 16 KB blocks moved with 1-D bulk copies (no tensor map).
//
// GEMM kernel: persistent, 1 CTA / SM, warp-specialized: warp 0 = bulk-copy
// producer, warp 1 = tcgen05.mma issuer (one thread) + TMEM owner, warps 2-5 =
// epilogue (tcgen05.ld -> mod m_l -> uint8).  A unit of work is (modulus l,
// 256-row block, column group); two M=128 MMAs share each B tile; int32
// accumulators live in TMEM (2 x N_g <= 512 columns).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace rlra {
namespace oz {

constexpr int kMaxMod = 16;
constexpr int kModuli[kMaxMod] = {249, 247, 245, 244, 241, 239, 233, 229,
                                  227, 223, 211, 199, 197, 193, 191, 181};
constexpr int kTile = 128;                 // rows / bytes per residue tile
constexpr int kTileBytes = kTile * kTile;  // 16 KB
constexpr int kMaxK = 133144;              // 127^2 * K < 2^31
constexpr int kStages = 3;
constexpr int kGemmThreads = 192;

__host__ __device__ constexpr int pow2mod(int e, int m) {
  int r = 1 % m;
  for (int i = 0; i < e; ++i) r = (r * 2) % m;
  return r;
}

typedef unsigned __int128 u128;

constexpr int kCrtLimbs = 7;  // 7 x 20 bits >= 125 bits (M for 16 moduli)

struct Crt {
  uint64_t M_lo, M_hi;        // M = prod m_l
  uint64_t H_lo, H_hi;        // floor(M / 2)
  uint64_t md_lo[kMaxMod];    // M / m_l
  uint64_t md_hi[kMaxMod];
  int y[kMaxMod];             // (M / m_l)^{-1} mod m_l
  int m[kMaxMod];
  float inv_m[kMaxMod];
  uint32_t limb[kCrtLimbs][kMaxMod];  // 20-bit limbs of M / m_l
  uint32_t d28[4][kMaxMod];           // 28-bit limbs of M / m_l (nmod <= 14: M < 2^112)
  uint32_t M28[4];                    // 28-bit limbs of M
  uint32_t H28[4];                    // 28-bit limbs of floor(M / 2)
  double inv_M;                     // ~1 / M
  int nmod;
};

// Precision split of the 128-bit budget: PA + PB = floor(log2 M) - 2, each <= 55.
struct Budget {
  int pa, pb;
};
static Budget budget(int nmod) {
  long double lg = 0;
  for (int l = 0; l < nmod; ++l) lg += std::log2((long double)kModuli[l]);
  int tot = (int)std::floor(lg) - 2;
  Budget b;
  b.pa = tot - tot / 2;
  b.pb = tot / 2;
  if (b.pa > 55) b.pa = 55;
  if (b.pb > 55) b.pb = 55;
  return b;
}

static Crt make_crt(int nmod) {
  Crt c{};
  u128 M = 1;
  for (int l = 0; l < nmod; ++l) M *= (u128)kModuli[l];
  c.M_lo = (uint64_t)M;
  c.M_hi = (uint64_t)(M >> 64);
  u128 H = M >> 1;
  c.H_lo = (uint64_t)H;
  c.H_hi = (uint64_t)(H >> 64);
  for (int l = 0; l < nmod; ++l) {
    const int m = kModuli[l];
    u128 md = M / (u128)m;
    c.md_lo[l] = (uint64_t)md;
    c.md_hi[l] = (uint64_t)(md >> 64);
    int r = (int)(md % (u128)m);
    int inv = 0;
    for (int y = 1; y < m; ++y)
      if ((r * y) % m == 1) {
        inv = y;
        break;
      }
    c.y[l] = inv;
    c.m[l] = m;
    c.inv_m[l] = 1.0f / (float)m;
    for (int q = 0; q < kCrtLimbs; ++q) c.limb[q][l] = (uint32_t)((md >> (20 * q)) & 0xFFFFF);
    for (int q = 0; q < 4; ++q) c.d28[q][l] = (uint32_t)((md >> (28 * q)) & 0xFFFFFFF);
  }
  for (int q = 0; q < 4; ++q) c.M28[q] = (uint32_t)((M >> (28 * q)) & 0xFFFFFFF);
  for (int q = 0; q < 4; ++q) c.H28[q] = (uint32_t)((H >> (28 * q)) & 0xFFFFFFF);
  c.inv_M = 1.0 / (double)M;
  c.nmod = nmod;
  return c;
}

// ----------------------------------------------------------------- residues
// x = rint(v * 2^e), |x| < 2^55, as four float parts x = p3 2^42 + p2 2^28 +
// p1 2^14 + p0 with p0..p2 in [0, 2^14) and p3 signed (two's complement split).
// Residue modulo m: v = p3 (2^42 mod m) + p2 (2^28 mod m) + p1 (2^14 mod m) + p0
// (exact in fp32, |v| < 2^24), q ~ rint(v / m), r = v - q m exact in
// [-m/2-1, m/2+1] (|r| <= 126), returned as the low byte of the float r + 1.5*2^23.
__device__ __forceinline__ unsigned pack4(unsigned b0, unsigned b1, unsigned b2, unsigned b3) {
  return __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
}

// ---- the same arithmetic on PAIRS of values with the packed fp32x2 pipe
// (FFMA2 / FADD2, sm_100): two values per instruction, half the instruction
// count of scalar fp32 -- the residue kernel is issue-bound, not HBM-bound,
// without it.
typedef unsigned long long f2_t;  // (lo = element 2i, hi = element 2i+1)
__device__ __forceinline__ f2_t f2_ffma(f2_t a, f2_t b, f2_t c) {
  f2_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2_t f2_fadd(f2_t a, f2_t b) {
  f2_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2_t f2_bits(unsigned lo, unsigned hi) { return ((f2_t)hi << 32) | lo; }
__device__ __forceinline__ f2_t f2_dup(float v) { return f2_bits(__float_as_uint(v), __float_as_uint(v)); }

struct Parts2 {
  f2_t p0, p1, p2, p3;
};
__device__ __forceinline__ Parts2 split_parts2(double va, double vb, double scale) {
  const long long xa = __double2ll_rn(va * scale), xb = __double2ll_rn(vb * scale);
  const unsigned la = (unsigned)xa, lb = (unsigned)xb;
  const unsigned ha = (unsigned)(xa >> 28), hb = (unsigned)(xb >> 28);
  const f2_t m23 = f2_dup(-8388608.0f);
  Parts2 p;
  p.p0 = f2_fadd(f2_bits(0x4B000000 | (la & 0x3FFF), 0x4B000000 | (lb & 0x3FFF)), m23);
  p.p1 = f2_fadd(f2_bits(0x4B000000 | ((la >> 14) & 0x3FFF), 0x4B000000 | ((lb >> 14) & 0x3FFF)), m23);
  p.p2 = f2_fadd(f2_bits(0x4B000000 | (ha & 0x3FFF), 0x4B000000 | (hb & 0x3FFF)), m23);
  p.p3 = f2_fadd(f2_bits(0x4B400000 + ((int)ha >> 14), 0x4B400000 + ((int)hb >> 14)), f2_dup(-12582912.0f));
  return p;
}

// residue_byte<L> of both values of a pair: the two floats' low bytes
template <int L>
__device__ __forceinline__ f2_t residue_pair(const Parts2& x) {
  constexpr int m = kModuli[L];
  const f2_t c1 = f2_dup((float)pow2mod(14, m)), c2 = f2_dup((float)pow2mod(28, m));
  const f2_t c3 = f2_dup((float)pow2mod(42, m)), inv = f2_dup(1.0f / (float)m);
  const f2_t big = f2_dup(12582912.0f), nbig = f2_dup(-12582912.0f), nm = f2_dup(-(float)m);
  const f2_t v = f2_ffma(x.p3, c3, f2_ffma(x.p2, c2, f2_ffma(x.p1, c1, x.p0)));  // exact, |v| < 2^24
  const f2_t q = f2_fadd(f2_ffma(v, inv, big), nbig);                             // ~rint(v / m)
  const f2_t r = f2_ffma(q, nm, v);                                               // exact
  return f2_fadd(r, big);                                                         // low bytes = r
}

template <int N>
struct Bytes;
template <>
struct Bytes<16> {
  typedef uint4 T;
};
template <>
struct Bytes<8> {
  typedef uint2 T;
};

// N (8 or 16) consecutive values (N/2 pairs) -> N residue bytes for modulus L.
template <int L, int N>
__device__ __forceinline__ typename Bytes<N>::T residue_chunk(const Parts2 (&x)[N / 2]) {
  unsigned w[N / 4];
#pragma unroll
  for (int q = 0; q < N / 4; ++q) {
    const f2_t a = residue_pair<L>(x[2 * q]), b = residue_pair<L>(x[2 * q + 1]);
    w[q] = pack4((unsigned)a, (unsigned)(a >> 32), (unsigned)b, (unsigned)(b >> 32));
  }
  typename Bytes<N>::T o;
  if constexpr (N == 16) {
    o.x = w[0]; o.y = w[1]; o.z = w[2]; o.w = w[3];
  } else {
    o.x = w[0]; o.y = w[1];
  }
  return o;
}

template <int L, int NMOD, int N>
struct ChunkWriter {
  __device__ __forceinline__ static void run(const Parts2 (&x)[N / 2], int8_t* base, size_t mod_stride) {
    *reinterpret_cast<typename Bytes<N>::T*>(base + (size_t)L * mod_stride) = residue_chunk<L, N>(x);
    ChunkWriter<L + 1, NMOD, N>::run(x, base, mod_stride);
  }
};
template <int NMOD, int N>
struct ChunkWriter<NMOD, NMOD, N> {
  __device__ __forceinline__ static void run(const Parts2 (&)[N / 2], int8_t*, size_t) {}
};

__device__ __forceinline__ int swz(int r, int c) {  // byte offset of 16-byte chunk c of row r
  return r * kTile + (((c ^ (r & 7)) & 7) << 4);
}

// Residues of A: one CTA per 128 x 128 block of A (tile (jb, ib)); each thread
// converts 8 x 8 consecutive rows of one column (half swizzle chunks), with the
// next group's loads in flight while the current one is converted.
template <int NMOD>
__global__ void __launch_bounds__(256, 3) residue_a_kernel(const double* __restrict__ a, int64_t lda, int64_t m,
                                                           int64_t n, const int* __restrict__ e_a,
                                                           int8_t* __restrict__ tiles, int64_t nib, int64_t njb,
                                                           int64_t jb0) {
  const int64_t ib = blockIdx.x, jb = blockIdx.y + jb0;
  const double scale = scalbn(1.0, e_a[0]);
  const size_t mod_stride = (size_t)njb * nib * kTileBytes;
  int8_t* tile = tiles + ((size_t)jb * nib + ib) * kTileBytes;
  const bool full = (ib + 1) * kTile <= m && (jb + 1) * kTile <= n;
  double cur[8], nxt[8];
  auto load = [&](int s, double (&d)[8]) {
    const int ch = threadIdx.x + 256 * s;  // 2048 half chunks per tile
    const int r = ch >> 4, h = ch & 15;
    const int64_t j = jb * kTile + r;
    const int64_t i0 = ib * kTile + h * 8;
    const double* src = a + i0 + j * lda;
    if (full) {
#pragma unroll
      for (int t = 0; t < 8; ++t) d[t] = __ldcs(src + t);
    } else {
#pragma unroll
      for (int t = 0; t < 8; ++t) d[t] = (j < n && i0 + t < m) ? __ldcs(src + t) : 0.0;
    }
  };
  load(0, cur);
#pragma unroll 1
  for (int s = 0; s < 8; ++s) {
    if (s + 1 < 8) load(s + 1, nxt);
    const int ch = threadIdx.x + 256 * s;
    const int r = ch >> 4, h = ch & 15;
    Parts2 x[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) x[t] = split_parts2(cur[2 * t], cur[2 * t + 1], scale);
    ChunkWriter<0, NMOD, 8>::run(x, tile + swz(r, h >> 1) + (h & 1) * 8, mod_stride);
#pragma unroll
    for (int t = 0; t < 8; ++t) cur[t] = nxt[t];
  }
}

// Per-column scale of the skinny operand B (K x ncols): one CTA per (padded)
// column.  One pass: max |b| and the sum of squares; only when that sum left
// [2^-900, 2^900] (squares that may have over- or underflowed) a second pass
// sums the squares of b 2^-s (s = exponent of the max), so no over/underflow
// can misplace the scale.  A column holding NaN/Inf
// gets kEbNonFinite: its residues are zero and the CRT writes NaN into the
// output column (every BLAS output touching it is non-finite too).  The scale
// may exceed 2^1023 (columns of norm < 2^-970): residue_b applies it with
// scalbn, the CRT unscales with scalbn.
constexpr int kEbNonFinite = -0x40000000;
__global__ void __launch_bounds__(256) bscale_kernel(const double* __restrict__ b, int64_t ldb, int64_t k,
                                                     int64_t ncols, int64_t cols_pad, int pb, int* __restrict__ e_b) {
  const int64_t jj = blockIdx.x;
  __shared__ double red[8], red2[8];
  __shared__ double s_mx;
  const double* col = b + jj * ldb;
  // pass 1: max |b|, non-finite flag and the plain sum of squares together;
  // the scaled second pass runs only when the plain sum left the safe range
  double mx = 0.0, ss = 0.0;
  bool bad = false;
  if (jj < ncols) {
    for (int64_t i = threadIdx.x; i < k; i += 256) {
      const double v = __ldg(col + i);
      const double av = fabs(v);
      bad |= !(av <= 1.7976931348623157e308);
      mx = fmax(mx, av);
      ss = fma(v, v, ss);
    }
  }
  bad = __syncthreads_or(bad);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = mx;
    red2[threadIdx.x >> 5] = ss;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0, t2 = 0.0;
    for (int w = 0; w < 8; ++w) {
      t = fmax(t, red[w]);
      t2 += red2[w];
    }
    s_mx = t;
    red2[0] = t2;
  }
  __syncthreads();
  mx = s_mx;
  const double plain = red2[0];
  if (bad || mx == 0.0) {
    if (threadIdx.x == 0) e_b[jj] = bad ? kEbNonFinite : 0;
    return;
  }
  if (plain >= 0x1p-900 && plain <= 0x1p900) {  // no over/underflow could have distorted it
    if (threadIdx.x == 0) {
      int ex;
      frexp(sqrt(plain) * (1.0 + 0x1p-40), &ex);  // ||b_j|| < 2^ex
      e_b[jj] = pb - ex;
    }
    return;
  }
  int s;
  frexp(mx, &s);  // mx < 2^s
  double s0 = 0.0, s1 = 0.0;
  for (int64_t i = threadIdx.x; i < k; i += 512) {
    const double v0 = scalbn(__ldg(col + i), -s);
    s0 = fma(v0, v0, s0);
    if (i + 256 < k) {
      const double v1 = scalbn(__ldg(col + i + 256), -s);
      s1 = fma(v1, v1, s1);
    }
  }
  ss = s0 + s1;
#pragma unroll
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < 8; ++w) tot += red[w];
    int ex;
    frexp(sqrt(tot) * (1.0 + 0x1p-40), &ex);  // ||b_j|| < 2^(ex + s)
    e_b[jj] = pb - (ex + s);
  }
}

// Residues of B: K-major tiles of n_g rows x 128 bytes per (l, group, kb);
// grid (padded column, chunk block), 16 consecutive k per thread.
template <int NMOD>
__global__ void __launch_bounds__(256) residue_b_kernel(const double* __restrict__ b, int64_t ldb, int64_t k,
                                                        int64_t ncols, int n_g, int64_t nkb,
                                                        const int* __restrict__ e_b, int8_t* __restrict__ tiles,
                                                        int ng) {
  const int64_t jj = blockIdx.x;
  const int g = (int)(jj / n_g), r = (int)(jj % n_g);
  const int eb = e_b[jj];
  const bool dead = eb == kEbNonFinite;  // NaN/Inf column: zero residues, NaN output (crt_kernel)
  const size_t mod_stride = (size_t)ng * nkb * n_g * kTile;
  int8_t* tile0 = tiles + (size_t)g * nkb * n_g * kTile;
  const int64_t ch = (int64_t)blockIdx.y * 256 + threadIdx.x;
  if (ch >= nkb * 8) return;
  const int64_t kb = ch >> 3;
  const int c = (int)(ch & 7);
  const int64_t i0 = kb * kTile + c * 16;
  double v[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const int64_t i = i0 + t;
    v[t] = (jj < ncols && i < k && !dead) ? scalbn(b[i + jj * ldb], eb) : 0.0;  // exact (|result| < 2^53)
  }
  Parts2 x[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) x[t] = split_parts2(v[2 * t], v[2 * t + 1], 1.0);
  ChunkWriter<0, NMOD, 16>::run(x, tile0 + (size_t)kb * n_g * kTile + swz(r, c), mod_stride);
}

// ----------------------------------------------------------------- A scale
// Row and column 2-norms of A in ONE read: CTA = 2048 rows x 256 columns;
// partial sums in fixed order (deterministic), then max -> eA, plus the
// guard statistics (header below); NaN / Inf propagate through the sums.  A
// row or column whose sum of squares is below DBL_MIN -- all zero, or tiny
// entries whose squares underflow -- is reported through the minimum as is
// (0 or subnormal), so the guard rejects that orientation: exact zero rows are
// rare in dense operands and only cost the faster engine.
constexpr int kNormRows = 2048, kNormCols = 256, kNormBlk = 8;
constexpr size_t kNormSmem = (8 * kNormCols + 8 * 32 * (kNormBlk + 1)) * sizeof(double);

// Header of the scale and prep workspaces (device, first 64 bytes).
struct OzHeader {
  int e_a;                       // scale of A (prep workspaces only)
  int pad;
  unsigned long long maxbits;    // max over rows and columns of the sum of squares (double bits)
  unsigned long long minrow;     // min over rows (~0ull: none)
  unsigned long long mincol;     // min over columns (~0ull: none)
  unsigned nonfinite;            // a row or column sum is NaN / Inf
  unsigned nonint;               // some entry is not an integer
  double fro2;                   // ||A||_F^2 from the column partials (fro2_kernel)
};

__global__ void __launch_bounds__(256, 4) norms_partial_kernel(const double* __restrict__ a, int64_t lda, int64_t m,
                                                            int64_t n, double* __restrict__ part_row,
                                                            double* __restrict__ part_col, OzHeader* hdr,
                                                            int64_t cb0) {
  // warp w owns rows r0 + 256 w + [0, 256) (8 chunks of 32, lane = row in
  // chunk); column blocks of 32: lane keeps its rows' partial sums per column,
  // then one shared-memory transpose per block sums them over the lanes
  const int64_t rb = blockIdx.x, cb = blockIdx.y + cb0;
  if (rb == 0 && cb == 0 && threadIdx.x == 0) {  // statistics reset (norms_final runs after this kernel)
    hdr->maxbits = 0ull;
    hdr->minrow = ~0ull;
    hdr->mincol = ~0ull;
    hdr->nonfinite = 0u;
    hdr->nonint = 0u;
  }
  const int64_t r0 = rb * kNormRows, c0 = cb * kNormCols;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  extern __shared__ double nsm[];
  double (*colw)[kNormCols] = reinterpret_cast<double (*)[kNormCols]>(nsm);
  double (*tile)[32][kNormBlk + 1] = reinterpret_cast<double (*)[32][kNormBlk + 1]>(nsm + 8 * kNormCols);
  double rs[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) rs[s] = 0.0;
  const int ncols = (int)(n - c0 < kNormCols ? n - c0 : kNormCols);
  const int64_t rw = r0 + 256 * warp + lane;
  const bool full = r0 + kNormRows <= m;
  for (int cb32 = 0; cb32 < ncols; cb32 += kNormBlk) {
    double cs[kNormBlk];
#pragma unroll
    for (int c = 0; c < kNormBlk; ++c) cs[c] = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int64_t i = rw + 32 * s;
      const bool rok = full || i < m;
#pragma unroll
      for (int c = 0; c < kNormBlk; ++c) {
        const double v = (rok && cb32 + c < ncols) ? __ldcs(a + i + (c0 + cb32 + c) * lda) : 0.0;
        rs[s] = fma(v, v, rs[s]);
        cs[c] = fma(v, v, cs[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < kNormBlk; ++c) tile[warp][lane][c] = cs[c];
    __syncwarp();
    if (lane < kNormBlk) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < 32; ++q) t += tile[warp][q][lane];
      if (cb32 + lane < ncols) colw[warp][cb32 + lane] = t;
    }
    __syncwarp();
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int64_t i = rw + 32 * s;
    if (i < m) part_row[cb * m + i] = rs[s];
  }
  if (threadIdx.x < ncols) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += colw[w][threadIdx.x];
    part_col[rb * n + c0 + threadIdx.x] = t;
  }
}

constexpr int kIntSampleCols = 16;

__global__ void norms_final_kernel(const double* __restrict__ part_row, int64_t ncb, int64_t m,
                                   const double* __restrict__ part_col, int64_t nrb, int64_t n,
                                   OzHeader* __restrict__ hdr, const double* __restrict__ a, int64_t lda) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < m) {  // integrality sample: row t of 16 evenly spread columns.  A non-integer
                // entry proves A is not integer-valued; an all-integer sample (possibly a
                // false "integer") only costs the faster engine (integer A goes to DMMA).
    bool frac = false;
#pragma unroll 4
    for (int q = 0; q < kIntSampleCols; ++q) {
      const double v = __ldg(a + t + ((int64_t)q * n / kIntSampleCols) * lda);
      frac |= v != rint(v);
    }
    if (__any_sync(__activemask(), frac) && (threadIdx.x & 31) == 0) atomicOr(&hdr->nonint, 1u);
  }
  double v = 0.0;
  if (t < m) {
    for (int64_t cb = 0; cb < ncb; ++cb) v += part_row[cb * m + t];
  } else if (t < m + n) {
    for (int64_t rb = 0; rb < nrb; ++rb) v += part_col[rb * n + (t - m)];
  }
  const bool bad = !(v <= 1.7976931348623157e308);  // NaN, Inf (or an overflowing sum of squares)
  const double inf = __longlong_as_double(0x7FF0000000000000ll);
  double mx = bad ? 0.0 : v;
  double mnr = (!bad && t < m) ? v : inf;
  double mnc = (!bad && t >= m && t < m + n) ? v : inf;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mnr = fmin(mnr, __shfl_xor_sync(0xffffffffu, mnr, o));
    mnc = fmin(mnc, __shfl_xor_sync(0xffffffffu, mnc, o));
  }
  const bool anybad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {  // v >= 0: bit order = value order
    atomicMax(&hdr->maxbits, (unsigned long long)__double_as_longlong(mx));
    if (mnr < inf) atomicMin(&hdr->minrow, (unsigned long long)__double_as_longlong(mnr));
    if (mnc < inf) atomicMin(&hdr->mincol, (unsigned long long)__double_as_longlong(mnc));
    if (anybad) atomicOr(&hdr->nonfinite, 1u);
  }
}

// ||A||_F^2 as a by-product of the norms pass (rlra/accessors.py:33-34 at
// rlra/fixedprec.py:72; north star (d): the Frobenius-norm reduction fused with
// the pass): the column partial sums (each over <= 2048 rows) are added in a
// fixed order in double-double, so no extra read of A.
__device__ __forceinline__ void oz_two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

__global__ void __launch_bounds__(1024) fro2_kernel(const double* __restrict__ part, int64_t count,
                                                    OzHeader* __restrict__ hdr) {
  __shared__ double sh[32], sl[32];
  double hi = 0.0, lo = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += 1024) {
    double s, e;
    oz_two_sum(hi, part[i], s, e);
    hi = s;
    lo += e;
  }
  auto merge = [](double& h, double& l, double h2, double l2) {
    double s, e;
    oz_two_sum(h, h2, s, e);
    h = s;
    l = l + l2 + e;
  };
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double h2 = __shfl_down_sync(0xffffffffu, hi, o), l2 = __shfl_down_sync(0xffffffffu, lo, o);
    merge(hi, lo, h2, l2);
  }
  if ((threadIdx.x & 31) == 0) {
    sh[threadIdx.x >> 5] = hi;
    sl[threadIdx.x >> 5] = lo;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    hi = sh[threadIdx.x];
    lo = sl[threadIdx.x];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double h2 = __shfl_down_sync(0xffffffffu, hi, o), l2 = __shfl_down_sync(0xffffffffu, lo, o);
      merge(hi, lo, h2, l2);
    }
    if (threadIdx.x == 0) hdr->fro2 = hi + lo;
  }
}

// Provisional scale from the first column chunk of a pipelined upload
// (columns [0, c1)): column norms of those columns exactly, row norms
// extrapolated by n / c1 (the remaining chunks are still on the PCIe bus).  The
// final norms decide whether it stands (oz_norms_finish: the residues are
// rebuilt when the final eA differs).
__global__ void __launch_bounds__(1024) scale_estimate_kernel(const double* __restrict__ part_row, int64_t m,
                                                              const double* __restrict__ part_col, int64_t nrb,
                                                              int64_t n, int64_t c1, int pa, OzHeader* __restrict__ hdr) {
  __shared__ double red[32];
  const int64_t ncb1 = (c1 + kNormCols - 1) / kNormCols;
  double mx = 0.0;
  for (int64_t t = threadIdx.x; t < m + c1; t += 1024) {
    double v = 0.0;
    if (t < m) {
      for (int64_t cb = 0; cb < ncb1; ++cb) v += part_row[cb * m + t];
      v *= (double)n / (double)c1;
    } else {
      for (int64_t rb = 0; rb < nrb; ++rb) v += part_col[rb * n + (t - m)];
    }
    mx = fmax(mx, v);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < 32; ++w) mx = fmax(mx, red[w]);
    int e = 0;
    if (mx > 0.0 && mx <= 1.7976931348623157e308) {
      int ex;
      frexp(sqrt(mx) * (1.0 + 0x1p-40), &ex);
      e = pa - ex;
    }
    hdr->e_a = e;
  }
}

__global__ void scale_a_kernel(const OzHeader* __restrict__ hdr, int pa, int* __restrict__ e_a) {
  const double t = __longlong_as_double((long long)hdr->maxbits);
  int e = 0;
  if (t > 0.0 && hdr->nonfinite == 0u) {
    int ex;
    frexp(sqrt(t) * (1.0 + 0x1p-40), &ex);
    e = pa - ex;
  }
  e_a[0] = e;
}

// ----------------------------------------------------------------- tcgen05 GEMM
struct GemmArgs {
  const int8_t* a_tiles;
  int64_t nib, njb;  // residue tile grid of A (both padded to even)
  int trans;         // 1: C = A^T B (M tiles = jb, K tiles = ib); 0: C = A B (M = ib, K = jb)
  const int8_t* b_tiles;
  int ng, n_g;  // column groups, columns per group (multiple of 32, <= 256)
  int64_t nkb;  // K tiles
  int64_t nmb;  // 256-row blocks
  uint8_t* out;  // t[l][col][row], rows padded to nmb*256, cols to ng*n_g
  int nmod;
  int accum;  // 1: t = (t + C_l) mod m_l (K split over several calls), 0: t = C_l mod m_l
  int mods[kMaxMod];
  int ys[kMaxMod];  // CRT weights (M/m_l)^-1 mod m_l, folded into the epilogue
};

__device__ __forceinline__ uint64_t sw128_desc(unsigned saddr, unsigned lbo, unsigned sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;  // 128-byte swizzle
  return d;
}

__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned mbar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(mbar), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void mma_i8(unsigned tmem_d, uint64_t adesc, uint64_t bdesc, unsigned idesc,
                                       unsigned acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_commit(unsigned mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(mbar)
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}

#define OZ_LD32(taddr, v)                                                                                      \
  asm volatile(                                                                                                \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                                     \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),       \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),             \
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),           \
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),           \
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                                                                 \
      : "r"(taddr))

// 32 accumulators of one TMEM row -> 32 bytes t = (c y) mod m in the warp's
// staging tile stg[col][lane] (see the epilogue comment in gemm_i8_kernel);
// ACCUM adds the previous K blocks' bytes staged at stg + 1024.  Straight-line
// code (no branch per element) so that the 16 pairs' chains interleave: an
// epilogue warp is alone on its scheduler, instruction-level parallelism is
// all the latency hiding there is.
template <bool ACCUM>
__device__ __forceinline__ void epi_chunk(const unsigned (&v)[32], uint8_t* stg, int lane, f2_t k1f, f2_t ycf,
                                          f2_t invf, f2_t nmf, float mf) {
  const f2_t big = f2_dup(12582912.0f), nbig = f2_dup(-12582912.0f), n23 = f2_dup(-8388608.0f);
  const float fix_neg = mf + 8388608.0f, fix_pos = 8388608.0f;  // exact: m + 2^23 < 2^24
  unsigned prev[ACCUM ? 32 : 1];
  if (ACCUM) {
#pragma unroll
    for (int e = 0; e < 32; ++e) prev[e] = stg[1024 + e * 32 + lane];
  }
#pragma unroll
  for (int e = 0; e < 32; e += 2) {
    const unsigned c0 = v[e], c1 = v[e + 1];
    const f2_t lof = f2_fadd(f2_bits(0x4B000000u | (c0 & 0xFFFFu), 0x4B000000u | (c1 & 0xFFFFu)), n23);
    const f2_t hif =
        f2_fadd(f2_bits(0x4B400000u + (unsigned)((int)c0 >> 16), 0x4B400000u + (unsigned)((int)c1 >> 16)), nbig);
    const f2_t sv = f2_ffma(hif, k1f, f2_ffma(lof, ycf, 0ull));  // exact: |s| < 2^24
    const f2_t qv = f2_fadd(f2_ffma(sv, invf, big), nbig);       // ~rint(s / m)
    const f2_t rv = f2_ffma(qv, nmf, sv);                        // exact, |r| <= 125
    const float r0 = __uint_as_float((unsigned)rv), r1 = __uint_as_float((unsigned)(rv >> 32));
    unsigned b0, b1;
    if (ACCUM) {  // exact modular sum with the previous K blocks (bytes in [0, m))
      float z0 = r0 + __uint_as_float(0x4B000000u | prev[e]);  // 2^23 + (r + prev), r + prev in (-m, 2m)
      float z1 = r1 + __uint_as_float(0x4B000000u | prev[ACCUM ? e + 1 : 0]);
      z0 += z0 < 8388608.0f ? mf : 0.0f;
      z1 += z1 < 8388608.0f ? mf : 0.0f;
      z0 -= z0 >= fix_neg ? mf : 0.0f;
      z1 -= z1 >= fix_neg ? mf : 0.0f;
      b0 = __float_as_uint(z0);
      b1 = __float_as_uint(z1);
    } else {
      b0 = __float_as_uint(r0 + (r0 < 0.0f ? fix_neg : fix_pos));
      b1 = __float_as_uint(r1 + (r1 < 0.0f ? fix_neg : fix_pos));
    }
    stg[e * 32 + lane] = (uint8_t)b0;
    stg[(e + 1) * 32 + lane] = (uint8_t)b1;
  }
}

__global__ void __launch_bounds__(kGemmThreads, 1) gemm_i8_kernel(const GemmArgs g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment of the stage buffers (swizzle atoms)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const unsigned b_bytes = (unsigned)g.n_g * kTile;
  const unsigned stage_bytes = 2 * kTileBytes + b_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * stage_bytes);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint64_t* tmem_empty = tmem_full + 1;
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(tmem_empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 128);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem_base = *tmem_slot;

  const int64_t mtiles = g.trans ? g.njb : g.nib;
  (void)mtiles;
  const int64_t units = (int64_t)g.nmod * g.nmb * g.ng;
  const size_t mod_stride_a = (size_t)g.njb * g.nib * kTileBytes;
  const size_t mod_stride_b = (size_t)g.ng * g.nkb * b_bytes;

  if (warp == 0) {
    if (lane == 0) {
      uint64_t pol_a, pol_b;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_a));
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_b));
      int stage = 0;
      unsigned phase = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int gi = (int)(u % g.ng);
        const int64_t mb = (u / g.ng) % g.nmb;
        const int l = (int)(u / ((int64_t)g.ng * g.nmb));
        const int8_t* abase = g.a_tiles + (size_t)l * mod_stride_a;
        const int8_t* bbase = g.b_tiles + (size_t)l * mod_stride_b + (size_t)gi * g.nkb * b_bytes;
        for (int64_t kb = 0; kb < g.nkb; ++kb) {
          mbar_wait_parity(empty + stage, phase ^ 1);
          uint8_t* st = smem + (size_t)stage * stage_bytes;
          const unsigned fb = smem_u32(full + stage);
          mbar_arrive_expect_tx(full + stage, stage_bytes);
          for (int t = 0; t < 2; ++t) {
            const int64_t mt = 2 * mb + t;
            const size_t tix = g.trans ? ((size_t)mt * g.nib + kb) : ((size_t)kb * g.nib + mt);
            bulk_g2s(smem_u32(st + t * kTileBytes), abase + tix * kTileBytes, kTileBytes, fb, pol_a);
          }
          bulk_g2s(smem_u32(st + 2 * kTileBytes), bbase + (size_t)kb * b_bytes, b_bytes, fb, pol_b);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // instruction descriptor: s32 accum, s8 x s8, A K-major (TN) or MN-major (NN), B K-major
      const unsigned idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((g.trans ? 0u : 1u) << 15) |
                             ((unsigned)(g.n_g >> 3) << 17) | ((unsigned)(128 >> 4) << 24);
      int stage = 0;
      unsigned phase = 0, acc_phase = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        mbar_wait_parity(tmem_empty, acc_phase ^ 1);
        tc_fence_after();
        for (int64_t kb = 0; kb < g.nkb; ++kb) {
          mbar_wait_parity(full + stage, phase);
          tc_fence_after();
          const unsigned sa = smem_u32(smem + (size_t)stage * stage_bytes);
          const unsigned sb = sa + 2 * kTileBytes;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t bdesc = sw128_desc(sb + 32 * k, 16, 1024);
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              const unsigned at = sa + t * kTileBytes;
              const uint64_t adesc =
                  g.trans ? sw128_desc(at + 32 * k, 16, 1024) : sw128_desc(at + 4096 * k, kTileBytes, 1024);
              mma_i8(tmem_base + (unsigned)(t * g.n_g), adesc, bdesc, idesc, (kb | k) ? 1u : 0u);
            }
          }
          mma_commit(smem_u32(empty + stage));
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(smem_u32(tmem_full));
        acc_phase ^= 1;
      }
    }
  } else {
    // epilogue: warps 2..5 -> TMEM lane quadrant (warp % 4).  t = (C_l y_l) mod
    // m_l on the fp32 pipes (packed FFMA2 / FADD2), every step exact:
    //   c = hi 2^16 + lo (hi signed, lo in [0, 2^16)); s = hi k1 + lo y' with the
    //   centred representatives k1 = (2^16 y) mod m, y' = y mod m in [-124, 124],
    //   so |s| <= 124 (2^15 + 2^16) < 2^24 is an exact fp32 integer = c y (mod m);
    //   q = rint(s / m) up to +-0.006 (magic-number rounding), r = s - q m exact,
    //   |r| <= 125 < m; t = r + m (r < 0).  The bytes go through a 32 x 32 staging
    //   tile per warp so that the global stores are 16-byte rows of t[l][col][row].
    const int q = warp & 3;
    const int64_t rows_pad = g.nmb * 256;
    const int64_t cols_pad = (int64_t)g.ng * g.n_g;
    uint8_t* stg = smem + (size_t)kStages * stage_bytes + 256 + (size_t)q * 2048;  // [2][32 cols][32 rows]
    unsigned acc_phase = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      const int gi = (int)(u % g.ng);
      const int64_t mb = (u / g.ng) % g.nmb;
      const int l = (int)(u / ((int64_t)g.ng * g.nmb));
      mbar_wait_parity(tmem_full, acc_phase);
      tc_fence_after();
      const int ml = g.mods[l], yl = g.ys[l] % ml;
      int k1 = (int)((65536ll * yl) % ml), yc = yl;
      if (2 * k1 > ml) k1 -= ml;
      if (2 * yc > ml) yc -= ml;
      const float mf = (float)ml;
      const f2_t k1f = f2_dup((float)k1), ycf = f2_dup((float)yc), invf = f2_dup(1.0f / mf), nmf = f2_dup(-mf);
      for (int t = 0; t < 2; ++t) {
        // rows mb*256 + t*128 + q*32 .. +32 of the 32 columns cc.. : 16-byte piece j = lane + 32 i of the
        // staging tile is rows (j % 2) * 16 .. +16 of column j / 2
        uint8_t* otile = g.out + ((size_t)l * cols_pad + (size_t)gi * g.n_g) * rows_pad + (mb * 256 + t * 128 + q * 32);
        for (int cc = 0; cc < g.n_g; cc += 32) {
          unsigned v[32];
          const unsigned taddr = tmem_base + ((unsigned)(q * 32) << 16) + (unsigned)(t * g.n_g + cc);
          OZ_LD32(taddr, v);
          if (g.accum) {  // previous K blocks' residues of this tile -> staging half 1
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int j = lane + 32 * i;
              const uint4 pv = *reinterpret_cast<const uint4*>(otile + (size_t)(cc + (j >> 1)) * rows_pad + (j & 1) * 16);
              *reinterpret_cast<uint4*>(stg + 1024 + j * 16) = pv;
            }
            __syncwarp();
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          if (g.accum) epi_chunk<true>(v, stg, lane, k1f, ycf, invf, nmf, mf);
          else epi_chunk<false>(v, stg, lane, k1f, ycf, invf, nmf, mf);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int j = lane + 32 * i;
            const uint4 ov = *reinterpret_cast<const uint4*>(stg + j * 16);
            *reinterpret_cast<uint4*>(otile + (size_t)(cc + (j >> 1)) * rows_pad + (j & 1) * 16) = ov;
          }
          __syncwarp();
        }
      }
      tc_fence_before();
      mbar_arrive(tmem_empty);
      acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem_base) : "memory");
  }
}

// ----------------------------------------------------------------- CRT
__device__ __forceinline__ double u128_to_double(u128 x) {
  if (x == 0) return 0.0;
  const uint64_t hi = (uint64_t)(x >> 64), lo = (uint64_t)x;
  const int lz = hi ? __clzll((long long)hi) : 64 + __clzll((long long)lo);
  const u128 y = x << lz;  // top bit at 127
  uint64_t top = (uint64_t)(y >> 64);
  top |= ((uint64_t)y != 0) ? 1ull : 0ull;  // sticky (below the rounding bit)
  return scalbn(__ull2double_rn(top), 64 - lz);
}

// CRT: s = sum_l t'_l (M / m_l) (t'_l < m_l, so every term is < M and the sum
// of nmod <= 15 terms stays below 2^122), in two 64-bit words; then one
// reduction modulo M and the signed representative as a double.
// One element of the CRT: residues tv[0..nmod) -> the signed integer A''B'' as a
// double (within 1 ulp; the sign in `neg`).
__device__ __forceinline__ double crt_value(const unsigned (&tv)[kMaxMod], const Crt& crt, bool& neg) {
  const int nm = crt.nmod;
  const u128 M = ((u128)crt.M_hi << 64) | crt.M_lo;
  const u128 H = ((u128)crt.H_hi << 64) | crt.H_lo;
  double v;
  if (nm <= 14) {
    // 28-bit limbs: every product t d < 2^36 and the 14-term sums < 2^40, one
    // 32x32->64 multiply-add each (IMAD.WIDE); then carries, one quotient
    // estimate (s < 14 * 256 * M / 181 < 20 M) and an exact limb subtraction
    constexpr int64_t MASK = (1ll << 28) - 1;
    uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
    for (int l = 0; l < 14; ++l) {
      const uint64_t tl = tv[l];
      a0 += tl * crt.d28[0][l];
      a1 += tl * crt.d28[1][l];
      a2 += tl * crt.d28[2][l];
      a3 += tl * crt.d28[3][l];
    }
    a1 += a0 >> 28;
    a2 += a1 >> 28;
    a3 += a2 >> 28;
    int64_t s0 = (int64_t)(a0 & MASK), s1 = (int64_t)(a1 & MASK), s2 = (int64_t)(a2 & MASK), s3 = (int64_t)a3;
    const double sd = fma((double)s3, 0x1p84, (double)s2 * 0x1p56);
    const int64_t q = (int64_t)(sd * crt.inv_M);  // floor(s / M) or one off
    s0 -= q * (int64_t)crt.M28[0];
    s1 -= q * (int64_t)crt.M28[1];
    s2 -= q * (int64_t)crt.M28[2];
    s3 -= q * (int64_t)crt.M28[3];
    auto norm = [&]() {  // signed limbs -> limbs in [0, 2^28) except the top
      s1 += s0 >> 28;
      s0 &= MASK;
      s2 += s1 >> 28;
      s1 &= MASK;
      s3 += s2 >> 28;
      s2 &= MASK;
    };
    norm();
    if (s3 < 0) {  // q one too large
      s0 += crt.M28[0]; s1 += crt.M28[1]; s2 += crt.M28[2]; s3 += crt.M28[3];
      norm();
    }
    const bool ge = s3 != (int64_t)crt.M28[3] ? s3 > (int64_t)crt.M28[3]
                    : s2 != (int64_t)crt.M28[2] ? s2 > (int64_t)crt.M28[2]
                    : s1 != (int64_t)crt.M28[1] ? s1 > (int64_t)crt.M28[1] : s0 >= (int64_t)crt.M28[0];
    if (ge) {  // q one too small
      s0 -= crt.M28[0]; s1 -= crt.M28[1]; s2 -= crt.M28[2]; s3 -= crt.M28[3];
      norm();
    }
    // s in [0, M): the signed representative is s - M when s > floor(M / 2)
    neg = s3 != (int64_t)crt.H28[3] ? s3 > (int64_t)crt.H28[3]
          : s2 != (int64_t)crt.H28[2] ? s2 > (int64_t)crt.H28[2]
          : s1 != (int64_t)crt.H28[1] ? s1 > (int64_t)crt.H28[1] : s0 > (int64_t)crt.H28[0];
    if (neg) {  // magnitude M - s
      s0 = crt.M28[0] - s0; s1 = crt.M28[1] - s1; s2 = crt.M28[2] - s2; s3 = crt.M28[3] - s3;
      norm();
    }
    const uint64_t top = ((uint64_t)s3 << 28) | (uint64_t)s2;  // < 2^54: exact in a double
    const uint64_t low = ((uint64_t)s1 << 28) | (uint64_t)s0;  // < 2^56
    v = fma((double)top, 0x1p56, (double)low);                  // within 1 ulp
  } else {
  u128 s = 0;
  if (nm <= 15) {
    uint64_t lo = 0, hi = 0;
#pragma unroll
    for (int l = 0; l < 15; ++l) {
      const uint64_t p0 = crt.md_lo[l] * (uint64_t)tv[l];
      const uint64_t p1 = __umul64hi(crt.md_lo[l], (uint64_t)tv[l]) + crt.md_hi[l] * (uint64_t)tv[l];
      lo += p0;
      hi += p1 + (lo < p0 ? 1ull : 0ull);
    }
    s = ((u128)hi << 64) | lo;
    const uint64_t q = (uint64_t)(fma((double)hi, 0x1p64, (double)lo) * crt.inv_M);  // floor(s / M) +- 1
    s -= (u128)q * M;
    if ((s >> 127) != 0) s += M;  // q was one too large
    if (s >= M) s -= M;
  } else {  // 16 moduli: M ~ 2^124.6; add the terms (< M) one by one, reducing
#pragma unroll
    for (int l = 0; l < kMaxMod; ++l) {
      s += (u128)tv[l] * (((u128)crt.md_hi[l] << 64) | crt.md_lo[l]);
      if (s >= M) s -= M;
    }
  }
  const u128 mag = (s > H) ? M - s : s;
  v = fma((double)(uint64_t)(mag >> 64), 0x1p64, (double)(uint64_t)mag);  // within 1 ulp
  neg = s > H;
  }
  return v;
}

// Double-double helpers of the fused column energies (same arithmetic as the
// K8 reduction in misc.cu).
struct DDv {
  double hi, lo;
};
__device__ __forceinline__ DDv dd_two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ DDv dd_plus(DDv x, DDv y) {
  const DDv s = dd_two_sum(x.hi, y.hi);
  return dd_two_sum(s.hi, s.lo + x.lo + y.lo);
}
__device__ __forceinline__ DDv dd_plus_sq(DDv acc, double x) {
  const double p = x * x, e = fma(x, x, -p);  // exact square = p + e
  const DDv s = dd_two_sum(acc.hi, p);
  return dd_two_sum(s.hi, s.lo + acc.lo + e);
}
__device__ __forceinline__ DDv dd_warp_sum(DDv v) {
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const DDv o{__shfl_down_sync(0xffffffffu, v.hi, off), __shfl_down_sync(0xffffffffu, v.lo, off)};
    v = dd_plus(v, o);
  }
  return v;
}

// 4 consecutive rows per thread: one 32-bit load per residue plane.
// colsq != nullptr (RLRA_B200_OZ_COLSQ; rlra/fixedprec.py:71-80, north star (d):
// the Frobenius-norm reduction fused with the product): the block also leaves
// the double-double sum of squares of the 1024 values it wrote at
// colsq[j * nblk + blockIdx.x] (fixed reduction tree: deterministic), so the
// column energies of G cost no second read of G.
template <bool COLSQ>
__global__ void __launch_bounds__(256) crt_kernel(const uint8_t* __restrict__ t, int64_t rows_pad, int64_t cols_pad,
                                                  int64_t mrows, int64_t ncols, const int* __restrict__ e_a,
                                                  const int* __restrict__ e_b, const Crt crt, double* __restrict__ c,
                                                  int64_t ldc, int add, double2* __restrict__ colsq) {
  const int64_t i0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  const int64_t j = blockIdx.y;
  DDv acc{0.0, 0.0};
  if (i0 < mrows) {
    const size_t lstride = (size_t)cols_pad * rows_pad;
    const uint32_t* tp = reinterpret_cast<const uint32_t*>(t + (size_t)j * rows_pad + i0);  // rows_pad % 256 == 0
    const int nm = crt.nmod;
    uint32_t w[kMaxMod];
#pragma unroll
    for (int l = 0; l < kMaxMod; ++l) w[l] = (l < nm) ? __ldcs(tp + (size_t)l * (lstride / 4)) : 0u;
    const int eb = e_b[j];
    const bool dead = eb == kEbNonFinite;  // non-finite column of B: NaN, like every BLAS output it touches
    const int sc = -(e_a[0] + (dead ? 0 : eb));
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (i0 + e >= mrows) break;
      unsigned tv[kMaxMod];
#pragma unroll
      for (int l = 0; l < kMaxMod; ++l) tv[l] = (w[l] >> (8 * e)) & 0xFFu;
      bool neg;
      const double v = crt_value(tv, crt, neg);
      double r = dead ? __longlong_as_double(0x7FF8000000000000ll) : scalbn(neg ? -v : v, sc);
      double* cp = c + (i0 + e) + j * ldc;
      if (add) r = *cp + r;  // add: C += A B (one rounding of the sum, like beta = 1)
      *cp = r;
      if (COLSQ) acc = dd_plus_sq(acc, r);
    }
  }
  if (!COLSQ) return;
  __shared__ double s_hi[8], s_lo[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  acc = dd_warp_sum(acc);
  if (lane == 0) {
    s_hi[warp] = acc.hi;
    s_lo[warp] = acc.lo;
  }
  __syncthreads();
  if (warp == 0) {
    DDv v = lane < 8 ? DDv{s_hi[lane], s_lo[lane]} : DDv{0.0, 0.0};
    v = dd_warp_sum(v);
    if (lane == 0) colsq[(size_t)j * gridDim.x + blockIdx.x] = make_double2(v.hi, v.lo);
  }
}

// Column energies from the CRT blocks' partials: one warp per column, partials
// added in a fixed order in double-double; out[j] = (or +=) the sum.
__global__ void __launch_bounds__(256) colsq_finish_kernel(const double2* __restrict__ part, int64_t nblk,
                                                           int64_t ncols, double* __restrict__ out, int accumulate) {
  const int lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= ncols) return;
  DDv acc{0.0, 0.0};
  for (int64_t b = lane; b < nblk; b += 32) {
    const double2 v = part[(size_t)j * nblk + b];
    acc = dd_plus(acc, DDv{v.x, v.y});
  }
  acc = dd_warp_sum(acc);
  if (lane == 0) {
    const double v = acc.hi + acc.lo;
    out[j] = accumulate ? out[j] + v : v;
  }
}

// ----------------------------------------------------------------- host side
struct PrepLayout {
  int64_t nib, njb, ncb, nrb;
  size_t off_hdr, off_prow, off_pcol, off_tiles, total;
};
static PrepLayout prep_layout(int64_t m, int64_t n, int nmod) {
  PrepLayout p;
  p.nib = ceil_div(m, kTile);
  p.nib += p.nib & 1;
  p.njb = ceil_div(n, kTile);
  p.njb += p.njb & 1;
  p.ncb = ceil_div(n, kNormCols);
  p.nrb = ceil_div(m, kNormRows);
  p.off_hdr = 0;
  p.off_prow = 256;
  p.off_pcol = p.off_prow + (size_t)p.ncb * m * sizeof(double);
  p.off_tiles = (p.off_pcol + (size_t)p.nrb * n * sizeof(double) + 1023) & ~size_t(1023);
  p.total = p.off_tiles + (size_t)nmod * p.njb * p.nib * kTileBytes;
  return p;
}

struct GemmLayout {
  int ng, n_g;
  int64_t nkb, nmb, rows_pad, cols_pad;
  size_t off_eb, off_b, off_t, off_tab, off_colsq, total;
  int64_t nblk;  // CRT blocks (1024 rows) per column: column-energy partials
};
static GemmLayout gemm_layout(const PrepLayout& p, int trans, int64_t ncols, int nmod) {
  GemmLayout g;
  g.ng = (int)ceil_div(ncols, 256);
  if (g.ng < 1) g.ng = 1;
  g.n_g = (int)ceil_div(ceil_div(ncols, g.ng), 32) * 32;
  if (g.n_g < 32) g.n_g = 32;
  g.nkb = trans ? p.nib : p.njb;
  g.nmb = (trans ? p.njb : p.nib) / 2;
  g.rows_pad = g.nmb * 256;
  g.cols_pad = (int64_t)g.ng * g.n_g;
  // t first: its offset depends only on the output block, so a K-split
  // sequence of calls (accumulating t) may pass workspaces sized for its
  // largest K block
  g.off_eb = 0;
  g.off_t = (((size_t)g.cols_pad * sizeof(int)) + 1023) & ~size_t(1023);
  g.off_b = (g.off_t + (size_t)nmod * g.cols_pad * g.rows_pad + 1023) & ~size_t(1023);
  g.off_tab = g.off_b + (size_t)nmod * g.cols_pad * g.nkb * kTile;
  g.nblk = ceil_div(g.rows_pad, 1024);
  g.off_colsq = (g.off_tab + 15) & ~size_t(15);
  g.total = g.off_colsq + (size_t)g.cols_pad * g.nblk * sizeof(double2);
  return g;
}

static size_t gemm_smem_bytes(int n_g) {  // stages + barriers (256) + the epilogue warps' staging tiles (4 x 2 KB)
  return 1024 + (size_t)kStages * (2 * kTileBytes + (size_t)n_g * kTile) + 256 + 8192;
}

template <int NMOD>
static void launch_residue_a(const double* a, int64_t lda, int64_t m, int64_t n, const int* e_a, int8_t* tiles,
                             const PrepLayout& p, cudaStream_t st) {
  residue_a_kernel<NMOD><<<dim3((unsigned)p.nib, (unsigned)p.njb), 256, 0, st>>>(a, lda, m, n, e_a, tiles, p.nib,
                                                                                  p.njb, 0);
}
// tile columns [jb0, jb1) only (the column chunks of a pipelined upload)
template <int NMOD>
static void launch_residue_a_cols(const double* a, int64_t lda, int64_t m, int64_t n, const int* e_a, int8_t* tiles,
                                  const PrepLayout& p, int64_t jb0, int64_t jb1, cudaStream_t st) {
  residue_a_kernel<NMOD><<<dim3((unsigned)p.nib, (unsigned)(jb1 - jb0)), 256, 0, st>>>(a, lda, m, n, e_a, tiles,
                                                                                        p.nib, p.njb, jb0);
}
template <int NMOD>
static void launch_residue_b(const double* b, int64_t ldb, int64_t k, int64_t ncols, const GemmLayout& g, int pb,
                             int* e_b, int8_t* tiles, bool scale, cudaStream_t st) {
  if (scale) bscale_kernel<<<(unsigned)g.cols_pad, 256, 0, st>>>(b, ldb, k, ncols, g.cols_pad, pb, e_b);
  residue_b_kernel<NMOD><<<dim3((unsigned)g.cols_pad, (unsigned)ceil_div(g.nkb * 8, 256)), 256, 0, st>>>(
      b, ldb, k, ncols, g.n_g, g.nkb, e_b, tiles, g.ng);
}

#define OZ_DISPATCH(NM, FN, ...)      \
  switch (NM) {                       \
    case 12: FN<12>(__VA_ARGS__); break; \
    case 13: FN<13>(__VA_ARGS__); break; \
    case 14: FN<14>(__VA_ARGS__); break; \
    case 15: FN<15>(__VA_ARGS__); break; \
    default: FN<16>(__VA_ARGS__); break; \
  }

}  // namespace oz

size_t oz_prep_workspace(int64_t m, int64_t n, int nmod) {
  if (nmod < 12 || nmod > oz::kMaxMod || m < 1 || n < 1) return 0;
  return oz::prep_layout(m, n, nmod).total;
}

static int oz_norms(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, int* e_a, oz::OzHeader* hdr,
                    double* prow, double* pcol, cudaStream_t st) {
  const int64_t ncb = ceil_div(n, oz::kNormCols), nrb = ceil_div(m, oz::kNormRows);
  RLRA_REQUIRE(nrb <= 2147483647 && ncb <= 65535, "oz: A too large for the norm grid");
  {
    static int attr_dev = -1;
    int dev = 0;
    RLRA_CHECK_CUDA(cudaGetDevice(&dev));
    if (attr_dev != dev) {
      RLRA_CHECK_CUDA(cudaFuncSetAttribute(oz::norms_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)oz::kNormSmem));
      attr_dev = dev;
    }
  }
  ktimer_mark(KT_OZ_NORMS, st, false);
  oz::norms_partial_kernel<<<dim3((unsigned)nrb, (unsigned)ncb), 256, oz::kNormSmem, st>>>(a, lda, m, n, prow,
                                                                                           pcol, hdr, 0);
  ktimer_mark(KT_OZ_NORMS, st, true);
  RLRA_LAUNCHED();
  oz::norms_final_kernel<<<(unsigned)ceil_div(m + n, 256), 256, 0, st>>>(prow, ncb, m, pcol, nrb, n, hdr, a, lda);
  RLRA_LAUNCHED();
  oz::scale_a_kernel<<<1, 1, 0, st>>>(hdr, oz::budget(nmod).pa, e_a);
  RLRA_LAUNCHED();
  oz::fro2_kernel<<<1, 1024, 0, st>>>(pcol, nrb * n, hdr);
  RLRA_LAUNCHED();
  return 0;
}

size_t oz_scale_workspace(int64_t m, int64_t n) {
  if (m < 1 || n < 1) return 0;
  return 256 + ((size_t)ceil_div(n, oz::kNormCols) * m + (size_t)ceil_div(m, oz::kNormRows) * n) * sizeof(double);
}

int oz_scale(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, int* e_a, void* ws, size_t ws_bytes,
             cudaStream_t st) {
  RLRA_REQUIRE(nmod >= 12 && nmod <= oz::kMaxMod, "oz_scale: nmod must be in [12, 16], got %d", nmod);
  RLRA_REQUIRE(m >= 1 && n >= 1 && lda >= m, "oz_scale: bad shape m=%lld n=%lld lda=%lld", (long long)m,
               (long long)n, (long long)lda);
  RLRA_REQUIRE(ws && e_a && ws_bytes >= oz_scale_workspace(m, n), "oz_scale: workspace too small");
  uint8_t* base = static_cast<uint8_t*>(ws);
  double* prow = reinterpret_cast<double*>(base + 256);
  double* pcol = prow + (size_t)ceil_div(n, oz::kNormCols) * m;
  return oz_norms(a, lda, m, n, nmod, e_a, reinterpret_cast<oz::OzHeader*>(base), prow, pcol, st);
}

// Dynamic-range guard (see the accuracy note at the top): T(K) = 2 (K-2)/sqrt(K) - 2.
double oz_guard_limit(int64_t k) { return k > 4 ? 2.0 * (double)(k - 2) / std::sqrt((double)k) - 2.0 : 0.0; }

int oz_guard(const void* hdr_host, int64_t m, int64_t n, int* ok_nn, int* ok_tn) {
  RLRA_REQUIRE(hdr_host && ok_nn && ok_tn && m >= 1 && n >= 1, "oz_guard: bad arguments");
  oz::OzHeader h;
  std::memcpy(&h, hdr_host, sizeof(h));
  double mx, mr, mc;
  std::memcpy(&mx, &h.maxbits, 8);
  std::memcpy(&mr, &h.minrow, 8);
  std::memcpy(&mc, &h.mincol, 8);
  *ok_nn = *ok_tn = 0;
  if (h.nonfinite) return 0;  // NaN / Inf (or |a| > ~1e154): the DMMA GEMM propagates them like BLAS
  if (mx == 0.0) {            // A = 0: exact either way
    *ok_nn = *ok_tn = 1;
    return 0;
  }
  if (mx < 0x1p-960) return 0;  // every row and column norm below 2^-480: the scale would leave the normal range
  // Integer-valued A: exact linear dependencies among its rows / columns survive
  // the engine's exactly-rounded products, so a rank-deficient sketch gets
  // EXACT zero pivots where BLAS's accumulation noise leaves tiny non-zero ones
  // (the reference then passes through instead of raising RankCollapse,
  // rlra/rangefinder.py:55-64).  Such inputs take the DMMA GEMM.
  if (h.nonint == 0u) return 0;
  // rho^2 = max / min of the sums of squares; a minimum below DBL_MIN (a zero
  // row, or squares that underflow) is rejected
  auto ok = [&](unsigned long long minbits, double mn, int64_t k) {
    if (minbits == ~0ull) return 1;
    const double lim = oz_guard_limit(k);
    return (mn >= 2.2250738585072014e-308 && mx <= lim * lim * mn) ? 1 : 0;
  };
  *ok_nn = ok(h.minrow, mr, n);  // C = A B: rows of A, K = n
  *ok_tn = ok(h.mincol, mc, m);  // C = A^T B: columns of A, K = m
  return 0;
}

int oz_prep_ex(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, const int* e_a_ext, void* prep,
               size_t prep_bytes, cudaStream_t st) {
  RLRA_REQUIRE(nmod >= 12 && nmod <= oz::kMaxMod, "oz_prep: nmod must be in [12, 16], got %d", nmod);
  RLRA_REQUIRE(m >= 1 && n >= 1 && lda >= m, "oz_prep: bad shape m=%lld n=%lld lda=%lld", (long long)m,
               (long long)n, (long long)lda);
  const oz::PrepLayout p = oz::prep_layout(m, n, nmod);
  RLRA_REQUIRE(prep && prep_bytes >= p.total, "oz_prep: workspace too small (%zu < %zu)", prep_bytes, p.total);
  RLRA_REQUIRE(p.njb <= 65535, "oz_prep: n too large (%lld)", (long long)n);
  uint8_t* base = static_cast<uint8_t*>(prep);
  oz::OzHeader* hdr = reinterpret_cast<oz::OzHeader*>(base + p.off_hdr);
  int* e_a = &hdr->e_a;
  double* prow = reinterpret_cast<double*>(base + p.off_prow);
  double* pcol = reinterpret_cast<double*>(base + p.off_pcol);
  int8_t* tiles = reinterpret_cast<int8_t*>(base + p.off_tiles);
  if (e_a_ext) {  // scale of an enclosing matrix (block-wise residues), or of this prep (oz_norms_prep)
    if (e_a_ext != e_a) RLRA_CHECK_CUDA(cudaMemcpyAsync(e_a, e_a_ext, sizeof(int), cudaMemcpyDeviceToDevice, st));
  } else {
    const int rc = oz_norms(a, lda, m, n, nmod, e_a, hdr, prow, pcol, st);
    if (rc) return rc;
  }
  ktimer_mark(KT_OZ_RESIDUE_A, st, false);
  OZ_DISPATCH(nmod, oz::launch_residue_a, a, lda, m, n, e_a, tiles, p, st);
  ktimer_mark(KT_OZ_RESIDUE_A, st, true);
  RLRA_LAUNCHED();
  return 0;
}

// Norms, scale and guard statistics into a prep workspace, without residues
// (the caller reads the header, then calls oz_prep_ex(e_a = the header's) for
// the residues only when an orientation passes the guard).
int oz_norms_prep(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, void* prep, size_t prep_bytes,
                  cudaStream_t st) {
  RLRA_REQUIRE(nmod >= 12 && nmod <= oz::kMaxMod, "oz_norms: nmod must be in [12, 16], got %d", nmod);
  RLRA_REQUIRE(m >= 1 && n >= 1 && lda >= m, "oz_norms: bad shape m=%lld n=%lld lda=%lld", (long long)m,
               (long long)n, (long long)lda);
  const oz::PrepLayout p = oz::prep_layout(m, n, nmod);
  RLRA_REQUIRE(prep && prep_bytes >= p.total, "oz_norms: workspace too small (%zu < %zu)", prep_bytes, p.total);
  uint8_t* base = static_cast<uint8_t*>(prep);
  oz::OzHeader* hdr = reinterpret_cast<oz::OzHeader*>(base + p.off_hdr);
  return oz_norms(a, lda, m, n, nmod, &hdr->e_a, hdr, reinterpret_cast<double*>(base + p.off_prow),
                  reinterpret_cast<double*>(base + p.off_pcol), st);
}

// ---- pipelined upload (column chunks of A land one after the other):
// norms per chunk, a provisional eA after the first chunk, residues per chunk,
// then the final norms / guard statistics and the final eA.
int oz_norms_cols(const double* a, int64_t lda, int64_t m, int64_t n, int64_t c0, int64_t c1, int nmod, void* prep,
                  size_t prep_bytes, cudaStream_t st) {
  const oz::PrepLayout p = oz::prep_layout(m, n, nmod);
  RLRA_REQUIRE(prep && prep_bytes >= p.total, "oz_norms_cols: workspace too small");
  RLRA_REQUIRE(c0 >= 0 && c0 < c1 && c1 <= n && c0 % oz::kNormCols == 0 && (c1 % oz::kNormCols == 0 || c1 == n),
               "oz_norms_cols: chunk [%lld, %lld) not aligned to %d columns", (long long)c0, (long long)c1,
               oz::kNormCols);
  uint8_t* base = static_cast<uint8_t*>(prep);
  const int64_t nrb = ceil_div(m, oz::kNormRows);
  const int64_t cb0 = c0 / oz::kNormCols, cb1 = ceil_div(c1, oz::kNormCols);
  RLRA_CHECK_CUDA(cudaFuncSetAttribute(oz::norms_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)oz::kNormSmem));
  oz::norms_partial_kernel<<<dim3((unsigned)nrb, (unsigned)(cb1 - cb0)), 256, oz::kNormSmem, st>>>(
      a, lda, m, n, reinterpret_cast<double*>(base + p.off_prow), reinterpret_cast<double*>(base + p.off_pcol),
      reinterpret_cast<oz::OzHeader*>(base + p.off_hdr), cb0);
  RLRA_LAUNCHED();
  return 0;
}

int oz_scale_provisional(int64_t m, int64_t n, int64_t c1, int nmod, void* prep, size_t prep_bytes, cudaStream_t st) {
  const oz::PrepLayout p = oz::prep_layout(m, n, nmod);
  RLRA_REQUIRE(prep && prep_bytes >= p.total && c1 >= 1 && c1 <= n, "oz_scale_provisional: bad arguments");
  uint8_t* base = static_cast<uint8_t*>(prep);
  oz::scale_estimate_kernel<<<1, 1024, 0, st>>>(reinterpret_cast<double*>(base + p.off_prow), m,
                                                reinterpret_cast<double*>(base + p.off_pcol),
                                                ceil_div(m, oz::kNormRows), n, c1, oz::budget(nmod).pa,
                                                reinterpret_cast<oz::OzHeader*>(base + p.off_hdr));
  RLRA_LAUNCHED();
  return 0;
}

int oz_residue_cols(const double* a, int64_t lda, int64_t m, int64_t n, int64_t c0, int64_t c1, int nmod, void* prep,
                    size_t prep_bytes, cudaStream_t st) {
  const oz::PrepLayout p = oz::prep_layout(m, n, nmod);
  RLRA_REQUIRE(prep && prep_bytes >= p.total, "oz_residue_cols: workspace too small");
  RLRA_REQUIRE(c0 >= 0 && c0 < c1 && c1 <= n && c0 % oz::kTile == 0 && (c1 % oz::kTile == 0 || c1 == n),
               "oz_residue_cols: chunk [%lld, %lld) not aligned to %d columns", (long long)c0, (long long)c1, oz::kTile);
  uint8_t* base = static_cast<uint8_t*>(prep);
  const int* e_a = &reinterpret_cast<oz::OzHeader*>(base + p.off_hdr)->e_a;
  int8_t* tiles = reinterpret_cast<int8_t*>(base + p.off_tiles);
  const int64_t jb0 = c0 / oz::kTile;
  int64_t jb1 = ceil_div(c1, oz::kTile);
  if (c1 == n) jb1 = p.njb;  // the padding tile column (njb is even) belongs to the last chunk
  OZ_DISPATCH(nmod, oz::launch_residue_a_cols, a, lda, m, n, e_a, tiles, p, jb0, jb1, st);
  RLRA_LAUNCHED();
  return 0;
}

int oz_norms_finish(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, void* prep, size_t prep_bytes,
                    int* e_a_final, cudaStream_t st) {
  const oz::PrepLayout p = oz::prep_layout(m, n, nmod);
  RLRA_REQUIRE(prep && prep_bytes >= p.total && e_a_final, "oz_norms_finish: bad arguments");
  uint8_t* base = static_cast<uint8_t*>(prep);
  oz::OzHeader* hdr = reinterpret_cast<oz::OzHeader*>(base + p.off_hdr);
  double* prow = reinterpret_cast<double*>(base + p.off_prow);
  double* pcol = reinterpret_cast<double*>(base + p.off_pcol);
  const int64_t ncb = ceil_div(n, oz::kNormCols), nrb = ceil_div(m, oz::kNormRows);
  oz::norms_final_kernel<<<(unsigned)ceil_div(m + n, 256), 256, 0, st>>>(prow, ncb, m, pcol, nrb, n, hdr, a, lda);
  RLRA_LAUNCHED();
  oz::scale_a_kernel<<<1, 1, 0, st>>>(hdr, oz::budget(nmod).pa, e_a_final);
  RLRA_LAUNCHED();
  oz::fro2_kernel<<<1, 1024, 0, st>>>(pcol, nrb * n, hdr);
  RLRA_LAUNCHED();
  return 0;
}

int oz_prep(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, void* prep, size_t prep_bytes,
            cudaStream_t st) {
  return oz_prep_ex(a, lda, m, n, nmod, nullptr, prep, prep_bytes, st);
}

int64_t oz_cols_pad(int64_t ncols) {
  const oz::PrepLayout p = oz::prep_layout(1, 1, 14);
  return oz::gemm_layout(p, 0, ncols < 1 ? 1 : ncols, 14).cols_pad;
}

int oz_bscale(const double* b, int64_t ldb, int64_t k, int64_t ncols, int nmod, int* e_b, cudaStream_t st) {
  RLRA_REQUIRE(nmod >= 12 && nmod <= oz::kMaxMod, "oz_bscale: nmod must be in [12, 16], got %d", nmod);
  RLRA_REQUIRE(k >= 1 && ncols >= 1 && ldb >= k && e_b, "oz_bscale: bad arguments");
  const int64_t cp = oz_cols_pad(ncols);
  oz::bscale_kernel<<<(unsigned)cp, 256, 0, st>>>(b, ldb, k, ncols, cp, oz::budget(nmod).pb, e_b);
  RLRA_LAUNCHED();
  return 0;
}

size_t oz_gemm_workspace(int trans, int64_t m, int64_t n, int64_t ncols, int nmod) {
  if (nmod < 12 || nmod > oz::kMaxMod || m < 1 || n < 1 || ncols < 1) return 0;
  const oz::PrepLayout p = oz::prep_layout(m, n, nmod);
  return oz::gemm_layout(p, trans, ncols, nmod).total;
}

int oz_gemm_ex(int trans, const void* prep, int64_t m, int64_t n, int nmod, const double* b, int64_t ldb,
               int64_t ncols, double* c, int64_t ldc, void* ws, size_t ws_bytes, const int* e_b_ext, int flags,
               cudaStream_t st) {
  RLRA_REQUIRE(nmod >= 12 && nmod <= oz::kMaxMod, "oz_gemm: nmod must be in [12, 16], got %d", nmod);
  const int64_t K = trans ? m : n, mrows = trans ? n : m;
  RLRA_REQUIRE(ncols >= 0 && ldb >= K && ldc >= mrows, "oz_gemm: bad leading dimensions");
  if (ncols == 0) return 0;
  const oz::PrepLayout p = oz::prep_layout(m, n, nmod);
  const oz::GemmLayout g = oz::gemm_layout(p, trans, ncols, nmod);
  RLRA_REQUIRE(ws && ws_bytes >= g.total, "oz_gemm: workspace too small (%zu < %zu)", ws_bytes, g.total);
  RLRA_REQUIRE(g.nkb * oz::kTile <= oz::kMaxK, "oz_gemm: K=%lld exceeds the exact int32 range",
               (long long)(g.nkb * oz::kTile));
  RLRA_REQUIRE(g.cols_pad <= 65535, "oz_gemm: too many columns (%lld)", (long long)ncols);
  const uint8_t* pb = static_cast<const uint8_t*>(prep);
  const int* e_a = reinterpret_cast<const int*>(pb + p.off_hdr);
  const int8_t* a_tiles = reinterpret_cast<const int8_t*>(pb + p.off_tiles);
  uint8_t* w = static_cast<uint8_t*>(ws);
  int* e_b = e_b_ext ? const_cast<int*>(e_b_ext) : reinterpret_cast<int*>(w + g.off_eb);
  int8_t* b_tiles = reinterpret_cast<int8_t*>(w + g.off_b);
  uint8_t* tout = w + g.off_t;
  const oz::Budget bud = oz::budget(nmod);
  if (!(flags & 16)) {  // RLRA_B200_OZ_REUSE_B: the workspace still holds this B's scales and residues
    ktimer_mark(KT_OZ_RESIDUE_B, st, false);
    OZ_DISPATCH(nmod, oz::launch_residue_b, b, ldb, K, ncols, g, bud.pb, e_b, b_tiles, e_b_ext == nullptr, st);
    ktimer_mark(KT_OZ_RESIDUE_B, st, true);
    RLRA_LAUNCHED();
    note_launch();  // bscale + residue_b
  }

  oz::GemmArgs ga;
  ga.a_tiles = a_tiles;
  ga.nib = p.nib;
  ga.njb = p.njb;
  ga.trans = trans;
  ga.b_tiles = b_tiles;
  ga.ng = g.ng;
  ga.n_g = g.n_g;
  ga.nkb = g.nkb;
  ga.nmb = g.nmb;
  ga.out = tout;
  ga.nmod = nmod;
  ga.accum = (flags & 1) ? 1 : 0;
  const oz::Crt crt = oz::make_crt(nmod);
  for (int l = 0; l < oz::kMaxMod; ++l) {
    ga.mods[l] = oz::kModuli[l];
    ga.ys[l] = l < nmod ? crt.y[l] : 1;
  }
  const size_t smem = oz::gemm_smem_bytes(g.n_g);
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(oz::gemm_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)oz::gemm_smem_bytes(256));
  });
  RLRA_CHECK_CUDA(attr_err);
  const int64_t units = (int64_t)nmod * g.nmb * g.ng;
  const int grid = (int)std::min<int64_t>(units, device_info().sm_count);
  ktimer_mark(KT_OZ_GEMM, st, false);
  oz::gemm_i8_kernel<<<grid, oz::kGemmThreads, smem, st>>>(ga);
  ktimer_mark(KT_OZ_GEMM, st, true);
  RLRA_LAUNCHED();

  if (flags & 2) return 0;  // RLRA_B200_OZ_NO_CRT: more K blocks follow
  ktimer_mark(KT_OZ_CRT, st, false);
  RLRA_REQUIRE(ceil_div(mrows, 1024) <= g.nblk, "oz_gemm: CRT grid exceeds the partial buffer");
  const dim3 cgrid((unsigned)ceil_div(mrows, 1024), (unsigned)ncols);
  if (flags & 8)
    oz::crt_kernel<true><<<cgrid, 256, 0, st>>>(tout, g.rows_pad, g.cols_pad, mrows, ncols, e_a, e_b, crt, c, ldc,
                                                (flags & 4) ? 1 : 0, reinterpret_cast<double2*>(w + g.off_colsq));
  else
    oz::crt_kernel<false><<<cgrid, 256, 0, st>>>(tout, g.rows_pad, g.cols_pad, mrows, ncols, e_a, e_b, crt, c, ldc,
                                                 (flags & 4) ? 1 : 0, nullptr);
  ktimer_mark(KT_OZ_CRT, st, true);
  RLRA_LAUNCHED();
  return 0;
}

// Column energies of the C written by the last oz_gemm_ex call with
// RLRA_B200_OZ_COLSQ on this workspace (same trans / m / n / nmod / ncols).
int oz_colsq(int trans, int64_t m, int64_t n, int nmod, int64_t ncols, const void* ws, size_t ws_bytes, double* out,
             int accumulate, cudaStream_t st) {
  RLRA_REQUIRE(nmod >= 12 && nmod <= oz::kMaxMod, "oz_colsq: nmod must be in [12, 16], got %d", nmod);
  if (ncols <= 0) return 0;
  const oz::PrepLayout p = oz::prep_layout(m, n, nmod);
  const oz::GemmLayout g = oz::gemm_layout(p, trans, ncols, nmod);
  RLRA_REQUIRE(ws && ws_bytes >= g.total && out, "oz_colsq: workspace too small (%zu < %zu)", ws_bytes, g.total);
  const int64_t mrows = trans ? n : m;
  const double2* part = reinterpret_cast<const double2*>(static_cast<const uint8_t*>(ws) + g.off_colsq);
  oz::colsq_finish_kernel<<<(unsigned)ceil_div(ncols, 8), 256, 0, st>>>(part, ceil_div(mrows, 1024), ncols, out,
                                                                        accumulate);
  RLRA_LAUNCHED();
  return 0;
}

int oz_gemm(int trans, const void* prep, int64_t m, int64_t n, int nmod, const double* b, int64_t ldb,
            int64_t ncols, double* c, int64_t ldc, void* ws, size_t ws_bytes, cudaStream_t st) {
  return oz_gemm_ex(trans, prep, m, n, nmod, b, ldb, ncols, c, ldc, ws, ws_bytes, nullptr, 0, st);
}

}  // namespace rlra
