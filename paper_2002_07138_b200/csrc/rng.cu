// Omega on the device, bit-identical to the reference's host draw
//   np.random.default_rng(seed).standard_normal(N)        (rlra/core.py:33-48)
// i.e. NumPy's PCG64 (128-bit LCG, XSL-RR output) feeding its 256-layer
// Marsaglia-Tsang ziggurat.  The draw is sequential by definition (a normal
// consumes a variable number of 64-bit words), so it is parallelised as:
//   1. raw stream: every thread jumps its PCG64 to its chunk (O(log k) 128-bit
//      LCG advance) and emits 64 consecutive XSL-RR words;
//   2. classify every word position s as the START of a normal: its length
//      len(s) (words consumed) and value, entirely on the device except the
//      rare tail draws (|x| > r, ~1 in 3900) whose log1p results must match
//      the host libm bit for bit -- those few are resolved by the host
//      (paper_2002_07138_b200/core.py) between the two phases;
//   3. the real starts are the path 0 -> 0+len(0) -> ...; chunks of 256
//      positions are summarised as functions entry offset -> (exit offset,
//      count) (a finite-state transducer, entry offsets < 16), composed by a
//      hierarchical fixed-order scan, and each chunk finally writes its
//      normals at their global indices (column-major Omega == flat order).
#include "common.cuh"

namespace rlra {

typedef unsigned __int128 u128;

constexpr int RNG_CHUNK = 256;  // positions per transducer chunk
constexpr int RNG_E = 16;       // entry offsets tracked per chunk (max len - 1 < 16)
constexpr int RNG_GROUP = 128;  // functions composed per scan thread
constexpr int RNG_WORDS_PER_THREAD = 64;
constexpr int LEN_TAIL = -1, LEN_CONT = -2, LEN_UNKNOWN = -3;

__host__ __device__ inline u128 make_u128(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const uint64_t x = hi ^ lo;
  const unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__global__ void pcg_stream_kernel(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                                  int64_t T, uint64_t* __restrict__ u) {
  const u128 MULT = make_u128(0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull);
  const u128 inc = make_u128(i_hi, i_lo);
  const int64_t p0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * RNG_WORDS_PER_THREAD;
  if (p0 >= T) return;
  // advance the state by p0 steps (Brown's LCG jump, as pcg_advance_lcg_128)
  u128 acc_mult = 1, acc_plus = 0, cur_mult = MULT, cur_plus = inc;
  uint64_t k = (uint64_t)p0;
  while (k) {
    if (k & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    k >>= 1;
  }
  u128 s = acc_mult * make_u128(s_hi, s_lo) + acc_plus;
  const int64_t p1 = min(T, p0 + RNG_WORDS_PER_THREAD);
  for (int64_t p = p0; p < p1; p++) {
    s = s * MULT + inc;  // NumPy steps first, then outputs the new state
    u[p] = xsl_rr(s);
  }
}

__device__ __forceinline__ double u64_to_double(uint64_t r) {
  return (double)(r >> 11) * (1.0 / 9007199254740992.0);
}

// len/val of a normal starting at word s (random_standard_normal, one pass of
// its outer loop); tails are left to the host, rejections chain to s + 2.
__global__ void zig_classify_kernel(const uint64_t* __restrict__ u, int64_t T, const uint64_t* __restrict__ ki,
                                    const double* __restrict__ wi, const double* __restrict__ fi,
                                    int* __restrict__ len, double* __restrict__ val,
                                    int64_t* __restrict__ tail_pos, unsigned long long* __restrict__ ntail,
                                    int64_t tail_cap) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < T;
       s += (int64_t)gridDim.x * blockDim.x) {
    uint64_t r = u[s];
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = __dmul_rn((double)rabs, wi[idx]);
    if (sign) x = -x;
    if (rabs < ki[idx]) {
      len[s] = 1;
      val[s] = x;
    } else if (idx == 0) {
      len[s] = LEN_TAIL;
      val[s] = 0.0;
      const unsigned long long slot = atomicAdd(ntail, 1ull);
      if ((int64_t)slot < tail_cap) tail_pos[slot] = s;
    } else if (s + 1 >= T) {
      len[s] = LEN_UNKNOWN;
      val[s] = 0.0;
    } else {
      // (fi[idx-1] - fi[idx]) * U + fi[idx] < exp(-0.5 * x * x), unfused like NumPy
      const double U = u64_to_double(u[s + 1]);
      const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(fi[idx - 1], fi[idx]), U), fi[idx]);
      const double rhs = exp(__dmul_rn(__dmul_rn(-0.5, x), x));
      if (lhs < rhs) {
        len[s] = 2;
        val[s] = x;
      } else {
        len[s] = LEN_CONT;  // outer loop restarts at s + 2
        val[s] = 0.0;
      }
    }
  }
}

__global__ void zig_scatter_tails_kernel(const int64_t* __restrict__ pos, const int* __restrict__ tl,
                                         const double* __restrict__ tv, int64_t n, int* __restrict__ len,
                                         double* __restrict__ val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    len[pos[i]] = tl[i];
    val[pos[i]] = tv[i];
  }
}

// Resolve rejection chains: len(s) = 2 + len(s + 2), value of the terminal.
// Reads `len`, writes `len2` (so chain walks never see half-updated entries);
// terminals are never CONT, so their `val` is only read here.
__global__ void zig_chain_kernel(int64_t T, const int* __restrict__ len, int* __restrict__ len2,
                                 double* __restrict__ val, int* __restrict__ flag) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < T;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int L0 = len[s];
    if (L0 != LEN_CONT) {
      len2[s] = L0;
      continue;
    }
    int64_t t = s;
    int total = 0;
    while (t < T && len[t] == LEN_CONT) {
      t += 2;
      total += 2;
    }
    const int L = (t < T) ? len[t] : LEN_UNKNOWN;
    if (L > 0 && total + L <= RNG_E) {
      len2[s] = total + L;
      val[s] = val[t];
    } else {
      len2[s] = LEN_UNKNOWN;
      if (L > 0) atomicOr(flag, 1);
    }
  }
}

// Chunk transducer: entry offset e -> (exit offset, number of normals started).
// One thread per chunk; the e = 0 path is walked once and remembered so the
// other entries stop as soon as they merge into it.
__global__ void zig_chunk_fn_kernel(const int* __restrict__ len, int64_t T, int64_t nchunks,
                                    int8_t* __restrict__ fexit, int32_t* __restrict__ fcnt,
                                    int* __restrict__ flag) {
  __shared__ int16_t kat[64][RNG_CHUNK];
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  int16_t* k_at = kat[threadIdx.x];
  for (int i = 0; i < RNG_CHUNK; i++) k_at[i] = -1;
  const int64_t base = c * RNG_CHUNK, end = base + RNG_CHUNK;
  int64_t pos = base;
  int cnt0 = 0;
  bool bad = false;
  while (pos < end) {
    k_at[pos - base] = (int16_t)cnt0;
    const int L = pos < T ? len[pos] : LEN_UNKNOWN;
    if (L <= 0) { bad = true; break; }
    pos += L;
    cnt0++;
  }
  const int exit0 = bad ? -1 : (int)(pos - end);
  for (int e = 0; e < RNG_E; e++) {
    int ex, cnt;
    if (e == 0) {
      ex = exit0;
      cnt = cnt0;
    } else {
      int64_t p = base + e;
      int steps = 0;
      bool b2 = false;
      while (p < end && k_at[p - base] < 0) {
        const int L = p < T ? len[p] : LEN_UNKNOWN;
        if (L <= 0) { b2 = true; break; }
        p += L;
        steps++;
      }
      if (b2) { ex = -1; cnt = 0; }
      else if (p >= end) { ex = (int)(p - end); cnt = steps; }
      else { ex = exit0; cnt = exit0 < 0 ? 0 : steps + (cnt0 - k_at[p - base]); }
    }
    if (ex >= RNG_E) atomicOr(flag, 2);
    fexit[c * RNG_E + e] = (int8_t)(ex < RNG_E ? ex : -1);
    fcnt[c * RNG_E + e] = cnt;
  }
}

// Compose groups of RNG_GROUP consecutive functions (fixed order).
__global__ void zig_compose_kernel(const int8_t* __restrict__ fe, const int32_t* __restrict__ fc, int64_t n,
                                   int8_t* __restrict__ ge, int64_t* __restrict__ gc) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t n_groups = ceil_div(n, RNG_GROUP);
  if (g >= n_groups) return;
  const int64_t i0 = g * RNG_GROUP, i1 = min(n, i0 + RNG_GROUP);
  for (int e = 0; e < RNG_E; e++) {
    int state = e;
    int64_t cnt = 0;
    for (int64_t i = i0; i < i1 && state >= 0; i++) {
      cnt += fc[i * RNG_E + state];
      state = fe[i * RNG_E + state];
    }
    ge[g * RNG_E + e] = (int8_t)state;
    gc[g * RNG_E + e] = state >= 0 ? cnt : 0;
  }
}
// Same, for 64-bit counts at the upper levels.
__global__ void zig_compose64_kernel(const int8_t* __restrict__ fe, const int64_t* __restrict__ fc, int64_t n,
                                     int8_t* __restrict__ ge, int64_t* __restrict__ gc) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t n_groups = ceil_div(n, RNG_GROUP);
  if (g >= n_groups) return;
  const int64_t i0 = g * RNG_GROUP, i1 = min(n, i0 + RNG_GROUP);
  for (int e = 0; e < RNG_E; e++) {
    int state = e;
    int64_t cnt = 0;
    for (int64_t i = i0; i < i1 && state >= 0; i++) {
      cnt += fc[i * RNG_E + state];
      state = fe[i * RNG_E + state];
    }
    ge[g * RNG_E + e] = (int8_t)state;
    gc[g * RNG_E + e] = state >= 0 ? cnt : 0;
  }
}

// Walk n functions from entry 0 sequentially (top level, one thread), writing
// each function's entry state and prefix count.
template <typename CNT>
__global__ void zig_top_scan_kernel(const int8_t* __restrict__ fe, const CNT* __restrict__ fc, int64_t n,
                                    int8_t* __restrict__ entry, int64_t* __restrict__ prefix) {
  if (threadIdx.x || blockIdx.x) return;
  int state = 0;
  int64_t cnt = 0;
  for (int64_t i = 0; i < n; i++) {
    entry[i] = (int8_t)state;
    prefix[i] = cnt;
    if (state < 0) continue;
    cnt += fc[i * RNG_E + state];
    state = fe[i * RNG_E + state];
  }
}

// Propagate a group's entry/prefix to its member functions.
template <typename CNT>
__global__ void zig_propagate_kernel(const int8_t* __restrict__ fe, const CNT* __restrict__ fc, int64_t n,
                                     const int8_t* __restrict__ gentry, const int64_t* __restrict__ gprefix,
                                     int8_t* __restrict__ entry, int64_t* __restrict__ prefix) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t n_groups = ceil_div(n, RNG_GROUP);
  if (g >= n_groups) return;
  int state = gentry[g];
  int64_t cnt = gprefix[g];
  const int64_t i0 = g * RNG_GROUP, i1 = min(n, i0 + RNG_GROUP);
  for (int64_t i = i0; i < i1; i++) {
    entry[i] = (int8_t)state;
    prefix[i] = cnt;
    if (state < 0) continue;
    cnt += fc[i * RNG_E + state];
    state = fe[i * RNG_E + state];
  }
}

// Final walk: chunk c emits its normals at global indices prefix[c] ...
__global__ void zig_emit_kernel(const int* __restrict__ len, const double* __restrict__ val, int64_t T,
                                int64_t nchunks, const int8_t* __restrict__ entry,
                                const int64_t* __restrict__ prefix, int64_t N, double* __restrict__ out,
                                unsigned long long* __restrict__ produced, int64_t* __restrict__ consumed) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  if (entry[c] < 0) return;
  const int64_t base = c * RNG_CHUNK, end = base + RNG_CHUNK;
  int64_t pos = base + entry[c];
  int64_t k = prefix[c];
  while (pos < end && k < N) {
    const int L = len[pos];
    if (L <= 0) break;
    out[k] = val[pos];
    k++;
    pos += L;
    if (k == N) *consumed = pos;  // words used by the N normals (stream continuation)
  }
  if (k >= N || pos >= end) {
    if (k > prefix[c]) atomicMax(produced, (unsigned long long)k);
  }
}

// ------------------------------------------------------------------ host side
static size_t al8(size_t x) { return (x + 255) & ~(size_t)255; }

struct RngLayout {
  size_t u, len, len2, val, tail_pos, ntail, flag, produced, levels, total;
};

static RngLayout rng_layout(int64_t T, int64_t tail_cap) {
  RngLayout L{};
  size_t o = 0;
  auto take = [&](size_t& off, size_t b) { off = o; o += al8(b); };
  take(L.u, (size_t)T * 8);
  take(L.len, (size_t)T * 4);
  take(L.len2, (size_t)T * 4);
  take(L.val, (size_t)T * 8);
  take(L.tail_pos, (size_t)tail_cap * 8);
  take(L.ntail, 8);
  take(L.flag, 8);
  take(L.produced, 8);
  // transducer levels: chunk functions + group functions + entries/prefixes
  const int64_t nch = ceil_div(T, RNG_CHUNK);
  size_t lv = 0;
  int64_t n = nch;
  lv += al8(n * RNG_E) + al8(n * RNG_E * 4) + al8(n) + al8(n * 8);
  while (n > 1) {
    n = ceil_div(n, RNG_GROUP);
    lv += al8(n * RNG_E) + al8(n * RNG_E * 8) + al8(n) + al8(n * 8);
  }
  take(L.levels, lv + 4096);
  L.total = o;
  return L;
}

int64_t normal_stream_words(int64_t N) { return N + N / 8 + 8192; }
int64_t normal_tail_cap(int64_t N) { return normal_stream_words(N) / 512 + 4096; }

size_t normal_workspace_bytes(int64_t N) {
  return rng_layout(normal_stream_words(N), normal_tail_cap(N)).total;
}

static int grid_of(int64_t n, int threads) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), (int64_t)device_info().sm_count * 32));
}

// Phase 1: raw stream + classification.  *ntail_dev (device u64) receives the
// number of tail starts, tail_pos_out (device int64[cap]) their positions;
// u_out points at the raw words (for the host tail resolution).
int normal_phase1(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, int64_t N,
                  const uint64_t* ki, const double* wi, const double* fi, void* ws, size_t ws_bytes,
                  cudaStream_t st) {
  const int64_t T = normal_stream_words(N), cap = normal_tail_cap(N);
  RngLayout L = rng_layout(T, cap);
  RLRA_REQUIRE(ws && ws_bytes >= L.total, "normal: workspace too small (%zu < %zu)", ws_bytes, L.total);
  char* b = static_cast<char*>(ws);
  uint64_t* u = reinterpret_cast<uint64_t*>(b + L.u);
  RLRA_CHECK_CUDA(cudaMemsetAsync(b + L.ntail, 0, 3 * 256, st));
  const int64_t nthreads = ceil_div(T, RNG_WORDS_PER_THREAD);
  pcg_stream_kernel<<<(unsigned)ceil_div(nthreads, 128), 128, 0, st>>>(s_hi, s_lo, i_hi, i_lo, T, u);
  RLRA_LAUNCHED();
  zig_classify_kernel<<<grid_of(T, 256), 256, 0, st>>>(
      u, T, ki, wi, fi, reinterpret_cast<int*>(b + L.len), reinterpret_cast<double*>(b + L.val),
      reinterpret_cast<int64_t*>(b + L.tail_pos), reinterpret_cast<unsigned long long*>(b + L.ntail), cap);
  RLRA_LAUNCHED();
  return 0;
}

// Workspace views for the host's tail step.
int normal_views(int64_t N, void* ws, uint64_t** u, int64_t** tail_pos, unsigned long long** ntail) {
  RngLayout L = rng_layout(normal_stream_words(N), normal_tail_cap(N));
  char* b = static_cast<char*>(ws);
  *u = reinterpret_cast<uint64_t*>(b + L.u);
  *tail_pos = reinterpret_cast<int64_t*>(b + L.tail_pos);
  *ntail = reinterpret_cast<unsigned long long*>(b + L.ntail);
  return 0;
}

// Phase 2: install the host-resolved tails, resolve rejection chains, run the
// transducer scan and emit N normals to out.  *status_dev (device int64):
// [0] normals produced (== N on success), [1] failure flags (0 on success),
// [2] 64-bit words consumed (to continue the stream in the next chunk).
int normal_phase2(int64_t N, const int64_t* tpos, const int* tlen, const double* tval, int64_t ntail,
                  double* out, int64_t* status_dev, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int64_t T = normal_stream_words(N), cap = normal_tail_cap(N);
  RngLayout L = rng_layout(T, cap);
  RLRA_REQUIRE(ws && ws_bytes >= L.total, "normal: workspace too small");
  char* b = static_cast<char*>(ws);
  int* len = reinterpret_cast<int*>(b + L.len);
  double* val = reinterpret_cast<double*>(b + L.val);
  int* flag = reinterpret_cast<int*>(b + L.flag);
  unsigned long long* produced = reinterpret_cast<unsigned long long*>(b + L.produced);
  if (ntail > 0) {
    zig_scatter_tails_kernel<<<grid_of(ntail, 256), 256, 0, st>>>(tpos, tlen, tval, ntail, len, val);
    RLRA_LAUNCHED();
  }
  int* len2 = reinterpret_cast<int*>(b + L.len2);
  zig_chain_kernel<<<grid_of(T, 256), 256, 0, st>>>(T, len, len2, val, flag);
  RLRA_LAUNCHED();
  len = len2;
  // ---- transducer levels
  const int64_t nch = ceil_div(T, RNG_CHUNK);
  char* lv = b + L.levels;
  auto carve = [&](size_t bytes) { char* p = lv; lv += al8(bytes); return p; };
  int8_t* fe0 = reinterpret_cast<int8_t*>(carve(nch * RNG_E));
  int32_t* fc0 = reinterpret_cast<int32_t*>(carve(nch * RNG_E * 4));
  int8_t* en0 = reinterpret_cast<int8_t*>(carve(nch));
  int64_t* pf0 = reinterpret_cast<int64_t*>(carve(nch * 8));
  zig_chunk_fn_kernel<<<(unsigned)ceil_div(nch, 64), 64, 0, st>>>(len, T, nch, fe0, fc0, flag);
  RLRA_LAUNCHED();
  // up-sweep
  struct Level { int8_t* fe; int64_t* fc; int8_t* en; int64_t* pf; int64_t n; };
  Level lvls[16];
  int nl = 0;
  int64_t n = nch;
  while (n > RNG_GROUP) {
    const int64_t ng = ceil_div(n, RNG_GROUP);
    Level g{reinterpret_cast<int8_t*>(carve(ng * RNG_E)), reinterpret_cast<int64_t*>(carve(ng * RNG_E * 8)),
            reinterpret_cast<int8_t*>(carve(ng)), reinterpret_cast<int64_t*>(carve(ng * 8)), ng};
    if (nl == 0)
      zig_compose_kernel<<<(unsigned)ceil_div(ng, 128), 128, 0, st>>>(fe0, fc0, n, g.fe, g.fc);
    else
      zig_compose64_kernel<<<(unsigned)ceil_div(ng, 128), 128, 0, st>>>(lvls[nl - 1].fe, lvls[nl - 1].fc, n,
                                                                         g.fe, g.fc);
    RLRA_LAUNCHED();
    lvls[nl++] = g;
    n = ng;
    RLRA_REQUIRE(nl < 15, "normal: too many scan levels");
  }
  // top: sequential scan of the last level (<= RNG_GROUP functions), then down-sweep
  if (nl == 0) {
    zig_top_scan_kernel<int32_t><<<1, 1, 0, st>>>(fe0, fc0, nch, en0, pf0);
    RLRA_LAUNCHED();
  } else {
    Level& top = lvls[nl - 1];
    zig_top_scan_kernel<int64_t><<<1, 1, 0, st>>>(top.fe, top.fc, top.n, top.en, top.pf);
    RLRA_LAUNCHED();
    for (int i = nl - 1; i >= 1; i--) {
      zig_propagate_kernel<int64_t><<<(unsigned)ceil_div(ceil_div(lvls[i - 1].n, RNG_GROUP), 128), 128, 0, st>>>(
          lvls[i - 1].fe, lvls[i - 1].fc, lvls[i - 1].n, lvls[i].en, lvls[i].pf, lvls[i - 1].en, lvls[i - 1].pf);
      RLRA_LAUNCHED();
    }
    zig_propagate_kernel<int32_t><<<(unsigned)ceil_div(ceil_div(nch, RNG_GROUP), 128), 128, 0, st>>>(
        fe0, fc0, nch, lvls[0].en, lvls[0].pf, en0, pf0);
    RLRA_LAUNCHED();
  }
  zig_emit_kernel<<<(unsigned)ceil_div(nch, 128), 128, 0, st>>>(len, val, T, nch, en0, pf0, N, out, produced,
                                                                 status_dev + 2);
  RLRA_LAUNCHED();
  // status_dev[0] = normals produced (== N on success), [1] failure flags, [2] set by emit
  RLRA_CHECK_CUDA(cudaMemcpyAsync(status_dev, produced, 8, cudaMemcpyDeviceToDevice, st));
  RLRA_CHECK_CUDA(cudaMemsetAsync(status_dev + 1, 0, 8, st));
  RLRA_CHECK_CUDA(cudaMemcpyAsync(status_dev + 1, flag, 4, cudaMemcpyDeviceToDevice, st));
  return 0;
}

}  // namespace rlra
