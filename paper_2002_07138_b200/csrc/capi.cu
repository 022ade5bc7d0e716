// extern "C" boundary of librlra_b200.so (declared in include/rlra_b200.h).
#include <atomic>
#include <cstdarg>
#include <mutex>
#include <vector>

#include "../../include/rlra_b200.h"
#include "common.cuh"

namespace rlra {

static thread_local char g_err[1024] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* last_error() { return g_err; }

static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static std::atomic<bool> g_ktimer{false};
static std::mutex g_ktimer_mu;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_ktimer_ev[KT_COUNT];
static const char* const kKTimerNames[KT_COUNT] = {"oz_gemm_i8", "oz_residue_a", "oz_norms", "oz_crt",
                                                   "oz_residue_b"};

bool ktimer_on() { return g_ktimer.load(std::memory_order_relaxed); }

void ktimer_mark(int id, cudaStream_t st, bool end) {
  if (!ktimer_on() || id < 0 || id >= KT_COUNT) return;
  std::lock_guard<std::mutex> lock(g_ktimer_mu);
  auto& v = g_ktimer_ev[id];
  if (!end) {
    cudaEvent_t a, b;
    if (cudaEventCreate(&a) != cudaSuccess) return;
    if (cudaEventCreate(&b) != cudaSuccess) {
      cudaEventDestroy(a);
      return;
    }
    cudaEventRecord(a, st);
    v.emplace_back(a, b);
  } else if (!v.empty()) {
    cudaEventRecord(v.back().second, st);
  }
}

const DeviceInfo& device_info() {
  static std::mutex mu;
  static std::vector<DeviceInfo> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if ((int)cache.size() <= dev) cache.resize(dev + 1);
  DeviceInfo& d = cache[dev];
  if (d.sm_count == 0) {
    cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (d.sm_count <= 0) d.sm_count = 148;
  }
  return d;
}

// implemented in the kernel translation units
int gemm(bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
         void* ws, size_t ws_bytes, cudaStream_t st);
size_t gemm_workspace_bytes(int64_t M, int64_t N, int64_t K);
size_t getrf_workspace_bytes(int64_t m, int64_t n);
int getrf(double* a, int64_t lda, int64_t m, int64_t n, int64_t* piv, int64_t* nonzero_diag_dev,
          int* zflag_out, void* ws, size_t ws_bytes, cudaStream_t st);
int fill_iota(int64_t* p, int64_t m, cudaStream_t st);
int getrf_block(double* a, int64_t lda, int64_t m, int64_t j0, int nbo, int64_t* piv, int* zflag_out,
                int64_t* ipiv_out, int64_t* nonzero_out, void* ws, size_t ws_bytes, cudaStream_t st);
int lu_trsm_rows(double* a, int64_t lda, int64_t j0, int nb, int64_t c0, int64_t c1, const int* zflag,
                 cudaStream_t st);
int lu_update_split(double* a, int64_t lda, const double* u, int64_t ldu, int64_t j0, int nb, int64_t r0, int64_t m,
                    int64_t c0, int64_t c1, const int* zflag, cudaStream_t st);
int count_nonzero_diag(const double* a, int64_t lda, int64_t r, int64_t* out_dev, cudaStream_t st);
int lu_basis(const double* lu, int64_t ldlu, int64_t m, int64_t k, const int64_t* piv,
             int64_t* pinv_ws, double* w, int64_t ldw, cudaStream_t st);
int extract_l(const double* lu, int64_t ldlu, int64_t m, int64_t k, double* l, int64_t ldl,
              cudaStream_t st);
int extract_u(const double* lu, int64_t ldlu, int64_t k, int64_t n, double* u, int64_t ldu,
              cudaStream_t st);
size_t geqrf_workspace_bytes(int64_t m, int64_t n);
int geqrf(double* a, int64_t lda, int64_t m, int64_t n, double* tau, void* ws, size_t ws_bytes,
          cudaStream_t st);
int orgqr(const double* a, int64_t lda, int64_t m, int64_t n, double* q, int64_t ldq, void* ws,
          size_t ws_bytes, cudaStream_t st);
int resid_sumsq_block(const double* a, int64_t lda, int64_t m, const int64_t* p, const int64_t* qb, int64_t w,
                      const double* lu, int64_t ldlu, double* partial, cudaStream_t st);
int dd_finish(const double* partial, int64_t nparts, double* out_dev, cudaStream_t st);
int spmm_csr(const int64_t* rowptr, const int64_t* colidx, const double* vals, int64_t rows, const double* x,
             int64_t ldx, int64_t l, double* y, int64_t ldy, cudaStream_t st);
int trsm_un(const double* r, int64_t ldr, int64_t l, double* x, int64_t ldx, int64_t ncols, void* ws,
            size_t ws_bytes, cudaStream_t st);
int apply_inv_row_perm(const int64_t* p, int64_t m, int64_t n, const double* x, int64_t ldx, int64_t* pinv_ws,
                       double* out, int64_t ldo, cudaStream_t st);
int svd_jacobi_max_l();
size_t svd_jacobi_workspace(int64_t m, int64_t l);
int svd_jacobi(const double* a, int64_t lda, int64_t m, int64_t l, double* u, int64_t ldu, double* s, double* v,
               int64_t ldv, int* sweeps_out, void* ws, size_t ws_bytes, cudaStream_t st);
int trsm_rt(const double* r, int64_t ldr, int64_t l, double* x, int64_t ldx, int64_t ncols,
            void* ws, size_t ws_bytes, cudaStream_t st);
int diag_absmin(const double* a, int64_t lda, int64_t r, double* out_dev, cudaStream_t st);
size_t sumsq_workspace_bytes(int64_t m, int64_t n);
int sumsq(const double* a, int64_t lda, int64_t m, int64_t n, double* out_dev, void* ws,
          size_t ws_bytes, cudaStream_t st);
int colsumsq(const double* a, int64_t lda, int64_t m, int64_t n, double* out_dev, cudaStream_t st);
int transpose(const double* in, int64_t ldi, int64_t m, int64_t n, double* out, int64_t ldo,
              cudaStream_t st);
int chol_inv_max_l();
int chol_shift_diag(double* g, int64_t ldg, int64_t l, double c, cudaStream_t st);
int diag_ratio_flag(const double* d, int64_t ldd, int64_t l, double cond_limit, int* flag, cudaStream_t st);
int gram_identity_flag(const double* g, int64_t ldg, int64_t l, double tol, int* flag, cudaStream_t st);
int chol_inv(double* g, int64_t ldg, int64_t l, double* x, int64_t ldx, int* flag, double cond_limit,
             cudaStream_t st);
size_t oz_prep_workspace(int64_t m, int64_t n, int nmod);
int oz_prep(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, void* prep, size_t prep_bytes,
            cudaStream_t st);
size_t oz_gemm_workspace(int trans, int64_t m, int64_t n, int64_t ncols, int nmod);
int oz_gemm(int trans, const void* prep, int64_t m, int64_t n, int nmod, const double* b, int64_t ldb,
            int64_t ncols, double* c, int64_t ldc, void* ws, size_t ws_bytes, cudaStream_t st);
size_t oz_scale_workspace(int64_t m, int64_t n);
int oz_scale(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, int* e_a, void* ws, size_t ws_bytes,
             cudaStream_t st);
int oz_prep_ex(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, const int* e_a_ext, void* prep,
               size_t prep_bytes, cudaStream_t st);
int oz_norms_prep(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, void* prep, size_t prep_bytes,
                  cudaStream_t st);
double oz_guard_limit(int64_t k);
int oz_norms_cols(const double* a, int64_t lda, int64_t m, int64_t n, int64_t c0, int64_t c1, int nmod, void* prep,
                  size_t prep_bytes, cudaStream_t st);
int oz_scale_provisional(int64_t m, int64_t n, int64_t c1, int nmod, void* prep, size_t prep_bytes, cudaStream_t st);
int oz_residue_cols(const double* a, int64_t lda, int64_t m, int64_t n, int64_t c0, int64_t c1, int nmod, void* prep,
                    size_t prep_bytes, cudaStream_t st);
int oz_norms_finish(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, void* prep, size_t prep_bytes,
                    int* e_a_final, cudaStream_t st);
int oz_guard(const void* hdr_host, int64_t m, int64_t n, int* ok_nn, int* ok_tn);
int64_t oz_cols_pad(int64_t ncols);
int oz_bscale(const double* b, int64_t ldb, int64_t k, int64_t ncols, int nmod, int* e_b, cudaStream_t st);
int oz_gemm_ex(int trans, const void* prep, int64_t m, int64_t n, int nmod, const double* b, int64_t ldb,
               int64_t ncols, double* c, int64_t ldc, void* ws, size_t ws_bytes, const int* e_b_ext, int flags,
               cudaStream_t st);
int oz_colsq(int trans, int64_t m, int64_t n, int nmod, int64_t ncols, const void* ws, size_t ws_bytes, double* out,
             int accumulate, cudaStream_t st);
size_t normal_workspace_bytes(int64_t N);
int64_t normal_stream_words(int64_t N);
int64_t normal_tail_cap(int64_t N);
int normal_phase1(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, int64_t N,
                  const uint64_t* ki, const double* wi, const double* fi, void* ws, size_t ws_bytes,
                  cudaStream_t st);
int normal_views(int64_t N, void* ws, uint64_t** u, int64_t** tail_pos, unsigned long long** ntail);
int normal_phase2(int64_t N, const int64_t* tpos, const int* tlen, const double* tval, int64_t ntail,
                  double* out, int64_t* status_dev, void* ws, size_t ws_bytes, cudaStream_t st);

}  // namespace rlra

using namespace rlra;

static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int rlra_b200_abi_version(void) { return RLRA_B200_ABI_VERSION; }
const char* rlra_b200_last_error(void) { return last_error(); }

long long rlra_b200_launch_count(void) { return g_launches.load(); }

int rlra_b200_ktimer_enable(int on) {
  g_ktimer.store(on != 0);
  return 0;
}

int rlra_b200_ktimer_read(const char* name, double* ms_total, long long* launches) {
  RLRA_REQUIRE(name && ms_total && launches, "ktimer_read: null argument");
  int id = -1;
  for (int i = 0; i < KT_COUNT; ++i)
    if (std::strcmp(name, kKTimerNames[i]) == 0) id = i;
  RLRA_REQUIRE(id >= 0, "ktimer_read: unknown kernel timer '%s'", name);
  std::lock_guard<std::mutex> lock(g_ktimer_mu);
  double tot = 0.0;
  long long cnt = 0;
  cudaError_t err = cudaSuccess;
  for (auto& pr : g_ktimer_ev[id]) {
    float ms = 0.0f;
    if (err == cudaSuccess) err = cudaEventSynchronize(pr.second);
    if (err == cudaSuccess) err = cudaEventElapsedTime(&ms, pr.first, pr.second);
    tot += ms;
    ++cnt;
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  g_ktimer_ev[id].clear();
  RLRA_CHECK_CUDA(err);
  *ms_total = tot;
  *launches = cnt;
  return 0;
}

int rlra_b200_device_count(int* out) {
  RLRA_CHECK_CUDA(cudaGetDeviceCount(out));
  return 0;
}

int rlra_b200_plu_inplace(double* lu, int64_t m, int64_t n, int64_t* piv) {
  RLRA_REQUIRE(lu != nullptr && piv != nullptr, "plu_inplace: null buffer");
  RLRA_REQUIRE(m >= 0 && n >= 0, "plu_inplace: negative shape");
  if (m == 0 || n == 0) return 0;
  cudaStream_t st;
  RLRA_CHECK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const size_t abytes = (size_t)m * n * sizeof(double), pbytes = (size_t)m * sizeof(int64_t);
  const size_t wbytes = getrf_workspace_bytes(m, n);
  char* dev = nullptr;
  int rc = 0;
  cudaError_t e = cudaMallocAsync(&dev, abytes + pbytes + wbytes + 512, st);
  if (e != cudaSuccess) {
    set_error("plu_inplace: device allocation failed: %s", cudaGetErrorString(e));
    cudaStreamDestroy(st);
    return -1;
  }
  double* da = reinterpret_cast<double*>(dev);
  int64_t* dp = reinterpret_cast<int64_t*>(dev + ((abytes + 255) & ~(size_t)255));
  void* dw = dev + ((abytes + 255) & ~(size_t)255) + ((pbytes + 255) & ~(size_t)255);
  do {
    if ((e = cudaMemcpyAsync(da, lu, abytes, cudaMemcpyHostToDevice, st)) != cudaSuccess) break;
    if ((e = cudaMemcpyAsync(dp, piv, pbytes, cudaMemcpyHostToDevice, st)) != cudaSuccess) break;
    rc = getrf(da, m, m, n, dp, nullptr, nullptr, dw, wbytes, st);
    if (rc) break;
    if ((e = cudaMemcpyAsync(lu, da, abytes, cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
    if ((e = cudaMemcpyAsync(piv, dp, pbytes, cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
    e = cudaStreamSynchronize(st);
  } while (0);
  cudaFreeAsync(dev, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (rc) return rc;
  if (e != cudaSuccess) {
    set_error("plu_inplace: %s", cudaGetErrorString(e));
    return -1;
  }
  return 0;
}

size_t rlra_b200_getrf_workspace(int64_t m, int64_t n) { return getrf_workspace_bytes(m, n); }

int rlra_b200_getrf_block(double* a, int64_t lda, int64_t m, int64_t j0, int nbo, int64_t* piv, int* zflag,
                          int64_t* ipiv, int64_t* nonzero, void* ws, size_t ws_bytes, void* stream) {
  return getrf_block(a, lda, m, j0, nbo, piv, zflag, ipiv, nonzero, ws, ws_bytes, S(stream));
}

int rlra_b200_lu_trsm_rows(double* a, int64_t lda, int64_t j0, int nb, int64_t c0, int64_t c1, const int* zflag,
                           void* stream) {
  return lu_trsm_rows(a, lda, j0, nb, c0, c1, zflag, S(stream));
}

int rlra_b200_lu_update_split(double* a, int64_t lda, const double* u, int64_t ldu, int64_t j0, int nb, int64_t r0,
                              int64_t m, int64_t c0, int64_t c1, const int* zflag, void* stream) {
  return lu_update_split(a, lda, u, ldu, j0, nb, r0, m, c0, c1, zflag, S(stream));
}

int rlra_b200_getrf(double* a, int64_t lda, int64_t m, int64_t n, int64_t* piv,
                    int64_t* nonzero_diag, void* ws, size_t ws_bytes, void* stream) {
  return getrf(a, lda, m, n, piv, nonzero_diag, nullptr, ws, ws_bytes, S(stream));
}

int rlra_b200_iota(int64_t* p, int64_t m, void* stream) { return fill_iota(p, m, S(stream)); }

int rlra_b200_count_nonzero_diag(const double* a, int64_t lda, int64_t r, int64_t* out,
                                 void* stream) {
  return count_nonzero_diag(a, lda, r, out, S(stream));
}

int rlra_b200_lu_basis(const double* lu, int64_t ldlu, int64_t m, int64_t k, const int64_t* piv,
                       int64_t* pinv_ws, double* w, int64_t ldw, void* stream) {
  return lu_basis(lu, ldlu, m, k, piv, pinv_ws, w, ldw, S(stream));
}

int rlra_b200_lu_extract(const double* lu, int64_t ldlu, int64_t m, int64_t n, double* l,
                         int64_t ldl, double* u, int64_t ldu, void* stream) {
  const int64_t r = m < n ? m : n;
  if (l && extract_l(lu, ldlu, m, r, l, ldl, S(stream))) return -1;
  if (u && extract_u(lu, ldlu, r, n, u, ldu, S(stream))) return -1;
  return 0;
}

int rlra_b200_chol_inv_max_l(void) { return chol_inv_max_l(); }

int rlra_b200_chol_shift_diag(double* g, int64_t ldg, int64_t l, double c, void* stream) {
  return chol_shift_diag(g, ldg, l, c, static_cast<cudaStream_t>(stream));
}

int rlra_b200_gram_identity_flag(const double* g, int64_t ldg, int64_t l, double tol, int* flag, void* stream) {
  return gram_identity_flag(g, ldg, l, tol, flag, static_cast<cudaStream_t>(stream));
}

int rlra_b200_diag_ratio_flag(const double* d, int64_t ldd, int64_t l, double cond_limit, int* flag,
                              void* stream) {
  return diag_ratio_flag(d, ldd, l, cond_limit, flag, static_cast<cudaStream_t>(stream));
}

int rlra_b200_chol_inv(double* g, int64_t ldg, int64_t l, double* rinv, int64_t ldr, int* flag,
                       double cond_limit, void* stream) {
  return chol_inv(g, ldg, l, rinv, ldr, flag, cond_limit, static_cast<cudaStream_t>(stream));
}

size_t rlra_b200_oz_prep_workspace(int64_t m, int64_t n, int nmod) { return oz_prep_workspace(m, n, nmod); }

int rlra_b200_oz_prep(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, void* prep,
                      size_t prep_bytes, void* stream) {
  return oz_prep(a, lda, m, n, nmod, prep, prep_bytes, static_cast<cudaStream_t>(stream));
}

size_t rlra_b200_oz_gemm_workspace(int trans, int64_t m, int64_t n, int64_t ncols, int nmod) {
  return oz_gemm_workspace(trans, m, n, ncols, nmod);
}

int rlra_b200_oz_gemm(int trans, const void* prep, int64_t m, int64_t n, int nmod, const double* b,
                      int64_t ldb, int64_t ncols, double* c, int64_t ldc, void* ws, size_t ws_bytes,
                      void* stream) {
  return oz_gemm(trans, prep, m, n, nmod, b, ldb, ncols, c, ldc, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

size_t rlra_b200_oz_scale_workspace(int64_t m, int64_t n) { return oz_scale_workspace(m, n); }

int rlra_b200_oz_scale(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, int* e_a, void* ws,
                       size_t ws_bytes, void* stream) {
  return oz_scale(a, lda, m, n, nmod, e_a, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int rlra_b200_oz_prep_ex(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, const int* e_a,
                         void* prep, size_t prep_bytes, void* stream) {
  return oz_prep_ex(a, lda, m, n, nmod, e_a, prep, prep_bytes, static_cast<cudaStream_t>(stream));
}

int rlra_b200_oz_norms(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, void* prep,
                       size_t prep_bytes, void* stream) {
  return oz_norms_prep(a, lda, m, n, nmod, prep, prep_bytes, static_cast<cudaStream_t>(stream));
}

double rlra_b200_oz_guard_limit(int64_t k) { return oz_guard_limit(k); }

int rlra_b200_oz_norms_cols(const double* a, int64_t lda, int64_t m, int64_t n, int64_t c0, int64_t c1, int nmod,
                            void* prep, size_t prep_bytes, void* stream) {
  return oz_norms_cols(a, lda, m, n, c0, c1, nmod, prep, prep_bytes, static_cast<cudaStream_t>(stream));
}

int rlra_b200_oz_scale_provisional(int64_t m, int64_t n, int64_t c1, int nmod, void* prep, size_t prep_bytes,
                                   void* stream) {
  return oz_scale_provisional(m, n, c1, nmod, prep, prep_bytes, static_cast<cudaStream_t>(stream));
}

int rlra_b200_oz_residue_cols(const double* a, int64_t lda, int64_t m, int64_t n, int64_t c0, int64_t c1, int nmod,
                              void* prep, size_t prep_bytes, void* stream) {
  return oz_residue_cols(a, lda, m, n, c0, c1, nmod, prep, prep_bytes, static_cast<cudaStream_t>(stream));
}

int rlra_b200_oz_norms_finish(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, void* prep,
                              size_t prep_bytes, int* e_a_final, void* stream) {
  return oz_norms_finish(a, lda, m, n, nmod, prep, prep_bytes, e_a_final, static_cast<cudaStream_t>(stream));
}

int rlra_b200_oz_guard(const void* header, int64_t m, int64_t n, int* ok_nn, int* ok_tn) {
  return oz_guard(header, m, n, ok_nn, ok_tn);
}

int64_t rlra_b200_oz_cols_pad(int64_t ncols) { return oz_cols_pad(ncols); }

int rlra_b200_oz_bscale(const double* b, int64_t ldb, int64_t k, int64_t ncols, int nmod, int* e_b,
                        void* stream) {
  return oz_bscale(b, ldb, k, ncols, nmod, e_b, static_cast<cudaStream_t>(stream));
}

int rlra_b200_oz_gemm_ex(int trans, const void* prep, int64_t m, int64_t n, int nmod, const double* b,
                         int64_t ldb, int64_t ncols, double* c, int64_t ldc, void* ws, size_t ws_bytes,
                         const int* e_b, int flags, void* stream) {
  return oz_gemm_ex(trans, prep, m, n, nmod, b, ldb, ncols, c, ldc, ws, ws_bytes, e_b, flags,
                    static_cast<cudaStream_t>(stream));
}

int rlra_b200_oz_colsq(int trans, int64_t m, int64_t n, int nmod, int64_t ncols, const void* ws, size_t ws_bytes,
                       double* out, int accumulate, void* stream) {
  return oz_colsq(trans, m, n, nmod, ncols, ws, ws_bytes, out, accumulate, static_cast<cudaStream_t>(stream));
}

size_t rlra_b200_gemm_workspace(int64_t m, int64_t n, int64_t k) { return gemm_workspace_bytes(m, n, k); }

int rlra_b200_dgemm(int transa, int transb, int64_t m, int64_t n, int64_t k, double alpha,
                    const double* a, int64_t lda, const double* b, int64_t ldb, double beta,
                    double* c, int64_t ldc, void* ws, size_t ws_bytes, void* stream) {
  return gemm(transa != 0, transb != 0, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc, ws, ws_bytes,
              S(stream));
}

size_t rlra_b200_geqrf_workspace(int64_t m, int64_t n) { return geqrf_workspace_bytes(m, n); }

int rlra_b200_geqrf(double* a, int64_t lda, int64_t m, int64_t n, double* tau, void* ws,
                    size_t ws_bytes, void* stream) {
  return geqrf(a, lda, m, n, tau, ws, ws_bytes, S(stream));
}

int rlra_b200_orgqr(const double* a, int64_t lda, int64_t m, int64_t n, double* q, int64_t ldq,
                    void* ws, size_t ws_bytes, void* stream) {
  return orgqr(a, lda, m, n, q, ldq, ws, ws_bytes, S(stream));
}

size_t rlra_b200_trsm_workspace(int64_t l, int64_t ncols) {
  (void)l;
  return (size_t)32 * 32 * (ncols > 0 ? ncols : 1) * sizeof(double);
}

int rlra_b200_trsm_rt(const double* r, int64_t ldr, int64_t l, double* x, int64_t ldx,
                      int64_t ncols, void* ws, size_t ws_bytes, void* stream) {
  return trsm_rt(r, ldr, l, x, ldx, ncols, ws, ws_bytes, S(stream));
}

int rlra_b200_trsm_un(const double* r, int64_t ldr, int64_t l, double* x, int64_t ldx, int64_t ncols, void* ws,
                      size_t ws_bytes, void* stream) {
  return trsm_un(r, ldr, l, x, ldx, ncols, ws, ws_bytes, S(stream));
}

int rlra_b200_apply_inv_row_perm(const int64_t* p, int64_t m, int64_t n, const double* x, int64_t ldx,
                                 int64_t* pinv_ws, double* out, int64_t ldo, void* stream) {
  return apply_inv_row_perm(p, m, n, x, ldx, pinv_ws, out, ldo, S(stream));
}

int rlra_b200_resid_sumsq_block(const double* a, int64_t lda, int64_t m, const int64_t* p, const int64_t* q_blk,
                                int64_t w, const double* lu, int64_t ldlu, double* partial, void* stream) {
  return resid_sumsq_block(a, lda, m, p, q_blk, w, lu, ldlu, partial, S(stream));
}

int rlra_b200_dd_finish(const double* partial, int64_t nparts, double* out, void* stream) {
  return dd_finish(partial, nparts, out, S(stream));
}

int rlra_b200_spmm_csr(const int64_t* rowptr, const int64_t* colidx, const double* vals, int64_t rows,
                       const double* x, int64_t ldx, int64_t l, double* y, int64_t ldy, void* stream) {
  return spmm_csr(rowptr, colidx, vals, rows, x, ldx, l, y, ldy, S(stream));
}

int rlra_b200_svd_jacobi_max_l(void) { return svd_jacobi_max_l(); }

size_t rlra_b200_svd_jacobi_workspace(int64_t m, int64_t l) { return svd_jacobi_workspace(m, l); }

int rlra_b200_svd_jacobi(const double* a, int64_t lda, int64_t m, int64_t l, double* u, int64_t ldu, double* s,
                         double* v, int64_t ldv, int* sweeps_out, void* ws, size_t ws_bytes, void* stream) {
  return svd_jacobi(a, lda, m, l, u, ldu, s, v, ldv, sweeps_out, ws, ws_bytes, S(stream));
}

int rlra_b200_diag_absmin(const double* a, int64_t lda, int64_t r, double* out, void* stream) {
  return diag_absmin(a, lda, r, out, S(stream));
}

size_t rlra_b200_sumsq_workspace(int64_t m, int64_t n) { return sumsq_workspace_bytes(m, n); }

int rlra_b200_sumsq(const double* a, int64_t lda, int64_t m, int64_t n, double* out, void* ws,
                    size_t ws_bytes, void* stream) {
  return sumsq(a, lda, m, n, out, ws, ws_bytes, S(stream));
}

int rlra_b200_colsumsq(const double* a, int64_t lda, int64_t m, int64_t n, double* out,
                       void* stream) {
  return colsumsq(a, lda, m, n, out, S(stream));
}

int rlra_b200_transpose(const double* in, int64_t ldi, int64_t m, int64_t n, double* out,
                        int64_t ldo, void* stream) {
  return transpose(in, ldi, m, n, out, ldo, S(stream));
}

size_t rlra_b200_normal_workspace(int64_t n) { return normal_workspace_bytes(n); }

int64_t rlra_b200_normal_stream_words(int64_t n) { return normal_stream_words(n); }

int64_t rlra_b200_normal_tail_cap(int64_t n) { return normal_tail_cap(n); }

int rlra_b200_normal_begin(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                           int64_t n, const uint64_t* ki, const double* wi, const double* fi, void* ws,
                           size_t ws_bytes, void* stream) {
  return normal_phase1(state_hi, state_lo, inc_hi, inc_lo, n, ki, wi, fi, ws, ws_bytes, S(stream));
}

int rlra_b200_normal_views(int64_t n, void* ws, uint64_t** words, int64_t** tail_pos,
                           unsigned long long** ntail) {
  return normal_views(n, ws, words, tail_pos, ntail);
}

int rlra_b200_normal_finish(int64_t n, const int64_t* tail_pos, const int* tail_len,
                            const double* tail_val, int64_t ntail, double* out, int64_t* status,
                            void* ws, size_t ws_bytes, void* stream) {
  return normal_phase2(n, tail_pos, tail_len, tail_val, ntail, out, status, ws, ws_bytes, S(stream));
}

}  // extern "C"
