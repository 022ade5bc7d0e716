/*
 * rlra_b200 — C ABI of the B200-native PowerLU hot path (sm_100a).
 *
 * Plain C: no torch or C++ types cross this boundary.  Every function returns
 * 0 on success and a negative status on failure; rlra_b200_last_error()
 * returns a thread-local description of the last failure.  Matrices are
 * column-major float64 with an explicit leading dimension (the reference's
 * canonical layout, rlra/core.py:25-30); permutations are int64 index vectors.
 * `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 * Device-pointer entry points are asynchronous on `stream`; the caller owns
 * every buffer and workspace (size queries are provided) and the library never
 * allocates on those paths.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/rlra):
 *   rlra_b200_plu_inplace      backend.plu_inplace            backend.py:32
 *                              -> _lu_cython.plu_inplace      _lu_cython.pyx:14-55
 *   rlra_b200_getrf            same kernel on device buffers  (kernels.plu, kernels.py:37-54)
 *   rlra_b200_lu_basis         rangefinder._lu_basis          rangefinder.py:73-77
 *                              (core.apply_inv_row_perm       core.py:103-109)
 *   rlra_b200_lu_extract       L/U extraction of kernels.plu  kernels.py:50-53
 *   rlra_b200_dgemm            DenseAccessor.matmul/rmatmul   accessors.py:27-31
 *                              and the assembly products      fixedrank.py:145-146, kernels.py:96
 *   rlra_b200_oz_prep/_gemm    the same two pass products     accessors.py:27-31
 *                              emulated on int8 tensor cores (Ozaki-II)
 *   rlra_b200_geqrf/_orgqr     kernels.eqr (np.linalg.qr)     kernels.py:57-61, :73
 *   rlra_b200_chol_inv         CholeskyQR2 basis (same range as  kernels.py:57-61
 *                              the Householder Q of eqr)
 *   rlra_b200_trsm_rt          solve_triangular(trans='T')    kernels.py:95
 *   rlra_b200_trsm_un          solve_triangular(R, C^T)       fixedrank.py:113 (randlu assembly)
 *   rlra_b200_apply_inv_row_perm core.apply_inv_row_perm      core.py:103-109, fixedrank.py:111
 *   rlra_b200_svd_jacobi       np.linalg.svd of the l x l     fixedrank.py:71 (randsvd)
 *   rlra_b200_resid_sumsq_block reconstruct + rel_fro_error    fixedrank.py:149-155, core.py:56-65
 *   rlra_b200_spmm_csr         SparseAccessor.matmul/rmatmul   accessors.py:40-64
 *                              triangular factor of B = Q^T A
 *   rlra_b200_diag_absmin      pinv_factor rank test          kernels.py:75-79
 *   rlra_b200_sumsq            DenseAccessor.fro_norm()**2    accessors.py:33-34, fixedprec.py:72
 *   rlra_b200_colsumsq         per-column energies of G       fixedprec.py:75-80, :105-107
 *   rlra_b200_transpose        U = L2^T                       fixedrank.py:146
 *   rlra_b200_normal_*         core.gaussian (NumPy PCG64     core.py:33-48
 *                              + ziggurat standard_normal)
 */
#ifndef RLRA_B200_H
#define RLRA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RLRA_B200_ABI_VERSION 1

#if defined(__GNUC__)
#define RLRA_B200_API __attribute__((visibility("default")))
#else
#define RLRA_B200_API
#endif

RLRA_B200_API int rlra_b200_abi_version(void);
RLRA_B200_API const char* rlra_b200_last_error(void);
RLRA_B200_API int rlra_b200_device_count(int* out);
/* number of kernels this library has launched in this process (instrumentation) */
RLRA_B200_API long long rlra_b200_launch_count(void);
/* per-kernel CUDA-event timing (instrumentation for bench.py's roofline):
 * while enabled, events are recorded on the launch stream around the named
 * kernels ("oz_gemm_i8", "oz_residue_a", "oz_norms", "oz_crt", "oz_residue_b");
 * read() waits for them, returns the summed milliseconds and launch count
 * since the last read, and clears the record. */
RLRA_B200_API int rlra_b200_ktimer_enable(int on);
RLRA_B200_API int rlra_b200_ktimer_read(const char* name, double* ms_total, long long* launches);

/* ---- host seam: drop-in for backend.plu_inplace(lu, piv) ---------------
 * lu: HOST F-contiguous float64 m x n (ld = m), overwritten with packed L\U;
 * piv: HOST int64[m], caller-preloaded (0..m-1) and permuted in place.
 * Bit-identical to the reference kernel.  Synchronous; runs on the current
 * CUDA device. */
RLRA_B200_API int rlra_b200_plu_inplace(double* lu, int64_t m, int64_t n, int64_t* piv);

/* ---- K3: GEPP on device buffers ---------------------------------------- */
RLRA_B200_API size_t rlra_b200_getrf_workspace(int64_t m, int64_t n);
/* nonzero_diag (device int64*, nullable) receives count_nonzero(diag(U)) */
RLRA_B200_API int rlra_b200_getrf(double* a, int64_t lda, int64_t m, int64_t n, int64_t* piv,
                    int64_t* nonzero_diag, void* ws, size_t ws_bytes, void* stream);
RLRA_B200_API int rlra_b200_iota(int64_t* p, int64_t m, void* stream);
/* Row-sharded exact GEPP primitives (distributed.dist_getrf_; bit-identical
 * to rlra_b200_getrf).  getrf_block factors the 32-column block [j0, j0+nbo)
 * of an m-row matrix whose VIRTUAL base `a` may be a gathered panel minus
 * j0*lda (only columns [j0, j0+nbo) are touched); rows < j0 enter the
 * zero-pivot column maxima only; piv (int64[m]) is permuted; zflag
 * (int32[>= j0+nbo]) receives the block's zero-pivot flags, ipiv
 * (int64[>= j0+nbo]) its interchange sequence (row j <-> ipiv[j]); *nonzero
 * (int64) accumulates count_nonzero(diag(U)).  ws: rlra_b200_getrf_workspace(m, j0+nbo).
 * lu_trsm_rows: U12 = L11^-1 A12 on rows [j0, j0+nb) of a virtual-row operand.
 * lu_update_split: A(r0:m, c0:c1) -= L(r0:m, j0:j0+nb) U(j0:j0+nb, c0:c1)
 * with L in `a` and U in `u`.  All follow the reference's rounding sequence
 * (rlra/_lu_cython.pyx:14-55). */
RLRA_B200_API int rlra_b200_getrf_block(double* a, int64_t lda, int64_t m, int64_t j0, int nbo, int64_t* piv,
                                        int* zflag, int64_t* ipiv, int64_t* nonzero, void* ws, size_t ws_bytes,
                                        void* stream);
RLRA_B200_API int rlra_b200_lu_trsm_rows(double* a, int64_t lda, int64_t j0, int nb, int64_t c0, int64_t c1,
                                         const int* zflag, void* stream);
RLRA_B200_API int rlra_b200_lu_update_split(double* a, int64_t lda, const double* u, int64_t ldu, int64_t j0, int nb,
                                            int64_t r0, int64_t m, int64_t c0, int64_t c1, const int* zflag,
                                            void* stream);
/* count_nonzero(diag(a)) over the leading r x r block -> device int64 *out
 * (rangefinder._check_width, rangefinder.py:55-64) */
RLRA_B200_API int rlra_b200_count_nonzero_diag(const double* a, int64_t lda, int64_t r, int64_t* out,
                                 void* stream);
/* W (m x k) = P^T L: row-unpermuted unit-lower factor; pinv_ws: int64[m] */
RLRA_B200_API int rlra_b200_lu_basis(const double* lu, int64_t ldlu, int64_t m, int64_t k, const int64_t* piv,
                       int64_t* pinv_ws, double* w, int64_t ldw, void* stream);
/* L (m x r, unit lower) and/or U (r x n, upper) of a packed LU; either may be NULL */
RLRA_B200_API int rlra_b200_lu_extract(const double* lu, int64_t ldlu, int64_t m, int64_t n, double* l,
                         int64_t ldl, double* u, int64_t ldu, void* stream);

/* ---- K1/K2/K5: FP64 DMMA GEMM  C = alpha op(A) op(B) + beta C ---------- */
RLRA_B200_API size_t rlra_b200_gemm_workspace(int64_t m, int64_t n, int64_t k);
RLRA_B200_API int rlra_b200_dgemm(int transa, int transb, int64_t m, int64_t n, int64_t k, double alpha,
                    const double* a, int64_t lda, const double* b, int64_t ldb, double beta,
                    double* c, int64_t ldc, void* ws, size_t ws_bytes, void* stream);

/* ---- K1/K2 emulated: the pass products on the int8 tensor cores --------
 * FP64 GEMM by the Ozaki-II scheme: A and B are scaled by powers of two and
 * rounded to integers (A'' = rint(2^eA A), B'' = rint(2^eB[j] B[:, j])), the
 * integer product is computed exactly modulo nmod pairwise-coprime moduli with
 * tcgen05 kind::i8 MMAs and reassembled by Chinese remaindering, then rounded
 * once to double.  Accuracy (nmod = 14, PA = 54, PB = 53): with N_A the
 * largest row or column 2-norm of A and A_i the i-th row of op(A),
 *   |error_ij| <= 2^-PA sqrt(K) N_A ||B_j|| + 2^-PB sqrt(K) ||A_i|| ||B_j|| + 2^-52 ||A_i|| ||B_j||,
 * normwise in N_A (one scale for all of A).  rlra_b200_oz_guard admits an
 * orientation when N_A / min ||A_i|| <= rlra_b200_oz_guard_limit(K), which
 * makes this at most K 2^-53 ||A_i|| ||B_j||, the classical DGEMM bound; the
 * drivers run the other products (graded rows / columns, NaN / Inf, norms
 * outside [2^-480, 2^512), integer-valued A) on the DMMA GEMM.  Results are exact functions of
 * the inputs.  A column of B holding NaN / Inf yields a NaN output column.
 * prep: residues of A, built once per A by rlra_b200_oz_prep (both
 * orientations); then any number of
 *   trans = 0: C (m x ncols) = A   B,  B n x ncols
 *   trans = 1: C (n x ncols) = A^T B,  B m x ncols
 * nmod in [12, 16] (14 = DGEMM accuracy); K (= n or m) <= 133144.
 * The first RLRA_B200_OZ_HEADER_BYTES of a prep (or oz_scale) workspace are
 * the guard header: int e_a, int pad, then three uint64 holding the double
 * bits of the largest row/column sum of squares, the smallest non-zero row
 * sum and the smallest non-zero column sum (all ones: none), then uint32
 * non-finite flag, uint32 "some entry is not an integer" flag and the double
 * ||A||_F^2 (fixed-order double-double sum of the column partials: the
 * Frobenius norm of rlra/fixedprec.py:72 fused into the norms pass)
 * (integer-valued A is routed to DMMA: exact products turn exact linear
 * dependencies into exact zero pivots where BLAS leaves rounding noise).  rlra_b200_oz_norms fills it (and e_a) without building
 * residues; copy it to the host and pass it to rlra_b200_oz_guard (host-only,
 * no GPU); then rlra_b200_oz_prep_ex(e_a = the prep's own header) builds the
 * residues. */
#define RLRA_B200_OZ_HEADER_BYTES 64
RLRA_B200_API int rlra_b200_oz_norms(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, void* prep,
                                     size_t prep_bytes, void* stream);
RLRA_B200_API double rlra_b200_oz_guard_limit(int64_t k);
/* Pipelined upload (A arriving in column chunks, the e2e path): norms of
 * chunk [c0, c1) (c0 a multiple of 256; chunks in ascending order, the first
 * at 0), a provisional eA after the first chunk (its column norms, row norms
 * extrapolated), residues of chunk [c0, c1) (multiple of 128) with the
 * header's eA, then the final norms / guard statistics / ||A||_F^2 with the
 * final eA in *e_a_final (device int): when it differs from the provisional
 * one the caller rebuilds the residues (rlra_b200_oz_prep_ex). */
RLRA_B200_API int rlra_b200_oz_norms_cols(const double* a, int64_t lda, int64_t m, int64_t n, int64_t c0, int64_t c1,
                                          int nmod, void* prep, size_t prep_bytes, void* stream);
RLRA_B200_API int rlra_b200_oz_scale_provisional(int64_t m, int64_t n, int64_t c1, int nmod, void* prep,
                                                 size_t prep_bytes, void* stream);
RLRA_B200_API int rlra_b200_oz_residue_cols(const double* a, int64_t lda, int64_t m, int64_t n, int64_t c0,
                                            int64_t c1, int nmod, void* prep, size_t prep_bytes, void* stream);
RLRA_B200_API int rlra_b200_oz_norms_finish(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, void* prep,
                                            size_t prep_bytes, int* e_a_final, void* stream);
RLRA_B200_API int rlra_b200_oz_guard(const void* header, int64_t m, int64_t n, int* ok_nn, int* ok_tn);
RLRA_B200_API size_t rlra_b200_oz_prep_workspace(int64_t m, int64_t n, int nmod);
RLRA_B200_API int rlra_b200_oz_prep(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, void* prep,
                                    size_t prep_bytes, void* stream);
RLRA_B200_API size_t rlra_b200_oz_gemm_workspace(int trans, int64_t m, int64_t n, int64_t ncols, int nmod);
RLRA_B200_API int rlra_b200_oz_gemm(int trans, const void* prep, int64_t m, int64_t n, int nmod, const double* b,
                                    int64_t ldb, int64_t ncols, double* c, int64_t ldc, void* ws,
                                    size_t ws_bytes, void* stream);
/* Block-wise pass products for operands whose residues do not fit next to A
 * (or whose K exceeds 133144): A is cut into rectangular blocks that share
 * ONE scale eA (rlra_b200_oz_scale over the whole A, passed to
 * rlra_b200_oz_prep_ex) and one per-column scale eB of the whole B
 * (rlra_b200_oz_bscale, int[rlra_b200_oz_cols_pad(ncols)]).  A K-split
 * product accumulates its residues exactly across calls
 * (RLRA_B200_OZ_ACCUMULATE on every call but the first, RLRA_B200_OZ_NO_CRT on
 * every call but the last, the same workspace throughout), so the result is
 * bit-identical to the one-block product. */
#define RLRA_B200_OZ_ACCUMULATE 1
#define RLRA_B200_OZ_NO_CRT 2
#define RLRA_B200_OZ_ADD_TO_C 4 /* C += A B (the single-pass H += panel G_j) */
RLRA_B200_API size_t rlra_b200_oz_scale_workspace(int64_t m, int64_t n);
RLRA_B200_API int rlra_b200_oz_scale(const double* a, int64_t lda, int64_t m, int64_t n, int nmod, int* e_a,
                                     void* ws, size_t ws_bytes, void* stream);
RLRA_B200_API int rlra_b200_oz_prep_ex(const double* a, int64_t lda, int64_t m, int64_t n, int nmod,
                                       const int* e_a, void* prep, size_t prep_bytes, void* stream);
RLRA_B200_API int64_t rlra_b200_oz_cols_pad(int64_t ncols);
RLRA_B200_API int rlra_b200_oz_bscale(const double* b, int64_t ldb, int64_t k, int64_t ncols, int nmod, int* e_b,
                                      void* stream);
RLRA_B200_API int rlra_b200_oz_gemm_ex(int trans, const void* prep, int64_t m, int64_t n, int nmod,
                                       const double* b, int64_t ldb, int64_t ncols, double* c, int64_t ldc,
                                       void* ws, size_t ws_bytes, const int* e_b, int flags, void* stream);
/* Column energies fused with the product (rlra/fixedprec.py:71-80 takes
 * sum(G[:, j]**2) of G = A V; north star (d)): with RLRA_B200_OZ_COLSQ the CRT
 * step of rlra_b200_oz_gemm_ex also leaves double-double partial sums of
 * squares of the C it writes (per column and 1024-row block) in the workspace;
 * rlra_b200_oz_colsq -- same trans / m / n / nmod / ncols / ws as that call --
 * adds them in a fixed order into out[ncols] (device; accumulate != 0: out +=,
 * for products cut into several output row blocks).  No second read of C. */
#define RLRA_B200_OZ_COLSQ 8
/* The workspace was last used by a product with the SAME skinny operand b,
 * trans, m, n, nmod and ncols: its scales and residues of b are still there
 * and are not rebuilt (the single-pass sweep multiplies every panel^T by the
 * same Omega, rlra/singlepass.py:112-117). */
#define RLRA_B200_OZ_REUSE_B 16
RLRA_B200_API int rlra_b200_oz_colsq(int trans, int64_t m, int64_t n, int nmod, int64_t ncols, const void* ws,
                                     size_t ws_bytes, double* out, int accumulate, void* stream);

/* ---- K4: Householder QR (m >= n) + explicit thin Q --------------------- */
RLRA_B200_API size_t rlra_b200_geqrf_workspace(int64_t m, int64_t n);
RLRA_B200_API int rlra_b200_geqrf(double* a, int64_t lda, int64_t m, int64_t n, double* tau, void* ws,
                    size_t ws_bytes, void* stream);
/* must receive geqrf's workspace, untouched since the geqrf call */
RLRA_B200_API int rlra_b200_orgqr(const double* a, int64_t lda, int64_t m, int64_t n, double* q, int64_t ldq,
                    void* ws, size_t ws_bytes, void* stream);

/* ---- K4 fast path: R^{-1} of R = chol(G), G symmetric positive definite l x l
 * (upper triangle read; g is used as workspace and overwritten).  rinv (l x l) receives R^{-1} (upper, zeros below).
 * *flag (device int) is set to 1 when G is not numerically SPD or when
 * max_i R_ii > cond_limit * min_i R_ii (rinv is then zero); it is never
 * cleared.  l <= rlra_b200_chol_inv_max_l() (one CTA, shared memory). */
RLRA_B200_API int rlra_b200_chol_inv_max_l(void);
/* Shifted CholeskyQR (sCholQR3's first step, sketches wider than
 * rlra_b200_chol_inv_max_l are factored by blocks of chol_inv + DMMA GEMMs in
 * ops.chol_inv_blocked): g_ii += c * trace(g).  Replaces rlra/kernels.py:57-61's
 * Householder QR for powerlu's final basis (rlra/rangefinder.py:67-70). */
RLRA_B200_API int rlra_b200_chol_shift_diag(double* g, int64_t ldg, int64_t l, double c, void* stream);
/* *flag := 1 when max |d_ii| > cond_limit * min |d_ii| (or a zero / non-finite
 * diagonal entry); never cleared. */
/* *flag := 1 when max |g_ij - delta_ij| > tol: CholeskyQR's second Gram far
 * from I means cond(Z) beyond ~u^-1/2 (the diagonal ratio is only a lower bound). */
RLRA_B200_API int rlra_b200_gram_identity_flag(const double* g, int64_t ldg, int64_t l, double tol, int* flag,
                                               void* stream);
RLRA_B200_API int rlra_b200_diag_ratio_flag(const double* d, int64_t ldd, int64_t l, double cond_limit, int* flag,
                                            void* stream);
RLRA_B200_API int rlra_b200_chol_inv(double* g, int64_t ldg, int64_t l, double* rinv, int64_t ldr, int* flag,
                                     double cond_limit, void* stream);

/* ---- K6: X = R^{-T} B in place over B (R upper l x l) ------------------- */
RLRA_B200_API size_t rlra_b200_trsm_workspace(int64_t l, int64_t ncols);
RLRA_B200_API int rlra_b200_trsm_rt(const double* r, int64_t ldr, int64_t l, double* x, int64_t ldx,
                      int64_t ncols, void* ws, size_t ws_bytes, void* stream);
RLRA_B200_API int rlra_b200_diag_absmin(const double* a, int64_t lda, int64_t r, double* out, void* stream);
/* X = R^{-1} B in place over B (R upper l x l; same workspace query). */
RLRA_B200_API int rlra_b200_trsm_un(const double* r, int64_t ldr, int64_t l, double* x, int64_t ldx,
                                    int64_t ncols, void* ws, size_t ws_bytes, void* stream);
/* out[p[i], :] = x[i, :] for a permutation p of 0..m-1 (pinv_ws: int64[m]). */
RLRA_B200_API int rlra_b200_apply_inv_row_perm(const int64_t* p, int64_t m, int64_t n, const double* x,
                                               int64_t ldx, int64_t* pinv_ws, double* out, int64_t ldo,
                                               void* stream);

/* ---- K9 validation residual ||A[p, :][:, q] - L U||_F^2 (rlra/fixedrank.py:149-155,
 * rlra/core.py:56-65) without materialising the m x n reconstruction: per block
 * of w columns of L U (m x w, caller-computed), partial[2j..2j+1] = the
 * double-double sum over i of (A[p[i], q_blk[j]] - LU[i, j])^2; dd_finish sums
 * nparts such pairs in a fixed order into out[0]. */
RLRA_B200_API int rlra_b200_resid_sumsq_block(const double* a, int64_t lda, int64_t m, const int64_t* p,
                                              const int64_t* q_blk, int64_t w, const double* lu, int64_t ldlu,
                                              double* partial, void* stream);
RLRA_B200_API int rlra_b200_dd_finish(const double* partial, int64_t nparts, double* out, void* stream);

/* ---- sparse operands (SparseAccessor, rlra/accessors.py:40-64): Y = S X for S
 * (rows x K) in CSR with int64 indices, X (K x l) and Y (rows x l) column-major;
 * A X uses the CSR of A, A^T X the CSR of A^T (the CSC arrays of A). */
RLRA_B200_API int rlra_b200_spmm_csr(const int64_t* rowptr, const int64_t* colidx, const double* vals,
                                     int64_t rows, const double* x, int64_t ldx, int64_t l, double* y,
                                     int64_t ldy, void* stream);

/* ---- randsvd's small SVD: one-sided Jacobi, A (m x l, m >= l, l <= max_l)
 * = U diag(s) V^T, s nonincreasing (ties by column index); sweeps_out
 * (device int, nullable) receives the number of sweeps. */
RLRA_B200_API int rlra_b200_svd_jacobi_max_l(void);
RLRA_B200_API size_t rlra_b200_svd_jacobi_workspace(int64_t m, int64_t l);
RLRA_B200_API int rlra_b200_svd_jacobi(const double* a, int64_t lda, int64_t m, int64_t l, double* u, int64_t ldu,
                                       double* s, double* v, int64_t ldv, int* sweeps_out, void* ws,
                                       size_t ws_bytes, void* stream);

/* ---- K8 / K2b: compensated deterministic energies ----------------------- */
RLRA_B200_API size_t rlra_b200_sumsq_workspace(int64_t m, int64_t n);
RLRA_B200_API int rlra_b200_sumsq(const double* a, int64_t lda, int64_t m, int64_t n, double* out, void* ws,
                    size_t ws_bytes, void* stream);
RLRA_B200_API int rlra_b200_colsumsq(const double* a, int64_t lda, int64_t m, int64_t n, double* out,
                       void* stream);

/* ---- a1: Omega on the device, bit-identical to the reference's host draw
 * np.random.default_rng(seed).standard_normal(n) (rlra/core.py:33-48): NumPy's
 * PCG64 (state/inc from the seed) + its 256-layer ziggurat (tables ki/wi/fi).
 * Two phases: begin() generates and classifies the word stream on the
 * device; the caller resolves the rare tail draws (|x| > r; positions and the
 * following words are exposed by views()) with the host libm log1p and passes
 * them to finish(), which emits the n normals (flat == column-major order).
 * status (device int64[3]): {normals produced (== n on success), flags, words consumed}. */
RLRA_B200_API size_t rlra_b200_normal_workspace(int64_t n);
RLRA_B200_API int64_t rlra_b200_normal_stream_words(int64_t n);
RLRA_B200_API int64_t rlra_b200_normal_tail_cap(int64_t n);
RLRA_B200_API int rlra_b200_normal_begin(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                                         uint64_t inc_lo, int64_t n, const uint64_t* ki,
                                         const double* wi, const double* fi, void* ws,
                                         size_t ws_bytes, void* stream);
RLRA_B200_API int rlra_b200_normal_views(int64_t n, void* ws, uint64_t** words, int64_t** tail_pos,
                                         unsigned long long** ntail);
RLRA_B200_API int rlra_b200_normal_finish(int64_t n, const int64_t* tail_pos, const int* tail_len,
                                          const double* tail_val, int64_t ntail, double* out,
                                          int64_t* status, void* ws, size_t ws_bytes, void* stream);

/* ---- layout helper ------------------------------------------------------ */
RLRA_B200_API int rlra_b200_transpose(const double* in, int64_t ldi, int64_t m, int64_t n, double* out,
                        int64_t ldo, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RLRA_B200_H */
