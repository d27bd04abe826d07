/*
 * ks.h -- C-ABI of the B200-native hot path of arXiv 1312.1869
 * ("blocked approximate inversion of large, nearly rank-deficient covariance
 * matrices"):
 *
 *     sketch       Y = K Omega            K generated on the fly, never stored
 *     tsqr         Y = Q R                blocked tall-skinny Householder QR
 *     lowrank      X = Omega R^{-1} Q^T A (truncated; K X = Q Q^T A)
 *
 * Citations are PAPER.md line numbers (the paper's LaTeX source); the readings
 * of silent or garbled passages (L1..L20) are listed in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Every pointer argument named *_dev / documented "device" is a CUDA device
 *    pointer on the current device; the caller owns all memory (inputs,
 *    outputs and workspaces).  The library never allocates or frees device
 *    memory and never frees caller buffers.
 *  - Matrices are row-major fp32, 16-byte aligned base pointers.
 *  - Every call is stream-ordered on `stream` and returns after enqueueing
 *    (no host synchronisation), except where documented (ks_trsolve tau == 0).
 *  - Errors: a ks_status is returned; ks_last_error() gives a thread-local
 *    message.  Invalid arguments are detected before anything is enqueued.
 *    No C++ exception crosses this boundary.
 *  - Determinism: Y is bitwise reproducible for given (inputs, seed) and its
 *    rows do not depend on the row range requested (multi-GPU sharding).
 *    R/Q are reproducible for fixed (rows, d, blocks).
 */
#ifndef KS_H_
#define KS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define KS_API __attribute__((visibility("default")))
#else
#define KS_API
#endif

typedef struct CUstream_st* ks_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum ks_status {
  KS_OK = 0,
  KS_ERR_INVALID_ARGUMENT = 1, /* any precondition violation */
  KS_ERR_SINGULAR = 2,         /* ks_trsolve, tau == 0: |r_jj| <= 1e-12 max|r_ii| */
  KS_ERR_CUDA = 3,             /* a CUDA runtime / driver call failed */
  KS_ERR_OOM = 4,              /* workspace smaller than the *_workspace_size answer */
  KS_ERR_UNSUPPORTED = 5,      /* valid request outside what the kernels implement */
  KS_ERR_NCCL = 6              /* reserved: collectives run in the Python layer */
} ks_status;

/* Covariance kernels (configs).  r^2 = sum_c (x_c - y_c)^2
 * by direct differences (reading L10).
 *   KS_KERNEL_SQEXP    k = sigma2 * exp(-r^2 / (2 ell^2))               (L7)
 *   KS_KERNEL_MATERN32 k = sigma2 * (1 + sqrt3 r/ell) exp(-sqrt3 r/ell) (L8) */
/*   KS_KERNEL_STORED   K is not generated: ks_sketch_stored reads it from device memory (NEXT-2, the
 *                      planted-spectrum workload K = E D E^T of PAPER.md:388); valid only there. */
typedef enum ks_kernel_kind { KS_KERNEL_SQEXP = 0, KS_KERNEL_MATERN32 = 1, KS_KERNEL_STORED = 2 } ks_kernel_kind;

/* Random projection Omega (n x d):
 *   KS_OMEGA_SRHT  Def. 1, T = Walsh-Hadamard (:74-89):
 *                  Omega = D_s H_N[:, S] / sqrt(N), natural order, N = 2^ceil(log2 n),
 *                  K zero-padded to N columns (readings L1-L4).
 *   KS_OMEGA_GAUSS PAPER.md:54: Omega_ij = fp16_RN(z_ij) / sqrt(d), z ~ N(0,1) (L6).
 *   KS_OMEGA_DHT / KS_OMEGA_DCT (NEXT-1): Def. 1 with T the orthonormal discrete Hartley
 *                  (cas(2 pi j k / n) / sqrt n) or cosine (DCT-II) transform (the
 *                  "HP" / "HC" projections of :403), for any n (no padding): Omega = D_s T[:, S],
 *                  S uniform without replacement from [0, n) (masked Philox draws >= n rejected).
 *                  Computed as a dense tensor-core contraction with Omega generated once per call in
 *                  fp16 hi + lo (scaled by sqrt n); same d limits as GAUSS. */
typedef enum ks_omega_kind { KS_OMEGA_SRHT = 0, KS_OMEGA_GAUSS = 1, KS_OMEGA_DHT = 2, KS_OMEGA_DCT = 3 } ks_omega_kind;

typedef struct ks_sketch_desc {
  int64_t n;       /* number of points = order of K, n >= 1 */
  int32_t dim;     /* point dimension, 1..3 */
  int32_t kernel;  /* ks_kernel_kind */
  float sigma2;    /* > 0 */
  float ell;       /* > 0 */
  float nugget;    /* >= 0, added to K's diagonal by index (L9) */
  int32_t d;       /* sketch width, 1 <= d <= N; SRHT: d <= 512; GAUSS/DHT/DCT: d <= n, d % 16 == 0, 16 <= d <= 256 */
  uint64_t seed;   /* Philox4x32-10 key */
  int32_t omega;   /* ks_omega_kind */
  int32_t reserved;
} ks_sketch_desc;

/* ------------------------------------------------------------------ sketch */

/* Device workspace bytes needed by ks_sketch / ks_omega_apply / ks_omega_export. */
KS_API ks_status ks_sketch_workspace_size(const ks_sketch_desc* desc, size_t* bytes);

/* Y = rows [row_begin, row_end) of K Omega  (PAPER.md:95 "K-hat = K Omega", :19).
 *   pts_dev : device, fp32 SoA, dim x n (coordinate c of point j at pts[c*n + j])
 *   Y_dev   : device, fp32, (row_end - row_begin) x d, row-major, 16-byte aligned
 *   ws_dev  : device workspace of ks_sketch_workspace_size bytes (contents
 *             after the call: the sketch randomness, reused by ks_omega_apply)
 * Generates the randomness (signs, selection, Gaussian Omega) in the workspace,
 * then runs the fused covariance-tile + transform kernel.  K is never stored.
 * Errors: INVALID_ARGUMENT (desc out of range, 0 <= row_begin <= row_end <= n
 * violated, null pointers), OOM (ws_bytes too small), UNSUPPORTED (d above the
 * kernel limits), CUDA. */
KS_API ks_status ks_sketch(const ks_sketch_desc* desc, const float* pts_dev, int64_t row_begin, int64_t row_end,
                    float* Y_dev, void* ws_dev, size_t ws_bytes, ks_stream_t stream);

/* NEXT-2: Y = rows [row_begin, row_end) of K Omega for a STORED K (PAPER.md:95 with the planted-spectrum
 * K = E D E^T of PAPER.md:388 "we start therefore with a known spectral decomposition"): the same Omega,
 * randomness and workspace as ks_sketch, but the sketch kernels stream K from HBM instead of evaluating
 * the covariance (an HBM-bound ingest of n^2 * 4 bytes).
 *   K_dev : device, fp32, row-major: rows [row_begin, row_end) of K, K[i][j] at K_dev[(i - row_begin) * ldk + j]
 *           (a rank passes just its row block); ldk >= n, ldk % 4 == 0, 16-byte aligned.  Columns [0, n)
 *           are read.  Not modified.
 *   desc  : kernel must be KS_KERNEL_STORED; dim and ell are ignored; sigma2 must bound max |K_ij| (it
 *           sets the fp16 scaling of the GAUSS / DHT / DCT tensor-core path; K itself is used unscaled);
 *           nugget is added to the diagonal by index as in ks_sketch (use 0 for K = E D E^T).
 * Errors: as ks_sketch; INVALID_ARGUMENT also for kernel != KS_KERNEL_STORED, ldk < n, ldk % 4 != 0 or a
 * misaligned K_dev. */
KS_API ks_status ks_sketch_stored(const ks_sketch_desc* desc, const float* K_dev, int64_t ldk, int64_t row_begin,
                                  int64_t row_end, float* Y_dev, void* ws_dev, size_t ws_bytes, ks_stream_t stream);

/* Export the sketch randomness for bit-exact tests (device outputs; any may be NULL):
 *   signs_dev  int8[N]       s_j in {-1,+1}      (Def. 1 "Rademacher")
 *   sel_dev    int32[d]      S sorted ascending  (Def. 1 "permutation submatrix", :70)
 *   gauss_dev  uint16[n*d]   fp16 bits of Omega_ij * sqrt(d), row-major n x d (GAUSS only) */
KS_API ks_status ks_omega_export(const ks_sketch_desc* desc, int8_t* signs_dev, int32_t* sel_dev, uint16_t* gauss_dev,
                          void* ws_dev, size_t ws_bytes, ks_stream_t stream);

/* X = rows [row_begin, row_end) of Omega Z  (reading L14: K X = Y Z).
 *   Z_dev : device, d x m fp32;  X_dev : device, (row_end-row_begin) x m fp32.
 *   1 <= m <= 64.  Regenerates the randomness into ws_dev (same size as ks_sketch). */
KS_API ks_status ks_omega_apply(const ks_sketch_desc* desc, const float* Z_dev, int32_t m, int64_t row_begin,
                         int64_t row_end, float* X_dev, void* ws_dev, size_t ws_bytes, ks_stream_t stream);

/* -------------------------------------------------------------------- TSQR */

/* Blocked TSQR, eqs. (1)-(4): the rows are split into `blocks`
 * contiguous, equal-as-possible blocks (L13); each block is factored by
 * Householder QR (internally as a binary sub-tree of row leaves of <= 1024
 * rows -- "any Householder-based scheme", R is unique); stacked R's are merged
 * pairwise, an odd one passing through.  R is upper triangular with exact
 * zeros below the diagonal and r_jj >= 0 (L12).
 * Limits: 1 <= d <= 512, every block must have >= d rows. */
typedef struct ks_tsqr_plan* ks_tsqr_handle;

/* Merge topology of the block R's: the pairwise tree (eqs. (2)-(3), the default) or the chain of
 * eq. (5) (the running R absorbs one block R per step).  R is the same (unique). */
/* KS_TSQR_MIXED: eq. (5) exactly as printed -- the blocks in two halves, a chain inside each half (advancing
 * side by side), then one merge of the two chains' R's: the paper's "mixture of the strategies". */
/* KS_TSQR_TRIANGULAR (a flag OR-ed into the topology): every block is exactly d rows and upper triangular -- a
 * stack of R factors, the second TSQR level (eqs. (2)-(3), :252).  Rows below a block's
 * diagonal are zero, so in panel k only its first 32 (k + 1) rows take part (the reflectors act as the identity
 * on the rest): the same R, less work and latency for the early panels.  Needs rows a multiple of d, whole R's
 * per block, d <= 512 (every R is its own leaf); ks_tsqr_merge uses it (one block: a flat merge of the P R's). */
typedef enum { KS_TSQR_TREE = 0, KS_TSQR_CHAIN = 1, KS_TSQR_MIXED = 2, KS_TSQR_TRIANGULAR = 16 } ks_tsqr_topology;

KS_API ks_status ks_tsqr_workspace_size(int64_t rows, int32_t d, int32_t blocks, size_t* bytes);
KS_API ks_status ks_tsqr_workspace_size_ex(int64_t rows, int32_t d, int32_t blocks, int32_t topology, size_t* bytes);

/* Create a plan over a caller-owned device workspace (kept until destroy).  _ex selects the topology
 * (KS_ERR_INVALID_ARGUMENT for an unknown one).  The plan metadata is copied into the workspace
 * synchronously (no stream argument): the workspace must be idle -- no kernel queued on any stream may
 * still be using it.  Plans are per device (create, run and destroy with the same current device). */
KS_API ks_status ks_tsqr_create(int64_t rows, int32_t d, int32_t blocks, void* ws_dev, size_t ws_bytes,
                         ks_tsqr_handle* out);
KS_API ks_status ks_tsqr_create_ex(int64_t rows, int32_t d, int32_t blocks, int32_t topology, void* ws_dev,
                            size_t ws_bytes, ks_tsqr_handle* out);
KS_API ks_status ks_tsqr_destroy(ks_tsqr_handle h);

/* The plan's working matrix (device, rows x d, row-major, inside the caller's workspace; valid until
 * destroy).  ks_tsqr factors a copy of Y_dev in it; passing this pointer itself as Y_dev skips the copy
 * (the sketch can be written there directly) -- Y is then overwritten by the factorisation. */
KS_API ks_status ks_tsqr_work_matrix(ks_tsqr_handle h, float** W_dev);

/* Factor Y (device, rows x d, not modified).  R_dev: d x d output.  If Q_dev is
 * non-NULL the explicit Q (rows x d, Q^T Q = I) is formed: Q-hat = Q^b_1 Q^b_2 ...
 * (eq. 4).  The implicit factors stay in the handle for ks_qform. */
KS_API ks_status ks_tsqr(ks_tsqr_handle h, const float* Y_dev, float* Q_dev, float* R_dev, ks_stream_t stream);

/* Q_dev (rows x d) = Q-hat * C, with C (d x d, device) or C = I if C_dev == NULL.
 * Multi-GPU second level: C = this rank's d x d block of the merge's Q2. */
KS_API ks_status ks_qform(ks_tsqr_handle h, const float* C_dev, float* Q_dev, ks_stream_t stream);

/* Implicit Q ("the matrix product for forming Q-hat need not be evaluated at all"),
 * valid after ks_tsqr on the handle; the stored reflectors are applied directly (4 rows d m flops
 * instead of forming Q):
 *   ks_tsqr_apply_qt: C_dev (d x m) = Q-hat^T X.  X_dev (rows x m, device) is overwritten (it holds
 *                     Q_full^T X on return; C is its first d rows).
 *   ks_tsqr_apply_q : X_dev (rows x m) = Q-hat C, C_dev d x m.
 * m >= 1; row-major fp32; stream-ordered. */
KS_API ks_status ks_tsqr_apply_qt(ks_tsqr_handle h, float* X_dev, int32_t m, float* C_dev, ks_stream_t stream);
KS_API ks_status ks_tsqr_apply_q(ks_tsqr_handle h, const float* C_dev, int32_t m, float* X_dev, ks_stream_t stream);

/* Second TSQR level (eq. (5)'s final merge of per-unit R's):
 * one QR of the stacked (P*d) x d matrix of per-rank R's (a single block: leaves of <= 512 stacked
 * rows merged by one flat level, not a second binary tree -- the latency of the merge is on every
 * rank's critical path).  Q2_dev: (P*d) x d
 * explicit, R_dev: d x d.  Run redundantly on every rank. */
KS_API ks_status ks_tsqr_merge_workspace_size(int32_t P, int32_t d, size_t* bytes);
KS_API ks_status ks_tsqr_merge(const float* Rstack_dev, int32_t P, int32_t d, float* Q2_dev, float* R_dev, void* ws_dev,
                        size_t ws_bytes, ks_stream_t stream);

/* ------------------------------------------------------------------- solve */

/* C = Q^T X (explicit Q, "Q-hat^T x ... evaluated via blocking").
 *   Q_dev rows x d, X_dev rows x m, C_dev d x m (1 <= m <= 64).  Deterministic
 *   two-stage reduction over row chunks (no atomics). */
KS_API ks_status ks_apply_qt_workspace_size(int64_t rows, int32_t d, int32_t m, size_t* bytes);
KS_API ks_status ks_apply_qt(const float* Q_dev, int64_t rows, int32_t d, const float* X_dev, int32_t m, float* C_dev,
                      void* ws_dev, size_t ws_bytes, ks_stream_t stream);

/* X = Q C (explicit Q; rows x d times d x m). */
KS_API ks_status ks_apply_q(const float* Q_dev, int64_t rows, int32_t d, const float* C_dev, int32_t m, float* X_dev,
                     ks_stream_t stream);

/* Truncated back substitution ("R^{-1} ... by backward substitution";
 * upper triangular per :95, reading L11; truncation L14):
 *   tau > 0 : k = largest prefix with |r_jj| >= tau * max_i |r_ii|;
 *             Z[:k] = R[:k,:k]^{-1} C[:k], Z[k:] = 0; *k_dev = k.  Async.
 *   tau == 0: strict; if any |r_jj| <= 1e-12 max|r_ii| returns KS_ERR_SINGULAR
 *             (message names the index).  Synchronises `stream`.
 *   R_dev d x d, C_dev/Z_dev d x m (device fp32); computed in fp64 on the GPU.
 *   k_dev: device int32 (may be NULL). */
KS_API ks_status ks_trsolve(const float* R_dev, const float* C_dev, int32_t d, int32_t m, float tau, float* Z_dev,
                     int32_t* k_dev, ks_stream_t stream);

/* ------------------------------------------------- NEXT-4: GP downstream */

/* Theorem 5's stability diagnostic (reading L19: the condition number of the linear
 * system K-hat R^{-1} with K-hat = K Omega = Y, "we are interested in the stability of the numerical
 * system, K-hat R_k^{-1}", :359).  X = Y R^{-1} (rows x d, == Q-hat in exact arithmetic), G = X^T X;
 *   out_dev (device float[4]) = { cond = sqrt(l_max / l_min) of G, i.e. c(X);  eps = ||G - I||_2
 *   (Theorem 5 bounds c by sqrt((1 + eps) / (1 - eps)));  l_min;  l_max }.
 *   Y_dev rows x d, R_dev d x d upper triangular with a nonzero diagonal (device fp32).  The extreme
 *   eigenvalues of G - I come from min(d, 256) Lanczos steps with full reorthogonalisation (one CTA) and a
 *   Sturm-count bisection of the tridiagonal (exact spectrum when d <= 256).
 * ks_cond_gram writes only G (d x d) for a row block -- ranks all-reduce their G's and call
 * ks_cond_from_gram (workspace >= 1024 * d bytes).  Errors: INVALID_ARGUMENT (null pointers, rows < 1,
 * d < 1 or d > 1024), OOM. */
KS_API ks_status ks_cond_diag_workspace_size(int64_t rows, int32_t d, size_t* bytes);
KS_API ks_status ks_cond_diag(const float* Y_dev, int64_t rows, int32_t d, const float* R_dev, float* out_dev,
                              void* ws_dev, size_t ws_bytes, ks_stream_t stream);
KS_API ks_status ks_cond_gram(const float* Y_dev, int64_t rows, int32_t d, const float* R_dev, float* G_dev,
                              void* ws_dev, size_t ws_bytes, ks_stream_t stream);
KS_API ks_status ks_cond_from_gram(const float* G_dev, int32_t d, float* out_dev, void* ws_dev, size_t ws_bytes,
                                   ks_stream_t stream);

/* Gaussian likelihood with the low-rank covariance plus a nugget ("evaluating a Gaussian
 * type likelihood"; SPEC.md:424-442 fixes the standard zero-mean form): Sigma = U diag(lam) U^T + sigma2 I,
 * U rows x r with orthonormal columns (e.g. the TSQR Q), lam >= 0 (device fp32[r]), sigma2 > 0.
 *   ks_gp_woodbury_solve: X = Sigma^{-1} B = (B - U diag(lam / (lam + sigma2)) U^T B) / sigma2
 *                         (Woodbury), B / X rows x q device fp32 (X may not alias B).
 *   ks_gp_loglik:         out_dev (device double[3]) = { -1/2 [n log 2 pi + log det Sigma + y^T Sigma^{-1} y],
 *                         y^T Sigma^{-1} y, log det Sigma = sum log(lam + sigma2) + (n - r) log sigma2 }
 *                         (determinant lemma), n = rows; y device fp32[rows].  The dot product is summed
 *                         in fp64 in a fixed order.
 * Workspace: ks_gp_workspace_size(rows, r, q) (q = 1 for the likelihood).  Errors: INVALID_ARGUMENT
 * (null pointers, sizes < 1, sigma2 <= 0), OOM. */
KS_API ks_status ks_gp_workspace_size(int64_t rows, int32_t r, int32_t q, size_t* bytes);
KS_API ks_status ks_gp_woodbury_solve(const float* U_dev, int64_t rows, int32_t r, const float* lam_dev, float sigma2,
                                      const float* B_dev, int32_t q, float* X_dev, void* ws_dev, size_t ws_bytes,
                                      ks_stream_t stream);
KS_API ks_status ks_gp_loglik(const float* U_dev, int64_t rows, int32_t r, const float* lam_dev, float sigma2,
                              const float* y_dev, double* out_dev, void* ws_dev, size_t ws_bytes, ks_stream_t stream);

/* The Nystrom core of the approximate spectral decomposition K ~ Q B Q^T ("approximate QR
 * decompositions are useful in obtaining other approximate matrix decompositions, such as approximate spectral
 * decompositions", citing Halko-Martinsson-Tropp's Alg. 5.3): a SECOND fused pass over K,
 *   W = K Q          (n x d; K generated on the fly from the points as in ks_sketch, never stored; the
 *                    tensor-core contraction of the Hartley / cosine path with Q split into fp16 hi + lo)
 *   B = (Q^T W + W^T Q) / 2   (d x d, deterministic split-K Q^T-apply, symmetrised)
 *   desc  : n, dim, kernel (SQEXP / MATERN32), sigma2, ell, nugget as for ks_sketch; d = Q's columns,
 *           d % 16 == 0, 16 <= d <= 256; omega and seed are ignored.
 *   pts_dev : device fp32 SoA dim x n;  Q_dev : device fp32 n x d row-major (all n rows, e.g. the TSQR Q),
 *           16-byte aligned;  W_dev : device fp32 n x d output, 16-byte aligned;  B_dev : device fp32 d x d.
 * Errors: INVALID_ARGUMENT (desc, NULL / misaligned pointers), UNSUPPORTED (d, stored kernel), OOM, CUDA. */
KS_API ks_status ks_nystrom_workspace_size(const ks_sketch_desc* desc, size_t* bytes);
KS_API ks_status ks_nystrom_core(const ks_sketch_desc* desc, const float* pts_dev, const float* Q_dev, float* W_dev,
                                 float* B_dev, void* ws_dev, size_t ws_bytes, ks_stream_t stream);

/* The Gaussian likelihood / solve of ks_gp_* with the core form Sigma = Q B Q^T + sigma2 I (Q rows x d with
 * orthonormal columns, B d x d symmetric positive semidefinite, e.g. from ks_nystrom_core; sigma2 > 0):
 *   ks_gp_loglik_core:   out_dev (device double[3]) = { log-likelihood, y^T Sigma^{-1} y, log det Sigma } with
 *                        y^T Sigma^{-1} y = (y^T y - c^T c) / sigma2 + c^T (B + sigma2 I)^{-1} c, c = Q^T y, and
 *                        log det Sigma = log det (B + sigma2 I) + (rows - d) log sigma2 (Woodbury and the
 *                        determinant lemma on the d x d core: a Cholesky factorisation in fp64 on the GPU).
 *   ks_gp_woodbury_core: Z_dev (rows x q) = Sigma^{-1} X = X / sigma2 + Q ((B + sigma2 I)^{-1} c - c / sigma2),
 *                        c = Q^T X; X / Z device fp32 rows x q, Z may not alias X.
 * Limits: d <= 256, q <= 64.  Workspace: ks_gp_core_workspace_size(rows, d, q) (q = 1 for the likelihood).
 * Errors: INVALID_ARGUMENT (NULL pointers, sizes < 1, sigma2 <= 0), UNSUPPORTED (limits), OOM. */
KS_API ks_status ks_gp_core_workspace_size(int64_t rows, int32_t d, int32_t q, size_t* bytes);
KS_API ks_status ks_gp_loglik_core(const float* Q_dev, int64_t rows, int32_t d, const float* B_dev, float sigma2,
                                   const float* y_dev, double* out_dev, void* ws_dev, size_t ws_bytes,
                                   ks_stream_t stream);
KS_API ks_status ks_gp_woodbury_core(const float* Q_dev, int64_t rows, int32_t d, const float* B_dev, float sigma2,
                                     const float* X_dev, int32_t q, float* Z_dev, void* ws_dev, size_t ws_bytes,
                                     ks_stream_t stream);

/* One-shot single-GPU path: sketch -> tsqr -> apply_qt -> trsolve -> omega_apply.
 *   A_dev n x m, X_dev n x m, Z_dev d x m, k_dev int32 (device, required: the truncation rank k < d is
 *   how a caller detects that the solve was truncated).  Workspace size from ks_lowrank_workspace_size.
 *   tau as in ks_trsolve: tau > 0 truncates (async); tau == 0 is the strict solve, which returns
 *   KS_ERR_SINGULAR (naming the index) when some |r_jj| <= 1e-12 max|r_ii| and synchronises `stream`. */
KS_API ks_status ks_lowrank_workspace_size(const ks_sketch_desc* desc, int32_t m, int32_t blocks, size_t* bytes);
KS_API ks_status ks_lowrank_solve(const ks_sketch_desc* desc, const float* pts_dev, const float* A_dev, int32_t m,
                           int32_t blocks, float tau, float* X_dev, float* Z_dev, int32_t* k_dev, void* ws_dev,
                           size_t ws_bytes, ks_stream_t stream);

/* Thread-local description of the last error ("" if none). */
KS_API const char* ks_last_error(void);

/* Library version string. */
KS_API const char* ks_version(void);

/* Number of kernels this library has enqueued since load (process-wide,
 * monotonically increasing; used by bench.py for its gpu_launches claim). */
KS_API uint64_t ks_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* KS_H_ */
