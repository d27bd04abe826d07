/*
 * ks_oracle.c -- CPU fp64 ORACLE for the arXiv 1312.1869 hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code with the CUDA path (paper_1312_1869_b200/): its own
 * Philox, its own kernel evaluation, its own transforms and QR.
 *
 * Plain, slow, obviously correct: materialise what the paper materialises,
 * textbook loops, fp64 throughout, no blocking beyond the paper's own TSQR
 * block scheme (eqs. 1-5).  Every function cites the passage it follows
 * (PAPER.md line numbers; readings of silent/garbled points are the ledger
 * L1..L20 of SURVEY.md 8(c), restated in DESIGN.md).
 *
 * Row parallelism (std threads) is used only where rows are independent
 * (sketch rows, TSQR leaves); results do not depend on the thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* RNG: Philox4x32-10 (Salmon et al. SC'11), stream layout of ledger L5.       */
/* The paper is silent on the generator ("independent Rademacher   */
/* entries", :70 "permutation submatrix", :54 "iid Gaussian").                 */
/* ------------------------------------------------------------------------- */
void ko_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    if (r != 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void draw(uint64_t seed, uint32_t stream, uint64_t idx, uint32_t w[4]) {
  uint32_t ctr[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), stream, 0u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  ko_philox(ctr, key, w);
}

enum { ST_SIGNS = 1, ST_SELECT = 2, ST_GAUSS = 3 };

/* Def. 1: "R is an n x n diagonal matrix whose diagonal elements
 * are independent Rademacher entries".  s_j = 1 - 2*bit(j&127) of draw(j>>7). */
void ko_signs(uint64_t seed, int64_t N, int8_t* s) {
  for (int64_t j = 0; j < N; ++j) {
    uint32_t w[4];
    draw(seed, ST_SIGNS, (uint64_t)j >> 7, w);
    int b = (int)(j & 127);
    uint32_t bit = (w[b >> 5] >> (b & 31)) & 1u;
    s[j] = (int8_t)(1 - 2 * (int)bit);
  }
}

/* Def. 1: "P is an n x r permutation submatrix".  Reading L4:
 * uniform without replacement = the first d distinct values of the masked draw
 * stream (N a power of two, so w0 & (N-1) is exactly uniform), sorted.
 * Returns 0 on success, -1 if d > N. */
int ko_selection(uint64_t seed, int64_t N, int32_t d, int32_t* S) {
  if (d > N || d < 0) return -1;
  uint8_t* used = (uint8_t*)calloc((size_t)N, 1);
  int32_t got = 0;
  for (uint64_t t = 0; got < d; ++t) {
    uint32_t w[4];
    draw(seed, ST_SELECT, t, w);
    uint32_t cand = w[0] & (uint32_t)(N - 1);
    if (!used[cand]) { used[cand] = 1; ++got; }
  }
  /* sorted ascending = enumerate the marked indices in order */
  int32_t k = 0;
  for (int64_t j = 0; j < N; ++j) if (used[j]) S[k++] = (int32_t)j;
  free(used);
  return 0;
}

static double u53(uint32_t a, uint32_t b) {
  double v = (double)(((uint64_t)(a >> 5) << 26) + (uint64_t)(b >> 6));
  return (v + 0.5) * 0x1p-53;
}

/* IEEE binary16 round-to-nearest-even of a double (no intermediate float). */
uint16_t ko_fp16_rn(double x) {
  uint16_t sign = signbit(x) ? 0x8000u : 0u;
  double a = fabs(x);
  if (isnan(x)) return 0x7E00u;
  if (a >= 65520.0) return sign | 0x7C00u;            /* rounds to inf */
  if (a < 0x1p-14) {                                   /* subnormal range, quantum 2^-24 */
    double q = a * 0x1p24;                             /* exact scaling */
    double r = nearbyint(q);                           /* default mode = RNE */
    return sign | (uint16_t)r;                         /* r == 1024 -> min normal, still right */
  }
  int e;
  double f = frexp(a, &e);                             /* a = f * 2^e, f in [0.5,1) */
  double q = ldexp(f, 11);                             /* 11 significant bits incl. hidden */
  double r = nearbyint(q);                             /* in [1024, 2048] */
  if (r >= 2048.0) { r /= 2.0; e += 1; }
  int exp16 = e - 1 + 15;                              /* value = r * 2^(e-11) = (r/1024) * 2^(e-1) */
  if (exp16 >= 31) return sign | 0x7C00u;
  return sign | (uint16_t)(exp16 << 10) | (uint16_t)((int)r - 1024);
}

double ko_fp16_to_double(uint16_t h) {
  int s = h >> 15, e = (h >> 10) & 31, m = h & 1023;
  double v;
  if (e == 0) v = ldexp((double)m, -24);
  else if (e == 31) v = m ? NAN : INFINITY;
  else v = ldexp((double)(m + 1024), e - 25);
  return s ? -v : v;
}

/* PAPER.md:54 "iid Gaussian random variables appropriately scaled"; reading L6:
 * Omega_ij = fp16_RN(z_ij) with z from fp64 Box-Muller, the 1/sqrt(d) applied
 * separately.  Output: n x d fp16 bit patterns, row-major. */
void ko_gauss_omega(uint64_t seed, int64_t n, int32_t d, uint16_t* om) {
  for (int64_t i = 0; i < n; ++i)
    for (int32_t t = 0; t < d; ++t) {
      uint32_t w[4];
      draw(seed, ST_GAUSS, (uint64_t)i * (uint64_t)d + (uint64_t)t, w);
      double z = sqrt(-2.0 * log(u53(w[0], w[1]))) * cos(6.283185307179586 * u53(w[2], w[3]));
      om[i * d + t] = ko_fp16_rn(z);
    }
}

/* ------------------------------------------------------------------------- */
/* Covariance kernel.  SE: PAPER.md:376 theta1*exp(-theta2*||x-y||^2) with     */
/* theta1 = sigma2, theta2 = 1/(2 ell^2) (reading L7).  Matern: PAPER.md:382    */
/* printed sqrt(2 nu) form; for half-integer nu = p + 1/2 the Bessel form has   */
/* the closed form exp(-a r) p!/(2p)! sum_i (p+i)!/(i!(p-i)!) (2 a r)^(p-i),     */
/* a = sqrt(2 nu)/ell (reading L8).  r^2 by direct differences (L10).           */
/* kind: 0 = SE, 1 = Matern-3/2, 2 = Matern-1/2, 3 = Matern-5/2.               */
/* ------------------------------------------------------------------------- */
static double fact(int k) { double f = 1; for (int i = 2; i <= k; ++i) f *= i; return f; }

double ko_kernel_r(int kind, double r2, double sigma2, double ell) {
  if (kind == 0) return sigma2 * exp(-r2 / (2.0 * ell * ell));
  int p = kind == 1 ? 1 : (kind == 2 ? 0 : 2);
  double nu = p + 0.5;
  double r = sqrt(r2);
  double a = sqrt(2.0 * nu) / ell;
  double sum = 0.0;
  for (int i = 0; i <= p; ++i)
    sum += fact(p + i) / (fact(i) * fact(p - i)) * pow(2.0 * a * r, p - i);
  return sigma2 * exp(-a * r) * fact(p) / fact(2 * p) * sum;
}

static double pt_r2(const float* pts, int64_t n, int dim, int64_t i, int64_t j) {
  double r2 = 0.0;
  for (int c = 0; c < dim; ++c) {
    double diff = (double)pts[c * n + i] - (double)pts[c * n + j];
    r2 += diff * diff;
  }
  return r2;
}

/* k(i,j) = C(x_i, x_j) plus the nugget on the diagonal by index
 * (reading L9).  pts is SoA fp32, dim x n. */
double ko_K_entry(const float* pts, int64_t n, int dim, int kind, double sigma2, double ell,
                  double nugget, int64_t i, int64_t j) {
  double k = ko_kernel_r(kind, pt_r2(pts, n, dim, i, j), sigma2, ell);
  return i == j ? k + nugget : k;
}

/* Tier A: materialise K (n x n). */
void ko_K_dense(const float* pts, int64_t n, int dim, int kind, double sigma2, double ell,
                double nugget, double* K) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j)
      K[i * n + j] = ko_K_entry(pts, n, dim, kind, sigma2, ell, nugget, i, j);
}

/* ------------------------------------------------------------------------- */
/* Walsh-Hadamard: H_n = [[H_{n/2}, H_{n/2}], [H_{n/2},        */
/* -H_{n/2}]], H_2 = [[1,1],[1,-1]] -- built literally by the recursion.        */
/* ------------------------------------------------------------------------- */
void ko_hadamard(int64_t N, double* H) {
  H[0] = 1.0;
  for (int64_t h = 1; h < N; h *= 2)
    for (int64_t i = 0; i < h; ++i)
      for (int64_t j = 0; j < h; ++j) {
        double v = H[i * N + j];
        H[i * N + (j + h)] = v;
        H[(i + h) * N + j] = v;
        H[(i + h) * N + (j + h)] = -v;
      }
}

/* The same recursion applied to a vector: v <- H_N v (textbook FWHT). */
void ko_fwht(double* v, int64_t N) {
  for (int64_t h = 1; h < N; h *= 2)
    for (int64_t i = 0; i < N; i += 2 * h)
      for (int64_t j = i; j < i + h; ++j) {
        double a = v[j], b = v[j + h];
        v[j] = a + b;
        v[j + h] = a - b;
      }
}

/* Def. 1 Omega = c R T P with T = H_N, c = 1/sqrt(N) (L1),
 * natural order (L2), zero padding to N = 2^ceil(log2 n) (L3): the first n rows
 * of diag(s) H_N[:, S] / sqrt(N).  Om is n x d row-major. */
void ko_omega_srht(const int8_t* s, const int32_t* S, int64_t n, int64_t N, int32_t d, double* Om) {
  double* H = (double*)malloc(sizeof(double) * (size_t)(N * N));
  ko_hadamard(N, H);
  double c = 1.0 / sqrt((double)N);
  for (int64_t j = 0; j < n; ++j)
    for (int32_t t = 0; t < d; ++t) Om[j * d + t] = c * (double)s[j] * H[j * N + S[t]];
  free(H);
}

/* Plain triple loop C (m x k) = A (m x p) B (p x k). */
void ko_matmul(const double* A, const double* B, int64_t m, int64_t p, int64_t k, double* C) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < k; ++j) {
      double acc = 0.0;
      for (int64_t l = 0; l < p; ++l) acc += A[i * p + l] * B[l * k + j];
      C[i * k + j] = acc;
    }
}

/* NEXT-1 structured Omega = R T P (Def. 1) with T the discrete Hartley or the discrete
 * cosine transform (PAPER.md:74 "discrete cosine matrix, discrete Hartley matrix", :91 "Hartley and
 * discrete cosine transforms ... do not have these problems"), both taken orthonormal so that c = 1
 * (L1) and for any n (no padding).  P: uniform without replacement from [0, n) -- the selection stream
 * masked to [0, N), N = 2^ceil(log2 n), out-of-range draws rejected (for n = N identical to
 * ko_selection), sorted ascending. */
int ko_selection_n(uint64_t seed, int64_t N, int64_t n, int32_t d, int32_t* S) {
  if (d > n || d < 0 || n > N) return -1;
  uint8_t* used = (uint8_t*)calloc((size_t)n, 1);
  int32_t got = 0;
  for (uint64_t t = 0; got < d; ++t) {
    uint32_t w[4];
    draw(seed, ST_SELECT, t, w);
    uint32_t cand = w[0] & (uint32_t)(N - 1);
    if (cand < (uint64_t)n && !used[cand]) { used[cand] = 1; ++got; }
  }
  int32_t k = 0;
  for (int64_t j = 0; j < n; ++j) if (used[j]) S[k++] = (int32_t)j;
  free(used);
  return 0;
}

/* T[j][k]: kind 2 = discrete Hartley, cas(2 pi j k / n) / sqrt(n), cas = cos + sin;
 *          kind 3 = discrete cosine (DCT-II), sqrt(2/n) eps_k cos(pi (2j+1) k / (2n)), eps_0 = 1/sqrt(2).
 * The angle's integer part is reduced exactly (j k mod n, (2j+1) k mod 4n) before the fp64 cos/sin. */
double ko_trig_entry(int kind, int64_t n, int64_t j, int64_t k) {
  const double pi = 3.14159265358979323846;
  if (kind == 2) {
    const double a = 2.0 * pi * (double)((j * k) % n) / (double)n;
    return (cos(a) + sin(a)) / sqrt((double)n);
  }
  const double a = pi * (double)(((2 * j + 1) * k) % (4 * n)) / (2.0 * (double)n);
  return sqrt(2.0 / (double)n) * (k == 0 ? 1.0 / sqrt(2.0) : 1.0) * cos(a);
}

/* Explicit Omega = diag(s) T[:, S] (n x d), row-major. */
void ko_omega_trig(int kind, const int8_t* s, const int32_t* S, int64_t n, int32_t d, double* Om) {
  for (int64_t j = 0; j < n; ++j)
    for (int32_t t = 0; t < d; ++t) Om[j * d + t] = (double)s[j] * ko_trig_entry(kind, n, j, S[t]);
}

/* ------------------------------------------------------------------------- */
/* Tier B sketch: per row, Y[i,:] = (1/sqrt N) (H_N (s o K[i,:]))[S]            */
/* (PAPER.md:19 "structured random matrices ... n log d", :61, :95).           */
/* ------------------------------------------------------------------------- */
typedef struct {
  const float* pts; int64_t n; int dim; int kind; double sigma2, ell, nugget;
  const int8_t* s; const int32_t* S; int64_t N; int32_t d;
  const uint16_t* om;                 /* gaussian omega (n x d fp16) or NULL */
  const double* omd;                  /* dense fp64 omega (n x d) or NULL (structured Hartley / cosine) */
  const int64_t* rows; int64_t nrows; double* Y;
  int tid, nthreads;
} sketch_job;

static void* sketch_worker(void* arg) {
  sketch_job* J = (sketch_job*)arg;
  if (J->omd != NULL) {
    double* krow = (double*)malloc(sizeof(double) * (size_t)J->n);
    for (int64_t r = J->tid; r < J->nrows; r += J->nthreads) {
      int64_t i = J->rows[r];
      for (int64_t j = 0; j < J->n; ++j)
        krow[j] = ko_K_entry(J->pts, J->n, J->dim, J->kind, J->sigma2, J->ell, J->nugget, i, j);
      for (int32_t t = 0; t < J->d; ++t) {
        double acc = 0.0;
        for (int64_t j = 0; j < J->n; ++j) acc += krow[j] * J->omd[j * J->d + t];
        J->Y[r * J->d + t] = acc;
      }
    }
    free(krow);
  } else if (J->om == NULL) {
    double* v = (double*)malloc(sizeof(double) * (size_t)J->N);
    double c = 1.0 / sqrt((double)J->N);
    for (int64_t r = J->tid; r < J->nrows; r += J->nthreads) {
      int64_t i = J->rows[r];
      for (int64_t j = 0; j < J->N; ++j)
        v[j] = j < J->n ? (double)J->s[j] *
                              ko_K_entry(J->pts, J->n, J->dim, J->kind, J->sigma2, J->ell, J->nugget, i, j)
                        : 0.0;
      ko_fwht(v, J->N);
      for (int32_t t = 0; t < J->d; ++t) J->Y[r * J->d + t] = c * v[J->S[t]];
    }
    free(v);
  } else {
    double* krow = (double*)malloc(sizeof(double) * (size_t)J->n);
    double c = 1.0 / sqrt((double)J->d);
    for (int64_t r = J->tid; r < J->nrows; r += J->nthreads) {
      int64_t i = J->rows[r];
      for (int64_t j = 0; j < J->n; ++j)
        krow[j] = ko_K_entry(J->pts, J->n, J->dim, J->kind, J->sigma2, J->ell, J->nugget, i, j);
      for (int32_t t = 0; t < J->d; ++t) {
        double acc = 0.0;
        for (int64_t j = 0; j < J->n; ++j) acc += krow[j] * ko_fp16_to_double(J->om[j * J->d + t]);
        J->Y[r * J->d + t] = c * acc;
      }
    }
    free(krow);
  }
  return NULL;
}

static void run_sketch(sketch_job* base, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  sketch_job* jobs = (sketch_job*)malloc(sizeof(sketch_job) * (size_t)nthreads);
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = *base; jobs[t].tid = t; jobs[t].nthreads = nthreads;
    pthread_create(&th[t], NULL, sketch_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th); free(jobs);
}

void ko_sketch_srht_rows(const float* pts, int64_t n, int dim, int kind, double sigma2, double ell,
                         double nugget, const int8_t* s, const int32_t* S, int64_t N, int32_t d,
                         const int64_t* rows, int64_t nrows, double* Y, int nthreads) {
  sketch_job J = {pts, n, dim, kind, sigma2, ell, nugget, s, S, N, d, NULL, NULL, rows, nrows, Y, 0, 1};
  run_sketch(&J, nthreads);
}

/* Gaussian Omega: Y[i,:] = K[i,:] Omega / sqrt(d), Omega the fp16
 * values promoted exactly to fp64 (L6). */
void ko_sketch_gauss_rows(const float* pts, int64_t n, int dim, int kind, double sigma2, double ell,
                          double nugget, const uint16_t* om, int32_t d, const int64_t* rows,
                          int64_t nrows, double* Y, int nthreads) {
  sketch_job J = {pts, n, dim, kind, sigma2, ell, nugget, NULL, NULL, 0, d, om, NULL, rows, nrows, Y, 0, 1};
  run_sketch(&J, nthreads);
}

/* Structured Hartley / cosine Omega (NEXT-1): Y[i,:] = K[i,:] Omega with the explicit fp64 Omega. */
void ko_sketch_dense_rows(const float* pts, int64_t n, int dim, int kind, double sigma2, double ell, double nugget,
                          const double* Om, int32_t d, const int64_t* rows, int64_t nrows, double* Y, int nthreads) {
  sketch_job J = {pts, n, dim, kind, sigma2, ell, nugget, NULL, NULL, 0, d, NULL, Om, rows, nrows, Y, 0, 1};
  run_sketch(&J, nthreads);
}

/* ------------------------------------------------------------------------- */
/* Householder QR, textbook unblocked (Golub & Van Loan, Alg. 5.1.1 house +     */
/* Alg. 5.2.1), the "QR decomposition" of PAPER.md:13 / :95.  house() is       */
/* chosen so that P x = ||x|| e1, i.e. r_jj >= 0 (reading L12).  Q is formed    */
/* explicitly by backward accumulation onto [I_d; 0].  A is m x d row-major;    */
/* internally column-major.  Q (m x d, row-major) may be NULL.                  */
/* ------------------------------------------------------------------------- */
static void house(const double* x, int64_t len, double* v, double* beta, double* mu_out) {
  double sigma = 0.0;
  for (int64_t i = 1; i < len; ++i) sigma += x[i] * x[i];
  v[0] = 1.0;
  for (int64_t i = 1; i < len; ++i) v[i] = x[i];
  if (sigma == 0.0) {
    if (x[0] >= 0.0) { *beta = 0.0; *mu_out = x[0]; }
    else { *beta = 2.0; *mu_out = -x[0]; }            /* P = I - 2 e1 e1^T flips the sign */
    return;
  }
  double mu = sqrt(x[0] * x[0] + sigma);
  double v0 = x[0] <= 0.0 ? x[0] - mu : -sigma / (x[0] + mu);
  *beta = 2.0 * v0 * v0 / (sigma + v0 * v0);
  for (int64_t i = 1; i < len; ++i) v[i] /= v0;
  *mu_out = mu;
}

void ko_householder_qr(const double* A, int64_t m, int32_t d, double* Q, double* R) {
  double* Ac = (double*)malloc(sizeof(double) * (size_t)(m * d));        /* column-major copy */
  for (int64_t i = 0; i < m; ++i)
    for (int32_t j = 0; j < d; ++j) Ac[(int64_t)j * m + i] = A[i * d + j];
  double* V = (double*)calloc((size_t)(m * d), sizeof(double));          /* reflectors, column j */
  double* betas = (double*)calloc((size_t)d, sizeof(double));
  int32_t kmax = (int32_t)(m < d ? m : d);
  for (int32_t j = 0; j < kmax; ++j) {
    double* x = Ac + (int64_t)j * m + j;
    double* v = V + (int64_t)j * m + j;
    int64_t len = m - j;
    double beta, mu;
    house(x, len, v, &beta, &mu);
    betas[j] = beta;
    /* A(j:m, j:d) = (I - beta v v^T) A(j:m, j:d) */
    for (int32_t c = j; c < d; ++c) {
      double* col = Ac + (int64_t)c * m + j;
      double w = 0.0;
      for (int64_t i = 0; i < len; ++i) w += v[i] * col[i];
      w *= beta;
      for (int64_t i = 0; i < len; ++i) col[i] -= w * v[i];
    }
    x[0] = mu;                                         /* exact value of the new diagonal */
    for (int64_t i = 1; i < len; ++i) x[i] = 0.0;      /* exact zeros below the diagonal */
  }
  for (int32_t i = 0; i < d; ++i)
    for (int32_t j = 0; j < d; ++j) R[i * d + j] = (j >= i && i < m) ? Ac[(int64_t)j * m + i] : 0.0;
  if (Q) {
    /* backward accumulation: Qc = H_0 H_1 ... H_{k-1} [I_d; 0] */
    double* Qc = (double*)calloc((size_t)(m * d), sizeof(double));
    for (int32_t j = 0; j < d && j < m; ++j) Qc[(int64_t)j * m + j] = 1.0;
    for (int32_t j = kmax - 1; j >= 0; --j) {
      const double* v = V + (int64_t)j * m + j;
      int64_t len = m - j;
      for (int32_t c = 0; c < d; ++c) {
        double* col = Qc + (int64_t)c * m + j;
        double w = 0.0;
        for (int64_t i = 0; i < len; ++i) w += v[i] * col[i];
        w *= betas[j];
        for (int64_t i = 0; i < len; ++i) col[i] -= w * v[i];
      }
    }
    for (int64_t i = 0; i < m; ++i)
      for (int32_t j = 0; j < d; ++j) Q[i * d + j] = Qc[(int64_t)j * m + i];
    free(Qc);
  }
  free(Ac); free(V); free(betas);
}

/* ------------------------------------------------------------------------- */
/* TSQR tree, eqs. (1)-(4): leaf QRs K_i = Q_i R_i (eq. 1),   */
/* pairwise QRs of stacked R's (eqs. 2-3) until one R remains; Q-hat =          */
/* Q^b_1 Q^b_2 Q^b_3 (eq. 4).  Block partition: contiguous, equal-as-possible   */
/* (L13); an odd R at a level passes through.  Q (m x d) may be NULL.           */
/* ------------------------------------------------------------------------- */
typedef struct node {
  int64_t rows;           /* rows of the matrix factored at this node */
  double* Qn;             /* rows x d explicit Q of this node's small QR */
  double* R;              /* d x d */
  struct node* kid[2];    /* children (NULL for a leaf); a pass-through has kid[1] == NULL */
  int64_t row0;           /* leaves: first row of the block */
} node;

/* Independent QRs run in batches of up to nthreads threads (rows of different blocks are independent;
 * results do not depend on the thread count). */
typedef struct { const double* A; int64_t d; node* nd; } qr_job;
static void* qr_worker(void* arg) {
  qr_job* L = (qr_job*)arg;
  node* nd = L->nd;
  ko_householder_qr(L->A, nd->rows, (int32_t)L->d, nd->Qn, nd->R);
  return NULL;
}

static void run_qr_jobs(qr_job* jobs, int32_t cnt, int nthreads) {
  for (int32_t i0 = 0; i0 < cnt; i0 += nthreads) {
    int c = (cnt - i0) < nthreads ? (cnt - i0) : nthreads;
    pthread_t th[64];
    for (int t = 0; t < c; ++t) pthread_create(&th[t], NULL, qr_worker, &jobs[i0 + t]);
    for (int t = 0; t < c; ++t) pthread_join(th[t], NULL);
  }
}

/* eq. (4) top-down: the d x d factor C that multiplies each leaf's Qn (Q-hat rows of the leaf =
 * Qn_leaf * C_leaf).  Internal nodes: (Qn_node * C) split into the children's d x d blocks. */
static void qform_collect(node* nd, const double* C, int32_t d, double* Cleaf, node** leaves, int32_t* nleaf) {
  if (nd->kid[0] == NULL) {
    memcpy(Cleaf + (int64_t)(*nleaf) * d * d, C, sizeof(double) * (size_t)d * d);
    leaves[(*nleaf)++] = nd;
    return;
  }
  double* QC = (double*)malloc(sizeof(double) * (size_t)(nd->rows * d));
  ko_matmul(nd->Qn, C, nd->rows, d, d, QC);
  if (nd->kid[1] == NULL) {
    qform_collect(nd->kid[0], QC, d, Cleaf, leaves, nleaf);
  } else {
    qform_collect(nd->kid[0], QC, d, Cleaf, leaves, nleaf);
    qform_collect(nd->kid[1], QC + (int64_t)d * d, d, Cleaf, leaves, nleaf);
  }
  free(QC);
}

typedef struct { const double* Qn; const double* C; int64_t rows; int32_t d; double* out; } mm_job;
static void* mm_worker(void* arg) {
  mm_job* J = (mm_job*)arg;
  ko_matmul(J->Qn, J->C, J->rows, J->d, J->d, J->out);
  return NULL;
}

static void free_tree(node* nd) {
  if (!nd) return;
  free_tree(nd->kid[0]);
  free_tree(nd->kid[1]);
  free(nd->Qn); free(nd->R); free(nd);
}

/* returns 0, or -1 if some block has fewer than d rows (L13 / SPEC.md:235) */
int ko_tsqr_tree(const double* A, int64_t m, int32_t d, int32_t b, double* R, double* Q, int nthreads) {
  if (b < 1 || m / b < d) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 64) nthreads = 64;
  node** level = (node**)malloc(sizeof(node*) * (size_t)b);
  node** leaves = (node**)malloc(sizeof(node*) * (size_t)b);
  qr_job* jobs = (qr_job*)malloc(sizeof(qr_job) * (size_t)b);
  for (int32_t i = 0; i < b; ++i) {
    node* nd = (node*)calloc(1, sizeof(node));
    int64_t r0 = (m * i) / b, r1 = (m * (i + 1)) / b;
    nd->row0 = r0; nd->rows = r1 - r0;
    nd->Qn = (double*)malloc(sizeof(double) * (size_t)(nd->rows * d));
    nd->R = (double*)malloc(sizeof(double) * (size_t)d * d);
    level[i] = nd;
    jobs[i].A = A + r0 * d; jobs[i].d = d; jobs[i].nd = nd;
  }
  /* eq. (1): independent leaf QRs */
  run_qr_jobs(jobs, b, nthreads);
  /* eqs. (2)-(3): pairwise QRs of stacked R's, the pairs of one level independent */
  int32_t cnt = b;
  while (cnt > 1) {
    int32_t nxt = 0;
    double** stk = (double**)malloc(sizeof(double*) * (size_t)(cnt / 2));
    for (int32_t i = 0; i + 1 < cnt; i += 2) {
      node* nd = (node*)calloc(1, sizeof(node));
      nd->rows = 2 * (int64_t)d;
      nd->kid[0] = level[i]; nd->kid[1] = level[i + 1];
      double* st = (double*)malloc(sizeof(double) * (size_t)(2 * d * d));
      memcpy(st, level[i]->R, sizeof(double) * (size_t)d * d);
      memcpy(st + (int64_t)d * d, level[i + 1]->R, sizeof(double) * (size_t)d * d);
      nd->Qn = (double*)malloc(sizeof(double) * (size_t)(2 * d * d));
      nd->R = (double*)malloc(sizeof(double) * (size_t)d * d);
      stk[nxt] = st;
      jobs[nxt].A = st; jobs[nxt].d = d; jobs[nxt].nd = nd;
      level[nxt++] = nd;
    }
    run_qr_jobs(jobs, nxt, nthreads);
    for (int32_t i = 0; i < nxt; ++i) free(stk[i]);
    free(stk);
    if (cnt & 1) level[nxt++] = level[cnt - 1];        /* odd one passes through */
    cnt = nxt;
  }
  node* root = level[0];
  memcpy(R, root->R, sizeof(double) * (size_t)d * d);
  if (Q) {
    /* eq. (4): Q-hat = Q^b_1 Q^b_2 ...: the node factors top-down, then Q rows of leaf i = Qn_i * C_i */
    double* I = (double*)calloc((size_t)d * d, sizeof(double));
    for (int32_t i = 0; i < d; ++i) I[i * d + i] = 1.0;
    double* Cleaf = (double*)malloc(sizeof(double) * (size_t)b * d * d);
    int32_t nleaf = 0;
    qform_collect(root, I, d, Cleaf, leaves, &nleaf);
    mm_job* mj = (mm_job*)malloc(sizeof(mm_job) * (size_t)nleaf);
    for (int32_t i0 = 0; i0 < nleaf; i0 += nthreads) {
      int c = (nleaf - i0) < nthreads ? (nleaf - i0) : nthreads;
      pthread_t th[64];
      for (int t = 0; t < c; ++t) {
        node* lf = leaves[i0 + t];
        mj[i0 + t] = (mm_job){lf->Qn, Cleaf + (int64_t)(i0 + t) * d * d, lf->rows, d, Q + lf->row0 * d};
        pthread_create(&th[t], NULL, mm_worker, &mj[i0 + t]);
      }
      for (int t = 0; t < c; ++t) pthread_join(th[t], NULL);
    }
    free(mj); free(Cleaf); free(I);
  }
  free_tree(root);
  free(level); free(leaves); free(jobs);
  return 0;
}

/* C (m x k) = A (m x p) B (p x k), the plain triple loop of ko_matmul with the rows of C split over
 * threads (each element summed in the same order: identical to ko_matmul). */
typedef struct { const double* A; const double* B; int64_t m0, m1, p, k; double* C; } mmr_job;
static void* mmr_worker(void* arg) {
  mmr_job* J = (mmr_job*)arg;
  ko_matmul(J->A + J->m0 * J->p, J->B, J->m1 - J->m0, J->p, J->k, J->C + J->m0 * J->k);
  return NULL;
}

void ko_matmul_mt(const double* A, const double* B, int64_t m, int64_t p, int64_t k, double* C, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 64) nthreads = 64;
  if (nthreads > m) nthreads = (int)(m > 0 ? m : 1);
  pthread_t th[64]; mmr_job J[64];
  for (int t = 0; t < nthreads; ++t) {
    J[t] = (mmr_job){A, B, (m * t) / nthreads, (m * (t + 1)) / nthreads, p, k, C};
    pthread_create(&th[t], NULL, mmr_worker, &J[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* Chain scheme, eq. (5): each of `chains` contiguous groups
 * of blocks is reduced sequentially, factoring [R_prev; K_next]; the chains'
 * final R's are then combined by one more QR of the stacked R's. */
int ko_tsqr_chain(const double* A, int64_t m, int32_t d, int32_t b, int32_t chains, double* R) {
  if (b < 1 || chains < 1 || chains > b || m / b < d) return -1;
  double* Rs = (double*)malloc(sizeof(double) * (size_t)chains * d * d);
  for (int32_t c = 0; c < chains; ++c) {
    int32_t b0 = (b * c) / chains, b1 = (b * (c + 1)) / chains;
    double* Rcur = Rs + (int64_t)c * d * d;
    for (int32_t i = b0; i < b1; ++i) {
      int64_t r0 = (m * i) / b, r1 = (m * (i + 1)) / b;
      if (i == b0) {
        ko_householder_qr(A + r0 * d, r1 - r0, d, NULL, Rcur);
      } else {
        int64_t rows = d + (r1 - r0);
        double* stk = (double*)malloc(sizeof(double) * (size_t)(rows * d));
        memcpy(stk, Rcur, sizeof(double) * (size_t)d * d);
        memcpy(stk + (int64_t)d * d, A + r0 * d, sizeof(double) * (size_t)((r1 - r0) * d));
        ko_householder_qr(stk, rows, d, NULL, Rcur);
        free(stk);
      }
    }
  }
  if (chains == 1) memcpy(R, Rs, sizeof(double) * (size_t)d * d);
  else ko_householder_qr(Rs, (int64_t)chains * d, d, NULL, R);
  free(Rs);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Solve ("evaluate the expression R^{-1} Q^T A ... backward       */
/* substitution"; upper triangular per :95 / :182, reading L11).  Truncation   */
/* rule L14: k = largest prefix with |r_jj| >= tau * max_i |r_ii|.             */
/* ------------------------------------------------------------------------- */
int32_t ko_truncation_rank(const double* R, int32_t d, double tau) {
  double mx = 0.0;
  for (int32_t i = 0; i < d; ++i) mx = fmax(mx, fabs(R[i * d + i]));
  int32_t k = 0;
  while (k < d && fabs(R[k * d + k]) >= tau * mx && R[k * d + k] != 0.0) ++k;
  return k;
}

/* Z[:k] = R[:k,:k]^{-1} C[:k], Z[k:] = 0.  C, Z are d x m row-major. */
void ko_back_substitute(const double* R, int32_t d, const double* C, int32_t m, int32_t k, double* Z) {
  for (int32_t c = 0; c < m; ++c) {
    for (int32_t i = d - 1; i >= k; --i) Z[i * m + c] = 0.0;
    for (int32_t i = k - 1; i >= 0; --i) {
      double acc = C[i * m + c];
      for (int32_t j = i + 1; j < k; ++j) acc -= R[i * d + j] * Z[j * m + c];
      Z[i * m + c] = acc / R[i * d + i];
    }
  }
}

/* X = Omega Z (reading L14: X = Omega Z so K X = Y Z).  SRHT: column by column,
 * scatter Z rows to S, textbook FWHT (H symmetric), x s / sqrt N, first n rows. */
void ko_omega_apply_srht(const int8_t* s, const int32_t* S, int64_t n, int64_t N, int32_t d,
                         const double* Z, int32_t m, double* X) {
  double* v = (double*)malloc(sizeof(double) * (size_t)N);
  double c = 1.0 / sqrt((double)N);
  for (int32_t col = 0; col < m; ++col) {
    for (int64_t j = 0; j < N; ++j) v[j] = 0.0;
    for (int32_t t = 0; t < d; ++t) v[S[t]] = Z[t * m + col];
    ko_fwht(v, N);
    for (int64_t j = 0; j < n; ++j) X[j * m + col] = c * (double)s[j] * v[j];
  }
  free(v);
}

void ko_omega_apply_gauss(const uint16_t* om, int64_t n, int32_t d, const double* Z, int32_t m, double* X) {
  double c = 1.0 / sqrt((double)d);
  for (int64_t j = 0; j < n; ++j)
    for (int32_t col = 0; col < m; ++col) {
      double acc = 0.0;
      for (int32_t t = 0; t < d; ++t) acc += ko_fp16_to_double(om[j * d + t]) * Z[t * m + col];
      X[j * m + col] = c * acc;
    }
}

/* X = Omega Z with an explicit fp64 Omega (n x d). */
void ko_omega_apply_dense(const double* Om, int64_t n, int32_t d, const double* Z, int32_t m, double* X) {
  for (int64_t j = 0; j < n; ++j)
    for (int32_t col = 0; col < m; ++col) {
      double acc = 0.0;
      for (int32_t t = 0; t < d; ++t) acc += Om[j * d + t] * Z[t * m + col];
      X[j * m + col] = acc;
    }
}
