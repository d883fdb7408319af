/* fp64 CPU restatement of the reference Muon path — see muon_oracle.h.
 * TEST INFRASTRUCTURE / CPU BASELINE ONLY (never linked into libosh.so).
 * Build: make -C oracle (gcc -O2 -fopenmp -ffp-contract=off). */
#define _GNU_SOURCE
#include "muon_oracle.h"

#include <dlfcn.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------ streams */
uint64_t orc_splitmix64(uint64_t x) { /* verify.hpp:39-44 */
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t orc_stream_seed(uint64_t seed, int kind, int step, int param_id, int rank) {
  /* verify.hpp:78-86 */
  uint64_t s = orc_splitmix64(seed ^ (0x100000001ULL * (uint64_t)(kind + 1)));
  s = orc_splitmix64(s ^ (uint64_t)(step + 1));
  s = orc_splitmix64(s ^ ((uint64_t)(param_id + 1) << 20));
  return orc_splitmix64(s ^ ((uint64_t)(rank + 1) << 40));
}

void orc_normal_fill(uint64_t seed, double scale, int64_t n, double* out) {
  /* NormalStream (verify.hpp:49-76): the state is replaced by each output;
   * every pair of raw draws yields cos (returned) then sin (spare). */
  uint64_t state = seed;
  int64_t k = 0;
  while (k < n) {
    state = orc_splitmix64(state);
    const double u1 = ((double)(state >> 11) + 1.0) * 0x1p-53;
    state = orc_splitmix64(state);
    const double u2 = (double)(state >> 11) * 0x1p-53;
    const double mag = sqrt(-2.0 * log(u1));
    const double ang = 2.0 * 3.14159265358979323846 * u2;
    out[k++] = mag * cos(ang) * scale;
    if (k < n) out[k++] = mag * sin(ang) * scale;
  }
}

static void filled_normal(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  /* verify.hpp:88-97 and :102-113: m(i,j) = next() * (1/sqrt(shape[0])) */
  const double scale = 1.0 / sqrt((double)rows);
  orc_normal_fill(seed, scale, rows * cols, out);
}

void orc_synth_gradient(int64_t rows, int64_t cols, int param_id, uint64_t seed, int step,
                        int rank, double* out) {
  filled_normal(rows, cols, orc_stream_seed(seed, 0, step, param_id, rank), out);
}

void orc_init_weight(int64_t rows, int64_t cols, int param_id, uint64_t seed, double* out) {
  filled_normal(rows, cols, orc_stream_seed(seed, 1, 0, param_id, 0), out);
}

void orc_reduced_gradient(int64_t rows, int64_t cols, int param_id, uint64_t seed, int step,
                          int contributors, double* out) {
  /* verify.hpp:180-186: g = g_0; g += g_r for r = 1.. in ascending order. The
   * per-rank streams are independent, so they are drawn in parallel and then
   * summed in rank order. */
  const int64_t n = rows * cols;
  orc_synth_gradient(rows, cols, param_id, seed, step, 0, out);
  if (contributors <= 1) return;
  double* tmp = (double*)malloc(sizeof(double) * (size_t)n * (size_t)(contributors - 1));
  int r;
#pragma omp parallel for schedule(dynamic)
  for (r = 1; r < contributors; ++r)
    orc_synth_gradient(rows, cols, param_id, seed, step, r, tmp + (size_t)(r - 1) * (size_t)n);
  int64_t k;
#pragma omp parallel for schedule(static)
  for (k = 0; k < n; ++k) /* per element, ranks ascending: the reference's order */
    for (int q = 1; q < contributors; ++q) out[k] += tmp[(size_t)(q - 1) * (size_t)n + (size_t)k];
  free(tmp);
}

/* ------------------------------------------------------------ kernels */
static int g_threads = 0;
void orc_set_threads(int n) { g_threads = n; }
int orc_get_threads(void) {
#ifdef _OPENMP
  return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
  return 1;
#endif
}

typedef void (*cblas_dgemm64_fn)(int, int, int, int64_t, int64_t, int64_t, double, const double*,
                                 int64_t, const double*, int64_t, double, double*, int64_t);
static cblas_dgemm64_fn g_dgemm = NULL;

int orc_set_blas(const char* path, const char* symbol) {
  g_dgemm = NULL;
  if (path == NULL) return 0;
  void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (h == NULL) return 1;
  g_dgemm = (cblas_dgemm64_fn)dlsym(h, symbol ? symbol : "scipy_cblas_dgemm64_");
  return g_dgemm == NULL ? 2 : 0;
}

double orc_norm(const double* x, int64_t rows, int64_t cols) {
  double s = 0.0;
  if (g_dgemm != NULL) { /* FAST mode: storage order */
    for (int64_t k = 0; k < rows * cols; ++k) s += x[k] * x[k];
    return sqrt(s);
  }
  for (int64_t j = 0; j < cols; ++j) /* Eigen column-major traversal */
    for (int64_t i = 0; i < rows; ++i) s += x[i * cols + j] * x[i * cols + j];
  return sqrt(s);
}

/* c[j] = (((c[j] + a0*b0[j]) + a1*b1[j]) + a2*b2[j]) + a3*b3[j]: four
 * ascending k steps per pass, identical to one-at-a-time accumulation. */
__attribute__((target_clones("avx512f", "avx2", "default"))) static void axpy4(
    double* restrict c, const double* restrict b0, const double* restrict b1,
    const double* restrict b2, const double* restrict b3, double a0, double a1, double a2,
    double a3, int64_t n) {
  for (int64_t j = 0; j < n; ++j) {
    double t = c[j];
    t = t + a0 * b0[j];
    t = t + a1 * b1[j];
    t = t + a2 * b2[j];
    t = t + a3 * b3[j];
    c[j] = t;
  }
}

__attribute__((target_clones("avx512f", "avx2", "default"))) static void axpy1(
    double* restrict c, const double* restrict b, double a, int64_t n) {
  for (int64_t j = 0; j < n; ++j) c[j] = c[j] + a * b[j];
}

/* C (MxN) = A (MxK) * B (KxN), row-major, k ascending per element. */
static void gemm(const double* A, const double* B, double* C, int64_t M, int64_t N, int64_t K) {
  if (g_dgemm != NULL) {
    g_dgemm(101 /*row major*/, 111, 111, M, N, K, 1.0, A, K, B, N, 0.0, C, N);
    return;
  }
  const int64_t IB = 16, JB = 1024, KB = 256;
  memset(C, 0, sizeof(double) * (size_t)(M * N));
  const int nth = orc_get_threads();
  int64_t ib;
#pragma omp parallel for schedule(dynamic) num_threads(nth)
  for (ib = 0; ib < M; ib += IB) {
    const int64_t ie = ib + IB < M ? ib + IB : M;
    for (int64_t kb = 0; kb < K; kb += KB) {
      const int64_t ke = kb + KB < K ? kb + KB : K;
      for (int64_t jb = 0; jb < N; jb += JB) {
        const int64_t jn = (jb + JB < N ? jb + JB : N) - jb;
        for (int64_t i = ib; i < ie; ++i) {
          double* c = C + i * N + jb;
          const double* a = A + i * K;
          int64_t k = kb;
          for (; k + 4 <= ke; k += 4)
            axpy4(c, B + k * N + jb, B + (k + 1) * N + jb, B + (k + 2) * N + jb,
                  B + (k + 3) * N + jb, a[k], a[k + 1], a[k + 2], a[k + 3], jn);
          for (; k < ke; ++k) axpy1(c, B + k * N + jb, a[k], jn);
        }
      }
    }
  }
}

static void transpose(const double* x, int64_t rows, int64_t cols, double* t) {
  int64_t i;
#pragma omp parallel for schedule(static)
  for (i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) t[j * rows + i] = x[i * cols + j];
}

int orc_newton_schulz(double* x, int64_t rows, int64_t cols, int steps) {
  /* verify.hpp:118-134 */
  const double a = 3.4445, b = -4.7750, c = 2.0315;
  const double norm = orc_norm(x, rows, cols);
  if (norm == 0.0) return 1;
  const int flip = rows > cols;
  const int64_t m = flip ? cols : rows, n = flip ? rows : cols;
  const size_t mn = (size_t)(m * n);
  double* X = (double*)malloc(sizeof(double) * mn);
  double* XT = (double*)malloc(sizeof(double) * mn);
  double* A = (double*)malloc(sizeof(double) * (size_t)(m * m));
  double* Bt = (double*)malloc(sizeof(double) * mn);
  double* Ct = (double*)malloc(sizeof(double) * mn);
  if (flip)
    transpose(x, rows, cols, X);
  else
    memcpy(X, x, sizeof(double) * mn);
  for (size_t k = 0; k < mn; ++k) X[k] /= norm;
  for (int s = 0; s < steps; ++s) {
    transpose(X, m, n, XT);
    gemm(X, XT, A, m, m, n);  /* xxt   = x * x^T   */
    gemm(A, X, Bt, m, n, m);  /* bterm = xxt * x   */
    gemm(A, Bt, Ct, m, n, m); /* cterm = xxt * bterm */
    size_t k;
#pragma omp parallel for schedule(static)
    for (k = 0; k < mn; ++k) {
      const double t = a * X[k] + b * Bt[k];
      X[k] = t + c * Ct[k];
    }
  }
  if (flip)
    transpose(X, m, n, x);
  else
    memcpy(x, X, sizeof(double) * mn);
  free(X);
  free(XT);
  free(A);
  free(Bt);
  free(Ct);
  return 0;
}

void orc_muon_apply(int64_t rows, int64_t cols, int is_matrix, double lr, double beta,
                    int ns_steps, double* w, double* m, const double* g, double* update_norm) {
  /* verify.hpp:138-147 */
  const int64_t n = rows * cols;
  double* before = NULL;
  if (update_norm != NULL) {
    before = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(before, w, sizeof(double) * (size_t)n);
  }
  /* elementwise loops are independent per element: threaded, same values */
  int64_t k;
#pragma omp parallel for schedule(static)
  for (k = 0; k < n; ++k) m[k] = beta * m[k] + g[k];
  if (is_matrix) {
    double* u = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(u, m, sizeof(double) * (size_t)n);
    orc_newton_schulz(u, rows, cols, ns_steps);
#pragma omp parallel for schedule(static)
    for (k = 0; k < n; ++k) w[k] -= lr * u[k];
    free(u);
  } else {
#pragma omp parallel for schedule(static)
    for (k = 0; k < n; ++k) w[k] -= lr * m[k];
  }
  if (update_norm != NULL) {
    for (int64_t k = 0; k < n; ++k) before[k] = w[k] - before[k];
    *update_norm = orc_norm(before, rows, cols);
    free(before);
  }
}
