/*
 * muon_oracle.h — fp64 CPU restatement of the reference's Muon path.
 *
 * TEST INFRASTRUCTURE / CPU BASELINE ONLY. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load liboracle.so; the product path
 * (libosh.so) never links or calls it.
 *
 * Follows proj/include/optishard/verify.hpp (reference checkout):
 *   orc_splitmix64        :39-44
 *   orc_normal_*          :49-76   (sequential splitmix64 chain, Box-Muller cos then sin)
 *   orc_stream_seed       :78-86
 *   orc_filled_normal     :88-97   (row-major fill order)
 *   orc_synth_gradient    :102-107 (scale 1/sqrt(shape[0]))
 *   orc_init_weight       :109-113
 *   orc_newton_schulz     :118-134 (zero-norm passthrough, transpose if rows>cols,
 *                                   reference 3-product form A=XX^T, B=AX, C=AB)
 *   orc_muon_apply        :138-147
 *   orc_reduced_gradient  :180-186 (ascending-rank fp64 sum)
 * Arrays are row-major. In EXACT mode every product accumulates k in
 * ascending order with separate multiply/add and norms sum in column-major
 * order — the evaluation order of oracle/eigen_shim, so results equal the
 * reference compiled against the shim bit for bit (tests/test_oracle.py).
 * FAST mode (orc_set_blas) routes products through an OpenBLAS dgemm for the
 * timed CPU baseline; values then differ from EXACT by fp64 rounding only.
 */
#ifndef MUON_ORACLE_H_
#define MUON_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_stream_seed(uint64_t seed, int kind, int step, int param_id, int rank);

/* n draws of the NormalStream seeded with `seed`. */
void orc_normal_fill(uint64_t seed, double scale, int64_t n, double* out);

/* shape = {rows, cols}; cols = 1 for vectors (ndim 1). */
void orc_synth_gradient(int64_t rows, int64_t cols, int param_id, uint64_t seed, int step,
                        int rank, double* out);
void orc_init_weight(int64_t rows, int64_t cols, int param_id, uint64_t seed, double* out);
void orc_reduced_gradient(int64_t rows, int64_t cols, int param_id, uint64_t seed, int step,
                          int contributors, double* out);

/* In place on x (rows x cols). Returns 0, or 1 when the input norm was 0. */
int orc_newton_schulz(double* x, int64_t rows, int64_t cols, int steps);

/* momentum = beta*momentum + grad; matrix: w -= lr*NS(momentum), vector:
 * w -= lr*momentum. is_matrix selects the branch (verify.hpp:142).
 * Writes ||w_new - w_old||_F (column-major sum) to *update_norm if non-NULL. */
void orc_muon_apply(int64_t rows, int64_t cols, int is_matrix, double lr, double beta,
                    int ns_steps, double* w, double* m, const double* g, double* update_norm);

/* Frobenius norm, column-major summation order (oracle/eigen_shim). */
double orc_norm(const double* x, int64_t rows, int64_t cols);

/* FAST mode: path to a library exporting an ILP64 cblas_dgemm under
 * `symbol` (numpy's bundled OpenBLAS: "scipy_cblas_dgemm64_"). NULL path
 * returns to EXACT mode. Returns 0 on success. */
int orc_set_blas(const char* path, const char* symbol);
/* OpenMP worker threads for EXACT-mode kernels (<= 0: runtime default). */
void orc_set_threads(int n);
int orc_get_threads(void);

#ifdef __cplusplus
}
#endif
#endif
