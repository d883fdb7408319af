// Elementwise and per-matrix kernels of the blocked SOAP step (DESIGN.md
// "SOAP"; specification: oracle/soap_oracle.py). The projections into and
// out of the eigenbasis, the statistics and the refresh's products (S Q,
// Q^T Q, L^-1 Q^T) run on the tcgen05 GEMM (ns_gemm.cu: SPLIT / STAT / GRAM
// epilogues, bf16x3 operands where precision matters); the Cholesky factor
// and its inverse come from soap_chol_inv (one CTA per matrix, fp32 CUDA
// cores). Everything else here is HBM-bound elementwise work.
//
//   soap_prep      g (tensor layout, bf16/fp32, optionally the NVLS multicast
//                  sum), M (fp32 tensor layout) -> M = b1 M + (1-b1) g and,
//                  per block, bf16x3 splits of G (column and row), G^T
//                  (column) and M (row)
//   soap_rot       V = b2 V + (1-b2) G'^2 ; N' = (M'/bc1) / (sqrt(V/bc2) + eps)
//                  over a class's [nb][p][ldq] block arrays (G', M', V fp32)
//   soap_apply     W -= lr * N (N per block, bf16) ; replica ; tile sums
//   soap_adam      vectors / vocabulary matrices: elementwise Adam
//   soap_basis     refresh helper, one CTA per matrix: Y += c Q (c = shift *
//                  ||S||_F), est_j = q_j . y_j, stable descending order,
//                  Q <- Y[:, order] with unit columns (column-major fp32)
//   soap_vperm     V'[i][j] = V[oL[i]][oR[j]] (the basis order change)
//   soap_qcast     fp32 column-major Q -> bf16 Q^T column-split, Q row-major,
//                  Q row-split
//   soap_eye       Q = I (column-major fp32, zero padding)
//   soap_split     fp32 matrix -> bf16x6 column / row splits (refresh operands)
//   soap_chol_inv  C = L L^T and L^-1 (blocked right-looking Cholesky, then a
//                  row-block forward substitution), one CTA per matrix
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "muon_kernels.cuh"
#include "shampoo_kernels.cuh"

namespace osh {

// bf16x3 split layouts (fp32-accurate tcgen05 products, ns_gemm kEpiSplit):
// a value x is stored as hi = bf16(x), lo = bf16(x - hi) in four segments
// (hi, lo, hi, hi) of `seg` elements each (zero padded from the logical size
// to seg). COLUMN-split [rows][4 seg]: the K-major A view is segments 0-2,
// the K-major B view segments 1-3. ROW-split [4 seg][cols]: the MN-major B
// view is row segments 1-3. A . B over the 3-segment K then sums
// hi*lo + lo*hi + hi*hi.
struct SoapPrepTask {
  const void* g;          // tensor base (or its multicast address when g_mc)
  float* m;               // fp32 momentum, tensor layout (same indexing as g)
  long long g_ld;         // tensor row stride (= cols)
  int g_mc, vec;
  int r0, c0, p, q;       // block origin and size inside the tensor
  __nv_bfloat16* gs;      // G   column-split [p][4 ldq]
  __nv_bfloat16* gts;     // G^T column-split [q][4 ldp]
  __nv_bfloat16* grs;     // G   row-split    [4 ldp][ldq]
  __nv_bfloat16* mrs;     // M   row-split    [4 ldp][ldq]
  long long ldq, ldp;
  long long tile_start;   // prefix over 64x64 tiles of ldp x ldq (pads written 0)
  int tiles_c;
  int exact;              // gradients exact in bf16: only the segments the fast
                          // path reads are written (G / G^T hi, G rows 2-3)
};

struct SoapRotTask {      // one class: nb blocks of [p][ldq] (elements = nb * p * ldq)
  const float* gp;
  const float* mp;
  float* v;
  __nv_bfloat16* nrot;
  long long ldq;          // row stride; columns [q, ldq) are padding (written 0)
  int q, pad_;
  long long elems;
  long long chunk_start;  // prefix over kSoapRotChunk-element chunks
};
constexpr int kSoapRotChunk = 8192;

struct SoapAdamTask {
  const void* g;
  int g_mc, rep_mc, vec, pad_;
  float* m;
  float* v;
  float* w;
  __nv_bfloat16* replica;
  long long n;
  long long tile_start;   // tiles of kShSgdTile elements
  double* partial;        // absolute
};

struct SoapBasisTask {    // one statistics matrix S (n x n) and its basis Q
  const float* s;         // [n][lds] fp32 (symmetric)
  long long lds;
  float* q;               // column-major [n][ldq]: column j at q + j * ldq
  float* y;               // S Q (column-major, same ld), from this library's tcgen05 STAT GEMM
  long long ldq;
  int* order;             // [n] out: new column k = old column order[k]
  int n, pad_;
};

struct SoapVpermTask {    // one block's V [p][ldq] permuted into dst
  const float* v;
  float* dst;
  const int* ol;          // [p]
  const int* orr;         // [q]
  int p, q;
  long long ldq;
  long long tile_start;   // 64x64 tiles of p x q
  int tiles_c, pad_;
};

struct SoapQcastTask {    // fp32 column-major Q (n x n) -> bf16 copies (each nullable)
  const float* q;
  long long ldq;
  __nv_bfloat16* qt_split;  // Q^T column-split [n][4 ldb]
  __nv_bfloat16* q_row;     // Q row-major hi   [n][ldb]
  __nv_bfloat16* q_rsplit;  // Q row-split      [4 ldb][ldb]
  long long ldb;
  int n, pad_;
  long long tile_start;
  int tiles_c, pad2_;
};

// bf16x6 (~24-bit) split for the basis refresh, whose power iteration
// amplifies operand rounding: x = h + m + l (three bf16 terms); the A layout
// stores segments (h, m, h, l, m, h) and the B layout (h, h, m, h, m, l), so
// one contraction over K = 6 seg sums h*h + m*h + h*m + l*h + m*m + h*l.
struct SoapSplitTask {    // fp32 [rows][lds] -> bf16x6 copies (each nullable), pads 0
  const float* src;
  long long lds;
  int rows, cols;         // logical size; tiles cover [rup(rows,64)] x [rup(cols,64)]
  __nv_bfloat16* col_a;   // column A layout [rows][6 ldd]
  __nv_bfloat16* col_b;   // column B layout [rows][6 ldd]
  __nv_bfloat16* row_b;   // row B layout    [6 ldd][ldd] (rows up to ldd, pads 0)
  long long ldd;
  long long tile_start;
  int tiles_c, pad_;
};
constexpr int kSoapSplitSegs = 6;

// Batched Cholesky + triangular inverse, one CTA per matrix (n <= 1024):
// C (SPD, fp32 [ld][ld], only [n][n] meaningful; the pad is made the identity)
// is factored in place as C = L L^T (lower) and L^-1 is written to linv
// ([ld][ld], upper part 0). Non-positive pivots are clamped to a tiny value.
struct SoapCholTask {
  float* c;
  float* linv;
  long long ld;
  int n, pad_;
};
constexpr int kSoapCholMaxN = 1024;

cudaError_t launch_soap_split(const SoapSplitTask* d, int n, long long tiles, cudaStream_t s);
cudaError_t launch_soap_chol_inv(const SoapCholTask* d, int n, cudaStream_t s);
cudaError_t launch_soap_prep(const SoapPrepTask* d, int n, long long tiles, int grad_dtype,
                             float beta1, cudaStream_t s);
cudaError_t launch_soap_rot(const SoapRotTask* d, int n, long long chunks, float beta2,
                            float inv_bc1, float inv_bc2, float eps, cudaStream_t s);
// tasks: ShApplyTask with m unused (nullptr); blocks[].scale unused
cudaError_t launch_soap_apply(const ShApplyTask* d, int n, long long tiles, float lr,
                              cudaStream_t s);
cudaError_t launch_soap_adam(const SoapAdamTask* d, int n, long long tiles, int grad_dtype,
                             float beta1, float beta2, float inv_bc1, float inv_bc2, float eps,
                             float lr, cudaStream_t s);
cudaError_t launch_soap_basis(const SoapBasisTask* d, int n, float shift, cudaStream_t s);
cudaError_t launch_soap_vperm(const SoapVpermTask* d, int n, long long tiles, cudaStream_t s);
cudaError_t launch_soap_qcast(const SoapQcastTask* d, int n, long long tiles, cudaStream_t s);
cudaError_t launch_soap_eye(float* q, long long ldq, long long bstride, int n, int batch,
                            cudaStream_t s);

}  // namespace osh
