// Elementwise kernels of the blocked Shampoo step (
// specification: oracle/shampoo_oracle.py). The contractions (statistics,
// coupled-Newton inverse roots, preconditioning) run on the tcgen05 GEMM
// (ns_gemm.cu epilogues STAT / SPLIT / UPDATE / GRAM); everything here is
// HBM-bound and works on 64x64 tiles with fixed-order fp64 tile partials, so
// results do not depend on which tensors share a launch.
//
//   sh_prep        g (tensor layout, bf16/fp32, optionally the NVLS multicast
//                  sum) -> G_b [p][ldq] and G_b^T [q][ldp] bf16 per block,
//                  tile sums of g^2
//   sh_sumsq       tile sums of x^2 of an fp32 or bf16 matrix
//   sh_root_init   A = S/||S|| + eps I and X = I in the split-bf16 layout
//                  [hi | lo | hi | hi] (identity when S = 0)
//   sh_root_scale  c^(-1/4) per statistics matrix (1 when S = 0)
//   sh_newton_t    T = (5 I - M) / 4 in the split layout
//   sh_extract     hi segment of the converged root -> compact bf16 P
//   sh_graft       per block scale ||G_b|| / ||U_b|| (0 when U_b = 0)
//   sh_apply       M = beta1 M + scale_b U_b ; W -= lr M ; replica ; tile sums
//   sh_sgd         vectors / vocabulary matrices: M = beta1 M + g ; W -= lr M
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "muon_kernels.cuh"

namespace osh {

struct ShPrepTask {
  const void* g;          // tensor base (or its multicast address when g_mc)
  long long g_ld;         // tensor row stride (= cols)
  int g_mc, vec;
  int r0, c0, p, q;       // block origin and size inside the tensor
  __nv_bfloat16* gb;      // [p][ldq]
  __nv_bfloat16* gbt;     // [q][ldp]
  long long ldq, ldp;
  long long tile_start;   // prefix over 64x64 tiles of p x q
  int tiles_c, pad_;
  double* partial;        // absolute: partial[tile_start + local]
};

template <typename T>
struct ShMatTask {        // a plain n_rows x n_cols matrix (sumsq / extract / root tasks)
  const T* src;
  long long ld;
  int rows, cols;
  long long tile_start;
  int tiles_c, pad_;
  double* partial;
};

struct ShRootTask {       // one statistics matrix of size n (split layout ld5 = 4 * seg)
  const float* s;         // fp32 statistics [n][lds]
  long long lds;
  __nv_bfloat16* a5;      // M0 = A (split)
  __nv_bfloat16* x5;      // X0 = I (split)
  long long ld5;
  int n, pad_;
  const double* sumsq;    // ||S||_F^2 (one value)
  long long tile_start;
  int tiles_c, pad2_;
  // the matrix's other split buffers (X1, M1, T, T2, T4): their pad columns
  // [n, seg) of every segment are zeroed with A's and X's, because the bf16x3
  // K dimension runs over them and the workspace is reused across waves
  __nv_bfloat16* others[5];
};

struct ShNewtonTask {     // T = (5I - M)/4, or P = hi(X) when extracting
  const __nv_bfloat16* src5;
  __nv_bfloat16* dst;     // split layout (newton_t) or compact [n][ldp] (extract)
  long long ld5, ldd;
  int n, pad_;
  long long tile_start;
  int tiles_c, pad2_;
};

struct ShBlockRef {       // one block as the apply kernel sees it
  const __nv_bfloat16* u; // [p][ldu]
  long long ldu;
  const float* scale;     // graft scale of this block
};

struct ShApplyTask {
  float* w;
  float* m;
  __nv_bfloat16* replica;
  int rep_mc, vec;
  int rows, cols;
  int block, blocks_c;    // block edge and blocks per block-row
  const ShBlockRef* blocks;
  long long tile_start;
  int tiles_c, pad_;
  double* partial;        // absolute
};

struct ShSgdTask {
  const void* g;
  int g_mc, rep_mc, vec, pad_;
  float* m;
  float* w;
  __nv_bfloat16* replica;
  long long n;
  long long tile_start;   // tiles of kShSgdTile elements
  double* partial;        // absolute
};
constexpr int kShSgdTile = 8192;

cudaError_t launch_sh_prep(const ShPrepTask* d, int n, long long tiles, int grad_dtype, cudaStream_t s);
cudaError_t launch_sh_sumsq_f32(const ShMatTask<float>* d, int n, long long tiles, cudaStream_t s);
cudaError_t launch_sh_sumsq_bf16(const ShMatTask<__nv_bfloat16>* d, int n, long long tiles,
                                 cudaStream_t s);
cudaError_t launch_sh_root_init(const ShRootTask* d, int n, long long tiles, float eps,
                                cudaStream_t s);
cudaError_t launch_sh_root_scale(const double* sumsq, float* scale, int n, cudaStream_t s);
cudaError_t launch_sh_newton_t(const ShNewtonTask* d, int n, long long tiles, cudaStream_t s);
cudaError_t launch_sh_extract(const ShNewtonTask* d, int n, long long tiles, cudaStream_t s);
cudaError_t launch_sh_graft(const double* gsq, const double* usq, float* scale, int n,
                            cudaStream_t s);
cudaError_t launch_sh_apply(const ShApplyTask* d, int n, long long tiles, float beta1, float lr,
                            cudaStream_t s);
cudaError_t launch_sh_sgd(const ShSgdTask* d, int n, long long tiles, int grad_dtype, float beta1,
                          float lr, cudaStream_t s);

}  // namespace osh
