// HBM-bound elementwise kernels around the Newton-Schulz GEMMs.
//
//  momentum_matrix_kernel  (SURVEY.md §2.2 K1+K2) per owned matrix tile:
//      m = beta*m + g            (fp32 state, g = reduced gradient bf16/fp32)
//      per-tile sum of m^2 (fp64, reduced in fixed order -> ||m||_F)
//      X0 = bf16(m) in the Newton-Schulz orientation (transposed through
//      shared memory when rows > cols, verify.hpp:123-124); the 1/||m|| scale
//      is folded into the first GEMM epilogues instead of a second pass.
//  momentum_vector_kernel  (K7) m = beta*m + g; w -= lr*m; replica = bf16(w)
//  ns_scales_kernel        s = 1/||m|| (0 for a zero matrix: the reference
//      returns the zero iterate unchanged, verify.hpp:122), s^2 for the Gram.
// Algorithmic HBM bytes per element: matrix pass 4+2 (g fp32/bf16 read) +
// 4 (m read) + 4 (m write) + 2 (X0 write); vector pass 4+2 + 4+4 + 4+4 + 2.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace osh {

enum GradDtype : int { kGradF32 = 0, kGradBF16 = 1 };

constexpr int kTile = 64;  // momentum tile edge (elements)

struct MomentumMatrixTask {
  const void* g;         // [rows][cols] reduced gradient (dtype per launch); with
                         // g_mc it is the NVLS multicast address of the local
                         // gradients and the kernel reads the cross-GPU sum
  int g_mc;              // 1: multimem.ld_reduce (RS-v fused into this kernel)
  int pad0_;
  float* m;              // [rows][cols] fp32 momentum
  __nv_bfloat16* x0;     // NS iterate: [rows][ldx] or, transposed, [cols][ldx]
  double* partial;       // [tiles of this task] per-tile sum of m^2 (fixed-order
                         // reduction in ns_scales keeps the step deterministic)
  int rows, cols;
  int ldx;
  int transposed;
  long long tile_start;  // first linear tile of this task (prefix sum)
  int tiles_c;           // column tiles
  int vec;               // 1: 128-bit path (cols % 8 == 0, 16-byte aligned rows)
};

struct MomentumVectorTask {
  int g_mc, rep_mc;            // NVLS fusion flags (see MomentumMatrixTask / ApplyTask)
  const void* g;
  float* m;
  float* w;
  __nv_bfloat16* replica;  // nullable
  double* sq_norm;         // += ||lr*m||^2, nullable
  long long n;
};

// Final Newton-Schulz output -> weight update, per 64x64 tile of W (original
// orientation): W -= lr * X (X read transposed through smem when the tensor
// is X^T), replica = bf16(W), per-tile sum of (lr*X)^2 for ||dW||.
// HBM bytes per element: 2 (X) + 4 + 4 (W) + 2 (replica) = 12.
struct ApplyTask {
  int rep_mc;                  // 1: replica is a multicast address: multimem.st (AG-v fused)
  int pad0_;
  const __nv_bfloat16* x;      // NS iterate [rows][ldx] or, transposed, [cols][ldx]
  const __nv_bfloat16* x_alt;  // the other ping-pong buffer (odd iteration counts)
  float* w;                // [rows][cols] fp32 master weight
  __nv_bfloat16* replica;  // [rows][cols] bf16 replica (nullable)
  double* partial;         // per-tile sums of (lr*x)^2 (rebased like MomentumMatrixTask)
  int rows, cols;
  int ldx;
  int transposed;
  long long tile_start;
  int tiles_c;
  int vec;                 // 1: 128-bit path (cols % 8 == 0, 16-byte aligned rows)
};

cudaError_t launch_apply_update(const ApplyTask* d_tasks, int n_tasks, long long total_tiles,
                                float lr, int use_alt, cudaStream_t s);
// Per slot i: out[target[i]] = sum(partial[begin_i .. begin_i + count_i)) (fixed order).
cudaError_t launch_partial_sums(const double* partial, const long long* begin, const int* count,
                                const int* target, double* out, int n, cudaStream_t s);

// Strided 2-D copies of 16-bit blocks (TP gather / scatter staging):
// dst[r*ldd + c] = src[r*lds + c], r < rows, c < cols, for every task.
// NVLS AG-v of fused FINAL tensors: the owner's freshly written local bf16
// slot is re-stored through the multicast address (every GPU's replica).
struct McCopyTask {
  const __nv_bfloat16* src;  // local replica slot
  __nv_bfloat16* dst;        // multicast address of the same slot
  long long n;               // elements (multiple of 8)
  long long vec_start;       // first 8-element vector of this task (prefix sum)
};
cudaError_t launch_mc_copy(const McCopyTask* d_tasks, int n_tasks, long long total_vecs,
                           cudaStream_t s);

// NVLS + TP: the DP owner's reduced gradient shard of a TP-plane tensor is
// read through the multicast address (the switch sums the DP group's
// gradients) and written over the owner's own local copy, which the TP
// gather then sends to the tensor's host. Only the owner reads its slice, so
// overwriting it in place is race-free; the step's end barrier keeps the
// peers' copies alive until then.
struct McReduceTask {
  const void* mc;            // multicast address of the slice
  void* dst;                 // the same slice in the local gradient buffer
  long long n;               // elements (multiple of 8)
  long long vec_start;       // first 8-element vector of this task (prefix sum)
};
cudaError_t launch_mc_reduce(const McReduceTask* d_tasks, int n_tasks, long long total_vecs,
                             int grad_bf16, cudaStream_t s);

// Completes symmetric fp32 matrices whose upper triangle alone is current
// (STAT GEMMs with symmetric = 2): S[i][j] = S[j][i] for i > j, 32 x 32 tiles
// of the lower triangle (diagonal tiles included), one CTA each.
struct SymFillTask {
  float* s;
  long long ld;
  int n;
  int tiles;                 // T (T + 1) / 2, T = ceil(n / 32)
  long long tile_start;      // prefix sum over the tasks
};
cudaError_t launch_sym_fill_lower(const SymFillTask* d_tasks, int n_tasks, long long total_tiles,
                                  cudaStream_t s);

struct CopyTask {
  const uint16_t* src;
  uint16_t* dst;
  long long lds, ldd;
  int rows, cols;
  long long tile_start;
  int tiles_c;
  int pad_;
};
cudaError_t launch_copy_blocks(const CopyTask* d_tasks, int n_tasks, long long total_tiles,
                               cudaStream_t s);

cudaError_t launch_momentum_matrix(const MomentumMatrixTask* d_tasks, int n_tasks,
                                   long long total_tiles, int grad_dtype, float beta,
                                   cudaStream_t s);
cudaError_t launch_momentum_vector(const MomentumVectorTask* d_tasks, int n_tasks, int grad_dtype,
                                   float beta, float lr, cudaStream_t s);
// Per slot i: s = 1/sqrt(sum(partial[begin_i .. begin_i+count_i))) (0 if the
// sum is 0); scale_update = s, scale_gram = s^2. Deterministic tree order.
cudaError_t launch_ns_scales(const double* partial, const long long* begin, const int* count,
                             float* scale_update, float* scale_gram, int n, cudaStream_t s);

}  // namespace osh
