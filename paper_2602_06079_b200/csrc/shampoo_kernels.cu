// Blocked-Shampoo elementwise kernels (see shampoo_kernels.cuh).
#include "shampoo_kernels.cuh"

#include "elementwise_util.cuh"

namespace osh {
namespace {

using namespace ew;

// task of linear tile t (tasks sorted by tile_start)
template <typename Task>
__device__ __forceinline__ int find_task(const Task* tasks, int n, long long t) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tasks[mid].tile_start <= t) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// ---------------------------------------------------------------- prep
template <typename G>
__global__ void __launch_bounds__(256) sh_prep_kernel(const ShPrepTask* tasks, int n) {
  __shared__ __nv_bfloat16 tile[kTile][kTile + 2];
  __shared__ double red[8];
  const long long t = blockIdx.x;
  const ShPrepTask T = tasks[find_task(tasks, n, t)];
  const long long local = t - T.tile_start;
  const int lr0 = static_cast<int>(local / T.tiles_c) * kTile;  // block-local
  const int lc0 = static_cast<int>(local % T.tiles_c) * kTile;
  float sq = 0.f;
  if (T.vec) {
    const int c8 = (threadIdx.x & 7) * 8, rr = threadIdx.x >> 3;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int lr = rr + 32 * h;
      const int r = lr0 + lr, c = lc0 + c8;
      float v[8];
      if (r < T.p && c < T.q) {
        const size_t idx = static_cast<size_t>(T.r0 + r) * T.g_ld + T.c0 + c;
        if (T.g_mc) mc_load_grad8<G>(T.g, idx, v);
        else load_grad8<G>(T.g, idx, v);
#pragma unroll
        for (int q = 0; q < 8; ++q) sq += v[q] * v[q];
        *reinterpret_cast<uint4*>(T.gb + static_cast<size_t>(r) * T.ldq + c) = pack_bf16x8(v);
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = 0.f;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) tile[lr][c8 + q] = __float2bfloat16_rn(v[q]);
    }
  } else {
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int i = 0; i < kTile / 8; ++i) {
      const int lr = ty + 8 * i, r = lr0 + lr;
      for (int j = 0; j < kTile / 32; ++j) {
        const int lc = tx + 32 * j, c = lc0 + lc;
        __nv_bfloat16 x = __float2bfloat16_rn(0.f);
        if (r < T.p && c < T.q) {
          const float v = load_grad<G>(T.g, static_cast<size_t>(T.r0 + r) * T.g_ld + T.c0 + c);
          sq += v * v;
          x = __float2bfloat16_rn(v);
          T.gb[static_cast<size_t>(r) * T.ldq + c] = x;
        }
        tile[lr][lc] = x;
      }
    }
  }
  __syncthreads();
  // transposed block: row = original column
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = 0; i < kTile / 8; ++i) {
    const int lc = ty + 8 * i, c = lc0 + lc;
    for (int j = 0; j < kTile / 32; ++j) {
      const int lr = tx + 32 * j, r = lr0 + lr;
      if (r < T.p && c < T.q) T.gbt[static_cast<size_t>(c) * T.ldp + r] = tile[lr][lc];
    }
  }
  const double s = block_sum(static_cast<double>(sq), red);
  if (threadIdx.x == 0) T.partial[t] = s;
}

// ---------------------------------------------------------------- sumsq
template <typename E>
__device__ __forceinline__ float to_f(E x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename E>
__global__ void __launch_bounds__(256) sh_sumsq_kernel(const ShMatTask<E>* tasks, int n) {
  __shared__ double red[8];
  const long long t = blockIdx.x;
  const ShMatTask<E> T = tasks[find_task(tasks, n, t)];
  const long long local = t - T.tile_start;
  const int r0 = static_cast<int>(local / T.tiles_c) * kTile;
  const int c0 = static_cast<int>(local % T.tiles_c) * kTile;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double sq = 0.0;  // fp64: statistics entries can be large
  for (int i = 0; i < kTile / 8; ++i) {
    const int r = r0 + ty + 8 * i;
    for (int j = 0; j < kTile / 32; ++j) {
      const int c = c0 + tx + 32 * j;
      if (r < T.rows && c < T.cols) {
        const double v = to_f<E>(T.src[static_cast<size_t>(r) * T.ld + c]);
        sq += v * v;
      }
    }
  }
  const double s = block_sum(sq, red);
  if (threadIdx.x == 0) T.partial[t] = s;
}

// ---------------------------------------------------------------- roots
__device__ __forceinline__ void store_split4(__nv_bfloat16* row_base, long long seg, int c, float v) {
  const __nv_bfloat16 hi = __float2bfloat16_rn(v);
  const __nv_bfloat16 lo = __float2bfloat16_rn(v - __bfloat162float(hi));
  row_base[c] = hi;
  row_base[seg + c] = lo;
  row_base[2 * seg + c] = hi;
  row_base[3 * seg + c] = hi;
}

__global__ void __launch_bounds__(256) sh_root_init_kernel(const ShRootTask* tasks, int n,
                                                           float eps) {
  const long long t = blockIdx.x;
  const ShRootTask T = tasks[find_task(tasks, n, t)];
  const long long local = t - T.tile_start;
  const int r0 = static_cast<int>(local / T.tiles_c) * kTile;
  const int c0 = static_cast<int>(local % T.tiles_c) * kTile;
  const double ss = *T.sumsq;
  const bool zero = !(ss > 0.0);
  const float inv_c = zero ? 0.f : static_cast<float>(1.0 / sqrt(ss));
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = 0; i < kTile / 8; ++i) {
    const int r = r0 + ty + 8 * i;
    if (r >= T.n) continue;
    __nv_bfloat16* arow = T.a5 + static_cast<size_t>(r) * T.ld5;
    __nv_bfloat16* xrow = T.x5 + static_cast<size_t>(r) * T.ld5;
    for (int j = 0; j < kTile / 32; ++j) {
      const int c = c0 + tx + 32 * j;
      if (c >= T.n) continue;
      const float d = r == c ? 1.f : 0.f;
      const float a = zero ? d : T.s[static_cast<size_t>(r) * T.lds + c] * inv_c + eps * d;
      store_split4(arow, T.ld5 / 4, c, a);  // segment width = n rounded up to 8
      store_split4(xrow, T.ld5 / 4, c, d);
    }
  }
  const int seg = static_cast<int>(T.ld5 / 4);
  if (seg > T.n && c0 + kTile >= T.n) {  // last column tile: zero the pad columns
    const __nv_bfloat16 z = __float2bfloat16_rn(0.f);
    for (int i = threadIdx.x; i < kTile * 4 * (seg - T.n); i += 256) {
      const int r = r0 + i / (4 * (seg - T.n));
      const int k = i % (4 * (seg - T.n));
      if (r >= T.n) continue;
      const size_t off = static_cast<size_t>(r) * T.ld5 + (k / (seg - T.n)) * seg + T.n + k % (seg - T.n);
      T.a5[off] = z;
      T.x5[off] = z;
      for (int b = 0; b < 5; ++b) T.others[b][off] = z;
    }
  }
}

__global__ void sh_root_scale_kernel(const double* sumsq, float* scale, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double ss = sumsq[i];
  scale[i] = ss > 0.0 ? static_cast<float>(pow(ss, -0.125)) : 1.f;  // (sqrt ss)^(-1/4)
}

__global__ void __launch_bounds__(256) sh_newton_t_kernel(const ShNewtonTask* tasks, int n) {
  const long long t = blockIdx.x;
  const ShNewtonTask T = tasks[find_task(tasks, n, t)];
  const long long local = t - T.tile_start;
  const int r0 = static_cast<int>(local / T.tiles_c) * kTile;
  const int c0 = static_cast<int>(local % T.tiles_c) * kTile;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = 0; i < kTile / 8; ++i) {
    const int r = r0 + ty + 8 * i;
    if (r >= T.n) continue;
    const __nv_bfloat16* mrow = T.src5 + static_cast<size_t>(r) * T.ld5;
    __nv_bfloat16* trow = T.dst + static_cast<size_t>(r) * T.ldd;
    for (int j = 0; j < kTile / 32; ++j) {
      const int c = c0 + tx + 32 * j;
      if (c >= T.n) continue;
      const long long seg = T.ld5 / 4;
      const float m = __bfloat162float(mrow[c]) + __bfloat162float(mrow[seg + c]);
      store_split4(trow, seg, c, ((r == c ? 5.f : 0.f) - m) * 0.25f);
    }
  }
}

__global__ void __launch_bounds__(256) sh_extract_kernel(const ShNewtonTask* tasks, int n) {
  const long long t = blockIdx.x;
  const ShNewtonTask T = tasks[find_task(tasks, n, t)];
  const long long local = t - T.tile_start;
  const int r0 = static_cast<int>(local / T.tiles_c) * kTile;
  const int c0 = static_cast<int>(local % T.tiles_c) * kTile;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = 0; i < kTile / 8; ++i) {
    const int r = r0 + ty + 8 * i;
    if (r >= T.n) continue;
    for (int j = 0; j < kTile / 32; ++j) {
      const int c = c0 + tx + 32 * j;
      // the Newton products are in the upper-tile form: (r, c) from the
      // upper triangle, so P is exactly symmetric
      if (c < T.n)
        T.dst[static_cast<size_t>(r) * T.ldd + c] =
            T.src5[static_cast<size_t>(min(r, c)) * T.ld5 + max(r, c)];
    }
  }
}

__global__ void sh_graft_kernel(const double* gsq, const double* usq, float* scale, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  scale[i] = usq[i] > 0.0 ? static_cast<float>(sqrt(gsq[i] / usq[i])) : 0.f;
}

// ---------------------------------------------------------------- apply
__global__ void __launch_bounds__(256) sh_apply_kernel(const ShApplyTask* tasks, int n,
                                                       float beta1, float lrate) {
  __shared__ double red[8];
  const long long t = blockIdx.x;
  const ShApplyTask T = tasks[find_task(tasks, n, t)];
  const long long local = t - T.tile_start;
  const int r0 = static_cast<int>(local / T.tiles_c) * kTile;
  const int c0 = static_cast<int>(local % T.tiles_c) * kTile;
  // a 64x64 tile never straddles blocks (block edges are multiples of 64)
  const int bi = r0 / T.block, bj = c0 / T.block;
  const ShBlockRef B = T.blocks[bi * T.blocks_c + bj];
  const float sc = *B.scale;
  const int br = r0 - bi * T.block, bc = c0 - bj * T.block;
  float sq = 0.f;
  if (T.vec) {
    const int c8 = (threadIdx.x & 7) * 8, rr = threadIdx.x >> 3;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int lr = rr + 32 * h;
      const int row = r0 + lr, col = c0 + c8;
      if (row >= T.rows || col >= T.cols) continue;
      float u[8], mv[8], wv[8];
      unpack_bf16x8(*reinterpret_cast<const uint4*>(B.u + static_cast<size_t>(br + lr) * B.ldu + bc + c8), u);
      const size_t idx = static_cast<size_t>(row) * T.cols + col;
      load_f8(T.m + idx, mv);
      load_f8(T.w + idx, wv);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        mv[q] = beta1 * mv[q] + sc * u[q];
        const float upd = lrate * mv[q];
        wv[q] -= upd;
        sq += upd * upd;
      }
      store_f8(T.m + idx, mv);
      store_f8(T.w + idx, wv);
      if (T.replica != nullptr) {
        if (T.rep_mc) mc_store16(T.replica + idx, pack_bf16x8(wv));
        else *reinterpret_cast<uint4*>(T.replica + idx) = pack_bf16x8(wv);
      }
    }
  } else {
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int i = 0; i < kTile / 8; ++i) {
      const int lr = ty + 8 * i, row = r0 + lr;
      if (row >= T.rows) continue;
      for (int j = 0; j < kTile / 32; ++j) {
        const int lc = tx + 32 * j, col = c0 + lc;
        if (col >= T.cols) continue;
        const float u = __bfloat162float(B.u[static_cast<size_t>(br + lr) * B.ldu + bc + lc]);
        const size_t idx = static_cast<size_t>(row) * T.cols + col;
        const float mv = beta1 * T.m[idx] + sc * u;
        T.m[idx] = mv;
        const float upd = lrate * mv;
        const float w = T.w[idx] - upd;
        T.w[idx] = w;
        if (T.replica != nullptr) T.replica[idx] = __float2bfloat16_rn(w);
        sq += upd * upd;
      }
    }
  }
  const double s = block_sum(static_cast<double>(sq), red);
  if (threadIdx.x == 0) {
    T.partial[t] = s;
    if (T.rep_mc) __threadfence_system();
  }
}

template <typename G>
__global__ void __launch_bounds__(256) sh_sgd_kernel(const ShSgdTask* tasks, int n, float beta1,
                                                     float lr) {
  __shared__ double red[8];
  const long long t = blockIdx.x;
  const ShSgdTask T = tasks[find_task(tasks, n, t)];
  const long long base = (t - T.tile_start) * kShSgdTile;
  float sq = 0.f;
  if (T.vec) {
    for (long long i = base + threadIdx.x * 8; i < base + kShSgdTile && i < T.n; i += 256 * 8) {
      float g[8], mv[8], wv[8];
      if (T.g_mc) mc_load_grad8<G>(T.g, static_cast<size_t>(i), g);
      else load_grad8<G>(T.g, static_cast<size_t>(i), g);
      load_f8(T.m + i, mv);
      load_f8(T.w + i, wv);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        mv[q] = beta1 * mv[q] + g[q];
        const float upd = lr * mv[q];
        wv[q] -= upd;
        sq += upd * upd;
      }
      store_f8(T.m + i, mv);
      store_f8(T.w + i, wv);
      if (T.replica != nullptr) {
        if (T.rep_mc) mc_store16(T.replica + i, pack_bf16x8(wv));
        else *reinterpret_cast<uint4*>(T.replica + i) = pack_bf16x8(wv);
      }
    }
  } else {
    for (long long i = base + threadIdx.x; i < base + kShSgdTile && i < T.n; i += 256) {
      const float mv = beta1 * T.m[i] + load_grad<G>(T.g, static_cast<size_t>(i));
      T.m[i] = mv;
      const float upd = lr * mv;
      const float w = T.w[i] - upd;
      T.w[i] = w;
      if (T.replica != nullptr) T.replica[i] = __float2bfloat16_rn(w);
      sq += upd * upd;
    }
  }
  const double s = block_sum(static_cast<double>(sq), red);
  if (threadIdx.x == 0) {
    T.partial[t] = s;
    if (T.rep_mc) __threadfence_system();
  }
}

bool bad_grid(long long tiles) { return tiles <= 0 || tiles > 0x7fffffffll; }

}  // namespace

cudaError_t launch_sh_prep(const ShPrepTask* d, int n, long long tiles, int grad_dtype, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(tiles)) return cudaErrorInvalidValue;
  if (grad_dtype == kGradBF16)
    sh_prep_kernel<__nv_bfloat16><<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n);
  else
    sh_prep_kernel<float><<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n);
  return cudaGetLastError();
}

cudaError_t launch_sh_sumsq_f32(const ShMatTask<float>* d, int n, long long tiles, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(tiles)) return cudaErrorInvalidValue;
  sh_sumsq_kernel<float><<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n);
  return cudaGetLastError();
}

cudaError_t launch_sh_sumsq_bf16(const ShMatTask<__nv_bfloat16>* d, int n, long long tiles,
                                 cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(tiles)) return cudaErrorInvalidValue;
  sh_sumsq_kernel<__nv_bfloat16><<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n);
  return cudaGetLastError();
}

cudaError_t launch_sh_root_init(const ShRootTask* d, int n, long long tiles, float eps,
                                cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(tiles)) return cudaErrorInvalidValue;
  sh_root_init_kernel<<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n, eps);
  return cudaGetLastError();
}

cudaError_t launch_sh_root_scale(const double* sumsq, float* scale, int n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  sh_root_scale_kernel<<<(n + 255) / 256, 256, 0, s>>>(sumsq, scale, n);
  return cudaGetLastError();
}

cudaError_t launch_sh_newton_t(const ShNewtonTask* d, int n, long long tiles, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(tiles)) return cudaErrorInvalidValue;
  sh_newton_t_kernel<<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n);
  return cudaGetLastError();
}

cudaError_t launch_sh_extract(const ShNewtonTask* d, int n, long long tiles, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(tiles)) return cudaErrorInvalidValue;
  sh_extract_kernel<<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n);
  return cudaGetLastError();
}

cudaError_t launch_sh_graft(const double* gsq, const double* usq, float* scale, int n,
                            cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  sh_graft_kernel<<<(n + 255) / 256, 256, 0, s>>>(gsq, usq, scale, n);
  return cudaGetLastError();
}

cudaError_t launch_sh_apply(const ShApplyTask* d, int n, long long tiles, float beta1, float lr,
                            cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(tiles)) return cudaErrorInvalidValue;
  sh_apply_kernel<<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n, beta1, lr);
  return cudaGetLastError();
}

cudaError_t launch_sh_sgd(const ShSgdTask* d, int n, long long tiles, int grad_dtype, float beta1,
                          float lr, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(tiles)) return cudaErrorInvalidValue;
  if (grad_dtype == kGradBF16)
    sh_sgd_kernel<__nv_bfloat16><<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n, beta1, lr);
  else
    sh_sgd_kernel<float><<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n, beta1, lr);
  return cudaGetLastError();
}

}  // namespace osh
