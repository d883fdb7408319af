// Elementwise Muon kernels (see muon_kernels.cuh for the math and bytes).
#include "muon_kernels.cuh"

#include <algorithm>

#include "elementwise_util.cuh"

namespace osh {
namespace {

using namespace ew;

// One 64x64 tile of one matrix per CTA; 256 threads = 8 rows x 32 columns
// per pass, so every global access is a coalesced 128-byte (fp32) or
// 64-byte (bf16) warp transaction.
#ifndef OSH_MOM_MINB
#define OSH_MOM_MINB 4
#endif
#ifndef OSH_MOM_STREAM
#define OSH_MOM_STREAM 1
#endif
// streaming (read-once / write-once) accesses of the momentum pass
__device__ __forceinline__ void load_f8_stream(const float* p, float (&v)[8]) {
#if OSH_MOM_STREAM
  // one 256-bit load (sm_100) per 8 values, evicted first from L2
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
                 "=f"(v[7])
               : "l"(p));
#else
  load_f8(p, v);
#endif
}
__device__ __forceinline__ void store_f8_stream(float* p, const float (&v)[8]) {
#if OSH_MOM_STREAM
  asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
               "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
#else
  store_f8(p, v);
#endif
}

template <typename G>
__global__ void __launch_bounds__(256, OSH_MOM_MINB) momentum_matrix_kernel(const MomentumMatrixTask* tasks,
                                                              int n_tasks, float beta) {
  __shared__ __nv_bfloat16 tile[kTile][kTile + 2];
  __shared__ double red[8];
  const long long t = blockIdx.x;
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tasks[mid].tile_start <= t) lo = mid;
    else hi = mid - 1;
  }
  const MomentumMatrixTask T = tasks[lo];
  const long long local = t - T.tile_start;
  const int r0 = static_cast<int>(local / T.tiles_c) * kTile;
  const int c0 = static_cast<int>(local % T.tiles_c) * kTile;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  float sq = 0.f;
  if (T.vec) {
    // 8 columns x 2 rows per thread: 128-bit loads / stores, 8 threads per
    // 64-element row segment (fully coalesced 256 B of fp32 per row)
    const int c8 = (threadIdx.x & 7) * 8, rr = threadIdx.x >> 3;
    // both rows' loads are issued before either is consumed: two 16-byte
    // requests in flight per thread (NVLS: each is a switch round trip)
    float g[2][8], mv[2][8];
    bool ok[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = r0 + rr + 32 * h, col = c0 + c8;
      ok[h] = row < T.rows && col < T.cols;
      if (ok[h]) {
        const size_t idx = static_cast<size_t>(row) * T.cols + col;
        if (T.g_mc) mc_load_grad8<G>(T.g, idx, g[h]);
        else load_grad8<G>(T.g, idx, g[h]);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (ok[h]) load_f8_stream(T.m + static_cast<size_t>(r0 + rr + 32 * h) * T.cols + c0 + c8, mv[h]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int lr = rr + 32 * h;
      const int row = r0 + lr, col = c0 + c8;
      float xv[8];
      if (ok[h]) {
        const size_t idx = static_cast<size_t>(row) * T.cols + col;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          mv[h][q] = beta * mv[h][q] + g[h][q];
          sq += mv[h][q] * mv[h][q];
          xv[q] = mv[h][q];
        }
        store_f8_stream(T.m + idx, mv[h]);
        if (!T.transposed)
          *reinterpret_cast<uint4*>(T.x0 + static_cast<size_t>(row) * T.ldx + col) = pack_bf16x8(xv);
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) xv[q] = 0.f;
      }
      if (T.transposed)
#pragma unroll
        for (int q = 0; q < 8; ++q) tile[lr][c8 + q] = __float2bfloat16_rn(xv[q]);
    }
    if (T.transposed) {
      __syncthreads();
      // output row = original column lc, 8 consecutive original rows per store
      const int lc = threadIdx.x >> 2, r8 = (threadIdx.x & 3) * 8;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int lr = r8 + 32 * h;
        const int col = c0 + lc, row = r0 + lr;
        if (col < T.cols && row < T.rows) {
          if (row + 8 <= T.rows && ((T.ldx & 7) == 0)) {
            float xv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) xv[q] = __bfloat162float(tile[lr + q][lc]);
            *reinterpret_cast<uint4*>(T.x0 + static_cast<size_t>(col) * T.ldx + row) = pack_bf16x8(xv);
          } else {
            for (int q = 0; q < 8 && row + q < T.rows; ++q)
              T.x0[static_cast<size_t>(col) * T.ldx + row + q] = tile[lr + q][lc];
          }
        }
      }
    }
    const double tile_sum = block_sum(static_cast<double>(sq), red);
    if (threadIdx.x == 0) T.partial[local] = tile_sum;
    return;
  }
#pragma unroll
  for (int i = 0; i < kTile / 8; ++i) {
    const int lr = ty + 8 * i;
    const int row = r0 + lr;
#pragma unroll
    for (int j = 0; j < kTile / 32; ++j) {
      const int lc = tx + 32 * j;
      const int col = c0 + lc;
      __nv_bfloat16 xv = __float2bfloat16_rn(0.f);
      if (row < T.rows && col < T.cols) {
        const size_t idx = static_cast<size_t>(row) * T.cols + col;
        const float mv = beta * T.m[idx] + load_grad<G>(T.g, idx);
        T.m[idx] = mv;
        sq += mv * mv;
        xv = __float2bfloat16_rn(mv);
        if (!T.transposed) T.x0[static_cast<size_t>(row) * T.ldx + col] = xv;
      }
      if (T.transposed) tile[lr][lc] = xv;
    }
  }
  if (T.transposed) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kTile / 8; ++i) {
      const int lc = ty + 8 * i;  // original column -> NS row
      const int col = c0 + lc;
#pragma unroll
      for (int j = 0; j < kTile / 32; ++j) {
        const int lr = tx + 32 * j;  // original row -> NS column (contiguous)
        const int row = r0 + lr;
        if (row < T.rows && col < T.cols)
          T.x0[static_cast<size_t>(col) * T.ldx + row] = tile[lr][lc];
      }
    }
  }
  const double tile_sum = block_sum(static_cast<double>(sq), red);
  if (threadIdx.x == 0) T.partial[local] = tile_sum;
}

__global__ void __launch_bounds__(256) apply_update_kernel(const ApplyTask* tasks, int n_tasks,
                                                          float lrate, int use_alt) {
  // X values are bf16, so a bf16 staging tile is exact and keeps the CTA at
  // 8.5 KB of shared memory: small enough to co-reside with a persistent
  // Newton-Schulz GEMM CTA when the update of one wave overlaps the next
  __shared__ __nv_bfloat16 tile[kTile][kTile + 2];
  __shared__ double red[8];
  const long long t = blockIdx.x;
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tasks[mid].tile_start <= t) lo = mid;
    else hi = mid - 1;
  }
  ApplyTask T = tasks[lo];
  if (use_alt) T.x = T.x_alt;
  const long long local = t - T.tile_start;
  const int r0 = static_cast<int>(local / T.tiles_c) * kTile;
  const int c0 = static_cast<int>(local % T.tiles_c) * kTile;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  if (T.vec) {
    if (T.transposed) {
      // X block [cols][rows]: 8 consecutive original rows per 16-byte load
      const int lc = threadIdx.x >> 2, r8 = (threadIdx.x & 3) * 8;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int lr = r8 + 32 * h;
        const int col = c0 + lc, row = r0 + lr;
        float xv[8];
        if (col < T.cols && row + 8 <= T.rows && (T.ldx & 7) == 0) {
          unpack_bf16x8(*reinterpret_cast<const uint4*>(T.x + static_cast<size_t>(col) * T.ldx + row), xv);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            xv[q] = (col < T.cols && row + q < T.rows)
                        ? __bfloat162float(T.x[static_cast<size_t>(col) * T.ldx + row + q])
                        : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) tile[lr + q][lc] = __float2bfloat16_rn(xv[q]);
      }
      __syncthreads();
    }
    float sq8 = 0.f;
    const int c8 = (threadIdx.x & 7) * 8, rr = threadIdx.x >> 3;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int lr = rr + 32 * h;
      const int row = r0 + lr, col = c0 + c8;
      if (row >= T.rows || col >= T.cols) continue;
      float xv[8], wv[8];
      if (T.transposed) {
#pragma unroll
        for (int q = 0; q < 8; ++q) xv[q] = __bfloat162float(tile[lr][c8 + q]);
      } else {
        unpack_bf16x8(*reinterpret_cast<const uint4*>(T.x + static_cast<size_t>(row) * T.ldx + col), xv);
      }
      const size_t idx = static_cast<size_t>(row) * T.cols + col;
      load_f8(T.w + idx, wv);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float upd = lrate * xv[q];
        wv[q] -= upd;
        sq8 += upd * upd;
      }
      store_f8(T.w + idx, wv);
      if (T.replica != nullptr) {
        if (T.rep_mc) mc_store16(T.replica + idx, pack_bf16x8(wv));
        else *reinterpret_cast<uint4*>(T.replica + idx) = pack_bf16x8(wv);
      }
    }
    const double tile_sum = block_sum(static_cast<double>(sq8), red);
    if (threadIdx.x == 0) {
      T.partial[local] = tile_sum;
      // the CTA's multicast stores (ordered before this by the barrier in
      // block_sum) are performed system-wide before the kernel can complete
      if (T.rep_mc) __threadfence_system();
    }
    return;
  }
  if (T.transposed) {
    // X is [cols][ldx]: read the 64x64 block along X's rows (= W's columns)
#pragma unroll
    for (int i = 0; i < kTile / 8; ++i) {
      const int lc = ty + 8 * i;
      const int col = c0 + lc;
#pragma unroll
      for (int j = 0; j < kTile / 32; ++j) {
        const int lr = tx + 32 * j;
        const int row = r0 + lr;
        tile[lr][lc] = (row < T.rows && col < T.cols) ? T.x[static_cast<size_t>(col) * T.ldx + row]
                                                      : __float2bfloat16_rn(0.f);
      }
    }
    __syncthreads();
  }
  float sq = 0.f;
#pragma unroll
  for (int i = 0; i < kTile / 8; ++i) {
    const int lr = ty + 8 * i;
    const int row = r0 + lr;
#pragma unroll
    for (int j = 0; j < kTile / 32; ++j) {
      const int lc = tx + 32 * j;
      const int col = c0 + lc;
      if (row < T.rows && col < T.cols) {
        const float x = __bfloat162float(T.transposed ? tile[lr][lc]
                                                      : T.x[static_cast<size_t>(row) * T.ldx + col]);
        const float upd = lrate * x;
        const size_t idx = static_cast<size_t>(row) * T.cols + col;
        const float w = T.w[idx] - upd;
        T.w[idx] = w;
        if (T.replica != nullptr) T.replica[idx] = __float2bfloat16_rn(w);
        sq += upd * upd;
      }
    }
  }
  const double tile_sum = block_sum(static_cast<double>(sq), red);
  if (threadIdx.x == 0) T.partial[local] = tile_sum;
}

__global__ void __launch_bounds__(256) mc_copy_kernel(const McCopyTask* tasks, int n_tasks,
                                                      long long total_vecs) {
  for (long long v = blockIdx.x * 256ll + threadIdx.x; v < total_vecs; v += 256ll * gridDim.x) {
    int lo = 0, hi = n_tasks - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tasks[mid].vec_start <= v) lo = mid;
      else hi = mid - 1;
    }
    const McCopyTask& T = tasks[lo];
    const long long i = 8 * (v - T.vec_start);
    mc_store16(T.dst + i, *reinterpret_cast<const uint4*>(T.src + i));
  }
  __threadfence_system();  // the multicast stores land before the step's end barrier
}

template <typename G>
__global__ void __launch_bounds__(256) mc_reduce_kernel(const McReduceTask* tasks, int n_tasks,
                                                        long long total_vecs) {
  for (long long v = blockIdx.x * 256ll + threadIdx.x; v < total_vecs; v += 256ll * gridDim.x) {
    int lo = 0, hi = n_tasks - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tasks[mid].vec_start <= v) lo = mid;
      else hi = mid - 1;
    }
    const McReduceTask& T = tasks[lo];
    const size_t i = 8 * static_cast<size_t>(v - T.vec_start);
    float x[8];
    mc_load_grad8<G>(T.mc, i, x);
    G* d = static_cast<G*>(T.dst) + i;
    if constexpr (sizeof(G) == 2) {
      // (the switch returned bf16 already: the conversion back is exact)
      uint4 u;
      u.x = (__float_as_uint(x[0]) >> 16) | (__float_as_uint(x[1]) & 0xFFFF0000u);
      u.y = (__float_as_uint(x[2]) >> 16) | (__float_as_uint(x[3]) & 0xFFFF0000u);
      u.z = (__float_as_uint(x[4]) >> 16) | (__float_as_uint(x[5]) & 0xFFFF0000u);
      u.w = (__float_as_uint(x[6]) >> 16) | (__float_as_uint(x[7]) & 0xFFFF0000u);
      *reinterpret_cast<uint4*>(d) = u;
    } else {
      reinterpret_cast<float4*>(d)[0] = make_float4(x[0], x[1], x[2], x[3]);
      reinterpret_cast<float4*>(d)[1] = make_float4(x[4], x[5], x[6], x[7]);
    }
  }
}

__global__ void __launch_bounds__(256) sym_fill_lower_kernel(const SymFillTask* tasks, int n_tasks) {
  __shared__ float t[32][33];
  const long long b = blockIdx.x;
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tasks[mid].tile_start <= b) lo = mid;
    else hi = mid - 1;
  }
  const SymFillTask T = tasks[lo];
  // lower-triangle tile (I, J), I >= J, from its index u = I (I + 1) / 2 + J
  const int u = static_cast<int>(b - T.tile_start);
  int I = static_cast<int>((sqrtf(8.f * u + 1.f) - 1.f) * 0.5f);
  while (I * (I + 1) / 2 > u) --I;
  while ((I + 1) * (I + 2) / 2 <= u) ++I;
  const int J = u - I * (I + 1) / 2;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  // read the mirror tile (J, I) of the upper triangle, coalesced along its rows
  for (int r = ty; r < 32; r += 8) {
    const int gr = J * 32 + r, gc = I * 32 + tx;
    t[r][tx] = (gr < T.n && gc < T.n) ? T.s[static_cast<long long>(gr) * T.ld + gc] : 0.f;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int gr = I * 32 + r, gc = J * 32 + tx;
    if (gr < T.n && gc < T.n && gr > gc) T.s[static_cast<long long>(gr) * T.ld + gc] = t[tx][r];
  }
}

__global__ void __launch_bounds__(256) partial_sums_kernel(const double* partial,
                                                           const long long* begin,
                                                           const int* count, const int* target,
                                                           double* out) {
  __shared__ double red[8];
  const int i = blockIdx.x;
  const double* p = partial + begin[i];
  double acc = 0.0;
  for (int t = threadIdx.x; t < count[i]; t += 256) acc += p[t];
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) out[target[i]] = s;
}

__global__ void __launch_bounds__(256) copy_blocks_kernel(const CopyTask* tasks, int n_tasks) {
  const long long t = blockIdx.x;
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tasks[mid].tile_start <= t) lo = mid;
    else hi = mid - 1;
  }
  const CopyTask T = tasks[lo];
  const long long local = t - T.tile_start;
  const int r0 = static_cast<int>(local / T.tiles_c) * kTile;
  const int c0 = static_cast<int>(local % T.tiles_c) * kTile;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < kTile / 8; ++i) {
    const int row = r0 + ty + 8 * i;
    if (row >= T.rows) continue;
#pragma unroll
    for (int j = 0; j < kTile / 32; ++j) {
      const int col = c0 + tx + 32 * j;
      if (col < T.cols) T.dst[row * T.ldd + col] = T.src[row * T.lds + col];
    }
  }
}

template <typename G>
__global__ void __launch_bounds__(256) momentum_vector_kernel(const MomentumVectorTask* tasks,
                                                              float beta, float lr) {
  __shared__ double red[8];
  const MomentumVectorTask T = tasks[blockIdx.y];
  float sq = 0.f;
  if (T.g_mc || T.rep_mc) {
    // NVLS-fused: n % 8 == 0 and 16-byte alignment are guaranteed by the runtime
    for (long long i = (blockIdx.x * 256ll + threadIdx.x) * 8; i < T.n; i += 256ll * gridDim.x * 8) {
      float g[8], mv[8], wv[8];
      if (T.g_mc) mc_load_grad8<G>(T.g, static_cast<size_t>(i), g);
      else load_grad8<G>(T.g, static_cast<size_t>(i), g);
      load_f8(T.m + i, mv);
      load_f8(T.w + i, wv);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        mv[q] = beta * mv[q] + g[q];
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
    block_add_double(sq, T.sq_norm, red);
    if (T.rep_mc && threadIdx.x == 0) __threadfence_system();
    return;
  }
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < T.n; i += 256ll * gridDim.x) {
    const float mv = beta * T.m[i] + load_grad<G>(T.g, static_cast<size_t>(i));
    T.m[i] = mv;
    const float upd = lr * mv;
    const float w = T.w[i] - upd;
    T.w[i] = w;
    if (T.replica != nullptr) T.replica[i] = __float2bfloat16_rn(w);
    sq += upd * upd;
  }
  block_add_double(sq, T.sq_norm, red);
}

__global__ void __launch_bounds__(256) ns_scales_kernel(const double* partial,
                                                        const long long* begin, const int* count,
                                                        float* su, float* sg) {
  __shared__ double red[8];
  const int i = blockIdx.x;
  const double* p = partial + begin[i];
  double acc = 0.0;
  for (int t = threadIdx.x; t < count[i]; t += 256) acc += p[t];
  const double ss = block_sum(acc, red);
  if (threadIdx.x == 0) {
    const double s = ss > 0.0 ? 1.0 / sqrt(ss) : 0.0;
    su[i] = static_cast<float>(s);
    sg[i] = static_cast<float>(s * s);
  }
}

}  // namespace

cudaError_t launch_momentum_matrix(const MomentumMatrixTask* d_tasks, int n_tasks,
                                   long long total_tiles, int grad_dtype, float beta,
                                   cudaStream_t s) {
  if (n_tasks == 0 || total_tiles == 0) return cudaSuccess;
  if (total_tiles > 0x7fffffffll) return cudaErrorInvalidValue;
  const dim3 grid(static_cast<unsigned>(total_tiles));
  if (grad_dtype == kGradBF16)
    momentum_matrix_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(d_tasks, n_tasks, beta);
  else
    momentum_matrix_kernel<float><<<grid, 256, 0, s>>>(d_tasks, n_tasks, beta);
  return cudaGetLastError();
}

cudaError_t launch_apply_update(const ApplyTask* d_tasks, int n_tasks, long long total_tiles,
                                float lr, int use_alt, cudaStream_t s) {
  if (n_tasks == 0 || total_tiles == 0) return cudaSuccess;
  if (total_tiles > 0x7fffffffll) return cudaErrorInvalidValue;
  apply_update_kernel<<<static_cast<unsigned>(total_tiles), 256, 0, s>>>(d_tasks, n_tasks, lr,
                                                                          use_alt);
  return cudaGetLastError();
}

cudaError_t launch_mc_copy(const McCopyTask* d_tasks, int n_tasks, long long total_vecs,
                           cudaStream_t s) {
  if (n_tasks == 0 || total_vecs == 0) return cudaSuccess;
  const long long blocks = std::min<long long>((total_vecs + 255) / 256, 148ll * 8);
  mc_copy_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(d_tasks, n_tasks, total_vecs);
  return cudaGetLastError();
}

cudaError_t launch_mc_reduce(const McReduceTask* d_tasks, int n_tasks, long long total_vecs,
                             int grad_bf16, cudaStream_t s) {
  if (n_tasks == 0 || total_vecs == 0) return cudaSuccess;
  // 2 CTAs per SM keep enough multicast loads in flight for the NVLink rate
  // while leaving the SMs to the DP waves' kernels running beside it
  const long long blocks = std::min<long long>((total_vecs + 255) / 256, 148ll * 2);
  if (grad_bf16)
    mc_reduce_kernel<__nv_bfloat16><<<static_cast<unsigned>(blocks), 256, 0, s>>>(d_tasks, n_tasks,
                                                                                  total_vecs);
  else
    mc_reduce_kernel<float><<<static_cast<unsigned>(blocks), 256, 0, s>>>(d_tasks, n_tasks,
                                                                          total_vecs);
  return cudaGetLastError();
}

cudaError_t launch_sym_fill_lower(const SymFillTask* d_tasks, int n_tasks, long long total_tiles,
                                  cudaStream_t s) {
  if (n_tasks == 0 || total_tiles == 0) return cudaSuccess;
  if (total_tiles > 0x7fffffffll) return cudaErrorInvalidValue;
  sym_fill_lower_kernel<<<static_cast<unsigned>(total_tiles), 256, 0, s>>>(d_tasks, n_tasks);
  return cudaGetLastError();
}

cudaError_t launch_partial_sums(const double* partial, const long long* begin, const int* count,
                                const int* target, double* out, int n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  partial_sums_kernel<<<n, 256, 0, s>>>(partial, begin, count, target, out);
  return cudaGetLastError();
}

cudaError_t launch_copy_blocks(const CopyTask* d_tasks, int n_tasks, long long total_tiles,
                               cudaStream_t s) {
  if (n_tasks == 0 || total_tiles == 0) return cudaSuccess;
  if (total_tiles > 0x7fffffffll) return cudaErrorInvalidValue;
  copy_blocks_kernel<<<static_cast<unsigned>(total_tiles), 256, 0, s>>>(d_tasks, n_tasks);
  return cudaGetLastError();
}

cudaError_t launch_momentum_vector(const MomentumVectorTask* d_tasks, int n_tasks, int grad_dtype,
                                   float beta, float lr, cudaStream_t s) {
  if (n_tasks == 0) return cudaSuccess;
  const dim3 grid(1, static_cast<unsigned>(n_tasks));  // one CTA per vector: deterministic norm
  if (grad_dtype == kGradBF16)
    momentum_vector_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(d_tasks, beta, lr);
  else
    momentum_vector_kernel<float><<<grid, 256, 0, s>>>(d_tasks, beta, lr);
  return cudaGetLastError();
}

cudaError_t launch_ns_scales(const double* partial, const long long* begin, const int* count,
                             float* su, float* sg, int n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  ns_scales_kernel<<<n, 256, 0, s>>>(partial, begin, count, su, sg);
  return cudaGetLastError();
}

}  // namespace osh
