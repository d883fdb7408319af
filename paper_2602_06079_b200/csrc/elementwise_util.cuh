// Device helpers shared by the elementwise kernels (muon_kernels.cu,
// shampoo_kernels.cu): gradient loads (bf16 / fp32 / NVLS multicast sums),
// 128-bit packing, multicast stores and fixed-order block reductions.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace osh {
namespace ew {

template <typename G>
__device__ __forceinline__ float load_grad(const void* g, size_t i);
template <>
__device__ __forceinline__ float load_grad<float>(const void* g, size_t i) {
  return __ldg(static_cast<const float*>(g) + i);
}
template <>
__device__ __forceinline__ float load_grad<__nv_bfloat16>(const void* g, size_t i) {
  return __bfloat162float(static_cast<const __nv_bfloat16*>(g)[i]);
}

// 8 consecutive gradient values (bf16: one 16-byte load; fp32: two).
template <typename G>
__device__ __forceinline__ void load_grad8(const void* g, size_t i, float (&v)[8]);
template <>
__device__ __forceinline__ void load_grad8<float>(const void* g, size_t i, float (&v)[8]) {
  const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(g) + i);
  const float4 a = __ldg(p), b = __ldg(p + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <>
__device__ __forceinline__ void load_grad8<__nv_bfloat16>(const void* g, size_t i, float (&v)[8]) {
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(g) + i));
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v[2 * q] = __uint_as_float(w[q] << 16);
    v[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
  }
}

// NVLS: sum over every GPU of the 8 gradient values at a multicast address
// (the NVSwitch reduces; bf16 accumulates in fp32).
template <typename G>
__device__ __forceinline__ void mc_load_grad8(const void* g, size_t i, float (&v)[8]);
template <>
__device__ __forceinline__ void mc_load_grad8<float>(const void* g, size_t i, float (&v)[8]) {
  const float* p = static_cast<const float*>(g) + i;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "l"(p));
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]) : "l"(p + 4));
}
template <>
__device__ __forceinline__ void mc_load_grad8<__nv_bfloat16>(const void* g, size_t i, float (&v)[8]) {
  const __nv_bfloat16* p = static_cast<const __nv_bfloat16*>(g) + i;
  uint32_t w[4];
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "l"(p));
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v[2 * q] = __uint_as_float(w[q] << 16);
    v[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
  }
}

// 16 bytes to the same offset of every GPU's buffer behind a multicast address.
__device__ __forceinline__ void mc_store16(void* p, uint4 u) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p),
               "f"(__uint_as_float(u.x)), "f"(__uint_as_float(u.y)), "f"(__uint_as_float(u.z)),
               "f"(__uint_as_float(u.w))
               : "memory");
}

__device__ __forceinline__ void load_f8(const float* p, float (&v)[8]) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

__device__ __forceinline__ void store_f8(float* p, const float (&v)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

__device__ __forceinline__ uint4 pack_bf16x8(const float (&v)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * q], v[2 * q + 1]);
    w[q] = *reinterpret_cast<uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ void unpack_bf16x8(uint4 u, float (&v)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v[2 * q] = __uint_as_float(w[q] << 16);
    v[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
  }
}

// Block sum in a fixed order (xor-shuffle tree, then warps in index order).
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w];
  return s;  // valid in thread 0
}

__device__ __forceinline__ void block_add_double(float v, double* dst, double* red) {
  const double s = block_sum(static_cast<double>(v), red);
  if (threadIdx.x == 0 && s != 0.0 && dst != nullptr) atomicAdd(dst, s);
}


}  // namespace ew
}  // namespace osh
