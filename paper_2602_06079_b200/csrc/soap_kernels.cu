// Blocked-SOAP kernels (see soap_kernels.cuh).
#include "soap_kernels.cuh"
#include "status.hpp"

#include "elementwise_util.cuh"

namespace osh {
namespace {

using namespace ew;

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

__device__ __forceinline__ int find_rot(const SoapRotTask* tasks, int n, long long t) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tasks[mid].chunk_start <= t) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// ---------------------------------------------------------------- prep
__device__ __forceinline__ void split8(const float (&v)[8], uint4& hi, uint4& lo) {
  float h[8], l[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    h[q] = __bfloat162float(__float2bfloat16_rn(v[q]));
    l[q] = v[q] - h[q];
  }
  hi = pack_bf16x8(h);
  lo = pack_bf16x8(l);
}

// One 64 x 64 tile of the padded block [ldp][ldq]: thread = 8 consecutive
// columns of one row (two row halves). Pads (r >= p or c >= q) are written 0.
template <typename G>
__global__ void __launch_bounds__(256) soap_prep_kernel(const SoapPrepTask* tasks, int n,
                                                        float beta1) {
  __shared__ float th[kTile][kTile + 1];  // hi / lo of g for the transposed split
  __shared__ float tl[kTile][kTile + 1];
  const long long t = blockIdx.x;
  const SoapPrepTask T = tasks[find_task(tasks, n, t)];
  const long long local = t - T.tile_start;
  const int lr0 = static_cast<int>(local / T.tiles_c) * kTile;  // block-local
  const int lc0 = static_cast<int>(local % T.tiles_c) * kTile;
  const float b1c = 1.f - beta1;
  const int c8 = (threadIdx.x & 7) * 8, rr = threadIdx.x >> 3;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int lr = rr + 32 * h;
    const int r = lr0 + lr, c = lc0 + c8;
    float v[8], mv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = mv[q] = 0.f;
    if (r < T.p && c < T.q) {
      const size_t idx = static_cast<size_t>(T.r0 + r) * T.g_ld + T.c0 + c;
      if (T.vec) {  // c + 8 <= q (q % 8 == 0)
        if (T.g_mc) mc_load_grad8<G>(T.g, idx, v);
        else load_grad8<G>(T.g, idx, v);
        load_f8(T.m + idx, mv);
#pragma unroll
        for (int q = 0; q < 8; ++q) mv[q] = beta1 * mv[q] + b1c * v[q];
        store_f8(T.m + idx, mv);
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (c + q < T.q) {
            v[q] = load_grad<G>(T.g, idx + q);
            mv[q] = beta1 * T.m[idx + q] + b1c * v[q];
            T.m[idx + q] = mv[q];
          }
      }
    }
    uint4 ghi, glo, mhi, mlo;
    split8(v, ghi, glo);
    split8(mv, mhi, mlo);
    const uint4 seg_g[4] = {ghi, glo, ghi, ghi};
    const uint4 seg_m[4] = {mhi, mlo, mhi, mhi};
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (r < T.p && (!T.exact || s == 0))  // (the column split has p rows; the row splits ldp)
        *reinterpret_cast<uint4*>(T.gs + static_cast<size_t>(r) * 4 * T.ldq + s * T.ldq + c) = seg_g[s];
      if (!T.exact || s >= 2)
        *reinterpret_cast<uint4*>(T.grs + (static_cast<size_t>(s) * T.ldp + r) * T.ldq + c) = seg_g[s];
      *reinterpret_cast<uint4*>(T.mrs + (static_cast<size_t>(s) * T.ldp + r) * T.ldq + c) = seg_m[s];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float hv = __bfloat162float(__float2bfloat16_rn(v[q]));
      th[lr][c8 + q] = hv;
      tl[lr][c8 + q] = v[q] - hv;
    }
  }
  __syncthreads();
  // G^T column-split: row = block column c (< q only), column = block row r
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = 0; i < kTile / 8; ++i) {
    const int lc = ty + 8 * i, c = lc0 + lc;
    if (c >= T.q) continue;
    __nv_bfloat16* row = T.gts + static_cast<size_t>(c) * 4 * T.ldp;
    for (int j = 0; j < kTile / 32; ++j) {
      const int lr = tx + 32 * j, r = lr0 + lr;
      const __nv_bfloat16 hi = __float2bfloat16_rn(th[lr][lc]);
      const __nv_bfloat16 lo = __float2bfloat16_rn(tl[lr][lc]);
      row[r] = hi;
      if (T.exact) continue;
      row[T.ldp + r] = lo;
      row[2 * T.ldp + r] = hi;
      row[3 * T.ldp + r] = hi;
    }
  }
}

// ---------------------------------------------------------------- rotated Adam
__global__ void __launch_bounds__(256) soap_rot_kernel(const SoapRotTask* tasks, int n,
                                                       float beta2, float ib1, float ib2,
                                                       float eps) {
  const long long t = blockIdx.x;
  const SoapRotTask T = tasks[find_rot(tasks, n, t)];
  const long long base = (t - T.chunk_start) * kSoapRotChunk;
  const float b2c = 1.f - beta2;
  for (long long i = base + threadIdx.x * 8; i < base + kSoapRotChunk && i < T.elems;
       i += 256 * 8) {
    float gp[8], mp[8], v[8], o[8];
    load_f8(T.gp + i, gp);
    load_f8(T.mp + i, mp);
    load_f8(T.v + i, v);
    const int col0 = static_cast<int>(i % T.ldq);  // ldq is a multiple of 8
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (col0 + q < T.q) {
        v[q] = beta2 * v[q] + b2c * gp[q] * gp[q];
        o[q] = (mp[q] * ib1) / (sqrtf(v[q] * ib2) + eps);
      } else {
        v[q] = 0.f;
        o[q] = 0.f;
      }
    }
    store_f8(T.v + i, v);
    *reinterpret_cast<uint4*>(T.nrot + i) = pack_bf16x8(o);
  }
}

// ---------------------------------------------------------------- apply
__global__ void __launch_bounds__(256) soap_apply_kernel(const ShApplyTask* tasks, int n,
                                                         float lrate) {
  __shared__ double red[8];
  const long long t = blockIdx.x;
  const ShApplyTask T = tasks[find_task(tasks, n, t)];
  const long long local = t - T.tile_start;
  const int r0 = static_cast<int>(local / T.tiles_c) * kTile;
  const int c0 = static_cast<int>(local % T.tiles_c) * kTile;
  const int bi = r0 / T.block, bj = c0 / T.block;  // block edges are multiples of 64
  const ShBlockRef B = T.blocks[bi * T.blocks_c + bj];
  const int br = r0 - bi * T.block, bc = c0 - bj * T.block;
  float sq = 0.f;
  if (T.vec) {
    const int c8 = (threadIdx.x & 7) * 8, rr = threadIdx.x >> 3;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int lr = rr + 32 * h;
      const int row = r0 + lr, col = c0 + c8;
      if (row >= T.rows || col >= T.cols) continue;
      float u[8], wv[8];
      unpack_bf16x8(*reinterpret_cast<const uint4*>(B.u + static_cast<size_t>(br + lr) * B.ldu + bc + c8), u);
      const size_t idx = static_cast<size_t>(row) * T.cols + col;
      load_f8(T.w + idx, wv);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float upd = lrate * u[q];
        wv[q] -= upd;
        sq += upd * upd;
      }
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
        const float upd = lrate * u;
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

// ---------------------------------------------------------------- elementwise Adam
template <typename G>
__global__ void __launch_bounds__(256) soap_adam_kernel(const SoapAdamTask* tasks, int n,
                                                        float beta1, float beta2, float ib1,
                                                        float ib2, float eps, float lr) {
  __shared__ double red[8];
  const long long t = blockIdx.x;
  const SoapAdamTask T = tasks[find_task(tasks, n, t)];
  const long long base = (t - T.tile_start) * kShSgdTile;
  const float b1c = 1.f - beta1, b2c = 1.f - beta2;
  float sq = 0.f;
  if (T.vec) {
    for (long long i = base + threadIdx.x * 8; i < base + kShSgdTile && i < T.n; i += 256 * 8) {
      float g[8], mv[8], vv[8], wv[8];
      if (T.g_mc) mc_load_grad8<G>(T.g, static_cast<size_t>(i), g);
      else load_grad8<G>(T.g, static_cast<size_t>(i), g);
      load_f8(T.m + i, mv);
      load_f8(T.v + i, vv);
      load_f8(T.w + i, wv);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        mv[q] = beta1 * mv[q] + b1c * g[q];
        vv[q] = beta2 * vv[q] + b2c * g[q] * g[q];
        const float upd = lr * (mv[q] * ib1) / (sqrtf(vv[q] * ib2) + eps);
        wv[q] -= upd;
        sq += upd * upd;
      }
      store_f8(T.m + i, mv);
      store_f8(T.v + i, vv);
      store_f8(T.w + i, wv);
      if (T.replica != nullptr) {
        if (T.rep_mc) mc_store16(T.replica + i, pack_bf16x8(wv));
        else *reinterpret_cast<uint4*>(T.replica + i) = pack_bf16x8(wv);
      }
    }
  } else {
    for (long long i = base + threadIdx.x; i < base + kShSgdTile && i < T.n; i += 256) {
      const float g = load_grad<G>(T.g, static_cast<size_t>(i));
      const float mv = beta1 * T.m[i] + b1c * g;
      const float vv = beta2 * T.v[i] + b2c * g * g;
      T.m[i] = mv;
      T.v[i] = vv;
      const float upd = lr * (mv * ib1) / (sqrtf(vv * ib2) + eps);
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

// ---------------------------------------------------------------- basis refresh
constexpr int kBasisThreads = 512;

__global__ void __launch_bounds__(kBasisThreads) soap_basis_kernel(const SoapBasisTask* tasks,
                                                                   float shift) {
  extern __shared__ float sm[];
  __shared__ double red[kBasisThreads / 32];
  __shared__ float s_c;
  const SoapBasisTask T = tasks[blockIdx.x];
  const int n = T.n;
  float* est = sm;
  float* nrm = sm + n;
  int* order = reinterpret_cast<int*>(sm + 2 * n);
  // (a) c = shift * ||S||_F (fixed-order fp64 block reduction)
  double ss = 0.0;
  const int warp0 = threadIdx.x >> 5, lane0 = threadIdx.x & 31;
  for (int r = warp0; r < n; r += kBasisThreads / 32) {  // warp per row, coalesced
    const float* row = T.s + static_cast<long long>(r) * T.lds;
    float acc = 0.f;
    for (int c = lane0; c < n; c += 32) acc += row[c] * row[c];
    ss += acc;
  }
  const double tot = block_sum(ss, red);
  if (threadIdx.x == 0) s_c = static_cast<float>(static_cast<double>(shift) * sqrt(tot));
  __syncthreads();
  const float c = s_c;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (c == 0.f) {  // no statistics yet: the basis is kept
    for (int j = threadIdx.x; j < n; j += kBasisThreads) T.order[j] = j;
    return;
  }
  // (b) y_j += c q_j ; est_j = q_j . y_j ; nrm_j = |y_j|^2  (warp per column)
  for (int j = warp; j < n; j += kBasisThreads / 32) {
    const float* qj = T.q + static_cast<size_t>(j) * T.ldq;
    float* yj = T.y + static_cast<size_t>(j) * T.ldq;
    float e = 0.f, r = 0.f;
    for (int i = lane; i < n; i += 32) {
      const float qv = qj[i];
      const float yv = yj[i] + c * qv;
      yj[i] = yv;
      e += qv * yv;
      r += yv * yv;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      e += __shfl_xor_sync(0xffffffffu, e, o);
      r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    if (lane == 0) {
      est[j] = e;
      nrm[j] = r;
    }
  }
  __syncthreads();
  // (c) stable descending order of est
  for (int j = threadIdx.x; j < n; j += kBasisThreads) {
    const float ej = est[j];
    int rank = 0;
    for (int k = 0; k < n; ++k) {
      const float ek = est[k];
      rank += (ek > ej || (ek == ej && k < j)) ? 1 : 0;
    }
    order[rank] = j;
  }
  __syncthreads();
  // (d) Q[:, k] = y_order[k] / |y_order[k]|  (Q is not read after (b))
  for (int k = warp; k < n; k += kBasisThreads / 32) {
    const int j = order[k];
    const float inv = nrm[j] > 0.f ? rsqrtf(nrm[j]) : 0.f;
    const float* yj = T.y + static_cast<size_t>(j) * T.ldq;
    float* qk = T.q + static_cast<size_t>(k) * T.ldq;
    for (int i = lane; i < n; i += 32) qk[i] = yj[i] * inv;
    if (lane == 0) T.order[k] = j;
  }
}

__global__ void __launch_bounds__(256) soap_vperm_kernel(const SoapVpermTask* tasks, int n) {
  const long long t = blockIdx.x;
  const SoapVpermTask T = tasks[find_task(tasks, n, t)];
  const long long local = t - T.tile_start;
  const int r0 = static_cast<int>(local / T.tiles_c) * kTile;
  const int c0 = static_cast<int>(local % T.tiles_c) * kTile;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = 0; i < kTile / 8; ++i) {
    const int r = r0 + ty + 8 * i;
    if (r >= T.p) continue;
    const float* src = T.v + static_cast<size_t>(T.ol[r]) * T.ldq;
    for (int j = 0; j < kTile / 32; ++j) {
      const int c = c0 + tx + 32 * j;
      if (c < T.q) T.dst[static_cast<size_t>(r) * T.ldq + c] = src[T.orr[c]];
    }
  }
}

__global__ void __launch_bounds__(256) soap_qcast_kernel(const SoapQcastTask* tasks, int n) {
  __shared__ float tile[kTile][kTile + 1];
  const long long t = blockIdx.x;
  const SoapQcastTask T = tasks[find_task(tasks, n, t)];
  const long long local = t - T.tile_start;
  const int r0 = static_cast<int>(local / T.tiles_c) * kTile;  // Q rows (i)
  const int c0 = static_cast<int>(local % T.tiles_c) * kTile;  // Q columns (j)
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  // tile[jj][ii] = Q(r0 + ii, c0 + jj), read along columns (coalesced in i)
  for (int a = 0; a < kTile / 8; ++a) {
    const int jj = ty + 8 * a, j = c0 + jj;
    for (int b = 0; b < kTile / 32; ++b) {
      const int ii = tx + 32 * b, i = r0 + ii;
      tile[jj][ii] = (i < T.n && j < T.n) ? T.q[static_cast<size_t>(j) * T.ldq + i] : 0.f;
    }
  }
  __syncthreads();
  if (T.qt_split != nullptr)  // Q^T row j = Q column j: qt[j][s*ldb + i], coalesced in i
    for (int a = 0; a < kTile / 8; ++a) {
      const int jj = ty + 8 * a, j = c0 + jj;
      if (j >= T.n) continue;
      __nv_bfloat16* row = T.qt_split + static_cast<size_t>(j) * 4 * T.ldb;
      for (int b = 0; b < kTile / 32; ++b) {
        const int ii = tx + 32 * b, i = r0 + ii;
        if (i >= T.n) continue;
        const float x = tile[jj][ii];
        const __nv_bfloat16 hi = __float2bfloat16_rn(x);
        const __nv_bfloat16 lo = __float2bfloat16_rn(x - __bfloat162float(hi));
        row[i] = hi;
        row[T.ldb + i] = lo;
        row[2 * T.ldb + i] = hi;
        row[3 * T.ldb + i] = hi;
      }
    }
  if (T.q_row != nullptr || T.q_rsplit != nullptr)  // row-major: [i][j], coalesced in j
    for (int a = 0; a < kTile / 8; ++a) {
      const int ii = ty + 8 * a, i = r0 + ii;
      if (i >= T.n) continue;
      for (int b = 0; b < kTile / 32; ++b) {
        const int jj = tx + 32 * b, j = c0 + jj;
        if (j >= T.n) continue;
        const float x = tile[jj][ii];
        const __nv_bfloat16 hi = __float2bfloat16_rn(x);
        if (T.q_row != nullptr) T.q_row[static_cast<size_t>(i) * T.ldb + j] = hi;
        if (T.q_rsplit != nullptr) {
          const __nv_bfloat16 lo = __float2bfloat16_rn(x - __bfloat162float(hi));
          const size_t seg = static_cast<size_t>(T.ldb) * T.ldb;
          __nv_bfloat16* d = T.q_rsplit + static_cast<size_t>(i) * T.ldb + j;
          d[0] = hi;
          d[seg] = lo;
          d[2 * seg] = hi;
          d[3 * seg] = hi;
        }
      }
    }
}

__global__ void soap_eye_kernel(float* q, long long ldq, long long bstride, int n, int batch) {
  const long long col = blockIdx.x;  // batch * n columns
  const int b = static_cast<int>(col / n), j = static_cast<int>(col % n);
  if (b >= batch) return;
  float* c = q + b * bstride + static_cast<long long>(j) * ldq;
  for (long long i = threadIdx.x; i < ldq; i += blockDim.x) c[i] = i == j ? 1.f : 0.f;
}

// ---------------------------------------------------------------- refresh factorizations
__global__ void __launch_bounds__(256) soap_split_kernel(const SoapSplitTask* tasks, int n) {
  const long long t = blockIdx.x;
  const SoapSplitTask T = tasks[find_task(tasks, n, t)];
  const long long local = t - T.tile_start;
  const int r0 = static_cast<int>(local / T.tiles_c) * kTile;
  const int c0 = static_cast<int>(local % T.tiles_c) * kTile;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = 0; i < kTile / 8; ++i) {
    const int r = r0 + ty + 8 * i;
    for (int j = 0; j < kTile / 32; ++j) {
      const int c = c0 + tx + 32 * j;
      const float v = (r < T.rows && c < T.cols) ? T.src[static_cast<size_t>(r) * T.lds + c] : 0.f;
      const __nv_bfloat16 h = __float2bfloat16_rn(v);
      const float r1 = v - __bfloat162float(h);
      const __nv_bfloat16 m = __float2bfloat16_rn(r1);
      const __nv_bfloat16 l = __float2bfloat16_rn(r1 - __bfloat162float(m));
      const __nv_bfloat16 sa[6] = {h, m, h, l, m, h};
      const __nv_bfloat16 sb[6] = {h, h, m, h, m, l};
      if (r < T.rows) {
        if (T.col_a != nullptr) {
          __nv_bfloat16* d = T.col_a + static_cast<size_t>(r) * 6 * T.ldd + c;
#pragma unroll
          for (int q = 0; q < 6; ++q) d[q * T.ldd] = sa[q];
        }
        if (T.col_b != nullptr) {
          __nv_bfloat16* d = T.col_b + static_cast<size_t>(r) * 6 * T.ldd + c;
#pragma unroll
          for (int q = 0; q < 6; ++q) d[q * T.ldd] = sb[q];
        }
      }
      if (T.row_b != nullptr) {
        const size_t seg = static_cast<size_t>(T.ldd) * T.ldd;
        __nv_bfloat16* d = T.row_b + static_cast<size_t>(r) * T.ldd + c;
#pragma unroll
        for (int q = 0; q < 6; ++q) d[q * seg] = sb[q];
      }
    }
  }
}

constexpr int kCholThreads = 1024;
constexpr int kCholLrs = kSoapCholMaxN + 4;  // row stride of the phase-2 row block (16 B aligned)
// panel [32][n] (phase 1) / row block [32][kCholLrs] (phase 2), diagonal block [32][33]
constexpr size_t kCholSmem =
    sizeof(float) * (static_cast<size_t>(kSoapCholMaxN) * 33 > 32ull * kCholLrs
                         ? static_cast<size_t>(kSoapCholMaxN) * 33
                         : 32ull * kCholLrs) +
    sizeof(float) * 32 * 33;

__global__ void __launch_bounds__(kCholThreads, 1) soap_chol_inv_kernel(const SoapCholTask* tasks) {
  extern __shared__ float sm[];
  float* P = sm;  // phase 1: transposed panel [32][kSoapCholMaxN]; phase 2: row block [32][kCholLrs]
  float* D = sm + (kCholSmem / sizeof(float) - 32 * 33);  // diagonal block [32][33]
  const SoapCholTask T = tasks[blockIdx.x];
  const int n = T.n;
  const int np = (n + 31) / 32 * 32;
  const long long ld = T.ld;
  float* C = T.c;
  float* X = T.linv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the pad [n, np) becomes the identity; L^-1 starts at 0
  for (int i = warp; i < np; i += kCholThreads / 32)  // warp per row, coalesced
    for (int j = lane; j < np; j += 32) {
      if (i >= n || j >= n) C[i * ld + j] = i == j ? 1.f : 0.f;
      X[i * ld + j] = 0.f;
    }
  __syncthreads();
  // ---- phase 1: right-looking blocked Cholesky, C = L L^T (lower, in place)
  for (int k0 = 0; k0 < np; k0 += 32) {
    if (warp == 0) {
      for (int r = 0; r < 32; ++r) D[r * 33 + lane] = lane <= r ? C[(k0 + r) * ld + k0 + lane] : 0.f;
      __syncwarp();
      for (int j = 0; j < 32; ++j) {
        if (lane == j) D[j * 33 + j] = sqrtf(fmaxf(D[j * 33 + j], 1e-30f));
        __syncwarp();
        if (lane > j) D[lane * 33 + j] /= D[j * 33 + j];
        __syncwarp();
        if (lane > j) {
          const float lij = D[lane * 33 + j];
          for (int l = j + 1; l <= lane; ++l) D[lane * 33 + l] -= lij * D[l * 33 + j];
        }
        __syncwarp();
      }
      for (int r = 0; r < 32; ++r)
        if (lane <= r) C[(k0 + r) * ld + k0 + lane] = D[r * 33 + lane];
    }
    __syncthreads();
    const int m = np - k0 - 32;  // rows below the diagonal block
    for (int t = threadIdx.x; t < m; t += kCholThreads) {
      const long long i = k0 + 32 + t;
      float x[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = C[i * ld + k0 + j];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float v = x[j];
#pragma unroll
        for (int q = 0; q < j; ++q) v -= x[q] * D[j * 33 + q];
        x[j] = v / D[j * 33 + j];
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        P[j * kSoapCholMaxN + t] = x[j];  // transposed panel: rows contiguous per j
        C[i * ld + k0 + j] = x[j];
      }
    }
    __syncthreads();
    const int mt = m / 4;  // m is a multiple of 32
    const int ntile = mt * (mt + 1) / 2;
    for (int id = threadIdx.x; id < ntile; id += kCholThreads) {
      int ti = static_cast<int>((sqrtf(8.f * id + 1.f) - 1.f) * 0.5f);
      while ((ti + 1) * (ti + 2) / 2 <= id) ++ti;
      while (ti * (ti + 1) / 2 > id) --ti;
      const int tj = id - ti * (ti + 1) / 2;
      // the tile's current values are loaded first, so their (L2 / HBM)
      // latency overlaps the 512 FMAs below
      float4 cur[4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
        cur[a] = *reinterpret_cast<const float4*>(C + (k0 + 32 + ti * 4 + a) * ld + k0 + 32 + tj * 4);
      float acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
#pragma unroll 4
      for (int q = 0; q < 32; ++q) {  // two 128-bit shared loads per 16 FMAs
        const float4 a4 = *reinterpret_cast<const float4*>(P + q * kSoapCholMaxN + ti * 4);
        const float4 b4 = *reinterpret_cast<const float4*>(P + q * kSoapCholMaxN + tj * 4);
        const float av[4] = {a4.x, a4.y, a4.z, a4.w}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] += av[a] * bv[b];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const long long i = k0 + 32 + ti * 4 + a, j0 = k0 + 32 + tj * 4;
        const float cv[4] = {cur[a].x, cur[a].y, cur[a].z, cur[a].w};
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (i >= j0 + b) C[i * ld + j0 + b] = cv[b] - acc[a][b];
      }
    }
    __syncthreads();
  }
  // ---- phase 2: X = L^-1 by row blocks: X[k..k+32) = Ldiag^-1 (E - L[k.., 0:k) X[0:k))
  float* Lr = P;
  for (int k = 0; k < np; k += 32) {
    const int w = k + 32;
    for (int e = threadIdx.x; e < 32 * w; e += kCholThreads) {
      const int r = e / w, mm = e % w;
      Lr[r * kCholLrs + mm] = mm <= k + r ? C[(k + r) * ld + mm] : 0.f;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < w; c += kCholThreads) {
      float x[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) x[r] = 0.f;
      if (c < k) {  // k is a multiple of 32: four X loads in flight per step,
                    // the row-block coefficients as broadcast 128-bit loads
        // software pipeline: the next four X values load while this step's
        // 128 FMAs run. X is lower triangular (X[mm][c] = 0 for mm < c), so
        // the contraction starts at row c (exactly: the skipped terms are 0)
        const int m0 = c & ~3;
        float n0 = X[static_cast<long long>(m0) * ld + c], n1 = X[static_cast<long long>(m0 + 1) * ld + c];
        float n2 = X[static_cast<long long>(m0 + 2) * ld + c], n3 = X[static_cast<long long>(m0 + 3) * ld + c];
        for (int mm = m0; mm < k; mm += 4) {
          const float x0 = n0, x1 = n1, x2 = n2, x3 = n3;
          if (mm + 4 < k) {
            n0 = X[static_cast<long long>(mm + 4) * ld + c];
            n1 = X[static_cast<long long>(mm + 5) * ld + c];
            n2 = X[static_cast<long long>(mm + 6) * ld + c];
            n3 = X[static_cast<long long>(mm + 7) * ld + c];
          }
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            const float4 l = *reinterpret_cast<const float4*>(Lr + r * kCholLrs + mm);
            x[r] -= l.x * x0 + l.y * x1 + l.z * x2 + l.w * x3;
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (c - k == r) x[r] += 1.f;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        float v = x[r];
#pragma unroll
        for (int q = 0; q < r; ++q) v -= Lr[r * kCholLrs + k + q] * x[q];
        x[r] = v / Lr[r * kCholLrs + k + r];
      }
#pragma unroll
      for (int r = 0; r < 32; ++r) X[static_cast<long long>(k + r) * ld + c] = x[r];
    }
    __syncthreads();
  }
}

bool bad_grid(long long tiles) { return tiles <= 0 || tiles > 0x7fffffffll; }

}  // namespace

cudaError_t launch_soap_prep(const SoapPrepTask* d, int n, long long tiles, int grad_dtype,
                             float beta1, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(tiles)) return cudaErrorInvalidValue;
  if (grad_dtype == kGradBF16)
    soap_prep_kernel<__nv_bfloat16><<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n, beta1);
  else
    soap_prep_kernel<float><<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n, beta1);
  return cudaGetLastError();
}

cudaError_t launch_soap_rot(const SoapRotTask* d, int n, long long chunks, float beta2,
                            float inv_bc1, float inv_bc2, float eps, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(chunks)) return cudaErrorInvalidValue;
  soap_rot_kernel<<<static_cast<unsigned>(chunks), 256, 0, s>>>(d, n, beta2, inv_bc1, inv_bc2, eps);
  return cudaGetLastError();
}

cudaError_t launch_soap_apply(const ShApplyTask* d, int n, long long tiles, float lr,
                              cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(tiles)) return cudaErrorInvalidValue;
  soap_apply_kernel<<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n, lr);
  return cudaGetLastError();
}

cudaError_t launch_soap_adam(const SoapAdamTask* d, int n, long long tiles, int grad_dtype,
                             float beta1, float beta2, float inv_bc1, float inv_bc2, float eps,
                             float lr, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(tiles)) return cudaErrorInvalidValue;
  if (grad_dtype == kGradBF16)
    soap_adam_kernel<__nv_bfloat16><<<static_cast<unsigned>(tiles), 256, 0, s>>>(
        d, n, beta1, beta2, inv_bc1, inv_bc2, eps, lr);
  else
    soap_adam_kernel<float><<<static_cast<unsigned>(tiles), 256, 0, s>>>(
        d, n, beta1, beta2, inv_bc1, inv_bc2, eps, lr);
  return cudaGetLastError();
}

cudaError_t launch_soap_basis(const SoapBasisTask* d, int n, float shift, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  // dynamic shared memory: est, nrm (float) and order (int) of the largest matrix
  constexpr int max_n = 4096;
  const size_t smem = static_cast<size_t>(max_n) * 12;
  if (cudaError_t e = set_max_dynamic_smem(reinterpret_cast<const void*>(soap_basis_kernel),
                                           static_cast<int>(smem));
      e != cudaSuccess)
    return e;
  soap_basis_kernel<<<n, kBasisThreads, smem, s>>>(d, shift);
  return cudaGetLastError();
}

cudaError_t launch_soap_vperm(const SoapVpermTask* d, int n, long long tiles, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(tiles)) return cudaErrorInvalidValue;
  soap_vperm_kernel<<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n);
  return cudaGetLastError();
}

cudaError_t launch_soap_qcast(const SoapQcastTask* d, int n, long long tiles, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(tiles)) return cudaErrorInvalidValue;
  soap_qcast_kernel<<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n);
  return cudaGetLastError();
}

cudaError_t launch_soap_split(const SoapSplitTask* d, int n, long long tiles, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (bad_grid(tiles)) return cudaErrorInvalidValue;
  soap_split_kernel<<<static_cast<unsigned>(tiles), 256, 0, s>>>(d, n);
  return cudaGetLastError();
}

cudaError_t launch_soap_chol_inv(const SoapCholTask* d, int n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (cudaError_t e = set_max_dynamic_smem(reinterpret_cast<const void*>(soap_chol_inv_kernel),
                                           static_cast<int>(kCholSmem));
      e != cudaSuccess)
    return e;
  soap_chol_inv_kernel<<<n, kCholThreads, kCholSmem, s>>>(d);
  return cudaGetLastError();
}

cudaError_t launch_soap_eye(float* q, long long ldq, long long bstride, int n, int batch,
                            cudaStream_t s) {
  if (batch == 0 || n == 0) return cudaSuccess;
  soap_eye_kernel<<<static_cast<unsigned>(static_cast<long long>(batch) * n), 256, 0, s>>>(
      q, ldq, bstride, n, batch);
  return cudaGetLastError();
}

}  // namespace osh
