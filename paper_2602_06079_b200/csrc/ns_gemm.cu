// Persistent, warp-specialised tcgen05 GEMM for the Newton-Schulz iteration
// (see ns_gemm.cuh for the math). Layout of one CTA (256 threads, 1 CTA/SM):
//   warp 0  lane 0 : TMA producer     (4-stage smem ring, full/empty mbarriers)
//   warp 1  lane 0 : tcgen05.mma issuer (UMMA 128x256x16, fp32 accum in TMEM)
//   warp 2         : TMEM allocator   (512 columns = 2 accumulator buffers)
//   warps 4-7      : epilogue         (tcgen05.ld -> fused math -> global)
// The two TMEM accumulators let the epilogue of tile i overlap the MMAs of
// tile i+1. Tiles of all problems are linearised and strided over the grid.
#include "ns_gemm.cuh"
#include "sm100.cuh"
#include "status.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace osh {
namespace {

using namespace osh::sm100;

// CG = CTAs per UMMA (cta_group::1 or ::2). With CG = 2 a cluster of two CTAs
// computes a 256 x 256 tile: each CTA stages its 128 rows of A and its half
// (128 rows / columns) of B; the leader CTA issues tcgen05.mma.cta_group::2
// and each CTA's TMEM receives its 128 accumulator rows.
template <int MODE, int CG>
struct Cfg {
  static constexpr uint32_t kRowsA = 128;                 // A rows per CTA
  static constexpr uint32_t kTileM = 128 * CG;            // output rows per tile
  static constexpr uint32_t kRowsB = kNsBN / CG;          // B rows (N) per CTA
  static constexpr uint32_t kStageA = kRowsA * kNsBK * 2; // 16 KiB
  static constexpr uint32_t kStageB = kRowsB * kNsBK * 2; // 32 or 16 KiB
#ifndef OSH_CG2_STAGES
#define OSH_CG2_STAGES 5  // 5 x 32 KiB leaves ~66 KiB for co-resident update kernels
#endif
#ifndef OSH_FINAL_STAGE_DROP
#define OSH_FINAL_STAGE_DROP 0
#endif
  // FINAL also stages W boxes (48 KiB); 5 stages still fit (209 KiB) and
  // measured 5 % faster than 4 (OSH_FINAL_STAGE_DROP=1: one stage fewer)
  // (1-CTA tiles stage 48 KiB per slot: FINAL keeps 3 of them there)
  static constexpr int kStages = CG == 1 ? (MODE == kEpiFinal ? 3 : 4)
                                         : OSH_CG2_STAGES - (MODE == kEpiFinal ? OSH_FINAL_STAGE_DROP : 0);
};
constexpr uint32_t kTmemCols = 512;
// kEpiFinal staging per epilogue warp: kFinBufs 32x32 fp32 W boxes in flight
#ifndef OSH_FIN_BUFS
#define OSH_FIN_BUFS 3
#endif
constexpr int kFinBufs = OSH_FIN_BUFS;
constexpr uint32_t kFinWBox = 32 * 32 * 4;
constexpr uint32_t kFinBytes = 4 * kFinBufs * kFinWBox;
// kEpiSplit (symmetric): per epilogue warp, its 32 x 32 chunk as bf16 hi and
// lo, transposed through shared memory (80 B row pitch: conflict-free 16 B
// reads) so the mirrored half leaves as 16 B row stores, not 2 B scalars
constexpr uint32_t kSplitPitch = 40;  // bf16 elements per staged row
constexpr uint32_t kSplitWarpBytes = 2 * 32 * kSplitPitch * 2;
constexpr uint32_t kSplitBytes = 4 * kSplitWarpBytes;
template <int MODE>
constexpr uint32_t epi_stage_bytes() {
  return MODE == kEpiFinal ? kFinBytes : MODE == kEpiSplit ? kSplitBytes : 0;
}
template <int MODE, int CG>
constexpr uint32_t smem_bytes();
static_assert(1024 + 5 * (16384 + 16384) + 4 * kFinBufs * 4096 + 256 <= 232448, "FINAL (2-CTA) exceeds smem");
static_assert(1024 + 3 * (16384 + 32768) + 4 * kFinBufs * 4096 + 256 <= 232448, "FINAL (1-CTA) exceeds smem");
template <int MODE, int CG>
constexpr uint32_t smem_bytes() {
  // [1 KiB align][stage ring][FINAL staging][barriers 256 B]
  return 1024 + Cfg<MODE, CG>::kStages * (Cfg<MODE, CG>::kStageA + Cfg<MODE, CG>::kStageB) +
         epi_stage_bytes<MODE>() + 256;
}
constexpr int kRasterGroup = 8;
// Tile rows per raster group: UPDATE sweeps 16 (a 4096-row iterate's X column
// panels are then read once, not twice: -0.9 % on the N=1 step, profiles/
// r02_update_raster16_ab.json); the other modes keep 8.
#ifndef OSH_UPDATE_RASTER
#define OSH_UPDATE_RASTER 16
#endif
#ifndef OSH_FINAL_RASTER
#define OSH_FINAL_RASTER 8
#endif
inline int raster_group(int mode) {
  return mode == kEpiUpdate ? OSH_UPDATE_RASTER : mode == kEpiFinal ? OSH_FINAL_RASTER : kRasterGroup;
}

struct TileCoord {
  int p, b, tm, tn;
};

__device__ __forceinline__ TileCoord decode_tile(const NsGemmParams& P, int t) {
  TileCoord c;
  c.p = 0;
  while (c.p + 1 < P.num_problems && t >= P.prob[c.p + 1].tile_start) ++c.p;
  const NsGemmProblem& pr = P.prob[c.p];
  const int local = t - pr.tile_start;
  const int per_batch = pr.tiles_per_batch;
  c.b = local / per_batch;
  int rem = local - c.b * per_batch;
  if (pr.symmetric) {
    // column-major over the tiles that touch the upper triangle: column tn
    // holds tiles tm = 0 .. min(tiles_m, (256*tn + 255) / tile_m + 1) - 1
    int tn = 0;
    for (;;) {
      const int cnt = min(pr.tiles_m, (kNsBN * tn + kNsBN - 1) / P.tile_m + 1);
      if (rem < cnt) break;
      rem -= cnt;
      ++tn;
    }
    c.tm = rem;
    c.tn = tn;
    return c;
  }
  // grouped rasterisation: P.raster tile-rows sweep one column panel
  const int rg = P.raster;
  const int span = rg * pr.tiles_n;
  const int group = rem / span;
  const int first_m = group * rg;
  const int gsz = min(pr.tiles_m - first_m, rg);
  const int r2 = rem - group * span;
  c.tm = first_m + r2 % gsz;
  c.tn = r2 / gsz;
  return c;
}

__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Loads 32 bf16 of one row (cols [col0, col0+32), masked at n) as floats.
__device__ __forceinline__ void load_row32(const __nv_bfloat16* src, int col0, int n,
                                           float (&v)[32]) {
  if (col0 + 32 <= n && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 u = __ldg(s4 + q);
      v[q * 8 + 0] = bf16_lo(u.x);
      v[q * 8 + 1] = bf16_hi(u.x);
      v[q * 8 + 2] = bf16_lo(u.y);
      v[q * 8 + 3] = bf16_hi(u.y);
      v[q * 8 + 4] = bf16_lo(u.z);
      v[q * 8 + 5] = bf16_hi(u.z);
      v[q * 8 + 6] = bf16_lo(u.w);
      v[q * 8 + 7] = bf16_hi(u.w);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = (col0 + j < n) ? __bfloat162float(src[j]) : 0.f;
  }
}

__device__ __forceinline__ void store_row32(__nv_bfloat16* dst, int col0, int n,
                                            const float (&v)[32]) {
  if (col0 + 32 <= n && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      u.x = pack_bf16(v[q * 8 + 0], v[q * 8 + 1]);
      u.y = pack_bf16(v[q * 8 + 2], v[q * 8 + 3]);
      u.z = pack_bf16(v[q * 8 + 4], v[q * 8 + 5]);
      u.w = pack_bf16(v[q * 8 + 6], v[q * 8 + 7]);
      d4[q] = u;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j < n) dst[j] = __float2bfloat16_rn(v[j]);
  }
}

// fp32 read-modify-write of 32 consecutive elements: dst = alpha * dst + v.
// All loads are issued before any store (no load-after-store chain).
__device__ __forceinline__ void rmw_row32(float* dst, int col0, int n, float alpha,
                                          const float (&v)[32]) {
  if (alpha == 0.f) {  // plain fp32 store (no read of the previous value)
    if (col0 + 32 <= n && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
      float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
      for (int q = 0; q < 8; ++q) d4[q] = make_float4(v[q * 4], v[q * 4 + 1], v[q * 4 + 2], v[q * 4 + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < n) dst[j] = v[j];
    }
    return;
  }
  if (col0 + 32 <= n && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    float4* d4 = reinterpret_cast<float4*>(dst);
    float4 o[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = d4[q];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      o[q].x = alpha * o[q].x + v[q * 4 + 0];
      o[q].y = alpha * o[q].y + v[q * 4 + 1];
      o[q].z = alpha * o[q].z + v[q * 4 + 2];
      o[q].w = alpha * o[q].w + v[q * 4 + 3];
      d4[q] = o[q];
    }
  } else {
    float o[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) o[j] = col0 + j < n ? dst[j] : 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j < n) dst[j] = alpha * o[j] + v[j];
  }
}

// Symmetric fp32 read-modify-write (same single-writer rule as below). The
// mirrored part reads its 32 old values first: for a fixed j the warp's lanes
// touch 32 consecutive floats of row col0 + j (coalesced), and no store sits
// between the loads.
__device__ __forceinline__ void rmw_row32_sym(float* out, long long ld, int row, int col0, int n,
                                              float alpha, const float (&v)[32]) {
  if (col0 >= row) {
    rmw_row32(out + row * ld + col0, col0, n, alpha, v);
  } else if (col0 + 31 >= row) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j >= row && col0 + j < n) {
        float* p = out + row * ld + col0 + j;
        *p = alpha * *p + v[j];
      }
  }
  if (col0 + 31 > row) {
    float o[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int c = col0 + j;
      o[j] = (c > row && c < n) ? out[static_cast<long long>(c) * ld + row] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int c = col0 + j;
      if (c > row && c < n) out[static_cast<long long>(c) * ld + row] = alpha * o[j] + v[j];
    }
  }
}

// Symmetric output: element (row, c) is written directly when c >= row and
// mirrored to (c, row) when c > row, so every element has exactly one writer.
__device__ __forceinline__ void store_row32_sym(__nv_bfloat16* out, long long ld, int row,
                                                int col0, int n, const float (&v)[32]) {
  if (col0 >= row) {
    store_row32(out + row * ld + col0, col0, n, v);
  } else if (col0 + 31 >= row) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j >= row && col0 + j < n) out[row * ld + col0 + j] = __float2bfloat16_rn(v[j]);
  }
  if (col0 + 31 > row) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int c = col0 + j;
      if (c > row && c < n) out[static_cast<long long>(c) * ld + row] = __float2bfloat16_rn(v[j]);
    }
  }
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_async16_evict_first(uint32_t smem_dst, const void* src,
                                                       uint32_t src_bytes, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(smem_dst),
               "l"(src), "r"(src_bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_global_v4_evict_first(void* dst, float4 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(dst),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_global_v4_evict_first(void* dst, uint4 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(dst),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// kEpiFinal epilogue of one warp (32 rows of the CTA's 128). W is staged per
// 32-column chunk as a 32 x 32 fp32 box in shared memory, kFinBufs - 1 chunks
// ahead, by cp.async (the LSU path: no contention with the operand TMA
// stream; the first boxes are requested before the tile's accumulator is
// ready). Box row r is one 128-byte segment of a W row; its 16-byte pieces
// are XOR-swizzled (piece k of row r at k ^ (r & 7)), so the coalesced copies
// (one instruction = 4 whole rows), a lane's walk along its own row and a
// lane's walk down a column are all free of bank conflicts. Not transposed
// (W = X, [M][N]) lane = X row = box row; transposed (W = X^T, [N][M]) box
// rows are W rows n and lane = m walks down its column. The updated box goes
// back to W, and its bf16 copy to the replica, with coalesced 16-byte stores.
// sum (lr*update)^2 of the warp goes to one partial slot per (tile, CTA,
// warp): the update norm is summed later in a fixed order.
template <int CG>
__device__ __forceinline__ void final_epilogue(const NsGemmParams& P, int it_begin, int it_end,
                                               int it_step, bool sched, uint32_t rank, int q,
                                               int lane, uint32_t tmem_base, uint64_t* tfull_bar,
                                               uint64_t* tempty_bar, uint8_t* fin) {
  float* box0 = reinterpret_cast<float*>(fin + q * kFinBufs * kFinWBox);
  const uint32_t box0_s = smem_u32(box0);
  const int sw = lane & 7;
  const int crow = lane >> 3, cpiece = lane & 7;  // coalesced W copies: 4 rows x 8 pieces
  const int rrow = lane >> 2, rpiece = lane & 3;  // coalesced replica stores: 8 rows x 4 pieces
  // W and the replica stream through L2 once: evict them first so the
  // operand panels the other tiles reuse stay resident
  const uint64_t pol = l2_policy_evict_first();
  uint32_t acc = 0, acc_phase = 0;
  for (int it = it_begin; it < it_end; it += it_step) {
    const int t = sched ? __ldg(P.sched + it) : it;
    const TileCoord c = decode_tile(P, t);
    const NsGemmProblem& pr = P.prob[c.p];
    const NsFinalTarget& ft = pr.final_targets[c.b];
    const int transposed = ft.transposed;
    float* const W = ft.w;
    __nv_bfloat16* const rep = ft.replica;
    const int M = pr.M, N = pr.N;
    const int x_row0 = c.tm * (128 * CG) + static_cast<int>(rank) * 128 + q * 32;  // X' rows (m)
    const int row = x_row0 + lane;
    const int nch = min(kNsBN / 32, (N - c.tn * kNsBN + 31) / 32);
    const float s = pr.scale != nullptr ? __ldg(pr.scale + c.b) : 1.f;
    // W geometry of chunk ch's box: box row r is W row (grow0 + r), columns
    // [gcol0, gcol0 + 32); the W row pitch is ld, valid rows < nrow, cols < ld
    const int ld = transposed ? M : N, nrow = transposed ? N : M;
    const auto geom = [&](int ch, int& grow0, int& gcol0) {
      const int xc = c.tn * kNsBN + ch * 32;
      if (transposed) { grow0 = xc; gcol0 = x_row0; } else { grow0 = x_row0; gcol0 = xc; }
    };
    const auto request = [&](int ch) {  // always commits a group (maybe empty)
      if (ch < nch) {
        int grow0, gcol0;
        geom(ch, grow0, gcol0);
        const uint32_t dst = box0_s + (ch % kFinBufs) * kFinWBox;
        const int gc = gcol0 + 4 * cpiece;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = 4 * i + crow;
          const bool v = grow0 + r < nrow && gc < ld;
          const float* src = v ? W + static_cast<long long>(grow0 + r) * ld + gc : W;
          cp_async16_evict_first(dst + r * 128 + 16 * (cpiece ^ (r & 7)), src, v ? 16u : 0u, pol);
        }
      }
      cp_async_commit();
    };
#pragma unroll
    for (int ch = 0; ch < kFinBufs - 1; ++ch) request(ch);
    mbar_wait(&tfull_bar[acc], acc_phase);
    tc_fence_after();
    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * kNsBN;
    float sq = 0.f;  // this lane's (lr*update)^2 over the tile (fixed order)
#pragma unroll 1
    for (int ch = 0; ch < nch; ++ch) {
      request(ch + kFinBufs - 1);  // the buffer it fills was released at the end of chunk ch - 1
      uint32_t r[32];
      tmem_ld_32x32b_x32(taddr + ch * 32, r);
      tmem_ld_wait();
      const int col0 = c.tn * kNsBN + ch * 32;
      float u[32];
      if (P.alpha != 0.f && row < M)
        load_row32(pr.aux + c.b * pr.aux_bstride + row * pr.aux_ld + col0, col0, N, u);
      else
#pragma unroll
        for (int j = 0; j < 32; ++j) u[j] = 0.f;
      float sq4[4] = {0.f, 0.f, 0.f, 0.f};  // four independent chains
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const bool ok = row < M && col0 + j < N;
        u[j] = ok ? P.lr * (s * (P.alpha * u[j] + __uint_as_float(r[j]))) : 0.f;
        sq4[j & 3] = fmaf(u[j], u[j], sq4[j & 3]);
      }
      sq += (sq4[0] + sq4[1]) + (sq4[2] + sq4[3]);
      cp_async_wait<kFinBufs - 1>();  // chunk ch's box: this lane's copies landed
      __syncwarp();                    // ... and every lane's
      float* box = box0 + (ch % kFinBufs) * (kFinWBox / 4);
      if (!transposed) {  // lane = box row
        float* br = box + lane * 32;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float4* p4 = reinterpret_cast<float4*>(br + 4 * (k ^ sw));
          float4 x = *p4;
          x.x -= u[4 * k + 0];
          x.y -= u[4 * k + 1];
          x.z -= u[4 * k + 2];
          x.w -= u[4 * k + 3];
          *p4 = x;
        }
      } else {  // lane = box column
#pragma unroll
        for (int j = 0; j < 32; ++j) box[j * 32 + 4 * ((lane >> 2) ^ (j & 7)) + (lane & 3)] -= u[j];
      }
      __syncwarp();
      int grow0, gcol0;
      geom(ch, grow0, gcol0);
      {  // W: 8 instructions of 4 whole box rows
        const int gc = gcol0 + 4 * cpiece;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = 4 * i + crow;
          if (grow0 + rr < nrow && gc < ld)
            st_global_v4_evict_first(W + static_cast<long long>(grow0 + rr) * ld + gc,
                                     *reinterpret_cast<const float4*>(box + rr * 32 + 4 * (cpiece ^ (rr & 7))),
                                     pol);
        }
      }
      if (rep != nullptr) {  // replica: 4 instructions of 8 whole box rows (64 bytes each)
        const int gc = gcol0 + 8 * rpiece;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int rr = 8 * i + rrow;
          if (grow0 + rr < nrow && gc < ld) {
            const float4 a = *reinterpret_cast<const float4*>(box + rr * 32 + 4 * ((2 * rpiece) ^ (rr & 7)));
            const float4 b = *reinterpret_cast<const float4*>(box + rr * 32 + 4 * ((2 * rpiece + 1) ^ (rr & 7)));
            uint4 h;
            h.x = pack_bf16(a.x, a.y);
            h.y = pack_bf16(a.z, a.w);
            h.z = pack_bf16(b.x, b.y);
            h.w = pack_bf16(b.z, b.w);
            st_global_v4_evict_first(rep + static_cast<long long>(grow0 + rr) * ld + gc, h, pol);
          }
        }
      }
      __syncwarp();  // the box is free for the request of chunk ch + kFinBufs
    }
    cp_async_wait<0>();  // (only empty groups remain)
    double dsq = static_cast<double>(sq);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dsq += __shfl_xor_sync(0xffffffffu, dsq, o);
    if (lane == 0) {
      const int tile_local = c.tm * pr.tiles_n + c.tn;
      ft.partial[(tile_local * CG + static_cast<int>(rank)) * 4 + q] = dsq;
    }
    tc_fence_before();
    if constexpr (CG == 2) mbar_arrive_leader(&tempty_bar[acc]);
    else mbar_arrive(&tempty_bar[acc]);
    acc ^= 1;
    if (acc == 0) acc_phase ^= 1;
  }
}

template <int MODE, int CG>
__global__ void __launch_bounds__(kNsThreads, 1)
    ns_gemm_kernel(const __grid_constant__ NsGemmParams P) {
  using C = Cfg<MODE, CG>;
  constexpr int kStages = C::kStages;
  constexpr uint32_t kStageBytesA = C::kStageA, kStageBytesB = C::kStageB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* smem_a = base;
  uint8_t* smem_b = base + kStages * kStageBytesA;
  uint8_t* fin = smem_b + kStages * kStageBytesB;  // 1 KiB aligned (kEpiFinal staging)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(fin + epi_stage_bytes<MODE>());
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;  // 0 = leader of the pair
  const int unit = blockIdx.x / CG, n_units = gridDim.x / CG;  // tiles are per cluster
  // tile sequence of this unit: the host's cost-balanced schedule when one is
  // attached for this grid, else static striding (t = unit, unit + n_units, ...)
  const bool sched = P.sched != nullptr && P.sched_units == n_units;
  const int it_begin = sched ? P.sched_off[unit] : unit;
  const int it_end = sched ? P.sched_off[unit + 1] : P.total_tiles;
  const int it_step = sched ? 1 : n_units;

  if (warp == 0 && lane == 0) {
    for (int p = 0; p < P.num_problems; ++p) {
      tma_prefetch_desc(&P.prob[p].tmA);
      tma_prefetch_desc(&P.prob[p].tmB);
    }
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 128 * CG);  // every epilogue thread of the pair
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CG == 2) tmem_alloc_cg2(tmem_slot, kTmemCols);
    else tmem_alloc(tmem_slot, kTmemCols);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      const auto load = [&](void* dst, const CUtensorMap* map, int c0, int c1, int c2) {
        if constexpr (CG == 2) tma_load_3d_cg2(dst, map, &full_bar[stage], c0, c1, c2);
        else tma_load_3d(dst, map, &full_bar[stage], c0, c1, c2);
      };
      for (int it = it_begin; it < it_end; it += it_step) {
        const int t = sched ? __ldg(P.sched + it) : it;
        const TileCoord c = decode_tile(P, t);
        const NsGemmProblem& pr = P.prob[c.p];
        int kb0 = 0, kb1 = (pr.K + kNsBK - 1) / kNsBK;
        if (sched && P.seg_kb != nullptr) {
          const int2 r = __ldg(P.seg_kb + it);
          kb0 = r.x;
          kb1 = r.y;
        }
        const int a_row = c.tm * C::kTileM + rank * C::kRowsA;
        const int b_row = c.tn * kNsBN + rank * C::kRowsB;
        // operands in the upper-tile form need the per-k-block mirror choice;
        // every other tile runs the plain loop (the choice costs issue slots)
        const bool up = (pr.a_upper && c.tm > 0) || (pr.b_upper && c.tn > 0);
        if (!up) {
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            // the leader's full barrier counts the bytes of both CTAs of the pair
            if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], CG * (kStageBytesA + kStageBytesB));
            load(smem_a + stage * kStageBytesA, &pr.tmA, kb * kNsBK, a_row, c.b);
            uint8_t* sb = smem_b + stage * kStageBytesB;
            if (!pr.b_mn_major) {
              load(sb, &pr.tmB, kb * kNsBK, b_row, c.b);
            } else {
#pragma unroll
              for (int q = 0; q < static_cast<int>(C::kRowsB) / 64; ++q)
                load(sb + q * 8192, &pr.tmB, b_row + q * 64, kb * kNsBK, c.b);
            }
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          continue;
        }
        // upper-tile operands: k-blocks left of the diagonal tile come from
        // the mirrored tile of the same K segment through the MN-major view
        int sgi = kb0 * kNsBK / pr.k_seg;                // segment, and column inside it
        int cc = kb0 * kNsBK - sgi * pr.k_seg;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], CG * (kStageBytesA + kStageBytesB));
          const int kv = kb * kNsBK;
          const int kt = cc / kNsBN;  // the k-block's tile column inside its segment
          uint8_t* sa = smem_a + stage * kStageBytesA;
          if (pr.a_upper && kt < c.tm) {
            const int col = (sgi + pr.a_seg0) * pr.k_seg + a_row;
#pragma unroll
            for (int q = 0; q < static_cast<int>(C::kRowsA) / 64; ++q)
              load(sa + q * 8192, &pr.tmA2, col + q * 64, cc, c.b);
          } else {
            load(sa, &pr.tmA, kv, a_row, c.b);
          }
          uint8_t* sb = smem_b + stage * kStageBytesB;
          if (pr.b_mn_major) {
#pragma unroll
            for (int q = 0; q < static_cast<int>(C::kRowsB) / 64; ++q)
              load(sb + q * 8192, &pr.tmB, b_row + q * 64, kv, c.b);
          } else if (pr.b_upper && kt < c.tn) {
            const int col = (sgi + pr.b_seg0) * pr.k_seg + b_row;
#pragma unroll
            for (int q = 0; q < static_cast<int>(C::kRowsB) / 64; ++q)
              load(sb + q * 8192, &pr.tmB2, col + q * 64, cc, c.b);
          } else {
            load(sb, &pr.tmB, kv, b_row, c.b);
          }
          if ((cc += kNsBK) == pr.k_seg) {
            cc = 0;
            ++sgi;
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------- tcgen05 issuer
    if (lane == 0 && rank == 0) {
      const uint32_t idesc_k = idesc_bf16_f32(C::kTileM, kNsBN, false, false);
      const uint32_t idesc_mn = idesc_bf16_f32(C::kTileM, kNsBN, false, true);
      const uint32_t idesc_ak = idesc_bf16_f32(C::kTileM, kNsBN, true, false);
      const uint32_t idesc_amn = idesc_bf16_f32(C::kTileM, kNsBN, true, true);
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      for (int it = it_begin; it < it_end; it += it_step) {
        const int t = sched ? __ldg(P.sched + it) : it;
        const TileCoord c = decode_tile(P, t);
        const NsGemmProblem& pr = P.prob[c.p];
        int kb0 = 0, kb1 = (pr.K + kNsBK - 1) / kNsBK;
        if (sched && P.seg_kb != nullptr) {
          const int2 r = __ldg(P.seg_kb + it);
          kb0 = r.x;
          kb1 = r.y;
        }
        const bool mn = pr.b_mn_major != 0;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kNsBN;
        const bool up = (pr.a_upper && c.tm > 0) || (pr.b_upper && c.tn > 0);
        if (!up) {  // (as the producer: the plain loop)
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            const uint32_t a0 = smem_u32(smem_a + stage * kStageBytesA);
            const uint32_t b0 = smem_u32(smem_b + stage * kStageBytesB);
#pragma unroll
            for (int k = 0; k < kNsBK / 16; ++k) {
              const uint64_t adesc = smem_desc_sw128(a0 + k * 32, 16, 1024);
              const uint64_t bdesc = mn ? smem_desc_sw128(b0 + k * 2048, 8192, 1024)
                                        : smem_desc_sw128(b0 + k * 32, 16, 1024);
              if constexpr (CG == 2)
                umma_bf16_cg2(d_tmem, adesc, bdesc, mn ? idesc_mn : idesc_k, (kb != kb0) || k != 0);
              else
                umma_bf16(d_tmem, adesc, bdesc, mn ? idesc_mn : idesc_k, (kb != kb0) || k != 0);
            }
            if constexpr (CG == 2) umma_commit_cg2_mc(&empty_bar[stage], 0x3);
            else umma_commit(&empty_bar[stage]);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        } else {
          int cc = kb0 * kNsBK - (kb0 * kNsBK / pr.k_seg) * pr.k_seg;
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            const uint32_t a0 = smem_u32(smem_a + stage * kStageBytesA);
            const uint32_t b0 = smem_u32(smem_b + stage * kStageBytesB);
            const int kt = cc / kNsBN;
            const bool amn = pr.a_upper && kt < c.tm;               // (as the producer)
            const bool bmn = mn || (pr.b_upper && kt < c.tn);
            const uint32_t idesc = amn ? (bmn ? idesc_amn : idesc_ak) : (bmn ? idesc_mn : idesc_k);
#pragma unroll
            for (int k = 0; k < kNsBK / 16; ++k) {
              const uint64_t adesc = amn ? smem_desc_sw128(a0 + k * 2048, 8192, 1024)
                                         : smem_desc_sw128(a0 + k * 32, 16, 1024);
              const uint64_t bdesc = bmn ? smem_desc_sw128(b0 + k * 2048, 8192, 1024)
                                         : smem_desc_sw128(b0 + k * 32, 16, 1024);
              if constexpr (CG == 2)
                umma_bf16_cg2(d_tmem, adesc, bdesc, idesc, (kb != kb0) || k != 0);
              else
                umma_bf16(d_tmem, adesc, bdesc, idesc, (kb != kb0) || k != 0);
            }
            if constexpr (CG == 2) umma_commit_cg2_mc(&empty_bar[stage], 0x3);
            else umma_commit(&empty_bar[stage]);
            if ((cc += kNsBK) == pr.k_seg) cc = 0;
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
        if constexpr (CG == 2) umma_commit_cg2_mc(&tfull_bar[acc], 0x3);
        else umma_commit(&tfull_bar[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4 && MODE == kEpiFinal) {
    final_epilogue<CG>(P, it_begin, it_end, it_step, sched, rank, warp & 3, lane, tmem_base,
                       tfull_bar, tempty_bar, fin);
  } else if (warp >= 4) {
    // ---------------------------------------------------------- epilogue
    const int quarter = warp & 3;
    const int row_in_tile = quarter * 32 + lane;
    uint32_t acc = 0, acc_phase = 0;
    for (int it = it_begin; it < it_end; it += it_step) {
      const int t = sched ? __ldg(P.sched + it) : it;
      const TileCoord c = decode_tile(P, t);
      const NsGemmProblem& pr = P.prob[c.p];
      const int row_base = c.tm * C::kTileM + rank * C::kRowsA;
      const int row = row_base + row_in_tile;
      const bool row_ok = row < pr.M;
      const float s = pr.scale != nullptr ? __ldg(pr.scale + c.b) : 1.f;
      // POLY: the aux row segment (b·A) of the next chunk is loaded one chunk
      // ahead — the first while waiting for the accumulator — so its L2/DRAM
      // latency hides behind the TMEM loads and stores of the current chunk
      uint4 ax_nxt[4];
      bool ax_nxt_ok = false;
      const __nv_bfloat16* ax_row =
          MODE == kEpiPoly && pr.aux != nullptr ? pr.aux + c.b * pr.aux_bstride + row * pr.aux_ld : nullptr;
      auto ax_prefetch = [&](int chunk) {
        const int col = c.tn * kNsBN + chunk * 32;
        ax_nxt_ok = MODE == kEpiPoly && P.alpha != 0.f && row_ok && col + 32 <= pr.N &&
                    ((reinterpret_cast<uintptr_t>(ax_row + col) & 15) == 0);
        if (ax_nxt_ok) {
          const uint4* s4 = reinterpret_cast<const uint4*>(ax_row + col);
#pragma unroll
          for (int q = 0; q < 4; ++q) ax_nxt[q] = __ldg(s4 + q);
        }
      };
      if constexpr (MODE == kEpiPoly) ax_prefetch(0);
      // STAT read-modify-write (alpha != 0) of a plain or upper-only output:
      // the old fp32 values of the next chunk are loaded one chunk ahead
      float4 so_nxt[8];
      bool so_nxt_ok = false;
      float* so_row = MODE == kEpiStat && pr.out32 != nullptr
                          ? pr.out32 + c.b * pr.out_bstride + row * pr.out_ld
                          : nullptr;
      auto so_prefetch = [&](int chunk) {
        const int col = c.tn * kNsBN + chunk * 32;
        so_nxt_ok = MODE == kEpiStat && P.alpha != 0.f && pr.symmetric != 1 && row_ok &&
                    col + 32 <= pr.N && (pr.symmetric == 0 || col >= row) &&
                    ((reinterpret_cast<uintptr_t>(so_row + col) & 15) == 0);
        if (so_nxt_ok) {
          const float4* s4 = reinterpret_cast<const float4*>(so_row + col);
#pragma unroll
          for (int q = 0; q < 8; ++q) so_nxt[q] = s4[q];
        }
      };
      if constexpr (MODE == kEpiStat) so_prefetch(0);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * kNsBN;
      // stream-K part of a tile: the raw accumulator to its partial slot
      const int slot = (MODE == kEpiGram && sched && P.seg_slot != nullptr) ? __ldg(P.seg_slot + it) : -1;
#pragma unroll 1
      for (int chunk = 0; chunk < kNsBN / 32; ++chunk) {
        uint4 ax_cur[4];
        bool ax_cur_ok = false;
        if constexpr (MODE == kEpiPoly) {
#pragma unroll
          for (int q = 0; q < 4; ++q) ax_cur[q] = ax_nxt[q];
          ax_cur_ok = ax_nxt_ok;
          if (chunk + 1 < kNsBN / 32) ax_prefetch(chunk + 1);
        }
        float4 so_cur[8];
        bool so_cur_ok = false;
        if constexpr (MODE == kEpiStat) {
#pragma unroll
          for (int q = 0; q < 8; ++q) so_cur[q] = so_nxt[q];
          so_cur_ok = so_nxt_ok;
          if (chunk + 1 < kNsBN / 32) so_prefetch(chunk + 1);
        }
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + chunk * 32, r);
        tmem_ld_wait();
        if (slot >= 0) {
          float4* d = reinterpret_cast<float4*>(
              P.seg_ws + (static_cast<size_t>(slot) * 256 + rank * C::kRowsA + row_in_tile) * kNsBN +
              chunk * 32);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            d[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                               __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
          continue;
        }
        const int col0 = c.tn * kNsBN + chunk * 32;
        if (col0 >= pr.N) continue;  // warp-uniform
        if (!row_ok) continue;
        float v[32];
        if constexpr (MODE == kEpiGram) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = s * __uint_as_float(r[j]);
          if (pr.symmetric && !(pr.symmetric == 3 && c.tn != c.tm))
            store_row32_sym(pr.out + c.b * pr.out_bstride, pr.out_ld, row, col0, pr.N, v);
          else  // (upper-tile form: an off-diagonal tile is stored as computed)
            store_row32(pr.out + c.b * pr.out_bstride + row * pr.out_ld + col0, col0, pr.N, v);
        } else if constexpr (MODE == kEpiPoly) {
          if (ax_cur_ok) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              v[q * 8 + 0] = bf16_lo(ax_cur[q].x);
              v[q * 8 + 1] = bf16_hi(ax_cur[q].x);
              v[q * 8 + 2] = bf16_lo(ax_cur[q].y);
              v[q * 8 + 3] = bf16_hi(ax_cur[q].y);
              v[q * 8 + 4] = bf16_lo(ax_cur[q].z);
              v[q * 8 + 5] = bf16_hi(ax_cur[q].z);
              v[q * 8 + 6] = bf16_lo(ax_cur[q].w);
              v[q * 8 + 7] = bf16_hi(ax_cur[q].w);
            }
          } else if (P.alpha != 0.f)
            load_row32(pr.aux + c.b * pr.aux_bstride + row * pr.aux_ld + col0, col0, pr.N, v);
          else
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = P.alpha * v[j] + P.beta * __uint_as_float(r[j]);
          // + lr * I (the Newton-Schulz 'a' folded into B, so UPDATE needs no aux read)
          if (P.lr != 0.f && row >= col0 && row < col0 + 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col0 + j == row) v[j] += P.lr;
          }
          if (pr.symmetric && !(pr.symmetric == 3 && c.tn != c.tm))
            store_row32_sym(pr.out + c.b * pr.out_bstride, pr.out_ld, row, col0, pr.N, v);
          else
            store_row32(pr.out + c.b * pr.out_bstride + row * pr.out_ld + col0, col0, pr.N, v);
        } else if constexpr (MODE == kEpiUpdate) {
          if (P.alpha != 0.f)
            load_row32(pr.aux + c.b * pr.aux_bstride + row * pr.aux_ld + col0, col0, pr.N, v);
          else
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = s * (P.alpha * v[j] + __uint_as_float(r[j]));
          store_row32(pr.out + c.b * pr.out_bstride + row * pr.out_ld + col0, col0, pr.N, v);
        } else if constexpr (MODE == kEpiStat) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = s * __uint_as_float(r[j]);
          float* o = pr.out32 + c.b * pr.out_bstride;
          if (so_cur_ok) {  // whole chunk on or above the diagonal, old values in registers
            float4* d4 = reinterpret_cast<float4*>(o + row * pr.out_ld + col0);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              d4[q] = make_float4(P.alpha * so_cur[q].x + v[q * 4 + 0], P.alpha * so_cur[q].y + v[q * 4 + 1],
                                  P.alpha * so_cur[q].z + v[q * 4 + 2], P.alpha * so_cur[q].w + v[q * 4 + 3]);
          } else if (pr.symmetric == 1) {
            rmw_row32_sym(o, pr.out_ld, row, col0, pr.N, P.alpha, v);
          } else if (pr.symmetric == 2) {
            // upper triangle only (the owner fills the lower one before reading
            // the whole matrix: launch_sym_fill_lower)
            if (col0 >= row) {
              rmw_row32(o + row * pr.out_ld + col0, col0, pr.N, P.alpha, v);
            } else if (col0 + 31 >= row) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (col0 + j >= row && col0 + j < pr.N) {
                  float* p = o + row * pr.out_ld + col0 + j;
                  *p = P.alpha == 0.f ? v[j] : P.alpha * *p + v[j];
                }
            }
          } else {
            rmw_row32(o + row * pr.out_ld + col0, col0, pr.N, P.alpha, v);
          }
        } else if constexpr (MODE == kEpiSplit) {
          float lo[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float x = s * __uint_as_float(r[j]);
            v[j] = __bfloat162float(__float2bfloat16_rn(x));
            lo[j] = x - v[j];
          }
          __nv_bfloat16* o = pr.out + c.b * pr.out_bstride;
          const long long sg = pr.out_seg;
          const int rblk = row_base + quarter * 32;  // this warp's 32 rows (32-aligned)
          const bool mirror = pr.symmetric == 1 || (pr.symmetric == 3 && c.tn == c.tm);
          if (mirror && col0 >= rblk + 32 && rblk + 32 <= pr.M && col0 + 32 <= pr.N &&
              (pr.out_ld & 7) == 0 && (sg & 7) == 0 &&
              (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
            // whole chunk above this warp's diagonal: rows leave as 16 B
            // stores; the mirrored block goes through shared memory
            __nv_bfloat16* d = o + row * pr.out_ld + col0;
            store_row32(d, col0, pr.N, v);
            store_row32(d + sg, col0, pr.N, lo);
            store_row32(d + 2 * sg, col0, pr.N, v);
            store_row32(d + 3 * sg, col0, pr.N, v);
            __nv_bfloat16* th = reinterpret_cast<__nv_bfloat16*>(fin + quarter * kSplitWarpBytes);
            __nv_bfloat16* tl = th + 32 * kSplitPitch;
            __syncwarp();  // the previous chunk's reads of the staging are done
#pragma unroll
            for (int j = 0; j < 32; ++j) {  // staged[j][lane] = value (row, col0 + j)
              th[j * kSplitPitch + lane] = __float2bfloat16_rn(v[j]);
              tl[j * kSplitPitch + lane] = __float2bfloat16_rn(lo[j]);
            }
            __syncwarp();
            // lane L: output row col0 + L, columns rblk .. rblk + 31
            const uint4* sh = reinterpret_cast<const uint4*>(th + lane * kSplitPitch);
            const uint4* sl = reinterpret_cast<const uint4*>(tl + lane * kSplitPitch);
            uint4* m = reinterpret_cast<uint4*>(o + static_cast<long long>(col0 + lane) * pr.out_ld + rblk);
            uint4* m1 = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(m) + sg);
            uint4* m2 = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(m) + 2 * sg);
            uint4* m3 = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(m) + 3 * sg);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 hv = sh[q], lv = sl[q];
              m[q] = hv;
              m1[q] = lv;
              m2[q] = hv;
              m3[q] = hv;
            }
          } else if (mirror) {
            store_row32_sym(o, pr.out_ld, row, col0, pr.N, v);
            store_row32_sym(o + sg, pr.out_ld, row, col0, pr.N, lo);
            store_row32_sym(o + 2 * sg, pr.out_ld, row, col0, pr.N, v);
            store_row32_sym(o + 3 * sg, pr.out_ld, row, col0, pr.N, v);
          } else {
            __nv_bfloat16* d = o + row * pr.out_ld + col0;
            store_row32(d, col0, pr.N, v);
            store_row32(d + sg, col0, pr.N, lo);
            store_row32(d + 2 * sg, col0, pr.N, v);
            store_row32(d + 3 * sg, col0, pr.N, v);
          }
        }
      }
      tc_fence_before();
      if constexpr (CG == 2) mbar_arrive_leader(&tempty_bar[acc]);
      else mbar_arrive(&tempty_bar[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_cg2(tmem_base, kTmemCols);
    else tmem_dealloc(tmem_base, kTmemCols);
  }
}

// Stream-K fixup: every tile that was cut across units is the fixed-order
// sum of its parts' partial slots, finished with the GRAM epilogue (scale,
// bf16, symmetric mirror). blockIdx.x = split tile, blockIdx.y = 8-row band;
// a thread sums 8 consecutive columns of one row.
__global__ void __launch_bounds__(256) stream_k_fixup_kernel(const __grid_constant__ NsGemmParams P,
                                                             const int* fix) {
  const int* f = fix + 6 * blockIdx.x;
  const NsGemmProblem& pr = P.prob[f[0]];
  const int b = f[1], tm = f[2], tn = f[3], slot0 = f[4], ns = f[5];
  const int lr = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int lc = (threadIdx.x & 31) * 8;
  if (lr >= P.tile_m) return;
  const int row = tm * P.tile_m + lr, col0 = tn * kNsBN + lc;
  if (row >= pr.M || col0 >= pr.N) return;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int k = 0; k < ns; ++k) {  // parts in k-block order
    const float4* src = reinterpret_cast<const float4*>(
        P.seg_ws + (static_cast<size_t>(slot0 + k) * 256 + lr) * kNsBN + lc);
    const float4 x = src[0], y = src[1];
    acc[0] += x.x; acc[1] += x.y; acc[2] += x.z; acc[3] += x.w;
    acc[4] += y.x; acc[5] += y.y; acc[6] += y.z; acc[7] += y.w;
  }
  const float sc = pr.scale != nullptr ? __ldg(pr.scale + b) : 1.f;
  __nv_bfloat16* out = pr.out + b * pr.out_bstride;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int col = col0 + j;
    if (col >= pr.N) break;
    const __nv_bfloat16 v = __float2bfloat16_rn(sc * acc[j]);
    if (!pr.symmetric) {
      out[row * pr.out_ld + col] = v;
    } else {
      if (col >= row) out[row * pr.out_ld + col] = v;
      if (col > row && (pr.symmetric != 3 || tm == tn))  // (upper-tile form: diagonal tiles only)
        out[static_cast<long long>(col) * pr.out_ld + row] = v;
    }
  }
}

// ------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// rows x cols per batch, row stride ld, batch stride bstride (elements);
// the tensor map's dim0 is `cols` (contiguous), dim1 `rows`, dim2 batch.
bool make_map(CUtensorMap* map, const NsMatrixRef& m, uint32_t box_cols, uint32_t box_rows) {
  EncodeFn enc = encode_fn();
  if (enc == nullptr) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(m.cols), static_cast<cuuint64_t>(m.rows),
                              static_cast<cuuint64_t>(m.batch)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(m.ld) * 2,
                                 static_cast<cuuint64_t>(m.bstride) * 2};
  const cuuint32_t box[3] = {box_cols, box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(m.ptr), dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

int sm_count() { return device_sm_count(); }

template <int MODE, int CG>
cudaError_t launch_mode(const NsGemmParams& P, cudaStream_t stream) {
  constexpr uint32_t smem = smem_bytes<MODE, CG>();
  if (cudaError_t e = set_max_dynamic_smem(reinterpret_cast<const void*>(ns_gemm_kernel<MODE, CG>),
                                           static_cast<int>(smem));
      e != cudaSuccess)
    return e;
  if constexpr (CG == 1) {
    const int grid = std::min(P.total_tiles, sm_count());
    ns_gemm_kernel<MODE, 1><<<grid, kNsThreads, smem, stream>>>(P);
    return cudaGetLastError();
  } else {
    // one 2-CTA cluster per pair of SMs; tiles are strided over clusters
    const int clusters = std::min(P.total_tiles, sm_count() / 2);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * clusters));
    cfg.blockDim = dim3(kNsThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, ns_gemm_kernel<MODE, 2>, P);
  }
}

int g_cta_group = 0;  // 0: not yet read from OSH_GEMM_CTA_GROUP (default 2)

int cta_group() {
  if (g_cta_group == 0) {
    const char* v = std::getenv("OSH_GEMM_CTA_GROUP");
    g_cta_group = (v != nullptr && v[0] == '1') ? 1 : 2;
  }
  return g_cta_group;
}

int sym_tiles(int tiles_m, int tiles_n, int tile_m) {
  int t = 0;
  for (int tn = 0; tn < tiles_n; ++tn)
    t += std::min(tiles_m, (kNsBN * tn + kNsBN - 1) / tile_m + 1);
  return t;
}

}  // namespace

bool final_target_ok(const void* w, const void* replica, int M, int N, int transposed) {
  const auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const int inner = transposed ? M : N;  // contiguous extent of W in elements
  if (w == nullptr || !a16(w) || inner % 4 != 0) return false;
  return replica == nullptr || (a16(replica) && inner % 8 == 0);
}

bool make_final_target(NsFinalTarget* t, float* w, __nv_bfloat16* replica, int M, int N,
                       int transposed, double* partial) {
  std::memset(t, 0, sizeof(*t));
  if (!final_target_ok(w, replica, M, N, transposed) || partial == nullptr) return false;
  t->w = w;
  t->replica = replica;
  t->partial = partial;
  t->transposed = transposed;
  return true;
}

int final_partials(int M, int N) {
  const int cg = cta_group();
  return ((M + 128 * cg - 1) / (128 * cg)) * ((N + kNsBN - 1) / kNsBN) * cg * 4;
}

void ns_gemm_set_cta_group(int cg) { g_cta_group = (cg == 1) ? 1 : 2; }
int ns_gemm_cta_group() { return cta_group(); }

double ns_gemm_executed_flops(const NsProblemDesc* probs, int num_problems) {
  double f = 0.0;
  for (int i = 0; i < num_problems; ++i) {
    const NsProblemDesc& d = probs[i];
    const double K = d.a.cols, M = d.a.rows;
    const double N = d.b_mn_major ? d.b.cols : d.b.rows;
    double frac = 1.0;
    if (d.symmetric) {
      const int tile_m = 128 * cta_group();
      const int tm = (d.a.rows + tile_m - 1) / tile_m;
      const int tn = (static_cast<int>(N) + kNsBN - 1) / kNsBN;
      frac = static_cast<double>(sym_tiles(tm, tn, tile_m)) / (static_cast<double>(tm) * tn);
    }
    f += 2.0 * M * N * K * d.a.batch * frac;
  }
  return f;
}

double ns_gemm_flops(const NsProblemDesc* probs, int num_problems) {
  double f = 0.0;
  for (int i = 0; i < num_problems; ++i) {
    const NsProblemDesc& d = probs[i];
    const double K = d.a.cols, M = d.a.rows;
    const double N = d.b_mn_major ? d.b.cols : d.b.rows;
    f += 2.0 * M * N * K * d.a.batch;
  }
  return f;
}

int ns_gemm_schedule(int mode, const NsProblemDesc* probs, int num_problems,
                     std::vector<int>* tiles_out, std::vector<int>* off_out, int* total_out) {
  if (num_problems < 1 || num_problems > kMaxProblems) return 0;
  const int cg = cta_group();
  const int tile_m = 128 * cg;
  std::vector<std::pair<long long, int>> cost;  // (cost, linear tile)
  int t = 0;
  for (int i = 0; i < num_problems; ++i) {
    const NsProblemDesc& d = probs[i];
    const int M = d.a.rows, K = d.a.cols, N = d.b_mn_major ? d.b.cols : d.b.rows;
    const bool sym = d.symmetric && M == N &&
                     (mode == kEpiGram || mode == kEpiPoly || mode == kEpiStat || mode == kEpiSplit);
    const int tm = (M + tile_m - 1) / tile_m, tn = (N + kNsBN - 1) / kNsBN;
    const int per = sym ? sym_tiles(tm, tn, tile_m) : tm * tn;
    const long long c = (K + kNsBK - 1) / kNsBK + 2;  // K blocks + epilogue
    for (int k = 0; k < d.a.batch * per; ++k) cost.emplace_back(c, t++);
  }
  const int units = std::min(t, cg == 2 ? sm_count() / 2 : sm_count());
  if (units < 1) return 0;
  std::stable_sort(cost.begin(), cost.end(),
                   [](const auto& a, const auto& b) { return a.first > b.first; });
  std::vector<long long> load(units, 0);
  std::vector<std::vector<int>> lists(units);
  for (const auto& ct : cost) {
    int u = 0;
    for (int v = 1; v < units; ++v)
      if (load[v] < load[u]) u = v;
    load[u] += ct.first;
    lists[u].push_back(ct.second);
  }
  tiles_out->clear();
  off_out->assign(1, 0);
  for (const auto& l : lists) {
    tiles_out->insert(tiles_out->end(), l.begin(), l.end());
    off_out->push_back(static_cast<int>(tiles_out->size()));
  }
  *total_out = t;
  return units;
}

int ns_gemm_stream_k_schedule(const NsProblemDesc* probs, int num_problems,
                              std::vector<int>* tiles_out, std::vector<int>* off_out,
                              std::vector<int2>* kb_out, std::vector<int>* slot_out,
                              std::vector<int>* fix_out, int* n_slots, int* total_out) {
  if (num_problems < 1 || num_problems > kMaxProblems) return 0;
  const int cg = cta_group();
  const int tile_m = 128 * cg;
  // linear tiles (the kernel's decode order: problem, batch, tile) and their k-blocks
  struct T {
    int p, b, tm, tn, nkb;
  };
  std::vector<T> ts;
  for (int i = 0; i < num_problems; ++i) {
    const NsProblemDesc& d = probs[i];
    const int M = d.a.rows, K = d.a.cols, N = d.b_mn_major ? d.b.cols : d.b.rows;
    const bool sym = d.symmetric && M == N;
    const int tmn = (M + tile_m - 1) / tile_m, tnn = (N + kNsBN - 1) / kNsBN;
    const int nkb = (K + kNsBK - 1) / kNsBK;
    for (int b = 0; b < d.a.batch; ++b) {
      if (sym) {  // column-major over the upper-triangle tiles (decode_tile)
        for (int tn = 0; tn < tnn; ++tn)
          for (int tm = 0; tm < std::min(tmn, (kNsBN * tn + kNsBN - 1) / tile_m + 1); ++tm)
            ts.push_back({i, b, tm, tn, nkb});
      } else {  // grouped rasterisation (decode_tile)
        for (int rem = 0; rem < tmn * tnn; ++rem) {
          const int rg = kRasterGroup;  // (stream-K: GRAM only)
          const int span = rg * tnn, group = rem / span, first_m = group * rg;
          const int gsz = std::min(tmn - first_m, rg), r2 = rem - group * span;
          ts.push_back({i, b, first_m + r2 % gsz, r2 / gsz, nkb});
        }
      }
    }
  }
  const int n_tiles = static_cast<int>(ts.size());
  const int units_max = cg == 2 ? sm_count() / 2 : sm_count();
  const int U = std::min(n_tiles, units_max);
  if (U < 2) return 0;
  // Tail split, cut PER MATRIX as if the matrix ran alone on the GPU: its
  // first (mt / U) * U tiles run whole (full rounds, every unit on the same
  // k-blocks of neighbouring tiles, so the operand panels are shared in L2);
  // the last mt % U tiles — a round that would leave units idle — are cut
  // into S equal k-parts, S chosen so the parts fill the units' rounds best,
  // and issued part-major (all tiles' part 0, then part 1, ...), so units
  // running together still read the same k-range. The cut points depend
  // only on the matrix's own shape — never on what shares the launch — so a
  // tensor's result does not depend on the plan (sharded == replicated bit
  // for bit). A stream-K cut with staggered k-phases was measured first: the
  // units' operand reads stopped sharing L2 (28 % hit rate, 7x the DRAM
  // traffic) and the launch got 37 % slower.
  struct Seg {
    int tile;
    int2 kb;
    long long cost;
  };
  std::vector<Seg> segs;
  std::vector<int> n_parts(static_cast<size_t>(n_tiles), 0);
  bool any = false, single = true;
  for (size_t first = 0; first < ts.size();) {
    size_t last = first;  // tiles of one matrix (problem, batch) are contiguous
    while (last < ts.size() && ts[last].p == ts[first].p && ts[last].b == ts[first].b) ++last;
    if (first != 0 || last != ts.size()) single = false;
    const int mt = static_cast<int>(last - first), nkb = ts[first].nkb;
    const int full = mt / units_max * units_max, rest = mt - full;
    // parts per tail tile: the S in 2..16 whose rounds ceil(rest*S/U)/S are
    // shortest (whole tiles: 1 round of 1), if that beats not splitting by > 5 %
    int best_s = 1;
    double best = 1.0;
    if (nkb >= 256 && full > 0 && rest > 0)
      for (int sp = 2; sp <= 16 && nkb / sp >= 32; ++sp) {
        const double r = static_cast<double>((rest * sp + units_max - 1) / units_max) / sp;
        if (r < best - 1e-9) {
          best = r;
          best_s = sp;
        }
      }
    if (best > 0.95) best_s = 1;
    for (int i = 0; i < full; ++i)
      segs.push_back({static_cast<int>(first) + i, make_int2(0, nkb), nkb + 2});
    if (best_s == 1) {
      for (int i = full; i < mt; ++i)
        segs.push_back({static_cast<int>(first) + i, make_int2(0, nkb), nkb + 2});
    } else {
      any = true;
      for (int j = 0; j < best_s; ++j) {
        const int k0 = static_cast<int>(static_cast<long long>(nkb) * j / best_s);
        const int k1 = static_cast<int>(static_cast<long long>(nkb) * (j + 1) / best_s);
        for (int i = full; i < mt; ++i)
          segs.push_back({static_cast<int>(first) + i, make_int2(k0, k1), (k1 - k0) + 2});
      }
    }
    first = last;
  }
  if (!any) return 0;
  for (const Seg& g : segs) ++n_parts[static_cast<size_t>(g.tile)];
  // units: one matrix alone takes its segments round-robin in order (whole
  // tiles first, then the parts part-major); mixed launches balance all
  // segments by LPT
  std::vector<std::vector<int>> lists(static_cast<size_t>(U));
  if (single && U == units_max) {
    for (size_t k = 0; k < segs.size(); ++k) lists[k % static_cast<size_t>(U)].push_back(static_cast<int>(k));
  } else {
    std::vector<size_t> order(segs.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](size_t x, size_t y) { return segs[x].cost > segs[y].cost; });
    std::vector<long long> load(static_cast<size_t>(U), 0);
    for (const size_t i : order) {
      int u = 0;
      for (int v = 1; v < U; ++v)
        if (load[static_cast<size_t>(v)] < load[static_cast<size_t>(u)]) u = v;
      load[static_cast<size_t>(u)] += segs[i].cost;
      lists[static_cast<size_t>(u)].push_back(static_cast<int>(i));
    }
  }
  tiles_out->clear();
  kb_out->clear();
  slot_out->clear();
  fix_out->clear();
  off_out->assign(1, 0);
  for (const auto& l : lists) {
    for (const int i : l) {
      tiles_out->push_back(segs[static_cast<size_t>(i)].tile);
      kb_out->push_back(segs[static_cast<size_t>(i)].kb);
      slot_out->push_back(-1);
    }
    off_out->push_back(static_cast<int>(tiles_out->size()));
  }
  std::vector<std::vector<int2>> pieces(static_cast<size_t>(n_tiles));  // parts of split tiles
  for (const Seg& g : segs)
    if (n_parts[static_cast<size_t>(g.tile)] > 1) pieces[static_cast<size_t>(g.tile)].push_back(g.kb);
  // slots for the parts of split tiles, in k order; fixup entries
  int slots = 0;
  std::vector<int> first_slot(static_cast<size_t>(n_tiles), -1);
  for (int i = 0; i < n_tiles; ++i) {
    if (pieces[static_cast<size_t>(i)].size() < 2) continue;
    first_slot[static_cast<size_t>(i)] = slots;
    const T& d = ts[static_cast<size_t>(i)];
    fix_out->insert(fix_out->end(), {d.p, d.b, d.tm, d.tn, slots,
                                     static_cast<int>(pieces[static_cast<size_t>(i)].size())});
    slots += static_cast<int>(pieces[static_cast<size_t>(i)].size());
  }
  // a part's slot = its rank in k order among its tile's parts (fixup order)
  for (size_t k = 0; k < tiles_out->size(); ++k) {
    const int ti = (*tiles_out)[k];
    if (first_slot[static_cast<size_t>(ti)] < 0) continue;
    int rank = 0;
    for (const int2& pc : pieces[static_cast<size_t>(ti)])
      if (pc.x < (*kb_out)[k].x) ++rank;
    (*slot_out)[k] = first_slot[static_cast<size_t>(ti)] + rank;
  }
  *n_slots = slots;
  *total_out = n_tiles;
  return U;
}

cudaError_t ns_gemm_launch(int mode, const NsProblemDesc* probs, int num_problems, float alpha,
                           float beta, float lr, cudaStream_t stream, const NsSchedule* sched) {
  if (num_problems < 1 || num_problems > kMaxProblems) return cudaErrorInvalidValue;
  NsGemmParams P{};
  P.num_problems = num_problems;
  P.alpha = alpha;
  P.beta = beta;
  P.lr = lr;
  const int cg = cta_group();
  P.tile_m = 128 * cg;
  int tiles = 0;
  for (int i = 0; i < num_problems; ++i) {
    const NsProblemDesc& d = probs[i];
    NsGemmProblem& pr = P.prob[i];
    pr.batch = d.a.batch;
    pr.M = d.a.rows;
    pr.K = d.a.cols;
    pr.N = d.b_mn_major ? d.b.cols : d.b.rows;
    const int kb = d.b_mn_major ? d.b.rows : d.b.cols;
    if (kb != pr.K || d.b.batch != pr.batch || pr.M < 1 || pr.N < 1 || pr.K < 1 || pr.batch < 1)
      return cudaErrorInvalidValue;
    pr.b_mn_major = d.b_mn_major;
    if (!make_map(&pr.tmA, d.a, kNsBK, 128)) return cudaErrorInvalidValue;
    if (!d.b_mn_major) {
      if (!make_map(&pr.tmB, d.b, kNsBK, kNsBN / cg)) return cudaErrorInvalidValue;
    } else {
      if (!make_map(&pr.tmB, d.b, 64, kNsBK)) return cudaErrorInvalidValue;
    }
    // upper-tile form: 2-CTA (256 x 256) tiles only; 1-CTA launches read and
    // write full matrices instead (same values)
    pr.a_upper = cg == 2 && d.a_upper ? 1 : 0;
    pr.b_upper = cg == 2 && d.b_upper ? 1 : 0;
    pr.k_seg = d.k_seg > 0 ? d.k_seg : pr.K;
    pr.a_seg0 = d.k_seg > 0 ? d.a_seg0 : 0;
    pr.b_seg0 = d.k_seg > 0 ? d.b_seg0 : 0;
    if ((pr.a_upper || pr.b_upper) && (pr.k_seg % kNsBK != 0 && pr.k_seg != pr.K))
      return cudaErrorInvalidValue;  // a k-block never straddles two segments
    if ((pr.a_upper && pr.M > pr.k_seg) || (pr.b_upper && (d.b_mn_major || pr.N > pr.k_seg)))
      return cudaErrorInvalidValue;  // each segment holds a square (padded) matrix
    // the MN-major mirror views span the whole segmented buffer of the operand
    const auto whole = [&](const NsMatrixRef& v, int seg0) {
      NsMatrixRef w = v;
      if (d.k_seg > 0) {
        w.ptr = static_cast<const __nv_bfloat16*>(v.ptr) - static_cast<long long>(seg0) * d.k_seg;
        w.cols = static_cast<int>(v.ld);
      }
      return w;
    };
    if (pr.a_upper && !make_map(&pr.tmA2, whole(d.a, pr.a_seg0), 64, kNsBK)) return cudaErrorInvalidValue;
    if (pr.b_upper && !make_map(&pr.tmB2, whole(d.b, pr.b_seg0), 64, kNsBK)) return cudaErrorInvalidValue;
    pr.tiles_m = (pr.M + P.tile_m - 1) / P.tile_m;
    pr.tiles_n = (pr.N + kNsBN - 1) / kNsBN;
    pr.symmetric = d.symmetric && pr.M == pr.N &&
                           (mode == kEpiGram || mode == kEpiPoly || mode == kEpiStat ||
                            mode == kEpiSplit)
                       ? (d.symmetric == 2 ? 2 : (d.symmetric == 3 && cg == 2 ? 3 : 1))
                       : 0;
    if (pr.symmetric == 3 && mode != kEpiGram && mode != kEpiPoly && mode != kEpiSplit)
      return cudaErrorInvalidValue;
    if (d.symmetric && !pr.symmetric) return cudaErrorInvalidValue;
    if (pr.symmetric == 2 && mode != kEpiStat) return cudaErrorInvalidValue;  // upper-only: STAT
    pr.tiles_per_batch =
        pr.symmetric ? sym_tiles(pr.tiles_m, pr.tiles_n, P.tile_m) : pr.tiles_m * pr.tiles_n;
    pr.tile_start = tiles;
    tiles += pr.batch * pr.tiles_per_batch;
    pr.out = static_cast<__nv_bfloat16*>(const_cast<void*>(d.out.ptr));
    pr.out_ld = d.out.ld;
    pr.out_bstride = d.out.bstride;
    pr.aux = static_cast<const __nv_bfloat16*>(d.aux.ptr);
    pr.aux_ld = d.aux.ld;
    pr.aux_bstride = d.aux.bstride;
    pr.scale = d.scale;
    pr.final_targets = d.final_targets;
    if (mode == kEpiFinal && pr.final_targets == nullptr) return cudaErrorInvalidValue;
    if ((mode == kEpiPoly || mode == kEpiUpdate || mode == kEpiFinal) && pr.aux == nullptr &&
        alpha != 0.f)
      return cudaErrorInvalidValue;
    pr.out32 = nullptr;
    pr.out_seg = d.out_seg;
    if (mode == kEpiStat) {
      pr.out32 = static_cast<float*>(const_cast<void*>(d.out.ptr));
      pr.out = nullptr;
      if (pr.out32 == nullptr) return cudaErrorInvalidValue;
    } else if (mode != kEpiFinal && pr.out == nullptr) {
      return cudaErrorInvalidValue;
    }
    if (mode == kEpiSplit && d.out_seg < pr.N) return cudaErrorInvalidValue;
  }
  P.total_tiles = tiles;
  P.raster = raster_group(mode);
  bool stream_k = false;
  if (sched != nullptr && sched->tiles != nullptr && sched->total_tiles == tiles &&
      sched->units == std::min(tiles, cg == 2 ? sm_count() / 2 : sm_count())) {
    P.sched = sched->tiles;
    P.sched_off = sched->off;
    P.sched_units = sched->units;
    if (sched->kb != nullptr && mode == kEpiGram) {
      P.seg_kb = sched->kb;
      P.seg_slot = sched->slot;
      P.seg_ws = sched->ws;
      stream_k = sched->n_fix > 0;
    }
  }
  if (stream_k) {
    const cudaError_t e = cg == 2 ? launch_mode<kEpiGram, 2>(P, stream) : launch_mode<kEpiGram, 1>(P, stream);
    if (e != cudaSuccess) return e;
    stream_k_fixup_kernel<<<dim3(static_cast<unsigned>(sched->n_fix), 32), 256, 0, stream>>>(P, sched->fix);
    return cudaGetLastError();
  }
  if (cg == 2) {
    switch (mode) {
      case kEpiGram: return launch_mode<kEpiGram, 2>(P, stream);
      case kEpiPoly: return launch_mode<kEpiPoly, 2>(P, stream);
      case kEpiUpdate: return launch_mode<kEpiUpdate, 2>(P, stream);
      case kEpiFinal: return launch_mode<kEpiFinal, 2>(P, stream);
      case kEpiStat: return launch_mode<kEpiStat, 2>(P, stream);
      case kEpiSplit: return launch_mode<kEpiSplit, 2>(P, stream);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (mode) {
    case kEpiGram: return launch_mode<kEpiGram, 1>(P, stream);
    case kEpiPoly: return launch_mode<kEpiPoly, 1>(P, stream);
    case kEpiUpdate: return launch_mode<kEpiUpdate, 1>(P, stream);
    case kEpiFinal: return launch_mode<kEpiFinal, 1>(P, stream);
    case kEpiStat: return launch_mode<kEpiStat, 1>(P, stream);
    case kEpiSplit: return launch_mode<kEpiSplit, 1>(P, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace osh
