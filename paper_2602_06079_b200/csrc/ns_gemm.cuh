// Batched, grouped tcgen05 GEMM for the Muon Newton-Schulz iteration.
//
// One Newton-Schulz step on X (m x n, m <= n, row-major bf16) is three
// contractions (reference verify.hpp:126-131):
//   GRAM   A  = s^2 * (X X^T)                 m x m, K = n, both operands K-major
//   POLY   B  = b*A + c*(A A^T)  (A = A^T)     m x m, K = m, both operands K-major
//   UPDATE X' = s*(a*X + B X)                  m x n, K = m, X read MN-major
//   FINAL  W -= lr * s*(a*X + B X)             last step: fused weight update
// s is a per-matrix scale (1/||M||_F on the first step, where the iterate is
// the raw momentum cast to bf16; 1 afterwards). The reference evaluates
// b*(A X) + c*(A (A X)); B = b*A + c*A*A is the same polynomial with
// 4m^2n + 2m^3 instead of 6m^2n flops per step.
//
// Up to kMaxProblems independent problems (shape classes) share one
// persistent launch; every problem is batched over same-shape matrices laid
// out as [batch][rows][ld] so a single 3-D TMA descriptor covers the class.
#pragma once

#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace osh {

constexpr int kNsBM = 128;       // UMMA M (one CTA, cta_group::1)
constexpr int kNsBN = 256;       // UMMA N
constexpr int kNsBK = 64;        // one 128-byte swizzle row of bf16
constexpr int kNsStages = 4;
constexpr int kNsThreads = 256;  // warps 0-3: TMA / MMA / TMEM alloc / spare, 4-7: epilogue
constexpr int kMaxProblems = 4;

enum NsEpilogue : int {
  kEpiGram = 0,    // out = s * acc                                  (bf16)
  kEpiPoly = 1,    // out = alpha * aux + beta * acc + lr * I         (bf16)
  kEpiUpdate = 2,  // out = s * (alpha * aux + acc)                  (bf16)
  kEpiFinal = 3,   // W -= lr * s * (alpha * aux + acc)              (fp32 master + replica)
  kEpiStat = 4,    // out32 = alpha * out32 + s * acc                (fp32 read-modify-write)
  kEpiSplit = 5,   // v = s * acc as bf16 hi/lo pairs in 4 segments of out_seg columns:
                   //   [hi | lo | hi | hi]; columns [0,3n) = (hi, lo, hi) are the A-operand view
                   //   and [n,4n) = (lo, hi, hi) the B-operand view of a bf16x3 product
                   //   (hi*lo + lo*hi + hi*hi)
};

// Where the last Newton-Schulz step of one matrix lands (kEpiFinal): the fp32
// master weight and its bf16 replica in the tensor's ORIGINAL orientation.
// The epilogue streams W through shared memory in 32 x 32 boxes (cp.async,
// prefetched while the tile's MMAs run) and writes W and the replica in
// 128 / 64-byte row segments, so the weight update costs one read and one
// write of W and one replica write — no separate streaming pass.
struct NsFinalTarget {
  float* w;                // fp32 W: not transposed [M][N], transposed [N][M]
  __nv_bfloat16* replica;  // bf16 replica, same geometry (nullable)
  double* partial;         // per (tile, CTA of the pair, epilogue warp): sum of (lr*update)^2
  int transposed;          // 1: the tensor is X^T (rows > cols in the reference)
  int pad_;
};

// One target for an M x N iterate (M <= N). W and the replica must be
// 16-byte aligned and their row pitch a multiple of 16 bytes
// (final_target_ok). `partial` needs final_partials(M, N) doubles.
bool final_target_ok(const void* w, const void* replica, int M, int N, int transposed);
bool make_final_target(NsFinalTarget* t, float* w, __nv_bfloat16* replica, int M, int N,
                       int transposed, double* partial);
int final_partials(int M, int N);  // tiles * CTAs per tile * 4 epilogue warps

struct alignas(64) NsGemmProblem {
  CUtensorMap tmA;  // [batch][M][K], K-major, box {64, 128, 1}
  CUtensorMap tmB;  // K-major: [batch][N][K] box {64, 256, 1}; MN-major: [batch][K][N] box {64, 64, 1}
  CUtensorMap tmA2;  // a_upper: the same square matrix as MN-major [batch][K][M] boxes {64, 64, 1}
  CUtensorMap tmB2;  // b_upper: likewise for B
  int batch, M, N, K;
  int b_mn_major;
  int a_upper, b_upper;  // operands in the upper-tile form (NsProblemDesc)
  int k_seg, a_seg0, b_seg0;  // K segments of the upper-form views (k_seg = K: one)
  int symmetric;      // output is symmetric (M == N): only tiles touching the
                      // upper triangle run; 1: the epilogue mirrors them,
                      // 2 (STAT): it writes the upper triangle only
  int tiles_m, tiles_n;
  int tiles_per_batch;
  int tile_start;
  __nv_bfloat16* out;
  long long out_ld, out_bstride;
  const __nv_bfloat16* aux;
  long long aux_ld, aux_bstride;
  const float* scale;                 // per-batch multiplier, nullable (= 1)
  const NsFinalTarget* final_targets; // per batch, kEpiFinal only
  float* out32;                       // kEpiStat: fp32 output (ld / bstride as out)
  long long out_seg;                  // kEpiSplit: segment width in elements
};

struct NsGemmParams {
  NsGemmProblem prob[kMaxProblems];
  int num_problems;
  int total_tiles;
  const int* sched;      // optional: tiles of unit u are sched[sched_off[u] .. sched_off[u+1])
  const int* sched_off;
  int sched_units;       // units (clusters / CTAs) the schedule was built for
  int raster;            // tile rows per raster group (non-symmetric problems)
  // stream-K (kEpiGram only, with a schedule): entry i covers k-blocks
  // [seg_kb[i].x, seg_kb[i].y) of its tile; seg_slot[i] >= 0 means a PART of
  // the tile, whose raw fp32 accumulator goes to seg_ws slot seg_slot[i]
  // ([256 rows][256 cols] per slot) for the fixup pass to sum in slot order
  const int2* seg_kb;
  const int* seg_slot;
  float* seg_ws;
  int tile_m;  // output rows per tile: 128 (cta_group::1) or 256 (cta_group::2)
  float alpha, beta, lr;
};

// Host-side description of one batched operand: batch x rows x cols bf16,
// row stride `ld` elements, batch stride `bstride` elements.
struct NsMatrixRef {
  const void* ptr;
  int batch, rows, cols;
  long long ld, bstride;
};

struct NsProblemDesc {
  NsMatrixRef a;        // M x K
  NsMatrixRef b;        // K-major: N x K ; MN-major: K x N
  int b_mn_major;
  NsMatrixRef out;      // M x N (bf16), unused for kEpiFinal
  NsMatrixRef aux;      // M x N (bf16) or nullptr
  const float* scale;   // device, per batch
  const NsFinalTarget* final_targets;  // device, per batch
  int symmetric = 0;    // GRAM / POLY / STAT / SPLIT: out = out^T, upper-triangle tiles only;
                        // 1: the epilogue mirrors them, 2 (STAT): upper triangle written
                        // only — launch_sym_fill_lower completes the matrix before a reader
  long long out_seg = 0;  // kEpiSplit segment width (elements)
  // Upper-tile form (2-CTA tiles only; 1-CTA launches fall back to the full
  // mirror): symmetric = 3 (GRAM / POLY) writes the 256 x 256 tiles on and
  // above the diagonal — diagonal tiles whole — and skips the mirror of the
  // others; an operand flagged a_upper / b_upper is such a matrix, its
  // k-blocks left of the diagonal are loaded from the mirrored upper tile
  // through an MN-major view (same values, no lower half needed).
  int a_upper = 0;
  int b_upper = 0;
  // K in segments (kEpiSplit views): the operand rows hold consecutive
  // segments of k_seg columns, each segment one symmetric matrix; the A / B
  // view starts at stored segment a_seg0 / b_seg0 of that buffer. k_seg 0:
  // one segment (K).
  int k_seg = 0;
  int a_seg0 = 0, b_seg0 = 0;
};

// A cost-balanced static tile schedule for one grouped launch (device arrays).
// Stream-K schedules (kEpiGram) also carry per-entry k-block ranges and
// partial slots, the fixup table of the split tiles (6 ints each: problem,
// batch, tile row, tile col, first slot, slot count) and the fp32 partial
// workspace (n_slots x 256 x 256).
struct NsSchedule {
  const int* tiles = nullptr;
  const int* off = nullptr;
  int units = 0;
  int total_tiles = 0;
  const int2* kb = nullptr;
  const int* slot = nullptr;
  const int* fix = nullptr;
  int n_fix = 0;
  int n_slots = 0;
  float* ws = nullptr;
};

// Launches one grouped GEMM. Returns a cudaError_t (cudaSuccess on success).
// `sched` (optional) must come from ns_gemm_schedule for the same problem
// shapes; it is ignored if the grid or tile count does not match.
cudaError_t ns_gemm_launch(int mode, const NsProblemDesc* probs, int num_problems, float alpha,
                           float beta, float lr, cudaStream_t stream,
                           const NsSchedule* sched = nullptr);

// Host-side LPT schedule of a grouped launch: every tile costs its problem's
// K-block count; tiles are taken heaviest first and given to the least-loaded
// unit (ties: lowest unit), so long-K problems (vocabulary Grams) do not form
// a tail. Fills per-unit tile lists; returns the unit count (0 on error).
int ns_gemm_schedule(int mode, const NsProblemDesc* probs, int num_problems,
                     std::vector<int>* tiles, std::vector<int>* off, int* total_tiles);

// Stream-K schedule of a GRAM launch with few, long-K tiles: the launch's
// k-blocks (tile by tile, in linear tile order) are cut into one contiguous
// range per unit, so every unit gets the same MMA work and no tile round is
// left half empty. Tiles cut across units are finished by a fixup pass that
// sums their parts in a fixed order (deterministic). Returns the unit count,
// or 0 when stream-K would not shorten the launch (enough tiles already).
int ns_gemm_stream_k_schedule(const NsProblemDesc* probs, int num_problems,
                              std::vector<int>* tiles, std::vector<int>* off,
                              std::vector<int2>* kb, std::vector<int>* slot,
                              std::vector<int>* fix, int* n_slots, int* total_tiles);

// UMMA CTA group used by subsequent launches: 2 (default; CTA pairs, 256x256
// tiles) or 1 (single-CTA 128x256 tiles). OSH_GEMM_CTA_GROUP=1 overrides.
void ns_gemm_set_cta_group(int cg);
int ns_gemm_cta_group();

// Algorithmic flops of a problem list (2*M*N*K per batch element).
double ns_gemm_flops(const NsProblemDesc* probs, int num_problems);
// Flops the tensor cores actually execute (symmetric problems skip the tiles
// strictly below the diagonal).
double ns_gemm_executed_flops(const NsProblemDesc* probs, int num_problems);

}  // namespace osh
