// MuonEngine: the per-rank Muon update of a fixed set of owned tensors.
//
// Built once per layout (the plan never changes between steps). Owned tensors
// are taken in declaration order (= bucket order) and cut into WAVES that fit
// the Newton-Schulz workspace; inside a wave, matrices of the same shape
// class (m = min side, n = max side) form one batched problem of a grouped
// GEMM launch (<= kMaxProblems classes per wave). Because waves follow bucket
// order, the runtime can start a wave as soon as the reduce-scatter of its
// last bucket has landed and all-gather a bucket as soon as the wave that
// finishes it is done (runtime.cu). One wave of a step is:
//   momentum_vector (1-D tensors) ; momentum_matrix (m = beta*m + g, tile
//   sums of m^2, X0 = bf16 m) -> ns_scales -> k x {GRAM, POLY, UPDATE}
//   -> apply_update (W -= lr*X_k, bf16 replica, tile sums of |dW|^2)
//   -> partial_sums (||dW||^2 per tensor, fixed order)
// All task tables live in device memory and are reused every step.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "muon_kernels.cuh"
#include "ns_gemm.cuh"
#include "osh.h"

namespace osh {

struct MuonTensorDesc {
  int rows = 0, cols = 1;   // cols == 1 and !is_matrix for vectors
  int is_matrix = 0;
  int bucket = 0;           // bucket index (declaration order)
  float* w = nullptr;       // fp32 master weight [rows][cols]
  float* m = nullptr;       // fp32 momentum
  const void* g = nullptr;  // reduced gradient (grad dtype of the engine)
  __nv_bfloat16* replica = nullptr;  // bf16 replica slot (nullable)
  int g_mc = 0;    // g is an NVLS multicast address (read the cross-GPU sum)
  int rep_mc = 0;  // replica is an NVLS multicast address (store to every GPU)
};

// profile modes >= kModeElementwise: momentum_vector, momentum_matrix,
// ns_scales, apply_update, partial_sums (GEMM modes are the OSH_EPI_* codes)
constexpr int kModeElementwise = 8;

struct NsLaunchStats {
  int launches_gemm = 0;
  int launches_elementwise = 0;
  double gemm_flops = 0.0;  // algorithmic 2MNK of the launched GEMMs
};

class MuonEngine {
 public:
  MuonEngine() = default;
  ~MuonEngine();
  MuonEngine(const MuonEngine&) = delete;
  MuonEngine& operator=(const MuonEngine&) = delete;

  // tensors must be in declaration order. min_waves > 1 cuts the work into at
  // least that many waves (finer RS/AG overlap) when tensors allow.
  // double_buffer: alternate waves between two workspace halves so run_pre of
  // wave w+1 may overlap run_ns of wave w on another stream.
  osh_status build(const std::vector<MuonTensorDesc>& tensors, int grad_dtype,
                   size_t workspace_budget_bytes, int min_waves, bool double_buffer = false);
  osh_status begin_step(cudaStream_t stream);  // clears the update norms / stats
  osh_status run_wave(int w, const osh_muon_cfg& cfg, cudaStream_t stream);  // pre+ns+post
  // The three phases of a wave. Ordering contract for overlapped schedules:
  // run_pre(w) -> run_ns(w) -> run_post(w); run_pre / run_post of all waves on
  // ONE stream in the order pre(0) pre(1) post(0) pre(2) post(1) ... (they
  // share the tile-partial buffer); run_ns(w+1) may overlap run_post(w) and,
  // with double buffering, run_pre(w+2) may not start before run_post(w).
  osh_status run_pre(int w, const osh_muon_cfg& cfg, cudaStream_t stream);   // momentum + scales
  osh_status run_ns(int w, const osh_muon_cfg& cfg, cudaStream_t stream);    // k x GRAM/POLY/UPDATE
  osh_status run_post(int w, const osh_muon_cfg& cfg, cudaStream_t stream);  // apply + norms
  bool double_buffered() const { return double_buffer_; }

  int num_waves() const { return static_cast<int>(waves_.size()); }
  int wave_first_bucket(int w) const { return waves_[w].first_bucket; }
  int wave_last_bucket(int w) const { return waves_[w].last_bucket; }

  // ||lr * update||^2 of tensor i from the last step (device array).
  const double* update_sq() const { return d_update_sq_; }
  size_t workspace_bytes() const { return ws_bytes_; }
  const NsLaunchStats& stats() const { return stats_; }  // since begin_step()
  int num_tensors() const { return n_tensors_; }

  // Per-launch CUDA-event timing of every launch (roofline reporting); the
  // read_profile totals cover the GEMMs only, profile_text lists all launches
  // (elementwise kernels report algorithmic bytes in the flops column).
  void set_profile(bool on) { profile_ = on; }
  void read_profile(int* launches, double* flops, double* exec_flops, double* ms, bool reset);
  // One line per recorded launch: "mode ms flops exec_flops shapes".
  std::string profile_text() const;
  // Symmetric GRAM / POLY tiles (default on; off reproduces the full GEMMs).
  void set_symmetric(bool on) { symmetric_ = on; }

 private:
  struct Chunk {
    int m = 0, n = 0, ldm = 0, ldn = 0, batch = 0;
    int slot0 = 0;                        // first matrix slot (chunk-contiguous)
    size_t x0 = 0, x1 = 0, a = 0, b = 0;  // byte offsets in the workspace
  };
  struct Wave {
    std::vector<int> chunks;
    int first_bucket = 0, last_bucket = 0;
    int task0 = 0, n_tasks = 0;  // momentum / apply tasks (same geometry)
    long long tiles = 0;
    int slot0 = 0, n_slots = 0;
    int vec0 = 0, n_vec = 0;
    double elems_matrix = 0.0, elems_vector = 0.0;  // owned elements (profile bytes)
  };
  struct Timed {
    cudaEvent_t a, b;
    double flops;
    double exec_flops;
    int mode;
    std::string what;  // e.g. "54x4096x4096x12288+2x4096x4096x151936"
  };
  void release();
  cudaEvent_t take_event();
  template <typename F>
  cudaError_t timed_elementwise(int mode, double bytes, double elems, cudaStream_t s, F&& launch);

  int n_tensors_ = 0;
  int grad_dtype_ = kGradF32;
  std::vector<Chunk> chunks_;
  std::vector<Wave> waves_;
  int n_slots_ = 0;
  size_t ws_bytes_ = 0;
  uint8_t* d_ws_ = nullptr;
  double* d_partial_ = nullptr;        // per momentum / apply tile of the largest wave
  long long* d_slot_begin_ = nullptr;  // per slot: first tile (wave-relative)
  int* d_slot_count_ = nullptr;        // per slot: tiles
  int* d_slot_tensor_ = nullptr;       // per slot: tensor index
  float* d_scale_update_ = nullptr;    // per slot
  float* d_scale_gram_ = nullptr;      // per slot
  double* d_update_sq_ = nullptr;      // per tensor
  MomentumMatrixTask* d_mtasks_ = nullptr;
  ApplyTask* d_atasks_ = nullptr;
  MomentumVectorTask* d_vtasks_ = nullptr;
  NsLaunchStats stats_;
  bool profile_ = false;
  bool symmetric_ = true;
  bool double_buffer_ = false;
  std::vector<Timed> timed_;
  std::vector<cudaEvent_t> event_pool_;
};

}  // namespace osh
