// MuonEngine: the per-rank Muon update of a fixed set of owned tensors.
//
// Built once per layout (the plan never changes between steps): matrices are
// grouped into shape classes (m = min side, n = max side), classes are cut
// into chunks that fit the Newton-Schulz workspace budget, and chunks are
// packed up to kMaxProblems per "wave". A step is then, per wave:
//   momentum_matrix (m = beta*m + g, ||m||^2, X0 = bf16 m)  -> ns_scales ->
//   k x { GRAM, POLY, UPDATE }  with the last UPDATE fused into the weight
//   update (FINAL: W -= lr*X_k, bf16 replica, ||dW||^2)
// plus one momentum_vector launch for every 1-D tensor. All task tables live
// in device memory and are reused every step (no host work on the hot path
// beyond the launches themselves).
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
  float* w = nullptr;       // fp32 master weight [rows][cols]
  float* m = nullptr;       // fp32 momentum
  const void* g = nullptr;  // reduced gradient (grad dtype of the engine)
  __nv_bfloat16* replica = nullptr;  // bf16 replica slot (nullable)
};

struct NsLaunchStats {
  int launches_gemm = 0;
  int launches_elementwise = 0;
  double gemm_flops = 0.0;      // algorithmic 2MNK of the launched GEMMs
  double elementwise_bytes = 0.0;
};

class MuonEngine {
 public:
  MuonEngine() = default;
  ~MuonEngine();
  MuonEngine(const MuonEngine&) = delete;
  MuonEngine& operator=(const MuonEngine&) = delete;

  // Plans classes / chunks / waves and allocates device tables + workspace.
  osh_status build(const std::vector<MuonTensorDesc>& tensors, int grad_dtype,
                   size_t workspace_budget_bytes);
  // One Muon update of every tensor on `stream`.
  osh_status run(const osh_muon_cfg& cfg, cudaStream_t stream);

  // ||lr * update||^2 of tensor i from the last run (device array).
  const double* update_sq() const { return d_update_sq_; }
  size_t workspace_bytes() const { return ws_bytes_; }
  const NsLaunchStats& stats() const { return stats_; }  // per run()
  int num_waves() const { return static_cast<int>(waves_.size()); }
  // Per-launch CUDA-event timing of the GEMMs (roofline reporting).
  void set_profile(bool on) { profile_ = on; }
  // Sums the recorded launches (host-synchronises on the events).
  void read_profile(int* launches, double* flops, double* exec_flops, double* ms, bool reset);
  // One line per recorded launch: "mode ms flops exec_flops shapes".
  std::string profile_text() const;
  // Symmetric GRAM / POLY tiles (default on; off reproduces the full GEMMs).
  void set_symmetric(bool on) { symmetric_ = on; }
  int num_tensors() const { return n_tensors_; }

 private:
  struct Chunk {
    int m = 0, n = 0, ldm = 0, ldn = 0, batch = 0;
    int slot0 = 0;  // first matrix slot (slots are chunk-contiguous)
    size_t x0 = 0, x1 = 0, a = 0, b = 0;  // byte offsets in the workspace
  };
  struct Wave {
    std::vector<int> chunks;
    int task0 = 0, n_tasks = 0;  // momentum_matrix tasks
    long long tiles = 0;
  };
  void release();

  int n_tensors_ = 0;
  int grad_dtype_ = kGradF32;
  std::vector<Chunk> chunks_;
  std::vector<Wave> waves_;
  int n_slots_ = 0;
  int n_vec_tasks_ = 0;
  size_t ws_bytes_ = 0;
  uint8_t* d_ws_ = nullptr;
  double* d_partial_ = nullptr;      // per momentum tile of the largest wave
  long long* d_slot_begin_ = nullptr;  // per slot: first partial (wave-relative)
  int* d_slot_count_ = nullptr;        // per slot: number of partials
  float* d_scale_update_ = nullptr;  // per slot
  float* d_scale_gram_ = nullptr;    // per slot
  double* d_update_sq_ = nullptr;    // per tensor
  MomentumMatrixTask* d_mtasks_ = nullptr;
  MomentumVectorTask* d_vtasks_ = nullptr;
  NsFinalTarget* d_final_ = nullptr;  // per slot
  NsLaunchStats stats_;
  bool profile_ = false;
  bool symmetric_ = true;
  struct Timed {
    cudaEvent_t a, b;
    double flops;
    double exec_flops;
    int mode;
    std::string what;  // e.g. "2x4096x12288+36x4096x4096"
  };
  std::vector<Timed> timed_;   // recorded since the last reset
  std::vector<cudaEvent_t> event_pool_;
  cudaEvent_t take_event();
};

}  // namespace osh
