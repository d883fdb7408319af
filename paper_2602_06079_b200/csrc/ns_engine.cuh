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
//   sums of m^2, X0 = bf16 m) -> ns_scales -> (k-1) x {GRAM, POLY, UPDATE}
//   -> GRAM, POLY, FINAL (W -= lr*X_k straight from the accumulator: W and
//   the bf16 replica move by TMA in the GEMM epilogue, per-tile |dW|^2)
//   -> partial_sums (||dW||^2 per tensor, fixed order)
// A wave whose tensors TMA cannot address (row pitch not a multiple of 16
// bytes, NVLS multicast replica) ends with UPDATE -> apply_update instead
// (OSH_FUSE_FINAL=0 forces that path everywhere).
// All task tables live in device memory and are reused every step.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "engine_base.cuh"
#include "muon_kernels.cuh"
#include "ns_gemm.cuh"
#include "osh.h"

namespace osh {

class MuonEngine : public OptimizerEngine {
 public:
  MuonEngine() = default;
  ~MuonEngine() override;
  MuonEngine(const MuonEngine&) = delete;
  MuonEngine& operator=(const MuonEngine&) = delete;

  // tensors must be in declaration order. min_waves > 1 cuts the work into at
  // least that many waves (finer RS/AG overlap) when tensors allow.
  // double_buffer: alternate waves between two workspace halves so run_pre of
  // wave w+1 may overlap run_ns of wave w on another stream.
  osh_status build(const std::vector<MuonTensorDesc>& tensors, int grad_dtype,
                   size_t workspace_budget_bytes, int min_waves, bool double_buffer) override;
  osh_status begin_step(cudaStream_t stream) override;  // clears the update norms / stats
  osh_status run_wave(int w, const osh_muon_cfg& cfg, cudaStream_t stream) override;  // pre+ns+post
  // The three phases of a wave. Ordering contract for overlapped schedules:
  // run_pre(w) -> run_ns(w) -> run_post(w); run_pre / run_post of all waves on
  // ONE stream in the order pre(0) pre(1) post(0) pre(2) post(1) ... (they
  // share the tile-partial buffer); run_ns(w+1) may overlap run_post(w) and,
  // with double buffering, run_pre(w+2) may not start before run_post(w).
  osh_status run_pre(int w, const osh_muon_cfg& cfg, cudaStream_t stream) override;   // momentum + scales
  osh_status run_ns(int w, const osh_muon_cfg& cfg, cudaStream_t stream) override;    // k x GRAM/POLY/UPDATE
  osh_status run_post(int w, const osh_muon_cfg& cfg, cudaStream_t stream) override;  // apply + norms
  bool double_buffered() const override { return double_buffer_; }

  int num_waves() const override { return static_cast<int>(waves_.size()); }
  int wave_first_bucket(int w) const override { return waves_[w].first_bucket; }
  int wave_last_bucket(int w) const override { return waves_[w].last_bucket; }

  // ||lr * update||^2 of tensor i from the last step (device array).
  const double* update_sq() const override { return d_update_sq_; }
  size_t workspace_bytes() const override { return ws_bytes_; }
  int num_tensors() const override { return n_tensors_; }

  void set_symmetric(bool on) override { symmetric_ = on; }
  void set_wave_reorder(bool on) override { reorder_ = on; }

 private:
  struct Chunk {
    int m = 0, n = 0, ldm = 0, ldn = 0, batch = 0;
    int slot0 = 0;                        // first matrix slot (chunk-contiguous)
    size_t x0 = 0, x1 = 0, a = 0, b = 0;  // byte offsets in the workspace
    int ftarget0 = -1;                    // fused waves: first NsFinalTarget of the batch
  };
  struct Wave {
    std::vector<int> chunks;
    int first_bucket = 0, last_bucket = 0;
    int task0 = 0, n_tasks = 0;  // momentum / apply tasks (same geometry)
    long long tiles = 0;
    int slot0 = 0, n_slots = 0;
    int vec0 = 0, n_vec = 0;
    double elems_matrix = 0.0, elems_vector = 0.0;  // owned elements (profile bytes)
    NsSchedule sched[4];  // per GEMM mode (kEpiGram / kEpiPoly / kEpiUpdate / kEpiFinal)
    // FINAL fusion (per tensor): the unfused chunks come first, so their
    // momentum / apply tasks, tiles and slots are a prefix of the wave's
    int nf_chunks = 0, nf_tasks = 0, nf_slots = 0;
    long long nf_tiles = 0;
    double nf_elems = 0.0;
    int fslot0 = 0;                  // first row of the fused partial-sum tables
    int mc0 = 0, n_mc = 0;           // NVLS: multicast re-store tasks of fused tensors
    long long mc_vecs = 0;
    NsSchedule sched_last_update;    // last iteration: UPDATE over the unfused prefix
  };
  void release();
  const char* elementwise_name(int mode) const override;
  void problems(const Wave& w, int it, NsProblemDesc* gram, NsProblemDesc* poly,
                NsProblemDesc* upd) const;

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
  // fused FINAL: per matrix slot a TMA target + its epilogue partials
  NsFinalTarget* d_ftargets_ = nullptr;
  McCopyTask* d_mctasks_ = nullptr;
  double* d_fpartial_ = nullptr;
  size_t fpartial_count_ = 0;
  long long* d_fslot_begin_ = nullptr;
  int* d_fslot_count_ = nullptr;
  int* d_fslot_tensor_ = nullptr;
  bool fuse_final_ = true;        // OSH_FUSE_FINAL=0: UPDATE + apply_update everywhere
  bool stream_k_ = false;         // OSH_STREAM_K=1: tail-split GRAM for few long-K tiles
  float* d_sk_ws_ = nullptr;      // stream-K partial tiles (fp32, 256 x 256 per slot)
  bool symmetric_ = true;
  bool upper_form_ = false;  // POLY output in the upper-tile form (ns_gemm.cuh; OSH_UPPER_FORM=1)
  bool double_buffer_ = false;
  bool reorder_ = false;          // small waves first and last (set_wave_reorder)
  bool lpt_ = true;               // cost-balanced tile schedules (OSH_GEMM_LPT=0: striding)
  bool fold_a_ = true;            // a*I folded into B (OSH_NS_AUX=1: aux read in UPDATE)
  bool sched_symmetric_ = true;   // symmetric_ when the schedules were built
  std::vector<int*> sched_mem_;
};

}  // namespace osh
