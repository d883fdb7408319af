// OptimizerEngine: what the per-rank runtime (runtime.cu) drives each step —
// the update of this rank's owned tensors in bucket-ordered WAVES — plus the
// CUDA-event profiling shared by the optimizers (MuonEngine, ShampooEngine).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ns_gemm.cuh"
#include "osh.h"

namespace osh {

struct MuonTensorDesc {
  int rows = 0, cols = 1;   // cols == 1 and !is_matrix for vectors
  int is_matrix = 0;
  int vocab_space = 0;      // Shampoo: vocabulary matrices take the momentum-SGD rule
  int bucket = 0;           // bucket index (declaration order)
  float* w = nullptr;       // fp32 master weight [rows][cols]
  float* m = nullptr;       // fp32 momentum
  const void* g = nullptr;  // reduced gradient (grad dtype of the engine)
  __nv_bfloat16* replica = nullptr;  // bf16 replica slot (nullable)
  int g_mc = 0;    // g is an NVLS multicast address (read the cross-GPU sum)
  int rep_mc = 0;  // replica is an NVLS multicast address (store to every GPU)
  __nv_bfloat16* replica_local = nullptr;  // rep_mc: this GPU's own copy of the slot
};

struct NsLaunchStats {
  int launches_gemm = 0;
  int launches_elementwise = 0;
  double gemm_flops = 0.0;  // algorithmic 2MNK of the launched GEMMs
};

// profile modes >= kModeElementwise are elementwise kernels (bytes in the
// flops column); GEMM modes are the kEpi* codes
constexpr int kModeElementwise = 8;

class OptimizerEngine {
 public:
  virtual ~OptimizerEngine();

  // tensors in declaration order; min_waves > 1 cuts the work into at least
  // that many waves when tensors allow; double_buffer: see MuonEngine.
  virtual osh_status build(const std::vector<MuonTensorDesc>& tensors, int grad_dtype,
                           size_t workspace_budget_bytes, int min_waves, bool double_buffer) = 0;
  virtual osh_status begin_step(cudaStream_t stream) = 0;  // clears norms / stats
  virtual osh_status run_wave(int w, const osh_muon_cfg& cfg, cudaStream_t stream) = 0;
  // Split phases for overlapped schedules (only when double_buffered()).
  virtual osh_status run_pre(int w, const osh_muon_cfg& cfg, cudaStream_t stream);
  virtual osh_status run_ns(int w, const osh_muon_cfg& cfg, cudaStream_t stream);
  virtual osh_status run_post(int w, const osh_muon_cfg& cfg, cudaStream_t stream);
  virtual bool double_buffered() const { return false; }

  virtual int num_waves() const = 0;
  virtual int wave_first_bucket(int w) const = 0;
  virtual int wave_last_bucket(int w) const = 0;
  virtual const double* update_sq() const = 0;  // ||lr * update||^2 per tensor (device)
  virtual size_t workspace_bytes() const = 0;
  virtual int num_tensors() const = 0;
  virtual void set_symmetric(bool) {}
  // Waves may run in any order (no bucket-ordered collective or host copy
  // depends on it): build() then puts small waves first and last, so the
  // exposed momentum of the first wave and update of the last are short.
  virtual void set_wave_reorder(bool) {}
  // Optimizer state beyond the per-tensor master / momentum (checkpointing):
  // a device buffer whose layout is a pure function of the tensors and the
  // configuration, plus the engine's step counter.
  virtual void* extra_state() { return nullptr; }
  virtual size_t extra_state_bytes() const { return 0; }
  virtual long long step_counter() const { return 0; }
  virtual void set_step_counter(long long) {}

  const NsLaunchStats& stats() const { return stats_; }  // since begin_step()
  // Engine tensor indices of wave w, in the order build() received them
  // (empty when the engine does not record them): lets a single-rank step
  // move host data wave by wave instead of bucket by bucket.
  const std::vector<int>& wave_tensors(int w) const {
    static const std::vector<int> kNone;
    return w >= 0 && w < static_cast<int>(wave_tensors_.size()) ? wave_tensors_[w] : kNone;
  }
  // Per-launch CUDA-event timing of every launch (roofline reporting); the
  // read_profile totals cover the GEMMs only, profile_text lists all launches.
  void set_profile(bool on) { profile_ = on; }
  void read_profile(int* launches, double* flops, double* exec_flops, double* ms, bool reset);
  // One line per recorded launch: "mode ms flops exec_flops shapes", plus
  // " @start" (ms after `ref`, a timing event recorded before the launches)
  // when ref is given.
  std::string profile_text(cudaEvent_t ref = nullptr) const;

 protected:
  struct Timed {
    cudaEvent_t a, b;
    double flops;
    double exec_flops;
    int mode;
    std::string what;
  };
  cudaEvent_t take_event();
  // one grouped GEMM launch, timed when profiling, counted in stats_
  cudaError_t timed_gemm(int mode, const NsProblemDesc* pd, int np, float alpha, float beta,
                         cudaStream_t s, const NsSchedule* sched = nullptr, float lr = 0.f);
  template <typename F>
  cudaError_t timed_elementwise(int mode, double bytes, double elems, cudaStream_t s, F&& launch) {
    const bool rec = profile_ && timed_.size() < 100000;
    Timed t{};
    if (rec) {
      t.a = take_event();
      t.b = take_event();
      t.flops = bytes;
      t.exec_flops = 0.0;
      t.mode = mode;
      t.what = std::to_string(static_cast<long long>(elems));
      cudaEventRecord(t.a, s);
    }
    const cudaError_t err = launch();
    if (rec) {
      cudaEventRecord(t.b, s);
      timed_.push_back(std::move(t));
    }
    ++stats_.launches_elementwise;
    return err;
  }
  // names of modes >= kModeElementwise for profile_text
  virtual const char* elementwise_name(int mode) const;

  NsLaunchStats stats_;
  std::vector<std::vector<int>> wave_tensors_;
  bool profile_ = false;
  std::vector<Timed> timed_;
  std::vector<cudaEvent_t> event_pool_;
};

}  // namespace osh
