// ShampooEngine: the builder-defined blocked Shampoo update of this rank's
// owned tensors (the reference only costs it, cost.hpp:47-48,
// 68-75). Specification and fp64 oracle: oracle/shampoo_oracle.py.
//
// Every 2-D non-vocabulary tensor is cut into blocks of <= cfg.block rows and
// columns; blocks of the same (p, q) within a wave form one batched GEMM
// problem. Per step and wave:
//   sh_prep              G_b, G_b^T (bf16) + ||G_b||^2 tile sums
//   STAT GEMMs           L = b2 L + G G^T, R = b2 R + G^T G          (fp32 state)
//   [refresh steps]      ||S||, A = S/||S|| + eps I, then newton_iters x
//                        { T = (5I - M)/4 ; X = X T, T2 = T T ; T4 = T2 T2 ;
//                          M = T4 M } as bf16x3 SPLIT GEMMs (fp32-accurate),
//                        P = hi(X) * ||S||^(-1/4)
//   UPDATE / GRAM GEMMs  U = (P_L G) P_R                              (bf16)
//   graft                s_b = ||G_b|| / ||U_b||
//   sh_apply / sh_sgd    M = b1 M + s_b U (or + g) ; W -= lr M ; replica
// Waves run back to back on one stream (no double buffering).
#pragma once

#include <vector>

#include "engine_base.cuh"
#include "shampoo_kernels.cuh"

namespace osh {

struct ShampooConfig {
  double beta2 = 0.95, eps = 1e-4;
  int block = 1024, precond_every = 10, newton_iters = 16;
};

class ShampooEngine : public OptimizerEngine {
 public:
  explicit ShampooEngine(const ShampooConfig& cfg) : cfg_(cfg) {}
  ~ShampooEngine() override;

  osh_status build(const std::vector<MuonTensorDesc>& tensors, int grad_dtype,
                   size_t workspace_budget_bytes, int min_waves, bool double_buffer) override;
  osh_status begin_step(cudaStream_t stream) override;
  osh_status run_wave(int w, const osh_muon_cfg& cfg, cudaStream_t stream) override;

  int num_waves() const override { return static_cast<int>(waves_.size()); }
  int wave_first_bucket(int w) const override { return waves_[w].first_bucket; }
  int wave_last_bucket(int w) const override { return waves_[w].last_bucket; }
  const double* update_sq() const override { return d_update_sq_; }
  size_t workspace_bytes() const override { return ws_bytes_; }
  int num_tensors() const override { return n_tensors_; }
  size_t state_bytes() const { return state_bytes_; }
  long long step_index() const { return step_; }
  void* extra_state() override { return d_state_; }
  size_t extra_state_bytes() const override { return state_bytes_; }
  long long step_counter() const override { return step_; }
  void set_step_counter(long long s) override { step_ = s; }

 private:
  struct Cls {                 // blocks of one (p, q) inside one wave
    int p = 0, q = 0, ldp = 0, ldq = 0, nb = 0, block0 = 0;
    size_t L = 0, R = 0, PL = 0, PR = 0;             // state offsets (bytes)
    size_t gb = 0, gbt = 0, u1 = 0, u = 0;           // workspace offsets (bytes)
    size_t xl[2] = {0, 0}, ml[2] = {0, 0}, tl = 0, t2l = 0, t4l = 0;  // split, [nb][p][4 seg]
    size_t xr[2] = {0, 0}, mr[2] = {0, 0}, tr = 0, t2r = 0, t4r = 0;  // split, [nb][q][4 seg]
    int stat0 = 0;             // first statistics-matrix index (L of block i = stat0 + i,
                               // R of block i = stat0 + nb + i)
  };
  struct Range {
    int first = 0, count = 0;
    long long tiles = 0;
  };
  struct Wave {
    int first_bucket = 0, last_bucket = 0;
    std::vector<Cls> cls;
    Range prep, usq, ssq, apply, sgd;     // task ranges (tiles = sum over the range)
    Range symf;                           // L / R lower-triangle fills (refresh steps)
    Range root_init[1], newton[2], extract[1];
    Range slot_g, slot_u, slot_s, slot_t; // partial-sum slot ranges
    int n_blocks = 0, n_stats = 0;
    double elems_pre = 0.0, elems_sgd = 0.0;
  };
  const char* elementwise_name(int mode) const override;
  void release();

  ShampooConfig cfg_;
  int n_tensors_ = 0, grad_dtype_ = 0;
  long long step_ = -1;
  std::vector<Wave> waves_;
  size_t ws_bytes_ = 0, state_bytes_ = 0;
  uint8_t* d_ws_ = nullptr;
  uint8_t* d_state_ = nullptr;
  double* d_partial_ = nullptr;  // all tile partials (absolute indices, disjoint per use)
  double* d_gsq_ = nullptr;      // per block
  double* d_usq_ = nullptr;      // per block
  double* d_ssq_ = nullptr;      // per statistics matrix
  float* d_sroot_ = nullptr;     // per statistics matrix: ||S||^(-1/4) (inside d_state_)
  float* d_graft_ = nullptr;     // per block
  double* d_update_sq_ = nullptr;
  ShPrepTask* d_prep_ = nullptr;
  ShMatTask<__nv_bfloat16>* d_usq_tasks_ = nullptr;
  ShMatTask<float>* d_ssq_tasks_ = nullptr;
  ShRootTask* d_root_ = nullptr;
  ShNewtonTask* d_newton_ = nullptr;   // [2 x stats]: from M0 and from M1
  ShNewtonTask* d_extract_ = nullptr;
  ShApplyTask* d_apply_ = nullptr;
  ShSgdTask* d_sgd_ = nullptr;
  ShBlockRef* d_blockrefs_ = nullptr;
  SymFillTask* d_symf_ = nullptr;
  long long* d_slot_begin_ = nullptr;
  int* d_slot_count_ = nullptr;
  int* d_slot_target_ = nullptr;
  int n_stats_total_ = 0;
};

}  // namespace osh
