// SoapEngine: the builder-defined blocked SOAP update of this rank's owned
// tensors (the reference only costs it, cost.hpp:47-48,
// 68-75). Specification and fp64 oracle: oracle/soap_oracle.py.
//
// Every 2-D non-vocabulary tensor is cut into blocks of <= cfg.block rows and
// columns; blocks of the same (p, q) within a wave form one batched GEMM
// problem. The first call only accumulates the statistics and computes the
// initial basis; every later call, per wave:
//   soap_prep            M = b1 M + (1-b1) g ; bf16x3 splits of G, G^T, M
//   SPLIT GEMMs          T1 = Q_L^T G, T2 = Q_L^T M      (bf16x3: fp32-accurate)
//   STAT GEMMs (a = 0)   G' = T1 Q_R, M' = T2 Q_R        (bf16x3 operands, fp32 out)
//   soap_rot             V = b2 V + (1-b2) G'^2 ; N' = M'/bc1 / (sqrt(V/bc2) + eps)
//   GRAM GEMMs           T3 = Q_L N', N = T3 Q_R^T                      (bf16)
//   soap_apply           W -= lr N ; replica ; ||lr N||^2
//   STAT GEMMs           L = bs L + (1-bs) G G^T, R = bs R + (1-bs) G^T G
//                        (bf16x3 operands, fp32 state)
// The rotated Adam ratio M'/sqrt(V) and the basis (a power iteration on the
// statistics) amplify operand rounding, so every product feeding them runs in
// bf16x3 (measured: bf16 operands there move the update 25-45 % away from the
// fp64 specification, bf16x3 ~1e-3); the back-projection N stays bf16.
//   [refresh calls]      per side, in sub-batches: bf16x6 splits of S and Q,
//                        Y = S Q (STAT, bf16x6), soap_basis (shift, order,
//                        unit columns), CholeskyQR2 = 2 x {Gram Q^T Q (STAT,
//                        bf16x6), soap_chol_inv (Cholesky + L^-1, one CTA per
//                        matrix), Q <- L^-1-applied Q (STAT, bf16x6)},
//                        V reordered, bf16 / bf16x3 copies of Q
//   soap_adam            vectors and vocabulary matrices: elementwise Adam
// Waves run back to back on one stream.
#pragma once

#include <vector>

#include "engine_base.cuh"
#include "soap_kernels.cuh"

namespace osh {

struct SoapConfig {
  double beta2 = 0.95;  // second moment and statistics decay (shampoo_beta = beta2)
  double eps = 1e-8;
  int block = 1024, precond_every = 10, init_iters = 4;
  float shift = 1e-3f;  // power-iteration shift, relative to ||S||_F
};

class SoapEngine : public OptimizerEngine {
 public:
  explicit SoapEngine(const SoapConfig& cfg) : cfg_(cfg) {}
  ~SoapEngine() override;

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
  void* extra_state() override { return d_state_; }
  size_t extra_state_bytes() const override { return state_bytes_; }
  long long step_counter() const override { return step_; }
  void set_step_counter(long long s) override { step_ = s; }

 private:
  struct RChunk {                  // refresh sub-batch: matrices [i0, i0 + b) of a side
    int i0 = 0, b = 0;
    int split_s = 0, split_q = 0, split_l = 0, chol = 0;  // first task of each kind
    long long tiles_s = 0, tiles_q = 0, tiles_l = 0;
  };
  struct Side {                    // one side (L or R) of a class: nb matrices of n x n
    int n = 0, ld = 0;
    bool frozen = false;           // elongated block: this side keeps Q = I (soap_oracle.frozen)
    size_t S = 0, Q = 0;           // state: statistics [n][ld] fp32, basis column-major fp32
    int order0 = 0;                // first order entry (d_order_)
    int basis0 = 0;                // first soap_basis task
    // refresh workspace (d_rws_), by kind for rb matrices (bf16x6 layouts,
    // soap_kernels.cuh): S (B), Q (A and B) and L^-1 (A) column layouts
    // [rb][n][6 ld], Q row B layout [rb][6 ld][ld], Y / Gram and L^-1 fp32
    // [rb][ld][ld]
    int rb = 1;
    size_t Sb = 0, Qa = 0, Qb = 0, La = 0, Qrb = 0, Y = 0, C = 0, Li = 0;
    std::vector<RChunk> chunks;
  };
  struct Cls {                     // blocks of one (p, q) inside one wave
    int p = 0, q = 0, ldp = 0, ldq = 0, nb = 0;
    Side l, r;
    // state: Q_L^T column-split [p][4 ldp], Q_L row-major [p][ldp],
    // Q_R row-split [4 ldq][ldq] (bf16x3 layouts, soap_kernels.cuh), V [p][ldq]
    size_t QLts = 0, QLb = 0, QRrs = 0, V = 0;
    // workspace: G column / G^T column / G row / M row splits, T1 / T2
    // column splits [p][4 ldq], G' M' fp32, N' T3 N bf16 [p][ldq]
    size_t Gs = 0, Gts = 0, Grs = 0, Mrs = 0, T1s = 0, T2s = 0, Gp = 0, Mp = 0;
    size_t Nr = 0, T3 = 0, Nb = 0;
    int rot = 0;                   // soap_rot task index
  };
  struct Range {
    int first = 0, count = 0;
    long long tiles = 0;
  };
  struct Wave {
    int first_bucket = 0, last_bucket = 0;
    std::vector<Cls> cls;
    Range prep, rot, apply, adam, basis, vperm, qcast, slots;
    Range symf;  // L / R lower-triangle fills before a refresh reads them
    double elems_pre = 0.0, elems_adam = 0.0;
  };
  const char* elementwise_name(int mode) const override;
  void release();
  osh_status refresh(const Wave& w, int iters, bool permute_v, cudaStream_t s);
  osh_status refresh_side(const Side& sd, int iters, cudaStream_t s);

  SoapConfig cfg_;
  int n_tensors_ = 0, grad_dtype_ = 0;
  long long step_ = -1;
  std::vector<Wave> waves_;
  size_t ws_bytes_ = 0, state_bytes_ = 0;
  uint8_t* d_ws_ = nullptr;
  uint8_t* d_state_ = nullptr;
  double* d_partial_ = nullptr;
  double* d_update_sq_ = nullptr;
  float* d_bscale_ = nullptr;     // (1 - beta2) per batch entry (statistics scale)
  int* d_order_ = nullptr;        // basis orders of every statistics matrix
  uint8_t* d_rws_ = nullptr;      // basis-refresh workspace (one sub-batch)
  size_t rws_bytes_ = 0;
  SoapSplitTask* d_split_ = nullptr;
  SoapCholTask* d_chol_ = nullptr;
  SoapPrepTask* d_prep_ = nullptr;
  SoapRotTask* d_rot_ = nullptr;
  ShApplyTask* d_apply_ = nullptr;
  ShBlockRef* d_blockrefs_ = nullptr;
  SoapAdamTask* d_adam_ = nullptr;
  SoapBasisTask* d_basis_ = nullptr;
  SoapVpermTask* d_vperm_ = nullptr;
  SoapQcastTask* d_qcast_ = nullptr;
  SymFillTask* d_symf_ = nullptr;
  long long* d_slot_begin_ = nullptr;
  int* d_slot_count_ = nullptr;
  int* d_slot_target_ = nullptr;
  int max_nb_ = 1;
  bool exact_grad_ = false;       // gradients exact in bf16 (statistics / T1 fast path)
};

}  // namespace osh
