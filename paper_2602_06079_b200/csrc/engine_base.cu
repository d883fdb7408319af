// OptimizerEngine: profiling shared by the optimizer engines.
#include "engine_base.cuh"

#include <cstdio>

#include "status.hpp"

namespace osh {

OptimizerEngine::~OptimizerEngine() {
  for (const Timed& t : timed_) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (cudaEvent_t ev : event_pool_) cudaEventDestroy(ev);
}

osh_status OptimizerEngine::run_pre(int, const osh_muon_cfg&, cudaStream_t) {
  return fail(OSH_ERR_UNSUPPORTED, "this optimizer engine has no split wave phases");
}
osh_status OptimizerEngine::run_ns(int, const osh_muon_cfg&, cudaStream_t) {
  return fail(OSH_ERR_UNSUPPORTED, "this optimizer engine has no split wave phases");
}
osh_status OptimizerEngine::run_post(int, const osh_muon_cfg&, cudaStream_t) {
  return fail(OSH_ERR_UNSUPPORTED, "this optimizer engine has no split wave phases");
}

cudaEvent_t OptimizerEngine::take_event() {
  if (!event_pool_.empty()) {
    cudaEvent_t ev = event_pool_.back();
    event_pool_.pop_back();
    return ev;
  }
  cudaEvent_t ev = nullptr;
  cudaEventCreate(&ev);
  return ev;
}

cudaError_t OptimizerEngine::timed_gemm(int mode, const NsProblemDesc* pd, int np, float alpha,
                                        float beta, cudaStream_t s, const NsSchedule* sched,
                                        float lr) {
  const bool rec = profile_ && timed_.size() < 100000;
  Timed t{};
  if (rec) {
    t.a = take_event();
    t.b = take_event();
    t.flops = ns_gemm_flops(pd, np);
    t.exec_flops = ns_gemm_executed_flops(pd, np);
    t.mode = mode;
    for (int q = 0; q < np; ++q) {
      if (q) t.what += "+";
      t.what += std::to_string(pd[q].a.batch) + "x" + std::to_string(pd[q].a.rows) + "x" +
                std::to_string(pd[q].b_mn_major ? pd[q].b.cols : pd[q].b.rows) + "x" +
                std::to_string(pd[q].a.cols);
    }
    if (sched != nullptr && sched->kb != nullptr && mode == kEpiGram) t.what += ":stream-k";
    cudaEventRecord(t.a, s);
  }
  const cudaError_t err = ns_gemm_launch(mode, pd, np, alpha, beta, lr, s, sched);
  if (rec) {
    cudaEventRecord(t.b, s);
    timed_.push_back(std::move(t));
  }
  stats_.gemm_flops += ns_gemm_flops(pd, np);
  ++stats_.launches_gemm;
  return err;
}

void OptimizerEngine::read_profile(int* launches, double* flops, double* exec_flops, double* ms,
                                   bool reset) {
  *launches = 0;
  *flops = *exec_flops = *ms = 0.0;
  for (const Timed& t : timed_) {
    float dt = 0.f;
    if (t.mode >= kModeElementwise) continue;
    cudaEventSynchronize(t.b);
    if (cudaEventElapsedTime(&dt, t.a, t.b) != cudaSuccess) continue;
    ++*launches;
    *flops += t.flops;
    *exec_flops += t.exec_flops;
    *ms += dt;
  }
  if (reset) {
    for (const Timed& t : timed_) {
      event_pool_.push_back(t.a);
      event_pool_.push_back(t.b);
    }
    timed_.clear();
  }
}

const char* OptimizerEngine::elementwise_name(int) const { return "elementwise"; }

std::string OptimizerEngine::profile_text(cudaEvent_t ref) const {
  static const char* kGemm[] = {"gram", "poly", "update", "final", "stat", "split", "?", "?"};
  std::string out;
  char line[512];
  for (const Timed& t : timed_) {
    float dt = 0.f;
    cudaEventSynchronize(t.b);
    if (cudaEventElapsedTime(&dt, t.a, t.b) != cudaSuccess) continue;
    const char* name = t.mode < kModeElementwise ? kGemm[t.mode] : elementwise_name(t.mode);
    std::snprintf(line, sizeof(line), "%s %.4f %.6e %.6e %s", name, dt, t.flops, t.exec_flops,
                  t.what.c_str());
    out += line;
    float t0 = 0.f;
    if (ref != nullptr && cudaEventElapsedTime(&t0, ref, t.a) == cudaSuccess) {
      std::snprintf(line, sizeof(line), " @%.4f", t0);
      out += line;
    }
    out += "\n";
  }
  return out;
}

}  // namespace osh
