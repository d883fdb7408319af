// C-ABI wrappers of the kernel-level entry points (osh.h, "kernel-level").
#include <cstring>
#include <string>

#include "ns_gemm.cuh"
#include "osh.h"
#include "status.hpp"

static_assert(sizeof(osh_final_target) == sizeof(osh::NsFinalTarget),
              "osh_final_target must mirror osh::NsFinalTarget");

namespace {

osh::NsMatrixRef to_ref(const osh_matrix_ref& m) {
  osh::NsMatrixRef r;
  r.ptr = m.ptr;
  r.batch = m.batch;
  r.rows = m.rows;
  r.cols = m.cols;
  r.ld = m.ld;
  r.bstride = m.bstride;
  return r;
}

}  // namespace

extern "C" osh_status osh_ns_gemm(int32_t epilogue, const osh_gemm_problem* problems,
                                  int32_t n_problems, float alpha, float beta, float lr,
                                  void* stream) {
  if (problems == nullptr || n_problems < 1 || n_problems > osh::kMaxProblems)
    return osh::fail(OSH_ERR_ARG, "osh_ns_gemm: need 1..4 problems");
  osh::NsProblemDesc d[osh::kMaxProblems];
  for (int i = 0; i < n_problems; ++i) {
    const osh_gemm_problem& p = problems[i];
    d[i].a = to_ref(p.a);
    d[i].b = to_ref(p.b);
    d[i].b_mn_major = p.b_mn_major;
    d[i].out = to_ref(p.out);
    d[i].aux = to_ref(p.aux);
    d[i].scale = p.scale;
    d[i].final_targets = reinterpret_cast<const osh::NsFinalTarget*>(p.final_targets);
    d[i].symmetric = p.symmetric;
    d[i].out_seg = p.out_seg;
  }
  const cudaError_t e = osh::ns_gemm_launch(epilogue, d, n_problems, alpha, beta, lr,
                                            static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess)
    return osh::fail(OSH_ERR_CUDA, std::string("osh_ns_gemm: ") + cudaGetErrorString(e));
  return OSH_OK;
}

extern "C" osh_status osh_set_gemm_cta_group(int32_t cg) {
  if (cg != 1 && cg != 2) return osh::fail(OSH_ERR_ARG, "cta group must be 1 or 2");
  osh::ns_gemm_set_cta_group(cg);
  return OSH_OK;
}

extern "C" int32_t osh_gemm_cta_group(void) { return osh::ns_gemm_cta_group(); }
