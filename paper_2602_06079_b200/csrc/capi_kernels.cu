// C-ABI wrappers of the kernel-level entry points (osh.h, "kernel-level").
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "ns_gemm.cuh"
#include "osh.h"
#include "status.hpp"

namespace {

// sq_norm[i] += sum of target i's epilogue partials (fixed order)
__global__ void add_partials_kernel(const double* partial, int stride, int per,
                                    double* const* out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || out[i] == nullptr) return;
  double s = 0.0;
  for (int k = 0; k < per; ++k) s += partial[static_cast<size_t>(i) * stride + k];
  *out[i] += s;
}

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
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // FINAL: the host targets become device NsFinalTarget entries (TMA maps of
  // W and the replica) with per-tile partials of the update norm
  std::vector<osh::NsFinalTarget> fts;
  std::vector<double*> sq_out;
  std::vector<int> per_prob(static_cast<size_t>(n_problems), 0), first(static_cast<size_t>(n_problems), 0);
  int stride = 0;
  double* d_partial = nullptr;
  osh::NsFinalTarget* d_ft = nullptr;
  double** d_sq = nullptr;
  if (epilogue == OSH_EPI_FINAL) {
    size_t total = 0;
    for (int i = 0; i < n_problems; ++i) {
      const osh_gemm_problem& p = problems[i];
      if (p.final_targets == nullptr) return osh::fail(OSH_ERR_ARG, "osh_ns_gemm: FINAL needs targets");
      const int M = p.a.rows, N = p.b_mn_major ? p.b.cols : p.b.rows;
      per_prob[static_cast<size_t>(i)] = osh::final_partials(M, N);
      stride = std::max(stride, per_prob[static_cast<size_t>(i)]);
      total += static_cast<size_t>(std::max(p.a.batch, 0));
    }
    if (cudaMallocAsync(reinterpret_cast<void**>(&d_partial), sizeof(double) * total * stride, st) != cudaSuccess ||
        cudaMallocAsync(reinterpret_cast<void**>(&d_ft), sizeof(osh::NsFinalTarget) * total, st) != cudaSuccess ||
        cudaMallocAsync(reinterpret_cast<void**>(&d_sq), sizeof(double*) * total, st) != cudaSuccess)
      return osh::fail(OSH_ERR_OOM, "osh_ns_gemm: FINAL staging");
    for (int i = 0; i < n_problems; ++i) {
      const osh_gemm_problem& p = problems[i];
      const int M = p.a.rows, N = p.b_mn_major ? p.b.cols : p.b.rows;
      first[static_cast<size_t>(i)] = static_cast<int>(fts.size());
      for (int b = 0; b < p.a.batch; ++b) {
        const osh_final_target& h = p.final_targets[b];
        osh::NsFinalTarget t;
        if (!osh::make_final_target(&t, h.w, static_cast<__nv_bfloat16*>(h.replica), M, N,
                                    h.transposed, d_partial + fts.size() * stride)) {
          cudaFreeAsync(d_partial, st);
          cudaFreeAsync(d_ft, st);
          cudaFreeAsync(d_sq, st);
          return osh::fail(OSH_ERR_ARG, "osh_ns_gemm: FINAL target needs 16-byte aligned W / "
                                        "replica and a row pitch of a multiple of 16 bytes");
        }
        fts.push_back(t);
        sq_out.push_back(h.sq_norm);
      }
    }
    cudaMemcpyAsync(d_ft, fts.data(), sizeof(osh::NsFinalTarget) * fts.size(), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_sq, sq_out.data(), sizeof(double*) * sq_out.size(), cudaMemcpyHostToDevice, st);
  }
  for (int i = 0; i < n_problems; ++i) {
    const osh_gemm_problem& p = problems[i];
    d[i].a = to_ref(p.a);
    d[i].b = to_ref(p.b);
    d[i].b_mn_major = p.b_mn_major;
    d[i].out = to_ref(p.out);
    d[i].aux = to_ref(p.aux);
    d[i].scale = p.scale;
    d[i].final_targets = d_ft != nullptr ? d_ft + first[static_cast<size_t>(i)] : nullptr;
    d[i].symmetric = p.symmetric;
    d[i].out_seg = p.out_seg;
    d[i].a_upper = p.a_upper;
    d[i].b_upper = p.b_upper;
  }
  cudaError_t e = osh::ns_gemm_launch(epilogue, d, n_problems, alpha, beta, lr, st);
  for (int i = 0; i < n_problems && e == cudaSuccess && epilogue == OSH_EPI_FINAL; ++i) {
    const int n = problems[i].a.batch, f = first[static_cast<size_t>(i)];
    add_partials_kernel<<<(n + 127) / 128, 128, 0, st>>>(d_partial + static_cast<size_t>(f) * stride,
                                                         stride, per_prob[static_cast<size_t>(i)],
                                                         d_sq + f, n);
    e = cudaGetLastError();
  }
  if (d_partial != nullptr) {
    cudaFreeAsync(d_partial, st);
    cudaFreeAsync(d_ft, st);
    cudaFreeAsync(d_sq, st);
  }
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
