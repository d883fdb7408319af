// NVLS-fused DP collectives.
//
// The NCCL path of runtime.cu runs RS-v and AG-v as NCCL kernels that take
// SMs from the persistent Newton-Schulz GEMMs while they overlap. On an
// NVSwitch node the same data movement can ride inside the update kernels:
//   * grad and replica live in NCCL symmetric windows (ncclMemAlloc +
//     ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC)); ncclDevCommCreate
//     with lsaMultimem gives each window a multicast address;
//   * the owner's momentum kernels read `multimem.ld_reduce` at the multicast
//     address of its slice: the NVSwitch sums the R ranks' gradients in
//     flight (RS-v, no reduced copy ever lands in HBM);
//   * the apply / vector kernels store the updated bf16 replica slice with
//     `multimem.st`: the switch writes it into every rank's replica (AG-v).
// A step is then: barrier -> waves -> barrier. The start barrier orders every
// rank's gradient writes before any remote read; the end barrier keeps a
// rank's gradients alive until every owner has read them and makes the
// replica complete on return. Bucket order / waves no longer matter for
// overlap, so the engine is built with the fewest waves the workspace allows.
//
// Same bits as the NCCL path for fp32 gradients only up to summation order:
// the switch's reduction order is fixed per element, so runs are
// deterministic, but bf16 gradients are summed with fp32 accumulation inside
// the switch (.acc::f32) rather than NCCL's bf16 ring/tree arithmetic.
#include <cstring>
#include <string>

#include <nccl.h>
#include <nccl_device.h>

#include "runtime.cuh"
#include "status.hpp"

namespace osh {
namespace {

__global__ void multicast_base_kernel(ncclWindow_t grad, ncclWindow_t replica, ncclDevComm dc,
                                      void** out) {
  out[0] = ncclGetLsaMultimemPointer(grad, 0, dc);
  out[1] = ncclGetLsaMultimemPointer(replica, 0, dc);
}

struct NvlsState {
  ncclWindow_t win_grad = nullptr, win_rep = nullptr;
  ncclDevComm devcomm{};
  bool devcomm_ok = false;
};

// Every rank learns whether every rank succeeded (min over ranks), so a
// failure on one GPU makes all of them fall back together instead of
// leaving the others blocked in a collective registration.
bool agree(osh_ctx* ctx, bool ok) {
  int32_t* d = nullptr;
  if (cudaMalloc(reinterpret_cast<void**>(&d), sizeof(int32_t)) != cudaSuccess) return false;
  const int32_t mine = ok ? 1 : 0;
  int32_t all = 0;
  bool good = cudaMemcpy(d, &mine, sizeof(mine), cudaMemcpyHostToDevice) == cudaSuccess &&
              ncclAllReduce(d, d, 1, ncclInt32, ncclMin, ctx->comm, ctx->compute) == ncclSuccess &&
              cudaStreamSynchronize(ctx->compute) == cudaSuccess &&
              cudaMemcpy(&all, d, sizeof(all), cudaMemcpyDeviceToHost) == cudaSuccess;
  cudaFree(d);
  return good && all == 1;
}

}  // namespace

// Allocates grad / replica as symmetric multicast-capable buffers. Returns
// OSH_OK with ctx->nvls == false when the node has no NVLS (the caller then
// allocates plain buffers); every rank must call it (collective).
osh_status nvls_setup(osh_ctx* ctx, size_t grad_bytes, size_t replica_bytes, bool required) {
  ctx->nvls = false;
  auto* st = new NvlsState();
  auto give_up = [&](const std::string& why) -> osh_status {
    if (st->devcomm_ok) ncclDevCommDestroy(ctx->comm, &st->devcomm);
    if (st->win_grad != nullptr) ncclCommWindowDeregister(ctx->comm, st->win_grad);
    if (st->win_rep != nullptr) ncclCommWindowDeregister(ctx->comm, st->win_rep);
    if (ctx->grad != nullptr) ncclMemFree(ctx->grad);
    if (ctx->replica != nullptr) ncclMemFree(ctx->replica);
    ctx->grad = nullptr;
    ctx->replica = nullptr;
    delete st;
    ctx->nvls_why = why;
    if (required) return fail(OSH_ERR_UNSUPPORTED, "NVLS collectives unavailable: " + why);
    return OSH_OK;
  };
  // each phase ends with an agreement so all ranks take the same branch
  bool ok = ncclMemAlloc(&ctx->grad, grad_bytes) == ncclSuccess &&
            ncclMemAlloc(reinterpret_cast<void**>(&ctx->replica), replica_bytes) == ncclSuccess;
  if (!agree(ctx, ok)) return give_up("ncclMemAlloc on some rank");
  ok = ncclCommWindowRegister(ctx->comm, ctx->grad, grad_bytes, &st->win_grad,
                              NCCL_WIN_COLL_SYMMETRIC) == ncclSuccess;
  ok = ncclCommWindowRegister(ctx->comm, ctx->replica, replica_bytes, &st->win_rep,
                              NCCL_WIN_COLL_SYMMETRIC) == ncclSuccess && ok;
  if (!agree(ctx, ok)) return give_up("symmetric window registration on some rank");
  ncclDevCommRequirements req;
  std::memset(&req, 0, sizeof(req));
  req.lsaMultimem = true;
  ok = ncclDevCommCreate(ctx->comm, &req, &st->devcomm) == ncclSuccess;
  st->devcomm_ok = ok;
  if (!agree(ctx, ok))
    return give_up(std::string("ncclDevCommCreate(lsaMultimem) on some rank: ") +
                   ncclGetLastError(ctx->comm));
  void** d_out = nullptr;
  void* h[2] = {nullptr, nullptr};
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&d_out), 2 * sizeof(void*));
  if (e == cudaSuccess) {
    multicast_base_kernel<<<1, 1>>>(st->win_grad, st->win_rep, st->devcomm, d_out);
    e = cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(d_out);
  }
  if (!agree(ctx, e == cudaSuccess && h[0] != nullptr && h[1] != nullptr))
    return give_up("multicast pointer lookup failed on some rank");
  ctx->mc_grad = h[0];
  ctx->mc_replica = static_cast<__nv_bfloat16*>(h[1]);
  ctx->nvls_state = st;
  ctx->nvls = true;
  return OSH_OK;
}

void nvls_free(osh_ctx* ctx) {
  auto* st = static_cast<NvlsState*>(ctx->nvls_state);
  if (st == nullptr) return;
  if (st->devcomm_ok) ncclDevCommDestroy(ctx->comm, &st->devcomm);
  if (st->win_grad != nullptr) ncclCommWindowDeregister(ctx->comm, st->win_grad);
  if (st->win_rep != nullptr) ncclCommWindowDeregister(ctx->comm, st->win_rep);
  ncclMemFree(ctx->grad);
  ncclMemFree(ctx->replica);
  ctx->grad = nullptr;
  ctx->replica = nullptr;
  ctx->mc_grad = nullptr;
  ctx->mc_replica = nullptr;
  delete st;
  ctx->nvls_state = nullptr;
  ctx->nvls = false;
}

}  // namespace osh
