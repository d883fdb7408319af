// Sharded optimizer-state checkpoint keyed by the plan.
//
// Each rank writes the state it owns — fp32 master + momentum of its owned
// tensors (and of the TP-plane tensors it hosts), plus the optimizer's extra
// state (Shampoo statistics / roots and step counter) — to its own file,
// behind a header that pins what the state means: format version, optimizer,
// dp / tp rank and size, grad dtype, and a 64-bit FNV-1a hash of the
// parameter shapes, bucket capacity layout and the plan's cut vectors. Loading
// into a ctx with a different plan or model fails with OSH_ERR_FORMAT (the
// reference's plan files are the on-disk contract for WHAT a rank owns,
// serialize.hpp:252-430; this file is the matching contract for its STATE).
// After loading, every rank rewrites the bf16 replica slots it owns and the
// replica is all-gathered, so the model the ranks forward with is restored too.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "runtime.cuh"
#include "status.hpp"

namespace {

constexpr char kMagic[8] = {'O', 'S', 'H', 'C', 'K', 'P', 'T', '1'};

struct Header {
  char magic[8];
  int32_t version, optimizer;
  int32_t dp_rank, dp_size, tp_rank, tp_size;
  int32_t n_params, grad_dtype;
  uint64_t plan_hash;
  int64_t step_counter;
  uint64_t n_records;    // (pid, numel) records that follow
  uint64_t extra_bytes;  // optimizer extra state after the records
};

uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const auto* b = static_cast<const uint8_t*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 1099511628211ull;
  }
  return h;
}

uint64_t plan_hash(const osh_ctx* ctx) {
  uint64_t h = 1469598103934665603ull;
  for (const auto& p : ctx->params_full) {
    for (const int64_t e : p.shape) h = fnv(h, &e, sizeof(e));
    const int32_t f[2] = {static_cast<int32_t>(p.tp_splittable), p.vocab_space ? 1 : 0};
    h = fnv(h, f, sizeof(f));
  }
  for (const auto& c : ctx->cuts) h = fnv(h, c.data(), sizeof(int64_t) * c.size());
  for (const auto& o : ctx->owner) h = fnv(h, &o, sizeof(o));
  const int32_t k[3] = {ctx->optimizer, ctx->shampoo.block, ctx->shampoo.newton_iters};
  return fnv(h, k, sizeof(k));
}

struct Region {
  int32_t pid;
  int64_t numel;
  float* w;
  float* m;
};

// every fp32 (w, m) region this rank holds, ascending parameter id
std::vector<Region> regions(osh_ctx* ctx) {
  std::vector<Region> out;
  for (size_t p = 0; p < ctx->params.size(); ++p) {
    if (ctx->owned_off[p] >= 0)
      out.push_back({static_cast<int32_t>(p), ctx->params[p].numel, ctx->w + ctx->owned_off[p],
                     ctx->m + ctx->owned_off[p]});
    const int ti = ctx->tp_item_of.empty() ? -1 : ctx->tp_item_of[p];
    if (ti >= 0 && ctx->tp_items[ti].w != nullptr) {
      const osh_ctx::TpItem& it = ctx->tp_items[ti];
      out.push_back({static_cast<int32_t>(p), it.full_rows * it.full_cols, it.w, it.m});
    }
  }
  return out;
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
  // flush + close, reporting a failed final write-back (ENOSPC, EIO)
  bool close() {
    FILE* g = f;
    f = nullptr;
    return g != nullptr && std::fflush(g) == 0 && std::fclose(g) == 0;
  }
};

}  // namespace

extern "C" osh_status osh_ctx_save_state(osh_ctx* ctx, const char* path) {
  if (ctx == nullptr || path == nullptr) return osh::fail(OSH_ERR_ARG, "null argument");
  if (!ctx->layout_ready) return osh::fail(OSH_ERR_PLAN, "osh_ctx_set_layout has not been called");
  OSH_CUDA_TRY(cudaSetDevice(ctx->device));
  if (osh_status st = osh_ctx_sync(ctx); st != OSH_OK) return st;
  const std::vector<Region> regs = regions(ctx);
  Header h{};
  std::memcpy(h.magic, kMagic, 8);
  h.version = 1;
  h.optimizer = ctx->optimizer;
  h.dp_rank = ctx->rank;
  h.dp_size = ctx->size;
  h.tp_rank = ctx->tp_rank;
  h.tp_size = ctx->tp_size;
  h.n_params = static_cast<int32_t>(ctx->params.size());
  h.grad_dtype = ctx->grad_dtype;
  h.plan_hash = plan_hash(ctx);
  h.step_counter = ctx->engine->step_counter();
  h.n_records = regs.size();
  h.extra_bytes = ctx->engine->extra_state_bytes();
  // written next to the target and renamed into place: a failed or
  // interrupted save never destroys the previous checkpoint
  const std::string tmp = std::string(path) + ".tmp";
  File out;
  out.f = std::fopen(tmp.c_str(), "wb");
  if (out.f == nullptr) return osh::fail(OSH_ERR_FORMAT, "cannot open " + tmp);
  bool ok = std::fwrite(&h, sizeof(h), 1, out.f) == 1;
  std::vector<float> buf;
  for (const Region& r : regs) {
    ok = ok && std::fwrite(&r.pid, sizeof(r.pid), 1, out.f) == 1 &&
         std::fwrite(&r.numel, sizeof(r.numel), 1, out.f) == 1;
    buf.resize(static_cast<size_t>(r.numel));
    for (float* src : {r.w, r.m}) {
      OSH_CUDA_TRY(cudaMemcpy(buf.data(), src, 4 * buf.size(), cudaMemcpyDeviceToHost));
      ok = ok && std::fwrite(buf.data(), 4, buf.size(), out.f) == buf.size();
    }
  }
  if (h.extra_bytes > 0) {
    std::vector<uint8_t> extra(h.extra_bytes);
    OSH_CUDA_TRY(cudaMemcpy(extra.data(), ctx->engine->extra_state(), extra.size(),
                            cudaMemcpyDeviceToHost));
    ok = ok && std::fwrite(extra.data(), 1, extra.size(), out.f) == extra.size();
  }
  if (!out.close() || !ok) {
    std::remove(tmp.c_str());
    return osh::fail(OSH_ERR_FORMAT, "short write to " + tmp);
  }
  if (std::rename(tmp.c_str(), path) != 0) {
    std::remove(tmp.c_str());
    return osh::fail(OSH_ERR_FORMAT, std::string("cannot rename ") + tmp + " to " + path);
  }
  return OSH_OK;
}

extern "C" osh_status osh_ctx_load_state(osh_ctx* ctx, const char* path) {
  if (ctx == nullptr || path == nullptr) return osh::fail(OSH_ERR_ARG, "null argument");
  if (!ctx->layout_ready) return osh::fail(OSH_ERR_PLAN, "osh_ctx_set_layout has not been called");
  OSH_CUDA_TRY(cudaSetDevice(ctx->device));
  if (osh_status st = osh_ctx_sync(ctx); st != OSH_OK) return st;
  File in;
  in.f = std::fopen(path, "rb");
  if (in.f == nullptr) return osh::fail(OSH_ERR_FORMAT, std::string("cannot open ") + path);
  Header h{};
  if (std::fread(&h, sizeof(h), 1, in.f) != 1 || std::memcmp(h.magic, kMagic, 8) != 0 ||
      h.version != 1)
    return osh::fail(OSH_ERR_FORMAT, std::string(path) + ": not an osh checkpoint (v1)");
  const std::vector<Region> regs = regions(ctx);
  if (h.optimizer != ctx->optimizer || h.dp_rank != ctx->rank || h.dp_size != ctx->size ||
      h.tp_rank != ctx->tp_rank || h.tp_size != ctx->tp_size ||
      h.n_params != static_cast<int32_t>(ctx->params.size()) || h.plan_hash != plan_hash(ctx) ||
      h.grad_dtype != ctx->grad_dtype || h.n_records != regs.size() ||
      h.extra_bytes != ctx->engine->extra_state_bytes())
    return osh::fail(OSH_ERR_FORMAT, std::string(path) +
                                         ": checkpoint belongs to a different rank, plan, model, "
                                         "gradient dtype or optimizer");
  // validation pass: every record header and the exact file length, before
  // any device state is touched (a bad file never leaves the ctx half restored)
  const long data0 = std::ftell(in.f);
  for (const Region& r : regs) {
    int32_t pid = -1;
    int64_t numel = -1;
    if (std::fread(&pid, sizeof(pid), 1, in.f) != 1 || std::fread(&numel, sizeof(numel), 1, in.f) != 1 ||
        pid != r.pid || numel != r.numel ||
        std::fseek(in.f, static_cast<long>(8 * numel), SEEK_CUR) != 0)
      return osh::fail(OSH_ERR_FORMAT, std::string(path) + ": tensor record mismatch");
  }
  const long expect_end = std::ftell(in.f) + static_cast<long>(h.extra_bytes);
  if (std::fseek(in.f, 0, SEEK_END) != 0 || std::ftell(in.f) != expect_end)
    return osh::fail(OSH_ERR_FORMAT, std::string(path) + ": truncated or oversized");
  if (std::fseek(in.f, data0, SEEK_SET) != 0)
    return osh::fail(OSH_ERR_FORMAT, std::string(path) + ": seek failed");
  std::vector<float> buf;
  for (const Region& r : regs) {
    int32_t pid = -1;
    int64_t numel = -1;
    if (std::fread(&pid, sizeof(pid), 1, in.f) != 1 || std::fread(&numel, sizeof(numel), 1, in.f) != 1 ||
        pid != r.pid || numel != r.numel)
      return osh::fail(OSH_ERR_FORMAT, std::string(path) + ": tensor record mismatch");
    buf.resize(static_cast<size_t>(numel));
    for (float* dst : {r.w, r.m}) {
      if (std::fread(buf.data(), 4, buf.size(), in.f) != buf.size())
        return osh::fail(OSH_ERR_FORMAT, std::string(path) + ": truncated");
      OSH_CUDA_TRY(cudaMemcpy(dst, buf.data(), 4 * buf.size(), cudaMemcpyHostToDevice));
    }
  }
  if (h.extra_bytes > 0) {
    std::vector<uint8_t> extra(h.extra_bytes);
    if (std::fread(extra.data(), 1, extra.size(), in.f) != extra.size())
      return osh::fail(OSH_ERR_FORMAT, std::string(path) + ": truncated optimizer state");
    OSH_CUDA_TRY(cudaMemcpy(ctx->engine->extra_state(), extra.data(), extra.size(),
                            cudaMemcpyHostToDevice));
  }
  ctx->engine->set_step_counter(h.step_counter);
  return osh::refresh_replica(ctx);
}
