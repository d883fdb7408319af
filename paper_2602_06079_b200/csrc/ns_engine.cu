// MuonEngine implementation (see ns_engine.cuh).
#include "ns_engine.cuh"

#include <algorithm>
#include <cstdio>
#include <map>
#include <string>

#include "status.hpp"

namespace osh {
namespace {

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

template <typename T>
cudaError_t upload(T** dst, const std::vector<T>& src) {
  *dst = nullptr;
  if (src.empty()) return cudaSuccess;
  cudaError_t e = osh::dev_alloc(reinterpret_cast<void**>(dst), sizeof(T) * src.size());
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice);
}

NsMatrixRef ref(const void* p, int batch, int rows, int cols, long long ld) {
  NsMatrixRef r;
  r.ptr = p;
  r.batch = batch;
  r.rows = rows;
  r.cols = cols;
  r.ld = ld;
  r.bstride = ld * rows;
  return r;
}

}  // namespace

MuonEngine::~MuonEngine() {
  release();
  for (const Timed& t : timed_) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (cudaEvent_t ev : event_pool_) cudaEventDestroy(ev);
}

std::string MuonEngine::profile_text() const {
  static const char* kNames[] = {"gram", "poly", "update", "final"};
  std::string out;
  char line[256];
  for (const Timed& t : timed_) {
    float dt = 0.f;
    cudaEventSynchronize(t.b);
    if (cudaEventElapsedTime(&dt, t.a, t.b) != cudaSuccess) continue;
    std::snprintf(line, sizeof(line), "%s %.4f %.6e %.6e %s\n", kNames[t.mode & 3], dt, t.flops,
                  t.exec_flops, t.what.c_str());
    out += line;
  }
  return out;
}

cudaEvent_t MuonEngine::take_event() {
  if (!event_pool_.empty()) {
    cudaEvent_t ev = event_pool_.back();
    event_pool_.pop_back();
    return ev;
  }
  cudaEvent_t ev = nullptr;
  cudaEventCreate(&ev);
  return ev;
}

void MuonEngine::read_profile(int* launches, double* flops, double* exec_flops, double* ms,
                              bool reset) {
  *launches = 0;
  *flops = 0.0;
  *exec_flops = 0.0;
  *ms = 0.0;
  for (const Timed& t : timed_) {
    float dt = 0.f;
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

void MuonEngine::release() {
  cudaFree(d_ws_);
  cudaFree(d_partial_);
  cudaFree(d_slot_begin_);
  cudaFree(d_slot_count_);
  cudaFree(d_scale_update_);
  cudaFree(d_scale_gram_);
  cudaFree(d_update_sq_);
  cudaFree(d_mtasks_);
  cudaFree(d_vtasks_);
  cudaFree(d_final_);
  d_ws_ = nullptr;
  d_partial_ = d_update_sq_ = nullptr;
  d_slot_begin_ = nullptr;
  d_slot_count_ = nullptr;
  d_scale_update_ = d_scale_gram_ = nullptr;
  d_mtasks_ = nullptr;
  d_vtasks_ = nullptr;
  d_final_ = nullptr;
  chunks_.clear();
  waves_.clear();
}

osh_status MuonEngine::build(const std::vector<MuonTensorDesc>& tensors, int grad_dtype,
                             size_t budget) {
  release();
  n_tensors_ = static_cast<int>(tensors.size());
  grad_dtype_ = grad_dtype;

  // ---- shape classes (m <= n), biggest total Newton-Schulz work first
  std::map<std::pair<int, int>, std::vector<int>> classes;
  std::vector<MomentumVectorTask> vtasks;
  for (int i = 0; i < n_tensors_; ++i) {
    const MuonTensorDesc& t = tensors[i];
    if (t.is_matrix) {
      classes[{std::min(t.rows, t.cols), std::max(t.rows, t.cols)}].push_back(i);
    } else {
      MomentumVectorTask v{};
      v.g = t.g;
      v.m = t.m;
      v.w = t.w;
      v.replica = t.replica;
      v.n = static_cast<long long>(t.rows) * t.cols;
      vtasks.push_back(v);
    }
  }
  std::vector<std::pair<std::pair<int, int>, std::vector<int>>> order(classes.begin(),
                                                                        classes.end());
  auto work = [](const std::pair<std::pair<int, int>, std::vector<int>>& c) {
    const double m = c.first.first, n = c.first.second;
    return (4.0 * m * m * n + 2.0 * m * m * m) * static_cast<double>(c.second.size());
  };
  std::stable_sort(order.begin(), order.end(),
                   [&](const auto& x, const auto& y) { return work(x) > work(y); });

  // ---- chunks within the workspace budget
  std::vector<std::vector<int>> chunk_members;
  for (const auto& [shape, members] : order) {
    Chunk c;
    c.m = shape.first;
    c.n = shape.second;
    c.ldm = static_cast<int>(round_up(static_cast<size_t>(c.m), 64));
    c.ldn = static_cast<int>(round_up(static_cast<size_t>(c.n), 64));
    const size_t per = 2 * (2ull * c.m * c.ldn) + 2 * (2ull * c.m * c.ldm);
    const size_t cap = std::max<size_t>(1, budget / std::max<size_t>(per, 1));
    const size_t pieces = (members.size() + cap - 1) / cap;
    const size_t base = members.size() / pieces, extra = members.size() % pieces;
    size_t k = 0;
    for (size_t p = 0; p < pieces; ++p) {
      const size_t take = base + (p < extra ? 1 : 0);
      c.batch = static_cast<int>(take);
      chunks_.push_back(c);
      chunk_members.emplace_back(members.begin() + static_cast<long>(k),
                                 members.begin() + static_cast<long>(k + take));
      k += take;
    }
  }
  auto chunk_bytes = [](const Chunk& c) {
    return static_cast<size_t>(c.batch) *
           (2 * round_up(2ull * c.m * c.ldn, 256) + 2 * round_up(2ull * c.m * c.ldm, 256));
  };

  // ---- waves: first-fit of chunks (largest first) into <= 4 problems / budget
  std::vector<int> by_size(chunks_.size());
  for (size_t i = 0; i < by_size.size(); ++i) by_size[i] = static_cast<int>(i);
  std::stable_sort(by_size.begin(), by_size.end(), [&](int x, int y) {
    return chunk_bytes(chunks_[x]) > chunk_bytes(chunks_[y]);
  });
  std::vector<size_t> wave_bytes;
  for (const int ci : by_size) {
    const size_t need = chunk_bytes(chunks_[ci]);
    bool placed = false;
    for (size_t w = 0; w < waves_.size() && !placed; ++w) {
      if (waves_[w].chunks.size() < static_cast<size_t>(kMaxProblems) &&
          wave_bytes[w] + need <= budget) {
        waves_[w].chunks.push_back(ci);
        wave_bytes[w] += need;
        placed = true;
      }
    }
    if (!placed) {
      Wave w;
      w.chunks.push_back(ci);
      waves_.push_back(w);
      wave_bytes.push_back(need);
    }
  }

  // ---- slots, workspace offsets, task tables
  std::vector<MomentumMatrixTask> mtasks;
  std::vector<NsFinalTarget> finals;
  ws_bytes_ = 0;
  int slot = 0;
  // The update norms are accumulated per tensor into d_update_sq_ (allocated
  // below); record the tensor index now, patch pointers after allocation.
  std::vector<int> slot_tensor;
  std::vector<long long> slot_begin;
  std::vector<int> slot_count;
  long long max_tiles = 1;
  std::vector<int> vec_tensor;
  for (int i = 0; i < n_tensors_; ++i)
    if (!tensors[i].is_matrix) vec_tensor.push_back(i);
  for (Wave& w : waves_) {
    size_t off = 0;
    w.task0 = static_cast<int>(mtasks.size());
    for (const int ci : w.chunks) {
      Chunk& c = chunks_[ci];
      c.slot0 = slot;
      const size_t xb = round_up(2ull * c.m * c.ldn, 256), ab = round_up(2ull * c.m * c.ldm, 256);
      c.x0 = off;
      off += xb * c.batch;
      c.x1 = off;
      off += xb * c.batch;
      c.a = off;
      off += ab * c.batch;
      c.b = off;
      off += ab * c.batch;
      for (int b = 0; b < c.batch; ++b) {
        const int ti = chunk_members[ci][b];
        const MuonTensorDesc& t = tensors[ti];
        MomentumMatrixTask mt{};
        mt.g = t.g;
        mt.m = t.m;
        mt.rows = t.rows;
        mt.cols = t.cols;
        mt.ldx = c.ldn;
        mt.transposed = t.rows > t.cols ? 1 : 0;
        mt.tiles_c = (t.cols + kTile - 1) / kTile;
        mt.tile_start = w.tiles;
        // x0 patched once the workspace base is known (offset stored as ptr)
        mt.x0 = reinterpret_cast<__nv_bfloat16*>(c.x0 + static_cast<size_t>(b) * (xb));
        const long long ntiles = static_cast<long long>((t.rows + kTile - 1) / kTile) * mt.tiles_c;
        // per-tile partial sums live at [tile_start, tile_start + ntiles) of
        // the wave's partial array; the task's pointer is rebased below
        mt.partial = nullptr;
        slot_begin.push_back(w.tiles);
        slot_count.push_back(static_cast<int>(ntiles));
        w.tiles += ntiles;
        mtasks.push_back(mt);
        NsFinalTarget ft{};
        ft.w = t.w;
        ft.replica = t.replica;
        ft.transposed = mt.transposed;
        finals.push_back(ft);
        slot_tensor.push_back(ti);
        ++slot;
      }
    }
    w.n_tasks = static_cast<int>(mtasks.size()) - w.task0;
    ws_bytes_ = std::max(ws_bytes_, off);
    max_tiles = std::max(max_tiles, w.tiles);
  }
  n_slots_ = slot;

  OSH_CUDA_TRY(osh::dev_alloc(reinterpret_cast<void**>(&d_ws_), std::max<size_t>(ws_bytes_, 256)));
  if (!debug_poison()) OSH_CUDA_TRY(cudaMemset(d_ws_, 0, std::max<size_t>(ws_bytes_, 256)));
  OSH_CUDA_TRY(osh::dev_alloc(reinterpret_cast<void**>(&d_partial_), sizeof(double) * static_cast<size_t>(max_tiles)));
  OSH_CUDA_TRY(upload(&d_slot_begin_, slot_begin));
  OSH_CUDA_TRY(upload(&d_slot_count_, slot_count));
  OSH_CUDA_TRY(osh::dev_alloc(reinterpret_cast<void**>(&d_scale_update_), sizeof(float) * std::max(n_slots_, 1)));
  OSH_CUDA_TRY(osh::dev_alloc(reinterpret_cast<void**>(&d_scale_gram_), sizeof(float) * std::max(n_slots_, 1)));
  OSH_CUDA_TRY(osh::dev_alloc(reinterpret_cast<void**>(&d_update_sq_), sizeof(double) * std::max(n_tensors_, 1)));
  OSH_CUDA_TRY(cudaMemset(d_update_sq_, 0, sizeof(double) * std::max(n_tensors_, 1)));
  for (MomentumMatrixTask& mt : mtasks) {
    mt.x0 = reinterpret_cast<__nv_bfloat16*>(d_ws_ + reinterpret_cast<uintptr_t>(mt.x0));
    mt.partial = d_partial_ + mt.tile_start;  // local tile index is added in-kernel
  }
  for (size_t s = 0; s < finals.size(); ++s) finals[s].sq_norm = d_update_sq_ + slot_tensor[s];
  for (size_t v = 0; v < vtasks.size(); ++v) vtasks[v].sq_norm = d_update_sq_ + vec_tensor[v];
  n_vec_tasks_ = static_cast<int>(vtasks.size());
  OSH_CUDA_TRY(upload(&d_mtasks_, mtasks));
  OSH_CUDA_TRY(upload(&d_vtasks_, vtasks));
  OSH_CUDA_TRY(upload(&d_final_, finals));
  return OSH_OK;
}

osh_status MuonEngine::run(const osh_muon_cfg& cfg, cudaStream_t s) {
  if (cfg.ns_steps < 1 && n_slots_ > 0)
    return fail(OSH_ERR_UNSUPPORTED, "MuonEngine: ns_steps must be >= 1 on the GPU path");
  stats_ = NsLaunchStats{};
  const float beta = static_cast<float>(cfg.beta), lr = static_cast<float>(cfg.lr);
  OSH_CUDA_TRY(cudaMemsetAsync(d_update_sq_, 0, sizeof(double) * std::max(n_tensors_, 1), s));
  if (n_vec_tasks_ > 0) {
    OSH_CUDA_TRY(launch_momentum_vector(d_vtasks_, n_vec_tasks_, grad_dtype_, beta, lr, s));
    ++stats_.launches_elementwise;
  }
  for (const Wave& w : waves_) {
    OSH_CUDA_TRY(launch_momentum_matrix(d_mtasks_ + w.task0, w.n_tasks, w.tiles, grad_dtype_,
                                        beta, s));
    const int slot0 = chunks_[w.chunks.front()].slot0;
    int nslots = 0;
    for (const int ci : w.chunks) nslots += chunks_[ci].batch;
    // slots of a wave are contiguous (assigned wave by wave, chunk by chunk)
    OSH_CUDA_TRY(launch_ns_scales(d_partial_, d_slot_begin_ + slot0, d_slot_count_ + slot0,
                                  d_scale_update_ + slot0, d_scale_gram_ + slot0, nslots, s));
    stats_.launches_elementwise += 2;
    const int np = static_cast<int>(w.chunks.size());
    for (int it = 0; it < cfg.ns_steps; ++it) {
      const bool first = it == 0, last = it == cfg.ns_steps - 1;
      NsProblemDesc gram[kMaxProblems], poly[kMaxProblems], upd[kMaxProblems];
      for (int q = 0; q < np; ++q) {
        const Chunk& c = chunks_[w.chunks[q]];
        uint8_t* xin = d_ws_ + ((it & 1) ? c.x1 : c.x0);
        uint8_t* xout = d_ws_ + ((it & 1) ? c.x0 : c.x1);
        uint8_t* A = d_ws_ + c.a;
        uint8_t* B = d_ws_ + c.b;
        const long long xb = static_cast<long long>(round_up(2ull * c.m * c.ldn, 256) / 2);
        const long long ab = static_cast<long long>(round_up(2ull * c.m * c.ldm, 256) / 2);
        NsMatrixRef X = ref(xin, c.batch, c.m, c.n, c.ldn);
        X.bstride = xb;
        NsMatrixRef Xo = ref(xout, c.batch, c.m, c.n, c.ldn);
        Xo.bstride = xb;
        NsMatrixRef Am = ref(A, c.batch, c.m, c.m, c.ldm);
        Am.bstride = ab;
        NsMatrixRef Bm = ref(B, c.batch, c.m, c.m, c.ldm);
        Bm.bstride = ab;
        gram[q] = NsProblemDesc{X, X, 0, Am, NsMatrixRef{}, first ? d_scale_gram_ + c.slot0 : nullptr,
                                nullptr, symmetric_ ? 1 : 0};
        poly[q] = NsProblemDesc{Am, Am, 0, Bm, Am, nullptr, nullptr, symmetric_ ? 1 : 0};
        upd[q] = NsProblemDesc{Bm, X, 1, Xo, X, first ? d_scale_update_ + c.slot0 : nullptr,
                               last ? d_final_ + c.slot0 : nullptr, 0};
      }
      const auto timed_launch = [&](int mode, const NsProblemDesc* pd, float a, float b,
                                    float l) {
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
          cudaEventRecord(t.a, s);
        }
        const cudaError_t err = ns_gemm_launch(mode, pd, np, a, b, l, s);
        if (rec) {
          cudaEventRecord(t.b, s);
          timed_.push_back(t);
        }
        return err;
      };
      cudaError_t e = timed_launch(kEpiGram, gram, 0.f, 0.f, 0.f);
      if (e == cudaSuccess)
        e = timed_launch(kEpiPoly, poly, static_cast<float>(cfg.ns_b),
                         static_cast<float>(cfg.ns_c), 0.f);
      if (e == cudaSuccess)
        e = timed_launch(last ? kEpiFinal : kEpiUpdate, upd, static_cast<float>(cfg.ns_a), 0.f, lr);
      if (e != cudaSuccess)
        return fail(OSH_ERR_CUDA, std::string("MuonEngine: ns_gemm_launch: ") +
                                      cudaGetErrorString(e));
      stats_.launches_gemm += 3;
      stats_.gemm_flops += ns_gemm_flops(gram, np) + ns_gemm_flops(poly, np) +
                           ns_gemm_flops(upd, np);
    }
  }
  return OSH_OK;
}

}  // namespace osh
