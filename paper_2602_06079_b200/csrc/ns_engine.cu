// MuonEngine implementation (see ns_engine.cuh).
#include "ns_engine.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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

NsMatrixRef ref(const void* p, int batch, int rows, int cols, long long ld, long long bstride) {
  NsMatrixRef r;
  r.ptr = p;
  r.batch = batch;
  r.rows = rows;
  r.cols = cols;
  r.ld = ld;
  r.bstride = bstride;
  return r;
}

struct Shape {
  int m, n, ldm, ldn;
  size_t xb, ab;  // bytes of one X / one A (256 B rounded)
};

Shape shape_of(int rows, int cols) {
  Shape s;
  s.m = std::min(rows, cols);
  s.n = std::max(rows, cols);
  s.ldm = static_cast<int>(round_up(static_cast<size_t>(s.m), 64));
  s.ldn = static_cast<int>(round_up(static_cast<size_t>(s.n), 64));
  s.xb = round_up(2ull * s.m * s.ldn, 256);
  s.ab = round_up(2ull * s.m * s.ldm, 256);
  return s;
}

}  // namespace

MuonEngine::~MuonEngine() { release(); }

const char* MuonEngine::elementwise_name(int mode) const {
  static const char* kNames[] = {"momentum_vector", "momentum_matrix", "ns_scales", "apply_update",
                                 "partial_sums", "mc_broadcast"};
  const int i = mode - kModeElementwise;
  return i >= 0 && i < 6 ? kNames[i] : "elementwise";
}

void MuonEngine::release() {
  for (void* p : {static_cast<void*>(d_ws_), static_cast<void*>(d_partial_),
                  static_cast<void*>(d_slot_begin_), static_cast<void*>(d_slot_count_),
                  static_cast<void*>(d_slot_tensor_), static_cast<void*>(d_scale_update_),
                  static_cast<void*>(d_scale_gram_), static_cast<void*>(d_update_sq_),
                  static_cast<void*>(d_mtasks_), static_cast<void*>(d_atasks_),
                  static_cast<void*>(d_vtasks_), static_cast<void*>(d_ftargets_),
                  static_cast<void*>(d_fpartial_), static_cast<void*>(d_fslot_begin_),
                  static_cast<void*>(d_fslot_count_), static_cast<void*>(d_fslot_tensor_),
                  static_cast<void*>(d_sk_ws_), static_cast<void*>(d_mctasks_)})
    cudaFree(p);
  d_sk_ws_ = nullptr;
  d_mctasks_ = nullptr;
  d_ftargets_ = nullptr;
  d_fpartial_ = nullptr;
  fpartial_count_ = 0;
  d_fslot_begin_ = nullptr;
  d_fslot_count_ = d_fslot_tensor_ = nullptr;
  d_ws_ = nullptr;
  d_partial_ = d_update_sq_ = nullptr;
  d_slot_begin_ = nullptr;
  d_slot_count_ = d_slot_tensor_ = nullptr;
  d_scale_update_ = d_scale_gram_ = nullptr;
  d_mtasks_ = nullptr;
  d_atasks_ = nullptr;
  d_vtasks_ = nullptr;
  for (int* p : sched_mem_) cudaFree(p);
  sched_mem_.clear();
  chunks_.clear();
  waves_.clear();
  wave_tensors_.clear();
}

osh_status MuonEngine::build(const std::vector<MuonTensorDesc>& tensors, int grad_dtype,
                             size_t budget, int min_waves, bool double_buffer) {
  release();
  n_tensors_ = static_cast<int>(tensors.size());
  grad_dtype_ = grad_dtype;

  // ---- waves: consecutive tensors (declaration order) within the budget
  size_t total_ws = 0, largest = 0;
  for (const MuonTensorDesc& t : tensors)
    if (t.is_matrix) {
      const Shape s = shape_of(t.rows, t.cols);
      total_ws += 2 * s.xb + 2 * s.ab;
      largest = std::max(largest, 2 * s.xb + 2 * s.ab);
    }
  if (largest > budget)
    return fail(OSH_ERR_OOM, "MuonEngine: one matrix needs " + std::to_string(largest) +
                                 " workspace bytes, budget is " + std::to_string(budget));
  // double buffering: odd waves use a second workspace half, so wave w+1's
  // momentum can run while wave w's GEMMs still read theirs
  double_buffer_ = double_buffer && largest <= budget / 2;
  size_t cap = double_buffer_ ? budget / 2 : budget;
  // a matrix larger than the wave target (a vocabulary matrix of a rank that
  // owns few others) forms a wave of its own; the rest keep the target size
  if (min_waves > 1) cap = std::min(cap, (total_ws + min_waves - 1) / min_waves);

  // FINAL fusion is a property of the TENSOR (vector-addressable W and
  // replica; with NVLS the epilogue writes this GPU's slot and run_post
  // re-stores it through the multicast address), never of the wave it lands
  // in, so results do not depend
  // on how the plan groups tensors (sharded == replicated bit for bit).
  const char* ff = std::getenv("OSH_FUSE_FINAL");
  fuse_final_ = !(ff != nullptr && std::strcmp(ff, "0") == 0);
  const char* uf = std::getenv("OSH_UPPER_FORM");
  upper_form_ = uf != nullptr && std::strcmp(uf, "1") == 0;  // opt-in (see problems())
  std::vector<char> fused_t(tensors.size(), 0);
  for (size_t i = 0; i < tensors.size(); ++i) {
    const MuonTensorDesc& t = tensors[i];
    if (!t.is_matrix || !fuse_final_) continue;
    const Shape s = shape_of(t.rows, t.cols);
    const __nv_bfloat16* rep = t.rep_mc ? t.replica_local : t.replica;
    fused_t[i] = (!t.rep_mc || t.replica_local != nullptr) &&
                         final_target_ok(t.w, rep, s.m, s.n, t.rows > t.cols ? 1 : 0)
                     ? 1
                     : 0;
  }
  // chunk key: (m, n), n negated for fused tensors (a class splits by fusion)
  const auto key_of = [&](int i) {
    const Shape s = shape_of(tensors[i].rows, tensors[i].cols);
    return std::pair<int, int>{s.m, fused_t[i] ? -s.n : s.n};
  };

  std::vector<std::vector<int>> wave_members(1);
  std::vector<std::vector<std::pair<int, int>>> wave_classes(1);
  size_t used = 0, half = 0;
  for (int i = 0; i < n_tensors_; ++i) {
    const MuonTensorDesc& t = tensors[i];
    if (t.is_matrix) {
      const Shape s = shape_of(t.rows, t.cols);
      const size_t need = 2 * s.xb + 2 * s.ab;
      const std::pair<int, int> cls = key_of(i);
      auto& classes = wave_classes.back();
      const bool new_class = std::find(classes.begin(), classes.end(), cls) == classes.end();
      const bool has_matrix = used > 0;
      if (has_matrix && (used + need > cap ||
                         (new_class && classes.size() == static_cast<size_t>(kMaxProblems)))) {
        wave_members.emplace_back();
        wave_classes.emplace_back();
        half = std::max(half, used);
        used = 0;
      }
      auto& cl = wave_classes.back();
      if (std::find(cl.begin(), cl.end(), cls) == cl.end()) cl.push_back(cls);
      used += need;
    }
    wave_members.back().push_back(i);
  }
  if (wave_members.back().empty()) wave_members.pop_back();
  half = (std::max(half, used) + 1023) / 1024 * 1024;
  if (reorder_ && wave_members.size() >= 3) {
    // The overlapped schedule exposes the momentum of the first wave and the
    // update of the last one (runtime.cu run_waves_local): run the smallest
    // wave first and the second smallest last, the rest in bucket order.
    std::vector<double> elems(wave_members.size(), 0.0);
    for (size_t wi = 0; wi < wave_members.size(); ++wi)
      for (const int ti : wave_members[wi])
        elems[wi] += static_cast<double>(tensors[ti].rows) * tensors[ti].cols;
    std::vector<size_t> idx(wave_members.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return elems[a] < elems[b]; });
    const char* tv = std::getenv("OSH_TAPER");
    const bool taper = !(tv != nullptr && std::strcmp(tv, "0") == 0);
    size_t first = idx[0], last = idx[1];
    if (taper)  // the tail is tapered below: last = the smallest wave of several tensors
      for (size_t k = 1; k < idx.size(); ++k)
        if (wave_members[idx[k]].size() >= 4) {
          last = idx[k];
          break;
        }
    std::vector<std::vector<int>> ordered;
    ordered.push_back(wave_members[first]);
    for (size_t wi = 0; wi < wave_members.size(); ++wi)
      if (wi != first && wi != last) ordered.push_back(wave_members[wi]);
    ordered.push_back(wave_members[last]);
    wave_members.swap(ordered);
    // Tapered tail: with host buffers the bf16 replica of a wave leaves (D2H)
    // while the next wave computes, so what stays exposed is the copy-out of
    // the LAST wave. The last wave is cut into parts shrinking by ~0.7x toward
    // the end (a part's compute covers the previous part's copy-out: D2H
    // moves ~1.4x more elements per ms than the step computes), the final part
    // <= 1/128 of the owned elements. OSH_TAPER=0 keeps the last wave whole.
    if (taper) {
      const auto numel = [&](int ti) { return static_cast<double>(tensors[ti].rows) * tensors[ti].cols; };
      double total = 0.0;
      for (const MuonTensorDesc& t : tensors) total += numel(static_cast<int>(&t - tensors.data()));
      std::vector<int> src = wave_members.back();
      wave_members.pop_back();
      std::vector<std::vector<int>> parts;  // built from the back: smallest first
      double target = total / 128.0;
      while (!src.empty()) {
        std::vector<int> part;
        double acc = 0.0;
        while (!src.empty() && (part.empty() || acc + numel(src.back()) <= target)) {
          acc += numel(src.back());
          part.insert(part.begin(), src.back());
          src.pop_back();
        }
        parts.push_back(part);
        target /= 0.7;
      }
      for (auto it = parts.rbegin(); it != parts.rend(); ++it) wave_members.push_back(*it);
    }
  }

  // fused FINAL targets: (tensor, m, n, partial offset) per fused matrix slot
  struct FTarget {
    int ti, m, n;
    size_t poff;
  };
  std::vector<FTarget> ftargets;
  std::vector<McCopyTask> mctasks;
  std::vector<long long> fslot_begin;
  std::vector<int> fslot_count, fslot_tensor;

  wave_tensors_ = wave_members;

  // ---- chunks (one per class per wave), slots, tables
  std::vector<MomentumMatrixTask> mtasks;
  std::vector<ApplyTask> atasks;
  std::vector<MomentumVectorTask> vtasks;
  std::vector<long long> slot_begin;
  std::vector<int> slot_count, slot_tensor;
  long long max_tiles = 1;
  ws_bytes_ = 0;
  int slot = 0;
  for (size_t wi = 0; wi < wave_members.size(); ++wi) {
    const std::vector<int>& mem = wave_members[wi];
    Wave w;
    w.first_bucket = tensors[mem.front()].bucket;
    w.last_bucket = tensors[mem.back()].bucket;
    w.task0 = static_cast<int>(mtasks.size());
    w.slot0 = slot;
    w.vec0 = static_cast<int>(vtasks.size());
    // group matrices by class, classes in order of first appearance
    std::vector<std::pair<int, int>> order;
    std::map<std::pair<int, int>, std::vector<int>> by_class;
    for (const int ti : mem) {
      const MuonTensorDesc& t = tensors[ti];
      if (!t.is_matrix) {
        MomentumVectorTask v{};
        v.g = t.g;
        v.m = t.m;
        v.w = t.w;
        v.replica = t.replica;
        v.n = static_cast<long long>(t.rows) * t.cols;
        w.elems_vector += static_cast<double>(v.n);
        v.g_mc = t.g_mc;
        v.rep_mc = t.rep_mc;
        v.sq_norm = reinterpret_cast<double*>(static_cast<uintptr_t>(ti));  // patched below
        vtasks.push_back(v);
        continue;
      }
      const std::pair<int, int> cls = key_of(ti);
      if (!by_class.count(cls)) order.push_back(cls);
      by_class[cls].push_back(ti);
    }
    // unfused chunks first: their momentum / apply tasks, tiles and slots form
    // a prefix of the wave's tables (the apply pass runs over that prefix)
    std::stable_partition(order.begin(), order.end(), [](const std::pair<int, int>& k) { return k.second > 0; });
    size_t off = double_buffer_ && (wi & 1) ? half : 0;
    w.fslot0 = static_cast<int>(fslot_begin.size());
    w.mc0 = static_cast<int>(mctasks.size());
    for (const auto& cls : order) {
      const bool cfused = cls.second < 0;
      if (!cfused) ++w.nf_chunks;
      const std::vector<int>& members = by_class[cls];
      const MuonTensorDesc& t0 = tensors[members.front()];
      const Shape s = shape_of(t0.rows, t0.cols);
      Chunk c;
      c.m = s.m;
      c.n = s.n;
      c.ldm = s.ldm;
      c.ldn = s.ldn;
      c.batch = static_cast<int>(members.size());
      c.slot0 = slot;
      c.x0 = off;
      off += s.xb * c.batch;
      c.x1 = off;
      off += s.xb * c.batch;
      c.a = off;
      off += s.ab * c.batch;
      c.b = off;
      off += s.ab * c.batch;
      if (cfused) c.ftarget0 = static_cast<int>(ftargets.size());
      for (int b = 0; b < c.batch; ++b) {
        const int ti = members[b];
        const MuonTensorDesc& t = tensors[ti];
        if (!cfused) {  // the unfused prefix of the wave's tables
          ++w.nf_tasks;
          ++w.nf_slots;
        }
        if (cfused) {
          // partial slots of both CTA-group variants (the larger count)
          const int cg0 = ns_gemm_cta_group();
          ns_gemm_set_cta_group(1);
          const int p1 = final_partials(s.m, s.n);
          ns_gemm_set_cta_group(2);
          const int p2 = final_partials(s.m, s.n);
          ns_gemm_set_cta_group(cg0);
          const int cnt = std::max(p1, p2);
          ftargets.push_back({ti, s.m, s.n, fpartial_count_});
          if (t.rep_mc) {  // NVLS: re-store the local slot through the multicast address
            const long long n = static_cast<long long>(t.rows) * t.cols;
            mctasks.push_back({t.replica_local, t.replica, n, w.mc_vecs});
            w.mc_vecs += n / 8;
            ++w.n_mc;
          }
          fslot_begin.push_back(static_cast<long long>(fpartial_count_));
          fslot_count.push_back(cnt);
          fslot_tensor.push_back(ti);
          fpartial_count_ += static_cast<size_t>(cnt);
        }
        const int tiles_c = (t.cols + kTile - 1) / kTile;
        const long long ntiles = static_cast<long long>((t.rows + kTile - 1) / kTile) * tiles_c;
        MomentumMatrixTask mt{};
        mt.g = t.g;
        mt.m = t.m;
        mt.rows = t.rows;
        mt.cols = t.cols;
        mt.ldx = c.ldn;
        mt.transposed = t.rows > t.cols ? 1 : 0;
        mt.tiles_c = tiles_c;
        mt.tile_start = w.tiles;
        const auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
        const bool vec = (t.cols % 8) == 0 && (c.ldn % 8) == 0 && a16(t.g) && a16(t.m) && a16(t.w) &&
                         (t.replica == nullptr || a16(t.replica));
        mt.vec = vec ? 1 : 0;
        mt.g_mc = t.g_mc;
        if (t.g_mc && !vec) return fail(OSH_ERR_UNSUPPORTED, "NVLS path needs the 128-bit layout");
        // workspace / partial pointers are offsets until the buffers exist
        mt.x0 = reinterpret_cast<__nv_bfloat16*>(c.x0 + static_cast<size_t>(b) * s.xb);
        ApplyTask at{};
        at.x = reinterpret_cast<const __nv_bfloat16*>(c.x0 + static_cast<size_t>(b) * s.xb);
        at.x_alt = reinterpret_cast<const __nv_bfloat16*>(c.x1 + static_cast<size_t>(b) * s.xb);
        at.w = t.w;
        at.replica = t.replica;
        at.rows = t.rows;
        at.cols = t.cols;
        at.ldx = c.ldn;
        at.transposed = mt.transposed;
        at.tile_start = w.tiles;
        at.tiles_c = tiles_c;
        at.vec = mt.vec;
        at.rep_mc = t.rep_mc;
        mtasks.push_back(mt);
        atasks.push_back(at);
        slot_begin.push_back(w.tiles);
        slot_count.push_back(static_cast<int>(ntiles));
        slot_tensor.push_back(ti);
        w.tiles += ntiles;
        if (!cfused) {
          w.nf_tiles = w.tiles;
          w.nf_elems += static_cast<double>(t.rows) * t.cols;
        }
        w.elems_matrix += static_cast<double>(t.rows) * t.cols;
        ++slot;
      }
      w.chunks.push_back(static_cast<int>(chunks_.size()));
      chunks_.push_back(c);
    }
    w.n_tasks = static_cast<int>(mtasks.size()) - w.task0;
    w.n_slots = slot - w.slot0;
    w.n_vec = static_cast<int>(vtasks.size()) - w.vec0;
    ws_bytes_ = std::max(ws_bytes_, off);
    max_tiles = std::max(max_tiles, w.tiles);
    waves_.push_back(w);
  }
  n_slots_ = slot;

  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_ws_), std::max<size_t>(ws_bytes_, 256)));
  if (!debug_poison()) OSH_CUDA_TRY(cudaMemset(d_ws_, 0, std::max<size_t>(ws_bytes_, 256)));
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_partial_),
                         sizeof(double) * static_cast<size_t>(max_tiles)));
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_scale_update_),
                         sizeof(float) * std::max(n_slots_, 1)));
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_scale_gram_),
                         sizeof(float) * std::max(n_slots_, 1)));
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_update_sq_),
                         sizeof(double) * std::max(n_tensors_, 1)));
  OSH_CUDA_TRY(cudaMemset(d_update_sq_, 0, sizeof(double) * std::max(n_tensors_, 1)));
  for (MomentumMatrixTask& mt : mtasks) {
    mt.x0 = reinterpret_cast<__nv_bfloat16*>(d_ws_ + reinterpret_cast<uintptr_t>(mt.x0));
    mt.partial = d_partial_ + mt.tile_start;  // local tile index is added in-kernel
  }
  for (ApplyTask& at : atasks) {
    at.x = reinterpret_cast<const __nv_bfloat16*>(d_ws_ + reinterpret_cast<uintptr_t>(at.x));
    at.x_alt = reinterpret_cast<const __nv_bfloat16*>(d_ws_ + reinterpret_cast<uintptr_t>(at.x_alt));
    at.partial = d_partial_ + at.tile_start;
  }
  for (MomentumVectorTask& v : vtasks)
    v.sq_norm = d_update_sq_ + reinterpret_cast<uintptr_t>(v.sq_norm);
  OSH_CUDA_TRY(upload(&d_mtasks_, mtasks));
  OSH_CUDA_TRY(upload(&d_atasks_, atasks));
  OSH_CUDA_TRY(upload(&d_vtasks_, vtasks));
  OSH_CUDA_TRY(upload(&d_slot_begin_, slot_begin));
  OSH_CUDA_TRY(upload(&d_slot_count_, slot_count));
  OSH_CUDA_TRY(upload(&d_slot_tensor_, slot_tensor));
  if (!ftargets.empty()) {
    OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_fpartial_), sizeof(double) * fpartial_count_));
    OSH_CUDA_TRY(cudaMemset(d_fpartial_, 0, sizeof(double) * fpartial_count_));
    std::vector<NsFinalTarget> ft(ftargets.size());
    for (size_t i = 0; i < ftargets.size(); ++i) {
      const MuonTensorDesc& t = tensors[ftargets[i].ti];
      // NVLS: FINAL writes this GPU's own slot; run_post re-stores it through
      // the multicast address (multimem.st from the epilogue stalls the MMAs)
      __nv_bfloat16* rep = t.rep_mc ? t.replica_local : t.replica;
      if (!make_final_target(&ft[i], t.w, rep, ftargets[i].m, ftargets[i].n,
                             t.rows > t.cols ? 1 : 0, d_fpartial_ + ftargets[i].poff))
        return fail(OSH_ERR_CUDA, "MuonEngine: cannot encode the FINAL TMA maps");
    }
    OSH_CUDA_TRY(upload(&d_ftargets_, ft));
    OSH_CUDA_TRY(upload(&d_mctasks_, mctasks));
    OSH_CUDA_TRY(upload(&d_fslot_begin_, fslot_begin));
    OSH_CUDA_TRY(upload(&d_fslot_count_, fslot_count));
    OSH_CUDA_TRY(upload(&d_fslot_tensor_, fslot_tensor));
  }
  // cost-balanced (LPT) tile schedules of the three GEMMs of every wave
  const char* aux = std::getenv("OSH_NS_AUX");
  fold_a_ = !(aux != nullptr && std::strcmp(aux, "1") == 0);
  const char* lpt = std::getenv("OSH_GEMM_LPT");
  lpt_ = !(lpt != nullptr && std::strcmp(lpt, "0") == 0);
  // tail-split GRAM (ns_gemm_stream_k_schedule) is opt-in: under the B200's
  // power cap the part-empty last round of a vocabulary GRAM costs nothing
  // measurable (idle SMs leave the busy ones more power), while the partial
  // slots cost traffic — DESIGN.md §3, profiles/r02_stream_k_ab.json
  const char* skv = std::getenv("OSH_STREAM_K");
  stream_k_ = skv != nullptr && std::strcmp(skv, "1") == 0;
  int sk_slots = 0;  // partial slots of the largest stream-K GRAM
  sched_symmetric_ = symmetric_;
  for (Wave& w : waves_) {
    if (w.n_tasks == 0 || !lpt_) continue;
    NsProblemDesc pd[3][kMaxProblems];
    problems(w, 0, pd[0], pd[1], pd[2]);
    const int modes[3] = {kEpiGram, kEpiPoly, kEpiUpdate};
    if (stream_k_) {  // GRAM of few long-K tiles (vocabulary matrices): stream-K
      std::vector<int> tl, off, slot, fix;
      std::vector<int2> kb;
      int total = 0, n_slots = 0;
      const int units = ns_gemm_stream_k_schedule(pd[0], static_cast<int>(w.chunks.size()), &tl, &off,
                                                  &kb, &slot, &fix, &n_slots, &total);
      if (units > 0) {
        NsSchedule& sc = w.sched[kEpiGram];
        int* d_tl = nullptr;
        int* d_off = nullptr;
        int* d_slot = nullptr;
        int* d_fix = nullptr;
        int2* d_kb = nullptr;
        OSH_CUDA_TRY(upload(&d_tl, tl));
        OSH_CUDA_TRY(upload(&d_off, off));
        OSH_CUDA_TRY(upload(&d_slot, slot));
        OSH_CUDA_TRY(upload(&d_fix, fix));
        OSH_CUDA_TRY(upload(&d_kb, kb));
        for (int* p : {d_tl, d_off, d_slot, d_fix}) sched_mem_.push_back(p);
        sched_mem_.push_back(reinterpret_cast<int*>(d_kb));
        sc.tiles = d_tl;
        sc.off = d_off;
        sc.units = units;
        sc.total_tiles = total;
        sc.kb = d_kb;
        sc.slot = d_slot;
        sc.fix = d_fix;
        sc.n_fix = static_cast<int>(fix.size() / 6);
        sc.n_slots = n_slots;
        sk_slots = std::max(sk_slots, n_slots);
      }
    }
    for (int m = 0; m < 3; ++m) {
      if (m == 0 && w.sched[kEpiGram].kb != nullptr) continue;  // stream-K above
      std::vector<int> tl, off;
      int total = 0;
      const int units = ns_gemm_schedule(modes[m], pd[m], static_cast<int>(w.chunks.size()), &tl, &off, &total);
      if (units == 0) continue;
      int* d_tl = nullptr;
      int* d_off = nullptr;
      OSH_CUDA_TRY(upload(&d_tl, tl));
      OSH_CUDA_TRY(upload(&d_off, off));
      sched_mem_.push_back(d_tl);
      sched_mem_.push_back(d_off);
      NsSchedule& sc = w.sched[modes[m]];
      sc.tiles = d_tl;
      sc.off = d_off;
      sc.units = units;
      sc.total_tiles = total;
    }
    // last iteration: UPDATE over the unfused prefix, FINAL over the fused rest
    const int nc = static_cast<int>(w.chunks.size());
    if (w.nf_chunks == nc) continue;  // nothing fused
    if (w.nf_chunks == 0) {
      w.sched[kEpiFinal] = w.sched[kEpiUpdate];  // the same tiles
      continue;
    }
    const std::pair<int, int> parts[2] = {{0, w.nf_chunks}, {w.nf_chunks, nc}};
    for (int part = 0; part < 2; ++part) {
      std::vector<int> tl, off;
      int total = 0;
      const int mode = part == 0 ? kEpiUpdate : kEpiFinal;
      const int units = ns_gemm_schedule(mode, pd[2] + parts[part].first,
                                         parts[part].second - parts[part].first, &tl, &off, &total);
      if (units == 0) continue;
      int* d_tl = nullptr;
      int* d_off = nullptr;
      OSH_CUDA_TRY(upload(&d_tl, tl));
      OSH_CUDA_TRY(upload(&d_off, off));
      sched_mem_.push_back(d_tl);
      sched_mem_.push_back(d_off);
      NsSchedule& sc = part == 0 ? w.sched_last_update : w.sched[kEpiFinal];
      sc.tiles = d_tl;
      sc.off = d_off;
      sc.units = units;
      sc.total_tiles = total;
    }
  }
  if (sk_slots > 0) {  // one fp32 partial workspace, reused by every wave's stream-K GRAM
    OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_sk_ws_),
                           sizeof(float) * static_cast<size_t>(sk_slots) * 256 * kNsBN));
    for (Wave& w : waves_)
      if (w.sched[kEpiGram].kb != nullptr) w.sched[kEpiGram].ws = d_sk_ws_;
  }
  OSH_CUDA_TRY(cudaDeviceSynchronize());
  return OSH_OK;
}

osh_status MuonEngine::begin_step(cudaStream_t s) {
  stats_ = NsLaunchStats{};
  OSH_CUDA_TRY(cudaMemsetAsync(d_update_sq_, 0, sizeof(double) * std::max(n_tensors_, 1), s));
  if (d_fpartial_ != nullptr)  // slots a CTA-group variant leaves unwritten stay zero
    OSH_CUDA_TRY(cudaMemsetAsync(d_fpartial_, 0, sizeof(double) * fpartial_count_, s));
  return OSH_OK;
}

osh_status MuonEngine::run_wave(int wi, const osh_muon_cfg& cfg, cudaStream_t s) {
  if (osh_status st = run_pre(wi, cfg, s); st != OSH_OK) return st;
  if (osh_status st = run_ns(wi, cfg, s); st != OSH_OK) return st;
  return run_post(wi, cfg, s);
}

// profile mode: CUDA events around each elementwise launch; `bytes` is the
// algorithmic HBM (or, NVLS, NVLink) traffic of the launch
osh_status MuonEngine::run_pre(int wi, const osh_muon_cfg& cfg, cudaStream_t s) {
  const Wave& w = waves_[wi];
  if (cfg.ns_steps < 1 && w.n_slots > 0)
    return fail(OSH_ERR_UNSUPPORTED, "MuonEngine: ns_steps must be >= 1 on the GPU path");
  const float beta = static_cast<float>(cfg.beta), lr = static_cast<float>(cfg.lr);
  const double ges = grad_dtype_ == kGradBF16 ? 2.0 : 4.0;
  const double elems = w.elems_matrix + w.elems_vector;
  const auto timed = [&](int mode, double bytes, auto&& launch) {
    return timed_elementwise(mode, bytes, elems, s, launch);
  };
  if (w.n_vec > 0)
    OSH_CUDA_TRY(timed(kModeElementwise + 0, w.elems_vector * (ges + 18.0), [&] {
      return launch_momentum_vector(d_vtasks_ + w.vec0, w.n_vec, grad_dtype_, beta, lr, s);
    }));
  if (w.n_tasks == 0) return OSH_OK;
  // g read, m read + write, bf16 X0 write
  OSH_CUDA_TRY(timed(kModeElementwise + 1, w.elems_matrix * (ges + 10.0), [&] {
    return launch_momentum_matrix(d_mtasks_ + w.task0, w.n_tasks, w.tiles, grad_dtype_, beta, s);
  }));
  OSH_CUDA_TRY(timed(kModeElementwise + 2, 0.0, [&] {
    return launch_ns_scales(d_partial_, d_slot_begin_ + w.slot0, d_slot_count_ + w.slot0,
                            d_scale_update_ + w.slot0, d_scale_gram_ + w.slot0, w.n_slots, s);
  }));
  return OSH_OK;
}

void MuonEngine::problems(const Wave& w, int it, NsProblemDesc* gram, NsProblemDesc* poly,
                          NsProblemDesc* upd) const {
  const bool first = it == 0;
  const int np = static_cast<int>(w.chunks.size());
  for (int q = 0; q < np; ++q) {
    const Chunk& c = chunks_[w.chunks[q]];
    const Shape sh = shape_of(c.m, c.n);
    uint8_t* xin = d_ws_ + ((it & 1) ? c.x1 : c.x0);
    uint8_t* xout = d_ws_ + ((it & 1) ? c.x0 : c.x1);
    const long long xbs = static_cast<long long>(sh.xb / 2), abs = static_cast<long long>(sh.ab / 2);
    const NsMatrixRef X = ref(xin, c.batch, c.m, c.n, c.ldn, xbs);
    const NsMatrixRef Xo = ref(xout, c.batch, c.m, c.n, c.ldn, xbs);
    const NsMatrixRef Am = ref(d_ws_ + c.a, c.batch, c.m, c.m, c.ldm, abs);
    const NsMatrixRef Bm = ref(d_ws_ + c.b, c.batch, c.m, c.m, c.ldm, abs);
    // OSH_UPPER_FORM=1 (opt-in): B = b A + c A^2 in the upper-tile form (no
    // lower-half stores; UPDATE / FINAL read the left-of-diagonal k-blocks of
    // B from the mirrored tiles). Measured against the mirrored step it is
    // slower inside the step (UPDATE / FINAL with MN-major A k-blocks beside
    // the momentum pass) though not in isolation, and POLY reading A through
    // the mirror is 13 % slower in isolation (profiles/r02_upper_form_ab.json),
    // so the Muon step keeps mirrored matrices by default; the Shampoo Newton
    // products use the form (shampoo_engine.cu).
    const int sym = symmetric_ ? 1 : 0;
    const int up = symmetric_ && upper_form_ ? 1 : 0;
    gram[q] = NsProblemDesc{X, X, 0, Am, NsMatrixRef{},
                            first ? d_scale_gram_ + c.slot0 : nullptr, nullptr, sym};
    poly[q] = NsProblemDesc{Am, Am, 0, Bm, Am, nullptr, nullptr, up ? 3 : sym};
    upd[q] = NsProblemDesc{Bm, X, 1, Xo, X, first ? d_scale_update_ + c.slot0 : nullptr,
                           nullptr, 0};
    upd[q].a_upper = up;
  }
}

osh_status MuonEngine::run_ns(int wi, const osh_muon_cfg& cfg, cudaStream_t s) {
  const Wave& w = waves_[wi];
  if (w.n_tasks == 0) return OSH_OK;
  const int np = static_cast<int>(w.chunks.size());
  for (int it = 0; it < cfg.ns_steps; ++it) {
    NsProblemDesc gram[kMaxProblems], poly[kMaxProblems], upd[kMaxProblems];
    problems(w, it, gram, poly, upd);
    const auto timed_launch = [&](int mode, const NsProblemDesc* pd, float a, float b, float l) {
      const NsSchedule* sc = lpt_ && sched_symmetric_ == symmetric_ ? &w.sched[mode] : nullptr;
      return timed_gemm(mode, pd, np, a, b, s, sc, l);
    };
    // B' = a I + b A + c A^2 in the POLY epilogue, X' = s B' X: the UPDATE
    // epilogue then reads no aux (one fewer pass over X per iteration);
    // OSH_NS_AUX=1 restores X' = s (a X + B X) with the aux read
    cudaError_t e = timed_launch(kEpiGram, gram, 0.f, 0.f, 0.f);
    if (e == cudaSuccess)
      e = timed_launch(kEpiPoly, poly, static_cast<float>(cfg.ns_b), static_cast<float>(cfg.ns_c),
                       fold_a_ ? static_cast<float>(cfg.ns_a) : 0.f);
    const int nf = w.nf_chunks;
    if (e == cudaSuccess && nf < np && it + 1 == cfg.ns_steps) {
      // last iteration: fused chunks apply W -= lr * X' in the FINAL epilogue
      // (no X' store, no apply pass); unfused ones (a prefix) UPDATE as usual
      const float alpha = fold_a_ ? 0.f : static_cast<float>(cfg.ns_a);
      for (int q = nf; q < np; ++q) upd[q].final_targets = d_ftargets_ + chunks_[w.chunks[q]].ftarget0;
      if (nf > 0) {
        const NsSchedule* sc = lpt_ && sched_symmetric_ == symmetric_ ? &w.sched_last_update : nullptr;
        e = timed_gemm(kEpiUpdate, upd, nf, alpha, 0.f, s, sc, 0.f);
      }
      if (e == cudaSuccess) {
        const NsSchedule* sc = lpt_ && sched_symmetric_ == symmetric_ ? &w.sched[kEpiFinal] : nullptr;
        e = timed_gemm(kEpiFinal, upd + nf, np - nf, alpha, 0.f, s, sc, static_cast<float>(cfg.lr));
      }
    } else if (e == cudaSuccess) {
      e = timed_launch(kEpiUpdate, upd, fold_a_ ? 0.f : static_cast<float>(cfg.ns_a), 0.f, 0.f);
    }
    if (e != cudaSuccess)
      return fail(OSH_ERR_CUDA, std::string("MuonEngine: ns_gemm_launch: ") + cudaGetErrorString(e));
  }
  return OSH_OK;
}

osh_status MuonEngine::run_post(int wi, const osh_muon_cfg& cfg, cudaStream_t s) {
  const Wave& w = waves_[wi];
  if (w.n_tasks == 0) return OSH_OK;
  const float lr = static_cast<float>(cfg.lr);
  const double elems = w.elems_matrix + w.elems_vector;
  const auto timed = [&](int mode, double bytes, auto&& launch) {
    return timed_elementwise(mode, bytes, elems, s, launch);
  };
  // fused tensors: W and the replica were written by FINAL (NVLS: this GPU's
  // slot, now spread to every GPU through the multicast address — the AG-v);
  // their norms are the FINAL epilogue partials
  if (w.n_mc > 0)
    OSH_CUDA_TRY(timed(kModeElementwise + 5, 2.0 * static_cast<double>(w.mc_vecs) * 8, [&] {
      return launch_mc_copy(d_mctasks_ + w.mc0, w.n_mc, w.mc_vecs, s);
    }));
  if (w.nf_slots < w.n_slots)
    OSH_CUDA_TRY(timed(kModeElementwise + 4, 0.0, [&] {
      return launch_partial_sums(d_fpartial_, d_fslot_begin_ + w.fslot0, d_fslot_count_ + w.fslot0,
                                 d_fslot_tensor_ + w.fslot0, d_update_sq_, w.n_slots - w.nf_slots, s);
    }));
  if (w.nf_tasks == 0) return OSH_OK;
  // unfused prefix: after k iterations the iterate sits in X0 (k even) or X1
  // (k odd); X read, w read + write, bf16 replica write
  OSH_CUDA_TRY(timed(kModeElementwise + 3, w.nf_elems * 12.0, [&] {
    return launch_apply_update(d_atasks_ + w.task0, w.nf_tasks, w.nf_tiles, lr, cfg.ns_steps & 1, s);
  }));
  OSH_CUDA_TRY(timed(kModeElementwise + 4, 0.0, [&] {
    return launch_partial_sums(d_partial_, d_slot_begin_ + w.slot0, d_slot_count_ + w.slot0,
                               d_slot_tensor_ + w.slot0, d_update_sq_, w.nf_slots, s);
  }));
  return OSH_OK;
}

}  // namespace osh
