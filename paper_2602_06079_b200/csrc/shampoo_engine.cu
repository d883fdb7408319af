// ShampooEngine implementation (see shampoo_engine.cuh).
#include "shampoo_engine.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>

#include "status.hpp"

namespace osh {
namespace {

size_t rup(size_t v, size_t a) { return (v + a - 1) / a * a; }
long long tiles_of(int rows, int cols) {
  return static_cast<long long>((rows + kTile - 1) / kTile) * ((cols + kTile - 1) / kTile);
}

template <typename T>
cudaError_t upload(T** dst, const std::vector<T>& src) {
  *dst = nullptr;
  if (src.empty()) return cudaSuccess;
  cudaError_t e = dev_alloc(reinterpret_cast<void**>(dst), sizeof(T) * src.size());
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice);
}

NsMatrixRef mref(const void* p, int batch, int rows, int cols, long long ld, long long bstride) {
  NsMatrixRef r;
  r.ptr = p;
  r.batch = batch;
  r.rows = rows;
  r.cols = cols;
  r.ld = ld;
  r.bstride = bstride;
  return r;
}

struct BlockGeom {
  int r0, p, c0, q;
};

std::vector<BlockGeom> blocks_of(int rows, int cols, int b) {
  std::vector<BlockGeom> out;
  for (int r0 = 0; r0 < rows; r0 += b)
    for (int c0 = 0; c0 < cols; c0 += b)
      out.push_back({r0, std::min(b, rows - r0), c0, std::min(b, cols - c0)});
  return out;
}

int seg_of(int n) { return static_cast<int>(rup(static_cast<size_t>(n), 8)); }

// per-block workspace: G, U1, U ([p][ldq]), G^T ([q][ldp]) and the split
// Newton matrices (7 per side)
size_t block_ws(int p, int q) {
  const size_t ldp = rup(p, 64), ldq = rup(q, 64);
  const size_t sp = seg_of(p), sq = seg_of(q);
  return rup(2 * p * ldq, 256) * 3 + rup(2 * q * ldp, 256) + 7 * rup(2 * p * 4 * sp, 256) +
         7 * rup(2 * q * 4 * sq, 256);
}

}  // namespace

ShampooEngine::~ShampooEngine() { release(); }

void ShampooEngine::release() {
  for (void* p : {static_cast<void*>(d_ws_), static_cast<void*>(d_state_),
                  static_cast<void*>(d_partial_), static_cast<void*>(d_gsq_),
                  static_cast<void*>(d_usq_), static_cast<void*>(d_ssq_),
                  static_cast<void*>(d_graft_),
                  static_cast<void*>(d_update_sq_), static_cast<void*>(d_prep_),
                  static_cast<void*>(d_usq_tasks_), static_cast<void*>(d_ssq_tasks_),
                  static_cast<void*>(d_root_), static_cast<void*>(d_newton_),
                  static_cast<void*>(d_extract_), static_cast<void*>(d_apply_),
                  static_cast<void*>(d_sgd_), static_cast<void*>(d_blockrefs_),
                  static_cast<void*>(d_symf_),
                  static_cast<void*>(d_slot_begin_), static_cast<void*>(d_slot_count_),
                  static_cast<void*>(d_slot_target_)})
    cudaFree(p);
  d_ws_ = d_state_ = nullptr;
  d_partial_ = d_gsq_ = d_usq_ = d_ssq_ = d_update_sq_ = nullptr;
  d_sroot_ = d_graft_ = nullptr;
  d_prep_ = nullptr;
  d_usq_tasks_ = nullptr;
  d_ssq_tasks_ = nullptr;
  d_root_ = nullptr;
  d_newton_ = d_extract_ = nullptr;
  d_apply_ = nullptr;
  d_sgd_ = nullptr;
  d_blockrefs_ = nullptr;
  d_symf_ = nullptr;
  d_slot_begin_ = nullptr;
  d_slot_count_ = d_slot_target_ = nullptr;
  waves_.clear();
}

const char* ShampooEngine::elementwise_name(int mode) const {
  static const char* kNames[] = {"sh_prep",   "sh_sumsq", "sh_root_init", "sh_newton_t",
                                 "sh_extract", "sh_graft", "sh_apply",     "sh_sgd",
                                 "partial_sums"};
  const int i = mode - kModeElementwise;
  return i >= 0 && i < 9 ? kNames[i] : "elementwise";
}

osh_status ShampooEngine::build(const std::vector<MuonTensorDesc>& tensors, int grad_dtype,
                                size_t budget, int min_waves, bool /*double_buffer*/) {
  release();
  if (cfg_.block < 64 || cfg_.block % 64 != 0)
    return fail(OSH_ERR_CONFIG, "Shampoo block size must be a positive multiple of 64");
  if (cfg_.precond_every < 1 || cfg_.newton_iters < 1)
    return fail(OSH_ERR_CONFIG, "Shampoo precond_every and newton_iters must be >= 1");
  n_tensors_ = static_cast<int>(tensors.size());
  grad_dtype_ = grad_dtype;
  step_ = -1;
  const int B = cfg_.block;
  auto pre = [&](const MuonTensorDesc& t) { return t.is_matrix && !t.vocab_space; };

  // ---- waves: consecutive tensors (declaration order) within the budget
  size_t total = 0, largest = 0;
  std::vector<size_t> cost(tensors.size(), 0);
  for (size_t i = 0; i < tensors.size(); ++i) {
    if (!pre(tensors[i])) continue;
    for (const BlockGeom& b : blocks_of(tensors[i].rows, tensors[i].cols, B)) cost[i] += block_ws(b.p, b.q);
    total += cost[i];
    largest = std::max(largest, cost[i]);
  }
  if (largest > budget)
    return fail(OSH_ERR_OOM, "ShampooEngine: one tensor needs " + std::to_string(largest) +
                                 " workspace bytes, budget is " + std::to_string(budget) +
                                 " (lower the block size)");
  // Waves run back to back (no overlap to feed): as large as the budget
  // allows, so the batched GEMMs and Newton iterations see full batches;
  // min_waves only matters for bucket-pipelined collectives (NCCL path).
  size_t cap = budget;
  if (min_waves > 1 && min_waves <= 4)
    cap = std::min(cap, std::max(largest, (total + min_waves - 1) / min_waves));
  std::vector<std::vector<int>> members(1);
  size_t used = 0;
  for (int i = 0; i < n_tensors_; ++i) {
    if (cost[i] > 0 && used > 0 && used + cost[i] > cap) {
      members.emplace_back();
      used = 0;
    }
    used += cost[i];
    members.back().push_back(i);
  }
  if (members.back().empty()) members.pop_back();

  // ---- classes, offsets and task tables
  std::vector<ShPrepTask> prep;
  std::vector<ShMatTask<__nv_bfloat16>> usq;
  std::vector<ShMatTask<float>> ssq;
  std::vector<SymFillTask> symf;
  std::vector<ShRootTask> root;
  std::vector<ShNewtonTask> newton0, newton1, extract;
  std::vector<ShApplyTask> apply;
  std::vector<ShSgdTask> sgd;
  std::vector<ShBlockRef> brefs;
  std::vector<long long> slot_begin;
  std::vector<int> slot_count, slot_target;
  size_t state_off = 0, partial_off = 0;
  int n_blocks = 0, n_stats = 0;
  ws_bytes_ = 0;
  // We build tasks with byte offsets stored in the pointer fields
  // (reinterpret_cast) and add the base addresses after allocation.
  auto off_ptr = [](size_t off) { return reinterpret_cast<void*>(off); };

  std::vector<size_t> apply_bref_index;

  for (size_t wi = 0; wi < members.size(); ++wi) {
    Wave w;
    w.first_bucket = tensors[members[wi].front()].bucket;
    w.last_bucket = tensors[members[wi].back()].bucket;
    std::map<std::pair<int, int>, int> cls_of;
    // blocks of every preconditioned tensor, grouped by class in first-seen order
    struct TB {
      int tensor, idx;  // idx = row-major block index within the tensor
      BlockGeom g;
    };
    std::vector<std::vector<TB>> by_cls;
    for (const int ti : members[wi]) {
      const MuonTensorDesc& t = tensors[ti];
      if (!pre(t)) continue;
      const auto bl = blocks_of(t.rows, t.cols, B);
      for (size_t k = 0; k < bl.size(); ++k) {
        const std::pair<int, int> key{bl[k].p, bl[k].q};
        auto it = cls_of.find(key);
        if (it == cls_of.end()) {
          it = cls_of.emplace(key, static_cast<int>(by_cls.size())).first;
          by_cls.emplace_back();
        }
        by_cls[it->second].push_back({ti, static_cast<int>(k), bl[k]});
      }
    }
    // global block id of (tensor, idx)
    std::map<std::pair<int, int>, int> gid;
    std::map<std::pair<int, int>, std::pair<size_t, long long>> u_of;  // -> (ws offset, ldq)
    size_t off = 0;
    w.prep.first = static_cast<int>(prep.size());
    w.usq.first = static_cast<int>(usq.size());
    w.ssq.first = static_cast<int>(ssq.size());
    w.symf.first = static_cast<int>(symf.size());
    w.root_init[0].first = static_cast<int>(root.size());
    w.newton[0].first = static_cast<int>(newton0.size());
    w.newton[1].first = static_cast<int>(newton1.size());
    w.extract[0].first = static_cast<int>(extract.size());
    const size_t prep_base = partial_off;
    long long prep_tiles = 0;
    for (size_t c = 0; c < by_cls.size(); ++c) {
      Cls k;
      k.p = by_cls[c].front().g.p;
      k.q = by_cls[c].front().g.q;
      k.ldp = static_cast<int>(rup(k.p, 64));
      k.ldq = static_cast<int>(rup(k.q, 64));
      k.nb = static_cast<int>(by_cls[c].size());
      k.block0 = n_blocks;
      k.stat0 = n_stats;
      const size_t gq = rup(2ull * k.p * k.ldq, 256), gtp = rup(2ull * k.q * k.ldp, 256);
      k.gb = off; off += gq * k.nb;
      k.gbt = off; off += gtp * k.nb;
      k.u1 = off; off += gq * k.nb;
      k.u = off; off += gq * k.nb;
      const size_t s5p = rup(2ull * k.p * 4 * seg_of(k.p), 256), s5q = rup(2ull * k.q * 4 * seg_of(k.q), 256);
      for (size_t* z : {&k.xl[0], &k.xl[1], &k.ml[0], &k.ml[1], &k.tl, &k.t2l, &k.t4l}) {
        *z = off;
        off += s5p * k.nb;
      }
      for (size_t* z : {&k.xr[0], &k.xr[1], &k.mr[0], &k.mr[1], &k.tr, &k.t2r, &k.t4r}) {
        *z = off;
        off += s5q * k.nb;
      }
      const size_t Lb = rup(4ull * k.p * k.ldp, 256), Rb = rup(4ull * k.q * k.ldq, 256);
      const size_t PLb = rup(2ull * k.p * k.ldp, 256), PRb = rup(2ull * k.q * k.ldq, 256);
      k.L = state_off; state_off += Lb * k.nb;
      k.R = state_off; state_off += Rb * k.nb;
      k.PL = state_off; state_off += PLb * k.nb;
      k.PR = state_off; state_off += PRb * k.nb;
      for (int i = 0; i < k.nb; ++i) {
        const TB& tb = by_cls[c][i];
        const MuonTensorDesc& t = tensors[tb.tensor];
        gid[{tb.tensor, tb.idx}] = n_blocks + i;
        u_of[{tb.tensor, tb.idx}] = {k.u + gq * i, k.ldq};
        ShPrepTask pt{};
        pt.g = static_cast<const uint8_t*>(t.g);  // real pointer (grad buffer)
        pt.g_ld = t.cols;
        pt.g_mc = t.g_mc;
        pt.vec = (t.cols % 8 == 0 && tb.g.c0 % 8 == 0 && tb.g.q % 8 == 0 &&
                  (reinterpret_cast<uintptr_t>(t.g) & 15) == 0)
                     ? 1
                     : 0;
        if (t.g_mc && !pt.vec) return fail(OSH_ERR_UNSUPPORTED, "NVLS path needs the 128-bit layout");
        pt.r0 = tb.g.r0;
        pt.c0 = tb.g.c0;
        pt.p = k.p;
        pt.q = k.q;
        pt.gb = static_cast<__nv_bfloat16*>(off_ptr(k.gb + gq * i));
        pt.gbt = static_cast<__nv_bfloat16*>(off_ptr(k.gbt + gtp * i));
        pt.ldq = k.ldq;
        pt.ldp = k.ldp;
        pt.tile_start = prep_tiles;
        pt.tiles_c = (k.q + kTile - 1) / kTile;
        pt.partial = reinterpret_cast<double*>(off_ptr(prep_base));  // patched: d_partial_ + base
        slot_begin.push_back(static_cast<long long>(prep_base) + prep_tiles);
        slot_count.push_back(static_cast<int>(tiles_of(k.p, k.q)));
        slot_target.push_back(n_blocks + i);
        prep_tiles += tiles_of(k.p, k.q);
        prep.push_back(pt);
      }
      n_blocks += k.nb;
      n_stats += 2 * k.nb;
      w.cls.push_back(k);
    }
    w.prep.count = static_cast<int>(prep.size()) - w.prep.first;
    w.prep.tiles = prep_tiles;
    w.slot_g = {static_cast<int>(slot_begin.size()) - w.prep.count, w.prep.count, 0};
    partial_off += static_cast<size_t>(prep_tiles);

    // U sums of squares, per block (same order as the blocks)
    const size_t u_base = partial_off;
    long long ut = 0;
    w.slot_u.first = static_cast<int>(slot_begin.size());
    for (const Cls& k : w.cls) {
      const size_t gq = rup(2ull * k.p * k.ldq, 256);
      for (int i = 0; i < k.nb; ++i) {
        ShMatTask<__nv_bfloat16> mt{};
        mt.src = static_cast<const __nv_bfloat16*>(off_ptr(k.u + gq * i));
        mt.ld = k.ldq;
        mt.rows = k.p;
        mt.cols = k.q;
        mt.tile_start = ut;
        mt.tiles_c = (k.q + kTile - 1) / kTile;
        mt.partial = reinterpret_cast<double*>(off_ptr(u_base));
        slot_begin.push_back(static_cast<long long>(u_base) + ut);
        slot_count.push_back(static_cast<int>(tiles_of(k.p, k.q)));
        slot_target.push_back(k.block0 + i);
        ut += tiles_of(k.p, k.q);
        usq.push_back(mt);
      }
    }
    w.usq.count = static_cast<int>(usq.size()) - w.usq.first;
    w.usq.tiles = ut;
    w.slot_u.count = static_cast<int>(slot_begin.size()) - w.slot_u.first;
    partial_off += static_cast<size_t>(ut);

    // statistics matrices: sums of squares, root init, Newton T, extract
    const size_t s_base = partial_off;
    long long st = 0, rt = 0;
    w.slot_s.first = static_cast<int>(slot_begin.size());
    for (const Cls& k : w.cls) {
      for (int side = 0; side < 2; ++side) {
        const int n = side == 0 ? k.p : k.q;
        const int ldn = side == 0 ? k.ldp : k.ldq;
        const int sg = seg_of(n);
        const size_t s5 = rup(2ull * n * 4 * sg, 256);
        const size_t Sb = rup(4ull * n * ldn, 256), Pb = rup(2ull * n * ldn, 256);
        for (int i = 0; i < k.nb; ++i) {
          const int stat = k.stat0 + side * k.nb + i;
          const size_t S = (side == 0 ? k.L : k.R) + Sb * i;
          ShMatTask<float> mt{};
          mt.src = static_cast<const float*>(off_ptr(S));
          mt.ld = ldn;
          mt.rows = n;
          mt.cols = n;
          mt.tile_start = st;
          mt.tiles_c = (n + kTile - 1) / kTile;
          mt.partial = reinterpret_cast<double*>(off_ptr(s_base));
          slot_begin.push_back(static_cast<long long>(s_base) + st);
          slot_count.push_back(static_cast<int>(tiles_of(n, n)));
          slot_target.push_back(stat);
          st += tiles_of(n, n);
          ssq.push_back(mt);
          {
            SymFillTask sf{};
            sf.s = static_cast<float*>(off_ptr(S));
            sf.ld = ldn;
            sf.n = n;
            const int T = (n + 31) / 32;
            sf.tiles = T * (T + 1) / 2;
            sf.tile_start = w.symf.tiles;
            w.symf.tiles += sf.tiles;
            symf.push_back(sf);
          }
          ShRootTask r{};
          r.s = static_cast<const float*>(off_ptr(S));
          r.lds = ldn;
          r.a5 = static_cast<__nv_bfloat16*>(off_ptr((side == 0 ? k.ml[0] : k.mr[0]) + s5 * i));
          r.x5 = static_cast<__nv_bfloat16*>(off_ptr((side == 0 ? k.xl[0] : k.xr[0]) + s5 * i));
          r.ld5 = 4ll * sg;
          r.n = n;
          r.sumsq = reinterpret_cast<const double*>(static_cast<uintptr_t>(stat));  // patched
          r.tile_start = rt;
          r.tiles_c = (n + kTile - 1) / kTile;
          {
            const size_t oth[5] = {side == 0 ? k.xl[1] : k.xr[1], side == 0 ? k.ml[1] : k.mr[1],
                                   side == 0 ? k.tl : k.tr, side == 0 ? k.t2l : k.t2r,
                                   side == 0 ? k.t4l : k.t4r};
            for (int o = 0; o < 5; ++o)
              r.others[o] = static_cast<__nv_bfloat16*>(off_ptr(oth[o] + s5 * i));
          }
          root.push_back(r);
          for (int par = 0; par < 2; ++par) {
            ShNewtonTask nt{};
            nt.src5 = static_cast<const __nv_bfloat16*>(
                off_ptr((side == 0 ? k.ml[par] : k.mr[par]) + s5 * i));
            nt.dst = static_cast<__nv_bfloat16*>(off_ptr((side == 0 ? k.tl : k.tr) + s5 * i));
            nt.ld5 = 4ll * sg;
            nt.ldd = 4ll * sg;
            nt.n = n;
            nt.tile_start = rt;
            nt.tiles_c = (n + kTile - 1) / kTile;
            (par == 0 ? newton0 : newton1).push_back(nt);
          }
          ShNewtonTask et{};
          const int fin = cfg_.newton_iters & 1;
          et.src5 = static_cast<const __nv_bfloat16*>(
              off_ptr((side == 0 ? k.xl[fin] : k.xr[fin]) + s5 * i));
          et.dst = static_cast<__nv_bfloat16*>(off_ptr((side == 0 ? k.PL : k.PR) + Pb * i));
          et.ld5 = 4ll * sg;
          et.ldd = ldn;
          et.n = n;
          et.tile_start = rt;
          et.tiles_c = (n + kTile - 1) / kTile;
          extract.push_back(et);
          rt += tiles_of(n, n);
        }
      }
    }
    w.ssq.count = static_cast<int>(ssq.size()) - w.ssq.first;
    w.symf.count = static_cast<int>(symf.size()) - w.symf.first;
    w.ssq.tiles = st;
    w.slot_s.count = static_cast<int>(slot_begin.size()) - w.slot_s.first;
    partial_off += static_cast<size_t>(st);
    w.root_init[0].count = static_cast<int>(root.size()) - w.root_init[0].first;
    w.root_init[0].tiles = rt;
    w.newton[0].count = w.newton[1].count = w.root_init[0].count;
    w.newton[0].tiles = w.newton[1].tiles = rt;
    w.extract[0].count = w.root_init[0].count;
    w.extract[0].tiles = rt;

    // apply (preconditioned tensors) and sgd (vectors / vocabulary matrices)
    const size_t t_base = partial_off;
    long long at = 0;
    w.apply.first = static_cast<int>(apply.size());
    w.sgd.first = static_cast<int>(sgd.size());
    w.slot_t.first = static_cast<int>(slot_begin.size());
    for (const int ti : members[wi]) {
      const MuonTensorDesc& t = tensors[ti];
      const long long t0 = at;
      if (pre(t)) {
        ShApplyTask a{};
        a.w = t.w;
        a.m = t.m;
        a.replica = t.replica;
        a.rep_mc = t.rep_mc;
        a.rows = t.rows;
        a.cols = t.cols;
        a.block = B;
        a.blocks_c = (t.cols + B - 1) / B;
        a.vec = (t.cols % 8 == 0 && (reinterpret_cast<uintptr_t>(t.w) & 15) == 0 &&
                 (reinterpret_cast<uintptr_t>(t.m) & 15) == 0 &&
                 (t.replica == nullptr || (reinterpret_cast<uintptr_t>(t.replica) & 15) == 0))
                    ? 1
                    : 0;
        if (t.rep_mc && !a.vec) return fail(OSH_ERR_UNSUPPORTED, "NVLS path needs the 128-bit layout");
        apply_bref_index.push_back(brefs.size());
        const int nbt = static_cast<int>(blocks_of(t.rows, t.cols, B).size());
        for (int k = 0; k < nbt; ++k) {
          const auto uo = u_of.at({ti, k});
          ShBlockRef br{};
          br.u = static_cast<const __nv_bfloat16*>(off_ptr(uo.first));
          br.ldu = uo.second;
          br.scale = reinterpret_cast<const float*>(static_cast<uintptr_t>(gid.at({ti, k})));
          brefs.push_back(br);
        }
        a.tile_start = at;
        a.tiles_c = (t.cols + kTile - 1) / kTile;
        a.partial = reinterpret_cast<double*>(off_ptr(t_base));
        at += tiles_of(t.rows, t.cols);
        apply.push_back(a);
        w.elems_pre += static_cast<double>(t.rows) * t.cols;
      }
      slot_begin.push_back(static_cast<long long>(t_base) + t0);
      slot_count.push_back(static_cast<int>(at - t0));
      slot_target.push_back(ti);
    }
    w.apply.count = static_cast<int>(apply.size()) - w.apply.first;
    w.apply.tiles = at;
    // sgd tensors: tiles after the apply tiles of this wave, same partial region
    long long sgt = 0;
    for (const int ti : members[wi]) {
      const MuonTensorDesc& t = tensors[ti];
      if (pre(t)) continue;
      ShSgdTask s{};
      s.g = t.g;
      s.g_mc = t.g_mc;
      s.rep_mc = t.rep_mc;
      s.m = t.m;
      s.w = t.w;
      s.replica = t.replica;
      s.n = static_cast<long long>(t.rows) * t.cols;
      s.vec = (s.n % 8 == 0 && (reinterpret_cast<uintptr_t>(t.g) & 15) == 0 &&
               (reinterpret_cast<uintptr_t>(t.w) & 15) == 0 &&
               (reinterpret_cast<uintptr_t>(t.m) & 15) == 0 &&
               (t.replica == nullptr || (reinterpret_cast<uintptr_t>(t.replica) & 15) == 0))
                  ? 1
                  : 0;
      if ((t.g_mc || t.rep_mc) && !s.vec)
        return fail(OSH_ERR_UNSUPPORTED, "NVLS path needs the 128-bit layout");
      s.tile_start = sgt;
      s.partial = reinterpret_cast<double*>(off_ptr(t_base + static_cast<size_t>(at)));
      const long long nt = (s.n + kShSgdTile - 1) / kShSgdTile;
      // the tensor's slot (pushed above with count 0) covers its sgd tiles
      for (int si = w.slot_t.first; si < static_cast<int>(slot_begin.size()); ++si)
        if (slot_target[si] == ti) {
          slot_begin[si] = static_cast<long long>(t_base + at) + sgt;
          slot_count[si] = static_cast<int>(nt);
        }
      sgt += nt;
      sgd.push_back(s);
      w.elems_sgd += static_cast<double>(s.n);
    }
    w.sgd.count = static_cast<int>(sgd.size()) - w.sgd.first;
    w.sgd.tiles = sgt;
    w.slot_t.count = static_cast<int>(slot_begin.size()) - w.slot_t.first;
    partial_off += static_cast<size_t>(at + sgt);
    w.n_blocks = 0;
    for (const Cls& k : w.cls) w.n_blocks += k.nb;
    w.n_stats = 2 * w.n_blocks;
    ws_bytes_ = std::max(ws_bytes_, off);
    waves_.push_back(std::move(w));
  }
  n_stats_total_ = n_stats;
  const size_t sroot_off = rup(state_off, 256);  // root scales live in the state buffer too
  state_off = sroot_off + rup(sizeof(float) * std::max(n_stats, 1), 256);
  state_bytes_ = state_off;

  // ---- allocate and patch
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_ws_), std::max<size_t>(ws_bytes_, 256)));
  OSH_CUDA_TRY(cudaMemset(d_ws_, 0, std::max<size_t>(ws_bytes_, 256)));  // split padding = 0
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_state_), std::max<size_t>(state_bytes_, 256)));
  OSH_CUDA_TRY(cudaMemset(d_state_, 0, std::max<size_t>(state_bytes_, 256)));
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_partial_), sizeof(double) * std::max<size_t>(partial_off, 1)));
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_gsq_), sizeof(double) * std::max(n_blocks, 1)));
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_usq_), sizeof(double) * std::max(n_blocks, 1)));
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_graft_), sizeof(float) * std::max(n_blocks, 1)));
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_ssq_), sizeof(double) * std::max(n_stats, 1)));
  d_sroot_ = reinterpret_cast<float*>(d_state_ + sroot_off);  // part of the checkpointed state
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_update_sq_), sizeof(double) * std::max(n_tensors_, 1)));
  OSH_CUDA_TRY(cudaMemset(d_update_sq_, 0, sizeof(double) * std::max(n_tensors_, 1)));
  auto ws = [&](const void* p) { return d_ws_ + reinterpret_cast<uintptr_t>(p); };
  auto stp = [&](const void* p) { return d_state_ + reinterpret_cast<uintptr_t>(p); };
  auto part = [&](const double* p) { return d_partial_ + reinterpret_cast<uintptr_t>(p); };
  for (ShPrepTask& t : prep) {
    t.gb = reinterpret_cast<__nv_bfloat16*>(ws(t.gb));
    t.gbt = reinterpret_cast<__nv_bfloat16*>(ws(t.gbt));
    t.partial = part(t.partial);
  }
  for (auto& t : usq) {
    t.src = reinterpret_cast<const __nv_bfloat16*>(ws(t.src));
    t.partial = part(t.partial);
  }
  for (auto& t : ssq) {
    t.src = reinterpret_cast<const float*>(stp(t.src));
    t.partial = part(t.partial);
  }
  for (auto& t : symf) t.s = reinterpret_cast<float*>(stp(t.s));
  for (auto& t : root) {
    t.s = reinterpret_cast<const float*>(stp(t.s));
    t.a5 = reinterpret_cast<__nv_bfloat16*>(ws(t.a5));
    t.x5 = reinterpret_cast<__nv_bfloat16*>(ws(t.x5));
    for (auto& o : t.others) o = reinterpret_cast<__nv_bfloat16*>(ws(o));
    t.sumsq = d_ssq_ + reinterpret_cast<uintptr_t>(t.sumsq);
  }
  for (auto* vec : {&newton0, &newton1})
    for (auto& t : *vec) {
      t.src5 = reinterpret_cast<const __nv_bfloat16*>(ws(t.src5));
      t.dst = reinterpret_cast<__nv_bfloat16*>(ws(t.dst));
    }
  for (auto& t : extract) {
    t.src5 = reinterpret_cast<const __nv_bfloat16*>(ws(t.src5));
    t.dst = reinterpret_cast<__nv_bfloat16*>(stp(t.dst));
  }
  for (auto& b : brefs) {
    b.u = reinterpret_cast<const __nv_bfloat16*>(ws(b.u));
    b.scale = d_graft_ + reinterpret_cast<uintptr_t>(b.scale);
  }
  for (auto& t : sgd) t.partial = part(t.partial);
  OSH_CUDA_TRY(upload(&d_blockrefs_, brefs));
  for (size_t i = 0; i < apply.size(); ++i) {
    apply[i].blocks = d_blockrefs_ + apply_bref_index[i];
    apply[i].partial = part(apply[i].partial);
  }
  std::vector<ShNewtonTask> newton(newton0);
  newton.insert(newton.end(), newton1.begin(), newton1.end());
  OSH_CUDA_TRY(upload(&d_prep_, prep));
  OSH_CUDA_TRY(upload(&d_usq_tasks_, usq));
  OSH_CUDA_TRY(upload(&d_ssq_tasks_, ssq));
  OSH_CUDA_TRY(upload(&d_symf_, symf));
  OSH_CUDA_TRY(upload(&d_root_, root));
  OSH_CUDA_TRY(upload(&d_newton_, newton));
  OSH_CUDA_TRY(upload(&d_extract_, extract));
  OSH_CUDA_TRY(upload(&d_apply_, apply));
  OSH_CUDA_TRY(upload(&d_sgd_, sgd));
  OSH_CUDA_TRY(upload(&d_slot_begin_, slot_begin));
  OSH_CUDA_TRY(upload(&d_slot_count_, slot_count));
  OSH_CUDA_TRY(upload(&d_slot_target_, slot_target));
  // newton1 tasks follow newton0 in one array
  for (Wave& w : waves_) w.newton[1].first += static_cast<int>(newton0.size());
  OSH_CUDA_TRY(cudaDeviceSynchronize());
  return OSH_OK;
}

osh_status ShampooEngine::begin_step(cudaStream_t s) {
  ++step_;
  stats_ = NsLaunchStats{};
  OSH_CUDA_TRY(cudaMemsetAsync(d_update_sq_, 0, sizeof(double) * std::max(n_tensors_, 1), s));
  return OSH_OK;
}

osh_status ShampooEngine::run_wave(int wi, const osh_muon_cfg& mcfg, cudaStream_t s) {
  const Wave& w = waves_[wi];
  const float beta1 = static_cast<float>(mcfg.beta), lr = static_cast<float>(mcfg.lr);
  const bool refresh = step_ % cfg_.precond_every == 0;
  const double ges = grad_dtype_ == kGradBF16 ? 2.0 : 4.0;
  const double elems = w.elems_pre + w.elems_sgd;
  auto ew = [&](int k, double bytes, auto&& launch) -> osh_status {
    OSH_CUDA_TRY(timed_elementwise(kModeElementwise + k, bytes, elems, s, launch));
    return OSH_OK;
  };
  auto sums = [&](const Range& r, double* out) -> osh_status {
    return ew(8, 0.0, [&] {
      return launch_partial_sums(d_partial_, d_slot_begin_ + r.first, d_slot_count_ + r.first,
                                 d_slot_target_ + r.first, out, r.count, s);
    });
  };
  auto gemm = [&](int mode, const NsProblemDesc* pd, int np, float a, float b) -> osh_status {
    const cudaError_t e = timed_gemm(mode, pd, np, a, b, s);
    if (e != cudaSuccess)
      return fail(OSH_ERR_CUDA, std::string("ShampooEngine: ns_gemm_launch: ") + cudaGetErrorString(e));
    return OSH_OK;
  };
  auto at = [&](size_t off) { return static_cast<void*>(d_ws_ + off); };
  auto st = [&](size_t off) { return static_cast<void*>(d_state_ + off); };

  if (w.prep.count > 0) {
    // g read, G and G^T bf16 writes
    if (osh_status e = ew(0, w.elems_pre * (ges + 4.0), [&] {
          return launch_sh_prep(d_prep_ + w.prep.first, w.prep.count, w.prep.tiles, grad_dtype_, s);
        }); e != OSH_OK)
      return e;
    if (osh_status e = sums(w.slot_g, d_gsq_); e != OSH_OK) return e;
    // statistics
    for (const Cls& k : w.cls) {
      const long long gq = static_cast<long long>(rup(2ull * k.p * k.ldq, 256) / 2);
      const long long gtp = static_cast<long long>(rup(2ull * k.q * k.ldp, 256) / 2);
      const long long Lb = static_cast<long long>(rup(4ull * k.p * k.ldp, 256) / 4);
      const long long Rb = static_cast<long long>(rup(4ull * k.q * k.ldq, 256) / 4);
      NsProblemDesc pd[2] = {};
      pd[0].a = mref(at(k.gb), k.nb, k.p, k.q, k.ldq, gq);
      pd[0].b = pd[0].a;
      pd[0].out = mref(st(k.L), k.nb, k.p, k.p, k.ldp, Lb);
      pd[0].symmetric = 2;  // upper triangle; filled below before the refresh reads
      pd[1].a = mref(at(k.gbt), k.nb, k.q, k.p, k.ldp, gtp);
      pd[1].b = pd[1].a;
      pd[1].out = mref(st(k.R), k.nb, k.q, k.q, k.ldq, Rb);
      pd[1].symmetric = 2;
      if (osh_status e = gemm(kEpiStat, pd, 2, static_cast<float>(cfg_.beta2), 0.f); e != OSH_OK)
        return e;
    }
    if (refresh) {
      const int s0 = w.cls.front().stat0;
      if (osh_status e = ew(1, 0.0, [&] {
            const cudaError_t r =
                launch_sym_fill_lower(d_symf_ + w.symf.first, w.symf.count, w.symf.tiles, s);
            if (r != cudaSuccess) return r;
            return launch_sh_sumsq_f32(d_ssq_tasks_ + w.ssq.first, w.ssq.count, w.ssq.tiles, s);
          }); e != OSH_OK)
        return e;
      if (osh_status e = sums(w.slot_s, d_ssq_); e != OSH_OK) return e;
      if (osh_status e = ew(2, 0.0, [&] {
            const cudaError_t r = launch_sh_root_scale(d_ssq_ + s0, d_sroot_ + s0, w.n_stats, s);
            if (r != cudaSuccess) return r;
            return launch_sh_root_init(d_root_ + w.root_init[0].first, w.root_init[0].count,
                                       w.root_init[0].tiles, static_cast<float>(cfg_.eps), s);
          }); e != OSH_OK)
        return e;
      for (int it = 0; it < cfg_.newton_iters; ++it) {
        const int cur = it & 1, nxt = cur ^ 1;
        const Range& nr = w.newton[cur];
        if (osh_status e = ew(3, 0.0, [&] {
              return launch_sh_newton_t(d_newton_ + nr.first, nr.count, nr.tiles, s);
            }); e != OSH_OK)
          return e;
        for (const Cls& k : w.cls) {
          auto split_ref = [&](size_t base, int n, bool bview) {
            const int sg = seg_of(n);
            const long long bs = static_cast<long long>(rup(2ull * n * 4 * sg, 256) / 2);
            return mref(static_cast<__nv_bfloat16*>(at(base)) + (bview ? sg : 0), k.nb, n,
                        3 * sg, 4ll * sg, bs);
          };
          auto out_ref = [&](size_t base, int n) {
            const int sg = seg_of(n);
            const long long bs = static_cast<long long>(rup(2ull * n * 4 * sg, 256) / 2);
            return mref(at(base), k.nb, n, n, 4ll * sg, bs);
          };
          auto prob = [&](size_t a, size_t b, size_t o, int n) {
            NsProblemDesc d{};
            d.a = split_ref(a, n, false);
            d.b = split_ref(b, n, true);
            d.out = out_ref(o, n);
            d.out_seg = seg_of(n);
            // upper-tile form (ns_gemm.cuh): no mirror stores off the diagonal;
            // the k-blocks left of it come from the mirrored tile of the same
            // segment (A view = stored segments 0..2, B view = 1..3). Needs
            // 64-wide segments (k-blocks inside one segment); ragged blocks
            // keep the mirrored form (same values either way)
            const bool upper = seg_of(n) % 64 == 0;
            d.symmetric = upper ? 3 : 1;
            d.a_upper = d.b_upper = upper ? 1 : 0;
            d.k_seg = upper ? seg_of(n) : 0;
            d.a_seg0 = 0;
            d.b_seg0 = upper ? 1 : 0;
            return d;
          };
          // X' = X T and T2 = T T (both sides), then T4 = T2 T2, then M' = T4 M
          NsProblemDesc p1[4] = {prob(k.xl[cur], k.tl, k.xl[nxt], k.p), prob(k.xr[cur], k.tr, k.xr[nxt], k.q),
                                 prob(k.tl, k.tl, k.t2l, k.p), prob(k.tr, k.tr, k.t2r, k.q)};
          if (osh_status e = gemm(kEpiSplit, p1, 4, 0.f, 0.f); e != OSH_OK) return e;
          NsProblemDesc p2[2] = {prob(k.t2l, k.t2l, k.t4l, k.p), prob(k.t2r, k.t2r, k.t4r, k.q)};
          if (osh_status e = gemm(kEpiSplit, p2, 2, 0.f, 0.f); e != OSH_OK) return e;
          NsProblemDesc p3[2] = {prob(k.t4l, k.ml[cur], k.ml[nxt], k.p),
                                 prob(k.t4r, k.mr[cur], k.mr[nxt], k.q)};
          if (osh_status e = gemm(kEpiSplit, p3, 2, 0.f, 0.f); e != OSH_OK) return e;
        }
      }
      if (osh_status e = ew(4, 0.0, [&] {
            return launch_sh_extract(d_extract_ + w.extract[0].first, w.extract[0].count,
                                     w.extract[0].tiles, s);
          }); e != OSH_OK)
        return e;
    }
    // preconditioning: U1 = (P_L G) * sL, U = (U1 P_R) * sR
    for (const Cls& k : w.cls) {
      const long long gq = static_cast<long long>(rup(2ull * k.p * k.ldq, 256) / 2);
      const long long PLb = static_cast<long long>(rup(2ull * k.p * k.ldp, 256) / 2);
      const long long PRb = static_cast<long long>(rup(2ull * k.q * k.ldq, 256) / 2);
      NsProblemDesc u1{};
      u1.a = mref(st(k.PL), k.nb, k.p, k.p, k.ldp, PLb);
      u1.b = mref(at(k.gb), k.nb, k.p, k.q, k.ldq, gq);  // [K = p][N = q], MN-major
      u1.b_mn_major = 1;
      u1.out = mref(at(k.u1), k.nb, k.p, k.q, k.ldq, gq);
      u1.scale = d_sroot_ + k.stat0;
      if (osh_status e = gemm(kEpiUpdate, &u1, 1, 0.f, 0.f); e != OSH_OK) return e;
      NsProblemDesc u2{};
      u2.a = mref(at(k.u1), k.nb, k.p, k.q, k.ldq, gq);
      u2.b = mref(st(k.PR), k.nb, k.q, k.q, k.ldq, PRb);  // symmetric: P_R^T = P_R
      u2.out = mref(at(k.u), k.nb, k.p, k.q, k.ldq, gq);
      u2.scale = d_sroot_ + k.stat0 + k.nb;
      if (osh_status e = gemm(kEpiGram, &u2, 1, 0.f, 0.f); e != OSH_OK) return e;
    }
    if (osh_status e = ew(1, w.elems_pre * 2.0, [&] {
          return launch_sh_sumsq_bf16(d_usq_tasks_ + w.usq.first, w.usq.count, w.usq.tiles, s);
        }); e != OSH_OK)
      return e;
    if (osh_status e = sums(w.slot_u, d_usq_); e != OSH_OK) return e;
    const int b0 = w.cls.front().block0;
    if (osh_status e = ew(5, 0.0, [&] {
          return launch_sh_graft(d_gsq_ + b0, d_usq_ + b0, d_graft_ + b0, w.n_blocks, s);
        }); e != OSH_OK)
      return e;
    // U read, M and W read + write, replica write
    if (osh_status e = ew(6, w.elems_pre * 20.0, [&] {
          return launch_sh_apply(d_apply_ + w.apply.first, w.apply.count, w.apply.tiles, beta1, lr, s);
        }); e != OSH_OK)
      return e;
  }
  if (std::getenv("OSH_SHAMPOO_DEBUG") != nullptr && w.n_blocks > 0) {
    cudaStreamSynchronize(s);
    const int b0 = w.cls.front().block0, s0 = w.cls.front().stat0;
    std::vector<double> g(w.n_blocks), u(w.n_blocks), ss(w.n_stats);
    std::vector<float> gr(w.n_blocks), sr(w.n_stats);
    cudaMemcpy(g.data(), d_gsq_ + b0, 8 * w.n_blocks, cudaMemcpyDeviceToHost);
    cudaMemcpy(u.data(), d_usq_ + b0, 8 * w.n_blocks, cudaMemcpyDeviceToHost);
    cudaMemcpy(gr.data(), d_graft_ + b0, 4 * w.n_blocks, cudaMemcpyDeviceToHost);
    cudaMemcpy(ss.data(), d_ssq_ + s0, 8 * w.n_stats, cudaMemcpyDeviceToHost);
    cudaMemcpy(sr.data(), d_sroot_ + s0, 4 * w.n_stats, cudaMemcpyDeviceToHost);
    for (int i = 0; i < w.n_blocks; ++i)
      std::fprintf(stderr, "block %d gsq %.6e usq %.6e graft %.6e\n", b0 + i, g[i], u[i], gr[i]);
    for (int i = 0; i < w.n_stats; ++i)
      std::fprintf(stderr, "stat %d ssq %.6e sroot %.6e\n", s0 + i, ss[i], sr[i]);
  }
  if (w.sgd.count > 0)
    if (osh_status e = ew(7, w.elems_sgd * (ges + 18.0), [&] {
          return launch_sh_sgd(d_sgd_ + w.sgd.first, w.sgd.count, w.sgd.tiles, grad_dtype_, beta1, lr, s);
        }); e != OSH_OK)
      return e;
  return sums(w.slot_t, d_update_sq_);
}

}  // namespace osh
