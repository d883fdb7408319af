// SoapEngine implementation (see soap_engine.cuh).
#include "soap_engine.cuh"

#include <algorithm>
#include <cmath>
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

// per-block workspace bytes (see SoapEngine::Cls)
size_t block_ws(int p, int q) {
  const size_t ldp = rup(p, 64), ldq = rup(q, 64);
  return rup(2 * p * 4 * ldq, 256) * 3 + rup(2 * q * 4 * ldp, 256) + 2 * rup(2 * 4 * ldp * ldq, 256) +
         2 * rup(4 * p * ldq, 256) + 3 * rup(2 * p * ldq, 256);
}

// refresh workspace bytes of one n x n matrix (see SoapEngine::Side)
size_t refresh_ws(int n, int ld) {
  const size_t seg = kSoapSplitSegs;
  return 3 * rup(2ull * n * seg * ld, 256) + rup(2ull * seg * ld * ld, 256) +
         2 * rup(4ull * ld * ld, 256);
}

}  // namespace

SoapEngine::~SoapEngine() { release(); }

void SoapEngine::release() {
  for (void* p : {static_cast<void*>(d_ws_), static_cast<void*>(d_state_),
                  static_cast<void*>(d_partial_), static_cast<void*>(d_update_sq_),
                  static_cast<void*>(d_bscale_), static_cast<void*>(d_order_),
                  static_cast<void*>(d_rws_), static_cast<void*>(d_split_),
                  static_cast<void*>(d_chol_),
                  static_cast<void*>(d_prep_), static_cast<void*>(d_rot_),
                  static_cast<void*>(d_apply_), static_cast<void*>(d_blockrefs_),
                  static_cast<void*>(d_adam_), static_cast<void*>(d_basis_),
                  static_cast<void*>(d_vperm_), static_cast<void*>(d_qcast_),
                  static_cast<void*>(d_symf_),
                  static_cast<void*>(d_slot_begin_), static_cast<void*>(d_slot_count_),
                  static_cast<void*>(d_slot_target_)})
    cudaFree(p);
  d_ws_ = d_state_ = nullptr;
  d_partial_ = d_update_sq_ = nullptr;
  d_bscale_ = nullptr;
  d_order_ = nullptr;
  d_rws_ = nullptr;
  d_split_ = nullptr;
  d_chol_ = nullptr;
  d_prep_ = nullptr;
  d_rot_ = nullptr;
  d_apply_ = nullptr;
  d_blockrefs_ = nullptr;
  d_adam_ = nullptr;
  d_basis_ = nullptr;
  d_vperm_ = nullptr;
  d_qcast_ = nullptr;
  d_symf_ = nullptr;
  d_slot_begin_ = nullptr;
  d_slot_count_ = d_slot_target_ = nullptr;
  waves_.clear();
}

const char* SoapEngine::elementwise_name(int mode) const {
  static const char* kNames[] = {"soap_prep",  "soap_rot",   "soap_apply", "soap_adam",
                                 "soap_basis", "soap_vperm", "soap_qcast", "soap_split_chol",
                                 "partial_sums"};
  const int i = mode - kModeElementwise;
  return i >= 0 && i < 9 ? kNames[i] : "elementwise";
}

osh_status SoapEngine::build(const std::vector<MuonTensorDesc>& tensors, int grad_dtype,
                             size_t budget, int min_waves, bool /*double_buffer*/) {
  release();
  const int B = cfg_.block;
  if (B < 64 || B % 64 != 0 || B > kSoapCholMaxN)  // (one CTA factors one block's statistics)
    return fail(OSH_ERR_CONFIG, "SOAP block size must be a multiple of 64 in [64, 1024]");
  if (cfg_.precond_every < 1 || cfg_.init_iters < 1)
    return fail(OSH_ERR_CONFIG, "SOAP precond_every and init_iters must be >= 1");
  n_tensors_ = static_cast<int>(tensors.size());
  grad_dtype_ = grad_dtype;
  step_ = -1;
  // bf16 gradients are exact in the hi segment (NVLS too: multimem.ld_reduce
  // accumulates in fp32 but returns the sum as bf16x2)
  exact_grad_ = grad_dtype == kGradBF16;
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
    return fail(OSH_ERR_OOM, "SoapEngine: one tensor needs " + std::to_string(largest) +
                                 " workspace bytes, budget is " + std::to_string(budget) +
                                 " (lower the block size)");
  // Waves run back to back here (no overlap to feed), so they are as large
  // as the budget allows: larger batches fill the GEMMs and give the
  // one-CTA-per-matrix refresh kernels enough matrices for every SM.
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

  // ---- pass 1: geometry and offsets
  struct TB {
    int tensor;
    BlockGeom g;
  };
  std::vector<std::vector<std::vector<TB>>> cls_blocks(members.size());  // [wave][cls] -> blocks
  size_t state_off = 0;
  int n_orders = 0;
  // refresh sub-batch budget: enough for 2 x 148 matrices (two CTA waves of
  // the one-CTA-per-matrix kernels) where the workspace budget allows
  const size_t rws_cap = std::min<size_t>(budget / 2, 12ull << 30);
  std::vector<size_t> vec_v(tensors.size(), 0);  // Adam second moment of non-preconditioned tensors
  for (size_t wi = 0; wi < members.size(); ++wi) {
    Wave w;
    w.first_bucket = tensors[members[wi].front()].bucket;
    w.last_bucket = tensors[members[wi].back()].bucket;
    std::map<std::pair<int, int>, int> cls_of;
    for (const int ti : members[wi]) {
      const MuonTensorDesc& t = tensors[ti];
      if (!pre(t)) {
        vec_v[ti] = state_off;
        state_off += rup(4ull * t.rows * t.cols, 256);
        continue;
      }
      for (const BlockGeom& g : blocks_of(t.rows, t.cols, B)) {
        auto it = cls_of.find({g.p, g.q});
        if (it == cls_of.end()) {
          it = cls_of.emplace(std::make_pair(g.p, g.q), static_cast<int>(cls_blocks[wi].size())).first;
          cls_blocks[wi].emplace_back();
        }
        cls_blocks[wi][it->second].push_back({ti, g});
      }
    }
    size_t off = 0;
    for (const auto& blocks : cls_blocks[wi]) {
      Cls k;
      k.p = blocks.front().g.p;
      k.q = blocks.front().g.q;
      k.ldp = static_cast<int>(rup(k.p, 64));
      k.ldq = static_cast<int>(rup(k.q, 64));
      k.nb = static_cast<int>(blocks.size());
      max_nb_ = std::max(max_nb_, k.nb);
      const size_t pq2 = rup(2ull * k.p * k.ldq, 256);
      const size_t pq4 = rup(4ull * k.p * k.ldq, 256);
      const size_t pp4 = rup(4ull * k.p * k.ldp, 256), qq4 = rup(4ull * k.q * k.ldq, 256);
      const size_t pp2 = rup(2ull * k.p * k.ldp, 256);
      const size_t cs_pq = rup(2ull * k.p * 4 * k.ldq, 256), cs_qp = rup(2ull * k.q * 4 * k.ldp, 256);
      const size_t rs_pq = rup(2ull * 4 * k.ldp * k.ldq, 256);
      const size_t cs_pp = rup(2ull * k.p * 4 * k.ldp, 256), rs_qq = rup(2ull * 4 * k.ldq * k.ldq, 256);
      // every [nb][rows][ld] array is addressed with the unrounded batch
      // stride rows * ld (a multiple of 64 elements); the 256 B rounding of
      // the per-block sizes only over-allocates
      k.Gs = off; off += cs_pq * k.nb;
      k.T1s = off; off += cs_pq * k.nb;
      k.T2s = off; off += cs_pq * k.nb;
      k.Gts = off; off += cs_qp * k.nb;
      k.Grs = off; off += rs_pq * k.nb;
      k.Mrs = off; off += rs_pq * k.nb;
      for (size_t* z : {&k.Nr, &k.T3, &k.Nb}) {
        *z = off;
        off += pq2 * k.nb;
      }
      k.Gp = off; off += pq4 * k.nb;
      k.Mp = off; off += pq4 * k.nb;
      k.l.n = k.p; k.l.ld = k.ldp;
      k.r.n = k.q; k.r.ld = k.ldq;
      // elongated blocks: the long side's statistics have rank <= the short
      // side, so its basis stays the identity (one-sided SOAP; soap_oracle.py)
      k.l.frozen = k.p > 2 * k.q;
      k.r.frozen = k.q > 2 * k.p;
      for (Side* sd : {&k.l, &k.r}) {  // refresh sub-batches
        sd->rb = static_cast<int>(std::max<size_t>(1, std::min<size_t>(
                                      static_cast<size_t>(k.nb), rws_cap / refresh_ws(sd->n, sd->ld))));
        const size_t rb = static_cast<size_t>(sd->rb);
        const size_t n = static_cast<size_t>(sd->n), ld = static_cast<size_t>(sd->ld);
        // S's split is dead once Y = S Q is formed, Y once soap_basis ran:
        // the L^-1 split aliases S's, the Gram matrix aliases Y
        const size_t sg = kSoapSplitSegs;
        size_t o = 0;
        sd->Sb = sd->La = o; o += rb * rup(2 * n * sg * ld, 256);
        sd->Qa = o; o += rb * rup(2 * n * sg * ld, 256);
        sd->Qb = o; o += rb * rup(2 * n * sg * ld, 256);
        sd->Qrb = o; o += rb * rup(2 * sg * ld * ld, 256);
        sd->Y = sd->C = o; o += rb * rup(4 * ld * ld, 256);
        sd->Li = o; o += rb * rup(4 * ld * ld, 256);
        rws_bytes_ = std::max(rws_bytes_, o);
      }
      k.l.S = state_off; state_off += pp4 * k.nb;
      k.r.S = state_off; state_off += qq4 * k.nb;
      k.l.Q = state_off; state_off += pp4 * k.nb;
      k.r.Q = state_off; state_off += qq4 * k.nb;
      k.QLts = state_off; state_off += cs_pp * k.nb;
      k.QLb = state_off; state_off += pp2 * k.nb;
      k.QRrs = state_off; state_off += rs_qq * k.nb;
      k.V = state_off; state_off += pq4 * k.nb;
      k.l.order0 = n_orders; n_orders += k.p * k.nb;
      k.r.order0 = n_orders; n_orders += k.q * k.nb;
      w.cls.push_back(k);
    }
    ws_bytes_ = std::max(ws_bytes_, off);
    waves_.push_back(w);
  }
  state_bytes_ = state_off;
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_ws_), std::max<size_t>(ws_bytes_, 256)));
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_state_), std::max<size_t>(state_bytes_, 256)));
  OSH_CUDA_TRY(cudaMemset(d_ws_, 0, std::max<size_t>(ws_bytes_, 256)));
  OSH_CUDA_TRY(cudaMemset(d_state_, 0, std::max<size_t>(state_bytes_, 256)));
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_rws_), std::max<size_t>(rws_bytes_, 256)));
  OSH_CUDA_TRY(cudaMemset(d_rws_, 0, std::max<size_t>(rws_bytes_, 256)));
  auto ws = [&](size_t o) { return d_ws_ + o; };
  auto st = [&](size_t o) { return d_state_ + o; };

  // ---- pass 2: task tables with real pointers
  std::vector<SoapPrepTask> prep;
  std::vector<SoapRotTask> rot;
  std::vector<ShApplyTask> apply;
  std::vector<ShBlockRef> brefs;
  std::vector<SoapAdamTask> adam;
  std::vector<SoapBasisTask> basis;
  std::vector<SoapVpermTask> vperm;
  std::vector<SoapQcastTask> qcast;
  std::vector<long long> slot_begin;
  std::vector<int> slot_count, slot_target;
  std::vector<SoapSplitTask> split;
  std::vector<SoapCholTask> chol;
  long long max_partial = 1;
  const auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  std::vector<size_t> apply_bref_first;  // per apply task: first ShBlockRef (patched below)
  for (size_t wi = 0; wi < members.size(); ++wi) {
    Wave& w = waves_[wi];
    std::map<std::pair<int, int>, std::pair<int, int>> where;  // (tensor, block idx) -> (cls, i)
    w.prep.first = static_cast<int>(prep.size());
    w.rot.first = static_cast<int>(rot.size());
    w.basis.first = static_cast<int>(basis.size());
    w.vperm.first = static_cast<int>(vperm.size());
    w.qcast.first = static_cast<int>(qcast.size());
    for (size_t c = 0; c < w.cls.size(); ++c) {
      Cls& k = w.cls[c];
      const auto& blocks = cls_blocks[wi][c];
      const long long pq = static_cast<long long>(k.p) * k.ldq;
      k.rot = static_cast<int>(rot.size());
      SoapRotTask rt{};
      rt.gp = reinterpret_cast<const float*>(ws(k.Gp));
      rt.mp = reinterpret_cast<const float*>(ws(k.Mp));
      rt.v = reinterpret_cast<float*>(st(k.V));
      rt.nrot = reinterpret_cast<__nv_bfloat16*>(ws(k.Nr));
      rt.ldq = k.ldq;
      rt.q = k.q;
      rt.elems = pq * k.nb;
      rt.chunk_start = w.rot.tiles;
      w.rot.tiles += (rt.elems + kSoapRotChunk - 1) / kSoapRotChunk;
      rot.push_back(rt);
      for (Side* sd : {&k.l, &k.r}) {
        sd->basis0 = static_cast<int>(basis.size());
        const long long n = sd->n, ld = sd->ld, nn = n * ld;
        uint8_t* R = d_rws_;
        auto bf = [&](size_t off, long long j, long long per) {
          return reinterpret_cast<__nv_bfloat16*>(R + off) + per * j;
        };
        auto f32 = [&](size_t off, long long j, long long per) {
          return reinterpret_cast<float*>(R + off) + per * j;
        };
        const long long tiles = tiles_of(sd->n, sd->n);
        for (int i0 = 0; i0 < k.nb; i0 += sd->rb) {
          RChunk ch;
          ch.i0 = i0;
          ch.b = std::min(sd->rb, k.nb - i0);
          ch.split_s = static_cast<int>(split.size());
          for (int j = 0; j < ch.b; ++j) {  // S -> column split
            SoapSplitTask t{};
            t.src = reinterpret_cast<const float*>(st(sd->S)) + nn * (i0 + j);
            t.lds = ld;
            t.rows = t.cols = sd->n;
            t.col_b = bf(sd->Sb, j, n * kSoapSplitSegs * ld);
            t.ldd = ld;
            t.tiles_c = (sd->n + kTile - 1) / kTile;
            t.tile_start = ch.tiles_s;
            ch.tiles_s += tiles;
            split.push_back(t);
          }
          ch.split_q = static_cast<int>(split.size());
          for (int j = 0; j < ch.b; ++j) {  // Q storage -> column and row splits
            SoapSplitTask t{};
            t.src = reinterpret_cast<const float*>(st(sd->Q)) + nn * (i0 + j);
            t.lds = ld;
            t.rows = t.cols = sd->n;
            t.col_a = bf(sd->Qa, j, n * kSoapSplitSegs * ld);
            t.col_b = bf(sd->Qb, j, n * kSoapSplitSegs * ld);
            t.row_b = bf(sd->Qrb, j, kSoapSplitSegs * ld * ld);
            t.ldd = ld;
            t.tiles_c = (sd->n + kTile - 1) / kTile;
            t.tile_start = ch.tiles_q;
            ch.tiles_q += tiles;
            split.push_back(t);
          }
          ch.split_l = static_cast<int>(split.size());
          for (int j = 0; j < ch.b; ++j) {  // L^-1 -> column split
            SoapSplitTask t{};
            t.src = f32(sd->Li, j, ld * ld);
            t.lds = ld;
            t.rows = t.cols = sd->n;
            t.col_a = bf(sd->La, j, n * kSoapSplitSegs * ld);
            t.ldd = ld;
            t.tiles_c = (sd->n + kTile - 1) / kTile;
            t.tile_start = ch.tiles_l;
            ch.tiles_l += tiles;
            split.push_back(t);
          }
          ch.chol = static_cast<int>(chol.size());
          for (int j = 0; j < ch.b; ++j) {
            SoapCholTask t{};
            t.c = f32(sd->C, j, ld * ld);
            t.linv = f32(sd->Li, j, ld * ld);
            t.ld = ld;
            t.n = sd->n;
            chol.push_back(t);
          }
          for (int j = 0; j < ch.b; ++j) {
            SoapBasisTask bt{};
            bt.s = reinterpret_cast<const float*>(st(sd->S)) + nn * (i0 + j);
            bt.lds = ld;
            bt.q = reinterpret_cast<float*>(st(sd->Q)) + nn * (i0 + j);
            bt.y = f32(sd->Y, j, nn);
            bt.ldq = ld;
            bt.order = nullptr;  // patched after d_order_ exists
            bt.n = sd->n;
            basis.push_back(bt);
          }
          sd->chunks.push_back(ch);
        }
      }
      for (int i = 0; i < k.nb; ++i) {
        const TB& tb = blocks[static_cast<size_t>(i)];
        const MuonTensorDesc& t = tensors[static_cast<size_t>(tb.tensor)];
        const BlockGeom& g = tb.g;
        const int bi = g.r0 / B, bj = g.c0 / B;
        const int blocks_c = (t.cols + B - 1) / B;
        where[{tb.tensor, bi * blocks_c + bj}] = {static_cast<int>(c), i};
        SoapPrepTask pt{};
        pt.g = t.g;
        pt.m = t.m;
        pt.g_ld = t.cols;
        pt.g_mc = t.g_mc;
        pt.r0 = g.r0;
        pt.c0 = g.c0;
        pt.p = g.p;
        pt.q = g.q;
        const long long cpq = static_cast<long long>(k.p) * 4 * k.ldq;
        const long long rpq = static_cast<long long>(4) * k.ldp * k.ldq;
        pt.gs = reinterpret_cast<__nv_bfloat16*>(ws(k.Gs)) + cpq * i;
        pt.gts = reinterpret_cast<__nv_bfloat16*>(ws(k.Gts)) + static_cast<long long>(k.q) * 4 * k.ldp * i;
        pt.grs = reinterpret_cast<__nv_bfloat16*>(ws(k.Grs)) + rpq * i;
        pt.mrs = reinterpret_cast<__nv_bfloat16*>(ws(k.Mrs)) + rpq * i;
        pt.ldq = k.ldq;
        pt.ldp = k.ldp;
        pt.vec = (t.cols % 8 == 0 && g.c0 % 8 == 0 && g.q % 8 == 0 && a16(t.g) && a16(t.m)) ? 1 : 0;
        pt.exact = exact_grad_ ? 1 : 0;
        if (t.g_mc && !pt.vec) return fail(OSH_ERR_UNSUPPORTED, "NVLS path needs the 128-bit layout");
        pt.tiles_c = (g.q + kTile - 1) / kTile;
        pt.tile_start = w.prep.tiles;
        w.prep.tiles += tiles_of(g.p, g.q);
        prep.push_back(pt);
        SoapVpermTask vt{};
        vt.v = reinterpret_cast<const float*>(st(k.V)) + pq * i;
        vt.dst = reinterpret_cast<float*>(ws(k.Gp)) + pq * i;
        vt.p = k.p;
        vt.q = k.q;
        vt.ldq = k.ldq;
        vt.tiles_c = (k.q + kTile - 1) / kTile;
        vt.tile_start = w.vperm.tiles;
        w.vperm.tiles += tiles_of(k.p, k.q);
        vperm.push_back(vt);
        const long long pp = static_cast<long long>(k.p) * k.ldp, qq = static_cast<long long>(k.q) * k.ldq;
        SoapQcastTask ql{};
        ql.q = reinterpret_cast<const float*>(st(k.l.Q)) + pp * i;
        ql.ldq = k.ldp;
        ql.qt_split = reinterpret_cast<__nv_bfloat16*>(st(k.QLts)) + static_cast<long long>(k.p) * 4 * k.ldp * i;
        ql.q_row = reinterpret_cast<__nv_bfloat16*>(st(k.QLb)) + pp * i;
        ql.q_rsplit = nullptr;
        ql.ldb = k.ldp;
        ql.n = k.p;
        ql.tiles_c = (k.p + kTile - 1) / kTile;
        ql.tile_start = w.qcast.tiles;
        w.qcast.tiles += tiles_of(k.p, k.p);
        qcast.push_back(ql);
        SoapQcastTask qr{};
        qr.q = reinterpret_cast<const float*>(st(k.r.Q)) + qq * i;
        qr.ldq = k.ldq;
        qr.qt_split = nullptr;
        qr.q_row = nullptr;
        qr.q_rsplit = reinterpret_cast<__nv_bfloat16*>(st(k.QRrs)) + static_cast<long long>(4) * k.ldq * k.ldq * i;
        qr.ldb = k.ldq;
        qr.n = k.q;
        qr.tiles_c = (k.q + kTile - 1) / kTile;
        qr.tile_start = w.qcast.tiles;
        w.qcast.tiles += tiles_of(k.q, k.q);
        qcast.push_back(qr);
      }
    }
    w.prep.count = static_cast<int>(prep.size()) - w.prep.first;
    w.rot.count = static_cast<int>(rot.size()) - w.rot.first;
    w.basis.count = static_cast<int>(basis.size()) - w.basis.first;
    w.vperm.count = static_cast<int>(vperm.size()) - w.vperm.first;
    w.qcast.count = static_cast<int>(qcast.size()) - w.qcast.first;
    // apply (preconditioned tensors) then Adam (the rest), one norm slot per tensor
    w.apply.first = static_cast<int>(apply.size());
    w.slots.first = static_cast<int>(slot_begin.size());
    for (const int ti : members[wi]) {
      const MuonTensorDesc& t = tensors[static_cast<size_t>(ti)];
      if (!pre(t)) continue;
      const int blocks_c = (t.cols + B - 1) / B, blocks_r = (t.rows + B - 1) / B;
      ShApplyTask at{};
      at.w = t.w;
      at.m = nullptr;
      at.replica = t.replica;
      at.rep_mc = t.rep_mc;
      at.rows = t.rows;
      at.cols = t.cols;
      at.block = B;
      at.blocks_c = blocks_c;
      at.tiles_c = (t.cols + kTile - 1) / kTile;
      at.tile_start = w.apply.tiles;
      at.partial = nullptr;  // d_partial_ (patched)
      apply_bref_first.push_back(brefs.size());
      bool vec = t.cols % 8 == 0 && a16(t.w) && (t.replica == nullptr || a16(t.replica));
      for (int bi = 0; bi < blocks_r; ++bi)
        for (int bj = 0; bj < blocks_c; ++bj) {
          const auto ci = where.at({ti, bi * blocks_c + bj});
          const Cls& k = w.cls[static_cast<size_t>(ci.first)];
          ShBlockRef br{};
          br.u = reinterpret_cast<const __nv_bfloat16*>(ws(k.Nb)) +
                 static_cast<long long>(k.p) * k.ldq * ci.second;
          br.ldu = k.ldq;
          br.scale = nullptr;
          vec = vec && a16(br.u);
          brefs.push_back(br);
        }
      at.vec = vec ? 1 : 0;
      if (t.rep_mc && !vec) return fail(OSH_ERR_UNSUPPORTED, "NVLS path needs the 128-bit layout");
      slot_begin.push_back(w.apply.tiles);
      slot_count.push_back(static_cast<int>(tiles_of(t.rows, t.cols)));
      slot_target.push_back(ti);
      w.apply.tiles += tiles_of(t.rows, t.cols);
      w.elems_pre += static_cast<double>(t.rows) * t.cols;
      apply.push_back(at);
    }
    w.apply.count = static_cast<int>(apply.size()) - w.apply.first;
    w.adam.first = static_cast<int>(adam.size());
    for (const int ti : members[wi]) {
      const MuonTensorDesc& t = tensors[static_cast<size_t>(ti)];
      if (pre(t)) continue;
      SoapAdamTask a{};
      a.g = t.g;
      a.g_mc = t.g_mc;
      a.rep_mc = t.rep_mc;
      a.m = t.m;
      a.v = reinterpret_cast<float*>(st(vec_v[static_cast<size_t>(ti)]));
      a.w = t.w;
      a.replica = t.replica;
      a.n = static_cast<long long>(t.rows) * t.cols;
      a.vec = (a.n % 8 == 0 && a16(t.g) && a16(t.m) && a16(t.w) &&
               (t.replica == nullptr || a16(t.replica))) ? 1 : 0;
      if ((t.g_mc || t.rep_mc) && !a.vec)
        return fail(OSH_ERR_UNSUPPORTED, "NVLS path needs the 128-bit layout");
      a.tile_start = w.adam.tiles;
      a.partial = nullptr;  // d_partial_ + apply tiles (patched)
      const long long tl = (a.n + kShSgdTile - 1) / kShSgdTile;
      slot_begin.push_back(w.apply.tiles + w.adam.tiles);
      slot_count.push_back(static_cast<int>(tl));
      slot_target.push_back(ti);
      w.adam.tiles += tl;
      w.elems_adam += static_cast<double>(a.n);
      adam.push_back(a);
    }
    w.adam.count = static_cast<int>(adam.size()) - w.adam.first;
    w.slots.count = static_cast<int>(slot_begin.size()) - w.slots.first;
    max_partial = std::max(max_partial, w.apply.tiles + w.adam.tiles);
  }
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_partial_), sizeof(double) * static_cast<size_t>(max_partial)));
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_update_sq_), sizeof(double) * std::max(n_tensors_, 1)));
  OSH_CUDA_TRY(cudaMemset(d_update_sq_, 0, sizeof(double) * std::max(n_tensors_, 1)));
  OSH_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&d_order_), sizeof(int) * static_cast<size_t>(std::max(n_orders, 1))));
  {  // identity orders: what a frozen side keeps (refreshed sides overwrite theirs)
    std::vector<int> ident(static_cast<size_t>(std::max(n_orders, 1)), 0);
    for (const Wave& w : waves_)
      for (const Cls& k : w.cls)
        for (const Side* sd : {&k.l, &k.r})
          for (int i = 0; i < k.nb; ++i)
            for (int j = 0; j < sd->n; ++j) ident[static_cast<size_t>(sd->order0 + sd->n * i + j)] = j;
    OSH_CUDA_TRY(cudaMemcpy(d_order_, ident.data(), sizeof(int) * ident.size(), cudaMemcpyHostToDevice));
  }
  {
    const std::vector<float> bs(static_cast<size_t>(max_nb_), static_cast<float>(1.0 - cfg_.beta2));
    OSH_CUDA_TRY(upload(&d_bscale_, bs));
  }
  for (size_t i = 0; i < apply.size(); ++i) {
    apply[i].partial = d_partial_;
    apply[i].blocks = nullptr;  // patched after d_blockrefs_ exists
  }
  for (size_t wi = 0; wi < waves_.size(); ++wi) {
    const Wave& w = waves_[wi];
    for (int i = 0; i < w.adam.count; ++i) adam[static_cast<size_t>(w.adam.first + i)].partial = d_partial_ + w.apply.tiles;
    for (const Cls& k : w.cls) {
      for (const Side* sd : {&k.l, &k.r})
        for (int i = 0; i < k.nb; ++i)
          basis[static_cast<size_t>(sd->basis0 + i)].order = d_order_ + sd->order0 + sd->n * i;
    }
    // vperm tasks follow the class / block order of prep
    int vi = w.vperm.first;
    for (const Cls& k : w.cls)
      for (int i = 0; i < k.nb; ++i, ++vi) {
        vperm[static_cast<size_t>(vi)].ol = d_order_ + k.l.order0 + k.p * i;
        vperm[static_cast<size_t>(vi)].orr = d_order_ + k.r.order0 + k.q * i;
      }
  }
  OSH_CUDA_TRY(upload(&d_blockrefs_, brefs));
  for (size_t i = 0; i < apply.size(); ++i) apply[i].blocks = d_blockrefs_ + apply_bref_first[i];
  OSH_CUDA_TRY(upload(&d_prep_, prep));
  OSH_CUDA_TRY(upload(&d_rot_, rot));
  OSH_CUDA_TRY(upload(&d_apply_, apply));
  OSH_CUDA_TRY(upload(&d_adam_, adam));
  OSH_CUDA_TRY(upload(&d_basis_, basis));
  OSH_CUDA_TRY(upload(&d_vperm_, vperm));
  OSH_CUDA_TRY(upload(&d_qcast_, qcast));
  {  // the statistics are accumulated upper-triangle only (STAT symmetric = 2)
    std::vector<SymFillTask> symf;
    for (Wave& w : waves_) {
      w.symf = Range{};
      w.symf.first = static_cast<int>(symf.size());
      for (const Cls& k : w.cls)
        for (int side = 0; side < 2; ++side) {
          const int n = side == 0 ? k.p : k.q, ld = side == 0 ? k.ldp : k.ldq;
          const Side& sd = side == 0 ? k.l : k.r;
          if (sd.frozen) continue;  // never read
          for (int i = 0; i < k.nb; ++i) {
            SymFillTask sf{};
            sf.s = reinterpret_cast<float*>(d_state_ + sd.S) + static_cast<size_t>(i) * n * ld;
            sf.ld = ld;
            sf.n = n;
            const int T = (n + 31) / 32;
            sf.tiles = T * (T + 1) / 2;
            sf.tile_start = w.symf.tiles;
            w.symf.tiles += sf.tiles;
            symf.push_back(sf);
          }
        }
      w.symf.count = static_cast<int>(symf.size()) - w.symf.first;
    }
    OSH_CUDA_TRY(upload(&d_symf_, symf));
  }
  OSH_CUDA_TRY(upload(&d_split_, split));
  OSH_CUDA_TRY(upload(&d_chol_, chol));
  OSH_CUDA_TRY(upload(&d_slot_begin_, slot_begin));
  OSH_CUDA_TRY(upload(&d_slot_count_, slot_count));
  OSH_CUDA_TRY(upload(&d_slot_target_, slot_target));
  // Q = I, bf16 copies
  for (const Wave& w : waves_) {
    for (const Cls& k : w.cls)
      for (const Side* sd : {&k.l, &k.r})
        OSH_CUDA_TRY(launch_soap_eye(reinterpret_cast<float*>(st(sd->Q)), sd->ld,
                                     static_cast<long long>(sd->n) * sd->ld, sd->n, k.nb, nullptr));
    OSH_CUDA_TRY(launch_soap_qcast(d_qcast_ + w.qcast.first, w.qcast.count, w.qcast.tiles, nullptr));
  }
  OSH_CUDA_TRY(cudaDeviceSynchronize());
  return OSH_OK;
}

osh_status SoapEngine::begin_step(cudaStream_t s) {
  stats_ = NsLaunchStats{};
  ++step_;
  OSH_CUDA_TRY(cudaMemsetAsync(d_update_sq_, 0, sizeof(double) * std::max(n_tensors_, 1), s));
  return OSH_OK;
}

// One side's basis refresh, `iters` times, in sub-batches (soap_engine.cuh):
// Y = S Q, soap_basis, then CholeskyQR2 on the result. All products are
// tcgen05 STAT GEMMs (fp32 out) over bf16x6 splits; the Cholesky factor and
// its inverse come from soap_chol_inv. Q (fp32) is stored column-major, i.e.
// its storage rows are Q's columns: Y^T = Q^T S, Gram = Q^T Q and
// Q' = Q (L^T)^-1  <=>  Q'^T = L^-1 Q^T are row-major products of the storage.
osh_status SoapEngine::refresh_side(const Side& sd, int iters, cudaStream_t s) {
  const long long n = sd.n, ld = sd.ld, nn = n * ld;
  auto gemm1 = [&](NsProblemDesc& d) -> osh_status {
    const cudaError_t e = timed_gemm(kEpiStat, &d, 1, 0.f, 0.f, s);
    if (e != cudaSuccess)
      return fail(OSH_ERR_CUDA, std::string("SoapEngine refresh: ns_gemm_launch: ") + cudaGetErrorString(e));
    return OSH_OK;
  };
  for (int it = 0; it < iters; ++it)
    for (const RChunk& ch : sd.chunks) {
      const int b = ch.b;
      float* Q = reinterpret_cast<float*>(d_state_ + sd.Q) + nn * ch.i0;
      OSH_CUDA_TRY(timed_elementwise(kModeElementwise + 7, 0.0, 0.0, s, [&] {
        cudaError_t e = launch_soap_split(d_split_ + ch.split_s, b, ch.tiles_s, s);
        if (e == cudaSuccess) e = launch_soap_split(d_split_ + ch.split_q, b, ch.tiles_q, s);
        return e;
      }));
      const long long sg = kSoapSplitSegs;
      {  // Y^T (= Y column-major) = Q^T S over the bf16x6 layouts (A: Q storage, B: S)
        NsProblemDesc d{};
        d.a = mref(d_rws_ + sd.Qa, b, sd.n, sg * sd.ld, sg * ld, n * sg * ld);
        d.b = mref(d_rws_ + sd.Sb, b, sd.n, sg * sd.ld, sg * ld, n * sg * ld);
        d.out = mref(d_rws_ + sd.Y, b, sd.n, sd.n, ld, nn);
        if (osh_status st = gemm1(d); st != OSH_OK) return st;
      }
      OSH_CUDA_TRY(timed_elementwise(kModeElementwise + 4, 0.0, 0.0, s, [&] {
        return launch_soap_basis(d_basis_ + sd.basis0 + ch.i0, b, cfg_.shift, s);
      }));
      for (int pass = 0; pass < 2; ++pass) {  // CholeskyQR2
        OSH_CUDA_TRY(timed_elementwise(kModeElementwise + 7, 0.0, 0.0, s, [&] {
          return launch_soap_split(d_split_ + ch.split_q, b, ch.tiles_q, s);
        }));
        NsProblemDesc g{};  // Gram = Q^T Q (symmetric)
        g.a = mref(d_rws_ + sd.Qa, b, sd.n, sg * sd.ld, sg * ld, n * sg * ld);
        g.b = mref(d_rws_ + sd.Qb, b, sd.n, sg * sd.ld, sg * ld, n * sg * ld);
        g.out = mref(d_rws_ + sd.C, b, sd.n, sd.n, ld, ld * ld);
        g.symmetric = 1;
        if (osh_status st = gemm1(g); st != OSH_OK) return st;
        OSH_CUDA_TRY(timed_elementwise(kModeElementwise + 7, 0.0, 0.0, s, [&] {
          cudaError_t e = launch_soap_chol_inv(d_chol_ + ch.chol, b, s);
          if (e == cudaSuccess) e = launch_soap_split(d_split_ + ch.split_l, b, ch.tiles_l, s);
          return e;
        }));
        NsProblemDesc u{};  // Q'^T = L^-1 Q^T: A = L^-1 (A layout), B = Q storage rows (B layout)
        u.a = mref(d_rws_ + sd.La, b, sd.n, sg * sd.ld, sg * ld, n * sg * ld);
        u.b = mref(d_rws_ + sd.Qrb, b, sg * sd.ld, sd.n, ld, sg * ld * ld);
        u.b_mn_major = 1;
        u.out = mref(Q, b, sd.n, sd.n, ld, nn);
        if (osh_status st = gemm1(u); st != OSH_OK) return st;
      }
    }
  return OSH_OK;
}

osh_status SoapEngine::refresh(const Wave& w, int iters, bool permute_v, cudaStream_t s) {
  OSH_CUDA_TRY(timed_elementwise(kModeElementwise + 7, 0.0, 0.0, s, [&] {
    return launch_sym_fill_lower(d_symf_ + w.symf.first, w.symf.count, w.symf.tiles, s);
  }));
  for (const Cls& k : w.cls)
    for (const Side* sd : {&k.l, &k.r})
      if (!sd->frozen)
        if (osh_status st = refresh_side(*sd, iters, s); st != OSH_OK) return st;
  if (permute_v && w.vperm.count > 0) {
    OSH_CUDA_TRY(timed_elementwise(kModeElementwise + 5, 0.0, 0.0, s, [&] {
      return launch_soap_vperm(d_vperm_ + w.vperm.first, w.vperm.count, w.vperm.tiles, s);
    }));
    for (const Cls& k : w.cls)
      OSH_CUDA_TRY(cudaMemcpyAsync(d_state_ + k.V, d_ws_ + k.Gp,
                                   4ull * k.p * k.ldq * k.nb, cudaMemcpyDeviceToDevice, s));
  }
  OSH_CUDA_TRY(timed_elementwise(kModeElementwise + 6, 0.0, 0.0, s, [&] {
    return launch_soap_qcast(d_qcast_ + w.qcast.first, w.qcast.count, w.qcast.tiles, s);
  }));
  return OSH_OK;
}

osh_status SoapEngine::run_wave(int wi, const osh_muon_cfg& cfg, cudaStream_t s) {
  const Wave& w = waves_[wi];
  // the first call only accumulates the statistics and computes the initial
  // basis (soap_oracle.py); Adam steps count from the second call
  const bool first = step_ == 0;
  const long long t = std::max<long long>(step_, 1);
  const double b1 = cfg.beta, b2 = cfg_.beta2;
  const float ib1 = static_cast<float>(1.0 / (1.0 - std::pow(b1, static_cast<double>(t))));
  const float ib2 = static_cast<float>(1.0 / (1.0 - std::pow(b2, static_cast<double>(t))));
  const float lr = static_cast<float>(cfg.lr), eps = static_cast<float>(cfg_.eps);
  const double ges = grad_dtype_ == kGradBF16 ? 2.0 : 4.0;
  const double elems = w.elems_pre + w.elems_adam;
  auto timed = [&](int mode, double bytes, auto&& launch) {
    return timed_elementwise(mode, bytes, elems, s, launch);
  };
  auto gemm = [&](int mode, std::vector<NsProblemDesc>& pd, float alpha) -> osh_status {
    for (size_t i = 0; i < pd.size(); i += kMaxProblems) {
      const int np = static_cast<int>(std::min<size_t>(kMaxProblems, pd.size() - i));
      const cudaError_t e = timed_gemm(mode, pd.data() + i, np, alpha, 0.f, s);
      if (e != cudaSuccess)
        return fail(OSH_ERR_CUDA, std::string("SoapEngine: ns_gemm_launch: ") + cudaGetErrorString(e));
    }
    return OSH_OK;
  };
  auto B16 = [&](size_t off, int nb, int rows, int cols, int ld) {
    return mref(d_ws_ + off, nb, rows, cols, ld, static_cast<long long>(rows) * ld);
  };
  auto S16 = [&](size_t off, int nb, int rows, int cols, int ld) {
    return mref(d_state_ + off, nb, rows, cols, ld, static_cast<long long>(rows) * ld);
  };
  if (w.prep.count > 0) {
    // g read, m read + write, G / G^T / bf16(M) written (first call: M kept)
    OSH_CUDA_TRY(timed(kModeElementwise + 0, w.elems_pre * (ges + 8.0 + 6.0), [&] {
      return launch_soap_prep(d_prep_ + w.prep.first, w.prep.count, w.prep.tiles, grad_dtype_,
                              first ? 1.f : static_cast<float>(b1), s);
    }));
    std::vector<NsProblemDesc> pd;
    if (!first) {
      // T1 = Q_L^T G, T2 = Q_L^T M in bf16x3: A = Q_L^T column-split view
      // (hi, lo, hi), B = G / M row-split view (lo, hi, hi); SPLIT epilogue
      // writes T1 / T2 column-split (their pad columns must be 0)
      for (const Cls& k : w.cls) {
        const long long cpq = static_cast<long long>(k.p) * 4 * k.ldq;
        if (k.q % 64 != 0)
          OSH_CUDA_TRY(cudaMemsetAsync(d_ws_ + k.T1s, 0, 2 * 2ull * cpq * k.nb, s));  // T1s, T2s
        for (size_t src : {k.Grs, k.Mrs}) {
          // bf16 gradients are exact in hi (lo = 0): T1 needs only the
          // (lo, hi) x (hi, hi) segment pairs, K = 2 ldp
          const int segs = (src == k.Grs && exact_grad_) ? 2 : 3;
          const int a0 = 3 - segs;  // first A segment: 0 (hi) or 1 (lo)
          NsProblemDesc d{};
          d.a = mref(d_state_ + k.QLts + 2ull * a0 * k.ldp, k.nb, k.p, segs * k.ldp, 4ll * k.ldp,
                     static_cast<long long>(k.p) * 4 * k.ldp);
          d.b = mref(d_ws_ + src + 2ull * (1 + a0) * k.ldp * k.ldq, k.nb, segs * k.ldp, k.q, k.ldq,
                     4ll * k.ldp * k.ldq);
          d.b_mn_major = 1;
          d.out = mref(d_ws_ + (src == k.Grs ? k.T1s : k.T2s), k.nb, k.p, k.q, 4ll * k.ldq, cpq);
          d.out_seg = k.ldq;
          pd.push_back(d);
        }
      }
      if (osh_status st = gemm(kEpiSplit, pd, 0.f); st != OSH_OK) return st;
      // G' = T1 Q_R, M' = T2 Q_R (fp32): A = T column-split view, B = Q_R row-split view
      pd.clear();
      for (const Cls& k : w.cls)
        for (size_t src : {k.T1s, k.T2s}) {
          NsProblemDesc d{};
          d.a = mref(d_ws_ + src, k.nb, k.p, 3 * k.ldq, 4ll * k.ldq,
                     static_cast<long long>(k.p) * 4 * k.ldq);
          d.b = mref(d_state_ + k.QRrs + 2ull * k.ldq * k.ldq, k.nb, 3 * k.ldq, k.q, k.ldq,
                     4ll * k.ldq * k.ldq);
          d.b_mn_major = 1;
          d.out = mref(d_ws_ + (src == k.T1s ? k.Gp : k.Mp), k.nb, k.p, k.q, k.ldq,
                       static_cast<long long>(k.p) * k.ldq);
          pd.push_back(d);
        }
      if (osh_status st = gemm(kEpiStat, pd, 0.f); st != OSH_OK) return st;
      // V update and the rotated Adam direction: G', M', V read, V and N' written
      OSH_CUDA_TRY(timed(kModeElementwise + 1, w.elems_pre * (4.0 * 4 + 2.0), [&] {
        return launch_soap_rot(d_rot_ + w.rot.first, w.rot.count, w.rot.tiles,
                               static_cast<float>(b2), ib1, ib2, eps, s);
      }));
      // T3 = Q_L N'
      pd.clear();
      for (const Cls& k : w.cls) {
        NsProblemDesc d{};
        d.a = S16(k.QLb, k.nb, k.p, k.p, k.ldp);
        d.b = B16(k.Nr, k.nb, k.p, k.q, k.ldq);
        d.b_mn_major = 1;
        d.out = B16(k.T3, k.nb, k.p, k.q, k.ldq);
        pd.push_back(d);
      }
      if (osh_status st = gemm(kEpiGram, pd, 0.f); st != OSH_OK) return st;
      // N = T3 Q_R^T (B K-major: [N][K] = Q_R row-major, the hi row segment of the split)
      pd.clear();
      for (const Cls& k : w.cls) {
        NsProblemDesc d{};
        d.a = B16(k.T3, k.nb, k.p, k.q, k.ldq);
        d.b = mref(d_state_ + k.QRrs, k.nb, k.q, k.q, k.ldq, 4ll * k.ldq * k.ldq);
        d.out = B16(k.Nb, k.nb, k.p, k.q, k.ldq);
        pd.push_back(d);
      }
      if (osh_status st = gemm(kEpiGram, pd, 0.f); st != OSH_OK) return st;
      // N read, w read + write, bf16 replica written
      OSH_CUDA_TRY(timed(kModeElementwise + 2, w.elems_pre * 12.0, [&] {
        return launch_soap_apply(d_apply_ + w.apply.first, w.apply.count, w.apply.tiles, lr, s);
      }));
    }
    // statistics L = bs L + (1 - bs) G G^T, R = bs R + (1 - bs) G^T G (after the step)
    pd.clear();
    for (const Cls& k : w.cls) {
      // bf16x3: A view (hi, lo, hi) at segment 0, B view (lo, hi, hi) at segment 1
      // (bf16 gradients: G is exact in hi, one segment hi x hi suffices)
      const bool exact = exact_grad_;
      const int ks = exact ? 1 : 3;
      const size_t b_off = exact ? 0 : 1;
      NsProblemDesc L{};
      const long long cpq = static_cast<long long>(k.p) * 4 * k.ldq;
      L.a = mref(d_ws_ + k.Gs, k.nb, k.p, ks * k.ldq, 4ll * k.ldq, cpq);
      L.b = mref(d_ws_ + k.Gs + 2ull * b_off * k.ldq, k.nb, k.p, ks * k.ldq, 4ll * k.ldq, cpq);
      L.out = S16(k.l.S, k.nb, k.p, k.p, k.ldp);
      L.scale = d_bscale_;
      L.symmetric = 2;  // upper triangle; refresh() fills the lower one first
      NsProblemDesc R{};
      const long long cqp = static_cast<long long>(k.q) * 4 * k.ldp;
      R.a = mref(d_ws_ + k.Gts, k.nb, k.q, ks * k.ldp, 4ll * k.ldp, cqp);
      R.b = mref(d_ws_ + k.Gts + 2ull * b_off * k.ldp, k.nb, k.q, ks * k.ldp, 4ll * k.ldp, cqp);
      R.out = S16(k.r.S, k.nb, k.q, k.q, k.ldq);
      R.scale = d_bscale_;
      R.symmetric = 2;
      pd.push_back(L);
      pd.push_back(R);
    }
    if (osh_status st = gemm(kEpiStat, pd, static_cast<float>(b2)); st != OSH_OK) return st;
    if (first || step_ % cfg_.precond_every == 0)
      if (osh_status st = refresh(w, first ? cfg_.init_iters : 1, !first, s); st != OSH_OK)
        return st;
  }
  if (first) return OSH_OK;  // update norms stay 0
  if (w.adam.count > 0)
    OSH_CUDA_TRY(timed(kModeElementwise + 3, w.elems_adam * (ges + 26.0), [&] {
      return launch_soap_adam(d_adam_ + w.adam.first, w.adam.count, w.adam.tiles, grad_dtype_,
                              static_cast<float>(b1), static_cast<float>(b2), ib1, ib2, eps, lr, s);
    }));
  if (w.slots.count > 0)
    OSH_CUDA_TRY(timed(kModeElementwise + 8, 0.0, [&] {
      return launch_partial_sums(d_partial_, d_slot_begin_ + w.slots.first,
                                 d_slot_count_ + w.slots.first, d_slot_target_ + w.slots.first,
                                 d_update_sq_, w.slots.count, s);
    }));
  return OSH_OK;
}

}  // namespace osh
