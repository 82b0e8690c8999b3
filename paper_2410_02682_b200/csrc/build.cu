// Kernel selection and cross-vertex fusion (ed_plan_h::build): maps every
// exec vertex of this rank onto a launch — region-fused tcgen05 GEMMs for
// mul/sum joins (kernel.cc:48-65), grouped memory-bound kernels, the exact
// generic kernel, aliases / rectangle folds for refinements
// (runtime.cc:198-269) — and fuses epilogue maps, the row softmax and the
// attention block where a region's chain runs on one rank.
#include "runtime.h"

namespace edrt {

// Merge the labels `cls` (in tensor order) of a row-major tensor into one
// strided dimension; fails if they are not one contiguous run.
bool merge_dim(const labels& tl, const shape& text, const labels& cls, Dim& out, labels& order) {
  shape strides(tl.size(), 1);
  for (int i = int(tl.size()) - 2; i >= 0; --i) strides[i] = strides[i + 1] * text[i + 1];
  std::vector<int> pos;
  for (size_t i = 0; i < tl.size(); ++i)
    if (std::find(cls.begin(), cls.end(), tl[i]) != cls.end() && text[i] > 1) pos.push_back(int(i));
  out = Dim{};
  order.clear();
  if (pos.empty()) return true;
  for (size_t j = 0; j + 1 < pos.size(); ++j)
    if (strides[pos[j]] != strides[pos[j + 1]] * text[pos[j + 1]]) return false;
  out.ext = 1;
  for (int q : pos) {
    out.ext *= text[q];
    order.push_back(tl[q]);
  }
  out.stride = strides[pos.back()];
  return true;
}

// merge_dim for a sub-box of a row-major tensor: the labels `cls` keep
// extents dst_ext of a tensor laid out with extents src_ext; fails if the kept
// part of the class is not one strided run (an inner label cut short).
static bool merge_sub(const labels& tl, const shape& src_ext, const shape& dst_ext, const labels& cls, Dim& out) {
  shape strides(tl.size(), 1);
  for (int i = int(tl.size()) - 2; i >= 0; --i) strides[i] = strides[i + 1] * src_ext[i + 1];
  std::vector<int> pos;
  for (size_t i = 0; i < tl.size(); ++i)
    if (std::find(cls.begin(), cls.end(), tl[i]) != cls.end() && dst_ext[i] > 1) pos.push_back(int(i));
  out = Dim{};
  if (pos.empty()) return true;
  for (size_t j = 0; j + 1 < pos.size(); ++j)
    if (strides[pos[j]] != strides[pos[j + 1]] * dst_ext[pos[j + 1]]) return false;
  out.ext = 1;
  for (int q : pos) out.ext *= dst_ext[q];
  out.stride = strides[pos.back()];
  return true;
}

bool map_gemm(const Vtx& v, const shape& local_xy, bool bf16, GemmMap& g, std::string& why) {
  if (v.arity != 2 || v.join != ED_JOIN_MUL || v.agg != ED_AGG_SUM) {
    why = "not mul/sum";
    return false;
  }
  std::map<int, int64_t> ext;
  for (size_t i = 0; i < v.lxy.size(); ++i) ext.emplace(v.lxy[i], local_xy[i]);
  auto extents = [&](const labels& ls) {
    shape r;
    for (auto l : ls) r.push_back(ext.at(l));
    return r;
  };
  auto has = [](const labels& ls, int l) { return std::find(ls.begin(), ls.end(), l) != ls.end(); };
  labels B, M, N, K;
  for (auto l : v.dls) {
    bool x = has(v.lx, l), y = has(v.ly, l), z = has(v.lz, l);
    if (x && y && z) B.push_back(l);
    else if (x && z) M.push_back(l);
    else if (y && z) N.push_back(l);
    else if (x && y) K.push_back(l);
    else if (ext.at(l) > 1) {
      why = "one-sided aggregation label";
      return false;
    }
  }
  // MMA-B must own the output's contiguous dimension.
  int inner = -1;
  for (int i = int(v.lz.size()) - 1; i >= 0; --i)
    if (ext.at(v.lz[i]) > 1) {
      inner = v.lz[i];
      break;
    }
  bool swap = inner >= 0 && has(M, inner);
  if (inner >= 0 && has(B, inner)) {
    why = "batch label is the output's contiguous dim";
    return false;
  }
  const labels& lA = swap ? v.ly : v.lx;
  const labels& lB = swap ? v.lx : v.ly;
  const labels& Mcls = swap ? N : M;
  const labels& Ncls = swap ? M : N;
  g.a_slot = swap ? 1 : 0;
  g.b_slot = swap ? 0 : 1;
  g.lA = lA;
  g.lB = lB;
  g.Mc = Mcls;
  g.Nc = Ncls;
  g.Kc = K;
  g.Bc = B;
  shape eA = extents(lA), eB = extents(lB), eZ = extents(v.lz);
  labels o1, o2, o3;
  bool ok = merge_dim(lA, eA, Mcls, g.am, o1) && merge_dim(v.lz, eZ, Mcls, g.cm, o2) && o1 == o2;
  ok = ok && merge_dim(lB, eB, Ncls, g.bn, o1) && merge_dim(v.lz, eZ, Ncls, g.cn, o2) && o1 == o2;
  ok = ok && merge_dim(lA, eA, K, g.ak, o1) && merge_dim(lB, eB, K, g.bk, o2) && o1 == o2;
  ok = ok && merge_dim(lA, eA, B, g.ab, o1) && merge_dim(lB, eB, B, g.bb, o2) && o1 == o2 &&
       merge_dim(v.lz, eZ, B, g.cb, o3) && o1 == o3;
  if (!ok) {
    why = "label classes are not contiguous runs";
    return false;
  }
  if (g.cn.ext > 1 && g.cn.stride != 1) {
    why = "output N not contiguous";
    return false;
  }
  g.a_mn = !(g.ak.ext == 1 || g.ak.stride == 1);
  if (g.a_mn && !(g.am.ext == 1 || g.am.stride == 1)) {
    why = "A has no unit-stride M or K";
    return false;
  }
  g.b_mn = !(g.bk.ext == 1 || g.bk.stride == 1);
  if (g.b_mn && !(g.bn.ext == 1 || g.bn.stride == 1)) {
    why = "B has no unit-stride N or K";
    return false;
  }
  const int es = bf16 ? 2 : 4;
  auto aligned = [&](const Dim& d) { return d.ext == 1 || (d.stride * es) % 16 == 0; };
  // outer (non-unit) strides of each TMA view must be 16-byte multiples
  if (!(aligned(g.a_mn ? g.ak : g.am) && aligned(g.ab) && aligned(g.b_mn ? g.bk : g.bn) && aligned(g.bb))) {
    why = "operand strides not 16-byte aligned";
    return false;
  }
  if (g.am.ext > INT32_MAX || g.bn.ext > INT32_MAX || g.ak.ext > INT32_MAX || g.ab.ext > 65535) {
    why = "extent too large";
    return false;
  }
  return true;
}

bool map_memory(const Vtx& v, const shape& local_xy, bool f64, MemMap& m) {
  std::map<int, int64_t> ext;
  for (size_t i = 0; i < v.lxy.size(); ++i) ext.emplace(v.lxy[i], local_xy[i]);
  auto prod_of = [&](const labels& ls, size_t from, size_t to) {
    int64_t r = 1;
    for (size_t i = from; i < to; ++i) r *= ext.at(ls[i]);
    return r;
  };
  const bool has_agg = v.agg >= 0;
  if (!has_agg) {
    if (v.lx != v.lz) return false;
    m.kind = OpKind::EWISE;
    if (v.arity == 1) return true;
    if (v.ly == v.lz) {
      m.y_mode = 1;
      return true;
    }
    // y's labels a prefix of z's: broadcast over the trailing block
    if (v.ly.size() < v.lz.size() && std::equal(v.ly.begin(), v.ly.end(), v.lz.begin())) {
      m.y_mode = 2;
      m.inner = prod_of(v.lz, v.ly.size(), v.lz.size());
      return m.inner % (f64 ? 2 : 4) == 0;
    }
    return false;
  }
  if (v.arity != 1) return false;
  // z's labels a prefix of x's: fold x's trailing labels (kernel_eval order)
  if (v.lz.size() >= v.lx.size() || !std::equal(v.lz.begin(), v.lz.end(), v.lx.begin())) return false;
  m.kind = OpKind::ROWREDUCE;
  m.rows = prod_of(v.lx, 0, v.lz.size());
  m.len = prod_of(v.lx, v.lz.size(), v.lx.size());
  return true;
}

}  // namespace edrt

void ed_plan_h::build() {
  const int ne = int(X.size());
  const int me = ctx->rank;
  owner.resize(ne);
  std::iota(owner.begin(), owner.end(), 0);
  local.assign(ne, 0);
  buf.assign(ne, Buffer{});
  for (int id = 0; id < ne; ++id) local[id] = rank_of(id) == me;

  const bool x3 = opt.precision == ED_PREC_F32X3;
  const bool tc = opt.precision == ED_PREC_TF32 || opt.precision == ED_PREC_BF16 || x3;
  const bool bf16 = opt.precision == ED_PREC_BF16;
  const int max_sib = kMaxSib;  // siblings K-concatenated into one accumulator (x3: one stage feeds all three products)

  // ---- per einsum: kernel class and region fusion ----
  std::map<int, GemmMap> gmap;
  std::map<int, std::string> why_not;
  std::vector<char> fused_head(ne, 0);       // join id -> emits the region's GEMM
  std::map<int, std::vector<int>> region_sibs;  // head join -> sibling joins (fold order)
  for (int w = 0; w < int(V.size()); ++w) {
    if (V[w].arity == 0) continue;
    GemmMap g;
    std::string why;
    if (tc && map_gemm(V[w], local_xy(w), bf16, g, why)) gmap[w] = g;
    else why_not[w] = why;
    MemMap mm;
    if (!gmap.count(w) && map_memory(V[w], local_xy(w), f64, mm)) memmap_[w] = mm;
  }
  {
    std::map<std::pair<int, shape>, std::vector<int>> regions;
    for (int id = 0; id < ne; ++id)
      if (X[id].kind == ED_EXEC_JOIN && local[id] && gmap.count(X[id].producer))
        regions[{X[id].producer, region_key(id)}].push_back(id);
    // consumers of each join (a sibling may only be folded into its region's
    // accumulator when everything that reads it runs on this rank)
    std::vector<char> remote_reader(ne, 0);
    for (int id = 0; id < ne; ++id)
      for (int d : X[id].deps)
        if (rank_of(id) != me) remote_reader[d] = 1;
    for (auto& [k, sibs] : regions) {
      bool all_local = std::none_of(sibs.begin(), sibs.end(), [&](int s) { return remote_reader[s]; });
      if (int(sibs.size()) <= max_sib && (all_local || sibs.size() == 1)) {
        fused_head[sibs[0]] = 1;
        region_sibs[sibs[0]] = sibs;
        for (int s : sibs) owner[s] = sibs[0];
      } else {
        for (int s : sibs) {
          fused_head[s] = 1;
          region_sibs[s] = {s};
        }
      }
    }
  }

  // remote dependencies become local copies received over NCCL
  std::vector<std::pair<int, int>> transfers;  // (dep, destination rank), global order
  {
    std::set<std::pair<int, int>> seen;
    for (int id = 0; id < ne; ++id) {
      if (X[id].kind == ED_EXEC_INPUT_CHUNK) continue;
      int dst = rank_of(id);
      for (int d : X[id].deps)
        if (rank_of(d) != dst && seen.insert({d, dst}).second) transfers.push_back({d, dst});
    }
  }

  // ---- refinements: effective sources, aliasing ----
  struct Src {
    int id;
    shape r0, ext;
  };
  std::vector<std::vector<Src>> srcs(ne);
  const std::vector<int> owner0 = owner;  // after sibling fusion
  std::vector<char> virt(ne, 0);          // exec vertices fused away (never computed)
  opaque_.assign(ne, 0);
  std::map<int, std::pair<int, double>> epi;  // GEMM einsum -> (map op, c) applied in its epilogue
  auto alias_pass = [&](const std::map<int, int>& virtual_join_src) {
    owner = owner0;
    for (int id = 0; id < ne; ++id) {
      srcs[id].clear();
      const Ex& u = X[id];
      if (!local[id]) continue;
      if (u.kind == ED_EXEC_JOIN) {
        auto it = virtual_join_src.find(id);
        if (it != virtual_join_src.end()) owner[id] = owner[u.deps[it->second]];
        continue;
      }
      if (u.kind != ED_EXEC_REFINEMENT) continue;
      const shape& bound = V[u.producer].bound;
      std::set<int> used;
      for (int d : u.deps) {
        int o = local[d] ? owner[d] : d;  // remote deps arrive as their own chunks
        if (!used.insert(o).second) continue;
        shape rk = region_key(d), dr = region_partition(d), r0(bound.size()), ext(bound.size());
        for (size_t i = 0; i < bound.size(); ++i) {
          ext[i] = bound[i] / dr[i];
          r0[i] = rk[i] * ext[i];
        }
        srcs[id].push_back({o, r0, ext});
      }
      // a refinement that is exactly one producer chunk is that chunk
      const shape dc = region_partition(id);
      if (srcs[id].size() == 1) {
        bool same = true;
        for (size_t i = 0; i < bound.size(); ++i)
          same = same && srcs[id][0].r0[i] == u.key[i] * (bound[i] / dc[i]) && srcs[id][0].ext[i] == u.cb[i];
        if (same) owner[id] = owner[srcs[id][0].id];
      }
    }
  };
  alias_pass({});

  // ---- cross-vertex fusion (tensor-core modes; exact modes keep every vertex) ----
  std::map<int, int> virtual_join_src;  // fused join -> dep slot whose buffer it becomes
  if (tc) {
    const int nv = int(V.size());
    std::vector<std::vector<int>> readers(nv);
    for (int w = 0; w < nv; ++w)
      for (int k = 0; k < V[w].arity; ++k) readers[V[w].inputs[k]].push_back(w);
    auto is_output = [&](int w) { return std::find(outputs.begin(), outputs.end(), w) != outputs.end(); };
    // Fusions are decided per rank: a vertex can be fused on this rank when it
    // has work here and none of the chunks it makes here is read by another
    // rank (what other ranks need is never fused away). With one rank this is
    // "all of its exec vertices are local".
    std::vector<char> remote_read(ne, 0);
    for (int id = 0; id < ne; ++id)
      if (!local[id])
        for (int d : X[id].deps) remote_read[d] = 1;
    // fused away on this rank: has work here, and no chunk it makes here is
    // read by another rank
    auto all_local = [&](int w) {
      bool any = false;
      for (int id = 0; id < ne; ++id) {
        if (X[id].producer != w || X[id].kind == ED_EXEC_INPUT_CHUNK || !local[id]) continue;
        if (remote_read[id]) return false;
        any = true;
      }
      return any;
    };
    // computed inside a fused kernel but still materialised: work here suffices
    auto has_local = [&](int w) {
      for (int id = 0; id < ne; ++id)
        if (X[id].producer == w && X[id].kind == ED_EXEC_JOIN && local[id]) return true;
      return false;
    };
    auto joins_of = [&](int w) {  // this rank's joins of w
      std::vector<int> r;
      for (int id = 0; id < ne; ++id)
        if (X[id].kind == ED_EXEC_JOIN && X[id].producer == w && local[id]) r.push_back(id);
      return r;
    };
    auto sole_reader = [&](int w, int r) {
      return readers[w].size() == 1 && readers[w][0] == r && !is_output(w);
    };
    // (1) map epilogue: v = map(u), u a region-fused GEMM read only by v
    for (int v = 0; v < nv; ++v) {
      if (!memmap_.count(v) || memmap_[v].kind != OpKind::EWISE || V[v].arity != 1) continue;
      const int u = V[v].inputs[0];
      if (!gmap.count(u) || !sole_reader(u, v) || !all_local(u) || !has_local(v)) continue;
      if (V[v].map == ED_MAP_EXP) continue;  // only cheap maps go into the epilogue
      bool ok = true;
      for (int j : joins_of(v)) {
        const int o = owner[X[j].deps[0]];
        ok = ok && fused_head[o] && X[o].producer == u;
      }
      if (!ok) continue;
      epi[u] = {V[v].map, V[v].c};
      for (int j : joins_of(v)) virtual_join_src[j] = 0;
      // u's own values never exist: its chunks hold map(u)
      for (int id = 0; id < ne; ++id)
        if (X[id].producer == u && X[id].kind != ED_EXEC_INPUT_CHUNK && local[id]) opaque_[id] = 1;
      memmap_.erase(v);
    }
    alias_pass(virtual_join_src);
    // (2) row softmax: M = max(X), S = sub(X, M), E = exp(S), Sg = sum(E), Y = div(E, Sg)
    for (int y = 0; y < nv; ++y) {
      auto is = [&](int w, OpKind k, int arity, int op) {
        return w >= 0 && memmap_.count(w) && memmap_[w].kind == k && V[w].arity == arity &&
               (arity == 2 ? V[w].join == op : (k == OpKind::ROWREDUCE ? V[w].agg == op : V[w].map == op));
      };
      if (!is(y, OpKind::EWISE, 2, ED_JOIN_DIV) || memmap_[y].y_mode != 2) continue;
      const int e = V[y].inputs[0], sg = V[y].inputs[1];
      if (!is(e, OpKind::EWISE, 1, ED_MAP_EXP) || !is(sg, OpKind::ROWREDUCE, 1, ED_AGG_SUM)) continue;
      if (V[sg].map != ED_MAP_IDENTITY || V[sg].inputs[0] != e) continue;
      const int sv = V[e].inputs[0];
      if (!is(sv, OpKind::EWISE, 2, ED_JOIN_SUB) || memmap_[sv].y_mode != 2) continue;
      const int xv = V[sv].inputs[0], m = V[sv].inputs[1];
      if (!sole_reader(sv, e) || !sole_reader(sg, y) || is_output(e) || readers[e].size() != 2) continue;
      if (!all_local(sv) || !all_local(e) || !all_local(sg) || !has_local(y)) continue;
      const int64_t L = memmap_[sg].len;
      if (memmap_[sv].inner != L || memmap_[y].inner != L) continue;
      if (L % 4 != 0 || L > 128 * 64 || f64) continue;  // the fused kernel keeps a row in registers
      // M joins the chain when it is the row max of the same, aligned x chunks;
      // otherwise (e.g. its label is split with a sibling fold) M is computed
      // as planned and the chain reads the materialised row maxima
      const bool m_max = is(m, OpKind::ROWREDUCE, 1, ED_AGG_MAX) && V[m].map == ED_MAP_IDENTITY &&
                         V[m].inputs[0] == xv && sole_reader(m, sv) && all_local(m);
      const bool m_fusable = m_max && memmap_[m].len == L;
      // M's reduced labels split over siblings (a max fold in its refinement):
      // when the chain's rows are whole rows of x, the row max the kernel
      // takes in registers IS M's value (max is exact and order-free), so M's
      // joins and fold are fused away too
      bool m_full_rows = false;
      if (m_max && !m_fusable) {
        int64_t ext = 1;
        for (size_t i = 0; i < V[m].lx.size(); ++i)
          if (std::find(V[m].lz.begin(), V[m].lz.end(), V[m].lx[i]) == V[m].lz.end()) ext *= V[xv].bound[i];
        m_full_rows = ext == L;
      }
      auto join_at = [&](int ref, int w) {
        const int o = owner[ref];
        return (X[o].kind == ED_EXEC_JOIN && X[o].producer == w && local[o]) ? o : -1;
      };
      Softmax sm;
      bool ok = true, internal = m_fusable || m_full_rows;
      for (int attempt = 0; attempt < 2 && !sm.pairs.size(); ++attempt) {
        ok = true;
        sm.pairs.clear();
        sm.m_refs.clear();
        for (int yj : joins_of(y)) {
          const int ej = join_at(X[yj].deps[0], e), sgj = join_at(X[yj].deps[1], sg);
          const int sj = ej >= 0 ? join_at(X[ej].deps[0], sv) : -1;
          ok = ok && ej >= 0 && sgj >= 0 && sj >= 0 && owner[X[sgj].deps[0]] == ej && X[yj].sz == X[sj].sz &&
               X[yj].sz % L == 0;
          if (ok && internal && !m_full_rows) {
            const int mj = join_at(X[sj].deps[1], m);
            ok = mj >= 0 && owner[X[mj].deps[0]] == owner[X[sj].deps[0]];
          }
          if (!ok) break;
          sm.pairs.push_back({yj, X[sj].deps[0]});
          if (!internal) sm.m_refs.push_back(X[sj].deps[1]);
        }
        if (!ok) {
          sm.pairs.clear();
          if (!internal) break;
          internal = false;  // retry with the row maxima read from memory
        }
      }
      if (!ok || sm.pairs.empty()) continue;
      sm.y = y;
      sm.x = xv;
      sm.len = L;
      softmax_[y] = sm;
      std::vector<int> gone = {sv, e, sg};
      if (internal) gone.push_back(m);
      for (int w : gone)
        for (int id = 0; id < ne; ++id)
          if (X[id].producer == w && X[id].kind != ED_EXEC_INPUT_CHUNK) virt[id] = 1;
      for (int w : gone) memmap_.erase(w);
    }
    // (3) attention block: T1 = Q K^T (GEMM, maybe with a fused scale), the
    // softmax chain on T1 (or its scaled map), O = T3 V (GEMM, K = the row
    // label) -> one kernel; T1 and T3 are never materialised (bf16:
    // attn_sm100.cu; fp32x3: attn_x3_sm100.cu)
    static const bool ftrace = std::getenv("ED_FUSE_TRACE") != nullptr;
#define REJECT(k)                                                                            \
  {                                                                                          \
    if (ftrace) std::fprintf(stderr, "[ed] rank %d: attention block at %s not fused (%d)\n", me, \
                             V[yv].name.c_str(), k);                                         \
    continue;                                                                                \
  }
    for (auto& [yv, sm] : softmax_) {
      if (!bf16 && !(x3 && x3_attention_fused())) break;
      if (readers[yv].size() != 1 || is_output(yv) || !sm.m_refs.empty()) REJECT(1)
      const int o = readers[yv][0];
      if (!gmap.count(o) || V[o].inputs[gmap[o].a_slot] != yv || !has_local(o) || !all_local(yv)) REJECT(2)
      int t1 = sm.x;
      float scale = 1.0f;
      if (!gmap.count(t1)) {
        // x is a map vertex fused into its GEMM's epilogue (T2 = scale(T1))
        const int u = V[t1].arity == 1 ? V[t1].inputs[0] : -1;
        if (u < 0 || !epi.count(u) || epi[u].first != ED_MAP_SCALE || !all_local(t1)) REJECT(3)
        scale = float(epi[u].second);
        t1 = u;
      } else if (epi.count(t1)) {
        REJECT(4)
      }
      if (!gmap.count(t1) || !all_local(t1)) REJECT(5)
      const GemmMap& gs = gmap[t1];
      const GemmMap& go = gmap[o];
      const int64_t H = gs.ab.ext, S = gs.am.ext, T = gs.bn.ext, Dd = gs.ak.ext;
      if (gs.a_mn || gs.b_mn || !go.b_mn || go.a_mn || go.ab.ext != H || go.am.ext != S || go.ak.ext != T ||
          go.bn.ext != Dd || T != sm.len ||
          !(x3 ? attn_x3_supported(int(S), int(T), int(Dd)) : attn_supported(int(S), int(T), int(Dd))))
        REJECT(6)
      // region correspondence: O region <- T3 chunk <- T1 region (single siblings)
      std::map<int, int> t1_of_y;
      for (auto& [yj, xr] : sm.pairs) t1_of_y[yj] = owner[xr];
      Flash f{t1, yv, o, scale, {}};
      bool ok = true;
      for (int oh = 0; oh < ne && ok; ++oh) {
        if (!fused_head[oh] || X[oh].producer != o) continue;
        ok = region_sibs[oh].size() == 1;
        const int yj = owner[X[oh].deps[go.a_slot]];
        auto it = t1_of_y.find(yj);
        ok = ok && it != t1_of_y.end();
        if (!ok) break;
        const int th = it->second;
        ok = fused_head[th] && X[th].producer == t1 && region_sibs[th].size() == 1;
        if (!ok && ftrace) std::fprintf(stderr, "[ed] rank %d: O region %d <- T1 join %d (head %d, sibs %zu)\n", me, oh, th, int(fused_head[th]), region_sibs[th].size());
        if (!ok) break;
        f.regions.push_back({X[th].deps[gs.a_slot], X[th].deps[gs.b_slot], X[oh].deps[go.b_slot], oh});
      }
      if (!ok || f.regions.empty()) REJECT(8)
#undef REJECT
      // K (T1's B) and V (O's B): read in place from their producers' regions
      // when the pasting refinement is a regular grid over (keys, d)
      auto tile = [&](int ref, const labels& lop, int keyl, int dl, int hl, KVTiles& t) {
        const Ex& R = X[ref];
        if (R.kind != ED_EXEC_REFINEMENT || !local[ref] || owner[ref] != ref || virt[ref] || srcs[ref].size() < 2 ||
            lop.size() != 3)
          return false;
        const int kd = int(std::find(lop.begin(), lop.end(), keyl) - lop.begin());
        const int dd = int(std::find(lop.begin(), lop.end(), dl) - lop.begin());
        const int hd = int(std::find(lop.begin(), lop.end(), hl) - lop.begin());
        if (kd > 2 || dd != 2 || hd > 2 || kd == hd) return false;  // d must be the contiguous label
        const shape& bound = V[R.producer].bound;
        const shape dc = region_partition(ref);
        shape cs(3);
        for (int i = 0; i < 3; ++i) cs[i] = R.key[i] * (bound[i] / dc[i]);
        const auto& S = srcs[ref];
        t.keys = S[0].ext[kd];
        t.dw = S[0].ext[dd];
        t.hoff = cs[hd] - S[0].r0[hd];
        t.ext = S[0].ext;
        if (t.keys % 128 || t.dw % 64 || R.cb[kd] % t.keys || R.cb[dd] % t.dw) return false;
        const int nk = int(R.cb[kd] / t.keys);
        t.nd = int(R.cb[dd] / t.dw);
        t.owners.assign(size_t(nk) * t.nd, -1);
        for (auto& sr : S) {
          if (!local[sr.id] || sr.ext != t.ext || cs[hd] - sr.r0[hd] != t.hoff || sr.r0[hd] > cs[hd] ||
              sr.r0[hd] + sr.ext[hd] < cs[hd] + R.cb[hd])
            return false;
          const int64_t ko = sr.r0[kd] - cs[kd], dof = sr.r0[dd] - cs[dd];
          if (ko % t.keys || dof % t.dw || ko < 0 || dof < 0) return false;
          int& cell = t.owners[size_t(ko / t.keys) * t.nd + size_t(dof / t.dw)];
          if (cell >= 0) return false;
          cell = sr.id;
        }
        for (int c : t.owners)
          if (c < 0) return false;
        t.tiled = true;
        return true;
      };
      const labels& lk = gs.b_slot == 0 ? V[t1].lx : V[t1].ly;
      const labels& lv = go.b_slot == 0 ? V[o].lx : V[o].ly;
      bool kv_ok = true;
      for (auto& r : f.regions) {
        KVTiles kt, vt;
        kv_ok = kv_ok && gs.Nc.size() == 1 && gs.Kc.size() == 1 && gs.Bc.size() == 1 && go.Kc.size() == 1 &&
                go.Nc.size() == 1 && go.Bc.size() == 1 && tile(r[1], lk, gs.Nc[0], gs.Kc[0], gs.Bc[0], kt) &&
                tile(r[2], lv, go.Kc[0], go.Nc[0], go.Bc[0], vt);
        f.ktiles.push_back(kt);
        f.vtiles.push_back(vt);
      }
      if (kv_ok) {
        for (auto& r : f.regions) {
          virt[r[1]] = 1;
          virt[r[2]] = 1;
        }
      } else {
        f.ktiles.assign(f.regions.size(), KVTiles{});
        f.vtiles.assign(f.regions.size(), KVTiles{});
      }
      flash_[o] = f;
      flash_skip_.insert(t1);
      flash_skip_.insert(yv);
      flash_skip_.insert(o);
      // T1's regions/refinements and T3's joins/refinements are never materialised
      for (int id = 0; id < ne; ++id) {
        const int w = X[id].producer;
        if ((w == t1 || w == yv) && X[id].kind != ED_EXEC_INPUT_CHUNK) virt[id] = 1;
      }
    }
  }

  // ---- K-segmented operands: a GEMM operand that is a refinement pasting
  // several producer regions along the contraction label is read straight
  // from those regions (one pseudo-sibling per segment), never copied ----
  kseg_.clear();
  for (auto& [c, g] : gmap) {
    if (flash_skip_.count(c)) continue;
    bool c_local = true;
    for (int id = 0; id < ne; ++id)
      if (X[id].producer == c && !local[id]) c_local = false;
    if (!c_local) continue;
    std::vector<int> kl;
    for (auto l : g.Kc) kl.push_back(l);
    if (kl.size() != 1) continue;
    for (int role = 0; role < 2 && !kseg_.count(c); ++role) {
      const int slot = role == 0 ? g.a_slot : g.b_slot;
      const labels& lop = slot == 0 ? V[c].lx : V[c].ly;
      const int kd = int(std::find(lop.begin(), lop.end(), kl[0]) - lop.begin());
      KSeg ks;
      ks.role = role;
      bool ok = true;
      std::vector<int> refs;
      int real_max = 1;
      for (int jid = 0; jid < ne && ok; ++jid) {
        if (X[jid].kind != ED_EXEC_JOIN || X[jid].producer != c) continue;
        const int ref = X[jid].deps[slot];
        const Ex& R = X[ref];
        ok = R.kind == ED_EXEC_REFINEMENT && local[ref] && owner[ref] == ref && !virt[ref] && srcs[ref].size() >= 2;
        if (!ok) break;
        const shape& bound = V[R.producer].bound;
        const shape dc = region_partition(ref);
        std::vector<Seg> segs;
        std::set<int64_t> starts;
        for (auto& sr : srcs[ref]) {
          for (size_t d = 0; d < bound.size() && ok; ++d) {
            const int64_t c0 = R.key[d] * (bound[d] / dc[d]);
            if (int(d) == kd) ok = sr.r0[d] >= c0 && sr.r0[d] + sr.ext[d] <= c0 + R.cb[d];
            else ok = sr.r0[d] == c0 && sr.ext[d] == R.cb[d];
          }
          ok = ok && starts.insert(sr.r0[kd]).second && local[sr.id];
          if (!ok) break;
          Seg sg;
          sg.owner = sr.id;
          sg.k0 = sr.r0[kd] - R.key[kd] * (bound[kd] / dc[kd]);
          sg.kext = sr.ext[kd];
          labels o1;
          const labels& mcls = role == 0 ? g.Mc : g.Nc;
          ok = merge_dim(lop, sr.ext, mcls, sg.mn, o1) && merge_dim(lop, sr.ext, g.Kc, sg.k, o1) &&
               merge_dim(lop, sr.ext, g.Bc, sg.b, o1);
          segs.push_back(sg);
        }
        if (!ok) break;
        std::sort(segs.begin(), segs.end(), [](const Seg& a, const Seg& b) { return a.k0 < b.k0; });
        int64_t covered = 0;
        for (auto& sg : segs) {
          ok = ok && sg.kext == segs[0].kext && sg.k0 == covered;
          covered += sg.kext;
        }
        ok = ok && covered == R.cb[kd];
        if (!ok) break;
        // the other operand is sliced along K: its segment starts must stay 16-byte aligned
        const Dim& ok_dim = role == 0 ? g.bk : g.ak;
        for (auto& sg : segs) ok = ok && (sg.k0 * ok_dim.stride * (bf16 ? 2 : 4)) % 16 == 0;
        if (ks.kseg < 0) ks.kseg = segs[0].kext;
        ok = ok && ks.kseg == segs[0].kext;
        ks.segs[jid] = segs;
        refs.push_back(ref);
        const int real = fused_head[owner[jid]] ? int(region_sibs[owner[jid]].size()) : 1;
        real_max = std::max(real_max, real);
        ok = ok && real * int(segs.size()) <= kMaxSib;
      }
      if (!ok || refs.empty()) continue;
      kseg_[c] = ks;
      for (int ref : refs) virt[ref] = 1;
    }
  }

  // ---- batch-segmented operands: a GEMM operand that is a refinement pasting
  // producer regions along the batch label (e.g. C2's repartition from
  // batch-sharded Z1 chunks to row-sharded Z2 inputs) is read in place: the
  // tiles of batch b load it from segment b / bseg through that segment's own
  // tensor map, offset to the sub-box the refinement keeps, so the pasted
  // chunk is never materialised (runtime.cc:198-269 copies it) ----
  bseg_.clear();
  for (auto& [c, g] : gmap) {
    if (flash_skip_.count(c) || kseg_.count(c) || g.Bc.size() != 1) continue;
    bool c_local = true;
    for (int id = 0; id < ne; ++id)
      if (X[id].producer == c && !local[id]) c_local = false;
    if (!c_local) continue;
    for (int role = 0; role < 2 && !bseg_.count(c); ++role) {
      const int slot = role == 0 ? g.a_slot : g.b_slot;
      const labels& lop = slot == 0 ? V[c].lx : V[c].ly;
      const int bd = int(std::find(lop.begin(), lop.end(), g.Bc[0]) - lop.begin());
      if (bd >= int(lop.size())) continue;
      const Dim& want_mn = role == 0 ? g.am : g.bn;
      const Dim& want_k = role == 0 ? g.ak : g.bk;
      BSeg bs;
      bs.role = role;
      bool ok = true;
      std::vector<int> refs;
      for (int jid = 0; jid < ne && ok; ++jid) {
        if (X[jid].kind != ED_EXEC_JOIN || X[jid].producer != c) continue;
        const int ref = X[jid].deps[slot];
        const Ex& R = X[ref];
        ok = R.kind == ED_EXEC_REFINEMENT && local[ref] && owner[ref] == ref && !virt[ref] && srcs[ref].size() >= 2 &&
             R.cb.size() == lop.size();
        if (!ok) break;
        const shape& bound = V[R.producer].bound;
        const shape dc = region_partition(ref);
        std::vector<Seg> segs;
        for (auto& sr : srcs[ref]) {
          shape de(lop.size());
          int64_t off = 0, st = 1;
          for (int d = int(lop.size()) - 1; d >= 0 && ok; --d) {
            const int64_t c0 = R.key[size_t(d)] * (bound[size_t(d)] / dc[size_t(d)]), ce = R.cb[size_t(d)];
            if (d == bd) {
              ok = sr.r0[d] >= c0 && sr.r0[d] + sr.ext[d] <= c0 + ce;
              de[d] = sr.ext[d];
            } else {
              ok = sr.r0[d] <= c0 && sr.r0[d] + sr.ext[d] >= c0 + ce;
              de[d] = ce;
              off += (c0 - sr.r0[d]) * st;
            }
            st *= sr.ext[d];
          }
          ok = ok && local[sr.id];
          if (!ok) break;
          Seg sg;
          sg.owner = sr.id;
          sg.k0 = sr.r0[bd] - R.key[size_t(bd)] * (bound[size_t(bd)] / dc[size_t(bd)]);
          sg.kext = sr.ext[bd];
          sg.off = off;
          const labels& mcls = role == 0 ? g.Mc : g.Nc;
          ok = merge_sub(lop, sr.ext, de, mcls, sg.mn) && merge_sub(lop, sr.ext, de, g.Kc, sg.k) &&
               merge_sub(lop, sr.ext, de, g.Bc, sg.b);
          // the segment must present exactly the GEMM's operand shape
          ok = ok && sg.mn.ext == want_mn.ext && sg.k.ext == want_k.ext && sg.b.ext == sg.kext &&
               (sg.off * (bf16 ? 2 : 4)) % 16 == 0;
          segs.push_back(sg);
        }
        if (!ok) break;
        std::sort(segs.begin(), segs.end(), [](const Seg& a, const Seg& b) { return a.k0 < b.k0; });
        int64_t covered = 0;
        for (auto& sg : segs) {
          ok = ok && sg.kext == segs[0].kext && sg.k0 == covered;
          covered += sg.kext;
        }
        ok = ok && covered == R.cb[size_t(bd)] && (bs.bseg == 0 || bs.bseg == segs[0].kext);
        if (!ok) break;
        bs.bseg = segs[0].kext;
        bs.segs[jid] = segs;
        refs.push_back(ref);
      }
      if (!ok || refs.empty()) continue;
      bseg_[c] = bs;
      for (int ref : refs) virt[ref] = 1;
    }
  }

  // softmax inputs that are a paste of column segments (rank 2) are read in place
  for (auto& [y, sm] : softmax_) {
    bool ok = true;
    std::vector<std::vector<Softmax::XSeg>> all;
    int w_all = 0;
    for (auto& [yj, xr] : sm.pairs) {
      const Ex& R = X[xr];
      ok = R.kind == ED_EXEC_REFINEMENT && local[xr] && owner[xr] == xr && !virt[xr] && srcs[xr].size() >= 2 &&
           R.cb.size() == 2 && R.cb[1] == sm.len;
      if (!ok) break;
      const shape& bound = V[R.producer].bound;
      const shape dc = region_partition(xr);
      const int64_t rs = R.key[0] * (bound[0] / dc[0]), cs = R.key[1] * (bound[1] / dc[1]);
      std::vector<std::pair<int64_t, Softmax::XSeg>> segs;
      for (auto& sr : srcs[xr]) {
        ok = ok && local[sr.id] && sr.r0[0] <= rs && sr.r0[0] + sr.ext[0] >= rs + R.cb[0] && sr.ext[1] % 4 == 0;
        segs.push_back({sr.r0[1] - cs, Softmax::XSeg{sr.id, rs - sr.r0[0], sr.ext[1]}});
      }
      std::sort(segs.begin(), segs.end(), [](auto& a, auto& b) { return a.first < b.first; });
      const int64_t wdt = srcs[xr][0].ext[1];
      for (size_t k = 0; k < segs.size() && ok; ++k) ok = segs[k].first == int64_t(k) * wdt && srcs[xr][k].ext[1] == wdt;
      ok = ok && int64_t(segs.size()) * wdt == sm.len && (w_all == 0 || w_all == wdt);
      if (!ok) break;
      w_all = int(wdt);
      std::vector<Softmax::XSeg> v;
      for (auto& q : segs) v.push_back(q.second);
      all.push_back(v);
    }
    if (!ok || all.empty()) continue;
    sm.xsegs = all;
    sm.seg_w = w_all;
    for (auto& pr : sm.pairs) virt[pr.second] = 1;
  }

  auto gemm_reads = [&](int jid) {
    std::vector<int> r;
    const int w = X[jid].producer;
    for (int k = 0; k < int(X[jid].deps.size()); ++k) {
      const int d = X[jid].deps[k];
      if (kseg_.count(w) && k == (kseg_[w].role == 0 ? gmap[w].a_slot : gmap[w].b_slot)) {
        for (auto& sg : kseg_[w].segs.at(jid)) r.push_back(sg.owner);
      } else if (bseg_.count(w) && k == (bseg_[w].role == 0 ? gmap[w].a_slot : gmap[w].b_slot)) {
        for (auto& sg : bseg_[w].segs.at(jid)) r.push_back(sg.owner);
      } else {
        r.push_back(local[d] ? owner[d] : d);
      }
    }
    return r;
  };

  // ---- buffer needs ----
  for (int id = 0; id < ne; ++id) {
    if (!local[id] || virt[id] || virtual_join_src.count(id)) continue;
    const Ex& u = X[id];
    if (u.kind == ED_EXEC_JOIN && flash_.count(u.producer)) {
      const Flash& f = flash_[u.producer];
      for (size_t q = 0; q < f.regions.size(); ++q) {
        const auto& r = f.regions[q];
        if (r[3] != id) continue;
        auto need = [&](int o2) {  // bf16: the shadow; fp32x3: the value and its lo shadow
          if (x3) {
            buf[o2].need_main = true;
            buf[o2].need_lo = true;
          } else {
            buf[o2].need_16 = true;
          }
        };
        need(local[r[0]] ? owner[r[0]] : r[0]);
        for (int k = 1; k < 3; ++k) {
          const KVTiles& t = k == 1 ? f.ktiles[q] : f.vtiles[q];
          if (t.tiled)
            for (int o2 : t.owners) need(o2);
          else
            need(local[r[k]] ? owner[r[k]] : r[k]);
        }
      }
      continue;
    }
    if (u.kind == ED_EXEC_JOIN && softmax_.count(u.producer)) {
      const Softmax& sm = softmax_[u.producer];
      for (size_t k = 0; k < sm.pairs.size(); ++k)
        if (sm.pairs[k].first == id) {
          if (!sm.xsegs.empty())
            for (auto& xs : sm.xsegs[k]) buf[xs.owner].need_main = true;
          else
            buf[owner[sm.pairs[k].second]].need_main = true;
          if (!sm.m_refs.empty()) buf[owner[sm.m_refs[k]]].need_main = true;
        }
      continue;
    }
    if (u.kind == ED_EXEC_INPUT_CHUNK) buf[owner[id]].need_main = true;
    if (u.kind == ED_EXEC_JOIN) {
      int w = u.producer;
      if (gmap.count(w)) {
        std::vector<int> reads;
        for (int k = 0; k < int(u.deps.size()); ++k) {
          const int d = u.deps[k];
          const bool segmented = kseg_.count(w) && k == (kseg_[w].role == 0 ? gmap[w].a_slot : gmap[w].b_slot);
          const bool bsegmented = bseg_.count(w) && k == (bseg_[w].role == 0 ? gmap[w].a_slot : gmap[w].b_slot);
          if (segmented) {
            for (auto& sg : kseg_[w].segs.at(id)) reads.push_back(sg.owner);
          } else if (bsegmented) {
            for (auto& sg : bseg_[w].segs.at(id)) reads.push_back(sg.owner);
          } else {
            reads.push_back(local[d] ? owner[d] : d);
          }
        }
        for (int o : reads) {
          if (bf16) buf[o].need_16 = true;
          else buf[o].need_main = true;
          if (x3) buf[o].need_lo = true;
        }
      } else {
        for (int d : u.deps) buf[local[d] ? owner[d] : d].need_main = true;
      }
    }
    if (u.kind == ED_EXEC_REFINEMENT) {
      if (owner[id] == id)
        for (auto& s : srcs[id]) buf[s.id].need_main = true;
      if (u.consumer < 0) buf[owner[id]].need_main = true;  // graph output / sink
    }
  }
  // data that leaves this rank travels in the storage dtype
  for (auto& [d, dst] : transfers)
    if (rank_of(d) == me) buf[owner[d]].need_main = true;
  for (auto& [d, dst] : transfers)
    if (dst == me) buf[d].need_main = true;
  // a received chunk only refinement folds read (fp32 / fp64, no shadows) can
  // be read where it lies on its producer once the peers are wired
  direct.assign(ne, 0);
  for (auto& [d, dst] : transfers) {
    if (dst != me || buf[d].need_16 || buf[d].need_lo) continue;
    bool ok = true;
    for (int u = 0; u < ne && ok; ++u)
      if (local[u] && std::find(X[u].deps.begin(), X[u].deps.end(), d) != X[u].deps.end())
        ok = X[u].kind == ED_EXEC_REFINEMENT && owner[u] == u && !virt[u];
    direct[d] = ok;
  }
  // every computed chunk keeps at least one representation
  for (int id = 0; id < ne; ++id)
    if (local[id] && !virt[id] && owner[id] == id && !buf[id].need_16) buf[id].need_main = true;

  // ---- allocation plan ----
  size_t off = 0;
  auto take = [&](int64_t elems, size_t esz) {
    size_t o = off;
    off += ((size_t(elems) * esz + 1023) / 1024) * 1024;
    return o;
  };
  for (int id = 0; id < ne; ++id) {
    bool here = (local[id] && owner[id] == id && !virt[id]);
    bool recv = false;
    for (auto& [d, dst] : transfers) recv = recv || (d == id && dst == me);
    if (!here && !recv) continue;
    if (buf[id].need_main) buf[id].off_main = take(X[id].sz, es);
    if (buf[id].need_16) buf[id].off_16 = take(X[id].sz, 2);
    if (buf[id].need_lo) buf[id].off_lo = take(X[id].sz, 4);
  }
  arena_bytes = std::max<size_t>(off, 1024);

  // ---- ops (exec-id order; transfers at their first consumer) ----
  const auto xfer_at = transfers_by_consumer();
  ops.clear();
  contraction_flops = 0;
  std::set<int> gemm_emitted;
  std::set<int> split_done;  // F32X3: chunks whose lo shadow exists (split, or written by their producer)
  for (int id = 0; id < ne; ++id) {
    for (auto& [d, dst] : xfer_at[id]) {
      if (rank_of(d) == me) {
        Op op{OpKind::SEND};
        op.name = "nccl_send";
        op.exec = d;
        op.peer = dst;
        op.ptr = reinterpret_cast<void*>(d);  // resolved after allocation
        op.count = size_t(X[d].sz);
        op.bytes = double(X[d].sz) * es;
        ops.push_back(op);
      } else if (dst == me) {
        Op op{OpKind::RECV};
        op.name = "nccl_recv";
        op.exec = d;
        op.peer = rank_of(d);
        op.ptr = reinterpret_cast<void*>(d);
        op.count = size_t(X[d].sz);
        op.bytes = double(X[d].sz) * es;
        ops.push_back(op);
        if (buf[d].need_16) {  // received operand of a bf16 GEMM
          Op cv{OpKind::CONVERT};
          cv.name = "convert_bf16";
          cv.ptr = reinterpret_cast<void*>(d);
          cv.bytes = double(X[d].sz) * (es + 2);
          ops.push_back(cv);
        }
      }
    }
    const Ex& u = X[id];
    if (!local[id] || u.kind == ED_EXEC_INPUT_CHUNK) continue;
    const Vtx& w = V[u.producer];
    if (u.kind == ED_EXEC_JOIN) {
      if (w.join == ED_JOIN_MUL && w.agg == ED_AGG_SUM) contraction_flops += 2.0 * double(u.fp);
      if (virt[id] || virtual_join_src.count(id)) continue;  // computed inside a fused kernel
      if (first_join < 0) first_join = id;
      if (softmax_.count(u.producer)) {
        if (gemm_emitted.count(u.producer)) continue;
        gemm_emitted.insert(u.producer);
        Op op{OpKind::SOFTMAX};
        op.name = "softmax_rows:" + w.name;
        op.ptr = reinterpret_cast<void*>(id);
        for (auto& [yj, xr] : softmax_[u.producer].pairs) {
          op.heads.push_back(yj);
          if (x3 && x3_lo_by_producer()) split_done.insert(yj);  // the kernel writes Y's lo shadow beside Y
        }
        ops.push_back(op);
        continue;
      }
      if (flash_.count(u.producer)) {
        if (!fused_head[id] || gemm_emitted.count(u.producer)) continue;
        gemm_emitted.insert(u.producer);
        const Flash& f = flash_.at(u.producer);
        if (x3) {
          // lo shadows of operands no producer wrote (receives, element-wise outputs)
          auto split = [&](int o2) {
            if ((X[o2].kind == ED_EXEC_INPUT_CHUNK && local[o2]) || !split_done.insert(o2).second) return;
            Op sp{OpKind::SPLIT};
            sp.name = "split_tf32";
            sp.ptr = reinterpret_cast<void*>(o2);
            sp.bytes = double(X[o2].sz) * 8;
            ops.push_back(sp);
          };
          for (size_t q = 0; q < f.regions.size(); ++q) {
            const auto& r = f.regions[q];
            split(local[r[0]] ? owner[r[0]] : r[0]);
            for (int k = 1; k < 3; ++k) {
              const KVTiles& t = k == 1 ? f.ktiles[q] : f.vtiles[q];
              if (t.tiled)
                for (int o2 : t.owners) split(o2);
              else
                split(local[r[k]] ? owner[r[k]] : r[k]);
            }
            split_done.insert(r[3]);  // the kernel writes O's lo shadow
          }
        }
        Op op{OpKind::FLASH};
        op.name = "attention_fused:" + V[f.t1].name + ".." + w.name;
        op.ptr = reinterpret_cast<void*>(id);
        for (auto& r : f.regions) op.heads.push_back(r[3]);
        for (int h = 0; h < ne; ++h)
          if (X[h].kind == ED_EXEC_JOIN && (X[h].producer == f.t1 || X[h].producer == f.o))
            op.flops += 2.0 * double(X[h].fp);
        ops.push_back(op);
        continue;
      }
      if (gmap.count(u.producer)) {
        if (!fused_head[id] || gemm_emitted.count(u.producer)) continue;
        gemm_emitted.insert(u.producer);
        // F32X3: lo shadows of produced operands are made just before use
        if (x3) {
          for (int h = 0; h < ne; ++h) {
            if (!fused_head[h] || X[h].producer != u.producer) continue;
            for (int sidx : region_sibs[h])
              for (int o0 : gemm_reads(sidx)) {
                const int o = o0;
                // (an input chunk's shadow is made at upload, on the rank that holds it:
                // one received from another rank is split here like any other receive)
                if ((X[o].kind == ED_EXEC_INPUT_CHUNK && local[o]) || !split_done.insert(o).second) continue;
                Op sp{OpKind::SPLIT};
                sp.name = "split_tf32";
                sp.ptr = reinterpret_cast<void*>(o);
                sp.bytes = double(X[o].sz) * 8;
                ops.push_back(sp);
              }
          }
        }
        // one persistent launch for every region of this einsum on this rank
        Op op{OpKind::GEMM};
        op.bf16 = bf16;
        op.einsum = u.producer;
        op.name = std::string(bf16 ? "gemm_bf16:" : "gemm_tf32:") + w.name;
        op.ptr = reinterpret_cast<void*>(id);
        for (int h = 0; h < ne; ++h)
          if (fused_head[h] && X[h].producer == u.producer) {
            op.heads.push_back(h);
            for (int s : region_sibs[h]) op.flops += 2.0 * double(X[s].fp);
            if (x3 && x3_lo_by_producer()) split_done.insert(h);  // the x3 epilogue writes the region's lo shadow
          }
        ops.push_back(op);
      } else if (memmap_.count(u.producer)) {
        if (gemm_emitted.count(u.producer)) continue;
        gemm_emitted.insert(u.producer);
        const MemMap& mm = memmap_.at(u.producer);
        Op op{mm.kind};
        op.name = std::string(mm.kind == OpKind::EWISE ? "ewise:" : "rowreduce:") + w.name;
        op.ptr = reinterpret_cast<void*>(id);
        for (int h = 0; h < ne; ++h)
          if (local[h] && X[h].kind == ED_EXEC_JOIN && X[h].producer == u.producer) {
            op.heads.push_back(h);
            op.flops += double(X[h].fp);
          }
        ops.push_back(op);
      } else {
        Op op{OpKind::GENERIC};
        op.name = "einsum_generic:" + w.name;
        op.ptr = reinterpret_cast<void*>(id);
        op.flops = double(u.fp);
        ops.push_back(op);
      }
      continue;
    }
    // refinement
    if (owner[id] != id || virt[id]) continue;  // aliased or fused away: no work
    Op op{OpKind::REFINE};
    op.name = "refine:" + w.name;
    op.ptr = reinterpret_cast<void*>(id);
    ops.push_back(op);
    if (x3 && x3_lo_by_producer()) split_done.insert(id);  // the fold writes the lo shadow beside the chunk
  }
  if (opt.corrupt && first_join >= 0 && local[first_join]) {
    // after the op that produced the first join
    size_t at = 0;
    for (size_t i = 0; i < ops.size(); ++i)
      if (((ops[i].kind == OpKind::GEMM || ops[i].kind == OpKind::EWISE || ops[i].kind == OpKind::ROWREDUCE ||
            ops[i].kind == OpKind::SOFTMAX || ops[i].kind == OpKind::FLASH) &&
           std::count(ops[i].heads.begin(), ops[i].heads.end(), owner[first_join])) ||
          (ops[i].kind == OpKind::GENERIC && reinterpret_cast<intptr_t>(ops[i].ptr) == owner[first_join])) {
        at = i + 1;
        break;
      }
    Op op{OpKind::CORRUPT};
    op.name = "corrupt_hook";
    op.ptr = reinterpret_cast<void*>(owner[first_join]);
    ops.insert(ops.begin() + at, op);
  }

  (void)0;
  // stash what allocate() needs
  // what each op writes (before allocate() turns some op.ptr ids into pointers)
  for (auto& op : ops) {
    op.writes.clear();
    switch (op.kind) {
      case OpKind::GEMM:
      case OpKind::SOFTMAX:
      case OpKind::FLASH:
      case OpKind::EWISE:
      case OpKind::ROWREDUCE: op.writes = op.heads; break;
      case OpKind::GENERIC:
      case OpKind::REFINE: op.writes.push_back(int(reinterpret_cast<intptr_t>(op.ptr))); break;
      default: break;
    }
  }
  this->srcs_.clear();
  for (int id = 0; id < ne; ++id)
    for (auto& s : srcs[id]) this->srcs_.push_back({id, s.id, s.r0, s.ext});
  this->gmap_ = gmap;
  this->epi_ = epi;
  this->region_sibs_ = region_sibs;
}
