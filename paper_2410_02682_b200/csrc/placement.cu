// GPU-aware re-placement of memory-bound exec vertices (ed_gpu_placement,
// SURVEY 8(f) row 1): host-only local search over placement_t::machine_of
// (placement.cc:132-178) under a device cost model.
#include "runtime.h"

namespace {

// Estimated per-machine busy time of a placement (seconds): each vertex's
// kernel time at the model's rates plus whole-chunk transfers, charged to
// sender and receiver once per (chunk, destination machine) like pull()
// (runtime.cc:157-172). Refinements the executor turns into aliases or
// folds inside a region-fused GEMM (all deps local) cost nothing.
struct SiteModel {
  const ed_plan_h& h;
  const ed_cost_model_c& cm;
  std::vector<char> contraction;  // exec id is a mul/sum join
  std::vector<char> fold_free;    // refinement free when co-located with all deps

  // co-located fusable chains (ed_gpu_placement with fuse_chains): members'
  // memory-bound work disappears into the fused kernel while the whole
  // group sits on one machine (the root and contractions are still charged)
  std::vector<std::vector<int>> groups;
  std::vector<int> group_of;
  std::vector<char> credited;

  SiteModel(const ed_plan_h& h_, const ed_cost_model_c& cm_) : h(h_), cm(cm_) {
    const int ne = int(h.X.size());
    contraction.assign(ne, 0);
    fold_free.assign(ne, 0);
    for (int id = 0; id < ne; ++id) {
      const Ex& u = h.X[id];
      if (u.kind == ED_EXEC_JOIN) {
        const Vtx& w = h.V[u.producer];
        contraction[id] = w.join == ED_JOIN_MUL && w.agg == ED_AGG_SUM;
      }
    }
    for (int id = 0; id < ne; ++id) {
      const Ex& u = h.X[id];
      if (u.kind != ED_EXEC_REFINEMENT || u.deps.empty()) continue;
      bool same = true;
      for (int d : u.deps) same = same && h.X[d].sz == u.sz;
      const bool identity = u.deps.size() == 1 && same;
      bool siblings = same;
      for (int d : u.deps) siblings = siblings && contraction[d] && h.X[d].producer == h.X[u.deps[0]].producer;
      fold_free[id] = identity || siblings;
    }
  }

  double comp(int id, const std::vector<int>& m, const std::vector<char>& together) const {
    const Ex& u = h.X[id];
    const double es = cm.elem_bytes;
    if (u.kind == ED_EXEC_INPUT_CHUNK) return 0.0;
    if (!group_of.empty() && group_of[id] >= 0 && together[size_t(group_of[id])] && credited[id]) return 0.0;
    if (u.kind == ED_EXEC_JOIN) {
      if (contraction[id]) return 2.0 * double(u.fp) / cm.tensor_flops;
      double el = double(u.sz);
      for (int d : u.deps) el += double(h.X[d].sz);
      return el * es / cm.hbm_bytes;
    }
    bool colocated = true;
    for (int d : u.deps) colocated = colocated && m[d] == m[id];
    if (fold_free[id] && colocated) return 0.0;
    double el = double(u.sz);
    for (int d : u.deps) el += double(std::min(h.X[d].sz, u.sz));
    return el * es / cm.hbm_bytes;
  }

  // (busiest machine seconds, total transferred elements)
  std::pair<double, double> eval(const std::vector<int>& m) const {
    std::vector<double> site(size_t(h.n_machines), 0.0);
    std::vector<char> together(groups.size(), 1);
    for (size_t g = 0; g < groups.size(); ++g)
      for (int id : groups[g]) together[g] = together[g] && m[id] == m[groups[g][0]];
    std::set<std::pair<int, int>> pulled;
    double moved = 0.0;
    for (int id = 0; id < int(h.X.size()); ++id) {
      const Ex& u = h.X[id];
      if (u.kind == ED_EXEC_INPUT_CHUNK) continue;
      site[size_t(m[id])] += comp(id, m, together);
      for (int d : u.deps)
        if (m[d] != m[id] && pulled.insert({d, m[id]}).second) {
          const double t = double(h.X[d].sz) * cm.elem_bytes / cm.link_bytes;
          site[size_t(m[id])] += t;
          site[size_t(m[d])] += t;
          moved += double(h.X[d].sz);
        }
    }
    return {*std::max_element(site.begin(), site.end()), moved};
  }
};

// Fusable chains the executor can run as one kernel per region when a
// region's exec vertices share a GPU (build.cu: epilogue map, row
// softmax, attention block). For each root join, the chain's exec vertices it
// reads (backwards through the chain's vertices) form one group; a chain
// whose groups overlap is left alone. Each group is moved onto its root's
// machine (m), registered with the cost model (members' memory-bound work is
// credited while the group stays together) and returned as a movable unit
// unless its root or a member is a contraction the re-placer may not move
// alone (then the group is fixed in place).
void fusable_groups(const ed_plan_h& h, SiteModel& sm, std::vector<int>& m, std::vector<std::vector<int>>& units,
                    std::vector<char>& fixed) {
  const auto& V = h.V;
  const auto& X = h.X;
  const int nv = int(V.size()), ne = int(X.size());
  std::vector<std::vector<int>> readers(static_cast<size_t>(nv));
  for (int w = 0; w < nv; ++w)
    for (int k = 0; k < V[w].arity; ++k) readers[size_t(V[w].inputs[k])].push_back(w);
  auto is_output = [&](int w) { return std::find(h.outputs.begin(), h.outputs.end(), w) != h.outputs.end(); };
  auto contr = [&](int w) { return V[w].arity == 2 && V[w].join == ED_JOIN_MUL && V[w].agg == ED_AGG_SUM; };
  auto reduces = [&](int w) { return V[w].arity == 1 && V[w].lz.size() < V[w].lx.size(); };
  auto sole = [&](int w, int r) { return readers[size_t(w)].size() == 1 && readers[size_t(w)][0] == r && !is_output(w); };
  sm.group_of.assign(size_t(ne), -1);
  sm.credited.assign(size_t(ne), 0);
  std::vector<char> taken(size_t(ne), 0);
  // members: the chain's vertices; credit: those whose work the fused kernel
  // removes; root: the vertex whose joins anchor the groups
  // One group per connected component of root joins and the chain vertices
  // they read (roots sharing a chunk, e.g. a row max split over column
  // blocks, land in one group).
  auto add_chain = [&](const std::set<int>& members, const std::set<int>& credit, int root) {
    std::vector<int> roots;
    for (int r = 0; r < ne; ++r)
      if (X[r].kind == ED_EXEC_JOIN && X[r].producer == root) roots.push_back(r);
    std::vector<int> parent(roots.size());
    for (size_t k = 0; k < roots.size(); ++k) parent[k] = int(k);
    std::function<int(int)> find = [&](int k) { return parent[size_t(k)] == k ? k : parent[size_t(k)] = find(parent[size_t(k)]); };
    std::vector<int> owner_of(static_cast<size_t>(ne), -1);
    for (size_t k = 0; k < roots.size(); ++k) {
      std::vector<int> stack = {roots[k]};
      while (!stack.empty()) {
        const int id = stack.back();
        stack.pop_back();
        for (int d : X[id].deps) {
          if (X[d].kind == ED_EXEC_INPUT_CHUNK || !members.count(X[d].producer)) continue;
          if (owner_of[size_t(d)] >= 0) {
            parent[size_t(find(int(k)))] = find(owner_of[size_t(d)]);
            continue;
          }
          owner_of[size_t(d)] = int(k);
          stack.push_back(d);
        }
      }
    }
    std::map<int, std::vector<int>> comp;
    for (size_t k = 0; k < roots.size(); ++k) comp[find(int(k))].push_back(roots[k]);
    for (int id = 0; id < ne; ++id)
      if (owner_of[size_t(id)] >= 0) comp[find(owner_of[size_t(id)])].push_back(id);
    for (auto& [c, g] : comp)
      for (int id : g)
        if (taken[size_t(id)]) return;  // overlaps another chain
    for (auto& [c, g] : comp) {
      const int gid = int(sm.groups.size());
      bool movable = true;
      for (int id : g) {
        taken[size_t(id)] = 1;
        sm.group_of[size_t(id)] = gid;
        sm.credited[size_t(id)] = credit.count(X[id].producer) && !sm.contraction[size_t(id)];
        m[size_t(id)] = m[size_t(g[0])];
        movable = movable && !sm.contraction[size_t(id)];
      }
      sm.groups.push_back(g);
      if (movable) units.push_back(g);
      else
        for (int id : g) fixed[size_t(id)] = 1;
    }
  };
  for (int y = 0; y < nv; ++y) {
    // row softmax: Y = div(E, Sg), E = exp(S), Sg = sum(E), S = sub(X, M), M = max(X)
    if (V[y].arity != 2 || V[y].join != ED_JOIN_DIV) continue;
    const int e = V[y].inputs[0], sg = V[y].inputs[1];
    if (V[e].arity != 1 || V[e].map != ED_MAP_EXP || reduces(e)) continue;
    if (!reduces(sg) || V[sg].agg != ED_AGG_SUM || V[sg].map != ED_MAP_IDENTITY || V[sg].inputs[0] != e) continue;
    const int sv = V[e].inputs[0];
    if (V[sv].arity != 2 || V[sv].join != ED_JOIN_SUB || !sole(sv, e) || !sole(sg, y)) continue;
    const int xv = V[sv].inputs[0], mx = V[sv].inputs[1];
    if (!reduces(mx) || V[mx].agg != ED_AGG_MAX || V[mx].inputs[0] != xv || !sole(mx, sv)) continue;
    std::set<int> chain = {mx, sv, e, sg};
    // attention block: X = T1 or scale(T1) with T1 = QK^T, O = T3 V the only reader of Y
    if (readers[size_t(y)].size() == 1 && !is_output(y) && contr(readers[size_t(y)][0])) {
      int t1 = xv;
      std::set<int> blk = chain;
      blk.insert(y);
      if (!contr(t1) && V[xv].arity == 1 && !reduces(xv) && contr(V[xv].inputs[0]) && sole(V[xv].inputs[0], xv)) {
        blk.insert(xv);
        t1 = V[xv].inputs[0];
      }
      const bool x_only_chain = readers[size_t(xv)].size() == 2 && !is_output(xv);
      if (contr(t1) && x_only_chain) {
        blk.insert(t1);
        add_chain(blk, blk, readers[size_t(y)][0]);
        continue;
      }
    }
    add_chain(chain, chain, y);
  }
  // map epilogue: V = map(U), U a contraction read only by V: V's joins follow U's
  for (int v = 0; v < nv; ++v) {
    if (V[v].arity != 1 || reduces(v) || V[v].map == ED_MAP_EXP) continue;
    const int u = V[v].inputs[0];
    if (!contr(u) || !sole(u, v)) continue;
    // one group per U join region: V's joins reading it, anchored on U's join
    for (int j = 0; j < ne; ++j) {
      if (X[j].kind != ED_EXEC_JOIN || X[j].producer != v || taken[size_t(j)]) continue;
      std::vector<int> g, stack = {j};
      std::set<int> mach;
      bool ok = true;
      while (!stack.empty() && ok) {
        const int id = stack.back();
        stack.pop_back();
        g.push_back(id);
        for (int d : X[id].deps) {
          if (X[d].kind == ED_EXEC_INPUT_CHUNK || X[d].producer != u) continue;
          if (X[d].kind == ED_EXEC_JOIN) mach.insert(m[size_t(d)]);
          else if (!taken[size_t(d)]) stack.push_back(d);
          else ok = false;
        }
      }
      if (!ok || mach.size() != 1) continue;
      const int gid = int(sm.groups.size());
      for (int id : g) {
        taken[size_t(id)] = 1;
        fixed[size_t(id)] = 1;
        sm.group_of[size_t(id)] = gid;
        m[size_t(id)] = *mach.begin();
      }
      sm.groups.push_back(g);
    }
  }
}

}  // namespace

extern "C" {

ed_status ed_gpu_placement(const ed_plan_c* plan, const ed_cost_model_c* model, int32_t* machine_of, double* est_ms,
                           char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!plan || !model || !machine_of) throw ed_error(ED_ERR_USAGE, "null argument");
    if (!(model->tensor_flops > 0 && model->hbm_bytes > 0 && model->link_bytes > 0 && model->elem_bytes > 0))
      throw ed_error(ED_ERR_USAGE, "cost model rates must be positive");
    ed_ctx c;
    c.world = std::max(1, plan->n_machines);
    ed_plan_h h;
    h.ctx = &c;
    h.copy_plan(plan);
    h.validate();
    const int ne = int(h.X.size());
    std::vector<int> m(static_cast<size_t>(ne));
    for (int id = 0; id < ne; ++id) m[size_t(id)] = h.X[id].machine;
    SiteModel sm(h, *model);
    std::vector<char> fixed(size_t(ne), 0);  // kept where the start placement put it
    std::vector<std::vector<int>> chain_units;
    const std::vector<int> m0 = m;
    if (model->fuse_chains) fusable_groups(h, sm, m, chain_units, fixed);
    const auto start = sm.eval(m0);
    auto better = [](std::pair<double, double> a, std::pair<double, double> b) {
      const double tol = 1e-12 * std::max(1.0, b.first);
      return a.first < b.first - tol || (std::abs(a.first - b.first) <= tol && a.second < b.second);
    };
    const int passes = model->max_passes > 0 ? model->max_passes : 4;
    // local search over units: a unit moves as a whole (a fusable chain and
    // its root, or one memory-bound exec vertex)
    auto search = [&](std::vector<int>& mm, const std::vector<std::vector<int>>& units) {
      auto cur = sm.eval(mm);
      for (int pass = 0; pass < passes; ++pass) {
        bool changed = false;
        for (const auto& un : units) {
          const int home = mm[size_t(un[0])];
          int best = home;
          auto best_c = cur;
          for (int l = 0; l < h.n_machines; ++l) {
            if (l == home) continue;
            for (int id : un) mm[size_t(id)] = l;
            auto cl = sm.eval(mm);
            if (better(cl, best_c)) {
              best_c = cl;
              best = l;
            }
          }
          for (int id : un) mm[size_t(id)] = best;
          if (best != home) {
            cur = best_c;
            changed = true;
          }
        }
        if (!changed) break;
      }
      return cur;
    };
    std::vector<std::vector<int>> singles;
    for (int id = 0; id < ne; ++id)
      if (h.X[id].kind != ED_EXEC_INPUT_CHUNK && !sm.contraction[size_t(id)]) singles.push_back({id});
    // (a) vertex by vertex from the start placement (chains may be split)
    std::vector<int> ma = m0;
    auto ca = search(ma, singles);
    if (!sm.groups.empty()) {
      // (b) chains co-located (fusable_groups moved them onto their roots'
      // machines), then units and the remaining vertices; the better wins
      std::vector<int> mb = m;
      std::vector<std::vector<int>> units = chain_units;
      std::vector<char> in_unit(size_t(ne), 0);
      for (auto& un : chain_units)
        for (int id : un) in_unit[size_t(id)] = 1;
      for (auto& sg : singles)
        if (!in_unit[size_t(sg[0])] && !fixed[size_t(sg[0])]) units.push_back(sg);
      auto cb = search(mb, units);
      if (better(cb, ca)) {
        ma = mb;
        ca = cb;
      }
    }
    for (int id = 0; id < ne; ++id) machine_of[id] = ma[size_t(id)];
    if (est_ms) {
      est_ms[0] = start.first * 1e3;
      est_ms[1] = ca.first * 1e3;
    }
  });
}

}  // extern "C"
