// The plan as the executor holds it: deep copy of ed_plan_c, execute()'s
// structural checks (runtime.cc:388-395), the refinement invariants compute()
// enforces per element (runtime.cc:230-268), the whole-chunk transfer
// accounting of pull() (runtime.cc:119-172), and a rank's logical schedule.
#include "runtime.h"

void ed_plan_h::copy_plan(const ed_plan_c* p) {
  if (!p || p->n_vertices <= 0 || !p->vertices || p->n_exec < 0 || (p->n_exec && !p->exec))
    throw ed_error(ED_ERR_USAGE, "ed_prepare: empty or null plan");
  V.resize(p->n_vertices);
  for (int i = 0; i < p->n_vertices; ++i) {
    const ed_vertex_c& s = p->vertices[i];
    Vtx& v = V[i];
    v.name = s.name ? s.name : ("v" + std::to_string(i));
    v.arity = s.arity;
    v.join = s.join_op;
    v.map = s.map_op;
    v.agg = s.agg_op;
    v.c = s.scale_c;
    v.bound.assign(s.bound, s.bound + s.rank);
    v.d.assign(s.d, s.d + s.rank_d);
    v.lz.assign(s.lz, s.lz + s.rank_z);
    v.lx.assign(s.lx, s.lx + s.rank_x);
    if (s.arity == 2) v.ly.assign(s.ly, s.ly + s.rank_y);
    v.inputs[0] = s.inputs[0];
    v.inputs[1] = s.inputs[1];
    v.lxy = v.lx;
    v.lxy.insert(v.lxy.end(), v.ly.begin(), v.ly.end());
    v.dls = v.lx;
    for (auto l : v.ly)
      if (std::find(v.dls.begin(), v.dls.end(), l) == v.dls.end()) v.dls.push_back(l);
  }
  X.resize(p->n_exec);
  for (int i = 0; i < p->n_exec; ++i) {
    const ed_exec_vertex_c& s = p->exec[i];
    Ex& x = X[i];
    x.kind = s.kind;
    x.owner = s.owner;
    x.producer = s.producer;
    x.consumer = s.consumer;
    x.slot = s.slot;
    x.machine = s.machine;
    x.key.assign(s.key, s.key + s.key_rank);
    x.cb.assign(s.chunk_bound, s.chunk_bound + s.chunk_rank);
    x.fp = s.fp;
    x.sz = s.sz;
    x.deps.assign(s.deps, s.deps + s.n_deps);
  }
  outputs.assign(p->outputs, p->outputs + p->n_outputs);
  n_machines = p->n_machines;
  alpha = p->alpha;
}

// execute()'s structural checks (runtime.cc:388-395) plus the refinement
// invariants compute() enforces per element (runtime.cc:230-268), which are
// data-independent and therefore checked once here.
void ed_plan_h::validate() {
  const int nv = int(V.size()), ne = int(X.size());
  if (n_machines < 1) throw ed_error(ED_ERR_PLAN, "execute: placement does not cover the exec graph");
  for (int w = 0; w < nv; ++w) {
    const Vtx& v = V[w];
    if (v.arity < 0 || v.arity > 2) throw ed_error(ED_ERR_PLAN, "bad arity for '" + v.name + "'");
    if (int(v.bound.size()) > kMaxRank) throw ed_error(ED_ERR_UNSUPPORTED, "rank > 8 for '" + v.name + "'");
    if (v.arity == 0) {
      if (v.d.size() != v.bound.size()) throw ed_error(ED_ERR_PLAN, "explode: vertex '" + v.name + "' is not labeled");
      continue;
    }
    if (v.d.size() != v.lxy.size()) throw ed_error(ED_ERR_PLAN, "partition vector rank mismatch for '" + v.name + "'");
    if (int(v.dls.size()) > kMaxRank) throw ed_error(ED_ERR_UNSUPPORTED, "more than 8 distinct labels");
    shape bxy;
    for (int s = 0; s < v.arity; ++s) {
      int in = v.inputs[s];
      if (in < 0 || in >= nv) throw ed_error(ED_ERR_PLAN, "graph: out-of-range input");
      bxy.insert(bxy.end(), V[in].bound.begin(), V[in].bound.end());
    }
    if (bxy.size() != v.lxy.size()) throw ed_error(ED_ERR_PLAN, "graph: ranks disagree with labels");
    for (size_t i = 0; i < bxy.size(); ++i) {
      if (v.d[i] < 1 || bxy[i] % v.d[i] != 0)
        throw ed_error(ED_ERR_PLAN, "partition entry does not divide bound");
      // shared labels must agree in extent and partition (first occurrence wins, indexing.cc:30-41)
      auto pos = positions({v.lxy[i]}, v.lxy)[0];
      if (bxy[pos] != bxy[i] || v.d[pos] != v.d[i]) throw ed_error(ED_ERR_PLAN, "inconsistent shared label");
    }
  }
  for (int id = 0; id < ne; ++id) {
    const Ex& u = X[id];
    if (u.machine < 0 || u.machine >= n_machines) throw ed_error(ED_ERR_PLAN, "execute: incomplete placement");
    if (u.producer < 0 || u.producer >= nv) throw ed_error(ED_ERR_PLAN, "exec vertex producer out of range");
    for (int d : u.deps)
      if (d < 0 || d >= id) throw ed_error(ED_ERR_PLAN, "exec graph is not in topological id order");
    if (prod(u.cb) != u.sz) throw ed_error(ED_ERR_PLAN, "exec vertex size mismatch");
    if (u.kind == ED_EXEC_JOIN) {
      if (int(u.deps.size()) != V[u.producer].arity) throw ed_error(ED_ERR_PLAN, "join arity mismatch");
    } else if (u.kind == ED_EXEC_REFINEMENT) {
      if (u.deps.size() > size_t(kMaxDeps)) throw ed_error(ED_ERR_UNSUPPORTED, "refinement with > 64 deps");
      // coverage: deps of one refinement share the producer's region partition,
      // so distinct region keys are disjoint and repeats are aggregation siblings
      const shape& bound = V[u.producer].bound;
      shape dc = region_partition(id);
      std::set<shape> seen;
      bool repeat = false;
      int64_t covered = 0;
      for (int d : u.deps) {
        shape rk = region_key(d), dr = region_partition(d);
        if (!seen.insert(rk).second) {
          repeat = true;
          continue;
        }
        int64_t vol = 1;
        for (size_t i = 0; i < bound.size(); ++i) {
          int64_t r0 = rk[i] * (bound[i] / dr[i]), r1 = r0 + bound[i] / dr[i];
          int64_t c0 = u.key[i] * (bound[i] / dc[i]), c1 = c0 + u.cb[i];
          vol *= std::max<int64_t>(0, std::min(r1, c1) - std::max(r0, c0));
        }
        covered += vol;
      }
      int agg = V[u.producer].arity == 0 ? -1 : V[u.producer].agg;
      if (repeat && agg < 0)
        throw ed_error(ED_ERR_PLAN, "execute: overlapping contributions without an aggregation op");
      if (covered != u.sz) throw ed_error(ED_ERR_PLAN, "execute: refinement chunk left partially unwritten");
    }
  }
  for (int o : outputs)
    if (o < 0 || o >= nv) throw ed_error(ED_ERR_PLAN, "output out of range");

  // transfer accounting: one whole-chunk pull per (chunk, machine)
  // (pull / pull_available, runtime.cc:119-172) — a pure function of the plan
  counters.assign(n_machines, ed_machine_c{0, 0, 0});
  std::set<std::pair<int, int>> pulled;
  total_transferred = 0;
  for (int id = 0; id < ne; ++id) {
    const Ex& v = X[id];
    if (v.kind == ED_EXEC_INPUT_CHUNK) continue;
    counters[v.machine].fp += v.fp;
    for (int d : v.deps)
      if (X[d].machine != v.machine && pulled.insert({d, v.machine}).second) {
        counters[X[d].machine].sent += X[d].sz;
        counters[v.machine].received += X[d].sz;
        total_transferred += X[d].sz;
      }
  }
  max_site_cost = 0;
  for (auto& c : counters)
    max_site_cost = std::max(max_site_cost, alpha * double(c.fp) + double(c.sent) + double(c.received));

  // run_round_robin's rounds (runtime.cc:281-298): each round, machine m in
  // order pulls every produced dependency of its waiting vertices, then runs
  // its first ready vertex. Data-independent, so replayed here once.
  std::vector<std::vector<int>> mine(static_cast<size_t>(n_machines));
  std::vector<char> done(size_t(ne), 0);
  std::vector<std::set<int>> resident(static_cast<size_t>(n_machines));
  int left = 0;
  for (int id = 0; id < ne; ++id) {
    if (X[id].kind == ED_EXEC_INPUT_CHUNK) {
      done[size_t(id)] = 1;
      resident[size_t(X[id].machine)].insert(id);
    } else {
      mine[size_t(X[id].machine)].push_back(id);
      ++left;
    }
  }
  std::vector<size_t> first_open(static_cast<size_t>(n_machines), 0);  // mine[m] before this index are done
  rr_rounds = 0;
  while (left > 0) {
    bool progressed = false;
    for (int m = 0; m < n_machines; ++m) {
      auto& mm = mine[size_t(m)];
      auto& res = resident[size_t(m)];
      while (first_open[size_t(m)] < mm.size() && done[size_t(mm[first_open[size_t(m)]])]) ++first_open[size_t(m)];
      for (size_t k = first_open[size_t(m)]; k < mm.size(); ++k)
        if (!done[size_t(mm[k])])
          for (int d : X[mm[k]].deps)
            if (done[size_t(d)]) res.insert(d);
      for (size_t k = first_open[size_t(m)]; k < mm.size(); ++k) {
        const int id = mm[k];
        if (done[size_t(id)]) continue;
        bool ready = true;
        for (int d : X[id].deps) ready = ready && res.count(d);
        if (!ready) continue;
        done[size_t(id)] = 1;
        res.insert(id);
        --left;
        progressed = true;
        break;  // one vertex per machine per round
      }
    }
    ++rr_rounds;
    if (!progressed) throw ed_error(ED_ERR_PLAN, "execute: no runnable vertex; graph is inconsistent");
  }
}

extern "C" {

ed_status ed_plan_schedule(const ed_plan_c* plan, int32_t rank, int32_t world, ed_sched_op_c* out, int32_t cap,
                           int32_t* n_out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!n_out || world < 1 || rank < 0 || rank >= world) throw ed_error(ED_ERR_USAGE, "bad rank/world");
    ed_ctx c;
    c.rank = rank;
    c.world = world;
    ed_plan_h h;
    h.ctx = &c;
    h.copy_plan(plan);
    h.validate();
    const auto at = h.transfers_by_consumer();
    std::vector<ed_sched_op_c> ops;
    for (int id = 0; id < int(h.X.size()); ++id) {
      for (auto& [d, dst] : at[id]) {
        if (h.rank_of(d) == rank) ops.push_back({ED_SCHED_SEND, d, dst, h.X[d].sz});
        else if (dst == rank) ops.push_back({ED_SCHED_RECV, d, h.rank_of(d), h.X[d].sz});
      }
      if (h.X[id].kind != ED_EXEC_INPUT_CHUNK && h.rank_of(id) == rank) ops.push_back({ED_SCHED_COMPUTE, id, -1, 0});
    }
    for (int i = 0; i < std::min<int>(cap, int(ops.size())); ++i) out[i] = ops[i];
    *n_out = int(ops.size());
  });
}

}  // extern "C"
