// Reference-side adapter (see execute_gpu.h): flattens exec_graph_t +
// placement_t into ed_plan_c, seeds the input chunks, runs, and rebuilds the
// reference's run_report_t — outputs, machine counters and the transfer audit.
#include "execute_gpu.h"

#include <memory>

namespace {

[[noreturn]] void rethrow(ed_status s, const char* err) {
  // status codes back to the reference's exception classes (setup.h:27-47)
  if (s == ED_ERR_PLAN) throw plan_error_t(err);
  if (s == ED_ERR_EVAL) throw eval_error_t(err);
  throw std::runtime_error(string("libed_gpu: ") + err);
}

#define ED_CALL(expr)                 \
  do {                                \
    ed_status s_ = (expr);            \
    if (s_ != ED_OK) rethrow(s_, err); \
  } while (0)

int join_code(join_op_t op) { return int(op); }
int agg_code(agg_op_t op) { return int(op); }
int map_code(unary_op_t const& op) { return int(op.kind); }

// engine_t::region_key / region_partition (runtime.cc:96-116), host side,
// for the transfer audit below
shape_t region_partition_of(exec_graph_t const& exec, exec_vertex_t const& u) {
  auto const& tg = exec.tg;
  if(u.kind == exec_kind_t::input_chunk) return tg.d[u.producer];
  if(u.kind == exec_kind_t::join_kernel) return tg.out_partition(u.producer);
  if(u.consumer >= 0) return tg.required_input_partition(u.consumer, u.slot);
  return tg.out_partition(u.producer);
}

shape_t region_key_of(exec_graph_t const& exec, exec_vertex_t const& u) {
  if(u.kind != exec_kind_t::join_kernel) return u.key;
  auto const& e = *exec.tg.graph.vertices[u.producer].expr;
  return project(u.key, e.out_labels, e.distinct_labels());
}

// The reference attributes every pulled chunk to join / aggregation /
// repartition traffic (runtime.cc:119-154). Replayed in exec-id order: one
// pull per (chunk, machine), triggered by its first consumer on that machine.
transfer_audit_t audit_of(exec_graph_t const& exec, placement_t const& placement) {
  transfer_audit_t audit;
  set<pair<int, int>> pulled;
  map<pair<tuple<int, int, int>, shape_t>, int> gatherer;
  auto const& tg = exec.tg;
  for(auto const& v: exec.vertices) {
    if(v.kind == exec_kind_t::input_chunk) continue;
    int m = placement.machine_of[v.id];
    for(int dep: v.deps) {
      auto const& u = exec.vertices[dep];
      if(placement.machine_of[dep] == m || !pulled.insert({dep, m}).second) continue;
      if(v.kind == exec_kind_t::join_kernel) {
        audit.join_in[v.owner] += u.sz;
        continue;
      }
      int w = v.producer;
      if(tg.graph.is_input(w)) {
        audit.repart_in[{w, v.consumer, v.slot}] += u.sz;
        continue;
      }
      shape_t dz = tg.out_partition(w);
      shape_t dc = v.consumer >= 0 ? tg.required_input_partition(v.consumer, v.slot) : dz;
      if(dc == dz) {
        audit.agg_in[w] += u.sz;
        continue;
      }
      tuple<int, int, int> edge{w, v.consumer, v.slot};
      auto [it, fresh] = gatherer.insert({{edge, region_key_of(exec, u)}, v.id});
      if(fresh || it->second != v.id) audit.repart_in[edge] += u.sz;
      else audit.agg_in[w] += u.sz;
    }
  }
  return audit;
}

}  // namespace

run_report_t execute_gpu(
  exec_graph_t const& exec,
  placement_t const& placement,
  map<int, tensor_relation_t> const& inputs,
  exec_options_t const& options,
  gpu_options_t const& gpu)
{
  char err[2048] = {0};
  auto const& tg = exec.tg;
  auto const& graph = tg.graph;
  if(placement.machine_of.size() != exec.vertices.size()) {
    throw plan_error_t("execute: placement does not cover the exec graph");
  }

  // ---- flatten the plan (labels interned per graph) ----
  map<string, int> label_id;
  auto intern = [&](labels_t const& ls) {
    vector<int32_t> r;
    for(auto const& l: ls) r.push_back(label_id.emplace(l, int(label_id.size())).first->second);
    return r;
  };
  size_t nv = graph.vertices.size();
  vector<ed_vertex_c> V(nv);
  vector<vector<int32_t>> lz(nv), lx(nv), ly(nv);
  for(size_t i = 0; i != nv; ++i) {
    auto const& gv = graph.vertices[i];
    ed_vertex_c& c = V[i];
    c.name = gv.name.c_str();
    c.rank = int32_t(gv.bound.size());
    c.bound = gv.bound.data();
    c.rank_d = int32_t(tg.d[i].size());
    c.d = tg.d[i].data();
    c.inputs[0] = gv.inputs.size() > 0 ? gv.inputs[0] : -1;
    c.inputs[1] = gv.inputs.size() > 1 ? gv.inputs[1] : -1;
    c.join_op = c.map_op = c.agg_op = -1;
    if(!gv.expr) {
      c.arity = 0;
      continue;
    }
    auto const& e = *gv.expr;
    c.arity = int32_t(e.in_labels.size());
    if(e.join) c.join_op = join_code(*e.join);
    if(e.map) {
      c.map_op = map_code(*e.map);
      c.scale_c = e.map->scale_c;
    }
    if(e.agg) c.agg_op = agg_code(*e.agg);
    lz[i] = intern(e.out_labels);
    lx[i] = intern(e.in_labels[0]);
    if(e.is_binary()) ly[i] = intern(e.in_labels[1]);
    c.rank_z = int32_t(lz[i].size());
    c.lz = lz[i].data();
    c.rank_x = int32_t(lx[i].size());
    c.lx = lx[i].data();
    c.rank_y = int32_t(ly[i].size());
    c.ly = ly[i].data();
  }
  vector<ed_exec_vertex_c> X(exec.vertices.size());
  for(auto const& v: exec.vertices) {
    ed_exec_vertex_c& c = X[v.id];
    c.kind = int32_t(v.kind);
    c.owner = v.owner;
    c.producer = v.producer;
    c.consumer = v.consumer;
    c.slot = v.slot;
    c.key_rank = int32_t(v.key.size());
    c.key = v.key.data();
    c.chunk_rank = int32_t(v.chunk_bound.size());
    c.chunk_bound = v.chunk_bound.data();
    c.fp = v.fp;
    c.sz = v.sz;
    c.n_deps = int32_t(v.deps.size());
    c.deps = v.deps.data();
    c.machine = placement.machine_of[v.id];
  }
  ed_plan_c plan{int32_t(nv), V.data(), int32_t(X.size()), X.data(), int32_t(graph.outputs.size()),
                 graph.outputs.data(), int32_t(placement.n_machines), placement.alpha};

  ed_options_c opt{};
  opt.precision = gpu.precision >= 0 ? gpu.precision : (options.f32 ? ED_PREC_FP32 : ED_PREC_FP64);
  opt.corrupt = options.corrupt ? 1 : 0;
  opt.sched_mode = options.mode == sched_mode_t::threaded ? ED_SCHED_THREADED : ED_SCHED_ROUND_ROBIN;

  ed_ctx* ctx = nullptr;
  if(gpu.devices.empty()) {
    ED_CALL(ed_ctx_create(gpu.device, 0, 1, nullptr, 0, &ctx, err, sizeof err));
  } else {
    ED_CALL(ed_ctx_create_multi(int32_t(gpu.devices.size()), gpu.devices.data(), &ctx, err, sizeof err));
  }
  std::unique_ptr<ed_ctx, void (*)(ed_ctx*)> ctx_guard(ctx, ed_ctx_destroy);
  ed_plan_h* h = nullptr;
  ED_CALL(ed_prepare(ctx, &plan, &opt, &h, err, sizeof err));
  std::unique_ptr<ed_plan_h, void (*)(ed_plan_h*)> plan_guard(h, ed_plan_destroy);

  // ---- seed the input chunks (engine_t ctor, runtime.cc:66-84) ----
  vector<ed_chunk_in_c> chunks;
  for(auto const& [vid, ids]: exec.input_chunks_of) {
    auto it = inputs.find(vid);
    if(it == inputs.end()) {
      throw plan_error_t("execute: no relation supplied for input '" + graph.vertices[vid].name + "'");
    }
    if(it->second.part != tg.d[vid] || it->second.bound != graph.vertices[vid].bound) {
      throw plan_error_t("execute: relation for '" + graph.vertices[vid].name + "' is not chunked as planned");
    }
    for(int cid: ids) {
      auto const& t = it->second.chunks.at(exec.vertices[cid].key);
      chunks.push_back({cid, ED_DTYPE_F64, t.values.data(), t.nelem()});
    }
  }
  ED_CALL(ed_upload(h, chunks.data(), int32_t(chunks.size()), err, sizeof err));

  // ---- run ----
  run_report_t report;
  vector<ed_machine_c> mc(placement.n_machines);
  ed_report_c rep{};
  rep.n_machines = int32_t(mc.size());
  rep.machines = mc.data();
  ED_CALL(ed_run(h, &rep, err, sizeof err));

  // ---- outputs (runtime.cc:432-448) and counters ----
  vector<tensor_t> outs;
  vector<ed_output_c> od;
  for(int o: graph.outputs) outs.push_back(tensor_t::zeros(graph.vertices[o].bound));
  for(size_t i = 0; i != outs.size(); ++i) {
    od.push_back({graph.outputs[i], ED_DTYPE_F64, outs[i].values.data(), outs[i].nelem()});
  }
  ED_CALL(ed_download(h, od.data(), int32_t(od.size()), err, sizeof err));
  for(size_t i = 0; i != outs.size(); ++i) report.outputs.insert({graph.outputs[i], std::move(outs[i])});
  report.machines.resize(mc.size());
  for(size_t m = 0; m != mc.size(); ++m) report.machines[m] = {mc[m].fp, mc[m].sent, mc[m].received};
  report.total_transferred = rep.total_transferred;
  report.wall_steps = rep.wall_steps;
  report.max_site_cost = rep.max_site_cost;
  report.audit = audit_of(exec, placement);
  return report;
}
