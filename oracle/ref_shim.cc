// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A thin C ABI over the UNMODIFIED reference sources (compiled in place from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libedref.so).
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg call it through ctypes to
//   * emit plans from the reference planner   (build_pipeline, runtime.cc:511-516)
//   * generate the reference's inputs         (generate_inputs, runtime.cc:552-571)
//   * run the reference CPU executor          (execute, runtime.cc:382-451)
//   * run the dense oracle                    (eval_reference, reference.cc:62-82)
// Plans are written as "edplan/1" JSON, a superset of the reference's
// execgraph/1 (json_io.cc:131-155) carrying everything execute() reads.
#include <chrono>
#include <cstdlib>
#include <cstring>

#include "eindecomp/json_io.h"
#include "eindecomp/parse.h"

namespace {

void set_err(char* err, size_t errlen, std::string const& msg) {
  if(err && errlen) {
    std::snprintf(err, errlen, "%s", msg.c_str());
  }
}

// Exception classes map onto the product's ed_status codes (include/ed_gpu.h).
template <typename F>
int guarded(char* err, size_t errlen, F&& f) {
  try {
    f();
    return 0;
  } catch(parse_error_t const& e) {
    set_err(err, errlen, e.what());
    return 2;
  } catch(plan_error_t const& e) {
    set_err(err, errlen, e.what());
    return 2;
  } catch(eval_error_t const& e) {
    set_err(err, errlen, e.what());
    return 4;
  } catch(std::exception const& e) {
    set_err(err, errlen, e.what());
    return 1;
  }
}

// Task graph: either the reference optimizer's plan or pinned d vectors
// (the test_runtime.cc:32-36 pattern: inputs take the partition their
// first consumer requires).
task_graph_t make_task_graph(eingraph_t const& g, int64_t p, const char* pinned_json) {
  if(pinned_json == nullptr || pinned_json[0] == 0) {
    return optimize_dag(g, p);
  }
  auto j = nlohmann::json::parse(pinned_json);
  task_graph_t tg { g, vector<shape_t>(g.vertices.size()), {}, 0 };
  tg.p_used.assign(g.vertices.size(), 0);
  for(size_t vid = 0; vid != g.vertices.size(); ++vid) {
    if(g.is_input(int(vid))) {
      continue;
    }
    auto const& name = g.vertices[vid].name;
    if(!j.contains(name)) {
      throw plan_error_t("pinned plan: no d for '" + name + "'");
    }
    tg.d[vid] = j.at(name).get<shape_t>();
  }
  vector<char> labeled(g.vertices.size(), 0);
  for(size_t vid = 0; vid != g.vertices.size(); ++vid) {
    if(g.is_input(int(vid))) {
      continue;
    }
    auto const& v = g.vertices[vid];
    for(size_t s = 0; s != v.inputs.size(); ++s) {
      int inn = v.inputs[s];
      if(g.is_input(inn) && !labeled[inn]) {
        tg.d[inn] = tg.required_input_partition(int(vid), int(s));
        labeled[inn] = 1;
      }
    }
  }
  for(size_t vid = 0; vid != g.vertices.size(); ++vid) {
    if(g.is_input(int(vid)) && !labeled[vid]) {
      tg.d[vid] = shape_t(g.vertices[vid].bound.size(), 1);
    }
  }
  return tg;
}

pipeline_t make_pipeline(eingraph_t const& g, int64_t p, int64_t L, double alpha, const char* pinned) {
  pipeline_t ret { g, make_task_graph(g, p, pinned), {}, {} };
  ret.exec = explode(ret.tg);
  ret.placement = place_all(ret.exec, L, alpha);
  return ret;
}

nlohmann::ordered_json expr_json(einsum_expr_t const& e) {
  nlohmann::ordered_json j;
  j["out"] = e.out_labels;
  j["in"] = e.in_labels;
  j["join"] = e.join ? nlohmann::ordered_json(join_op_name(*e.join)) : nlohmann::ordered_json(nullptr);
  if(e.map) {
    string name = unary_op_name(*e.map);
    j["map"] = name.rfind("scale(", 0) == 0 ? string("scale") : name;
    j["scale_c"] = e.map->scale_c;
  } else {
    j["map"] = nullptr;
    j["scale_c"] = 0.0;
  }
  j["agg"] = e.agg ? nlohmann::ordered_json(agg_op_name(*e.agg)) : nlohmann::ordered_json(nullptr);
  return j;
}

string plan_json(pipeline_t const& pipe, int64_t p) {
  auto const& g = pipe.graph;
  nlohmann::ordered_json j;
  j["schema"] = "edplan/1";
  j["p"] = p;
  j["n_machines"] = pipe.placement.n_machines;
  j["alpha"] = pipe.placement.alpha;
  nlohmann::ordered_json verts = nlohmann::ordered_json::array();
  for(size_t vid = 0; vid != g.vertices.size(); ++vid) {
    auto const& v = g.vertices[vid];
    nlohmann::ordered_json jv;
    jv["name"] = v.name;
    jv["bound"] = v.bound;
    jv["inputs"] = v.inputs;
    jv["expr"] = v.expr ? expr_json(*v.expr) : nlohmann::ordered_json(nullptr);
    jv["d"] = pipe.tg.d[vid];
    jv["out_partition"] = pipe.tg.out_partition(int(vid));
    verts.push_back(std::move(jv));
  }
  j["vertices"] = std::move(verts);
  j["outputs"] = g.outputs;
  j["objective"] = pipe.tg.objective;
  nlohmann::ordered_json ev = nlohmann::ordered_json::array();
  for(auto const& v: pipe.exec.vertices) {
    nlohmann::ordered_json jv;
    jv["id"] = v.id;
    jv["kind"] = int(v.kind);
    jv["owner"] = v.owner;
    jv["producer"] = v.producer;
    jv["consumer"] = v.consumer;
    jv["slot"] = v.slot;
    jv["key"] = v.key;
    jv["chunk_bound"] = v.chunk_bound;
    jv["fp"] = v.fp;
    jv["sz"] = v.sz;
    jv["deps"] = v.deps;
    jv["machine"] = pipe.placement.machine_of[v.id];
    ev.push_back(std::move(jv));
  }
  j["exec"] = std::move(ev);
  auto idx = [](map<int, vector<int>> const& m) {
    nlohmann::ordered_json r = nlohmann::ordered_json::object();
    for(auto const& [k, v]: m) {
      r[std::to_string(k)] = v;
    }
    return r;
  };
  j["input_chunks_of"] = idx(pipe.exec.input_chunks_of);
  j["joins_of"] = idx(pipe.exec.joins_of);
  j["refinements_of"] = idx(pipe.exec.refinements_of);
  j["input_refines_of"] = idx(pipe.exec.input_refines_of);
  j["output_refines_of"] = idx(pipe.exec.output_refines_of);
  return j.dump();
}

char* dup_string(string const& s) {
  char* r = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(r, s.data(), s.size() + 1);
  return r;
}

map<int, tensor_t> wrap_inputs(eingraph_t const& g, const double* const* inputs) {
  map<int, tensor_t> ret;
  for(size_t vid = 0; vid != g.vertices.size(); ++vid) {
    if(!g.is_input(int(vid))) {
      continue;
    }
    tensor_t t = tensor_t::zeros(g.vertices[vid].bound);
    std::memcpy(t.values.data(), inputs[vid], sizeof(double) * t.values.size());
    ret.insert({ int(vid), std::move(t) });
  }
  return ret;
}

} // namespace

extern "C" {

void edref_free(void* p) { std::free(p); }

int edref_plan(const char* graph_text, int64_t p, int64_t n_machines, double alpha,
               const char* pinned_json, char** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto g = parse_eingraph(graph_text);
    auto pipe = make_pipeline(g, p, n_machines, alpha, pinned_json);
    *out = dup_string(plan_json(pipe, p));
  });
}

// The reference's own on-disk artifacts for a plan: taskgraph/1
// (json_io.cc:63-103, what `eindecomp optimize --out` writes) and execgraph/1
// with machines (json_io.cc:131-155, what `eindecomp place --out` writes).
int edref_artifacts(const char* graph_text, int64_t p, int64_t n_machines, double alpha,
                    const char* pinned_json, char** taskgraph, char** execgraph, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto g = parse_eingraph(graph_text);
    auto pipe = make_pipeline(g, p, n_machines, alpha, pinned_json);
    *taskgraph = dup_string(taskgraph_to_json(pipe.tg).dump());
    *execgraph = dup_string(execgraph_to_json(pipe.exec, &pipe.placement).dump());
  });
}

// Element count of graph vertex vid (so callers can size buffers).
int64_t edref_vertex_numel(const char* graph_text, int vid) {
  try {
    auto g = parse_eingraph(graph_text);
    return product(g.vertices.at(vid).bound);
  } catch(...) {
    return -1;
  }
}

int edref_generate_input(const char* graph_text, uint64_t seed, int vid,
                         double* out, int64_t n, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto g = parse_eingraph(graph_text);
    if(!g.is_input(vid)) {
      throw plan_error_t("not an input vertex");
    }
    // generate_inputs (runtime.cc:552-571) seeds each input vertex's stream
    // with mt19937_64(seed*7919+vid); the integer/real choice looks only at
    // the expressions. Shrinking the OTHER inputs to all-ones bounds keeps
    // this vertex's draw identical while skipping their (possibly GiB) draws.
    eingraph_t one = g;
    for(size_t u = 0; u != one.vertices.size(); ++u) {
      if(int(u) != vid && one.is_input(int(u))) {
        one.vertices[u].bound.assign(one.vertices[u].bound.size(), 1);
      }
    }
    auto all = generate_inputs(one, seed);
    auto const& t = all.at(vid);
    if(int64_t(t.values.size()) != n) {
      throw plan_error_t("size mismatch");
    }
    std::memcpy(out, t.values.data(), sizeof(double) * size_t(n));
  });
}

// Reference run_end_to_end flow (runtime.cc:518-550) with execute() timed
// alone. inputs: one full row-major tensor per graph vertex (nullptr for
// expression vertices). outputs: one buffer per graph output, in
// graph.outputs order. counters: 3 per machine (fp, sent, received).
// machine_of (nullable, one entry per exec vertex) overrides the planner's
// placement_t::machine_of — e.g. a GPU-aware re-placement under test.
int edref_execute_placed(const char* graph_text, int64_t p, int64_t n_machines, double alpha,
                         const char* pinned_json, const double* const* inputs,
                         int threaded, int f32, int corrupt, const int32_t* machine_of, int32_t n_machine_of,
                         double* const* outputs, double* exec_seconds,
                         int64_t* counters, int64_t* total_transferred,
                         char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto g = parse_eingraph(graph_text);
    auto pipe = make_pipeline(g, p, n_machines, alpha, pinned_json);
    if(machine_of) {
      if(size_t(n_machine_of) != pipe.placement.machine_of.size()) {
        throw std::runtime_error("machine_of size differs from the exec graph");
      }
      for(size_t i = 0; i != pipe.placement.machine_of.size(); ++i) {
        pipe.placement.machine_of[i] = machine_of[i];
      }
    }
    auto ins = wrap_inputs(g, inputs);
    map<int, tensor_relation_t> chunked;
    for(auto const& [vid, t]: ins) {
      chunked.insert({ vid, chunk(t, pipe.tg.d[vid]) });
    }
    exec_options_t opt;
    opt.mode = threaded ? sched_mode_t::threaded : sched_mode_t::round_robin;
    opt.f32 = f32 != 0;
    opt.corrupt = corrupt != 0;
    auto t0 = std::chrono::steady_clock::now();
    auto report = execute(pipe.exec, pipe.placement, chunked, opt);
    auto t1 = std::chrono::steady_clock::now();
    if(exec_seconds) {
      *exec_seconds = std::chrono::duration<double>(t1 - t0).count();
    }
    for(size_t i = 0; i != g.outputs.size(); ++i) {
      auto const& t = report.outputs.at(g.outputs[i]);
      if(outputs && outputs[i]) {
        std::memcpy(outputs[i], t.values.data(), sizeof(double) * t.values.size());
      }
    }
    if(counters) {
      for(size_t m = 0; m != report.machines.size(); ++m) {
        counters[3 * m + 0] = report.machines[m].fp;
        counters[3 * m + 1] = report.machines[m].sent;
        counters[3 * m + 2] = report.machines[m].received;
      }
    }
    if(total_transferred) {
      *total_transferred = report.total_transferred;
    }
  });
}

int edref_execute(const char* graph_text, int64_t p, int64_t n_machines, double alpha,
                  const char* pinned_json, const double* const* inputs,
                  int threaded, int f32, int corrupt,
                  double* const* outputs, double* exec_seconds,
                  int64_t* counters, int64_t* total_transferred,
                  char* err, size_t errlen) {
  return edref_execute_placed(graph_text, p, n_machines, alpha, pinned_json, inputs, threaded, f32, corrupt,
                              nullptr, 0, outputs, exec_seconds, counters, total_transferred, err, errlen);
}

// Dense oracle over the whole graph: outs has one buffer per graph vertex
// (nullptr to skip).
int edref_eval_reference(const char* graph_text, const double* const* inputs,
                         double* const* outs, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto g = parse_eingraph(graph_text);
    auto res = eval_reference(g, wrap_inputs(g, inputs));
    for(auto const& [vid, t]: res) {
      if(outs[vid]) {
        std::memcpy(outs[vid], t.values.data(), sizeof(double) * t.values.size());
      }
    }
  });
}

// One expression vertex, given its (full) input tensors: eval_expr
// (reference.cc:3-60). Used for per-vertex parity.
int edref_eval_vertex(const char* graph_text, int vid, const double* x, const double* y,
                      double* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto g = parse_eingraph(graph_text);
    auto const& v = g.vertices.at(vid);
    if(!v.expr) {
      throw plan_error_t("not an expression vertex");
    }
    tensor_t tx = tensor_t::zeros(g.vertices[v.inputs[0]].bound);
    std::memcpy(tx.values.data(), x, sizeof(double) * tx.values.size());
    tensor_t ty;
    if(v.inputs.size() == 2) {
      ty = tensor_t::zeros(g.vertices[v.inputs[1]].bound);
      std::memcpy(ty.values.data(), y, sizeof(double) * ty.values.size());
    }
    auto r = eval_expr(*v.expr, tx, v.inputs.size() == 2 ? &ty : nullptr, v.name);
    std::memcpy(out, r.values.data(), sizeof(double) * r.values.size());
  });
}

// One expression vertex through the reference's own kernel_eval (kernel.cc:15-68)
// as a single unpartitioned chunk, in f64 (f32 = 0) or the reference's f32
// mode (f32 = 1: every operand and result rounded through float, folds in
// odometer order) — the reference's f32 arithmetic on a vertex slice.
int edref_kernel_vertex(const char* graph_text, int vid, int f32, const double* x, const double* y,
                        double* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto g = parse_eingraph(graph_text);
    auto const& v = g.vertices.at(vid);
    if(!v.expr) {
      throw plan_error_t("not an expression vertex");
    }
    kernel_spec_t spec{*v.expr, g.bxy(vid)};
    tensor_t tx = tensor_t::zeros(spec.in_bound(0));
    std::memcpy(tx.values.data(), x, sizeof(double) * tx.values.size());
    tensor_t ty;
    if(v.expr->is_binary()) {
      ty = tensor_t::zeros(spec.in_bound(1));
      std::memcpy(ty.values.data(), y, sizeof(double) * ty.values.size());
    }
    auto r = kernel_eval(spec, tx, v.expr->is_binary() ? &ty : nullptr, f32 != 0);
    std::memcpy(out, r.values.data(), sizeof(double) * r.values.size());
  });
}

} // extern "C"
