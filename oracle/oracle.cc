// TEST INFRASTRUCTURE ONLY — see oracle.h. A CPU restatement of the
// reference executor, written against ed_plan_c. Never part of the product.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

using shape = std::vector<int64_t>;
using labels = std::vector<int32_t>;

struct plan_err : std::runtime_error { using std::runtime_error::runtime_error; };
struct eval_err : std::runtime_error { using std::runtime_error::runtime_error; };

int64_t prod(shape const& s) {
  int64_t r = 1;
  for(auto x: s) r *= x;
  return r;
}

// row-major offset (indexing.cc:11-17)
int64_t offset_of(shape const& idx, shape const& bound) {
  int64_t r = 0;
  for(size_t i = 0; i != bound.size(); ++i) r = r * bound[i] + idx[i];
  return r;
}

// lexicographic odometer, last index fastest (indexing.cc:19-28)
bool advance(shape& idx, shape const& bound) {
  for(int i = int(bound.size()) - 1; i >= 0; --i) {
    if(++idx[i] < bound[i]) return true;
    idx[i] = 0;
  }
  return false;
}

// first occurrence of each of l1 in l2 (indexing.cc:30-41)
std::vector<int> positions(labels const& l1, labels const& l2) {
  std::vector<int> r;
  for(auto l: l1) {
    auto it = std::find(l2.begin(), l2.end(), l);
    if(it == l2.end()) throw plan_err("unknown label in projection");
    r.push_back(int(it - l2.begin()));
  }
  return r;
}

shape pick(shape const& b, std::vector<int> const& pos) {
  shape r;
  for(int p: pos) r.push_back(b[p]);
  return r;
}

// The scalar operator sets (ops.cc:5-38).
double join_op(int op, double x, double y) {
  switch(op) {
    case ED_JOIN_MUL: return x * y;
    case ED_JOIN_ADD: return x + y;
    case ED_JOIN_SUB: return x - y;
    case ED_JOIN_DIV:
      if(y == 0.0) throw eval_err("division by zero");
      return x / y;
    case ED_JOIN_SQDIFF: return (x - y) * (x - y);
    case ED_JOIN_ABSDIFF: return std::abs(x - y);
  }
  throw std::runtime_error("bad join op");
}

double map_op(int op, double c, double x) {
  switch(op) {
    case ED_MAP_RELU: return x > 0.0 ? x : 0.0;
    case ED_MAP_EXP: return std::exp(x);
    case ED_MAP_NEG: return -x;
    case ED_MAP_SCALE: return c * x;
    case ED_MAP_IDENTITY: return x;
  }
  throw std::runtime_error("bad map op");
}

double agg_op(int op, double x, double y) {
  return op == ED_AGG_SUM ? x + y : std::max(x, y);
}

// One expression in label space (einsum.cc:31-52).
struct expr_view {
  const ed_vertex_c* v;
  labels lz, lx, ly, lxy, dls;
  bool binary;

  explicit expr_view(const ed_vertex_c* vv) : v(vv) {
    binary = v->arity == 2;
    lz.assign(v->lz, v->lz + v->rank_z);
    lx.assign(v->lx, v->lx + v->rank_x);
    if(binary) ly.assign(v->ly, v->ly + v->rank_y);
    lxy = lx;
    lxy.insert(lxy.end(), ly.begin(), ly.end());
    dls = lx;
    for(auto l: ly) {
      if(std::find(dls.begin(), dls.end(), l) == dls.end()) dls.push_back(l);
    }
  }
};

// The shared nested loop of kernel_eval (kernel.cc:32-65) and eval_expr
// (reference.cc:18-56): `bxy` is the extent over l_XY (chunk-local for a
// kernel call, global for the dense oracle).
void einsum_loop(expr_view const& e, shape const& bxy, const double* x, const double* y,
                 double* out, bool f32) {
  shape dbound = pick(bxy, positions(e.dls, e.lxy));
  auto xp = positions(e.lx, e.dls);
  auto yp = e.binary ? positions(e.ly, e.dls) : std::vector<int>{};
  auto zp = positions(e.lz, e.dls);
  shape xb = pick(dbound, xp), yb = pick(dbound, yp), zb = pick(dbound, zp);
  int64_t nz = prod(zb);
  std::vector<char> touched(size_t(nz), 0);
  auto r32 = [f32](double v) { return f32 ? double(float(v)) : v; };
  if(prod(dbound) == 0) return;
  shape idx(dbound.size(), 0), xi(xp.size()), yi(yp.size()), zi(zp.size());
  do {
    for(size_t i = 0; i != xp.size(); ++i) xi[i] = idx[xp[i]];
    double val;
    if(e.binary) {
      for(size_t i = 0; i != yp.size(); ++i) yi[i] = idx[yp[i]];
      val = r32(join_op(e.v->join_op, r32(x[offset_of(xi, xb)]), r32(y[offset_of(yi, yb)])));
    } else {
      val = r32(map_op(e.v->map_op, e.v->scale_c, r32(x[offset_of(xi, xb)])));
    }
    for(size_t i = 0; i != zp.size(); ++i) zi[i] = idx[zp[i]];
    int64_t o = offset_of(zi, zb);
    if(!touched[size_t(o)]) {
      out[o] = val;
      touched[size_t(o)] = 1;
    } else {
      out[o] = r32(agg_op(e.v->agg_op, out[o], val));
    }
  } while(advance(idx, dbound));
}

void set_err(char* err, size_t errlen, const char* msg) {
  if(err && errlen) std::snprintf(err, errlen, "%s", msg);
}

template <typename F>
int guarded(char* err, size_t errlen, F&& f) {
  try {
    f();
    return ED_OK;
  } catch(plan_err const& e) {
    set_err(err, errlen, e.what());
    return ED_ERR_PLAN;
  } catch(eval_err const& e) {
    set_err(err, errlen, e.what());
    return ED_ERR_EVAL;
  } catch(std::exception const& e) {
    set_err(err, errlen, e.what());
    return ED_ERR_USAGE;
  }
}

// Block copy between a whole tensor and chunk `key` of partition d
// (relation.cc:31-78: global = key * (bound/d) + local).
void block_copy(shape const& bound, shape const& d, shape const& key,
                const double* src, double* dst, bool to_chunk) {
  shape cb(bound.size());
  for(size_t i = 0; i != bound.size(); ++i) cb[i] = bound[i] / d[i];
  shape local(cb.size(), 0), global(cb.size());
  do {
    for(size_t i = 0; i != cb.size(); ++i) global[i] = key[i] * cb[i] + local[i];
    if(to_chunk) dst[offset_of(local, cb)] = src[offset_of(global, bound)];
    else dst[offset_of(global, bound)] = src[offset_of(local, cb)];
  } while(advance(local, cb));
}

// Plan-level helpers shared by the whole-plan and per-vertex entry points.
struct plan_view {
  const ed_plan_c* plan;
  explicit plan_view(const ed_plan_c* p) : plan(p) {}
  shape bound_of(int vid) const { auto const& v = plan->vertices[vid]; return shape(v.bound, v.bound + v.rank); }
  shape d_of(int vid) const { auto const& v = plan->vertices[vid]; return shape(v.d, v.d + v.rank_d); }
  shape key_of(int id) const { auto const& x = plan->exec[id]; return shape(x.key, x.key + x.key_rank); }
  shape cb_of(int id) const { auto const& x = plan->exec[id]; return shape(x.chunk_bound, x.chunk_bound + x.chunk_rank); }

  // task_graph_t::out_partition / required_input_partition (decomp.cc:3-14)
  shape out_partition(int vid) const {
    if(plan->vertices[vid].arity == 0) return d_of(vid);
    expr_view e(&plan->vertices[vid]);
    return pick(d_of(vid), positions(e.lz, e.lxy));
  }
  shape required_partition(int vid, int slot) const {
    expr_view e(&plan->vertices[vid]);
    return pick(d_of(vid), positions(slot == 0 ? e.lx : e.ly, e.lxy));
  }
  // engine_t::region_key / region_partition (runtime.cc:96-116)
  shape region_key(int id) const {
    auto const& u = plan->exec[id];
    if(u.kind != ED_EXEC_JOIN) return key_of(id);
    expr_view e(&plan->vertices[u.producer]);
    return pick(key_of(id), positions(e.lz, e.dls));
  }
  shape region_partition(int id) const {
    auto const& u = plan->exec[id];
    if(u.kind == ED_EXEC_INPUT_CHUNK) return d_of(u.producer);
    if(u.kind == ED_EXEC_JOIN) return out_partition(u.producer);
    if(u.consumer >= 0) return required_partition(u.consumer, u.slot);
    return out_partition(u.producer);
  }

  // compute() (runtime.cc:183-270) for one join or refinement, given its
  // dependency chunks in dep order
  void compute(int id, const double* const* deps, double* out, bool r32) const {
    auto const& v = plan->exec[id];
    auto const* V = plan->vertices;
    std::fill(out, out + v.sz, 0.0);
    if(v.kind == ED_EXEC_JOIN) {
      // join branch: spec.local_xy = b_XY / d (runtime.cc:51-63, 185-196)
      int w = v.producer;
      expr_view e(&V[w]);
      shape bxy;
      for(int s = 0; s != V[w].arity; ++s) {
        auto b = bound_of(V[w].inputs[s]);
        bxy.insert(bxy.end(), b.begin(), b.end());
      }
      shape d = d_of(w);
      for(size_t i = 0; i != bxy.size(); ++i) bxy[i] /= d[i];
      einsum_loop(e, bxy, deps[0], e.binary ? deps[1] : nullptr, out, r32);
      return;
    }
    // refinement branch: paste each dep's overlap rectangle, folding
    // aggregation siblings in dep order (runtime.cc:198-269)
    int w = v.producer;
    shape bound = bound_of(w);
    shape dc = region_partition(id);
    int agg = V[w].arity == 0 ? -1 : V[w].agg_op;
    shape cbound = cb_of(id), ckey = key_of(id);
    std::vector<char> touched(size_t(v.sz), 0);
    shape c0(bound.size());
    for(size_t i = 0; i != bound.size(); ++i) c0[i] = ckey[i] * (bound[i] / dc[i]);
    for(int k = 0; k != v.n_deps; ++k) {
      int uid = v.deps[k];
      shape rk = region_key(uid), dr = region_partition(uid);
      shape r0(bound.size()), lo(bound.size()), span(bound.size());
      bool empty = false;
      for(size_t i = 0; i != bound.size(); ++i) {
        r0[i] = rk[i] * (bound[i] / dr[i]);
        lo[i] = std::max(r0[i], c0[i]);
        int64_t hi = std::min(r0[i] + bound[i] / dr[i], c0[i] + cbound[i]);
        span[i] = hi - lo[i];
        if(span[i] <= 0) empty = true;
      }
      if(empty) continue;
      shape ub = cb_of(uid);
      shape rel(bound.size(), 0), ui(bound.size()), ci(bound.size());
      const double* u = deps[k];
      do {
        for(size_t i = 0; i != bound.size(); ++i) {
          ui[i] = lo[i] + rel[i] - r0[i];
          ci[i] = lo[i] + rel[i] - c0[i];
        }
        double val = u[offset_of(ui, ub)];
        int64_t off = offset_of(ci, cbound);
        if(!touched[size_t(off)]) {
          out[off] = val;
          touched[size_t(off)] = 1;
        } else {
          if(agg < 0) throw plan_err("execute: overlapping contributions without an aggregation op");
          double r = agg_op(agg, out[off], val);
          out[off] = r32 ? double(float(r)) : r;
        }
      } while(advance(rel, span));
    }
    for(char t: touched) {
      if(!t) throw plan_err("execute: refinement chunk left partially unwritten");
    }
  }
};

} // namespace

extern "C" {

int oracle_kernel_eval(const ed_vertex_c* v, const int64_t* local_xy, const double* cx,
                       const double* cy, double* out, int f32, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    expr_view e(v);
    shape lxy(local_xy, local_xy + e.lxy.size());
    einsum_loop(e, lxy, cx, cy, out, f32 != 0);
  });
}

int oracle_eval_expr(const ed_vertex_c* v, const int64_t* bxy, const double* x,
                     const double* y, double* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    expr_view e(v);
    shape b(bxy, bxy + e.lxy.size());
    einsum_loop(e, b, x, y, out, false);
  });
}

void oracle_chunk(int32_t rank, const int64_t* bound, const int64_t* d, const double* t,
                  double* out) {
  shape b(bound, bound + rank), dd(d, d + rank), key(size_t(rank), 0);
  int64_t csz = prod(b) / prod(dd);
  int64_t k = 0;
  do {
    block_copy(b, dd, key, t, out + k * csz, true);
    ++k;
  } while(advance(key, dd));
}

void oracle_assemble(int32_t rank, const int64_t* bound, const int64_t* d,
                     const double* chunks, double* out) {
  shape b(bound, bound + rank), dd(d, d + rank), key(size_t(rank), 0);
  int64_t csz = prod(b) / prod(dd);
  int64_t k = 0;
  do {
    block_copy(b, dd, key, chunks + k * csz, out, false);
    ++k;
  } while(advance(key, dd));
}

double oracle_max_rel_err(const double* got, const double* expect, int64_t n) {
  double r = 0.0;
  for(int64_t i = 0; i != n; ++i) {
    r = std::max(r, std::abs(got[i] - expect[i]) / std::max(1.0, std::abs(expect[i])));
  }
  return r;
}

void oracle_generate_input(int64_t n, int32_t integer_valued, uint64_t seed, int32_t vid,
                           double* out) {
  std::mt19937_64 gen(seed * 7919 + uint64_t(vid));
  if(integer_valued) {
    std::uniform_int_distribution<int> dist(-4, 4);
    for(int64_t i = 0; i != n; ++i) out[i] = dist(gen);
  } else {
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for(int64_t i = 0; i != n; ++i) out[i] = dist(gen);
  }
}

int oracle_execute(const ed_plan_c* plan, const ed_tensor_in_c* inputs, int32_t n_inputs,
                   int32_t f32, ed_output_c* outputs, int32_t n_outputs,
                   double* const* chunk_out, ed_machine_c* counters,
                   int64_t* total_transferred, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    plan_view pv(plan);
    int ne = plan->n_exec;
    auto const* X = plan->exec;
    std::vector<std::vector<double>> produced{size_t(ne)};
    // seed: chunk each input tensor (engine_t ctor, runtime.cc:66-84)
    std::map<int, const double*> in_data;
    for(int i = 0; i != n_inputs; ++i) {
      if(inputs[i].dtype != ED_DTYPE_F64) throw plan_err("oracle: inputs must be f64");
      in_data[inputs[i].vertex_id] = static_cast<const double*>(inputs[i].data);
    }
    for(int id = 0; id != ne; ++id) {
      if(X[id].kind != ED_EXEC_INPUT_CHUNK) continue;
      int vid = X[id].producer;
      auto it = in_data.find(vid);
      if(it == in_data.end()) throw plan_err("execute: no relation supplied for an input");
      produced[id].resize(size_t(X[id].sz));
      block_copy(pv.bound_of(vid), pv.d_of(vid), pv.key_of(id), it->second, produced[id].data(), true);
    }
    for(int id = 0; id != ne; ++id) {
      if(X[id].kind == ED_EXEC_INPUT_CHUNK) continue;
      produced[id].assign(size_t(X[id].sz), 0.0);
      std::vector<const double*> deps;
      for(int k = 0; k != X[id].n_deps; ++k) deps.push_back(produced[X[id].deps[k]].data());
      pv.compute(id, deps.data(), produced[id].data(), f32 != 0);
    }

    // counters: one whole-chunk pull per (chunk, machine) (runtime.cc:119-172)
    if(counters) {
      for(int m = 0; m != plan->n_machines; ++m) counters[m] = ed_machine_c{0, 0, 0};
      std::set<std::pair<int, int>> pulled;
      int64_t total = 0;
      for(int id = 0; id != ne; ++id) {
        auto const& v = X[id];
        if(v.kind == ED_EXEC_INPUT_CHUNK) continue;
        counters[v.machine].fp += v.fp;
        for(int k = 0; k != v.n_deps; ++k) {
          int dep = v.deps[k];
          if(X[dep].machine != v.machine && pulled.insert({dep, v.machine}).second) {
            counters[X[dep].machine].sent += X[dep].sz;
            counters[v.machine].received += X[dep].sz;
            total += X[dep].sz;
          }
        }
      }
      if(total_transferred) *total_transferred = total;
    }

    if(chunk_out) {
      for(int id = 0; id != ne; ++id) {
        if(chunk_out[id]) std::memcpy(chunk_out[id], produced[id].data(), sizeof(double) * produced[id].size());
      }
    }

    // output assembly (runtime.cc:432-448)
    for(int i = 0; i != n_outputs; ++i) {
      int vid = outputs[i].vertex_id;
      if(outputs[i].dtype != ED_DTYPE_F64) throw plan_err("oracle: outputs must be f64");
      double* dst = static_cast<double*>(outputs[i].data);
      shape bound = pv.bound_of(vid);
      shape part = pv.out_partition(vid);
      for(int id = 0; id != ne; ++id) {
        auto const& u = X[id];
        bool mine = plan->vertices[vid].arity == 0
          ? (u.kind == ED_EXEC_INPUT_CHUNK && u.producer == vid)
          : (u.kind == ED_EXEC_REFINEMENT && u.producer == vid && u.consumer < 0);
        if(mine) block_copy(bound, part, pv.key_of(id), produced[id].data(), dst, false);
      }
    }
  });
}

int oracle_exec_vertex(const ed_plan_c* plan, int32_t exec_id, const double* const* deps, double* out,
                       int32_t f32, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if(exec_id < 0 || exec_id >= plan->n_exec) throw plan_err("exec id out of range");
    if(plan->exec[exec_id].kind == ED_EXEC_INPUT_CHUNK) throw plan_err("input chunks are not computed");
    plan_view(plan).compute(exec_id, deps, out, f32 != 0);
  });
}

} // extern "C"
