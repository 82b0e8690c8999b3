// libed_gpu: the B200 executor behind include/ed_gpu.h.
//
// Replaces execute() (runtime.cc:382-451). ed_prepare turns the placed
// ExecGraph into a static schedule of kernel launches on a compute stream:
//   * mul/sum joins of one output region -> ONE tcgen05 GEMM whose K loop
//     runs over the region's aggregation siblings, so the sibling fold of the
//     refinement (runtime.cc:242-261) happens in the TMEM accumulator;
//   * every other join -> the exact generic inner-EinSum kernel;
//   * refinements that are a single same-shape dependency -> aliases (no
//     copy); all others -> the ordered gather/fold kernel;
//   * remote dependencies (world > 1) -> NCCL send/recv groups on a comm
//     stream that forks from / joins the compute stream (enqueue()).
// The schedule is captured once into a CUDA graph and replayed by ed_run.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>
#include <functional>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "ed_gpu.h"
#include "gemm_sm100.h"
#include "attn_sm100.h"
#include "ewise.h"
#include "kernels.h"

using namespace ed;

namespace {

using shape = std::vector<int64_t>;
using labels = std::vector<int32_t>;

struct ed_error : std::runtime_error {
  ed_status code;
  ed_error(ed_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CUDA_OK(expr)                                                                         \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      throw ed_error(e_ == cudaErrorMemoryAllocation ? ED_ERR_OOM : ED_ERR_CUDA,              \
                     std::string(#expr) + ": " + cudaGetErrorString(e_));                     \
  } while (0)

#define NCCL_OK(expr)                                                                         \
  do {                                                                                        \
    ncclResult_t r_ = (expr);                                                                 \
    if (r_ != ncclSuccess) throw ed_error(ED_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
  } while (0)

void set_err(char* err, size_t errlen, const std::string& m) {
  if (err && errlen) std::snprintf(err, errlen, "%s", m.c_str());
}

template <typename F>
ed_status guarded(char* err, size_t errlen, F&& f) {
  try {
    f();
    return ED_OK;
  } catch (ed_error const& e) {
    set_err(err, errlen, e.what());
    return e.code;
  } catch (std::exception const& e) {
    set_err(err, errlen, e.what());
    return ED_ERR_USAGE;
  }
}

int64_t prod(const shape& s) {
  int64_t r = 1;
  for (auto x : s) r *= x;
  return r;
}

std::vector<int> positions(const labels& l1, const labels& l2) {
  std::vector<int> r;
  for (auto l : l1) {
    auto it = std::find(l2.begin(), l2.end(), l);
    if (it == l2.end()) throw ed_error(ED_ERR_PLAN, "unknown label in projection");
    r.push_back(int(it - l2.begin()));
  }
  return r;
}

shape pick(const shape& b, const std::vector<int>& pos) {
  shape r;
  for (int p : pos) r.push_back(b[p]);
  return r;
}

// ---- deep copy of the plan ----------------------------------------------------
struct Vtx {
  std::string name;
  int arity, join, map, agg;
  double c;
  shape bound, d;
  labels lz, lx, ly, lxy, dls;
  int inputs[2];
};

struct Ex {
  int kind, owner, producer, consumer, slot, machine;
  shape key, cb;
  int64_t fp, sz;
  std::vector<int> deps;
};

// ---- label -> GEMM mapping ----------------------------------------------------
struct Dim {
  int64_t ext = 1, stride = 0;
};

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

struct GemmMap {
  int a_slot, b_slot;  // which einsum input feeds MMA-A / MMA-B
  Dim am, ak, ab, bn, bk, bb, cm, cn, cb;
  bool a_mn, b_mn;
  labels lA, lB, Mc, Nc, Kc, Bc;  // operand label lists and the label classes
};

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

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    CUDA_OK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p) throw ed_error(ED_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D tensor map {inner, outer, batch} with a 128-byte swizzled box.
void make_map(CUtensorMap* m, const void* base, bool bf16, int64_t inner, int64_t outer, int64_t outer_stride,
              int64_t batch, int64_t batch_stride, uint32_t box_inner, uint32_t box_outer,
              CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  const int es = bf16 ? 2 : 4;
  cuuint64_t dims[3] = {cuuint64_t(inner), cuuint64_t(outer), cuuint64_t(batch)};
  auto fix = [&](int64_t s, int64_t prev_bytes) -> cuuint64_t {
    int64_t b = s * es;
    if (b <= 0 || b % 16) b = ((prev_bytes + 15) / 16) * 16;  // unit extent: stride unused
    return cuuint64_t(b);
  };
  cuuint64_t s1 = fix(outer > 1 ? outer_stride : 0, inner * es);
  cuuint64_t s2 = fix(batch > 1 ? batch_stride : 0, int64_t(s1) * outer);
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {box_inner, box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                           const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw ed_error(ED_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
}

// ---- schedule -------------------------------------------------------------------
enum class OpKind { GEMM, GENERIC, REFINE, CORRUPT, SEND, RECV, CONVERT, EWISE, ROWREDUCE, SOFTMAX, FLASH, SPLIT };

struct Op {
  OpKind kind;
  std::string name;   // launch class, e.g. "gemm_bf16:Z1"
  double flops = 0, bytes = 0;
  GemmLaunch gemm{};
  AttnLaunch attn{};
  std::vector<AttnRegion> aregions;
  std::vector<RowSeg> rowsegs;         // SOFTMAX: x read in place from column segments
  std::vector<int> heads;              // GEMM: region heads (join ids), fold order
  std::vector<CUtensorMap> maps;       // GEMM: host copies, uploaded by allocate()
  std::vector<GemmRegion> regions;
  bool bf16 = false;
  GenericParams gen;
  RefineParams ref;
  EwiseParams ew{};
  RectParams rect{};
  std::vector<RectGroup> groups;       // REFINE fast path (empty: generic fold kernel)
  int64_t max_rows = 0;
  RowReduceParams rr{};
  SoftmaxParams sm{};
  std::vector<JoinPtrs> jptrs;         // EWISE / ROWREDUCE: per-join operands
  void* ptr = nullptr;
  DT dt = DT::F32;
  int peer = -1;
  size_t count = 0;
  int exec = -1;      // SEND / RECV: the chunk's exec id
  int einsum = -1;    // GEMM: the graph vertex it computes
};

struct Buffer {
  size_t off_main = SIZE_MAX, off_16 = SIZE_MAX, off_lo = SIZE_MAX;
  bool need_main = false, need_16 = false, need_lo = false;
  void* main = nullptr;
  void* b16 = nullptr;
  void* lo = nullptr;   // F32X3: x - tf32(x)
};

// Memory-bound join shapes with a dedicated grouped kernel (ewise.cu).
struct MemMap {
  OpKind kind;
  int y_mode = 0;
  int64_t inner = 1, rows = 1, len = 1;
};

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

}  // namespace

struct ed_ctx {
  int device = 0, rank = 0, world = 1, num_sms = 148;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr, comm_stream = nullptr;
};

struct ed_plan_h {
  ed_ctx* ctx = nullptr;
  ed_options_c opt{};
  std::vector<Vtx> V;
  std::vector<Ex> X;
  std::vector<int> outputs;
  int n_machines = 1;
  double alpha = 0.0;
  bool f64 = false;
  DT store = DT::F32;
  size_t es = 4;

  std::vector<int> owner;          // exec id -> exec id holding its data
  std::vector<char> local;         // exec id runs (or is received) on this rank
  std::vector<Buffer> buf;         // indexed by exec id (meaningful at owners)
  std::vector<Op> ops;
  std::vector<ed_machine_c> counters;
  int64_t total_transferred = 0, peer_bytes = 0;
  double max_site_cost = 0.0, contraction_flops = 0.0;
  int first_join = -1;

  void* arena = nullptr;
  size_t arena_bytes = 0;
  DepRect* d_deps = nullptr;
  void* d_maps = nullptr;          // CUtensorMap[] of all GEMM launches
  void* d_regions = nullptr;       // GemmRegion[] of all GEMM launches
  void** d_ptrs = nullptr;         // chunk-pointer tables for scatter/gather
  int* d_err = nullptr;
  void* staging = nullptr;
  size_t staging_bytes = 0;
  // ed_run_steps: copy streams, double-buffered staging, cached copy descriptors
  struct CopyPlan {
    void* d = nullptr;  // BlockCopy[] on the device
    int n = 0, rank = 0;
    int64_t max_rows = 1;
  };
  std::map<std::tuple<int, int, const void*, int>, CopyPlan> copy_cache;
  cudaStream_t cs_in = nullptr, cs_out = nullptr;
  void* stg_in[2] = {nullptr, nullptr};
  void* stg_out[2] = {nullptr, nullptr};
  size_t stg_in_bytes = 0, stg_out_bytes = 0;
  cudaEvent_t ev_pipe[8] = {};  // in_full[2], in_free[2], out_full[2], out_free[2]
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<cudaEvent_t> op_events;
  std::vector<ed_kernel_stat_c> stats;

  struct SrcRec {
    int ref, src;
    shape r0, ext;
  };
  std::vector<SrcRec> srcs_;                      // refinement sources, fold order
  std::map<int, GemmMap> gmap_;                   // einsum -> GEMM mapping
  std::map<int, std::vector<int>> region_sibs_;   // GEMM head join -> siblings
  std::map<int, MemMap> memmap_;                  // einsum -> memory-bound kernel shape
  struct Softmax {
    int y;
    int x;                                        // the chain's input vertex
    int64_t len;
    std::vector<std::pair<int, int>> pairs;       // (Y join, x chunk ref)
    std::vector<int> m_refs;                      // row-max chunk refs when M stays unfused
    struct XSeg {
      int owner;
      int64_t row0, stride;
    };
    std::vector<std::vector<XSeg>> xsegs;         // per pair: x read in place from column segments
    int seg_w = 0;
  };
  struct KVTiles {                                // K or V read in place from producer regions
    bool tiled = false;
    std::vector<int> owners;                      // grid (key block, d block), row-major
    int nd = 1;
    int64_t keys = 0, dw = 0, hoff = 0;
    shape ext;                                    // source region extents (operand label order)
  };
  struct Flash {                                  // T1 -> softmax -> O in one kernel
    int t1, y, o;
    float scale;
    std::vector<std::array<int, 4>> regions;      // (Q ref, K ref, V ref, O region head)
    std::vector<KVTiles> ktiles, vtiles;          // per region
  };
  std::map<int, Flash> flash_;                    // O vertex -> fused attention block
  struct Seg {
    int owner;                                    // source region buffer
    int64_t k0, kext;                             // its range along the contraction label
    Dim mn, k, b;                                 // its layout for the GEMM classes
  };
  struct KSeg {
    int role = 0;                                 // 0: MMA-A operand segmented, 1: MMA-B
    int64_t kseg = -1;
    std::map<int, std::vector<Seg>> segs;         // join -> segments in K order
  };
  std::map<int, KSeg> kseg_;                      // GEMM einsum -> K-segmented operand
  std::set<int> flash_skip_;                      // einsums computed inside a Flash op
  std::map<int, Softmax> softmax_;                // Y vertex -> fused row-softmax chain
  std::map<int, std::pair<int, double>> epi_;     // GEMM einsum -> epilogue map (op, c)
  std::vector<char> opaque_;                      // exec id whose value was fused into a consumer
  void* d_joinptrs = nullptr;                     // JoinPtrs[] of grouped memory-bound launches
  void* d_rects = nullptr;                        // RectGroup[] of fast refinements
  void* d_copy_desc = nullptr;                    // BlockCopy[] scratch for upload / download
  void* d_attn = nullptr;                         // tensor maps + regions of fused attention launches
  void* d_rowsegs = nullptr;                      // RowSeg[] of softmax launches reading in place
  size_t copy_desc_bytes = 0;

  int rank_of(int id) const { return X[id].machine % ctx->world; }
  shape out_partition(int w) const {
    if (V[w].arity == 0) return V[w].d;
    return pick(V[w].d, positions(V[w].lz, V[w].lxy));
  }
  shape required_partition(int w, int slot) const {
    return pick(V[w].d, positions(slot == 0 ? V[w].lx : V[w].ly, V[w].lxy));
  }
  // engine_t::region_key / region_partition (runtime.cc:96-116)
  shape region_key(int id) const {
    const Ex& u = X[id];
    if (u.kind != ED_EXEC_JOIN) return u.key;
    return pick(u.key, positions(V[u.producer].lz, V[u.producer].dls));
  }
  shape region_partition(int id) const {
    const Ex& u = X[id];
    if (u.kind == ED_EXEC_INPUT_CHUNK) return V[u.producer].d;
    if (u.kind == ED_EXEC_JOIN) return out_partition(u.producer);
    if (u.consumer >= 0) return required_partition(u.consumer, u.slot);
    return out_partition(u.producer);
  }
  shape local_xy(int w) const {
    shape b;
    for (int s = 0; s < V[w].arity; ++s) {
      const shape& bi = V[V[w].inputs[s]].bound;
      b.insert(b.end(), bi.begin(), bi.end());
    }
    for (size_t i = 0; i < b.size(); ++i) b[i] /= V[w].d[i];
    return b;
  }
  void* main_of(int id) { return buf[owner[id]].main; }
  void* b16_of(int id) { return buf[owner[id]].b16; }

  // Remote dependencies: (dep, destination rank), placed before the dep's
  // first consumer on that rank — where the consumer is LAUNCHED: the joins
  // of one einsum run as one grouped launch at the position of its first
  // join, so a transfer feeding any of them goes before that position. The
  // positions depend on the plan only, so every rank derives the same
  // global transfer order.
  std::vector<std::vector<std::pair<int, int>>> transfers_by_consumer() const {
    const int ne = int(X.size());
    std::map<int, int> first_join;  // einsum -> its lowest join id
    for (int id = 0; id < ne; ++id)
      if (X[id].kind == ED_EXEC_JOIN) first_join.emplace(X[id].producer, id);
    std::vector<std::vector<std::pair<int, int>>> at(ne);
    std::map<std::pair<int, int>, int> pos;  // (dep, dst) -> launch position of its first consumer
    for (int id = 0; id < ne; ++id) {
      if (X[id].kind == ED_EXEC_INPUT_CHUNK) continue;
      const int dst = rank_of(id);
      const int lp = X[id].kind == ED_EXEC_JOIN ? first_join.at(X[id].producer) : id;
      for (int d : X[id].deps) {
        if (rank_of(d) == dst) continue;
        auto it = pos.find({d, dst});
        if (it == pos.end()) pos.emplace(std::make_pair(d, dst), lp);
        else it->second = std::min(it->second, lp);
      }
    }
    // within one position, transfers keep the consumers' exec-id order
    std::vector<std::tuple<int, int, int, int>> order;  // (position, first consumer, dep, dst)
    std::set<std::pair<int, int>> seen;
    for (int id = 0; id < ne; ++id) {
      if (X[id].kind == ED_EXEC_INPUT_CHUNK) continue;
      const int dst = rank_of(id);
      for (int d : X[id].deps)
        if (rank_of(d) != dst && seen.insert({d, dst}).second) order.emplace_back(pos.at({d, dst}), id, d, dst);
    }
    std::stable_sort(order.begin(), order.end(),
                     [](const auto& a, const auto& b) { return std::get<0>(a) < std::get<0>(b); });
    for (auto& [p, c, d, dst] : order) {
      (void)c;
      if (d >= p) throw ed_error(ED_ERR_PLAN, "transfer scheduled before its chunk is produced");
      at[p].push_back({d, dst});
    }
    return at;
  }
  void copy_plan(const ed_plan_c* p);
  void validate();
  void build();
  void allocate();
  void record();
  void launch_op(size_t i, cudaStream_t s);
  void enqueue(cudaStream_t s);
  std::vector<cudaEvent_t> comm_events;  // fork / join points of the comm stream
  cudaStream_t aux[2] = {nullptr, nullptr};  // independent GEMMs run as parallel graph branches
  // graph vertex a is an ancestor of b (data flows from a to b)
  bool ancestor(int a, int b) const {
    std::vector<int> todo{b};
    std::vector<char> seen(V.size(), 0);
    while (!todo.empty()) {
      const int w = todo.back();
      todo.pop_back();
      for (int k = 0; k < V[w].arity; ++k) {
        const int in = V[w].inputs[k];
        if (in == a) return true;
        if (in >= 0 && !seen[size_t(in)]) {
          seen[size_t(in)] = 1;
          todo.push_back(in);
        }
      }
    }
    return false;
  }
  // peer transport (ED_TRANSPORT_PEER): run epoch, exported flag words
  // [0] run done, [1] outputs downloaded, [2 + id] chunk id ready; the peers'
  // arenas, flags and chunk offsets as mapped by ed_peer_import
  bool peer = false, peer_ready = false;
  int* d_epoch = nullptr;
  int* d_pflags = nullptr;
  int* d_perr = nullptr;  // a peer wait that timed out: 1 + tag * 64 + flag
  void check_peer_error() {
    if (!d_perr) return;
    int e = 0;
    CUDA_OK(cudaMemcpy(&e, d_perr, sizeof(int), cudaMemcpyDeviceToHost));
    if (!e) return;
    CUDA_OK(cudaMemset(d_perr, 0, sizeof(int)));
    const int tag = (e - 1) / 64, i = (e - 1) % 64, ne = int(X.size());
    std::string what = tag < ne   ? "chunk " + std::to_string(tag) + " from rank " + std::to_string(rank_of(tag))
                       : tag == ne ? "the run-start barrier (rank " + std::to_string(i) + ")"
                       : tag == ne + 1 ? "rank " + std::to_string(i) + " finishing the run (download)"
                                       : "rank 0's download";
    throw ed_error(ED_ERR_CUDA, "peer transport: timed out waiting for " + what);
  }
  std::vector<char*> peer_arena;
  std::vector<int*> peer_flags;
  std::vector<std::vector<int64_t>> peer_off;
  int64_t arena_offset(int id) const {
    const Buffer& b = buf[owner[id]];
    return b.main ? int64_t(static_cast<char*>(b.main) - static_cast<char*>(arena)) : -1;
  }
  void destroy();
};

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
}

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
  const int max_sib = x3 ? kMaxSib / 3 : kMaxSib;  // F32X3 runs 3 products per sibling

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
    // label) -> one kernel; T1 and T3 are never materialised (bf16 only)
    static const bool ftrace = std::getenv("ED_FUSE_TRACE") != nullptr;
#define REJECT(k)                                                                            \
  {                                                                                          \
    if (ftrace) std::fprintf(stderr, "[ed] rank %d: attention block at %s not fused (%d)\n", me, \
                             V[yv].name.c_str(), k);                                         \
    continue;                                                                                \
  }
    for (auto& [yv, sm] : softmax_) {
      if (!bf16) break;
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
          go.bn.ext != Dd || T != sm.len || !attn_supported(int(S), int(T), int(Dd)))
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
        ok = ok && real * int(segs.size()) * (x3 ? 3 : 1) <= kMaxSib;
      }
      if (!ok || refs.empty()) continue;
      kseg_[c] = ks;
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
        buf[local[r[0]] ? owner[r[0]] : r[0]].need_16 = true;
        for (int k = 1; k < 3; ++k) {
          const KVTiles& t = k == 1 ? f.ktiles[q] : f.vtiles[q];
          if (t.tiled)
            for (int o2 : t.owners) buf[o2].need_16 = true;
          else
            buf[local[r[k]] ? owner[r[k]] : r[k]].need_16 = true;
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
          if (segmented) {
            for (auto& sg : kseg_[w].segs.at(id)) reads.push_back(sg.owner);
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
  std::set<int> split_done;
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
        for (auto& [yj, xr] : softmax_[u.producer].pairs) op.heads.push_back(yj);
        ops.push_back(op);
        continue;
      }
      if (flash_.count(u.producer)) {
        if (!fused_head[id] || gemm_emitted.count(u.producer)) continue;
        gemm_emitted.insert(u.producer);
        const Flash& f = flash_.at(u.producer);
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
                if (X[o].kind == ED_EXEC_INPUT_CHUNK || !split_done.insert(o).second) continue;
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
  this->srcs_.clear();
  for (int id = 0; id < ne; ++id)
    for (auto& s : srcs[id]) this->srcs_.push_back({id, s.id, s.r0, s.ext});
  this->gmap_ = gmap;
  this->epi_ = epi;
  this->region_sibs_ = region_sibs;
}

void ed_plan_h::allocate() {
  const int ne = int(X.size());
  CUDA_OK(cudaMalloc(&arena, arena_bytes));
  char* base = static_cast<char*>(arena);
  for (int id = 0; id < ne; ++id) {
    if (buf[id].off_main != SIZE_MAX) buf[id].main = base + buf[id].off_main;
    if (buf[id].off_16 != SIZE_MAX) buf[id].b16 = base + buf[id].off_16;
    if (buf[id].off_lo != SIZE_MAX) buf[id].lo = base + buf[id].off_lo;
  }
  CUDA_OK(cudaMalloc(&d_err, sizeof(int)));
  CUDA_OK(cudaMemset(d_err, 0, sizeof(int)));
  CUDA_OK(cudaMalloc(&d_ptrs, sizeof(void*) * 2 * std::max(1, ne)));

  // refinement dependency tables, one contiguous device array
  std::vector<DepRect> host_deps;
  std::map<int, size_t> dep_off;
  for (auto& s : srcs_) {
    if (!dep_off.count(s.ref)) dep_off[s.ref] = host_deps.size();
    DepRect r{};
    r.src = buf[s.src].main;
    for (size_t i = 0; i < s.r0.size(); ++i) {
      r.r0[i] = s.r0[i];
      r.ext[i] = s.ext[i];
    }
    host_deps.push_back(r);
  }
  if (!host_deps.empty()) {
    CUDA_OK(cudaMalloc(&d_deps, sizeof(DepRect) * host_deps.size()));
    CUDA_OK(cudaMemcpy(d_deps, host_deps.data(), sizeof(DepRect) * host_deps.size(), cudaMemcpyHostToDevice));
  }

  auto resolve = [&](int dep) { return local[dep] ? owner[dep] : dep; };
  size_t gemm_maps_total = 0, gemm_regions_total = 0, jptrs_total = 0, rect_total = 0;
  size_t attn_maps_total = 0, attn_regions_total = 0, rowseg_total = 0;
  for (auto& op : ops) {
    const int id = int(reinterpret_cast<intptr_t>(op.ptr));
    switch (op.kind) {
      case OpKind::GEMM: {
        const Ex& u = X[id];
        const GemmMap& g = gmap_.at(u.producer);
        GemmLaunch& p = op.gemm;
        const bool b16 = op.bf16;
        p.bf16 = b16;
        p.M = int(g.am.ext);
        p.N = int(g.bn.ext);
        p.K = int(kseg_.count(u.producer) ? kseg_.at(u.producer).kseg : g.ak.ext);
        p.batch = int(g.ab.ext);
        p.a_mn = g.a_mn;
        p.b_mn = g.b_mn;
        p.c_sm = g.cm.ext > 1 ? g.cm.stride : 0;
        p.c_sb = g.cb.ext > 1 ? g.cb.stride : 0;
        p.vec_ok = (p.c_sm % 8 == 0) && (p.c_sb % 8 == 0);
        p.epi_map = -1;
        if (epi_.count(u.producer)) {
          p.epi_map = epi_.at(u.producer).first;
          p.epi_c = float(epi_.at(u.producer).second);
          op.name += "+map";
        }
        p.bn = gemm_pick_bn(p.M, p.N, p.batch, int(op.heads.size()), ctx->num_sms);
        p.x3 = opt.precision == ED_PREC_F32X3;
        p.group_m = 8;
        if (const char* gm = std::getenv("ED_GEMM_GROUP_M")) p.group_m = std::max(1, std::atoi(gm));  // experiments
        const uint32_t BK = uint32_t(gemm_bk(b16)), BM = uint32_t(gemm_bm());
        const uint32_t ATOM = 128u / (b16 ? 2u : 4u);
        op.maps.clear();
        op.regions.clear();
        int total_sib = 0;
        for (int head : op.heads) {
          const auto& sibs = region_sibs_.at(head);
          GemmRegion r{};
          r.n_sib = int(sibs.size());
          r.map0 = int(op.maps.size());
          const bool x3 = opt.precision == ED_PREC_F32X3;
          const KSeg* ks = kseg_.count(u.producer) ? &kseg_.at(u.producer) : nullptr;
          const int nseg = ks ? int(ks->segs.at(sibs[0]).size()) : 1;
          r.n_sib = int(sibs.size()) * nseg;
          // MN-major fp32 operands need the 32-byte-atom swizzle (see gemm_sm100.cu)
          const CUtensorMapSwizzle mn_swz = b16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
          const int es_op = b16 ? 2 : 4;
          for (int pseudo = 0; pseudo < r.n_sib; ++pseudo) {
            const int sidx = sibs[pseudo / nseg];
            const int seg = pseudo % nseg;
            const Ex& j = X[sidx];
            int da = resolve(j.deps[g.a_slot]), db = resolve(j.deps[g.b_slot]);
            Dim am = g.am, ak = g.ak, ab = g.ab, bn = g.bn, bk = g.bk, bb = g.bb;
            int64_t aoff = 0, boff = 0;
            if (ks) {
              const Seg& sg = ks->segs.at(sidx)[seg];
              if (ks->role == 0) {
                da = sg.owner;
                am = sg.mn;
                ak = sg.k;
                ab = sg.b;
                bk.ext = sg.kext;
                boff = sg.k0 * g.bk.stride;
              } else {
                db = sg.owner;
                bn = sg.mn;
                bk = sg.k;
                bb = sg.b;
                ak.ext = sg.kext;
                aoff = sg.k0 * g.ak.stride;
              }
            }
            // F32X3: A, B, then their lo copies (x - tf32(x)); the kernel feeds
            // hi*hi + hi*lo + lo*hi from one stage into the accumulator
            for (int part = 0; part < (x3 ? 2 : 1); ++part) {
              const char* pa = static_cast<const char*>(b16 ? buf[da].b16 : part ? buf[da].lo : buf[da].main);
              const char* pb = static_cast<const char*>(b16 ? buf[db].b16 : part ? buf[db].lo : buf[db].main);
              if (!pa || !pb) throw ed_error(ED_ERR_PLAN, "GEMM operand buffer missing");
              pa += aoff * es_op;
              pb += boff * es_op;
              CUtensorMap ma, mb;
              if (!g.a_mn) make_map(&ma, pa, b16, ak.ext, am.ext, am.stride, ab.ext, ab.stride, BK, BM);
              else make_map(&ma, pa, b16, am.ext, ak.ext, ak.stride, ab.ext, ab.stride, ATOM, BK, mn_swz);
              if (!g.b_mn)
                make_map(&mb, pb, b16, bk.ext, bn.ext, bn.stride, bb.ext, bb.stride, BK, uint32_t(gemm_b_box(p.M, p.bn)));
              else make_map(&mb, pb, b16, bn.ext, bk.ext, bk.stride, bb.ext, bb.stride, ATOM, BK, mn_swz);
              op.maps.push_back(ma);
              op.maps.push_back(mb);
            }
            total_sib += x3 ? 2 : 1;
          }
          r.c32 = static_cast<float*>(buf[head].main);
          r.c16 = buf[head].b16;
          // output tensor maps for the TMA-store epilogue (16-byte strides only)
          auto out_map = [&](void* base, bool o16) {
            const int oes = o16 ? 2 : 4;
            bool ok = base && (g.cm.ext == 1 || (g.cm.stride * oes) % 16 == 0) &&
                      (g.cb.ext == 1 || (g.cb.stride * oes) % 16 == 0);
            if (!ok) return -1;
            CUtensorMap mc;
            make_map(&mc, base, o16, g.bn.ext, g.am.ext, g.cm.stride, g.ab.ext, g.cb.stride, o16 ? 64u : 32u,
                     uint32_t(kStoreRows));
            op.maps.push_back(mc);
            return int(op.maps.size()) - 1;
          };
          r.cmap32 = out_map(r.c32, false);
          r.cmap16 = out_map(r.c16, true);
          op.regions.push_back(r);
        }
        p.n_regions = int(op.regions.size());
        const double ab = double(g.am.ext) * g.ak.ext * g.ab.ext + double(g.bn.ext) * g.bk.ext * g.bb.ext;
        const double cbytes = double(g.am.ext) * g.bn.ext * g.ab.ext *
                              ((op.regions[0].c32 ? 4 : 0) + (op.regions[0].c16 ? 2 : 0));
        op.bytes = ab * (b16 ? 2 : 4) * total_sib + cbytes * p.n_regions;
        gemm_maps_total += op.maps.size();
        gemm_regions_total += op.regions.size();
        break;
      }
      case OpKind::GENERIC: {
        const Ex& u = X[id];
        const Vtx& w = V[u.producer];
        GenericParams& p = op.gen;
        std::memset(&p, 0, sizeof(p));
        shape lxy = local_xy(u.producer);
        std::map<int, int64_t> ext;
        for (size_t i = 0; i < w.lxy.size(); ++i) ext.emplace(w.lxy[i], lxy[i]);
        auto strides_of = [&](const labels& ls) {
          std::map<int, int64_t> st;
          int64_t s = 1;
          for (int i = int(ls.size()) - 1; i >= 0; --i) {
            st[ls[i]] = s;
            s *= ext.at(ls[i]);
          }
          return st;
        };
        auto xs = strides_of(w.lx);
        auto ys = w.arity == 2 ? strides_of(w.ly) : std::map<int, int64_t>{};
        auto get = [](const std::map<int, int64_t>& m, int l) {
          auto it = m.find(l);
          return it == m.end() ? int64_t(0) : it->second;
        };
        p.nz = int(w.lz.size());
        for (int i = 0; i < p.nz; ++i) {
          p.zext[i] = ext.at(w.lz[i]);
          p.xs_z[i] = get(xs, w.lz[i]);
          p.ys_z[i] = get(ys, w.lz[i]);
        }
        p.na = 0;
        for (auto l : w.dls)
          if (std::find(w.lz.begin(), w.lz.end(), l) == w.lz.end()) {
            p.aext[p.na] = ext.at(l);
            p.xs_a[p.na] = get(xs, l);
            p.ys_a[p.na] = get(ys, l);
            ++p.na;
          }
        p.join = w.join;
        p.map = w.map;
        p.agg = w.agg;
        p.c = w.c;
        p.x = buf[resolve(u.deps[0])].main;
        p.y = w.arity == 2 ? buf[resolve(u.deps[1])].main : nullptr;
        p.out = buf[id].main;
        p.out16 = buf[id].b16;
        p.n_out = u.sz;
        p.err = d_err;
        int64_t xin = prod(pick(lxy, positions(w.lx, w.lxy)));
        int64_t yin = w.arity == 2 ? prod(pick(lxy, positions(w.ly, w.lxy))) : 0;
        op.bytes = double(xin + yin + u.sz) * es;
        break;
      }
      case OpKind::REFINE: {
        const Ex& u = X[id];
        const Vtx& w = V[u.producer];
        RefineParams& p = op.ref;
        std::memset(&p, 0, sizeof(p));
        const shape& bound = w.bound;
        shape dc = region_partition(id);
        p.rank = int(bound.size());
        p.agg = w.arity == 0 ? -1 : w.agg;
        for (int i = 0; i < p.rank; ++i) {
          p.cext[i] = u.cb[i];
          p.c0[i] = u.key[i] * (bound[i] / dc[i]);
        }
        p.n_out = u.sz;
        size_t first = dep_off.at(id), n = 0;
        for (auto& s : srcs_) n += s.ref == id;
        p.deps = d_deps + first;
        p.n_deps = int(n);
        p.out = buf[id].main;
        p.out16 = buf[id].b16;
        op.bytes = double(u.sz) * (es + (p.out16 ? 2 : 0));
        double rd = 0;
        for (auto& s : srcs_)
          if (s.ref == id) {
            double vol = 1;
            for (int i = 0; i < p.rank; ++i)
              vol *= double(std::max<int64_t>(0, std::min(s.r0[i] + s.ext[i], p.c0[i] + p.cext[i]) -
                                                     std::max(s.r0[i], p.c0[i])));
            rd += vol;
          }
        op.bytes += rd * es;
        // fast path: group sources by region (siblings fold in dep order)
        op.groups.clear();
        op.max_rows = 0;
        bool fast = true;
        std::vector<std::pair<shape, std::vector<const void*>>> regions;
        std::vector<const SrcRec*> firsts;
        for (auto& sr : srcs_) {
          if (sr.ref != id) continue;
          auto it = std::find_if(regions.begin(), regions.end(), [&](auto& q) { return q.first == sr.r0; });
          if (it == regions.end()) {
            regions.push_back({sr.r0, {}});
            firsts.push_back(&sr);
            it = regions.end() - 1;
          }
          it->second.push_back(buf[sr.src].main);
        }
        const int V = int(16 / es);
        bool vec = true;
        for (size_t gi = 0; gi < regions.size() && fast; ++gi) {
          const SrcRec& f = *firsts[gi];
          if (int(regions[gi].second.size()) > kRectSrc) {
            fast = false;
            break;
          }
          RectGroup rg{};
          rg.n_src = int(regions[gi].second.size());
          for (int k = 0; k < rg.n_src; ++k) rg.src[k] = regions[gi].second[k];
          int64_t ss = 1, ds = 1;
          for (int i = p.rank - 1; i >= 0; --i) {
            rg.sstr[i] = ss;
            rg.dstr[i] = ds;
            ss *= f.ext[i];
            ds *= p.cext[i];
          }
          rg.src_off = rg.dst_off = 0;
          rg.rows = 1;
          for (int i = 0; i < p.rank; ++i) {
            int64_t lo = std::max(f.r0[i], p.c0[i]);
            int64_t hi = std::min(f.r0[i] + f.ext[i], p.c0[i] + p.cext[i]);
            rg.ext[i] = hi - lo;
            rg.src_off += (lo - f.r0[i]) * rg.sstr[i];
            rg.dst_off += (lo - p.c0[i]) * rg.dstr[i];
            if (i < p.rank - 1) rg.rows *= rg.ext[i];
          }
          if (std::any_of(rg.ext, rg.ext + p.rank, [](int64_t e) { return e <= 0; })) continue;
          vec = vec && rg.ext[p.rank - 1] % V == 0 && rg.src_off % V == 0 && rg.dst_off % V == 0 &&
                (p.rank == 1 || (f.ext[p.rank - 1] % V == 0 && p.cext[p.rank - 1] % V == 0));
          op.max_rows = std::max(op.max_rows, rg.rows);
          op.groups.push_back(rg);
        }
        if (fast && !op.groups.empty() && p.rank >= 1) {
          op.rect.rank = p.rank;
          op.rect.agg = p.agg;
          op.rect.vec = vec;
          const int64_t inner = op.groups[0].ext[p.rank - 1];
          // ~32 KiB of output per block
          op.rect.rows_per_block = int(std::max<int64_t>(1, (32768 / int64_t(es)) / std::max<int64_t>(1, inner)));
          op.rect.out = p.out;
          op.rect.out16 = p.out16;
          rect_total += op.groups.size();
        } else {
          op.groups.clear();
        }
        break;
      }
      case OpKind::SPLIT:
        op.gen.x = buf[id].main;
        op.gen.out = buf[id].lo;
        op.gen.n_out = X[id].sz;
        break;
      case OpKind::CORRUPT:
        op.dt = buf[id].main ? store : DT::BF16;
        op.ptr = buf[id].main ? buf[id].main : buf[id].b16;
        break;
      case OpKind::SEND:
        op.ptr = buf[resolve(id)].main;
        break;
      case OpKind::RECV:
        op.ptr = buf[id].main;
        break;
      case OpKind::CONVERT:
        op.gen.x = buf[id].main;
        op.gen.out16 = buf[id].b16;
        op.gen.n_out = X[id].sz;
        break;
      case OpKind::FLASH: {
        const Flash& f = flash_.at(X[id].producer);
        const GemmMap& gs = gmap_.at(f.t1);
        const GemmMap& go = gmap_.at(f.o);
        AttnLaunch& a = op.attn;
        a.H = int(gs.ab.ext);
        a.S = int(gs.am.ext);
        a.T = int(gs.bn.ext);
        a.D = int(gs.ak.ext);
        a.scale = f.scale;
        op.maps.clear();
        op.aregions.clear();
        for (auto& r : f.regions) {
          AttnRegion ar{};
          const void* q = buf[resolve(r[0])].b16;
          const void* k = f.ktiles[size_t(&r - f.regions.data())].tiled ? nullptr : buf[resolve(r[1])].b16;
          const void* v = f.vtiles[size_t(&r - f.regions.data())].tiled ? nullptr : buf[resolve(r[2])].b16;
          if (!q) throw ed_error(ED_ERR_PLAN, "attention operand buffer missing");
          CUtensorMap m;
          make_map(&m, q, true, gs.ak.ext, gs.am.ext, gs.am.stride, gs.ab.ext, gs.ab.stride, 64, 128);
          ar.q = int(op.maps.size());
          op.maps.push_back(m);
          const size_t ri = size_t(&r - f.regions.data());
          // K: {d, keys, h}; V: {d, keys, h} — from the pasted chunk, or from each
          // source region of the grid with that region's own strides
          auto kv_maps = [&](const KVTiles& t, const void* chunk, const Dim& dk, const Dim& keys, const Dim& hb,
                             const labels& lop, int keyl, int hl, AttnSrc& out) {
            out.base = int(op.maps.size());
            if (!t.tiled) {
              make_map(&m, chunk, true, dk.ext, keys.ext, keys.stride, hb.ext, hb.stride, 64, 128);
              op.maps.push_back(m);
              out.nd = 1;
              out.keys = int(keys.ext);
              out.dw = int(dk.ext);
              out.hoff = 0;
              return;
            }
            const int kd = int(std::find(lop.begin(), lop.end(), keyl) - lop.begin());
            const int hd = int(std::find(lop.begin(), lop.end(), hl) - lop.begin());
            shape st(3, 1);
            for (int i = 1; i >= 0; --i) st[i] = st[i + 1] * t.ext[i + 1];
            for (int o2 : t.owners) {
              const void* b = buf[o2].b16;
              if (!b) throw ed_error(ED_ERR_PLAN, "attention source buffer missing");
              make_map(&m, b, true, t.ext[2], t.ext[kd], st[kd], t.ext[hd], st[hd], 64, 128);
              op.maps.push_back(m);
            }
            out.nd = t.nd;
            out.keys = int(t.keys);
            out.dw = int(t.dw);
            out.hoff = int(t.hoff);
          };
          const labels& lk = gs.b_slot == 0 ? V[f.t1].lx : V[f.t1].ly;
          const labels& lv = go.b_slot == 0 ? V[f.o].lx : V[f.o].ly;
          kv_maps(f.ktiles[ri], k, gs.bk, gs.bn, gs.bb, lk, gs.Nc.empty() ? -1 : gs.Nc[0], gs.Bc.empty() ? -1 : gs.Bc[0],
                  ar.k);
          kv_maps(f.vtiles[ri], v, go.bn, go.bk, go.bb, lv, go.Kc.empty() ? -1 : go.Kc[0], go.Bc.empty() ? -1 : go.Bc[0],
                  ar.v);
          auto out_map = [&](void* base, bool o16) {
            const int oes = o16 ? 2 : 4;
            bool ok = base && (go.cm.ext == 1 || (go.cm.stride * oes) % 16 == 0) &&
                      (go.cb.ext == 1 || (go.cb.stride * oes) % 16 == 0);
            if (!ok) return -1;
            CUtensorMap mc;
            make_map(&mc, base, o16, go.bn.ext, go.am.ext, go.cm.stride, go.ab.ext, go.cb.stride, o16 ? 64u : 32u,
                     uint32_t(kStoreRows));
            op.maps.push_back(mc);
            return int(op.maps.size()) - 1;
          };
          ar.o32 = out_map(buf[r[3]].main, false);
          ar.o16 = out_map(buf[r[3]].b16, true);
          if ((buf[r[3]].main && ar.o32 < 0) || (buf[r[3]].b16 && ar.o16 < 0))
            throw ed_error(ED_ERR_UNSUPPORTED, "attention output not 16-byte aligned");
          op.aregions.push_back(ar);
        }
        a.n_regions = int(op.aregions.size());
        op.bytes = 0;
        for (auto& r : f.regions)
          op.bytes += double(X[r[0]].sz + X[r[1]].sz + X[r[2]].sz) * 2 + double(X[r[3]].sz) * (buf[r[3]].main ? 4 : 0) +
                      double(X[r[3]].sz) * (buf[r[3]].b16 ? 2 : 0);
        attn_maps_total += op.maps.size();
        attn_regions_total += op.aregions.size();
        break;
      }
      case OpKind::SOFTMAX: {
        const Softmax& sm = softmax_.at(X[id].producer);
        op.jptrs.clear();
        for (size_t k = 0; k < sm.pairs.size(); ++k) {
          const int yj = sm.pairs[k].first, xr = sm.pairs[k].second;
          JoinPtrs jp{};
          jp.x = buf[resolve(xr)].main;
          jp.y = sm.m_refs.empty() ? nullptr : buf[resolve(sm.m_refs[k])].main;
          jp.out = buf[yj].main;
          jp.out16 = buf[yj].b16;
          op.jptrs.push_back(jp);
          op.bytes += double(X[yj].sz) * (es + (jp.out ? es : 0) + (jp.out16 ? 2 : 0));
        }
        op.sm.rows = X[sm.pairs[0].first].sz / sm.len;
        op.sm.len = int(sm.len);
        op.rowsegs.clear();
        if (!sm.xsegs.empty()) {
          op.sm.n_seg = int(sm.xsegs[0].size());
          op.sm.seg_w = sm.seg_w;
          for (auto& v : sm.xsegs)
            for (auto& xs : v) op.rowsegs.push_back(RowSeg{static_cast<const float*>(buf[xs.owner].main), xs.row0, xs.stride});
          rowseg_total += op.rowsegs.size();
        }
        jptrs_total += op.jptrs.size();
        break;
      }
      case OpKind::EWISE:
      case OpKind::ROWREDUCE: {
        const Ex& u = X[id];
        const Vtx& w = V[u.producer];
        const MemMap& mm = memmap_.at(u.producer);
        op.jptrs.clear();
        double in_el = 0;
        shape lxy = local_xy(u.producer);
        int64_t xin = prod(pick(lxy, positions(w.lx, w.lxy)));
        int64_t yin = w.arity == 2 ? prod(pick(lxy, positions(w.ly, w.lxy))) : 0;
        for (int h : op.heads) {
          const Ex& j = X[h];
          JoinPtrs jp{};
          jp.x = buf[resolve(j.deps[0])].main;
          jp.y = w.arity == 2 ? buf[resolve(j.deps[1])].main : nullptr;
          jp.out = buf[h].main;
          jp.out16 = buf[h].b16;
          op.jptrs.push_back(jp);
          in_el += double(xin + yin);
          op.bytes += double(j.sz) * ((jp.out ? es : 0) + (jp.out16 ? 2 : 0));
        }
        op.bytes += in_el * es;
        if (mm.kind == OpKind::EWISE) {
          EwiseParams& p = op.ew;
          p.n = u.sz;
          p.binary = w.arity == 2;
          p.y_mode = mm.y_mode;
          p.inner = mm.inner;
          p.join = w.join;
          p.map = w.map;
          p.c = w.c;
          p.err = d_err;
        } else {
          RowReduceParams& p = op.rr;
          p.rows = mm.rows;
          p.len = mm.len;
          p.map = w.map;
          p.agg = w.agg;
          p.c = w.c;
        }
        jptrs_total += op.jptrs.size();
        break;
      }
    }
  }
  if (rowseg_total) {
    CUDA_OK(cudaMalloc(&d_rowsegs, sizeof(RowSeg) * rowseg_total));
    size_t o = 0;
    for (auto& op : ops) {
      if (op.rowsegs.empty()) continue;
      RowSeg* d = static_cast<RowSeg*>(d_rowsegs) + o;
      CUDA_OK(cudaMemcpy(d, op.rowsegs.data(), sizeof(RowSeg) * op.rowsegs.size(), cudaMemcpyHostToDevice));
      op.sm.segs = d;
      o += op.rowsegs.size();
    }
  }
  if (attn_maps_total) {
    CUDA_OK(cudaMalloc(&d_attn, sizeof(CUtensorMap) * attn_maps_total + sizeof(AttnRegion) * attn_regions_total));
    size_t mo = 0, ro = 0;
    CUtensorMap* maps = static_cast<CUtensorMap*>(d_attn);
    AttnRegion* regs = reinterpret_cast<AttnRegion*>(maps + attn_maps_total);
    for (auto& op : ops) {
      if (op.kind != OpKind::FLASH) continue;
      CUDA_OK(cudaMemcpy(maps + mo, op.maps.data(), sizeof(CUtensorMap) * op.maps.size(), cudaMemcpyHostToDevice));
      CUDA_OK(cudaMemcpy(regs + ro, op.aregions.data(), sizeof(AttnRegion) * op.aregions.size(),
                         cudaMemcpyHostToDevice));
      op.attn.maps = maps + mo;
      op.attn.regions = regs + ro;
      mo += op.maps.size();
      ro += op.aregions.size();
    }
  }
  if (rect_total) {
    CUDA_OK(cudaMalloc(&d_rects, sizeof(RectGroup) * rect_total));
    size_t o = 0;
    for (auto& op : ops) {
      if (op.groups.empty()) continue;
      RectGroup* d = static_cast<RectGroup*>(d_rects) + o;
      CUDA_OK(cudaMemcpy(d, op.groups.data(), sizeof(RectGroup) * op.groups.size(), cudaMemcpyHostToDevice));
      op.rect.groups = d;
      o += op.groups.size();
    }
  }
  if (jptrs_total) {
    CUDA_OK(cudaMalloc(&d_joinptrs, sizeof(JoinPtrs) * jptrs_total));
    size_t o = 0;
    for (auto& op : ops) {
      if (op.jptrs.empty()) continue;
      JoinPtrs* d = static_cast<JoinPtrs*>(d_joinptrs) + o;
      CUDA_OK(cudaMemcpy(d, op.jptrs.data(), sizeof(JoinPtrs) * op.jptrs.size(), cudaMemcpyHostToDevice));
      op.ew.joins = d;
      op.rr.joins = d;
      op.sm.joins = d;
      o += op.jptrs.size();
    }
  }
  // tensor maps and region tables of every GEMM launch, in device memory
  if (gemm_maps_total) {
    CUDA_OK(cudaMalloc(&d_maps, sizeof(CUtensorMap) * gemm_maps_total));
    CUDA_OK(cudaMalloc(&d_regions, sizeof(GemmRegion) * gemm_regions_total));
    size_t mo = 0, ro = 0;
    for (auto& op : ops) {
      if (op.kind != OpKind::GEMM) continue;
      CUtensorMap* dm = static_cast<CUtensorMap*>(d_maps) + mo;
      GemmRegion* dr = static_cast<GemmRegion*>(d_regions) + ro;
      CUDA_OK(cudaMemcpy(dm, op.maps.data(), sizeof(CUtensorMap) * op.maps.size(), cudaMemcpyHostToDevice));
      CUDA_OK(cudaMemcpy(dr, op.regions.data(), sizeof(GemmRegion) * op.regions.size(), cudaMemcpyHostToDevice));
      op.gemm.maps = dm;
      op.gemm.regions = dr;
      mo += op.maps.size();
      ro += op.regions.size();
    }
  }
  if (peer) {
    CUDA_OK(cudaMalloc(&d_epoch, sizeof(int)));
    CUDA_OK(cudaMemset(d_epoch, 0, sizeof(int)));
    CUDA_OK(cudaMalloc(&d_pflags, sizeof(int) * (X.size() + 2)));
    CUDA_OK(cudaMemset(d_pflags, 0, sizeof(int) * (X.size() + 2)));
    CUDA_OK(cudaMalloc(&d_perr, sizeof(int)));
    CUDA_OK(cudaMemset(d_perr, 0, sizeof(int)));
  }
}

void ed_plan_h::launch_op(size_t i, cudaStream_t s) {
  Op& op = ops[i];
  switch (op.kind) {
    case OpKind::GEMM: CUDA_OK(launch_gemm(op.gemm, ctx->num_sms, s)); break;
    case OpKind::GENERIC: CUDA_OK(launch_generic(op.gen, f64, s)); break;
    case OpKind::REFINE:
      if (!op.groups.empty()) CUDA_OK(launch_rect(op.rect, int(op.groups.size()), op.max_rows, f64, s));
      else CUDA_OK(launch_refine(op.ref, f64, s));
      break;
    case OpKind::CORRUPT: CUDA_OK(launch_add_one(op.ptr, op.dt, s)); break;
    case OpKind::EWISE:
      CUDA_OK(launch_ewise(op.ew, int(op.jptrs.size()), f64, opt.precision == ED_PREC_FP32, s));
      break;
    case OpKind::FLASH: CUDA_OK(launch_attn(op.attn, ctx->num_sms, s)); break;
    case OpKind::SPLIT:
      CUDA_OK(launch_split_lo(static_cast<const float*>(op.gen.x), static_cast<float*>(op.gen.out), op.gen.n_out, s));
      break;
    case OpKind::SOFTMAX: CUDA_OK(launch_softmax(op.sm, int(op.jptrs.size()), s)); break;
    case OpKind::ROWREDUCE:
      CUDA_OK(launch_rowreduce(op.rr, int(op.jptrs.size()), f64, opt.precision == ED_PREC_FP32, s));
      break;
    case OpKind::CONVERT: CUDA_OK(launch_convert(op.gen.x, store, op.gen.out16, DT::BF16, op.gen.n_out, s)); break;
    case OpKind::SEND:
      if (peer) CUDA_OK(launch_peer_signal(d_pflags + 2 + op.exec, d_epoch, s));  // chunk ready for the peer
      else NCCL_OK(ncclSend(op.ptr, op.count, f64 ? ncclFloat64 : ncclFloat32, op.peer, ctx->comm, s));
      break;
    case OpKind::RECV:
      if (peer) {
        int* f = peer_flags[size_t(op.peer)] + 2 + op.exec;
        CUDA_OK(launch_peer_wait(&f, 1, d_epoch, 0, s, d_perr, op.exec));
        const int64_t off = peer_off[size_t(op.peer)][size_t(op.exec)];
        if (off < 0) throw ed_error(ED_ERR_PLAN, "peer transport: chunk not resident on its producer rank");
        CUDA_OK(cudaMemcpyAsync(op.ptr, peer_arena[size_t(op.peer)] + off, op.count * es, cudaMemcpyDeviceToDevice, s));
      } else {
        NCCL_OK(ncclRecv(op.ptr, op.count, f64 ? ncclFloat64 : ncclFloat32, op.peer, ctx->comm, s));
      }
      break;
  }
}

// Every op in schedule order on the compute stream, except that each run of
// consecutive transfers goes to the comm stream as ONE NCCL group (the
// exchange of a repartition proceeds with all peers at once). The comm
// stream forks from the compute stream before every run (a send's operand
// is produced by then, and the fork keeps the comm stream inside the CUDA
// graph capture) and the compute stream joins it right after the run: transfers sit just before their data's first consumer, so
// the sender keeps computing while its sends drain and a receiver's recvs
// are posted as soon as the comm stream reaches them, ahead of its compute.
// Buffers are never reused within a run (linear arena), so an early recv
// cannot overwrite live data. Ranks enqueue the same transfers in the same
// global order (transfers_by_consumer), so the groups match.
void ed_plan_h::enqueue(cudaStream_t s) {
  cudaStream_t cs = ctx->comm_stream;
  size_t ev = 0;
  if (peer) {
    // new run: advance the epoch, then wait until every rank has finished its
    // previous run (its receives from our chunks are complete: write-after-read)
    CUDA_OK(launch_peer_tick(d_epoch, s));
    std::vector<int*> done(peer_flags.size());
    for (size_t r = 0; r < done.size(); ++r) done[r] = peer_flags[r];
    CUDA_OK(launch_peer_wait(done.data(), int(done.size()), d_epoch, -1, s, d_perr, int(X.size())));
  }
  auto next_event = [&]() {
    if (ev == comm_events.size()) {
      cudaEvent_t e;
      CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      comm_events.push_back(e);
    }
    return comm_events[ev++];
  };
  auto is_comm = [&](size_t i) { return ops[i].kind == OpKind::SEND || ops[i].kind == OpKind::RECV; };
  for (size_t i = 0; i < ops.size();) {
    // consecutive GEMMs of mutually independent einsums (e.g. attention's Q, K, V
    // projections) run as parallel branches: each persistent grid's last,
    // partial wave leaves SMs the next one fills
    size_t g = i;
    if (!opt.profile) {
      while (g < ops.size() && ops[g].kind == OpKind::GEMM && g - i < 3) {
        bool indep = true;
        for (size_t a = i; a < g && indep; ++a) indep = !ancestor(ops[a].einsum, ops[g].einsum);
        if (!indep) break;
        ++g;
      }
    }
    if (g - i >= 2) {
      cudaEvent_t fork = next_event();
      CUDA_OK(cudaEventRecord(fork, s));
      std::vector<cudaEvent_t> joins;
      for (size_t k = i + 1; k < g; ++k) {
        cudaStream_t a = aux[k - i - 1];
        if (!a) {
          CUDA_OK(cudaStreamCreateWithFlags(&aux[k - i - 1], cudaStreamNonBlocking));
          a = aux[k - i - 1];
        }
        CUDA_OK(cudaStreamWaitEvent(a, fork, 0));
        launch_op(k, a);
        joins.push_back(next_event());
        CUDA_OK(cudaEventRecord(joins.back(), a));
      }
      launch_op(i, s);
      for (cudaEvent_t e : joins) CUDA_OK(cudaStreamWaitEvent(s, e, 0));
      i = g;
      continue;
    }
    if (!is_comm(i)) {
      if (opt.profile) CUDA_OK(cudaEventRecord(op_events[i], s));
      launch_op(i, s);
      ++i;
      continue;
    }
    size_t j = i;
    while (j < ops.size() && is_comm(j)) ++j;
    if (opt.profile)
      for (size_t k = i; k < j; ++k) CUDA_OK(cudaEventRecord(op_events[k], s));
    {
      // every run forks from the compute stream: a send's chunk is produced by
      // then, and a receive must follow the run's start (epoch, graph capture)
      cudaEvent_t fork = next_event();
      CUDA_OK(cudaEventRecord(fork, s));
      CUDA_OK(cudaStreamWaitEvent(cs, fork, 0));
    }
    if (!peer) NCCL_OK(ncclGroupStart());
    for (size_t k = i; k < j; ++k) launch_op(k, cs);
    if (!peer) NCCL_OK(ncclGroupEnd());
    cudaEvent_t join = next_event();
    CUDA_OK(cudaEventRecord(join, cs));
    CUDA_OK(cudaStreamWaitEvent(s, join, 0));
    i = j;
  }
  if (opt.profile) CUDA_OK(cudaEventRecord(op_events[ops.size()], s));
  if (peer) CUDA_OK(launch_peer_signal(d_pflags, d_epoch, s));  // this run is done on this rank
}

void ed_plan_h::record() {
  CUDA_OK(gemm_prepare());
  CUDA_OK(attn_prepare());
  if (!ev0) CUDA_OK(cudaEventCreate(&ev0));
  if (!ev1) CUDA_OK(cudaEventCreate(&ev1));
  if (opt.no_graph || opt.profile || (peer && !peer_ready)) return;  // peer: recorded by ed_peer_import
  cudaStream_t s = ctx->stream;
  CUDA_OK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  try {
    enqueue(s);
  } catch (...) {
    cudaGraph_t g;
    cudaStreamEndCapture(s, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  CUDA_OK(cudaStreamEndCapture(s, &graph));
  CUDA_OK(cudaGraphInstantiate(&gexec, graph, 0));
}

void ed_plan_h::destroy() {
  if (gexec) cudaGraphExecDestroy(gexec);
  if (graph) cudaGraphDestroy(graph);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  for (auto e : op_events) cudaEventDestroy(e);
  for (auto e : comm_events) cudaEventDestroy(e);
  for (auto a : aux)
    if (a) cudaStreamDestroy(a);
  for (size_t r = 0; r < peer_arena.size(); ++r)
    if (int(r) != ctx->rank) {
      if (peer_arena[r]) cudaIpcCloseMemHandle(peer_arena[r]);
      if (peer_flags[r]) cudaIpcCloseMemHandle(peer_flags[r]);
    }
  if (d_epoch) cudaFree(d_epoch);
  if (d_perr) cudaFree(d_perr);
  if (d_pflags) cudaFree(d_pflags);
  if (arena) cudaFree(arena);
  if (d_deps) cudaFree(d_deps);
  if (d_maps) cudaFree(d_maps);
  if (d_joinptrs) cudaFree(d_joinptrs);
  if (d_rects) cudaFree(d_rects);
  if (d_copy_desc) cudaFree(d_copy_desc);
  if (d_attn) cudaFree(d_attn);
  if (d_rowsegs) cudaFree(d_rowsegs);
  if (d_regions) cudaFree(d_regions);
  if (d_ptrs) cudaFree(d_ptrs);
  if (d_err) cudaFree(d_err);
  if (staging) cudaFree(staging);
  for (auto& [k, c] : copy_cache)
    if (c.d) cudaFree(c.d);
  for (void* b : stg_in)
    if (b) cudaFree(b);
  for (void* b : stg_out)
    if (b) cudaFree(b);
  for (auto e : ev_pipe)
    if (e) cudaEventDestroy(e);
  if (cs_in) cudaStreamDestroy(cs_in);
  if (cs_out) cudaStreamDestroy(cs_out);
}

namespace {

void ensure_staging(ed_plan_h* h, size_t bytes) {
  if (h->staging_bytes >= bytes) return;
  if (h->staging) CUDA_OK(cudaFree(h->staging));
  h->staging = nullptr;
  CUDA_OK(cudaMalloc(&h->staging, bytes));
  h->staging_bytes = bytes;
}

size_t dt_size(int dtype) {
  if (dtype == ED_DTYPE_F64) return 8;
  if (dtype == ED_DTYPE_F32) return 4;
  throw ed_error(ED_ERR_USAGE, "unknown dtype");
}

DT dt_of(int dtype) { return dtype == ED_DTYPE_F64 ? DT::F64 : DT::F32; }

// chunk <-> whole-tensor rectangle copies (BlockCopy) for graph vertex w over
// partition `part`; to_chunks: whole (staging) -> chunk buffers, else back.
std::vector<BlockCopy> copy_groups(ed_plan_h* h, int w, const shape& part, const std::vector<int>& ids,
                                   bool to_chunks, const void* whole_src, void* whole_dst,
                                   const std::vector<void*>* remote, int64_t& max_rows) {
  const shape& bound = h->V[w].bound;
  const int rank = int(bound.size());
  if (rank == 0) throw ed_error(ED_ERR_UNSUPPORTED, "rank-0 tensors");
  shape cb(rank), ws(rank), cs(rank);
  for (int i = 0; i < rank; ++i) cb[i] = bound[i] / part[i];
  int64_t a = 1, b = 1;
  for (int i = rank - 1; i >= 0; --i) {
    ws[i] = a;
    cs[i] = b;
    a *= bound[i];
    b *= cb[i];
  }
  std::vector<BlockCopy> groups;
  max_rows = 1;
  for (size_t n = 0; n < ids.size(); ++n) {
    const int id = ids[n];
    void* chunk = (remote && (*remote)[n]) ? (*remote)[n] : (h->local[id] ? h->buf[h->owner[id]].main : nullptr);
    if (!chunk) continue;
    BlockCopy g{};
    int64_t woff = 0, rows = 1;
    for (int i = 0; i < rank; ++i) {
      woff += h->X[id].key[i] * cb[i] * ws[i];
      g.ext[i] = cb[i];
      if (i < rank - 1) rows *= cb[i];
    }
    g.rows = rows;
    max_rows = std::max(max_rows, rows);
    if (to_chunks) {
      g.src = whole_src;
      g.dst = chunk;
      g.dst16 = h->buf[h->owner[id]].b16;
      g.src_off = woff;
      g.dst_off = 0;
      for (int i = 0; i < rank; ++i) {
        g.sstr[i] = ws[i];
        g.dstr[i] = cs[i];
      }
    } else {
      g.src = chunk;
      g.dst = whole_dst;
      g.src_off = 0;
      g.dst_off = woff;
      for (int i = 0; i < rank; ++i) {
        g.sstr[i] = cs[i];
        g.dstr[i] = ws[i];
      }
    }
    groups.push_back(g);
  }
  return groups;
}

void block_copies(ed_plan_h* h, int w, const shape& part, const std::vector<int>& ids, bool to_chunks,
                  const void* whole_src, void* whole_dst, DT whole_dt, cudaStream_t s,
                  const std::vector<void*>* remote = nullptr) {
  int64_t max_rows = 1;
  const std::vector<BlockCopy> groups = copy_groups(h, w, part, ids, to_chunks, whole_src, whole_dst, remote, max_rows);
  const int rank = int(h->V[w].bound.size());
  if (groups.empty()) return;
  const size_t need = sizeof(BlockCopy) * groups.size();
  if (h->copy_desc_bytes < need) {
    if (h->d_copy_desc) CUDA_OK(cudaFree(h->d_copy_desc));
    CUDA_OK(cudaMalloc(&h->d_copy_desc, need));
    h->copy_desc_bytes = need;
  }
  CUDA_OK(cudaMemcpyAsync(h->d_copy_desc, groups.data(), need, cudaMemcpyHostToDevice, s));
  BlockCopyParams p{};
  p.rank = rank;
  p.in_dt = int(to_chunks ? whole_dt : h->store);
  p.out_dt = int(to_chunks ? h->store : whole_dt);
  p.groups = static_cast<const BlockCopy*>(h->d_copy_desc);
  CUDA_OK(launch_blockcopy(p, int(groups.size()), max_rows, s));
}

// chunk <-> whole-tensor mapping for graph vertex w over partition `part`
// and the exec ids holding its chunks (any order; keyed by their key).
void chunk_map(ed_plan_h* h, int w, const shape& part, const std::vector<int>& ids, bool want_shadow,
               ChunkMapParams& p, const std::vector<void*>* remote = nullptr) {
  const shape& bound = h->V[w].bound;
  std::memset(&p, 0, sizeof(p));
  p.rank = int(bound.size());
  p.n = prod(bound);
  int64_t nkeys = prod(part);
  std::vector<void*> ptrs(size_t(2 * nkeys), nullptr);
  for (int i = 0; i < p.rank; ++i) {
    p.bound[i] = bound[i];
    p.part[i] = part[i];
    p.cb[i] = bound[i] / part[i];
  }
  for (size_t n = 0; n < ids.size(); ++n) {
    const int id = ids[n];
    int64_t k = 0;
    for (int i = 0; i < p.rank; ++i) k = k * part[i] + h->X[id].key[i];
    if (remote && (*remote)[n]) {
      ptrs[size_t(k)] = (*remote)[n];
    } else if (h->local[id]) {
      ptrs[size_t(k)] = h->buf[h->owner[id]].main;
      if (want_shadow) ptrs[size_t(nkeys + k)] = h->buf[h->owner[id]].b16;
    }
  }
  if (size_t(2 * nkeys) > 2 * std::max<size_t>(1, h->X.size())) {
    CUDA_OK(cudaFree(h->d_ptrs));
    CUDA_OK(cudaMalloc(&h->d_ptrs, sizeof(void*) * 2 * nkeys));
  }
  CUDA_OK(cudaMemcpy(h->d_ptrs, ptrs.data(), sizeof(void*) * 2 * nkeys, cudaMemcpyHostToDevice));
  p.chunks = h->d_ptrs;
  p.shadows = want_shadow ? h->d_ptrs + nkeys : nullptr;
}

}  // namespace

extern "C" {

int32_t ed_abi_version(void) { return ED_ABI_VERSION; }

ed_status ed_nccl_unique_id(void* out, size_t len, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!out || len < sizeof(ncclUniqueId)) throw ed_error(ED_ERR_USAGE, "buffer too small for ncclUniqueId");
    ncclUniqueId id;
    NCCL_OK(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
  });
}

ed_status ed_ctx_create(int32_t device, int32_t rank, int32_t world, const void* nccl_id, size_t nccl_id_len,
                        ed_ctx** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!out || world < 1 || rank < 0 || rank >= world) throw ed_error(ED_ERR_USAGE, "bad rank/world");
    int n = 0;
    CUDA_OK(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw ed_error(ED_ERR_USAGE, "no such CUDA device");
    CUDA_OK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_OK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw ed_error(ED_ERR_UNSUPPORTED, "libed_gpu is built for sm_100a (B200)");
    auto* c = new ed_ctx;
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    c->rank = rank;
    c->world = world;
    try {
      CUDA_OK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      CUDA_OK(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
      if (world > 1 && nccl_id) {
        if (nccl_id_len < sizeof(ncclUniqueId)) throw ed_error(ED_ERR_USAGE, "NCCL id too short");
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        NCCL_OK(ncclCommInitRank(&c->comm, world, id, rank));
      }
    } catch (...) {
      ed_ctx_destroy(c);
      throw;
    }
    *out = c;
  });
}

void ed_ctx_destroy(ed_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  delete c;
}

ed_status ed_prepare(ed_ctx* ctx, const ed_plan_c* plan, const ed_options_c* options, ed_plan_h** out,
                     char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!ctx || !out) throw ed_error(ED_ERR_USAGE, "null context or output");
    CUDA_OK(cudaSetDevice(ctx->device));
    auto* h = new ed_plan_h;
    h->ctx = ctx;
    if (options) h->opt = *options;
    if (h->opt.precision < 0 || h->opt.precision > 4) {
      delete h;
      throw ed_error(ED_ERR_USAGE, "unknown precision");
    }
    h->peer = ctx->world > 1 && h->opt.transport == ED_TRANSPORT_PEER;
    if (ctx->world > 1 && !h->peer && !ctx->comm) {
      delete h;
      throw ed_error(ED_ERR_USAGE, "world > 1 without an NCCL communicator needs ED_TRANSPORT_PEER");
    }
    h->f64 = h->opt.precision == ED_PREC_FP64;
    h->store = h->f64 ? DT::F64 : DT::F32;
    h->es = h->f64 ? 8 : 4;
    try {
      h->copy_plan(plan);
      h->validate();
      h->build();
      h->allocate();
      h->record();
    } catch (...) {
      h->destroy();
      delete h;
      throw;
    }
    *out = h;
  });
}

void ed_plan_destroy(ed_plan_h* h) {
  if (!h) return;
  cudaSetDevice(h->ctx->device);
  h->destroy();
  delete h;
}

ed_status ed_upload(ed_plan_h* h, const ed_chunk_in_c* chunks, int32_t n, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h || (n && !chunks)) throw ed_error(ED_ERR_USAGE, "null argument");
    CUDA_OK(cudaSetDevice(h->ctx->device));
    cudaStream_t s = h->ctx->stream;
    for (int i = 0; i < n; ++i) {
      const ed_chunk_in_c& c = chunks[i];
      if (c.exec_id < 0 || c.exec_id >= int(h->X.size()) || h->X[c.exec_id].kind != ED_EXEC_INPUT_CHUNK)
        throw ed_error(ED_ERR_PLAN, "ed_upload: not an input chunk");
      if (c.n != h->X[c.exec_id].sz) throw ed_error(ED_ERR_PLAN, "ed_upload: chunk size mismatch");
      if (!h->local[c.exec_id]) continue;
      size_t bytes = size_t(c.n) * dt_size(c.dtype);
      ensure_staging(h, bytes);
      CUDA_OK(cudaMemcpyAsync(h->staging, c.data, bytes, cudaMemcpyHostToDevice, s));
      Buffer& b = h->buf[c.exec_id];
      CUDA_OK(launch_convert(h->staging, dt_of(c.dtype), b.main, h->store, c.n, s));
      if (b.b16) CUDA_OK(launch_convert(h->staging, dt_of(c.dtype), b.b16, DT::BF16, c.n, s));
      if (b.lo) CUDA_OK(launch_split_lo(static_cast<const float*>(b.main), static_cast<float*>(b.lo), c.n, s));
    }
    CUDA_OK(cudaStreamSynchronize(s));
  });
}

ed_status ed_upload_tensors(ed_plan_h* h, const ed_tensor_in_c* ts, int32_t n, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h || (n && !ts)) throw ed_error(ED_ERR_USAGE, "null argument");
    CUDA_OK(cudaSetDevice(h->ctx->device));
    cudaStream_t s = h->ctx->stream;
    for (int i = 0; i < n; ++i) {
      const ed_tensor_in_c& t = ts[i];
      if (t.vertex_id < 0 || t.vertex_id >= int(h->V.size()) || h->V[t.vertex_id].arity != 0)
        throw ed_error(ED_ERR_PLAN, "execute: no relation supplied for an input");
      if (t.n != prod(h->V[t.vertex_id].bound)) throw ed_error(ED_ERR_PLAN, "ed_upload_tensors: size mismatch");
      std::vector<int> ids;
      bool shadow = false;
      for (int id = 0; id < int(h->X.size()); ++id)
        if (h->X[id].kind == ED_EXEC_INPUT_CHUNK && h->X[id].producer == t.vertex_id) {
          ids.push_back(id);
          shadow = shadow || (h->local[id] && h->buf[id].b16);
        }
      size_t bytes = size_t(t.n) * dt_size(t.dtype);
      ensure_staging(h, bytes);
      CUDA_OK(cudaMemcpyAsync(h->staging, t.data, bytes, cudaMemcpyHostToDevice, s));
      (void)shadow;
      block_copies(h, t.vertex_id, h->V[t.vertex_id].d, ids, true, h->staging, nullptr, dt_of(t.dtype), s);
      for (int id : ids)
        if (h->local[id] && h->buf[id].lo)
          CUDA_OK(launch_split_lo(static_cast<const float*>(h->buf[id].main), static_cast<float*>(h->buf[id].lo),
                                  h->X[id].sz, s));
      CUDA_OK(cudaStreamSynchronize(s));
    }
  });
}

namespace {
std::vector<int> io_chunks(const ed_plan_h* h, int w, bool input);
}  // namespace

ed_status ed_generate_inputs(ed_plan_h* h, uint64_t seed, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h) throw ed_error(ED_ERR_USAGE, "null plan");
    CUDA_OK(cudaSetDevice(h->ctx->device));
    // uses_only_sum_mul (runtime.cc:358-378): generate_inputs' distribution switch
    bool integer_valued = true;
    for (const Vtx& v : h->V) {
      if (v.arity == 0) continue;
      if (v.join >= 0 && v.join != ED_JOIN_MUL && v.join != ED_JOIN_ADD) integer_valued = false;
      if (v.map >= 0 && v.map != ED_MAP_IDENTITY && v.map != ED_MAP_RELU && v.map != ED_MAP_NEG) integer_valued = false;
      if (v.agg >= 0 && v.agg != ED_AGG_SUM && v.agg != ED_AGG_MAX) integer_valued = false;
    }
    cudaStream_t s = h->ctx->stream;
    std::vector<GenTensor> jobs;
    std::vector<int> vids;
    for (int w = 0; w < int(h->V.size()); ++w) {
      if (h->V[w].arity != 0) continue;
      bool any_local = false;
      for (int id : io_chunks(h, w, true)) any_local = any_local || h->local[id];
      if (!any_local) continue;  // a rank only materialises the inputs it holds chunks of
      GenTensor g{};
      g.n = prod(h->V[w].bound);
      g.seed = seed * 7919ULL + uint64_t(w);
      CUDA_OK(cudaMallocAsync(&g.out, size_t(g.n) * h->es, s));
      jobs.push_back(g);
      vids.push_back(w);
    }
    if (jobs.empty()) return;
    GenTensor* d_jobs = nullptr;
    int* d_flag = nullptr;
    CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&d_jobs), sizeof(GenTensor) * jobs.size(), s));
    CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&d_flag), sizeof(int), s));
    CUDA_OK(cudaMemsetAsync(d_flag, 0, sizeof(int), s));
    CUDA_OK(cudaMemcpyAsync(d_jobs, jobs.data(), sizeof(GenTensor) * jobs.size(), cudaMemcpyHostToDevice, s));
    CUDA_OK(launch_generate(d_jobs, int(jobs.size()), integer_valued, h->store, d_flag, s));
    // chunk() (relation.cc:31-53) into this rank's input chunks (+ bf16 / lo shadows)
    for (size_t k = 0; k < jobs.size(); ++k) {
      const std::vector<int> ids = io_chunks(h, vids[k], true);
      block_copies(h, vids[k], h->V[vids[k]].d, ids, true, jobs[k].out, nullptr, h->store, s);
      for (int id : ids)
        if (h->local[id] && h->buf[id].lo)
          CUDA_OK(launch_split_lo(static_cast<const float*>(h->buf[id].main), static_cast<float*>(h->buf[id].lo),
                                  h->X[id].sz, s));
      CUDA_OK(cudaStreamSynchronize(s));  // block_copies' descriptor buffer is reused per tensor
    }
    int flag = 0;
    CUDA_OK(cudaMemcpyAsync(&flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    for (auto& g : jobs) CUDA_OK(cudaFreeAsync(g.out, s));
    CUDA_OK(cudaFreeAsync(d_jobs, s));
    CUDA_OK(cudaFreeAsync(d_flag, s));
    CUDA_OK(cudaStreamSynchronize(s));
    if (flag)
      throw ed_error(ED_ERR_UNSUPPORTED,
                     "generate_inputs: a rejected integer draw (p = 7/2^64) shifted the stream; generate on the host");
  });
}

ed_status ed_run(ed_plan_h* h, ed_report_c* rep, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h) throw ed_error(ED_ERR_USAGE, "null plan");
    if (h->peer && !h->peer_ready) throw ed_error(ED_ERR_USAGE, "ED_TRANSPORT_PEER: call ed_peer_import first");
    CUDA_OK(cudaSetDevice(h->ctx->device));
    cudaStream_t s = h->ctx->stream;
    CUDA_OK(cudaMemsetAsync(h->d_err, 0, sizeof(int), s));
    if (h->opt.profile && h->op_events.size() != h->ops.size() + 1) {
      for (auto e : h->op_events) cudaEventDestroy(e);
      h->op_events.assign(h->ops.size() + 1, nullptr);
      for (auto& e : h->op_events) CUDA_OK(cudaEventCreate(&e));
    }
    CUDA_OK(cudaEventRecord(h->ev0, s));
    if (h->gexec) CUDA_OK(cudaGraphLaunch(h->gexec, s));
    else h->enqueue(s);
    CUDA_OK(cudaEventRecord(h->ev1, s));
    CUDA_OK(cudaEventSynchronize(h->ev1));
    h->check_peer_error();
    int flag = 0;
    CUDA_OK(cudaMemcpy(&flag, h->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    float ms = 0;
    CUDA_OK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    if (h->opt.profile) {
      std::map<std::string, size_t> idx;
      h->stats.clear();
      for (size_t i = 0; i < h->ops.size(); ++i) {
        float t = 0;
        CUDA_OK(cudaEventElapsedTime(&t, h->op_events[i], h->op_events[i + 1]));
        const Op& op = h->ops[i];
        auto it = idx.find(op.name);
        if (it == idx.end()) {
          ed_kernel_stat_c st{};
          std::snprintf(st.name, sizeof(st.name), "%s", op.name.c_str());
          it = idx.emplace(op.name, h->stats.size()).first;
          h->stats.push_back(st);
        }
        auto& st = h->stats[it->second];
        st.launches += 1;
        st.ms += t;
        st.flops += op.flops;
        st.bytes += op.bytes;
      }
    }
    if (flag) throw ed_error(ED_ERR_EVAL, "division by zero");
    if (rep) {
      if (rep->machines)
        for (int m = 0; m < std::min(rep->n_machines, h->n_machines); ++m) rep->machines[m] = h->counters[m];
      rep->total_transferred = h->total_transferred;
      rep->wall_steps = int64_t(h->X.size());
      rep->max_site_cost = h->max_site_cost;
      rep->device_ms = ms;
      int64_t pb = 0;
      int launches = 0;
      for (auto& op : h->ops) {
        if (op.kind == OpKind::SEND) pb += int64_t(op.count) * int64_t(h->es);
        if (op.kind != OpKind::SEND && op.kind != OpKind::RECV) ++launches;
      }
      rep->peer_bytes = pb;
      rep->contraction_flops = h->contraction_flops;
      rep->gpu_launches = launches;
    }
  });
}

ed_status ed_download(ed_plan_h* h, ed_output_c* outs, int32_t n, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h || (n && !outs)) throw ed_error(ED_ERR_USAGE, "null argument");
    CUDA_OK(cudaSetDevice(h->ctx->device));
    cudaStream_t s = h->ctx->stream;
    const int me = h->ctx->rank, world = h->ctx->world;
    for (int i = 0; i < n; ++i) {
      int w = outs[i].vertex_id;
      if (w < 0 || w >= int(h->V.size())) throw ed_error(ED_ERR_USAGE, "output vertex out of range");
      if (outs[i].n != prod(h->V[w].bound)) throw ed_error(ED_ERR_USAGE, "output size mismatch");
      std::vector<int> ids;
      for (int id = 0; id < int(h->X.size()); ++id) {
        const Ex& u = h->X[id];
        bool mine = h->V[w].arity == 0 ? (u.kind == ED_EXEC_INPUT_CHUNK && u.producer == w)
                                        : (u.kind == ED_EXEC_REFINEMENT && u.producer == w && u.consumer < 0);
        if (mine) ids.push_back(id);
      }
      if (ids.empty()) throw ed_error(ED_ERR_PLAN, "no final refinement layer for output");
      // world > 1: every rank calls; chunks held elsewhere travel to rank 0
      std::vector<void*> remote(ids.size(), nullptr);
      if (world > 1 && h->peer) {
        if (me != 0) continue;  // rank 0 reads our chunks; we wait for it below
        // once every rank has finished the run, copy its chunks out of its HBM
        std::vector<int*> done(h->peer_flags.begin(), h->peer_flags.end());
        CUDA_OK(launch_peer_wait(done.data(), int(done.size()), h->d_epoch, 0, s, h->d_perr, int(h->X.size()) + 1));
        for (size_t k = 0; k < ids.size(); ++k) {
          const int id = ids[k], src = h->rank_of(id);
          if (src == 0) continue;
          const int64_t off = h->peer_off[size_t(src)][size_t(id)];
          if (off < 0) throw ed_error(ED_ERR_PLAN, "peer transport: output chunk not resident on its rank");
          CUDA_OK(cudaMallocAsync(&remote[k], size_t(h->X[id].sz) * h->es, s));
          CUDA_OK(cudaMemcpyAsync(remote[k], h->peer_arena[size_t(src)] + off, size_t(h->X[id].sz) * h->es,
                                  cudaMemcpyDeviceToDevice, s));
        }
      } else if (world > 1) {
        NCCL_OK(ncclGroupStart());
        for (size_t k = 0; k < ids.size(); ++k) {
          int id = ids[k], src = h->rank_of(id);
          if (src == 0) continue;
          if (me == src)
            NCCL_OK(ncclSend(h->main_of(id), size_t(h->X[id].sz), h->f64 ? ncclFloat64 : ncclFloat32, 0,
                             h->ctx->comm, s));
          if (me == 0) {
            CUDA_OK(cudaMallocAsync(&remote[k], size_t(h->X[id].sz) * h->es, s));
            NCCL_OK(ncclRecv(remote[k], size_t(h->X[id].sz), h->f64 ? ncclFloat64 : ncclFloat32, src,
                             h->ctx->comm, s));
          }
        }
        NCCL_OK(ncclGroupEnd());
        if (me != 0) {
          CUDA_OK(cudaStreamSynchronize(s));
          continue;
        }
      }
      shape part = h->V[w].arity == 0 ? h->V[w].d : h->out_partition(w);
      size_t bytes = size_t(outs[i].n) * dt_size(outs[i].dtype);
      ensure_staging(h, bytes);
      block_copies(h, w, part, ids, false, nullptr, h->staging, dt_of(outs[i].dtype), s, &remote);
      CUDA_OK(cudaMemcpyAsync(outs[i].data, h->staging, bytes, cudaMemcpyDeviceToHost, s));
      for (void* r : remote)
        if (r) CUDA_OK(cudaFreeAsync(r, s));
      CUDA_OK(cudaStreamSynchronize(s));
    }
    if (world > 1 && h->peer) {
      // rank 0 has copied every remote output chunk once its flag [1] carries
      // this run's epoch; until then the other ranks must not start a new run
      if (me == 0) CUDA_OK(launch_peer_signal(h->d_pflags + 1, h->d_epoch, s));
      else {
        int* f = h->peer_flags[0] + 1;
        CUDA_OK(launch_peer_wait(&f, 1, h->d_epoch, 0, s, h->d_perr, int(h->X.size()) + 2));
      }
      CUDA_OK(cudaStreamSynchronize(s));
      h->check_peer_error();
    }
  });
}

namespace {

// exec ids holding graph vertex w's chunks for upload (input chunks) or
// download (its final refinement layer), runtime.cc:432-448
std::vector<int> io_chunks(const ed_plan_h* h, int w, bool input) {
  std::vector<int> ids;
  for (int id = 0; id < int(h->X.size()); ++id) {
    const Ex& u = h->X[id];
    const bool mine = input ? (u.kind == ED_EXEC_INPUT_CHUNK && u.producer == w)
                            : (h->V[w].arity == 0 ? (u.kind == ED_EXEC_INPUT_CHUNK && u.producer == w)
                                                  : (u.kind == ED_EXEC_REFINEMENT && u.producer == w && u.consumer < 0));
    if (mine) ids.push_back(id);
  }
  return ids;
}

// whole tensor <-> chunks through a staging buffer with descriptors built
// once and kept on the device (no host->device copy inside the pipeline)
void cached_copy(ed_plan_h* h, int w, bool to_chunks, void* whole, int dtype, cudaStream_t s) {
  const auto key = std::make_tuple(w, int(to_chunks), static_cast<const void*>(whole), dtype);
  auto it = h->copy_cache.find(key);
  if (it == h->copy_cache.end()) {
    ed_plan_h::CopyPlan c;
    const shape part = (h->V[w].arity == 0 || to_chunks) ? h->V[w].d : h->out_partition(w);
    const std::vector<int> ids = io_chunks(h, w, to_chunks);
    const std::vector<BlockCopy> g =
        copy_groups(h, w, part, ids, to_chunks, to_chunks ? whole : nullptr, to_chunks ? nullptr : whole, nullptr,
                    c.max_rows);
    c.n = int(g.size());
    c.rank = int(h->V[w].bound.size());
    if (c.n) {
      CUDA_OK(cudaMalloc(&c.d, sizeof(BlockCopy) * g.size()));
      CUDA_OK(cudaMemcpy(c.d, g.data(), sizeof(BlockCopy) * g.size(), cudaMemcpyHostToDevice));
    }
    it = h->copy_cache.emplace(key, c).first;
  }
  const ed_plan_h::CopyPlan& c = it->second;
  if (!c.n) return;
  BlockCopyParams p{};
  p.rank = c.rank;
  p.in_dt = int(to_chunks ? dt_of(dtype) : h->store);
  p.out_dt = int(to_chunks ? h->store : dt_of(dtype));
  p.groups = static_cast<const BlockCopy*>(c.d);
  CUDA_OK(launch_blockcopy(p, c.n, c.max_rows, s));
}

void throw_status(ed_status st, const char* msg) {
  if (st != ED_OK) throw ed_error(st, msg);
}

}  // namespace

ed_status ed_run_steps(ed_plan_h* h, int32_t n_steps, const ed_tensor_in_c* ins, int32_t n_in, ed_output_c* outs,
                       int32_t n_out, ed_report_c* rep, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h || n_steps < 0 || n_in < 0 || n_out < 0 || (n_in && !ins) || (n_out && !outs))
      throw ed_error(ED_ERR_USAGE, "null argument");
    if (h->ctx->world > 1) {  // collective download: the plain sequence, step by step
      char e2[512];
      for (int st = 0; st < n_steps; ++st) {
        throw_status(ed_upload_tensors(h, ins + size_t(st) * n_in, n_in, e2, sizeof e2), e2);
        throw_status(ed_run(h, rep, e2, sizeof e2), e2);
        throw_status(ed_download(h, outs + size_t(st) * n_out, n_out, e2, sizeof e2), e2);
      }
      return;
    }
    CUDA_OK(cudaSetDevice(h->ctx->device));
    size_t in_b = 0, out_b = 0;
    for (int64_t i = 0; i < int64_t(n_steps) * n_in; ++i) {
      const ed_tensor_in_c& t = ins[i];
      if (t.vertex_id < 0 || t.vertex_id >= int(h->V.size()) || h->V[t.vertex_id].arity != 0)
        throw ed_error(ED_ERR_PLAN, "execute: no relation supplied for an input");
      if (t.n != prod(h->V[t.vertex_id].bound)) throw ed_error(ED_ERR_PLAN, "ed_run_steps: input size mismatch");
      in_b = std::max(in_b, size_t(t.n) * dt_size(t.dtype));
    }
    for (int64_t i = 0; i < int64_t(n_steps) * n_out; ++i) {
      const ed_output_c& o = outs[i];
      if (o.vertex_id < 0 || o.vertex_id >= int(h->V.size())) throw ed_error(ED_ERR_USAGE, "output vertex out of range");
      if (o.n != prod(h->V[o.vertex_id].bound)) throw ed_error(ED_ERR_USAGE, "output size mismatch");
      if (io_chunks(h, o.vertex_id, false).empty()) throw ed_error(ED_ERR_PLAN, "no final refinement layer for output");
      out_b = std::max(out_b, size_t(o.n) * dt_size(o.dtype));
    }
    if (!h->cs_in) {
      CUDA_OK(cudaStreamCreateWithFlags(&h->cs_in, cudaStreamNonBlocking));
      CUDA_OK(cudaStreamCreateWithFlags(&h->cs_out, cudaStreamNonBlocking));
      for (auto& e : h->ev_pipe) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    auto grow = [&](void* (&b)[2], size_t& have, size_t need) {
      if (have >= need) return;
      CUDA_OK(cudaDeviceSynchronize());
      for (void*& x : b) {
        if (x) CUDA_OK(cudaFree(x));
        CUDA_OK(cudaMalloc(&x, need));
      }
      have = need;
      // descriptors point into the old buffers
      for (auto& [k, c] : h->copy_cache)
        if (c.d) cudaFree(c.d);
      h->copy_cache.clear();
    };
    grow(h->stg_in, h->stg_in_bytes, in_b);
    grow(h->stg_out, h->stg_out_bytes, out_b);
    cudaEvent_t* in_full = h->ev_pipe;
    cudaEvent_t* in_free = h->ev_pipe + 2;
    cudaEvent_t* out_full = h->ev_pipe + 4;
    cudaEvent_t* out_free = h->ev_pipe + 6;
    cudaStream_t s = h->ctx->stream;
    CUDA_OK(cudaMemsetAsync(h->d_err, 0, sizeof(int), s));
    CUDA_OK(cudaEventRecord(h->ev0, s));
    int bi = 0, bo = 0;
    for (int st = 0; st < n_steps; ++st) {
      // inputs: H2D on the copy-in stream, chunk() on the compute stream
      // (after the previous step's run has read the input chunks)
      for (int k = 0; k < n_in; ++k) {
        const ed_tensor_in_c& t = ins[size_t(st) * n_in + k];
        const int b = bi++ & 1;
        const size_t bytes = size_t(t.n) * dt_size(t.dtype);
        CUDA_OK(cudaStreamWaitEvent(h->cs_in, in_free[b], 0));
        CUDA_OK(cudaMemcpyAsync(h->stg_in[b], t.data, bytes, cudaMemcpyHostToDevice, h->cs_in));
        CUDA_OK(cudaEventRecord(in_full[b], h->cs_in));
        CUDA_OK(cudaStreamWaitEvent(s, in_full[b], 0));
        cached_copy(h, t.vertex_id, true, h->stg_in[b], t.dtype, s);
        for (int id : io_chunks(h, t.vertex_id, true))
          if (h->local[id] && h->buf[id].lo)
            CUDA_OK(launch_split_lo(static_cast<const float*>(h->buf[id].main), static_cast<float*>(h->buf[id].lo),
                                    h->X[id].sz, s));
        CUDA_OK(cudaEventRecord(in_free[b], s));
      }
      if (h->gexec) CUDA_OK(cudaGraphLaunch(h->gexec, s));
      else h->enqueue(s);
      // outputs: assemble on the compute stream, D2H on the copy-out stream,
      // overlapping the next step's uploads
      for (int k = 0; k < n_out; ++k) {
        const ed_output_c& o = outs[size_t(st) * n_out + k];
        const int b = bo++ & 1;
        CUDA_OK(cudaStreamWaitEvent(s, out_free[b], 0));
        cached_copy(h, o.vertex_id, false, h->stg_out[b], o.dtype, s);
        CUDA_OK(cudaEventRecord(out_full[b], s));
        CUDA_OK(cudaStreamWaitEvent(h->cs_out, out_full[b], 0));
        CUDA_OK(cudaMemcpyAsync(o.data, h->stg_out[b], size_t(o.n) * dt_size(o.dtype), cudaMemcpyDeviceToHost,
                                h->cs_out));
        CUDA_OK(cudaEventRecord(out_free[b], h->cs_out));
      }
    }
    CUDA_OK(cudaEventRecord(h->ev1, s));
    CUDA_OK(cudaStreamSynchronize(h->cs_out));
    CUDA_OK(cudaStreamSynchronize(s));
    CUDA_OK(cudaStreamSynchronize(h->cs_in));
    int flag = 0;
    CUDA_OK(cudaMemcpy(&flag, h->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (flag) throw ed_error(ED_ERR_EVAL, "division by zero");
    if (rep) {
      if (rep->machines)
        for (int m = 0; m < std::min(rep->n_machines, h->n_machines); ++m) rep->machines[m] = h->counters[m];
      rep->total_transferred = h->total_transferred;
      rep->wall_steps = int64_t(h->X.size());
      rep->max_site_cost = h->max_site_cost;
      float ms = 0;
      CUDA_OK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
      rep->device_ms = ms;
      rep->peer_bytes = 0;
      rep->contraction_flops = h->contraction_flops;
      int launches = 0;
      for (auto& op : h->ops)
        if (op.kind != OpKind::SEND && op.kind != OpKind::RECV) ++launches;
      rep->gpu_launches = launches;
    }
  });
}

ed_status ed_download_chunk(ed_plan_h* h, int32_t exec_id, int32_t dtype, void* data, int64_t n, char* err,
                            size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h || !data) throw ed_error(ED_ERR_USAGE, "null argument");
    if (exec_id < 0 || exec_id >= int(h->X.size())) throw ed_error(ED_ERR_USAGE, "exec id out of range");
    if (n != h->X[exec_id].sz) throw ed_error(ED_ERR_USAGE, "chunk size mismatch");
    if (!h->local[exec_id]) throw ed_error(ED_ERR_USAGE, "chunk not resident on this rank");
    const Ex& u = h->X[exec_id];
    int o = h->owner[exec_id];
    if (u.kind == ED_EXEC_JOIN && o != exec_id && h->X[o].producer == u.producer)
      throw ed_error(ED_ERR_USAGE, "join partial was folded into its region's accumulator");
    if (h->opaque_[exec_id]) throw ed_error(ED_ERR_USAGE, "chunk was fused into its consumer's kernel");
    CUDA_OK(cudaSetDevice(h->ctx->device));
    cudaStream_t s = h->ctx->stream;
    size_t bytes = size_t(n) * dt_size(dtype);
    ensure_staging(h, bytes);
    const Buffer& b = h->buf[o];
    if (!b.main && !b.b16) throw ed_error(ED_ERR_USAGE, "chunk was fused into a consumer kernel and never materialised");
    if (b.main) CUDA_OK(launch_convert(b.main, h->store, h->staging, dt_of(dtype), n, s));
    else CUDA_OK(launch_convert(b.b16, DT::BF16, h->staging, dt_of(dtype), n, s));
    CUDA_OK(cudaMemcpyAsync(data, h->staging, bytes, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
  });
}

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
// region's exec vertices share a GPU (runtime.cu, prepare: epilogue map, row
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

namespace {

struct PeerBlobHead {
  int32_t magic, rank, world, n_exec;
  cudaIpcMemHandle_t arena, flags;
};
constexpr int32_t kPeerMagic = 0x45445031;  // "EDP1"

size_t peer_blob_len(const ed_plan_h* h) { return sizeof(PeerBlobHead) + sizeof(int64_t) * h->X.size(); }

}  // namespace

ed_status ed_peer_export(ed_plan_h* h, void* out, size_t cap, size_t* len, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h || !len) throw ed_error(ED_ERR_USAGE, "null argument");
    if (!h->peer) throw ed_error(ED_ERR_USAGE, "plan was not prepared with ED_TRANSPORT_PEER in a world > 1");
    *len = peer_blob_len(h);
    if (!out) return;
    if (cap < *len) throw ed_error(ED_ERR_USAGE, "ed_peer_export: buffer too small");
    CUDA_OK(cudaSetDevice(h->ctx->device));
    PeerBlobHead hd{};
    hd.magic = kPeerMagic;
    hd.rank = h->ctx->rank;
    hd.world = h->ctx->world;
    hd.n_exec = int32_t(h->X.size());
    CUDA_OK(cudaIpcGetMemHandle(&hd.arena, h->arena));
    CUDA_OK(cudaIpcGetMemHandle(&hd.flags, h->d_pflags));
    std::memcpy(out, &hd, sizeof hd);
    auto* off = reinterpret_cast<int64_t*>(static_cast<char*>(out) + sizeof hd);
    for (int id = 0; id < int(h->X.size()); ++id) off[id] = h->local[id] ? h->arena_offset(id) : -1;
  });
}

ed_status ed_peer_import(ed_plan_h* h, const void* blobs, size_t blob_len, int32_t n, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h || !blobs) throw ed_error(ED_ERR_USAGE, "null argument");
    if (!h->peer) throw ed_error(ED_ERR_USAGE, "plan was not prepared with ED_TRANSPORT_PEER in a world > 1");
    if (h->peer_ready) throw ed_error(ED_ERR_USAGE, "ed_peer_import: already imported");
    if (n != h->ctx->world || blob_len != peer_blob_len(h)) throw ed_error(ED_ERR_USAGE, "ed_peer_import: need one blob per rank");
    CUDA_OK(cudaSetDevice(h->ctx->device));
    const int world = h->ctx->world, me = h->ctx->rank;
    h->peer_arena.assign(size_t(world), nullptr);
    h->peer_flags.assign(size_t(world), nullptr);
    h->peer_off.assign(size_t(world), {});
    for (int r = 0; r < world; ++r) {
      const char* b = static_cast<const char*>(blobs) + size_t(r) * blob_len;
      PeerBlobHead hd;
      std::memcpy(&hd, b, sizeof hd);
      if (hd.magic != kPeerMagic || hd.rank != r || hd.world != world || hd.n_exec != int32_t(h->X.size()))
        throw ed_error(ED_ERR_USAGE, "ed_peer_import: blob " + std::to_string(r) + " does not belong to this plan");
      h->peer_off[size_t(r)].resize(h->X.size());
      std::memcpy(h->peer_off[size_t(r)].data(), b + sizeof hd, sizeof(int64_t) * h->X.size());
      if (r == me) {
        h->peer_arena[size_t(r)] = static_cast<char*>(h->arena);
        h->peer_flags[size_t(r)] = h->d_pflags;
        continue;
      }
      void* a = nullptr;
      void* f = nullptr;
      CUDA_OK(cudaIpcOpenMemHandle(&a, hd.arena, cudaIpcMemLazyEnablePeerAccess));
      CUDA_OK(cudaIpcOpenMemHandle(&f, hd.flags, cudaIpcMemLazyEnablePeerAccess));
      h->peer_arena[size_t(r)] = static_cast<char*>(a);
      h->peer_flags[size_t(r)] = static_cast<int*>(f);
    }
    h->peer_ready = true;
    h->record();
  });
}

ed_status ed_kernel_stats(ed_plan_h* h, ed_kernel_stat_c* out, int32_t cap, int32_t* n_out, char* err,
                          size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h || !n_out) throw ed_error(ED_ERR_USAGE, "null argument");
    int k = std::min<int>(cap, int(h->stats.size()));
    for (int i = 0; i < k; ++i) out[i] = h->stats[i];
    *n_out = int(h->stats.size());
  });
}

}  // extern "C"
