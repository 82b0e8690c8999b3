// Internal header of libed_gpu's host runtime (not part of the C ABI).
//
// The runtime replaces execute() (runtime.cc:382-451). Its translation units:
//   plan.cu       deep copy of the plan, execute()'s structural checks and the
//                 transfer accounting (runtime.cc:96-172, 388-395), schedules
//   build.cu      label -> kernel mapping and cross-vertex fusion: which launch
//                 runs every exec vertex of this rank
//   alloc.cu      the chunk arena, tensor maps and launch descriptors in HBM
//   exec.cu       launches, the per-run stream schedule (CUDA graph), ed_run
//   io.cu         uploads, device input generation, downloads, ed_run_steps
//   api.cu        contexts, ed_prepare, the peer transport's bootstrap
//   placement.cu  GPU-aware re-placement (ed_gpu_placement, host-only)
#pragma once
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

namespace edrt {


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


inline void set_err(char* err, size_t errlen, const std::string& m) {
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

inline int64_t prod(const shape& s) {
  int64_t r = 1;
  for (auto x : s) r *= x;
  return r;
}

inline std::vector<int> positions(const labels& l1, const labels& l2) {
  std::vector<int> r;
  for (auto l : l1) {
    auto it = std::find(l2.begin(), l2.end(), l);
    if (it == l2.end()) throw ed_error(ED_ERR_PLAN, "unknown label in projection");
    r.push_back(int(it - l2.begin()));
  }
  return r;
}

inline shape pick(const shape& b, const std::vector<int>& pos) {
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
bool merge_dim(const labels& tl, const shape& text, const labels& cls, Dim& out, labels& order);

struct GemmMap {
  int a_slot, b_slot;  // which einsum input feeds MMA-A / MMA-B
  Dim am, ak, ab, bn, bk, bb, cm, cn, cb;
  bool a_mn, b_mn;
  labels lA, lB, Mc, Nc, Kc, Bc;  // operand label lists and the label classes
};

bool map_gemm(const Vtx& v, const shape& local_xy, bool bf16, GemmMap& g, std::string& why);

// 3-D tensor map {inner, outer, batch} with a 128-byte swizzled box.
void make_map(CUtensorMap* m, const void* base, bool bf16, int64_t inner, int64_t outer, int64_t outer_stride,
              int64_t batch, int64_t batch_stride, uint32_t box_inner, uint32_t box_outer,
              CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B);

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
  bool direct = false;  // RECV: no copy, readers use the producer's chunk (bind_direct)
  std::vector<int> writes;  // exec ids whose data this op writes (the peer transport's early ready signals)
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

bool map_memory(const Vtx& v, const shape& local_xy, bool f64, MemMap& m);

// F32X3: producers (x3 GEMM epilogue, softmax, refinement folds) write the lo
// shadow x - tf32(x) of a chunk a later contraction reads; ED_X3_LO_EPI=0
// falls back to a separate split launch before the consumer (A/B experiments)
// F32X3: the attention block runs fused (attn_x3_sm100.cu); ED_ATTN_X3=0 keeps
// it as three einsums through HBM (A/B experiments)
inline bool x3_attention_fused() {
  static const bool on = [] {
    const char* e = std::getenv("ED_ATTN_X3");
    return !(e && e[0] == '0');
  }();
  return on;
}
// peer transport: every receive of a run is issued on the comm stream at the
// run's start (each waits for its chunk's ready flag, then copies), and the
// compute stream waits for it only at the chunk's first consumer; a chunk's
// ready flag is raised right after the op that produces it. ED_PEER_PREFETCH=0
// keeps each receive at its consumer (A/B experiments).
inline bool peer_prefetch() {
  static const bool on = [] {
    const char* e = std::getenv("ED_PEER_PREFETCH");
    return !(e && e[0] == '0');
  }();
  return on;
}
inline bool x3_lo_by_producer() {
  static const bool on = [] {
    const char* e = std::getenv("ED_X3_LO_EPI");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace edrt

using namespace edrt;

struct ed_ctx {
  int device = 0, rank = 0, world = 1, num_sms = 148;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr, comm_stream = nullptr;
  // ed_ctx_create_multi: one process drives every rank (machine % world) on
  // its own device — the reference's single execute() over L machines
  // (runtime.cc:301-355). Ranks exchange chunks through the peer transport
  // with plain device pointers (no IPC); several ranks may share a device.
  std::vector<ed_ctx*> subs;
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
  std::vector<char> direct;        // received chunk read by refinement folds only: with prefetched
                                   // receives they read the producer's copy in place (bind_direct)
  std::vector<DepRect> host_deps;  // host copy of d_deps (rebound by bind_direct)
  bool direct_bound = false;       // bind_direct rebound at least one receive
  std::vector<Buffer> buf;         // indexed by exec id (meaningful at owners)
  std::vector<Op> ops;
  std::vector<ed_machine_c> counters;
  int64_t total_transferred = 0, peer_bytes = 0;
  int64_t rr_rounds = 0;           // run_round_robin's wall_steps for this plan (runtime.cc:281-298)
  double max_site_cost = 0.0, contraction_flops = 0.0;
  int first_join = -1;

  void* arena = nullptr;
  size_t arena_bytes = 0;
  DepRect* d_deps = nullptr;
  void* d_maps = nullptr;          // CUtensorMap[] of all GEMM launches
  void* d_regions = nullptr;       // GemmRegion[] of all GEMM launches
  void* d_sync = nullptr;          // producer lockstep counters of GEMM launches (ED_GEMM_SYNC)
  void* d_split = nullptr;         // x3 tail split-K workspaces and counters
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
  bool prefetch_ok = true;                // peer receives may be prefetched (not time-sliced processes)
  bool shared_device = false;             // another rank runs on this GPU (same-device functional mode)
  bool profile_traced = false;            // ED_PEER_TRACE printed this plan's schedule
  std::vector<cudaEvent_t> recv_events;  // profile, peer transport: [2k], [2k+1] around the k-th receive copy
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
    int64_t k0, kext;                             // its range along the contraction (KSeg) / batch (BSeg) label
    Dim mn, k, b;                                 // its layout for the GEMM classes
    int64_t off = 0;                              // BSeg: element offset of the kept sub-box in the source
  };
  struct KSeg {
    int role = 0;                                 // 0: MMA-A operand segmented, 1: MMA-B
    int64_t kseg = -1;
    std::map<int, std::vector<Seg>> segs;         // join -> segments in K order
  };
  std::map<int, KSeg> kseg_;                      // GEMM einsum -> K-segmented operand
  struct BSeg {
    int role = 0;                                 // 0: MMA-A operand segmented, 1: MMA-B
    int64_t bseg = 0;                             // batches per segment
    std::map<int, std::vector<Seg>> segs;         // join -> segments in batch order
  };
  std::map<int, BSeg> bseg_;                      // GEMM einsum -> batch-segmented operand
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
  void bind_direct();  // peer transport: point direct receives' readers at the producers' chunks
  void launch_op(size_t i, cudaStream_t s, bool branch = false);  // branch: runs beside other launches
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
                       : tag == ne + 3 ? "rank " + std::to_string(i) + " finishing the run (new inputs / teardown)"
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
  // group plan (prepared on an ed_ctx_create_multi context): one sub-plan per
  // rank; entry points dispatch to them. peer_inproc: peer pointers are the
  // sibling sub-plans' own allocations, not IPC mappings.
  std::vector<ed_plan_h*> subs;
  bool peer_inproc = false;
};

namespace edrt {
// io.cu helpers shared with exec.cu / api.cu
size_t dt_size(int dtype);
DT dt_of(int dtype);
void ensure_staging(ed_plan_h* h, size_t bytes);
std::vector<int> io_chunks(const ed_plan_h* h, int w, bool input);
// peer transport: block the stream until every rank has finished the current
// run, so this rank's exported chunks may be overwritten or freed
void wait_peers_idle(ed_plan_h* h, cudaStream_t s);
// rethrow a nested entry point's status (group plans forward to sub-plans)
void throw_status(ed_status st, const char* msg);
}  // namespace edrt
