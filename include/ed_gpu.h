/*
 * ed_gpu.h — C ABI of the B200-native EinDecomp executor (libed_gpu.so).
 *
 * Drop-in replacement for the reference's CPU executor
 *
 *   run_report_t execute(exec_graph_t const&, placement_t const&,
 *                        map<int, tensor_relation_t> const&,
 *                        exec_options_t const& = {});     // runtime.h:45-49
 *                                                          // runtime.cc:382-451
 *
 * The reference planner (parse -> optimize_dag -> explode -> place_all,
 * runtime.cc:511-516) is unchanged; its products are flattened into
 * ed_plan_c by the host adapter and executed here on
 * B200s. No C++ or torch types cross this boundary: plain structs,
 * pointers and sizes, status codes plus a NUL-terminated message.
 *
 * Ownership: the caller owns every host buffer; the library owns device
 * memory, streams, CUDA graphs and NCCL communicators. ed_prepare deep-
 * copies the plan. A context / plan handle is single-caller (not
 * re-entrant); calls block until their work is complete, like execute().
 *
 * Multi-GPU: rank r runs the exec vertices whose machine
 * (placement_t::machine_of, placement.h:9-15) maps to it (machine % world
 * == r). Either one process drives every rank (ed_ctx_create_multi, the
 * drop-in for the reference's single execute() over L machines), or one
 * process per GPU (ed_ctx_create + ed_peer_export / ed_peer_import). Remote
 * dependencies move over the peer transport (the consumer reads the
 * producer's HBM over NVLink once its ready flag carries the run's epoch);
 * ED_TRANSPORT_NCCL is an opt-in alternative for one-process-per-GPU worlds.
 */
#ifndef ED_GPU_H
#define ED_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ED_ABI_VERSION 1

#if defined(__GNUC__)
#define ED_API __attribute__((visibility("default")))
#else
#define ED_API
#endif

/* Errors. The adapter rethrows ED_ERR_PLAN as plan_error_t (setup.h:40-42),
 * ED_ERR_EVAL as eval_error_t (setup.h:45-47; division by zero, ops.cc:10-14,
 * detected on device), everything else as std::runtime_error. */
typedef enum {
  ED_OK = 0,
  ED_ERR_USAGE = 1,
  ED_ERR_PLAN = 2,
  ED_ERR_EVAL = 4,
  ED_ERR_CUDA = 5,
  ED_ERR_NCCL = 6,
  ED_ERR_OOM = 7,
  ED_ERR_UNSUPPORTED = 8
} ed_status;

/* Arithmetic of the run (exec_options_t::f32, runtime.h:39-43, generalised).
 *   FP64 : f64 storage, every op in double, folds in dep order — reproduces
 *          the reference's default execute() bit for bit.
 *   FP32 : f32 storage; non-contraction vertices reproduce the reference's
 *          f32 mode bit for bit; contractions on fp32 CUDA cores.
 *   TF32 : f32 storage; mul/sum contractions on tcgen05 kind::tf32.
 *   BF16 : f32 storage, bf16 contraction operands (written by their
 *          producers), tcgen05 kind::f16 with fp32 accumulation in TMEM.
 *   F32X3: f32 storage; contractions as three kind::tf32 products
 *          hi*hi + hi*lo + lo*hi (lo = x - tf32(x)) accumulated in TMEM:
 *          fp32-level accuracy at tensor-core speed. */
typedef enum {
  ED_PREC_FP32 = 0,
  ED_PREC_TF32 = 1,
  ED_PREC_BF16 = 2,
  ED_PREC_FP64 = 3,
  ED_PREC_F32X3 = 4
} ed_precision;

/* Operator enums, in the order of ops.h:8-22. -1 = absent. */
typedef enum { ED_JOIN_MUL = 0, ED_JOIN_ADD, ED_JOIN_SUB, ED_JOIN_DIV, ED_JOIN_SQDIFF, ED_JOIN_ABSDIFF } ed_join_op;
typedef enum { ED_AGG_SUM = 0, ED_AGG_MAX } ed_agg_op;
typedef enum { ED_MAP_RELU = 0, ED_MAP_EXP, ED_MAP_NEG, ED_MAP_SCALE, ED_MAP_IDENTITY } ed_map_op;

/* exec_kind_t, execgraph.h:12 */
typedef enum { ED_EXEC_INPUT_CHUNK = 0, ED_EXEC_JOIN = 1, ED_EXEC_REFINEMENT = 2 } ed_exec_kind;

typedef enum { ED_DTYPE_F64 = 0, ED_DTYPE_F32 = 1 } ed_dtype;

/* One EinGraph vertex: ein_vertex_t (einsum.h:42-47) + einsum_expr_t
 * (einsum.h:9-38) + task_graph_t::d (decomp.h:21-30). Labels are interned
 * as small non-negative ints (equal strings -> equal ids within a vertex). */
typedef struct {
  const char* name;
  int32_t arity;            /* 0 = graph input, 1 = unary map, 2 = binary join */
  int32_t join_op;          /* ed_join_op or -1 */
  int32_t map_op;           /* ed_map_op or -1 */
  int32_t agg_op;           /* ed_agg_op or -1 */
  double scale_c;           /* unary_op_t::scale_c */
  int32_t rank;             /* rank of bound */
  const int64_t* bound;     /* b of this vertex */
  int32_t rank_z, rank_x, rank_y;
  const int32_t* lz;        /* out_labels */
  const int32_t* lx;        /* in_labels[0] */
  const int32_t* ly;        /* in_labels[1] (binary only) */
  int32_t rank_d;
  const int64_t* d;         /* exprs: over l_XY; inputs: storage partition */
  int32_t inputs[2];        /* graph vertex ids, -1 when absent */
} ed_vertex_c;

/* exec_vertex_t (execgraph.h:14-34) + placement_t::machine_of. */
typedef struct {
  int32_t kind;             /* ed_exec_kind */
  int32_t owner, producer, consumer, slot;
  int32_t key_rank;
  const int64_t* key;
  int32_t chunk_rank;
  const int64_t* chunk_bound;
  int64_t fp, sz;
  int32_t n_deps;
  const int32_t* deps;      /* fixed order: refinements fold in this order */
  int32_t machine;
} ed_exec_vertex_c;

typedef struct {
  int32_t n_vertices;
  const ed_vertex_c* vertices;
  int32_t n_exec;
  const ed_exec_vertex_c* exec;   /* ids = array positions, topological */
  int32_t n_outputs;
  const int32_t* outputs;         /* eingraph_t::outputs */
  int32_t n_machines;             /* placement_t::n_machines */
  double alpha;                   /* placement_t::alpha (max_site_cost) */
} ed_plan_c;

typedef struct {
  int32_t precision;        /* ed_precision */
  int32_t corrupt;          /* exec_options_t::corrupt test hook: +1 on one join output */
  int32_t profile;          /* 1: time every launch with CUDA events (ed_kernel_stats) */
  int32_t no_graph;         /* 1: launch eagerly instead of replaying a CUDA graph */
  int32_t transport;        /* ed_transport: how remote dependencies move (world > 1) */
  int32_t sched_mode;       /* ed_sched_mode: which of the reference's schedulers wall_steps reports */
  int32_t reserved[2];
} ed_options_c;

/* sched_mode_t (runtime.h:23): wall_steps of run_report_t counts rounds in
 * round_robin (the reference's default, runtime.cc:281-298) and vertices in
 * threaded mode (runtime.cc:353). The device schedule is the same for both. */
typedef enum { ED_SCHED_ROUND_ROBIN = 0, ED_SCHED_THREADED = 1 } ed_sched_mode;

/* ED_TRANSPORT_NCCL: ncclSend / ncclRecv groups on a comm stream (needs the
 *   context's NCCL communicator).
 * ED_TRANSPORT_PEER: the consumer copies the producer's chunk straight out of
 *   the producer's HBM (CUDA IPC mapping; NVLink between GPUs) once a ready
 *   flag in the producer's memory carries this run's epoch. Needs
 *   ed_peer_export / ed_peer_import before the first ed_run; works with several
 *   ranks on one GPU too (tests). */
typedef enum { ED_TRANSPORT_NCCL = 0, ED_TRANSPORT_PEER = 1 } ed_transport;

/* One input chunk (tensor_relation_t::chunks entry, relation.h:13-19),
 * row-major over exec vertex exec_id's chunk_bound. */
typedef struct {
  int32_t exec_id;
  int32_t dtype;            /* ed_dtype */
  const void* data;
  int64_t n;
} ed_chunk_in_c;

/* One whole input tensor of graph vertex vertex_id; the library performs
 * chunk() (relation.cc:31-53) on the device. */
typedef struct {
  int32_t vertex_id;
  int32_t dtype;
  const void* data;
  int64_t n;
} ed_tensor_in_c;

/* One graph output, assembled (relation.cc:55-78) row-major. */
typedef struct {
  int32_t vertex_id;
  int32_t dtype;
  void* data;
  int64_t n;
} ed_output_c;

/* machine_counters_t, runtime.h:16-20 */
typedef struct {
  int64_t fp, sent, received;
} ed_machine_c;

/* run_report_t (runtime.h:27-37) minus the tensors (see ed_download). */
typedef struct {
  int32_t n_machines;        /* capacity of machines[] (caller-owned) */
  ed_machine_c* machines;    /* counters equal the reference's whole-chunk accounting */
  int64_t total_transferred;
  int64_t wall_steps;
  double max_site_cost;
  double device_ms;          /* event-timed ed_run on this rank */
  int64_t peer_bytes;        /* bytes this rank actually sent to peers */
  double contraction_flops;  /* 2 * sum fp of mul/sum joins run by this rank */
  int32_t gpu_launches;      /* kernels launched by this rank's ed_run */
} ed_report_c;

/* Per-launch-class timing from a profiled run (options.profile = 1). */
typedef struct {
  char name[64];             /* kernel class + graph vertex, e.g. "gemm_bf16:Z1" */
  int32_t launches;
  double ms;                 /* summed CUDA-event time */
  double flops;              /* algorithmic flops summed over launches */
  double bytes;              /* algorithmic HBM bytes summed over launches */
} ed_kernel_stat_c;

/* One step of a rank's logical schedule (ed_plan_schedule). */
typedef enum { ED_SCHED_COMPUTE = 0, ED_SCHED_SEND = 1, ED_SCHED_RECV = 2 } ed_sched_kind;
typedef struct {
  int32_t kind;              /* ed_sched_kind */
  int32_t exec_id;           /* vertex computed, or chunk sent / received */
  int32_t peer;              /* SEND: destination rank, RECV: source rank, else -1 */
  int64_t elems;             /* chunk elements moved (SEND / RECV) */
} ed_sched_op_c;

struct ed_ctx;
struct ed_plan_h;

ED_API int32_t ed_abi_version(void);

/* NCCL bootstrap id (128 bytes) for world > 1, made on rank 0 and
 * broadcast by the caller. ed_ctx_create takes nccl_id = NULL for a world
 * that only uses the peer transport. */
ED_API ed_status ed_nccl_unique_id(void* out, size_t len, char* err, size_t errlen);

ED_API ed_status ed_ctx_create(int32_t device, int32_t rank, int32_t world,
                        const void* nccl_id, size_t nccl_id_len,
                        struct ed_ctx** out, char* err, size_t errlen);
/* One process, several ranks: the reference's single execute() call drives
 * all L machines (runtime.cc:301-355, runtime.cc:518-550), so the drop-in
 * does too. Rank r (machine % n) runs on device_ids[r] (a device may repeat:
 * several ranks then share it); ranks exchange remote chunks through the
 * peer transport with plain device pointers (peer access is enabled between
 * distinct devices, NVLink on an HGX board). Every plan call on such a
 * context drives all ranks from the calling thread: ed_run starts every
 * rank's run before waiting for any; ed_download assembles on rank 0.
 * ed_peer_export / ed_peer_import are not used. */
ED_API ed_status ed_ctx_create_multi(int32_t n, const int32_t* device_ids, struct ed_ctx** out, char* err,
                                     size_t errlen);
ED_API void ed_ctx_destroy(struct ed_ctx* ctx);

/* Validates the plan (execute()'s checks, runtime.cc:388-395), maps each
 * expression onto a kernel, allocates every chunk buffer in HBM, builds
 * tensor maps and the transfer schedule, and records the CUDA graph. */
ED_API ed_status ed_prepare(struct ed_ctx* ctx, const ed_plan_c* plan, const ed_options_c* options,
                     struct ed_plan_h** out, char* err, size_t errlen);
ED_API void ed_plan_destroy(struct ed_plan_h* h);

/* Seed input chunks (engine_t ctor, runtime.cc:66-84): H2D + convert. */
ED_API ed_status ed_upload(struct ed_plan_h* h, const ed_chunk_in_c* chunks, int32_t n,
                    char* err, size_t errlen);
/* Whole input tensors; chunked on device. */
ED_API ed_status ed_upload_tensors(struct ed_plan_h* h, const ed_tensor_in_c* tensors, int32_t n,
                            char* err, size_t errlen);

/* generate_inputs(graph, seed) (runtime.cc:552-571) on the device: every input
 * tensor this rank holds chunks of is drawn from std::mt19937_64(seed * 7919 +
 * vertex) through libstdc++'s uniform_int_distribution<int>(-4, 4) (graphs
 * that only sum and multiply, runtime.cc:358-378) or
 * uniform_real_distribution<double>(-1, 1), bit for bit, then chunked in
 * place of ed_upload_tensors. */
ED_API ed_status ed_generate_inputs(struct ed_plan_h* h, uint64_t seed, char* err, size_t errlen);

/* Run every exec vertex of this rank; device-resident. report may be NULL. */
ED_API ed_status ed_run(struct ed_plan_h* h, ed_report_c* report, char* err, size_t errlen);

/* Assemble graph outputs from their final refinement layers (runtime.cc:432-448)
 * and copy D2H. With world > 1 this is collective: every rank calls it, chunks
 * held by other ranks travel to rank 0 over NCCL, and only rank 0's buffers
 * are written. */
ED_API ed_status ed_download(struct ed_plan_h* h, ed_output_c* outputs, int32_t n,
                      char* err, size_t errlen);

/* n_steps end-to-end steps of a serving loop in one call: for step s, upload
 * inputs[s*n_in .. s*n_in+n_in) (chunked on the device), run, and assemble and
 * copy outputs[s*n_out .. s*n_out+n_out) to the host. The host-to-device copies
 * of step s+1 run on a copy stream while step s computes and its outputs
 * travel device-to-host on another (double-buffered staging), so a step costs
 * about max(H2D, D2H) + compute instead of their sum. Host buffers should be
 * pinned for the copies to overlap. Blocks until every output is written;
 * report (nullable) as ed_run, device_ms spanning all steps. With world > 1
 * this is the plain upload / run / collective-download sequence per step. */
ED_API ed_status ed_run_steps(struct ed_plan_h* h, int32_t n_steps, const ed_tensor_in_c* inputs, int32_t n_in,
                              ed_output_c* outputs, int32_t n_out, ed_report_c* report, char* err, size_t errlen);

/* Copy one exec vertex's produced chunk D2H (per-vertex parity tests).
 * Returns ED_ERR_USAGE if the chunk is not resident on this rank. */
ED_API ed_status ed_download_chunk(struct ed_plan_h* h, int32_t exec_id, int32_t dtype,
                            void* data, int64_t n, char* err, size_t errlen);

/* Host-only (no GPU needed): rank `rank`'s logical schedule in a world of
 * `world` processes — its exec vertices in execution order, interleaved with
 * the NCCL sends/receives of remote dependencies, which every rank issues in
 * the same global order (a transfer is placed before its first consumer).
 * ed_run executes exactly this order (with joins grouped into launches). */
ED_API ed_status ed_plan_schedule(const ed_plan_c* plan, int32_t rank, int32_t world, ed_sched_op_c* out,
                                  int32_t cap, int32_t* n_out, char* err, size_t errlen);

/* Device cost model for ed_gpu_placement (rates in units per second). */
typedef struct {
  double tensor_flops;       /* contraction rate per GPU (e.g. measured bf16 peak) */
  double hbm_bytes;          /* memory-bound kernel rate per GPU (measured copy bandwidth) */
  double link_bytes;         /* GPU-to-GPU rate per direction (NVLink 5) */
  int32_t elem_bytes;        /* bytes per stored element (4: f32, 8: f64) */
  int32_t max_passes;        /* local-search passes (0: default 4) */
  int32_t fuse_chains;       /* 1: keep each region of a fusable chain (attention block, row softmax,
                                map epilogue) on one GPU so the executor can fuse it per rank */
  int32_t reserved;
} ed_cost_model_c;

/* Host-only (no GPU needed). GPU-aware re-placement:
 * starting from the plan's machine_of (place_all, placement.cc:132-178),
 * moves memory-bound exec vertices (non-contraction joins and refinements)
 * between machines to minimise the estimated busiest-GPU time — compute at
 * the cost model's rates plus whole-chunk transfers over the links — ties
 * broken by transfer volume. Input chunks and mul/sum contraction joins keep
 * their machines (with fuse_chains, the QK^T joins of an attention block move
 * with the block: each region of a fusable chain is kept on one GPU so the
 * executor can fuse it there, and the chain's memory-bound work is credited
 * while it stays together); the exec graph, keys and fold order are untouched,
 * so the results are bitwise those of the original placement
 * (acceptance.cc:241-250).
 * machine_of: n_exec entries, written. est_ms (nullable, 2 entries): the
 * estimated busiest-GPU milliseconds before and after. */
ED_API ed_status ed_gpu_placement(const ed_plan_c* plan, const ed_cost_model_c* model, int32_t* machine_of,
                                  double* est_ms, char* err, size_t errlen);

/* Peer transport bootstrap (ED_TRANSPORT_PEER, world > 1). ed_peer_export
 * writes this rank's blob (IPC handles of its chunk arena and flag words, and
 * the arena offset of every chunk it holds) into out (capacity cap, *len set;
 * call with out = NULL to get the size). The caller all-gathers the blobs
 * (any bootstrap: torch.distributed, MPI, files) and hands every rank the
 * world's blobs in rank order: ed_peer_import maps the peers' memory and
 * records the CUDA graph. */
ED_API ed_status ed_peer_export(struct ed_plan_h* h, void* out, size_t cap, size_t* len, char* err, size_t errlen);
ED_API ed_status ed_peer_import(struct ed_plan_h* h, const void* blobs, size_t blob_len, int32_t n, char* err,
                                size_t errlen);

/* Per-launch-class timings of the last profiled ed_run. A plan over several
 * ranks in one process (ed_ctx_create_multi) lists the classes summed over its
 * ranks, then each rank's own as "r<rank>/<class>". With the peer transport,
 * "nccl_recv" is the time the compute stream waited for its received chunks
 * and "peer_recv_copy" the copies themselves (prefetched on the comm stream). */
ED_API ed_status ed_kernel_stats(struct ed_plan_h* h, ed_kernel_stat_c* out, int32_t cap,
                          int32_t* n_out, char* err, size_t errlen);

#ifdef __cplusplus
}
#endif

#endif /* ED_GPU_H */
