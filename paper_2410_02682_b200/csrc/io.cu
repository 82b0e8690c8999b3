// Data in and out of a prepared plan: input chunks (engine_t ctor,
// runtime.cc:66-84) and whole tensors chunked on the device (relation.cc:31-53),
// generate_inputs on the device (runtime.cc:552-571), output assembly
// (runtime.cc:432-448, relation.cc:55-78), and the pipelined serving loop.
#include <vector>

#include "runtime.h"

namespace edrt {

void ensure_staging(ed_plan_h* h, size_t bytes) {
  if (h->staging_bytes >= bytes) return;
  if (h->staging) CUDA_OK(cudaFree(h->staging));
  h->staging = nullptr;
  CUDA_OK(cudaMalloc(&h->staging, bytes));
  h->staging_bytes = bytes;
}

void wait_peers_idle(ed_plan_h* h, cudaStream_t s) {
  if (!h->peer || !h->peer_ready) return;
  // peers copy our input chunks during a run (write-after-read): new inputs
  // are written only once every rank's run-done flag carries this epoch
  std::vector<int*> done(h->peer_flags.begin(), h->peer_flags.end());
  CUDA_OK(launch_peer_wait(done.data(), int(done.size()), h->d_epoch, 0, s, h->d_perr, int(h->X.size()) + 3));
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

}  // namespace edrt

namespace edrt {

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
  if (st != ED_OK) throw ed_error(st, msg ? msg : "");
}

}  // namespace edrt

extern "C" {

ed_status ed_upload(ed_plan_h* h, const ed_chunk_in_c* chunks, int32_t n, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (h && !h->subs.empty()) {  // group plan: every rank's sub-plan, in rank order
      for (ed_plan_h* q : h->subs) throw_status(ed_upload(q, chunks, n, err, errlen), err);
      return;
    }
    if (!h || (n && !chunks)) throw ed_error(ED_ERR_USAGE, "null argument");
    CUDA_OK(cudaSetDevice(h->ctx->device));
    cudaStream_t s = h->ctx->stream;
    wait_peers_idle(h, s);
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
    if (h && !h->subs.empty()) {  // group plan: every rank's sub-plan, in rank order
      for (ed_plan_h* q : h->subs) throw_status(ed_upload_tensors(q, ts, n, err, errlen), err);
      return;
    }
    if (!h || (n && !ts)) throw ed_error(ED_ERR_USAGE, "null argument");
    CUDA_OK(cudaSetDevice(h->ctx->device));
    cudaStream_t s = h->ctx->stream;
    wait_peers_idle(h, s);
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

ed_status ed_generate_inputs(ed_plan_h* h, uint64_t seed, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (h && !h->subs.empty()) {  // group plan: every rank's sub-plan, in rank order
      for (ed_plan_h* q : h->subs) throw_status(ed_generate_inputs(q, seed, err, errlen), err);
      return;
    }
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
    wait_peers_idle(h, s);
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

ed_status ed_download(ed_plan_h* h, ed_output_c* outs, int32_t n, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (h && !h->subs.empty()) {  // group plan: every rank's sub-plan, in rank order (rank 0 assembles)
      for (ed_plan_h* q : h->subs) throw_status(ed_download(q, outs, n, err, errlen), err);
      return;
    }
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

ed_status ed_run_steps(ed_plan_h* h, int32_t n_steps, const ed_tensor_in_c* ins, int32_t n_in, ed_output_c* outs,
                       int32_t n_out, ed_report_c* rep, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (h && h->subs.size() == 1) {
      throw_status(ed_run_steps(h->subs[0], n_steps, ins, n_in, outs, n_out, rep, err, errlen), err);
      return;
    }
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
    // ED_STEPS_TRACE=1: per step, when each copy and the run start / end (ms from the first step)
    static const bool trace = std::getenv("ED_STEPS_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t q) {
      if (!trace) return;
      cudaEvent_t e;
      CUDA_OK(cudaEventCreate(&e));
      CUDA_OK(cudaEventRecord(e, q));
      tev.push_back(e);
    };
    int bi = 0, bo = 0;
    for (int st = 0; st < n_steps; ++st) {
      // inputs: H2D on the copy-in stream, chunk() on the compute stream
      // (after the previous step's run has read the input chunks)
      for (int k = 0; k < n_in; ++k) {
        const ed_tensor_in_c& t = ins[size_t(st) * n_in + k];
        const int b = bi++ & 1;
        const size_t bytes = size_t(t.n) * dt_size(t.dtype);
        CUDA_OK(cudaStreamWaitEvent(h->cs_in, in_free[b], 0));
        mark(h->cs_in);
        CUDA_OK(cudaMemcpyAsync(h->stg_in[b], t.data, bytes, cudaMemcpyHostToDevice, h->cs_in));
        mark(h->cs_in);
        CUDA_OK(cudaEventRecord(in_full[b], h->cs_in));
        CUDA_OK(cudaStreamWaitEvent(s, in_full[b], 0));
        cached_copy(h, t.vertex_id, true, h->stg_in[b], t.dtype, s);
        for (int id : io_chunks(h, t.vertex_id, true))
          if (h->local[id] && h->buf[id].lo)
            CUDA_OK(launch_split_lo(static_cast<const float*>(h->buf[id].main), static_cast<float*>(h->buf[id].lo),
                                    h->X[id].sz, s));
        CUDA_OK(cudaEventRecord(in_free[b], s));
      }
      mark(s);
      if (h->gexec) CUDA_OK(cudaGraphLaunch(h->gexec, s));
      else h->enqueue(s);
      mark(s);
      // outputs: assemble on the compute stream, D2H on the copy-out stream,
      // overlapping the next step's uploads
      for (int k = 0; k < n_out; ++k) {
        const ed_output_c& o = outs[size_t(st) * n_out + k];
        const int b = bo++ & 1;
        CUDA_OK(cudaStreamWaitEvent(s, out_free[b], 0));
        cached_copy(h, o.vertex_id, false, h->stg_out[b], o.dtype, s);
        CUDA_OK(cudaEventRecord(out_full[b], s));
        CUDA_OK(cudaStreamWaitEvent(h->cs_out, out_full[b], 0));
        mark(h->cs_out);
        CUDA_OK(cudaMemcpyAsync(o.data, h->stg_out[b], size_t(o.n) * dt_size(o.dtype), cudaMemcpyDeviceToHost,
                                h->cs_out));
        mark(h->cs_out);
        CUDA_OK(cudaEventRecord(out_free[b], h->cs_out));
      }
    }
    CUDA_OK(cudaEventRecord(h->ev1, s));
    CUDA_OK(cudaStreamSynchronize(h->cs_out));
    CUDA_OK(cudaStreamSynchronize(s));
    CUDA_OK(cudaStreamSynchronize(h->cs_in));
    if (trace && !tev.empty()) {
      // per step: n_in x (H2D start, end), run start, end, n_out x (D2H start, end)
      const size_t per = size_t(2 * n_in + 2 + 2 * n_out);
      for (size_t st = 0; st * per < tev.size(); ++st) {
        std::fprintf(stderr, "[ed] step %zu:", st);
        for (size_t k = 0; k < per && st * per + k < tev.size(); ++k) {
          float ms = 0;
          CUDA_OK(cudaEventElapsedTime(&ms, tev[0], tev[st * per + k]));
          std::fprintf(stderr, " %.2f", ms);
        }
        std::fprintf(stderr, "\n");
      }
      for (auto e : tev) cudaEventDestroy(e);
    }
    int flag = 0;
    CUDA_OK(cudaMemcpy(&flag, h->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (flag) throw ed_error(ED_ERR_EVAL, "division by zero");
    if (rep) {
      if (rep->machines)
        for (int m = 0; m < std::min(rep->n_machines, h->n_machines); ++m) rep->machines[m] = h->counters[m];
      rep->total_transferred = h->total_transferred;
      rep->wall_steps = h->opt.sched_mode == ED_SCHED_THREADED ? int64_t(h->X.size()) : h->rr_rounds;
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
    if (h && !h->subs.empty()) {  // group plan: the rank holding the chunk
      if (exec_id < 0 || exec_id >= int(h->X.size())) throw ed_error(ED_ERR_USAGE, "exec id out of range");
      ed_plan_h* q = h->subs[size_t(h->X[exec_id].machine % int(h->subs.size()))];
      throw_status(ed_download_chunk(q, exec_id, dtype, data, n, err, errlen), err);
      return;
    }
    if (!h || !data) throw ed_error(ED_ERR_USAGE, "null argument");
    if (exec_id < 0 || exec_id >= int(h->X.size())) throw ed_error(ED_ERR_USAGE, "exec id out of range");
    if (n != h->X[exec_id].sz) throw ed_error(ED_ERR_USAGE, "chunk size mismatch");
    if (!h->local[exec_id]) throw ed_error(ED_ERR_USAGE, "chunk not resident on this rank");
    const Ex& u = h->X[exec_id];
    int o = h->owner[exec_id];
    if (u.kind == ED_EXEC_JOIN && o != exec_id && h->X[o].producer == u.producer)
      throw ed_error(ED_ERR_USAGE, "join partial was folded into its region's accumulator");
    if (h->opaque_[exec_id]) throw ed_error(ED_ERR_USAGE, "chunk was fused into its consumer's kernel");
    if (h->direct_bound && h->direct[exec_id])
      throw ed_error(ED_ERR_USAGE, "chunk is read in place on its producer rank (peer transport): download it there");
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

}  // extern "C"
