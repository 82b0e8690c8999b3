// Running a prepared plan: one launch per op on the compute stream, transfer
// runs on the comm stream, independent GEMMs as parallel branches, all
// captured once into a CUDA graph (record) and replayed by ed_run.
#include <algorithm>
#include <cstring>

#include "runtime.h"

void ed_plan_h::launch_op(size_t i, cudaStream_t s, bool branch) {
  Op& op = ops[i];
  switch (op.kind) {
    case OpKind::GEMM:
      if (branch && (op.gemm.sync || op.gemm.split)) {
        // a parallel branch shares the SMs: no producer lockstep, no split tiles
        // (a half waiting for its partner while the partner waits for SMs)
        GemmLaunch g = op.gemm;
        g.sync = nullptr;
        g.split = 0;
        CUDA_OK(launch_gemm(g, ctx->num_sms, s));
      } else {
        CUDA_OK(launch_gemm(op.gemm, ctx->num_sms, s));
      }
      break;
    case OpKind::GENERIC: CUDA_OK(launch_generic(op.gen, f64, s)); break;
    case OpKind::REFINE:
      if (!op.groups.empty()) CUDA_OK(launch_rect(op.rect, int(op.groups.size()), op.max_rows, f64, s));
      else CUDA_OK(launch_refine(op.ref, f64, s));
      break;
    case OpKind::CORRUPT: CUDA_OK(launch_add_one(op.ptr, op.dt, s)); break;
    case OpKind::EWISE:
      CUDA_OK(launch_ewise(op.ew, int(op.jptrs.size()), f64, opt.precision == ED_PREC_FP32, s));
      break;
    case OpKind::FLASH:
      CUDA_OK(op.attn.x3 ? launch_attn_x3(op.attn, ctx->num_sms, s) : launch_attn(op.attn, ctx->num_sms, s));
      break;
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
  const bool prefetch = peer && peer_prefetch() && prefetch_ok;
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

  // Peer transport, prefetched: a chunk's ready signal goes right after the op
  // that writes it (input chunks: at the start), every receive is issued on
  // the comm stream at the run's start in schedule order (flag wait, then the
  // copy), and the compute stream waits for a receive only where its chunk's
  // first consumer launches — so copies run under this rank's compute.
  std::vector<cudaEvent_t> recv_done;
  std::vector<std::vector<size_t>> signal_after;
  std::vector<char> moved;
  bool recv_fork = false;
  auto signal = [&](size_t k) { CUDA_OK(launch_peer_signal(d_pflags + 2 + ops[k].exec, d_epoch, s)); };
  if (prefetch) {
    recv_done.assign(ops.size(), nullptr);
    signal_after.assign(ops.size(), {});
    moved.assign(ops.size(), 0);
    for (size_t k = 0; k < ops.size(); ++k) {
      if (ops[k].kind != OpKind::SEND) continue;
      const int o = owner[size_t(ops[k].exec)];
      for (size_t q = k; q-- > 0;) {
        const auto& w = ops[q].writes;
        if (std::find(w.begin(), w.end(), o) != w.end()) {
          signal_after[q].push_back(k);
          moved[k] = 1;
          break;
        }
      }
      if (!moved[k] && X[size_t(o)].kind == ED_EXEC_INPUT_CHUNK) {
        signal(k);  // uploaded before the run
        moved[k] = 1;
      }
    }
    static const bool trace = std::getenv("ED_PEER_TRACE") != nullptr;
    if (trace && !profile_traced) {
      profile_traced = true;
      for (size_t q = 0; q < ops.size(); ++q) {
        std::fprintf(stderr, "[ed] rank %d op %zu %s", ctx->rank, q, ops[q].name.c_str());
        if (ops[q].kind == OpKind::SEND || ops[q].kind == OpKind::RECV)
          std::fprintf(stderr, " exec %d owner %d peer %d moved %d", ops[q].exec, owner[size_t(ops[q].exec)], ops[q].peer,
                       moved[q]);
        for (size_t k : signal_after[q]) std::fprintf(stderr, " -> signal exec %d", ops[k].exec);
        std::fprintf(stderr, "\n");
      }
    }
    size_t r = 0;
    for (size_t k = 0; k < ops.size(); ++k) {
      if (ops[k].kind != OpKind::RECV) continue;
      if (!recv_fork) {
        cudaEvent_t fork = next_event();
        CUDA_OK(cudaEventRecord(fork, s));
        CUDA_OK(cudaStreamWaitEvent(cs, fork, 0));
        recv_fork = true;
      }
      const Op& op = ops[k];
      int* f = peer_flags[size_t(op.peer)] + 2 + op.exec;
      CUDA_OK(launch_peer_wait(&f, 1, d_epoch, 0, cs, d_perr, op.exec));
      const int64_t off = peer_off[size_t(op.peer)][size_t(op.exec)];
      if (off < 0) throw ed_error(ED_ERR_PLAN, "peer transport: chunk not resident on its producer rank");
      if (op.direct) {  // its readers take the producer's chunk in place: the flag wait is the receive
        recv_done[k] = next_event();
        CUDA_OK(cudaEventRecord(recv_done[k], cs));
        continue;
      }
      if (opt.profile) {
        if (recv_events.size() < 2 * (r + 1)) {
          for (int e2 = 0; e2 < 2; ++e2) {
            cudaEvent_t e;
            CUDA_OK(cudaEventCreate(&e));
            recv_events.push_back(e);
          }
        }
        CUDA_OK(cudaEventRecord(recv_events[2 * r], cs));
      }
      CUDA_OK(cudaMemcpyAsync(op.ptr, peer_arena[size_t(op.peer)] + off, op.count * es, cudaMemcpyDeviceToDevice, cs));
      if (opt.profile) CUDA_OK(cudaEventRecord(recv_events[2 * r + 1], cs));
      recv_done[k] = next_event();
      CUDA_OK(cudaEventRecord(recv_done[k], cs));
      ++r;
    }
  }
  auto signals_after = [&](size_t q) {
    if (prefetch)
      for (size_t k : signal_after[q]) signal(k);
  };

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
        launch_op(k, a, true);
        joins.push_back(next_event());
        CUDA_OK(cudaEventRecord(joins.back(), a));
      }
      launch_op(i, s, true);
      for (cudaEvent_t e : joins) CUDA_OK(cudaStreamWaitEvent(s, e, 0));
      for (size_t k = i; k < g; ++k) signals_after(k);
      i = g;
      continue;
    }
    if (!is_comm(i)) {
      if (opt.profile) CUDA_OK(cudaEventRecord(op_events[i], s));
      launch_op(i, s);
      signals_after(i);
      ++i;
      continue;
    }
    if (prefetch) {
      // the compute stream takes its received chunk (the copy ran on the comm stream)
      if (opt.profile) CUDA_OK(cudaEventRecord(op_events[i], s));
      if (ops[i].kind == OpKind::RECV) CUDA_OK(cudaStreamWaitEvent(s, recv_done[i], 0));
      else if (!moved[i]) signal(i);
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
  if (recv_fork) {  // the comm stream rejoins (graph capture; every copy has landed anyway)
    cudaEvent_t join = next_event();
    CUDA_OK(cudaEventRecord(join, cs));
    CUDA_OK(cudaStreamWaitEvent(s, join, 0));
  }
  if (opt.profile) CUDA_OK(cudaEventRecord(op_events[ops.size()], s));
  if (peer) CUDA_OK(launch_peer_signal(d_pflags, d_epoch, s));  // this run is done on this rank
}

void ed_plan_h::record() {
  if (shared_device)
    // ranks sharing one GPU run their kernels side by side: a split tile's second
    // half could spin on an SM its partner half needs while that one waits for
    // another rank's kernel to leave — split tiles need every cluster of the launch
    for (Op& op : ops)
      if (op.kind == OpKind::GEMM) op.gemm.split = 0;
  CUDA_OK(gemm_prepare());
  CUDA_OK(attn_prepare());
  CUDA_OK(attn_x3_prepare());
  if (!ev0) CUDA_OK(cudaEventCreate(&ev0));
  if (!ev1) CUDA_OK(cudaEventCreate(&ev1));
  if (opt.profile && op_events.size() != ops.size() + 1) {  // every entry point that enqueues (ed_run, ed_run_steps)
    for (auto e : op_events) cudaEventDestroy(e);
    op_events.assign(ops.size() + 1, nullptr);
    for (auto& e : op_events) CUDA_OK(cudaEventCreate(&e));
  }
  if (peer && !peer_ready) return;  // peer: recorded by ed_peer_import
  cudaStream_t s = ctx->stream;
  if (opt.no_graph || opt.profile) {
    if (peer) {
      // launched op by op, a rank's first launch of a kernel loads it (lazy
      // module loading), and a load can wait for running kernels — among them
      // a wait spinning on a rank sharing this context whose own launches have
      // not been issued yet. Instantiating a throwaway capture loads them all.
      cudaGraph_t g = nullptr;
      cudaGraphExec_t ge = nullptr;
      CUDA_OK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      try {
        enqueue(s);
      } catch (...) {
        cudaStreamEndCapture(s, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      CUDA_OK(cudaStreamEndCapture(s, &g));
      CUDA_OK(cudaGraphInstantiate(&ge, g, 0));
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
    return;
  }
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
  if (peer && peer_ready && ctx->stream) {
    // peers may still be reading our arena (their last run's receives): wait
    // until every rank has finished it before the exported memory goes away
    try {
      wait_peers_idle(this, ctx->stream);
      cudaStreamSynchronize(ctx->stream);
    } catch (...) {
    }
  }
  if (gexec) cudaGraphExecDestroy(gexec);
  if (graph) cudaGraphDestroy(graph);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  for (auto e : op_events) cudaEventDestroy(e);
  for (auto e : comm_events) cudaEventDestroy(e);
  for (auto e : recv_events) cudaEventDestroy(e);
  if (d_split) cudaFree(d_split);
  for (auto a : aux)
    if (a) cudaStreamDestroy(a);
  for (size_t r = 0; r < peer_arena.size() && !peer_inproc; ++r)
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
  if (d_sync) cudaFree(d_sync);
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

extern "C" {

namespace {

// ed_run in two halves, so a group plan can start every rank's run before
// waiting for any of them (they exchange chunks while running)
void start_run(ed_plan_h* h) {
  if (h->peer && !h->peer_ready) throw ed_error(ED_ERR_USAGE, "ED_TRANSPORT_PEER: call ed_peer_import first");
  CUDA_OK(cudaSetDevice(h->ctx->device));
  cudaStream_t s = h->ctx->stream;
  CUDA_OK(cudaMemsetAsync(h->d_err, 0, sizeof(int), s));
  CUDA_OK(cudaEventRecord(h->ev0, s));
  if (h->gexec) CUDA_OK(cudaGraphLaunch(h->gexec, s));
  else h->enqueue(s);
  CUDA_OK(cudaEventRecord(h->ev1, s));
}

void finish_run(ed_plan_h* h, ed_report_c* rep) {
  CUDA_OK(cudaSetDevice(h->ctx->device));
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
    // prefetched receives: the copies themselves (on the comm stream); the
    // receive ops above count only what the compute stream waited for them
    if (h->peer && peer_prefetch() && h->prefetch_ok) {
      ed_kernel_stat_c st{};
      std::snprintf(st.name, sizeof(st.name), "%s", "peer_recv_copy");
      size_t r = 0;
      for (const Op& op : h->ops) {
        if (op.kind != OpKind::RECV || op.direct) continue;
        float t = 0;
        CUDA_OK(cudaEventElapsedTime(&t, h->recv_events[2 * r], h->recv_events[2 * r + 1]));
        st.launches += 1;
        st.ms += t;
        st.bytes += double(op.count) * double(h->es);
        ++r;
      }
      if (st.launches) h->stats.push_back(st);
    }
  }
  if (flag) throw ed_error(ED_ERR_EVAL, "division by zero");
  if (rep) {
    if (rep->machines)
      for (int m = 0; m < std::min(rep->n_machines, h->n_machines); ++m) rep->machines[m] = h->counters[m];
    rep->total_transferred = h->total_transferred;
    rep->wall_steps = h->opt.sched_mode == ED_SCHED_THREADED ? int64_t(h->X.size()) : h->rr_rounds;
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
}

}  // namespace

ed_status ed_run(ed_plan_h* h, ed_report_c* rep, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h) throw ed_error(ED_ERR_USAGE, "null plan");
    if (h->subs.empty()) {
      start_run(h);
      finish_run(h, rep);
      return;
    }
    // group plan: every rank's run is in flight before any is waited for;
    // device_ms is the slowest rank's, counts sum over ranks
    for (ed_plan_h* s : h->subs) start_run(s);
    double ms = 0;
    int64_t pb = 0;
    double cf = 0;
    int launches = 0;
    std::map<std::string, size_t> idx;
    h->stats.clear();
    for (ed_plan_h* s : h->subs) {
      ed_report_c r{};
      r.n_machines = rep ? rep->n_machines : 0;
      r.machines = rep ? rep->machines : nullptr;
      finish_run(s, &r);
      ms = std::max(ms, r.device_ms);
      pb += r.peer_bytes;
      cf += r.contraction_flops;
      launches += r.gpu_launches;
      if (rep) {
        rep->total_transferred = r.total_transferred;
        rep->wall_steps = r.wall_steps;
        rep->max_site_cost = r.max_site_cost;
      }
      for (const auto& st : s->stats) {
        auto it = idx.find(st.name);
        if (it == idx.end()) {
          it = idx.emplace(st.name, h->stats.size()).first;
          h->stats.push_back(st);
          continue;
        }
        auto& t = h->stats[it->second];
        t.launches += st.launches;
        t.ms += st.ms;
        t.flops += st.flops;
        t.bytes += st.bytes;
      }
    }
    if (rep) {
      rep->device_ms = ms;
      rep->peer_bytes = pb;
      rep->contraction_flops = cf;
      rep->gpu_launches = launches;
    }
  });
}

ed_status ed_kernel_stats(ed_plan_h* h, ed_kernel_stat_c* out, int32_t cap, int32_t* n_out, char* err,
                          size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h || !n_out) throw ed_error(ED_ERR_USAGE, "null argument");
    std::vector<ed_kernel_stat_c> all = h->stats;
    for (size_t r = 0; r < h->subs.size(); ++r)  // one process over L ranks: "r<rank>/<launch class>"
      for (ed_kernel_stat_c st : h->subs[r]->stats) {
        char name[sizeof st.name];
        std::snprintf(name, sizeof name, "r%zu/%s", r, st.name);
        std::memcpy(st.name, name, sizeof name);
        all.push_back(st);
      }
    int k = std::min<int>(cap, int(all.size()));
    for (int i = 0; i < k; ++i) out[i] = all[i];
    *n_out = int(all.size());
  });
}

}  // extern "C"
