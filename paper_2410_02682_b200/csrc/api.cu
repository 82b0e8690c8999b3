// Contexts and plan lifetime (ed_ctx_create, ed_prepare, ed_plan_destroy) and
// the peer transport's bootstrap (ed_peer_export / ed_peer_import).
#include "runtime.h"

namespace {

struct PeerBlobHead {
  int32_t magic, rank, world, n_exec;
  cudaIpcMemHandle_t arena, flags;
};
constexpr int32_t kPeerMagic = 0x45445031;  // "EDP1"

size_t peer_blob_len(const ed_plan_h* h) { return sizeof(PeerBlobHead) + sizeof(int64_t) * h->X.size(); }

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

ed_status ed_ctx_create_multi(int32_t n, const int32_t* device_ids, ed_ctx** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!out || n < 1 || !device_ids) throw ed_error(ED_ERR_USAGE, "ed_ctx_create_multi: need n >= 1 device ids");
    auto* g = new ed_ctx;
    try {
      for (int r = 0; r < n; ++r) {
        ed_ctx* c = nullptr;
        char e2[512];
        const ed_status st = ed_ctx_create(device_ids[r], r, n, nullptr, 0, &c, e2, sizeof e2);
        if (st != ED_OK) throw ed_error(st, e2);
        g->subs.push_back(c);
      }
      // every rank reads its peers' chunks in place: enable peer access
      // between the distinct devices of the group (NVLink on an HGX board)
      for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
          const int da = device_ids[a], db = device_ids[b];
          if (da == db) continue;
          int can = 0;
          CUDA_OK(cudaDeviceCanAccessPeer(&can, da, db));
          if (!can) throw ed_error(ED_ERR_UNSUPPORTED, "devices " + std::to_string(da) + " and " +
                                                            std::to_string(db) + " have no peer access");
          CUDA_OK(cudaSetDevice(da));
          const cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          else CUDA_OK(e);
        }
      g->device = device_ids[0];
      g->world = n;
      g->num_sms = g->subs[0]->num_sms;
    } catch (...) {
      ed_ctx_destroy(g);
      throw;
    }
    *out = g;
  });
}

void ed_ctx_destroy(ed_ctx* c) {
  if (!c) return;
  if (!c->subs.empty()) {
    for (ed_ctx* s : c->subs) ed_ctx_destroy(s);
    delete c;
    return;
  }
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
    if (!ctx->subs.empty()) {
      // one sub-plan per rank, peer transport over plain device pointers
      auto* g = new ed_plan_h;
      g->ctx = ctx;
      if (options) g->opt = *options;
      g->opt.transport = ED_TRANSPORT_PEER;
      try {
        for (ed_ctx* c : ctx->subs) {
          ed_plan_h* h = nullptr;
          char e2[1024];
          const ed_status st = ed_prepare(c, plan, &g->opt, &h, e2, sizeof e2);
          if (st != ED_OK) throw ed_error(st, e2);
          g->subs.push_back(h);
        }
        g->copy_plan(plan);
        g->counters = g->subs[0]->counters;
        g->total_transferred = g->subs[0]->total_transferred;
        g->max_site_cost = g->subs[0]->max_site_cost;
        g->rr_rounds = g->subs[0]->rr_rounds;
        const int world = int(g->subs.size());
        for (ed_plan_h* h : g->subs) {
          if (!h->peer) continue;  // world 1: nothing to exchange
          h->peer_arena.assign(size_t(world), nullptr);
          h->peer_flags.assign(size_t(world), nullptr);
          h->peer_off.assign(size_t(world), {});
          for (int r = 0; r < world; ++r) {
            ed_plan_h* q = g->subs[size_t(r)];
            h->peer_arena[size_t(r)] = static_cast<char*>(q->arena);
            h->peer_flags[size_t(r)] = q->d_pflags;
            auto& off = h->peer_off[size_t(r)];
            off.resize(q->X.size());
            for (int id = 0; id < int(q->X.size()); ++id) off[size_t(id)] = q->local[id] ? q->arena_offset(id) : -1;
          }
          h->peer_inproc = true;
          for (ed_plan_h* q : g->subs)
            if (q != h && q->ctx->device == h->ctx->device) h->shared_device = true;
          h->peer_ready = true;
          CUDA_OK(cudaSetDevice(h->ctx->device));
          h->bind_direct();
          h->record();
        }
      } catch (...) {
        for (ed_plan_h* h : g->subs) ed_plan_destroy(h);
        delete g;
        throw;
      }
      *out = g;
      return;
    }
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
  if (!h->subs.empty()) {
    for (ed_plan_h* s : h->subs) ed_plan_destroy(s);
    delete h;
    return;
  }
  cudaSetDevice(h->ctx->device);
  h->destroy();
  delete h;
}

ed_status ed_peer_export(ed_plan_h* h, void* out, size_t cap, size_t* len, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h || !len) throw ed_error(ED_ERR_USAGE, "null argument");
    if (!h->subs.empty()) throw ed_error(ED_ERR_USAGE, "a multi-device context exchanges in-process (no export)");
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
    if (!h->subs.empty()) throw ed_error(ED_ERR_USAGE, "a multi-device context exchanges in-process (no import)");
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
      // another process on this same GPU (a functional test without MPS): the
      // contexts time-slice, and a receive that spins from the run's start
      // holds the GPU for its slice while the producer's context waits —
      // receives then stay at their consumers (no prefetch)
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, a) == cudaSuccess && at.device == h->ctx->device) {
        h->prefetch_ok = false;
        h->shared_device = true;
      }
      cudaGetLastError();
    }
    h->peer_ready = true;
    h->bind_direct();
    h->record();
  });
}

}  // extern "C"
