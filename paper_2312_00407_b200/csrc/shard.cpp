// Native ZeRO sharders over NCCL (SURVEY 8(b) "mco_shard_step", 8(e)): the stage-2
// branch of ParallelWorker::train_step (parallel.cpp:656-666),
//
//   owned_grads = reduce_scatter(flat_grads, SUM, ZeroPlan parts)   parallel.cpp:657-658
//   FlatOptimizer::step(params[owned], owned_grads, lr)             parallel.cpp:660
//   params      = all_gather(params[owned])                         parallel.cpp:661-663
//
// stream-ordered on the caller's stream, so a C / C++ host (the reference's own
// parallel engine) gets the sharded step without torch.
//   mco_shard_step[_mixed]  one reduce-scatter of the whole flat gradient, the update of
//                           the ZeroPlan part, one all-gather (P mod N != 0: per-part
//                           ncclReduce / ncclBroadcast, the reference's ownership).
//   mco_zb_*                the bucketed, double-buffered form: the
//                           gradient arrives bucket by bucket (as backward produces it,
//                           no full-length gradient needs to be resident); per bucket a
//                           reduce-scatter on the library's comm stream, the update of
//                           this rank's piece on its update stream, an all-gather of
//                           the bucket's replicas -- RS(k+1) is issued before AG(k), so
//                           it overlaps update(k).
//
// Failure handling (comm.cpp:126-132 timeouts, comm.cpp:330-348 rank-attributed abort):
// every communicator is created non-blocking with a deadline (MCO_NCCL_TIMEOUT_S, or
// mco_comm_create_timeout); an init that does not complete in time (a rank that never
// joined), and a stream wait (mco_comm_wait) whose collectives do not finish in time,
// abort the communicator (ncclCommAbort) and return MCO_PROTOCOL naming this rank and
// what it was waiting for.
//
// NCCL is resolved at run time (dlopen): the libnccl.so.2 already mapped into the
// process (torch's build) is reused, never a second copy; otherwise MCO_NCCL_LIB, then
// the system libnccl.so.2.  libmco.so has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "abi_internal.h"

namespace mco {
namespace {

struct NcclApi {
  void* so = nullptr;
  std::string from;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank_config)(ncclComm_t*, int, ncclUniqueId, int,
                                        ncclConfig_t*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_abort)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_get_async_error)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*get_error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                 ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int,
                         ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                             ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
};

template <class F>
void sym(void* so, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(so, name));
  if (!out) throw Error(MCO_IO, std::string("NCCL: missing symbol ") + name);
}

const NcclApi& nccl() {
  static std::mutex mu;
  static NcclApi api;
  std::lock_guard<std::mutex> lock(mu);
  if (api.so) return api;
  void* so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's own NCCL
  std::string from = "already loaded";
  if (!so) {
    if (const char* env = getenv("MCO_NCCL_LIB")) {
      so = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
      from = env;
    }
  }
  if (!so) {
    so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    from = "libnccl.so.2";
  }
  if (!so) throw Error(MCO_IO, std::string("NCCL: cannot load libnccl.so.2: ") + dlerror());
  NcclApi a;
  a.so = so;
  a.from = from;
  sym(so, "ncclGetUniqueId", a.get_unique_id);
  sym(so, "ncclCommInitRankConfig", a.comm_init_rank_config);
  sym(so, "ncclCommDestroy", a.comm_destroy);
  sym(so, "ncclCommAbort", a.comm_abort);
  sym(so, "ncclCommGetAsyncError", a.comm_get_async_error);
  sym(so, "ncclGetErrorString", a.get_error_string);
  sym(so, "ncclReduceScatter", a.reduce_scatter);
  sym(so, "ncclAllGather", a.all_gather);
  sym(so, "ncclReduce", a.reduce);
  sym(so, "ncclBroadcast", a.broadcast);
  sym(so, "ncclAllReduce", a.all_reduce);
  sym(so, "ncclGroupStart", a.group_start);
  sym(so, "ncclGroupEnd", a.group_end);
  api = a;
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess && r != ncclInProgress)
    throw Error(MCO_PROTOCOL, std::string(what) + ": " + nccl().get_error_string(r));
}

ncclDataType_t nccl_type(int dt) {
  switch (dt) {
    case MCO_F32: return ncclFloat32;
    case MCO_BF16: return ncclBfloat16;
    case MCO_F64: return ncclFloat64;
  }
  throw Error(MCO_CONTRACT, "NCCL: unsupported dtype " + std::to_string(dt));
}

size_t dt_size(int dt) { return dt == MCO_F64 ? 8 : dt == MCO_BF16 ? 2 : 4; }

// bf16 -> fp32 (exact): the mixed sharder's master initialised from bf16 replicas
__global__ void widen_bf16_kernel(float* out, const uint16_t* in, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = __uint_as_float((uint32_t)in[i] << 16);
}

void widen_bf16(float* out, const uint16_t* in, uint64_t n, cudaStream_t st) {
  if (!n) return;
  const int blocks = (int)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  widen_bf16_kernel<<<blocks, 256, 0, st>>>(out, in, n);
  MCO_CUDA_CHECK(cudaGetLastError());
}

double default_timeout() {
  if (const char* e = getenv("MCO_NCCL_TIMEOUT_S")) {
    const double v = atof(e);
    if (v > 0) return v;
  }
  return 600.0;
}

}  // namespace
}  // namespace mco

using namespace mco;

struct mco_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
  double timeout_s = 600.0;
  bool aborted = false;
  void* scratch = nullptr;  // reduced owned gradient (ZeroPlan part of this rank)
  size_t scratch_bytes = 0;
  ~mco_comm() {
    if (scratch) cudaFree(scratch);
    if (comm) {
      if (aborted)
        ;  // ncclCommAbort already released it
      else
        nccl().comm_destroy(comm);
    }
  }

  std::string who() const {
    return "[rank " + std::to_string(rank) + " of " + std::to_string(nranks) + "] ";
  }

  // Abort the communicator (releases this side's pending collectives) and raise the
  // rank-attributed error (comm.cpp:330-348).
  [[noreturn]] void fail(const std::string& what) {
    if (comm && !aborted) {
      nccl().comm_abort(comm);
      aborted = true;
    }
    throw Error(MCO_PROTOCOL, who() + what);
  }

  // A non-blocking NCCL call returned: wait (bounded) until it is enqueued / complete.
  void settle(ncclResult_t r, const char* what) {
    if (aborted) throw Error(MCO_PROTOCOL, who() + "communicator was aborted");
    if (r == ncclSuccess) return;
    if (r != ncclInProgress) fail(std::string(what) + ": " + nccl().get_error_string(r));
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      ncclResult_t a = ncclSuccess;
      nccl().comm_get_async_error(comm, &a);
      if (a == ncclSuccess) return;
      if (a != ncclInProgress) fail(std::string(what) + ": " + nccl().get_error_string(a));
      const double dt =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (dt > timeout_s)
        fail(std::string(what) + ": timed out after " + std::to_string(timeout_s) + " s");
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }

  // Host wait for `stream` (its collectives) with the deadline.
  void wait(cudaStream_t st, const char* what) {
    if (aborted) throw Error(MCO_PROTOCOL, who() + "communicator was aborted");
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      const cudaError_t q = cudaStreamQuery(st);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) cuda_check(q, what);
      ncclResult_t a = ncclSuccess;
      nccl().comm_get_async_error(comm, &a);
      if (a != ncclSuccess && a != ncclInProgress)
        fail(std::string(what) + ": " + nccl().get_error_string(a));
      const double dt =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (dt > timeout_s)
        fail(std::string(what) + ": collectives did not complete within " +
             std::to_string(timeout_s) + " s (a peer rank did not take part)");
      std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
  }
};

#define MCO_NCALL(c, x) (c)->settle((x), #x)

extern "C" {

mco_status mco_comm_unique_id(void* id_out) {
  return guard([&] {
    if (!id_out) throw Error(MCO_CONTRACT, "comm unique id: null output");
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof(id));
  });
}

mco_status mco_comm_create_timeout(const void* id, int nranks, int rank, int device,
                                   double timeout_s, mco_comm** out) {
  return guard([&] {
    if (!id || !out) throw Error(MCO_CONTRACT, "comm create: null argument");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks)
      throw Error(MCO_CONFIG, "comm create: rank " + std::to_string(rank) + " of " +
                                  std::to_string(nranks));
    device = resolve_device(device);
    DeviceGuard ds(device);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    auto c = std::make_unique<mco_comm>();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    c->timeout_s = timeout_s > 0 ? timeout_s : default_timeout();
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;  // init and every call return at once; settle() bounds the wait
    const ncclResult_t r = nccl().comm_init_rank_config(&c->comm, nranks, uid, rank, &cfg);
    if (r != ncclSuccess && r != ncclInProgress) {
      c->comm = nullptr;
      throw Error(MCO_PROTOCOL, c->who() + "ncclCommInitRank: " + nccl().get_error_string(r));
    }
    c->settle(r, "ncclCommInitRank (waiting for every rank to join)");
    *out = c.release();
  });
}

mco_status mco_comm_create(const void* id, int nranks, int rank, int device, mco_comm** out) {
  return mco_comm_create_timeout(id, nranks, rank, device, 0.0, out);
}

mco_status mco_comm_destroy(mco_comm* c) {
  return guard([&] {
    if (!c) return;
    DeviceGuard ds(c->device);
    delete c;
  });
}

mco_status mco_comm_check(mco_comm* c) {
  return guard([&] {
    if (!c) throw Error(MCO_CONTRACT, "mco_comm_check: null handle");
    if (c->aborted) throw Error(MCO_PROTOCOL, c->who() + "communicator was aborted");
    ncclResult_t r = ncclSuccess;
    nccl_check(nccl().comm_get_async_error(c->comm, &r), "ncclCommGetAsyncError");
    if (r != ncclSuccess && r != ncclInProgress)
      c->fail(std::string("NCCL asynchronous error: ") + nccl().get_error_string(r));
  });
}

mco_status mco_comm_wait(mco_comm* c, void* stream) {
  return guard([&] {
    if (!c) throw Error(MCO_CONTRACT, "mco_comm_wait: null handle");
    DeviceGuard ds(c->device);
    c->wait((cudaStream_t)stream, "stream wait");
  });
}

mco_status mco_comm_abort(mco_comm* c) {
  return guard([&] {
    if (!c) throw Error(MCO_CONTRACT, "mco_comm_abort: null handle");
    DeviceGuard ds(c->device);
    if (c->comm && !c->aborted) {
      nccl().comm_abort(c->comm);
      c->aborted = true;
    }
  });
}

mco_status mco_comm_allreduce_sum(mco_comm* c, void* buf, int dtype, uint64_t n, void* stream) {
  return guard([&] {
    if (!c) throw Error(MCO_CONTRACT, "mco_comm_allreduce_sum: null handle");
    DeviceGuard ds(c->device);
    MCO_NCALL(c, nccl().all_reduce(buf, buf, n, nccl_type(dtype), ncclSum, c->comm,
                                   (cudaStream_t)stream));
  });
}

}  // extern "C"

namespace {
// RS (or grouped reduce) of flat_grads into a scratch slice whose element phase (mod 8)
// matches `phase_ref` -> step(gdst, owned_len) -> AG (or grouped broadcast) of ag_buf,
// whose element type is ag_dtype.  Argument checks come first, before any collective
// (every rank fails the same way).
template <class StepFn>
void shard_run(mco_flat* h, mco_comm* c, const void* flat_grads, int grad_dtype,
               uint64_t total_len, void* ag_buf, int ag_dtype, const void* phase_ref,
               size_t phase_es, void* stream, StepFn step) {
  if (!h || !c || !flat_grads || !ag_buf) throw Error(MCO_CONTRACT, "shard step: null argument");
  const int N = c->nranks, me = c->rank;
  std::vector<uint64_t> parts(N), offs(N + 1);
  const mco_status zs = mco_zero_plan(total_len, N, 2, parts.data(), offs.data());
  if (zs != MCO_OK) throw Error(zs, "shard step: zero plan");
  // the owned length straight from the handle: the public mco_flat_buffer() would mark
  // the state exposed and freeze its layout before the first step re-phases it to the
  // parameters' alignment (abi_flat.cpp align_state_to)
  const uint64_t nbuf = h->n;
  // the handle's owned length must be this rank's ZeroPlan part (parallel.cpp:330)
  if (nbuf != parts[me])
    throw Error(MCO_CONTRACT, "shard step: optimizer owns " + std::to_string(nbuf) +
                                  " elements but ZeroPlan gives rank " + std::to_string(me) +
                                  " " + std::to_string(parts[me]));
  const ncclDataType_t gt = nccl_type(grad_dtype), at = nccl_type(ag_dtype);
  const size_t gs = dt_size(grad_dtype), as = dt_size(ag_dtype);
  DeviceGuard ds(c->device);
  // reduced gradient in the stepped slice's alignment phase (mod 8 elements): the update
  // then vectorises after a short head (flat.cu launch_flat_step)
  const uintptr_t u = (uintptr_t)phase_ref;
  const size_t phase = (u % phase_es) ? 0 : (u / phase_es) % 8;
  const size_t need = (parts[me] + 8) * gs + 256;
  if (c->scratch_bytes < need) {
    if (c->scratch) MCO_CUDA_CHECK(cudaFree(c->scratch));
    c->scratch = nullptr;
    MCO_CUDA_CHECK(cudaMalloc(&c->scratch, need));
    c->scratch_bytes = need;
  }
  auto s = (cudaStream_t)stream;
  char* gdst = (char*)c->scratch + phase * gs;
  const char* algo = getenv("MCO_SHARD_ALGO");  // "p2p": force the per-part path (tests)
  const bool even = total_len % (uint64_t)N == 0 && !(algo && std::string(algo) == "p2p");
  const auto& api = nccl();
  if (even) {
    MCO_NCALL(c, api.reduce_scatter(flat_grads, gdst, parts[me], gt, ncclSum, c->comm, s));
  } else {
    MCO_NCALL(c, api.group_start());
    for (int r = 0; r < N; ++r)
      MCO_NCALL(c, api.reduce((const char*)flat_grads + offs[r] * gs, gdst, parts[r], gt,
                              ncclSum, r, c->comm, s));
    MCO_NCALL(c, api.group_end());
  }
  step(gdst, parts[me], (char*)ag_buf + offs[me] * as);
  if (even) {
    MCO_NCALL(c, api.all_gather((char*)ag_buf + offs[me] * as, ag_buf, parts[me], at,
                                c->comm, s));
  } else {
    MCO_NCALL(c, api.group_start());
    for (int r = 0; r < N; ++r) {
      char* part = (char*)ag_buf + offs[r] * as;
      MCO_NCALL(c, api.broadcast(part, part, parts[r], at, r, c->comm, s));
    }
    MCO_NCALL(c, api.group_end());
  }
}
}  // namespace

extern "C" {

mco_status mco_shard_step(mco_flat* h, mco_comm* c, void* flat_params, int param_dtype,
                          const void* flat_grads, int grad_dtype, uint64_t total_len, double lr,
                          void* stream) {
  return guard([&] {
    if (!h || !c) throw Error(MCO_CONTRACT, "mco_shard_step: null handle");
    const size_t ps = dt_size(param_dtype);
    std::vector<uint64_t> parts(c->nranks), offs(c->nranks + 1);
    if (mco_zero_plan(total_len, c->nranks, 2, parts.data(), offs.data()) != MCO_OK)
      throw Error(MCO_CONFIG, "shard step: zero plan");
    const char* mine = (const char*)flat_params + offs[c->rank] * ps;
    shard_run(h, c, flat_grads, grad_dtype, total_len, flat_params, param_dtype, mine, ps,
              stream, [&](void* g, uint64_t n, void* p_owned) {
                const mco_status st =
                    mco_flat_step(h, p_owned, param_dtype, n, g, grad_dtype, n, lr, stream);
                if (st != MCO_OK) throw Error(st, mco_last_error());
              });
  });
}

// Mixed-precision stage 2: fp32 master + state for the owned part,
// bf16 replicas.  RS(grads) -> mco_flat_step_mixed(master, g, bf16 replica slice) ->
// AG of the bf16 replicas (2 B/param on the wire instead of 4).
mco_status mco_shard_step_mixed(mco_flat* h, mco_comm* c, float* master_owned,
                                uint16_t* flat_params_bf16, const void* flat_grads,
                                int grad_dtype, uint64_t total_len, double lr, void* stream) {
  return guard([&] {
    if (!h || !c) throw Error(MCO_CONTRACT, "mco_shard_step_mixed: null handle");
    if (!master_owned) throw Error(MCO_CONTRACT, "shard step: null master");
    shard_run(h, c, flat_grads, grad_dtype, total_len, flat_params_bf16, MCO_BF16,
              master_owned, sizeof(float), stream,
              [&](void* g, uint64_t n, void* replica_owned) {
                const mco_status st = mco_flat_step_mixed(h, master_owned, g, grad_dtype,
                                                          (uint16_t*)replica_owned, n, lr,
                                                          stream);
                if (st != MCO_OK) throw Error(st, mco_last_error());
              });
  });
}

}  // extern "C"

// ---- bucketed, double-buffered ZeRO step --------------------------
// Buckets: [k B, min(P, (k+1) B)) of the registry-order flat vector, B rounded up to a
// multiple of 8 N.  Inside bucket k, rank i owns piece i of ZeroPlan(len_k, N)
// (parallel.cpp:20-34 applied per bucket): every rank updates its share of every
// bucket, so all ranks work on bucket k while bucket k+1 is being reduced.  The update
// is elementwise, so the gathered parameters equal the whole-vector ZeroPlan step's
// (and the serial FlatOptimizer's on the summed gradient); the state of rank i is its
// pieces in bucket order (mco_zb_piece maps them back to registry offsets).  With
// bucket_elems >= P there is one bucket and the ownership is ZeroPlan's exactly.
struct mco_zb {
  mco_comm* comm = nullptr;
  mco_flat* flat = nullptr;  // state of this rank's pieces, bucket order
  uint64_t P = 0, B = 0;
  int nb = 0;
  int gdt = MCO_F32, rdt = MCO_F32;  // gradient / replica dtypes
  bool mixed = false;                 // bf16 replicas + fp32 master
  float* master = nullptr;            // fp32 master of this rank's pieces (mixed)
  std::vector<uint64_t> state_off;    // per bucket: this rank's piece in the state
  cudaStream_t cs = nullptr, us = nullptr;  // comm stream, update stream
  void* stage[2] = {nullptr, nullptr};      // gradient staging buckets (lazy)
  void* red[2] = {nullptr, nullptr};        // reduced pieces
  cudaEvent_t ev_grad = nullptr, ev_rs[2] = {}, ev_upd[2] = {}, ev_stage_free[2] = {},
              ev_done = nullptr;
  // ring mode (begin with replicas == NULL; bf16 replicas only): no full replica is
  // resident -- bucket k is gathered into ring slot k mod 2 (the stage-3 layout: fp32
  // master + state of the owned pieces persist, parameters are gathered on demand)
  bool ring = false;
  void* ring_buf[2] = {nullptr, nullptr};
  cudaEvent_t ev_ag[2] = {};
  // step state
  bool open = false;
  double lr = 0;
  void* replicas = nullptr;
  int last = -1;   // bucket whose all-gather is still to be issued
  int issued = 0;  // buckets reduced this step
  std::vector<char> seen;

  uint64_t len(int k) const { return std::min(P, (uint64_t)(k + 1) * B) - (uint64_t)k * B; }
  void piece(int k, int r, uint64_t* off, uint64_t* n) const {
    const uint64_t L = len(k), N = (uint64_t)comm->nranks, q = L / N, rem = L % N;
    *off = (uint64_t)r * q + std::min<uint64_t>((uint64_t)r, rem);
    *n = q + ((uint64_t)r < rem ? 1 : 0);
  }
  ~mco_zb() {
    for (void* p : {stage[0], stage[1], red[0], red[1], (void*)master, ring_buf[0], ring_buf[1]})
      if (p) cudaFree(p);
    for (cudaEvent_t e : {ev_grad, ev_rs[0], ev_rs[1], ev_upd[0], ev_upd[1], ev_stage_free[0],
                          ev_stage_free[1], ev_done, ev_ag[0], ev_ag[1]})
      if (e) cudaEventDestroy(e);
    if (cs) cudaStreamDestroy(cs);
    if (us) cudaStreamDestroy(us);
    if (flat) mco_flat_destroy(flat);
  }

  // bucket k's parameters: its range of the replicas, or its ring slot
  char* bucket_base(int k) const {
    return ring ? (char*)ring_buf[k % 2] : (char*)replicas + (uint64_t)k * B * dt_size(rdt);
  }

  // all-gather of bucket k's replicas (after its update) on the comm stream
  void all_gather(int k) {
    const int N = comm->nranks, me = comm->rank;
    const size_t rs = dt_size(rdt);
    MCO_CUDA_CHECK(cudaStreamWaitEvent(cs, ev_upd[k % 2], 0));
    char* base = bucket_base(k);
    const auto& api = nccl();
    const ncclDataType_t at = nccl_type(rdt);
    if (len(k) % (uint64_t)N == 0) {
      uint64_t off, n;
      piece(k, me, &off, &n);
      MCO_NCALL(comm, api.all_gather(base + off * rs, base, n, at, comm->comm, cs));
    } else {
      MCO_NCALL(comm, api.group_start());
      for (int r = 0; r < N; ++r) {
        uint64_t off, n;
        piece(k, r, &off, &n);
        MCO_NCALL(comm, api.broadcast(base + off * rs, base + off * rs, n, at, r, comm->comm,
                                      cs));
      }
      MCO_NCALL(comm, api.group_end());
    }
    if (ring) MCO_CUDA_CHECK(cudaEventRecord(ev_ag[k % 2], cs));
  }
};

extern "C" {

// The bucket plan alone (host arithmetic, no communicator): the rounded bucket size,
// the bucket count, and piece `rank` of bucket k.
mco_status mco_zb_plan(uint64_t total_len, int nranks, uint64_t bucket_elems, int k, int rank,
                       uint64_t* bucket_rounded, int* nbuckets, uint64_t* bucket_off,
                       uint64_t* bucket_len, uint64_t* off, uint64_t* n) {
  return guard([&] {
    if (nranks < 1 || total_len == 0)
      throw Error(MCO_CONFIG, "bucket plan: needs >= 1 rank and a non-empty set");
    const uint64_t unit = 8 * (uint64_t)nranks;
    uint64_t B = bucket_elems ? std::min<uint64_t>(bucket_elems, total_len) : total_len;
    B = (B + unit - 1) / unit * unit;
    const int nb = (int)((total_len + B - 1) / B);
    if (bucket_rounded) *bucket_rounded = B;
    if (nbuckets) *nbuckets = nb;
    if (k < 0 || k >= nb || rank < 0 || rank >= nranks)
      throw Error(MCO_CONTRACT, "bucket plan: bucket / rank out of range");
    const uint64_t L = std::min(total_len, (uint64_t)(k + 1) * B) - (uint64_t)k * B;
    const uint64_t q = L / nranks, rem = L % nranks;
    if (bucket_off) *bucket_off = (uint64_t)k * B;
    if (bucket_len) *bucket_len = L;
    if (off) *off = (uint64_t)rank * q + std::min<uint64_t>((uint64_t)rank, rem);
    if (n) *n = q + ((uint64_t)rank < rem ? 1 : 0);
  });
}

mco_status mco_zb_create(const mco_config* cfg, mco_comm* c, uint64_t total_len,
                         uint64_t bucket_elems, int grad_dtype, int replica_dtype,
                         mco_zb** out) {
  return guard([&] {
    if (!cfg || !c || !out) throw Error(MCO_CONTRACT, "mco_zb_create: null argument");
    *out = nullptr;
    if (fused(cfg->kind))
      throw Error(MCO_CONTRACT, "bucketed shard step: " + kind_str(cfg->kind) +
                                    " is a fused optimizer and keeps no flat state");
    if (grad_dtype != MCO_F32 && grad_dtype != MCO_BF16)
      throw Error(MCO_CONTRACT, "bucketed shard step: gradients must be f32 or bf16");
    if (replica_dtype != MCO_F32 && replica_dtype != MCO_BF16)
      throw Error(MCO_CONTRACT, "bucketed shard step: replicas must be f32 or bf16");
    if (total_len == 0) throw Error(MCO_CONTRACT, "bucketed shard step: empty parameter set");
    DeviceGuard dg(c->device);
    auto z = std::make_unique<mco_zb>();
    z->comm = c;
    z->P = total_len;
    const uint64_t unit = 8 * (uint64_t)c->nranks;
    uint64_t B = bucket_elems ? std::min<uint64_t>(bucket_elems, total_len) : total_len;
    B = (B + unit - 1) / unit * unit;
    z->B = B;
    z->nb = (int)((total_len + B - 1) / B);
    z->gdt = grad_dtype;
    z->rdt = replica_dtype;
    z->mixed = replica_dtype == MCO_BF16;
    uint64_t own = 0, pmax = 0;
    z->state_off.resize(z->nb);
    for (int k = 0; k < z->nb; ++k) {
      uint64_t off, n;
      z->piece(k, c->rank, &off, &n);
      z->state_off[k] = own;
      own += n;
      z->piece(k, 0, &off, &n);  // rank 0's piece is the largest of the bucket
      pmax = std::max(pmax, n);
    }
    mco_flat* h = nullptr;
    const mco_status st = mco_flat_create(cfg, own, c->device, MCO_F32, &h);
    if (st != MCO_OK) throw Error(st, mco_last_error());
    z->flat = h;
    if (z->mixed) MCO_CUDA_CHECK(cudaMalloc(&z->master, (std::max<uint64_t>(own, 1) + 8) * 4));
    for (auto& r : z->red) MCO_CUDA_CHECK(cudaMalloc(&r, (pmax + 8) * dt_size(grad_dtype)));
    MCO_CUDA_CHECK(cudaStreamCreateWithFlags(&z->cs, cudaStreamNonBlocking));
    MCO_CUDA_CHECK(cudaStreamCreateWithFlags(&z->us, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&z->ev_grad, &z->ev_rs[0], &z->ev_rs[1], &z->ev_upd[0],
                           &z->ev_upd[1], &z->ev_stage_free[0], &z->ev_stage_free[1],
                           &z->ev_done})
      MCO_CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    *out = z.release();
  });
}

mco_status mco_zb_destroy(mco_zb* z) {
  return guard([&] {
    if (!z) return;
    DeviceGuard dg(z->comm->device);
    cudaStreamSynchronize(z->cs);
    cudaStreamSynchronize(z->us);
    delete z;
  });
}

// Layout: the (rounded) bucket size and count, this rank's owned element count, its
// state handle (named buffers m, v, n, h, g_prev over its pieces; steps) and the fp32
// master (mixed mode, else null).
mco_status mco_zb_info(const mco_zb* z, uint64_t* bucket_elems, int* nbuckets,
                       uint64_t* owned, mco_flat** flat, float** master) {
  return guard([&] {
    if (!z) throw Error(MCO_CONTRACT, "mco_zb_info: null handle");
    if (bucket_elems) *bucket_elems = z->B;
    if (nbuckets) *nbuckets = z->nb;
    if (owned) *owned = z->flat->n;
    if (flat) *flat = z->flat;
    if (master) *master = z->master;
  });
}

// Piece of rank r in bucket k: registry elements [bucket_off + off, + n); state_off =
// its offset in this rank's state (UINT64_MAX for other ranks).
mco_status mco_zb_piece(const mco_zb* z, int k, int rank, uint64_t* bucket_off,
                        uint64_t* bucket_len, uint64_t* off, uint64_t* n,
                        uint64_t* state_off) {
  return guard([&] {
    if (!z || !bucket_off || !bucket_len || !off || !n)
      throw Error(MCO_CONTRACT, "mco_zb_piece: null argument");
    if (k < 0 || k >= z->nb || rank < 0 || rank >= z->comm->nranks)
      throw Error(MCO_CONTRACT, "bucketed shard step: bucket / rank out of range");
    z->piece(k, rank, off, n);
    *bucket_off = (uint64_t)k * z->B;
    *bucket_len = z->len(k);
    if (state_off) *state_off = rank == z->comm->rank ? z->state_off[k] : UINT64_MAX;
  });
}

// Mixed mode: the fp32 master of this rank's pieces from a full registry-order buffer
// (f32, or bf16 widened exactly), stream-ordered.
mco_status mco_zb_load_master(mco_zb* z, const void* full, int dtype, void* stream) {
  return guard([&] {
    if (!z || !full) throw Error(MCO_CONTRACT, "mco_zb_load_master: null argument");
    if (!z->mixed) throw Error(MCO_CONTRACT, "bucketed shard step: no master (f32 replicas)");
    if (dtype != MCO_F32 && dtype != MCO_BF16)
      throw Error(MCO_CONTRACT, "bucketed shard step: master source must be f32 or bf16");
    DeviceGuard dg(z->comm->device);
    for (int k = 0; k < z->nb; ++k) {
      uint64_t off, n;
      z->piece(k, z->comm->rank, &off, &n);
      const uint64_t src = (uint64_t)k * z->B + off;
      if (dtype == MCO_F32) {
        MCO_CUDA_CHECK(cudaMemcpyAsync(z->master + z->state_off[k], (const float*)full + src,
                                       n * 4, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
      } else {
        widen_bf16(z->master + z->state_off[k], (const uint16_t*)full + src, n,
                   (cudaStream_t)stream);
      }
    }
  });
}

// Begin a step: ++t of the owned state (optim.cpp:104); `replicas` (replica dtype, P
// elements, registry order) receive the gathered parameters -- or, NULL (bf16 replicas
// only), ring mode: bucket k is gathered into ring slot k mod 2 (mco_zb_gathered).
mco_status mco_zb_begin(mco_zb* z, void* replicas, double lr, void* stream) {
  return guard([&] {
    if (!z) throw Error(MCO_CONTRACT, "mco_zb_begin: null handle");
    if (!replicas && !z->mixed)
      throw Error(MCO_CONTRACT, "bucketed shard step: ring mode (no replicas) needs bf16 "
                                "replicas over an fp32 master");
    if (z->open) throw Error(MCO_CONTRACT, "bucketed shard step: step already open");
    if (z->flat->gdev) throw Error(MCO_CONTRACT, "bucketed shard step: graph mode unsupported");
    DeviceGuard dg(z->comm->device);
    z->ring = replicas == nullptr;
    if (z->ring && !z->ring_buf[0])
      for (int s = 0; s < 2; ++s) {
        MCO_CUDA_CHECK(cudaMalloc(&z->ring_buf[s], z->B * dt_size(z->rdt)));
        MCO_CUDA_CHECK(cudaEventCreateWithFlags(&z->ev_ag[s], cudaEventDisableTiming));
      }
    ++z->flat->t;
    z->flat->stepped = true;
    z->open = true;
    z->lr = lr;
    z->replicas = replicas;
    z->last = -1;
    z->issued = 0;
    z->seen.assign(z->nb, 0);
    // the caller's prior work (replica / master writes) happens-before the step
    MCO_CUDA_CHECK(cudaEventRecord(z->ev_grad, (cudaStream_t)stream));
    MCO_CUDA_CHECK(cudaStreamWaitEvent(z->cs, z->ev_grad, 0));
    MCO_CUDA_CHECK(cudaStreamWaitEvent(z->us, z->ev_grad, 0));
  });
}

// Staging buffer for bucket k's local gradient (len(k) elements of the gradient dtype,
// slot k mod 2); `stream` waits until the slot's previous bucket has been reduced.
mco_status mco_zb_grad_buffer(mco_zb* z, int k, void** ptr, uint64_t* len, void* stream) {
  return guard([&] {
    if (!z || !ptr) throw Error(MCO_CONTRACT, "mco_zb_grad_buffer: null argument");
    if (k < 0 || k >= z->nb) throw Error(MCO_CONTRACT, "bucketed shard step: bucket out of range");
    DeviceGuard dg(z->comm->device);
    const int s = k % 2;
    if (!z->stage[s]) {
      MCO_CUDA_CHECK(cudaMalloc(&z->stage[s], z->B * dt_size(z->gdt)));
      MCO_CUDA_CHECK(cudaEventRecord(z->ev_stage_free[s], z->cs));
    }
    MCO_CUDA_CHECK(cudaStreamWaitEvent((cudaStream_t)stream, z->ev_stage_free[s], 0));
    *ptr = z->stage[s];
    if (len) *len = z->len(k);
  });
}

// Bucket k's local gradient is complete on `stream` (at `grad`, or in its staging slot
// when grad is null): reduce-scatter on the comm stream, the piece's update on the
// update stream, then the previous bucket's all-gather (issued after this bucket's
// reduce-scatter, so that reduce-scatter overlaps the previous update).  Every rank
// must hand in the buckets in the same order (NCCL's per-communicator ordering).
mco_status mco_zb_grad_ready(mco_zb* z, int k, const void* grad, void* stream) {
  return guard([&] {
    if (!z) throw Error(MCO_CONTRACT, "mco_zb_grad_ready: null handle");
    if (!z->open) throw Error(MCO_CONTRACT, "bucketed shard step: mco_zb_begin first");
    if (k < 0 || k >= z->nb || z->seen[k])
      throw Error(MCO_CONTRACT, "bucketed shard step: bucket " + std::to_string(k) +
                                    " out of range or already reduced this step");
    const int s = k % 2;
    if (!grad) {
      if (!z->stage[s]) throw Error(MCO_CONTRACT, "bucketed shard step: no staged gradient");
      grad = z->stage[s];
    }
    DeviceGuard dg(z->comm->device);
    z->seen[k] = 1;
    const int N = z->comm->nranks, me = z->comm->rank;
    const size_t gs = dt_size(z->gdt), rs = dt_size(z->rdt);
    uint64_t off, n;
    z->piece(k, me, &off, &n);
    // the reduced piece takes the phase (mod 8 elements) of the parameters it updates
    const uint64_t pel = (uint64_t)k * z->B + off;
    char* rpiece = z->bucket_base(k) + off * rs;  // this rank's piece of the replicas
    const char* pptr = z->mixed ? (const char*)(z->master + z->state_off[k]) : rpiece;
    const size_t pes = z->mixed ? 4 : rs;
    const size_t phase = ((uintptr_t)pptr / pes) % 8;
    char* red = (char*)z->red[s] + phase * gs;
    MCO_CUDA_CHECK(cudaEventRecord(z->ev_grad, (cudaStream_t)stream));
    MCO_CUDA_CHECK(cudaStreamWaitEvent(z->cs, z->ev_grad, 0));
    const auto& api = nccl();
    const ncclDataType_t gt = nccl_type(z->gdt);
    if (z->len(k) % (uint64_t)N == 0) {
      MCO_NCALL(z->comm, api.reduce_scatter(grad, red, n, gt, ncclSum, z->comm->comm, z->cs));
    } else {
      MCO_NCALL(z->comm, api.group_start());
      for (int r = 0; r < N; ++r) {
        uint64_t o, m;
        z->piece(k, r, &o, &m);
        MCO_NCALL(z->comm, api.reduce((const char*)grad + o * gs, red, m, gt, ncclSum, r,
                                      z->comm->comm, z->cs));
      }
      MCO_NCALL(z->comm, api.group_end());
    }
    MCO_CUDA_CHECK(cudaEventRecord(z->ev_rs[s], z->cs));
    if (grad == z->stage[s]) MCO_CUDA_CHECK(cudaEventRecord(z->ev_stage_free[s], z->cs));
    // this rank's piece: fused update (and the bf16 replica write in mixed mode)
    MCO_CUDA_CHECK(cudaStreamWaitEvent(z->us, z->ev_rs[s], 0));
    if (z->mixed) {
      flat_step_range(z->flat, z->master + z->state_off[k], MCO_F32, red, z->gdt,
                      (uint16_t*)rpiece, n, z->state_off[k], z->lr, z->us);
    } else {
      flat_step_range(z->flat, rpiece, MCO_F32, red, z->gdt, nullptr, n, z->state_off[k],
                      z->lr, z->us);
    }
    (void)pel;
    MCO_CUDA_CHECK(cudaEventRecord(z->ev_upd[s], z->us));
    if (z->last >= 0) z->all_gather(z->last);
    z->last = k;
    ++z->issued;
  });
}

// End the step: the last all-gather, then `stream` waits for every collective.
mco_status mco_zb_end(mco_zb* z, void* stream) {
  return guard([&] {
    if (!z) throw Error(MCO_CONTRACT, "mco_zb_end: null handle");
    if (!z->open) throw Error(MCO_CONTRACT, "bucketed shard step: no open step");
    z->open = false;
    if (z->issued != z->nb)
      throw Error(MCO_CONTRACT, "bucketed shard step: " + std::to_string(z->issued) + " of " +
                                    std::to_string(z->nb) + " buckets reduced");
    DeviceGuard dg(z->comm->device);
    if (z->last >= 0) z->all_gather(z->last);
    MCO_CUDA_CHECK(cudaEventRecord(z->ev_done, z->cs));
    MCO_CUDA_CHECK(cudaStreamWaitEvent((cudaStream_t)stream, z->ev_done, 0));
  });
}

// Ring mode: bucket k's gathered parameters (ring slot k mod 2, len_k bf16 elements);
// `stream` waits for its all-gather.  Valid until bucket k+2's update overwrites the slot.
mco_status mco_zb_gathered(mco_zb* z, int k, void** ptr, void* stream) {
  return guard([&] {
    if (!z || !ptr) throw Error(MCO_CONTRACT, "mco_zb_gathered: null argument");
    if (!z->ring) throw Error(MCO_CONTRACT, "bucketed shard step: not in ring mode");
    if (k < 0 || k >= z->nb) throw Error(MCO_CONTRACT, "bucketed shard step: bucket out of range");
    DeviceGuard dg(z->comm->device);
    MCO_CUDA_CHECK(cudaStreamWaitEvent((cudaStream_t)stream, z->ev_ag[k % 2], 0));
    *ptr = z->ring_buf[k % 2];
  });
}

// The same step's update kernels without the collectives (every piece updated from this
// rank's own local gradient, on the caller's stream): the shard-local cost the
// collectives are added to (bench.py reports it beside the whole step).
mco_status mco_zb_step_local(mco_zb* z, void* replicas, const void* flat_grads, double lr,
                             void* stream) {
  return guard([&] {
    if (!z || !replicas || !flat_grads)
      throw Error(MCO_CONTRACT, "mco_zb_step_local: null argument");
    if (z->open) throw Error(MCO_CONTRACT, "bucketed shard step: step already open");
    DeviceGuard dg(z->comm->device);
    ++z->flat->t;
    z->flat->stepped = true;
    const size_t gs = dt_size(z->gdt), rs = dt_size(z->rdt);
    for (int k = z->nb - 1; k >= 0; --k) {
      uint64_t off, n;
      z->piece(k, z->comm->rank, &off, &n);
      const uint64_t pel = (uint64_t)k * z->B + off;
      const char* g = (const char*)flat_grads + pel * gs;
      char* rp = (char*)replicas + pel * rs;
      if (z->mixed)
        flat_step_range(z->flat, z->master + z->state_off[k], MCO_F32, g, z->gdt,
                        (uint16_t*)rp, n, z->state_off[k], lr, (cudaStream_t)stream);
      else
        flat_step_range(z->flat, rp, MCO_F32, g, z->gdt, nullptr, n, z->state_off[k], lr,
                        (cudaStream_t)stream);
    }
  });
}

// The whole step from a full local gradient buffer: buckets in reverse registry order,
// as backward produces them.
mco_status mco_zb_step(mco_zb* z, void* replicas, const void* flat_grads, double lr,
                       void* stream) {
  return guard([&] {
    if (!z || !flat_grads) throw Error(MCO_CONTRACT, "mco_zb_step: null argument");
    auto chk = [](mco_status s) {
      if (s != MCO_OK) throw Error(s, mco_last_error());
    };
    chk(mco_zb_begin(z, replicas, lr, stream));
    const size_t gs = dt_size(z->gdt);
    for (int k = z->nb - 1; k >= 0; --k)
      chk(mco_zb_grad_ready(z, k, (const char*)flat_grads + (uint64_t)k * z->B * gs, stream));
    chk(mco_zb_end(z, stream));
  });
}

}  // extern "C"
