// Native ZeRO sharder over NCCL (SURVEY 8(b) "mco_shard_step", 8(e)): the stage-2
// branch of ParallelWorker::train_step (parallel.cpp:656-666) as one C-ABI call,
//
//   owned_grads = reduce_scatter(flat_grads, SUM, ZeroPlan parts)   parallel.cpp:657-658
//   FlatOptimizer::step(params[owned], owned_grads, lr)             parallel.cpp:660
//   params      = all_gather(params[owned])                         parallel.cpp:661-663
//
// stream-ordered on the caller's stream, so a C / C++ host (the reference's own
// parallel engine) gets the sharded step without torch.  Equal ZeroPlan parts use
// ncclReduceScatter / ncclAllGather (in place); unequal parts (P mod N != 0: the first
// P mod N ranks own one more element, parallel.cpp:25-32) use one ncclReduce and one
// ncclBroadcast per part inside a group, which keeps the reference's ownership.
//
// NCCL is resolved at run time (dlopen): the libnccl.so.2 already mapped into the
// process (torch's build) is reused, never a second copy; otherwise MCO_NCCL_LIB, then
// the system libnccl.so.2.  libmco.so has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "abi_internal.h"

namespace mco {
namespace {

struct NcclApi {
  void* so = nullptr;
  std::string from;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
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
  sym(so, "ncclCommInitRank", a.comm_init_rank);
  sym(so, "ncclCommDestroy", a.comm_destroy);
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
  if (r != ncclSuccess)
    throw Error(MCO_PROTOCOL, std::string(what) + ": " + nccl().get_error_string(r));
}
#define MCO_NCCL_CHECK(x) nccl_check((x), #x)

ncclDataType_t nccl_type(int dt) {
  switch (dt) {
    case MCO_F32: return ncclFloat32;
    case MCO_BF16: return ncclBfloat16;
    case MCO_F64: return ncclFloat64;
  }
  throw Error(MCO_CONTRACT, "NCCL: unsupported dtype " + std::to_string(dt));
}

size_t dt_size(int dt) { return dt == MCO_F64 ? 8 : dt == MCO_BF16 ? 2 : 4; }


}  // namespace
}  // namespace mco

using namespace mco;

struct mco_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
  void* scratch = nullptr;  // reduced owned gradient (ZeroPlan part of this rank)
  size_t scratch_bytes = 0;
  ~mco_comm() {
    if (scratch) cudaFree(scratch);
    if (comm) nccl().comm_destroy(comm);
  }
};

extern "C" {

mco_status mco_comm_unique_id(void* id_out) {
  return guard([&] {
    if (!id_out) throw Error(MCO_CONTRACT, "comm unique id: null output");
    ncclUniqueId id;
    MCO_NCCL_CHECK(nccl().get_unique_id(&id));
    std::memcpy(id_out, &id, sizeof(id));
  });
}

mco_status mco_comm_create(const void* id, int nranks, int rank, int device, mco_comm** out) {
  return guard([&] {
    if (!id || !out) throw Error(MCO_CONTRACT, "comm create: null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks)
      throw Error(MCO_CONFIG, "comm create: rank " + std::to_string(rank) + " of " +
                                  std::to_string(nranks));
    device = resolve_device(device);
    DeviceGuard ds(device);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    auto* c = new mco_comm;
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    const ncclResult_t r = nccl().comm_init_rank(&c->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
      c->comm = nullptr;
      delete c;
      nccl_check(r, "ncclCommInitRank");
    }
    *out = c;
  });
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
    ncclResult_t r = ncclSuccess;
    MCO_NCCL_CHECK(nccl().comm_get_async_error(c->comm, &r));
    nccl_check(r, "NCCL asynchronous error");
  });
}

mco_status mco_comm_allreduce_sum(mco_comm* c, void* buf, int dtype, uint64_t n, void* stream) {
  return guard([&] {
    if (!c) throw Error(MCO_CONTRACT, "mco_comm_allreduce_sum: null handle");
    DeviceGuard ds(c->device);
    MCO_NCCL_CHECK(nccl().all_reduce(buf, buf, n, nccl_type(dtype), ncclSum, c->comm,
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
    MCO_NCCL_CHECK(api.reduce_scatter(flat_grads, gdst, parts[me], gt, ncclSum, c->comm, s));
  } else {
    MCO_NCCL_CHECK(api.group_start());
    for (int r = 0; r < N; ++r)
      MCO_NCCL_CHECK(api.reduce((const char*)flat_grads + offs[r] * gs, gdst, parts[r], gt,
                                ncclSum, r, c->comm, s));
    MCO_NCCL_CHECK(api.group_end());
  }
  step(gdst, parts[me], (char*)ag_buf + offs[me] * as);
  if (even) {
    MCO_NCCL_CHECK(api.all_gather((char*)ag_buf + offs[me] * as, ag_buf, parts[me], at,
                                  c->comm, s));
  } else {
    MCO_NCCL_CHECK(api.group_start());
    for (int r = 0; r < N; ++r) {
      char* part = (char*)ag_buf + offs[r] * as;
      MCO_NCCL_CHECK(api.broadcast(part, part, parts[r], at, r, c->comm, s));
    }
    MCO_NCCL_CHECK(api.group_end());
  }
}
}  // namespace

extern "C" {

mco_status mco_shard_step(mco_flat* h, mco_comm* c, void* flat_params, int param_dtype,
                          const void* flat_grads, int grad_dtype, uint64_t total_len, double lr,
                          void* stream) {
  return guard([&] {
    if (!h || !c) throw Error(MCO_CONTRACT, "mco_shard_step: null handle");
    if (!c) throw Error(MCO_CONTRACT, "shard step: null argument");
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
