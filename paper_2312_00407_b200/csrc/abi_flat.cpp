// C-ABI: FlatOptimizer (optim.cpp:74-181), LOMO (optim.cpp:185-190, 291-303) and the
// ZeRO step fused with its collectives over peer memory (parallel.cpp:656-666).
#include "abi_internal.h"

using namespace mco;

extern "C" {

// ---- FlatOptimizer ---------------------------------------------------------------
// optim.cpp:74-98
mco_status mco_flat_create(const mco_config* cfg, uint64_t owned_len, int device,
                           int state_dtype, mco_flat** out) {
  return guard([&] {
    *out = nullptr;
    if (fused(cfg->kind))
      throw Error(MCO_CONTRACT, "FlatOptimizer: " + kind_str(cfg->kind) +
                                    " is a fused optimizer and keeps no flat state");
    kind_str(cfg->kind);
    // the reference's Sophia evaluates (t - 1) % update_interval every step
    // (optim.cpp:161): an interval < 1 would divide by zero there and on the device here
    if (cfg->kind == MCO_SOPHIA && cfg->update_interval < 1)
      throw Error(MCO_CONFIG, "optimizer: update_interval must be >= 1");
    if (state_dtype != MCO_F32 && state_dtype != MCO_F64 && state_dtype != MCO_F32M64)
      throw Error(MCO_CONTRACT, "FlatOptimizer: state dtype must be f32, f64 or f32m64");
    if (state_dtype == MCO_F32M64 && cfg->kind != MCO_SOPHIA)
      throw Error(MCO_CONTRACT, "FlatOptimizer: the fp64-m state (precise-m) is Sophia's");
    device = resolve_device(device);
    DeviceGuard dg(device);
    auto h = std::make_unique<mco_flat>();
    h->cfg = *cfg;
    h->n = owned_len;
    h->device = device;
    h->state_dtype = state_dtype;
    // slots s0..s3 and the reference's buffers() names / order (optim.cpp:173-181)
    const char* names[4] = {nullptr, nullptr, nullptr, nullptr};
    int nslots = 0;
    switch (cfg->kind) {
      case MCO_ADAMW: names[0] = "m"; names[1] = "v"; nslots = 2; break;
      case MCO_LION: names[0] = "m"; nslots = 1; break;
      case MCO_ADAN: names[0] = "m"; names[1] = "v"; names[2] = "n"; names[3] = "g_prev";
        nslots = 4; break;
      case MCO_SOPHIA: names[0] = "m"; names[1] = "h"; nslots = 2; break;
    }
    // 8 elements of slack: the state is shifted to the parameters' alignment phase at
    // the first step (align_state_to), so shard views at odd offsets stay vectorised
    for (int i = 0; i < nslots; ++i) {
      const size_t bytes = (std::max<uint64_t>(owned_len, 1) + 8) * h->slot_es(i);
      MCO_CUDA_CHECK(cudaMalloc(&h->base[i], bytes));
      MCO_CUDA_CHECK(cudaMemset(h->base[i], 0, bytes));
      h->slot[i] = h->base[i];
      h->named.emplace_back(names[i], h->slot[i]);
    }
    *out = h.release();
  });
}

mco_status mco_flat_destroy(mco_flat* h) {
  return guard([&] {
    if (!h) return;
    DeviceGuard dg(h->device);
    delete h;
  });
}

namespace {
// n > 0 elements behind a null pointer would fault on the device: a contract error
void check_data(uint64_t n, const void* a, const void* b, const char* what) {
  if (n && (!a || !b)) throw Error(MCO_CONTRACT, std::string(what) + ": null data pointer");
}

void check_lengths(const mco_flat* h, uint64_t np, uint64_t ng) {
  if (np != ng)  // optim.cpp:101-103
    throw Error(MCO_CONTRACT, "optimizer step: params/grads length mismatch: " +
                                  std::to_string(np) + " vs " + std::to_string(ng));
  if (np > h->n)
    throw Error(MCO_CONTRACT, "optimizer step: " + std::to_string(np) +
                                  " elements exceed the owned state of " + std::to_string(h->n));
}

// Before the first step (state still all zero, never handed out) the state buffers are
// shifted within their slack so that state[i] has the same address phase (mod 8
// elements) as params[i]: the launch can then peel a short head and run the rest
// aligned (flat.cu, launch_flat_step).
void align_state_to(mco_flat* h, const void* params) {
  if (h->exposed || h->stepped || h->t != 0 || !params) return;
  const size_t es = h->state_dtype == MCO_F64 ? 8 : 4;  // the parameters' element size
  const uintptr_t u = (uintptr_t)params;
  if (u % es) return;
  const int want = (int)((u / es) % 8);
  if (want == h->phase) return;
  h->phase = want;
  for (int i = 0; i < 4; ++i)
    if (h->base[i]) h->slot[i] = (char*)h->base[i] + (size_t)want * h->slot_es(i);
  for (size_t i = 0; i < h->named.size(); ++i) h->named[i].second = h->slot[i];
}

// Graph mode: the kernels read t and advance it (common.cuh); eager: empty.
GraphStep graph_step(const mco_flat* h, double lr) {
  GraphStep gs{};
  if (!h->gdev) return gs;
  gs.d = h->gdev;
  gs.rows = h->state_dtype == MCO_F64 ? (const void*)h->grow_d : (const void*)h->grow_f;
  gs.nrows = h->grows;
  gs.lr = h->glr;
  gs.lr_host = lr;
  gs.wd = h->cfg.weight_decay;
  gs.interval = h->cfg.update_interval;
  gs.bump = 1;
  return gs;
}

void flat_launch(mco_flat* h, void* p, int pdt, const void* g, int gdt, uint16_t* pout,
                 uint64_t n, uint64_t state_off, double lr, cudaStream_t st) {
  FlatArgs a{};
  a.kind = h->cfg.kind;
  a.state_dtype = h->state_dtype;
  a.p = p;
  a.p_dtype = pdt;
  a.g = g;
  a.g_dtype = gdt;
  for (int i = 0; i < 4; ++i)
    a.s[i] = h->slot[i] ? (char*)h->slot[i] + state_off * h->slot_es(i) : nullptr;
  a.p_out_bf16 = pout;
  a.n = n;
  const auto kf = make_consts<float>(h->cfg, h->t, lr);
  const auto kd = make_consts<double>(h->cfg, h->t, lr);
  a.gs = graph_step(h, lr);
  if (h->state_dtype == MCO_F32M64) {  // Sophia precise-m (sophia_m64.cu)
    if (pout || a.gs.d)
      throw Error(MCO_CONTRACT, "precise-m Sophia: no mixed / graph-mode step");
    launch_sophia_m64((float*)p, g, gdt, (double*)a.s[0], (float*)a.s[1], n, kd, st);
  } else {
    launch_flat_step(a, kf, kd, st);
  }
  h->stepped = true;
}

void no_m64(const mco_flat* h, const char* what) {
  if (h->state_dtype == MCO_F32M64)
    throw Error(MCO_CONTRACT, std::string(what) + ": not available for the precise-m (f32m64) "
                              "state");
}

void no_graph(const mco_flat* h, const char* what) {
  if (h->gdev)
    throw Error(MCO_CONTRACT, std::string(what) + ": not available in graph mode "
                              "(mco_flat_graph_disable first)");
}

// Device step counter <-> host (graph mode); the device may still be running steps.
int64_t graph_steps(const mco_flat* h) {
  int64_t t = 0;
  MCO_CUDA_CHECK(cudaDeviceSynchronize());
  MCO_CUDA_CHECK(cudaMemcpy(&t, &h->gdev->t, sizeof(t), cudaMemcpyDeviceToHost));
  return t;
}

void check_dtypes(const mco_flat* h, int pdt, int gdt) {
  if (h->state_dtype == MCO_F64) {
    if (pdt != MCO_F64 || gdt != MCO_F64)
      throw Error(MCO_CONTRACT, "optimizer step: f64 state takes f64 params and grads");
  } else if (pdt != MCO_F32 || (gdt != MCO_F32 && gdt != MCO_BF16)) {
    throw Error(MCO_CONTRACT, "optimizer step: f32 state takes f32 params and f32/bf16 grads");
  }
}
}  // namespace

}  // extern "C"

namespace mco {
// Sharders (shard.cpp): one piece of a step -- params [0, n) against the state slice at
// state_off, at the handle's current step counter (the caller advanced it once for the
// whole step, optim.cpp:104).
void flat_step_range(mco_flat* h, void* p, int pdt, const void* g, int gdt, uint16_t* pout,
                     uint64_t n, uint64_t state_off, double lr, cudaStream_t st) {
  if (state_off + n > h->n)
    throw Error(MCO_CONTRACT, "optimizer step: piece [" + std::to_string(state_off) + ", " +
                                  std::to_string(state_off + n) + ") exceeds the owned state of " +
                                  std::to_string(h->n));
  check_dtypes(h, pdt, gdt);
  no_m64(h, "sharded step");
  if (pout && h->state_dtype != MCO_F32) throw Error(MCO_CONTRACT, "mixed step needs f32 state");
  flat_launch(h, p, pdt, g, gdt, pout, n, state_off, lr, st);
}
}  // namespace mco

extern "C" {

// optim.cpp:100-112
mco_status mco_flat_step(mco_flat* h, void* params, int pdt, uint64_t np, const void* grads,
                         int gdt, uint64_t ng, double lr, void* stream) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_flat_step: null handle");
    check_lengths(h, np, ng);
    check_data(np, params, grads, "optimizer step");
    check_dtypes(h, pdt, gdt);
    DeviceGuard dg(h->device);
    align_state_to(h, params);
    if (!h->gdev) ++h->t;  // optim.cpp:104 (graph mode: on the device)
    flat_launch(h, params, pdt, grads, gdt, nullptr, np, 0, lr, (cudaStream_t)stream);
  });
}

mco_status mco_flat_step_mixed(mco_flat* h, float* master, const void* grads, int gdt,
                               uint16_t* pout, uint64_t n, double lr, void* stream) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_flat_step_mixed: null handle");
    check_lengths(h, n, n);
    check_data(n, master, grads, "mixed step");
    check_dtypes(h, MCO_F32, gdt);
    no_m64(h, "mixed step");
    if (h->state_dtype != MCO_F32) throw Error(MCO_CONTRACT, "mixed step needs f32 state");
    if (!pout) throw Error(MCO_CONTRACT, "mixed step: param_out is null");
    DeviceGuard dg(h->device);
    align_state_to(h, master);
    if (!h->gdev) ++h->t;
    flat_launch(h, master, MCO_F32, grads, gdt, pout, n, 0, lr, (cudaStream_t)stream);
  });
}

// List form (beyond the reference's flat spans): the model's parameter tensors and their
// gradients at separate device pointers, stepped in one launch per kListMax tensors
// over the handle's flat state -- tensor i's state is the slice the flattened vector
// would give it (registry order), so the result and the state equal a flat step over
// the concatenation bit for bit, without the flatten / scatter copies
// (parallel.cpp:468-494).
mco_status mco_flat_step_list(mco_flat* h, int count, void* const* params, int pdt,
                              const void* const* grads, int gdt, const uint64_t* lens,
                              double lr, void* stream) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_flat_step_list: null handle");
    if (count < 0 || (count > 0 && (!params || !grads || !lens)))
      throw Error(MCO_CONTRACT, "step list: null table");
    uint64_t total = 0;
    for (int i = 0; i < count; ++i) {
      if (lens[i] && (!params[i] || !grads[i]))
        throw Error(MCO_CONTRACT, "step list: null tensor " + std::to_string(i));
      total += lens[i];
    }
    if (total > h->n)
      throw Error(MCO_CONTRACT, "step list: " + std::to_string(total) +
                                    " elements exceed the owned state of " + std::to_string(h->n));
    check_dtypes(h, pdt, gdt);
    no_m64(h, "list step");
    DeviceGuard dg(h->device);
    if (count > 0) align_state_to(h, params[0]);
    if (!h->gdev) ++h->t;
    FlatListArgs a{};
    a.kind = h->cfg.kind;
    a.state_dtype = h->state_dtype;
    a.p_dtype = pdt;
    a.g_dtype = gdt;
    a.count = count;
    a.p = params;
    a.g = grads;
    a.len = lens;
    for (int i = 0; i < 4; ++i) a.s[i] = h->slot[i];
    const auto kf = make_consts<float>(h->cfg, h->t, lr);
    const auto kd = make_consts<double>(h->cfg, h->t, lr);
    a.gs = graph_step(h, lr);
    launch_flat_step_list(a, kf, kd, (cudaStream_t)stream);
    h->stepped = true;
  });
}

// Host-span overload: pipelined H2D(p,g) -> step -> D2H(p) over chunks on two
// streams, so PCIe traffic in both directions overlaps the kernels.
mco_status mco_flat_step_host(mco_flat* h, void* params, int pdt, uint64_t np, const void* grads,
                              int gdt, uint64_t ng, double lr) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_flat_step_host: null handle");
    check_lengths(h, np, ng);
    check_data(np, params, grads, "optimizer step");
    check_dtypes(h, pdt, gdt);
    no_graph(h, "host-span step");
    DeviceGuard dg(h->device);
    ++h->t;
    host_pipeline(h->device, params, dtype_size(pdt), grads, dtype_size(gdt), np, true,
                  [&](void* dp, void* dg_, uint64_t off, uint64_t m, cudaStream_t st) {
                    flat_launch(h, dp, pdt, dg_, gdt, nullptr, m, off, lr, st);
                  });
  });
}

mco_status mco_flat_get_steps(const mco_flat* h, int64_t* t) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_flat_get_steps: null handle");
    if (h->gdev) {
      DeviceGuard dg(h->device);
      *t = graph_steps(h);
    } else {
      *t = h->t;
    }
  });
}
mco_status mco_flat_set_steps(mco_flat* h, int64_t t) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_flat_set_steps: null handle");
    h->t = t;
    if (h->gdev) {
      DeviceGuard dg(h->device);
      MCO_CUDA_CHECK(cudaDeviceSynchronize());
      MCO_CUDA_CHECK(cudaMemcpy(&h->gdev->t, &t, sizeof(t), cudaMemcpyHostToDevice));
    }
  });
}

// Graph mode: the step counter moves to the device; the step kernels derive the step's
// scalars from it and the step's last launch advances it (common.cuh step_consts /
// graph_bump), so a step captured into a CUDA graph replays as the next step -- bit-identical to eager steps (the t-dependent scalars are the
// host's own, tabulated up to the step where every 1 - beta_k^t has rounded to 1.0).
mco_status mco_flat_graph_enable(mco_flat* h, const double* dev_lr) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_flat_graph_enable: null handle");
    no_m64(h, "graph mode");
    DeviceGuard dg(h->device);
    if (h->gdev) {  // already on: only the lr source changes
      h->glr = dev_lr;
      return;
    }
    constexpr int64_t kMaxRows = int64_t(1) << 25;
    std::vector<GraphRow<float>> rf(1);
    std::vector<GraphRow<double>> rd(1);
    for (int64_t t = 1;; ++t) {
      const auto f = make_consts<float>(h->cfg, t, 0.0);
      const auto d = make_consts<double>(h->cfg, t, 0.0);
      rf.push_back({f.c1, f.c2, f.c3, f.sthr, f.rc1, f.rc2, f.rc3});
      rd.push_back({d.c1, d.c2, d.c3, d.sthr, d.rc1, d.rc2, d.rc3});
      if (d.c1 == 1.0 && d.c2 == 1.0 && d.c3 == 1.0) break;  // 1 - beta^t is 1.0 from here on
      if (t + 1 >= kMaxRows)
        throw Error(MCO_CONFIG, "graph mode: betas too close to 1 (1 - beta^t still below "
                                "1.0 after 2^25 steps)");
    }
    rf[0] = rf[1];
    rd[0] = rd[1];
    mco_flat g;  // allocation holder: released into h on success
    MCO_CUDA_CHECK(cudaMalloc(&g.gdev, sizeof(FlatGraphDev)));
    MCO_CUDA_CHECK(cudaMalloc(&g.grow_f, rf.size() * sizeof(GraphRow<float>)));
    MCO_CUDA_CHECK(cudaMalloc(&g.grow_d, rd.size() * sizeof(GraphRow<double>)));
    MCO_CUDA_CHECK(cudaDeviceSynchronize());
    FlatGraphDev init{};
    init.t = h->t;
    MCO_CUDA_CHECK(cudaMemcpy(g.gdev, &init, sizeof(init), cudaMemcpyHostToDevice));
    MCO_CUDA_CHECK(cudaMemcpy(g.grow_f, rf.data(), rf.size() * sizeof(GraphRow<float>),
                              cudaMemcpyHostToDevice));
    MCO_CUDA_CHECK(cudaMemcpy(g.grow_d, rd.data(), rd.size() * sizeof(GraphRow<double>),
                              cudaMemcpyHostToDevice));
    h->gdev = g.gdev, h->grow_f = g.grow_f, h->grow_d = g.grow_d;
    h->grows = (int64_t)rf.size();
    h->glr = dev_lr;
    g.gdev = nullptr, g.grow_f = nullptr, g.grow_d = nullptr;
  });
}

mco_status mco_flat_graph_disable(mco_flat* h) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_flat_graph_disable: null handle");
    if (!h->gdev) return;
    DeviceGuard dg(h->device);
    h->t = graph_steps(h);
    h->free_graph();
  });
}
mco_status mco_flat_state_bytes(const mco_flat* h, uint64_t* out) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_flat_state_bytes: null handle");
    uint64_t b = 0;
    for (size_t i = 0; i < h->named.size(); ++i) b += h->n * h->slot_es((int)i);
    *out = b;
  });
}
mco_status mco_flat_config(const mco_flat* h, mco_config* out) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_flat_config: null handle");
    *out = h->cfg;
  });
}
mco_status mco_flat_num_buffers(const mco_flat* h, int* out) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_flat_num_buffers: null handle");
    *out = (int)h->named.size();
  });
}
mco_status mco_flat_buffer(mco_flat* h, int i, const char** name, void** ptr, uint64_t* len,
                           int* dtype) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_flat_buffer: null handle");
    if (i < 0 || i >= (int)h->named.size())
      throw Error(MCO_CONTRACT, "buffers(): index out of range");
    h->exposed = true;  // callers may keep the pointer: no more relayout
    *name = h->named[i].first;
    *ptr = h->named[i].second;
    *len = h->n;
    *dtype = h->slot_dtype(i);
  });
}

// ---- ZeRO step fused with RS / AG over peer memory (peer.cu) ------------------------
mco_status mco_flat_step_peers(mco_flat* h, const void* const* grad_bufs, int grad_dtype,
                               void* const* param_bufs, int param_dtype, int npeers,
                               float* master, uint64_t offset, uint64_t n, double lr,
                               void* stream) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_flat_step_peers: null handle");
    check_lengths(h, n, n);
    if (h->state_dtype != MCO_F32)
      throw Error(MCO_CONTRACT, "peer step: f32 optimizer state required");
    if (!master) throw Error(MCO_CONTRACT, "peer step: master is null");
    if (npeers < 1 || npeers > kMaxPeers)
      throw Error(MCO_CONTRACT, "peer step: npeers must be 1.." + std::to_string(kMaxPeers));
    PeerPtrs pp{};
    pp.n = npeers;
    for (int r = 0; r < npeers; ++r) {
      if (!grad_bufs[r] || !param_bufs[r])
        throw Error(MCO_CONTRACT, "peer step: null peer buffer");
      pp.g[r] = grad_bufs[r];
      pp.p[r] = param_bufs[r];
    }
    no_graph(h, "peer step");
    no_m64(h, "peer step");
    DeviceGuard dg(h->device);
    ++h->t;
    const auto kf = make_consts<float>(h->cfg, h->t, lr);
    launch_peer_step(h->cfg.kind, pp, grad_dtype, param_dtype, master, h->slot, offset, n, kf,
                     (cudaStream_t)stream);
  });
}

namespace {
PeerPtrs make_peers(const void* const* grad_bufs, void* const* param_bufs, int npeers) {
  if (npeers < 1 || npeers > kMaxPeers)
    throw Error(MCO_CONTRACT, "peer step: npeers must be 1.." + std::to_string(kMaxPeers));
  PeerPtrs pp{};
  pp.n = npeers;
  for (int r = 0; r < npeers; ++r) {
    if (!grad_bufs[r] || (param_bufs && !param_bufs[r]))
      throw Error(MCO_CONTRACT, "peer step: null peer buffer");
    pp.g[r] = grad_bufs[r];
    pp.p[r] = param_bufs ? param_bufs[r] : nullptr;
  }
  return pp;
}
}  // namespace

// (sum over ranks of g_r)^2 summed over this rank's owned range, into *dev_out.
mco_status mco_sumsq_peers(const void* const* grad_bufs, int grad_dtype, int npeers,
                           uint64_t offset, uint64_t n, double* dev_out, void* stream) {
  return guard([&] {
    const PeerPtrs pp = make_peers(grad_bufs, nullptr, npeers);
    cudaStream_t st = (cudaStream_t)stream;
    launch_peer_sumsq(pp, grad_dtype, offset, n, dev_out, sumsq_ws(st), st);
  });
}

// LOMO fused with its collectives: p = p - f * sum_r g_r over the owned range,
// written into every rank's replica; f = lr*scale, or from the all-reduced
// dev_sumsq and clip (optim.cpp:302-303) when dev_sumsq is not null.
mco_status mco_lomo_apply_peers(const void* const* grad_bufs, int grad_dtype,
                                void* const* param_bufs, int param_dtype, int npeers,
                                float* master, uint64_t offset, uint64_t n, double lr,
                                double scale, const double* dev_sumsq, double clip,
                                void* stream) {
  return guard([&] {
    const PeerPtrs pp = make_peers(grad_bufs, param_bufs, npeers);
    launch_peer_lomo(pp, grad_dtype, param_dtype, master, offset, n, lr, scale, dev_sumsq, clip,
                     (cudaStream_t)stream);
  });
}

// Symmetric buffers for the peer step: allocation + CUDA IPC export / import.
mco_status mco_peer_alloc(uint64_t bytes, int device, void** out) {
  return guard([&] {
    DeviceGuard dg(device);
    MCO_CUDA_CHECK(cudaMalloc(out, std::max<uint64_t>(bytes, 1)));
  });
}
mco_status mco_peer_free(void* p) {
  return guard([&] { MCO_CUDA_CHECK(cudaFree(p)); });
}
mco_status mco_peer_export(void* p, void* handle_out) {
  return guard([&] {
    cudaIpcMemHandle_t h;
    MCO_CUDA_CHECK(cudaIpcGetMemHandle(&h, p));
    static_assert(sizeof(h) == 64, "CUDA IPC handle is 64 bytes");
    std::memcpy(handle_out, &h, sizeof(h));
  });
}
mco_status mco_peer_import(const void* handle, int device, void** out) {
  return guard([&] {
    DeviceGuard dg(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    MCO_CUDA_CHECK(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  });
}
mco_status mco_peer_close(void* p) {
  return guard([&] { MCO_CUDA_CHECK(cudaIpcCloseMemHandle(p)); });
}

// ---- LOMO -------------------------------------------------------------------------
mco_status mco_lomo_apply(void* p, int pdt, const void* g, int gdt, uint64_t n, double lr,
                          double scale, void* stream) {
  return guard([&] {
    check_data(n, p, g, "lomo_apply");
    launch_lomo(p, pdt, g, gdt, n, lr, scale, nullptr, 0.0, (cudaStream_t)stream);
  });
}

// LOMO list form: `count` tensors at separate device pointers in one launch per 40
// tensors -- each tensor's update is lomo_apply's, bit for bit (optim.cpp:185-190);
// dev_sumsq != null applies the global-norm clip rule (optim.cpp:291-303).
mco_status mco_lomo_apply_list(int count, void* const* params, int pdt,
                               const void* const* grads, int gdt, const uint64_t* lens,
                               double lr, double scale, const double* dev_sumsq, double clip,
                               void* stream) {
  return guard([&] {
    if (count < 0 || (count > 0 && (!params || !grads || !lens)))
      throw Error(MCO_CONTRACT, "lomo_apply_list: null table");
    for (int i = 0; i < count; ++i)
      check_data(lens[i], params[i], grads[i], "lomo_apply_list");
    launch_lomo_list(count, params, pdt, grads, gdt, lens, lr, scale, dev_sumsq, clip,
                     (cudaStream_t)stream);
  });
}

mco_status mco_lomo_apply_clipped(void* p, int pdt, const void* g, int gdt, uint64_t n, double lr,
                                  const double* dev_sumsq, double clip, void* stream) {
  return guard([&] {
    if (!dev_sumsq) throw Error(MCO_CONTRACT, "lomo clip: device sum of squares is null");
    check_data(n, p, g, "lomo_apply_clipped");
    launch_lomo(p, pdt, g, gdt, n, lr, 1.0, dev_sumsq, clip, (cudaStream_t)stream);
  });
}

// lomo_apply on host spans (the reference's Tensor data is host memory).
// clip >= 0: the norm needs every gradient before any parameter moves.  When the device
// has room, the gradient goes up once into a resident buffer (its sum of squares chunk by
// chunk as it lands), then the parameters stream up / update / down against it: 8 B/param
// up instead of 12.  The buffer stays allocated for the next call (mco_host_release).  Otherwise two passes over the host gradient.  The chunking and the
// accumulation order are the same either way (bit-identical norms).
mco_status mco_lomo_apply_host(void* p, int pdt, const void* g, int gdt, uint64_t n, double lr,
                               double scale, double clip) {
  return guard([&] {
    check_data(n, p, g, "lomo_apply_host");
    const int dev = current_device();
    const size_t gsz = dtype_size(gdt), psz = dtype_size(pdt);
    host_trace(nullptr);
    const double* dnorm = nullptr;
    double* acc = nullptr;
    void* gres = nullptr;  // device-resident gradient (clip only), HostStage::gres
    HostStage& hs = host_stage(dev);
    std::unique_lock<std::mutex> gres_lock(hs.gres_mu, std::defer_lock);
    if (clip >= 0) {
      MCO_CUDA_CHECK(cudaMalloc(&acc, sizeof(double)));
      MCO_CUDA_CHECK(cudaMemset(acc, 0, sizeof(double)));
      gres_lock.lock();
      const uint64_t need = n * gsz;
      if (hs.gres_bytes < need) {  // grow (or first use): only with room to spare
        if (hs.gres) {
          MCO_CUDA_CHECK(cudaFree(hs.gres));
          hs.gres = nullptr;
          hs.gres_bytes = 0;
        }
        size_t free_b = 0, total_b = 0;
        MCO_CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
        if (need + (2ull << 30) < free_b) {
          if (cudaMalloc(&hs.gres, need) == cudaSuccess) {
            hs.gres_bytes = need;
          } else {
            cudaGetLastError();  // out of memory: the two-pass form
            hs.gres = nullptr;
          }
        }
      }
      gres = hs.gres;
      if (!gres) gres_lock.unlock();
      if (gres) {
        std::lock_guard<std::mutex> lock(hs.mu);
        const uint64_t C = hs.chunk_bytes / 8;
        cudaStream_t up = hs.st[1], red = hs.st[0];
        cudaEvent_t ev[2];
        for (auto& e : ev) MCO_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        int k = 0;
        for (uint64_t off = 0; off < n; off += C, k ^= 1) {
          const uint64_t m = std::min(C, n - off);
          char* dg_ = (char*)gres + off * gsz;
          MCO_CUDA_CHECK(cudaMemcpyAsync(dg_, (const char*)g + off * gsz, m * gsz,
                                         cudaMemcpyHostToDevice, up));
          MCO_CUDA_CHECK(cudaEventRecord(ev[k], up));
          MCO_CUDA_CHECK(cudaStreamWaitEvent(red, ev[k], 0));
          launch_sumsq(dg_, gdt, m, acc, 1, sumsq_ws(red), red);  // chunk order, one stream
        }
        MCO_CUDA_CHECK(cudaStreamSynchronize(up));
        MCO_CUDA_CHECK(cudaStreamSynchronize(red));
        for (auto& e : ev) MCO_CUDA_CHECK(cudaEventDestroy(e));
        host_trace("lomo_apply_host: gradient resident + sum of squares");
      } else {
        host_pipeline(dev, const_cast<void*>(g), gsz, nullptr, 0, n, false,
                      [&](void* dg_, void*, uint64_t, uint64_t m, cudaStream_t st) {
                        // one accumulator, chunks strictly ordered through stream 0
                        if (st != hs.st[0]) {
                          cudaEvent_t ev;
                          MCO_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                          MCO_CUDA_CHECK(cudaEventRecord(ev, hs.st[0]));
                          MCO_CUDA_CHECK(cudaStreamWaitEvent(st, ev, 0));
                          MCO_CUDA_CHECK(cudaEventDestroy(ev));
                        }
                        launch_sumsq(dg_, gdt, m, acc, 1, sumsq_ws(st), st);
                        if (st != hs.st[0]) {
                          cudaEvent_t ev;
                          MCO_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                          MCO_CUDA_CHECK(cudaEventRecord(ev, st));
                          MCO_CUDA_CHECK(cudaStreamWaitEvent(hs.st[0], ev, 0));
                          MCO_CUDA_CHECK(cudaEventDestroy(ev));
                        }
                      });
      }
      dnorm = acc;
    }
    if (gres) {
      host_pipeline(dev, p, psz, nullptr, 0, n, true,
                    [&](void* dp, void*, uint64_t off, uint64_t m, cudaStream_t st) {
                      launch_lomo(dp, pdt, (const char*)gres + off * gsz, gdt, m, lr, scale,
                                  dnorm, clip, st);
                    });
    } else {
      host_pipeline(dev, p, psz, g, gsz, n, true,
                    [&](void* dp, void* dg_, uint64_t, uint64_t m, cudaStream_t st) {
                      launch_lomo(dp, pdt, dg_, gdt, m, lr, scale, dnorm, clip, st);
                    });
    }
    host_trace("lomo_apply_host: parameters up / update / down");
    if (acc) cudaFree(acc);
  });
}

mco_status mco_sumsq(const void* x, int dtype, uint64_t n, double* out, int accumulate,
                     void* stream) {
  return guard([&] {
    dtype_size(dtype);
    check_data(n, x, x, "sumsq");
    if (!out) throw Error(MCO_CONTRACT, "sumsq: null output");
    cudaStream_t st = (cudaStream_t)stream;
    launch_sumsq(x, dtype, n, out, accumulate, sumsq_ws(st), st);
  });
}

}  // extern "C"
