// C-ABI: AdaLomoState (optim.cpp:192-282) -- hook, list, multi-tensor, host-span and
// row-split (phase) forms.
#include <cstdlib>

#include "abi_internal.h"

using namespace mco;

extern "C" {

// ---- AdaLomo ----------------------------------------------------------------------
// optim.cpp:192-207
mco_status mco_adalomo_create(const mco_config* cfg, int ntensors, const int* ndims,
                              const int64_t* dims, int device, mco_adalomo** out) {
  return guard([&] {
    *out = nullptr;
    device = resolve_device(device);
    DeviceGuard dg(device);
    auto h = std::make_unique<mco_adalomo>();
    auto& pl = h->plan;
    pl.cfg = *cfg;
    pl.device = device;
    std::vector<std::vector<int64_t>> shapes;
    const int64_t* d = dims;
    for (int k = 0; k < ntensors; ++k) {
      shapes.emplace_back(d, d + ndims[k]);
      d += ndims[k];
    }
    build_adalomo_plan(pl, shapes, device_info(device).sms);
    auto alloc = [](auto** p, size_t count, size_t esz) {
      MCO_CUDA_CHECK(cudaMalloc((void**)p, std::max<size_t>(count, 1) * esz));
      MCO_CUDA_CHECK(cudaMemset(*p, 0, std::max<size_t>(count, 1) * esz));
    };
    alloc(&pl.d_tiles, pl.h_tiles.size(), sizeof(Tile));
    alloc(&pl.d_chunks, pl.h_chunks.size(), sizeof(Chunk));
    alloc(&pl.d_chunk_sc, pl.h_chunks.size(), sizeof(double));
    alloc(&pl.d_tensors, pl.h_tensors.size(), sizeof(TensorInfo));
    alloc(&pl.d_item_off, pl.h_item_off.size(), sizeof(int64_t));
    alloc(&pl.d_col_off, pl.h_col_off.size(), sizeof(int64_t));
    alloc(&pl.d_payload, pl.stats_len + pl.usq_len, sizeof(double));
    alloc(&pl.d_state, pl.state_len, sizeof(double));
    alloc(&pl.d_colpart, pl.colpart_len, sizeof(float));
    alloc(&pl.d_rowpart, pl.rowpart_len, sizeof(double));
    alloc(&pl.d_tile_sc, pl.h_tiles.size() * 4, sizeof(double));
    alloc(&pl.d_tens_sc, pl.h_tensors.size() * 8, sizeof(double));
    alloc(&pl.d_fa, pl.fa_len, sizeof(float));
    alloc(&pl.d_fb, pl.fb_len, sizeof(float));
    alloc(&pl.d_fra, pl.fa_len, sizeof(float));
    alloc(&pl.d_frb, pl.fb_len, sizeof(float));
    alloc(&pl.d_mins, 2 * pl.h_tensors.size(), sizeof(unsigned));
    alloc(&pl.d_glob, 6, sizeof(double));  // s, G, host-clip sum, K4 / KR tickets
    MCO_CUDA_CHECK(cudaMemcpy(pl.d_tiles, pl.h_tiles.data(), pl.h_tiles.size() * sizeof(Tile),
                              cudaMemcpyHostToDevice));
    MCO_CUDA_CHECK(cudaMemcpy(pl.d_chunks, pl.h_chunks.data(),
                              pl.h_chunks.size() * sizeof(Chunk), cudaMemcpyHostToDevice));
    MCO_CUDA_CHECK(cudaMemcpy(pl.d_tensors, pl.h_tensors.data(),
                              pl.h_tensors.size() * sizeof(TensorInfo), cudaMemcpyHostToDevice));
    MCO_CUDA_CHECK(cudaMemcpy(pl.d_col_off, pl.h_col_off.data(),
                              pl.h_col_off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    MCO_CUDA_CHECK(cudaMemcpy(pl.d_item_off, pl.h_item_off.data(),
                              pl.h_item_off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    *out = h.release();
  });
}

mco_status mco_adalomo_destroy(mco_adalomo* h) {
  return guard([&] {
    if (!h) return;
    DeviceGuard dg(h->plan.device);
    delete h;
  });
}

namespace {
void check_ada_dtypes(int pdt, int gdt) {
  const bool ok = (pdt == MCO_F32 && (gdt == MCO_F32 || gdt == MCO_BF16)) ||
                  (pdt == MCO_BF16 && gdt == MCO_BF16);
  if (!ok)
    throw Error(MCO_CONTRACT,
                "adalomo: params / grads must be f32 / f32, f32 / bf16 or bf16 / bf16");
}

// Consecutive hook-form calls overlap (the next tensor's K1 under the previous K6);
// MCO_ADALOMO_HOOK_OVERLAP=0 turns it off (A/B knob).
int hook_overlap() {
  static const int on = [] {
    const char* e = getenv("MCO_ADALOMO_HOOK_OVERLAP");
    return e ? atoi(e) : 1;
  }();
  return on;
}

// Hook forms clip with a caller-supplied global Σg² only when the handle opted in.
int hook_clip(const AdaLomoPlan& pl, const double* dev_grad_sumsq) {
  if (!dev_grad_sumsq) return 0;
  if (!pl.grad_clip_on)
    throw Error(MCO_CONTRACT, "adalomo: a gradient sum of squares was passed but the "
                              "grad-norm clip is off (mco_adalomo_set_grad_clip)");
  return 1;
}
}  // namespace

// Opt-in global grad-norm clip for AdaLomo (BASELINE C3; no reference counterpart: the
// reference's AdaLomoState::apply ignores cfg.clip_threshold, optim.cpp:215-275, which
// only LOMO reads, optim.cpp:288-304).  enable = 0 turns it off.
mco_status mco_adalomo_set_grad_clip(mco_adalomo* h, int enable, double clip) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_adalomo_set_grad_clip: null handle");
    if (enable && !(clip >= 0))  // the LOMO rule accepts any threshold >= 0
      throw Error(MCO_CONFIG, "adalomo: grad-norm clip threshold must be >= 0");
    h->plan.grad_clip_on = enable ? 1 : 0;
    h->plan.grad_clip = enable ? clip : 0.0;
  });
}

// optim.cpp:215-275 (hook form: one tensor)
mco_status mco_adalomo_apply(mco_adalomo* h, int idx, void* param, int pdt, const void* grad,
                             int gdt, double lr, const double* dev_grad_sumsq, void* stream) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_adalomo_apply: null handle");
    if (idx < 0 || idx >= (int)h->plan.h_tensors.size())  // optim.cpp:212
      throw Error(MCO_CONTRACT, "adalomo: unknown parameter '" + std::to_string(idx) + "'");
    check_ada_dtypes(pdt, gdt);
    if (!param || !grad) throw Error(MCO_CONTRACT, "adalomo: null data pointer");
    DeviceGuard dg(h->plan.device);
    AdaLomoCall c{};
    c.t0 = idx;
    c.t1 = idx + 1;
    c.p = param;
    c.p_dtype = pdt;
    c.g = grad;
    c.g_dtype = gdt;
    c.single = 1;
    c.lr = lr;
    c.use_clip = hook_clip(h->plan, dev_grad_sumsq);
    c.ext_sumsq = dev_grad_sumsq;
    c.trigger = hook_overlap();
    c.early = c.trigger && h->last_hook >= 0 && h->last_hook != idx && h->last_stream == stream;
    launch_adalomo(h->plan, c, (cudaStream_t)stream);
    h->plan.h_tensors[idx].t += 1;
    h->last_hook = idx;
    h->last_stream = stream;
  });
}

// List form of the hook: tensors t0..t1-1 at separate device pointers, one launch chain
// per kMaxTab tensors (AdaLomo's statistics are per tensor, so the split is exact).
mco_status mco_adalomo_apply_list(mco_adalomo* h, int t0, int t1, void* const* params,
                                  int pdt, const void* const* grads, int gdt, double lr,
                                  const double* dev_grad_sumsq, void* stream) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_adalomo_apply_list: null handle");
    const int nt = (int)h->plan.h_tensors.size();
    if (t0 < 0 || t1 > nt || t0 > t1)
      throw Error(MCO_CONTRACT, "adalomo: tensor range [" + std::to_string(t0) + ", " +
                                    std::to_string(t1) + ") outside 0.." + std::to_string(nt));
    check_ada_dtypes(pdt, gdt);
    if (t1 > t0 && (!params || !grads)) throw Error(MCO_CONTRACT, "adalomo: null table");
    for (int k = t0; k < t1; ++k)
      if (!params[k - t0] || !grads[k - t0])
        throw Error(MCO_CONTRACT, "adalomo: null tensor pointer for index " + std::to_string(k));
    DeviceGuard dg(h->plan.device);
    for (int a = t0; a < t1; a += kMaxTab) {
      const int b = std::min(t1, a + kMaxTab);
      AdaLomoCall c{};
      c.t0 = a;
      c.t1 = b;
      c.p_dtype = pdt;
      c.g_dtype = gdt;
      c.lr = lr;
      c.use_clip = hook_clip(h->plan, dev_grad_sumsq);
      c.ext_sumsq = dev_grad_sumsq;
      c.ntab = b - a;
      for (int k = a; k < b; ++k) {
        c.ptab[k - a] = params[k - t0];
        c.gtab[k - a] = grads[k - t0];
      }
      launch_adalomo(h->plan, c, (cudaStream_t)stream);
    }
    for (int k = t0; k < t1; ++k) h->plan.h_tensors[k].t += 1;
  });
}

mco_status mco_adalomo_apply_all(mco_adalomo* h, void* flat_p, int pdt, const void* flat_g,
                                 int gdt, double lr, void* stream) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_adalomo_apply_all: null handle");
    check_ada_dtypes(pdt, gdt);
    if (!flat_p || !flat_g) throw Error(MCO_CONTRACT, "adalomo: null data pointer");
    DeviceGuard dg(h->plan.device);
    AdaLomoCall c{};
    c.t0 = 0;
    c.t1 = (int)h->plan.h_tensors.size();
    c.p = flat_p;
    c.p_dtype = pdt;
    c.g = flat_g;
    c.g_dtype = gdt;
    c.single = 0;
    c.lr = lr;
    c.use_clip = h->plan.grad_clip_on;
    c.ext_sumsq = nullptr;
    launch_adalomo(h->plan, c, (cudaStream_t)stream);
    for (auto& T : h->plan.h_tensors) T.t += 1;
  });
}

// Host spans (the reference's Tensor data lives in host memory): per tensor,
// H2D(p_k, g_k) -> hook-form apply(k) -> D2H(p_k) on three streams, so tensor
// k+1's upload overlaps tensor k's update and tensor k-1's download.  With a
// global clip every gradient must be seen first: gradients up (with their statistics),
// then per tensor parameters up -> update -> parameters down (below).
mco_status mco_adalomo_apply_all_host(mco_adalomo* h, void* p, int pdt, const void* g, int gdt,
                                      double lr) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_adalomo_apply_all_host: null handle");
    check_ada_dtypes(pdt, gdt);
    if (!p || !g) throw Error(MCO_CONTRACT, "adalomo: null data pointer");
    auto& pl = h->plan;
    DeviceGuard dg(pl.device);
    const int nt = (int)pl.h_tensors.size();
    const uint64_t total = nt ? (uint64_t)(pl.h_tensors.back().elem_off +
                                           pl.h_tensors.back().numel) : 0;
    const size_t gs = dtype_size(gdt), ps = dtype_size(pdt);
    if (!h->hp) {
      MCO_CUDA_CHECK(cudaMalloc(&h->hp, std::max<uint64_t>(total, 1) * 4));
      MCO_CUDA_CHECK(cudaMalloc(&h->hg, std::max<uint64_t>(total, 1) * 4));
      for (auto& st : h->hst) MCO_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      h->ev_in.resize(nt);
      h->ev_out.resize(nt);
      for (int k = 0; k < nt; ++k) {
        MCO_CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_in[k], cudaEventDisableTiming));
        MCO_CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_out[k], cudaEventDisableTiming));
      }
    }
    cudaStream_t up = h->hst[0], comp = h->hst[1], down = h->hst[2];
    AdaLomoCall c{};
    c.p_dtype = pdt;
    c.g_dtype = gdt;
    c.lr = lr;
    if (pl.grad_clip_on) {
      // The clip needs every gradient before any parameter moves, so the step streams in
      // two halves.  A: the gradients go up tensor by tensor and each tensor's gradient
      // statistics (K1 in its gradient-only mode) run as it lands; then the global sum of
      // g^2.  B: per tensor, its parameters go up, sum p^2 (K1 parameter-only mode), the
      // rest of the update, and the parameters come back down -- B's uploads share the
      // link with its downloads (full duplex) instead of following them.  The statistics
      // keep MODE 3's loops and order and the global sum K2's, so the result equals the
      // device apply_all on the uploaded buffers bit for bit.
      double* gsum = pl.d_glob + 2;
      for (int k = 0; k < nt; ++k) {
        const TensorInfo& T = pl.h_tensors[k];
        const uint64_t off = (uint64_t)T.elem_off, n = (uint64_t)T.numel;
        MCO_CUDA_CHECK(cudaMemcpyAsync((char*)h->hg + off * gs, (const char*)g + off * gs,
                                       n * gs, cudaMemcpyHostToDevice, up));
        MCO_CUDA_CHECK(cudaEventRecord(h->ev_in[k], up));
        MCO_CUDA_CHECK(cudaStreamWaitEvent(comp, h->ev_in[k], 0));
        c.t0 = k;
        c.t1 = k + 1;
        c.p = (char*)h->hp + off * ps;
        c.g = (char*)h->hg + off * gs;
        c.single = 1;
        c.stats_mode = 1;
        launch_adalomo_phase(pl, c, 1, comp);
      }
      launch_adalomo_gsumsq(pl, 0, nt, gsum, comp);
      c.stats_mode = 2;
      c.use_clip = 1;
      c.ext_sumsq = gsum;
      c.fuse_usq = 1;
      for (int k = 0; k < nt; ++k) {
        const TensorInfo& T = pl.h_tensors[k];
        const uint64_t off = (uint64_t)T.elem_off, n = (uint64_t)T.numel;
        char* dp = (char*)h->hp + off * ps;
        MCO_CUDA_CHECK(cudaMemcpyAsync(dp, (const char*)p + off * ps, n * ps,
                                       cudaMemcpyHostToDevice, up));
        MCO_CUDA_CHECK(cudaEventRecord(h->ev_in[k], up));
        MCO_CUDA_CHECK(cudaStreamWaitEvent(comp, h->ev_in[k], 0));
        c.t0 = k;
        c.t1 = k + 1;
        c.p = dp;
        c.g = (char*)h->hg + off * gs;
        for (int phase = 1; phase <= 3; ++phase) launch_adalomo_phase(pl, c, phase, comp);
        MCO_CUDA_CHECK(cudaEventRecord(h->ev_out[k], comp));
        MCO_CUDA_CHECK(cudaStreamWaitEvent(down, h->ev_out[k], 0));
        MCO_CUDA_CHECK(cudaMemcpyAsync((char*)p + off * ps, dp, n * ps, cudaMemcpyDeviceToHost,
                                       down));
      }
    } else {
      for (int k = 0; k < nt; ++k) {
        const TensorInfo& T = pl.h_tensors[k];
        const uint64_t off = (uint64_t)T.elem_off, n = (uint64_t)T.numel;
        char* dp = (char*)h->hp + off * ps;
        char* dgp = (char*)h->hg + off * gs;
        MCO_CUDA_CHECK(cudaMemcpyAsync(dp, (const char*)p + off * ps, n * ps,
                                       cudaMemcpyHostToDevice, up));
        MCO_CUDA_CHECK(cudaMemcpyAsync(dgp, (const char*)g + off * gs, n * gs,
                                       cudaMemcpyHostToDevice, up));
        MCO_CUDA_CHECK(cudaEventRecord(h->ev_in[k], up));
        MCO_CUDA_CHECK(cudaStreamWaitEvent(comp, h->ev_in[k], 0));
        c.t0 = k;
        c.t1 = k + 1;
        c.p = dp;
        c.g = dgp;
        c.single = 1;
        c.use_clip = 0;
        launch_adalomo(pl, c, comp);
        MCO_CUDA_CHECK(cudaEventRecord(h->ev_out[k], comp));
        MCO_CUDA_CHECK(cudaStreamWaitEvent(down, h->ev_out[k], 0));
        MCO_CUDA_CHECK(cudaMemcpyAsync((char*)p + off * ps, dp, n * ps, cudaMemcpyDeviceToHost,
                                       down));
      }
    }
    for (auto st : h->hst) MCO_CUDA_CHECK(cudaStreamSynchronize(st));
    for (auto& T : pl.h_tensors) T.t += 1;
  });
}

// ---- AdaLomo row-split sharding ---------------------------------------------------
// Tensor `idx` holds a row slice of a global (global_rows x C) matrix (or a
// replica of a 1-D tensor): statistics normalise by the global shape and the
// payload contribution is scaled by `weight` (1 for a row slice, 1 on exactly
// one rank for a replica, 0 elsewhere).
mco_status mco_adalomo_set_shard(mco_adalomo* h, int idx, int64_t global_rows, double weight) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_adalomo_set_shard: null handle");
    auto& pl = h->plan;
    if (idx < 0 || idx >= (int)pl.h_tensors.size())
      throw Error(MCO_CONTRACT, "adalomo: tensor index out of range");
    TensorInfo& T = pl.h_tensors[idx];
    if (global_rows < T.rows)
      throw Error(MCO_CONTRACT, "adalomo: global rows smaller than the local slice");
    DeviceGuard dg(pl.device);
    // keep the device-side step counter (advanced by k2_scalars)
    MCO_CUDA_CHECK(cudaMemcpy(&T.t, &pl.d_tensors[idx].t, sizeof(int64_t),
                              cudaMemcpyDeviceToHost));
    T.rows_global = global_rows;
    T.numel_global = T.factored ? global_rows * T.cols : T.numel;
    T.weight = weight;
    MCO_CUDA_CHECK(cudaMemcpy(&pl.d_tensors[idx], &T, sizeof(TensorInfo),
                              cudaMemcpyHostToDevice));
  });
}

// One phase of apply_all (1: stats, 2: moments + sum u^2, 3: update).  A
// row-split caller all-reduces payload 0 after phase 1 and payload 1 after phase 2.
mco_status mco_adalomo_phase(mco_adalomo* h, int phase, void* flat_p, int pdt,
                             const void* flat_g, int gdt, double lr, void* stream) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_adalomo_phase: null handle");
    check_ada_dtypes(pdt, gdt);
    if (phase < 1 || phase > 3) throw Error(MCO_CONTRACT, "adalomo: phase must be 1, 2 or 3");
    DeviceGuard dg(h->plan.device);
    AdaLomoCall c{};
    c.t0 = 0;
    c.t1 = (int)h->plan.h_tensors.size();
    c.p = flat_p;
    c.p_dtype = pdt;
    c.g = flat_g;
    c.g_dtype = gdt;
    c.single = 0;
    c.lr = lr;
    c.use_clip = h->plan.grad_clip_on;
    launch_adalomo_phase(h->plan, c, phase, (cudaStream_t)stream);
    if (phase == 3)
      for (auto& T : h->plan.h_tensors) T.t += 1;
  });
}

// which 0: stats payload (3 per tensor + column sums), 1: sum u^2 payload.
mco_status mco_adalomo_payload(mco_adalomo* h, int which, double** dev_ptr, uint64_t* len) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_adalomo_payload: null handle");
    if (which == 0) {
      *dev_ptr = h->plan.d_payload;
      *len = (uint64_t)h->plan.stats_len;
    } else if (which == 1) {
      *dev_ptr = h->plan.d_payload + h->plan.stats_len;
      *len = (uint64_t)h->plan.usq_len;
    } else {
      throw Error(MCO_CONTRACT, "adalomo: payload must be 0 or 1");
    }
  });
}

// optim.cpp:277-282 (fp64 state, as the reference)
mco_status mco_adalomo_state_bytes(const mco_adalomo* h, uint64_t* out) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_adalomo_state_bytes: null handle");
    *out = (uint64_t)h->plan.state_len * sizeof(double);
  });
}

mco_status mco_adalomo_get_steps(const mco_adalomo* h, int idx, int64_t* t) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_adalomo_get_steps: null handle");
    if (idx < 0 || idx >= (int)h->plan.h_tensors.size())
      throw Error(MCO_CONTRACT, "adalomo: tensor index out of range");
    // the device counter is the truth (K2 advances it): steps replayed from a captured
    // CUDA graph count too, which a host mirror would miss
    DeviceGuard dg(h->plan.device);
    MCO_CUDA_CHECK(cudaDeviceSynchronize());
    const TensorInfo* dT = reinterpret_cast<const TensorInfo*>(h->plan.d_tensors) + idx;
    MCO_CUDA_CHECK(cudaMemcpy(t, &dT->t, sizeof(int64_t), cudaMemcpyDeviceToHost));
  });
}

mco_status mco_adalomo_buffer(mco_adalomo* h, int idx, int which, void** ptr, uint64_t* len) {
  return guard([&] {
    if (!h) throw Error(MCO_CONTRACT, "mco_adalomo_buffer: null handle");
    if (idx < 0 || idx >= (int)h->plan.h_tensors.size())
      throw Error(MCO_CONTRACT, "adalomo: tensor index out of range");
    const TensorInfo& T = h->plan.h_tensors[idx];
    int64_t off = -1, n = 0;
    if (which == 0 && T.factored) off = T.vrow_off, n = T.rows;
    if (which == 1 && T.factored) off = T.vcol_off, n = T.cols;
    if (which == 2 && !T.factored) off = T.vfull_off, n = T.numel;
    *ptr = off >= 0 ? (void*)(h->plan.d_state + off) : nullptr;
    *len = (uint64_t)n;
  });
}

}  // extern "C"
