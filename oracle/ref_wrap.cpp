// ORACLE -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference optimizer path
// (/root/reference/proj/core/src/optim.cpp, parallel.cpp ZeroPlan), compiled
// from the reference sources by oracle/Makefile into oracle/_ref/libmco_ref.so.
// This file adds no arithmetic of its own: every optimizer number it returns is
// computed by minicollie::optim.  It exists so that tests/ and bench.py's
// reference arm can drive the reference from Python (ctypes), and so the CPU
// baseline can run the reference on all host cores (one FlatOptimizer per
// thread over disjoint slices -- valid because the four stored-state updates
// are elementwise with a uniform step counter).
#include <algorithm>
#include <atomic>
#include <barrier>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "minicollie/errors.hpp"
#include "minicollie/optim.hpp"
#include "minicollie/parallel.hpp"
#include "minicollie/tensor.hpp"

using namespace minicollie;
using namespace minicollie::optim;

extern "C" {
// Same layout as mco_config (include/mco.h) and orc_config (mco_oracle.c).
struct ref_config {
  int kind;
  double lr, weight_decay, beta1, beta2, beta3, eps;
  int has_clip_threshold;
  double clip_threshold;
  double adalomo_clip;
  double sophia_rho;
  int update_interval;
};
// from mco_oracle.c (synthetic inputs, identical generator to the product's)
uint64_t orc_synth_key(uint64_t seed, uint32_t role, uint32_t tensor, uint32_t step);
void orc_synth_f64(double* out, uint64_t n, uint64_t key, int64_t cols, int scale_log2,
                   int zero_log2, int rowcol);
}

namespace {
thread_local std::string g_err;

OptimizerConfig to_cfg(const ref_config& c) {
  OptimizerConfig o;
  o.kind = static_cast<Kind>(c.kind);
  o.lr = c.lr;
  o.weight_decay = c.weight_decay;
  o.beta1 = c.beta1;
  o.beta2 = c.beta2;
  o.beta3 = c.beta3;
  o.eps = c.eps;
  if (c.has_clip_threshold) o.clip_threshold = c.clip_threshold;
  o.adalomo_clip = c.adalomo_clip;
  o.sophia_rho = c.sophia_rho;
  o.update_interval = c.update_interval;
  return o;
}

void from_cfg(const OptimizerConfig& o, ref_config* c) {
  c->kind = static_cast<int>(o.kind);
  c->lr = o.lr;
  c->weight_decay = o.weight_decay;
  c->beta1 = o.beta1;
  c->beta2 = o.beta2;
  c->beta3 = o.beta3;
  c->eps = o.eps;
  c->has_clip_threshold = o.clip_threshold.has_value();
  c->clip_threshold = o.clip_threshold.value_or(0.0);
  c->adalomo_clip = o.adalomo_clip;
  c->sophia_rho = o.sophia_rho;
  c->update_interval = o.update_interval;
}

// Status codes mirror mco_status (errors.hpp taxonomy).
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const DataError& e) {
    g_err = e.what();
    return 3;
  } catch (const ContractError& e) {
    g_err = e.what();
    return 4;
  } catch (const ProtocolError& e) {
    g_err = e.what();
    return 5;
  } catch (const IoError& e) {
    g_err = e.what();
    return 6;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

Shape make_shape(int ndim, const int64_t* dims) { return Shape(dims, dims + ndim); }

// A parameter tensor with a gradient attached, the way the reference's hooks
// see it (Tensor::leaf + mark_param + grad()).
Tensor make_param(const Shape& s, const double* p, const double* g, const std::string& name) {
  const size_t n = static_cast<size_t>(shape_numel(s));
  Tensor t = Tensor::leaf(s, std::vector<double>(p, p + n), true);
  t.mark_param(name);
  t.grad().assign(g, g + n);
  return t;
}

struct AdaLomoHandle {
  OptimizerConfig cfg;
  std::vector<Tensor> params;
  std::unique_ptr<AdaLomoState> state;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_parse_kind(const char* name, int* out) {
  return guard([&] { *out = static_cast<int>(parse_kind(name)); });
}
const char* ref_kind_name(int kind) {
  static thread_local std::string s;
  s = kind_name(static_cast<Kind>(kind));
  return s.c_str();
}
int ref_is_fused(int kind) { return is_fused(static_cast<Kind>(kind)) ? 1 : 0; }
int ref_defaults_for(int kind, ref_config* out) {
  return guard([&] { from_cfg(OptimizerConfig::defaults_for(static_cast<Kind>(kind)), out); });
}
int ref_validate(const ref_config* c) { return guard([&] { to_cfg(*c).validate(); }); }

// ---- FlatOptimizer ----------------------------------------------------------
int ref_flat_create(const ref_config* c, size_t n, void** out) {
  return guard([&] { *out = new FlatOptimizer(to_cfg(*c), n); });
}
void ref_flat_destroy(void* h) { delete static_cast<FlatOptimizer*>(h); }
int ref_flat_step(void* h, double* p, const double* g, size_t np, size_t ng, double lr) {
  return guard([&] {
    static_cast<FlatOptimizer*>(h)->step(std::span<double>(p, np),
                                          std::span<const double>(g, ng), lr);
  });
}
int64_t ref_flat_steps(void* h) { return static_cast<FlatOptimizer*>(h)->steps_taken(); }
void ref_flat_set_steps(void* h, int64_t t) { static_cast<FlatOptimizer*>(h)->set_steps_taken(t); }
uint64_t ref_flat_state_bytes(void* h) {
  return static_cast<FlatOptimizer*>(h)->state_bytes_runtime();
}
int ref_flat_num_buffers(void* h) {
  return static_cast<int>(static_cast<FlatOptimizer*>(h)->buffers().size());
}
const char* ref_flat_buffer(void* h, int i, double** ptr, size_t* len) {
  static thread_local std::string name;
  auto bufs = static_cast<FlatOptimizer*>(h)->buffers();
  name = bufs[static_cast<size_t>(i)].first;
  *ptr = bufs[static_cast<size_t>(i)].second->data();
  *len = bufs[static_cast<size_t>(i)].second->size();
  return name.c_str();
}

// ---- LOMO -------------------------------------------------------------------
int ref_lomo_apply(double* p, const double* g, size_t n, double lr, double scale) {
  return guard([&] {
    Tensor t = make_param({static_cast<int64_t>(n)}, p, g, "w");
    lomo_apply(t, lr, scale);
    std::memcpy(p, t.data().data(), n * sizeof(double));
  });
}

// Runs the reference's own two-pass lomo_fused_backward_step (optim.cpp:284-318)
// with a loss whose gradient w.r.t. param k is exactly g_k:
//   loss = sum_k sum(p_k * G_k),  G_k a constant leaf holding g_k.
// (mul's backward gives grad_p = 1.0 * G exactly; tensor.cpp.)  Params are
// updated in place.  clip < 0 means "no clip".
int ref_lomo_fused_step(int ntensors, const int64_t* numels, double* const* ps,
                        const double* const* gs, double lr, double clip) {
  return guard([&] {
    std::vector<Tensor> params, consts;
    for (int k = 0; k < ntensors; ++k) {
      const size_t n = static_cast<size_t>(numels[k]);
      Tensor t = Tensor::leaf({numels[k]}, std::vector<double>(ps[k], ps[k] + n), true);
      t.mark_param("p" + std::to_string(k));
      params.push_back(t);
      consts.push_back(Tensor::leaf({numels[k]}, std::vector<double>(gs[k], gs[k] + n), false));
    }
    auto loss_fn = [&](Tape& tape) {
      Tensor acc;
      for (size_t k = 0; k < params.size(); ++k) {
        Tensor s = sum(tape, mul(tape, params[k], consts[k]));
        acc = acc.defined() ? add(tape, acc, s) : s;
      }
      return acc;
    };
    std::optional<double> c;
    if (clip >= 0) c = clip;
    lomo_fused_backward_step(params, loss_fn, lr, c);
    for (int k = 0; k < ntensors; ++k)
      std::memcpy(ps[k], params[static_cast<size_t>(k)].data().data(),
                  static_cast<size_t>(numels[k]) * sizeof(double));
  });
}

// ---- AdaLomo -------------------------------------------------------------------
int ref_adalomo_create(const ref_config* c, int ntensors, const int* ndims, const int64_t* dims,
                       void** out) {
  return guard([&] {
    auto h = std::make_unique<AdaLomoHandle>();
    h->cfg = to_cfg(*c);
    const int64_t* d = dims;
    for (int k = 0; k < ntensors; ++k) {
      Shape s = make_shape(ndims[k], d);
      d += ndims[k];
      const size_t n = static_cast<size_t>(shape_numel(s));
      Tensor t = Tensor::leaf(s, std::vector<double>(n, 0.0), true);
      t.mark_param("t" + std::to_string(k));
      h->params.push_back(t);
    }
    h->state = std::make_unique<AdaLomoState>(h->cfg, h->params);
    *out = h.release();
  });
}
void ref_adalomo_destroy(void* h) { delete static_cast<AdaLomoHandle*>(h); }

// The per-tensor hook body (optim.cpp:215-275) on caller data: copy in, apply,
// copy the updated parameter out.
int ref_adalomo_apply(void* hv, int idx, double* p, const double* g, double lr) {
  return guard([&] {
    auto* h = static_cast<AdaLomoHandle*>(hv);
    Tensor& t = h->params.at(static_cast<size_t>(idx));
    const size_t n = static_cast<size_t>(t.numel());
    std::memcpy(t.data().data(), p, n * sizeof(double));
    t.grad().assign(g, g + n);
    h->state->apply(t, lr);
    t.drop_grad();
    std::memcpy(p, t.data().data(), n * sizeof(double));
  });
}
uint64_t ref_adalomo_state_bytes(void* hv) {
  return static_cast<AdaLomoHandle*>(hv)->state->state_bytes_runtime();
}

// ---- accounting / plan ------------------------------------------------------------
int ref_state_bytes(int kind, uint64_t count, int param_bytes, int grad_bytes, int master,
                    int nshapes, const int* ndims, const int64_t* dims, uint64_t* out) {
  return guard([&] {
    PrecisionPolicy pol;
    pol.param_dtype_bytes = param_bytes;
    pol.grad_dtype_bytes = grad_bytes;
    pol.master_copy = master != 0;
    std::vector<Shape> shapes;
    const int64_t* d = dims;
    for (int k = 0; k < nshapes; ++k) {
      shapes.push_back(make_shape(ndims[k], d));
      d += ndims[k];
    }
    *out = state_bytes(static_cast<Kind>(kind), count, pol, shapes);
  });
}

int ref_zero_plan(size_t total, int dp, int stage, size_t* part_sizes, size_t* offsets) {
  return guard([&] {
    auto plan = parallel::ZeroPlan::make(total, dp, stage);
    for (int i = 0; i < dp; ++i) part_sizes[i] = plan.part_sizes[static_cast<size_t>(i)];
    for (int i = 0; i <= dp; ++i) offsets[i] = plan.offsets[static_cast<size_t>(i)];
  });
}

// ---- CPU baseline timing (reference code on all host cores) ------------------------
// Flat kinds: `threads` FlatOptimizers over disjoint slices of an n-element set.
// Fused kinds: the registry tensors (shapes) spread over threads largest-first onto the
// least-loaded thread (LPT), so every thread gets work when there are more tensors than
// threads; lomo_apply / AdaLomoState::apply per tensor.  clip >= 0 adds the global
// gradient-norm pass of lomo_fused_backward_step (optim.cpp:291-303): every thread sums
// g^2 over its tensors in the reference hook's order (`sum_sq += g * g`, optim.cpp:297),
// the partials are combined in thread order, scale = clip / norm iff norm > clip and
// norm > 0; LOMO then runs lomo_apply(t, lr, scale), AdaLomo scales the gradient by it
// before AdaLomoState::apply (the composed oracle of SURVEY 8(c) "parity unpinned" 1).
// The sum and the gradient scaling are the only arithmetic this file restates; every
// update is the reference's.  Inputs are the synthetic generator's values (params
// role 0, grads role 1).  Returns mean seconds per step over `steps` timed steps after
// `warmup` untimed ones.
int ref_bench(const ref_config* c, int ntensors, const int* ndims, const int64_t* dims,
              int threads, int warmup, int steps, uint64_t seed, double clip,
              double* sec_per_step) {
  return guard([&] {
    const OptimizerConfig cfg = to_cfg(*c);
    std::vector<Shape> shapes;
    const int64_t* d = dims;
    for (int k = 0; k < ntensors; ++k) {
      shapes.push_back(make_shape(ndims[k], d));
      d += ndims[k];
    }
    const int T = std::max(1, threads);
    std::barrier sync(T + 1);
    std::barrier workers(T);
    std::atomic<int> failed{0};
    std::vector<std::thread> pool;
    const bool fused = is_fused(cfg.kind);
    const bool clipped = fused && clip >= 0;
    std::vector<double> partial(static_cast<size_t>(T), 0.0);
    // LPT assignment of tensors to threads (fused kinds)
    std::vector<int> owner(static_cast<size_t>(ntensors), 0);
    {
      std::vector<int> order(static_cast<size_t>(ntensors));
      for (int k = 0; k < ntensors; ++k) order[static_cast<size_t>(k)] = k;
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        return shape_numel(shapes[static_cast<size_t>(a)]) >
               shape_numel(shapes[static_cast<size_t>(b)]);
      });
      std::vector<int64_t> load(static_cast<size_t>(T), 0);
      for (int k : order) {
        const size_t w = static_cast<size_t>(std::min_element(load.begin(), load.end()) -
                                             load.begin());
        owner[static_cast<size_t>(k)] = static_cast<int>(w);
        load[w] += shape_numel(shapes[static_cast<size_t>(k)]);
      }
    }
    auto make_tensor = [&](int k) {
      const Shape& s = shapes[static_cast<size_t>(k)];
      const size_t n = static_cast<size_t>(shape_numel(s));
      std::vector<double> pv(n), gv(n);
      orc_synth_f64(pv.data(), n, orc_synth_key(seed, 0, static_cast<uint32_t>(k), 0),
                    s.size() == 2 ? s[1] : 0, s.size() == 2 ? -6 : 0, 0, 0);
      if (s.size() != 2) std::fill(pv.begin(), pv.end(), 1.0);
      orc_synth_f64(gv.data(), n, orc_synth_key(seed, 1, static_cast<uint32_t>(k), 1),
                    s.size() == 2 ? s[1] : 0, -7, 10, s.size() == 2);
      Tensor t = Tensor::leaf(s, std::move(pv), true);
      t.mark_param("t" + std::to_string(k));
      t.grad() = std::move(gv);
      return t;
    };
    std::unique_ptr<AdaLomoState> ada;
    std::vector<Tensor> ada_params;
    std::vector<std::vector<Tensor>> owned(static_cast<size_t>(T));
    if (cfg.kind == Kind::kAdaLomo) {
      // AdaLomoState keys entries on tensor identity; build every tensor up front so
      // one state serves all threads (entries are disjoint per tensor).
      for (int k = 0; k < ntensors; ++k) {
        Tensor t = make_tensor(k);
        ada_params.push_back(t);
        owned[static_cast<size_t>(owner[static_cast<size_t>(k)])].push_back(t);
      }
      ada = std::make_unique<AdaLomoState>(cfg, ada_params);
    }
    uint64_t total = 0;
    for (const Shape& s : shapes) total += static_cast<uint64_t>(shape_numel(s));

    for (int w = 0; w < T; ++w) {
      pool.emplace_back([&, w] {
        try {
          std::unique_ptr<FlatOptimizer> opt;
          std::vector<double> p, g;
          if (!fused) {  // per-thread setup inside the thread (first-touch locality)
            const uint64_t q = total / T, r = total % T;
            const uint64_t len = q + (static_cast<uint64_t>(w) < r ? 1 : 0);
            const uint64_t off = static_cast<uint64_t>(w) * q + std::min<uint64_t>(w, r);
            p.resize(len);
            g.resize(len);
            orc_synth_f64(p.data(), len, orc_synth_key(seed, 0, 0xffffu, 0) + off * 0x9E3779B97F4A7C15ULL, 0, -6, 0, 0);
            orc_synth_f64(g.data(), len, orc_synth_key(seed, 1, 0xffffu, 1) + off * 0x9E3779B97F4A7C15ULL, 0, -7, 10, 0);
            opt = std::make_unique<FlatOptimizer>(cfg, len);
          } else if (cfg.kind == Kind::kLomo) {
            for (int k = 0; k < ntensors; ++k)
              if (owner[static_cast<size_t>(k)] == w)
                owned[static_cast<size_t>(w)].push_back(make_tensor(k));
          }
          auto& mine = owned[static_cast<size_t>(w)];
          for (int it = 0; it < warmup + steps; ++it) {
            sync.arrive_and_wait();  // start of step
            if (!fused) {
              opt->step(p, g, cfg.lr);
            } else {
              double scale = 1.0;
              if (clipped) {
                double sum_sq = 0.0;
                for (Tensor& t : mine)
                  for (double x : t.grad()) sum_sq += x * x;
                partial[static_cast<size_t>(w)] = sum_sq;
                workers.arrive_and_wait();
                double all = 0.0;
                for (double x : partial) all += x;  // thread order
                const double norm = std::sqrt(all);
                if (norm > clip && norm > 0) scale = clip / norm;
                workers.arrive_and_wait();  // partials read before the next step
              }
              for (Tensor& t : mine) {
                if (cfg.kind == Kind::kLomo) {
                  lomo_apply(t, cfg.lr, scale);
                } else {
                  if (scale != 1.0)
                    for (double& x : t.grad()) x *= scale;
                  ada->apply(t, cfg.lr);
                }
              }
            }
            sync.arrive_and_wait();  // end of step
          }
        } catch (...) {
          // keep the barrier phases aligned; the caller reports the failure
          failed = 1;
          for (int it = 0; it < warmup + steps; ++it) {
            sync.arrive_and_wait();
            if (clipped) {
              workers.arrive_and_wait();
              workers.arrive_and_wait();
            }
            sync.arrive_and_wait();
          }
        }
      });
    }
    double timed = 0.0;
    for (int it = 0; it < warmup + steps; ++it) {
      sync.arrive_and_wait();
      auto t0 = std::chrono::steady_clock::now();
      sync.arrive_and_wait();
      auto t1 = std::chrono::steady_clock::now();
      if (it >= warmup) timed += std::chrono::duration<double>(t1 - t0).count();
    }
    for (auto& th : pool) th.join();
    if (failed) throw std::runtime_error("ref_bench: worker failed");
    *sec_per_step = timed / std::max(1, steps);
  });
}

}  // extern "C"
