// minicollie_b200/optim.hpp -- header-only C++ shim that re-exposes the
// reference's optimizer API (namespace minicollie::optim,
// /root/reference/proj/core/include/minicollie/optim.hpp) on top of the C-ABI
// (include/mco.h, libmco.so).  Host code written against the reference
// compiles against this header with the same class / function names; link
// with -lmco.  It also provides the reference's error taxonomy
// (minicollie/errors.hpp) because exceptions are how the reference reports
// failures: every mco_status is rethrown as the matching exception type with
// the reference's message.
//
//   reference                                    this shim
//   FlatOptimizer(cfg, owned_len)                FlatOptimizer(cfg, owned_len[, device, precision])
//   step(span<double>, span<const double>, lr)   same (host spans, staged through the GPU)
//                                                + step(float* dev_p, const float* dev_g, n, lr, stream)
//   buffers() -> {name, vector<double>*}         buffers() -> {name, DeviceBuffer};
//                                                buffer_to_host(name) -> vector<double>
//   lomo_apply(Tensor&, lr, scale)               lomo_apply(DeviceTensor&, lr, scale)
//   AdaLomoState(cfg, vector<Tensor>)            AdaLomoState(cfg, vector<DeviceTensor>)
//   apply(Tensor&, lr)                           apply(DeviceTensor&, lr[, stream])
//   state_bytes(kind, n, policy, shapes)         same
//
// Like the reference, instances are not thread-safe; use one per device/thread.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mco.h"

namespace minicollie {

// errors.hpp:11-32
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct DataError : std::runtime_error {
  explicit DataError(const std::string& m) : std::runtime_error(m) {}
};
struct ContractError : std::logic_error {
  explicit ContractError(const std::string& m) : std::logic_error(m) {}
};
struct ProtocolError : std::runtime_error {
  explicit ProtocolError(const std::string& m) : std::runtime_error(m) {}
};
struct IoError : std::runtime_error {
  explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
struct DeviceError : std::runtime_error {
  explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

using Shape = std::vector<int64_t>;

inline void mco_throw(mco_status s) {
  if (s == MCO_OK) return;
  const std::string m = mco_last_error();
  switch (s) {
    case MCO_CONFIG: throw ConfigError(m);
    case MCO_DATA: throw DataError(m);
    case MCO_CONTRACT: throw ContractError(m);
    case MCO_PROTOCOL: throw ProtocolError(m);
    case MCO_IO: throw IoError(m);
    default: throw DeviceError(m);
  }
}

// A parameter living on the GPU: data + gradient device pointers (fp32), shape.
// Stands in for the reference's Tensor on the update path.
struct DeviceTensor {
  float* data = nullptr;
  const float* grad = nullptr;
  Shape shape;
  std::string name;
  int64_t numel() const {
    int64_t n = 1;
    for (int64_t d : shape) n *= d;
    return n;
  }
  int ndim() const { return static_cast<int>(shape.size()); }
  int64_t dim(int i) const { return shape.at(static_cast<size_t>(i)); }
};

namespace optim {

enum class Kind { kAdamW, kLion, kAdan, kSophia, kLomo, kAdaLomo };  // optim.hpp:14

inline Kind parse_kind(const std::string& name) {
  int k = 0;
  mco_throw(mco_parse_kind(name.c_str(), &k));
  return static_cast<Kind>(k);
}
inline std::string kind_name(Kind kind) {
  const char* s = mco_kind_name(static_cast<int>(kind));
  if (!s) throw ConfigError("unknown optimizer kind");
  return s;
}
inline bool is_fused(Kind kind) { return mco_is_fused(static_cast<int>(kind)) != 0; }

struct OptimizerConfig {  // optim.hpp:20-35
  Kind kind = Kind::kAdamW;
  double lr = 1e-3;
  double weight_decay = 0.0;
  double beta1 = 0.9;
  double beta2 = 0.999;
  double beta3 = 0.99;
  double eps = 1e-8;
  std::optional<double> clip_threshold;
  double adalomo_clip = 1.0;
  double sophia_rho = 0.04;
  int update_interval = 10;

  static OptimizerConfig defaults_for(Kind kind) {
    mco_config c{};
    mco_throw(mco_defaults_for(static_cast<int>(kind), &c));
    return from_c(c);
  }
  void validate() const {
    const mco_config c = to_c();
    mco_throw(mco_validate(&c));
  }
  mco_config to_c() const {
    mco_config c{};
    c.kind = static_cast<int>(kind);
    c.lr = lr;
    c.weight_decay = weight_decay;
    c.beta1 = beta1;
    c.beta2 = beta2;
    c.beta3 = beta3;
    c.eps = eps;
    c.has_clip_threshold = clip_threshold.has_value();
    c.clip_threshold = clip_threshold.value_or(0.0);
    c.adalomo_clip = adalomo_clip;
    c.sophia_rho = sophia_rho;
    c.update_interval = update_interval;
    return c;
  }
  static OptimizerConfig from_c(const mco_config& c) {
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
};

// State precision: kF64 reproduces the reference bit for bit on double host
// spans (the drop-in default); kF32 is the HBM-roofline product path.
enum class Precision { kF64, kF32 };

// Device argument default: the calling thread's current CUDA device (resolved inside the
// C-ABI), so a rank that called cudaSetDevice(r) gets its state on GPU r.
constexpr int kCurrentDevice = -1;

struct DeviceBuffer {
  void* ptr = nullptr;
  uint64_t len = 0;
  int dtype = MCO_F32;
};

class FlatOptimizer {  // optim.hpp:40-64
 public:
  FlatOptimizer(const OptimizerConfig& cfg, size_t owned_len, int device = kCurrentDevice,
                Precision precision = Precision::kF64)
      : cfg_(cfg), precision_(precision) {
    const mco_config c = cfg.to_c();
    mco_throw(mco_flat_create(&c, owned_len, device,
                              precision == Precision::kF64 ? MCO_F64 : MCO_F32, &h_));
  }
  ~FlatOptimizer() {
    if (h_) mco_flat_destroy(h_);
  }
  FlatOptimizer(const FlatOptimizer&) = delete;
  FlatOptimizer& operator=(const FlatOptimizer&) = delete;
  FlatOptimizer(FlatOptimizer&& o) noexcept : cfg_(o.cfg_), precision_(o.precision_), h_(o.h_) {
    o.h_ = nullptr;
  }
  FlatOptimizer& operator=(FlatOptimizer&& o) noexcept {
    std::swap(h_, o.h_);
    cfg_ = o.cfg_;
    precision_ = o.precision_;
    return *this;
  }

  // Host spans, as the reference (synchronous; staged through the device).
  void step(std::span<double> params, std::span<const double> grads, double lr) {
    if (precision_ == Precision::kF64) {
      mco_throw(mco_flat_step_host(h_, params.data(), MCO_F64, params.size(), grads.data(),
                                   MCO_F64, grads.size(), lr));
      return;
    }
    if (params.size() != grads.size())
      throw ContractError("optimizer step: params/grads length mismatch: " +
                          std::to_string(params.size()) + " vs " + std::to_string(grads.size()));
    std::vector<float> p(params.begin(), params.end()), g(grads.begin(), grads.end());
    mco_throw(mco_flat_step_host(h_, p.data(), MCO_F32, p.size(), g.data(), MCO_F32, g.size(),
                                 lr));
    for (size_t i = 0; i < p.size(); ++i) params[i] = p[i];
  }
  // Device path (kF32): stream-ordered, asynchronous.
  void step(float* dev_params, const float* dev_grads, size_t n, double lr,
            void* stream = nullptr) {
    mco_throw(mco_flat_step(h_, dev_params, MCO_F32, n, dev_grads, MCO_F32, n, lr, stream));
  }
  void step(double* dev_params, const double* dev_grads, size_t n, double lr,
            void* stream = nullptr) {
    mco_throw(mco_flat_step(h_, dev_params, MCO_F64, n, dev_grads, MCO_F64, n, lr, stream));
  }
  // List form (mco_flat_step_list): a model's tensors in registry order over the flat
  // state -- == step() over their concatenation, without flattening.
  void step(std::span<DeviceTensor> tensors, double lr, void* stream = nullptr) {
    std::vector<void*> p;
    std::vector<const void*> g;
    std::vector<uint64_t> len;
    for (auto& t : tensors) {
      p.push_back(t.data);
      g.push_back(t.grad);
      len.push_back(static_cast<uint64_t>(t.numel()));
    }
    mco_throw(mco_flat_step_list(h_, static_cast<int>(tensors.size()), p.data(), MCO_F32,
                                 g.data(), MCO_F32, len.data(), lr, stream));
  }

  int64_t steps_taken() const {
    int64_t t = 0;
    mco_throw(mco_flat_get_steps(h_, &t));
    return t;
  }
  void set_steps_taken(int64_t t) { mco_throw(mco_flat_set_steps(h_, t)); }
  // CUDA-graph mode (mco_flat_graph_enable): dev_lr = optional device double
  void enable_graph(const double* dev_lr = nullptr) { mco_throw(mco_flat_graph_enable(h_, dev_lr)); }
  void disable_graph() { mco_throw(mco_flat_graph_disable(h_)); }
  uint64_t state_bytes_runtime() const {
    uint64_t b = 0;
    mco_throw(mco_flat_state_bytes(h_, &b));
    return b;
  }
  std::vector<std::pair<std::string, DeviceBuffer>> buffers() {
    int n = 0;
    mco_throw(mco_flat_num_buffers(h_, &n));
    std::vector<std::pair<std::string, DeviceBuffer>> out;
    for (int i = 0; i < n; ++i) {
      const char* name = nullptr;
      DeviceBuffer b;
      mco_throw(mco_flat_buffer(h_, i, &name, &b.ptr, &b.len, &b.dtype));
      out.emplace_back(name, b);
    }
    return out;
  }
  const OptimizerConfig& config() const { return cfg_; }
  mco_flat* handle() { return h_; }

 private:
  OptimizerConfig cfg_;
  Precision precision_;
  mco_flat* h_ = nullptr;
};

// optim.hpp:71 -- p -= (lr*scale) * g on the device.
inline void lomo_apply(DeviceTensor& param, double lr, double scale, void* stream = nullptr) {
  mco_throw(mco_lomo_apply(param.data, MCO_F32, param.grad, MCO_F32,
                           static_cast<uint64_t>(param.numel()), lr, scale, stream));
}

class AdaLomoState {  // optim.hpp:76-96
 public:
  AdaLomoState(const OptimizerConfig& cfg, const std::vector<DeviceTensor>& params,
               int device = kCurrentDevice)
      : cfg_(cfg) {
    std::vector<int> nd;
    std::vector<int64_t> dims;
    for (const DeviceTensor& t : params) {
      nd.push_back(t.ndim());
      dims.insert(dims.end(), t.shape.begin(), t.shape.end());
      ids_.push_back(t.data);
      names_.push_back(t.name);
    }
    const mco_config c = cfg.to_c();
    mco_throw(mco_adalomo_create(&c, static_cast<int>(params.size()), nd.data(), dims.data(),
                                 device, &h_));
  }
  ~AdaLomoState() {
    if (h_) mco_adalomo_destroy(h_);
  }
  AdaLomoState(const AdaLomoState&) = delete;
  AdaLomoState& operator=(const AdaLomoState&) = delete;

  // Consumes param.grad (device); entry looked up by storage identity (optim.cpp:209-213).
  void apply(DeviceTensor& param, double lr, void* stream = nullptr) {
    for (size_t i = 0; i < ids_.size(); ++i)
      if (ids_[i] == param.data) {
        mco_throw(mco_adalomo_apply(h_, static_cast<int>(i), param.data, MCO_F32, param.grad,
                                    MCO_F32, lr, nullptr, stream));
        return;
      }
    throw ContractError("adalomo: unknown parameter '" + param.name + "'");
  }
  // Opt-in global grad-norm clip (beyond the reference, whose AdaLomoState ignores
  // cfg.clip_threshold): mco_adalomo_set_grad_clip.
  void set_grad_clip(std::optional<double> clip) {
    mco_throw(mco_adalomo_set_grad_clip(h_, clip.has_value() ? 1 : 0, clip.value_or(0.0)));
  }
  // Every registered tensor at once over registry-order flat device buffers.
  void apply_all(float* flat_params, const float* flat_grads, double lr, void* stream = nullptr) {
    mco_throw(mco_adalomo_apply_all(h_, flat_params, MCO_F32, flat_grads, MCO_F32, lr, stream));
  }
  uint64_t state_bytes_runtime() const {
    uint64_t b = 0;
    mco_throw(mco_adalomo_state_bytes(h_, &b));
    return b;
  }

 private:
  OptimizerConfig cfg_;
  mco_adalomo* h_ = nullptr;
  std::vector<const void*> ids_;
  std::vector<std::string> names_;
};

struct PrecisionPolicy {  // optim.hpp:113-119
  int param_dtype_bytes = 2;
  int grad_dtype_bytes = 4;
  bool master_copy = true;
  bool needs_master() const { return master_copy && param_dtype_bytes < 4; }
};

inline uint64_t state_bytes(Kind kind, uint64_t param_count, const PrecisionPolicy& policy,
                            const std::vector<Shape>& shapes = {}) {
  std::vector<int> nd;
  std::vector<int64_t> dims;
  for (const Shape& s : shapes) {
    nd.push_back(static_cast<int>(s.size()));
    dims.insert(dims.end(), s.begin(), s.end());
  }
  uint64_t out = 0;
  mco_throw(mco_state_bytes(static_cast<int>(kind), param_count, policy.param_dtype_bytes,
                            policy.grad_dtype_bytes, policy.master_copy ? 1 : 0,
                            static_cast<int>(shapes.size()), nd.data(), dims.data(), &out));
  return out;
}

}  // namespace optim

namespace parallel {
struct ZeroPlan {  // parallel.hpp:22-29
  int stage = 0;
  std::vector<size_t> part_sizes;
  std::vector<size_t> offsets;
  static ZeroPlan make(size_t total_len, int dp_size, int stage) {
    ZeroPlan p;
    p.stage = stage;
    std::vector<uint64_t> ps(static_cast<size_t>(dp_size > 0 ? dp_size : 1)),
        off(ps.size() + 1);
    mco_throw(mco_zero_plan(total_len, dp_size, stage, ps.data(), off.data()));
    p.part_sizes.assign(ps.begin(), ps.end());
    p.offsets.assign(off.begin(), off.end());
    return p;
  }
  std::pair<size_t, size_t> owned_range(int dp_index) const {
    return {offsets[static_cast<size_t>(dp_index)], offsets[static_cast<size_t>(dp_index) + 1]};
  }
};

// The sharder's NCCL communicator (libmco's mco_comm; the CommHub group of
// comm.hpp:77-135).  NCCL is loaded at run time by libmco (no link dependency).
class NcclComm {
 public:
  using Id = std::array<char, 128>;
  static Id unique_id() {  // on one rank; ship the bytes to the others
    Id id{};
    mco_throw(mco_comm_unique_id(id.data()));
    return id;
  }
  NcclComm(const Id& id, int nranks, int rank, int device = optim::kCurrentDevice) {
    mco_throw(mco_comm_create(id.data(), nranks, rank, device, &h_));
  }
  ~NcclComm() {
    if (h_) mco_comm_destroy(h_);
  }
  NcclComm(const NcclComm&) = delete;
  NcclComm& operator=(const NcclComm&) = delete;
  mco_comm* handle() const { return h_; }
  void check() const { mco_throw(mco_comm_check(h_)); }

 private:
  mco_comm* h_ = nullptr;
};

// Stage-2 ZeRO step of ParallelWorker::train_step (parallel.cpp:656-666) on device
// flat buffers: reduce-scatter(SUM) -> step of the owned ZeroPlan part -> all-gather.
// `opt` must own exactly this rank's part (ZeroPlan::make(total_len, nranks)).
inline void shard_step(optim::FlatOptimizer& opt, const NcclComm& comm, float* flat_params,
                       const float* flat_grads, size_t total_len, double lr,
                       void* stream = nullptr) {
  mco_throw(mco_shard_step(opt.handle(), comm.handle(), flat_params, MCO_F32, flat_grads,
                           MCO_F32, total_len, lr, stream));
}
// Mixed precision: fp32 master of the owned part, bf16 replicas (mco_shard_step_mixed).
inline void shard_step_mixed(optim::FlatOptimizer& opt, const NcclComm& comm,
                             float* master_owned, uint16_t* flat_params_bf16,
                             const float* flat_grads, size_t total_len, double lr,
                             void* stream = nullptr) {
  mco_throw(mco_shard_step_mixed(opt.handle(), comm.handle(), master_owned, flat_params_bf16,
                                 flat_grads, MCO_F32, total_len, lr, stream));
}
}  // namespace parallel

}  // namespace minicollie
