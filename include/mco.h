/*
 * mco.h -- C-ABI of the B200-native optimizer-update hot path.
 *
 * Drop-in boundary for the reference's C++ optimizer operator API,
 * namespace minicollie::optim (/root/reference/proj/core/include/minicollie/optim.hpp).
 * Every entry point below names the reference interface it replaces.
 * Plain C types only: device buffers are `void*` device pointers, streams are
 * `void*` holding a cudaStream_t (NULL = legacy default stream).  A `device`
 * argument < 0 means the calling thread's current CUDA device.
 *
 * Error model (errors.hpp:8-32): each call returns an mco_status; the message
 * of the last failure on the calling thread is mco_last_error() and equals the
 * reference's exception what() text where the reference throws.  Argument and
 * contract errors are reported synchronously; device-side CUDA errors surface
 * as MCO_CUDA on the failing launch or on the next synchronising call
 * (mco_sync).  Stream-ordered calls are asynchronous with respect to the host.
 *
 * Numerics: fp32 state and arithmetic by default (bf16 accepted for gradients,
 * bf16 parameter storage for LOMO and the bf16 parameter copy of the mixed
 * step); fp64 state for the bit-exact parity mode.  Kernels are compiled with
 * no multiply-add contraction, so every fp32 / fp64 elementwise update is
 * bit-identical to the operation order of optim.cpp.
 */
#ifndef MCO_H_
#define MCO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* errors.hpp:8-32 taxonomy; CLI exit-code mapping Config->2, Data->3 kept. */
typedef enum mco_status {
  MCO_OK = 0,
  MCO_CONFIG = 2,   /* ConfigError   */
  MCO_DATA = 3,     /* DataError     */
  MCO_CONTRACT = 4, /* ContractError */
  MCO_PROTOCOL = 5, /* ProtocolError */
  MCO_IO = 6,       /* IoError       */
  MCO_CUDA = 7      /* device / runtime failure (no reference counterpart) */
} mco_status;

/* optim.hpp:14  enum class Kind { kAdamW, kLion, kAdan, kSophia, kLomo, kAdaLomo } */
typedef enum mco_kind {
  MCO_ADAMW = 0,
  MCO_LION = 1,
  MCO_ADAN = 2,
  MCO_SOPHIA = 3,
  MCO_LOMO = 4,
  MCO_ADALOMO = 5
} mco_kind;

/* MCO_F32M64 is a FlatOptimizer state layout only: fp32 state with an fp64 first
 * moment m (Sophia's opt-in "precise-m" mode, see mco_flat_create). */
typedef enum mco_dtype { MCO_F32 = 0, MCO_BF16 = 1, MCO_F64 = 2, MCO_F32M64 = 3 } mco_dtype;

/* optim.hpp:20-35  struct OptimizerConfig, field for field
 * (std::optional<double> clip_threshold -> has_clip_threshold + clip_threshold). */
typedef struct mco_config {
  int kind;
  double lr;
  double weight_decay;
  double beta1;
  double beta2;
  double beta3;
  double eps;
  int has_clip_threshold;
  double clip_threshold;
  double adalomo_clip;
  double sophia_rho;
  int update_interval;
} mco_config;

const char* mco_last_error(void);
const char* mco_version(void);

/* optim.hpp:16  Kind parse_kind(const std::string&)  (ConfigError on unknown) */
mco_status mco_parse_kind(const char* name, int* kind_out);
/* optim.hpp:17  std::string kind_name(Kind)  (NULL on unknown kind) */
const char* mco_kind_name(int kind);
/* optim.hpp:18  bool is_fused(Kind) */
int mco_is_fused(int kind);
/* optim.hpp:33  static OptimizerConfig defaults_for(Kind) */
mco_status mco_defaults_for(int kind, mco_config* out);
/* optim.hpp:34  void validate() const */
mco_status mco_validate(const mco_config* cfg);

/* optim.hpp:113-127  state_bytes(kind, param_count, PrecisionPolicy, shapes).
 * shapes: nshapes entries, entry k has ndims[k] dims taken consecutively from dims. */
mco_status mco_state_bytes(int kind, uint64_t param_count, int param_dtype_bytes,
                           int grad_dtype_bytes, int master_copy, int nshapes,
                           const int* ndims, const int64_t* dims, uint64_t* out);

/* ---- FlatOptimizer (optim.hpp:40-64, optim.cpp:74-181) ------------------- */
typedef struct mco_flat mco_flat;

/* FlatOptimizer(cfg, owned_len): zero-initialised SoA state on `device`
 * (m,v | m | m,v,n,g_prev | m,h).  state_dtype MCO_F32 (default product path)
 * or MCO_F64 (bit-exact parity mode), or -- Sophia only -- MCO_F32M64: fp32 h with an
 * fp64 m and fp64 per-element arithmetic on fp32 params ("precise-m": the fp32 m's
 * cancellation error, amplified by 1/(rho h), otherwise pushes ~0.06 % of elements past
 * 1e-5 of the fp64 reference; 32 B/param instead of 24; mco_flat_step and the host-span
 * step only).  Fused kinds -> MCO_CONTRACT. */
mco_status mco_flat_create(const mco_config* cfg, uint64_t owned_len, int device,
                           int state_dtype, mco_flat** out);
mco_status mco_flat_destroy(mco_flat* h);

/* FlatOptimizer::step(span<double> params, span<const double> grads, lr),
 * device pointers, stream-ordered.  n_params != n_grads -> MCO_CONTRACT with
 * the reference's message (optim.cpp:101-103); n_params > owned_len ->
 * MCO_CONTRACT (the reference would index past its state).  ++t happens
 * before the update (optim.cpp:104).
 * dtypes: state F32 -> params F32, grads F32 or BF16; state F64 -> F64/F64. */
mco_status mco_flat_step(mco_flat* h, void* params, int param_dtype, uint64_t n_params,
                         const void* grads, int grad_dtype, uint64_t n_grads, double lr,
                         void* stream);

/* Mixed-precision step (ZeRO shard, SURVEY 8(d) "mixed"): fp32 master params
 * updated in place and written once more as bf16 into param_out. */
mco_status mco_flat_step_mixed(mco_flat* h, float* master, const void* grads, int grad_dtype,
                               uint16_t* param_out_bf16, uint64_t n, double lr, void* stream);

/* The reference's host-span overload: params / grads are HOST arrays (F64 for
 * an F64-state optimizer, F32 for an F32-state one); streamed through the
 * device in pipelined chunks; returns when params hold the updated values. */
mco_status mco_flat_step_host(mco_flat* h, void* params, int param_dtype, uint64_t n_params,
                              const void* grads, int grad_dtype, uint64_t n_grads, double lr);

/* List form (beyond the reference's flat spans): `count` parameter tensors and their
 * gradients at separate device pointers (lens[i] elements each, registry order) over
 * the handle's flat state -- tensor i's state is the slice at the sum of the preceding
 * lengths, so results and state equal mco_flat_step over the concatenation bit for bit,
 * without flattening.  sum(lens) <= owned_len.  One launch per 40 tensors. */
mco_status mco_flat_step_list(mco_flat* h, int count, void* const* params, int param_dtype,
                              const void* const* grads, int grad_dtype, const uint64_t* lens,
                              double lr, void* stream);
mco_status mco_flat_get_steps(const mco_flat* h, int64_t* t);  /* steps_taken()     */
mco_status mco_flat_set_steps(mco_flat* h, int64_t t);          /* set_steps_taken() */
/* Graph mode (beyond the reference: CUDA-graph capture of the step).  The step counter
 * moves to the device: the kernels of mco_flat_step / mco_flat_step_mixed derive the
 * step's scalars from it and advance it, so a step captured into a CUDA graph replays
 * as the next step, bit-identical to eager steps (no extra launch per step).  dev_lr: optional device
 * double read at every step (a schedule updates it between replays); null = the lr
 * argument of each call (baked into a captured graph).  Host-span and peer steps are
 * refused in graph mode.  get/set_steps synchronise the device.  Calling enable again
 * only changes dev_lr; disable brings t back to the host. */
mco_status mco_flat_graph_enable(mco_flat* h, const double* dev_lr);
mco_status mco_flat_graph_disable(mco_flat* h);
mco_status mco_flat_state_bytes(const mco_flat* h, uint64_t* out); /* state_bytes_runtime() */
mco_status mco_flat_config(const mco_flat* h, mco_config* out);   /* config()          */
/* buffers(): names in the reference's fixed order m, v, n, h, g_prev (optim.cpp:173-181). */
mco_status mco_flat_num_buffers(const mco_flat* h, int* out);
mco_status mco_flat_buffer(mco_flat* h, int index, const char** name, void** dev_ptr,
                           uint64_t* len, int* dtype);

/* ---- ZeRO step fused with its collectives (parallel.cpp:656-666) ------------
 * One kernel per rank over NVLink peer memory: for the owned flat range
 * [offset, offset+n): g = sum over r of grad_bufs[r][offset+i] (rank order),
 * update master (f32, n elements, may alias this rank's f32 replica) and the
 * optimizer state, then store the new parameter into param_bufs[r][offset+i]
 * for every r (param_dtype F32 or BF16).  grad_bufs / param_bufs are device
 * pointers valid on this device (own buffers or mco_peer_import'ed peers).
 * The caller orders the ranks around the call (grads final before; replicas
 * not read until every rank's call completed). */
mco_status mco_flat_step_peers(mco_flat* h, const void* const* grad_bufs, int grad_dtype,
                               void* const* param_bufs, int param_dtype, int npeers,
                               float* master, uint64_t offset, uint64_t n, double lr,
                               void* stream);
/* LOMO fused with its collectives (C5): sum of squares of the rank-summed
 * gradient over the owned range (all-reduce it across ranks for the global
 * norm), then p = p - f * sum_r g_r written into every rank's replica, f =
 * lr*scale or the clip rule on dev_sumsq.  master: f32 owned copy or NULL
 * (then param_bufs[0] supplies the current value). */
mco_status mco_sumsq_peers(const void* const* grad_bufs, int grad_dtype, int npeers,
                           uint64_t offset, uint64_t n, double* dev_out, void* stream);
mco_status mco_lomo_apply_peers(const void* const* grad_bufs, int grad_dtype,
                                void* const* param_bufs, int param_dtype, int npeers,
                                float* master, uint64_t offset, uint64_t n, double lr,
                                double scale, const double* dev_sumsq, double clip,
                                void* stream);
/* Symmetric buffers: cudaMalloc'ed base allocations and their 64-byte CUDA IPC handles. */
mco_status mco_peer_alloc(uint64_t bytes, int device, void** out);
mco_status mco_peer_free(void* p);
mco_status mco_peer_export(void* p, void* handle_out_64);
mco_status mco_peer_import(const void* handle_64, int device, void** out);
mco_status mco_peer_close(void* p);

/* ---- LOMO (optim.cpp:185-190, 284-318) ------------------------------------ */
/* lomo_apply(Tensor& param, lr, scale): p -= (lr*scale) * g.
 * dtypes: F32/F32, BF16/BF16 (fp32 math, RNE store), F32/BF16, F64/F64. */
mco_status mco_lomo_apply(void* params, int param_dtype, const void* grads, int grad_dtype,
                          uint64_t n, double lr, double scale, void* stream);
/* Same, with the clip scale computed on the device from a device Σg²
 * (optim.cpp:302-303: scale = clip/‖g‖ iff ‖g‖ > clip and ‖g‖ > 0). */
/* LOMO list form: `count` tensors at separate device pointers (lens[i] elements each) in
 * one launch per 40 tensors; each tensor's update equals mco_lomo_apply's bit for bit.
 * dev_sumsq (nullable): device global sum of squares -> clip scale as
 * mco_lomo_apply_clipped (then `scale` is ignored). */
mco_status mco_lomo_apply_list(int count, void* const* params, int param_dtype,
                               const void* const* grads, int grad_dtype, const uint64_t* lens,
                               double lr, double scale, const double* dev_sumsq, double clip,
                               void* stream);
mco_status mco_lomo_apply_clipped(void* params, int param_dtype, const void* grads,
                                  int grad_dtype, uint64_t n, double lr, const double* dev_sumsq,
                                  double clip, void* stream);
/* lomo_apply over HOST arrays (the reference's Tensor data is host memory),
 * pipelined through the device in chunks; clip >= 0 adds the global-norm pass
 * (lomo_fused_backward_step's two passes, optim.cpp:291-316). Synchronous.
 * With clip >= 0 and room on the device, the gradient is held in a device buffer that
 * the library keeps for the next call (see mco_host_release). */
mco_status mco_lomo_apply_host(void* params, int param_dtype, const void* grads, int grad_dtype,
                               uint64_t n, double lr, double scale, double clip);
/* Frees the device buffers the host-span calls keep between calls on every device
 * (mco_lomo_apply_host's resident gradient); waits for a running call to finish. */
mco_status mco_host_release(void);
/* Σx² into *dev_out (fp64, deterministic fixed-order reduction);
 * accumulate != 0 adds to the existing value (optim.cpp:294-300 hook sum). */
mco_status mco_sumsq(const void* x, int dtype, uint64_t n, double* dev_out, int accumulate,
                     void* stream);

/* ---- AdaLomo (optim.hpp:76-96, optim.cpp:192-282) ------------------------- */
typedef struct mco_adalomo mco_adalomo;

/* AdaLomoState(cfg, params): one entry per tensor in registry order;
 * ndim == 2 -> factored v_row[R], v_col[C]; otherwise v_full[numel].
 * State is fp64 on `device`. */
mco_status mco_adalomo_create(const mco_config* cfg, int ntensors, const int* ndims,
                              const int64_t* dims, int device, mco_adalomo** out);
mco_status mco_adalomo_destroy(mco_adalomo* h);
/* Opt-in global grad-norm clip of the gradients before the AdaLomo update (BASELINE
 * C3; no reference counterpart -- the reference's AdaLomoState ignores
 * cfg.clip_threshold, which only LOMO reads, optim.hpp:28, optim.cpp:288-304).  The
 * LOMO rule (optim.cpp:302-303): g *= clip/||g|| iff ||g|| > clip and ||g|| > 0, with
 * ||g|| over every tensor of the call (multi-tensor / phase / host forms) or from the
 * caller's device sum of squares (hook forms).  enable = 0: off (the default). */
mco_status mco_adalomo_set_grad_clip(mco_adalomo* h, int enable, double clip);
/* AdaLomoState::apply(Tensor& param, lr) -- the per-tensor hook form.
 * dev_grad_sumsq: optional device Σg² over ALL tensors (global grad-norm clip; needs
 * mco_adalomo_set_grad_clip, else MCO_CONTRACT); NULL = no clip.  dtypes (param/grad) F32/F32,
 * F32/BF16, BF16/BF16 (bf16 parameters: fp32 arithmetic, RNE store). */
mco_status mco_adalomo_apply(mco_adalomo* h, int tensor_index, void* param, int param_dtype,
                             const void* grad, int grad_dtype, double lr,
                             const double* dev_grad_sumsq, void* stream);
/* List form of the hook: tensors t0..t1-1 (consecutive registry indices) at separate
 * device pointers params[i] / grads[i] -- a bucket of backward-completed gradients
 * applied with one launch chain per 64 tensors instead of one per tensor.  Same
 * result as t1 - t0 mco_adalomo_apply calls. */
mco_status mco_adalomo_apply_list(mco_adalomo* h, int t0, int t1, void* const* params,
                                  int param_dtype, const void* const* grads, int grad_dtype,
                                  double lr, const double* dev_grad_sumsq, void* stream);
/* Multi-tensor form: every tensor at once over registry-order flat buffers
 * (tensor k at element offset sum_{j<k} numel_j).  With mco_adalomo_set_grad_clip
 * the global grad norm over the whole set is computed in the same pass and
 * applied (clip fused into pass 1). */
mco_status mco_adalomo_apply_all(mco_adalomo* h, void* flat_params, int param_dtype,
                                 const void* flat_grads, int grad_dtype, double lr,
                                 void* stream);
/* apply_all over HOST arrays: per-tensor H2D -> apply -> D2H pipeline on three
 * streams (whole-set upload first with the grad-norm clip on).  Synchronous. */
mco_status mco_adalomo_apply_all_host(mco_adalomo* h, void* flat_params, int param_dtype,
                                      const void* flat_grads, int grad_dtype, double lr);
mco_status mco_adalomo_state_bytes(const mco_adalomo* h, uint64_t* out); /* fp64 accounting */
/* Row-split sharding across GPUs: tensor idx is a row slice of a
 * (global_rows x C) matrix or a 1-D replica; weight scales its contribution to
 * the all-reduced statistics (1 for slices; 1 on one rank, 0 elsewhere for replicas). */
mco_status mco_adalomo_set_shard(mco_adalomo* h, int tensor_index, int64_t global_rows,
                                 double weight);
/* apply_all in phases: 1 = pass 1 + statistics payload, 2 = moments + sum u^2
 * payload, 3 = update.  Sharded callers all-reduce (SUM) payload 0 between
 * phases 1 and 2 and payload 1 between phases 2 and 3. */
mco_status mco_adalomo_phase(mco_adalomo* h, int phase, void* flat_params, int param_dtype,
                             const void* flat_grads, int grad_dtype, double lr, void* stream);
mco_status mco_adalomo_payload(mco_adalomo* h, int which, double** dev_ptr, uint64_t* len);
mco_status mco_adalomo_get_steps(const mco_adalomo* h, int tensor_index, int64_t* t);
/* which: 0 v_row, 1 v_col, 2 v_full (fp64 device arrays; len 0 if absent). */
mco_status mco_adalomo_buffer(mco_adalomo* h, int tensor_index, int which, void** dev_ptr,
                              uint64_t* len);

/* ---- ZeRO partition (parallel.cpp:20-38) ------------------------------------ */
/* ZeroPlan::make(total_len, dp_size, stage): part_sizes[dp_size], offsets[dp_size+1]. */
mco_status mco_zero_plan(uint64_t total_len, int dp_size, int stage, uint64_t* part_sizes,
                         uint64_t* offsets);

/* ---- native sharder over NCCL (parallel.cpp:656-666, comm.cpp:193-246) -------
 * NCCL is resolved at run time: the libnccl.so.2 already loaded in the process
 * (e.g. torch's) is reused, else $MCO_NCCL_LIB, else the system libnccl.so.2;
 * failure -> MCO_IO.  NCCL errors -> MCO_PROTOCOL with NCCL's message. */
typedef struct mco_comm mco_comm;
/* 128-byte ncclUniqueId, created on one rank and shipped to the others by the caller. */
mco_status mco_comm_unique_id(void* id_out_128);
mco_status mco_comm_create(const void* id_128, int nranks, int rank, int device,
                           mco_comm** out);
mco_status mco_comm_destroy(mco_comm* c);
/* Failure handling (comm.cpp:126-132 collective timeouts, comm.cpp:330-348 abort with
 * the failing rank named): communicators are non-blocking with a deadline --
 * timeout_s (<= 0: $MCO_NCCL_TIMEOUT_S, default 600 s).  An init that does not complete
 * in time (a rank never joined), an NCCL error, or a mco_comm_wait whose collectives do
 * not finish in time aborts the communicator (ncclCommAbort) and returns MCO_PROTOCOL
 * with "[rank r of N] <what it waited for>"; later calls on it fail the same way. */
mco_status mco_comm_create_timeout(const void* id_128, int nranks, int rank, int device,
                                   double timeout_s, mco_comm** out);
/* Host wait until `stream` (its collectives) completes, bounded by the deadline. */
mco_status mco_comm_wait(mco_comm* c, void* stream);
/* ncclCommAbort (idempotent); the handle still has to be destroyed. */
mco_status mco_comm_abort(mco_comm* c);
/* ncclCommGetAsyncError: MCO_PROTOCOL if the communicator has failed. */
mco_status mco_comm_check(mco_comm* c);
/* In-place SUM all-reduce (LOMO global sum of squares, AdaLomo statistic payloads). */
mco_status mco_comm_allreduce_sum(mco_comm* c, void* buf, int dtype, uint64_t n, void* stream);
/* Stage-2 ZeRO step of ParallelWorker::train_step, stream-ordered:
 * reduce-scatter(SUM) of flat_grads over ZeroPlan(total_len, nranks) parts ->
 * FlatOptimizer step of this rank's part of flat_params (h owns exactly that part:
 * MCO_CONTRACT otherwise) -> all-gather of flat_params in place.  Equal parts use
 * ncclReduceScatter / ncclAllGather; P mod N != 0 uses per-part ncclReduce /
 * ncclBroadcast (the reference's uneven ownership, parallel.cpp:25-32). */
mco_status mco_shard_step(mco_flat* h, mco_comm* c, void* flat_params, int param_dtype,
                          const void* flat_grads, int grad_dtype, uint64_t total_len,
                          double lr, void* stream);
/* Mixed-precision stage 2 (beyond the reference's fp64): the handle
 * (fp32 state) and master_owned (fp32, this rank's ZeroPlan part) cover the owned part;
 * flat_params_bf16 are the bf16 replicas.  RS(grads) -> mco_flat_step_mixed(master,
 * g, replica slice) -> all-gather of the bf16 replicas.  For the vector path, allocate
 * master_owned with the element phase (address / elem size mod 8) of the replica
 * slice it writes. */
mco_status mco_shard_step_mixed(mco_flat* h, mco_comm* c, float* master_owned,
                                uint16_t* flat_params_bf16, const void* flat_grads,
                                int grad_dtype, uint64_t total_len, double lr, void* stream);

/* ---- bucketed, double-buffered stage-2 step (parallel.cpp:656-666) --
 * The registry-order flat vector is cut into buckets of B elements (bucket_elems rounded
 * up to a multiple of 8 N; 0 = one bucket); inside bucket k rank i owns piece i of
 * ZeroPlan(len_k, N) (parallel.cpp:20-34 per bucket), so every rank updates its share of
 * every bucket.  Per bucket, as its local gradient becomes ready: ncclReduceScatter(SUM)
 * on the library's comm stream -> the fused update of this rank's piece on its update
 * stream -> ncclAllGather of the bucket's replicas, issued after the NEXT bucket's
 * reduce-scatter (which therefore overlaps this update).  No full-length gradient has to
 * be resident: a caller can produce bucket k into the library's staging slot
 * (mco_zb_grad_buffer, double-buffered) right before handing it in.  Results equal the
 * whole-vector stage-2 step (elementwise update) and the serial FlatOptimizer on the
 * rank-summed gradient.  replica_dtype F32 (params = replicas) or BF16 (fp32 master of
 * the owned pieces + bf16 replicas: the C4 mixed layout).  State is fp32. */
typedef struct mco_zb mco_zb;
/* The bucket plan alone (host arithmetic): rounded bucket size, bucket count, and rank's
 * piece of bucket k -- registry elements [bucket_off + off, bucket_off + off + n). */
mco_status mco_zb_plan(uint64_t total_len, int nranks, uint64_t bucket_elems, int k, int rank,
                       uint64_t* bucket_rounded, int* nbuckets, uint64_t* bucket_off,
                       uint64_t* bucket_len, uint64_t* off, uint64_t* n);
mco_status mco_zb_create(const mco_config* cfg, mco_comm* c, uint64_t total_len,
                         uint64_t bucket_elems, int grad_dtype, int replica_dtype,
                         mco_zb** out);
mco_status mco_zb_destroy(mco_zb* z);
/* Rounded bucket size, bucket count, owned elements, the state handle (buffers() names /
 * steps over the owned pieces in bucket order; owned by z) and the fp32 master (BF16
 * replicas; NULL otherwise). */
mco_status mco_zb_info(const mco_zb* z, uint64_t* bucket_elems, int* nbuckets,
                       uint64_t* owned, mco_flat** flat, float** master);
/* Rank r's piece of bucket k: registry elements [bucket_off + off, bucket_off + off + n);
 * state_off = its offset in this rank's state (UINT64_MAX for another rank). */
mco_status mco_zb_piece(const mco_zb* z, int k, int rank, uint64_t* bucket_off,
                        uint64_t* bucket_len, uint64_t* off, uint64_t* n, uint64_t* state_off);
/* BF16 replicas: load the fp32 master of the owned pieces from a full registry-order
 * buffer (F32, or BF16 widened exactly). */
mco_status mco_zb_load_master(mco_zb* z, const void* full, int dtype, void* stream);
/* One step: begin (++t, optim.cpp:104) -> grad_ready for every bucket exactly once, in
 * the same order on every rank -> end (stream waits for the last all-gather). */
mco_status mco_zb_begin(mco_zb* z, void* replicas, double lr, void* stream);
/* Staging slot (k mod 2) for bucket k's local gradient; stream waits until it is free. */
mco_status mco_zb_grad_buffer(mco_zb* z, int k, void** dev_ptr, uint64_t* len, void* stream);
/* Bucket k's local gradient is complete on `stream`, at `grad` (len_k elements) or, when
 * grad is NULL, in its staging slot. */
mco_status mco_zb_grad_ready(mco_zb* z, int k, const void* grad, void* stream);
mco_status mco_zb_end(mco_zb* z, void* stream);
/* Ring mode (mco_zb_begin with replicas == NULL; BF16 replicas only, the stage-3 layout
 * for sets whose full replicas do not fit, e.g. 65B Sophia at N = 8): bucket k is
 * gathered into ring slot k mod 2; this returns it (len_k bf16 elements) and makes
 * `stream` wait for its all-gather.  Valid until bucket k+2's update. */
mco_status mco_zb_gathered(mco_zb* z, int k, void** dev_ptr, void* stream);
/* The step's update kernels alone (each piece from this rank's own local gradient, no
 * collectives): the shard-local cost the collectives add to (benchmarks). */
mco_status mco_zb_step_local(mco_zb* z, void* replicas, const void* flat_grads, double lr,
                             void* stream);
/* Whole step from a full local gradient buffer (buckets in reverse registry order;
 * replicas may be NULL in ring mode). */
mco_status mco_zb_step(mco_zb* z, void* replicas, const void* flat_grads, double lr,
                       void* stream);

/* ---- synthetic inputs ------------------------------------------ */
/* Counter-based, stateless generator; values exact in fp32 (bf16 grid for BF16). */
mco_status mco_synth_fill(void* dst, int dtype, uint64_t n, uint64_t seed, uint32_t role,
                          uint32_t tensor, uint32_t step, int64_t cols, int scale_log2,
                          int zero_log2, int rowcol, void* stream);

/* ---- misc -------------------------------------------------------------------- */
mco_status mco_sync(void* stream);                 /* cudaStreamSynchronize + error check */
mco_status mco_device_count(int* out);
/* Tuning knob (no reference counterpart): data-movement variant of the fp32
 * stored-state kernels, process-wide.  "tma" (default: cp.async.bulk + mbarrier
 * producer/consumer pipeline when the call is eligible -- fp32 params / grads / state,
 * 16 B aligned, >= one tile -- else "ldg") or "ldg" (256-bit LDG/STG, persistent
 * grid-stride); other names are the measured alternatives listed in DESIGN.md.
 * Results are bit-identical across variants.  Initial value from the
 * MCO_FLAT_VARIANT environment variable.  CONFIG on an unknown name. */
mco_status mco_set_flat_variant(const char* name);
const char* mco_flat_variant(void);
/* Kernel launches issued by this library on the calling process (counter). */
uint64_t mco_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* MCO_H_ */
