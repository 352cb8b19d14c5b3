/*
 * diloco_cuda.h — C ABI of the B200-native DiLoCo optimizer hot path.
 *
 * Drop-in boundary for the reference C++ library (diloco-cpp,
 * /root/reference/proj).  Plain pointers and sizes, `int` status codes, no
 * C++ or torch types.  Every entry point names the reference interface it
 * replaces (file:line under proj/).  Implemented by libdiloco_cuda.so
 * (paper_2407_07852_b200/csrc, sm_100a kernels + NCCL); there is no CPU
 * fallback: without a CUDA device every compute call fails with DLC_ECUDA.
 *
 * Errors.  C cannot throw, so each reference exception maps to a status
 * (errors.hpp:12-51); dlc_last_error() returns the calling thread's message:
 *   DLC_ESHAPE      ShapeError       layout / length mismatch
 *   DLC_ECONFIG     ConfigError      bad hyperparameter / config
 *   DLC_ENUMERIC    NumericError     non-finite input where finite math is required
 *   DLC_ECOLLECTIVE CollectiveError  epoch mismatch, no contributions
 *   DLC_ENCCL       CollectiveError  NCCL failure
 *   DLC_EQUORUM     QuorumError      membership below quorum_min (errors.hpp:42)
 *   DLC_ECUDA       Error            CUDA failure / no device
 *   DLC_EINVAL      Error            null pointer or out-of-range argument
 * Overflow is a signal, not an error (UnscaleResult.overflow,
 * Fp16Buffer.overflow, OuterStepResult.applied), exactly as in the reference.
 *
 * Threading (reduce.hpp:84-85).  One engine per worker thread
 * and GPU; no internal locking.  Host-buffer calls block the caller; engine
 * calls are stream-ordered on the engine's stream and return immediately
 * unless a result struct is requested.
 */
#ifndef DILOCO_CUDA_H_
#define DILOCO_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DLC_ABI_VERSION 1

#if defined(__GNUC__)
#define DLC_API __attribute__((visibility("default")))
#else
#define DLC_API
#endif

enum dlc_status {
  DLC_OK = 0,
  DLC_ESHAPE = 1,
  DLC_ECONFIG = 2,
  DLC_ENUMERIC = 3,
  DLC_ECOLLECTIVE = 4,
  DLC_ECUDA = 5,
  DLC_ENCCL = 6,
  DLC_EINVAL = 7,
  DLC_ESERIAL = 8, /* SerializationError, errors.hpp:48 (wire frames) */
  DLC_EQUORUM = 9  /* QuorumError, errors.hpp:42 (membership change below quorum) */
};

/* Precision, reduce.hpp:22 */
enum dlc_precision { DLC_FP32 = 0, DLC_FP16 = 1 };
/* LrDecay, optim.hpp:38 */
enum dlc_lr_decay { DLC_LR_NONE = 0, DLC_LR_COSINE = 1 };

DLC_API int dlc_abi_version(void);
/* Message of the last failing call on this thread ("" if none). */
DLC_API const char* dlc_last_error(void);
DLC_API int dlc_device_count(int* count);
/* Selects the calling thread's device for the host-buffer math below. */
DLC_API int dlc_set_device(int device);

/* =========================================================================
 * 1. Reference math over HOST buffers.  Same argument meaning, ownership and
 *    error behaviour as the reference free functions; each call stages
 *    through the calling thread's current device and synchronises.
 * ========================================================================= */

/* AdamWState, optim.hpp:17-28 (m, v: host arrays of n, updated in place). */
typedef struct {
  float* m;
  float* v;
  uint64_t step_count;
  float beta1, beta2, eps, weight_decay;
} dlc_adamw_state;

/* NesterovState, optim.hpp:30-36 (momentum_buf: host array of n). */
typedef struct {
  float* momentum_buf;
  float lr;
  float momentum;
} dlc_nesterov_state;

/* LrSchedule, optim.hpp:40-45 */
typedef struct {
  uint64_t warmup_steps;
  uint64_t total_steps;
  float base_lr;
  int decay; /* dlc_lr_decay */
} dlc_lr_schedule;

/* LossScaler, optim.hpp:52-56 */
typedef struct {
  float scale;
  uint64_t growth_interval;
  uint64_t consecutive_good;
} dlc_loss_scaler;

/* axpy, tensor.hpp:108 / tensor.cpp:118-129: out = y + alpha * x. */
DLC_API int dlc_axpy(float alpha, const float* x, const float* y, size_t n, float* out);
/* encode_fp16, tensor.hpp:111 / tensor.cpp:131-140 (RNE, overflow -> inf). */
DLC_API int dlc_encode_fp16(const float* v, size_t n, uint16_t* out, int* overflow);
/* decode_fp16, tensor.hpp:115 / tensor.cpp:142-154 (exact). */
DLC_API int dlc_decode_fp16(const uint16_t* bits, size_t n, float* out);
/* ParamVector::all_finite, tensor.hpp:86 / tensor.cpp:97-104. */
DLC_API int dlc_all_finite(const float* v, size_t n, int* all_finite);
/* lr_at, optim.hpp:49 / optim.cpp:37-56 (host scalar). */
DLC_API float dlc_lr_at(const dlc_lr_schedule* schedule, uint64_t step);
/* adamw_step, optim.hpp:61-62 / optim.cpp:58-93: out = new params; state m, v,
 * step_count updated.  DLC_ECONFIG on lr < 0, DLC_ENUMERIC on a non-finite
 * gradient (state untouched). */
DLC_API int dlc_adamw_step(dlc_adamw_state* state, const float* params, const float* grad, size_t n,
                   float lr, float* out);
/* nesterov_step, optim.hpp:65-66 / optim.cpp:95-115. */
DLC_API int dlc_nesterov_step(dlc_nesterov_state* state, const float* params, const float* pseudo_grad,
                      size_t n, float* out);
/* scaler_scale_loss, optim.hpp:68 / optim.cpp:117-119. */
DLC_API float dlc_scaler_scale_loss(const dlc_loss_scaler* scaler, float loss);
/* scaler_unscale_and_check, optim.hpp:76-77 / optim.cpp:121-135. */
DLC_API int dlc_scaler_unscale_and_check(const dlc_loss_scaler* scaler, const float* grad, size_t n,
                                 float* out, int* overflow);
/* scaler_update, optim.hpp:80 / optim.cpp:137-148 (host scalar). */
DLC_API void dlc_scaler_update(dlc_loss_scaler* scaler, int overflow);
/* reduce_average, reduce.hpp:65-66 / reduce.cpp:46-89: mean of k host vectors
 * folded in index order; DLC_FP16 reproduces the wire path (one encode per
 * contribution, one of the mean).  DLC_ECOLLECTIVE when k == 0. */
DLC_API int dlc_reduce_average(const float* const* contributions, size_t k, size_t n, int precision,
                       float* out);
/* partition_ranges / per_peer_reduce_bytes / fleet_reduce_bytes,
 * reduce.hpp:55,78-82 / reduce.cpp:20-31,91-111 (host integers). */
DLC_API void dlc_partition_ranges(size_t n, size_t k, size_t* offsets, size_t* lengths);
DLC_API uint64_t dlc_per_peer_reduce_bytes(size_t n, size_t k, size_t rank, int precision);
DLC_API uint64_t dlc_fleet_reduce_bytes(size_t n, size_t k, int precision);

/* =========================================================================
 * 2. Collective plugin, class Collective (reduce.hpp:86-97).
 * ========================================================================= */

typedef struct dlc_collective dlc_collective;

/* ReduceReport, reduce.hpp:37-46 */
typedef struct {
  uint64_t outer_epoch;
  size_t contributors;
  uint64_t data_bytes_sent;
  uint64_t data_bytes_received;
  uint64_t wire_bytes_sent;
  uint64_t wire_bytes_received;
  double wall_ms;
  uint32_t attempts;
} dlc_reduce_report;

/* DLC_MODE_ORDERED: NCCL grouped send/recv scatter -> owner fold in rank order
 *   (K3) -> NCCL all-gather; bit-identical to reduce_average in rank order.
 * DLC_MODE_ALLREDUCE: ncclAllReduce(ncclAvg) on the flat buffer; NCCL's
 *   reduction order, within the tolerance stated in DESIGN.md. */
enum dlc_reduce_mode { DLC_MODE_ORDERED = 0, DLC_MODE_ALLREDUCE = 1, DLC_MODE_P2P = 2 };
/* DLC_MODE_P2P: the same rank-ordered fold as ORDERED, fused with the data
 *   movement over NVLink peer memory (CUDA IPC): each owner folds its slot
 *   straight out of the peers' send buffers, and the outer Nesterov kernel
 *   reads every owner's mean slot in place, so there are no recv / gather
 *   copies in HBM.  Flag barriers over NVLink order the phases; they are also
 *   the failure detector (a peer silent for reduce_timeout_ms fails the round
 *   with DLC_ECOLLECTIVE and leaves the engine's state unchanged).  Bitwise
 *   equal to ORDERED.  Engine path only; the host-buffer plugin call uses
 *   ORDERED semantics. */

/* 128-byte ncclUniqueId, created on rank 0 and shipped to every rank. */
DLC_API int dlc_nccl_unique_id(uint8_t id[128]);
/* SocketCollective replacement: one rank per process and GPU. */
DLC_API int dlc_collective_create_nccl(int rank, int world, const uint8_t id[128], int device, int mode,
                               dlc_collective** out);
/* SoloCollective, reduce.hpp:101-106. */
DLC_API int dlc_collective_create_solo(int device, dlc_collective** out);
DLC_API int dlc_collective_destroy(dlc_collective* c);
DLC_API size_t dlc_collective_world_size(const dlc_collective* c);
DLC_API int dlc_collective_rank(const dlc_collective* c);
/* Collective::all_reduce_avg on a HOST pseudo-gradient (reduce.hpp:95-96). */
DLC_API int dlc_collective_all_reduce_avg(dlc_collective* c, const float* local_delta, size_t n,
                                  int precision, uint64_t outer_epoch, float* out,
                                  dlc_reduce_report* report);

/* Membership.  The reference's Node restarts a failed
 * round over the live members minus the suspects: contributors sorted, quorum
 * checked, rank = position, divisor = contributor count
 * (collective.cpp:1369-1395; test_collective.cpp:460-531).  On one NVLink box:
 *
 *   dlc_collective_shrink   called by the SURVIVORS only (ncclCommShrink):
 *                           a new collective over the world minus
 *                           `exclude_ranks` (ranks of `c`), survivors keeping
 *                           their relative order.  DLC_ECOLLECTIVE "excluded
 *                           from round" when the caller is in the list,
 *                           DLC_EQUORUM when fewer than max(quorum_min, 1)
 *                           ranks remain.  DLC_SHRINK_ABORT first aborts
 *                           operations still pending on `c`.  An engine made
 *                           for num_workers_k >= the new world re-lays its
 *                           owner slots at its next outer step on the new
 *                           collective (ReduceReport::contributors = survivors,
 *                           attempts = failed tries at this epoch + 1).
 *                           `c` stays valid (destroy aborts its communicator).
 *   dlc_collective_members  original ranks of the current members, sorted;
 *                           returns the member count.
 *   dlc_collective_set_reduce_timeout_ms
 *                           NodeOptions::reduce_timeout_ms (default 20000):
 *                           how long a DLC_MODE_P2P barrier waits for a peer
 *                           (on the device; the round then fails on every
 *                           rank with the state unchanged), and how long after
 *                           it was enqueued an ORDERED / ALLREDUCE round may
 *                           take before a host wait on the engine (a result,
 *                           a download, dlc_engine_synchronize) declares it
 *                           failed: DLC_ECOLLECTIVE "timed out".  NCCL never
 *                           times out, so that round's device work stays
 *                           blocked until the survivors call
 *                           dlc_collective_shrink with DLC_SHRINK_ABORT; it
 *                           then finishes without changing the engine state
 *                           (speculative K4, error-gated finish), and the
 *                           same epoch is retried on the shrunk collective
 *                           (ReduceReport::attempts = 2).  A timed-out
 *                           collective is marked broken: destroying it aborts
 *                           the blocked work too (do that before destroying
 *                           the engine, whose destroy waits for its stream).
 *   dlc_collective_inject_stall
 *                           fault injection (SocketCollective::set_stage_hook,
 *                           test_collective.cpp:485-492): this rank stops
 *                           arriving from its `barrier_index`-th P2P barrier
 *                           on (counted from now; < 0 disables), so its round
 *                           and its peers' rounds fail with DLC_ECOLLECTIVE. */
enum dlc_shrink_flags { DLC_SHRINK_DEFAULT = 0, DLC_SHRINK_ABORT = 1 };
DLC_API int dlc_collective_shrink(dlc_collective* c, const int* exclude_ranks, size_t n_exclude, size_t quorum_min,
                                  int flags, dlc_collective** out);
DLC_API size_t dlc_collective_members(const dlc_collective* c, int* ranks, size_t cap);
DLC_API int dlc_collective_set_reduce_timeout_ms(dlc_collective* c, uint64_t ms);
DLC_API int dlc_collective_inject_stall(dlc_collective* c, int64_t barrier_index);

/* DLC_MODE_P2P tuning (development sweeps; no reference counterpart).  All
 * fields zero = the measured defaults: piece plan 1,2,3,2,1
 * (1,2,2,1 below 400M params per worker, 16 equal pieces on the host-buffer
 * path), max(16, 320 / K) fold CTAs, 128 / 256 / 512 fold threads for
 * K <= 4 / <= 6 / <= 8, one piece-kernel CTA per 256-vector window.
 * Process-wide; applies from the next outer step.  NULL restores the defaults. */
typedef struct {
  uint32_t plan[32]; /* relative piece weights inside an owner slot (1..1024 each) */
  uint32_t plan_len; /* 0 = default plan */
  int32_t fold_ctas;    /* TMA fold CTAs, 0 = default */
  int32_t fold_threads; /* 128, 256 or 512; 0 = default by K */
  int32_t piece_ctas;   /* K2 / K4 piece kernels' grid, 0 = one CTA per window */
  int32_t fold_kernel;  /* 0 = single-leader TMA fold (default), 1 = warp-specialised TMA fold */
} dlc_p2p_tuning;
DLC_API int dlc_p2p_set_tuning(const dlc_p2p_tuning* t);
DLC_API int dlc_p2p_get_tuning(dlc_p2p_tuning* t);

/* =========================================================================
 * 3. Device-resident engine: DilocoEngine (engine.hpp:76-116) with theta_t,
 *    theta_local, AdamW m/v, Nesterov buffer, loss scaler and counters all in
 *    HBM.  The inner step, pseudo-gradient, collective and outer step never
 *    leave the GPU.
 * ========================================================================= */

/* DilocoConfig, engine.hpp:22-32 (batch_size belongs to the out-of-scope
 * gradient producer). */
typedef struct {
  uint64_t local_steps_h;
  size_t num_workers_k;
  int reduce_precision; /* dlc_precision */
  uint64_t total_inner_steps;
} dlc_config;

/* OptimHyperparams, engine.hpp:34-46 */
typedef struct {
  float inner_lr;
  uint64_t warmup_steps;
  int lr_decay;
  float weight_decay, beta1, beta2, adam_eps;
  float outer_lr, outer_momentum;
  float scaler_init_scale;
  uint64_t scaler_growth_interval;
} dlc_hyperparams;

/* Engine scalars (EngineState engine.hpp:48-56 minus the vectors). */
typedef struct {
  uint64_t step_count;      /* AdamWState::step_count */
  uint64_t inner_step;      /* data cursor */
  uint64_t outer_epoch;
  float scale;              /* LossScaler::scale */
  uint64_t consecutive_good;
  uint64_t overflow_skips;
  uint64_t outer_skips;
  float last_lr;            /* InnerStepResult::lr */
  int last_overflow;        /* InnerStepResult::overflow_skipped */
  int last_applied;         /* OuterStepResult::applied */
} dlc_engine_scalars;

/* K1 variants.  PINGPONG: one HBM pass (28 B/param), p/m/v alternate between
 * two buffers and the live one is picked on the device.  INPLACE: fixed
 * addresses, an overflow pre-pass over the gradient then a gated in-place
 * update (32 B/param). */
enum dlc_inner_mode { DLC_INNER_PINGPONG = 0, DLC_INNER_INPLACE = 1 };

/* Buffers of one engine. */
enum dlc_buffer {
  DLC_THETA_T = 0,
  DLC_THETA_LOCAL = 1,
  DLC_ADAM_M = 2,
  DLC_ADAM_V = 3,
  DLC_MOMENTUM = 4,
  DLC_GRAD = 5 /* gradient staging buffer owned by the engine */
};

typedef struct dlc_engine dlc_engine;

DLC_API void dlc_hyperparams_default(dlc_hyperparams* h);
/* Allocates every buffer on `device` (theta zero-initialised; load weights with
 * dlc_engine_upload(DLC_THETA_T) and (DLC_THETA_LOCAL)).  DLC_ECONFIG per
 * DilocoConfig::validate (engine.cpp:31-48). */
DLC_API int dlc_engine_create(const dlc_config* cfg, const dlc_hyperparams* hyper, size_t n_params,
                      int device, int inner_mode, dlc_engine** out);
DLC_API int dlc_engine_destroy(dlc_engine* e);
DLC_API size_t dlc_engine_size(const dlc_engine* e);
/* The engine's CUDA stream (cudaStream_t), for producers of gradients. */
DLC_API int dlc_engine_stream(dlc_engine* e, void** stream);
/* Host <-> device copies of one buffer (synchronous). */
DLC_API int dlc_engine_upload(dlc_engine* e, int which, const float* host, size_t n);
DLC_API int dlc_engine_download(dlc_engine* e, int which, float* host, size_t n);
/* Elements [offset, offset + count) of one buffer (synchronous). */
DLC_API int dlc_engine_download_range(dlc_engine* e, int which, size_t offset, float* host, size_t count);
DLC_API int dlc_engine_upload_range(dlc_engine* e, int which, size_t offset, const float* host, size_t count);
/* Current device address of a buffer (synchronises: the live p/m/v buffer is
 * chosen on the device in PINGPONG mode). */
DLC_API int dlc_engine_device_ptr(dlc_engine* e, int which, float** dev);
DLC_API int dlc_engine_get_scalars(dlc_engine* e, dlc_engine_scalars* out);
DLC_API int dlc_engine_set_scalars(dlc_engine* e, const dlc_engine_scalars* in);
DLC_API int dlc_engine_synchronize(dlc_engine* e);

/* InnerStepResult, engine.hpp:58-62 (loss belongs to the producer). */
typedef struct {
  float lr;
  int overflow_skipped;
} dlc_inner_result;

/* apply_inner_step minus the producer (engine.cpp:50-69): unscale + overflow
 * check + AdamW + scaler update, skip semantics on overflow.  `grad` is a
 * device pointer on the engine's device; `grad_is_scaled` = 1 when it is
 * already multiplied by the current loss scale (backward of the scaled loss),
 * 0 to have the engine apply scale_gradient (engine.cpp:20-27) first.
 * `result` may be NULL (asynchronous); otherwise the call synchronises. */
DLC_API int dlc_engine_inner_step(dlc_engine* e, const float* grad, int grad_is_scaled,
                          dlc_inner_result* result);
/* Same with a HOST gradient (copied to DLC_GRAD first). */
DLC_API int dlc_engine_inner_step_host(dlc_engine* e, const float* host_grad, int grad_is_scaled,
                               dlc_inner_result* result);

/* OuterStepResult, engine.hpp:64-66 */
typedef struct {
  int applied;
  uint64_t outer_epoch; /* epoch after the step */
} dlc_outer_result;

/* DilocoOptimizer::step's outer part (engine.cpp:165-172): K2 pseudo-gradient
 * -> Collective::all_reduce_avg on device buffers -> K4 outer Nesterov +
 * theta_local refresh.  `c` NULL or solo => K = 1.  DLC_ECOLLECTIVE when the
 * collective's world size differs from num_workers_k or when called
 * mid-window (engine.cpp:116-120).  `result` / `report` may be NULL. */
DLC_API int dlc_engine_outer_step(dlc_engine* e, dlc_collective* c, dlc_outer_result* result,
                          dlc_reduce_report* report);
/* Outer step whose theta(t+h) comes from a caller-owned DEVICE buffer (a model
 * trained outside the engine); the engine's theta_local is refreshed as usual. */
DLC_API int dlc_engine_outer_step_from(dlc_engine* e, dlc_collective* c, const float* theta_local_dev,
                                       dlc_outer_result* result, dlc_reduce_report* report);
/* Host-buffer outer round for drop-in callers whose inner loop runs on the
 * host: theta_local is uploaded, the outer step runs, theta_t is downloaded. */
DLC_API int dlc_engine_outer_step_host(dlc_engine* e, dlc_collective* c, const float* host_theta_local,
                               float* host_theta_t, dlc_outer_result* result);
/* The outer step split around a collective that runs outside this library
 * (e.g. the reference's SocketCollective between boxes,
 * fed from D2H-staged buffers):
 *   dlc_engine_compute_pseudo_gradient = DilocoEngine::compute_pseudo_gradient
 *     (engine.cpp:115-126): the raw FP32 delta = theta_t - theta_local into a
 *     host buffer of n, plus the engine's outer epoch (the PseudoGradient tag);
 *     Error when mid-window.
 *   dlc_engine_apply_outer_step = DilocoEngine::outer_step (engine.cpp:128-146)
 *     on a host FP32 mean: CollectiveError on an epoch mismatch, Nesterov only
 *     when every element is finite, theta_local := theta_t always. */
DLC_API int dlc_engine_compute_pseudo_gradient(dlc_engine* e, float* host_delta, uint64_t* outer_epoch);
DLC_API int dlc_engine_apply_outer_step(dlc_engine* e, const float* host_mean, uint64_t outer_epoch,
                                        dlc_outer_result* result);
/* K engines of one process on one device (in-process fleet, the device
 * analogue of run_simulated's outer round, netsim.cpp:325-357): pseudo-grads,
 * one fold in index order, K outer steps. */
DLC_API int dlc_engines_outer_step_local(dlc_engine* const* engines, size_t k, dlc_outer_result* result);

/* Single-process multi-GPU world: K engines, engine r on devices[r], driven by
 * ONE host thread (the device analogue of run_simulated's K workers,
 * netsim.cpp:325-357, and of SURVEY.md §8b's dlc_world_create).  DLC_MODE_P2P
 * joins the engines by direct NVLink peer access (no IPC, no communicator);
 * ORDERED / ALLREDUCE use communicators from ncclCommInitAll with the
 * per-rank calls grouped, and need one device per rank; in DLC_MODE_P2P the
 * ranks synchronise through CUDA events, so several may share a device.
 * The engines belong to the world (use dlc_world_engine for inner steps,
 * uploads and downloads; do not destroy them).  dlc_world_outer_step runs
 * every rank's outer step; `result` (may be NULL: asynchronous) is rank 0's,
 * checked equal on every rank. */
typedef struct dlc_world dlc_world;
DLC_API int dlc_world_create(const dlc_config* cfg, const dlc_hyperparams* hyper, size_t n_params, const int* devices,
                             int inner_mode, int mode, dlc_world** out);
DLC_API int dlc_world_destroy(dlc_world* w);
DLC_API int dlc_world_engine(dlc_world* w, int rank, dlc_engine** e);
DLC_API int dlc_world_outer_step(dlc_world* w, dlc_outer_result* result);
/* Membership change of a world: the next rounds run
 * over the current ranks minus `exclude_ranks`, survivors kept in order and
 * renumbered 0..k'-1, divisor k' (collective.cpp:1369-1395).  The excluded
 * engines are destroyed; the survivors re-lay their owner slots for k'
 * (ReduceReport::contributors = k').  The window rule of the reference holds:
 * call it between rounds (every engine at a window boundary).  DLC_EQUORUM when
 * fewer than max(quorum_min, 1) ranks would remain, DLC_ECONFIG for a rank out
 * of range; on error nothing changes.  ORDERED / ALLREDUCE worlds get fresh
 * communicators over the survivors' devices.  The failure detector of a
 * one-thread world is its caller (every rank is driven by it), so this is the
 * planned exclusion of the reference's fleet; the flag-barrier timeout
 * (dlc_collective_set_reduce_timeout_ms) detects silent peers of the one
 * process per GPU path. */
DLC_API int dlc_world_shrink(dlc_world* w, const int* exclude_ranks, size_t n_exclude, size_t quorum_min);
/* Original ranks (at dlc_world_create) of the current members, in rank order;
 * returns the member count. */
DLC_API size_t dlc_world_members(const dlc_world* w, int* ranks, size_t cap);

/* DilocoOptimizer::step (engine.cpp:162-174): one inner step, then the outer
 * step when the window boundary is reached.  `round_completed` may be NULL. */
DLC_API int dlc_optimizer_step(dlc_engine* e, dlc_collective* c, const float* grad, int grad_is_scaled,
                       int* round_completed);

/* run_training (engine.cpp:176-240): total_inner_steps inner steps with an
 * outer round every H, one record per step and per round (and per skip
 * event) through `sink` with the fields of MetricsRecord (metrics.hpp:19-34),
 * `on_round` after every completed round (the checkpoint hook).  The gradient
 * producer (task.cpp, out of scope here) is the caller's `producer`: given the
 * inner step, it returns a DEVICE gradient on the engine's device (loss-scaled
 * when *grad_is_scaled), the step's loss, and 0 (non-zero aborts with
 * DLC_EINVAL).  `sink` / `on_round` may be NULL.  Result: RunResult
 * (engine.hpp:142-150).  The loop keeps up to two steps queued on the GPU:
 * the producer is called for step t + 2 before step t's records reach the
 * sink.  Every step the producer depends on is enqueued by then, and engine
 * reads (downloads) synchronize the stream, so a producer sees theta_local
 * after step t + 1.  It drains at a window boundary when K > 1 or `on_round`
 * is set, so the hook sees the boundary's state. */
enum dlc_record_kind { DLC_RECORD_STEP = 0, DLC_RECORD_ROUND = 1, DLC_RECORD_EVENT = 2 };
typedef struct {
  int kind;
  int worker;
  uint64_t inner_step, outer_epoch;
  float loss, perplexity, lr;
  double compute_ms, comm_ms;
  uint64_t bytes_sent;
  size_t contributors;
  const char* event; /* kind == DLC_RECORD_EVENT: "inner_overflow_skip" | "outer_skip_nonfinite" */
} dlc_metrics_record;
typedef struct {
  uint64_t steps_done, rounds_done;
  float final_train_loss;
  uint64_t reduce_data_bytes, reduce_wire_bytes;
  double comm_ms, compute_ms;
} dlc_run_result;
typedef int (*dlc_grad_producer)(void* user, uint64_t inner_step, const float** grad, int* grad_is_scaled,
                                 float* loss);
typedef void (*dlc_metrics_sink)(void* user, const dlc_metrics_record* record);
typedef void (*dlc_round_hook)(void* user, uint64_t rounds_done);
DLC_API int dlc_run_training(dlc_engine* e, dlc_collective* c, dlc_grad_producer producer, dlc_metrics_sink sink,
                             dlc_round_hook on_round, void* user, int worker_index, dlc_run_result* out);

/* Checkpoint / resume of device-resident engines in the reference's ODLCKPT1
 * format (save_checkpoint / load_checkpoint, checkpoint.cpp:17,74-198):
 * magic, config hash, completed rounds, clock, reduce bytes, utilization
 * ledger, then per engine the FP64-text scalar header (checkpoint.cpp:74-91)
 * and serialize_param_vector blocks (tensor.cpp:188-200) of theta_t,
 * theta_local, m, v and the momentum buffer.  Files are interchangeable with
 * the reference's.  The Layout is `nseg` named segments of `seg_lengths`
 * (NULL names: one segment "p" covering the vector).  Vectors stream through
 * a pinned staging buffer. */
typedef struct {
  uint64_t config_hash;
  uint64_t completed_rounds;
  double clock_seconds;
  uint64_t reduce_data_bytes;
  size_t ledger_workers;  /* entries in `ledger` (compute, comm, idle seconds each) */
  const double* ledger;   /* save: 3 * ledger_workers doubles, may be NULL when 0 */
} dlc_checkpoint_meta;
DLC_API int dlc_checkpoint_save(dlc_engine* const* engines, size_t count, const char* path,
                                const dlc_checkpoint_meta* meta, const char* const* seg_names,
                                const uint64_t* seg_lengths, size_t nseg);
/* Restores `count` engines (sizes must match, ShapeError otherwise);
 * meta_out (may be NULL) receives the header fields (ledger = NULL).  All or
 * nothing: the whole file is parsed and validated first (SerializationError
 * for a truncated file, a missing key or a bad number; ShapeError for a
 * layout or length mismatch), and no engine changes unless every engine
 * restores.  The _layout variant also checks every vector's segment names and
 * lengths against the caller's Layout (restore_state, engine.cpp:148-155). */
DLC_API int dlc_checkpoint_load(dlc_engine* const* engines, size_t count, const char* path,
                                dlc_checkpoint_meta* meta_out);
DLC_API int dlc_checkpoint_load_layout(dlc_engine* const* engines, size_t count, const char* path,
                                       const char* const* seg_names, const uint64_t* seg_lengths, size_t nseg,
                                       dlc_checkpoint_meta* meta_out);

/* Per-phase device timing with CUDA events on the engine stream (ncu-free
 * evidence for the roofline): phase 0 = K1 inner AdamW, 1 = K2 pseudo-grad,
 * 2 = collective (C1 + K3 fold), 3 = K4 outer Nesterov.  dlc_engine_phase_times
 * synchronises, returns the summed milliseconds and launch counts since the
 * previous call, and resets them. */
enum { DLC_PHASE_INNER = 0, DLC_PHASE_PSEUDO = 1, DLC_PHASE_COLLECTIVE = 2, DLC_PHASE_OUTER = 3 };
DLC_API int dlc_engine_set_timing(dlc_engine* e, int on);
DLC_API int dlc_engine_phase_times(dlc_engine* e, double total_ms[4], uint64_t count[4]);

/* One worker (num_workers_k = 1, solo collective, either inner mode): dlc_optimizer_step
 * and dlc_run_training run the window's last inner step and the outer step as
 * ONE fused pass (K1 + K2 + K4, 40 B/param instead of 28 + 20; INPLACE
 * engines 48 instead of 32 + 24; the result is bit-identical, and an overflow
 * on that inner step reruns the outer step from the unchanged theta_local).
 * On by default; `on` = 0 runs them as two steps.
 * num_workers_k > 1: K2 fused into the window's last inner step (opt-in,
 * default off).  The inner step that completes a window of H also
 * writes delta = theta_t - theta_local' (engine.cpp:115-126, in the reduce
 * precision) into the collective's send buffer, so the outer step starts with
 * the exchange instead of a separate 10-12 B/param K2 pass.  Results are
 * bit-identical either way: the outer step still runs a gated K2 that
 * recomputes the delta when that inner step overflowed (theta_local kept its
 * old value), and every engine call that writes theta_t / theta_local or the
 * send buffer between the two (uploads, set_scalars, checkpoint load, wire
 * rounds, host-buffer and explicit-source outer steps) drops the fused delta.
 * Writes through a pointer from dlc_engine_device_ptr made AFTER that inner
 * step are not seen: make them before it, or leave fusion off.  Off by
 * default because the window boundary (that inner step + the outer step) is
 * not faster with it on this pool's B200 boxes: the P2P outer step is bound by
 * the NVLink exchange and K4, not by K2. */
DLC_API int dlc_engine_set_fused_delta(dlc_engine* e, int on);

/* =========================================================================
 * 4. Synthetic inputs and test probes (bench / parity tests).  Counter-based
 *    streams identical to the reference's CounterRng (rng.hpp:38-74).
 * ========================================================================= */

/* key of CounterRng(seed, purpose, index) */
DLC_API uint64_t dlc_rng_key(uint64_t seed, const char* purpose, uint64_t index);
/* dev[i] = draw (first + i) of the stream `key`, uniform in [lo, hi). */
DLC_API int dlc_rng_fill_device(dlc_engine* e, int which, uint64_t key, uint64_t first, float lo, float hi);
/* dst = theta_t - U(lo, hi) drawn from `key` (synthetic end-of-window weights);
 * dst = NULL writes the engine's own theta_local, else a caller device buffer of n. */
DLC_API int dlc_rng_perturb(dlc_engine* e, float* dst, uint64_t key, float lo, float hi);
/* FP16 codes of the 2^32 FP32 bit patterns [start, start + n) (host out). */
DLC_API int dlc_fp16_encode_bits(uint32_t start, size_t n, uint16_t* out);
/* The P2P owner fold (K3 + push) on HOST buffers staged through the current
 * device: k contributions of n elements (FP32 values or FP16 codes per
 * `precision`, n a multiple of 64) folded in order into `out` by the
 * per-thread kernel (tma = 0), the single-leader TMA kernel (tma = 1) or the
 * warp-specialised TMA kernel (tma = 2; TMA needs k in 2..8, else the
 * per-thread kernel runs); *nonfinite = the mark the owner pushes.  Probe for
 * the kernels every world size uses. */
DLC_API int dlc_fold_push_probe(const void* const* contribs, int k, size_t n, int precision, int tma, void* out,
                                int* nonfinite);

/* Kernel probe for the K > 1 outer step on ONE device (development / ncu tool,
 * no reference counterpart): allocates full-size synthetic buffers for n
 * parameters and k owner slots and times, each averaged over `reps` launches,
 * ms3[0] = K2 pseudo_grad_piece over a whole slot range (10 / 12 B/param FP16 /
 * FP32), ms3[1] = the owner fold + mean push over k local rows (the DRAM bytes
 * one GPU serves and receives in the exchange: 2w B/param), ms3[2] = K4
 * nesterov_p2p_piece (16 + w B/param).  Lets ncu capture the multi-GPU kernels
 * in a single process. */
DLC_API int dlc_p2p_kernels_probe(int k, size_t n, int precision, int reps, float* ms3);
/* The same, plus overlap_ms[0] = K4 per launch while the fold (fold_ctas CTAs,
 * 0 = one per SM) runs back to back on a second stream, overlap_ms[1] = the
 * fold per launch meanwhile: on-chip interference without NVLink. */
DLC_API int dlc_p2p_overlap_probe(int k, size_t n, int precision, int reps, int fold_ctas, float* ms3,
                                  float* overlap_ms);

/* =========================================================================
 * 5. Wire codec for cross-box transports.
 *
 *    The reference's TCP collective moves pseudo-gradient slices as framed
 *    messages.  These calls produce and consume exactly those bytes straight
 *    from / into DEVICE buffers, so a transport between boxes (the
 *    reference's Node, or any socket code) never touches a host copy of the
 *    vector: frames are assembled in the caller's (ideally pinned) host
 *    buffer by strided copy-engine transfers, one per run of full chunks.
 *    Byte-exact with:
 *      encode_frame            wire.cpp:10-22   "ODLC" | 1 | type | u64 len | payload
 *      encode_reduce_payload   wire.cpp:74-88   epoch u64 | chunk_index u32 | precision u8 | segment
 *      encode_chunk_segment    collective.cpp:63-81  u64 1 | u64 name_len | name | u64 offset | u64 length | scalars
 *      chunk_name              collective.cpp:126-131, PeerId::hex collective.cpp:214-220
 *      send_chunk_span         collective.cpp:1318-1345 (max(1, chunk_size_bytes / width) elements per frame)
 *    and, on receipt, FrameParser::next (wire.cpp:38-72), decode_reduce_payload
 *    (wire.cpp:90-104), decode_chunk_segment (collective.cpp:90-118) and the
 *    drop rules of handle_reduce_chunk (collective.cpp:1017-1047).
 * ========================================================================= */

enum dlc_msg_type { DLC_MSG_REDUCE_CHUNK = 5, DLC_MSG_REDUCE_RESULT = 6 }; /* MsgType, wire.hpp:31-41 */

typedef struct {
  uint8_t msg_type;          /* DLC_MSG_REDUCE_CHUNK (scatter) | DLC_MSG_REDUCE_RESULT (all-gather) */
  int precision;             /* DLC_FP32 | DLC_FP16: element width 4 | 2 */
  uint64_t outer_epoch;
  uint32_t attempt;          /* barrier attempt of the round */
  uint32_t partition;        /* owner range index */
  uint64_t from_hi, from_lo; /* PeerId of the producer (the scatter sender, or the owner for results) */
  uint64_t chunk_size_bytes; /* NodeOptions::chunk_size_bytes (collective.hpp:93, default 1 MiB) */
} dlc_wire_tags;

typedef struct {
  uint8_t msg_type;
  uint8_t precision;
  int accepted;              /* 1: scalars copied to the device; 0: dropped (see dlc_wire_decode) */
  uint32_t chunk_index;
  uint32_t attempt, partition;
  uint64_t outer_epoch;
  uint64_t from_hi, from_lo;
  uint64_t offset, length;   /* global element range of the chunk */
  uint64_t frame_offset, frame_bytes;
} dlc_wire_chunk;

/* Bytes and frames send_chunk_span produces for `elems` elements. */
DLC_API int dlc_wire_frames_size(uint64_t elems, const dlc_wire_tags* tags, size_t* bytes, uint64_t* frames);
/* Frames for the DEVICE scalars dev[0, elems) (FP16 codes or FP32 values),
 * element `global_offset` first, into host_out (cap bytes; DLC_ESHAPE when
 * short).  Synchronous with respect to `stream` (NULL: the legacy stream). */
DLC_API int dlc_wire_encode(const void* dev_scalars, uint64_t global_offset, uint64_t elems, const dlc_wire_tags* tags,
                            uint8_t* host_out, size_t cap, size_t* used, void* stream);
/* Parses the complete frames at the front of host_in and copies each accepted
 * chunk's scalars to dev_out[offset - base_offset] (capacity elements).
 * DLC_ESERIAL on a malformed frame (bad magic / version / length / type,
 * truncated payload or segment, segment count != 1), with *consumed = the
 * bytes before it.  A trailing incomplete frame is left unconsumed.  Dropped,
 * not errors: frames of other message types, unparsable chunk names and size
 * mismatches (collective.cpp:1022-1029), a precision other than `precision`,
 * ranges outside [base_offset, base_offset + capacity).  `chunks` (may be NULL)
 * receives up to max_chunks descriptors.  Synchronous. */
DLC_API int dlc_wire_decode(const uint8_t* host_in, size_t bytes, int precision, uint64_t base_offset,
                            uint64_t capacity, void* dev_out, dlc_wire_chunk* chunks, size_t max_chunks,
                            size_t* n_chunks, size_t* consumed, void* stream);

/* Engine side of a wire round (the device data plane of Node::Impl::all_reduce,
 * collective.cpp:1347-1595; the control plane - barrier, commit, membership -
 * stays with the transport):
 *   begin   K2 over the whole vector into the DELTA buffer in the engine's
 *           precision (encode once at the source, collective.cpp:1356-1366);
 *           returns the outer epoch that tags the round.  Error when mid-window.
 *   encode  frames of DELTA or MEAN [offset, offset + length) (scatter a
 *           partition to its owner / relay an owner's mean).
 *   decode  frames into fold ROW `row` (contributor index, base = the owned
 *           range's offset) or into MEAN (base 0).
 *   fold    owner fold (collective.cpp:1456-1489): contributors 0..k-1 in
 *           order, row `rank` read from DELTA, mean encoded once into
 *           MEAN[offset, offset + length).
 *   finish  DilocoEngine::outer_step on MEAN (engine.cpp:128-146): epoch
 *           guard, finite gate, Nesterov, theta_local := theta_t. */
enum dlc_wire_buffer { DLC_WIRE_DELTA = 0, DLC_WIRE_MEAN = 1, DLC_WIRE_ROW = 2 };
DLC_API int dlc_engine_wire_begin(dlc_engine* e, uint64_t* outer_epoch);
DLC_API int dlc_engine_wire_encode(dlc_engine* e, int which, uint64_t offset, uint64_t length,
                                   const dlc_wire_tags* tags, uint8_t* host_out, size_t cap, size_t* used);
DLC_API int dlc_engine_wire_decode(dlc_engine* e, int which, int row, uint64_t base_offset, uint64_t capacity,
                                   const uint8_t* host_in, size_t bytes, dlc_wire_chunk* chunks, size_t max_chunks,
                                   size_t* n_chunks, size_t* consumed);
DLC_API int dlc_engine_wire_fold(dlc_engine* e, int rank, int k, uint64_t offset, uint64_t length);
DLC_API int dlc_engine_wire_finish(dlc_engine* e, uint64_t outer_epoch, dlc_outer_result* result);

#ifdef __cplusplus
}
#endif

#endif /* DILOCO_CUDA_H_ */
