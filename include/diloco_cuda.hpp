// diloco_cuda.hpp — C++ drop-in layer over the C ABI (include/diloco_cuda.h).
//
// Header-only.  Include it in the reference code base (diloco-cpp) after its
// own headers; it provides the reference's signatures backed by the B200
// kernels, so call sites swap `diloco::adamw_step` for
// `diloco::cuda::adamw_step` (or bring the names in with a using-declaration):
//
//   adamw_step / nesterov_step / scaler_unscale_and_check   (optim.hpp:61-77)
//   axpy / encode_fp16 / decode_fp16                         (tensor.hpp:108-115)
//   reduce_average                                           (reduce.hpp:65-66)
//   NcclCollective final : Collective                        (reduce.hpp:86-97)
//   DeviceEngine: DilocoEngine's state and steps resident in HBM (engine.hpp:76-116)
//
// Status codes from the C ABI are rethrown as the reference's exception
// classes (errors.hpp:12-51), so error behaviour is unchanged for callers.
#pragma once

#include <algorithm>
#include <cstdint>
#include <exception>
#include <functional>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "diloco/errors.hpp"
#include "diloco/metrics.hpp"
#include "diloco/optim.hpp"
#include "diloco/reduce.hpp"
#include "diloco/tensor.hpp"
#include "diloco_cuda.h"

namespace diloco::cuda {

inline void throw_status(int st) {
  if (st == DLC_OK) return;
  const std::string msg = dlc_last_error();
  switch (st) {
    case DLC_ESHAPE: throw ShapeError(msg);
    case DLC_ECONFIG: throw ConfigError(msg);
    case DLC_ENUMERIC: throw NumericError(msg);
    case DLC_ECOLLECTIVE:
    case DLC_ENCCL: throw CollectiveError(msg);
    case DLC_ESERIAL: throw SerializationError(msg);
    case DLC_EQUORUM: throw QuorumError(msg);
    default: throw Error(msg);
  }
}

inline int to_c(Precision p) { return p == Precision::fp16 ? DLC_FP16 : DLC_FP32; }

/// adamw_step (optim.hpp:61-62): new params; state.m, state.v, step_count in place.
inline ParamVector adamw_step(AdamWState& state, const ParamVector& params, const ParamVector& grad, float lr) {
  if (!params.same_layout(grad) || !params.same_layout(state.m)) throw ShapeError("adamw_step: layout mismatch");
  dlc_adamw_state s{state.m.mutable_values().data(), state.v.mutable_values().data(), state.step_count,
                    state.beta1, state.beta2, state.eps, state.weight_decay};
  std::vector<float> out(params.size());
  throw_status(dlc_adamw_step(&s, params.values().data(), grad.values().data(), params.size(), lr, out.data()));
  state.step_count = s.step_count;
  return ParamVector(params.layout(), std::move(out));
}

/// nesterov_step (optim.hpp:65-66).
inline ParamVector nesterov_step(NesterovState& state, const ParamVector& params, const ParamVector& pseudo_grad) {
  if (!params.same_layout(pseudo_grad) || !params.same_layout(state.momentum_buf))
    throw ShapeError("nesterov_step: layout mismatch");
  dlc_nesterov_state s{state.momentum_buf.mutable_values().data(), state.lr, state.momentum};
  std::vector<float> out(params.size());
  throw_status(dlc_nesterov_step(&s, params.values().data(), pseudo_grad.values().data(), params.size(), out.data()));
  return ParamVector(params.layout(), std::move(out));
}

/// scaler_unscale_and_check (optim.hpp:76-77).
inline UnscaleResult scaler_unscale_and_check(const LossScaler& scaler, const ParamVector& grad) {
  dlc_loss_scaler s{scaler.scale, scaler.growth_interval, scaler.consecutive_good};
  std::vector<float> out(grad.size());
  int overflow = 0;
  throw_status(dlc_scaler_unscale_and_check(&s, grad.values().data(), grad.size(), out.data(), &overflow));
  UnscaleResult r;
  r.grad = ParamVector(grad.layout(), std::move(out));
  r.overflow = overflow != 0;
  return r;
}

/// axpy (tensor.hpp:108).
inline ParamVector axpy(float alpha, const ParamVector& x, const ParamVector& y) {
  if (!x.same_layout(y)) throw ShapeError("axpy: layout mismatch");
  std::vector<float> out(x.size());
  throw_status(dlc_axpy(alpha, x.values().data(), y.values().data(), x.size(), out.data()));
  return ParamVector(x.layout(), std::move(out));
}

/// encode_fp16 (tensor.hpp:111).
inline Fp16Buffer encode_fp16(const ParamVector& v) {
  Fp16Buffer b;
  b.bits.resize(v.size());
  int overflow = 0;
  throw_status(dlc_encode_fp16(v.values().data(), v.size(), b.bits.data(), &overflow));
  b.overflow = overflow != 0;
  return b;
}

/// decode_fp16 (tensor.hpp:115).
inline ParamVector decode_fp16(const Fp16Buffer& buffer, LayoutPtr layout) {
  if (buffer.bits.size() != layout->total_length()) throw ShapeError("decode_fp16: length mismatch");
  std::vector<float> out(buffer.bits.size());
  throw_status(dlc_decode_fp16(buffer.bits.data(), buffer.bits.size(), out.data()));
  return ParamVector(std::move(layout), std::move(out));
}

/// reduce_average (reduce.hpp:65-66).
inline ParamVector reduce_average(std::span<const ParamVector* const> contributions, Precision precision) {
  if (contributions.empty()) throw CollectiveError("reduce_average: no contributions");
  const ParamVector& first = *contributions.front();
  std::vector<const float*> ptrs;
  for (const ParamVector* c : contributions) {
    if (!c->same_layout(first)) throw ShapeError("reduce_average: contribution layout mismatch");
    ptrs.push_back(c->values().data());
  }
  std::vector<float> out(first.size());
  throw_status(dlc_reduce_average(ptrs.data(), ptrs.size(), first.size(), to_c(precision), out.data()));
  return ParamVector(first.layout(), std::move(out));
}

/// Collective plugin over NCCL: one rank per process and GPU (replaces
/// SocketCollective, collective.hpp:160-178).  Rank 0 creates the id with
/// make_unique_id() and ships it to the other ranks out of band.
class NcclCollective final : public Collective {
 public:
  static std::vector<uint8_t> make_unique_id() {
    std::vector<uint8_t> id(128);
    throw_status(dlc_nccl_unique_id(id.data()));
    return id;
  }

  NcclCollective(int rank, int world, const std::vector<uint8_t>& id, int device,
                 dlc_reduce_mode mode = DLC_MODE_ORDERED) {
    if (id.size() != 128) throw ConfigError("NcclCollective: unique id must be 128 bytes");
    throw_status(dlc_collective_create_nccl(rank, world, id.data(), device, mode, &c_));
  }
  ~NcclCollective() override { dlc_collective_destroy(c_); }
  NcclCollective(const NcclCollective&) = delete;
  NcclCollective& operator=(const NcclCollective&) = delete;

  size_t world_size() const override { return dlc_collective_world_size(c_); }

  PseudoGradient all_reduce_avg(const PseudoGradient& local, ReduceReport* report) override {
    PseudoGradient out;
    std::vector<float> mean(local.delta.size());
    dlc_reduce_report rep{};
    throw_status(dlc_collective_all_reduce_avg(c_, local.delta.values().data(), local.delta.size(),
                                               to_c(local.precision), local.outer_epoch, mean.data(), &rep));
    out.delta = ParamVector(local.delta.layout(), std::move(mean));
    out.precision = local.precision;
    out.outer_epoch = local.outer_epoch;
    if (report) {
      *report = ReduceReport{};
      report->outer_epoch = rep.outer_epoch;
      report->contributors = rep.contributors;
      report->data_bytes_sent = rep.data_bytes_sent;
      report->data_bytes_received = rep.data_bytes_received;
      report->wire_bytes_sent = rep.wire_bytes_sent;
      report->wire_bytes_received = rep.wire_bytes_received;
      report->wall_ms = rep.wall_ms;
      report->attempts = rep.attempts;
    }
    return out;
  }

  dlc_collective* handle() const { return c_; }

  /// Survivors-only membership change (collective.cpp:1369-1395): this world
  /// minus `exclude`, survivors in order; QuorumError below `quorum_min`,
  /// CollectiveError("excluded from round") for an excluded caller.
  std::unique_ptr<NcclCollective> shrink(const std::vector<int>& exclude, size_t quorum_min = 1,
                                         bool abort_pending = false) {
    dlc_collective* n = nullptr;
    throw_status(dlc_collective_shrink(c_, exclude.data(), exclude.size(), quorum_min,
                                       abort_pending ? DLC_SHRINK_ABORT : DLC_SHRINK_DEFAULT, &n));
    return std::unique_ptr<NcclCollective>(new NcclCollective(n));
  }

  /// Original ranks of the current members (the round's sorted contributors).
  std::vector<int> members() const {
    std::vector<int> r(32);
    r.resize(std::min<size_t>(dlc_collective_members(c_, r.data(), r.size()), r.size()));
    return r;
  }

  void set_reduce_timeout_ms(uint64_t ms) { throw_status(dlc_collective_set_reduce_timeout_ms(c_, ms)); }

 private:
  explicit NcclCollective(dlc_collective* c) : c_(c) {}
  dlc_collective* c_ = nullptr;
};

/// DilocoEngine's optimizer state resident in HBM (engine.hpp:76-116).  The
/// gradient producer (task/model) stays with the caller: inner_step takes the
/// gradient of one batch; outer_step runs pseudo-gradient -> all-reduce ->
/// Nesterov on the device.
class DeviceEngine {
 public:
  DeviceEngine(const dlc_config& cfg, const dlc_hyperparams& hyper, const ParamVector& theta0, int device,
               dlc_inner_mode mode = DLC_INNER_PINGPONG)
      : layout_(theta0.layout()) {
    throw_status(dlc_engine_create(&cfg, &hyper, theta0.size(), device, mode, &e_));
    throw_status(dlc_engine_upload(e_, DLC_THETA_T, theta0.values().data(), theta0.size()));
    throw_status(dlc_engine_upload(e_, DLC_THETA_LOCAL, theta0.values().data(), theta0.size()));
  }
  ~DeviceEngine() { dlc_engine_destroy(e_); }
  DeviceEngine(const DeviceEngine&) = delete;
  DeviceEngine& operator=(const DeviceEngine&) = delete;

  /// apply_inner_step with the gradient of one batch (engine.cpp:50-69).
  dlc_inner_result inner_step(const ParamVector& grad) {
    if (!grad.layout() || !(*grad.layout() == *layout_)) throw ShapeError("inner_step: layout mismatch");
    dlc_inner_result r{};
    throw_status(dlc_engine_inner_step_host(e_, grad.values().data(), 0, &r));
    return r;
  }

  /// compute_pseudo_gradient -> all_reduce_avg -> outer_step (engine.cpp:165-172).
  dlc_outer_result outer_step(NcclCollective* collective = nullptr) {
    dlc_outer_result r{};
    throw_status(dlc_engine_outer_step(e_, collective ? collective->handle() : nullptr, &r, nullptr));
    return r;
  }

  /// The same outer round through ANY reference Collective, e.g. a
  /// SocketCollective between boxes: the pseudo-gradient
  /// is staged to the host, averaged by `collective`, and applied on the device.
  /// Returns OuterStepResult::applied (engine.hpp:64-66).
  bool outer_step(Collective& collective, Precision precision, ReduceReport* report = nullptr) {
    std::vector<float> d(layout_->total_length());
    uint64_t epoch = 0;
    throw_status(dlc_engine_compute_pseudo_gradient(e_, d.data(), &epoch));
    PseudoGradient pg;
    pg.delta = ParamVector(layout_, std::move(d));
    pg.precision = precision;
    pg.outer_epoch = epoch;
    const PseudoGradient reduced = collective.all_reduce_avg(pg, report);
    if (!reduced.delta.same_layout(pg.delta)) throw ShapeError("outer_step: reduced layout mismatch");
    dlc_outer_result r{};
    throw_status(dlc_engine_apply_outer_step(e_, reduced.delta.values().data(), reduced.outer_epoch, &r));
    return r.applied != 0;
  }

  ParamVector download(dlc_buffer which) const {
    std::vector<float> h(layout_->total_length());
    throw_status(dlc_engine_download(e_, which, h.data(), h.size()));
    return ParamVector(layout_, std::move(h));
  }

  dlc_engine_scalars scalars() const {
    dlc_engine_scalars s{};
    throw_status(dlc_engine_get_scalars(e_, &s));
    return s;
  }

  dlc_engine* handle() const { return e_; }

  // ---- wire rounds for the reference's TCP Node (diloco_cuda.h section 5) ----
  /// K2 into the DELTA buffer in the engine's precision; returns the outer epoch.
  uint64_t wire_begin() {
    uint64_t epoch = 0;
    throw_status(dlc_engine_wire_begin(e_, &epoch));
    return epoch;
  }
  /// The bytes send_chunk_span (collective.cpp:1318-1345) puts on the wire for
  /// DELTA / MEAN [offset, offset + length).
  std::vector<uint8_t> wire_encode(int which, uint64_t offset, uint64_t length, const dlc_wire_tags& tags) {
    size_t bytes = 0;
    throw_status(dlc_wire_frames_size(length, &tags, &bytes, nullptr));
    std::vector<uint8_t> out(bytes);
    size_t used = 0;
    throw_status(dlc_engine_wire_encode(e_, which, offset, length, &tags, out.data(), out.size(), &used));
    out.resize(used);
    return out;
  }
  /// Decodes the complete frames of `bytes` into a fold row / MEAN; returns the bytes consumed.
  size_t wire_decode(int which, int row, uint64_t base_offset, uint64_t capacity, const std::vector<uint8_t>& bytes,
                     std::vector<dlc_wire_chunk>* chunks = nullptr) {
    size_t n_chunks = 0, consumed = 0;
    std::vector<dlc_wire_chunk> scratch(chunks ? 4096 : 0);
    throw_status(dlc_engine_wire_decode(e_, which, row, base_offset, capacity, bytes.data(), bytes.size(),
                                        chunks ? scratch.data() : nullptr, scratch.size(), &n_chunks, &consumed));
    if (chunks) chunks->assign(scratch.begin(), scratch.begin() + std::min(n_chunks, scratch.size()));
    return consumed;
  }
  void wire_fold(int rank, int k, uint64_t offset, uint64_t length) {
    throw_status(dlc_engine_wire_fold(e_, rank, k, offset, length));
  }
  dlc_outer_result wire_finish(uint64_t epoch) {
    dlc_outer_result r{};
    throw_status(dlc_engine_wire_finish(e_, epoch, &r));
    return r;
  }

 private:
  LayoutPtr layout_;
  dlc_engine* e_ = nullptr;
};

/// DilocoOptimizer (engine.hpp:122-140, engine.cpp:162-174) on a DeviceEngine:
/// step() runs one inner step and, after every H-th, the outer round; for a
/// single worker the window's last inner step and the outer step run as one
/// fused pass (dlc_optimizer_step).  The producer (task.cpp) stays with the
/// caller, so step() takes the raw gradient of one batch instead of a Batch.
class DeviceOptimizer {
 public:
  explicit DeviceOptimizer(DeviceEngine& engine, NcclCollective* collective = nullptr)
      : engine_(engine), collective_(collective) {
    throw_status(dlc_engine_device_ptr(engine_.handle(), DLC_GRAD, &grad_));
  }

  /// InnerStepResult's lr and overflow_skipped (engine.hpp:58-62).
  dlc_inner_result step(const ParamVector& grad) {
    throw_status(dlc_engine_upload(engine_.handle(), DLC_GRAD, grad.values().data(), grad.size()));
    int done = 0;
    throw_status(dlc_optimizer_step(engine_.handle(), collective_ ? collective_->handle() : nullptr, grad_, 0, &done));
    const dlc_engine_scalars s = engine_.scalars();
    round_completed_ = done != 0;
    if (round_completed_) last_applied_ = s.last_applied != 0;
    dlc_inner_result r{};
    r.lr = s.last_lr;
    r.overflow_skipped = s.last_overflow;
    return r;
  }
  void zero_grad() {}
  bool round_just_completed() const { return round_completed_; }
  bool last_round_applied() const { return last_applied_; }

 private:
  DeviceEngine& engine_;
  NcclCollective* collective_ = nullptr;
  float* grad_ = nullptr;
  bool round_completed_ = false;
  bool last_applied_ = false;
};

/// One sample of the gradient producer (task.cpp's loss_and_grad, out of
/// scope here): a DEVICE gradient on the engine's device and its loss.
struct GradSample {
  const float* grad = nullptr;
  bool scaled = false;  // already multiplied by the current loss scale
  float loss = 0.0f;
};

/// run_training (engine.cpp:176-240) on a DeviceEngine: the same loop, the
/// same MetricsRecord stream into the reference's MetricsSink, the same
/// on_round hook; returns the RunResult fields (engine.hpp:142-150).
inline dlc_run_result run_training(DeviceEngine& engine, NcclCollective* collective,
                                   const std::function<GradSample(uint64_t)>& producer, const MetricsSink& sink,
                                   int worker_index = 0, const std::function<void(uint64_t)>& on_round = {}) {
  struct Ctx {
    const std::function<GradSample(uint64_t)>* producer;
    const MetricsSink* sink;
    const std::function<void(uint64_t)>* on_round;
    std::exception_ptr error;
  } ctx{&producer, &sink, &on_round, nullptr};
  auto produce = [](void* u, uint64_t step, const float** grad, int* scaled, float* loss) -> int {
    auto* c = static_cast<Ctx*>(u);
    try {
      const GradSample g = (*c->producer)(step);
      *grad = g.grad;
      *scaled = g.scaled ? 1 : 0;
      *loss = g.loss;
      return 0;
    } catch (...) {
      c->error = std::current_exception();
      return 1;
    }
  };
  auto emit = [](void* u, const dlc_metrics_record* r) {
    auto* c = static_cast<Ctx*>(u);
    if (!*c->sink) return;
    MetricsRecord m;
    m.kind = r->kind == DLC_RECORD_STEP ? RecordKind::step
             : r->kind == DLC_RECORD_ROUND ? RecordKind::round
                                           : RecordKind::event;
    m.worker = r->worker;
    m.inner_step = r->inner_step;
    m.outer_epoch = r->outer_epoch;
    m.loss = r->loss;
    m.perplexity = r->perplexity;
    m.lr = r->lr;
    m.compute_ms = r->compute_ms;
    m.comm_ms = r->comm_ms;
    m.bytes_sent = r->bytes_sent;
    m.contributors = r->contributors;
    if (r->event) m.event = r->event;
    (*c->sink)(m);
  };
  auto round = [](void* u, uint64_t n) {
    auto* c = static_cast<Ctx*>(u);
    if (*c->on_round) (*c->on_round)(n);
  };
  dlc_run_result res{};
  const int st = dlc_run_training(engine.handle(), collective ? collective->handle() : nullptr, produce, emit, round,
                                  &ctx, worker_index, &res);
  if (ctx.error) std::rethrow_exception(ctx.error);
  throw_status(st);
  return res;
}

}  // namespace diloco::cuda
