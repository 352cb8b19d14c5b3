// training.cu — run_training (engine.cpp:176-240) around the device engine:
// the reference's training loop with its metrics records, the gradient
// producer (task.cpp, out of scope) supplied by the caller.
#include <chrono>
#include <cmath>
#include <string>

#include "engine_impl.hpp"

using namespace dlc;

namespace {

using Clock = std::chrono::steady_clock;

double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

}  // namespace

extern "C" {

int dlc_run_training(dlc_engine* e, dlc_collective* c, dlc_grad_producer producer, dlc_metrics_sink sink,
                     dlc_round_hook on_round, void* user, int worker_index, dlc_run_result* out) {
  return guard([&] {
    if (!e || !producer || !out) fail(DLC_EINVAL, "dlc_run_training: null argument");
    if (c && c->kind == 0) c = nullptr;
    DeviceGuard dg(e->device);
    *out = dlc_run_result{};
    while (e->issued_inner < e->cfg.total_inner_steps) {  // !engine.finished()
      const auto compute_start = Clock::now();
      const float* grad = nullptr;
      int grad_is_scaled = 1;
      float loss = 0.0f;
      if (producer(user, e->issued_inner, &grad, &grad_is_scaled, &loss) != 0)
        fail(DLC_EINVAL, "run_training: the gradient producer failed at inner step " +
                             std::to_string(e->issued_inner));
      if (e->n && !grad) fail(DLC_EINVAL, "run_training: the gradient producer returned no gradient");
      // DilocoOptimizer::step (engine.cpp:162-174)
      engine_inner(e, grad, grad_is_scaled);
      const bool boundary = e->issued_inner % e->cfg.local_steps_h == 0;
      dlc_reduce_report report{};
      bool applied = false;
      if (boundary) {
        check_collective(e, c);
        const uint64_t epoch = read_state(e).outer_epoch;
        outer_round(e, c, nullptr, &report);
        fill_report(e, c, &report, epoch);
      }
      const DevState s = read_state(e);  // synchronises: the step's result is final
      if (boundary) {
        check_barrier(e);
        applied = s.last_applied != 0;
      }
      const double total_ms = ms_since(compute_start);
      out->steps_done += 1;
      out->final_train_loss = loss;

      dlc_metrics_record record{};
      record.kind = DLC_RECORD_STEP;
      record.worker = worker_index;
      record.inner_step = s.inner_step;
      record.outer_epoch = s.outer_epoch;
      record.loss = loss;
      record.perplexity = std::exp(loss);  // task.cpp:544-546
      record.lr = s.last_lr;
      if (s.last_overflow && sink) {
        dlc_metrics_record event = record;
        event.kind = DLC_RECORD_EVENT;
        event.event = "inner_overflow_skip";
        sink(user, &event);
      }
      if (boundary) {
        out->rounds_done += 1;
        out->reduce_data_bytes += report.data_bytes_sent;
        out->reduce_wire_bytes += report.wire_bytes_sent;
        out->comm_ms += report.wall_ms;
        record.compute_ms = total_ms - report.wall_ms;
        out->compute_ms += record.compute_ms;
        if (sink) {
          sink(user, &record);
          dlc_metrics_record round = record;
          round.kind = DLC_RECORD_ROUND;
          round.comm_ms = report.wall_ms;
          round.bytes_sent = report.data_bytes_sent;
          round.contributors = report.contributors;
          sink(user, &round);
          if (!applied) {
            dlc_metrics_record event = round;
            event.kind = DLC_RECORD_EVENT;
            event.event = "outer_skip_nonfinite";
            sink(user, &event);
          }
        }
        if (on_round) on_round(user, out->rounds_done);
      } else {
        record.compute_ms = total_ms;
        out->compute_ms += total_ms;
        if (sink) sink(user, &record);
      }
    }
  });
}

}  // extern "C"
