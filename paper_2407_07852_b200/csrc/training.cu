// training.cu — run_training (engine.cpp:176-240) around the device engine:
// the reference's training loop with its metrics records, the gradient
// producer (task.cpp, out of scope) supplied by the caller.
#include <cmath>
#include <deque>
#include <string>

#include "engine_impl.hpp"

using namespace dlc;


extern "C" {

// The loop never waits for the GPU between inner steps: each step's K1 (and,
// at a window boundary, the outer round) is enqueued, followed by an
// asynchronous copy of the engine's device scalars into a pinned ring slot and
// a timing event.  A step's records are emitted two steps behind, once its
// event has completed, so the GPU always has the next two steps queued while
// the host formats records and calls the producer (one step of slack was not
// enough to hide the Python callbacks of 0.7 ms steps).  At a window boundary the loop
// drains when a fleet's barrier check (K > 1) must raise before the next inner
// step is queued, or when an on_round hook (a checkpoint) must see the
// boundary's state; otherwise a boundary is emitted two steps behind like any
// other step.  The record stream is the reference's (engine.cpp:181-238); only the
// interleaving of producer calls and sink calls differs (producer(t + 2) runs
// before step t's records are emitted).  compute_ms / comm_ms are CUDA-event
// times of the step and of its collective on the device, not host wall time.
int dlc_run_training(dlc_engine* e, dlc_collective* c, dlc_grad_producer producer, dlc_metrics_sink sink,
                     dlc_round_hook on_round, void* user, int worker_index, dlc_run_result* out) {
  return guard([&] {
    if (!e || !producer || !out) fail(DLC_EINVAL, "dlc_run_training: null argument");
    if (c && c->kind == 0) c = nullptr;
    DeviceGuard dg(e->device);
    *out = dlc_run_result{};
    constexpr int kRing = dlc_engine::kRing;
    if (!e->ring_host) {
      DLC_CUDA(cudaMallocHost(&e->ring_host, kRing * sizeof(DevState)));
      for (int i = 0; i < kRing; ++i) {
        DLC_CUDA(cudaEventCreate(&e->ring_a[i]));
        DLC_CUDA(cudaEventCreate(&e->ring_b[i]));
      }
    }
    struct {
      DevState* host;
      cudaEvent_t *a, *b;
    } ring{e->ring_host, e->ring_a, e->ring_b};
    struct Pending {
      int slot;
      float loss;
      bool boundary;
    };
    std::deque<Pending> pending;
    auto emit = [&](const Pending& p) {
      if (p.boundary && e->k > 1) stream_wait(e);  // a timed-out NCCL round raises instead of blocking
      DLC_CUDA(cudaEventSynchronize(ring.b[p.slot]));
      const DevState s = ring.host[p.slot];
      float step_ms = 0.0f;
      DLC_CUDA(cudaEventElapsedTime(&step_ms, ring.a[p.slot], ring.b[p.slot]));
      dlc_reduce_report report{};
      bool applied = false;
      if (p.boundary) {
        if (e->k > 1) check_barrier(e);  // a failed round raises CollectiveError here
        fill_report(e, c, &report, s.outer_epoch - 1);
        applied = s.last_applied != 0;
      }
      out->steps_done += 1;
      out->final_train_loss = p.loss;
      dlc_metrics_record record{};
      record.kind = DLC_RECORD_STEP;
      record.worker = worker_index;
      record.inner_step = s.inner_step;
      record.outer_epoch = s.outer_epoch;
      record.loss = p.loss;
      record.perplexity = std::exp(p.loss);  // task.cpp:544-546
      record.lr = s.last_lr;
      if (s.last_overflow && sink) {
        dlc_metrics_record event = record;
        event.kind = DLC_RECORD_EVENT;
        event.event = "inner_overflow_skip";
        sink(user, &event);
      }
      if (p.boundary) {
        out->rounds_done += 1;
        out->reduce_data_bytes += report.data_bytes_sent;
        out->reduce_wire_bytes += report.wire_bytes_sent;
        out->comm_ms += report.wall_ms;
        record.compute_ms = step_ms - report.wall_ms;
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
        record.compute_ms = step_ms;
        out->compute_ms += step_ms;
        if (sink) sink(user, &record);
      }
    };
    while (e->issued_inner < e->cfg.total_inner_steps) {  // !engine.finished()
      const uint64_t t = e->issued_inner;
      const float* grad = nullptr;
      int grad_is_scaled = 1;
      float loss = 0.0f;
      if (producer(user, t, &grad, &grad_is_scaled, &loss) != 0)
        fail(DLC_EINVAL, "run_training: the gradient producer failed at inner step " + std::to_string(t));
      if (e->n && !grad) fail(DLC_EINVAL, "run_training: the gradient producer returned no gradient");
      const int slot = (int)(t % kRing);
      DLC_CUDA(cudaEventRecord(ring.a[slot], e->stream));
      // DilocoOptimizer::step (engine.cpp:162-174); a single worker's window
      // boundary runs as one fused pass (engine_boundary_solo)
      const bool fused = boundary_solo_ok(e, c);
      if (fused)
        engine_boundary_solo(e, grad, grad_is_scaled);
      else
        engine_inner(e, grad, grad_is_scaled);
      const bool boundary = e->issued_inner % e->cfg.local_steps_h == 0;
      dlc_reduce_report rep{};
      if (boundary && !fused) {
        check_collective(e, c);
        outer_round(e, c, nullptr, &rep);  // records the collective's events for fill_report
      }
      DLC_CUDA(cudaMemcpyAsync(&ring.host[slot], e->st, sizeof(DevState), cudaMemcpyDeviceToHost, e->stream));
      DLC_CUDA(cudaEventRecord(ring.b[slot], e->stream));
      pending.push_back({slot, loss, boundary});
      // two steps behind (kRing = 4 slots: at most 3 in flight); drain at a boundary when a fleet's failed round must
      // raise before the next inner step runs, or when the on_round hook (the
      // checkpoint hook, engine.hpp:154) must see the state of that boundary
      const bool drain = boundary && (e->k > 1 || on_round);
      while (!pending.empty() && (drain || pending.size() > 2)) {
        const Pending p = pending.front();
        pending.pop_front();
        emit(p);
      }
    }
    while (!pending.empty()) {
      const Pending p = pending.front();
      pending.pop_front();
      emit(p);
    }
  });
}

}  // extern "C"
