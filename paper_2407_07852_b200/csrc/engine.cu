// engine.cu — section 3 of include/diloco_cuda.h: the C ABI of the
// device-resident DilocoEngine (engine.hpp:76-157).  Its state is
// engine_impl.hpp; the outer step's collectives are p2p.cu.
//
// HBM layout of one engine (one worker, one GPU), every buffer 256-B aligned:
//   theta_t[2][N], buf[2][N]       outer weights, momentum  FP32 ping-pong pair
//   p[2][N], m[2][N], v[2][N]      theta_local + AdamW      FP32 ping-pong pair
//                                  (one buffer each in INPLACE mode; theta_local
//                                  may follow theta_t[ocur], Pair::follow)
//   grad[N]                        gradient staging          FP32
//   send[K*S]                      pseudo-gradient, padded   FP32 | FP16 codes
//   recv[K*S], gather[K*S]         scatter / all-gather      (K > 1)
//   flags[kMaxK], DevState, lr/corr tables
// S = ceil(N / K) rounded up to 512 elements: rank r owns send[r*S, (r+1)*S).
// The partition differs from partition_ranges (reduce.cpp:20-31) only by the
// padding; results are independent of the split because the fold is
// elementwise, and the scalar bytes on the wire are the same
// 2(K-1)/K*N*{4,2} per peer.
#include <chrono>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "engine_impl.hpp"

using namespace dlc;

extern "C" {

void dlc_hyperparams_default(dlc_hyperparams* h) {
  // OptimHyperparams defaults, engine.hpp:34-46
  h->inner_lr = 4e-4f;
  h->warmup_steps = 1000;
  h->lr_decay = DLC_LR_NONE;
  h->weight_decay = 0.1f;
  h->beta1 = 0.9f;
  h->beta2 = 0.95f;
  h->adam_eps = 1e-8f;
  h->outer_lr = 0.7f;
  h->outer_momentum = 0.9f;
  h->scaler_init_scale = 65536.0f;
  h->scaler_growth_interval = 2000;
}

int dlc_engine_create(const dlc_config* cfg, const dlc_hyperparams* hyper, size_t n, int device, int inner_mode,
                      dlc_engine** out) {
  dlc_engine* e = nullptr;
  const int st = guard([&] {
    if (!cfg || !hyper || !out) fail(DLC_EINVAL, "dlc_engine_create: null argument");
    *out = nullptr;
    // DilocoConfig::validate, engine.cpp:31-48
    if (cfg->local_steps_h < 1) fail(DLC_ECONFIG, "local_steps must be >= 1");
    if (cfg->num_workers_k < 1) fail(DLC_ECONFIG, "num_workers must be >= 1");
    if (cfg->total_inner_steps == 0 || cfg->total_inner_steps % cfg->local_steps_h != 0)
      fail(DLC_ECONFIG, "total_inner_steps (" + std::to_string(cfg->total_inner_steps) +
                            ") must be a positive multiple of local_steps (" + std::to_string(cfg->local_steps_h) +
                            ")");
    if (cfg->num_workers_k > (size_t)kMaxK) fail(DLC_ECONFIG, "num_workers_k exceeds 32");
    if (cfg->reduce_precision != DLC_FP32 && cfg->reduce_precision != DLC_FP16)
      fail(DLC_ECONFIG, "unknown reduce precision");
    if (inner_mode != DLC_INNER_PINGPONG && inner_mode != DLC_INNER_INPLACE) fail(DLC_ECONFIG, "unknown inner mode");
    DeviceGuard dg(device);
    e = new dlc_engine();
    e->device = device;
    e->cfg = *cfg;
    e->hyper = *hyper;
    e->inner_mode = inner_mode;
    e->n = n;
    e->k = cfg->num_workers_k;
    e->prec = cfg->reduce_precision;
    e->fuse_delta = e->k == 1;  // K = 1: the fused window boundary; K > 1: opt-in
    e->S = slot_elems(n, e->k);
    // the collective buffers also fit every smaller fleet a membership change
    // (dlc_collective_shrink) can leave behind
    e->k_cap = e->k;
    for (size_t kk = 1; kk <= e->k; ++kk) e->slot_cap = std::max(e->slot_cap, kk * slot_elems(n, kk));
    DLC_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    DLC_CUDA(cudaEventCreate(&e->ev0));
    DLC_CUDA(cudaEventCreate(&e->ev1));
    const size_t vb = n * sizeof(float);
    // theta_t / momentum ping-pong: the fused solo step (K = 1) and the pipelined
    // P2P step (K > 1) write the new values speculatively into the idle buffer
    for (int i = 0; i < 2; ++i) {
      e->theta_t[i] = (float*)dalloc(e, vb);
      e->buf[i] = (float*)dalloc(e, vb);
    }
    const int pairs = inner_mode == DLC_INNER_PINGPONG ? 2 : 1;
    for (int i = 0; i < pairs; ++i) {
      e->p[i] = (float*)dalloc(e, vb);
      e->m[i] = (float*)dalloc(e, vb);
      e->v[i] = (float*)dalloc(e, vb);
    }
    if (pairs == 1) {
      e->p[1] = e->p[0];
      e->m[1] = e->m[0];
      e->v[1] = e->v[0];
    }
    e->grad = (float*)dalloc(e, vb);
    const size_t pb = e->slot_cap * elem_width(e->prec);
    e->send = dalloc(e, pb);
    DLC_CUDA(cudaMemsetAsync(e->send, 0, pb, e->stream));  // padding stays zero
    if (e->k > 1) {
      e->recv = dalloc(e, pb);
      e->gather = dalloc(e, pb);
      DLC_CUDA(cudaMemsetAsync(e->gather, 0, pb, e->stream));
      e->barrier_buf = (int*)dalloc(e, 256);
      e->sig = (uint64_t*)dalloc(e, kMaxK * sizeof(uint64_t));
      e->sig_err = (int*)dalloc(e, 256);
      DLC_CUDA(cudaMemsetAsync(e->sig, 0, kMaxK * sizeof(uint64_t), e->stream));
      DLC_CUDA(cudaMemsetAsync(e->sig_err, 0, 256, e->stream));
    }
    e->flags = (int*)dalloc(e, kMaxK * sizeof(int));
    e->st = (DevState*)dalloc(e, sizeof(DevState));
    for (int i = 0; i < pairs; ++i) {
      DLC_CUDA(cudaMemsetAsync(e->p[i], 0, vb, e->stream));
      DLC_CUDA(cudaMemsetAsync(e->m[i], 0, vb, e->stream));  // AdamWState::init zeros, optim.cpp:17-27
      DLC_CUDA(cudaMemsetAsync(e->v[i], 0, vb, e->stream));
    }
    for (int i = 0; i < 2; ++i) {
      DLC_CUDA(cudaMemsetAsync(e->theta_t[i], 0, vb, e->stream));
      DLC_CUDA(cudaMemsetAsync(e->buf[i], 0, vb, e->stream));  // NesterovState::init, optim.cpp:29-35
    }
    DLC_CUDA(cudaMemsetAsync(e->flags, 0, kMaxK * sizeof(int), e->stream));
    DevState s{};
    s.scale = hyper->scaler_init_scale;
    s.growth = hyper->scaler_growth_interval;
    DLC_CUDA(cudaMemcpyAsync(e->st, &s, sizeof(s), cudaMemcpyHostToDevice, e->stream));
    ensure_tables(e, std::min<uint64_t>(cfg->total_inner_steps + 2, 1u << 16));
    DLC_CUDA(cudaStreamSynchronize(e->stream));
    *out = e;
  });
  if (st != DLC_OK && e) dlc_engine_destroy(e);
  return st;
}

int dlc_engine_destroy(dlc_engine* e) {
  if (!e) return DLC_OK;
  return guard([&] {
    DeviceGuard dg(e->device);
    if (e->stream) cudaStreamSynchronize(e->stream);
    if (e->cstream) cudaStreamSynchronize(e->cstream);
    if (e->p2p_bound && e->p2p_bound->comm && !e->p2p_bound->broken) {
      // peers may still be reading this engine's slot / send buffer: wait for
      // the whole fleet (engines are destroyed collectively; a collective
      // destroyed first unbinds its engines, which then skip this barrier)
      fleet_barrier(e, const_cast<dlc_collective*>(e->p2p_bound));
      cudaStreamSynchronize(e->stream);
    }
    p2p_unbind(e);
    unwatch(e);
    if (e->watch_ev) cudaEventDestroy(e->watch_ev);
    for (void* p : e->allocs) cudaFree(p);
    if (e->wire_rows) cudaFree(e->wire_rows);
    for (const auto& mk : e->pending) {
      cudaEventDestroy(mk.a);
      cudaEventDestroy(mk.b);
    }
    for (cudaEvent_t ev : e->pool) cudaEventDestroy(ev);
    if (e->tab) cudaFree(e->tab);
    if (e->ring_host) cudaFreeHost(e->ring_host);
    for (int i = 0; i < dlc_engine::kRing; ++i) {
      if (e->ring_a[i]) cudaEventDestroy(e->ring_a[i]);
      if (e->ring_b[i]) cudaEventDestroy(e->ring_b[i]);
    }
    if (e->ev0) cudaEventDestroy(e->ev0);
    if (e->ev1) cudaEventDestroy(e->ev1);
    for (cudaEvent_t ev : e->chunk_ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : e->piece_ev) cudaEventDestroy(ev);
    if (e->cstream) cudaStreamDestroy(e->cstream);
    if (e->h2d) cudaStreamDestroy(e->h2d);
    if (e->d2h) cudaStreamDestroy(e->d2h);
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
  });
}

size_t dlc_engine_size(const dlc_engine* e) { return e ? e->n : 0; }

int dlc_engine_stream(dlc_engine* e, void** stream) {
  return guard([&] {
    if (!e || !stream) fail(DLC_EINVAL, "dlc_engine_stream: null argument");
    *stream = (void*)e->stream;
  });
}

int dlc_engine_upload(dlc_engine* e, int which, const float* host, size_t n) {
  return guard([&] {
    if (!e || (n && !host)) fail(DLC_EINVAL, "dlc_engine_upload: null argument");
    if (n != e->n) fail(DLC_ESHAPE, "upload length " + std::to_string(n) + " != engine size " + std::to_string(e->n));
    DeviceGuard dg(e->device);
    float* d = writable(e, which);
    DLC_CUDA(cudaMemcpyAsync(d, host, n * sizeof(float), cudaMemcpyHostToDevice, e->stream));
    stream_wait(e);
  });
}

int dlc_engine_download(dlc_engine* e, int which, float* host, size_t n) {
  return guard([&] {
    if (!e || (n && !host)) fail(DLC_EINVAL, "dlc_engine_download: null argument");
    if (n != e->n) fail(DLC_ESHAPE, "download length " + std::to_string(n) + " != engine size " + std::to_string(e->n));
    DeviceGuard dg(e->device);
    float* d = live(e, which);
    DLC_CUDA(cudaMemcpyAsync(host, d, n * sizeof(float), cudaMemcpyDeviceToHost, e->stream));
    stream_wait(e);
  });
}

int dlc_engine_download_range(dlc_engine* e, int which, size_t offset, float* host, size_t count) {
  return guard([&] {
    if (!e || (count && !host)) fail(DLC_EINVAL, "dlc_engine_download_range: null argument");
    if (offset > e->n || count > e->n - offset)
      fail(DLC_ESHAPE, "download range [" + std::to_string(offset) + ", +" + std::to_string(count) + ") outside " +
                           std::to_string(e->n) + " elements");
    DeviceGuard dg(e->device);
    const float* d = live(e, which);
    DLC_CUDA(cudaMemcpyAsync(host, d + offset, count * sizeof(float), cudaMemcpyDeviceToHost, e->stream));
    stream_wait(e);
  });
}

int dlc_engine_upload_range(dlc_engine* e, int which, size_t offset, const float* host, size_t count) {
  return guard([&] {
    if (!e || (count && !host)) fail(DLC_EINVAL, "dlc_engine_upload_range: null argument");
    if (offset > e->n || count > e->n - offset)
      fail(DLC_ESHAPE, "upload range [" + std::to_string(offset) + ", +" + std::to_string(count) + ") outside " +
                           std::to_string(e->n) + " elements");
    DeviceGuard dg(e->device);
    float* d = writable(e, which);
    DLC_CUDA(cudaMemcpyAsync(d + offset, host, count * sizeof(float), cudaMemcpyHostToDevice, e->stream));
    stream_wait(e);
  });
}

int dlc_engine_device_ptr(dlc_engine* e, int which, float** dev) {
  return guard([&] {
    if (!e || !dev) fail(DLC_EINVAL, "dlc_engine_device_ptr: null argument");
    DeviceGuard dg(e->device);
    *dev = writable(e, which);  // the caller may write through it
  });
}

int dlc_engine_get_scalars(dlc_engine* e, dlc_engine_scalars* out) {
  return guard([&] {
    if (!e || !out) fail(DLC_EINVAL, "dlc_engine_get_scalars: null argument");
    DeviceGuard dg(e->device);
    const DevState s = read_state(e);
    out->step_count = s.step_count;
    out->inner_step = s.inner_step;
    out->outer_epoch = s.outer_epoch;
    out->scale = s.scale;
    out->consecutive_good = s.good;
    out->overflow_skips = s.overflow_skips;
    out->outer_skips = s.outer_skips;
    out->last_lr = s.last_lr;
    out->last_overflow = s.last_overflow;
    out->last_applied = s.last_applied;
  });
}

int dlc_engine_set_scalars(dlc_engine* e, const dlc_engine_scalars* in) {
  return guard([&] {
    if (!e || !in) fail(DLC_EINVAL, "dlc_engine_set_scalars: null argument");
    if (in->inner_step > e->cfg.total_inner_steps) fail(DLC_ECONFIG, "inner_step beyond total_inner_steps");
    DeviceGuard dg(e->device);
    DevState s = read_state(e);
    s.step_count = in->step_count;
    s.inner_step = in->inner_step;
    s.outer_epoch = in->outer_epoch;
    s.scale = in->scale;
    s.good = in->consecutive_good;
    s.overflow_skips = in->overflow_skips;
    s.outer_skips = in->outer_skips;
    s.last_lr = in->last_lr;
    s.last_overflow = in->last_overflow;
    s.last_applied = in->last_applied;
    e->delta_fused = false;
    ensure_tables(e, in->step_count + 2);
    DLC_CUDA(cudaMemcpy(e->st, &s, sizeof(s), cudaMemcpyHostToDevice));
    e->issued_inner = in->inner_step;
  });
}

int dlc_engine_synchronize(dlc_engine* e) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_engine_synchronize: null engine");
    DeviceGuard dg(e->device);
    stream_wait(e);
    check_barrier(e);
  });
}

int dlc_engine_inner_step(dlc_engine* e, const float* grad, int grad_is_scaled, dlc_inner_result* result) {
  return guard([&] {
    if (!e || (e->n && !grad)) fail(DLC_EINVAL, "dlc_engine_inner_step: null argument");
    DeviceGuard dg(e->device);
    engine_inner(e, grad, grad_is_scaled);
    if (result) {
      const DevState s = read_state(e);
      result->lr = s.last_lr;
      result->overflow_skipped = s.last_overflow;
    }
  });
}

int dlc_engine_inner_step_host(dlc_engine* e, const float* host_grad, int grad_is_scaled,
                               dlc_inner_result* result) {
  return guard([&] {
    if (!e || (e->n && !host_grad)) fail(DLC_EINVAL, "dlc_engine_inner_step_host: null argument");
    DeviceGuard dg(e->device);
    DLC_CUDA(cudaMemcpyAsync(e->grad, host_grad, e->n * sizeof(float), cudaMemcpyHostToDevice, e->stream));
    engine_inner(e, e->grad, grad_is_scaled);
    if (result) {
      const DevState s = read_state(e);
      result->lr = s.last_lr;
      result->overflow_skipped = s.last_overflow;
    }
  });
}

int dlc_engine_outer_step(dlc_engine* e, dlc_collective* c, dlc_outer_result* result, dlc_reduce_report* report) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_engine_outer_step: null engine");
    if (c && c->kind == 0) c = nullptr;
    check_collective(e, c);
    DeviceGuard dg(e->device);
    const uint64_t epoch = report ? read_state(e).outer_epoch : 0;
    outer_round(e, c, nullptr, report);
    fill_report(e, c, report, epoch);
    outer_result(e, result);
  });
}

int dlc_engine_outer_step_from(dlc_engine* e, dlc_collective* c, const float* theta_local_dev,
                               dlc_outer_result* result, dlc_reduce_report* report) {
  return guard([&] {
    if (!e || (e->n && !theta_local_dev)) fail(DLC_EINVAL, "dlc_engine_outer_step_from: null argument");
    if (c && c->kind == 0) c = nullptr;
    check_collective(e, c);
    DeviceGuard dg(e->device);
    const uint64_t epoch = report ? read_state(e).outer_epoch : 0;
    float* src = const_cast<float*>(theta_local_dev);
    outer_round(e, c, src, report);
    fill_report(e, c, report, epoch);
    outer_result(e, result);
  });
}

int dlc_engine_set_fused_delta(dlc_engine* e, int on) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_engine_set_fused_delta: null engine");
    e->fuse_delta = on != 0;
    if (!e->fuse_delta) e->delta_fused = false;
  });
}

int dlc_engine_set_timing(dlc_engine* e, int on) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_engine_set_timing: null engine");
    DeviceGuard dg(e->device);
    harvest(e);
    e->timing = on != 0;
  });
}

int dlc_engine_phase_times(dlc_engine* e, double total_ms[4], uint64_t count[4]) {
  return guard([&] {
    if (!e || !total_ms || !count) fail(DLC_EINVAL, "dlc_engine_phase_times: null argument");
    DeviceGuard dg(e->device);
    harvest(e);
    for (int i = 0; i < 4; ++i) {
      total_ms[i] = e->phase_ms[i];
      count[i] = e->phase_n[i];
      e->phase_ms[i] = 0.0;
      e->phase_n[i] = 0;
    }
  });
}

int dlc_engine_outer_step_host(dlc_engine* e, dlc_collective* c, const float* host_theta_local, float* host_theta_t,
                               dlc_outer_result* result) {
  return guard([&] {
    if (!e || (e->n && (!host_theta_local || !host_theta_t))) fail(DLC_EINVAL, "dlc_engine_outer_step_host: null argument");
    if (c && c->kind == 0) c = nullptr;
    check_collective(e, c);
    DeviceGuard dg(e->device);
    e->delta_fused = false;  // theta_local comes from the host: the full K2 runs
    // theta_local arrives chunk by chunk in the staging buffer (copy stream);
    // each chunk's kernel starts as soon as its bytes land, and for a single
    // worker each finished chunk of the new theta_t streams back on a second
    // copy stream, so H2D, compute and D2H overlap.  K4 refreshes the engine's
    // own theta_local from the new theta_t.
    ensure_copy_streams(e);
    const DevState s0 = read_state(e);
    if (e->k > 1 && c->mode == DLC_MODE_P2P) {  // piece-pipelined H2D / step / D2H
      outer_p2p_pipelined(e, c, e->grad, nullptr, host_theta_local, host_theta_t, s0.ocur);
      DLC_CUDA(cudaStreamSynchronize(e->h2d));
      DLC_CUDA(cudaStreamSynchronize(e->d2h));
      const DevState s1 = read_state(e);
      if (!s1.last_applied)  // skipped: theta_t did not move
        DLC_CUDA(cudaMemcpy(host_theta_t, e->theta_t[s1.ocur], e->n * sizeof(float), cudaMemcpyDeviceToHost));
      outer_result(e, result);
      return;
    }
    const size_t n = e->n, C = kHostChunk, nch = (n + C - 1) / C;
    ensure_chunk_events(e, 2 * nch + 1);
    reset_flags(e);
    DLC_CUDA(cudaEventRecord(e->chunk_ev[2 * nch], e->stream));  // staging buffer free to overwrite
    DLC_CUDA(cudaStreamWaitEvent(e->h2d, e->chunk_ev[2 * nch], 0));
    float* staged = e->grad;
    for (size_t ci = 0; ci < nch; ++ci) {
      const size_t off = ci * C, len = std::min(C, n - off);
      DLC_CUDA(cudaMemcpyAsync(staged + off, host_theta_local + off, len * sizeof(float), cudaMemcpyHostToDevice,
                               e->h2d));
      DLC_CUDA(cudaEventRecord(e->chunk_ev[2 * ci], e->h2d));
      DLC_CUDA(cudaStreamWaitEvent(e->stream, e->chunk_ev[2 * ci], 0));
      if (e->k == 1) {
        launch_outer_solo_chunk(tt_pair(e), buf_pair(e), local_pair(e), staged, e->prec, e->st, e->hyper.outer_lr,
                                e->hyper.outer_momentum, off, len, e->stream);
        launched("outer_solo_chunk");
        DLC_CUDA(cudaEventRecord(e->chunk_ev[2 * ci + 1], e->stream));
        DLC_CUDA(cudaStreamWaitEvent(e->d2h, e->chunk_ev[2 * ci + 1], 0));
        // speculative: the idle theta_t buffer holds the new weights if the step applies
        DLC_CUDA(cudaMemcpyAsync(host_theta_t + off, e->theta_t[s0.ocur ^ 1] + off, len * sizeof(float),
                                 cudaMemcpyDeviceToHost, e->d2h));
      } else {
        launch_pseudo_grad(tt_pair(e), Pair{{staged, staged}}, e->st, e->send, e->prec, &e->st->delta_nonfinite,
                           off, len, e->stream);
        launched("pseudo_grad_chunk");
      }
    }
    if (e->k == 1) {
      launch_outer_solo_finish(tt_pair(e), local_pair(e), e->st, n, e->stream);
      launched("outer_solo_finish");
    } else {
      outer_collective(e, c, nullptr);  // ORDERED / ALLREDUCE: K4 speculative into theta_t[ocur ^ 1]
      DLC_CUDA(cudaMemcpyAsync(host_theta_t, e->theta_t[s0.ocur ^ 1], n * sizeof(float), cudaMemcpyDeviceToHost,
                               e->stream));
    }
    DLC_CUDA(cudaStreamSynchronize(e->h2d));
    DLC_CUDA(cudaStreamSynchronize(e->d2h));
    const DevState s1 = read_state(e);
    if (!s1.last_applied)  // skipped: theta_t did not move
      DLC_CUDA(cudaMemcpy(host_theta_t, e->theta_t[s1.ocur], n * sizeof(float), cudaMemcpyDeviceToHost));
    outer_result(e, result);
  });
}

int dlc_engine_compute_pseudo_gradient(dlc_engine* e, float* host_delta, uint64_t* outer_epoch) {
  return guard([&] {
    if (!e || (e->n && !host_delta)) fail(DLC_EINVAL, "dlc_engine_compute_pseudo_gradient: null argument");
    if (e->issued_inner % e->cfg.local_steps_h != 0)  // engine.cpp:116-120
      fail(DLC_EINVAL, "pseudo-gradient requested mid-window (inner_step " + std::to_string(e->issued_inner) +
                           ", H " + std::to_string(e->cfg.local_steps_h) + ")");
    DeviceGuard dg(e->device);
    // raw FP32 delta (axpy(-1, theta_local, theta_t), engine.cpp:122) into the staging buffer
    launch_pseudo_grad(tt_pair(e), local_pair(e), e->st, e->grad, DLC_FP32, &e->st->delta_nonfinite, 0, e->n,
                       e->stream);
    launched("pseudo_grad");
    DLC_CUDA(cudaMemcpyAsync(host_delta, e->grad, e->n * sizeof(float), cudaMemcpyDeviceToHost, e->stream));
    const DevState s = read_state(e);
    if (outer_epoch) *outer_epoch = s.outer_epoch;
  });
}

int dlc_engine_apply_outer_step(dlc_engine* e, const float* host_mean, uint64_t outer_epoch,
                                dlc_outer_result* result) {
  return guard([&] {
    if (!e || (e->n && !host_mean)) fail(DLC_EINVAL, "dlc_engine_apply_outer_step: null argument");
    DeviceGuard dg(e->device);
    const DevState s = read_state(e);
    if (outer_epoch != s.outer_epoch)  // engine.cpp:129-134
      fail(DLC_ECOLLECTIVE, "outer_step: reduced pseudo-gradient from epoch " + std::to_string(outer_epoch) +
                                " applied at epoch " + std::to_string(s.outer_epoch));
    e->delta_fused = false;
    DLC_CUDA(cudaMemcpyAsync(e->grad, host_mean, e->n * sizeof(float), cudaMemcpyHostToDevice, e->stream));
    DLC_CUDA(cudaMemsetAsync(e->flags, 0, sizeof(int), e->stream));
    launch_nonfinite(e->grad, e->flags, e->n, e->stream);  // engine.cpp:136
    launch_nesterov_outer(tt_pair(e), buf_pair(e), local_pair(e), e->grad, DLC_FP32, e->flags, 1, e->st,
                          e->hyper.outer_lr, e->hyper.outer_momentum, e->n, e->stream);
    launched("apply_outer_step");
    outer_result(e, result);
  });
}

int dlc_engines_outer_step_local(dlc_engine* const* engines, size_t k, dlc_outer_result* result) {
  return guard([&] {
    if (!engines || k == 0) fail(DLC_ECOLLECTIVE, "outer_step_local: no engines");
    if (k > (size_t)kMaxK) fail(DLC_ECONFIG, "outer_step_local: more than 32 engines");
    dlc_engine* e0 = engines[0];
    for (size_t j = 0; j < k; ++j) {
      dlc_engine* e = engines[j];
      if (!e) fail(DLC_EINVAL, "outer_step_local: null engine");
      if (e->n != e0->n || e->prec != e0->prec || e->device != e0->device)
        fail(DLC_ESHAPE, "outer_step_local: engines differ in size, precision or device");  // reduce.cpp:52-56
      if (e->k != k) fail(DLC_ECOLLECTIVE, "outer_step_local: num_workers_k != fleet size");
      if (e->issued_inner % e->cfg.local_steps_h != 0) fail(DLC_EINVAL, "pseudo-gradient requested mid-window");
    }
    DeviceGuard dg(e0->device);
    cudaEvent_t ev;
    DLC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    for (size_t j = 1; j < k; ++j) {  // everything below runs on engine 0's stream
      DLC_CUDA(cudaEventRecord(ev, engines[j]->stream));
      DLC_CUDA(cudaStreamWaitEvent(e0->stream, ev, 0));
    }
    cudaStream_t s = e0->stream;
    for (size_t j = 0; j < k; ++j)
      DLC_CUDA(cudaMemsetAsync(&engines[j]->st->delta_nonfinite, 0, sizeof(int), s));
    PtrList in{};
    for (size_t j = 0; j < k; ++j) {
      dlc_engine* e = engines[j];
      if (take_fused_delta(e) && k > 1)  // the window's last K1 wrote the delta (k = 1 needs the flag below)
        launch_pseudo_grad_gated(tt_pair(e), local_pair(e), e->st, e->send, e->prec, e->n, s);
      else
        launch_pseudo_grad(tt_pair(e), local_pair(e), e->st, e->send, e->prec, &e->st->delta_nonfinite, 0, e->n,
                           s);
      in.ptr[j] = e->send;
    }
    DLC_CUDA(cudaMemsetAsync(e0->flags, 0, kMaxK * sizeof(int), s));
    void* dbar = k > 1 ? e0->gather : e0->send;
    if (k > 1) {
      launch_fold(in, (int)k, e0->prec, e0->gather, e0->prec, e0->flags, e0->n, s);
    } else {
      DLC_CUDA(cudaMemcpyAsync(e0->flags, &e0->st->delta_nonfinite, sizeof(int), cudaMemcpyDeviceToDevice, s));
    }
    for (size_t j = 0; j < k; ++j) {
      dlc_engine* e = engines[j];
      launch_nesterov_outer(tt_pair(e), buf_pair(e), local_pair(e), dbar, e->prec, e0->flags, 1, e->st,
                            e->hyper.outer_lr, e->hyper.outer_momentum, e->n, s);
    }
    launched("outer_step_local");
    DLC_CUDA(cudaEventRecord(ev, s));
    for (size_t j = 1; j < k; ++j) DLC_CUDA(cudaStreamWaitEvent(engines[j]->stream, ev, 0));
    DLC_CUDA(cudaEventDestroy(ev));
    outer_result(e0, result);
  });
}

int dlc_optimizer_step(dlc_engine* e, dlc_collective* c, const float* grad, int grad_is_scaled, int* round_completed) {
  return guard([&] {
    if (!e || (e->n && !grad)) fail(DLC_EINVAL, "dlc_optimizer_step: null argument");
    if (c && c->kind == 0) c = nullptr;
    DeviceGuard dg(e->device);
    if (boundary_solo_ok(e, c)) {  // K = 1: the window's last inner step and the outer step in one pass
      engine_boundary_solo(e, grad, grad_is_scaled);
      if (round_completed) *round_completed = 1;
      return;
    }
    engine_inner(e, grad, grad_is_scaled);  // engine.cpp:163
    const bool boundary = e->issued_inner % e->cfg.local_steps_h == 0;
    if (round_completed) *round_completed = boundary ? 1 : 0;
    if (boundary) {  // engine.cpp:165-172
      check_collective(e, c);
      outer_round(e, c, nullptr, nullptr);
    }
  });
}

int dlc_rng_fill_device(dlc_engine* e, int which, uint64_t key, uint64_t first, float lo, float hi) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_rng_fill_device: null engine");
    DeviceGuard dg(e->device);
    float* d = writable(e, which);
    launch_rng_fill(key, first, lo, hi, d, e->n, e->stream);
    launched("rng_fill");
  });
}

int dlc_rng_perturb(dlc_engine* e, float* dst, uint64_t key, float lo, float hi) {
  return guard([&] {
    if (!e) fail(DLC_EINVAL, "dlc_rng_perturb: null engine");
    DeviceGuard dg(e->device);
    float* d = dst ? dst : writable(e, DLC_THETA_LOCAL);
    launch_rng_perturb(live(e, DLC_THETA_T), key, lo, hi, d, e->n, e->stream);
    launched("rng_perturb");
  });
}
}  // extern "C"
