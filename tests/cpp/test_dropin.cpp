// test_dropin.cpp — the C++ drop-in layer (include/diloco_cuda.hpp) against the
// reference implementation, with the reference's own types (TEST INFRASTRUCTURE).
//
// Built by oracle/Makefile (target `dropin`) from the reference's hot-path
// sources under /root/reference/proj/src plus libdiloco_cuda.so, into
// oracle/_ref/test_dropin; run on the GPU box by tests/test_dropin_gpu.py.
// Every check compares diloco::X (reference CPU) with diloco::cuda::X (B200)
// using the reference's bitwise ParamVector equality (tensor.cpp:106-116).
#include <cmath>
#include <cstring>
#include <span>
#include <cstdio>
#include <string>
#include <vector>

#include "diloco/rng.hpp"
#include "diloco/wire.hpp"
#include "diloco_cuda.hpp"

using namespace diloco;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (cond) {                                                       \
      ++g_pass;                                                       \
    } else {                                                          \
      ++g_fail;                                                       \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
    }                                                                 \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static void throw_status_ok(int st) {
  if (st != DLC_OK) throw Error(dlc_last_error());
}

static ParamVector random_vec(LayoutPtr layout, uint64_t seed, const char* purpose, float lo, float hi) {
  CounterRng rng(seed, purpose, 0);
  std::vector<float> d(layout->total_length());
  for (float& f : d) f = rng.next_uniform(lo, hi);
  return ParamVector(std::move(layout), std::move(d));
}

int main() {
  if (dlc_set_device(0) != DLC_OK) {
    std::printf("no device: %s\n", dlc_last_error());
    return 2;
  }
  // Multi-segment layout: the drop-in must preserve the caller's layout.
  auto layout = Layout::make({{"w", 0, 70001}, {"b", 70001, 33}});
  const size_t n = layout->total_length();

  // adamw_step over 6 steps, state evolving on both sides (optim.cpp:58-93)
  {
    AdamWState ref = AdamWState::init(layout, 0.9f, 0.95f, 1e-8f, 0.1f);
    AdamWState gpu = AdamWState::init(layout, 0.9f, 0.95f, 1e-8f, 0.1f);
    ParamVector p_ref = random_vec(layout, 1, "p", -2, 2), p_gpu = p_ref;
    for (int t = 0; t < 6; ++t) {
      const ParamVector g = random_vec(layout, 10 + t, "g", -1, 1);
      p_ref = adamw_step(ref, p_ref, g, 1e-3f * (t + 1));
      p_gpu = cuda::adamw_step(gpu, p_gpu, g, 1e-3f * (t + 1));
      CHECK(p_ref == p_gpu);
      CHECK(ref.m == gpu.m && ref.v == gpu.v && ref.step_count == gpu.step_count);
    }
    std::vector<float> bad(n, 0.0f);
    bad[n - 1] = INFINITY;
    const uint64_t before = gpu.step_count;
    CHECK(throws<NumericError>([&] { cuda::adamw_step(gpu, p_gpu, ParamVector(layout, bad), 1e-3f); }));
    CHECK(gpu.step_count == before);
    CHECK(throws<ConfigError>([&] { cuda::adamw_step(gpu, p_gpu, p_gpu, -1.0f); }));
    CHECK(throws<ShapeError>([&] { cuda::adamw_step(gpu, p_gpu, random_vec(Layout::single("x", n), 1, "g", 0, 1), 1e-3f); }));
  }
  // nesterov_step (optim.cpp:95-115)
  {
    NesterovState ref = NesterovState::init(layout, 0.7f, 0.9f), gpu = NesterovState::init(layout, 0.7f, 0.9f);
    ParamVector th_ref = random_vec(layout, 2, "th", -5, 5), th_gpu = th_ref;
    for (int t = 0; t < 4; ++t) {
      const ParamVector g = random_vec(layout, 20 + t, "d", -1, 1);
      th_ref = nesterov_step(ref, th_ref, g);
      th_gpu = cuda::nesterov_step(gpu, th_gpu, g);
      CHECK(th_ref == th_gpu && ref.momentum_buf == gpu.momentum_buf);
    }
  }
  // scaler, axpy, codec (optim.cpp:121-135; tensor.cpp:118-154)
  {
    LossScaler s;
    s.scale = 0x1p-3f;
    ParamVector g = random_vec(layout, 3, "g", -1e30f, 1e30f);
    const UnscaleResult a = scaler_unscale_and_check(s, g), b = cuda::scaler_unscale_and_check(s, g);
    CHECK(a.overflow == b.overflow && a.grad == b.grad);
    const ParamVector x = random_vec(layout, 4, "x", -1, 1), y = random_vec(layout, 5, "y", -1, 1);
    CHECK(axpy(-1.0f, x, y) == cuda::axpy(-1.0f, x, y));
    const ParamVector wide = random_vec(layout, 6, "wide", -7e4f, 7e4f);
    const Fp16Buffer e1 = encode_fp16(wide), e2 = cuda::encode_fp16(wide);
    CHECK(e1.bits == e2.bits && e1.overflow == e2.overflow && e1.overflow);
    CHECK(decode_fp16(e1, layout) == cuda::decode_fp16(e2, layout));
  }
  // reduce_average, K = 1..9, both precisions (reduce.cpp:46-89)
  for (size_t k = 1; k <= 9; ++k) {
    std::vector<ParamVector> cs;
    for (size_t j = 0; j < k; ++j) cs.push_back(random_vec(layout, 100 + j, "c", -1e-2f, 1e-2f));
    std::vector<const ParamVector*> ptrs;
    for (const auto& c : cs) ptrs.push_back(&c);
    for (Precision p : {Precision::fp32, Precision::fp16}) {
      CHECK(reduce_average(ptrs, p) == cuda::reduce_average(ptrs, p));
    }
  }
  CHECK(throws<CollectiveError>([&] { cuda::reduce_average({}, Precision::fp32); }));
  // NcclCollective with a world of one == SoloCollective (reduce.cpp:113-126)
  {
    cuda::NcclCollective nccl(0, 1, cuda::NcclCollective::make_unique_id(), 0);
    SoloCollective solo;
    CHECK(nccl.world_size() == 1);
    for (Precision p : {Precision::fp32, Precision::fp16}) {
      PseudoGradient pg;
      pg.delta = random_vec(layout, 7, "delta", -1, 1);
      pg.precision = p;
      pg.outer_epoch = 5;
      ReduceReport r1, r2;
      const PseudoGradient a = solo.all_reduce_avg(pg, &r1), b = nccl.all_reduce_avg(pg, &r2);
      CHECK(a.delta == b.delta && b.outer_epoch == 5 && r2.contributors == 1);
    }
  }
  // DeviceEngine: H=4 window + outer step vs the reference's functions sequenced as
  // apply_inner_step + compute_pseudo_gradient + SoloCollective + outer_step (engine.cpp:50-146)
  for (Precision prec : {Precision::fp32, Precision::fp16}) {
    const ParamVector theta0 = random_vec(layout, 8, "theta", -0.05f, 0.05f);
    dlc_config cfg{4, 1, cuda::to_c(prec), 8};
    dlc_hyperparams hp;
    dlc_hyperparams_default(&hp);
    hp.warmup_steps = 3;
    cuda::DeviceEngine eng(cfg, hp, theta0, 0);
    ParamVector theta_t = theta0, theta_local = theta0;
    AdamWState adam = AdamWState::init(layout, hp.beta1, hp.beta2, hp.adam_eps, hp.weight_decay);
    NesterovState outer = NesterovState::init(layout, hp.outer_lr, hp.outer_momentum);
    LossScaler scaler;
    LrSchedule sched;
    sched.warmup_steps = hp.warmup_steps;
    sched.total_steps = cfg.total_inner_steps;
    sched.base_lr = hp.inner_lr;
    SoloCollective solo;
    for (int round = 0; round < 2; ++round) {
      for (int t = 0; t < 4; ++t) {
        ParamVector g = random_vec(layout, 1000 + round * 10 + t, "grad", -1e-2f, 1e-2f);
        if (round == 1 && t == 2) {
          std::vector<float> d(g.values().begin(), g.values().end());
          d[17] = NAN;
          g = ParamVector(layout, d);
        }
        std::vector<float> scaled(n);
        for (size_t i = 0; i < n; ++i) scaled[i] = g.values()[i] * scaler.scale;  // engine.cpp:20-27
        const UnscaleResult un = scaler_unscale_and_check(scaler, ParamVector(layout, scaled));
        if (!un.overflow) theta_local = adamw_step(adam, theta_local, un.grad, lr_at(sched, adam.step_count + 1));
        scaler_update(scaler, un.overflow);
        const dlc_inner_result r = eng.inner_step(g);
        CHECK((r.overflow_skipped != 0) == un.overflow);
      }
      PseudoGradient pg;
      pg.delta = axpy(-1.0f, theta_local, theta_t);
      pg.precision = prec;
      const PseudoGradient red = solo.all_reduce_avg(pg, nullptr);
      if (red.delta.all_finite()) theta_t = nesterov_step(outer, theta_t, red.delta);
      theta_local = theta_t;
      const dlc_outer_result o = eng.outer_step();
      CHECK(o.applied == 1 && o.outer_epoch == (uint64_t)round + 1);
    }
    CHECK(eng.download(DLC_THETA_T) == theta_t);
    CHECK(eng.download(DLC_THETA_LOCAL) == theta_local);
    CHECK(eng.download(DLC_ADAM_M) == adam.m && eng.download(DLC_ADAM_V) == adam.v);
    CHECK(eng.download(DLC_MOMENTUM) == outer.momentum_buf);
    const dlc_engine_scalars s = eng.scalars();
    CHECK(s.step_count == adam.step_count && s.scale == scaler.scale && s.overflow_skips == 1);
  }
  // DeviceOptimizer (DilocoOptimizer::step, engine.cpp:162-174): one worker's
  // window boundary as one fused pass, against the same reference sequence,
  // with overflows on a window's last step (the gated rerun) and mid-window
  for (Precision prec : {Precision::fp32, Precision::fp16}) {
    const ParamVector theta0 = random_vec(layout, 9, "theta", -0.05f, 0.05f);
    dlc_config cfg{3, 1, cuda::to_c(prec), 9};
    dlc_hyperparams hp;
    dlc_hyperparams_default(&hp);
    hp.warmup_steps = 2;
    cuda::DeviceEngine eng(cfg, hp, theta0, 0);
    cuda::DeviceOptimizer opt(eng);
    ParamVector theta_t = theta0, theta_local = theta0;
    AdamWState adam = AdamWState::init(layout, hp.beta1, hp.beta2, hp.adam_eps, hp.weight_decay);
    NesterovState outer = NesterovState::init(layout, hp.outer_lr, hp.outer_momentum);
    LossScaler scaler;
    LrSchedule sched;
    sched.warmup_steps = hp.warmup_steps;
    sched.total_steps = cfg.total_inner_steps;
    sched.base_lr = hp.inner_lr;
    SoloCollective solo;
    for (int round = 0; round < 3; ++round) {
      for (int t = 0; t < 3; ++t) {
        ParamVector g = random_vec(layout, 2000 + round * 10 + t, "grad", -1e-2f, 1e-2f);
        if ((round == 0 && t == 2) || (round == 1 && t == 0)) {
          std::vector<float> d(g.values().begin(), g.values().end());
          d[5] = INFINITY;
          g = ParamVector(layout, d);
        }
        std::vector<float> scaled(n);
        for (size_t i = 0; i < n; ++i) scaled[i] = g.values()[i] * scaler.scale;  // engine.cpp:20-27
        const UnscaleResult un = scaler_unscale_and_check(scaler, ParamVector(layout, scaled));
        if (!un.overflow) theta_local = adamw_step(adam, theta_local, un.grad, lr_at(sched, adam.step_count + 1));
        scaler_update(scaler, un.overflow);
        const dlc_inner_result r = opt.step(g);
        CHECK((r.overflow_skipped != 0) == un.overflow);
        CHECK(opt.round_just_completed() == (t == 2));
      }
      PseudoGradient pg;
      pg.delta = axpy(-1.0f, theta_local, theta_t);
      pg.precision = prec;
      const PseudoGradient red = solo.all_reduce_avg(pg, nullptr);
      const bool applied = red.delta.all_finite();
      if (applied) theta_t = nesterov_step(outer, theta_t, red.delta);
      theta_local = theta_t;
      CHECK(opt.last_round_applied() == applied);
      CHECK(eng.download(DLC_THETA_T) == theta_t && eng.download(DLC_THETA_LOCAL) == theta_local);
    }
    CHECK(eng.download(DLC_ADAM_M) == adam.m && eng.download(DLC_ADAM_V) == adam.v);
    CHECK(eng.download(DLC_MOMENTUM) == outer.momentum_buf);
    const dlc_engine_scalars s = eng.scalars();
    CHECK(s.step_count == adam.step_count && s.scale == scaler.scale && s.overflow_skips == 2 && s.outer_epoch == 3);
  }
  // DeviceEngine's outer round through the reference's own Collective class
  // (SoloCollective here; SocketCollective plugs in the same way across boxes),
  // with an epoch-guard violation and a non-finite skip.
  for (Precision prec : {Precision::fp32, Precision::fp16}) {
    const ParamVector theta0 = random_vec(layout, 31, "theta", -0.05f, 0.05f);
    dlc_config cfg{2, 1, cuda::to_c(prec), 6};
    dlc_hyperparams hp;
    dlc_hyperparams_default(&hp);
    cuda::DeviceEngine eng(cfg, hp, theta0, 0);
    ParamVector theta_t = theta0, theta_local = theta0;
    AdamWState adam = AdamWState::init(layout, hp.beta1, hp.beta2, hp.adam_eps, hp.weight_decay);
    NesterovState outer = NesterovState::init(layout, hp.outer_lr, hp.outer_momentum);
    LossScaler scaler;
    LrSchedule sched;
    sched.warmup_steps = hp.warmup_steps;
    sched.total_steps = cfg.total_inner_steps;
    sched.base_lr = hp.inner_lr;
    SoloCollective solo;
    for (int round = 0; round < 3; ++round) {
      for (int t = 0; t < 2; ++t) {
        const ParamVector g = random_vec(layout, 2000 + round * 10 + t, "grad", -1e-2f, 1e-2f);
        std::vector<float> scaled(n);
        for (size_t i = 0; i < n; ++i) scaled[i] = g.values()[i] * scaler.scale;
        const UnscaleResult un = scaler_unscale_and_check(scaler, ParamVector(layout, scaled));
        if (!un.overflow) theta_local = adamw_step(adam, theta_local, un.grad, lr_at(sched, adam.step_count + 1));
        scaler_update(scaler, un.overflow);
        eng.inner_step(g);
      }
      PseudoGradient pg;
      pg.delta = axpy(-1.0f, theta_local, theta_t);
      pg.precision = prec;
      PseudoGradient red = solo.all_reduce_avg(pg, nullptr);
      bool applied = red.delta.all_finite();
      if (applied) theta_t = nesterov_step(outer, theta_t, red.delta);
      theta_local = theta_t;
      CHECK(eng.outer_step(solo, prec) == applied);
    }
    CHECK(eng.download(DLC_THETA_T) == theta_t && eng.download(DLC_THETA_LOCAL) == theta_local);
    CHECK(eng.download(DLC_MOMENTUM) == outer.momentum_buf);
    // a reduction tagged with the wrong epoch is a CollectiveError (engine.cpp:129-134)
    std::vector<float> zeros(n, 0.0f);
    dlc_outer_result r{};
    CHECK(dlc_engine_apply_outer_step(eng.handle(), zeros.data(), 99, &r) == DLC_ECOLLECTIVE);
    // a non-finite mean skips Nesterov but re-snapshots theta_local (engine.cpp:136-144)
    std::vector<float> bad(n, 0.0f);
    bad[3] = NAN;
    CHECK(dlc_engine_apply_outer_step(eng.handle(), bad.data(), eng.scalars().outer_epoch, &r) == DLC_OK);
    CHECK(r.applied == 0 && eng.download(DLC_THETA_T) == theta_t && eng.download(DLC_THETA_LOCAL) == theta_t);
  }
  // ---- wire codec: frames from the device engine through the reference's own
  // FrameParser / decode_reduce_payload (wire.cpp); scalars = encode_fp16 of the
  // reference's axpy pseudo-gradient; then a 2-worker round whose only exchange
  // is those bytes, against reduce_average + nesterov_step.
  {
    const size_t n = 5003;
    auto layout = Layout::single("p", n);
    const ParamVector theta0 = random_vec(layout, 31, "theta", -1.0f, 1.0f);
    dlc_config cfg{1, 2, DLC_FP16, 4};
    dlc_hyperparams hp;
    dlc_hyperparams_default(&hp);
    cuda::DeviceEngine e0(cfg, hp, theta0, 0, DLC_INNER_PINGPONG), e1(cfg, hp, theta0, 0, DLC_INNER_PINGPONG);
    std::vector<ParamVector> locals;
    for (int j = 0; j < 2; ++j) {
      std::vector<float> l(theta0.values().begin(), theta0.values().end());
      const ParamVector noise = random_vec(layout, 40 + j, "local", -1e-2f, 1e-2f);
      for (size_t i = 0; i < n; ++i) l[i] -= noise.values()[i];
      locals.emplace_back(layout, std::move(l));
    }
    throw_status_ok(dlc_engine_upload(e0.handle(), DLC_THETA_LOCAL, locals[0].values().data(), n));
    throw_status_ok(dlc_engine_upload(e1.handle(), DLC_THETA_LOCAL, locals[1].values().data(), n));
    cuda::DeviceEngine* eng[2] = {&e0, &e1};
    const uint64_t epoch = e0.wire_begin();
    CHECK(e1.wire_begin() == epoch);
    const auto ranges = partition_ranges(n, 2);
    const dlc_wire_tags t{DLC_MSG_REDUCE_CHUNK, DLC_FP16, epoch, 0, 1, 0x11, 0x22, 4096};
    const std::vector<uint8_t> frames = e0.wire_encode(DLC_WIRE_DELTA, ranges[1].offset, ranges[1].length, t);
    FrameParser parser;
    parser.feed(frames);
    const Fp16Buffer want = encode_fp16(axpy(-1.0f, locals[0], theta0));
    size_t elems = 0, chunks = 0;
    while (auto m = parser.next()) {
      std::span<const uint8_t> seg;
      const ReduceChunkHeader h = decode_reduce_payload(m->payload, seg);
      CHECK(m->type == MsgType::reduce_chunk && h.outer_epoch == epoch && h.chunk_index == chunks && h.precision == 1);
      const size_t header = 32 + std::string("a0.p1.f00000000000000110000000000000022").size();
      const size_t count = (seg.size() - header) / 2;
      CHECK(std::memcmp(seg.data() + header, want.bits.data() + ranges[1].offset + elems, count * 2) == 0);
      elems += count;
      ++chunks;
    }
    CHECK(elems == ranges[1].length && chunks == (ranges[1].length + 2047) / 2048);
    // the round: scatter, fold, ring all-gather, outer step
    for (int r = 0; r < 2; ++r) {
      const int p = 1 - r;
      const dlc_wire_tags ts{DLC_MSG_REDUCE_CHUNK, DLC_FP16, epoch, 0, (uint32_t)p, 0x11, (uint64_t)r, 4096};
      const auto bytes = eng[r]->wire_encode(DLC_WIRE_DELTA, ranges[p].offset, ranges[p].length, ts);
      CHECK(eng[p]->wire_decode(DLC_WIRE_ROW, r, ranges[p].offset, ranges[p].length, bytes) == bytes.size());
    }
    for (int r = 0; r < 2; ++r) eng[r]->wire_fold(r, 2, ranges[r].offset, ranges[r].length);
    for (int r = 0; r < 2; ++r) {
      const dlc_wire_tags ts{DLC_MSG_REDUCE_RESULT, DLC_FP16, epoch, 0, (uint32_t)r, 0x11, (uint64_t)r, 4096};
      const auto bytes = eng[r]->wire_encode(DLC_WIRE_MEAN, ranges[r].offset, ranges[r].length, ts);
      CHECK(eng[1 - r]->wire_decode(DLC_WIRE_MEAN, 0, 0, n, bytes) == bytes.size());
    }
    const ParamVector d0 = axpy(-1.0f, locals[0], theta0), d1 = axpy(-1.0f, locals[1], theta0);
    std::vector<const ParamVector*> ptrs{&d0, &d1};
    const ParamVector dbar = reduce_average(ptrs, Precision::fp16);
    NesterovState outer = NesterovState::init(layout, hp.outer_lr, hp.outer_momentum);
    const ParamVector theta1 = nesterov_step(outer, theta0, dbar);
    for (int r = 0; r < 2; ++r) {
      const dlc_outer_result o = eng[r]->wire_finish(epoch);
      CHECK(o.applied == 1 && o.outer_epoch == epoch + 1);
      CHECK(eng[r]->download(DLC_THETA_T) == theta1 && eng[r]->download(DLC_THETA_LOCAL) == theta1);
      CHECK(eng[r]->download(DLC_MOMENTUM) == outer.momentum_buf);
    }
    std::vector<uint8_t> bad = frames;
    bad[0] = 'X';
    CHECK(throws<SerializationError>([&] { e1.wire_decode(DLC_WIRE_MEAN, 0, 0, n, bad); }));
  }
  // ---- run_training (engine.cpp:176-240) on a DeviceEngine: the record stream
  // and the final state of the same window sequence driven step by step
  {
    const size_t n = 3001;
    auto layout = Layout::single("p", n);
    const ParamVector theta0 = random_vec(layout, 51, "theta", -1.0f, 1.0f);
    dlc_config cfg{3, 1, DLC_FP16, 9};
    dlc_hyperparams hp;
    dlc_hyperparams_default(&hp);
    hp.warmup_steps = 2;
    cuda::DeviceEngine a(cfg, hp, theta0, 0, DLC_INNER_PINGPONG), b(cfg, hp, theta0, 0, DLC_INNER_PINGPONG);
    std::vector<ParamVector> grads;
    for (int t = 0; t < 9; ++t) grads.push_back(random_vec(layout, 60 + t, "grad", -1e-2f, 1e-2f));
    for (int t = 0; t < 9; ++t) {  // step by step
      a.inner_step(grads[t]);
      if ((t + 1) % 3 == 0) a.outer_step(nullptr);
    }
    float* gdev = nullptr;
    throw_status_ok(dlc_engine_device_ptr(b.handle(), DLC_GRAD, &gdev));
    std::vector<MetricsRecord> records;
    std::vector<uint64_t> rounds;
    const dlc_run_result res = cuda::run_training(
        b, nullptr,
        [&](uint64_t step) {
          throw_status_ok(dlc_engine_upload(b.handle(), DLC_GRAD, grads[step].values().data(), n));
          return cuda::GradSample{gdev, false, 0.5f * (float)step};
        },
        [&](const MetricsRecord& r) { records.push_back(r); }, 0, [&](uint64_t k) { rounds.push_back(k); });
    CHECK(res.steps_done == 9 && res.rounds_done == 3 && res.final_train_loss == 4.0f);
    size_t steps = 0, round_records = 0;
    for (const MetricsRecord& r : records) {
      steps += r.kind == RecordKind::step;
      round_records += r.kind == RecordKind::round;
    }
    CHECK(steps == 9 && round_records == 3 && rounds == std::vector<uint64_t>({1, 2, 3}));
    CHECK(a.download(DLC_THETA_T) == b.download(DLC_THETA_T));
    CHECK(a.download(DLC_THETA_LOCAL) == b.download(DLC_THETA_LOCAL));
    CHECK(a.download(DLC_MOMENTUM) == b.download(DLC_MOMENTUM) && a.download(DLC_ADAM_V) == b.download(DLC_ADAM_V));
  }
  std::printf("test_dropin: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
