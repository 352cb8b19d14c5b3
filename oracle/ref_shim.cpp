// ref_shim.cpp — extern "C" wrappers around the REFERENCE implementation.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference's own hot-path sources, straight from /root/reference/proj/src
// (fp16.cpp tensor.cpp optim.cpp reduce.cpp), into oracle/_ref/libdiloco_ref.so
// with the reference's flags (-ffp-contract=off, proj/CMakeLists.txt:18).  No
// reference source is copied into this repository.  The .so is linked with
// hidden visibility so only the ref_* symbols below are exported.
//
// Uses: (1) pin the C restatement (oracle/diloco_oracle.c) bit-for-bit,
// (2) generate tests/golden fixtures, (3) the CPU baseline / `bench.py --impl
// reference` arm (ref_bench_*), timing the reference's own functions.
#include <algorithm>
#include <atomic>
#include <stdexcept>
#include <barrier>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <thread>
#include <vector>

#include "diloco/fp16.hpp"
#include "diloco/optim.hpp"
#include "diloco/reduce.hpp"
#include "diloco/rng.hpp"
#include "diloco/tensor.hpp"
#include "diloco/wire.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

using namespace diloco;

namespace {

enum { kOk = 0, kShape = 1, kConfig = 2, kNumeric = 3, kCollective = 4, kSerial = 5, kOther = 9 };

ParamVector pv(const float* data, size_t n) {
  return ParamVector(Layout::single("p", n), std::vector<float>(data, data + n));
}

void put(const ParamVector& v, float* out) {
  std::memcpy(out, v.values().data(), v.size() * sizeof(float));
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const ShapeError&) {
    return kShape;
  } catch (const ConfigError&) {
    return kConfig;
  } catch (const NumericError&) {
    return kNumeric;
  } catch (const CollectiveError&) {
    return kCollective;
  } catch (const SerializationError&) {
    return kSerial;
  } catch (const std::exception&) {
    return kOther;
  }
}

}  // namespace

REF_API uint16_t ref_fp16_encode(float v) { return fp16_encode(v); }
REF_API float ref_fp16_decode(uint16_t b) { return fp16_decode(b); }

REF_API int ref_encode_fp16(const float* v, size_t n, uint16_t* out) {
  const Fp16Buffer b = encode_fp16(pv(v, n));
  std::memcpy(out, b.bits.data(), n * sizeof(uint16_t));
  return b.overflow ? 1 : 0;
}

REF_API int ref_decode_fp16(const uint16_t* b, size_t n, float* out) {
  Fp16Buffer buf;
  buf.bits.assign(b, b + n);
  return guarded([&] { put(decode_fp16(buf, Layout::single("p", n)), out); });
}

REF_API int ref_all_finite(const float* v, size_t n) { return pv(v, n).all_finite() ? 1 : 0; }

REF_API int ref_axpy(float alpha, const float* x, const float* y, size_t n, float* out) {
  return guarded([&] { put(axpy(alpha, pv(x, n), pv(y, n)), out); });
}

REF_API float ref_lr_at(uint64_t warmup, uint64_t total, float base_lr, int cosine,
                        uint64_t step) {
  LrSchedule s;
  s.warmup_steps = warmup;
  s.total_steps = total;
  s.base_lr = base_lr;
  s.decay = cosine ? LrDecay::cosine : LrDecay::none;
  return lr_at(s, step);
}

// adamw_step (optim.hpp:61-62): p -> out; m, v, step_count updated in place.
REF_API int ref_adamw_step(const float* p, const float* g, float* m, float* v, size_t n,
                           float b1, float b2, float eps, float wd, uint64_t* step_count,
                           float lr, float* out) {
  auto layout = Layout::single("p", n);
  AdamWState st;
  st.m = ParamVector(layout, std::vector<float>(m, m + n));
  st.v = ParamVector(layout, std::vector<float>(v, v + n));
  st.step_count = *step_count;
  st.beta1 = b1;
  st.beta2 = b2;
  st.eps = eps;
  st.weight_decay = wd;
  const ParamVector params(layout, std::vector<float>(p, p + n));
  const ParamVector grad(layout, std::vector<float>(g, g + n));
  return guarded([&] {
    const ParamVector o = adamw_step(st, params, grad, lr);
    put(o, out);
    put(st.m, m);
    put(st.v, v);
    *step_count = st.step_count;
  });
}

// nesterov_step (optim.hpp:65-66): p -> out; momentum buffer in place.
REF_API int ref_nesterov_step(const float* p, const float* g, float* buf, size_t n,
                              float lr, float mu, float* out) {
  auto layout = Layout::single("p", n);
  NesterovState st;
  st.momentum_buf = ParamVector(layout, std::vector<float>(buf, buf + n));
  st.lr = lr;
  st.momentum = mu;
  const ParamVector params(layout, std::vector<float>(p, p + n));
  const ParamVector grad(layout, std::vector<float>(g, g + n));
  return guarded([&] {
    const ParamVector o = nesterov_step(st, params, grad);
    put(o, out);
    put(st.momentum_buf, buf);
  });
}

REF_API int ref_scaler_unscale_and_check(float scale, const float* g, size_t n, float* out) {
  LossScaler s;
  s.scale = scale;
  const UnscaleResult r = scaler_unscale_and_check(s, pv(g, n));
  put(r.grad, out);
  return r.overflow ? 1 : 0;
}

REF_API void ref_scaler_update(float* scale, uint64_t* good, uint64_t growth, int overflow) {
  LossScaler s;
  s.scale = *scale;
  s.consecutive_good = *good;
  s.growth_interval = growth;
  scaler_update(s, overflow != 0);
  *scale = s.scale;
  *good = s.consecutive_good;
}

// reduce_average (reduce.hpp:65-66) over k contributions of n floats.
REF_API int ref_reduce_average(const float* const* contribs, size_t k, size_t n,
                               int precision, float* out) {
  auto layout = Layout::single("delta", n);
  std::vector<ParamVector> vs;
  vs.reserve(k);
  for (size_t j = 0; j < k; ++j) {
    vs.emplace_back(layout, std::vector<float>(contribs[j], contribs[j] + n));
  }
  std::vector<const ParamVector*> ptrs;
  for (const auto& v : vs) ptrs.push_back(&v);
  return guarded([&] {
    put(reduce_average(ptrs, precision ? Precision::fp16 : Precision::fp32), out);
  });
}

REF_API void ref_partition_ranges(size_t n, size_t k, size_t* offsets, size_t* lengths) {
  const std::vector<Range> r = partition_ranges(n, k);
  for (size_t i = 0; i < k; ++i) {
    offsets[i] = r[i].offset;
    lengths[i] = r[i].length;
  }
}

REF_API uint64_t ref_per_peer_reduce_bytes(size_t n, size_t k, size_t rank, int precision) {
  return per_peer_reduce_bytes(n, k, rank, precision ? Precision::fp16 : Precision::fp32);
}

REF_API uint64_t ref_fleet_reduce_bytes(size_t n, size_t k, int precision) {
  return fleet_reduce_bytes(n, k, precision ? Precision::fp16 : Precision::fp32);
}

// SoloCollective::all_reduce_avg (reduce.cpp:113-126).
REF_API int ref_solo_all_reduce_avg(const float* delta, size_t n, int precision, float* out) {
  SoloCollective solo;
  PseudoGradient pg;
  pg.delta = pv(delta, n);
  pg.precision = precision ? Precision::fp16 : Precision::fp32;
  return guarded([&] { put(solo.all_reduce_avg(pg, nullptr).delta, out); });
}

// ---------------------------------------------------------------------------
// CPU baseline harness: the reference's own functions, one engine set per
// host thread on a disjoint slice (every op on the path is elementwise, so a
// slice is an exact sub-problem).  Inputs follow SURVEY.md §8(d):
//   theta_0 ~ U(-0.05, 0.05)  CounterRng(4242, "theta", 0)
//   theta_local_w = theta_0 - U(-1e-3, 1e-3)  CounterRng(4242, "local", w)
//   grad_w ~ U(-1e-2, 1e-2)   CounterRng(4242, "grad", w)
// Returns seconds per outer step (max over threads of the per-iteration wall
// time, averaged over iters) in *sec_per_iter.
// ---------------------------------------------------------------------------

namespace {

std::vector<float> fill(uint64_t seed, const char* purpose, uint64_t stream, size_t first,
                        size_t n, float lo, float hi) {
  CounterRng rng(seed, purpose, stream);
  // skip `first` draws: each draw advances the (only) state word by the
  // splitmix64 increment (rng.hpp:43-46), so add first x increment directly
  static_assert(sizeof(CounterRng) == sizeof(uint64_t), "CounterRng holds one state word");
  uint64_t state;
  std::memcpy(&state, &rng, sizeof state);
  state += 0x9E3779B97F4A7C15ull * (uint64_t)first;
  std::memcpy(static_cast<void*>(&rng), &state, sizeof state);
  std::vector<float> out(n);
  for (float& f : out) f = rng.next_uniform(lo, hi);
  return out;
}

}  // namespace

// Thread t takes elements [lo_t, lo_t + len_t) of an n-element vector
// (balanced split).  `warmup` untimed iterations, then `iters` timed ones;
// per_iter[i] = wall seconds of timed iteration i, from the moment every
// thread starts it until the last one finishes (main-thread clock between
// the two barriers).
namespace {

struct Split {
  size_t lo, len;
};
Split split(size_t n, int threads, int t) {
  const size_t base = n / threads, extra = n % threads;
  return Split{t * base + std::min<size_t>(t, extra), base + ((size_t)t < extra ? 1 : 0)};
}

template <typename Body>
int run_timed(int threads, int warmup, int iters, double* per_iter, Body&& body) {
  std::barrier sync(threads + 1);
  std::atomic<int> err{0};
  auto work = [&](int tid) {
    try {
      body.setup(tid);
    } catch (...) {
      err = 1;
    }
    for (int it = 0; it < warmup + iters; ++it) {
      body.prepare(tid);  // untimed
      sync.arrive_and_wait();
      try {
        if (!err) body.step(tid);
      } catch (...) {
        err = 1;
      }
      sync.arrive_and_wait();
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
  for (int it = 0; it < warmup + iters; ++it) {
    sync.arrive_and_wait();
    const auto t0 = std::chrono::steady_clock::now();
    sync.arrive_and_wait();
    if (it >= warmup) per_iter[it - warmup] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  for (auto& th : pool) th.join();
  return err ? kOther : kOk;
}

}  // namespace

// run_simulated's outer round (netsim.cpp:325-357) over n parameters per
// worker, K workers: K x axpy pseudo-gradients, one reduce_average, K x
// (all_finite, nesterov_step, theta_local = theta_t).
REF_API int ref_bench_outer(int threads, size_t n, size_t k, int precision, int warmup, int iters, float lr,
                            float mu, double* per_iter) {
  if (threads < 1 || k < 1 || iters < 1 || warmup < 0 || n < (size_t)threads || !per_iter) return kConfig;
  const Precision prec = precision ? Precision::fp16 : Precision::fp32;
  struct Body {
    size_t n, k;
    Precision prec;
    float lr, mu;
    struct Slice {
      std::vector<ParamVector> theta_t, local, pristine;
      std::vector<NesterovState> outer;
    };
    std::vector<Slice> sl;
    int threads;
    void setup(int tid) {
      const Split sp = split(n, threads, tid);
      auto layout = Layout::single("p", sp.len);
      const std::vector<float> theta0 = fill(4242, "theta", 0, sp.lo, sp.len, -0.05f, 0.05f);
      Slice& s = sl[tid];
      for (size_t w = 0; w < k; ++w) {
        std::vector<float> noise = fill(4242, "local", w, sp.lo, sp.len, -1e-3f, 1e-3f);
        std::vector<float> loc(sp.len);
        for (size_t i = 0; i < sp.len; ++i) loc[i] = theta0[i] - noise[i];
        s.theta_t.emplace_back(layout, theta0);
        s.pristine.emplace_back(layout, std::move(loc));
        s.local.push_back(s.pristine.back());
        s.outer.push_back(NesterovState::init(layout, lr, mu));
      }
    }
    void prepare(int tid) {  // a fresh end-of-window theta_local
      Slice& s = sl[tid];
      for (size_t w = 0; w < k; ++w) s.local[w] = s.pristine[w];
    }
    void step(int tid) {
      Slice& s = sl[tid];
      std::vector<ParamVector> deltas;
      deltas.reserve(k);
      for (size_t w = 0; w < k; ++w) deltas.push_back(axpy(-1.0f, s.local[w], s.theta_t[w]));  // engine.cpp:122
      std::vector<const ParamVector*> ptrs;
      for (const auto& d : deltas) ptrs.push_back(&d);
      const ParamVector dbar = reduce_average(ptrs, prec);
      for (size_t w = 0; w < k; ++w) {  // DilocoEngine::outer_step, engine.cpp:136-144
        if (dbar.all_finite()) s.theta_t[w] = nesterov_step(s.outer[w], s.theta_t[w], dbar);
        s.local[w] = s.theta_t[w];
      }
    }
  } body{n, k, prec, lr, mu, std::vector<Body::Slice>(threads), threads};
  return run_timed(threads, warmup, iters, per_iter, body);
}

// apply_inner_step (engine.cpp:50-69) over n parameters: scale_gradient
// (engine.cpp:20-27), scaler_unscale_and_check, lr_at, adamw_step,
// scaler_update.
REF_API int ref_bench_inner(int threads, size_t n, int warmup, int iters, double* per_iter) {
  if (threads < 1 || iters < 1 || warmup < 0 || n < (size_t)threads || !per_iter) return kConfig;
  struct Body {
    size_t n;
    int threads;
    struct Slice {
      std::vector<ParamVector> params, grad;
      std::vector<AdamWState> adam;
      LossScaler scaler;
      LrSchedule sched;
    };
    std::vector<Slice> sl;
    void setup(int tid) {
      const Split sp = split(n, threads, tid);
      auto layout = Layout::single("p", sp.len);
      Slice& s = sl[tid];
      s.params.emplace_back(layout, fill(4242, "theta", 0, sp.lo, sp.len, -0.05f, 0.05f));
      s.grad.emplace_back(layout, fill(4242, "grad", 0, sp.lo, sp.len, -1e-2f, 1e-2f));
      s.adam.push_back(AdamWState::init(layout, 0.9f, 0.95f, 1e-8f, 0.1f));
    }
    void prepare(int) {}
    void step(int tid) {
      Slice& s = sl[tid];
      const auto g = s.grad[0].values();
      std::vector<float> scaled(g.size());
      for (size_t i = 0; i < g.size(); ++i) scaled[i] = g[i] * s.scaler.scale;
      UnscaleResult un = scaler_unscale_and_check(s.scaler, ParamVector(s.grad[0].layout(), std::move(scaled)));
      if (!un.overflow) s.params[0] = adamw_step(s.adam[0], s.params[0], un.grad, lr_at(s.sched, s.adam[0].step_count + 1));
      scaler_update(s.scaler, un.overflow);
    }
  } body{n, threads, std::vector<Body::Slice>(threads)};
  return run_timed(threads, warmup, iters, per_iter, body);
}

// ---------------------------------------------------------------------------
// Checkpoint files through the reference's own save/load (checkpoint.cpp).
// ---------------------------------------------------------------------------
#include "diloco/checkpoint.hpp"

// Reads engine `idx` of a checkpoint with load_checkpoint (checkpoint.cpp:162-198).
// u[0..5] = step_count, growth_interval, consecutive_good, inner_step,
// outer_epoch, engine count; d[0..7] = beta1, beta2, eps, weight_decay,
// outer_lr, outer_momentum, scale, clock_seconds; h[0..2] = config_hash,
// completed_rounds, reduce_data_bytes.  Vectors are copied when non-null and n
// matches.
REF_API int ref_checkpoint_read(const char* path, size_t idx, size_t n, float* tt, float* tl, float* m, float* v,
                                float* buf, uint64_t* u, double* d, uint64_t* h) {
  return guarded([&] {
    const Checkpoint ck = load_checkpoint(path);
    h[0] = ck.config_hash;
    h[1] = ck.completed_rounds;
    h[2] = ck.reduce_data_bytes;
    u[5] = ck.engines.size();
    d[7] = ck.clock_seconds;
    if (idx >= ck.engines.size()) throw ShapeError("engine index");
    const EngineState& s = ck.engines[idx];
    if (s.theta_t.size() != n) throw ShapeError("size");
    if (tt) put(s.theta_t, tt);
    if (tl) put(s.theta_local, tl);
    if (m) put(s.inner.m, m);
    if (v) put(s.inner.v, v);
    if (buf) put(s.outer.momentum_buf, buf);
    u[0] = s.inner.step_count;
    u[1] = s.scaler.growth_interval;
    u[2] = s.scaler.consecutive_good;
    u[3] = s.inner_step;
    u[4] = s.outer_epoch;
    d[0] = s.inner.beta1;
    d[1] = s.inner.beta2;
    d[2] = s.inner.eps;
    d[3] = s.inner.weight_decay;
    d[4] = s.outer.lr;
    d[5] = s.outer.momentum;
    d[6] = s.scaler.scale;
  });
}

// Writes a one-engine checkpoint with save_checkpoint (checkpoint.cpp:131-160).
REF_API int ref_checkpoint_write(const char* path, size_t n, const float* tt, const float* tl, const float* m,
                                 const float* v, const float* buf, const uint64_t* u, const double* d,
                                 const uint64_t* h) {
  return guarded([&] {
    Checkpoint ck;
    ck.config_hash = h[0];
    ck.completed_rounds = h[1];
    ck.reduce_data_bytes = h[2];
    ck.clock_seconds = d[7];
    EngineState s;
    s.theta_t = pv(tt, n);
    s.theta_local = pv(tl, n);
    s.inner.m = pv(m, n);
    s.inner.v = pv(v, n);
    s.outer.momentum_buf = pv(buf, n);
    s.inner.step_count = u[0];
    s.scaler.growth_interval = u[1];
    s.scaler.consecutive_good = u[2];
    s.inner_step = u[3];
    s.outer_epoch = u[4];
    s.inner.beta1 = (float)d[0];
    s.inner.beta2 = (float)d[1];
    s.inner.eps = (float)d[2];
    s.inner.weight_decay = (float)d[3];
    s.outer.lr = (float)d[4];
    s.outer.momentum = (float)d[5];
    s.scaler.scale = (float)d[6];
    ck.engines.push_back(std::move(s));
    save_checkpoint(ck, path);
  });
}

// ---- wire codec (wire.cpp:10-104): frames and reduce payloads -------------------

REF_API int ref_encode_frame(uint8_t type, const uint8_t* payload, size_t len, uint8_t* out, size_t* out_len) {
  return guarded([&] {
    WireMessage m;
    m.type = static_cast<MsgType>(type);
    m.payload.assign(payload, payload + len);
    const std::vector<uint8_t> f = encode_frame(m);
    std::memcpy(out, f.data(), f.size());
    *out_len = f.size();
  });
}

REF_API int ref_encode_reduce_payload(uint64_t epoch, uint32_t chunk_index, uint8_t precision, const uint8_t* seg,
                                      size_t seglen, uint8_t* out, size_t* out_len) {
  return guarded([&] {
    ReduceChunkHeader h;
    h.outer_epoch = epoch;
    h.chunk_index = chunk_index;
    h.precision = precision;
    const std::vector<uint8_t> p = encode_reduce_payload(h, std::span<const uint8_t>(seg, seglen));
    std::memcpy(out, p.data(), p.size());
    *out_len = p.size();
  });
}

// Feeds `in` to a FrameParser in pieces of `feed` bytes and pops every complete
// frame: types[i], payload lengths, and each payload's reduce header when it
// decodes (ok[i] = 0 when decode_reduce_payload throws).
REF_API int ref_parse_frames(const uint8_t* in, size_t n, size_t feed, uint8_t* types, uint64_t* payload_lens,
                             uint64_t* epochs, uint32_t* chunk_indices, uint8_t* precisions, int* ok,
                             size_t max_frames, size_t* nframes) {
  return guarded([&] {
    FrameParser parser;
    size_t count = 0;
    for (size_t at = 0; at < n;) {
      const size_t take = std::min(feed ? feed : n, n - at);
      parser.feed(std::span<const uint8_t>(in + at, take));
      at += take;
      while (auto m = parser.next()) {
        if (count >= max_frames) throw std::runtime_error("too many frames");
        types[count] = static_cast<uint8_t>(m->type);
        payload_lens[count] = m->payload.size();
        ok[count] = 0;
        try {
          std::span<const uint8_t> seg;
          const ReduceChunkHeader h = decode_reduce_payload(m->payload, seg);
          epochs[count] = h.outer_epoch;
          chunk_indices[count] = h.chunk_index;
          precisions[count] = h.precision;
          ok[count] = 1;
        } catch (const SerializationError&) {
        }
        ++count;
      }
    }
    *nframes = count;
  });
}

// ---- CPU baseline of the wire path: the scatter side of Node::Impl::all_reduce ----
// Per thread slice: axpy pseudo-gradient (engine.cpp:122), encode_fp16 once at the
// source (collective.cpp:1356-1366), then send_chunk_span's framing of the slice
// (collective.cpp:1318-1345) with the reference's encode_reduce_payload /
// encode_frame (wire.cpp); the chunk segment header (collective.cpp:63-81, in an
// anonymous namespace there) is rebuilt inline.  Frames go to a byte vector in
// place of the socket.
REF_API int ref_bench_wire(int threads, size_t slice, int precision, size_t chunk_bytes, int iters,
                           double* sec_per_iter, uint64_t* frame_bytes) {
  if (threads < 1 || iters < 1 || slice < 1) return kConfig;
  std::barrier sync(threads + 1);
  std::vector<double> t_thread(threads, 0.0);
  std::vector<uint64_t> bytes_thread(threads, 0);
  std::atomic<int> err{0};
  auto work = [&](int tid) {
    try {
      auto layout = Layout::single("p", slice);
      const ParamVector tt(layout, fill(4242, "theta", 0, tid * slice, slice, -0.05f, 0.05f));
      std::vector<float> loc = tt.values().size() ? std::vector<float>(tt.values().begin(), tt.values().end())
                                                  : std::vector<float>();
      const std::vector<float> noise = fill(4242, "local", 0, tid * slice, slice, -1e-3f, 1e-3f);
      for (size_t i = 0; i < slice; ++i) loc[i] -= noise[i];
      const ParamVector tl(layout, std::move(loc));
      const std::string name = "a0.p1.f0123456789abcdeffedcba9876543210";
      for (int it = 0; it < iters; ++it) {
        sync.arrive_and_wait();
        const auto t0 = std::chrono::steady_clock::now();
        const ParamVector delta = axpy(-1.0f, tl, tt);
        Fp16Buffer codes;
        const uint8_t* bytes = reinterpret_cast<const uint8_t*>(delta.values().data());
        size_t width = 4;
        if (precision) {
          codes = encode_fp16(delta);
          bytes = reinterpret_cast<const uint8_t*>(codes.bits.data());
          width = 2;
        }
        const uint64_t max_elems = std::max<uint64_t>(1, chunk_bytes / width);
        uint64_t total = 0;
        uint32_t chunk_index = 0;
        for (uint64_t start = 0; start < slice; start += max_elems) {
          const uint64_t count = std::min<uint64_t>(max_elems, slice - start);
          std::vector<uint8_t> seg;
          seg.reserve(32 + name.size() + count * width);
          auto put_u64 = [&seg](uint64_t v) {
            for (int i = 0; i < 8; ++i) seg.push_back(static_cast<uint8_t>(v >> (8 * i)));
          };
          put_u64(1);
          put_u64(name.size());
          seg.insert(seg.end(), name.begin(), name.end());
          put_u64(start);
          put_u64(count);
          seg.insert(seg.end(), bytes + start * width, bytes + (start + count) * width);
          ReduceChunkHeader h;
          h.outer_epoch = 0;
          h.chunk_index = chunk_index++;
          h.precision = precision ? 1 : 0;
          WireMessage m;
          m.type = MsgType::reduce_chunk;
          m.payload = encode_reduce_payload(h, seg);
          total += encode_frame(m).size();
        }
        t_thread[tid] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        bytes_thread[tid] = total;
        sync.arrive_and_wait();
      }
    } catch (...) {
      err = 1;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
  for (int it = 0; it < iters; ++it) {
    sync.arrive_and_wait();
    sync.arrive_and_wait();
  }
  for (auto& th : pool) th.join();
  if (err) return kOther;
  double worst = 0.0;
  uint64_t total = 0;
  for (int t = 0; t < threads; ++t) {
    worst = t_thread[t] > worst ? t_thread[t] : worst;
    total += bytes_thread[t];
  }
  *sec_per_iter = worst / iters;
  *frame_bytes = total;
  return kOk;
}
