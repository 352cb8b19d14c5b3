// checkpoint.cu — checkpoint / resume of device engines in the reference's
// ODLCKPT1 format (checkpoint.cpp:17-198).
#include <chrono>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <array>
#include <stdexcept>
#include <map>
#include <string>
#include <vector>

#include "engine_impl.hpp"

using namespace dlc;

// ---- checkpoint / resume, ODLCKPT1 (checkpoint.cpp:17-198) -------------------------

namespace {

constexpr char kCkptMagic[8] = {'O', 'D', 'L', 'C', 'K', 'P', 'T', '1'};
constexpr size_t kCkptStage = size_t(16) << 20;  // floats per staging round trip

struct File {
  FILE* f = nullptr;
  std::string path;
  File(const char* p, const char* mode) : path(p) {
    f = std::fopen(p, mode);
    if (!f) fail(DLC_ECONFIG, std::string("cannot open checkpoint file '") + p + "'");
  }
  ~File() {
    if (f) std::fclose(f);
  }
  uint64_t size() {
    const long here = std::ftell(f);
    std::fseek(f, 0, SEEK_END);
    const long end = std::ftell(f);
    std::fseek(f, here, SEEK_SET);
    return end < 0 ? 0 : (uint64_t)end;
  }
  void write(const void* d, size_t b) {
    if (b && std::fwrite(d, 1, b, f) != b) fail(DLC_EINVAL, "checkpoint write failed: " + path);
  }
  void read(void* d, size_t b) {
    if (b && std::fread(d, 1, b, f) != b) fail(DLC_ESERIAL, "checkpoint truncated: " + path);  // checkpoint.cpp:45,60
  }
  void u64(uint64_t v) {
    uint8_t b[8];
    for (int i = 0; i < 8; ++i) b[i] = (uint8_t)(v >> (8 * i));
    write(b, 8);
  }
  uint64_t u64() {
    uint8_t b[8];
    read(b, 8);
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)b[i] << (8 * i);
    return v;
  }
  void f64(double d) {
    uint64_t v;
    std::memcpy(&v, &d, 8);
    u64(v);
  }
  double f64() {
    const uint64_t v = u64();
    double d;
    std::memcpy(&d, &v, 8);
    return d;
  }
};

struct Seg {
  std::string name;
  uint64_t offset, length;
};

// scalar_header, checkpoint.cpp:74-91 (same printf formats, FP64 text).
std::string ckpt_header(const dlc_engine* e, const DevState& s) {
  char buf[512];
  std::snprintf(buf, sizeof(buf),
                "step_count=%" PRIu64 "\nbeta1=%.17g\nbeta2=%.17g\neps=%.17g\n"
                "weight_decay=%.17g\nouter_lr=%.17g\nouter_momentum=%.17g\n"
                "scale=%.17g\ngrowth_interval=%" PRIu64 "\nconsecutive_good=%" PRIu64
                "\ninner_step=%" PRIu64 "\nouter_epoch=%" PRIu64 "\n",
                s.step_count, (double)e->hyper.beta1, (double)e->hyper.beta2, (double)e->hyper.adam_eps,
                (double)e->hyper.weight_decay, (double)e->hyper.outer_lr, (double)e->hyper.outer_momentum,
                (double)s.scale, s.growth, s.good, s.inner_step, s.outer_epoch);
  return buf;
}

// serialize_layout + FP32 payload (tensor.cpp:156-200), streamed from the device.
void ckpt_write_vector(File& f, const std::vector<Seg>& segs, const float* dev, size_t n, float* stage,
                       cudaStream_t s) {
  uint64_t layout_bytes = 8;
  for (const Seg& g : segs) layout_bytes += 8 + g.name.size() + 16;
  f.u64(layout_bytes + 4 * (uint64_t)n);  // put_block length prefix (checkpoint.cpp:31-34)
  f.u64(segs.size());
  for (const Seg& g : segs) {
    f.u64(g.name.size());
    f.write(g.name.data(), g.name.size());
    f.u64(g.offset);
    f.u64(g.length);
  }
  for (size_t off = 0; off < n; off += kCkptStage) {  // little-endian FP32 (x86 host order)
    const size_t len = std::min(kCkptStage, n - off);
    DLC_CUDA(cudaMemcpyAsync(stage, dev + off, len * 4, cudaMemcpyDeviceToHost, s));
    DLC_CUDA(cudaStreamSynchronize(s));
    f.write(stage, len * 4);
  }
}

// deserialize_param_vector (tensor.cpp:202-218), first pass: the layout of one
// vector block, checked against the engine's size (and the caller's layout,
// restore_state's same_layout check, engine.cpp:148-155, when one is given);
// returns the file offset of the FP32 payload and skips it.
long ckpt_parse_vector(File& f, size_t n, const std::vector<Seg>* expect, std::vector<Seg>& got) {
  const uint64_t block = f.u64();
  const uint64_t nseg = f.u64();
  if (nseg > (1u << 20)) fail(DLC_ESERIAL, "checkpoint: implausible segment count");
  uint64_t used = 8, total = 0, next = 0;
  got.clear();
  for (uint64_t i = 0; i < nseg; ++i) {
    const uint64_t len = f.u64();
    if (len > (1u << 20)) fail(DLC_ESERIAL, "checkpoint: implausible segment name");  // tensor.cpp:169-176
    std::string name(len, '\0');
    f.read(name.data(), len);
    const uint64_t off = f.u64(), length = f.u64();
    if (off != next) fail(DLC_ESHAPE, "checkpoint: segments must be contiguous and ordered");  // tensor.cpp:36-47
    next += length;
    total += length;
    used += 8 + len + 16;
    got.push_back({name, off, length});
  }
  if (total != n) fail(DLC_ESHAPE, "checkpoint vector of " + std::to_string(total) + " scalars, engine holds " +
                                       std::to_string(n));
  if (block != used + 4 * total) fail(DLC_ESHAPE, "checkpoint: block length mismatch");
  if (expect) {
    bool same = expect->size() == got.size();
    for (size_t i = 0; same && i < got.size(); ++i)
      same = (*expect)[i].name == got[i].name && (*expect)[i].length == got[i].length;
    if (!same) fail(DLC_ESHAPE, "restore_state: checkpoint layout mismatch");  // engine.cpp:148-155
  }
  const long at = std::ftell(f.f);
  if (at < 0 || (uint64_t)at + 4 * total > f.size() || std::fseek(f.f, (long)(4 * total), SEEK_CUR) != 0)
    fail(DLC_ESERIAL, "checkpoint truncated: " + f.path);  // checkpoint.cpp:45,60
  return at;
}

// Second pass: the FP32 payload at `at` into a device buffer of n.
void ckpt_read_payload(File& f, long at, float* dev, size_t n, float* stage, cudaStream_t s) {
  if (std::fseek(f.f, at, SEEK_SET) != 0) fail(DLC_ESERIAL, "checkpoint seek failed: " + f.path);
  for (size_t off = 0; off < n; off += kCkptStage) {
    const size_t len = std::min(kCkptStage, n - off);
    f.read(stage, len * 4);
    DLC_CUDA(cudaMemcpyAsync(dev + off, stage, len * 4, cudaMemcpyHostToDevice, s));
    DLC_CUDA(cudaStreamSynchronize(s));
  }
}

// parse_scalar_header, checkpoint.cpp:93-129, into the values load commits.
struct EngineHeader {
  uint64_t step_count, growth, good, inner_step, outer_epoch;
  float beta1, beta2, eps, wd, outer_lr, outer_mu, scale;
};

EngineHeader ckpt_parse_header(const std::string& text) {
  std::map<std::string, std::string> kv;
  size_t pos = 0;
  while (pos < text.size()) {
    const size_t nl = text.find('\n', pos);
    const std::string line = text.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos);
    pos = nl == std::string::npos ? text.size() : nl + 1;
    const size_t eq = line.find('=');
    if (eq != std::string::npos) kv[line.substr(0, eq)] = line.substr(eq + 1);
  }
  auto need = [&](const char* key) {
    const auto it = kv.find(key);
    if (it == kv.end()) fail(DLC_ESERIAL, std::string("checkpoint header missing '") + key + "'");  // checkpoint.cpp:109
    return it->second;
  };
  EngineHeader h{};
  try {
    h.step_count = std::stoull(need("step_count"));
    h.beta1 = (float)std::stod(need("beta1"));
    h.beta2 = (float)std::stod(need("beta2"));
    h.eps = (float)std::stod(need("eps"));
    h.wd = (float)std::stod(need("weight_decay"));
    h.outer_lr = (float)std::stod(need("outer_lr"));
    h.outer_mu = (float)std::stod(need("outer_momentum"));
    h.scale = (float)std::stod(need("scale"));
    h.growth = std::stoull(need("growth_interval"));
    h.good = std::stoull(need("consecutive_good"));
    h.inner_step = std::stoull(need("inner_step"));
    h.outer_epoch = std::stoull(need("outer_epoch"));
  } catch (const std::logic_error& x) {  // std::stoull / std::stod: not a number, out of range
    fail(DLC_ESERIAL, std::string("checkpoint header: bad number (") + x.what() + ")");
  }
  return h;
}

struct Pinned {
  float* p = nullptr;
  Pinned() { DLC_CUDA(cudaMallocHost(&p, kCkptStage * 4)); }
  ~Pinned() { cudaFreeHost(p); }
};

}  // namespace

extern "C" {

int dlc_checkpoint_save(dlc_engine* const* engines, size_t count, const char* path, const dlc_checkpoint_meta* meta,
                        const char* const* seg_names, const uint64_t* seg_lengths, size_t nseg) {
  return guard([&] {
    if (!engines || !path || !meta) fail(DLC_EINVAL, "dlc_checkpoint_save: null argument");
    if (meta->ledger_workers && !meta->ledger) fail(DLC_EINVAL, "dlc_checkpoint_save: ledger missing");
    for (size_t i = 0; i < count; ++i)
      if (!engines[i]) fail(DLC_EINVAL, "dlc_checkpoint_save: null engine");
    File f(path, "wb");
    f.write(kCkptMagic, 8);  // save_checkpoint, checkpoint.cpp:131-160
    f.u64(meta->config_hash);
    f.u64(meta->completed_rounds);
    f.f64(meta->clock_seconds);
    f.u64(meta->reduce_data_bytes);
    f.u64(meta->ledger_workers);
    for (size_t w = 0; w < meta->ledger_workers; ++w)
      for (int j = 0; j < 3; ++j) f.f64(meta->ledger[3 * w + j]);
    f.u64(count);
    Pinned stage;
    for (size_t i = 0; i < count; ++i) {
      dlc_engine* e = engines[i];
      DeviceGuard dg(e->device);
      std::vector<Seg> segs;
      if (seg_names && nseg) {
        uint64_t off = 0;
        for (size_t j = 0; j < nseg; ++j) {
          segs.push_back({seg_names[j], off, seg_lengths[j]});
          off += seg_lengths[j];
        }
        if (off != e->n) fail(DLC_ESHAPE, "checkpoint layout does not cover the engine's vector");
      } else {
        segs.push_back({"p", 0, e->n});
      }
      const DevState s = read_state(e);
      const std::string header = ckpt_header(e, s);
      f.u64(header.size());
      f.write(header.data(), header.size());
      for (int which : {DLC_THETA_T, DLC_THETA_LOCAL, DLC_ADAM_M, DLC_ADAM_V, DLC_MOMENTUM})
        ckpt_write_vector(f, segs, live(e, which), e->n, stage.p, e->stream);
    }
  });
}

// load_checkpoint (checkpoint.cpp:162-198) + restore_state, all or nothing:
// pass 1 parses and validates the whole file (headers, numbers, every vector's
// layout and length, the file's size) before anything is touched; pass 2
// streams the vectors into each engine's IDLE ping-pong buffers (theta_t[ocur^1],
// buf[ocur^1], p/m/v[cur^1]), and only once every engine's vectors are in does
// the commit swap them in (flip cur / ocur) with the hyperparameters and
// counters.  INPLACE engines have no idle p / m / v: they are written in place
// after the validation pass.
int dlc_checkpoint_load_layout(dlc_engine* const* engines, size_t count, const char* path,
                               const char* const* seg_names, const uint64_t* seg_lengths, size_t nseg,
                               dlc_checkpoint_meta* meta_out) {
  return guard([&] {
    if (!engines || !path) fail(DLC_EINVAL, "dlc_checkpoint_load: null argument");
    if (nseg && (!seg_names || !seg_lengths)) fail(DLC_EINVAL, "dlc_checkpoint_load: layout arrays missing");
    for (size_t i = 0; i < count; ++i)
      if (!engines[i]) fail(DLC_EINVAL, "dlc_checkpoint_load: null engine");
    std::vector<Seg> expect;
    for (size_t j = 0; j < nseg; ++j) expect.push_back({seg_names[j], 0, seg_lengths[j]});
    File f(path, "rb");
    char magic[8];
    f.read(magic, 8);
    if (std::memcmp(magic, kCkptMagic, 8) != 0) fail(DLC_ESERIAL, "not a checkpoint file: bad magic");  // checkpoint.cpp:170
    dlc_checkpoint_meta m{};
    m.config_hash = f.u64();
    m.completed_rounds = f.u64();
    m.clock_seconds = f.f64();
    m.reduce_data_bytes = f.u64();
    m.ledger_workers = f.u64();
    if (m.ledger_workers > (1u << 20)) fail(DLC_ESERIAL, "checkpoint: implausible ledger");
    for (size_t w = 0; w < 3 * m.ledger_workers; ++w) (void)f.f64();
    const uint64_t n_eng = f.u64();
    if (n_eng != count)
      fail(DLC_ESHAPE, "checkpoint holds " + std::to_string(n_eng) + " engines, " + std::to_string(count) + " given");
    // ---- pass 1: validate everything ----
    std::vector<EngineHeader> hdr(count);
    std::vector<std::array<long, 5>> at(count);
    std::vector<Seg> layout;
    for (size_t i = 0; i < count; ++i) {
      dlc_engine* e = engines[i];
      const uint64_t hl = f.u64();
      if (hl > 4096) fail(DLC_ESERIAL, "checkpoint: implausible scalar header");
      std::string text(hl, '\0');
      f.read(text.data(), hl);
      hdr[i] = ckpt_parse_header(text);
      if (hdr[i].inner_step > e->cfg.total_inner_steps)
        fail(DLC_ECONFIG, "checkpoint inner_step beyond total_inner_steps");
      std::vector<Seg> first;
      for (int v = 0; v < 5; ++v) {
        at[i][v] = ckpt_parse_vector(f, e->n, nseg ? &expect : (v ? &first : nullptr), layout);
        if (v == 0) first = layout;  // without a caller layout: one layout for all five vectors
      }
    }
    // ---- pass 2: vectors into the idle buffers (live state untouched) ----
    Pinned stage;
    std::vector<DevState> st(count);
    for (size_t i = 0; i < count; ++i) {
      dlc_engine* e = engines[i];
      DeviceGuard dg(e->device);
      st[i] = read_state(e);
      const bool pp = e->inner_mode == DLC_INNER_PINGPONG;
      const int oc = st[i].ocur ^ 1, cu = pp ? st[i].cur ^ 1 : st[i].cur;
      if (!pp) unalias(e);
      float* dst[5] = {e->theta_t[oc], e->p[cu], e->m[cu], e->v[cu], e->buf[oc]};
      for (int v = 0; v < 5; ++v) ckpt_read_payload(f, at[i][v], dst[v], e->n, stage.p, e->stream);
    }
    // ---- commit ----
    for (size_t i = 0; i < count; ++i) {
      dlc_engine* e = engines[i];
      DeviceGuard dg(e->device);
      const EngineHeader& h = hdr[i];
      DevState s = st[i];
      s.ocur ^= 1;
      if (e->inner_mode == DLC_INNER_PINGPONG) s.cur ^= 1;
      s.lalias = 0;
      s.step_count = h.step_count;
      s.scale = h.scale;
      s.growth = h.growth;
      s.good = h.good;
      s.inner_step = h.inner_step;
      s.outer_epoch = h.outer_epoch;
      s.found_inf = 0;
      s.delta_nonfinite = 0;
      s.delta_ready = 0;
      e->delta_fused = false;
      e->hyper.beta1 = h.beta1;
      e->hyper.beta2 = h.beta2;
      e->hyper.adam_eps = h.eps;
      e->hyper.weight_decay = h.wd;
      e->hyper.outer_lr = h.outer_lr;
      e->hyper.outer_momentum = h.outer_mu;
      e->hyper.scaler_growth_interval = h.growth;
      // betas may differ from the engine's: rebuild the per-step tables
      if (e->tab) cudaFree(e->tab);
      e->tab = nullptr;
      e->tab_cap = 0;
      ensure_tables(e, std::max<uint64_t>(s.step_count + 2, h.inner_step + 2));
      DLC_CUDA(cudaMemcpy(e->st, &s, sizeof(s), cudaMemcpyHostToDevice));
      e->issued_inner = s.inner_step;
    }
    if (meta_out) *meta_out = m;
  });
}

int dlc_checkpoint_load(dlc_engine* const* engines, size_t count, const char* path, dlc_checkpoint_meta* meta_out) {
  return dlc_checkpoint_load_layout(engines, count, path, nullptr, nullptr, 0, meta_out);
}

}  // extern "C"
