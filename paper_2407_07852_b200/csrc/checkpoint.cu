// checkpoint.cu — checkpoint / resume of device engines in the reference's
// ODLCKPT1 format (checkpoint.cpp:17-198).
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

// deserialize_param_vector (tensor.cpp:202-218) into a device buffer of n.
void ckpt_read_vector(File& f, float* dev, size_t n, float* stage, cudaStream_t s) {
  const uint64_t block = f.u64();
  const uint64_t nseg = f.u64();
  uint64_t used = 8, total = 0, expect = 0;
  for (uint64_t i = 0; i < nseg; ++i) {
    const uint64_t len = f.u64();
    if (len > (1u << 20)) fail(DLC_ESERIAL, "checkpoint: implausible segment name");  // tensor.cpp:169-176
    std::string name(len, '\0');
    f.read(name.data(), len);
    const uint64_t off = f.u64(), length = f.u64();
    if (off != expect) fail(DLC_ESHAPE, "checkpoint: segments must be contiguous and ordered");  // tensor.cpp:36-47
    expect += length;
    total += length;
    used += 8 + len + 16;
  }
  if (total != n) fail(DLC_ESHAPE, "checkpoint vector of " + std::to_string(total) + " scalars, engine holds " +
                                       std::to_string(n));
  if (block != used + 4 * total) fail(DLC_ESHAPE, "checkpoint: block length mismatch");
  for (size_t off = 0; off < n; off += kCkptStage) {
    const size_t len = std::min(kCkptStage, n - off);
    f.read(stage, len * 4);
    DLC_CUDA(cudaMemcpyAsync(dev + off, stage, len * 4, cudaMemcpyHostToDevice, s));
    DLC_CUDA(cudaStreamSynchronize(s));
  }
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

int dlc_checkpoint_load(dlc_engine* const* engines, size_t count, const char* path, dlc_checkpoint_meta* meta_out) {
  return guard([&] {
    if (!engines || !path) fail(DLC_EINVAL, "dlc_checkpoint_load: null argument");
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
    for (size_t w = 0; w < 3 * m.ledger_workers; ++w) (void)f.f64();
    const uint64_t n_eng = f.u64();
    if (n_eng != count)
      fail(DLC_ESHAPE, "checkpoint holds " + std::to_string(n_eng) + " engines, " + std::to_string(count) + " given");
    Pinned stage;
    for (size_t i = 0; i < count; ++i) {
      dlc_engine* e = engines[i];
      if (!e) fail(DLC_EINVAL, "dlc_checkpoint_load: null engine");
      DeviceGuard dg(e->device);
      const uint64_t hl = f.u64();
      if (hl > 4096) fail(DLC_ESERIAL, "checkpoint: implausible scalar header");
      std::string text(hl, '\0');
      f.read(text.data(), hl);
      std::map<std::string, std::string> kv;  // parse_scalar_header, checkpoint.cpp:93-129
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
      unalias(e);
      DevState s = read_state(e);
      s.step_count = std::stoull(need("step_count"));
      e->hyper.beta1 = (float)std::stod(need("beta1"));
      e->hyper.beta2 = (float)std::stod(need("beta2"));
      e->hyper.adam_eps = (float)std::stod(need("eps"));
      e->hyper.weight_decay = (float)std::stod(need("weight_decay"));
      e->hyper.outer_lr = (float)std::stod(need("outer_lr"));
      e->hyper.outer_momentum = (float)std::stod(need("outer_momentum"));
      s.scale = (float)std::stod(need("scale"));
      s.growth = std::stoull(need("growth_interval"));
      e->hyper.scaler_growth_interval = s.growth;
      s.good = std::stoull(need("consecutive_good"));
      s.inner_step = std::stoull(need("inner_step"));
      s.outer_epoch = std::stoull(need("outer_epoch"));
      s.found_inf = 0;
      s.delta_nonfinite = 0;
      if (s.inner_step > e->cfg.total_inner_steps) fail(DLC_ECONFIG, "checkpoint inner_step beyond total_inner_steps");
      for (int which : {DLC_THETA_T, DLC_THETA_LOCAL, DLC_ADAM_M, DLC_ADAM_V, DLC_MOMENTUM})
        ckpt_read_vector(f, live(e, which), e->n, stage.p, e->stream);
      // betas may differ from the engine's: rebuild the per-step tables
      if (e->tab) cudaFree(e->tab);
      e->tab = nullptr;
      e->tab_cap = 0;
      ensure_tables(e, std::max<uint64_t>(s.step_count + 2, e->issued_inner + 2));
      DLC_CUDA(cudaMemcpy(e->st, &s, sizeof(s), cudaMemcpyHostToDevice));
      e->issued_inner = s.inner_step;
    }
    if (meta_out) *meta_out = m;
  });
}

}  // extern "C"
