// wire.cu — section 5 of include/diloco_cuda.h: the reference's transport
// framing produced from / consumed into device buffers.
//
// Frame of one reduce chunk (all integers little-endian):
//   "ODLC" | version 1 | type | u64 payload_len          encode_frame, wire.cpp:10-22
//   epoch u64 | chunk_index u32 | precision u8           encode_reduce_payload, wire.cpp:74-88
//   u64 1 | u64 name_len | name | u64 offset | u64 len   encode_chunk_segment, collective.cpp:63-81
//   scalars (len * width bytes)
// send_chunk_span (collective.cpp:1318-1345) cuts a range into chunks of
// max(1, chunk_size_bytes / width) elements.  Every full chunk has the same
// frame size, so the scalars of all full chunks land in the caller's host
// buffer with ONE strided copy-engine transfer (cudaMemcpy2DAsync: source
// pitch = chunk bytes, destination pitch = frame bytes); the host writes only
// the 59 + name_len header bytes of each frame.  Decoding mirrors it: headers
// are parsed on the host, and runs of equally spaced chunks go to the device
// in one strided transfer each.
#include <cstring>
#include <string>
#include <vector>

#include "internal.hpp"

using namespace dlc;

namespace {

constexpr size_t kFrameHeader = 14;    // kFrameHeaderBytes, wire.hpp:29
constexpr size_t kReduceHeader = 13;   // wire.cpp:76-86
constexpr size_t kSegmentFixed = 32;   // count, name_len, offset, length

size_t width_of(int precision) { return precision == DLC_FP16 ? 2 : 4; }

void put_le(uint8_t* out, uint64_t v, int nbytes) {
  for (int i = 0; i < nbytes; ++i) out[i] = static_cast<uint8_t>(v >> (8 * i));
}

uint64_t get_le(const uint8_t* in, int nbytes) {
  uint64_t v = 0;
  for (int i = 0; i < nbytes; ++i) v |= static_cast<uint64_t>(in[i]) << (8 * i);
  return v;
}

// chunk_name (collective.cpp:126-131) with PeerId::hex (collective.cpp:214-220)
std::string chunk_name(uint32_t attempt, uint32_t partition, uint64_t hi, uint64_t lo) {
  char hex[33];
  std::snprintf(hex, sizeof(hex), "%016llx%016llx", static_cast<unsigned long long>(hi),
                static_cast<unsigned long long>(lo));
  return "a" + std::to_string(attempt) + ".p" + std::to_string(partition) + ".f" + std::string(hex, 32);
}

// std::stoul(s) (base 10): leading white space, optional sign, digits; false
// where stoul would throw.  The caller truncates to uint32 like the reference.
bool parse_stoul(const std::string& s, uint64_t* out) {
  size_t i = 0;
  while (i < s.size() && (s[i] == ' ' || (s[i] >= '\t' && s[i] <= '\r'))) ++i;
  bool neg = false;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  uint64_t v = 0;
  size_t digits = 0;
  for (; i < s.size() && s[i] >= '0' && s[i] <= '9'; ++i, ++digits) {
    const uint64_t d = static_cast<uint64_t>(s[i] - '0');
    if (v > (UINT64_MAX - d) / 10) return false;  // out_of_range
    v = v * 10 + d;
  }
  if (!digits) return false;  // invalid_argument
  *out = neg ? (0 - v) : v;
  return true;
}

// std::from_chars(p, p + 16, v, 16): leading hex digits; false when none.
bool parse_hex16(const char* p, uint64_t* out) {
  uint64_t v = 0;
  int digits = 0;
  for (; digits < 16; ++digits) {
    const char c = p[digits];
    int d;
    if (c >= '0' && c <= '9')
      d = c - '0';
    else if (c >= 'a' && c <= 'f')
      d = c - 'a' + 10;
    else if (c >= 'A' && c <= 'F')
      d = c - 'A' + 10;
    else
      break;
    v = (v << 4) | static_cast<uint64_t>(d);
  }
  if (!digits) return false;
  *out = v;
  return true;
}

// parse_chunk_name, collective.cpp:133-152 (+ PeerId::from_hex :221-238)
bool parse_chunk_name(const std::string& name, uint32_t* attempt, uint32_t* partition, uint64_t* hi, uint64_t* lo) {
  if (name.empty() || name[0] != 'a') return false;
  const size_t p = name.find(".p");
  const size_t f = name.find(".f");
  if (p == std::string::npos || f == std::string::npos || f < p) return false;
  uint64_t a = 0, q = 0;
  if (!parse_stoul(name.substr(1, p - 1), &a)) return false;
  if (!parse_stoul(name.substr(p + 2, f - p - 2), &q)) return false;
  const std::string hex = name.substr(f + 2);
  if (hex.size() != 32) return false;
  if (!parse_hex16(hex.data(), hi) || !parse_hex16(hex.data() + 16, lo)) return false;
  *attempt = static_cast<uint32_t>(a);
  *partition = static_cast<uint32_t>(q);
  return true;
}

void check_tags(const dlc_wire_tags* t) {
  if (!t) fail(DLC_EINVAL, "wire: null tags");
  if (t->precision != DLC_FP32 && t->precision != DLC_FP16) fail(DLC_ECONFIG, "wire: unknown precision");
}

}  // namespace

namespace dlc {

// Frame geometry of one send_chunk_span call.
struct WireGeometry {
  size_t width, header, max_elems, full_frames, tail_elems, full_frame_bytes, bytes;
};

WireGeometry wire_geometry(uint64_t elems, const dlc_wire_tags* t, size_t name_len) {
  WireGeometry g{};
  g.width = width_of(t->precision);
  g.max_elems = std::max<uint64_t>(1, t->chunk_size_bytes / g.width);  // collective.cpp:1325-1326
  g.header = kFrameHeader + kReduceHeader + kSegmentFixed + name_len;
  g.full_frames = elems / g.max_elems;
  g.tail_elems = elems % g.max_elems;
  g.full_frame_bytes = g.header + g.max_elems * g.width;
  g.bytes = g.full_frames * g.full_frame_bytes + (g.tail_elems ? g.header + g.tail_elems * g.width : 0);
  return g;
}

void wire_encode_impl(const void* dev, uint64_t global_offset, uint64_t elems, const dlc_wire_tags* t,
                      uint8_t* host_out, size_t cap, size_t* used, cudaStream_t stream) {
  check_tags(t);
  if (t->msg_type < 1 || t->msg_type > 9) fail(DLC_ECONFIG, "wire: unknown message type");
  const std::string name = chunk_name(t->attempt, t->partition, t->from_hi, t->from_lo);
  const WireGeometry g = wire_geometry(elems, t, name.size());
  if (used) *used = g.bytes;
  if (!elems) return;
  if (!dev || !host_out) fail(DLC_EINVAL, "wire encode: null buffer");
  if (cap < g.bytes) fail(DLC_ESHAPE, "wire encode: output holds " + std::to_string(cap) + " bytes, frames need " +
                                          std::to_string(g.bytes));
  // scalars first (the copy engine runs while the host writes the headers)
  const uint8_t* src = static_cast<const uint8_t*>(dev);
  const size_t row = g.max_elems * g.width;
  if (g.full_frames)
    DLC_CUDA(cudaMemcpy2DAsync(host_out + g.header, g.full_frame_bytes, src, row, row, g.full_frames,
                               cudaMemcpyDeviceToHost, stream));
  if (g.tail_elems)
    DLC_CUDA(cudaMemcpyAsync(host_out + g.full_frames * g.full_frame_bytes + g.header, src + g.full_frames * row,
                             g.tail_elems * g.width, cudaMemcpyDeviceToHost, stream));
  const uint64_t frames = g.full_frames + (g.tail_elems ? 1 : 0);
  for (uint64_t i = 0; i < frames; ++i) {
    uint8_t* f = host_out + i * g.full_frame_bytes;
    const uint64_t count = i < g.full_frames ? g.max_elems : g.tail_elems;
    const uint64_t payload = kReduceHeader + kSegmentFixed + name.size() + count * g.width;
    std::memcpy(f, "ODLC", 4);
    f[4] = 1;  // kWireVersion, wire.hpp:27
    f[5] = t->msg_type;
    put_le(f + 6, payload, 8);
    uint8_t* p = f + kFrameHeader;
    put_le(p, t->outer_epoch, 8);
    put_le(p + 8, static_cast<uint32_t>(i), 4);  // chunk_index counts from 0 per call (:1328, :1336)
    p[12] = t->precision == DLC_FP16 ? 1 : 0;
    uint8_t* s = p + kReduceHeader;
    put_le(s, 1, 8);
    put_le(s + 8, name.size(), 8);
    std::memcpy(s + 16, name.data(), name.size());
    put_le(s + 16 + name.size(), global_offset + i * g.max_elems, 8);
    put_le(s + 24 + name.size(), count, 8);
  }
  DLC_CUDA(cudaStreamSynchronize(stream));
}

void wire_decode_impl(const uint8_t* in, size_t bytes, int precision, uint64_t base, uint64_t capacity, void* dev_out,
                      dlc_wire_chunk* chunks, size_t max_chunks, size_t* n_chunks, size_t* consumed,
                      cudaStream_t stream) {
  if (precision != DLC_FP32 && precision != DLC_FP16) fail(DLC_ECONFIG, "wire: unknown precision");
  if (bytes && !in) fail(DLC_EINVAL, "wire decode: null input");
  const size_t w = width_of(precision);
  uint8_t* dst = static_cast<uint8_t*>(dev_out);
  size_t at = 0, count = 0;
  bool copied = false;  // header-only work (all dropped / errors) never touches the device
  // pending strided run of accepted chunks: equal sizes, equal source spacing,
  // destinations back to back
  struct Run {
    const uint8_t* src = nullptr;
    size_t spitch = 0, bytes = 0, rows = 0;
    uint64_t dst_elem = 0;
  } run;
  auto flush = [&] {
    if (!run.rows) return;
    copied = true;
    if (run.rows == 1)
      DLC_CUDA(cudaMemcpyAsync(dst + run.dst_elem * w, run.src, run.bytes, cudaMemcpyHostToDevice, stream));
    else
      DLC_CUDA(cudaMemcpy2DAsync(dst + run.dst_elem * w, run.bytes, run.src, run.spitch, run.bytes, run.rows,
                                 cudaMemcpyHostToDevice, stream));
    run = Run{};
  };
  auto add = [&](const uint8_t* src, size_t nbytes, uint64_t dst_elem) {
    if (run.rows) {
      const bool same = nbytes == run.bytes && dst_elem == run.dst_elem + run.rows * (run.bytes / w) &&
                        (run.rows == 1 ? src > run.src : src == run.src + run.rows * run.spitch);
      if (same) {
        if (run.rows == 1) run.spitch = static_cast<size_t>(src - run.src);
        run.rows += 1;
        return;
      }
      flush();
    }
    run.src = src;
    run.bytes = nbytes;
    run.rows = 1;
    run.dst_elem = dst_elem;
  };
  auto done = [&] {
    flush();
    if (copied) DLC_CUDA(cudaStreamSynchronize(stream));
    if (n_chunks) *n_chunks = count;
    if (consumed) *consumed = at;
  };
  try {
    while (bytes - at >= kFrameHeader) {  // FrameParser::next, wire.cpp:38-72
      const uint8_t* f = in + at;
      if (std::memcmp(f, "ODLC", 4) != 0) fail(DLC_ESERIAL, "bad frame magic");
      if (f[4] != 1) fail(DLC_ESERIAL, "unsupported wire version " + std::to_string(f[4]));
      const uint64_t len = get_le(f + 6, 8);
      if (len > (1ull << 33)) fail(DLC_ESERIAL, "implausible frame length");
      if (bytes - at < kFrameHeader + len) break;  // incomplete: wait for more bytes
      const uint8_t type = f[5];
      if (type < 1 || type > 9) fail(DLC_ESERIAL, "unknown message type " + std::to_string(type));
      dlc_wire_chunk c{};
      c.msg_type = type;
      c.frame_offset = at;
      c.frame_bytes = kFrameHeader + len;
      if (type == DLC_MSG_REDUCE_CHUNK || type == DLC_MSG_REDUCE_RESULT) {
        const uint8_t* p = f + kFrameHeader;
        if (len < kReduceHeader) fail(DLC_ESERIAL, "truncated reduce payload");  // wire.cpp:92-94
        c.outer_epoch = get_le(p, 8);
        c.chunk_index = static_cast<uint32_t>(get_le(p + 8, 4));
        c.precision = p[12];
        // decode_chunk_segment, collective.cpp:90-118
        const uint8_t* s = p + kReduceHeader;
        const uint64_t slen = len - kReduceHeader;
        if (slen < 8) fail(DLC_ESERIAL, "truncated chunk segment");
        if (get_le(s, 8) != 1) fail(DLC_ESERIAL, "chunk segment must hold exactly one segment");
        if (slen < 16) fail(DLC_ESERIAL, "truncated chunk segment");
        const uint64_t nl = get_le(s + 8, 8);
        if (nl > slen - 16) fail(DLC_ESERIAL, "truncated chunk segment name");
        if (slen - 16 - nl < 16) fail(DLC_ESERIAL, "truncated chunk segment");
        const std::string name(reinterpret_cast<const char*>(s + 16), nl);
        c.offset = get_le(s + 16 + nl, 8);
        c.length = get_le(s + 24 + nl, 8);
        const uint8_t* scalars = s + 32 + nl;
        const uint64_t sbytes = slen - 32 - nl;
        // handle_reduce_chunk's drops (collective.cpp:1022-1029), then this
        // buffer's own: precision and range
        const uint64_t cw = c.precision == 1 ? 2 : 4;
        const bool named = parse_chunk_name(name, &c.attempt, &c.partition, &c.from_hi, &c.from_lo);
        const bool sized = c.length <= (UINT64_MAX / cw) && sbytes == c.length * cw;
        const bool prec_ok = c.precision == (precision == DLC_FP16 ? 1 : 0);
        const bool in_range = c.offset >= base && c.offset - base <= capacity && c.length <= capacity - (c.offset - base);
        if (named && sized && prec_ok && in_range) {
          c.accepted = 1;
          if (c.length) {
            if (!dev_out) fail(DLC_EINVAL, "wire decode: null device buffer");
            add(scalars, sbytes, c.offset - base);
          }
        }
      }
      if (chunks && count < max_chunks) chunks[count] = c;
      ++count;
      at += kFrameHeader + len;
    }
  } catch (...) {
    done();
    throw;
  }
  done();
}

}  // namespace dlc

extern "C" {

int dlc_wire_frames_size(uint64_t elems, const dlc_wire_tags* tags, size_t* bytes, uint64_t* frames) {
  return guard([&] {
    check_tags(tags);
    const std::string name = chunk_name(tags->attempt, tags->partition, tags->from_hi, tags->from_lo);
    const WireGeometry g = wire_geometry(elems, tags, name.size());
    if (bytes) *bytes = g.bytes;
    if (frames) *frames = g.full_frames + (g.tail_elems ? 1 : 0);
  });
}

int dlc_wire_encode(const void* dev_scalars, uint64_t global_offset, uint64_t elems, const dlc_wire_tags* tags,
                    uint8_t* host_out, size_t cap, size_t* used, void* stream) {
  return guard([&] {
    wire_encode_impl(dev_scalars, global_offset, elems, tags, host_out, cap, used,
                     static_cast<cudaStream_t>(stream));
  });
}

int dlc_wire_decode(const uint8_t* host_in, size_t bytes, int precision, uint64_t base_offset, uint64_t capacity,
                    void* dev_out, dlc_wire_chunk* chunks, size_t max_chunks, size_t* n_chunks, size_t* consumed,
                    void* stream) {
  return guard([&] {
    wire_decode_impl(host_in, bytes, precision, base_offset, capacity, dev_out, chunks, max_chunks, n_chunks,
                     consumed, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
