// Drop-in host API (namespace pact::io) — binary raster and signal files.
//
// Same functions, formats and error messages as the reference's
// proj/include/pact/io.hpp (write_pgrid 80-91, read_pgrid 93-112,
// write_sigset 114-127, read_sigset 129-150).  Both formats are little-endian
// with a 4-byte magic and f32 payloads:
//
//   PGRID  "PGRD" u32 width, u32 height, f64 pitch_mm, f64 origin_x_mm,
//          f64 origin_y_mm, then width*height f32 (row-major)
//   SIGSET "SIGS" u32 N_t, u32 n_samples, f64 dt_s, f64 t0_s, f64 ring_radius_mm,
//          f64 angle_offset_rad, f64 background_sos_mps, then N_t*n_samples f32
//          (transducer-major)
//
// Implementation: a file is encoded into / decoded from one in-memory byte
// image (one write, one read), and the decoder walks a field cursor that
// reports the first field a truncated file cuts, exactly as the reference's
// field-by-field reads do.  Host-only; no device work.
#ifndef PACT_B200_IO_HPP
#define PACT_B200_IO_HPP

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pact/core.hpp"

namespace pact::io {

#if defined(__BYTE_ORDER__) && __BYTE_ORDER__ != __ORDER_LITTLE_ENDIAN__
#error "file I/O assumes a little-endian host"
#endif

namespace detail {

/// Byte image being encoded.
struct Encoder {
  std::vector<unsigned char> bytes;
  void raw(const void* p, size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    bytes.insert(bytes.end(), b, b + n);
  }
  template <typename T>
  void put(T v) {
    raw(&v, sizeof(T));
  }
  void put_f32_array(const std::vector<double>& v) {
    const size_t at = bytes.size();
    bytes.resize(at + 4 * v.size());
    for (size_t i = 0; i < v.size(); ++i) {
      const float f = static_cast<float>(v[i]);
      std::memcpy(bytes.data() + at + 4 * i, &f, 4);
    }
  }
  void save(const std::string& path) const {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw ValidationError("cannot open for writing: " + path);
    const size_t n = std::fwrite(bytes.data(), 1, bytes.size(), f);
    const bool ok = n == bytes.size() && std::fflush(f) == 0;
    std::fclose(f);
    if (!ok) throw ValidationError("write failed: " + path);
  }
};

/// Cursor over a file's bytes; every read names its field for the
/// truncation message.
struct Decoder {
  std::string path;
  std::vector<unsigned char> bytes;
  size_t pos = 0;

  explicit Decoder(const std::string& p) : path(p) {
    std::FILE* f = std::fopen(p.c_str(), "rb");
    if (!f) throw ValidationError("cannot open for reading: " + p);
    unsigned char buf[1 << 16];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) bytes.insert(bytes.end(), buf, buf + n);
    std::fclose(f);
  }
  void magic(const char* m) {
    if (bytes.size() < 4 || std::memcmp(bytes.data(), m, 4) != 0)
      throw ValidationError("bad magic in " + path + " (expected " + m + ")");
    pos = 4;
  }
  template <typename T>
  T get(const char* field) {
    if (bytes.size() - pos < sizeof(T))
      throw ValidationError("truncated file while reading " + path + " " + field);
    T v;
    std::memcpy(&v, bytes.data() + pos, sizeof(T));
    pos += sizeof(T);
    return v;
  }
  /// n f32 values widened to f64; `bad` is the message for a non-finite one.
  /// (Values before a truncation are checked first, as the reference's
  /// value-by-value reads do; nothing is allocated beyond the file.)
  std::vector<double> f32_array(size_t n, const char* field, const std::string& bad) {
    const size_t avail = (bytes.size() - pos) / 4, m = n < avail ? n : avail;
    std::vector<double> out(m);
    for (size_t i = 0; i < m; ++i) {
      float v;
      std::memcpy(&v, bytes.data() + pos + 4 * i, 4);
      if (!std::isfinite(v)) throw ValidationError(bad);
      out[i] = v;
    }
    if (m < n) throw ValidationError("truncated file while reading " + path + " " + field);
    pos += 4 * n;
    return out;
  }
};

}  // namespace detail

inline void write_pgrid(const std::string& path, const RasterGrid& g) {
  g.spec().validate();
  detail::Encoder e;
  e.raw("PGRD", 4);
  e.put<uint32_t>(static_cast<uint32_t>(g.width));
  e.put<uint32_t>(static_cast<uint32_t>(g.height));
  e.put<double>(g.pitch);
  e.put<double>(g.origin.x);
  e.put<double>(g.origin.y);
  e.put_f32_array(g.values);
  e.save(path);
}

inline RasterGrid read_pgrid(const std::string& path) {
  detail::Decoder d(path);
  d.magic("PGRD");
  RasterGrid g;
  g.width = static_cast<int>(d.get<uint32_t>("width"));
  g.height = static_cast<int>(d.get<uint32_t>("height"));
  g.pitch = d.get<double>("pitch");
  g.origin.x = d.get<double>("origin_x");
  g.origin.y = d.get<double>("origin_y");
  g.spec().validate();
  g.values = d.f32_array(static_cast<size_t>(g.width) * g.height, "values",
                         "non-finite value in " + path);
  return g;
}

inline void write_sigset(const std::string& path, const SignalSet& s) {
  s.validate();
  detail::Encoder e;
  e.raw("SIGS", 4);
  e.put<uint32_t>(static_cast<uint32_t>(s.geom.n_transducers));
  e.put<uint32_t>(static_cast<uint32_t>(s.n_samples));
  e.put<double>(s.dt);
  e.put<double>(s.t0);
  e.put<double>(s.geom.radius);
  e.put<double>(s.geom.angle_offset);
  e.put<double>(s.background_sos);
  e.put_f32_array(s.data);
  e.save(path);
}

inline SignalSet read_sigset(const std::string& path) {
  detail::Decoder d(path);
  d.magic("SIGS");
  SignalSet s;
  s.geom.n_transducers = static_cast<int>(d.get<uint32_t>("N_t"));
  s.n_samples = static_cast<int>(d.get<uint32_t>("n_samples"));
  s.dt = d.get<double>("dt");
  s.t0 = d.get<double>("t0");
  s.geom.radius = d.get<double>("ring_radius");
  s.geom.angle_offset = d.get<double>("angle_offset");
  s.background_sos = d.get<double>("background_sos");
  if (!(s.background_sos > 0.0)) throw ValidationError("non-positive SOS in " + path);
  s.data = d.f32_array(static_cast<size_t>(s.geom.n_transducers) * s.n_samples, "data",
                       "non-finite sample in " + path);
  s.validate();
  return s;
}

}  // namespace pact::io

#endif  // PACT_B200_IO_HPP
