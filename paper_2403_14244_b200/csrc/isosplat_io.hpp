// isosplat_io.hpp — the reference's scene / camera file formats for the C++ drop-in
// (/root/reference/proj/include/isosplat/particle_io.hpp:18-57, src/particle_io.cpp:151-298),
// so the reference's render3d flow (tools/isosplat_main.cpp:357-398: load_particles ->
// load_camera -> render -> write_png) runs on the B200 path unchanged.
//
// The reference parses JSON with nlohmann-json, which is not available here; a small reader
// for the subset these files use (objects, arrays, numbers, strings, booleans, null) is
// included.  Errors are std::runtime_error with the reference's messages; an invalid camera
// throws std::domain_error from Camera::validate.  Only isotropic 3D sets are materialised.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "isosplat_b200.hpp"

namespace isosplat {

// ---- minimal JSON -----------------------------------------------------------------------
namespace json {

// JSON syntax / access errors (nlohmann::json::exception in the reference).
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Value {
  enum Type { Null, Bool, Number, String, Array, Object } type = Null;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;

  bool contains(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return true;
    return false;
  }
  const Value& at(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return kv.second;
    throw Error("json: missing key '" + k + "'");
  }
  const Value& at(std::size_t i) const {
    if (type != Array || i >= arr.size()) throw Error("json: index out of range");
    return arr[i];
  }
  std::size_t size() const { return type == Array ? arr.size() : obj.size(); }
  double number() const {
    if (type != Number) throw Error("json: expected a number");
    return num;
  }
  const std::string& string() const {
    if (type != String) throw Error("json: expected a string");
    return str;
  }
};

class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}
  Value parse() {
    Value v = value();
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  std::size_t i_ = 0;
  [[noreturn]] void fail(const char* what) {
    throw Error(std::string("json parse error at ") + std::to_string(i_) + ": " + what);
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\r' || s_[i_] == '\t')) ++i_;
  }
  bool lit(const char* w) {
    const std::size_t n = std::strlen(w);
    if (s_.compare(i_, n, w) == 0) {
      i_ += n;
      return true;
    }
    return false;
  }
  std::string str() {
    if (s_[i_] != '"') fail("expected string");
    ++i_;
    std::string out;
    while (i_ < s_.size() && s_[i_] != '"') {
      char c = s_[i_++];
      if (c == '\\') {
        if (i_ >= s_.size()) fail("bad escape");
        char e = s_[i_++];
        switch (e) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (i_ + 4 > s_.size()) fail("bad \\u escape");
            const unsigned cp = (unsigned)std::stoul(s_.substr(i_, 4), nullptr, 16);
            i_ += 4;
            if (cp < 0x80) out += (char)cp;
            else if (cp < 0x800) { out += (char)(0xC0 | (cp >> 6)); out += (char)(0x80 | (cp & 0x3F)); }
            else { out += (char)(0xE0 | (cp >> 12)); out += (char)(0x80 | ((cp >> 6) & 0x3F)); out += (char)(0x80 | (cp & 0x3F)); }
            break;
          }
          default: out += e;
        }
      } else {
        out += c;
      }
    }
    if (i_ >= s_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
  Value value() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end");
    Value v;
    const char c = s_[i_];
    if (c == '{') {
      v.type = Value::Object;
      ++i_;
      ws();
      if (s_[i_] == '}') { ++i_; return v; }
      while (true) {
        ws();
        std::string k = str();
        ws();
        if (s_[i_] != ':') fail("expected ':'");
        ++i_;
        v.obj.emplace_back(std::move(k), value());
        ws();
        if (s_[i_] == ',') { ++i_; continue; }
        if (s_[i_] == '}') { ++i_; break; }
        fail("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.type = Value::Array;
      ++i_;
      ws();
      if (s_[i_] == ']') { ++i_; return v; }
      while (true) {
        v.arr.push_back(value());
        ws();
        if (s_[i_] == ',') { ++i_; continue; }
        if (s_[i_] == ']') { ++i_; break; }
        fail("expected ',' or ']'");
      }
    } else if (c == '"') {
      v.type = Value::String;
      v.str = str();
    } else if (lit("true")) {
      v.type = Value::Bool;
      v.b = true;
    } else if (lit("false")) {
      v.type = Value::Bool;
    } else if (lit("null")) {
      v.type = Value::Null;
    } else {
      char* end = nullptr;
      v.type = Value::Number;
      v.num = std::strtod(s_.c_str() + i_, &end);
      if (end == s_.c_str() + i_) fail("unexpected character");
      i_ = (std::size_t)(end - s_.c_str());
    }
    return v;
  }
};

inline Value parse(const std::string& s) { return Parser(s).parse(); }

inline void dump_number(std::ostringstream& o, double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  o << buf;
}
}  // namespace json

// ---- particle sets (iso 3D) -----------------------------------------------------------------
struct ParticleSet {
  int format_version = 1;
  std::string kind = "iso";
  int dimension = 3;
  int channels = 3;
  std::vector<IsoSplat3D> iso3d;
  std::string metadata_json = "{}";  // raw JSON object, passed through
  std::size_t count() const { return iso3d.size(); }
  int values_per_record() const {  // particle_io.cpp:32-35
    if (dimension == 2) return (kind == "iso" ? 3 : 5) + channels;
    return kind == "iso" ? 8 : 14;
  }
};

namespace detail {
inline std::string header_json(const ParticleSet& s) {
  std::ostringstream o;
  o << "{\"version\":" << s.format_version << ",\"kernel_kind\":\"" << s.kind
    << "\",\"dimension\":" << s.dimension << ",\"channels\":" << s.channels
    << ",\"count\":" << s.count() << ",\"metadata\":" << s.metadata_json << "}";
  return o.str();
}

inline std::size_t set_from_header(const json::Value& h, ParticleSet& s) {  // :128-147
  s.format_version = (int)h.at("version").number();
  if (s.format_version != 1)
    throw std::runtime_error("unknown particle file version " + std::to_string(s.format_version));
  s.kind = h.at("kernel_kind").string();
  if (s.kind != "iso" && s.kind != "aniso") throw std::runtime_error("unknown kernel_kind: " + s.kind);
  s.dimension = (int)h.at("dimension").number();
  if (s.dimension != 2 && s.dimension != 3)
    throw std::runtime_error("particle file: dimension must be 2 or 3");
  s.channels = (int)h.at("channels").number();
  if (s.channels != 1 && s.channels != 3)
    throw std::runtime_error("particle file: channels must be 1 or 3");
  return (std::size_t)h.at("count").number();
}

inline void fill_iso3d(ParticleSet& s, const std::vector<double>& v, std::size_t count) {
  if (s.kind != "iso" || s.dimension != 3)
    throw std::runtime_error("scene file must hold isotropic 3D splats (kernel_kind=iso, dimension=3)");
  s.iso3d.resize(count);
  for (std::size_t i = 0; i < count; ++i) {
    const double* p = v.data() + 8 * i;
    s.iso3d[i].mu = {p[0], p[1], p[2]};
    s.iso3d[i].sigma = p[3];
    s.iso3d[i].color = {p[4], p[5], p[6]};
    s.iso3d[i].opacity = p[7];
  }
}
}  // namespace detail

// save_particles, particle_io.cpp:151-182 (iso 3D)
inline void save_particles(const std::string& path, const ParticleSet& s, bool as_json = false) {
  std::vector<double> v;
  v.reserve(8 * s.count());
  for (const auto& p : s.iso3d)
    for (double x : {p.mu[0], p.mu[1], p.mu[2], p.sigma, p.color[0], p.color[1], p.color[2], p.opacity})
      v.push_back(x);
  if (as_json) {
    std::ostringstream o;
    std::string h = detail::header_json(s);
    h.pop_back();
    o << h << ",\"format\":\"ISPL-json\",\"particles\":[";
    for (std::size_t i = 0; i < s.count(); ++i) {
      o << (i ? ",[" : "[");
      for (int k = 0; k < 8; ++k) {
        if (k) o << ",";
        json::dump_number(o, v[8 * i + k]);
      }
      o << "]";
    }
    o << "]}\n";
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot write particle file: " + path);
    out << o.str();
    return;
  }
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write particle file: " + path);
  const std::string header = detail::header_json(s);
  const uint32_t len = (uint32_t)header.size();
  out.write("ISPL", 4);
  out.write(reinterpret_cast<const char*>(&len), 4);  // little endian host (documented format)
  out.write(header.data(), (std::streamsize)header.size());
  out.write(reinterpret_cast<const char*>(v.data()), (std::streamsize)(v.size() * sizeof(double)));
  if (!out) throw std::runtime_error("short write: " + path);
}

// load_particles, particle_io.cpp:184-236
inline ParticleSet load_particles(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open particle file: " + path);
  std::string data((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  ParticleSet s;
  if (data.size() >= 4 && data.compare(0, 4, "ISPL") == 0) {
    if (data.size() < 8) throw std::runtime_error("truncated particle file: " + path);
    uint32_t len = 0;
    std::memcpy(&len, data.data() + 4, 4);
    if (data.size() < 8ull + len) throw std::runtime_error("truncated particle file: " + path);
    const std::size_t count = detail::set_from_header(json::parse(data.substr(8, len)), s);
    const std::size_t nbytes = count * (std::size_t)s.values_per_record() * sizeof(double);
    if (data.size() < 8ull + len + nbytes) throw std::runtime_error("truncated particle file: " + path);
    std::vector<double> v(count * (std::size_t)s.values_per_record());
    std::memcpy(v.data(), data.data() + 8 + len, nbytes);
    detail::fill_iso3d(s, v, count);
    return s;
  }
  json::Value j;
  try {
    j = json::parse(data);
  } catch (const json::Error&) {
    throw std::runtime_error("unrecognized particle file format: " + path);
  }
  if (j.type != json::Value::Object || !j.contains("format") ||
      j.at("format").type != json::Value::String || j.at("format").str != "ISPL-json")
    throw std::runtime_error("unrecognized particle file format: " + path);
  const std::size_t count = detail::set_from_header(j, s);
  const json::Value& recs = j.at("particles");
  if (recs.size() != count) throw std::runtime_error("particle file: count mismatch");
  std::vector<double> v;
  for (const auto& r : recs.arr) {
    if ((int)r.size() != s.values_per_record()) throw std::runtime_error("particle file: bad record arity");
    for (const auto& x : r.arr) v.push_back(x.number());
  }
  detail::fill_iso3d(s, v, count);
  return s;
}

// camera_from_json, particle_io.cpp:238-268
inline Camera camera_from_json(const json::Value& j) {
  Camera cam;
  if (j.contains("rotation")) {
    const auto& r = j.at("rotation");
    if (r.size() != 3) throw std::runtime_error("camera: rotation must be 3 rows");
    for (int i = 0; i < 3; ++i)
      for (int k = 0; k < 3; ++k) cam.rotation(i, k) = r.at(i).at(k).number();
  } else if (j.contains("quaternion")) {
    const auto& q = j.at("quaternion");
    if (q.size() != 4) throw std::runtime_error("camera: quaternion must be [w,x,y,z]");
    const double w = q.at(0).number(), x = q.at(1).number(), y = q.at(2).number(), z = q.at(3).number();
    if (std::abs(std::sqrt(w * w + x * x + y * y + z * z) - 1.0) > 1e-9)
      throw std::runtime_error("camera: quaternion norm must be 1 within 1e-9");
    const double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)},
                            {2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)},
                            {2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)}};
    for (int i = 0; i < 3; ++i)
      for (int k = 0; k < 3; ++k) cam.rotation(i, k) = R[i][k];
  } else {
    throw std::runtime_error("camera: missing rotation or quaternion");
  }
  const auto& t = j.at("translation");
  for (int i = 0; i < 3; ++i) cam.translation[i] = t.at(i).number();
  cam.focal = j.at("focal").number();
  const auto& pp = j.at("principal_point");
  cam.principal_point = {pp.at(0).number(), pp.at(1).number()};
  const auto& size = j.at("image_size");
  cam.width = (int)size.at(0).number();
  cam.height = (int)size.at(1).number();
  cam.validate();
  return cam;
}

inline Camera load_camera(const std::string& path) {  // particle_io.cpp:270-284
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open camera file: " + path);
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  json::Value j;
  try {
    j = json::parse(text);
  } catch (const json::Error& e) {
    throw std::runtime_error("camera JSON parse error in " + path + ": " + e.what());
  }
  try {
    return camera_from_json(j);
  } catch (const json::Error& e) {
    throw std::runtime_error("camera JSON field error in " + path + ": " + e.what());
  }
}

// write_loss_csv, particle_io.cpp:286-298
inline void write_loss_csv(const std::string& path, double initial_loss, int initial_count,
                           const std::vector<double>& loss_history,
                           const std::vector<int>& count_history) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write csv: " + path);
  out << "epoch,loss,particles\n";
  out.precision(17);
  out << 0 << "," << initial_loss << "," << initial_count << "\n";
  for (std::size_t i = 0; i < loss_history.size(); ++i)
    out << (i + 1) << "," << loss_history[i] << ","
        << (i < count_history.size() ? count_history[i] : initial_count) << "\n";
}

// 8-bit RGB PNG with the reference's quantisation (clamp, round half up: png_io.hpp:17-21),
// zlib "stored" blocks so no compression library is needed.
inline void write_png(const std::string& path, const ImageGrid& img) {
  auto crc32 = [](const unsigned char* p, std::size_t n, uint32_t c) {
    static uint32_t table[256];
    static bool init = false;
    if (!init) {
      for (uint32_t i = 0; i < 256; ++i) {
        uint32_t r = i;
        for (int k = 0; k < 8; ++k) r = (r & 1) ? 0xEDB88320u ^ (r >> 1) : r >> 1;
        table[i] = r;
      }
      init = true;
    }
    c = ~c;
    for (std::size_t i = 0; i < n; ++i) c = table[(c ^ p[i]) & 0xFF] ^ (c >> 8);
    return ~c;
  };
  std::vector<unsigned char> raw;
  raw.reserve((std::size_t)img.height * (1 + 3 * img.width));
  for (int y = 0; y < img.height; ++y) {
    raw.push_back(0);
    for (int x = 0; x < img.width; ++x)
      for (int c = 0; c < 3; ++c) {
        const double v = img.at(x, y, img.channels == 3 ? c : 0);
        raw.push_back((unsigned char)std::floor(std::fmin(std::fmax(v, 0.0), 1.0) * 255.0 + 0.5));
      }
  }
  std::vector<unsigned char> z = {0x78, 0x01};
  uint32_t a = 1, b = 0;
  for (unsigned char ch : raw) {
    a = (a + ch) % 65521;
    b = (b + a) % 65521;
  }
  for (std::size_t off = 0; off < raw.size() || off == 0; off += 65535) {
    const std::size_t n = std::min<std::size_t>(65535, raw.size() - off);
    const bool last = off + n >= raw.size();
    z.push_back(last ? 1 : 0);
    z.push_back(n & 0xFF);
    z.push_back(n >> 8);
    z.push_back(~n & 0xFF);
    z.push_back((~n >> 8) & 0xFF);
    z.insert(z.end(), raw.begin() + off, raw.begin() + off + n);
    if (last) break;
  }
  const uint32_t adler = (b << 16) | a;
  for (int s = 24; s >= 0; s -= 8) z.push_back((adler >> s) & 0xFF);
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write png: " + path);
  auto be32 = [&](uint32_t v) {
    const unsigned char b4[4] = {(unsigned char)(v >> 24), (unsigned char)(v >> 16),
                                 (unsigned char)(v >> 8), (unsigned char)v};
    out.write(reinterpret_cast<const char*>(b4), 4);
  };
  auto chunk = [&](const char* tag, const std::vector<unsigned char>& d) {
    be32((uint32_t)d.size());
    std::vector<unsigned char> td(tag, tag + 4);
    td.insert(td.end(), d.begin(), d.end());
    out.write(reinterpret_cast<const char*>(td.data()), (std::streamsize)td.size());
    be32(crc32(td.data(), td.size(), 0));
  };
  out.write("\x89PNG\r\n\x1a\n", 8);
  std::vector<unsigned char> ihdr = {0, 0, 0, 0, 0, 0, 0, 0, 8, 2, 0, 0, 0};
  for (int i = 0; i < 4; ++i) {
    ihdr[i] = (unsigned char)(img.width >> (24 - 8 * i));
    ihdr[4 + i] = (unsigned char)(img.height >> (24 - 8 * i));
  }
  chunk("IHDR", ihdr);
  chunk("IDAT", z);
  chunk("IEND", {});
}

}  // namespace isosplat
