// io.cpp — scene I/O of the C ABI (include/odgs_b200.h "scene I/O"): the reference's
// polygon point clouds and checkpoints (reference src/io.cpp:1-362, io.hpp).
//
// Host code by nature (file formats); it reads into / writes from plain binary64
// column-major arrays so an Eigen caller passes .data(). Behaviour mirrors the
// reference line by line where a caller can observe it: accepted header grammar,
// property types, value conversion, the first error and its message (with the byte
// offset where the reference reports one), and the exact bytes written.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "odgs_b200.h"

namespace {

thread_local std::string g_io_error;

constexpr double kSh0 = 0.28209479177387814;  // io.hpp:14
constexpr int kCheckpointVersion = 1;         // io.hpp:19
const char* const kCheckpointFields[14] = {"x",       "y",       "z",       "f_dc_0", "f_dc_1",
                                           "f_dc_2",  "opacity", "scale_0", "scale_1", "scale_2",
                                           "rot_0",   "rot_1",   "rot_2",   "rot_3"};

// std::runtime_error "<path>: <what>[ (byte N)]" (io.cpp:23-30).
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
[[noreturn]] void fail(const std::string& path, const std::string& what) { throw IoError(path + ": " + what); }
[[noreturn]] void fail_at(const std::string& path, const std::string& what, std::streamoff byte) {
  fail(path, what + " (byte " + std::to_string(byte) + ")");
}

// Bytes per value of a vertex property type; 0 for unsupported (io.cpp:32-37).
int type_bytes(const std::string& t) {
  if (t == "float" || t == "float32") return 4;
  if (t == "double" || t == "float64") return 8;
  if (t == "uchar" || t == "uint8") return 1;
  return 0;
}

struct Property {
  std::string type, name;
  int bytes;
};

// The vertex element of a polygon file: header grammar of parse_ply_header
// (io.cpp:41-118) and the column reader of read_ply (io.cpp:141-199).
class PolygonFile {
 public:
  explicit PolygonFile(const std::string& path) : path_(path), in_(path, std::ios::binary) {
    if (!in_) fail(path_, "cannot open file");
    parse_header();
  }

  int64_t vertex_count() const { return count_; }
  const std::vector<std::string>& comments() const { return comments_; }

  // Reads every vertex into one binary64 column per distinct property name (a
  // repeated name keeps its first column and later ones overwrite its values, as the
  // reference's map::emplace does).
  void read_columns() {
    std::vector<std::vector<double>*> dst;
    for (const Property& p : props_) {
      auto it = columns_.find(p.name);
      if (it == columns_.end()) it = columns_.emplace(p.name, std::vector<double>((size_t)count_)).first;
      dst.push_back(&it->second);
    }
    if (binary_) {
      std::vector<char> row((size_t)stride_);
      for (int64_t v = 0; v < count_; ++v) {
        const std::streamoff at = data_start_ + std::streamoff(v) * stride_;
        if (!in_.read(row.data(), stride_)) fail_at(path_, "truncated vertex data", at);
        size_t o = 0;
        for (size_t k = 0; k < props_.size(); ++k) {
          (*dst[k])[(size_t)v] = decode(props_[k].bytes, row.data() + o);
          o += (size_t)props_[k].bytes;
        }
      }
    } else {
      std::string line;
      for (int64_t v = 0; v < count_; ++v) {
        const std::streamoff at = in_.tellg();
        if (!std::getline(in_, line)) fail_at(path_, "truncated vertex data", at);
        std::istringstream fields(line);
        for (size_t k = 0; k < props_.size(); ++k) {
          double x;
          if (!(fields >> x)) fail_at(path_, "malformed vertex line", at);
          (*dst[k])[(size_t)v] = x;
        }
      }
    }
  }

  const std::vector<double>& column(const std::string& name) const {
    auto it = columns_.find(name);
    if (it == columns_.end()) throw IoError(path_ + ": missing required property '" + name + "'");
    return it->second;
  }

  bool byte_valued(const std::string& name) const {
    for (const Property& p : props_)
      if (p.name == name) return p.type == "uchar" || p.type == "uint8";
    return false;
  }

 private:
  static double decode(int bytes, const char* at) {
    if (bytes == 4) {
      float f;
      std::memcpy(&f, at, 4);
      return f;
    }
    if (bytes == 8) {
      double d;
      std::memcpy(&d, at, 8);
      return d;
    }
    return (double)static_cast<unsigned char>(*at);
  }

  void parse_header() {
    std::string line;
    std::streamoff at = in_.tellg();
    if (!std::getline(in_, line) || line != "ply") fail_at(path_, "not a polygon file (missing 'ply' magic)", at);
    bool have_format = false, in_vertex = false;
    for (;;) {
      at = in_.tellg();
      if (!std::getline(in_, line)) fail_at(path_, "header ended before 'end_header'", at);
      std::istringstream words(line);
      std::string key;
      words >> key;
      if (key.empty() || key == "comment" || key == "obj_info") {
        if (key == "comment") comments_.push_back(line.substr(line.find("comment") + 8));
        continue;
      }
      if (key == "format") {
        std::string kind, version;
        words >> kind >> version;
        if (kind == "ascii") binary_ = false;
        else if (kind == "binary_little_endian") binary_ = true;
        else fail_at(path_, "unsupported format '" + kind + "'", at);
        have_format = true;
      } else if (key == "element") {
        std::string name;
        long long count = 0;
        words >> name >> count;
        if (name == "vertex") {
          count_ = count;
          in_vertex = true;
        } else if (in_vertex) {
          in_vertex = false;  // a later element: vertices come first, read them and stop
        } else {
          fail_at(path_, "element '" + name + "' precedes the vertex element", at);
        }
      } else if (key == "property") {
        if (!in_vertex) continue;
        std::string type;
        words >> type;
        if (type == "list") fail_at(path_, "list properties are not supported on vertices", at);
        std::string name;
        words >> name;
        const int b = type_bytes(type);
        if (b == 0) fail_at(path_, "unsupported property type '" + type + "'", at);
        props_.push_back({type, name, b});
      } else if (key == "end_header") {
        break;
      } else {
        fail_at(path_, "unrecognized header line '" + line + "'", at);
      }
    }
    if (!have_format) fail(path_, "header has no format line");
    if (props_.empty()) fail(path_, "no vertex properties declared");
    data_start_ = in_.tellg();
    for (const Property& p : props_) stride_ += p.bytes;
  }

  std::string path_;
  std::ifstream in_;
  bool binary_ = false;
  int64_t count_ = 0;
  int stride_ = 0;
  std::streamoff data_start_ = 0;
  std::vector<Property> props_;
  std::vector<std::string> comments_;
  std::map<std::string, std::vector<double>> columns_;
};

template <class F>
odgs_status guarded(F&& body) {
  try {
    body();
    g_io_error.clear();
    return ODGS_OK;
  } catch (const std::invalid_argument& e) {
    g_io_error = e.what();
    return ODGS_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_io_error = e.what();
    return ODGS_ERR_RUNTIME;
  }
}

void require_count(const std::string& path, int64_t have, int64_t want) {
  if (have != want)
    throw std::invalid_argument(path + ": buffer holds " + std::to_string(want) + " rows, the file has " +
                                std::to_string(have));
}

void put_f32(std::ofstream& out, double v) {
  const float f = static_cast<float>(v);
  out.write(reinterpret_cast<const char*>(&f), 4);
}

// save_pointcloud's colour quantisation (io.cpp:238-241).
unsigned char colour_byte(double v) { return static_cast<unsigned char>(std::lround(std::clamp(v, 0.0, 1.0) * 255.0)); }

}  // namespace

extern "C" {

size_t odgs_io_last_error(char* message, size_t message_len) {
  if (message && message_len) {
    const size_t k = std::min(message_len - 1, g_io_error.size());
    std::memcpy(message, g_io_error.data(), k);
    message[k] = '\0';
  }
  return g_io_error.size();
}

odgs_status odgs_ply_vertex_count(const char* path, int64_t* n) {
  return guarded([&] {
    if (!path || !n) throw std::invalid_argument("odgs_ply_vertex_count: null argument");
    *n = PolygonFile(path).vertex_count();
  });
}

odgs_status odgs_load_pointcloud(const char* path, int64_t n, double* positions, double* colors) {
  return guarded([&] {
    if (!path || !positions || !colors) throw std::invalid_argument("odgs_load_pointcloud: null argument");
    PolygonFile f(path);
    f.read_columns();
    const int64_t m = f.vertex_count();
    if (m < 1) fail(path, "point cloud is empty");
    const char* xyz[3] = {"x", "y", "z"};
    const char* rgb[3] = {"red", "green", "blue"};
    std::vector<const std::vector<double>*> cols;
    for (const char* c : xyz) cols.push_back(&f.column(c));
    for (const char* c : rgb) cols.push_back(&f.column(c));
    require_count(path, m, n);
    for (int c = 0; c < 3; ++c) std::copy(cols[c]->begin(), cols[c]->end(), positions + c * n);
    for (int c = 0; c < 3; ++c) {
      const bool scaled = f.byte_valued(rgb[c]);
      const std::vector<double>& src = *cols[3 + c];
      for (int64_t i = 0; i < n; ++i) colors[c * n + i] = scaled ? src[(size_t)i] / 255.0 : src[(size_t)i];
    }
  });
}

odgs_status odgs_save_pointcloud(const char* path, int64_t n, const double* positions, const double* colors,
                                 int32_t binary) {
  return guarded([&] {
    if (!path || (n > 0 && (!positions || !colors))) throw std::invalid_argument("odgs_save_pointcloud: null argument");
    std::ofstream out(path, std::ios::binary);
    if (!out) fail(path, "cannot open file for writing");
    out.precision(17);
    out << "ply\n" << (binary ? "format binary_little_endian 1.0\n" : "format ascii 1.0\n") << "element vertex "
        << n << "\n"
        << "property float x\nproperty float y\nproperty float z\n"
        << "property uchar red\nproperty uchar green\nproperty uchar blue\n"
        << "end_header\n";
    for (int64_t i = 0; i < n; ++i) {
      if (binary) {
        for (int c = 0; c < 3; ++c) put_f32(out, positions[c * n + i]);
        for (int c = 0; c < 3; ++c) {
          const unsigned char b = colour_byte(colors[c * n + i]);
          out.write(reinterpret_cast<const char*>(&b), 1);
        }
      } else {
        for (int c = 0; c < 3; ++c) out << static_cast<float>(positions[c * n + i]) << " ";
        for (int c = 0; c < 3; ++c) out << int(colour_byte(colors[c * n + i])) << (c < 2 ? " " : "\n");
      }
    }
    if (!out) fail(path, "write failed");
  });
}

odgs_status odgs_save_checkpoint(const char* path, const odgs_cloud64* cloud) {
  return guarded([&] {
    if (!path || !cloud) throw std::invalid_argument("odgs_save_checkpoint: null argument");
    const int64_t n = cloud->n;
    std::ofstream out(path, std::ios::binary);
    if (!out) fail(path, "cannot open file for writing");
    out << "ply\nformat binary_little_endian 1.0\ncomment odgs_checkpoint_version " << kCheckpointVersion
        << "\nelement vertex " << n << "\n";
    for (const char* name : kCheckpointFields) out << "property float " << name << "\n";
    out << "end_header\n";
    for (int64_t i = 0; i < n; ++i) {
      for (int c = 0; c < 3; ++c) put_f32(out, cloud->means[c * n + i]);
      for (int c = 0; c < 3; ++c) {
        // Degree-zero coefficient, flushed to zero below 2^-27 (io.cpp:317-326).
        const float f_dc = static_cast<float>((cloud->colors[c * n + i] - 0.5) / kSh0);
        const float v = std::abs(f_dc) < 0x1p-27f ? 0.0f : f_dc;
        out.write(reinterpret_cast<const char*>(&v), 4);
      }
      put_f32(out, cloud->raw_opacities[i]);
      for (int c = 0; c < 3; ++c) put_f32(out, cloud->log_scales[c * n + i]);
      for (int c = 0; c < 4; ++c) put_f32(out, cloud->rotations[c * n + i]);
    }
    if (!out) fail(path, "write failed");
  });
}

odgs_status odgs_load_checkpoint(const char* path, const odgs_cloud64* cloud) {
  return guarded([&] {
    if (!path || !cloud) throw std::invalid_argument("odgs_load_checkpoint: null argument");
    PolygonFile f(path);
    f.read_columns();
    for (const std::string& comment : f.comments()) {
      std::istringstream words(comment);
      std::string tag;
      int version = 0;
      if (words >> tag >> version && tag == "odgs_checkpoint_version" && version > kCheckpointVersion)
        fail(path, "checkpoint version " + std::to_string(version) + " is newer than this build understands (" +
                       std::to_string(kCheckpointVersion) + ")");
    }
    const int64_t n = f.vertex_count();
    std::vector<const std::vector<double>*> cols;
    for (const char* name : kCheckpointFields) cols.push_back(&f.column(name));
    require_count(path, n, cloud->n);
    double* dst[14];
    for (int c = 0; c < 3; ++c) dst[c] = cloud->means + c * n;
    for (int c = 0; c < 3; ++c) dst[3 + c] = cloud->colors + c * n;
    dst[6] = cloud->raw_opacities;
    for (int c = 0; c < 3; ++c) dst[7 + c] = cloud->log_scales + c * n;
    for (int c = 0; c < 4; ++c) dst[10 + c] = cloud->rotations + c * n;
    for (int k = 0; k < 14; ++k) {
      const std::vector<double>& src = *cols[k];
      for (int64_t i = 0; i < n; ++i) dst[k][i] = (k >= 3 && k < 6) ? 0.5 + kSh0 * src[(size_t)i] : src[(size_t)i];
    }
  });
}

}  // extern "C"
