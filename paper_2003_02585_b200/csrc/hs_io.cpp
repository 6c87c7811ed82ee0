// On-disk formats of the reference, byte for byte:
//   HSVG velocity grid   include/helmsweep/media.hpp:22-27, src/media.cpp:58-100
//                        "HSVG", u32 version = 1, u32 dim, u32 n[3], f64 origin[3], f64 spacing[3],
//                        then f32 samples, axis 0 fastest; CSV fallback src/media.cpp:102-130
//   HSFD field dump      src/harness.cpp:32-83
//                        "HSFD", u32 version = 1, u32 dim, u32 n[3], i32 lo[3], f64 h[3],
//                        f64 origin[3], then complex128 values (re, im), axis 0 fastest
// Little-endian host layout, as the reference writes it. Errors use the reference's classes
// (DataError for I/O and content, ConfigError for size mismatches).
#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "helmsweep_b200.h"
#include "hs_common.hpp"

namespace hsb {
std::string& last_error_ref();
}

namespace {

using hsb::Error;

constexpr char kVelMagic[4] = {'H', 'S', 'V', 'G'};
constexpr char kFieldMagic[4] = {'H', 'S', 'F', 'D'};
constexpr std::uint32_t kVersion = 1;

template <class F>
int io_guarded(F&& fn) {
  try {
    fn();
    return HS_OK;
  } catch (const Error& e) {
    hsb::last_error_ref() = e.what();
    return e.code;
  } catch (const std::exception& e) {
    hsb::last_error_ref() = e.what();
    return HS_ERR_INTERNAL;
  }
}
using hsb::data_error;

struct Velocity {
  int dim = 2;
  int n[3] = {2, 2, 1};
  double origin[3] = {0, 0, 0}, spacing[3] = {1, 1, 0};
  std::vector<float> c;
  std::int64_t count() const {
    std::int64_t k = 1;
    for (int a = 0; a < dim; ++a) k *= n[a];
    return k;
  }
  void validate() const {  // VelocityGrid::validate, src/media.cpp:16-28
    if (dim != 2 && dim != 3) data_error("VelocityGrid: dim must be 2 or 3");
    for (int a = 0; a < dim; ++a) {
      if (n[a] < 2) data_error("VelocityGrid: need at least 2 samples per axis");
      if (spacing[a] <= 0.0) data_error("VelocityGrid: spacing must be positive");
    }
    if (static_cast<std::int64_t>(c.size()) != count()) data_error("VelocityGrid: sample count does not match dims");
    for (float v : c)
      if (!(v > 0.0f)) data_error("VelocityGrid: non-positive velocity sample");
  }
};

void export_velocity(const Velocity& g, int* dim, int n[3], double origin[3], double spacing[3], float* c,
                     std::int64_t cap, std::int64_t* count) {
  *dim = g.dim;
  for (int a = 0; a < 3; ++a) {
    n[a] = g.n[a];
    origin[a] = g.origin[a];
    spacing[a] = g.spacing[a];
  }
  *count = static_cast<std::int64_t>(g.c.size());
  if (c && cap >= *count) std::memcpy(c, g.c.data(), g.c.size() * sizeof(float));
}

}  // namespace

extern "C" {

int hs_read_velocity_grid(const char* path, int* dim, int n[3], double origin[3], double spacing[3], float* c,
                          int64_t cap, int64_t* count) {
  return io_guarded([&] {
    std::ifstream f(path, std::ios::binary);
    if (!f) data_error(std::string("read_velocity_grid: cannot open ") + path);
    char magic[4];
    f.read(magic, 4);
    if (!f || std::memcmp(magic, kVelMagic, 4) != 0) data_error(std::string("read_velocity_grid: bad magic in ") + path);
    std::uint32_t version = 0, d = 0, nn[3] = {0, 0, 0};
    f.read(reinterpret_cast<char*>(&version), 4);
    f.read(reinterpret_cast<char*>(&d), 4);
    f.read(reinterpret_cast<char*>(nn), 12);
    if (version != kVersion) data_error("read_velocity_grid: unsupported version");
    Velocity g;
    g.dim = static_cast<int>(d);
    for (int a = 0; a < 3; ++a) g.n[a] = static_cast<int>(nn[a]);
    f.read(reinterpret_cast<char*>(g.origin), 24);
    f.read(reinterpret_cast<char*>(g.spacing), 24);
    if (g.dim != 2 && g.dim != 3) data_error("read_velocity_grid: bad dim");
    const std::int64_t k = g.count();
    if (k <= 0) data_error("read_velocity_grid: bad dims");
    g.c.resize(k);
    f.read(reinterpret_cast<char*>(g.c.data()), k * 4);
    if (!f) data_error(std::string("read_velocity_grid: truncated payload in ") + path);
    g.validate();
    export_velocity(g, dim, n, origin, spacing, c, cap, count);
  });
}

int hs_write_velocity_grid(const char* path, int dim, const int n[3], const double origin[3], const double spacing[3],
                           const float* c) {
  return io_guarded([&] {
    Velocity g;
    g.dim = dim;
    for (int a = 0; a < 3; ++a) {
      g.n[a] = n[a];
      g.origin[a] = origin[a];
      g.spacing[a] = spacing[a];
    }
    if (dim == 2 || dim == 3) {
      const std::int64_t k = g.count();
      if (k > 0) g.c.assign(c, c + k);
    }
    g.validate();
    std::ofstream f(path, std::ios::binary);
    if (!f) data_error(std::string("write_velocity_grid: cannot open ") + path);
    f.write(kVelMagic, 4);
    const std::uint32_t version = kVersion, d = static_cast<std::uint32_t>(g.dim);
    std::uint32_t nn[3];
    for (int a = 0; a < 3; ++a) nn[a] = static_cast<std::uint32_t>(g.n[a]);
    f.write(reinterpret_cast<const char*>(&version), 4);
    f.write(reinterpret_cast<const char*>(&d), 4);
    f.write(reinterpret_cast<const char*>(nn), 12);
    f.write(reinterpret_cast<const char*>(g.origin), 24);
    f.write(reinterpret_cast<const char*>(g.spacing), 24);
    f.write(reinterpret_cast<const char*>(g.c.data()), static_cast<std::streamsize>(g.c.size() * 4));
    if (!f) data_error(std::string("write_velocity_grid: write failed for ") + path);
  });
}

int hs_read_velocity_csv(const char* path, int* dim, int n[3], double origin[3], double spacing[3], float* c,
                         int64_t cap, int64_t* count) {
  return io_guarded([&] {
    std::ifstream f(path);
    if (!f) data_error(std::string("read_velocity_csv: cannot open ") + path);
    std::string header;
    if (!std::getline(f, header)) data_error("read_velocity_csv: empty file");
    std::vector<double> fields;
    std::stringstream ss(header);
    std::string tok;
    while (std::getline(ss, tok, ',')) fields.push_back(std::stod(tok));
    if (fields.empty()) data_error("read_velocity_csv: bad header");
    Velocity g;
    g.dim = static_cast<int>(fields[0]);
    if (g.dim != 2 && g.dim != 3) data_error("read_velocity_csv: dim must be 2 or 3");
    if (static_cast<int>(fields.size()) != 1 + 3 * g.dim)
      data_error("read_velocity_csv: header needs dim, n, origin, spacing");
    for (int a = 0; a < g.dim; ++a) {
      g.n[a] = static_cast<int>(fields[1 + a]);
      g.origin[a] = fields[1 + g.dim + a];
      g.spacing[a] = fields[1 + 2 * g.dim + a];
    }
    std::string line;
    while (std::getline(f, line)) {
      if (line.empty()) continue;
      g.c.push_back(std::stof(line));
    }
    g.validate();
    export_velocity(g, dim, n, origin, spacing, c, cap, count);
  });
}

int hs_write_field(const char* path, int dim, const int lo[3], const int hi[3], const double h[3],
                   const double origin[3], const double* u) {
  return io_guarded([&] {
    if (dim != 2 && dim != 3) throw Error(hsb::kConfig, "write_field: dim must be 2 or 3");
    std::uint32_t nn[3];
    std::int32_t l[3];
    std::int64_t k = 1;
    for (int a = 0; a < 3; ++a) {
      nn[a] = a < dim ? static_cast<std::uint32_t>(hi[a] - lo[a] + 1) : 1;
      l[a] = a < dim ? lo[a] : 0;
      if (a < dim) k *= hi[a] - lo[a] + 1;
    }
    if (k <= 0) throw Error(hsb::kConfig, "write_field: size mismatch");
    std::ofstream f(path, std::ios::binary);
    if (!f) data_error(std::string("write_field: cannot open ") + path);
    f.write(kFieldMagic, 4);
    const std::uint32_t version = kVersion, d = static_cast<std::uint32_t>(dim);
    f.write(reinterpret_cast<const char*>(&version), 4);
    f.write(reinterpret_cast<const char*>(&d), 4);
    f.write(reinterpret_cast<const char*>(nn), 12);
    f.write(reinterpret_cast<const char*>(l), 12);
    f.write(reinterpret_cast<const char*>(h), 24);
    f.write(reinterpret_cast<const char*>(origin), 24);
    f.write(reinterpret_cast<const char*>(u), static_cast<std::streamsize>(k * 16));
    if (!f) data_error(std::string("write_field: write failed for ") + path);
  });
}

int hs_read_field(const char* path, int* dim, int lo[3], int hi[3], double h[3], double origin[3], double* u,
                  int64_t cap, int64_t* count) {
  return io_guarded([&] {
    std::ifstream f(path, std::ios::binary);
    if (!f) data_error(std::string("read_field: cannot open ") + path);
    char magic[4];
    f.read(magic, 4);
    if (!f || std::memcmp(magic, kFieldMagic, 4) != 0) data_error(std::string("read_field: bad magic in ") + path);
    std::uint32_t version = 0, d = 0, nn[3] = {0, 0, 0};
    std::int32_t l[3] = {0, 0, 0};
    f.read(reinterpret_cast<char*>(&version), 4);
    f.read(reinterpret_cast<char*>(&d), 4);
    f.read(reinterpret_cast<char*>(nn), 12);
    f.read(reinterpret_cast<char*>(l), 12);
    if (version != kVersion) data_error("read_field: unsupported version");
    double hh[3], oo[3];
    f.read(reinterpret_cast<char*>(hh), 24);
    f.read(reinterpret_cast<char*>(oo), 24);
    const int dm = static_cast<int>(d);
    std::int64_t k = 1;
    for (int a = 0; a < 3; ++a) {
      lo[a] = a < dm ? l[a] : 0;
      hi[a] = a < dm ? l[a] + static_cast<int>(nn[a]) - 1 : 0;
      if (a < dm) k *= nn[a];
      h[a] = hh[a];
      origin[a] = oo[a];
    }
    *dim = dm;
    std::vector<double> vals(static_cast<size_t>(2 * k));
    f.read(reinterpret_cast<char*>(vals.data()), static_cast<std::streamsize>(k * 16));
    if (!f) data_error(std::string("read_field: truncated payload in ") + path);
    *count = k;
    if (u && cap >= k) std::memcpy(u, vals.data(), vals.size() * sizeof(double));
  });
}

}  // extern "C"
