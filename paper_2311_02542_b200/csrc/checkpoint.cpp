// checkpoint.cpp -- LUMICKPT v1 ingest and export (the on-disk model format feeding the render
// path): proj/src/scene.cpp:286-394 (header, config, grid table, density / colour parameters,
// per-camera vignetting) and proj/src/occupancy.cpp:200-243 (RLE occupancy bits + trackers).
// Host-only; the parsed arrays go straight to lumi_model_create.
#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "lumi_cuda.h"

extern "C" int lumi_set_error(int code, const char* msg);

namespace {

struct Reader {
  std::ifstream is;
  template <typename T>
  bool get(T* v) {
    is.read(reinterpret_cast<char*>(v), sizeof(T));
    return static_cast<bool>(is);
  }
};

int err(const std::string& m) { return lumi_set_error(LUMI_ERR_INVALID, m.c_str()); }

}  // namespace

extern "C" int lumi_checkpoint_read(const char* path, LumiCheckpointInfo* info, float* table,
                                    float* dparams, float* cparams, uint8_t* occupancy) {
  if (!path || !info) return err("checkpoint: null argument");
  Reader r;
  r.is.open(path, std::ios::binary);
  if (!r.is.good()) return err(std::string("checkpoint: cannot open ") + path);
  char magic[8];
  r.is.read(magic, 8);
  if (!r.is || std::memcmp(magic, "LUMICKPT", 8) != 0)
    return err(std::string("checkpoint: bad magic in ") + path);
  uint32_t version = 0;
  if (!r.get(&version) || version != 1)
    return err(std::string("checkpoint: unsupported version in ") + path);
  LumiCheckpointInfo ci{};
  int32_t i32;
  double f64;
  uint32_t u32;
  uint8_t u8, contraction;
  bool ok = r.get(&i32) && ((ci.field.levels = i32), true) && r.get(&i32) &&
            ((ci.field.features_per_level = i32), true) && r.get(&i32) &&
            ((ci.field.base_resolution = i32), true) && r.get(&f64) &&
            ((ci.field.per_level_scale = f64), true) && r.get(&u32) &&
            ((ci.field.table_size = u32), true) && r.get(&i32) &&
            ((ci.field.hidden_width = i32), true) && r.get(&i32) &&
            ((ci.field.bottleneck = i32), true) && r.get(&u8) &&
            ((ci.field.color_space = u8 == 0 ? 0 : 1), true) && r.get(&contraction) &&
            r.get(&ci.samples_per_ray) && r.get(&ci.background[0]) && r.get(&ci.background[1]) &&
            r.get(&ci.background[2]);
  if (!ok) return err("checkpoint: truncated header");
  ci.contraction = contraction == 0 ? 1 : 0;  // 0 = kLInfCubic in the file (scene.cpp:332)
  LumiGridLayout lay;
  int rc = lumi_field_layout(&ci.field, &lay);
  if (rc) return rc;
  ci.table_floats = lay.total_floats;
  ci.density_params = lay.density_params;
  ci.color_params = lay.color_params;

  auto floats = [&](uint64_t expect, float* dst, const char* what) -> int {
    uint64_t n = 0;
    if (!r.get(&n)) return err("checkpoint: truncated stream");
    if (n != expect) return err(std::string("checkpoint: ") + what + " size mismatch");
    if (dst) {
      r.is.read(reinterpret_cast<char*>(dst), static_cast<std::streamsize>(n * sizeof(float)));
    } else {
      r.is.seekg(static_cast<std::streamoff>(n * sizeof(float)), std::ios::cur);
    }
    return r.is ? LUMI_OK : err("checkpoint: truncated stream");
  };
  if ((rc = floats(lay.total_floats, table, "grid"))) return rc;
  if ((rc = floats(lay.density_params, dparams, "density net"))) return rc;
  if ((rc = floats(lay.color_params, cparams, "color net"))) return rc;
  uint64_t ncam = 0;
  if (!r.get(&ncam)) return err("checkpoint: truncated stream");
  ci.n_cameras = static_cast<int32_t>(ncam);
  r.is.seekg(static_cast<std::streamoff>(ncam * sizeof(double)), std::ios::cur);

  // OccupancyGrid::load (occupancy.cpp:224-243)
  int32_t res = 0;
  uint64_t runs = 0;
  if (!r.get(&res) || !r.get(&runs)) return err("occupancy: truncated stream");
  if (res < 1 || res > 1024) return err("occupancy: bad resolution");
  ci.occ_res = res;
  const uint64_t n = static_cast<uint64_t>(res) * res * res;
  uint64_t at = 0;
  for (uint64_t k = 0; k < runs; ++k) {
    uint8_t v;
    uint64_t len;
    if (!r.get(&v) || !r.get(&len)) return err("occupancy: truncated stream");
    if (at + len > n) return err("occupancy: corrupt RLE stream");
    if (occupancy) std::memset(occupancy + at, v ? 1 : 0, len);
    at += len;
  }
  if (at != n) return err("occupancy: truncated RLE stream");
  // carved bytes + history + probe trackers follow (training state, not rendering); the
  // reference requires them present (occupancy.cpp:241)
  std::vector<char> rest(n * (1 + 2 * sizeof(float)));
  r.is.read(rest.data(), static_cast<std::streamsize>(rest.size()));
  if (!r.is) return err("occupancy: truncated stream");
  *info = ci;
  return LUMI_OK;
}

namespace {
struct Writer {
  std::ofstream os;
  template <typename T>
  void put(const T& v) {
    os.write(reinterpret_cast<const char*>(&v), sizeof(T));
  }
  void floats(const float* p, uint64_t n) {  // put_floats (scene.cpp:309-312)
    put(n);
    os.write(reinterpret_cast<const char*>(p), static_cast<std::streamsize>(n * sizeof(float)));
  }
};
}  // namespace

// save_checkpoint (scene.cpp:320-351) + OccupancyGrid::save (occupancy.cpp:200-222) of a
// rendering model: training trackers (carved bytes, history, probe maxima) are written as zeros.
extern "C" int lumi_checkpoint_write(const char* path, const LumiCheckpointInfo* info,
                                     const float* table, const float* dparams, const float* cparams,
                                     const double* alpha_v, const uint8_t* occupancy) {
  if (!path || !info || !table || !dparams || !cparams || !occupancy)
    return err("checkpoint: null argument");
  LumiGridLayout lay;
  int rc = lumi_field_layout(&info->field, &lay);
  if (rc) return rc;
  if (info->occ_res < 1 || info->occ_res > 1024) return err("occupancy: bad resolution");
  if (info->n_cameras < 0) return err("checkpoint: bad camera count");
  Writer w;
  w.os.open(path, std::ios::binary);
  if (!w.os.good()) return err(std::string("checkpoint: cannot write ") + path);
  w.os.write("LUMICKPT", 8);
  w.put<uint32_t>(1);
  const LumiFieldDesc& f = info->field;
  w.put<int32_t>(f.levels);
  w.put<int32_t>(f.features_per_level);
  w.put<int32_t>(f.base_resolution);
  w.put<double>(f.per_level_scale);
  w.put<uint32_t>(f.table_size);
  w.put<int32_t>(f.hidden_width);
  w.put<int32_t>(f.bottleneck);
  w.put<uint8_t>(f.color_space == 0 ? 0 : 1);
  w.put<uint8_t>(info->contraction == 1 ? 0 : 1);  // 0 = kLInfCubic in the file
  w.put<int32_t>(info->samples_per_ray);
  for (int k = 0; k < 3; ++k) w.put<double>(info->background[k]);
  w.floats(table, lay.total_floats);
  w.floats(dparams, lay.density_params);
  w.floats(cparams, lay.color_params);
  w.put<uint64_t>(static_cast<uint64_t>(info->n_cameras));
  for (int k = 0; k < info->n_cameras; ++k) w.put<double>(alpha_v ? alpha_v[k] : 0.0);
  const int32_t res = info->occ_res;
  const uint64_t n = static_cast<uint64_t>(res) * res * res;
  w.put<int32_t>(res);
  std::vector<std::pair<uint8_t, uint64_t>> rle;
  for (uint64_t i = 0; i < n;) {
    const uint8_t v = occupancy[i] ? 1 : 0;
    uint64_t len = 1;
    while (i + len < n && (occupancy[i + len] ? 1 : 0) == v) ++len;
    rle.emplace_back(v, len);
    i += len;
  }
  w.put<uint64_t>(rle.size());
  for (const auto& r : rle) {
    w.put<uint8_t>(r.first);
    w.put<uint64_t>(r.second);
  }
  const std::vector<char> zeros(n * (1 + 2 * sizeof(float)), 0);
  w.os.write(zeros.data(), static_cast<std::streamsize>(zeros.size()));
  w.os.flush();
  if (!w.os.good()) return err(std::string("checkpoint: write failed ") + path);
  return LUMI_OK;
}
