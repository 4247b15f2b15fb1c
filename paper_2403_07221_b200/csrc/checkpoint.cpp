// checkpoint.cpp -- the reference's "LFFN" v1 checkpoint as the on-disk input
// of the device path.
//
// Format (checkpoint.hpp:17-26, checkpoint.cpp:52-138), little endian:
//   "LFFN" | u32 version (1) | u32 d_in, d_out, h, tau | u8 variant |
//   u8 projection kind | u32 m (bh stages / acdc depth) | u32 b (bh block) |
//   float64 projection blob | float64 tables T [h][2^tau][d_out]
// Blob lengths are implied by the header.  Loading validates exactly what the
// reference validates (magic, version, variant/kind bytes, config, blob
// length, truncation, trailing bytes) with the same UsageError messages.
// lffn_ctx_create_from_checkpoint streams the float64 tables in slices
// straight into the device copy (a c4 checkpoint is 4.3 GB of doubles).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "lffn_gpu.h"
#include "lffn_internal.h"

namespace lffn_gpu {
namespace {

struct File {
  FILE* f = nullptr;
  explicit File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

bool get_u32(FILE* f, uint32_t* v) {
  unsigned char b[4];
  if (std::fread(b, 1, 4, f) != 4) return false;
  *v = uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
  return true;
}

bool get_u8(FILE* f, uint8_t* v) { return std::fread(v, 1, 1, f) == 1; }

bool get_f64s(FILE* f, double* out, size_t n) {
  // little-endian host (x86-64 / aarch64): raw copy
  return std::fread(out, sizeof(double), n, f) == n;
}

void put_u32(FILE* f, uint32_t v) {
  const unsigned char b[4] = {uint8_t(v), uint8_t(v >> 8), uint8_t(v >> 16), uint8_t(v >> 24)};
  std::fwrite(b, 1, 4, f);
}

// Reads the header; on success leaves the file positioned at the blob.
int read_header(FILE* f, const std::string& path, lffn_cfg* cfg, lffn_proj* proj) {
  char magic[4];
  if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "LFFN", 4) != 0)
    return fail(LFFN_ERR_USAGE, "checkpoint load: bad magic in " + path);
  uint32_t version = 0, d_in = 0, d_out = 0, h = 0, tau = 0, m = 0, b = 0;
  uint8_t variant = 0, kind = 0;
  if (!get_u32(f, &version)) return fail(LFFN_ERR_USAGE, "checkpoint load: truncated file " + path);
  if (version != 1)
    return fail(LFFN_ERR_USAGE, "checkpoint load: unsupported version " + std::to_string(version));
  if (!get_u32(f, &d_in) || !get_u32(f, &d_out) || !get_u32(f, &h) || !get_u32(f, &tau) ||
      !get_u8(f, &variant) || !get_u8(f, &kind) || !get_u32(f, &m) || !get_u32(f, &b))
    return fail(LFFN_ERR_USAGE, "checkpoint load: truncated file " + path);
  if (variant > LFFN_GELU_TAU1) return fail(LFFN_ERR_USAGE, "checkpoint load: bad variant byte");
  if (kind > LFFN_PROJ_SIGNFLIP) return fail(LFFN_ERR_USAGE, "checkpoint load: bad projection kind byte");
  *cfg = lffn_cfg{};
  cfg->d_in = d_in;
  cfg->d_out = d_out;
  cfg->tables = h;
  cfg->code_bits = tau;
  cfg->variant = variant;
  cfg->neighbor_count = 1;
  if (int rc = validate_cfg(cfg)) return rc;
  *proj = lffn_proj{};
  proj->kind = kind;
  proj->d_in = d_in;
  proj->d_out = int64_t(h) * int64_t(tau);
  proj->stages = 4;
  proj->block = 0;
  proj->depth = 1;
  if (kind == LFFN_PROJ_BH) {
    proj->stages = m;
    proj->block = b;
  } else if (kind == LFFN_PROJ_ACDC) {
    proj->depth = m;
  }
  if (int rc = validate_proj(proj)) return rc;
  proj->blob_len = blob_size(proj);
  return LFFN_OK;
}

}  // namespace
}  // namespace lffn_gpu

using namespace lffn_gpu;

extern "C" {

int lffn_checkpoint_header(const char* path, lffn_cfg* cfg, lffn_proj* proj,
                           int64_t* tables_len) {
  if (!path || !cfg || !proj) return fail(LFFN_ERR_USAGE, "checkpoint: null argument");
  File f(path, "rb");
  if (!f.f) return fail(LFFN_ERR_USAGE, std::string("checkpoint load: cannot open ") + path);
  if (int rc = read_header(f.f, path, cfg, proj)) return rc;
  if (tables_len) *tables_len = cfg->tables * (int64_t(1) << cfg->code_bits) * cfg->d_out;
  return LFFN_OK;
}

int lffn_checkpoint_load(const char* path, double* blob, double* tables) {
  if (!path || !blob || !tables) return fail(LFFN_ERR_USAGE, "checkpoint: null argument");
  File f(path, "rb");
  if (!f.f) return fail(LFFN_ERR_USAGE, std::string("checkpoint load: cannot open ") + path);
  lffn_cfg cfg;
  lffn_proj proj;
  if (int rc = read_header(f.f, path, &cfg, &proj)) return rc;
  const size_t nt = size_t(cfg.tables) * (size_t(1) << cfg.code_bits) * size_t(cfg.d_out);
  if (!get_f64s(f.f, blob, size_t(proj.blob_len)) || !get_f64s(f.f, tables, nt))
    return fail(LFFN_ERR_USAGE, std::string("checkpoint load: truncated file ") + path);
  if (std::fgetc(f.f) != EOF)
    return fail(LFFN_ERR_USAGE, std::string("checkpoint load: trailing bytes in ") + path);
  return LFFN_OK;
}

int lffn_checkpoint_save(const char* path, const lffn_cfg* cfg, const lffn_proj* proj,
                         const double* tables) {
  if (!path || !cfg || !proj || !proj->blob || !tables)
    return fail(LFFN_ERR_USAGE, "checkpoint: null argument");
  if (int rc = validate_cfg(cfg)) return rc;
  if (int rc = validate_proj(proj)) return rc;
  if (proj->d_in != cfg->d_in || proj->d_out != cfg->tables * cfg->code_bits)
    return fail(LFFN_ERR_USAGE, "checkpoint save: projection spec inconsistent with config");
  File f(path, "wb");
  if (!f.f) return fail(LFFN_ERR_USAGE, std::string("checkpoint save: cannot open ") + path);
  std::fwrite("LFFN", 1, 4, f.f);
  put_u32(f.f, 1);
  put_u32(f.f, uint32_t(cfg->d_in));
  put_u32(f.f, uint32_t(cfg->d_out));
  put_u32(f.f, uint32_t(cfg->tables));
  put_u32(f.f, uint32_t(cfg->code_bits));
  const uint8_t variant = uint8_t(cfg->variant), kind = uint8_t(proj->kind);
  std::fwrite(&variant, 1, 1, f.f);
  std::fwrite(&kind, 1, 1, f.f);
  uint32_t m = 0, b = 0;
  if (proj->kind == LFFN_PROJ_BH) {
    m = uint32_t(proj->stages);
    b = uint32_t(proj->block);
  } else if (proj->kind == LFFN_PROJ_ACDC) {
    m = uint32_t(proj->depth);
  }
  put_u32(f.f, m);
  put_u32(f.f, b);
  std::fwrite(proj->blob, sizeof(double), size_t(proj->blob_len), f.f);
  const size_t nt = size_t(cfg->tables) * (size_t(1) << cfg->code_bits) * size_t(cfg->d_out);
  std::fwrite(tables, sizeof(double), nt, f.f);
  if (std::ferror(f.f)) return fail(LFFN_ERR_USAGE, std::string("checkpoint save: write failed for ") + path);
  return LFFN_OK;
}

int lffn_ctx_create_from_checkpoint(lffn_ctx** out, int device, int64_t max_tokens,
                                    const char* path, int store_dtype, int64_t table_begin,
                                    int64_t table_end) {
  if (!out) return fail(LFFN_ERR_USAGE, "checkpoint: null output");
  *out = nullptr;
  lffn_cfg cfg;
  lffn_proj proj;
  {
    File f(path, "rb");
    if (!f.f) return fail(LFFN_ERR_USAGE, std::string("checkpoint load: cannot open ") + (path ? path : ""));
    if (int rc = read_header(f.f, path, &cfg, &proj)) return rc;
    std::vector<double> blob(size_t(proj.blob_len));
    if (!get_f64s(f.f, blob.data(), blob.size()))
      return fail(LFFN_ERR_USAGE, std::string("checkpoint load: truncated file ") + path);
    proj.blob = blob.data();
    if (table_begin == 0 && table_end == 0) table_end = cfg.tables;
    // the whole file must hold exactly header + blob + tables, as
    // load_checkpoint requires (checkpoint.cpp:134-136), even though only the
    // owned slice is read
    {
      const size_t per = (size_t(1) << cfg.code_bits) * size_t(cfg.d_out);
      const long here = std::ftell(f.f);
      if (here < 0 || std::fseek(f.f, 0, SEEK_END) != 0)
        return fail(LFFN_ERR_USAGE, std::string("checkpoint load: truncated file ") + path);
      const long end = std::ftell(f.f);
      const long long want = (long long)here + (long long)(size_t(cfg.tables) * per * sizeof(double));
      if (end < want) return fail(LFFN_ERR_USAGE, std::string("checkpoint load: truncated file ") + path);
      if (end > want) return fail(LFFN_ERR_USAGE, std::string("checkpoint load: trailing bytes in ") + path);
      if (std::fseek(f.f, here, SEEK_SET) != 0)
        return fail(LFFN_ERR_USAGE, std::string("checkpoint load: truncated file ") + path);
    }
    lffn_ctx* ctx = nullptr;
    if (int rc = lffn_ctx_create_shard(&ctx, device, max_tokens, &cfg, &proj, table_begin, table_end))
      return rc;
    // stream the owned table slice through a bounded host buffer
    const size_t per_table = (size_t(1) << cfg.code_bits) * size_t(cfg.d_out);
    if (std::fseek(f.f, long(table_begin * per_table * sizeof(double)), SEEK_CUR) != 0) {
      lffn_ctx_destroy(ctx);
      return fail(LFFN_ERR_USAGE, std::string("checkpoint load: truncated file ") + path);
    }
    const int64_t nloc = table_end - table_begin;
    const int64_t chunk_tables = std::max<int64_t>(1, int64_t((size_t(64) << 20) / (per_table * 8)));
    std::vector<double> buf;
    for (int64_t k0 = 0; k0 < nloc; k0 += chunk_tables) {
      const int64_t nk = std::min(chunk_tables, nloc - k0);
      buf.resize(size_t(nk) * per_table);
      if (!get_f64s(f.f, buf.data(), buf.size())) {
        lffn_ctx_destroy(ctx);
        return fail(LFFN_ERR_USAGE, std::string("checkpoint load: truncated file ") + path);
      }
      if (int rc = tables_upload_range(ctx, buf.data(), LFFN_F64, store_dtype, k0, nk)) {
        lffn_ctx_destroy(ctx);
        return rc;
      }
    }
    *out = ctx;
  }
  return LFFN_OK;
}

}  // extern "C"
