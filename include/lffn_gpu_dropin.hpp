// lffn_gpu_dropin.hpp -- reference-side C++ drop-in over the lffn C-ABI.
//
// A maintainer of the reference library (lookupffn, namespace lffn) adds this
// header to their tree and links liblffn_gpu.so.  It restates the
// reference's public forward entry points with the same signatures, argument
// meaning and exception types, and runs them on a B200:
//
//   lffn::gpu::lookup_forward(x, proj, tables, cfg)   ~ lffn::lookup_forward
//                                                       (lookup.hpp:124-125)
//   lffn::gpu::Layer                                   a device-resident layer
//                                                       for repeated calls
//
// It includes the reference's own headers (lookupffn/lookup.hpp,
// projection.hpp, matrix.hpp, common.hpp) for DenseMatrix / Projection /
// HashTables / LookupConfig and the error types; nothing here depends on the
// reference's implementation files.  There is no CPU fallback: a missing
// device surfaces as std::runtime_error, a LookupCache (training) as
// UsageError, neighbor_count above the device limit (256) as SizeError; the
// other validation failures throw SizeError or UsageError exactly where the
// reference does (lffn_last_error_class).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "lffn_gpu.h"
#include "lookupffn/common.hpp"
#include "lookupffn/lookup.hpp"
#include "lookupffn/matrix.hpp"
#include "lookupffn/projection.hpp"

namespace lffn {
namespace gpu {

/// Status -> the reference's exception types (common.hpp:13-37): status 1
/// is SizeError or UsageError as lffn_last_error_class() says, 2 NumericError.
inline void check(int status) {
  if (status == LFFN_OK) return;
  const std::string msg = lffn_last_error();
  if (status == LFFN_ERR_USAGE) {
    if (lffn_last_error_class() == LFFN_CLASS_SIZE) throw SizeError(msg);
    throw UsageError(msg);
  }
  if (status == LFFN_ERR_NUMERIC) throw NumericError(msg);
  throw std::runtime_error("lffn_gpu: " + msg);
}

/// 64-bit content hash of a float64 array (multi-threaded): the drop-in
/// reuses its device copy of the tables only while they are unchanged.
inline uint64_t content_hash(const std::vector<double>& v) {
  const std::size_t n = v.size();
  const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<uint64_t> part(nt, 0);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      const std::size_t b = n * t / nt, e = n * (t + 1) / nt;
      uint64_t h = 0x9e3779b97f4a7c15ull ^ (uint64_t(t) << 32);
      for (std::size_t i = b; i < e; ++i) {
        uint64_t u;
        std::memcpy(&u, &v[i], 8);
        h = (h ^ u) * 0x100000001b3ull;
        h ^= h >> 29;
      }
      part[t] = h;
    });
  for (auto& x : th) x.join();
  uint64_t h = n;
  for (uint64_t p : part) h = (h ^ p) * 0x9e3779b97f4a7c15ull;
  return h;
}

inline lffn_cfg to_c(const LookupConfig& c) {
  lffn_cfg o{};
  o.d_in = int64_t(c.d_in);
  o.d_out = int64_t(c.d_out);
  o.tables = int64_t(c.tables);
  o.code_bits = int64_t(c.code_bits);
  o.variant = int32_t(c.variant);
  o.neighbor_count = int32_t(c.neighbor_count);
  return o;
}

inline lffn_proj to_c(const Projection& p) {
  lffn_proj o{};
  const ProjectionSpec& s = p.spec();
  o.kind = int32_t(s.kind);
  o.d_in = int64_t(s.d_in);
  o.d_out = int64_t(s.d_out);
  o.stages = int64_t(s.stages);
  o.block = int64_t(s.block);
  o.depth = int64_t(s.depth);
  o.blob = p.blob().data();
  o.blob_len = int64_t(p.blob_size());
  return o;
}

/// A device-resident LookupFFN layer (one lffn_ctx): tables uploaded once,
/// then forward() per batch with host DenseMatrix in/out.
class Layer {
 public:
  Layer(const Projection& proj, const HashTables& tables, const LookupConfig& cfg,
        std::size_t max_tokens, int device = 0, bool bf16_tables = false)
      : cfg_(cfg) {
    const lffn_cfg c = to_c(cfg);
    const lffn_proj p = to_c(proj);
    lffn_ctx* ctx = nullptr;
    check(lffn_ctx_create(&ctx, device, int64_t(max_tokens), &c, &p));
    ctx_.reset(ctx);
    if (tables.tables != cfg.tables || tables.code_bits != cfg.code_bits ||
        tables.d_out != cfg.d_out)
      throw SizeError("lookup forward: table stack shape mismatch");
    check(lffn_tables_upload(ctx, tables.data.data(), LFFN_F64,
                             bf16_tables ? LFFN_BF16 : LFFN_F32));
  }

  /// y = lookup_forward(x): x rows are rounded to float32 on the way in (the
  /// reference's own inference path, bench.cpp:115-217, is float32 too).
  DenseMatrix forward(const DenseMatrix& x) const {
    if (x.cols != cfg_.d_in) throw SizeError("lookup forward: input width mismatch");
    std::vector<float> xf(x.data.begin(), x.data.end());
    std::vector<float> yf(x.rows * cfg_.d_out);
    check(lffn_forward_host(ctx_.get(), xf.data(), int64_t(x.rows), yf.data()));
    DenseMatrix y(x.rows, cfg_.d_out);
    for (std::size_t i = 0; i < yf.size(); ++i) y.data[i] = double(yf[i]);
    return y;
  }

 private:
  struct Deleter {
    void operator()(lffn_ctx* c) const { lffn_ctx_destroy(c); }
  };
  LookupConfig cfg_;
  std::unique_ptr<lffn_ctx, Deleter> ctx_;
};

/// Drop-in for lffn::lookup_forward (lookup.hpp:124-125), any neighbor_count <= 256.
/// The reference call is stateless; the device layer (context, converted
/// tables) is cached per thread and reused while the configuration, the
/// projection and the table contents are unchanged (content hashes), and
/// the batch fits its max_tokens -- repeated calls skip the table upload.
inline DenseMatrix lookup_forward(const DenseMatrix& x, const Projection& proj,
                                  const HashTables& tables, const LookupConfig& cfg,
                                  LookupCache* cache = nullptr) {
  if (cache) throw UsageError("lffn::gpu: LookupCache (training) is not supported on the device");
  cfg.validate();
  if (x.cols != cfg.d_in) throw SizeError("lookup forward: input width mismatch");
  if (proj.spec().d_in != cfg.d_in || proj.spec().d_out != cfg.code_width())
    throw SizeError("lookup forward: projection must map d_in to h*tau");
  struct Cached {
    std::unique_ptr<Layer> layer;
    std::size_t max_tokens = 0;
    uint64_t key[8] = {};
  };
  static thread_local Cached c;
  const uint64_t key[8] = {uint64_t(cfg.d_in), uint64_t(cfg.d_out), uint64_t(cfg.tables),
                           uint64_t(cfg.code_bits) | (uint64_t(cfg.variant) << 32),
                           uint64_t(cfg.neighbor_count) | (uint64_t(proj.spec().kind) << 32),
                           content_hash(proj.blob()), content_hash(tables.data),
                           uint64_t(tables.data.size())};
  const std::size_t rows = x.rows > 0 ? x.rows : 1;
  const bool same = c.layer && std::memcmp(key, c.key, sizeof(key)) == 0;
  if (!same || rows > c.max_tokens) {
    c.max_tokens = same ? std::max(rows, c.max_tokens) : rows;
    c.layer.reset();
    c.layer.reset(new Layer(proj, tables, cfg, c.max_tokens));
    std::memcpy(c.key, key, sizeof(key));
  }
  return c.layer->forward(x);
}

}  // namespace gpu
}  // namespace lffn
