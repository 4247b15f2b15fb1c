// host_params.cpp -- configuration checks and seeded parameter generation of
// the lffn C-ABI (include/lffn_gpu.h).
//
// Parameters are generated on the host with the same engine and libstdc++
// distributions the reference uses (std::mt19937_64, std::normal_distribution,
// std::bernoulli_distribution; common.hpp:44-55), so a context built from
// lffn_proj_init / lffn_tables_init holds bit-identical parameters to the
// reference's Projection::init / HashTables::init for the same seed.  The
// device never generates parameters: the reference's distributions are
// implementation-defined and sequential.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "lffn_gpu.h"
#include "lffn_internal.h"

namespace lffn_gpu {

int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

int64_t transform_width(const lffn_proj* p) {
  return next_pow2(p->d_in > p->d_out ? p->d_in : p->d_out);
}

int64_t blob_size(const lffn_proj* p) {
  const int64_t D = transform_width(p);
  switch (p->kind) {
    case LFFN_PROJ_DENSE: return p->d_in * p->d_out;
    case LFFN_PROJ_BH: {
      const int64_t b = p->block == 0 ? D : p->block;
      return p->stages * (D / b) * b * b;
    }
    case LFFN_PROJ_ACDC: return 2 * p->depth * D;
    case LFFN_PROJ_SIGNFLIP: return 3 * D;
  }
  return 0;
}

namespace {

void gaussian(std::mt19937_64& rng, double* out, int64_t n, double stddev) {
  std::normal_distribution<double> dist(0.0, stddev);
  for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
}

void signs(std::mt19937_64& rng, double* out, int64_t n) {
  std::bernoulli_distribution coin(0.5);
  for (int64_t i = 0; i < n; ++i) out[i] = coin(rng) ? 1.0 : -1.0;
}

// Random orthogonal b x b block: Gaussian draw (fresh distribution), then
// modified Gram-Schmidt over the columns with a basis-column fallback for
// degenerate columns -- the construction of projection.cpp:60-79.
void orthogonal_block(double* m, int64_t b, std::mt19937_64& rng) {
  gaussian(rng, m, b * b, 1.0);
  for (int64_t c = 0; c < b; ++c) {
    for (int64_t prev = 0; prev < c; ++prev) {
      double dot = 0.0;
      for (int64_t r = 0; r < b; ++r) dot += m[r * b + c] * m[r * b + prev];
      for (int64_t r = 0; r < b; ++r) m[r * b + c] -= dot * m[r * b + prev];
    }
    double norm = 0.0;
    for (int64_t r = 0; r < b; ++r) norm += m[r * b + c] * m[r * b + c];
    norm = std::sqrt(norm);
    if (norm < 1e-12) {
      for (int64_t r = 0; r < b; ++r) m[r * b + c] = (r == c) ? 1.0 : 0.0;
      continue;
    }
    for (int64_t r = 0; r < b; ++r) m[r * b + c] /= norm;
  }
}

}  // namespace

int validate_cfg(const lffn_cfg* c) {
  if (!c) return fail(LFFN_ERR_USAGE, "lookup config: null");
  if (c->d_in <= 0 || c->d_out <= 0)
    return fail(LFFN_ERR_USAGE, "lookup config: d_in and d_out must be positive");
  if (c->tables <= 0) return fail(LFFN_ERR_USAGE, "lookup config: table count must be >= 1");
  if (c->code_bits < 1 || c->code_bits > 24)
    return fail(LFFN_ERR_USAGE, "lookup config: code bits must be in [1, 24]");
  if (c->neighbor_count < 1 || int64_t(c->neighbor_count) > (int64_t(1) << c->code_bits))
    return fail(LFFN_ERR_USAGE, "lookup config: neighbor count must be in [1, 2^tau]");
  if ((c->variant == LFFN_SIGMOID_TAU1 || c->variant == LFFN_GELU_TAU1) && c->code_bits != 1)
    return fail(LFFN_ERR_USAGE, "lookup config: tau-1 variants require code_bits == 1");
  if (c->variant < LFFN_SOFTMAX || c->variant > LFFN_GELU_TAU1)
    return fail(LFFN_ERR_USAGE, "unknown lookup variant");
  return LFFN_OK;
}

int validate_proj(const lffn_proj* p) {
  if (!p) return fail(LFFN_ERR_USAGE, "projection: null");
  if (p->kind < LFFN_PROJ_DENSE || p->kind > LFFN_PROJ_SIGNFLIP)
    return fail(LFFN_ERR_USAGE, "unknown projection kind");
  if (p->d_in <= 0 || p->d_out <= 0)
    return fail(LFFN_ERR_USAGE, "projection: d_in and d_out must be positive");
  const int64_t D = transform_width(p);
  if (p->kind == LFFN_PROJ_BH) {
    const int64_t b = p->block == 0 ? D : p->block;
    if (p->stages <= 0) return fail(LFFN_ERR_USAGE, "bh projection: stage count must be >= 1");
    if (b <= 0 || b > D || D % b != 0)
      return fail(LFFN_ERR_USAGE, "bh projection: block size " + std::to_string(b) +
                                      " must divide transform width " + std::to_string(D));
  }
  if (p->kind == LFFN_PROJ_ACDC && p->depth <= 0)
    return fail(LFFN_ERR_USAGE, "acdc projection: depth must be >= 1");
  if (p->blob && p->blob_len != blob_size(p))
    return fail(LFFN_ERR_USAGE, "projection blob: expected " + std::to_string(blob_size(p)) +
                                    " values, got " + std::to_string(p->blob_len));
  return LFFN_OK;
}

}  // namespace lffn_gpu

using namespace lffn_gpu;

extern "C" {

int lffn_cfg_validate(const lffn_cfg* cfg) { return validate_cfg(cfg); }

int lffn_proj_validate(const lffn_proj* proj) { return validate_proj(proj); }

int64_t lffn_transform_width(const lffn_proj* proj) {
  return proj ? transform_width(proj) : -1;
}

int64_t lffn_proj_blob_size(const lffn_proj* proj) {
  if (!proj || validate_proj(proj) != LFFN_OK) return -1;
  return blob_size(proj);
}

int lffn_proj_init(const lffn_proj* spec, uint64_t seed, double* blob_out) {
  lffn_proj s = *spec;
  s.blob = nullptr;
  if (int rc = validate_proj(&s)) return rc;
  if (!blob_out) return fail(LFFN_ERR_USAGE, "projection init: null output");
  const int64_t n = blob_size(&s);
  const int64_t D = transform_width(&s);
  std::memset(blob_out, 0, size_t(n) * sizeof(double));
  std::mt19937_64 rng(seed);
  switch (s.kind) {
    case LFFN_PROJ_DENSE:
      gaussian(rng, blob_out, n, 1.0 / std::sqrt(double(s.d_in)));
      break;
    case LFFN_PROJ_BH: {
      const int64_t b = s.block == 0 ? D : s.block;
      const double scale = 1.0 / std::sqrt(double(D));
      for (int64_t blk = 0; blk < n / (b * b); ++blk) {
        double* m = blob_out + blk * b * b;
        orthogonal_block(m, b, rng);
        for (int64_t i = 0; i < b * b; ++i) m[i] *= scale;
      }
      break;
    }
    case LFFN_PROJ_ACDC: {
      signs(rng, blob_out, n);
      const double scale = 1.0 / std::sqrt(double(D));
      for (int64_t i = 0; i < n; ++i) blob_out[i] *= scale;
      break;
    }
    case LFFN_PROJ_SIGNFLIP:
      signs(rng, blob_out, n);
      break;
  }
  return LFFN_OK;
}

int lffn_fill_gaussian(uint64_t seed, double* out, int64_t n, double stddev) {
  if (!out || n < 0) return fail(LFFN_ERR_USAGE, "fill_gaussian: bad arguments");
  std::mt19937_64 rng(seed);
  gaussian(rng, out, n, stddev);
  return LFFN_OK;
}

int lffn_fill_gaussian_slice(uint64_t seed, int64_t skip, double* out, int64_t n, double stddev) {
  if (!out || n < 0 || skip < 0) return fail(LFFN_ERR_USAGE, "fill_gaussian_slice: bad arguments");
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> dist(0.0, stddev);
  for (int64_t i = 0; i < skip; ++i) (void)dist(rng);
  for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
  return LFFN_OK;
}

int lffn_fill_signs(uint64_t seed, double* out, int64_t n) {
  if (!out || n < 0) return fail(LFFN_ERR_USAGE, "fill_signs: bad arguments");
  std::mt19937_64 rng(seed);
  signs(rng, out, n);
  return LFFN_OK;
}

int lffn_tables_init(const lffn_cfg* cfg, uint64_t seed, double* out) {
  if (int rc = validate_cfg(cfg)) return rc;
  if (!out) return fail(LFFN_ERR_USAGE, "tables init: null output");
  const int64_t n = cfg->tables * (int64_t(1) << cfg->code_bits) * cfg->d_out;
  std::mt19937_64 rng(seed);
  gaussian(rng, out, n, 1.0 / std::sqrt(double(cfg->tables)));
  return LFFN_OK;
}

}  // extern "C"
