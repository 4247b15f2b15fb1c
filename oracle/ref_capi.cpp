// ref_capi.cpp -- extern "C" shim over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference's own sources (read in place from /root/reference/proj, never
// copied) into oracle/_ref/liblffn_ref.so.  tests/ use it to pin the C
// restatement (oracle/lffn_oracle.c) and to generate tests/golden/; bench.py's
// reference arm and cpu_baseline time the reference's float32 inference
// kernels through it.
//
// The float32 kernels live in an anonymous namespace in src/bench.cpp
// (bench.cpp:115-217); including that translation unit here is the only way
// to call them without copying them.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "lookupffn/checkpoint.hpp"
#include "lookupffn/common.hpp"
#include "lookupffn/flops.hpp"
#include "lookupffn/fwht.hpp"
#include "lookupffn/lookup.hpp"
#include "lookupffn/projection.hpp"
#include "src/bench.cpp"  // NOLINT: exposes lookup_hash_f32 & co.

#if defined(_OPENMP)
#include <omp.h>
#endif

using namespace lffn;

namespace {

ProjectionSpec make_spec(int kind, int64_t d_in, int64_t d_out, int64_t stages, int64_t block,
                         int64_t depth) {
  ProjectionSpec s;
  s.d_in = size_t(d_in);
  s.d_out = size_t(d_out);
  s.kind = ProjKind(kind);
  s.stages = size_t(stages);
  s.block = size_t(block);
  s.depth = size_t(depth);
  return s;
}

LookupConfig make_cfg(int64_t d_in, int64_t d_out, int64_t h, int64_t tau, int variant,
                      int64_t nc) {
  LookupConfig c;
  c.d_in = size_t(d_in);
  c.d_out = size_t(d_out);
  c.tables = size_t(h);
  c.code_bits = size_t(tau);
  c.variant = LookupVariant(variant);
  c.neighbor_count = size_t(nc);
  return c;
}

thread_local std::string g_err;

int map_exc(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const SizeError*>(&e) || dynamic_cast<const UsageError*>(&e)) return 1;
  if (dynamic_cast<const NumericError*>(&e)) return 2;
  return 3;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// make_rng(seed) + fill_gaussian(std)  (common.hpp:44-49); DenseMatrix::gaussian
// (matrix.hpp:37-42) is the same call on a fresh rng.
void ref_fill_gaussian(uint64_t seed, double* out, size_t n, double stddev) {
  auto rng = make_rng(seed);
  fill_gaussian(std::span<double>(out, n), rng, stddev);
}

void ref_fill_signs(uint64_t seed, double* out, size_t n) {
  auto rng = make_rng(seed);
  fill_signs(std::span<double>(out, n), rng);
}

// Projection::init (projection.cpp:97-135). Returns blob size, or -1.
int64_t ref_proj_init(int kind, int64_t d_in, int64_t d_out, int64_t stages, int64_t block,
                      int64_t depth, uint64_t seed, double* blob, int64_t cap) {
  try {
    Projection p = Projection::init(make_spec(kind, d_in, d_out, stages, block, depth), seed);
    if (blob && cap >= int64_t(p.blob_size()))
      std::memcpy(blob, p.blob().data(), p.blob_size() * sizeof(double));
    return int64_t(p.blob_size());
  } catch (const std::exception& e) {
    map_exc(e);
    return -1;
  }
}

// HashTables::init (lookup.cpp:39-49), std 1/sqrt(h).
int ref_tables_init(int64_t d_in, int64_t d_out, int64_t h, int64_t tau, uint64_t seed,
                    double* out) {
  try {
    HashTables t = HashTables::init(make_cfg(d_in, d_out, h, tau, 0, 1), seed);
    std::memcpy(out, t.data.data(), t.data.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

void ref_fwht(double* v, size_t n) { fwht_kernel(v, n); }

uint32_t ref_sign_code(const double* z, size_t tau) {
  return sign_code(std::span<const double>(z, tau));
}

double ref_log_denominator(const double* z, size_t tau) {
  return log_denominator(std::span<const double>(z, tau));
}

double ref_code_dot(const double* z, size_t tau, uint32_t code) {
  return code_dot(std::span<const double>(z, tau), code);
}

int64_t ref_neighbor_codes(const double* z, size_t tau, size_t count, uint32_t* out) {
  try {
    auto v = neighbor_codes(std::span<const double>(z, tau), count);
    std::memcpy(out, v.data(), v.size() * sizeof(uint32_t));
    return int64_t(v.size());
  } catch (const std::exception& e) {
    map_exc(e);
    return -1;
  }
}

// compute_codes (lookup.cpp:81-100)
int ref_compute_codes(const double* z, size_t n, size_t h, size_t tau, uint32_t* codes,
                      double* abs_z) {
  try {
    SoftCodes soft;
    soft.n = n;
    soft.tables = h;
    soft.code_bits = tau;
    soft.z.assign(z, z + n * h * tau);
    SignCodes s = compute_codes(soft);
    std::memcpy(codes, s.codes.data(), s.codes.size() * sizeof(uint32_t));
    if (abs_z) std::memcpy(abs_z, s.abs_z.data(), s.abs_z.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

// Projection::forward (projection.cpp:268-270)
int ref_proj_forward(int kind, int64_t d_in, int64_t d_out, int64_t stages, int64_t block,
                     int64_t depth, const double* blob, int64_t blob_len, const double* x,
                     size_t n, double* z) {
  try {
    ProjectionSpec s = make_spec(kind, d_in, d_out, stages, block, depth);
    Projection p = Projection::from_blob(s, std::vector<double>(blob, blob + blob_len));
    DenseMatrix xm(n, size_t(d_in));
    std::memcpy(xm.data.data(), x, n * size_t(d_in) * sizeof(double));
    DenseMatrix out = p.forward(xm);
    std::memcpy(z, out.data.data(), out.data.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

// lookup_forward (lookup.cpp:279-282) with a LookupCache to expose z, codes,
// weights and dots.  All optional outputs may be NULL.
int ref_lookup_forward(int64_t d_in, int64_t d_out, int64_t h, int64_t tau, int variant,
                       int64_t nc, int kind, int64_t stages, int64_t block, int64_t depth,
                       const double* blob, int64_t blob_len, const double* tables, const double* x,
                       size_t n, double* y, double* z_out, uint32_t* codes_out,
                       double* weights_out, double* dots_out) {
  try {
    LookupConfig cfg = make_cfg(d_in, d_out, h, tau, variant, nc);
    ProjectionSpec s = make_spec(kind, d_in, h * tau, stages, block, depth);
    Projection p = Projection::from_blob(s, std::vector<double>(blob, blob + blob_len));
    HashTables t = HashTables::zeros_like(cfg);
    std::memcpy(t.data.data(), tables, t.data.size() * sizeof(double));
    DenseMatrix xm(n, size_t(d_in));
    std::memcpy(xm.data.data(), x, n * size_t(d_in) * sizeof(double));
    LookupCache cache;
    DenseMatrix out = lookup_forward(xm, p, t, cfg, &cache);
    std::memcpy(y, out.data.data(), out.data.size() * sizeof(double));
    if (z_out) std::memcpy(z_out, cache.soft.z.data(), cache.soft.z.size() * sizeof(double));
    if (codes_out)
      std::memcpy(codes_out, cache.codes.data(), cache.codes.size() * sizeof(uint32_t));
    if (weights_out)
      std::memcpy(weights_out, cache.weights.data(), cache.weights.size() * sizeof(double));
    if (dots_out) std::memcpy(dots_out, cache.dots.data(), cache.dots.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

// lookup_forward with a cache, then lookup_backward (lookup.cpp:292-347):
// grad_x [n x d_in], grad_tables [h][2^tau][d_out], grad_proj [param_count].
int ref_lookup_backward(int64_t d_in, int64_t d_out, int64_t h, int64_t tau, int variant,
                        int64_t nc, int kind, int64_t stages, int64_t block, int64_t depth,
                        const double* blob, int64_t blob_len, const double* tables, const double* x,
                        size_t n, const double* grad_y, double* grad_x, double* grad_tables,
                        double* grad_proj) {
  try {
    LookupConfig cfg = make_cfg(d_in, d_out, h, tau, variant, nc);
    ProjectionSpec s = make_spec(kind, d_in, h * tau, stages, block, depth);
    Projection p = Projection::from_blob(s, std::vector<double>(blob, blob + blob_len));
    HashTables t = HashTables::zeros_like(cfg);
    std::memcpy(t.data.data(), tables, t.data.size() * sizeof(double));
    DenseMatrix xm(n, size_t(d_in));
    std::memcpy(xm.data.data(), x, n * size_t(d_in) * sizeof(double));
    LookupCache cache;
    lookup_forward(xm, p, t, cfg, &cache);
    DenseMatrix gy(n, size_t(d_out));
    std::memcpy(gy.data.data(), grad_y, n * size_t(d_out) * sizeof(double));
    LookupGrads g = lookup_backward(gy, cache, p, t, cfg);
    std::memcpy(grad_x, g.grad_x.data.data(), g.grad_x.data.size() * sizeof(double));
    std::memcpy(grad_tables, g.grad_tables.data(), g.grad_tables.size() * sizeof(double));
    std::memcpy(grad_proj, g.grad_proj.data(), g.grad_proj.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

// Projection::backward (projection.cpp:279-386) with the forward's cache.
int ref_proj_backward(int kind, int64_t d_in, int64_t d_out, int64_t stages, int64_t block,
                      int64_t depth, const double* blob, int64_t blob_len, const double* x, size_t n,
                      const double* grad_out, double* grad_x, double* grad_params) {
  try {
    ProjectionSpec s = make_spec(kind, d_in, d_out, stages, block, depth);
    Projection p = Projection::from_blob(s, std::vector<double>(blob, blob + blob_len));
    DenseMatrix xm(n, size_t(d_in));
    std::memcpy(xm.data.data(), x, n * size_t(d_in) * sizeof(double));
    ProjectionCache cache;
    p.forward(xm, &cache);
    DenseMatrix go(n, size_t(d_out));
    std::memcpy(go.data.data(), grad_out, n * size_t(d_out) * sizeof(double));
    std::vector<double> gp(p.param_count(), 0.0);
    DenseMatrix gx = p.backward(go, xm, cache, gp);
    std::memcpy(grad_x, gx.data.data(), gx.data.size() * sizeof(double));
    std::memcpy(grad_params, gp.data(), gp.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

// save_checkpoint / load_checkpoint (checkpoint.cpp:52-138).  load returns
// the header fields in hdr[8] = {d_in, d_out, h, tau, variant, kind, m, b}
// and copies blob / tables when the pointers are non-null.
int ref_save_checkpoint(const char* path, int64_t d_in, int64_t d_out, int64_t h, int64_t tau,
                        int variant, int kind, int64_t stages, int64_t block, int64_t depth,
                        const double* blob, int64_t blob_len, const double* tables) {
  try {
    CheckpointModel m;
    m.cfg = make_cfg(d_in, d_out, h, tau, variant, 1);
    m.proj = Projection::from_blob(make_spec(kind, d_in, h * tau, stages, block, depth),
                                   std::vector<double>(blob, blob + blob_len));
    m.tables = HashTables::zeros_like(m.cfg);
    std::memcpy(m.tables.data.data(), tables, m.tables.data.size() * sizeof(double));
    save_checkpoint(path, m);
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

int ref_load_checkpoint(const char* path, int64_t* hdr, double* blob, double* tables) {
  try {
    CheckpointModel m = load_checkpoint(path);
    const ProjectionSpec& s = m.proj.spec();
    hdr[0] = int64_t(m.cfg.d_in);
    hdr[1] = int64_t(m.cfg.d_out);
    hdr[2] = int64_t(m.cfg.tables);
    hdr[3] = int64_t(m.cfg.code_bits);
    hdr[4] = int64_t(m.cfg.variant);
    hdr[5] = int64_t(s.kind);
    hdr[6] = int64_t(s.kind == ProjKind::acdc ? s.depth : s.stages);
    hdr[7] = int64_t(s.block);
    if (blob) std::memcpy(blob, m.proj.blob().data(), m.proj.blob_size() * sizeof(double));
    if (tables) std::memcpy(tables, m.tables.data.data(), m.tables.data.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

// lookup_flops (flops.cpp:51-60) -> MFLOP per token {hash, gather, other}
int ref_lookup_flops(int64_t d_in, int64_t d_out, int64_t h, int64_t tau, int64_t nc, int kind,
                     int64_t stages, int64_t block, int64_t depth, double* out3) {
  try {
    LookupConfig cfg = make_cfg(d_in, d_out, h, tau, 0, nc);
    ProjectionSpec s = make_spec(kind, d_in, h * tau, stages, block, depth);
    FlopReport r = lookup_flops(cfg, s);
    out3[0] = r.hash_mflop;
    out3[1] = r.gather_mflop;
    out3[2] = r.other_mflop;
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

// The reference float32 inference pipeline (bench.cpp:366-386: per tile of
// <= 256 rows, lookup_hash_f32 -> lookup_weights_f32 -> lookup_gather_f32 or
// lookup_gather_sorted_f32) over caller-provided inputs.  The reference runs
// the tiles one after another on one core; with threads > 1 the independent
// tiles are spread over OpenMP threads, each with its own row buffers.
// Returns the wall time in ms of the last of `reps` repetitions.
double ref_pipeline_f32(int64_t d_in, int64_t d_out, int64_t h, int64_t tau, int variant,
                        int kind, int64_t stages, int64_t block, int64_t depth,
                        const float* blob, const float* tables, const float* x, size_t rows,
                        float* y, int threads, int sorted, int reps) {
  LookupConfig cfg = make_cfg(d_in, d_out, h, tau, variant, 1);
  ProjectionSpec spec = make_spec(kind, d_in, h * tau, stages, block, depth);
  const size_t D = spec.transform_width();
  std::vector<float> z(rows * cfg.code_width());
  std::vector<std::uint32_t> codes(rows * cfg.tables);
  std::vector<float> weights(rows * cfg.tables);
  const size_t tile = std::min<size_t>(rows, 256);
  const size_t ntiles = (rows + tile - 1) / tile;
  if (threads < 1) threads = 1;
  double ms = 0.0;
  for (int rep = 0; rep < reps; ++rep) {
    const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel num_threads(threads)
    {
      std::vector<float> buf(D), tmp(D);
      std::vector<std::uint32_t> order(tile);
#pragma omp for schedule(dynamic, 1)
      for (long tix = 0; tix < long(ntiles); ++tix) {
        const size_t r0 = size_t(tix) * tile;
        const size_t r1 = std::min(rows, r0 + tile);
        lookup_hash_f32(x, r0, r1, spec, blob, z.data(), cfg.code_width(), cfg.d_in, buf.data(),
                        tmp.data());
        lookup_weights_f32(z.data(), r0, r1, cfg.tables, cfg.code_bits, cfg.scaled_numerator(),
                           codes.data(), weights.data());
        if (sorted)
          lookup_gather_sorted_f32(tables, cfg.tables, cfg.table_rows(), cfg.d_out, codes.data(),
                                   weights.data(), r0, r1, order.data(), y);
        else
          lookup_gather_f32(tables, cfg.tables, cfg.table_rows(), cfg.d_out, codes.data(),
                            weights.data(), r0, r1, y);
      }
    }
    ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return ms;
}

// The stock public benchmark driver bench_lookup_ffn (bench.cpp:264-350),
// unmodified: its own inputs (seeded), its own timing.  out: {median_ms,
// mean_ms, hash_ms, gather_ms, other_ms, mflop_per_token, gflops,
// timed_allocs}.
int ref_bench_lookup_ffn(int64_t d_in, int64_t d_out, int64_t h, int64_t tau, int variant,
                         int kind, int64_t stages, int64_t block, int64_t depth, size_t rows,
                         size_t reps, size_t warmup, int threads, int sorted, uint64_t seed,
                         double* out8) {
  try {
    BenchSpec bs;
    bs.rows = rows;
    bs.reps = reps;
    bs.warmup = warmup;
    bs.threads = threads;
    bs.sorted_gather = sorted != 0;
    LookupConfig cfg = make_cfg(d_in, d_out, h, tau, variant, 1);
    ProjectionSpec spec = make_spec(kind, d_in, h * tau, stages, block, depth);
    BenchResult r = bench_lookup_ffn(bs, cfg, spec, seed);
    out8[0] = r.median_ms;
    out8[1] = r.mean_ms;
    out8[2] = r.hash_ms;
    out8[3] = r.gather_ms;
    out8[4] = r.other_ms;
    out8[5] = r.mflop_per_token;
    out8[6] = r.gflops;
    out8[7] = double(r.timed_allocs);
    return 0;
  } catch (const std::exception& e) {
    return map_exc(e);
  }
}

}  // extern "C"
