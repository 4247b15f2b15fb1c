// dropin_test.cpp -- the reference's own forward-path checks, re-pointed at
// the GPU through the C++ drop-in (include/lffn_gpu_dropin.hpp).
//
// TEST INFRASTRUCTURE ONLY.  Built by `make -C oracle dropin` against the
// reference headers and sources (the checker side) and liblffn_gpu.so (the
// product side) into oracle/_ref/dropin_test; run by tests/test_gpu_dropin.py
// on the GPU box.  Every case computes lffn::lookup_forward (reference, CPU,
// float64) and lffn::gpu::lookup_forward (device) on the same inputs.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>

#include "lffn_gpu_dropin.hpp"
#include "lookupffn/lookup.hpp"

using namespace lffn;

static int failures = 0;

#define EXPECT(cond, ...)                      \
  do {                                         \
    if (!(cond)) {                             \
      ++failures;                              \
      std::printf("FAIL %s:%d ", __FILE__, __LINE__); \
      std::printf(__VA_ARGS__);                \
      std::printf("\n");                       \
    }                                          \
  } while (0)

static void round_to_f32(DenseMatrix& m) {
  for (double& v : m.data) v = double(float(v));
}

static double l2_rel(const DenseMatrix& a, const DenseMatrix& b) { return l2_rel_diff(a.data, b.data); }

static double maxabs_rel(const DenseMatrix& a, const DenseMatrix& b) {
  double m = 0.0, r = 0.0;
  for (std::size_t i = 0; i < a.data.size(); ++i) {
    m = std::max(m, std::abs(a.data[i] - b.data[i]));
    r = std::max(r, std::abs(b.data[i]));
  }
  return m / std::max(r, 1e-300);
}

static void parity_case(const char* name, const LookupConfig& cfg, const ProjectionSpec& spec,
                        std::size_t n, std::uint64_t seed, double table_std) {
  auto rng = make_rng(seed);
  DenseMatrix x = DenseMatrix::gaussian(n, cfg.d_in, rng);
  round_to_f32(x);
  Projection p = Projection::init(spec, seed + 1);
  HashTables t = HashTables::zeros_like(cfg);
  auto trng = make_rng(seed + 2);
  fill_gaussian(t.data, trng, table_std);
  HashTables t32 = t;  // the device stores float32 tables
  for (double& v : t32.data) v = double(float(v));
  const DenseMatrix y_ref = lookup_forward(x, p, t32, cfg);
  const DenseMatrix y_gpu = gpu::lookup_forward(x, p, t, cfg);
  const double e1 = l2_rel(y_gpu, y_ref), e2 = maxabs_rel(y_gpu, y_ref);
  std::printf("%-28s n=%zu l2_rel=%.2e maxabs_rel=%.2e\n", name, n, e1, e2);
  EXPECT(e1 <= 1e-5 && e2 <= 1e-5, "%s parity", name);
}

int main() {
  // BASELINE c1 and c2-shaped forwards, all device projection kinds
  {
    LookupConfig c1{.d_in = 64, .d_out = 64, .tables = 8, .code_bits = 4};
    parity_case("c1 signflip", c1, ProjectionSpec::signflip(64, 32), 1024, 0, 0.02);
    parity_case("c1 dense", c1, ProjectionSpec::dense(64, 32), 512, 0, 0.02);
    parity_case("c1 acdc", c1, ProjectionSpec::acdc(64, 32, 2), 512, 0, 0.02);
    LookupConfig c2{.d_in = 768, .d_out = 768, .tables = 256, .code_bits = 8};
    parity_case("c2 signflip (256 tok)", c2, ProjectionSpec::signflip(768, 2048), 256, 0, 0.02);
    LookupConfig sc{.d_in = 50, .d_out = 30, .tables = 12, .code_bits = 10,
                    .variant = LookupVariant::scaled};
    parity_case("scaled, pad+truncate", sc, ProjectionSpec::signflip(50, 120), 33, 5, 0.02);
  }
  // test_lookup.cpp:207-230 -- zero projection spreads mass as 2^-tau
  {
    LookupConfig cfg{.d_in = 6, .d_out = 5, .tables = 3, .code_bits = 4};
    Projection proj = Projection::from_blob(ProjectionSpec::dense(6, 12), std::vector<double>(72, 0.0));
    HashTables tables = HashTables::init(cfg, 31);
    auto rng = make_rng(30);
    DenseMatrix x = DenseMatrix::gaussian(2, 6, rng);
    const DenseMatrix y = gpu::lookup_forward(x, proj, tables, cfg);
    for (std::size_t i = 0; i < 2; ++i)
      for (std::size_t j = 0; j < 5; ++j) {
        double expected = 0.0;
        for (std::size_t k = 0; k < 3; ++k) expected += double(float(tables.row(k, 15)[j])) / 16.0;
        EXPECT(std::abs(y.at(i, j) - expected) <= 1e-6 * std::abs(expected) + 1e-9, "zero proj");
      }
  }
  // neighbor_count > 1 (lookup.cpp:118-165, 231-262) against the reference
  {
    LookupConfig n3{.d_in = 64, .d_out = 64, .tables = 8, .code_bits = 4, .neighbor_count = 3};
    parity_case("c1 signflip nc=3", n3, ProjectionSpec::signflip(64, 32), 512, 0, 0.02);
    LookupConfig n5{.d_in = 50, .d_out = 30, .tables = 12, .code_bits = 10,
                    .variant = LookupVariant::scaled, .neighbor_count = 5};
    parity_case("scaled nc=5 pad+truncate", n5, ProjectionSpec::signflip(50, 120), 33, 5, 0.02);
    LookupConfig n4{.d_in = 64, .d_out = 64, .tables = 8, .code_bits = 4, .neighbor_count = 4};
    parity_case("dense nc=4", n4, ProjectionSpec::dense(64, 32), 128, 3, 0.02);
  }
  // test_lookup.cpp:251-272 -- full-neighbour forward (nc = 2^tau), bh, both variants
  for (LookupVariant variant : {LookupVariant::softmax, LookupVariant::scaled}) {
    LookupConfig cfg{.d_in = 8, .d_out = 6, .tables = 2, .code_bits = 3, .variant = variant,
                     .neighbor_count = 8};
    parity_case(variant == LookupVariant::softmax ? "full codebook softmax" : "full codebook scaled",
                cfg, ProjectionSpec::bh(8, 6, 2, 4), 16, 33, 0.5);
  }
  // test_lookup.cpp:274-342 -- tau = 1 sigmoid / GELU constructions (nc = 2)
  for (LookupVariant variant : {LookupVariant::sigmoid_tau1, LookupVariant::gelu_tau1}) {
    const std::size_t d = 7, units = 9, d_out = 4;
    auto rng = make_rng(36);
    const DenseMatrix w = DenseMatrix::gaussian(units, d, rng);
    const DenseMatrix v = DenseMatrix::gaussian(units, d_out, rng);
    LookupConfig cfg{.d_in = d, .d_out = d_out, .tables = units, .code_bits = 1,
                     .variant = variant, .neighbor_count = 2};
    const double sw = variant == LookupVariant::sigmoid_tau1 ? 0.5 : 0.851;
    const double sv = variant == LookupVariant::sigmoid_tau1 ? 1.0 : 1.175;
    std::vector<double> blob(d * units);
    for (std::size_t k = 0; k < units; ++k)
      for (std::size_t c = 0; c < d; ++c) blob[c * units + k] = sw * w.at(k, c);
    Projection proj = Projection::from_blob(ProjectionSpec::dense(d, units), blob);
    HashTables tables = HashTables::zeros_like(cfg);
    for (std::size_t k = 0; k < units; ++k)
      for (std::size_t j = 0; j < d_out; ++j) tables.row(k, 1)[j] = double(float(sv * v.at(k, j)));
    DenseMatrix x = DenseMatrix::gaussian(12, d, rng);
    round_to_f32(x);
    const DenseMatrix y_ref = lookup_forward(x, proj, tables, cfg);
    const DenseMatrix y_gpu = gpu::lookup_forward(x, proj, tables, cfg);
    const double e1 = l2_rel(y_gpu, y_ref), e2 = maxabs_rel(y_gpu, y_ref);
    std::printf("%-28s l2_rel=%.2e maxabs_rel=%.2e\n",
                variant == LookupVariant::sigmoid_tau1 ? "tau1 sigmoid nc=2" : "tau1 gelu nc=2", e1, e2);
    EXPECT(e1 <= 1e-5 && e2 <= 1e-5, "tau1 construction parity");
    if (variant == LookupVariant::gelu_tau1) {
      // GELU(0) = 0: the scaled numerator zeroes at z = 0
      const DenseMatrix zeros(3, d);
      const DenseMatrix y0 = gpu::lookup_forward(zeros, proj, tables, cfg);
      for (double val : y0.data) EXPECT(val == 0.0, "gelu(0) == 0");
    }
  }
  // test_lookup.cpp:232-249 -- tau = 1 with equal rows halves the sum
  {
    LookupConfig cfg{.d_in = 4, .d_out = 3, .tables = 5, .code_bits = 1};
    Projection proj = Projection::from_blob(ProjectionSpec::dense(4, 5), std::vector<double>(20, 0.0));
    HashTables tables = HashTables::zeros_like(cfg);
    const double v[3] = {0.5, -1.0, 2.0};
    for (std::size_t k = 0; k < 5; ++k)
      for (std::uint32_t c = 0; c < 2; ++c) std::copy(v, v + 3, tables.row(k, c));
    DenseMatrix x(1, 4);
    x.at(0, 1) = 0.3;
    const DenseMatrix y = gpu::lookup_forward(x, proj, tables, cfg);
    for (std::size_t j = 0; j < 3; ++j) EXPECT(std::abs(y.at(0, j) - 2.5 * v[j]) < 1e-6, "tau1");
  }
  // test_lookup.cpp:477-500 -- validation errors keep the reference's types
  {
    LookupConfig cfg{.d_in = 8, .d_out = 4, .tables = 2, .code_bits = 3};
    Projection bad = Projection::init(ProjectionSpec::dense(8, 5), 1);
    HashTables tables = HashTables::init(cfg, 2);
    DenseMatrix x(2, 8);
    bool threw = false;
    try {
      gpu::lookup_forward(x, bad, tables, cfg);
    } catch (const SizeError&) {
      threw = true;
    }
    EXPECT(threw, "SizeError on projection width");
    cfg.neighbor_count = 9;
    threw = false;
    try {
      gpu::lookup_forward(x, bad, tables, cfg);
    } catch (const SizeError&) {
      threw = true;
    }
    EXPECT(threw, "SizeError on neighbor count");
  }
  // NumericError names the stage (lookup.cpp:204, projection.cpp:172)
  {
    LookupConfig cfg{.d_in = 8, .d_out = 4, .tables = 2, .code_bits = 3};
    Projection proj = Projection::init(ProjectionSpec::signflip(8, 6), 1);
    HashTables tables = HashTables::init(cfg, 2);
    DenseMatrix x(2, 8);
    x.at(1, 3) = std::nan("");
    std::string what;
    try {
      gpu::lookup_forward(x, proj, tables, cfg);
    } catch (const NumericError& e) {
      what = e.what();
    }
    EXPECT(what.find("projection forward input") != std::string::npos, "NumericError stage: %s",
           what.c_str());
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
