/*
 * lffn_oracle.h -- CPU restatement of the reference LookupFFN forward path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity oracle for the B200 kernels
 * in paper_2403_07221_b200/csrc.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it, and only as the
 * checker.  The product path never links or calls it.
 *
 * Every function restates the reference C++ library (namespace lffn,
 * /root/reference/proj) in plain C11, float64 like the reference's
 * verification path, with the same operation order so that results are
 * bit-identical to the reference built with the same compiler/libm.
 * Pinned against the reference itself (oracle/_ref, built from the reference
 * sources by oracle/Makefile) by tests/test_oracle_pin.py and against the
 * committed fixtures in tests/golden/.
 */
#ifndef LFFN_ORACLE_H
#define LFFN_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG: std::mt19937_64 + libstdc++ distributions (common.hpp:44-55) ---- */
typedef struct orc_rng {
  uint64_t mt[312];
  int idx;
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_canonical(orc_rng* r);
/* fill_gaussian: a fresh std::normal_distribution per call (common.hpp:46-49) */
void orc_fill_gaussian(orc_rng* r, double* out, size_t n, double stddev);
/* fill_signs: std::bernoulli_distribution(0.5) -> +1/-1 (common.hpp:52-55) */
void orc_fill_signs(orc_rng* r, double* out, size_t n);

/* ---- projection (projection.hpp:13-95, projection.cpp) ---- */
enum { ORC_DENSE = 0, ORC_BH = 1, ORC_ACDC = 2, ORC_SIGNFLIP = 3 };

typedef struct orc_proj_spec {
  int64_t d_in, d_out;
  int32_t kind;
  int64_t stages, block, depth;
} orc_proj_spec;

size_t orc_next_pow2(size_t n);
size_t orc_transform_width(const orc_proj_spec* s);
size_t orc_proj_blob_size(const orc_proj_spec* s);
int orc_proj_validate(const orc_proj_spec* s);
int orc_proj_init(const orc_proj_spec* s, uint64_t seed, double* blob);
void orc_fwht(double* v, size_t n);
void orc_block_diag_apply(const double* in, double* out, const double* blocks, size_t D, size_t b);
/* z[n x d_out] = forward(x[n x d_in]); returns 0, or 2 on non-finite input/output */
int orc_proj_forward(const orc_proj_spec* s, const double* blob, const double* x, size_t n,
                     double* z);

/* ---- lookup core (lookup.hpp, lookup.cpp) ---- */
enum { ORC_SOFTMAX = 0, ORC_SCALED = 1, ORC_SIGMOID_TAU1 = 2, ORC_GELU_TAU1 = 3 };

typedef struct orc_cfg {
  int64_t d_in, d_out, tables, code_bits;
  int32_t variant;
  int64_t neighbor_count;
} orc_cfg;

int orc_cfg_validate(const orc_cfg* c);
uint32_t orc_sign_code(const double* z, size_t tau);
void orc_compute_codes(const double* z, size_t n, size_t h, size_t tau, uint32_t* codes,
                       double* abs_z);
double orc_top1_weight(const double* abs_z, size_t tau);
double orc_log_denominator(const double* z, size_t tau);
double orc_code_dot(const double* z, size_t tau, uint32_t code);
/* returns number of codes written (== count) or 0 on error */
size_t orc_neighbor_codes(const double* z, size_t tau, size_t count, uint32_t* out);

/*
 * Full forward (lookup.cpp:191-282).  tables: [h][2^tau][d_out].
 * Optional outputs (may be NULL): z [n x h*tau], codes / weights / dots
 * [n x h x nc] (the LookupCache fields).  Returns 0 ok, 1 size/usage error,
 * 2 non-finite ("hash stage" / "gather stage").
 */
int orc_lookup_forward(const orc_cfg* c, const orc_proj_spec* ps, const double* blob,
                       const double* tables, const double* x, size_t n, double* y, double* z_out,
                       uint32_t* codes_out, double* weights_out, double* dots_out);

/*
 * Projection::backward (projection.cpp:279-386): grad_x [n x d_in] and
 * grad_params [param_count] (accumulated, caller zero-fills) from grad_out
 * [n x d_out]; the bh / acdc stage inputs are recomputed from x as the
 * forward cache holds them (projection.cpp:201-245).  0 ok, 1 usage, 2
 * non-finite ("projection backward input/output").
 */
int orc_proj_backward(const orc_proj_spec* s, const double* blob, const double* x, size_t n,
                      const double* grad_out, double* grad_x, double* grad_params);

/*
 * lookup_backward (lookup.cpp:292-347) at the forward's neighbour selection
 * (recomputed from x): grad_tables [h][2^tau][d_out] and grad_params
 * (accumulated, caller zero-fills), grad_x [n x d_in]; grad_z [n x h*tau]
 * (optional) exposes the straight-through z gradient.
 */
int orc_lookup_backward(const orc_cfg* c, const orc_proj_spec* ps, const double* blob,
                        const double* tables, const double* x, size_t n, const double* grad_y,
                        double* grad_x, double* grad_tables, double* grad_params, double* grad_z);

/* y = sum_k coeff[i,k] * T[k][code[i,k]] for precomputed codes/coeffs (the gather half) */
void orc_gather(const double* tables, size_t h, size_t rows, size_t d_out, const uint32_t* codes,
                const double* coeff, size_t n, double* y);

#ifdef __cplusplus
}
#endif
#endif
