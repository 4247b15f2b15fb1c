/*
 * lffn_oracle.c -- plain-C restatement of the reference LookupFFN forward.
 *
 * TEST INFRASTRUCTURE ONLY (the parity checker).  See lffn_oracle.h.
 * Each function cites the reference file:line it restates; paths are
 * relative to /root/reference/proj.  Arithmetic is float64 in the same
 * operation order as the reference so that, compiled for baseline x86-64
 * (no FMA contraction) against the same libm, outputs are bit-identical to
 * the reference library (checked by tests/test_oracle_pin.py).
 */
#include "lffn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (the engine behind make_rng, include/lookupffn/common.hpp:44) */
/* ------------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ull
#define MT_LOWER 0x000000007FFFFFFFull

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
}

static void mt_twist(orc_rng* r) {
  for (int i = 0; i < MT_N; ++i) {
    uint64_t y = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
    uint64_t v = r->mt[(i + MT_M) % MT_N] ^ (y >> 1);
    if (y & 1ull) v ^= 0xB5026F5AA96619E9ull;
    r->mt[i] = v;
  }
  r->idx = 0;
}

uint64_t orc_rng_next(orc_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t z = r->mt[r->idx++];
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= z >> 43;
  return z;
}

/* std::generate_canonical<double, 53>(mt19937_64): one 64-bit draw / 2^64,
 * clamped below 1 (libstdc++ <bits/random.tcc>). */
double orc_canonical(orc_rng* r) {
  double sum = (double)orc_rng_next(r);
  double ret = sum / 18446744073709551616.0;
  if (ret >= 1.0) ret = nextafter(1.0, 0.0);
  return ret;
}

/* fill_gaussian (common.hpp:46-49): std::normal_distribution<double>, which
 * libstdc++ implements with the Marsaglia polar method, caching the second
 * deviate inside the distribution object (one object per fill call). */
void orc_fill_gaussian(orc_rng* r, double* out, size_t n, double stddev) {
  int saved_ok = 0;
  double saved = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double ret;
    if (saved_ok) {
      saved_ok = 0;
      ret = saved;
    } else {
      double x, y, r2;
      do {
        x = 2.0 * orc_canonical(r) - 1.0;
        y = 2.0 * orc_canonical(r) - 1.0;
        r2 = x * x + y * y;
      } while (r2 > 1.0 || r2 == 0.0);
      const double mult = sqrt(-2 * log(r2) / r2);
      saved = x * mult;
      saved_ok = 1;
      ret = y * mult;
    }
    out[i] = ret * stddev + 0.0;
  }
}

/* fill_signs (common.hpp:52-55): bernoulli_distribution(0.5) is
 * canonical() < 0.5. */
void orc_fill_signs(orc_rng* r, double* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = (orc_canonical(r) < 0.5) ? 1.0 : -1.0;
}

/* ------------------------------------------------------------------------ */
/* Projection                                                               */
/* ------------------------------------------------------------------------ */

/* next_power_of_two (common.hpp:66-70) */
size_t orc_next_pow2(size_t n) {
  size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

/* ProjectionSpec::transform_width (projection.hpp:30) */
size_t orc_transform_width(const orc_proj_spec* s) {
  size_t a = (size_t)s->d_in, b = (size_t)s->d_out;
  return orc_next_pow2(a > b ? a : b);
}

/* ProjectionSpec::validate (projection.cpp:29-40); 1 = SizeError */
int orc_proj_validate(const orc_proj_spec* s) {
  if (s->d_in <= 0 || s->d_out <= 0) return 1;
  const size_t D = orc_transform_width(s);
  if (s->kind == ORC_BH) {
    const size_t b = s->block == 0 ? D : (size_t)s->block;
    if (s->stages <= 0) return 1;
    if (b > D || D % b != 0) return 1;
  }
  if (s->kind == ORC_ACDC && s->depth <= 0) return 1;
  if (s->kind < 0 || s->kind > 3) return 1;
  return 0;
}

/* blob_size_for (projection.cpp:81-93) */
size_t orc_proj_blob_size(const orc_proj_spec* s) {
  const size_t D = orc_transform_width(s);
  switch (s->kind) {
    case ORC_DENSE: return (size_t)s->d_in * (size_t)s->d_out;
    case ORC_BH: {
      const size_t b = s->block == 0 ? D : (size_t)s->block;
      return (size_t)s->stages * (D / b) * b * b;
    }
    case ORC_ACDC: return 2 * (size_t)s->depth * D;
    case ORC_SIGNFLIP: return 3 * D;
  }
  return 0;
}

/* fill_orthogonal (projection.cpp:60-79): Gaussian draw from a fresh
 * normal_distribution, then modified Gram-Schmidt over columns. */
static void fill_orthogonal(double* out, size_t b, orc_rng* rng) {
  orc_fill_gaussian(rng, out, b * b, 1.0);
  for (size_t c = 0; c < b; ++c) {
    for (size_t prev = 0; prev < c; ++prev) {
      double dot = 0.0;
      for (size_t r = 0; r < b; ++r) dot += out[r * b + c] * out[r * b + prev];
      for (size_t r = 0; r < b; ++r) out[r * b + c] -= dot * out[r * b + prev];
    }
    double norm = 0.0;
    for (size_t r = 0; r < b; ++r) norm += out[r * b + c] * out[r * b + c];
    norm = sqrt(norm);
    if (norm < 1e-12) {
      for (size_t r = 0; r < b; ++r) out[r * b + c] = (r == c) ? 1.0 : 0.0;
      continue;
    }
    for (size_t r = 0; r < b; ++r) out[r * b + c] /= norm;
  }
}

/* Projection::init (projection.cpp:97-135) */
int orc_proj_init(const orc_proj_spec* s, uint64_t seed, double* blob) {
  if (orc_proj_validate(s)) return 1;
  const size_t n = orc_proj_blob_size(s);
  memset(blob, 0, n * sizeof(double));
  orc_rng rng;
  orc_rng_seed(&rng, seed);
  const size_t D = orc_transform_width(s);
  switch (s->kind) {
    case ORC_DENSE:
      orc_fill_gaussian(&rng, blob, n, 1.0 / sqrt((double)s->d_in));
      break;
    case ORC_BH: {
      const size_t b = s->block == 0 ? D : (size_t)s->block;
      const double scale = 1.0 / sqrt((double)D);
      for (size_t blk = 0; blk < n / (b * b); ++blk) {
        double* out = blob + blk * b * b;
        fill_orthogonal(out, b, &rng);
        for (size_t i = 0; i < b * b; ++i) out[i] *= scale;
      }
      break;
    }
    case ORC_ACDC: {
      orc_fill_signs(&rng, blob, n);
      const double scale = 1.0 / sqrt((double)D);
      for (size_t i = 0; i < n; ++i) blob[i] *= scale;
      break;
    }
    case ORC_SIGNFLIP:
      orc_fill_signs(&rng, blob, n);
      break;
  }
  return 0;
}

/* fwht_kernel (include/lookupffn/fwht.hpp:28-41): unnormalized Sylvester
 * transform, stage order half = 1, 2, 4, ... */
void orc_fwht(double* v, size_t n) {
  for (size_t half = 1; half < n; half <<= 1) {
    for (size_t block = 0; block < n; block += half << 1) {
      for (size_t j = block; j < block + half; ++j) {
        double x = v[j];
        double y = v[j + half];
        v[j] = x + y;
        v[j + half] = x - y;
      }
    }
  }
}

/* detail::block_diag_apply (projection.hpp:101-119) */
void orc_block_diag_apply(const double* in, double* out, const double* blocks, size_t D,
                          size_t b) {
  const size_t groups = D / b;
  for (size_t g = 0; g < groups; ++g) {
    const double* blk = blocks + g * b * b;
    const double* src = in + g * b;
    double* dst = out + g * b;
    for (size_t c = 0; c < b; ++c) dst[c] = 0.0;
    for (size_t r = 0; r < b; ++r) {
      const double sv = src[r];
      const double* brow = blk + r * b;
      for (size_t c = 0; c < b; ++c) dst[c] += sv * brow[c];
    }
  }
}

static int all_finite(const double* v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

/* Projection::forward_impl (projection.cpp:167-266); rows are independent,
 * so the row loop may run in parallel without changing any result. */
int orc_proj_forward(const orc_proj_spec* s, const double* blob, const double* x, size_t n,
                     double* z) {
  if (orc_proj_validate(s)) return 1;
  const size_t d_in = (size_t)s->d_in, d_out = (size_t)s->d_out;
  if (!all_finite(x, n * d_in)) return 2; /* "projection forward input" */
  const size_t D = orc_transform_width(s);
  if (s->kind == ORC_DENSE) {
    const double* w = blob; /* d_in x d_out */
#pragma omp parallel for schedule(static)
    for (long i = 0; i < (long)n; ++i) {
      const double* xi = x + (size_t)i * d_in;
      double* zi = z + (size_t)i * d_out;
      for (size_t j = 0; j < d_out; ++j) zi[j] = 0.0;
      for (size_t k = 0; k < d_in; ++k) {
        const double sv = xi[k];
        const double* wrow = w + k * d_out;
        for (size_t j = 0; j < d_out; ++j) zi[j] += sv * wrow[j];
      }
    }
    return all_finite(z, n * d_out) ? 0 : 2; /* "projection forward output" */
  }
#pragma omp parallel
  {
    double* buf = (double*)malloc(D * sizeof(double));
    double* tmp = (double*)malloc(D * sizeof(double));
#pragma omp for schedule(static)
    for (long i = 0; i < (long)n; ++i) {
      for (size_t j = 0; j < D; ++j) buf[j] = 0.0;
      memcpy(buf, x + (size_t)i * d_in, d_in * sizeof(double));
      if (s->kind == ORC_BH) {
        const size_t b = s->block == 0 ? D : (size_t)s->block;
        const size_t stage_size = (D / b) * b * b;
        for (int64_t st = 0; st < s->stages; ++st) {
          orc_block_diag_apply(buf, tmp, blob + (size_t)st * stage_size, D, b);
          double* t = buf;
          buf = tmp;
          tmp = t;
          orc_fwht(buf, D);
        }
      } else if (s->kind == ORC_ACDC) {
        for (int64_t st = 0; st < s->depth; ++st) {
          const double* a = blob + 2 * (size_t)st * D;
          const double* d = a + D;
          for (size_t j = 0; j < D; ++j) buf[j] *= a[j];
          orc_fwht(buf, D);
          for (size_t j = 0; j < D; ++j) buf[j] *= d[j];
          orc_fwht(buf, D);
        }
      } else { /* signflip (projection.cpp:248-258) */
        for (size_t st = 0; st < 3; ++st) {
          const double* sv = blob + st * D;
          for (size_t j = 0; j < D; ++j) buf[j] *= sv[j];
          orc_fwht(buf, D);
        }
      }
      memcpy(z + (size_t)i * d_out, buf, d_out * sizeof(double));
    }
    free(buf);
    free(tmp);
  }
  return all_finite(z, n * d_out) ? 0 : 2;
}

/* ------------------------------------------------------------------------ */
/* Lookup core                                                              */
/* ------------------------------------------------------------------------ */

/* LookupConfig::validate (lookup.cpp:27-37); 1 = SizeError */
int orc_cfg_validate(const orc_cfg* c) {
  if (c->d_in <= 0 || c->d_out <= 0) return 1;
  if (c->tables <= 0) return 1;
  if (c->code_bits < 1 || c->code_bits > 24) return 1;
  if (c->neighbor_count < 1 || c->neighbor_count > ((int64_t)1 << c->code_bits)) return 1;
  if ((c->variant == ORC_SIGMOID_TAU1 || c->variant == ORC_GELU_TAU1) && c->code_bits != 1)
    return 1;
  if (c->variant < 0 || c->variant > 3) return 1;
  return 0;
}

/* sign_code (lookup.cpp:74-79): bit j <- [z_j >= 0], LSB first */
uint32_t orc_sign_code(const double* z, size_t tau) {
  uint32_t code = 0;
  for (size_t j = 0; j < tau; ++j)
    if (z[j] >= 0.0) code |= (1u << j);
  return code;
}

/* compute_codes (lookup.cpp:81-100) */
void orc_compute_codes(const double* z, size_t n, size_t h, size_t tau, uint32_t* codes,
                       double* abs_z) {
  for (size_t ik = 0; ik < n * h; ++ik) {
    const double* zz = z + ik * tau;
    uint32_t code = 0;
    for (size_t j = 0; j < tau; ++j) {
      if (zz[j] >= 0.0) code |= (1u << j);
      if (abs_z) abs_z[ik * tau + j] = fabs(zz[j]);
    }
    codes[ik] = code;
  }
}

/* top1_weight (lookup.cpp:185-189): prod_j 1/(1+exp(-2|z_j|)) by repeated division */
double orc_top1_weight(const double* abs_z, size_t tau) {
  double w = 1.0;
  for (size_t j = 0; j < tau; ++j) w /= 1.0 + exp(-2.0 * abs_z[j]);
  return w;
}

/* log_denominator (lookup.cpp:102-109) */
double orc_log_denominator(const double* z, size_t tau) {
  double acc = 0.0;
  for (size_t j = 0; j < tau; ++j) {
    const double a = fabs(z[j]);
    acc += a + log1p(exp(-2.0 * a));
  }
  return acc;
}

/* code_dot (lookup.cpp:111-116) */
double orc_code_dot(const double* z, size_t tau, uint32_t code) {
  double acc = 0.0;
  for (size_t j = 0; j < tau; ++j) acc += ((code >> j) & 1u) ? z[j] : -z[j];
  return acc;
}

/* neighbor_codes (lookup.cpp:118-165).  The frontier is a
 * std::priority_queue<Node, vector, greater<Node>>; ties in cost are broken
 * by the heap layout, so the libstdc++ push_heap / pop_heap (<bits/stl_heap.h>)
 * sift order is restated exactly. */
typedef struct nb_node {
  double cost;
  uint32_t mask;
  uint32_t last;
} nb_node;

static int nb_greater(const nb_node* a, const nb_node* b) { return a->cost > b->cost; }

static void nb_push_up(nb_node* first, long hole, long top, nb_node value) {
  long parent = (hole - 1) / 2;
  while (hole > top && nb_greater(&first[parent], &value)) {
    first[hole] = first[parent];
    hole = parent;
    parent = (hole - 1) / 2;
  }
  first[hole] = value;
}

static void nb_push(nb_node* heap, long* len, nb_node v) {
  heap[*len] = v;
  *len += 1;
  nb_push_up(heap, *len - 1, 0, heap[*len - 1]);
}

static void nb_adjust(nb_node* first, long hole, long len, nb_node value) {
  const long top = hole;
  long second = hole;
  while (second < (len - 1) / 2) {
    second = 2 * (second + 1);
    if (nb_greater(&first[second], &first[second - 1])) second--;
    first[hole] = first[second];
    hole = second;
  }
  if ((len & 1) == 0 && second == (len - 2) / 2) {
    second = 2 * (second + 1);
    first[hole] = first[second - 1];
    hole = second - 1;
  }
  nb_push_up(first, hole, top, value);
}

static nb_node nb_pop(nb_node* heap, long* len) {
  nb_node top = heap[0];
  if (*len > 1) {
    long last = *len - 1;
    nb_node value = heap[last];
    heap[last] = heap[0];
    nb_adjust(heap, 0, last, value);
  }
  *len -= 1;
  return top;
}

typedef struct nb_mag {
  double a;
  uint32_t j;
} nb_mag;

static int nb_mag_cmp(const void* pa, const void* pb) {
  const nb_mag* a = (const nb_mag*)pa;
  const nb_mag* b = (const nb_mag*)pb;
  if (a->a < b->a) return -1;
  if (b->a < a->a) return 1;
  return (a->j < b->j) ? -1 : (a->j > b->j);
}

size_t orc_neighbor_codes(const double* z, size_t tau, size_t count, uint32_t* out) {
  if (tau == 0 || tau > 24) return 0;
  const size_t total = (size_t)1 << tau;
  if (count > total) return 0;
  size_t nout = 0;
  const uint32_t base = orc_sign_code(z, tau);
  out[nout++] = base;
  if (count == 1) return 1;
  nb_mag mag[24];
  for (size_t j = 0; j < tau; ++j) {
    mag[j].a = fabs(z[j]);
    mag[j].j = (uint32_t)j;
  }
  qsort(mag, tau, sizeof(nb_mag), nb_mag_cmp);
  nb_node* heap = (nb_node*)malloc(sizeof(nb_node) * (2 * count + 4));
  long len = 0;
  nb_node first = {mag[0].a, 1u, 0u};
  nb_push(heap, &len, first);
  while (nout < count && len > 0) {
    const nb_node node = nb_pop(heap, &len);
    uint32_t code = base;
    for (size_t p = 0; p < tau; ++p)
      if ((node.mask >> p) & 1u) code ^= (1u << mag[p].j);
    out[nout++] = code;
    if (node.last + 1 < tau) {
      nb_node a = {node.cost + mag[node.last + 1].a, node.mask | (1u << (node.last + 1)),
                   node.last + 1};
      nb_push(heap, &len, a);
      nb_node b = {node.cost - mag[node.last].a + mag[node.last + 1].a,
                   (node.mask ^ (1u << node.last)) | (1u << (node.last + 1)), node.last + 1};
      nb_push(heap, &len, b);
    }
  }
  free(heap);
  return nout;
}

/* forward_impl (lookup.cpp:191-275) + lookup_forward (:279-282).  The
 * reference walks rows serially; every row is independent, so rows are split
 * across threads here with identical per-row arithmetic. */
int orc_lookup_forward(const orc_cfg* c, const orc_proj_spec* ps, const double* blob,
                       const double* tables, const double* x, size_t n, double* y, double* z_out,
                       uint32_t* codes_out, double* weights_out, double* dots_out) {
  if (orc_cfg_validate(c)) return 1;                                   /* check_shapes */
  if (ps->d_in != c->d_in || ps->d_out != c->tables * c->code_bits) return 1;
  const size_t h = (size_t)c->tables, tau = (size_t)c->code_bits;
  const size_t nc = (size_t)c->neighbor_count, d_out = (size_t)c->d_out;
  const size_t rows = (size_t)1 << tau;
  const int scaled = (c->variant == ORC_SCALED || c->variant == ORC_GELU_TAU1);
  double* z = z_out ? z_out : (double*)malloc(sizeof(double) * n * h * tau + 8);
  int rc = orc_proj_forward(ps, blob, x, n, z);
  if (rc != 0) {
    if (!z_out) free(z);
    return rc; /* "hash stage" */
  }
  int bad = 0;
#pragma omp parallel reduction(| : bad)
  {
    uint32_t* local = (uint32_t*)malloc(sizeof(uint32_t) * (nc + 1));
    double absz[24];
#pragma omp for schedule(static)
    for (long i = 0; i < (long)n; ++i) {
      double* yi = y + (size_t)i * d_out;
      for (size_t j = 0; j < d_out; ++j) yi[j] = 0.0;
      for (size_t k = 0; k < h; ++k) {
        const size_t ik = (size_t)i * h + k;
        const double* zk = z + ik * tau;
        uint32_t top = orc_sign_code(zk, tau);
        for (size_t j = 0; j < tau; ++j) absz[j] = fabs(zk[j]);
        const uint32_t* codes = &top;
        size_t count = 1;
        if (nc > 1) {
          count = orc_neighbor_codes(zk, tau, nc, local);
          codes = local;
        }
        double logden = 0.0, sum_abs = 0.0;
        if (nc > 1)
          logden = orc_log_denominator(zk, tau);
        else
          for (size_t j = 0; j < tau; ++j) sum_abs += absz[j];
        for (size_t cc = 0; cc < count; ++cc) {
          const uint32_t code = codes[cc];
          const double dot = (nc == 1) ? sum_abs : orc_code_dot(zk, tau, code);
          const double w = (nc == 1) ? orc_top1_weight(absz, tau) : exp(dot - logden);
          const double coeff = scaled ? w * dot : w;
          const double* trow = tables + (k * rows + code) * d_out;
          for (size_t j = 0; j < d_out; ++j) yi[j] += coeff * trow[j];
          const size_t slot = ik * nc + cc;
          if (codes_out) codes_out[slot] = code;
          if (weights_out) weights_out[slot] = w;
          if (dots_out) dots_out[slot] = dot;
        }
      }
      if (!all_finite(yi, d_out)) bad = 1; /* "gather stage" */
    }
    free(local);
  }
  if (!z_out) free(z);
  return bad ? 2 : 0;
}

/* block_diag_apply_transposed (projection.hpp:122-137) */
static void orc_block_diag_apply_transposed(const double* in, double* out, const double* blocks,
                                            size_t D, size_t b) {
  const size_t groups = D / b;
  for (size_t g = 0; g < groups; ++g) {
    const double* blk = blocks + g * b * b;
    const double* src = in + g * b;
    double* dst = out + g * b;
    for (size_t r = 0; r < b; ++r) {
      double acc = 0.0;
      const double* brow = blk + r * b;
      for (size_t c = 0; c < b; ++c) acc += brow[c] * src[c];
      dst[r] = acc;
    }
  }
}

/* Projection::backward (projection.cpp:279-386).  Rows are visited in order
 * (the reference's gradient accumulation over rows is sequential). */
int orc_proj_backward(const orc_proj_spec* s, const double* blob, const double* x, size_t n,
                      const double* grad_out, double* grad_x, double* grad_params) {
  if (orc_proj_validate(s)) return 1;
  const size_t d_in = (size_t)s->d_in, d_out = (size_t)s->d_out;
  if (!all_finite(grad_out, n * d_out)) return 2; /* "projection backward input" */
  const size_t D = orc_transform_width(s);
  if (s->kind == ORC_DENSE) {
    for (size_t i = 0; i < n; ++i) {
      const double* gi = grad_out + i * d_out;
      const double* xi = x + i * d_in;
      double* gxi = grad_x + i * d_in;
      for (size_t k = 0; k < d_in; ++k) {
        const double* wrow = blob + k * d_out;
        double* gwrow = grad_params + k * d_out;
        double acc = 0.0;
        const double xv = xi[k];
        for (size_t j = 0; j < d_out; ++j) {
          acc += gi[j] * wrow[j];
          gwrow[j] += xv * gi[j];
        }
        gxi[k] = acc;
      }
    }
    return all_finite(grad_x, n * d_in) ? 0 : 2;
  }
  double* g = (double*)malloc(D * sizeof(double));
  double* tmp = (double*)malloc(D * sizeof(double));
  const size_t nst = s->kind == ORC_BH ? (size_t)s->stages : s->kind == ORC_ACDC ? 2 * (size_t)s->depth : 0;
  double* stage_in = nst ? (double*)malloc(nst * D * sizeof(double)) : NULL;
  for (size_t i = 0; i < n; ++i) {
    if (nst) {
      /* the forward's cached stage inputs for row i (projection.cpp:216-245) */
      double* buf = g;
      for (size_t j = 0; j < D; ++j) buf[j] = 0.0;
      memcpy(buf, x + i * d_in, d_in * sizeof(double));
      if (s->kind == ORC_BH) {
        const size_t b = s->block == 0 ? D : (size_t)s->block;
        const size_t stage_size = (D / b) * b * b;
        for (size_t st = 0; st < nst; ++st) {
          memcpy(stage_in + st * D, buf, D * sizeof(double));
          orc_block_diag_apply(buf, tmp, blob + st * stage_size, D, b);
          memcpy(buf, tmp, D * sizeof(double));
          orc_fwht(buf, D);
        }
      } else {
        for (size_t st = 0; st < (size_t)s->depth; ++st) {
          const double* a = blob + 2 * st * D;
          const double* d = a + D;
          memcpy(stage_in + 2 * st * D, buf, D * sizeof(double));
          for (size_t j = 0; j < D; ++j) buf[j] *= a[j];
          orc_fwht(buf, D);
          memcpy(stage_in + (2 * st + 1) * D, buf, D * sizeof(double));
          for (size_t j = 0; j < D; ++j) buf[j] *= d[j];
          orc_fwht(buf, D);
        }
      }
    }
    for (size_t j = 0; j < D; ++j) g[j] = 0.0;
    memcpy(g, grad_out + i * d_out, d_out * sizeof(double));
    if (s->kind == ORC_BH) {
      const size_t b = s->block == 0 ? D : (size_t)s->block;
      const size_t groups = D / b, stage_size = groups * b * b;
      for (size_t st = (size_t)s->stages; st-- > 0;) {
        orc_fwht(g, D);
        const double* in = stage_in + st * D;
        double* gblk = grad_params + st * stage_size;
        for (size_t grp = 0; grp < groups; ++grp) {
          const double* src = in + grp * b;
          const double* gdst = g + grp * b;
          double* gb = gblk + grp * b * b;
          for (size_t r = 0; r < b; ++r) {
            const double sv = src[r];
            double* gbrow = gb + r * b;
            for (size_t c = 0; c < b; ++c) gbrow[c] += sv * gdst[c];
          }
        }
        orc_block_diag_apply_transposed(g, tmp, blob + st * stage_size, D, b);
        memcpy(g, tmp, D * sizeof(double));
      }
    } else if (s->kind == ORC_ACDC) {
      for (size_t st = (size_t)s->depth; st-- > 0;) {
        const double* a = blob + 2 * st * D;
        const double* d = a + D;
        double* ga = grad_params + 2 * st * D;
        double* gd = ga + D;
        const double* pre_a = stage_in + 2 * st * D;
        const double* pre_d = stage_in + (2 * st + 1) * D;
        orc_fwht(g, D);
        for (size_t j = 0; j < D; ++j) {
          gd[j] += pre_d[j] * g[j];
          g[j] *= d[j];
        }
        orc_fwht(g, D);
        for (size_t j = 0; j < D; ++j) {
          ga[j] += pre_a[j] * g[j];
          g[j] *= a[j];
        }
      }
    } else { /* signflip */
      for (size_t st = 3; st-- > 0;) {
        const double* sv = blob + st * D;
        orc_fwht(g, D);
        for (size_t j = 0; j < D; ++j) g[j] *= sv[j];
      }
    }
    memcpy(grad_x + i * d_in, g, d_in * sizeof(double));
  }
  free(g);
  free(tmp);
  free(stage_in);
  return all_finite(grad_x, n * d_in) ? 0 : 2; /* "projection backward output" */
}

/* lookup_backward (lookup.cpp:292-347) */
int orc_lookup_backward(const orc_cfg* c, const orc_proj_spec* ps, const double* blob,
                        const double* tables, const double* x, size_t n, const double* grad_y,
                        double* grad_x, double* grad_tables, double* grad_params, double* grad_z) {
  if (orc_cfg_validate(c)) return 1;
  const size_t h = (size_t)c->tables, tau = (size_t)c->code_bits, nc = (size_t)c->neighbor_count;
  const size_t d_out = (size_t)c->d_out, rows = (size_t)1 << tau, cw = h * tau;
  const int scaled = (c->variant == ORC_SCALED || c->variant == ORC_GELU_TAU1);
  if (!all_finite(grad_y, n * d_out)) return 2; /* "lookup backward input" */
  double* y = (double*)malloc(sizeof(double) * (n * d_out + 1));
  double* z = (double*)malloc(sizeof(double) * (n * cw + 1));
  uint32_t* codes = (uint32_t*)malloc(sizeof(uint32_t) * (n * h * nc + 1));
  double* w = (double*)malloc(sizeof(double) * (n * h * nc + 1));
  double* dots = (double*)malloc(sizeof(double) * (n * h * nc + 1));
  double* gz = grad_z ? grad_z : (double*)malloc(sizeof(double) * (n * cw + 1));
  int rc = orc_lookup_forward(c, ps, blob, tables, x, n, y, z, codes, w, dots);
  if (rc == 0) {
    for (size_t q = 0; q < n * cw; ++q) gz[q] = 0.0;
    for (size_t i = 0; i < n; ++i) {
      const double* gy = grad_y + i * d_out;
      for (size_t k = 0; k < h; ++k) {
        const size_t ik = i * h + k;
        const double* zk = z + ik * tau;
        double* g = gz + i * cw + k * tau;
        for (size_t cc = 0; cc < nc; ++cc) {
          const size_t slot = ik * nc + cc;
          const uint32_t code = codes[slot];
          const double wt = w[slot], dot = dots[slot];
          const double coeff = scaled ? wt * dot : wt;
          const double* trow = tables + (k * rows + code) * d_out;
          double* gtrow = grad_tables + (k * rows + code) * d_out;
          double gdott = 0.0;
          for (size_t j = 0; j < d_out; ++j) {
            gdott += gy[j] * trow[j];
            gtrow[j] += coeff * gy[j];
          }
          for (size_t j = 0; j < tau; ++j) {
            const double sg = ((code >> j) & 1u) ? 1.0 : -1.0;
            const double th = tanh(zk[j]);
            const double dcoeff = scaled ? wt * (sg * (1.0 + dot) - dot * th) : wt * (sg - th);
            g[j] += gdott * dcoeff;
          }
        }
      }
    }
    rc = orc_proj_backward(ps, blob, x, n, gz, grad_x, grad_params);
    if (rc == 0 && !all_finite(grad_tables, h * rows * d_out)) rc = 2; /* "lookup backward tables" */
  }
  free(y);
  free(z);
  free(codes);
  free(w);
  free(dots);
  if (!grad_z) free(gz);
  return rc;
}

void orc_gather(const double* tables, size_t h, size_t rows, size_t d_out, const uint32_t* codes,
                const double* coeff, size_t n, double* y) {
#pragma omp parallel for schedule(static)
  for (long i = 0; i < (long)n; ++i) {
    double* yi = y + (size_t)i * d_out;
    for (size_t j = 0; j < d_out; ++j) yi[j] = 0.0;
    for (size_t k = 0; k < h; ++k) {
      const double cf = coeff[(size_t)i * h + k];
      const double* trow = tables + (k * rows + codes[(size_t)i * h + k]) * d_out;
      for (size_t j = 0; j < d_out; ++j) yi[j] += cf * trow[j];
    }
  }
}
