/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference optimizer-update path
 * (minicollie::optim, /root/reference/proj/core/src/optim.cpp). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this file's
 * library, and only as the checker. The product path
 * (paper_2312_00407_b200/csrc) never links or calls it.
 *
 * Parity pinning: the f64 functions below follow the reference loops operation
 * for operation and are checked BIT-EXACT against the reference itself compiled
 * from /root/reference into oracle/_ref (tests/test_oracle.py), and against the
 * reference's own known-answer tests (tests/test_optim.cpp) restated in
 * tests/test_oracle.py.  The f32 / bf16 functions are the same operation order
 * at single precision with the per-step scalars derived in double on the host
 * and rounded once to float -- the contract the CUDA kernels implement.  Build
 * with -ffp-contract=off so no multiply-add is fused (the kernels are compiled
 * with --fmad=false for the same reason).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* Mirrors minicollie::optim::OptimizerConfig (optim.hpp:20-35) field for field;
 * identical layout to mco_config in include/mco.h. */
typedef struct {
  int kind; /* 0 adamw, 1 lion, 2 adan, 3 sophia, 4 lomo, 5 adalomo (optim.hpp:14) */
  double lr, weight_decay, beta1, beta2, beta3, eps;
  int has_clip_threshold;
  double clip_threshold;
  double adalomo_clip;
  double sophia_rho;
  int update_interval;
} orc_config;

/* ------------------------------------------------------------------------ */
/* Synthetic inputs: counter-based, stateless, exact in fp32 / bf16.          */
/* (SURVEY.md 8(d) "Values"; independent restatement of csrc/synth.cu.)       */
/* ------------------------------------------------------------------------ */
#define ORC_GOLDEN 0x9E3779B97F4A7C15ULL

uint64_t orc_fmix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

uint64_t orc_synth_key(uint64_t seed, uint32_t role, uint32_t tensor, uint32_t step) {
  uint64_t a = orc_fmix64(seed + (uint64_t)role * ORC_GOLDEN);
  return orc_fmix64(a ^ (((uint64_t)tensor << 32) | (uint64_t)step));
}

/* Value of element idx. bf16_grid: 8 significant bits (exact in bf16). */
static double synth_value(uint64_t key, uint64_t idx, int64_t cols, int scale_log2,
                          int zero_log2, int rowcol, int bf16_grid) {
  uint64_t x = orc_fmix64(key + (idx + 1) * ORC_GOLDEN);
  double v;
  if (bf16_grid)
    v = (double)((int32_t)(x >> 56) - 128) * 0x1.0p-7;
  else
    v = (double)((int32_t)(x >> 40) - (1 << 23)) * 0x1.0p-23;
  if (zero_log2 > 0 && (x & ((1ULL << zero_log2) - 1)) == 0) v = 0.0;
  int e = scale_log2;
  if (rowcol && cols > 0) {
    uint64_t r = idx / (uint64_t)cols, c = idx % (uint64_t)cols;
    e += (int)(orc_fmix64(key ^ (0xA5A5A5A5A5A5A5A5ULL + r * ORC_GOLDEN)) >> 62) - 1;
    e += (int)(orc_fmix64(key ^ (0x5A5A5A5A5A5A5A5AULL + c * ORC_GOLDEN)) >> 62) - 1;
  }
  return ldexp(v, e);
}

void orc_synth_f32(float* out, uint64_t n, uint64_t key, int64_t cols, int scale_log2,
                   int zero_log2, int rowcol) {
  for (uint64_t i = 0; i < n; ++i)
    out[i] = (float)synth_value(key, i, cols, scale_log2, zero_log2, rowcol, 0);
}

void orc_synth_f64(double* out, uint64_t n, uint64_t key, int64_t cols, int scale_log2,
                   int zero_log2, int rowcol) {
  for (uint64_t i = 0; i < n; ++i)
    out[i] = synth_value(key, i, cols, scale_log2, zero_log2, rowcol, 0);
}

/* bf16 bit patterns (upper half of the exact float). */
void orc_synth_bf16(uint16_t* out, uint64_t n, uint64_t key, int64_t cols, int scale_log2,
                    int zero_log2, int rowcol) {
  for (uint64_t i = 0; i < n; ++i) {
    float f = (float)synth_value(key, i, cols, scale_log2, zero_log2, rowcol, 1);
    uint32_t u;
    memcpy(&u, &f, 4);
    out[i] = (uint16_t)(u >> 16);
  }
}

/* ------------------------------------------------------------------------ */
/* bf16 helpers                                                             */
/* ------------------------------------------------------------------------ */
float orc_bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* Round-to-nearest-even; any NaN -> canonical 0x7fff (the cvt.rn.bf16 rule). */
uint16_t orc_f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)0x7fffu;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

/* ------------------------------------------------------------------------ */
/* f64: operation-for-operation restatement of optim.cpp                    */
/* ------------------------------------------------------------------------ */

/* optim.cpp:114-125 */
void orc_adamw_f64(double* p, const double* g, double* m, double* v, uint64_t n,
                   const orc_config* c, int64_t t, double lr) {
  const double b1 = c->beta1, b2 = c->beta2;
  const double c1 = 1.0 - pow(b1, (double)t);
  const double c2 = 1.0 - pow(b2, (double)t);
  for (uint64_t i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + (1 - b1) * g[i];
    v[i] = b2 * v[i] + (1 - b2) * g[i] * g[i];
    const double mhat = m[i] / c1;
    const double vhat = v[i] / c2;
    p[i] -= lr * (mhat / (sqrt(vhat) + c->eps) + c->weight_decay * p[i]);
  }
}

/* optim.cpp:127-135 */
void orc_lion_f64(double* p, const double* g, double* m, uint64_t n, const orc_config* c,
                  double lr) {
  const double b1 = c->beta1, b2 = c->beta2;
  for (uint64_t i = 0; i < n; ++i) {
    const double u = b1 * m[i] + (1 - b1) * g[i];
    const double s = u > 0 ? 1.0 : (u < 0 ? -1.0 : 0.0); /* sign(0) = 0 */
    p[i] -= lr * (s + c->weight_decay * p[i]);
    m[i] = b2 * m[i] + (1 - b2) * g[i];
  }
}

/* optim.cpp:137-155 */
void orc_adan_f64(double* p, const double* g, double* m, double* v, double* nb, double* gp,
                  uint64_t n, const orc_config* c, int64_t t, double lr) {
  const double b1 = c->beta1, b2 = c->beta2, b3 = c->beta3;
  const double c1 = 1.0 - pow(b1, (double)t);
  const double c2 = 1.0 - pow(b2, (double)t);
  const double c3 = 1.0 - pow(b3, (double)t);
  for (uint64_t i = 0; i < n; ++i) {
    const double gd = t == 1 ? 0.0 : g[i] - gp[i];
    m[i] = b1 * m[i] + (1 - b1) * g[i];
    v[i] = b2 * v[i] + (1 - b2) * gd;
    const double nu = g[i] + b2 * gd;
    nb[i] = b3 * nb[i] + (1 - b3) * nu * nu;
    const double mhat = m[i] / c1;
    const double vhat = v[i] / c2;
    const double nhat = nb[i] / c3;
    p[i] = (p[i] - lr * (mhat + b2 * vhat) / (sqrt(nhat) + c->eps)) /
           (1.0 + lr * c->weight_decay);
    gp[i] = g[i];
  }
}

static double clampd(double x, double lo, double hi) { return x < lo ? lo : (hi < x ? hi : x); }
static double maxd(double a, double b) { return a < b ? b : a; } /* std::max(a, b) */

/* optim.cpp:157-167 */
void orc_sophia_f64(double* p, const double* g, double* m, double* h, uint64_t n,
                    const orc_config* c, int64_t t, double lr) {
  const double b1 = c->beta1, b2 = c->beta2;
  const int refresh = ((t - 1) % c->update_interval) == 0;
  for (uint64_t i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + (1 - b1) * g[i];
    if (refresh) h[i] = b2 * h[i] + (1 - b2) * g[i] * g[i];
    const double denom = maxd(c->sophia_rho * h[i], c->eps);
    const double u = clampd(m[i] / denom, -1.0, 1.0);
    p[i] -= lr * u + lr * c->weight_decay * p[i];
  }
}

/* optim.cpp:185-190 */
void orc_lomo_f64(double* p, const double* g, uint64_t n, double lr, double scale) {
  const double f = lr * scale;
  for (uint64_t i = 0; i < n; ++i) p[i] -= f * g[i];
}

/* optim.cpp:294-303: sequential sum of squares and the clip rule. */
double orc_sumsq_f64(const double* g, uint64_t n) {
  double s = 0.0;
  for (uint64_t i = 0; i < n; ++i) s += g[i] * g[i];
  return s;
}

double orc_clip_scale(double sum_sq, double clip) {
  const double norm = sqrt(sum_sq);
  return (norm > clip && norm > 0) ? clip / norm : 1.0;
}

/*
 * optim.cpp:215-275, one tensor. factored => v_row[R], v_col[C]; else v_full[n].
 * *t is the entry's step counter (incremented here, optim.cpp:219).
 * grad_scale multiplies g first (1.0 = the reference exactly): the composed
 * oracle for "AdaLomo + global grad-norm clip" (SURVEY.md 8(c) unpinned #1).
 */
void orc_adalomo_f64(double* p, const double* g_in, int64_t R, int64_t C, int factored,
                     double* v_row, double* v_col, double* v_full, int64_t* t,
                     const orc_config* c, double lr, double grad_scale, double* u /* scratch n */) {
  const uint64_t n = factored ? (uint64_t)(R * C) : (uint64_t)R;
  const double b2 = c->beta2;
  /* g = scale * g_in; materialised in u's slot first only when scaling */
  const double* g = g_in;
  double* gs = 0;
  if (grad_scale != 1.0) {
    gs = u + n; /* caller provides 2n scratch when scaling */
    for (uint64_t i = 0; i < n; ++i) gs[i] = grad_scale * g_in[i];
    g = gs;
  }
  *t += 1;
  const double corr = 1.0 - pow(b2, (double)*t);
  double theta_sq = 0.0;
  for (uint64_t i = 0; i < n; ++i) theta_sq += p[i] * p[i];
  const double rms_theta = sqrt(theta_sq / (double)n);
  const double lr_t = lr * maxd(1e-3, rms_theta);
  if (factored) {
    for (int64_t i = 0; i < R; ++i) {
      double acc = 0.0;
      for (int64_t j = 0; j < C; ++j) {
        const double gij = g[i * C + j];
        acc += gij * gij;
      }
      v_row[i] = b2 * v_row[i] + (1 - b2) * (acc / (double)C);
    }
    for (int64_t j = 0; j < C; ++j) {
      double acc = 0.0;
      for (int64_t i = 0; i < R; ++i) {
        const double gij = g[i * C + j];
        acc += gij * gij;
      }
      v_col[j] = b2 * v_col[j] + (1 - b2) * (acc / (double)R);
    }
    double row_mean = 0.0;
    for (int64_t i = 0; i < R; ++i) row_mean += v_row[i];
    row_mean /= (double)R * corr;
    for (int64_t i = 0; i < R; ++i) {
      const double vr = v_row[i] / corr;
      for (int64_t j = 0; j < C; ++j) {
        const double vc = v_col[j] / corr;
        const double vhat = vr * vc / maxd(row_mean, 1e-300);
        u[i * C + j] = g[i * C + j] / sqrt(vhat + c->eps);
      }
    }
  } else {
    for (uint64_t i = 0; i < n; ++i) {
      v_full[i] = b2 * v_full[i] + (1 - b2) * g[i] * g[i];
      u[i] = g[i] / sqrt(v_full[i] / corr + c->eps);
    }
  }
  double u_sq = 0.0;
  for (uint64_t i = 0; i < n; ++i) u_sq += u[i] * u[i];
  const double rms_u = sqrt(u_sq / (double)n);
  const double damp = maxd(1.0, rms_u / c->adalomo_clip);
  const double f = lr_t / damp;
  for (uint64_t i = 0; i < n; ++i) p[i] -= f * u[i];
}

/* ------------------------------------------------------------------------ */
/* f32: same operation order; per-step scalars derived in double, rounded   */
/* once to float. This is the bit-exact target of the fp32 CUDA kernels.    */
/* ------------------------------------------------------------------------ */

void orc_adamw_f32(float* p, const float* g, float* m, float* v, uint64_t n,
                   const orc_config* c, int64_t t, double lr) {
  const float b1 = (float)c->beta1, b2 = (float)c->beta2;
  const float omb1 = (float)(1.0 - c->beta1), omb2 = (float)(1.0 - c->beta2);
  const float c1 = (float)(1.0 - pow(c->beta1, (double)t));
  const float c2 = (float)(1.0 - pow(c->beta2, (double)t));
  const float lrf = (float)lr, eps = (float)c->eps, wd = (float)c->weight_decay;
  for (uint64_t i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + omb1 * g[i];
    v[i] = b2 * v[i] + omb2 * g[i] * g[i];
    const float mhat = m[i] / c1;
    const float vhat = v[i] / c2;
    p[i] = p[i] - lrf * (mhat / (sqrtf(vhat) + eps) + wd * p[i]);
  }
}

void orc_lion_f32(float* p, const float* g, float* m, uint64_t n, const orc_config* c,
                  double lr) {
  const float b1 = (float)c->beta1, b2 = (float)c->beta2;
  const float omb1 = (float)(1.0 - c->beta1), omb2 = (float)(1.0 - c->beta2);
  const float lrf = (float)lr, wd = (float)c->weight_decay;
  for (uint64_t i = 0; i < n; ++i) {
    const float u = b1 * m[i] + omb1 * g[i];
    const float s = u > 0 ? 1.0f : (u < 0 ? -1.0f : 0.0f);
    p[i] = p[i] - lrf * (s + wd * p[i]);
    m[i] = b2 * m[i] + omb2 * g[i];
  }
}

void orc_adan_f32(float* p, const float* g, float* m, float* v, float* nb, float* gp,
                  uint64_t n, const orc_config* c, int64_t t, double lr) {
  const float b1 = (float)c->beta1, b2 = (float)c->beta2, b3 = (float)c->beta3;
  const float omb1 = (float)(1.0 - c->beta1), omb2 = (float)(1.0 - c->beta2),
              omb3 = (float)(1.0 - c->beta3);
  /* fp32 product form (update.cuh): the bias corrections 1 / (1 - beta^t) and the
   * decay 1 / (1 + lr wd) are reciprocals rounded once and multiplied (the f64
   * functions keep optim.cpp's divisions) */
  const float rc1 = (float)(1.0 / (1.0 - pow(c->beta1, (double)t)));
  const float rc2 = (float)(1.0 / (1.0 - pow(c->beta2, (double)t)));
  const float rc3 = (float)(1.0 / (1.0 - pow(c->beta3, (double)t)));
  const float lrf = (float)lr, eps = (float)c->eps;
  const float rden = (float)(1.0 / (1.0 + lr * c->weight_decay));
  for (uint64_t i = 0; i < n; ++i) {
    const float gd = t == 1 ? 0.0f : g[i] - gp[i];
    m[i] = b1 * m[i] + omb1 * g[i];
    v[i] = b2 * v[i] + omb2 * gd;
    const float nu = g[i] + b2 * gd;
    nb[i] = b3 * nb[i] + omb3 * nu * nu;
    const float mhat = m[i] * rc1;
    const float vhat = v[i] * rc2;
    const float nhat = nb[i] * rc3;
    p[i] = (p[i] - lrf * (mhat + b2 * vhat) / (sqrtf(nhat) + eps)) * rden;
    gp[i] = g[i];
  }
}

static float clampf_(float x, float lo, float hi) { return x < lo ? lo : (hi < x ? hi : x); }
static float maxf_(float a, float b) { return a < b ? b : a; }

void orc_sophia_f32(float* p, const float* g, float* m, float* h, uint64_t n,
                    const orc_config* c, int64_t t, double lr) {
  const float b1 = (float)c->beta1, b2 = (float)c->beta2;
  const float omb1 = (float)(1.0 - c->beta1), omb2 = (float)(1.0 - c->beta2);
  const float rho = (float)c->sophia_rho, eps = (float)c->eps, lrf = (float)lr;
  const float lrwd = (float)(lr * c->weight_decay);
  const int refresh = ((t - 1) % c->update_interval) == 0;
  for (uint64_t i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + omb1 * g[i];
    if (refresh) h[i] = b2 * h[i] + omb2 * g[i] * g[i];
    const float denom = maxf_(rho * h[i], eps);
    const float u = clampf_(m[i] / denom, -1.0f, 1.0f);
    p[i] = p[i] - (lrf * u + lrwd * p[i]);
  }
}

/* Sophia "precise-m" (state MCO_F32M64, sophia_m64.cu): fp32 p, g, h with an fp64 m and
 * fp64 per-element arithmetic in optim.cpp:160-166's order; h and p rounded once. */
void orc_sophia_m64(float* p, const float* g, double* m, float* h, uint64_t n,
                    const orc_config* c, int64_t t, double lr) {
  const double b1 = c->beta1, b2 = c->beta2, omb1 = 1.0 - c->beta1, omb2 = 1.0 - c->beta2;
  const double rho = c->sophia_rho, eps = c->eps, lrwd = lr * c->weight_decay;
  const int refresh = ((t - 1) % c->update_interval) == 0;
  for (uint64_t i = 0; i < n; ++i) {
    const double gd = (double)g[i];
    m[i] = b1 * m[i] + omb1 * gd;
    if (refresh) h[i] = (float)(b2 * (double)h[i] + omb2 * gd * gd);
    const double rh = rho * (double)h[i];
    const double denom = rh < eps ? eps : rh;
    const double q = m[i] / denom;
    const double u = q < -1.0 ? -1.0 : (1.0 < q ? 1.0 : q);
    const double pd = (double)p[i];
    p[i] = (float)(pd - (lr * u + lrwd * pd));
  }
}

void orc_lomo_f32(float* p, const float* g, uint64_t n, double lr, double scale) {
  const float f = (float)(lr * scale);
  for (uint64_t i = 0; i < n; ++i) p[i] = p[i] - f * g[i];
}

void orc_lomo_bf16(uint16_t* p, const uint16_t* g, uint64_t n, double lr, double scale) {
  const float f = (float)(lr * scale);
  for (uint64_t i = 0; i < n; ++i)
    p[i] = orc_f32_to_bf16(orc_bf16_to_f32(p[i]) - f * orc_bf16_to_f32(g[i]));
}

/* Σg² of fp32 / bf16 data in double (order-independent up to double rounding). */
double orc_sumsq_f32(const float* g, uint64_t n) {
  double s = 0.0;
  for (uint64_t i = 0; i < n; ++i) s += (double)g[i] * (double)g[i];
  return s;
}

double orc_sumsq_bf16(const uint16_t* g, uint64_t n) {
  double s = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    const double x = orc_bf16_to_f32(g[i]);
    s += x * x;
  }
  return s;
}

/* ZeroPlan::make (parallel.cpp:20-34): q = P/N, first P%N ranks get one more. */
int orc_zero_plan(uint64_t total, int dp, uint64_t* part_sizes, uint64_t* offsets) {
  if (dp < 1) return 2;
  const uint64_t q = total / (uint64_t)dp, r = total % (uint64_t)dp;
  offsets[0] = 0;
  for (int i = 0; i < dp; ++i) {
    part_sizes[i] = q + ((uint64_t)i < r ? 1 : 0);
    offsets[i + 1] = offsets[i] + part_sizes[i];
  }
  return 0;
}
