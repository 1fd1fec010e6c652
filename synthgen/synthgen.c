/*
 * synthgen.c — seeded synthetic inputs for the dense product C = A·B.
 *
 * This module is shared by the oracle side (tests/, oracle checks) and the
 * product side (bench.py, smoke()).  It holds NONE of the method's
 * arithmetic: no products, no sums over k.  It only turns (seed, role,
 * index) into matrix entries, and hashes matrices into checksums.
 *
 * Recipe:
 *   key        = fmix64(4*seed + role)       role: A=1, B=2, row-sample=3, col-sample=4
 *   w(idx)     = fmix64(key + (idx+1)*0x9E3779B97F4A7C15)   (SplitMix64 output #idx)
 *   idx        = i*cols + j  (row-major, "C ... stores data in row-major order")
 *   FP64 U[-1,1)        : (w>>11)*2^-52 - 1                      (BASELINE.json configs 0,1,4)
 *   INT8 U{-127..127}   : (((w>>32)*255)>>32) - 127              (BASELINE.json config 2)
 *   BF16 N(0,1)         : Box-Muller, PAPER.md:158-168 (eqs. Z0, Z1) and Fig. 5
 *                          on the pair q = idx>>1:
 *                           u1 = ((w(2q)>>12) + 0.5)*2^-52,  u2 likewise from w(2q+1)
 *                           (both strictly inside (0,1): "in the range (0, 1)")
 *                           r = sqrt(-2.0*log(u1)), t = 2.0*pi*u2
 *                           even idx -> r*cos(t), odd idx -> r*sin(t)
 *                         then double -> bf16 by ONE round-to-nearest-even (reading R9).
 *   exact-int pins      : (((w>>32)*K)>>32) - (K-1)/2   (K odd: 3, 9, 2049, ...)
 *   checksum            : sum_idx fmix64(bits(x_idx) + (idx+1)*0x9E3779B97F4A7C15) mod 2^64,
 *                         bits zero-extended, FP -0.0 canonicalised to +0.0.
 *
 * Compiled -O2 -fopenmp (no -ffast-math): libm log/cos/sin from glibc.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t fmix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

uint64_t sg_fmix64(uint64_t z) { return fmix64(z); }

uint64_t sg_key(uint64_t seed, uint64_t role) { return fmix64(4 * seed + role); }

uint64_t sg_word(uint64_t key, uint64_t idx) { return fmix64(key + (idx + 1) * GOLDEN); }

static inline double u_m1_1(uint64_t w) { return (double)(w >> 11) * 0x1p-52 - 1.0; }

/* double -> bf16 bits, one round-to-nearest-even directly from double.
 * Values here are finite normal numbers of modest magnitude (|z| < 10) or 0. */
static inline uint16_t bf16_rne_from_double(double x) {
  if (x == 0.0) return signbit(x) ? 0x8000 : 0;
  int e;
  double m = frexp(x, &e);             /* x = m * 2^e, 0.5 <= |m| < 1 */
  double r = ldexp(rint(ldexp(m, 8)), e - 8); /* 8 significant bits, RNE */
  float f = (float)r;                   /* exact: r has <= 8 significant bits */
  uint32_t u;
  memcpy(&u, &f, 4);
  return (uint16_t)(u >> 16);
}

uint16_t sg_bf16_from_double(double x) { return bf16_rne_from_double(x); }

static inline double box_muller_at(uint64_t key, uint64_t idx) {
  uint64_t q = idx >> 1;
  uint64_t w1 = fmix64(key + (2 * q + 1) * GOLDEN);
  uint64_t w2 = fmix64(key + (2 * q + 2) * GOLDEN);
  double u1 = ((double)(w1 >> 12) + 0.5) * 0x1p-52;
  double u2 = ((double)(w2 >> 12) + 0.5) * 0x1p-52;
  double r = sqrt(-2.0 * log(u1));
  double t = 2.0 * M_PI * u2;
  return (idx & 1) ? r * sin(t) : r * cos(t);
}

/* Box-Muller on given uniforms (test pin SPEC.md:126-128). */
void sg_box_muller(double u1, double u2, double* z0, double* z1) {
  double r = sqrt(-2.0 * log(u1));
  double t = 2.0 * M_PI * u2;
  *z0 = r * cos(t);
  *z1 = r * sin(t);
}

/* ---- generators: out has rows*cols entries, row-major ---- */

void sg_gen_f64(uint64_t seed, uint64_t role, int64_t rows, int64_t cols, double* out) {
  const uint64_t key = sg_key(seed, role);
  const int64_t N = rows * cols;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) out[i] = u_m1_1(sg_word(key, (uint64_t)i));
}

void sg_gen_i8(uint64_t seed, uint64_t role, int64_t rows, int64_t cols, int8_t* out) {
  const uint64_t key = sg_key(seed, role);
  const int64_t N = rows * cols;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    uint64_t w = sg_word(key, (uint64_t)i);
    out[i] = (int8_t)((int64_t)(((w >> 32) * 255ULL) >> 32) - 127);
  }
}

/* bf16 Box-Muller normals, returned as raw bf16 bit patterns. */
void sg_gen_bf16_normal(uint64_t seed, uint64_t role, int64_t rows, int64_t cols, uint16_t* out) {
  const uint64_t key = sg_key(seed, role);
  const int64_t N = rows * cols;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) out[i] = bf16_rne_from_double(box_muller_at(key, (uint64_t)i));
}

/* The unrounded Box-Muller double (test use: bf16 rounding pin). */
void sg_gen_normal_f64(uint64_t seed, uint64_t role, int64_t rows, int64_t cols, double* out) {
  const uint64_t key = sg_key(seed, role);
  const int64_t N = rows * cols;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) out[i] = box_muller_at(key, (uint64_t)i);
}

static inline int64_t exact_int(uint64_t w, uint64_t K) {
  return (int64_t)(((w >> 32) * K) >> 32) - (int64_t)((K - 1) / 2);
}

/* Exact-integer pin inputs, K odd: values in [-(K-1)/2, (K-1)/2]. */
void sg_gen_exact_f64(uint64_t seed, uint64_t role, uint64_t K, int64_t rows, int64_t cols, double* out) {
  const uint64_t key = sg_key(seed, role);
  const int64_t N = rows * cols;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) out[i] = (double)exact_int(sg_word(key, (uint64_t)i), K);
}

void sg_gen_exact_bf16(uint64_t seed, uint64_t role, uint64_t K, int64_t rows, int64_t cols, uint16_t* out) {
  const uint64_t key = sg_key(seed, role);
  const int64_t N = rows * cols;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i)
    out[i] = bf16_rne_from_double((double)exact_int(sg_word(key, (uint64_t)i), K));
}

void sg_gen_exact_i8(uint64_t seed, uint64_t role, uint64_t K, int64_t rows, int64_t cols, int8_t* out) {
  const uint64_t key = sg_key(seed, role);
  const int64_t N = rows * cols;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) out[i] = (int8_t)exact_int(sg_word(key, (uint64_t)i), K);
}

/* Seeded sample of `count` distinct-ish indices in [0, limit) (role 3 = rows, 4 = cols).
 * Duplicates are allowed; the caller dedups. */
void sg_sample_indices(uint64_t seed, uint64_t role, int64_t count, int64_t limit, int64_t* out) {
  const uint64_t key = sg_key(seed, role);
  for (int64_t i = 0; i < count; ++i) {
    uint64_t w = sg_word(key, (uint64_t)i);
    out[i] = (int64_t)(((w >> 32) * (uint64_t)limit) >> 32);
  }
}

/* ---- checksums ---- */

static inline uint64_t cs_term(uint64_t bits, int64_t idx) { return fmix64(bits + (uint64_t)(idx + 1) * GOLDEN); }

/* `off` = global row-major index of x[0] (checksums of row blocks add up mod 2^64). */
uint64_t sg_checksum_f64_off(const double* x, int64_t N, int64_t off) {
  uint64_t s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    double v = x[i] + 0.0; /* -0.0 -> +0.0 */
    uint64_t b;
    memcpy(&b, &v, 8);
    s += cs_term(b, off + i);
  }
  return s;
}
uint64_t sg_checksum_f64(const double* x, int64_t N) { return sg_checksum_f64_off(x, N, 0); }

uint64_t sg_checksum_f32_off(const float* x, int64_t N, int64_t off) {
  uint64_t s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    float v = x[i] + 0.0f;
    uint32_t b;
    memcpy(&b, &v, 4);
    s += cs_term((uint64_t)b, off + i);
  }
  return s;
}
uint64_t sg_checksum_f32(const float* x, int64_t N) { return sg_checksum_f32_off(x, N, 0); }

/* checksum of doubles as if they had been stored as fp32 / int32 (exact-int results) */
uint64_t sg_checksum_f64_as_f32_off(const double* x, int64_t N, int64_t off) {
  uint64_t s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    float v = (float)x[i] + 0.0f;
    uint32_t b;
    memcpy(&b, &v, 4);
    s += cs_term((uint64_t)b, off + i);
  }
  return s;
}

uint64_t sg_checksum_i32_off(const int32_t* x, int64_t N, int64_t off) {
  uint64_t s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (int64_t i = 0; i < N; ++i) s += cs_term((uint64_t)(uint32_t)x[i], off + i);
  return s;
}
uint64_t sg_checksum_i32(const int32_t* x, int64_t N) { return sg_checksum_i32_off(x, N, 0); }

uint64_t sg_checksum_bf16(const uint16_t* x, int64_t N) {
  uint64_t s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    uint16_t b = x[i];
    if (b == 0x8000) b = 0; /* -0 -> +0 */
    s += cs_term((uint64_t)b, i);
  }
  return s;
}

uint64_t sg_checksum_i8(const int8_t* x, int64_t N) {
  uint64_t s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (int64_t i = 0; i < N; ++i) s += cs_term((uint64_t)(uint8_t)x[i], i);
  return s;
}
