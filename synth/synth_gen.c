/*
 * synth_gen.c — seeded, counter-based synthetic inputs shared by the tests, bench.py and the oracle
 * harness. It holds NONE of the method's arithmetic (no reduction, no rounding routine of the
 * collectives): each element is a pure function of (seed, rank, index) via splitmix64, so any
 * sub-range of any rank can be regenerated independently.
 * bf16 values are produced by TRUNCATING the binary32 bit pattern (round toward zero) — a
 * deliberately different rule from the method's round-to-nearest-even narrowing.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

static inline uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint64_t key(uint64_t seed, int rank, size_t i) {
  return splitmix64(splitmix64(seed * 0x100000001B3ull + (uint64_t)rank) ^ (uint64_t)i * 0xD1B54A32D192ED03ull);
}

/* 24-bit uniform in [0,1) */
static inline double u01(uint32_t b) { return (double)(b >> 8) * (1.0 / 16777216.0); }

static inline float normal_at(uint64_t seed, int rank, size_t i) {
  uint64_t h = key(seed, rank, i);
  double u1 = u01((uint32_t)h) + (1.0 / 33554432.0); /* (0,1) */
  double u2 = u01((uint32_t)(h >> 32));
  return (float)(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
}

void synth_normal_f32(uint64_t seed, int rank, size_t start, size_t n, float scale, float* out) {
  for (size_t t = 0; t < n; t++) out[t] = normal_at(seed, rank, start + t) * scale;
}

void synth_normal_bf16(uint64_t seed, int rank, size_t start, size_t n, float scale, uint16_t* out) {
  for (size_t t = 0; t < n; t++) {
    float f = normal_at(seed, rank, start + t) * scale;
    uint32_t u;
    memcpy(&u, &f, 4);
    out[t] = (uint16_t)(u >> 16); /* truncation */
  }
}

void synth_uniform_f32(uint64_t seed, int rank, size_t start, size_t n, float lo, float hi, float* out) {
  for (size_t t = 0; t < n; t++) {
    double u = u01((uint32_t)key(seed, rank, start + t));
    out[t] = (float)(lo + (hi - lo) * u);
  }
}

void synth_bits_u32(uint64_t seed, int rank, size_t start, size_t n, uint32_t* out) {
  for (size_t t = 0; t < n; t++) out[t] = (uint32_t)(key(seed, rank, start + t) >> 16);
}
