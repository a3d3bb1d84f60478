/*
 * oracle/synth.c -- TEST INFRASTRUCTURE (part of the CPU oracle, never the
 * product).  A plain-C restatement of the reference's parameter synthesis
 * (nf/weights.py:58-94, SplitMix64 counter draws nf/halfnum.py:35-59) followed
 * by binary16 round-to-nearest-even (nf/halfnum.py:80-111), i.e. exactly
 * neox_oracle.f16_params(neox_oracle.synth_block(...)) -- "what the GPU
 * stores" -- but ~50x faster than numpy, so the multi-layer Pythia-2.8B /
 * 6.9B parity tests can synthesize 32 layers of oracle weights in seconds.
 * Pinned bit-exact against the numpy oracle (itself pinned to the reference
 * fixtures) by tests/test_oracle_golden.py::test_c_synth_matches_numpy_oracle.
 */
#include <stdint.h>
#include <string.h>

static inline uint64_t splitmix(uint64_t seed, uint64_t c) {
  uint64_t z = seed + (c + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* binary16 RNE of a double (bit algorithm of nf/halfnum.py:80-111), then
 * the double value of that half, built from its bits. */
static inline double f16_round(double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  const uint64_t sign = b & 0x8000000000000000ull;
  const int ex = (int)((b >> 52) & 0x7ff);
  const uint64_t frac = b & 0xfffffffffffffull;
  if (ex == 0x7ff) return x;
  const int e = ex - 1023;
  uint32_t hv; /* half without sign: exponent << 10 | mantissa */
  if (e >= 16) {
    hv = 0x7c00;
  } else if (e >= -14) {
    hv = ((uint32_t)(e + 15) << 10) | (uint32_t)(frac >> 42);
    const uint64_t rest = frac & ((1ull << 42) - 1), tie = 1ull << 41;
    if (rest > tie || (rest == tie && (hv & 1u))) ++hv; /* carries into the exponent */
  } else if (e < -26) {
    hv = 0;
  } else {
    const uint64_t sig = (1ull << 52) | frac;
    const int sh = 28 - e;
    uint64_t q = sig >> sh;
    const uint64_t rest = sig & ((1ull << sh) - 1), tie = 1ull << (sh - 1);
    if (rest > tie || (rest == tie && (q & 1ull))) ++q;
    hv = (uint32_t)q; /* 0x400 = the smallest normal */
  }
  uint64_t o;
  const uint32_t he = hv >> 10, hm = hv & 0x3ffu;
  if (he >= 31) {
    o = 0x7ff0000000000000ull;
  } else if (he == 0) {
    double v = (double)hm * 0x1p-24;
    memcpy(&o, &v, 8);
  } else {
    o = ((uint64_t)(he - 15 + 1023) << 52) | ((uint64_t)hm << 42);
  }
  o |= sign;
  double r;
  memcpy(&r, &o, 8);
  return r;
}

/* kind: 0 weight u/div, 1 gain 1+0.1u, 2 LN bias 0.1u, 3 bias 0.02u, 4 plain u, 5 KV 0.8660254037844386u */
/* elements [start, start + n) of one tensor stream */
void oracle_synth_f16_range(uint64_t seed, uint32_t stream, uint64_t start, uint64_t n, int kind, double div,
                            double* out) {
  const uint64_t base = ((uint64_t)stream << 32) + start;
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < n; ++i) {
    const double u = (double)(splitmix(seed, base + i) >> 11) * 0x1p-52 - 1.0;
    double v;
    switch (kind) {
      case 0: v = u / div; break;
      case 1: v = 1.0 + 0.1 * u; break;
      case 2: v = 0.1 * u; break;
      case 3: v = 0.02 * u; break;
      case 5: v = 0.8660254037844386 * u; break;
      default: v = u;
    }
    out[i] = f16_round(v);
  }
}

void oracle_synth_f16(uint64_t seed, uint32_t stream, uint64_t n, int kind, double div, double* out) {
  oracle_synth_f16_range(seed, stream, 0, n, kind, div, out);
}

/* f16_round over an array (pinned against the reference's half.npz fixture). */
void oracle_f16_round(const double* x, uint64_t n, double* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = f16_round(x[i]);
}
