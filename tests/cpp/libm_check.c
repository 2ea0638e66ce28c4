/* Bit-for-bit check of glibc_libm.cuh (the device port of glibc 2.39 exp/log)
 * against this host's libm, which the reference links. Inputs: the
 * distributions the path produces (lognormal noise N*sigma for exp; the polar
 * method's r2 = a*a + b*b in (0,1] for log) plus uniform ranges, values near 1
 * and random bit patterns. Prints "<checked> <mismatches>" and the first
 * mismatches. Built by tests/test_libm_port.py with -mfma -ffp-contract=off
 * (fma() is then one vfmadd, nothing else contracts). */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "glibc_libm.cuh"

static uint64_t s[2] = {0x9E3779B97F4A7C15ULL, 0xD1B54A32D192ED03ULL};
static uint64_t next(void) { /* xorshift128+ */
  uint64_t a = s[0], b = s[1];
  s[0] = b;
  a ^= a << 23;
  s[1] = a ^ b ^ (a >> 17) ^ (b >> 26);
  return s[1] + b;
}
static double unif(void) { return (double)(next() >> 11) * 0x1p-53; }
static double bits(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static uint64_t ubits(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }

static long bad = 0, checked = 0;
static void cmp(const char* f, double x, double got, double want) {
  ++checked;
  if (ubits(got) != ubits(want) && !(isnan(got) && isnan(want))) {
    if (bad < 10) printf("MISMATCH %s(%a) = %a, libm %a\n", f, x, got, want);
    ++bad;
  }
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 10000000;
  const double sig[] = {0.05, 0.1, 0.2, 0.3, 0.6, 1.0, 3.0};
  for (long i = 0; i < n; ++i) {
    /* exp: the predictor's noise, wide uniform ranges, random bits */
    double a = 2.0 * unif() - 1.0, b = 2.0 * unif() - 1.0, r2 = a * a + b * b;
    if (r2 > 1.0 || r2 == 0.0) r2 = unif();
    double x = b * sqrt(-2 * log(r2) / r2) * sig[i % 7] + 0.0;
    cmp("exp", x, econo_libm::exp(x), exp(x));
    x = unif() * 1500.0 - 750.0;
    cmp("exp", x, econo_libm::exp(x), exp(x));
    x = bits(next());
    cmp("exp", x, econo_libm::exp(x), exp(x));
    x = (unif() - 0.5) * 0x1p-50;
    cmp("exp", x, econo_libm::exp(x), exp(x));
    /* log: the polar method's r2, near 1, (0,1], random positive bits, subnormals */
    cmp("log", r2, econo_libm::log(r2), log(r2));
    x = 1.0 + (unif() - 0.5) * 0.2;
    cmp("log", x, econo_libm::log(x), log(x));
    x = unif();
    cmp("log", x, econo_libm::log(x), log(x));
    x = bits(next() >> 1);
    cmp("log", x, econo_libm::log(x), log(x));
    x = bits(next() >> 12);
    cmp("log", x, econo_libm::log(x), log(x));
  }
  const double sp[] = {0.0, -0.0, 1.0, -1.0, INFINITY, -INFINITY, NAN, 709.78, 709.79, -745.13, -745.14,
                       -708.4, -708.3, 1e-300, 5e-324, 0x1p-54, -0x1p-54, 0x1.fffffffffffffp-1, 0x1.0000000000001p0};
  for (unsigned k = 0; k < sizeof(sp) / sizeof(sp[0]); ++k) {
    cmp("exp", sp[k], econo_libm::exp(sp[k]), exp(sp[k]));
    cmp("log", sp[k], econo_libm::log(sp[k]), log(sp[k]));
  }
  printf("%ld %ld\n", checked, bad);
  return bad != 0;
}
