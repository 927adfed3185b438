/* Exhaustive pin of the oracle's fp32 -> bf16 round-to-nearest-even
 * (test plan item 1): every one of the 2^32
 * fp32 bit patterns through or_f32_to_bf16 (liboracle.so) against a rounding
 * written independently here.  The oracle adds 0x7fff + lsb and truncates;
 * this reference instead measures the exact fp64 distance to the two bf16
 * neighbours of x, ties going to the even mantissa, with IEEE overflow (a
 * finite x whose upper neighbour is infinite rounds to inf iff it is at least
 * halfway to 2^128).  NaN must stay NaN with its sign; +-inf must stay +-inf.
 * Test infrastructure only (tests/test_oracle_numerics.py builds and runs it).
 * Prints "checked N mismatches M first F". */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

uint16_t or_f32_to_bf16(float x);

static double f32_of(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

static uint16_t ref_bf16(uint32_t u) {
  const uint32_t mag = u & 0x7fffffffu;
  if (mag > 0x7f800000u) return 0xffffu; /* NaN: checked by class below */
  if (mag == 0x7f800000u) return (uint16_t)(u >> 16);
  const uint32_t lo = u & 0xffff0000u;   /* bf16 neighbour toward zero */
  const uint32_t hi = lo + 0x10000u;     /* the next one away from zero */
  const double x = fabs(f32_of(u));
  const double dlo = x - fabs(f32_of(lo));
  const double fhi = ((hi & 0x7fffffffu) == 0x7f800000u) ? ldexp(1.0, 128) : fabs(f32_of(hi));
  const double dhi = fhi - x;
  const int lo_even = ((lo >> 16) & 1u) == 0;
  const uint32_t pick = (dhi < dlo || (dhi == dlo && !lo_even)) ? hi : lo;
  return (uint16_t)(pick >> 16);
}

int main(void) {
  unsigned long long bad = 0, first = 0xffffffffffffffffull;
#pragma omp parallel for schedule(static, 1 << 20) reduction(+ : bad)
  for (long long i = 0; i < (1ll << 32); ++i) {
    const uint32_t u = (uint32_t)i;
    float x;
    memcpy(&x, &u, 4);
    const uint16_t got = or_f32_to_bf16(x);
    int ok;
    if ((u & 0x7fffffffu) > 0x7f800000u) /* NaN in: NaN out, same sign */
      ok = (got & 0x7fffu) > 0x7f80u && (got >> 15) == (u >> 31);
    else
      ok = got == ref_bf16(u);
    if (!ok) {
      ++bad;
#pragma omp critical
      if ((unsigned long long)i < first) first = (unsigned long long)i;
    }
  }
  printf("checked %llu mismatches %llu first %llx\n", 1ull << 32, bad, bad ? first : 0ull);
  return bad != 0;
}
