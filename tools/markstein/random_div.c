/* Exhaustive-random check of the tracer's division by a known divisor (tracer.cu Divisor):
   RN(q + (a - b q) y) with y = RN(1/b), q = RN(a y) against IEEE a / b, over random
   operands with edge-case significands (all ones, near zero).  gcc -O2 -mfma -ffp-contract=off
   random_div.c -lm && ./a.out 200000000   ->  bad=0 (200 M cases). */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>
static uint64_t s = 0x9E3779B97F4A7C15ull;
static uint64_t nx(void) { uint64_t z = (s += 0x9E3779B97F4A7C15ull); z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31); }
static double bits(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static double rnd_in(int emin, int emax) { /* random sign-positive double with exponent in [emin, emax] */
  uint64_t m = nx() & 0xFFFFFFFFFFFFFull; int e = emin + (int)(nx() % (uint64_t)(emax - emin + 1));
  int mode = nx() % 8; if (mode == 0) m = 0xFFFFFFFFFFFFFull; else if (mode == 1) m = 0; else if (mode == 2) m = (nx() % 64); else if (mode == 3) m = 0xFFFFFFFFFFFFFull - (nx() % 64);
  return bits(((uint64_t)(e + 1023) << 52) | m); }
int main(int argc, char** argv) {
  long long N = argc > 1 ? atoll(argv[1]) : 100000000LL, bad = 0;
  for (long long i = 0; i < N; ++i) {
    double b = rnd_in(-60, 60), a = rnd_in(-200, 200);
    if (nx() & 1) a = -a;
    if (nx() & 1) b = -b;
    volatile double one = 1.0;
    double y = one / b;            /* RN(1/b) */
    double q = a * y;
    double r = fma(-b, q, a);
    double q2 = fma(r, y, q);
    double t = a / b;
    if (q2 != t) { if (bad < 10) printf("a=%a b=%a got %a want %a\n", a, b, q2, t); ++bad; }
  }
  printf("N=%lld bad=%lld\n", N, bad);
  return 0;
}
