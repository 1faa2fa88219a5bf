/* spec_exhaustive.c — exhaustive accuracy pins of the oracle's sin_spec and exp_spec (ARITH
 * §B2, §C) against libm in fp64 (test infrastructure: links the oracle library only).
 * sin_spec: max |error| over every fp32 x in [0, pi_f] (the form is odd).
 * exp_spec: max error in units of the last place over every fp32 x in [-80, 0].
 * Prints the two maxima. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

float oracle_sin_spec(float x);
float oracle_exp_spec(float x);

int main(void) {
  const float pif = 3.14159274101257324f, lo = -80.0f;
  uint32_t lim, blo;
  memcpy(&lim, &pif, 4);
  memcpy(&blo, &lo, 4);
  double es = 0.0, ee = 0.0;
#pragma omp parallel for reduction(max : es) schedule(static)
  for (int64_t bi = 0; bi <= (int64_t)lim; ++bi) {
    const uint32_t b = (uint32_t)bi;
    float x;
    memcpy(&x, &b, 4);
    const double e = fabs((double)oracle_sin_spec(x) - sin((double)x));
    if (e > es) es = e;
  }
#pragma omp parallel for reduction(max : ee) schedule(static)
  for (int64_t bi = 0x80000000ll; bi <= (int64_t)blo; ++bi) {
    const uint32_t b = (uint32_t)bi;
    float x;
    memcpy(&x, &b, 4);
    const double ref = exp((double)x);
    const double ulp = ldexp(1.0, ilogb((float)ref) - 23);
    const double e = fabs((double)oracle_exp_spec(x) - ref) / ulp;
    if (e > ee) ee = e;
  }
  printf("%.9e %.6f\n", es, ee);
  return 0;
}
