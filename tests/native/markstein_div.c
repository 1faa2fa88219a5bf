/* The division the SST kernel uses for unclipped windows (params.cu k_smooth_rs): with
 * y = RN(1/b), q0 = RN(a y), rem = a - b q0 (exact by fma), q = RN(q0 + rem y), q equals
 * the IEEE quotient RN(a/b) (Markstein's theorem). Checked here for every unclipped window
 * count b = w * ncol (w = 3..17 odd, ncol = (w+1)/2..w) and random window sums a = k 2^-40
 * over every magnitude up to 2^53; exit status 1 on any mismatch.
 *   usage: markstein_div [samples per divisor] */
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
static uint64_t s = 88172645463325252ull;
static inline uint64_t xr(void){ s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
int main(int argc, char **argv){
  const long per = argc > 1 ? atol(argv[1]) : 4000000;
  long long bad = 0, n = 0;
  for (int w = 3; w <= 17; w += 2)
    for (int ncol = (w+1)/2; ncol <= w; ++ncol) {
      double full = (double)(w * ncol);
      double y = 1.0 / full;
      for (long k = 0; k < per; ++k) {
        /* window sums: integers up to 2^53 spread over magnitudes */
        int e = (int)(xr() % 54);
        uint64_t m = xr() & ((e >= 63) ? ~0ull : ((1ull << e) - 1));
        m |= (1ull << (e > 0 ? e - 1 : 0));
        double a = (double)(int64_t)m * 0x1p-40;
        double q0 = a * y;
        double rem = fma(-full, q0, a);
        double q = fma(rem, y, q0);
        double ref = a / full;
        ++n;
        if (q != ref) { if (bad < 5) printf("mismatch w=%d ncol=%d a=%a q=%a ref=%a\n", w, ncol, a, q, ref); ++bad; }
      }
    }
  printf("%lld mismatches in %lld\n", bad, n);
  return bad != 0;
}
