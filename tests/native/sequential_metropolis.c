/* sequential_metropolis.c — an independent sampler for SPEC acceptance criterion 6 (test
 * infrastructure, shares nothing with oracle/ or the CUDA path): random-order single-site
 * Metropolis on an open Lx x Ly lattice of the MPR Hamiltonian H = -J sum_<ij> cos(q(phi_i -
 * phi_j)) (Eq.(1)), fp64 with libm, proposals phi' ~ U[0, 2pi) (reading R1),
 * acceptance min(1, exp(-dE / T)); the sites with mask != 0 stay frozen.
 * Input on stdin: Lx Ly T q J chains burn sweeps seed, then Lx*Ly lines "mask phi".
 * Output: per chain, the mean whole-lattice specific energy e = H / (J N_bonds) over the
 * measured sweeps (one sweep = as many random site picks as free sites). */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

static uint64_t st;
static uint64_t next_u64(void) {  /* splitmix64 */
  uint64_t z = (st += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static double uniform(void) { return (double)(next_u64() >> 11) * 0x1p-53; }

int main(void) {
  int Lx, Ly, chains, burn, sweeps;
  double T, q, J;
  unsigned long long seed;
  if (scanf("%d %d %lf %lf %lf %d %d %d %llu", &Lx, &Ly, &T, &q, &J, &chains, &burn, &sweeps, &seed) != 9) return 2;
  const int n = Lx * Ly;
  int *mask = malloc(sizeof(int) * n), *freeidx = malloc(sizeof(int) * n);
  double *phi0 = malloc(sizeof(double) * n), *phi = malloc(sizeof(double) * n);
  int nfree = 0;
  for (int i = 0; i < n; ++i) {
    if (scanf("%d %lf", &mask[i], &phi0[i]) != 2) return 2;
    if (!mask[i]) freeidx[nfree++] = i;
  }
  const double nbonds = (double)(2 * Lx * Ly - Lx - Ly);
  const double pi2 = 2.0 * acos(-1.0);
  for (int ch = 0; ch < chains; ++ch) {
    st = seed * 1000003ull + (uint64_t)ch;
    for (int i = 0; i < n; ++i) phi[i] = phi0[i];
    double esum = 0.0;
    for (int s = 0; s < burn + sweeps; ++s) {
      for (int k = 0; k < nfree; ++k) {
        const int i = freeidx[(int)(uniform() * nfree)];
        const int r = i / Lx, c = i % Lx;
        const double prop = uniform() * pi2;
        double dE = 0.0;
        const int nb[4] = {r > 0 ? i - Lx : -1, r + 1 < Ly ? i + Lx : -1, c > 0 ? i - 1 : -1, c + 1 < Lx ? i + 1 : -1};
        for (int t = 0; t < 4; ++t)
          if (nb[t] >= 0) dE += -J * (cos(q * (prop - phi[nb[t]])) - cos(q * (phi[i] - phi[nb[t]])));
        if (dE <= 0.0 || uniform() < exp(-dE / T)) phi[i] = prop;
      }
      if (s >= burn) {
        double H = 0.0;
        for (int r = 0; r < Ly; ++r)
          for (int c = 0; c < Lx; ++c) {
            const int i = r * Lx + c;
            if (c + 1 < Lx) H -= cos(q * (phi[i] - phi[i + 1]));
            if (r + 1 < Ly) H -= cos(q * (phi[i] - phi[i + Lx]));
          }
        esum += H / nbonds;
      }
    }
    printf("%.12f\n", esum / sweeps);
  }
  return 0;
}
