/*
 * fill.c — using libmpr.so from plain C (no Python, no torch): fill the gaps of a small
 * synthetic grid through the C-ABI of include/mpr.h.
 *
 *   gcc -O2 -I include examples/fill.c -L paper_2212_01317_b200 -lmpr \
 *       -Wl,-rpath,$PWD/paper_2212_01317_b200 -o /tmp/mpr_fill_c
 *   /tmp/mpr_fill_c paper_2212_01317_b200/data/calib_q0.5.txt
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "mpr.h"

static int read_table(const char *path, float *T, float *e, int cap) {
  FILE *f = fopen(path, "r");
  if (!f) return -1;
  char line[512];
  int k = 0;
  while (k < cap && fgets(line, sizeof line, f)) {
    if (line[0] == '#') continue;
    char *end = NULL;
    T[k] = strtof(line, &end);
    e[k] = strtof(end, NULL);
    ++k;
  }
  fclose(f);
  return k;
}

int main(int argc, char **argv) {
  const char *table = argc > 1 ? argv[1] : "paper_2212_01317_b200/data/calib_q0.5.txt";
  float T[256], e[256];
  int K = read_table(table, T, e, 256);
  if (K < 2) {
    fprintf(stderr, "cannot read calibration table %s\n", table);
    return 2;
  }
  const int64_t Lx = 96, Ly = 80, n = Lx * Ly;
  float *grid = malloc(sizeof(float) * n), *truth = malloc(sizeof(float) * n), *out = malloc(sizeof(float) * n);
  uint8_t *mask = malloc(n);
  uint32_t s = 12345u;
  for (int64_t i = 0; i < n; ++i) {  /* smooth field + every other site missing at random */
    const int64_t r = i / Lx, c = i % Lx;
    truth[i] = (float)(10.0 + 3.0 * sin(0.11 * r) * cos(0.07 * c) + 0.5 * sin(0.5 * (r + c)));
    s = s * 1664525u + 1013904223u;
    mask[i] = (s >> 31) ? 1 : 0;
    grid[i] = mask[i] ? truth[i] : NAN;
  }
  mpr_config cfg;
  mpr_config_default(&cfg);
  cfg.calib_T = T;
  cfg.calib_e = e;
  cfg.calib_n = K;
  mpr_ctx *ctx = NULL;
  mpr_status st = mpr_init(&cfg, &ctx);
  if (st != MPR_OK) {
    fprintf(stderr, "mpr_init failed: %d\n", (int)st);
    return 1;
  }
#define CHECK(call)                                                     \
  do {                                                                  \
    mpr_status s_ = (call);                                             \
    if (s_ != MPR_OK) {                                                 \
      fprintf(stderr, "%s -> %d: %s\n", #call, (int)s_, mpr_last_error(ctx)); \
      return 1;                                                         \
    }                                                                   \
  } while (0)
  CHECK(mpr_set_data(ctx, grid, mask, Lx, Ly));
  CHECK(mpr_estimate_local_params(ctx, NULL));
  CHECK(mpr_simulate(ctx, 20, 30, 7));
  CHECK(mpr_predict(ctx, out));
  double mae = 0.0;
  int64_t P = 0, bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (mask[i]) {
      if (out[i] != grid[i]) ++bad;  /* samples come back bitwise */
      continue;
    }
    mae += fabs((double)out[i] - (double)truth[i]);
    ++P;
  }
  mpr_info info;
  CHECK(mpr_get_info(ctx, &info));
  printf("%s\nfilled %lld gaps of a %lldx%lld grid, MAE %.4f, %lld sample mismatches, %lld kernel launches\n",
         mpr_version(), (long long)P, (long long)Lx, (long long)Ly, mae / (double)P, (long long)bad,
         (long long)info.total_launches);
  mpr_destroy(ctx);
  free(grid); free(truth); free(out); free(mask);
  return bad == 0 ? 0 : 1;
}
