/*
 * fill_slabs.c — the multi-rank path of libmpr.so from plain C: W ranks fill one grid as
 * row slabs (MPR_SHARD_ROWS), each rank a context driven by its own host thread and joined
 * by libmpr's in-process communicator (mpr_group_create). Rank w runs on device w % ndev,
 * so the same program drives W GPUs of one node, or W contexts on one GPU. Every rank makes
 * the same SPMD calls; the decomposition (slab-local memory, the distributed parameter
 * stage, the halo exchange per colour half-sweep, the all-gathered prediction) runs inside
 * the library. The program checks that every rank returns the prediction a single context
 * computes, bit for bit.
 *
 * With NCCL across processes instead (one process per GPU), each rank would draw the id
 * with mpr_nccl_unique_id on rank 0, distribute it (e.g. MPI_Bcast), create the
 * communicator with mpr_nccl_comm_init(W, rank, id, device, &comm) and set cfg.nccl_comm.
 *
 *   gcc -O2 -I include examples/fill_slabs.c -L paper_2212_01317_b200 -lmpr -lpthread \
 *       -Wl,-rpath,$PWD/paper_2212_01317_b200 -lm -o /tmp/mpr_fill_slabs
 *   /tmp/mpr_fill_slabs paper_2212_01317_b200/data/calib_q0.5.txt 4
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mpr.h"

#define MAXW 16

static float T_tab[256], e_tab[256];
static int K_tab;
static int64_t Lx = 160, Ly = 123;
static float *grid;
static uint8_t *mask;
static float *outs[MAXW];
static mpr_group *group;
static int W, ndev = 1;
static int rank_status[MAXW];

static int read_table(const char *path) {
  FILE *f = fopen(path, "r");
  if (!f) return -1;
  char line[512];
  int k = 0;
  while (k < 256 && fgets(line, sizeof line, f)) {
    if (line[0] == '#') continue;
    char *end = NULL;
    T_tab[k] = strtof(line, &end);
    e_tab[k] = strtof(end, NULL);
    ++k;
  }
  fclose(f);
  return k;
}

/* one fill on a context; shard < 0: a single context without a communicator */
static int fill(int rank, int shard, float *out) {
  mpr_config cfg;
  mpr_config_default(&cfg);
  cfg.calib_T = T_tab;
  cfg.calib_e = e_tab;
  cfg.calib_n = K_tab;
  if (shard >= 0) {
    cfg.device = rank % ndev;
    cfg.group = group;
    cfg.group_rank = rank;
    cfg.shard = shard;
  }
  mpr_ctx *ctx = NULL;
  mpr_status st = mpr_init(&cfg, &ctx);
  if (st != MPR_OK) {
    fprintf(stderr, "rank %d: mpr_init -> %d\n", rank, (int)st);
    return 1;
  }
  const char *where = "";
  if ((st = mpr_set_data(ctx, grid, mask, Lx, Ly)) != MPR_OK) where = "mpr_set_data";
  else if ((st = mpr_estimate_local_params(ctx, NULL)) != MPR_OK) where = "mpr_estimate_local_params";
  else if ((st = mpr_simulate(ctx, 12, 20, 7)) != MPR_OK) where = "mpr_simulate";
  else if ((st = mpr_predict(ctx, out)) != MPR_OK) where = "mpr_predict";
  if (st != MPR_OK) fprintf(stderr, "rank %d: %s -> %d: %s\n", rank, where, (int)st, mpr_last_error(ctx));
  mpr_destroy(ctx);
  return st == MPR_OK ? 0 : 1;
}

static void *rank_main(void *arg) {
  const int rank = (int)(intptr_t)arg;
  rank_status[rank] = fill(rank, MPR_SHARD_ROWS, outs[rank]);
  return NULL;
}

int main(int argc, char **argv) {
  const char *table = argc > 1 ? argv[1] : "paper_2212_01317_b200/data/calib_q0.5.txt";
  W = argc > 2 ? atoi(argv[2]) : 4;
  if (W < 1 || W > MAXW) return 2;
  if (argc > 3) ndev = atoi(argv[3]);
  if (ndev < 1) ndev = 1;
  K_tab = read_table(table);
  if (K_tab < 2) {
    fprintf(stderr, "cannot read calibration table %s\n", table);
    return 2;
  }
  const int64_t n = Lx * Ly;
  grid = malloc(sizeof(float) * n);
  mask = malloc(n);
  uint32_t s = 4242u;
  for (int64_t i = 0; i < n; ++i) {  /* a smooth field with a variance step, 45 % missing */
    const int64_t r = i / Lx, c = i % Lx;
    const double amp = c < Lx / 2 ? 1.0 : 6.0;
    s = s * 1664525u + 1013904223u;
    mask[i] = (s >> 8) % 100 >= 45;
    grid[i] = mask[i] ? (float)(amp * sin(0.09 * r) * cos(0.13 * c) + 0.2 * sin(0.7 * (r - c))) : NAN;
  }
  float *ref = malloc(sizeof(float) * n);
  if (fill(0, -1, ref)) return 1;
  if (mpr_group_create(W, &group) != MPR_OK) return 1;
  pthread_t th[MAXW];
  for (int w = 0; w < W; ++w) {
    outs[w] = malloc(sizeof(float) * n);
    pthread_create(&th[w], NULL, rank_main, (void *)(intptr_t)w);
  }
  for (int w = 0; w < W; ++w) pthread_join(th[w], NULL);
  mpr_group_destroy(group);
  int64_t mismatches = 0;
  int failed = 0;
  for (int w = 0; w < W; ++w) {
    failed |= rank_status[w];
    if (!rank_status[w])
      for (int64_t i = 0; i < n; ++i)
        if (memcmp(&outs[w][i], &ref[i], sizeof(float)) != 0) ++mismatches;
  }
  printf("%s\n%d row slabs on %d device(s), %lldx%lld grid: %lld mismatches against one context\n", mpr_version(), W,
         ndev, (long long)Lx, (long long)Ly, (long long)mismatches);
  return failed || mismatches ? 1 : 0;
}
