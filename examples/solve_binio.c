/* A C caller of libddnm.so with no Python anywhere: build a GPU context from
 * a binio instance file pair (written by RomInstance.save_binio, see
 * include/ddnm.h: ddnm_ctx_create_binio), solve a batch of seeded parameters
 * mu = (a, lambda) with the reference's SqpConfig defaults (sqp.py:68-81), and
 * write the latents/multipliers as a binio file -- the layout of the
 * reference CLI's latent.bin (cli.py:327-329), one column per parameter.
 *
 *   gcc -O2 -Iinclude examples/solve_binio.c -Lpaper_2305_15163_b200 -lddnm \
 *       -Wl,-rpath,'$ORIGIN/../paper_2305_15163_b200' -o build/solve_binio
 *   build/solve_binio inst.bin B out.bin
 */
#include <stdio.h>
#include <stdlib.h>

#include "ddnm.h"

/* parameters in the reference's box, a ~ U[1, 1e4], lambda ~ U[5, 25]
 * (SURVEY.md §8(d1)); a fixed LCG keeps the example dependency-free */
static double lcg(unsigned long long* s) {
  *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
  return (double)(*s >> 11) / 9007199254740992.0;
}

#define CHECK(x)                                                          \
  do {                                                                    \
    int rc_ = (x);                                                        \
    if (rc_) {                                                            \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, ddnm_last_error()); \
      return 1;                                                           \
    }                                                                     \
  } while (0)

int main(int argc, char** argv) {
  if (argc < 4) {
    fprintf(stderr, "usage: %s inst.bin B out.bin\n", argv[0]);
    return 2;
  }
  const int B = atoi(argv[2]);
  ddnm_ctx* ctx = NULL;
  CHECK(ddnm_ctx_create_binio(-1, argv[1], 0, &ctx));
  ddnm_info info;
  CHECK(ddnm_ctx_info(ctx, &info));
  const int nD = info.n_primal, nC = info.n_mult;
  double* mu = malloc(sizeof(double) * 2 * B);
  double* x = malloc(sizeof(double) * nD * B);
  double* lam = malloc(sizeof(double) * nC * B);
  int* n_iter = malloc(sizeof(int) * B);
  int* status = malloc(sizeof(int) * B);
  unsigned long long seed = 2305151630ULL;
  for (int k = 0; k < B; ++k) {
    mu[2 * k] = 1.0 + (1e4 - 1.0) * lcg(&seed);
    mu[2 * k + 1] = 5.0 + 20.0 * lcg(&seed);
  }
  ddnm_sqp_cfg cfg = {1e-4, 15, 1e-4, 0.5, 25, 1e-12};
  ddnm_solve_out out = {0};
  out.x = x;
  out.lam = lam;
  out.n_iter = n_iter;
  out.status = status;
  CHECK(ddnm_solve_batch(ctx, B, mu, NULL, NULL, &cfg, &out));
  int64_t evals = 0, kkts = 0;
  CHECK(ddnm_last_counters(ctx, &evals, &kkts));
  int ok = 0;
  for (int k = 0; k < B; ++k) ok += status[k] == DDNM_STATUS_OK;
  /* binio stores column-major: x is [B][nD] row-major = [nD x B] column-major */
  const char* names[3] = {"latent", "multipliers", "mu"};
  const int64_t rows[3] = {nD, nC, 2}, cols[3] = {B, B, B};
  const double* data[3] = {x, lam, mu};
  CHECK(ddnm_binio_write(argv[3], 3, names, NULL, rows, cols, data));
  printf("solved %d parameters: %d ok, %lld block evaluations, %lld KKT solves, n_iter[0] = %d\n",
         B, ok, (long long)evals, (long long)kkts, n_iter[0]);
  ddnm_ctx_destroy(ctx);
  free(mu); free(x); free(lam); free(n_iter); free(status);
  return 0;
}
