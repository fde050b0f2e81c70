/* C client of include/pdcs.h (plain C99, no framework types): the ABI is
 * exercised from C, not only through ctypes.  Usage: pdcs_c_smoke [gpu]
 * Without "gpu": host-only calls and the documented no-device error path.
 * With "gpu": solve min x1 + x2 s.t. x1 + 2 x2 >= 2, x in [0, inf)^2 (optimum 1
 * at (0, 1)) through pdcs_create / pdcs_set_cones / pdcs_solve. */
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "pdcs.h"

static int fails = 0;
#define CHECK(c) do { if (!(c)) { fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); ++fails; } } while (0)

int main(int argc, char **argv) {
  const int gpu = argc > 1 && strcmp(argv[1], "gpu") == 0;
  pdcs_params p;
  pdcs_default_params(&p);
  CHECK(p.check_interval == 40 && p.ruiz_iters == 10 && p.tol == 1e-6);
  /* host-only layout diagnostic on a 2 x 3 structure */
  const int64_t ptr[3] = {0, 2, 3};
  const int32_t col[3] = {0, 2, 1};
  double st[16];
  CHECK(pdcs_tiled_layout_stats(ptr, col, 2, 3, 2, st, 16) > 0 && st[0] == 3.0);
  /* argument errors that need no device */
  pdcs_loopback *grp = NULL;
  CHECK(pdcs_loopback_create(&grp, 0) == PDCS_ERR_ARG);
  CHECK(pdcs_loopback_create(&grp, 2) == PDCS_OK && grp != NULL);
  pdcs_loopback_destroy(grp);
  CHECK(pdcs_set_allocator(NULL, (pdcs_free_fn)0x1, NULL) == PDCS_ERR_ARG);
  /* the LP: G = [1 2], rows NonNeg (G x - h >= 0), h = 2, c = (1, 1), x >= 0 */
  const int64_t rp[2] = {0, 2};
  const int32_t cl[2] = {0, 1};
  const double val[2] = {1.0, 2.0}, c[2] = {1.0, 1.0}, h[1] = {2.0}, l[2] = {0.0, 0.0};
  const double u[2] = {INFINITY, INFINITY};
  pdcs_ctx *ctx = NULL;
  p.tol = 1e-8;
  pdcs_status s = pdcs_create(&ctx, 1, 2, 2, 0, 1, rp, cl, val, c, h, l, u, &p, 0, NULL, PDCS_MEM_HOST, NULL,
                              0, 1);
  if (!gpu) {
    CHECK(s == PDCS_ERR_CUDA && ctx == NULL && strlen(pdcs_last_error(NULL)) > 0);
  } else {
    CHECK(s == PDCS_OK && ctx != NULL);
    const int32_t rk[1] = {PDCS_CONE_NONNEG};
    const int64_t rd[1] = {1};
    CHECK(pdcs_set_cones(ctx, NULL, NULL, 0, rk, rd, 1) == PDCS_OK);
    pdcs_result_t r;
    CHECK(pdcs_solve(ctx, &r) == PDCS_OK);
    CHECK(r.status == PDCS_OPTIMAL && fabs(r.kkt.pobj - 1.0) < 1e-6);
    double x[2], y[1];
    CHECK(pdcs_get_iterate(ctx, PDCS_BEST, PDCS_ORIGINAL, x, y) == PDCS_OK);
    CHECK(fabs(x[0]) < 1e-5 && fabs(x[1] - 1.0) < 1e-5 && fabs(y[0] - 0.5) < 1e-5);
    printf("solve: status %d, objective %.9f, x = (%.3g, %.6f), y = %.6f, %lld iterations\n", r.status,
           r.kkt.pobj, x[0], x[1], y[0], (long long)r.iters);
    pdcs_destroy(ctx);
  }
  printf("%s: %d failures\n", gpu ? "gpu" : "host", fails);
  return fails != 0;
}
