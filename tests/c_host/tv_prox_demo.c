/* A C host using libpsb200 through include/psb200.h alone -- no CUDA runtime
 * calls and no torch: context, device buffers, upload, the TV prox
 * (tv.py:53-89 -> psb_tv_prox2d, fp64 bit-exact path), download.
 *
 *   tv_prox_demo H W inner weight in.bin out.bin
 * in.bin: H*W float64 (x); out.bin: H*W float64 (u). */
#include <stdio.h>
#include <stdlib.h>

#include "psb200.h"

#define CHECK(call)                                                    \
  do {                                                                 \
    int rc_ = (call);                                                  \
    if (rc_ != PSB_OK) {                                               \
      fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, psb_last_error()); \
      return 1;                                                        \
    }                                                                  \
  } while (0)

int main(int argc, char** argv) {
  if (argc != 7) {
    fprintf(stderr, "usage: %s H W inner weight in.bin out.bin\n", argv[0]);
    return 2;
  }
  const int H = atoi(argv[1]), W = atoi(argv[2]), inner = atoi(argv[3]);
  const double weight = atof(argv[4]);
  const int64_t HW = (int64_t)H * W;
  double* x = malloc(sizeof(double) * HW);
  double* u = malloc(sizeof(double) * HW);
  FILE* f = fopen(argv[5], "rb");
  if (!f || fread(x, sizeof(double), HW, f) != (size_t)HW) return 3;
  fclose(f);

  psb_ctx* ctx = NULL;
  void *dx = NULL, *dq = NULL, *du = NULL;
  CHECK(psb_ctx_create(0, &ctx));
  CHECK(psb_buf_alloc(ctx, sizeof(double) * HW, &dx));
  CHECK(psb_buf_alloc(ctx, sizeof(double) * 6 * HW, &dq)); /* 3 dual slots, zero = cold start */
  CHECK(psb_buf_alloc(ctx, sizeof(double) * HW, &du));
  CHECK(psb_upload(ctx, dx, x, sizeof(double) * HW));
  /* two calls: the second is warm-started from the first's dual (tv.py:60-89) */
  for (int call = 0; call < 2; ++call)
    CHECK(psb_tv_prox2d(PSB_F64, dx, HW, dq, 6 * HW, NULL, 1, weight, NULL, 0, NULL, H, W, inner,
                        1, 0, 0.125, du, HW, psb_ctx_stream(ctx)));
  CHECK(psb_download(ctx, u, du, sizeof(double) * HW));
  CHECK(psb_buf_free(ctx, dx));
  CHECK(psb_buf_free(ctx, dq));
  CHECK(psb_buf_free(ctx, du));
  CHECK(psb_ctx_destroy(ctx));

  f = fopen(argv[6], "wb");
  if (!f || fwrite(u, sizeof(double), HW, f) != (size_t)HW) return 4;
  fclose(f);
  free(x);
  free(u);
  return 0;
}
