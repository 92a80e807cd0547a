/* C99 translation unit against include/cafxg.h: proves the boundary is plain
 * C (no C++ types, extern "C" linkage) and links against libcafxg.so. Built
 * (not run) by tests/test_abi.py; run on a GPU box it opens a context and
 * checks run_mandelbrot(256, 100)'s golden checksum through the C ABI. */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "cafxg.h"

static void on_done(void* user, int status) {
  *(int*)user = status + 1;
}

int main(void) {
  cafxg_ctx* ctx = NULL;
  int s = cafxg_open(0, &ctx);
  if (s != CAFXG_OK) {
    printf("open: %s (%s)\n", cafxg_status_string(s), cafxg_last_error());
    return s == CAFXG_E_SPAWN ? 0 : 1; /* no GPU: fails loudly, not silently */
  }
  uint64_t h = 0;
  double ms = 0;
  s = cafxg_run_mandelbrot(ctx, 256, 100, &h, &ms);
  printf("run_mandelbrot(256,100) = %llu in %.3f ms\n", (unsigned long long)h, ms);
  int ok = s == CAFXG_OK && h == 12958954340663424292ull;
  /* one async request through the actor facade */
  cafxg_actor* a = NULL;
  cafxg_mandel_desc d;
  memset(&d, 0, sizeof d);
  d.x0 = -2; d.x1 = 1; d.y0 = -1; d.y1 = 1;
  d.width = d.ncols = 32; d.height = d.nrows = 16; d.max_iter = 50;
  d.precision = CAFXG_FP32; d.sampling = CAFXG_CENTRE;
  uint32_t* out = NULL;
  int fired = 0;
  ok = ok && cafxg_spawn(ctx, "mandelbrot", NULL, 0, &a) == CAFXG_OK;
  ok = ok && cafxg_host_alloc(ctx, 32 * 16 * 4, (void**)&out) == CAFXG_OK;
  const void* in[1] = {&d};
  size_t in_bytes[1] = {sizeof d};
  ok = ok && cafxg_actor_enqueue(a, in, in_bytes, 1, out, 32 * 16 * 4, on_done, &fired) ==
                 CAFXG_OK;
  ok = ok && cafxg_sync(ctx) == CAFXG_OK && fired == CAFXG_OK + 1;
  cafxg_actor_release(a);
  cafxg_host_free(ctx, out);
  cafxg_close(ctx);
  printf("%s\n", ok ? "C ABI OK" : "C ABI FAILED");
  return ok ? 0 : 1;
}
