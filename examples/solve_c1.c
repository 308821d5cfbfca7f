/*
 * solve_c1.c -- the C ABI without Python or PyTorch: a C1-shaped PnP-MS2G
 * solve (64^2 ellipse-free disk phantom, 90 views x 96 bins, stages 2x:10 ->
 * full:10, Gaussian denoiser, alpha 0.5) through include/ms2g.h, with device
 * buffers from the CUDA runtime.  Prints the data residual before and after.
 *
 *   gcc -O2 examples/solve_c1.c -Iinclude -I$CUDA/include -Lpaper_2203_07308_b200 -lms2g \
 *       -L$CUDA/lib64 -lcudart -Wl,-rpath,$PWD/paper_2203_07308_b200 -o solve_c1
 *
 * Exit status: 0 on success, the ms2g error code otherwise.
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "ms2g.h"

#define CHECK(call)                                                        \
  do {                                                                     \
    int rc_ = (call);                                                      \
    if (rc_ != MS2G_OK) {                                                  \
      fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, ms2g_last_error()); \
      return rc_;                                                          \
    }                                                                      \
  } while (0)

static double norm2(const float* h, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += (double)h[i] * h[i];
  return sqrt(s);
}

int main(void) {
  const int n = 64, V = 90, B = 96;
  ms2g_geom_desc d = {0};
  d.n = n; d.fov = 2.0; d.n_views = V; d.arc_rad = 2.0 * M_PI; d.n_bins = B;
  d.sod = 4.0; d.sdd = 8.0; d.bin_pitch = 0.0; d.view_begin = 0; d.view_end = V; d.batch = 1;
  const int32_t factors[2] = {2, 1};
  ms2g_plan* plan = NULL;
  CHECK(ms2g_plan_geometry(&d, factors, 2, &plan));

  /* phantom: a centred disk of radius 0.5 (value 1) on the pixel centres */
  const size_t np = (size_t)n * n, ns = (size_t)V * B;
  float* hx = (float*)calloc(np, sizeof(float));
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double y = -1.0 + (i + 0.5) * 2.0 / n, x = -1.0 + (j + 0.5) * 2.0 / n;
      hx[(size_t)i * n + j] = (x * x + y * y <= 0.25) ? 1.f : 0.f;
    }
  float *x = NULL, *b = NULL, *x0 = NULL, *xo = NULL, *r = NULL;
  if (cudaMalloc((void**)&x, np * 4) || cudaMalloc((void**)&b, ns * 4) || cudaMalloc((void**)&x0, np * 4) ||
      cudaMalloc((void**)&xo, np * 4) || cudaMalloc((void**)&r, ns * 4)) {
    fprintf(stderr, "cudaMalloc failed\n");
    return MS2G_ERR_CUDA;
  }
  cudaMemcpy(x, hx, np * 4, cudaMemcpyHostToDevice);
  cudaMemset(x0, 0, np * 4);
  CHECK(ms2g_forward_project(plan, 1, x, NULL, b, NULL, 0, NULL));   /* noiseless data b = A x */

  ms2g_stage stages[2] = {{2, 10, 0}, {1, 10, 0}};
  ms2g_solve_desc sd = {0};
  sd.stages = stages; sd.n_stages = 2; sd.option = 1; sd.n_subsets = 1; sd.seed = 0;
  sd.den.kind = 1; sd.den.sigma = 0.8f; sd.alpha = 0.5f; sd.power_iters = 20; sd.resampler = MS2G_RESAMPLE_MEAN;
  ms2g_sched_entry trace[20];
  CHECK(ms2g_pnp_ms2g_solve(plan, &sd, b, x0, xo, trace, NULL));

  float* hr = (float*)malloc(ns * 4);
  CHECK(ms2g_forward_project(plan, 1, x0, b, r, NULL, 0, NULL));      /* A x0 - b = -b */
  cudaMemcpy(hr, r, ns * 4, cudaMemcpyDeviceToHost);
  const double r0 = norm2(hr, ns);
  CHECK(ms2g_forward_project(plan, 1, xo, b, r, NULL, 0, NULL));      /* A x_20 - b */
  cudaMemcpy(hr, r, ns * 4, cudaMemcpyDeviceToHost);
  const double r1 = norm2(hr, ns);
  printf("steps %d, eta(stage 0) %.6g, eta(stage 1) %.6g, residual %.4g -> %.4g, kernels launched %llu\n",
         trace[19].i, trace[0].eta, trace[19].eta, r0, r1, (unsigned long long)ms2g_launch_count());
  ms2g_plan_destroy(plan);
  cudaFree(x); cudaFree(b); cudaFree(x0); cudaFree(xo); cudaFree(r);
  free(hx); free(hr);
  return (r1 < 0.5 * r0) ? 0 : 1;
}
