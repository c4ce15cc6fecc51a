/* Plain-C use of the library (no Python): the exact rank-2 QTT of the cyclic
 * shift (PAPER P:1226-1231 family of closed forms; SURVEY pin P4) applied to a
 * vector through include/qtt.h, checked bitwise against the shifted input.
 *
 *   gcc -std=c99 -Iinclude -I/usr/local/cuda/include examples/qtt_c_example.c \
 *       -Lpaper_1511_06029_b200 -lqtt_b200 -L/usr/local/cuda/lib64 -lcudart -o qtt_c_example
 *   ./qtt_c_example            # needs an sm_100 GPU
 *   ./qtt_c_example --plan     # host only: the stage schedule of a rank profile
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "qtt.h"

#define D 12

/* core k (0-based, acts on bit k) of the shift by +1: carry chain from the LSB.
 * G[a][i][j][b] row-major, i = output digit, j = input digit. */
static double* shift_core(int k, int d, int64_t* ra, int64_t* rb) {
  *ra = (k == 0) ? 1 : 2;
  *rb = (k == d - 1) ? 1 : 2;
  double* g = calloc((size_t)(*ra) * 4 * (*rb), sizeof(double));
  for (int a = 0; a < *ra; ++a)
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) {
        const int c = (k == 0) ? 1 : a;           /* carry in (the +1 enters at bit 0) */
        if (i != (j ^ c)) continue;
        const int cout = j & c;                     /* carry out */
        if (k == d - 1) {
          g[((a * 2 + i) * 2 + j) * (*rb) + 0] = 1.0;   /* cyclic: drop the final carry */
        } else {
          g[((a * 2 + i) * 2 + j) * (*rb) + cout] = 1.0;
        }
      }
  return g;
}

int main(int argc, char** argv) {
  int64_t ranks[D + 1];
  double* cores[D];
  ranks[0] = 1;
  for (int k = 0; k < D; ++k) {
    int64_t ra, rb;
    cores[k] = shift_core(k, D, &ra, &rb);
    ranks[k + 1] = rb;
  }
  if (argc > 1 && strcmp(argv[1], "--plan") == 0) {
    int n = 0, kf[D], kl[D], var[D], ks[D];
    qtt_status_t s = qtt_plan_stages_split(D, ranks, 0, 10, &n, kf, kl, var, ks);
    printf("%s: %d stages:", qtt_status_string(s), n);
    for (int i = 0; i < n; ++i) printf(" [%d-%d v%d s%d]", kf[i], kl[i], var[i], ks[i]);
    printf("\n");
    return s == QTT_SUCCESS ? 0 : 1;
  }
  const size_t N = (size_t)1 << D;
  qtt_handle_t h = NULL;
  qtt_status_t s = qtt_create(&h, D, ranks, (const double* const*)cores);
  for (int k = 0; k < D; ++k) free(cores[k]);     /* the library copied them */
  if (s != QTT_SUCCESS) {
    fprintf(stderr, "qtt_create: %s\n", qtt_status_string(s));
    return 1;
  }
  double* x = malloc(N * sizeof(double));
  double* y = malloc(N * sizeof(double));
  for (size_t i = 0; i < N; ++i) x[i] = (double)(i * 7919 % 1000) - 500.0;
  double *dx = NULL, *dy = NULL;
  if (cudaMalloc((void**)&dx, N * sizeof(double)) != cudaSuccess ||
      cudaMalloc((void**)&dy, N * sizeof(double)) != cudaSuccess) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 1;
  }
  cudaMemcpy(dx, x, N * sizeof(double), cudaMemcpyHostToDevice);
  {   /* what one apply launches: at this size one fused persistent launch */
    int launches = 0, n = 0, kf[D], kl[D], var[D];
    if (qtt_get_apply_plan(h, 1, &launches, &n, kf, kl, var) == QTT_SUCCESS) {
      printf("apply plan: %d launch(es), %d stage(s):", launches, n);
      for (int i = 0; i < n; ++i) printf(" [%d-%d v%d]", kf[i], kl[i], var[i]);
      printf("\n");
    }
  }
  s = qtt_apply(h, dx, dy, 1, NULL);
  if (s == QTT_SUCCESS && cudaDeviceSynchronize() != cudaSuccess) s = QTT_ERROR_CUDA;
  cudaMemcpy(y, dy, N * sizeof(double), cudaMemcpyDeviceToHost);
  size_t bad = 0;
  for (size_t i = 0; i < N; ++i)
    if (y[(i + 1) % N] != x[i]) ++bad;               /* y = roll(x, +1), bitwise */
  printf("qtt_apply: %s, %zu of %zu entries differ from roll(x, 1)\n", qtt_status_string(s), bad, N);
  qtt_destroy(h);
  cudaFree(dx);
  cudaFree(dy);
  free(x);
  free(y);
  return (s == QTT_SUCCESS && bad == 0) ? 0 : 1;
}
