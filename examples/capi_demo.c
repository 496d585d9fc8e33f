/* Plain-C consumer of the C-ABI (no Python, no torch): pivots of the paper's
 * 8-point support, then hidft + hidft_to_dft of a band-limited signal
 * synthesised on the device, checked against the planted coefficients.
 *   gcc -O2 examples/capi_demo.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2211_15299_b200 -lsfft_b200 -L/usr/local/cuda/lib64 -lcudart -lm -o capi_demo
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "structfft_b200.h"

#define CHECK(x)                                                              \
  do {                                                                        \
    int rc_ = (x);                                                            \
    if (rc_) {                                                                \
      fprintf(stderr, "%s -> %d: %s\n", #x, rc_, sfft_last_error());         \
      return 1;                                                               \
    }                                                                         \
  } while (0)

int main(void) {
  const int M = 10, k = 8;
  const int64_t J[8] = {23, 187, 190, 247, 386, 731, 990, 994}; /* tests/test_hidft.py:111-118 */
  uint64_t mask = 0;
  int homog = 0;
  CHECK(sfft_analyze(J, k, M, &mask, &homog, 0));
  printf("pivots mask 0x%llx homogeneous %d\n", (unsigned long long)mask, homog);
  if (mask != 0x25ull || !homog) return 2; /* pivots (0, 2, 5) */

  int32_t r[3] = {0, 2, 5};
  sfft_plan* plan = NULL;
  CHECK(sfft_plan_create(J, k, M, r, 3, 0, SFFT_C128, 0, &plan));

  /* planted spectrum -> full signal on the device (sfft_synthesize at all N locations) */
  const int64_t N = 1 << M;
  double c[16];
  for (int i = 0; i < k; ++i) {
    c[2 * i] = cos(0.7 * i + 0.1);
    c[2 * i + 1] = sin(1.3 * i);
  }
  int64_t *dJ, *dloc;
  double *dc, *dsig, *dout;
  cudaMalloc((void**)&dJ, sizeof J);
  cudaMalloc((void**)&dc, sizeof c);
  cudaMalloc((void**)&dloc, 8 * N);
  cudaMalloc((void**)&dsig, 16 * N);
  cudaMalloc((void**)&dout, 16 * k);
  int64_t* loc = (int64_t*)malloc(8 * N);
  for (int64_t i = 0; i < N; ++i) loc[i] = i;
  cudaMemcpy(dJ, J, sizeof J, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, c, sizeof c, cudaMemcpyHostToDevice);
  cudaMemcpy(dloc, loc, 8 * N, cudaMemcpyHostToDevice);
  CHECK(sfft_synthesize(dJ, dc, k, M, dloc, N, dsig, 0));
  CHECK(sfft_hidft(plan, dsig, 1, N, 0, SFFT_OUT_DFT, dout, k, NULL, 0, 0));
  double out[16];
  cudaMemcpy(out, dout, sizeof out, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 2 * k; ++i) err = fmax(err, fabs(out[i] - c[i]));
  printf("max |coeff - planted| = %.3e\n", err);

  /* the same transform from a plain host array, results to a host array */
  double* hsig = (double*)malloc(16 * N);
  cudaMemcpy(hsig, dsig, 16 * N, cudaMemcpyDeviceToHost);
  double hout[16];
  CHECK(sfft_hidft_host(plan, hsig, 1, N, 0, SFFT_OUT_DFT, hout, k, NULL, 0, 0, 0, 0));
  double herr = 0;
  for (int i = 0; i < 2 * k; ++i) herr = fmax(herr, fabs(hout[i] - out[i]));
  printf("host-array path: max |diff| vs device path = %.3e\n", herr);
  free(hsig);
  if (herr != 0.0) return 4;

  /* the same signal stored sample-major (an (N, 2) batch: two copies side by side),
   * inside a PDL chain scope on the default stream */
  double* dnb;
  cudaMalloc((void**)&dnb, 32 * N);
  cudaMemcpy2D(dnb, 32, dsig, 16, 16, N, cudaMemcpyDeviceToDevice);
  cudaMemcpy2D((char*)dnb + 16, 32, dsig, 16, 16, N, cudaMemcpyDeviceToDevice);
  CHECK(sfft_stream_chain(0, 1));
  double* dout2;
  cudaMalloc((void**)&dout2, 32 * k);
  CHECK(sfft_hidft_interleaved(plan, dnb, 2, 2, 0, SFFT_OUT_DFT, dout2, k, 0));
  CHECK(sfft_stream_chain(0, 0));
  double out2[32];
  cudaMemcpy(out2, dout2, sizeof out2, cudaMemcpyDeviceToHost);
  double ierr = 0;
  for (int i = 0; i < 2 * k; ++i) ierr = fmax(ierr, fmax(fabs(out2[i] - out[i]), fabs(out2[2 * k + i] - out[i])));
  printf("interleaved layout: max |diff| vs row-major = %.3e\n", ierr);
  if (ierr != 0.0) return 5;

  /* congruence tree, levels 0..3, host outputs (congruence.py:134-222) */
  int64_t members[4 * 8];
  int32_t node_off[4 * 9], n_nodes[4];
  CHECK(sfft_tree_build(J, k, M, 0, 3, members, node_off, n_nodes, 0));
  printf("tree nodes per level: %d %d %d %d\n", n_nodes[0], n_nodes[1], n_nodes[2], n_nodes[3]);
  if (n_nodes[0] != 1 || n_nodes[1] != 2 || n_nodes[2] != 2 || n_nodes[3] != 4) return 6; /* pivots 0, 2 */

  /* the contract errors come back as status codes */
  int32_t bad[1] = {5};
  sfft_plan* p2 = NULL;
  int rc = sfft_plan_create(J, k, M, bad, 1, 0, SFFT_C128, 0, &p2);
  printf("non-part-homogeneous r -> status %d (%s)\n", rc, sfft_last_error());
  sfft_plan_destroy(plan);
  free(loc);
  return (err < 1e-12 && rc == SFFT_ERR_CONTRACT) ? 0 : 3;
}
