/* Plain C use of the C ABI (include/tsf.h): no torch, no Python.  Runs a
 * [K, N, H, d] block on a constant input x = c, whose output is known
 * exactly (identical keys give uniform softmax weights, so T(x) = x and
 * S(X_t) = X_t: y = 4c), and checks the capability and aliasing errors. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime.h>
#include "tsf.h"

int main(void) {
  const int K = 4, N = 64, H = 2, d = 32;
  const size_t E = (size_t)K * N * H * d;
  tsf_handle* h = NULL;
  if (tsf_create(K, N, H, d, &h) != TSF_OK) { printf("create failed: %s\n", tsf_last_error(NULL)); return 1; }
  tsf_handle* bad = NULL;
  if (tsf_create(K, N, H, 48, &bad) != TSF_ERR_UNSUPPORTED) { printf("expected TSF_ERR_UNSUPPORTED\n"); return 1; }
  tsf_bf16* x; float* y;
  cudaMalloc((void**)&x, E * sizeof(tsf_bf16));
  cudaMalloc((void**)&y, E * sizeof(float));
  tsf_bf16* hx = (tsf_bf16*)malloc(E * sizeof(tsf_bf16));
  float* hy = (float*)malloc(E * sizeof(float));
  for (size_t i = 0; i < E; ++i) hx[i] = 0x3F40;  /* bf16 0.75 */
  cudaMemcpy(x, hx, E * sizeof(tsf_bf16), cudaMemcpyHostToDevice);
  if (tsf_spacetime_block(h, x, y, NULL) != TSF_OK) { printf("block failed: %s\n", tsf_last_error(h)); return 1; }
  cudaMemcpy(hy, y, E * sizeof(float), cudaMemcpyDeviceToHost);
  for (size_t i = 0; i < E; ++i)
    if (hy[i] != 3.0f) { printf("y[%zu] = %.9g, expected 3 (X_t = 2 x, y = 2 X_t)\n", i, hy[i]); return 1; }
  if (tsf_spacetime_block(h, x, (float*)x, NULL) != TSF_ERR_CONFIG) { printf("aliasing not rejected\n"); return 1; }
  tsf_destroy(h);
  cudaFree(x); cudaFree(y); free(hx); free(hy);
  printf("C ABI OK\n");
  return 0;
}
