// Microbenchmark of the softmax instruction mix on sm_100a: issue cost per
// warp-instruction per SM sub-partition for MUFU.EX2 (f32, f16x2), F2FP
// packing, FFMA2, FMNMX3 and the polynomial exp2.  One CTA, W warps.
// nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -I paper_2604_16590_b200/csrc tools/ubench.cu -o tools/ubench
#include <cstdio>
#include <cuda_fp16.h>
#include "sm100.cuh"
using namespace tsf;

constexpr int ITERS = 4096;

template <int OP>
__global__ void bench(float* out, long long* cyc) {
  float a[8];
  uint32_t h[8];
  for (int i = 0; i < 8; ++i) { a[i] = -0.001f * (threadIdx.x + i); h[i] = 0x3c003c00u + i; }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (OP == 0) a[i] = ex2(a[i]);                                  // MUFU.EX2 f32
      if constexpr (OP == 1) h[i] = ex2_f16x2(h[i]);                            // MUFU.EX2 f16x2
      if constexpr (OP == 2) { __half2 v = __floats2half2_rn(a[i], a[(i + 1) & 7]); h[i] ^= *reinterpret_cast<uint32_t*>(&v); a[i] += 1e-7f; }  // F2FP
      if constexpr (OP == 3) ffma2(a[i], a[(i + 4) & 7], a[i], a[(i + 4) & 7], 1.0001f, 1.0001f, -1e-7f, -1e-7f);
      if constexpr (OP == 4) a[i] = max3(a[i], a[(i + 1) & 7], a[(i + 2) & 7]);
      if constexpr (OP == 5) { float y0, y1; ex2_poly2(y0, y1, a[i], a[(i + 3) & 7]); a[i] = y0 - 1.0f; a[(i + 3) & 7] = y1 - 1.0f; }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + (float)h[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 1024);
  const char* names[6] = {"MUFU.EX2 f32", "MUFU.EX2 f16x2", "F2FP pack (+FADD)", "FFMA2", "FMNMX3", "ex2_poly2 (pair)"};
  for (int warps : {4, 8}) {
    for (int op = 0; op < 6; ++op) {
      void (*k)(float*, long long*) = nullptr;
      switch (op) {
        case 0: k = bench<0>; break; case 1: k = bench<1>; break; case 2: k = bench<2>; break;
        case 3: k = bench<3>; break; case 4: k = bench<4>; break; default: k = bench<5>; break;
      }
      k<<<1, 32 * warps>>>(out, cyc);
      k<<<1, 32 * warps>>>(out, cyc);
      cudaDeviceSynchronize();
      const double per_smsp_inst = (double)ITERS * 8 * warps / 4;  // op-units per SMSP
      printf("%-20s warps=%d: %.2f cycles per op-unit per SMSP (%.2f per warp-op)\n", names[op], warps,
             (double)cyc[0] / per_smsp_inst, (double)cyc[0] / (ITERS * 8.0));
    }
  }
  return 0;
}
