// Which pipe does F2FP (fp32 pair -> packed 16-bit) share with MUFU.EX2?
// Independent streams, 2 warps per SMSP; cycles per inner iteration.
// nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -I paper_2604_16590_b200/csrc tools/ubench2.cu -o tools/ubench2
#include <cstdio>
#include <cuda_fp16.h>
#include "sm100.cuh"
using namespace tsf;
constexpr int ITERS = 2048;

template <int OP>
__global__ void bench(float* out, long long* cyc) {
  float a[16];
  uint32_t h[16];
  for (int i = 0; i < 16; ++i) { a[i] = -0.001f * (threadIdx.x + i); h[i] = 0x3c003c00u + i; }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (OP == 0 || OP == 2) a[i] = ex2(a[i]);                      // MUFU f32
      if constexpr (OP == 1 || OP == 2) {                                       // F2FP f16x2
        __half2 v = __floats2half2_rn(a[8 + i], a[8 + ((i + 1) & 7)]);
        h[i] += *reinterpret_cast<uint32_t*>(&v);
      }
      if constexpr (OP == 3 || OP == 4) {                                       // F2FP bf16x2
        __nv_bfloat162 v = __floats2bfloat162_rn(a[8 + i], a[8 + ((i + 1) & 7)]);
        h[i] += *reinterpret_cast<uint32_t*>(&v);
      }
      if constexpr (OP == 4) a[i] = ex2(a[i]);
      if constexpr (OP == 5) h[i] += __byte_perm(__float_as_uint(a[8 + i]), __float_as_uint(a[8 + ((i + 1) & 7)]), 0x7632);  // PRMT
      if constexpr (OP == 6) { h[i] += __byte_perm(__float_as_uint(a[8 + i]), __float_as_uint(a[8 + ((i + 1) & 7)]), 0x7632); a[i] = ex2(a[i]); }
      if constexpr (OP == 7) h[i] += 1u;                                        // IADD baseline
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 16; ++i) s += a[i] + (float)h[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 1024);
  const char* names[8] = {"MUFU f32 x8", "F2FP.F16 x8 (+IADD)", "MUFU x8 + F2FP.F16 x8", "F2FP.BF16 x8 (+IADD)",
                          "MUFU x8 + F2FP.BF16 x8", "PRMT x8 (+IADD)", "MUFU x8 + PRMT x8", "IADD x8"};
  void (*ks[8])(float*, long long*) = {bench<0>, bench<1>, bench<2>, bench<3>, bench<4>, bench<5>, bench<6>, bench<7>};
  for (int op = 0; op < 8; ++op) {
    ks[op]<<<1, 256>>>(out, cyc); ks[op]<<<1, 256>>>(out, cyc);
    cudaDeviceSynchronize();
    printf("%-26s: %.1f cycles per iteration (8 warps, per SMSP: %.2f per op-slot)\n", names[op],
           (double)cyc[0] / ITERS, (double)cyc[0] / ITERS / 16.0);
  }
  return 0;
}
