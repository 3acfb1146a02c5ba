// TMEM load/store throughput on sm_100a: W warps each issue tcgen05.ld/st
// 32x32b.x32 (4 KB per warp-instruction) in a loop.  Prints bytes/clk/SM.
// nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -I paper_2604_16590_b200/csrc tools/ubench3.cu -o tools/ubench3
#include <cstdio>
#include "sm100.cuh"
using namespace tsf;
constexpr int ITERS = 1024;

template <int MODE>  // 0 = ld, 1 = st, 2 = ld+st
__global__ void bench(long long* cyc, float* out) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder + (((warp & 3) * 32) << 16) + (warp / 4) * 64;
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = i;
  float acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    if (MODE != 1) {
      tmem_ld_x32(tm + (it & 1) * 32, r);
      tmem_wait_ld();
      acc += __uint_as_float(r[it & 31]);
    }
    if (MODE != 0) {
      tmem_st_x32(tm + (it & 1) * 32, r);
      tmem_wait_st();
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(holder);
}

int main() {
  long long* cyc; float* out;
  cudaMallocManaged(&cyc, 64); cudaMalloc(&out, 4096 * 4);
  const char* names[3] = {"tcgen05.ld x32", "tcgen05.st x32", "ld + st x32"};
  for (int mode = 0; mode < 3; ++mode)
    for (int w : {4, 8, 16}) {
      void (*k)(long long*, float*) = mode == 0 ? bench<0> : mode == 1 ? bench<1> : bench<2>;
      k<<<1, 32 * w>>>(cyc, out); k<<<1, 32 * w>>>(cyc, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      const double bytes = (double)ITERS * w * 4096 * (mode == 2 ? 2 : 1);
      printf("%-16s warps=%2d: %.1f cycles/iter, %.1f bytes/clk/SM\n", names[mode], w, (double)cyc[0] / ITERS,
             bytes / cyc[0]);
    }
  return 0;
}
