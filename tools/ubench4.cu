// TMEM read bandwidth by shape / batching (tcgen05.ld), 4 or 8 warps, one CTA.
#include <cstdio>
#include "sm100.cuh"
using namespace tsf;
constexpr int ITERS = 512;

__device__ __forceinline__ void ld16x256_x8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(taddr));
}

template <int MODE>
__global__ void bench(long long* cyc, float* out) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = holder + (((warp & 3) * 32) << 16) + (warp / 4) * 128;
  uint32_t r[128];
  float acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    if (MODE == 0) {  // 4 x (32x32b.x32) then one wait: 16 KB per warp
#pragma unroll
      for (int k = 0; k < 4; ++k) tmem_ld_x32(base + 32 * k, r + 32 * k);
      tmem_wait_ld();
    } else if (MODE == 1) {  // 2 x x32 then wait: 8 KB
      tmem_ld_x32(base, r);
      tmem_ld_x32(base + 32, r + 32);
      tmem_wait_ld();
    } else if (MODE == 2) {  // 16x256b.x8: 32 regs, 4 KB per warp
      ld16x256_x8(base, r);
      tmem_wait_ld();
    } else {  // 32x32b.x32 single, 4 KB
      tmem_ld_x32(base, r);
      tmem_wait_ld();
    }
#pragma unroll
    for (int k = 0; k < 128; k += 16) acc += __uint_as_float(r[k]);
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
  const char* names[4] = {"4x x32 + 1 wait (16 KB)", "2x x32 + 1 wait (8 KB)", "16x256b.x8 (4 KB)", "x32 (4 KB)"};
  const int kb[4] = {16, 8, 4, 4};
  for (int mode = 0; mode < 4; ++mode)
    for (int w : {4, 8}) {
      void (*k)(long long*, float*) = mode == 0 ? bench<0> : mode == 1 ? bench<1> : mode == 2 ? bench<2> : bench<3>;
      k<<<1, 32 * w>>>(cyc, out); k<<<1, 32 * w>>>(cyc, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      printf("%-26s warps=%d: %.1f cycles/iter, %.1f bytes/clk/SM\n", names[mode], w, (double)cyc[0] / ITERS,
             (double)ITERS * w * kb[mode] * 1024 / cyc[0]);
    }
  return 0;
}
