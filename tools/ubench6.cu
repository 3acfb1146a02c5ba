// Microbenchmark of the flash softmax's exponential phase in isolation: per
// warp, 128 fp32 scores -> scale/subtract (FFMA2) -> exp2 (MUFU, EMU of 16 on
// the polynomial) -> fp16 pack (F2FP) [-> tcgen05.st to TMEM], the same
// three-pass structure as attn_flash.cuh.  Reports cycles per 128-column row
// per warp with W warps on each SM sub-partition (W = 1: ping-pong, one
// warpgroup at a time; W = 2: both softmax warpgroups at once).
// nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_16590_b200/csrc tools/ubench6.cu -o tools/ubench6
#include <cstdio>
#include <cuda_fp16.h>
#include "sm100.cuh"
#include "attn_common.cuh"
using namespace tsf;

constexpr int ITERS = 512;

template <int EMU, bool STORE, int PASSW, bool LDMAX = false>
__global__ void __launch_bounds__(256, 1) bench(const float* in, uint32_t* out, long long* cyc) {
  __shared__ uint32_t holder;
  if (threadIdx.x < 32) tmem_alloc<512>(&holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  const uint32_t warp = threadIdx.x / 32;
  const uint32_t lane_base = ((warp & 3) * 32) << 16;
  const uint32_t tP = tmem + lane_base + 128 * (warp >> 2);
  uint32_t sv[128];
#pragma unroll
  for (int c = 0; c < 128; ++c) sv[c] = __float_as_uint(in[(threadIdx.x * 7 + c) & 1023]);
  const float sl2 = 0.18033688f;
  float nmb = -1.0f;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
    nmb = fmaf(nmb, 0.999f, -1e-3f);   // loop-carried: nothing can be hoisted
    if constexpr (LDMAX) {
      // the sub-step's S load and row max as in the kernel (4 FMNMX3 chains)
#pragma unroll
      for (int c = 0; c < 128; c += 32) tmem_ld_x32(tP - 128 * (warp >> 2) + 256 + c, sv + c);
      tmem_wait_ld();
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 128; c += 8)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          m4[q] = max3(m4[q], __uint_as_float(sv[c + 2 * q]), __uint_as_float(sv[c + 2 * q + 1]));
      nmb = fminf(nmb, -max3(m4[0], m4[1], fmaxf(m4[2], m4[3])) * 1e-3f);
    }
#pragma unroll
    for (int c0 = 0; c0 < 128; c0 += PASSW) {
      float xv[PASSW], pv[PASSW];
      uint32_t pk[PASSW / 2];
#pragma unroll
      for (int c = 0; c < PASSW; c += 2)
        ffma2(xv[c], xv[c + 1], __uint_as_float(sv[c0 + c]), __uint_as_float(sv[c0 + c + 1]), sl2, sl2, nmb, nmb);
#pragma unroll
      for (int c = 0; c < PASSW; c += 2) {
        if (((c >> 1) & 7) >= 8 - EMU / 2) {
          ex2_poly2(pv[c], pv[c + 1], xv[c], xv[c + 1]);
        } else {
          pv[c] = ex2(xv[c]);
          pv[c + 1] = ex2(xv[c + 1]);
        }
      }
#pragma unroll
      for (int c = 0; c < PASSW; c += 2) pk[c / 2] = pack2<true>(pv[c], pv[c + 1]);
      if constexpr (STORE) {
#pragma unroll
        for (int c = 0; c < PASSW / 2; c += 16) tmem_st_x16(tP + 64 + (c0 / 2) + c, pk + c);
      } else {
#pragma unroll
        for (int c = 0; c < PASSW / 2; ++c) acc ^= pk[c];
      }
    }
    if constexpr (STORE) tmem_wait_st();
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int EMU, bool STORE, int PASSW, bool LDMAX = false>
void run(const float* in, uint32_t* out, long long* cyc) {
  for (int w : {1, 2}) {
    bench<EMU, STORE, PASSW, LDMAX><<<1, 128 * w>>>(in, out, cyc);
    bench<EMU, STORE, PASSW, LDMAX><<<1, 128 * w>>>(in, out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
    const double per_row = (double)cyc[0] / ITERS;   // every warp did ITERS rows
    printf("ldmax=%d EMU=%d store=%d passw=%3d warps/SMSP=%d: %7.1f cycles per iteration = %6.1f per row-tile per SMSP "
           "(MUFU bound %5.1f)\n", (int)LDMAX, EMU, STORE, PASSW, w, per_row, per_row / w, 128 * (16 - EMU) / 16 * 8.0);
  }
}

int main() {
  float* in;
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&in, 4096 * 4);
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 1024);
  float h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = (float)((i * 37) % 200) * 0.05f - 5.0f;
  cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  run<0, false, 32>(in, out, cyc);
  run<4, false, 32>(in, out, cyc);
  run<6, false, 32>(in, out, cyc);
  run<8, false, 32>(in, out, cyc);
  run<4, true, 32>(in, out, cyc);
  run<6, true, 32>(in, out, cyc);
  run<4, true, 64>(in, out, cyc);
  run<4, true, 128>(in, out, cyc);
  run<0, true, 32>(in, out, cyc);
  run<4, true, 32, true>(in, out, cyc);
  run<6, true, 32, true>(in, out, cyc);
  run<8, true, 32, true>(in, out, cyc);
  return 0;
}
