// Probe: does tcgen05.mma kind::f16 accept A = fp16 with B = bf16 (mixed
// formats in the instruction descriptor)?  D[128x16] = A[128x64] * B[16x64]^T.
// Build: nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -I paper_2604_16590_b200/csrc tools/mma_mixed_test.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>
#include "sm100.cuh"
using namespace tsf;

__device__ uint32_t swz(uint32_t r, uint32_t c) {  // element (r, c) of a 64-wide 16-bit SW128 tile
  const uint32_t byte = c * 2;
  return r * 128 + (((byte >> 4) ^ (r & 7)) << 4) + (byte & 15);
}

__global__ void probe(const float* A, const float* B, float* D, int a_f16, int b_f16) {
  __shared__ __align__(1024) uint8_t sa[128 * 128];
  __shared__ __align__(1024) uint8_t sb[16 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int t = threadIdx.x;
  for (int i = t; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, c = i % 64;
    uint16_t v;
    if (a_f16) { __half h = __float2half_rn(A[i]); v = *reinterpret_cast<uint16_t*>(&h); }
    else { __nv_bfloat16 h = __float2bfloat16_rn(A[i]); v = *reinterpret_cast<uint16_t*>(&h); }
    *reinterpret_cast<uint16_t*>(sa + swz(r, c)) = v;
  }
  for (int i = t; i < 16 * 64; i += blockDim.x) {
    const int r = i / 64, c = i % 64;
    uint16_t v;
    if (b_f16) { __half h = __float2half_rn(B[i]); v = *reinterpret_cast<uint16_t*>(&h); }
    else { __nv_bfloat16 h = __float2bfloat16_rn(B[i]); v = *reinterpret_cast<uint16_t*>(&h); }
    *reinterpret_cast<uint16_t*>(sb + swz(r, c)) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (t < 32) tmem_alloc<32>(&holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder;
  if (t == 0) {
    const uint32_t idesc = (1u << 4) | ((a_f16 ? 0u : 1u) << 7) | ((b_f16 ? 0u : 1u) << 10) | ((16u >> 3) << 17) |
                           ((128u >> 4) << 24);
    for (int k = 0; k < 4; ++k)
      mma_ss(tm, make_sdesc(smem_u32(sa) + 32 * k, 16, 1024, SWZ_128B),
             make_sdesc(smem_u32(sb) + 32 * k, 16, 1024, SWZ_128B), idesc, k > 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[16];
  tmem_ld_x16(tm + (((t / 32) * 32) << 16), r);
  tmem_wait_ld();
  for (int j = 0; j < 16; ++j) D[t * 16 + j] = __uint_as_float(r[j]);
  tc_fence_before();
  __syncthreads();
  if (t < 32) tmem_dealloc<32>(tm);
}

int main() {
  float *A, *B, *D;
  cudaMallocManaged(&A, 128 * 64 * 4);
  cudaMallocManaged(&B, 16 * 64 * 4);
  cudaMallocManaged(&D, 128 * 16 * 4);
  srand(1);
  for (int i = 0; i < 128 * 64; ++i) A[i] = (rand() % 17 - 8) / 8.0f;   // exact in fp16 and bf16
  for (int i = 0; i < 16 * 64; ++i) B[i] = (rand() % 17 - 8) / 4.0f;
  const char* names[4] = {"bf16 x bf16", "bf16 x f16", "f16 x bf16", "f16 x f16"};
  for (int mode = 0; mode < 4; ++mode) {
    const int af = mode >> 1, bf = mode & 1;
    probe<<<1, 128>>>(A, B, D, af, bf);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: CUDA error %s\n", names[mode], cudaGetErrorString(e)); return 1; }
    double err = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 16; ++n) {
        double ref = 0;
        for (int k = 0; k < 64; ++k) ref += (double)A[m * 64 + k] * B[n * 64 + k];
        err = fmax(err, fabs(ref - D[m * 16 + n]));
      }
    printf("A=%s: max err %g\n", names[mode], err);
  }
  return 0;
}
