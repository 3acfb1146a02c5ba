// tcgen05.mma issue/throughput: cycles per MMA (M=128, K=16) vs N, SS and TS
// (A from TMEM) forms; one CTA, one issuing thread.
#include <cstdio>
#include "sm100.cuh"
using namespace tsf;
constexpr int NMMA = 2048;

template <int N, bool TS>
__global__ void bench(long long* cyc) {
  __shared__ __align__(1024) uint8_t sab[256 * 128];  // B up to N = 256 rows; A aliases it
  uint8_t* sa = sab;
  uint8_t* sb = sab;
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  for (int i = threadIdx.x; i < 128 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sa)[i] = 0x3c003c00u;
  for (int i = threadIdx.x; i < 256 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sb)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc(128, N, 0, TS ? 1 : 0, true);
    const uint64_t da = make_sdesc(smem_u32(sa), 16, 1024, SWZ_128B);
    const uint64_t db = TS ? make_sdesc(smem_u32(sb), 16384, 1024, SWZ_128B) : make_sdesc(smem_u32(sb), 16, 1024, SWZ_128B);
    long long t0 = clock64();
    for (int i = 0; i < NMMA; ++i) {
      if (TS) mma_ts(tm + 256, tm, db, idesc, 1);
      else mma_ss(tm + 256, da, db, idesc, 1);
    }
    long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tm);
}

template <int N, bool TS>
void run(long long* cyc) {
  bench<N, TS><<<1, 128>>>(cyc);
  bench<N, TS><<<1, 128>>>(cyc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  printf("%s N=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma (ideal %d)\n", TS ? "TS" : "SS", N,
         (double)cyc[0] / NMMA, (double)cyc[1] / NMMA, 128 * N / 256);
}

int main() {
  long long* cyc;
  cudaMallocManaged(&cyc, 64);
  run<16, false>(cyc); run<32, false>(cyc); run<64, false>(cyc); run<96, false>(cyc); run<128, false>(cyc);
  run<192, false>(cyc); run<256, false>(cyc);
  run<16, true>(cyc); run<64, true>(cyc); run<80, true>(cyc); run<96, true>(cyc); run<128, true>(cyc); run<144, true>(cyc); run<256, true>(cyc);
  return 0;
}
