// HBM-bound layout kernels (SURVEY 8(a) a5 unpack/pack, a10 transpose).
//
// All of them move whole rows of R = H*d bf16 elements (the contiguous inner
// run of a [K, N, H, d] tensor) with 16-byte vector loads/stores: thread i of
// a row copies bytes [16 i, 16 i + 16), so both the read and the write side
// are fully coalesced whenever R*2 >= 512 bytes (every BASELINE config).
// Grid-stride loops over rows, grid sized to a multiple of the SM count.
#pragma once
#include <cstdint>

namespace tsf {

// out[b][a] = in[a][b] for rows of `vecs` 16-byte vectors; A x B rows.
// Up to two tensors per launch (in1/out1 may be null).
__global__ void __launch_bounds__(256) transpose_rows_kernel(const uint4* __restrict__ in0, uint4* __restrict__ out0,
                                                             const uint4* __restrict__ in1, uint4* __restrict__ out1,
                                                             long long A, long long B, int vecs) {
  const long long total = A * B * vecs;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / vecs;
    const int v = (int)(i - row * vecs);
    const long long a = row / B, b = row - a * B;
    const long long o = (b * A + a) * vecs + v;
    const uint4 x0 = in0[i];
    uint4 x1;
    if (in1) x1 = in1[i];
    out0[o] = x0;
    if (in1) out1[o] = x1;
  }
}

// Same permutation, 4 independent 16-byte loads in flight per thread before
// the stores, and the (a, b) decomposition done once per 1024-vector chunk
// instead of with two 64-bit divisions per vector.
__global__ void __launch_bounds__(256) transpose_rows_ilp_kernel(const uint4* __restrict__ in, uint4* __restrict__ out,
                                                                 long long A, long long B, int vecs) {
  constexpr int U = 4, CHUNK = 256 * U;
  const long long total = A * B * vecs;
  for (long long c0 = (long long)blockIdx.x * CHUNK; c0 < total; c0 += (long long)gridDim.x * CHUNK) {
    const long long row0 = c0 / vecs;
    const int v0 = (int)(c0 - row0 * vecs);
    const long long a0 = row0 / B, b0 = row0 - a0 * B;
    uint4 x[U];
    long long o[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = c0 + threadIdx.x + u * 256;
      o[u] = -1;
      if (i < total) {
        x[u] = in[i];
        const int e = v0 + (int)threadIdx.x + u * 256;  // vectors past the chunk's first row start
        const int dr = e / vecs, v = e - dr * vecs;
        long long a = a0, b = b0 + dr;
        while (b >= B) { b -= B; ++a; }
        o[u] = (b * A + a) * vecs + v;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (o[u] >= 0) out[o[u]] = x[u];
  }
}

// Chunked reshard permutation between [P][Kc][Nc] row blocks and [Kc][P*Nc]:
//   pack   (UNPACK=false): out[(p*Kc + k)*Nc + n] = in[k*(P*Nc) + p*Nc + n]
//   unpack (UNPACK=true):  out[k*(P*Nc) + p*Nc + n] = in[(p*Kc + k)*Nc + n]
// One row = `vecs` 16-byte vectors.  Up to two tensors per launch.
template <bool UNPACK>
__global__ void __launch_bounds__(256) reshard_perm_kernel(const uint4* __restrict__ in0, uint4* __restrict__ out0,
                                                           const uint4* __restrict__ in1, uint4* __restrict__ out1,
                                                           int P, long long Kc, long long Nc, int vecs) {
  const long long total = (long long)P * Kc * Nc * vecs;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / vecs;
    const int v = (int)(i - row * vecs);
    long long p, k, n;
    if (UNPACK) {  // i walks the input [P][Kc][Nc]
      n = row % Nc;
      k = (row / Nc) % Kc;
      p = row / (Nc * Kc);
    } else {  // i walks the input [Kc][P][Nc]
      n = row % Nc;
      p = (row / Nc) % P;
      k = row / (Nc * P);
    }
    const long long blk = ((p * Kc + k) * Nc + n) * vecs + v;     // [P][Kc][Nc]
    const long long flat = ((k * P + p) * Nc + n) * vecs + v;     // [Kc][P*Nc]
    const long long dst = UNPACK ? flat : blk;  // the source index is i itself
    const uint4 x0 = in0[i];
    uint4 x1;
    if (in1) x1 = in1[i];
    out0[dst] = x0;
    if (in1) out1[dst] = x1;
  }
}

}  // namespace tsf
