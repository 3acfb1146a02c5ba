// tcgen05 GEMM with fused epilogues for the full TimeSformer divided block
// (per-stage Q/K/V/O projections and the MLP around the
// factorized attention of PAPER.md P:64).
//
//   C[M, N] = A[M, K] . W[N, K]^T  (+ bias[N])  (+ GELU | + residual R[M, N])
//
// A (activations) and W (nn.Linear layout [out, in]) are bf16, K-major, loaded
// by TMA in 128-byte-swizzled 64-column k-blocks; the accumulator lives in
// TMEM (fp32), double-buffered across tiles so the epilogue of tile i
// overlaps the MMAs of tile i+1.  Persistent CTAs, one per SM; tiles are
// walked M-fastest inside an N band so a band's weight tile stays in L2.
//
// Warp roles (192 threads): warps 0-3 epilogue (thread = TMEM lane = tile
// row), warp 4 TMA producer, warp 5 MMA issuer (+ TMEM allocation).
#pragma once
#include "sm100.cuh"
#include <cuda_bf16.h>

namespace tsf {

enum GemmEpi : int {
  GEPI_BIAS_BF16 = 0,   // C bf16 = acc + bias
  GEPI_GELU_BF16 = 1,   // C bf16 = gelu(acc + bias), exact erf form
  GEPI_RES_F32 = 2,     // C fp32 = acc + bias + R (R fp32)
  GEPI_RESB_F32 = 3,    // C fp32 = acc + bias + R (R bf16)
};

struct GemmParams {
  int M, N, K;
  const float* bias;    // [N]
  const void* res;      // [M, N] residual (GEPI_RES*), row stride ldc
  void* c;              // [M, N] output, row stride ldc (elements)
  long long ldc;
  int tiles_m, tiles_n;
};

template <int BN>
struct GemmCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;             // 16 KB
  static constexpr int B_BYTES = BN * BK * 2;             // 16 / 32 KB
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int NST = (BN == 256) ? 4 : 6;
  static constexpr int SMEM = NST * STAGE + 256 + 1024;
  static constexpr int TCOLS = 2 * BN;                    // double-buffered accumulator
};

__device__ __forceinline__ float gelu_erf(float x) { return 0.5f * x * (1.f + erff(x * 0.70710678118654752f)); }

template <int BN, int EPI>
__global__ void __launch_bounds__(192, 1)
gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tw, const GemmParams p) {
  using C = GemmCfg<BN>;
  constexpr int NST = C::NST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * C::STAGE);
  uint64_t* full = bars;                  // [NST]
  uint64_t* empty = bars + NST;           // [NST]
  uint64_t* acc_full = bars + 2 * NST;    // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2] (4 epilogue warps)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int ntiles = p.tiles_m * p.tiles_n;
  const int nk = p.K / C::BK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<C::TCOLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 4) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      tma_prefetch_desc(&ta);
      tma_prefetch_desc(&tw);
      int g = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int tm = tile % p.tiles_m, tn = tile / p.tiles_m;
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % NST;
          if (g >= NST) mbar_wait_sleep(&empty[s], ((g / NST) - 1) & 1);
          uint8_t* st = smem + s * C::STAGE;
          mbar_arrive_expect_tx(&full[s], C::STAGE);
          tma_load_2d(st, &ta, &full[s], kb * C::BK, tm * C::BM);
          tma_load_2d(st + C::A_BYTES, &tw, &full[s], kb * C::BK, tn * BN);
        }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ===================== MMA issuer =====================
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc(128, BN, 0, 0, false);
      int g = 0, it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int b = it & 1;
        if (it >= 2) mbar_wait_sleep(&acc_empty[b], ((it >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t dacc = tmem + b * BN;
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % NST;
          mbar_wait_sleep(&full[s], (g / NST) & 1);
          tc_fence_after();
          const uint32_t aa = smem_u32(smem + s * C::STAGE), ba = aa + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k)
            mma_ss(dacc, make_sdesc(aa + 32 * k, 16, 1024, SWZ_128B), make_sdesc(ba + 32 * k, 16, 1024, SWZ_128B),
                   idesc, (kb > 0 || k > 0) ? 1u : 0u);
          mma_commit(&empty[s]);  // the stage is free once these MMAs retire
        }
        mma_commit(&acc_full[b]);
      }
    }
    __syncwarp();
  } else {
    // ===================== epilogue (warps 0-3) =====================
    const uint32_t r = warp * 32 + lane;
    const uint32_t lane_base = (warp * 32) << 16;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int b = it & 1;
      const int tm = tile % p.tiles_m, tn = tile / p.tiles_m;
      mbar_wait(&acc_full[b], (it >> 1) & 1);
      tc_fence_after();
      const int row = tm * C::BM + (int)r;
      const bool ok = row < p.M;
      const int col0 = tn * BN;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld_x32(tmem + lane_base + b * BN + c0, v);
        tmem_wait_ld();
        if (ok) {
          float f[32];
          const float4* b4 = reinterpret_cast<const float4*>(p.bias + col0 + c0);
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 bb = __ldg(b4 + j / 4);
            f[j] = __uint_as_float(v[j]) + bb.x;
            f[j + 1] = __uint_as_float(v[j + 1]) + bb.y;
            f[j + 2] = __uint_as_float(v[j + 2]) + bb.z;
            f[j + 3] = __uint_as_float(v[j + 3]) + bb.w;
          }
          const long long off = (long long)row * p.ldc + col0 + c0;
          if constexpr (EPI == GEPI_BIAS_BF16 || EPI == GEPI_GELU_BF16) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              float g8[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) g8[e] = (EPI == GEPI_GELU_BF16) ? gelu_erf(f[j + e]) : f[j + e];
              uint4 w;
              __nv_bfloat162 h0 = __floats2bfloat162_rn(g8[0], g8[1]), h1 = __floats2bfloat162_rn(g8[2], g8[3]),
                             h2 = __floats2bfloat162_rn(g8[4], g8[5]), h3 = __floats2bfloat162_rn(g8[6], g8[7]);
              w.x = *reinterpret_cast<uint32_t*>(&h0);
              w.y = *reinterpret_cast<uint32_t*>(&h1);
              w.z = *reinterpret_cast<uint32_t*>(&h2);
              w.w = *reinterpret_cast<uint32_t*>(&h3);
              *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.c) + off + j) = w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              float4 rr;
              if constexpr (EPI == GEPI_RES_F32) {
                rr = *reinterpret_cast<const float4*>(static_cast<const float*>(p.res) + off + j);
              } else {
                const uint2 rb = *reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(p.res) + off + j);
                rr.x = __uint_as_float(rb.x << 16); rr.y = __uint_as_float(rb.x & 0xFFFF0000u);
                rr.z = __uint_as_float(rb.y << 16); rr.w = __uint_as_float(rb.y & 0xFFFF0000u);
              }
              float4 o4 = make_float4(f[j] + rr.x, f[j + 1] + rr.y, f[j + 2] + rr.z, f[j + 3] + rr.w);
              *reinterpret_cast<float4*>(static_cast<float*>(p.c) + off + j) = o4;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<C::TCOLS>(tmem);
  }
}

// LayerNorm over the last dimension (the pre-LN of TimeSformer's block, cited
// at PAPER.md P:64; reading G21): one warp per row, fp32 statistics (two-pass:
// mean, then centred variance), eps = 1e-5, bf16 output.  IN = float or
// __nv_bfloat16; D % 8 == 0 and D <= 8192 (lane l owns the 8-element chunks
// l, l + 32, ...: 16- / 32-byte vector loads, 16-byte stores); MAXC >= D / 256
// bounds the per-lane chunks so they stay in registers.
template <typename IN, int MAXC>
__global__ void __launch_bounds__(256) layernorm_kernel(const IN* __restrict__ x, const float* __restrict__ gamma,
                                                        const float* __restrict__ beta, __nv_bfloat16* __restrict__ y,
                                                        long long rows, int D) {
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int nq = D / 8;                                     // chunks of 8; at most MAXC per lane
  float v[MAXC][8];
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    if (c * 32 + lane < nq) {
      const long long col = (long long)(c * 32 + lane) * 8;
      if constexpr (sizeof(IN) == 4) {
        const float4 a = *reinterpret_cast<const float4*>(x + row * D + col);
        const float4 b = *reinterpret_cast<const float4*>(x + row * D + col + 4);
        v[c][0] = a.x; v[c][1] = a.y; v[c][2] = a.z; v[c][3] = a.w;
        v[c][4] = b.x; v[c][5] = b.y; v[c][6] = b.z; v[c][7] = b.w;
      } else {
        const uint4 w = *reinterpret_cast<const uint4*>(x + row * D + col);
        const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[c][2 * e] = __uint_as_float(u[e] << 16);
          v[c][2 * e + 1] = __uint_as_float(u[e] & 0xFFFF0000u);
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) s += v[c][e];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / D;
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < MAXC; ++c)
    if (c * 32 + lane < nq) {
#pragma unroll
      for (int e = 0; e < 8; ++e) { const float t = v[c][e] - mean; q += t * t; }
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rstd = rsqrtf(q / D + 1e-5f);
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    if (c * 32 + lane < nq) {
      const int col = (c * 32 + lane) * 8;
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float y0 = (v[c][2 * e] - mean) * rstd * gamma[col + 2 * e] + beta[col + 2 * e];
        const float y1 = (v[c][2 * e + 1] - mean) * rstd * gamma[col + 2 * e + 1] + beta[col + 2 * e + 1];
        __nv_bfloat162 h = __floats2bfloat162_rn(y0, y1);
        w[e] = *reinterpret_cast<uint32_t*>(&h);
      }
      *reinterpret_cast<uint4*>(y + row * D + col) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

}  // namespace tsf
