// Shared definitions of the two attention kernels (packed short-sequence and
// flash long-sequence): "temporal attention at each spatial
// location ... followed by spatial attention at each time frame".
//
// A "view" presents a [K, N, H, d] bf16 tensor (d fastest) as groups of
// sequences: element (l, a, b, e) lives at l*sL + a*sA + b*sB + e, where l is
// the attention axis (frames for temporal, tokens for spatial) and (a, b) name
// the group.  Temporal view: L = K, (a, b) = (h, n).  Spatial view: L = N,
// (a, b) = (h, t).  The TMA tensor maps use the dims (d, L, A, B) in that
// order, so a box (d, L, Ab, Bb) lands in shared memory group-major: row
// r = l + L * (ai + Ab * bi).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

namespace tsf {

enum EpiMode : int {
  EPI_BF16 = 0,     // o = bf16(O / l)                          (tsf_*_attn)
  EPI_BLOCK_T = 1,  // X_t = x + O/l -> hi = bf16(X_t), lo = bf16(X_t - hi)
  EPI_BLOCK_S = 2,  // y = (hi + lo) + O/l, fp32                 (tsf_spacetime_block)
};

struct AttnParams {
  int L, A, B;               // sequence length, group dims
  long long sL, sA, sB;      // element strides of the view
  float scale_log2;          // log2(e) / sqrt(d)
  __nv_bfloat16* o;          // EPI_BF16: output; EPI_BLOCK_T: hi
  __nv_bfloat16* o2;         // EPI_BLOCK_T: lo
  const __nv_bfloat16* res_lo;  // EPI_BLOCK_S: lo part of the residual
  float* y;                  // EPI_BLOCK_S: fp32 output
  // packed kernel: G = Ab * Bb groups per 128-row tile, rows used L * G
  int Ab, Bb, tiles_a, num_tiles;
  // flash kernel: pairs of 128-row query tiles per group, 128-row KV tiles
  int n_qpairs, nkv;
};

// Byte offset of 16-byte unit u of row r in a TMA/UMMA swizzled tile whose
// rows are SWB bytes (128 -> SWIZZLE_128B, 64 -> SWIZZLE_64B).
template <int SWB>
__device__ __forceinline__ uint32_t swz_off(uint32_t r, uint32_t u) {
  if constexpr (SWB == 128) return r * 128u + ((u ^ (r & 7u)) << 4);
  else return r * 64u + ((u ^ ((r >> 1) & 3u)) << 4);
}

// Read element chunk [8u, 8u+8) of row r of a d-wide bf16 tile stored as
// NCH column chunks of ROWS x SWB bytes.
template <int D, int ROWS>
__device__ __forceinline__ uint4 tile_row_u4(const uint8_t* tile, uint32_t r, uint32_t u) {
  constexpr int SWB = (2 * D < 128) ? 2 * D : 128;
  constexpr int UPC = SWB / 16;  // 16-byte units per chunk row
  const uint32_t c = u / UPC, uu = u % UPC;
  return *reinterpret_cast<const uint4*>(tile + c * (ROWS * SWB) + swz_off<SWB>(r, uu));
}

__device__ __forceinline__ float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

// Epilogue for one row: o_acc[0..D) = unnormalised O row, inv_l = 1/l.
// res_tile: the row's bf16 input (x or hi) in shared memory (swizzled tile).
template <int D, int ROWS, int EPI>
__device__ __forceinline__ void epilogue_row(const AttnParams& p, const float* o_acc, float inv_l,
                                             long long off, const uint8_t* res_tile, uint32_t r) {
#pragma unroll
  for (int u = 0; u < D / 8; ++u) {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = o_acc[8 * u + i] * inv_l;
    if constexpr (EPI == EPI_BF16) {
      uint4 w;
      w.x = pack_bf16x2(v[0], v[1]);
      w.y = pack_bf16x2(v[2], v[3]);
      w.z = pack_bf16x2(v[4], v[5]);
      w.w = pack_bf16x2(v[6], v[7]);
      *reinterpret_cast<uint4*>(p.o + off + 8 * u) = w;
    } else {
      const uint4 rr = tile_row_u4<D, ROWS>(res_tile, r, u);
      float x[8] = {bf16lo(rr.x), bf16hi(rr.x), bf16lo(rr.y), bf16hi(rr.y),
                    bf16lo(rr.z), bf16hi(rr.z), bf16lo(rr.w), bf16hi(rr.w)};
      if constexpr (EPI == EPI_BLOCK_S) {
        const uint4 lo = *reinterpret_cast<const uint4*>(p.res_lo + off + 8 * u);
        const float l8[8] = {bf16lo(lo.x), bf16hi(lo.x), bf16lo(lo.y), bf16hi(lo.y),
                             bf16lo(lo.z), bf16hi(lo.z), bf16lo(lo.w), bf16hi(lo.w)};
        float4 y0, y1;
        y0.x = (x[0] + l8[0]) + v[0]; y0.y = (x[1] + l8[1]) + v[1];
        y0.z = (x[2] + l8[2]) + v[2]; y0.w = (x[3] + l8[3]) + v[3];
        y1.x = (x[4] + l8[4]) + v[4]; y1.y = (x[5] + l8[5]) + v[5];
        y1.z = (x[6] + l8[6]) + v[6]; y1.w = (x[7] + l8[7]) + v[7];
        *reinterpret_cast<float4*>(p.y + off + 8 * u) = y0;
        *reinterpret_cast<float4*>(p.y + off + 8 * u + 4) = y1;
      } else {  // EPI_BLOCK_T
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float a = x[2 * i] + v[2 * i], b = x[2 * i + 1] + v[2 * i + 1];
          hw[i] = pack_bf16x2(a, b);
          lw[i] = pack_bf16x2(a - bf16lo(hw[i]), b - bf16hi(hw[i]));
        }
        *reinterpret_cast<uint4*>(p.o + off + 8 * u) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(p.o2 + off + 8 * u) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      }
    }
  }
}

}  // namespace tsf
