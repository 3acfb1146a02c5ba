// Shared definitions of the two attention kernels (packed short-sequence and
// flash long-sequence): "temporal attention at each spatial
// location ... followed by spatial attention at each time frame".
//
// A "view" presents a [K, N, H, d] tensor (d fastest) as groups of sequences:
// element (l, a, b, e) lives at l*sL + a*sA + b*sB + e, where l is the
// attention axis (frames for temporal, tokens for spatial) and (a, b) name the
// group.  Temporal view: L = K, (a, b) = (h, n).  Spatial view: L = N,
// (a, b) = (h, t).  The TMA tensor maps use the dims (d, L, A, B) in that
// order, so a box (d, L, Ab, Bb) lands in shared memory group-major: row
// r = l + L * (ai + Ab * bi).
//
// Operand precision (reading G8): the standalone calls run on bf16
// operands with bf16 P.  Both stages of the block run on fp16 operands with
// fp16 P (11-bit mantissa, 8x bf16's): the temporal stage converts its bf16 x
// tiles to fp16 in shared memory (exact for 2^-14 <= |x| <= 65504), and X_t =
// x + T(x) is stored in fp16 for the spatial stage.  bf16 P in the block's
// temporal stage perturbs X_t enough to move near-tied spatial logits (~35 at
// C2) by 2e-2 in y; fp16 P keeps y within 1e-2 (tools/sim notes in DESIGN.md).
// The softmax denominator l is always the sum of the ROUNDED P that the PV
// MMA consumes, so the weights applied to V sum to one exactly.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace tsf {

enum EpiMode : int {
  EPI_OUT16 = 0,    // o = bf16(O / l)                (tsf_*_attn), bf16 operands, bf16 P
  EPI_BLOCK_T = 1,  // X_t = x + O/l -> fp16 X_t       (block, temporal stage): x arrives bf16 and
                    //   is converted to fp16 in shared memory; fp16 operands, fp16 P
  EPI_BLOCK_S = 2,  // y = X_t + O/l -> fp32 y         (block, spatial stage), fp16 operands, fp16 P
  EPI_STORM_X = 3,  // y = u + g O/l -> fp32 y         (STORM cross-attention, q = u, k = v = ctx), bf16
  EPI_STORM_S = 4,  // y += (1 - g) O/l (fp32 y)       (STORM self-attention, q = k = v = u), bf16
};
template <int EPI> struct EpiTraits {
  static constexpr bool F16 = (EPI == EPI_BLOCK_T || EPI == EPI_BLOCK_S);  // MMA operand / P type fp16 (else bf16)
  static constexpr bool CONVERT = (EPI == EPI_BLOCK_T);  // tiles land as bf16, converted in smem
  static constexpr bool SHARED = (EPI == EPI_BLOCK_T || EPI == EPI_BLOCK_S || EPI == EPI_STORM_S);  // q = k = v
};

// In-place bf16 -> fp16 conversion of one 16-byte unit (8 elements).  Exact
// for 2^-14 <= |v| <= 65504; smaller magnitudes become fp16 subnormals
// (absolute error < 2^-25).
__device__ __forceinline__ void cvt_unit_bf16_to_f16(uint8_t* p) {
  uint4 w = *reinterpret_cast<uint4*>(p);
  uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float lo = __uint_as_float(u[i] << 16), hi = __uint_as_float(u[i] & 0xFFFF0000u);
    __half2 h = __floats2half2_rn(lo, hi);
    u[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  *reinterpret_cast<uint4*>(p) = w;
}

struct AttnParams {
  int L, A, B;               // sequence length, group dims
  long long sL, sA, sB;      // element strides of the input view (TMA maps)
  long long osL, osA, osB;   // element strides of the output (per-thread stores)
  float scale_log2;          // log2(e) / sqrt(d)
  void* o;                   // EPI_OUT16: bf16 output; EPI_BLOCK_T: fp16 X_t
  float* y;                  // EPI_BLOCK_S: fp32 output
  // packed kernel: G = Ab * Bb groups per 128-row tile, rows used L * G
  int Ab, Bb, tiles_a, num_tiles;
  // flash kernel: pairs of 128-row query tiles per group, 128-row KV tiles
  int n_qpairs, nkv;
  // diagnostics (builds with -DTSF_TRACE only): clock64 stamps of CTA 0
  unsigned long long* trace;
  // distributed block, temporal stage (P > 1): X_t rows of frame l go straight
  // to rank l / Kc's frame-shard buffer (NVLink, CUDA IPC mapping):
  // peer_out[r] + (l % Kc) * osL + a * osA + (b + b_off) * osB
  int P, Kc, b_off;
  void* peer_out[8];
  // flash kernel: the block residual is read from global memory (the input
  // tensor, input-view strides): x (bf16) for EPI_BLOCK_T, X_t (fp16) for EPI_BLOCK_S
  const void* res;
  int num_items;  // flash kernel work items (pairs of query tiles x groups), persistent CTAs
  // flash kernel schedule: FLASH_PINGPONG (the two softmax warpgroups take
  // turns for the exponential phase)
  int flags;
  // block temporal stage: set to 1 (plain store, host-mapped memory) when a
  // stored fp16 X_t element is +-inf or NaN (|x + T(x)| beyond the fp16 range,
  // or a non-finite input); reported as TSF_ERR_NUMERIC by tsf_sync
  unsigned int* nonfinite;
  // joint attention over all K*N tokens (tsf_joint_attn, flash kernel MASK = 1):
  // mask_mode 1 = temporal block mask [n' = n], 2 = spatial block mask
  // [t' = t], 3 = causal frames [t' <= t]; mask_n = N tokens per frame
  int mask_mode, mask_n;
  // key/value sequence length (= L except for cross-attention, EPI_STORM_X)
  int Lk;
  // STORM epilogue weight: g for EPI_STORM_X, 1 - g for EPI_STORM_S
  float gate;
  // backward recompute (EPI_OUT16 flash path only, when lse != null): per query
  // row, lse2 = log2 sum_j 2^(s_j log2e / sqrt d) (log2 units) and, when dO is
  // given, D = sum_e O_e dO_e; stored group-major at (gb * A + ga) * lse_pitch + l
  float* lse;
  float* drow;
  const void* dO;
  int lse_pitch;
};
constexpr int FLASH_PINGPONG = 2;     // (builds with -DTSF_FLASH_PINGPONG_AB only)
constexpr int FLASH_RES_GLOBAL = 4;  // flash kernel: block residual from global memory, not the Q tile (diagnostics)
constexpr int FLASH_INPLACE_EXP = 8; // flash kernel (SEP), builds with -DTSF_FLASH_INPLACE_AB only: the exponential phase as one in-place pass over the row

constexpr int MAX_PEERS = 8;
// per-destination output tensor maps (packed kernel, distributed temporal stage)
struct PeerMaps {
  CUtensorMap m[MAX_PEERS];
};

#ifdef TSF_TRACE
constexpr int TRACE_PER_WARP = 1024;
#define TSF_STAMP(p, w, k)                                                        \
  do {                                                                           \
    if ((p).trace && blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (k) < TRACE_PER_WARP) \
      (p).trace[(w) * TRACE_PER_WARP + (k)] = clock64();                         \
  } while (0)
#else
#define TSF_STAMP(p, w, k) \
  do {                     \
  } while (0)
#endif

// ---- 16-bit pairs ----
template <bool F16>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  if constexpr (F16) {
    __half2 v = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
  } else {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);  // .x (low half) = lo
    return *reinterpret_cast<uint32_t*>(&v);
  }
}
template <bool F16>
__device__ __forceinline__ float2 unpack2(uint32_t w) {
  if constexpr (F16) {
    return __half22float2(*reinterpret_cast<__half2*>(&w));
  } else {
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
  }
}

// Non-finite detector for a pair of fp16 values: an fp16 is +-inf or NaN iff
// its exponent field is all ones (0x7C00); adding 0x0400 to the masked
// exponent then carries into bit 15 of that half (and only then; no carry
// crosses into the upper half).  OR-accumulate and test once per row.
__device__ __forceinline__ uint32_t f16x2_nonfinite_bits(uint32_t w) {
  return ((w & 0x7C007C00u) + 0x04000400u) & 0x80008000u;
}
__device__ __forceinline__ uint32_t u4_nonfinite_bits(const uint4& w) {
  return f16x2_nonfinite_bits(w.x) | f16x2_nonfinite_bits(w.y) | f16x2_nonfinite_bits(w.z) |
         f16x2_nonfinite_bits(w.w);
}
// Report a row's accumulated non-finite bits (rare path: one plain store).
__device__ __forceinline__ void report_nonfinite(const AttnParams& p, uint32_t nf) {
  if (__builtin_expect(nf != 0u, 0) && p.nonfinite) *reinterpret_cast<volatile unsigned int*>(p.nonfinite) = 1u;
}

// Byte offset of 16-byte unit u of row r in a TMA/UMMA swizzled tile whose
// rows are SWB bytes (128 -> SWIZZLE_128B, 64 -> SWIZZLE_64B).
template <int SWB>
__device__ __forceinline__ uint32_t swz_off(uint32_t r, uint32_t u) {
  if constexpr (SWB == 128) return r * 128u + ((u ^ (r & 7u)) << 4);
  else return r * 64u + ((u ^ ((r >> 1) & 3u)) << 4);
}

// 16-byte unit u (elements [8u, 8u+8)) of row r of a d-wide 16-bit tile
// stored as NCH column chunks of ROWS x SWB bytes.
template <int D, int ROWS>
__device__ __forceinline__ uint4 tile_row_u4(const uint8_t* tile, uint32_t r, uint32_t u) {
  constexpr int SWB = (2 * D < 128) ? 2 * D : 128;
  constexpr int UPC = SWB / 16;  // 16-byte units per chunk row
  const uint32_t c = u / UPC, uu = u % UPC;
  return *reinterpret_cast<const uint4*>(tile + c * (ROWS * SWB) + swz_off<SWB>(r, uu));
}

// Epilogue for one row: o_acc[0..D) = unnormalised O row, inv_l = 1/l.
// res_tile: the row's 16-bit input (x for BLOCK_T, X_t for BLOCK_S) in shared
// memory (the swizzled Q tile).
// NU 16-byte units starting at unit u0 (o_acc holds those 8 * NU values).
template <int D, int ROWS, int EPI, int NU = D / 8>
__device__ __forceinline__ uint32_t epilogue_row(const AttnParams& p, const float* o_acc, float inv_l,
                                             long long off, const uint8_t* res_tile, uint32_t r, int u0 = 0) {
  constexpr bool F16 = EpiTraits<EPI>::F16;
  uint32_t nf = 0;
  off += 8 * u0;
  // residual units loaded before any store (generic pointers: see epilogue_row_stage)
  uint4 res[NU];
  if constexpr (EPI != EPI_OUT16 && EPI != EPI_STORM_S) {
#pragma unroll
    for (int u = 0; u < NU; ++u) res[u] = tile_row_u4<D, ROWS>(res_tile, r, u0 + u);
  }
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = o_acc[8 * u + i] * inv_l;
    if constexpr (EPI == EPI_OUT16) {
      uint4 w;
      w.x = pack2<false>(v[0], v[1]);
      w.y = pack2<false>(v[2], v[3]);
      w.z = pack2<false>(v[4], v[5]);
      w.w = pack2<false>(v[6], v[7]);
      *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.o) + off + 8 * u) = w;
    } else if constexpr (EPI == EPI_STORM_S) {  // y += (1 - g) O/l
      float4* yp = reinterpret_cast<float4*>(p.y + off + 8 * u);
      float4 y0 = yp[0], y1 = yp[1];
      const float w = p.gate;
      y0.x = fmaf(w, v[0], y0.x); y0.y = fmaf(w, v[1], y0.y); y0.z = fmaf(w, v[2], y0.z); y0.w = fmaf(w, v[3], y0.w);
      y1.x = fmaf(w, v[4], y1.x); y1.y = fmaf(w, v[5], y1.y); y1.z = fmaf(w, v[6], y1.z); y1.w = fmaf(w, v[7], y1.w);
      yp[0] = y0;
      yp[1] = y1;
    } else {
      const uint4 rr = res[u];
      const float2 x0 = unpack2<F16>(rr.x), x1 = unpack2<F16>(rr.y), x2 = unpack2<F16>(rr.z),
                   x3 = unpack2<F16>(rr.w);
      if constexpr (EPI == EPI_STORM_X) {  // y = u + g O/l
        const float w = p.gate;
        float4 y0, y1;
        y0.x = fmaf(w, v[0], x0.x); y0.y = fmaf(w, v[1], x0.y); y0.z = fmaf(w, v[2], x1.x); y0.w = fmaf(w, v[3], x1.y);
        y1.x = fmaf(w, v[4], x2.x); y1.y = fmaf(w, v[5], x2.y); y1.z = fmaf(w, v[6], x3.x); y1.w = fmaf(w, v[7], x3.y);
        *reinterpret_cast<float4*>(p.y + off + 8 * u) = y0;
        *reinterpret_cast<float4*>(p.y + off + 8 * u + 4) = y1;
      } else if constexpr (EPI == EPI_BLOCK_S) {
        float4 y0, y1;
        y0.x = x0.x + v[0]; y0.y = x0.y + v[1]; y0.z = x1.x + v[2]; y0.w = x1.y + v[3];
        y1.x = x2.x + v[4]; y1.y = x2.y + v[5]; y1.z = x3.x + v[6]; y1.w = x3.y + v[7];
        *reinterpret_cast<float4*>(p.y + off + 8 * u) = y0;
        *reinterpret_cast<float4*>(p.y + off + 8 * u + 4) = y1;
      } else {  // EPI_BLOCK_T: X_t = x + O/l, stored fp16
        uint4 w;
        w.x = pack2<true>(x0.x + v[0], x0.y + v[1]);
        w.y = pack2<true>(x1.x + v[2], x1.y + v[3]);
        w.z = pack2<true>(x2.x + v[4], x2.y + v[5]);
        w.w = pack2<true>(x3.x + v[6], x3.y + v[7]);
        nf |= u4_nonfinite_bits(w);
        *reinterpret_cast<uint4*>(reinterpret_cast<__half*>(p.o) + off + 8 * u) = w;
      }
    }
  }
  return nf;
}

// Flash-kernel epilogue for NU units starting at unit u0 of one row, residual
// read from global memory at element offset in_off (EPI_BLOCK_T: bf16 x,
// EPI_BLOCK_S: fp16 X_t); output at element offset off of p.o / p.y.
template <int D, int EPI, int NU>
__device__ __forceinline__ uint32_t epilogue_row_g(const AttnParams& p, const float* o_acc, float inv_l, long long off,
                                               long long in_off, int u0) {
  uint32_t nf = 0;
  off += 8 * u0;
  in_off += 8 * u0;
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = o_acc[8 * u + i] * inv_l;
    if constexpr (EPI == EPI_OUT16) {
      uint4 w;
      w.x = pack2<false>(v[0], v[1]);
      w.y = pack2<false>(v[2], v[3]);
      w.z = pack2<false>(v[4], v[5]);
      w.w = pack2<false>(v[6], v[7]);
      *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.o) + off + 8 * u) = w;
    } else if constexpr (EPI == EPI_STORM_S) {  // y += (1 - g) O/l
      float4* yp = reinterpret_cast<float4*>(p.y + off + 8 * u);
      float4 y0 = yp[0], y1 = yp[1];
      const float w = p.gate;
      y0.x = fmaf(w, v[0], y0.x); y0.y = fmaf(w, v[1], y0.y); y0.z = fmaf(w, v[2], y0.z); y0.w = fmaf(w, v[3], y0.w);
      y1.x = fmaf(w, v[4], y1.x); y1.y = fmaf(w, v[5], y1.y); y1.z = fmaf(w, v[6], y1.z); y1.w = fmaf(w, v[7], y1.w);
      yp[0] = y0;
      yp[1] = y1;
    } else {
      constexpr bool RES_F16 = (EPI == EPI_BLOCK_S);
      const uint4 rr = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(p.res) + in_off + 8 * u);
      const float2 x0 = unpack2<RES_F16>(rr.x), x1 = unpack2<RES_F16>(rr.y), x2 = unpack2<RES_F16>(rr.z),
                   x3 = unpack2<RES_F16>(rr.w);
      if constexpr (EPI == EPI_STORM_X) {  // y = u + g O/l
        const float w = p.gate;
        float4 y0, y1;
        y0.x = fmaf(w, v[0], x0.x); y0.y = fmaf(w, v[1], x0.y); y0.z = fmaf(w, v[2], x1.x); y0.w = fmaf(w, v[3], x1.y);
        y1.x = fmaf(w, v[4], x2.x); y1.y = fmaf(w, v[5], x2.y); y1.z = fmaf(w, v[6], x3.x); y1.w = fmaf(w, v[7], x3.y);
        *reinterpret_cast<float4*>(p.y + off + 8 * u) = y0;
        *reinterpret_cast<float4*>(p.y + off + 8 * u + 4) = y1;
      } else if constexpr (EPI == EPI_BLOCK_S) {
        float4 y0, y1;
        y0.x = x0.x + v[0]; y0.y = x0.y + v[1]; y0.z = x1.x + v[2]; y0.w = x1.y + v[3];
        y1.x = x2.x + v[4]; y1.y = x2.y + v[5]; y1.z = x3.x + v[6]; y1.w = x3.y + v[7];
        *reinterpret_cast<float4*>(p.y + off + 8 * u) = y0;
        *reinterpret_cast<float4*>(p.y + off + 8 * u + 4) = y1;
      } else {  // EPI_BLOCK_T: X_t = x + O/l, stored fp16
        uint4 w;
        w.x = pack2<true>(x0.x + v[0], x0.y + v[1]);
        w.y = pack2<true>(x1.x + v[2], x1.y + v[3]);
        w.z = pack2<true>(x2.x + v[4], x2.y + v[5]);
        w.w = pack2<true>(x3.x + v[6], x3.y + v[7]);
        nf |= u4_nonfinite_bits(w);
        *reinterpret_cast<uint4*>(reinterpret_cast<__half*>(p.o) + off + 8 * u) = w;
      }
    }
  }
  return nf;
}

// Epilogue for one row written back IN PLACE into its swizzled shared-memory
// row (the tile the row's input came from), for a TMA store of the whole tile.
// EPI_OUT16: bf16(O/l); EPI_BLOCK_T: fp16(x + O/l) with x read from the same row.
template <int D, int ROWS, int EPI>
__device__ __forceinline__ uint32_t epilogue_row_smem(const float* o_acc, float inv_l, uint8_t* tile, uint32_t r) {
  constexpr int SWB = (2 * D < 128) ? 2 * D : 128;
  constexpr int UPC = SWB / 16;
  uint32_t nf = 0;
#pragma unroll
  for (int u = 0; u < D / 8; ++u) {
    uint4* ptr = reinterpret_cast<uint4*>(tile + (u / UPC) * (ROWS * SWB) + swz_off<SWB>(r, u % UPC));
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = o_acc[8 * u + i] * inv_l;
    uint4 w;
    if constexpr (EPI == EPI_OUT16) {
      w.x = pack2<false>(v[0], v[1]);
      w.y = pack2<false>(v[2], v[3]);
      w.z = pack2<false>(v[4], v[5]);
      w.w = pack2<false>(v[6], v[7]);
    } else {
      const uint4 rr = *ptr;
      const float2 x0 = unpack2<true>(rr.x), x1 = unpack2<true>(rr.y), x2 = unpack2<true>(rr.z),
                   x3 = unpack2<true>(rr.w);
      w.x = pack2<true>(x0.x + v[0], x0.y + v[1]);
      w.y = pack2<true>(x1.x + v[2], x1.y + v[3]);
      w.z = pack2<true>(x2.x + v[4], x2.y + v[5]);
      w.w = pack2<true>(x3.x + v[6], x3.y + v[7]);
      nf |= u4_nonfinite_bits(w);
    }
    *ptr = w;
  }
  return nf;
}

// EPI_BLOCK_T epilogue into a separate staging tile: x from res_tile row r,
// X_t = fp16(x + O/l) written to row orow of out_tile (same swizzled layout).
template <int D, int ROWS_IN, int ROWS_OUT>
__device__ __forceinline__ uint32_t epilogue_row_stage(const float* o_acc, float inv_l, const uint8_t* res_tile,
                                                   uint32_t r, uint8_t* out_tile, uint32_t orow) {
  constexpr int SWB = (2 * D < 128) ? 2 * D : 128;
  constexpr int UPC = SWB / 16;
  uint32_t nf = 0;
  // residual units are loaded four at a time before their stores: the tiles are
  // reached through generic pointers, so a load after a store could not be
  // hoisted by the compiler (four keeps the register footprint small)
  constexpr int GU = (D / 8 < 4) ? D / 8 : 4;
  uint4 res[GU];
#pragma unroll
  for (int u = 0; u < D / 8; ++u) {
    if (u % GU == 0) {
#pragma unroll
      for (int e = 0; e < GU; ++e) res[e] = tile_row_u4<D, ROWS_IN>(res_tile, r, u + e);
    }
    const uint4 rr = res[u % GU];
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = o_acc[8 * u + i] * inv_l;
    const float2 x0 = unpack2<true>(rr.x), x1 = unpack2<true>(rr.y), x2 = unpack2<true>(rr.z),
                 x3 = unpack2<true>(rr.w);
    uint4 w;
    w.x = pack2<true>(x0.x + v[0], x0.y + v[1]);
    w.y = pack2<true>(x1.x + v[2], x1.y + v[3]);
    w.z = pack2<true>(x2.x + v[4], x2.y + v[5]);
    w.w = pack2<true>(x3.x + v[6], x3.y + v[7]);
    nf |= u4_nonfinite_bits(w);
    *reinterpret_cast<uint4*>(out_tile + (u / UPC) * (ROWS_OUT * SWB) + swz_off<SWB>(orow, u % UPC)) = w;
  }
  return nf;
}

}  // namespace tsf
