// Streaming temporal stage of the block (SURVEY 8(a) rows a1-a5 for K <= 128):
// X_t = x + T(x, x, x), "temporal attention at each spatial
// location", stored fp16 (G8), optionally scattered straight into
// the owning ranks' frame shards (row a5, fused exchange).
//
// The stage is HBM-bound (K/2 flop/B): every byte of x is read once and every
// byte of X_t written once, so the kernel is organised as a stream in which
// every role works on a different tile at the same time:
//
//   warp 16      TMA producer: x tiles into an NST-deep input ring
//   warps 12-15  converters: bf16 -> fp16 in place (the MMA operands and the
//                residual are fp16, reading G8); tile i by warp 12 + i % 4
//   warp 17      QK^T issuer: S[b] = X X^T of tile i into TMEM slot b = i % 2
//   warps 0-3    softmax: block-diagonal window softmax of S[b] -> P[b] (TMEM),
//                row sums l of the rounded P -> shared memory
//   warp 18      PV issuer: O[b] = P[b] X
//   warps 4-7,   epilogue warpgroup b (slot b's tiles): X_t = x + O[b] / l into
//   8-11         an fp16 staging tile (regrouped by destination rank when
//                distributed), one TMA store per tile (per destination),
//                input stage released
//
// Measured on B200 (tools/trace_stream.py): converting one 16 KB tile costs a
// warp ~2300 cycles and the epilogue of one tile ~1700, against a ~1400-cycle
// per-tile budget at the HBM roofline, hence four converters and two
// epilogue warpgroups.
//
// A 128-row tile holds G = Ab * Bb whole groups of L = K rows (group-major,
// see attn_common.cuh); one 128x128 QK^T and one 128xD PV MMA cover all of
// them, the softmax restricts each row to its own diagonal block.
//
// TMEM: two slots of [S 128 | P 64 | O D] columns (512 at D = 64), so the
// softmax of tile i+1 and the epilogue of tile i run concurrently, and the
// QK^T of tile i+2 is issued as soon as the softmax of tile i is done.
// The older attn_packed kernel (one slot, softmax and epilogue in the same
// warps) serves the other modes and shapes.
#pragma once
#include "sm100.cuh"
#include "attn_common.cuh"

namespace tsf {

template <int D, int WIN, int NST, int NS = 2>
struct StreamCfg {
  static constexpr int SWB = (2 * D < 128) ? 2 * D : 128;
  static constexpr int CH = SWB / 2;
  static constexpr int NCH = D / CH;
  static constexpr int CHUNK_BYTES = 128 * SWB;
  static constexpr int TILE_BYTES = NCH * CHUNK_BYTES;        // 128 x D 16-bit
  // NS = 2: slot = [S 128 | P 64 | O 64];  NS = 4: slot = 128 columns, S
  // [0,128) -> P over [0,64) after the softmax read S -> O over [64,128)
  static constexpr int SLOT = 512 / NS;                       // TMEM columns per slot
  static constexpr int COL_S = 0, COL_P = (NS == 4) ? 0 : 128, COL_O = (NS == 4) ? 64 : 192;
  static_assert(NS == 2 || NS == 4, "TMEM slots");
  static_assert(COL_O + D <= SLOT, "TMEM slot layout needs D <= 64");
  static_assert(WIN == 32 || WIN == 64, "softmax window");
  static constexpr int LBUF_BYTES = NS * 128 * 4;             // l per row per slot
  static constexpr int BAR_BYTES = 512;
  static constexpr int SMEM = NST * TILE_BYTES + 2 * TILE_BYTES + LBUF_BYTES + BAR_BYTES + 1024;
  static constexpr int THREADS = 640;
  static constexpr int W_EPI = 4, W_CONV = 12, NCONV = 4, W_TMA = 16, W_QK = 17, W_PV = 18;
};

template <int D, int WIN, int NST, int LT, int NS>
__global__ void __launch_bounds__(640, 1)
attn_stream_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap to,
                   const __grid_constant__ PeerMaps pm, const AttnParams p) {
  using C = StreamCfg<D, WIN, NST, NS>;
  static_assert(LT == 0 || (WIN == 32 && 32 % LT == 0 && LT >= 2), "compact softmax: L divides 32");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sIn = smem;                                   // NST input tiles (x, bf16 -> fp16 in place)
  uint8_t* sOut = smem + NST * C::TILE_BYTES;            // fp16 X_t staging tile of each epilogue warpgroup
  float* lbuf = reinterpret_cast<float*>(sOut + 2 * C::TILE_BYTES);   // [NS][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOut + 2 * C::TILE_BYTES + C::LBUF_BYTES);
  uint64_t* in_full = bars;              // [NST] TMA
  uint64_t* in_conv = bars + NST;        // [NST] converter
  uint64_t* in_empty = bars + 2 * NST;   // [NST] epilogue read the residual (4 warps)
  uint64_t* s_full = bars + 3 * NST;     // [NS] QK^T committed
  uint64_t* p_full = s_full + NS;        // [NS] softmax stored P and l (4 warps)
  uint64_t* o_full = s_full + 2 * NS;    // [NS] PV committed
  uint64_t* o_empty = s_full + 3 * NS;   // [NS] epilogue read O and l (4 warps)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_full + 4 * NS);
  static_assert(sizeof(uint64_t) * (3 * NST + 4 * NS) + 4 <= C::BAR_BYTES, "barrier space");

  const uint32_t warp = warp_id(), lane = lane_id();
  const int L = p.L;
  const int G = p.Ab * p.Bb;
  const int rows_used = L * G;
  const int ntiles = p.num_tiles;
  const int my_tiles = (ntiles > (int)blockIdx.x) ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

  // rows >= rows_used of the input ring are never written by TMA: zero them
  // once (0 * NaN in PV must not happen)
  if (rows_used < 128) {
    for (uint32_t i = threadIdx.x; i < NST * C::TILE_BYTES / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&in_full[s], 1);
      mbar_init(&in_conv[s], 1);
      mbar_init(&in_empty[s], 4);
    }
    for (int b = 0; b < NS; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 4);
      mbar_init(&o_full[b], 1);
      mbar_init(&o_empty[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == C::W_QK) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == C::W_TMA) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      tma_prefetch_desc(&tx);
      const uint32_t bytes = (uint32_t)(C::CH * 2) * (uint32_t)rows_used * C::NCH;
      for (int i = 0; i < my_tiles; ++i) {
        const int tile = blockIdx.x + i * gridDim.x;
        const int s = i % NST;
        if (i >= NST) mbar_wait_sleep(&in_empty[s], ((i / NST) - 1) & 1);
        TSF_STAMP(p, 12 + (C::W_TMA), i);
        const int a0 = (tile % p.tiles_a) * p.Ab, b0 = (tile / p.tiles_a) * p.Bb;
        mbar_arrive_expect_tx(&in_full[s], bytes);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_4d(sIn + s * C::TILE_BYTES + c * C::CHUNK_BYTES, &tx, &in_full[s], c * C::CH, 0, a0, b0);
      }
    }
    __syncwarp();
  } else if (warp >= C::W_CONV && warp < C::W_CONV + C::NCONV) {
    // ===================== converters: bf16 -> fp16 in place =====================
    constexpr int UPR = D / 8;                 // 16-byte units per row
    constexpr int UPC = C::SWB / 16;           // units per chunk row
    const int units = rows_used * UPR;         // rows are whole units: the swizzle does not matter
    for (int i = (int)(warp - C::W_CONV); i < my_tiles; i += C::NCONV) {
      const int s = i % NST;
      mbar_wait(&in_full[s], (i / NST) & 1);
      TSF_STAMP(p, 12 + (warp), 2 * (i / C::NCONV));
      uint8_t* tile = sIn + s * C::TILE_BYTES;
      constexpr int BATCH = 8;
      for (int u0 = (int)lane; u0 < units; u0 += 32 * BATCH) {
        uint4 w[BATCH];
        uint8_t* ptr[BATCH];
#pragma unroll
        for (int k = 0; k < BATCH; ++k) {
          const int u = u0 + 32 * k;
          const int r = u / UPR, c = u % UPR;
          ptr[k] = tile + (c / UPC) * C::CHUNK_BYTES + r * C::SWB + (c % UPC) * 16;
          if (u < units) w[k] = *reinterpret_cast<const uint4*>(ptr[k]);
        }
#pragma unroll
        for (int k = 0; k < BATCH; ++k) {
          if (u0 + 32 * k < units) {
            uint32_t* q = reinterpret_cast<uint32_t*>(&w[k]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float lo = __uint_as_float(q[e] << 16), hi = __uint_as_float(q[e] & 0xFFFF0000u);
              __half2 hv = __floats2half2_rn(lo, hi);
              q[e] = *reinterpret_cast<uint32_t*>(&hv);
            }
            *reinterpret_cast<uint4*>(ptr[k]) = w[k];
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&in_conv[s]);
      TSF_STAMP(p, 12 + (warp), 2 * (i / C::NCONV) + 1);
    }
  } else if (warp == C::W_QK) {
    // ===================== QK^T issuer =====================
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc(128, 128, 0, 0, true);
      constexpr uint32_t swz = C::SWB == 128 ? SWZ_128B : SWZ_64B;
      for (int i = 0; i < my_tiles; ++i) {
        const int s = i % NST, b = i % NS;
        mbar_wait_sleep(&in_conv[s], (i / NST) & 1);
        if constexpr (NS == 2) {  // S[b] is free once the softmax of tile i - 2 has loaded it (and stored P)
          if (i >= 2) mbar_wait_sleep(&p_full[b], ((i - 2) >> 1) & 1);
        } else {                  // the whole slot is free once the epilogue of tile i - 4 has read O
          if (i >= NS) mbar_wait_sleep(&o_empty[b], ((i - NS) / NS) & 1);
        }
        TSF_STAMP(p, 12 + (C::W_QK), i);
        tc_fence_after();
        const uint32_t xa = smem_u32(sIn + s * C::TILE_BYTES);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k * 16 / C::CH) * C::CHUNK_BYTES + (k * 16 % C::CH) * 2;
          mma_ss(tmem + b * C::SLOT + C::COL_S, make_sdesc(xa + off, 16, 8 * C::SWB, swz),
                 make_sdesc(xa + off, 16, 8 * C::SWB, swz), idesc, k > 0);
        }
        mma_commit(&s_full[b]);
      }
    }
    __syncwarp();
  } else if (warp == C::W_PV) {
    // ===================== PV issuer =====================
    if (elect_one()) {
      constexpr uint32_t idesc = make_idesc(128, D, 0, 1, true);
      constexpr uint32_t swz = C::SWB == 128 ? SWZ_128B : SWZ_64B;
      for (int i = 0; i < my_tiles; ++i) {
        const int s = i % NST, b = i % NS;
        mbar_wait_sleep(&p_full[b], (i / NS) & 1);
        // O[b] is free once the epilogue of tile i - NS has read it (NS = 4:
        // implied, the QK^T of this tile waited for it)
        if (NS == 2 && i >= 2) mbar_wait_sleep(&o_empty[b], ((i - 2) >> 1) & 1);
        TSF_STAMP(p, 12 + (C::W_PV), i);
        tc_fence_after();
        const uint32_t va = smem_u32(sIn + s * C::TILE_BYTES);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          mma_ts(tmem + b * C::SLOT + C::COL_O, tmem + b * C::SLOT + C::COL_P + 8 * k,
                 make_sdesc(va + k * 16 * C::SWB, C::CHUNK_BYTES, 8 * C::SWB, swz), idesc, k > 0);
        mma_commit(&o_full[b]);
      }
    }
    __syncwarp();
  } else if (warp < C::W_EPI) {
    // ===================== softmax (warps 0-3) =====================
    const uint32_t r = warp * 32 + lane;                 // tile row == TMEM lane
    const uint32_t lane_base = (warp * 32) << 16;
    const int colstart = (int)((warp * 32) & ~(uint32_t)(WIN - 1));
    const bool row_ok = (int)r < rows_used;
    const int g = (int)r / L;
    const int lo = g * L - colstart, hi = lo + L;        // this row's window columns [lo, hi)
    const float sl2 = p.scale_log2;
    if constexpr (NS == 2) {  // P columns outside the windows stay zero in both slots
      uint32_t z[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) z[i] = 0;
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        tmem_st_x32(tmem + lane_base + b * C::SLOT + C::COL_P, z);
        tmem_st_x32(tmem + lane_base + b * C::SLOT + C::COL_P + 32, z);
      }
      tmem_wait_st();
    }
    for (int i = 0; i < my_tiles; ++i) {
      const int b = i % NS;
      mbar_wait(&s_full[b], (i / NS) & 1);
      TSF_STAMP(p, 12 + (warp), 4 * i);
      tc_fence_after();
      uint32_t sv[WIN];
#pragma unroll
      for (int c = 0; c < WIN; c += 32) tmem_ld_x32(tmem + lane_base + b * C::SLOT + C::COL_S + colstart + c, sv + c);
      tmem_wait_ld();
      float l = 0.f;
      uint32_t pk[WIN / 2];
      if constexpr (LT > 0) {
        // compact path (L = LT divides 32): the row's LT valid scores are the
        // LT-column block number gsel of its 32-column window; only those are
        // exponentiated (LT instead of 32 exps per row)
        const int gsel = (int)lane / LT;
        float v[LT];
#pragma unroll
        for (int k = 0; k < LT; ++k) {
          uint32_t x = sv[k];
#pragma unroll
          for (int g2 = 1; g2 < 32 / LT; ++g2) x = (gsel == g2) ? sv[g2 * LT + k] : x;
          v[k] = __uint_as_float(x);
        }
        float m = v[0];
#pragma unroll
        for (int k = 1; k < LT; ++k) m = fmaxf(m, v[k]);
        const float mb = m * sl2;
        uint32_t pw[LT / 2];
#pragma unroll
        for (int k = 0; k < LT; k += 2) {
          pw[k / 2] = pack2<true>(ex2(fmaf(v[k], sl2, -mb)), ex2(fmaf(v[k + 1], sl2, -mb)));
          const float2 pr = unpack2<true>(pw[k / 2]);
          l += pr.x + pr.y;                              // l sums the rounded P (reading G9)
        }
#pragma unroll
        for (int c = 0; c < WIN / 2; ++c)
          pk[c] = (row_ok && c / (LT / 2) == gsel) ? pw[c % (LT / 2)] : 0u;
      } else {
        float m = -INFINITY;
#pragma unroll
        for (int c = 0; c < WIN; ++c) {
          const bool ok = row_ok && c >= lo && c < hi;
          m = ok ? fmaxf(m, __uint_as_float(sv[c])) : m;
        }
        const float mb = (m == -INFINITY) ? 0.f : m * sl2;
#pragma unroll
        for (int c = 0; c < WIN; c += 2) {
          const bool ok0 = row_ok && c >= lo && c < hi;
          const bool ok1 = row_ok && c + 1 >= lo && c + 1 < hi;
          const float p0 = ok0 ? ex2(fmaf(__uint_as_float(sv[c]), sl2, -mb)) : 0.f;
          const float p1 = ok1 ? ex2(fmaf(__uint_as_float(sv[c + 1]), sl2, -mb)) : 0.f;
          pk[c / 2] = pack2<true>(p0, p1);
          const float2 pr = unpack2<true>(pk[c / 2]);
          l += pr.x + pr.y;                              // l sums the rounded P (reading G9)
        }
      }
      // P[b] and l[b] are free once the epilogue of tile i - 2 has read O[b] and
      // l[b] (which also means PV(i - 2) has consumed P[b])
      TSF_STAMP(p, 12 + (warp), 4 * i + 1);
      if (NS == 2 && i >= 2) {
        mbar_wait(&o_empty[b], ((i - 2) >> 1) & 1);
        tc_fence_after();
      }
      TSF_STAMP(p, 12 + (warp), 4 * i + 2);
      if constexpr (NS == 2) {
#pragma unroll
        for (int c = 0; c < WIN / 2; c += 16)
          tmem_st_x16(tmem + lane_base + b * C::SLOT + C::COL_P + colstart / 2 + c, pk + c);
      } else {
        // P over the slot's first 64 columns: this row's window, zeros elsewhere
        // (those columns still hold S values of this lane)
        uint32_t z[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) z[e] = 0u;
#pragma unroll
        for (int c = 0; c < 64; c += 16) {
          const int w = c - colstart / 2;
          if (w >= 0 && w < WIN / 2) tmem_st_x16(tmem + lane_base + b * C::SLOT + C::COL_P + c, pk + (w & (WIN / 2 - 1)));
          else tmem_st_x16(tmem + lane_base + b * C::SLOT + C::COL_P + c, z);
        }
      }
      lbuf[b * 128 + r] = l;
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);
      TSF_STAMP(p, 12 + (warp), 4 * i + 3);
    }
  } else if (warp < C::W_CONV) {
    // ===================== epilogue (warpgroup e = slot e: warps 4-7, 8-11) =====================
    const uint32_t e = (warp - C::W_EPI) >> 2;          // slot of this warpgroup
    const uint32_t q4 = warp & 3;                       // TMEM lane quarter
    const uint32_t r = q4 * 32 + lane;
    const uint32_t lane_base = (q4 * 32) << 16;
    const uint32_t et = threadIdx.x - 32 * (C::W_EPI + 4 * e);  // 0..127
    const bool row_ok = (int)r < rows_used;
    const int gi = (int)r / L, li = (int)r - gi * L;
    const bool dist = p.P > 1;
    uint8_t* stg = sOut + e * C::TILE_BYTES;
    const uint32_t bar_id = 1 + e;
    for (int i = (int)e; i < my_tiles; i += 2) {
      const int tile = blockIdx.x + i * gridDim.x;
      const int s = i % NST, b = i % NS;
      const uint32_t tcol = tmem + lane_base + b * C::SLOT;
      const uint32_t ph = (i / NS) & 1;
      mbar_wait(&o_full[b], ph);
      mbar_wait(&p_full[b], ph);                         // l[b] written (release by the softmax warps)
      mbar_wait(&in_conv[s], (i / NST) & 1);             // residual rows converted (release by the converter)
      TSF_STAMP(p, 12 + (warp), 4 * (i >> 1));
      tc_fence_after();
      float o[D];
#pragma unroll
      for (int c = 0; c < D; c += 32) tmem_ld_x32(tcol + C::COL_O + c, reinterpret_cast<uint32_t*>(o + c));
      const float l = lbuf[b * 128 + r];
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[b]);
      TSF_STAMP(p, 12 + (warp), 4 * (i >> 1) + 1);
      // this warpgroup's staging tile is free once its previous store has read it
      if (et == 0) bulk_wait_read0();
      named_bar_sync(bar_id, 128);
      uint32_t nf = 0;
      if (row_ok) {
        const uint32_t orow = dist ? (uint32_t)((li / p.Kc) * (p.Kc * G) + (li % p.Kc) + p.Kc * gi) : r;
        nf = epilogue_row_stage<D, 128, 128>(o, 1.0f / l, sIn + s * C::TILE_BYTES, r, stg, orow);
      }
      report_nonfinite(p, nf);
      TSF_STAMP(p, 12 + (warp), 4 * (i >> 1) + 2);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&in_empty[s]);        // the residual rows of this warp are read
      named_bar_sync(bar_id, 128);
      if (et == 0) {
        const int a0 = (tile % p.tiles_a) * p.Ab, b0 = (tile / p.tiles_a) * p.Bb;
        if (dist) {
          const int rows_per_dst = p.Kc * G;
          for (int dst = 0; dst < p.P; ++dst)
#pragma unroll
            for (int c = 0; c < C::NCH; ++c)
              tma_store_4d(&pm.m[dst], stg + c * C::CHUNK_BYTES + dst * rows_per_dst * C::SWB, c * C::CH, 0, a0, b0);
        } else {
#pragma unroll
          for (int c = 0; c < C::NCH; ++c) tma_store_4d(&to, stg + c * C::CHUNK_BYTES, c * C::CH, 0, a0, b0);
        }
        bulk_commit();
      }
      TSF_STAMP(p, 12 + (warp), 4 * (i >> 1) + 3);
    }
    if (et == 0) bulk_wait0();                           // every X_t store has landed
  }

  tc_fence_before();
  __syncthreads();
  if (warp == C::W_QK) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace tsf
