// Packed short-sequence attention (L <= 128): one 128-row tile holds
// G = Ab * Bb whole groups of L rows each (group-major rows, see
// attn_common.cuh), so one QK^T (128 x 128) and one PV (128 x d) tcgen05 MMA
// cover G independent attentions.  The softmax is restricted to each row's own
// group (block-diagonal mask); P outside the diagonal blocks stays zero.
//
// Used for temporal attention with K <= 128 frames (C1-C4: K = 4, 8, 32, 128)
// and spatial attention with N <= 128 tokens (C1).  This stage is HBM-bound
// (arithmetic intensity ~L/2 flop/B), so the kernel is a persistent stream:
// TMA prefetches NST tiles ahead while the MMA warp and the softmax warpgroup
// work on the current one; two CTAs per SM interleave.
//
// Warp roles (192 threads): warps 0-3 softmax + epilogue (thread r owns tile
// row r = TMEM lane r), warp 4 TMA producer (+ TMEM allocation), warp 5 MMA.
#pragma once
#include "sm100.cuh"
#include "attn_common.cuh"

namespace tsf {

template <int D, int WIN, int EPI, bool SHARED, int NST>
struct PackedCfg {
  static constexpr int SWB = (2 * D < 128) ? 2 * D : 128;  // swizzle width (bytes)
  static constexpr int CH = SWB / 2;                        // elements per column chunk
  static constexpr int NCH = D / CH;                        // column chunks per row
  static constexpr int CHUNK_BYTES = 128 * SWB;             // one chunk of a 128-row tile
  static constexpr int TILE_BYTES = NCH * CHUNK_BYTES;      // 128 x D bf16
  static constexpr int NT = SHARED ? 1 : 3;                 // tiles per stage (q,k,v)
  static constexpr int STAGE_BYTES = NT * TILE_BYTES;
  static constexpr int TCOLS = (192 + D <= 256) ? 256 : 512;  // S(128) + P(64) + O(D)
  static constexpr int COL_S = 0, COL_P = 128, COL_O = 192;
  static constexpr int SMEM = NST * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  // + one output staging tile when the distributed temporal stage scatters X_t
  static constexpr int SMEM_DIST = SMEM + TILE_BYTES;
  static constexpr int THREADS = 192;
};

template <int D, int WIN, int EPI, bool SHARED, int NST>
__global__ void __launch_bounds__(192, (192 + D <= 256) ? 2 : 1)
attn_packed_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                   const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap to,
                   const __grid_constant__ PeerMaps pm, const AttnParams p) {
  using C = PackedCfg<D, WIN, EPI, SHARED, NST>;
  constexpr bool F16 = EpiTraits<EPI>::F16;
  constexpr bool CONVERT = EpiTraits<EPI>::CONVERT;
  // 16-bit outputs go through shared memory and one TMA store per tile (rows of
  // a tile are scattered in HBM: per-thread row stores touch 32 lines per
  // instruction); the fp32 y of EPI_BLOCK_S is stored per thread.
  constexpr bool TMA_OUT = (EPI != EPI_BLOCK_S);
  static_assert(SHARED == EpiTraits<EPI>::SHARED, "q = k = v exactly in the block modes");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * C::STAGE_BYTES);
  uint8_t* stage_out = smem + NST * C::STAGE_BYTES + 1024;  // distributed temporal stage only (1024-aligned)
  uint64_t* full = bars;               // [NST] TMA -> MMA
  uint64_t* empty = bars + NST;        // [NST] epilogue -> TMA
  uint64_t* s_full = bars + 2 * NST;   // MMA -> softmax
  uint64_t* p_full = s_full + 1;       // softmax -> MMA
  uint64_t* o_full = s_full + 2;       // MMA -> epilogue
  uint64_t* o_empty = s_full + 3;      // epilogue -> MMA
  uint64_t* conv_full = s_full + 4;    // softmax warps converted the stage to fp16 -> MMA
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_full + 5);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int L = p.L;
  const int G = p.Ab * p.Bb;
  const int rows_used = L * G;

  // Zero the stage buffers once: rows >= rows_used are never written by TMA
  // and must not hold NaN bit patterns (0 * NaN in PV).
  for (uint32_t i = threadIdx.x; i < NST * C::STAGE_BYTES / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 4);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 4);
    mbar_init(conv_full, 4);
    fence_barrier_init();
  }
  if (warp == 4) tmem_alloc<C::TCOLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const uint32_t tS = tmem + C::COL_S, tP = tmem + C::COL_P, tO = tmem + C::COL_O;

  const int ntiles = p.num_tiles;
  const int my_tiles = (ntiles > (int)blockIdx.x) ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

  if (warp == 4) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      tma_prefetch_desc(&tq);
      if (!SHARED) { tma_prefetch_desc(&tk); tma_prefetch_desc(&tv); }
      if (TMA_OUT) tma_prefetch_desc(&to);
      const uint32_t box_bytes = (uint32_t)(C::CH * 2) * (uint32_t)rows_used;
      for (int i = 0; i < my_tiles; ++i) {
        const int tile = blockIdx.x + i * gridDim.x;
        const int s = i % NST;
        if (i >= NST) mbar_wait(&empty[s], ((i / NST) - 1) & 1);
        const int a0 = (tile % p.tiles_a) * p.Ab, b0 = (tile / p.tiles_a) * p.Bb;
        uint8_t* st = smem + s * C::STAGE_BYTES;
        TSF_STAMP(p, 16 + 4, 2 * i);
        mbar_arrive_expect_tx(&full[s], box_bytes * C::NCH * C::NT);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c) {
          tma_load_4d(st + c * C::CHUNK_BYTES, &tq, &full[s], c * C::CH, 0, a0, b0);
          if (!SHARED) {
            tma_load_4d(st + C::TILE_BYTES + c * C::CHUNK_BYTES, &tk, &full[s], c * C::CH, 0, a0, b0);
            tma_load_4d(st + 2 * C::TILE_BYTES + c * C::CHUNK_BYTES, &tv, &full[s], c * C::CH, 0, a0, b0);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ===================== MMA issuer =====================
    if (elect_one()) {
      constexpr uint32_t idesc_qk = make_idesc(128, 128, 0, 0, F16);
      constexpr uint32_t idesc_pv = make_idesc(128, D, 0, 1, F16);
      for (int i = 0; i < my_tiles; ++i) {
        const int s = i % NST;
        if constexpr (CONVERT) mbar_wait(conv_full, i & 1);
        else mbar_wait(&full[s], (i / NST) & 1);
        tc_fence_after();
        const uint32_t qa = smem_u32(smem + s * C::STAGE_BYTES);
        const uint32_t ka = SHARED ? qa : qa + C::TILE_BYTES;
        const uint32_t va = SHARED ? qa : qa + 2 * C::TILE_BYTES;
        // S = Q K^T   (M=128, N=128, K=D in steps of 16)
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k * 16 / C::CH) * C::CHUNK_BYTES + (k * 16 % C::CH) * 2;
          mma_ss(tS, make_sdesc(qa + off, 16, 8 * C::SWB, C::SWB == 128 ? SWZ_128B : SWZ_64B),
                 make_sdesc(ka + off, 16, 8 * C::SWB, C::SWB == 128 ? SWZ_128B : SWZ_64B), idesc_qk, k > 0);
        }
        mma_commit(s_full);
        TSF_STAMP(p, 16 + 5, 4 * i);
        mbar_wait(p_full, i & 1);
        tc_fence_after();
        if (i > 0) { mbar_wait(o_empty, (i - 1) & 1); tc_fence_after(); }
        // O = P V   (M=128, N=D, K=128 kv rows in steps of 16; V is MN-major)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          mma_ts(tO, tP + 8 * k,
                 make_sdesc(va + k * 16 * C::SWB, C::CHUNK_BYTES, 8 * C::SWB, C::SWB == 128 ? SWZ_128B : SWZ_64B),
                 idesc_pv, k > 0);
        }
        mma_commit(o_full);
        TSF_STAMP(p, 16 + 5, 4 * i + 1);
      }
    }
    __syncwarp();
  } else {
    // ===================== softmax + epilogue (warps 0-3) =====================
    const uint32_t r = warp * 32 + lane;                 // tile row == TMEM lane
    const uint32_t lane_base = (warp * 32) << 16;
    const int colstart = (int)((warp * 32) & ~(uint32_t)(WIN - 1));
    // zero P once (columns outside this warp's window stay zero)
    {
      uint32_t z[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) z[i] = 0;
      tmem_st_x32(tP + lane_base, z);
      tmem_st_x32(tP + lane_base + 32, z);
      tmem_wait_st();
    }
    const bool row_ok = (int)r < rows_used;
    const int g = (int)r / L;                            // group of this row
    const int lo = g * L - colstart, hi = lo + L;        // valid window columns [lo, hi)
    const int gi = g, li = (int)r - g * L;
    const float sl2 = p.scale_log2;

    // x tile (bf16 from TMA) -> fp16 in place, each thread its own row; done
    // for tile i+1 before the epilogue of tile i so the MMA of i+1 overlaps it
    auto convert = [&](int i) {
      const int s = i % NST;
      mbar_wait(&full[s], (i / NST) & 1);
      uint8_t* tile = smem + s * C::STAGE_BYTES;
      // the warp converts its own 32 rows; consecutive lanes take consecutive
      // 16-byte units of a row (bank-conflict free)
      constexpr int UPR = D / 8, UPC = C::SWB / 16;
#pragma unroll
      for (int k = 0; k < UPR; ++k) {
        const uint32_t idx = lane + 32 * k;
        const uint32_t row = warp * 32 + idx / UPR, u = idx % UPR;
        cvt_unit_bf16_to_f16(tile + (u / UPC) * C::CHUNK_BYTES + row * C::SWB + (u % UPC) * 16);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(conv_full);
    };
    if (CONVERT && my_tiles > 0) convert(0);

    for (int i = 0; i < my_tiles; ++i) {
      const int tile = blockIdx.x + i * gridDim.x;
      const int s = i % NST;
      TSF_STAMP(p, 16 + warp, 6 * i + 0);
      mbar_wait(s_full, i & 1);
      TSF_STAMP(p, 16 + warp, 6 * i + 1);
      tc_fence_after();
      uint32_t sv[WIN];
#pragma unroll
      for (int c = 0; c < WIN; c += 32) tmem_ld_x32(tS + lane_base + colstart + c, sv + c);
      tmem_wait_ld();
      float m = -INFINITY;
#pragma unroll
      for (int c = 0; c < WIN; ++c) {
        const bool ok = row_ok && c >= lo && c < hi;
        m = ok ? fmaxf(m, __uint_as_float(sv[c])) : m;
      }
      const float mb = (m == -INFINITY) ? 0.f : m * sl2;
      // l sums the rounded P the PV MMA consumes (weights sum to one exactly)
      float l = 0.f;
      uint32_t pk[WIN / 2];
#pragma unroll
      for (int c = 0; c < WIN; c += 2) {
        const bool ok0 = row_ok && c >= lo && c < hi;
        const bool ok1 = row_ok && c + 1 >= lo && c + 1 < hi;
        const float p0 = ok0 ? ex2(fmaf(__uint_as_float(sv[c]), sl2, -mb)) : 0.f;
        const float p1 = ok1 ? ex2(fmaf(__uint_as_float(sv[c + 1]), sl2, -mb)) : 0.f;
        pk[c / 2] = pack2<F16>(p0, p1);
        const float2 pr = unpack2<F16>(pk[c / 2]);
        l += pr.x + pr.y;
      }
#pragma unroll
      for (int c = 0; c < WIN / 2; c += 16) tmem_st_x16(tP + lane_base + colstart / 2 + c, pk + c);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      TSF_STAMP(p, 16 + warp, 6 * i + 2);

      if (CONVERT && i + 1 < my_tiles) convert(i + 1);
      TSF_STAMP(p, 16 + warp, 6 * i + 3);

      // ---- epilogue ----
      mbar_wait(o_full, i & 1);
      TSF_STAMP(p, 16 + warp, 6 * i + 4);
      tc_fence_after();
      float o[D];
#pragma unroll
      for (int c = 0; c < D; c += 32) tmem_ld_x32(tO + lane_base + c, reinterpret_cast<uint32_t*>(o + c));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_empty);

      const int a0 = (tile % p.tiles_a) * p.Ab, b0 = (tile / p.tiles_a) * p.Bb;
      if (EPI == EPI_BLOCK_T && p.P > 1) {
        // distributed: rows regrouped by destination rank (frame l -> rank
        // l / Kc) into P dense boxes of Kc * G rows, one TMA store per rank
        // straight into that rank's frame shard (NVLink peer memory)
        const int Kc = p.Kc, rows_per_dst = Kc * G;
        if (threadIdx.x == 0) bulk_wait_read0();   // previous tile's stores have read the staging tile
        named_bar_sync(1, 128);
        if (row_ok) {
          const int dst = li / Kc, orow = dst * rows_per_dst + (li - dst * Kc) + Kc * gi;
          report_nonfinite(p, epilogue_row_stage<D, 128, 128>(o, 1.0f / l, smem + s * C::STAGE_BYTES, r, stage_out, orow));
        }
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (threadIdx.x == 0) {
          mbar_arrive(&empty[s]);                  // the input stage is no longer read
          for (int dst = 0; dst < p.P; ++dst)
#pragma unroll
            for (int c = 0; c < C::NCH; ++c)
              tma_store_4d(&pm.m[dst], stage_out + c * C::CHUNK_BYTES + dst * rows_per_dst * C::SWB, c * C::CH, 0,
                           a0, b0);
          bulk_commit();
        }
      } else if constexpr (TMA_OUT) {
        // rows into the stage's (first) tile in place, then one TMA store
        if (row_ok) report_nonfinite(p, epilogue_row_smem<D, 128, EPI>(o, 1.0f / l, smem + s * C::STAGE_BYTES, r));
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (threadIdx.x == 0) {
#pragma unroll
          for (int c = 0; c < C::NCH; ++c)
            tma_store_4d(&to, smem + s * C::STAGE_BYTES + c * C::CHUNK_BYTES, c * C::CH, 0, a0, b0);
          bulk_commit();
          // release the PREVIOUS tile's stage once its store has read smem
          // (at most one store group in flight), so this wait overlaps work
          if (i > 0) {
            bulk_wait_read1();
            mbar_arrive(&empty[(i - 1) % NST]);
          }
          if (i == my_tiles - 1) {
            bulk_wait_read0();
            mbar_arrive(&empty[s]);
          }
        }
      } else {
        const int a = a0 + gi % p.Ab, b = b0 + gi / p.Ab;
        if (row_ok && b < p.B && l > 0.f) {
          const long long off = (long long)li * p.osL + (long long)a * p.osA + (long long)b * p.osB;
          report_nonfinite(p, epilogue_row<D, 128, EPI>(p, o, 1.0f / l, off, smem + s * C::STAGE_BYTES, r));
        }
        named_bar_sync(1, 128);
        if (threadIdx.x == 0) mbar_arrive(&empty[s]);
      }
      TSF_STAMP(p, 16 + warp, 6 * i + 5);
    }
  }

  if (TMA_OUT && threadIdx.x == 0) bulk_wait0();  // all output stores complete
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<C::TCOLS>(tmem);
  }
}

}  // namespace tsf
