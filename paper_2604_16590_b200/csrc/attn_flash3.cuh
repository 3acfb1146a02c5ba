// Flash attention with one 128-row query tile per CTA and three CTAs per SM
// (spatial stage of the block, "spatial attention at each time
// frame").
//
// Why (measured, tools/trace_flash.py on B200): in the two-tile-per-CTA
// kernel (attn_flash.cuh) the two softmax warps of an SM sub-partition run
// in lockstep, so per 96-key step ~1060 of ~1940 cycles have neither the
// MUFU nor the tensor pipe busy, and a lone warp's exponential phase is
// latency-bound (ping-pong does not help).  Here each CTA is a plain
// serial chain QK^T(g) -> softmax(g) -> PV(g) -> QK^T(g+1) over 64-key tiles,
// and THREE independent CTAs per SM interleave their chains on the shared
// tensor pipe, MUFU and issue ports.
//
// TMEM per CTA: 128 columns = O (D = 64 fp32) | S (64 fp32); the softmax
// writes P (fp16 pairs) over the first 32 columns of S after loading S.  The
// tensor pipe executes one CTA's MMAs in issue order, so QK^T(g+1) (issued
// after PV(g)) never overwrites P(g) before PV(g) has read it, and S(g) being
// ready implies PV(g-1) retired (O may be rescaled, P(g) may be stored).
//
// Softmax: online, log2 domain, conditional rescale (threshold 2^8, exact
// since l uses the same stale max), EMU of 16 exponentials on the FMA pipe
// (ex2_poly2), l accumulated in fp32 from the unrounded P.  Residual of the
// block's spatial epilogue: X_t from global memory (L2).
//
// Warps (192 threads, <= 112 registers each at 3 CTAs per SM): 0-3 softmax +
// epilogue (thread = TMEM lane = query row), 4 TMA producer, 5 MMA issuer
// (+ TMEM allocation).
#pragma once
#include "sm100.cuh"
#include "attn_common.cuh"

namespace tsf {

constexpr float F3_RESCALE_LOG2 = 8.0f;  // same threshold as attn_flash.cuh

template <int D, int EPI, int NST>
struct Flash3Cfg {
  static_assert(D == 64, "flash3: d = 64");
  static constexpr int SUB = 64;                            // keys per step
  static constexpr int SWB = 128;
  static constexpr int Q_BYTES = 128 * SWB;                 // 16 KB
  static constexpr int KV_TILE = SUB * SWB;                 // 8 KB
  static constexpr bool SHARED = EpiTraits<EPI>::SHARED;
  static constexpr int STAGE_BYTES = (SHARED ? 1 : 2) * KV_TILE;
  static constexpr int BAR_BYTES = 256;
  static constexpr int SMEM = Q_BYTES + NST * STAGE_BYTES + BAR_BYTES + 1024;
  static constexpr int THREADS = 192;
  static constexpr uint32_t COL_O = 0, COL_S = D;          // 128 TMEM columns
};

template <int D, int EPI, int NST, int EMU, int CPS>
__global__ void __launch_bounds__(192, CPS)
attn_flash3_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                   const __grid_constant__ CUtensorMap tv, const AttnParams p) {
  using C = Flash3Cfg<D, EPI, NST>;
  constexpr int SUB = C::SUB;
  constexpr bool F16 = EpiTraits<EPI>::F16;
  constexpr bool SHARED = C::SHARED;
  static_assert(!EpiTraits<EPI>::CONVERT, "flash3 takes 16-bit operands as stored");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + C::Q_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + NST * C::STAGE_BYTES);
  uint64_t* kv_full = bars;              // [NST] TMA
  uint64_t* kv_empty = bars + NST;       // [NST] PV retired
  uint64_t* q_full = bars + 2 * NST;     // TMA
  uint64_t* q_empty = q_full + 1;        // last QK^T of the item retired
  uint64_t* s_full = q_full + 2;         // QK^T retired (per step)
  uint64_t* p_full = q_full + 3;         // P stored (4 softmax warps)
  uint64_t* o_full = q_full + 4;         // last PV of the item retired
  uint64_t* o_empty = q_full + 5;        // epilogue read O (4 softmax warps)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(q_full + 6);
  static_assert(sizeof(uint64_t) * (2 * NST + 6) + 4 <= C::BAR_BYTES, "barrier space");

  const uint32_t warp = warp_id(), lane = lane_id();
  const int L = p.L, Lk = p.Lk, nkv = p.nkv;
  const int my_items = (p.num_items > (int)blockIdx.x) ? (p.num_items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  auto item_coords = [&](int k, int& qt, int& ga, int& gb) {
    const int item = blockIdx.x + k * gridDim.x;
    qt = item % p.n_qpairs;              // here: 128-row query tiles per group
    const int grp = item / p.n_qpairs;
    ga = grp % p.A;
    gb = grp / p.A;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(p_full, 4);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 4);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<128>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 4) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      tma_prefetch_desc(&tq);
      tma_prefetch_desc(&tk);
      if (!SHARED) tma_prefetch_desc(&tv);
      int G = 0;
      for (int k = 0; k < my_items; ++k) {
        int qt, ga, gb;
        item_coords(k, qt, ga, gb);
        if (k > 0) mbar_wait_sleep(q_empty, (k - 1) & 1);
        mbar_arrive_expect_tx(q_full, C::Q_BYTES);
        tma_load_4d(sQ, &tq, q_full, 0, qt * 128, ga, gb);
        for (int j = 0; j < nkv; ++j, ++G) {
          const int s = G % NST;
          if (G >= NST) mbar_wait_sleep(&kv_empty[s], ((G / NST) - 1) & 1);
          uint8_t* st = sKV + s * C::STAGE_BYTES;
          mbar_arrive_expect_tx(&kv_full[s], C::STAGE_BYTES);
          tma_load_4d(st, &tk, &kv_full[s], 0, j * SUB, ga, gb);
          if constexpr (!SHARED) tma_load_4d(st + C::KV_TILE, &tv, &kv_full[s], 0, j * SUB, ga, gb);
        }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ===================== MMA issuer =====================
    if (elect_one()) {
      constexpr uint32_t idesc_qk = make_idesc(128, SUB, 0, 0, F16);
      constexpr uint32_t idesc_pv = make_idesc(128, D, 0, 1, F16);
      const uint32_t qa = smem_u32(sQ);
      const uint32_t tS = tmem + C::COL_S, tO = tmem + C::COL_O;
      int G = 0;
      for (int k = 0; k < my_items; ++k) {
        mbar_wait_sleep(q_full, k & 1);
        for (int j = 0; j < nkv; ++j, ++G) {
          const int s = G % NST;
          mbar_wait_sleep(&kv_full[s], (G / NST) & 1);
          tc_fence_after();
          const uint32_t ka = smem_u32(sKV + s * C::STAGE_BYTES);
          // S = Q K_j^T  (M = 128, N = 64, K = d in steps of 16; both K-major)
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            mma_ss(tS, make_sdesc(qa + 32 * kk, 16, 8 * C::SWB, SWZ_128B),
                   make_sdesc(ka + 32 * kk, 16, 8 * C::SWB, SWZ_128B), idesc_qk, kk > 0);
          mma_commit(s_full);
          if (j == nkv - 1) mma_commit(q_empty);  // Q read by every QK^T of the item
          mbar_wait(p_full, G & 1);             // critical path: spin, do not sleep
          TSF_STAMP(p, 5, 2 * (j & 511));
          tc_fence_after();
          if (j == 0 && k > 0) {                 // the epilogue of the previous item has read O
            mbar_wait_sleep(o_empty, (k - 1) & 1);
            tc_fence_after();
          }
          // O (+)= P V_j  (M = 128, N = d, K = 64 keys; P from TMEM, V MN-major)
          const uint32_t va = ka + (SHARED ? 0 : C::KV_TILE);
#pragma unroll
          for (int kk = 0; kk < SUB / 16; ++kk)
            mma_ts(tO, tS + 8 * kk, make_sdesc(va + kk * 16 * C::SWB, C::KV_TILE, 8 * C::SWB, SWZ_128B), idesc_pv,
                   (j > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&kv_empty[s]);
          if (j == nkv - 1) mma_commit(o_full);
          TSF_STAMP(p, 5, 2 * (j & 511) + 1);
        }
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ===================== softmax + epilogue =====================
    const uint32_t row = warp * 32 + lane;
    const uint32_t lane_base = (warp * 32) << 16;
    const uint32_t tSrow = tmem + lane_base + C::COL_S, tOrow = tmem + lane_base + C::COL_O;
    const float sl2 = p.scale_log2;
    int G = 0;
    for (int k = 0; k < my_items; ++k) {
      int qt, ga, gb;
      item_coords(k, qt, ga, gb);
      float m_run = -INFINITY;
      float l0 = 0.f, l1 = 0.f;
      for (int j = 0; j < nkv; ++j, ++G) {
        mbar_wait(s_full, G & 1);
        TSF_STAMP(p, warp, 4 * (j & 255));
        tc_fence_after();
        const int valid = Lk - j * SUB;          // keys >= valid are beyond the sequence (-inf)
        // pass 1: the row max over the 64 scores (two 32-column halves)
        float mx = -INFINITY;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          uint32_t sv[32];
          tmem_ld_x32(tSrow + 32 * h2, sv);
          tmem_wait_ld();
          if (valid < SUB) {
#pragma unroll
            for (int c = 0; c < 32; ++c) sv[c] = (32 * h2 + c < valid) ? sv[c] : 0xFF800000u;
          }
          float m4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) m4[q] = fmaxf(__uint_as_float(sv[2 * q]), __uint_as_float(sv[2 * q + 1]));
#pragma unroll
          for (int c = 8; c < 32; c += 8)
#pragma unroll
            for (int q = 0; q < 4; ++q)
              m4[q] = max3(m4[q], __uint_as_float(sv[c + 2 * q]), __uint_as_float(sv[c + 2 * q + 1]));
          mx = max3(mx, fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        }
        const float m_new = fmaxf(m_run, mx * sl2);
        if (j == 0) {
          m_run = m_new;
        } else if (__any_sync(0xffffffffu, (m_new - m_run) > F3_RESCALE_LOG2)) {
          // O (PV(j-1) retired: S(j) is ready) and l move to the new max
          const float alpha = ex2(m_run - m_new);
          l0 *= alpha;
          l1 *= alpha;
          m_run = m_new;
#pragma unroll
          for (int c = 0; c < D; c += 32) {
            uint32_t ov[32];
            tmem_ld_x32(tOrow + c, ov);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
            tmem_st_x32(tOrow + c, ov);
          }
        }
        const float nmb = -m_run;
        TSF_STAMP(p, warp, 4 * (j & 255) + 1);
        // pass 2: 16-column chunks reloaded from TMEM: scale, exponentiate, pack,
        // store P over S (P of keys c0.. lands in columns c0/2.., below the next chunk)
        uint32_t sb[2][16];                      // chunk c0 + 16 loads while chunk c0 computes
        tmem_ld_x16(tSrow, sb[0]);
        tmem_wait_ld();
#pragma unroll
        for (int c0 = 0; c0 < SUB; c0 += 16) {
          uint32_t* sv = sb[(c0 / 16) & 1];
          if (c0 + 16 < SUB) tmem_ld_x16(tSrow + c0 + 16, sb[((c0 / 16) + 1) & 1]);
          if (valid < SUB) {
#pragma unroll
            for (int c = 0; c < 16; ++c) sv[c] = (c0 + c < valid) ? sv[c] : 0xFF800000u;
          }
          float xv[16], pv[16];
          uint32_t pk[8];
#pragma unroll
          for (int c = 0; c < 16; c += 2)
            ffma2(xv[c], xv[c + 1], __uint_as_float(sv[c]), __uint_as_float(sv[c + 1]), sl2, sl2, nmb, nmb);
#pragma unroll
          for (int c = 0; c < 16; c += 2) {
            if (((c >> 1) & 7) >= 8 - EMU / 2) {
              ex2_poly2(pv[c], pv[c + 1], xv[c], xv[c + 1]);
            } else {
              pv[c] = ex2(xv[c]);
              pv[c + 1] = ex2(xv[c + 1]);
            }
          }
#pragma unroll
          for (int c = 0; c < 16; c += 2) {
            pk[c / 2] = pack2<F16>(pv[c], pv[c + 1]);
            add2(l0, l1, pv[c], pv[c + 1]);
          }
          tmem_st_x8(tSrow + c0 / 2, pk);
          if (c0 + 16 < SUB) tmem_wait_ld();
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        TSF_STAMP(p, warp, 4 * (j & 255) + 2);
      }
      // ---- epilogue of item k, in two 32-column halves ----
      mbar_wait(o_full, k & 1);
      tc_fence_after();
      const int l_idx = qt * 128 + (int)row;
      const float inv_l = 1.0f / (l0 + l1);
      const long long in_off = (long long)l_idx * p.sL + (long long)ga * p.sA + (long long)gb * p.sB;
      const long long off = (long long)l_idx * p.osL + (long long)ga * p.osA + (long long)gb * p.osB;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        float o[32];
        tmem_ld_x32(tOrow + 32 * h2, reinterpret_cast<uint32_t*>(o));
        tmem_wait_ld();
        if (h2 == 1) {                           // O read: the next item's PV may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(o_empty);
        }
        if (l_idx < L) report_nonfinite(p, epilogue_row_g<D, EPI, 4>(p, o, inv_l, off, in_off, 4 * h2));
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

}  // namespace tsf
