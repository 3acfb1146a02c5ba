// Flash (online-softmax) attention for long sequences (L > 128): spatial
// attention over N tokens of each frame (C2-C5) and temporal attention over
// K = 1024 frames (C5).  Tensor-core bound: 4 d L^2 flops per group against
// 8 d L bytes.
//
// One persistent CTA per SM loops over work items (two 128-row query tiles of
// one group).  The group's K/V stream through an NST-deep TMA ring in tiles of
// SUB rows shared by both query tiles (halves K/V smem/L2 traffic per flop).
//
// Score buffers rotate.  TMEM holds O_0 | O_1 (OW columns each: d, + 16 l
// columns when d = 64) and NB score buffers of SUB fp32 columns.  Score tile
// number m = 2 g + t (KV tile g, query tile t, counted over all items of the
// CTA) lives in buffer m % NB; its P (16-bit pairs, SUB/2 columns) overwrites
// the buffer's upper half after the softmax has read it.  One MMA warp issues,
// in order:
//     S(0) .. S(NB-1);  then for m = 0, 1, ...:  PV(m), S(m + NB)
// S(m + NB) reuses buffer m % NB right after PV(m) consumed its P (the tensor
// pipe executes in order).  With NB = 3 (d = 64, SUB = 96) a query tile's next
// scores S_t(g+1) are issued as soon as the OTHER tile's P_t'(g) is consumed,
// so they are resident before the softmax of S_t(g) ends: the QK^T -> softmax
// -> PV chain no longer serialises a warpgroup (with one buffer per tile the
// warpgroup waited ~30% of the time for its next S).
//
// Online softmax in the log2 domain with conditional rescaling: the running
// max only moves (and O_t is rescaled in TMEM) when a row max grows by more
// than RESCALE_LOG2; O/l is exact either way because l is accumulated against
// the same stale max.
//
// Softmax denominator: for d = 64 the V operand of the PV MMA carries a second
// MN atom of ones (descriptor LBO points from the V tile to a tile of ones),
// so one N = d + 16 MMA yields O and l = sum of the ROUNDED P (exact fp32), and
// the softmax warps spend no ALU on it; for d = 32 / 128 the warps sum P.
//
// exp2: EMU of every 16 exponentials per row go to a polynomial on the FMA/ALU
// pipes (ex2_poly2) instead of MUFU (16 ex2/clk/SM vs 4 d MMA flops per score).
//
// Warp roles (384 threads): warps 0-3 softmax of query tile 0, warps 4-7 of
// tile 1 (thread owns TMEM lane = tile row), warp 8 TMA producer, warp 9 MMA
// issuer (owns TMEM), warp 10 idle, warp 11 converts bf16 tiles to fp16 in the
// block's temporal stage.  In the block modes q = k = v, so one TMA tile per
// stage serves as K (K-major view for QK^T) and V (MN-major view for PV).
#pragma once
#include "sm100.cuh"
#include "attn_common.cuh"

namespace tsf {

constexpr float RESCALE_LOG2 = 8.0f;

template <int D, int EPI, int NST, int SUB>
struct FlashCfg {
  static constexpr int SWB = (2 * D < 128) ? 2 * D : 128;  // bytes per swizzled row chunk
  static constexpr int CH = SWB / 2;                       // 16-bit elements per chunk row
  static constexpr int NCH = D / CH;
  static constexpr int QCHUNK = 128 * SWB;                 // Q tiles: 128 rows
  static constexpr int Q_TILE = NCH * QCHUNK;
  static constexpr int Q_BYTES = 2 * Q_TILE;
  static constexpr int KCHUNK = SUB * SWB;                 // K/V tiles: SUB rows
  static constexpr int KV_TILE = NCH * KCHUNK;
  static constexpr bool SHARED = EpiTraits<EPI>::SHARED;  // block: K_j = V_j (one tile per stage)
  static constexpr int STAGE_BYTES = (SHARED ? 1 : 2) * KV_TILE;
  static constexpr bool ONES = (D == 64);
  static constexpr int ONES_BYTES = ONES ? SUB * SWB : 0;
  static constexpr int SMEM = Q_BYTES + NST * STAGE_BYTES + ONES_BYTES + 1024 + 256;
  static_assert(SMEM <= 227 * 1024, "shared memory");
  static_assert(SUB % 32 == 0 && SUB >= 64 && SUB <= 128, "KV tile rows");
  static constexpr uint32_t OW = ONES ? D + 16 : D;
  static constexpr uint32_t COL_O0 = 0, COL_O1 = OW, COL_S = 2 * OW;
  // rotating score buffers, at most 3: the rescale of O_t at S_t(g) waits for
  // PV_t(g-1) on o_full[t] by parity, which needs PV_t(g-2) retired; S(m)
  // is issued after PV(m - NB), which implies that only for NB <= 3
  static constexpr int NB_FIT = (512 - 2 * (int)OW) / SUB;
  static constexpr int NB = NB_FIT < 3 ? NB_FIT : 3;
  static_assert(NB >= 2, "TMEM budget");
  static constexpr int W_TMA = 8, W_MMA = 9, W_CONV = 11;
  static constexpr int THREADS = 384;                       // whole warpgroups (setmaxnreg is per warpgroup)
  // setmaxnreg must balance: (168 - 56) x 128 released >= (224 - 168) x 256 gained
  static constexpr int REG_SOFTMAX = 224, REG_PRODUCER = 56;
};

template <int D, int EPI, int NST, int EMU, int SUB>
__global__ void __launch_bounds__(384, 1)
attn_flash_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                  const __grid_constant__ CUtensorMap tv, const AttnParams p) {
  using C = FlashCfg<D, EPI, NST, SUB>;
  constexpr int NB = C::NB;
  constexpr bool F16 = EpiTraits<EPI>::F16;
  constexpr bool CONVERT = EpiTraits<EPI>::CONVERT;
  constexpr bool SHARED = C::SHARED;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                        // Q0 | Q1
  uint8_t* sKV = smem + C::Q_BYTES;          // NST x (K | V)
  uint8_t* sOnes = sKV + NST * C::STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOnes + C::ONES_BYTES);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;               // [NST]
  uint64_t* v_full = k_full + NST;           // [NST]
  uint64_t* kv_empty = v_full + NST;         // [NST]
  uint64_t* kv_conv = kv_empty + NST;        // [NST] converter -> MMA (CONVERT only)
  uint64_t* s_full = kv_conv + NST;          // [NB] score buffer written (MMA commit)
  uint64_t* p_full = s_full + NB;            // [NB] P stored (4 softmax warps)
  uint64_t* o_full = p_full + NB;            // [2] one phase per PV of the tile
  uint64_t* o_done = o_full + 2;             // [2] last PV of the item retired (one phase per item)
  uint64_t* o_empty = o_done + 2;            // [2] epilogue read O -> next item's PV may overwrite
  uint64_t* q_empty = o_empty + 2;           // last QK^T of the item retired -> next Q may load
  uint64_t* q_conv = q_empty + 1;            // converter warp -> MMA (CONVERT only)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(q_conv + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int L = p.L, nkv = p.nkv;  // nkv = ceil(L / SUB) KV tiles per group
  // persistent: CTA handles work items blockIdx.x, blockIdx.x + gridDim.x, ...;
  // item = (query-tile pair qp, group (ga, gb)), group-major so consecutive
  // CTAs share a group's K/V in L2
  const int my_items = (p.num_items > (int)blockIdx.x) ? (p.num_items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  auto item_coords = [&](int k, int& qp, int& ga, int& gb) {
    const int item = blockIdx.x + k * gridDim.x;
    qp = item % p.n_qpairs;
    const int grp = item / p.n_qpairs;
    ga = grp % p.A;
    gb = grp / p.A;
  };

  if constexpr (C::ONES) {
    const uint32_t one2 = F16 ? 0x3C003C00u : 0x3F803F80u;
    for (uint32_t i = threadIdx.x; i < C::ONES_BYTES / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(one2, one2, one2, one2);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < NST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&kv_empty[s], 2);  // one commit after each query tile's PV
      mbar_init(&kv_conv[s], 1);
    }
    mbar_init(q_conv, 1);
    for (int b = 0; b < NB; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 4);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&o_full[t], 1);
      mbar_init(&o_done[t], 1);
      mbar_init(&o_empty[t], 4);
    }
    mbar_init(q_empty, 2);
    fence_barrier_init();
  }
  if (warp == C::W_MMA) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  // registers (setmaxnreg, per role branch): softmax warpgroups 224/thread,
  // producer warpgroup (TMA, MMA, idle, converter) 56/thread
  if (warp == C::W_TMA) {
    // ===================== TMA producer =====================
    reg_dealloc<C::REG_PRODUCER>();
    if (elect_one()) {
      tma_prefetch_desc(&tq);
      tma_prefetch_desc(&tk);
      tma_prefetch_desc(&tv);
      int g = 0;  // KV tiles loaded so far (all items)
      for (int k = 0; k < my_items; ++k) {
        int qp, ga, gb;
        item_coords(k, qp, ga, gb);
        if (k > 0) mbar_wait_sleep(q_empty, (k - 1) & 1);
        mbar_arrive_expect_tx(q_full, C::Q_BYTES);
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int c = 0; c < C::NCH; ++c)
            tma_load_4d(sQ + t * C::Q_TILE + c * C::QCHUNK, &tq, q_full, c * C::CH, qp * 256 + t * 128, ga, gb);
        for (int j = 0; j < nkv; ++j, ++g) {
          const int s = g % NST;
          if (g >= NST) mbar_wait_sleep(&kv_empty[s], ((g / NST) - 1) & 1);
          uint8_t* sk = sKV + s * C::STAGE_BYTES;
          mbar_arrive_expect_tx(&k_full[s], C::KV_TILE);
#pragma unroll
          for (int c = 0; c < C::NCH; ++c)
            tma_load_4d(sk + c * C::KCHUNK, &tk, &k_full[s], c * C::CH, j * SUB, ga, gb);
          if constexpr (!SHARED) {
            mbar_arrive_expect_tx(&v_full[s], C::KV_TILE);
#pragma unroll
            for (int c = 0; c < C::NCH; ++c)
              tma_load_4d(sk + C::KV_TILE + c * C::KCHUNK, &tv, &v_full[s], c * C::CH, j * SUB, ga, gb);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == C::W_MMA || warp == C::W_MMA + 1) {
    // ===================== MMA issuer (warp 10 idle) =====================
    reg_dealloc<C::REG_PRODUCER>();
    if (warp == C::W_MMA && elect_one()) {
      constexpr uint32_t idesc_qk = make_idesc(128, SUB, 0, 0, F16);
      constexpr uint32_t idesc_pv = make_idesc(128, C::OW, 0, 1, F16);
      constexpr uint32_t swz = (C::SWB == 128) ? SWZ_128B : SWZ_64B;
      const uint32_t q_addr = smem_u32(sQ);
      // S(m) = Q_t K_j^T -> buffer m % NB   (j: global KV tile index)
      auto issue_s = [&](int t, int j, int m) {
        const uint32_t ka = smem_u32(sKV + (j % NST) * C::STAGE_BYTES);
        const uint32_t qa = q_addr + t * C::Q_TILE;
        const uint32_t dS = tmem + C::COL_S + SUB * (m % NB);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t e = k * 16 / C::CH, w = (k * 16 % C::CH) * 2;
          mma_ss(dS, make_sdesc(qa + e * C::QCHUNK + w, 16, 8 * C::SWB, swz),
                 make_sdesc(ka + e * C::KCHUNK + w, 16, 8 * C::SWB, swz), idesc_qk, k > 0);
        }
        mma_commit(&s_full[m % NB]);
      };
      // O_t (+)= P(m) V_j  (+ l_t (+)= P(m) 1)
      auto issue_pv = [&](int t, int j, int m, bool first, bool last) {
        const uint32_t va = smem_u32(sKV + (j % NST) * C::STAGE_BYTES + (SHARED ? 0 : C::KV_TILE));
        const uint32_t aP = tmem + C::COL_S + SUB * (m % NB) + SUB / 2;
        // second MN atom of the B operand: the next V chunk (d = 128) or the ones tile
        const uint32_t vlbo = C::ONES ? smem_u32(sOnes) - va : (uint32_t)C::KCHUNK;
        const uint32_t dO = tmem + (t ? C::COL_O1 : C::COL_O0);
#pragma unroll
        for (int k = 0; k < SUB / 16; ++k)
          mma_ts(dO, aP + 8 * k, make_sdesc(va + k * 16 * C::SWB, vlbo, 8 * C::SWB, swz), idesc_pv,
                 (!first || k > 0) ? 1u : 0u);
        mma_commit(&o_full[t]);
        if (last) mma_commit(&o_done[t]);
      };
      // K tile j (and, separately, V tile j) of stage j % NST usable
      auto wait_k = [&](int j) {
        if constexpr (CONVERT) mbar_wait_sleep(&kv_conv[j % NST], (j / NST) & 1);
        else mbar_wait_sleep(&k_full[j % NST], (j / NST) & 1);
      };
      auto wait_v = [&](int j) {
        if constexpr (!SHARED) mbar_wait_sleep(&v_full[j % NST], (j / NST) & 1);
        else wait_k(j);
      };
      const int nS = 2 * nkv;  // score tiles per item
      int g0 = 0;              // global KV tile index of the item's first tile
      for (int k = 0; k < my_items; ++k, g0 += nkv) {
        const int M0 = 2 * g0;  // global score-tile index of the item's first S
        if constexpr (CONVERT) mbar_wait_sleep(q_conv, k & 1);
        else mbar_wait_sleep(q_full, k & 1);
        for (int n = 0; n < NB && n < nS; ++n) {
          const int t = n & 1, i = n >> 1;
          if (t == 0) wait_k(g0 + i);
          tc_fence_after();
          issue_s(t, g0 + i, M0 + n);
          if (i == nkv - 1) mma_commit(q_empty);  // Q_t no longer read once this retires
        }
        for (int n = 0; n < nS; ++n) {
          const int t = n & 1, i = n >> 1, m = M0 + n;
          if (t == 0) wait_v(g0 + i);
          mbar_wait_sleep(&p_full[m % NB], (m / NB) & 1);
          TSF_STAMP(p, C::W_MMA, 2 * n);
          tc_fence_after();
          if (i == 0 && k > 0) {  // the epilogue of the previous item has read O_t
            mbar_wait_sleep(&o_empty[t], (k - 1) & 1);
            tc_fence_after();
          }
          issue_pv(t, g0 + i, m, i == 0, i == nkv - 1);
          mma_commit(&kv_empty[(g0 + i) % NST]);  // K_j/V_j free once both tiles' PVs retire
          const int n2 = n + NB;
          if (n2 < nS) {
            const int t2 = n2 & 1, i2 = n2 >> 1;
            if (t2 == 0) {
              wait_k(g0 + i2);
              tc_fence_after();
            }
            issue_s(t2, g0 + i2, M0 + n2);  // reuses buffer m % NB after PV(m) (in order)
            if (i2 == nkv - 1) mma_commit(q_empty);
          }
          TSF_STAMP(p, C::W_MMA, 2 * n + 1);
        }
      }
    }
    __syncwarp();
  } else if (warp < 8) {
    // ===================== softmax warps =====================
    reg_alloc<C::REG_SOFTMAX>();
    const int t = warp >> 2;                                   // query tile
    const uint32_t row = (warp & 3) * 32 + lane;               // tile row == TMEM lane
    const uint32_t lane_base = ((warp & 3) * 32) << 16;
    const uint32_t tSrow = tmem + lane_base + C::COL_S;
    const uint32_t tOrow = tmem + lane_base + (t ? C::COL_O1 : C::COL_O0);
    const float sl2 = p.scale_log2;
    const bool pingpong = (p.flags & FLASH_PINGPONG) != 0;
    int G0 = 0;  // global KV tile index of the item's first tile
    for (int k = 0; k < my_items; ++k, G0 += nkv) {
      int qp, ga, gb;
      item_coords(k, qp, ga, gb);
      float m_run = -INFINITY;  // running max, log2-scaled units
      float l_run = 0.f;        // used when !ONES

      for (int i = 0; i < nkv; ++i) {
        const int G = G0 + i, m = 2 * G + t, b = m % NB;
        const uint32_t tSb = tSrow + SUB * b;
        TSF_STAMP(p, warp, 6 * i + 0);
        mbar_wait(&s_full[b], (m / NB) & 1);
        TSF_STAMP(p, warp, 6 * i + 1);
        tc_fence_after();
        uint32_t sv[SUB];
#pragma unroll
        for (int c = 0; c < SUB; c += 32) tmem_ld_x32(tSb + c, sv + c);
        tmem_wait_ld();
        TSF_STAMP(p, warp, 6 * i + 2);
        const int valid = L - i * SUB;  // columns >= valid are beyond the sequence
        if (valid < SUB) {
#pragma unroll
          for (int c = 0; c < SUB; ++c) sv[c] = (c < valid) ? sv[c] : 0xFF800000u;  // -inf
        }
        // row max: 8 independent FMNMX3 chains
        float m8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) m8[q] = fmaxf(__uint_as_float(sv[2 * q]), __uint_as_float(sv[2 * q + 1]));
#pragma unroll
        for (int c = 16; c < SUB; c += 16)
#pragma unroll
          for (int q = 0; q < 8; ++q)
            m8[q] = max3(m8[q], __uint_as_float(sv[c + 2 * q]), __uint_as_float(sv[c + 2 * q + 1]));
        const float mx = fmaxf(max3(m8[0], m8[1], m8[2]), max3(m8[3], max3(m8[4], m8[5], m8[6]), m8[7]));
        if (i == nkv - 1 && EPI != EPI_OUT16) {
          // the epilogue's residual row: start its global read now (L1 prefetch)
          const int l_idx = qp * 256 + t * 128 + (int)row;
          if (l_idx < L) {
            const long long in_off = (long long)l_idx * p.sL + (long long)ga * p.sA + (long long)gb * p.sB;
            const uint8_t* rp = reinterpret_cast<const uint8_t*>(p.res) + 2 * in_off;
#pragma unroll
            for (int c = 0; c < 2 * D; c += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(rp + c));
          }
        }
        const float m_new = fmaxf(m_run, mx * sl2);
        TSF_STAMP(p, warp, 6 * i + 3);
        if (i == 0) {
          m_run = m_new;
        } else {
          const bool need = (m_new - m_run) > RESCALE_LOG2;
          if (__any_sync(0xffffffffu, need)) {
            // Move the max for the whole warp (exact for every row); rescale O_t
            // (and its l columns) once PV_t(i-1) has retired.
            const float alpha = ex2(m_run - m_new);
            l_run *= alpha;
            m_run = m_new;
            mbar_wait(&o_full[t], (G - 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < D; c += 32) {
              uint32_t ov[32];
              tmem_ld_x32(tOrow + c, ov);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
              tmem_st_x32(tOrow + c, ov);
            }
            if (C::ONES) {
              uint32_t lv[8];
              tmem_ld_x8(tOrow + D, lv);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 8; ++e) lv[e] = __float_as_uint(__uint_as_float(lv[e]) * alpha);
              tmem_st_x8(tOrow + D, lv);
            }
          }
        }
        // ping-pong: the two warpgroups take turns for the exponential phase
        // (MUFU-bound), so one's exps overlap the other's waits / max / stores
        if (pingpong && !(t == 0 && G == 0)) named_bar_sync(1 + t, 256);
        const float nmb = -m_run;
        float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
        for (int c0 = 0; c0 < SUB; c0 += 32) {
          // three passes over 32 columns (scale, exponentiate, pack) so no
          // MUFU result is consumed right after it is issued (in-order issue)
          float xv[32], pv[32];
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 32; c += 2)
            ffma2(xv[c], xv[c + 1], __uint_as_float(sv[c0 + c]), __uint_as_float(sv[c0 + c + 1]), sl2, sl2, nmb,
                  nmb);
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            if (((c >> 1) & 7) >= 8 - EMU / 2) {
              ex2_poly2(pv[c], pv[c + 1], xv[c], xv[c + 1]);   // FMA/ALU pipes
            } else {
              pv[c] = ex2(xv[c]);                              // MUFU
              pv[c + 1] = ex2(xv[c + 1]);
            }
          }
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            pk[c / 2] = pack2<F16>(pv[c], pv[c + 1]);
            if constexpr (!C::ONES) { ls0 += pv[c]; ls1 += pv[c + 1]; }
          }
          tmem_st_x16(tSb + SUB / 2 + c0 / 2, pk);
        }
        if (pingpong) named_bar_arrive(2 - t, 256);
        l_run += ls0 + ls1;
        TSF_STAMP(p, warp, 6 * i + 4);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b]);
        TSF_STAMP(p, warp, 6 * i + 5);
      }

      // ---- epilogue of item k ----
      mbar_wait(&o_done[t], k & 1);
      tc_fence_after();
      float o[D];
#pragma unroll
      for (int c = 0; c < D; c += 32) tmem_ld_x32(tOrow + c, reinterpret_cast<uint32_t*>(o + c));
      if constexpr (C::ONES) {
        uint32_t lv[8];
        tmem_ld_x8(tOrow + D, lv);
        tmem_wait_ld();
        l_run = __uint_as_float(lv[0]);
      } else {
        tmem_wait_ld();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[t]);  // the next item's PV may overwrite O_t
      const int l_idx = qp * 256 + t * 128 + (int)row;
      if (l_idx < L) {
        const long long in_off = (long long)l_idx * p.sL + (long long)ga * p.sA + (long long)gb * p.sB;
        if (EPI == EPI_BLOCK_T && p.P > 1) {
          // distributed temporal stage: frame l_idx belongs to rank l_idx / Kc
          const int dst = l_idx / p.Kc;
          AttnParams q = p;
          q.o = p.peer_out[dst];
          const long long off = (long long)(l_idx - dst * p.Kc) * p.osL + (long long)ga * p.osA +
                                (long long)(gb + p.b_off) * p.osB;
          epilogue_row_g<D, EPI, D / 8>(q, o, 1.0f / l_run, off, in_off, 0);
        } else {
          const long long off = (long long)l_idx * p.osL + (long long)ga * p.osA + (long long)gb * p.osB;
          epilogue_row_g<D, EPI, D / 8>(p, o, 1.0f / l_run, off, in_off, 0);
        }
      }
    }  // items
    if (pingpong && t == 0 && my_items > 0) named_bar_sync(1, 256);  // consume tile 1's last turn
  } else {
    // ===================== converter warp (block temporal stage) =====================
    reg_dealloc<C::REG_PRODUCER>();
    if constexpr (CONVERT) {
      // bf16 tiles from TMA -> fp16 in place (rows are whole 16-byte units, so
      // the swizzle does not matter); 32 threads, 8 loads in flight per lane
      constexpr int UPR = 2 * D / 16;  // 16-byte units per row
      constexpr int UPC = C::SWB / 16;
      const uint32_t ct = threadIdx.x - 32 * C::W_CONV;
      auto convert_tile = [&](uint8_t* tile, int rows) {
        const int chunk = rows * C::SWB;
        const int per = rows * UPR / 32;  // units per lane
        constexpr int BATCH = 8;
#pragma unroll 1
        for (int b0 = 0; b0 < per; b0 += BATCH) {
          uint4 w[BATCH];
          uint8_t* ptr[BATCH];
#pragma unroll
          for (int k = 0; k < BATCH; ++k) {
            const uint32_t i = ct + 32 * (b0 + k);
            const uint32_t r = i / UPR, u = i % UPR;
            ptr[k] = tile + (u / UPC) * chunk + r * C::SWB + (u % UPC) * 16;
            w[k] = *reinterpret_cast<const uint4*>(ptr[k]);
          }
#pragma unroll
          for (int k = 0; k < BATCH; ++k) {
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
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
      };
      static_assert((SUB * 2 * D / 16 / 32) % 8 == 0, "conversion batching");
      int g = 0;
      for (int k = 0; k < my_items; ++k) {
        mbar_wait(q_full, k & 1);
        convert_tile(sQ, 128);
        convert_tile(sQ + C::Q_TILE, 128);
        if (lane == 0) mbar_arrive(q_conv);
        for (int j = 0; j < nkv; ++j, ++g) {
          const int s = g % NST;
          mbar_wait(&k_full[s], (g / NST) & 1);
          convert_tile(sKV + s * C::STAGE_BYTES, SUB);
          if (lane == 0) mbar_arrive(&kv_conv[s]);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == C::W_MMA) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace tsf
