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

template <int D, int EPI, int NST, int SUB, int SPLIT_ = 1>
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
  static constexpr uint32_t OW = ONES ? D + 16 : D;
  // SEP: each query tile owns an S buffer (SUB fp32 columns) and a separate P
  // buffer (SUB / 2 columns of 16-bit pairs).  The softmax releases S as soon
  // as it has loaded it, so S_t(g+1) is computed while the softmax of S_t(g)
  // is still exponentiating.  Needs 2 OW + 3 SUB <= 512 TMEM columns (d = 32,
  // 64); d = 128 uses rotating S/P buffers instead (below).
  static constexpr bool SEP = (2 * (int)OW + 3 * SUB) <= 512;
  // SPLIT = 2: two softmax warps per tile row group, each owning half of the
  // score columns (row maxima exchanged through shared memory), i.e. four
  // softmax warps per SM sub-partition to keep MUFU busy.  Needs SEP and the
  // ones-column denominator (no partial row sums to combine).
  static constexpr int SPLIT = SPLIT_;
  static constexpr int NSOFT_ = 8 * SPLIT_;
  static_assert(SPLIT == 1 || (SPLIT == 2 && SEP && ONES), "SPLIT = 2 needs SEP and d = 64");
  static constexpr int CW = SUB / SPLIT;                   // score columns per softmax warp
  static_assert(CW % 16 == 0, "columns per warp");
  static constexpr int QST = SEP ? 2 : 1;                  // Q stages (double-buffered when SMEM allows)
  static constexpr int XMAX_BYTES = SPLIT > 1 ? 2 * 2 * SPLIT * 128 * 4 : 0;  // [parity][tile][half][row]
  static constexpr int BAR_BYTES = 1024;
  // distributed block temporal stage: each softmax warp stages its 32 X_t rows
  // in shared memory so the stores to peer ranks go out as whole 2d-byte rows
  // (UPR lanes per row) instead of one 16-byte piece per thread and row
  static constexpr int EPI_STAGE = (SEP && SPLIT == 1 && EPI == EPI_BLOCK_T) ? NSOFT_ * 32 * 2 * D : 0;
  static constexpr int SMEM =
      QST * Q_BYTES + NST * STAGE_BYTES + ONES_BYTES + XMAX_BYTES + EPI_STAGE + BAR_BYTES + 1024;
  static_assert(SMEM <= 227 * 1024, "shared memory");
  static_assert(SUB % 32 == 0 && SUB >= 64 && SUB <= 128, "KV tile rows");
  static constexpr uint32_t COL_O0 = 0, COL_O1 = OW, COL_S = 2 * OW;
  static constexpr uint32_t COL_P = 2 * OW + 2 * SUB;      // SEP: P_0 | P_1 after S_0 | S_1
  // rotating score buffers, at most 3: the rescale of O_t at S_t(g) waits for
  // PV_t(g-1) on o_full[t] by parity, which needs PV_t(g-2) retired; S(m)
  // is issued after PV(m - NB), which implies that only for NB <= 3
  static constexpr int NB_FIT = (512 - 2 * (int)OW) / SUB;
  static constexpr int NB = SEP ? 2 : (NB_FIT < 3 ? NB_FIT : 3);
  static_assert(NB >= 2, "TMEM budget");
  static constexpr int NSOFT = 8 * SPLIT;                   // softmax warps: tile t = w / (4 SPLIT)
  static constexpr int W_TMA = NSOFT, W_MMA = NSOFT + 1, W_CONV = NSOFT + 3;
  static constexpr int THREADS = 32 * (NSOFT + 4);          // whole warpgroups (setmaxnreg is per warpgroup)
  // setmaxnreg must balance within the launch allocation (65536 / THREADS,
  // rounded down to 8): SPLIT 1: 168 -> 224 / 56; SPLIT 2: 96 -> 104 / 48
  static constexpr int REG_SOFTMAX = SPLIT == 1 ? 224 : 104, REG_PRODUCER = SPLIT == 1 ? 56 : 48;
};

template <int D, int EPI, int NST, int EMU, int SUB, int SPLIT, int MASK = 0>
__global__ void __launch_bounds__(FlashCfg<D, EPI, NST, SUB, SPLIT>::THREADS, 1)
attn_flash_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                  const __grid_constant__ CUtensorMap tv, const AttnParams p) {
  using C = FlashCfg<D, EPI, NST, SUB, SPLIT>;
  constexpr int NB = C::NB;
  constexpr bool F16 = EpiTraits<EPI>::F16;
  constexpr bool CONVERT = EpiTraits<EPI>::CONVERT;
  constexpr bool SHARED = C::SHARED;
  // block spatial stage: the residual X_t row is the query row itself (q = X_t),
  // so the epilogue reads it from the Q tile in shared memory (Q double-buffered)
  // (block temporal stage: the Q tile holds fp16(x), converted in place; equal
  // to the bf16 x except below 2^-14 in magnitude, where it differs by < 2^-25)
  constexpr bool RES_SMEM_OK = C::SEP && EPI != EPI_OUT16;
#ifdef TSF_FLASH_RESGLOBAL_AB
  const bool RES_SMEM = RES_SMEM_OK && !(p.flags & FLASH_RES_GLOBAL);
#else
  // (the global-residual diagnostic is compiled in only for A/B builds: its
  // prefetch branch sits in the step loop)
  constexpr bool RES_SMEM = RES_SMEM_OK;
#endif
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                        // QST x (Q0 | Q1)
  uint8_t* sKV = smem + C::QST * C::Q_BYTES; // NST x (K | V)
  uint8_t* sOnes = sKV + NST * C::STAGE_BYTES;
  float* xmax = reinterpret_cast<float*>(sOnes + C::ONES_BYTES);  // SPLIT > 1: [2][2][SPLIT][128]
  uint8_t* sEpi = sOnes + C::ONES_BYTES + C::XMAX_BYTES;  // EPI_STAGE: [softmax warp][32 rows][2 d bytes]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + C::EPI_STAGE);
  uint64_t* q_full = bars;                   // [QST]
  uint64_t* k_full = bars + C::QST;          // [NST]
  uint64_t* v_full = k_full + NST;           // [NST]
  uint64_t* kv_empty = v_full + NST;         // [NST]
  uint64_t* kv_conv = kv_empty + NST;        // [NST] converter -> MMA (CONVERT only)
  uint64_t* s_full = kv_conv + NST;          // [NB] score buffer written (MMA commit)
  uint64_t* p_full = s_full + NB;            // [NB] P stored (4 softmax warps)
  uint64_t* s_free = p_full + NB;            // [2] SEP: S_t loaded into registers (4 softmax warps)
  uint64_t* o_full = s_free + 2;             // [2] one phase per PV of the tile
  uint64_t* o_done = o_full + 2;             // [2] last PV of the item retired (one phase per item)
  uint64_t* o_empty = o_done + 2;            // [2] epilogue read O -> next item's PV may overwrite
  uint64_t* q_empty = o_empty + 2;           // [QST] last QK^T of the item retired -> next Q may load
  uint64_t* q_conv = q_empty + C::QST;       // [QST] converter warp -> MMA (CONVERT only)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(q_conv + C::QST);
  static_assert(sizeof(uint64_t) * (3 * C::QST + 4 * NST + 2 * NB + 8) + 4 <= C::BAR_BYTES, "barrier space");

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
    for (int q = 0; q < C::QST; ++q) {
      mbar_init(&q_full[q], 1);
      mbar_init(&q_conv[q], 1);
      mbar_init(&q_empty[q], 2 + (RES_SMEM ? C::NSOFT : 0));  // last S of both tiles (+ every softmax warp's epilogue)
    }
    for (int s = 0; s < NST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&kv_empty[s], 2);  // one commit after each query tile's PV
      mbar_init(&kv_conv[s], 1);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 4 * SPLIT);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&o_full[t], 1);
      mbar_init(&o_done[t], 1);
      mbar_init(&o_empty[t], 4 * SPLIT);
      mbar_init(&s_free[t], 4 * SPLIT);
    }
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
        const int qs = k % C::QST;
        if (k >= C::QST) mbar_wait_sleep(&q_empty[qs], ((k / C::QST) - 1) & 1);
        mbar_arrive_expect_tx(&q_full[qs], C::Q_BYTES);
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int c = 0; c < C::NCH; ++c)
            tma_load_4d(sQ + qs * C::Q_BYTES + t * C::Q_TILE + c * C::QCHUNK, &tq, &q_full[qs], c * C::CH,
                        qp * 256 + t * 128, ga, gb);
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
    // ===================== MMA issuers =====================
    // SEP: warp W_MMA issues the QK^T MMAs, warp W_MMA + 1 the PV MMAs (an
    // issuing thread blocks while the tensor pipe is busy, so one role's
    // issue never delays the other's); otherwise warp W_MMA issues both
    reg_dealloc<C::REG_PRODUCER>();
    if ((warp == C::W_MMA || C::SEP) && elect_one()) {
      constexpr uint32_t idesc_qk = make_idesc(128, SUB, 0, 0, F16);
      constexpr uint32_t idesc_pv = make_idesc(128, C::OW, 0, 1, F16);
      constexpr uint32_t swz = (C::SWB == 128) ? SWZ_128B : SWZ_64B;
      const uint32_t q_addr = smem_u32(sQ);
      // S = Q_t K_j^T of item k into TMEM column dS   (j: global KV tile index)
      auto issue_s = [&](int t, int j, int k, uint32_t dS, uint64_t* bar) {
        const uint32_t ka = smem_u32(sKV + (j % NST) * C::STAGE_BYTES);
        const uint32_t qa = q_addr + (k % C::QST) * C::Q_BYTES + t * C::Q_TILE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t e = kk * 16 / C::CH, w = (kk * 16 % C::CH) * 2;
          mma_ss(dS, make_sdesc(qa + e * C::QCHUNK + w, 16, 8 * C::SWB, swz),
                 make_sdesc(ka + e * C::KCHUNK + w, 16, 8 * C::SWB, swz), idesc_qk, kk > 0);
        }
        mma_commit(bar);
      };
      // O_t (+)= P V_j  (+ l_t (+)= P 1), P at TMEM column aP
      auto issue_pv = [&](int t, int j, uint32_t aP, bool first, bool last) {
        const uint32_t va = smem_u32(sKV + (j % NST) * C::STAGE_BYTES + (SHARED ? 0 : C::KV_TILE));
        // second MN atom of the B operand: the next V chunk (d = 128) or the ones tile
        const uint32_t vlbo = C::ONES ? smem_u32(sOnes) - va : (uint32_t)C::KCHUNK;
        const uint32_t dO = tmem + (t ? C::COL_O1 : C::COL_O0);
#pragma unroll
        for (int kk = 0; kk < SUB / 16; ++kk)
          mma_ts(dO, aP + 8 * kk, make_sdesc(va + kk * 16 * C::SWB, vlbo, 8 * C::SWB, swz), idesc_pv,
                 (!first || kk > 0) ? 1u : 0u);
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
      auto wait_q = [&](int k) {
        if constexpr (CONVERT) mbar_wait_sleep(&q_conv[k % C::QST], (k / C::QST) & 1);
        else mbar_wait_sleep(&q_full[k % C::QST], (k / C::QST) & 1);
      };
      if constexpr (C::SEP) {
        // Per global step G (item G / nkv, KV tile G % nkv), in issue order:
        //   S_0(G+1) once softmax 0 has loaded S_0(G);  S_1(G+1) likewise;
        //   PV_0(G) once P_0(G) is stored;  PV_1(G) likewise.
        // Each tile's next scores are thus computed a full step ahead, and
        // the tensor pipe (in order) runs PV_t(G) right behind them.
        const int total = my_items * nkv;
        if (warp == C::W_MMA) {
          // QK^T issuer: S_t(G+1) once softmax t has loaded S_t(G)
          auto issue_next_s = [&](int t, int Gn) {  // S_t(Gn), Gn a global step
            const int k = Gn / nkv, i = Gn - k * nkv;
            if (t == 0) {
              if (i == 0) wait_q(k);
              wait_k(Gn);
            }
            tc_fence_after();
            issue_s(t, Gn, k, tmem + C::COL_S + SUB * t, &s_full[t]);
            if (i == nkv - 1) mma_commit(&q_empty[k % C::QST]);  // Q_t of item k no longer read by MMAs
          };
          if (total > 0) {
            issue_next_s(0, 0);
            issue_next_s(1, 0);
          }
          for (int G = 0; G + 1 < total; ++G) {
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              mbar_wait_sleep(&s_free[t], G & 1);
              issue_next_s(t, G + 1);
            }
          }
        } else {
          // PV issuer: PV_t(G) once P_t(G) is stored
          for (int G = 0; G < total; ++G) {
            const int k = G / nkv, i = G - k * nkv;
            wait_v(G);
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              mbar_wait_sleep(&p_full[t], G & 1);
              TSF_STAMP(p, C::W_MMA, 2 * (2 * i + t));
              tc_fence_after();
              if (i == 0 && k > 0) {  // the epilogue of the previous item has read O_t
                mbar_wait_sleep(&o_empty[t], (k - 1) & 1);
                tc_fence_after();
              }
              issue_pv(t, G, tmem + C::COL_P + (SUB / 2) * t, i == 0, i == nkv - 1);
              mma_commit(&kv_empty[G % NST]);  // K_j/V_j free once both tiles' PVs retire
              TSF_STAMP(p, C::W_MMA, 2 * (2 * i + t) + 1);
            }
          }
        }
      } else {
        // rotating score buffers: score tile m = 2 g + t in buffer m % NB, its
        // P in the buffer's upper half; S(m + NB) is issued right after PV(m)
        const int nS = 2 * nkv;  // score tiles per item
        int g0 = 0;              // global KV tile index of the item's first tile
        for (int k = 0; k < my_items; ++k, g0 += nkv) {
          const int M0 = 2 * g0;  // global score-tile index of the item's first S
          wait_q(k);
          for (int n = 0; n < NB && n < nS; ++n) {
            const int t = n & 1, i = n >> 1, m = M0 + n;
            if (t == 0) wait_k(g0 + i);
            tc_fence_after();
            issue_s(t, g0 + i, k, tmem + C::COL_S + SUB * (m % NB), &s_full[m % NB]);
            if (i == nkv - 1) mma_commit(&q_empty[k % C::QST]);
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
            issue_pv(t, g0 + i, tmem + C::COL_S + SUB * (m % NB) + SUB / 2, i == 0, i == nkv - 1);
            mma_commit(&kv_empty[(g0 + i) % NST]);
            const int n2 = n + NB;
            if (n2 < nS) {
              const int t2 = n2 & 1, i2 = n2 >> 1, m2 = M0 + n2;
              if (t2 == 0) {
                wait_k(g0 + i2);
                tc_fence_after();
              }
              issue_s(t2, g0 + i2, k, tmem + C::COL_S + SUB * (m2 % NB), &s_full[m2 % NB]);
              if (i2 == nkv - 1) mma_commit(&q_empty[k % C::QST]);
            }
            TSF_STAMP(p, C::W_MMA, 2 * n + 1);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < C::W_TMA) {
    // ===================== softmax warps =====================
    // warp w: query tile t = w / (4 SPLIT), column part hf = (w / 4) % SPLIT,
    // rows (w % 4) * 32 + lane (TMEM lanes are tied to the sub-partition)
    reg_alloc<C::REG_SOFTMAX>();
    constexpr int CW = C::CW;                                  // score columns of this warp
    constexpr int PW = (CW % 32 == 0) ? 32 : 16;               // exponential pass width
    const int t = warp / (4 * SPLIT);
    const int hf = (warp >> 2) % SPLIT;
    const uint32_t quarter = warp & 3;
    const uint32_t row = quarter * 32 + lane;                  // tile row == TMEM lane
    const uint32_t lane_base = (quarter * 32) << 16;
    const uint32_t tSrow = tmem + lane_base + C::COL_S + hf * CW;
    const uint32_t tOrow = tmem + lane_base + (t ? C::COL_O1 : C::COL_O0);
    constexpr int OCOLS = D / SPLIT;                           // O columns this warp rescales / stores
    const float sl2 = p.scale_log2;
#ifdef TSF_FLASH_PINGPONG_AB
    const bool pingpong = (p.flags & FLASH_PINGPONG) != 0;
#else
    // ping-pong (measured no faster) is compiled in only for A/B builds: its
    // bar.arrive sits between the exponentials and the P store, and even never
    // taken, that asm (a memory clobber) constrains the scheduling of every
    // step (C2 spatial 690 -> 727 us with it compiled in, profiles/r07/c5_regression)
    constexpr bool pingpong = false;
#endif
    int G0 = 0;  // global KV tile index of the item's first tile
    for (int k = 0; k < my_items; ++k, G0 += nkv) {
      int qp, ga, gb;
      item_coords(k, qp, ga, gb);
      if (k < 256) TSF_STAMP(p, warp, 512 + 2 * k);      // item start
      float m_run = -INFINITY;  // running max, log2-scaled units
      float l_run = 0.f;        // used when !ONES

      for (int i = 0; i < nkv; ++i) {
        const int G = G0 + i, m = 2 * G + t;
        // SEP: S_t in its own buffer, P_t in a separate one; else rotating
        // buffer m % NB with P in its upper half
        const int b = C::SEP ? t : m % NB;
        const uint32_t sphase = C::SEP ? (G & 1) : ((m / NB) & 1);
        const uint32_t tSb = tSrow + SUB * b;
        const uint32_t tPb = C::SEP ? tmem + lane_base + C::COL_P + (SUB / 2) * t + hf * (CW / 2)
                                    : tSb + SUB / 2;
        TSF_STAMP(p, warp, 7 * i + 0);
        mbar_wait(&s_full[b], sphase);
        TSF_STAMP(p, warp, 7 * i + 1);
        tc_fence_after();
        uint32_t sv[CW];
#pragma unroll
        for (int c = 0; c < CW; c += 32) {
          if (c + 32 <= CW) tmem_ld_x32(tSb + c, sv + c);
          else tmem_ld_x16(tSb + c, sv + c);
        }
        tmem_wait_ld();
        if constexpr (C::SEP) {  // S_t may now be overwritten by S_t(G+1)
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_free[t]);
        }
        TSF_STAMP(p, warp, 7 * i + 2);
        const int valid = p.Lk - i * SUB - hf * CW;  // columns >= valid are beyond the key sequence
        if (valid < CW) {
#pragma unroll
          for (int c = 0; c < CW; ++c) sv[c] = (c < valid) ? sv[c] : 0xFF800000u;  // -inf
        }
        if constexpr (MASK) {
          // joint attention over the flattened tokens j = t' N + n' (tsf_joint_attn):
          // query qi = t N + n, key j of this tile = j0 + c
          const int Nf = p.mask_n;
          const int qi = qp * 256 + t * 128 + (int)row;
          const int ti = qi / Nf, ni = qi - ti * Nf;
          const int j0 = i * SUB + hf * CW;
          if (p.mask_mode == 1) {  // [n' = n]: keys j0 + c with (j0 + c - ni) % Nf == 0
            int first = (ni - j0) % Nf;
            if (first < 0) first += Nf;
            uint32_t b0 = 0, b1 = 0, b2 = 0, b3 = 0;
            for (int c = first; c < CW; c += Nf) {
              const uint32_t bit = 1u << (c & 31);
              if (c < 32) b0 |= bit;
              else if (c < 64) b1 |= bit;
              else if (c < 96) b2 |= bit;
              else b3 |= bit;
            }
#pragma unroll
            for (int c = 0; c < CW; ++c) {
              const uint32_t w = c < 32 ? b0 : c < 64 ? b1 : c < 96 ? b2 : b3;
              sv[c] = ((w >> (c & 31)) & 1u) ? sv[c] : 0xFF800000u;
            }
          } else {  // 2: [t' = t] -> j in [ti Nf, ti Nf + Nf);  3: [t' <= t] -> j < (ti + 1) Nf
            const int lo = (p.mask_mode == 2 ? ti * Nf : 0) - j0, hi = (ti + 1) * Nf - j0;
#pragma unroll
            for (int c = 0; c < CW; ++c) sv[c] = (c >= lo && c < hi) ? sv[c] : 0xFF800000u;
          }
        }
        // row max: 8 independent FMNMX3 chains
        float m8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) m8[q] = fmaxf(__uint_as_float(sv[2 * q]), __uint_as_float(sv[2 * q + 1]));
#pragma unroll
        for (int c = 16; c < CW; c += 16)
#pragma unroll
          for (int q = 0; q < 8; ++q)
            m8[q] = max3(m8[q], __uint_as_float(sv[c + 2 * q]), __uint_as_float(sv[c + 2 * q + 1]));
        float mx = fmaxf(max3(m8[0], m8[1], m8[2]), max3(m8[3], max3(m8[4], m8[5], m8[6]), m8[7]));
        if constexpr (SPLIT > 1) {
          // the row's other column part: partial maxima through shared memory
          // (slot by step parity: a partner one step ahead writes the other slot)
          float* xm = xmax + ((G & 1) * 2 + t) * SPLIT * 128;
          xm[hf * 128 + row] = mx;
          named_bar_sync(3 + t * 4 + quarter, 32 * SPLIT);
#pragma unroll
          for (int h2 = 0; h2 < SPLIT; ++h2)
            if (h2 != hf) mx = fmaxf(mx, xm[h2 * 128 + row]);
        }
        if (i == nkv - 1 && EPI != EPI_OUT16 && !RES_SMEM) {
          // the epilogue's residual row: start its global read now (L1 prefetch)
          const int l_idx = qp * 256 + t * 128 + (int)row;
          if (l_idx < L) {
            const long long in_off = (long long)l_idx * p.sL + (long long)ga * p.sA + (long long)gb * p.sB;
            const uint8_t* rp = reinterpret_cast<const uint8_t*>(p.res) + 2 * in_off + hf * (2 * OCOLS);
#pragma unroll
            for (int c = 0; c < 2 * OCOLS; c += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(rp + c));
          }
        }
        const float m_new = fmaxf(m_run, mx * sl2);
        TSF_STAMP(p, warp, 7 * i + 3);
        // Move the max for the whole warp (exact for every row) when some row's
        // max grew by more than RESCALE_LOG2; O_t (and its l columns) is
        // rescaled by alpha before P_t is stored, once PV_t(G-1) has retired.
        // The warps sharing rows see the same maxima, so they decide alike.
        bool rescale = false;
        float alpha = 1.f;
        if (i == 0) {
          m_run = m_new;
        } else if (__any_sync(0xffffffffu, (m_new - m_run) > RESCALE_LOG2)) {
          rescale = true;
          alpha = ex2(m_run - m_new);
          if constexpr (MASK) alpha = (m_new == -INFINITY) ? 1.f : alpha;  // row still fully masked
          l_run *= alpha;
          m_run = m_new;
        }
        auto before_p_store = [&]() {
          // SEP: P_t's buffer is free once PV_t(G-1) retired (every step); the
          // rescale needs the same (O_t final for this step)
          if ((C::SEP && G > 0) || rescale) {
            mbar_wait(&o_full[t], (G - 1) & 1);
            tc_fence_after();
          }
          if (rescale) {
#pragma unroll
            for (int c = hf * OCOLS; c < (hf + 1) * OCOLS; c += 32) {
              uint32_t ov[32];
              tmem_ld_x32(tOrow + c, ov);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
              tmem_st_x32(tOrow + c, ov);
            }
            if (C::ONES && hf == SPLIT - 1) {
              uint32_t lv[8];
              tmem_ld_x8(tOrow + D, lv);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 8; ++e) lv[e] = __float_as_uint(__uint_as_float(lv[e]) * alpha);
              tmem_st_x8(tOrow + D, lv);
            }
          }
        };
        // ping-pong: the two tiles' warps take turns for the exponential phase
        // (MUFU-bound), so one's exps overlap the other's waits / max / stores
        if (pingpong && !(t == 0 && G == 0)) named_bar_sync(1 + t, 256 * SPLIT);
        // a row whose keys so far are all masked (MASK only) has m_run = -inf:
        // its scores are all -inf and exponentiate against 0 to exactly 0
        const float nmb = (MASK && m_run == -INFINITY) ? 0.f : -m_run;
        float ls0 = 0.f, ls1 = 0.f;
        // SEP: all of P_t is packed in registers and stored after the last
        // exponential, so the wait for PV_t(G-1) (P_t's buffer) is at the end
        uint32_t pk_all[C::SEP ? CW / 2 : 1];
#ifdef TSF_FLASH_INPLACE_AB
        // (A/B builds only: compiled in, this branch alone costs the default path
        // stack frame and 13% of the C5 temporal stage)
        if (C::SEP && (p.flags & FLASH_INPLACE_EXP)) {
          // one dependency graph over all CW columns, transformed in place
          // (scores -> log2-domain exponents -> P -> packed pairs), so the
          // scheduler can keep the MUFU queue full across the whole row
          // instead of draining it at the end of each 32-column pass
          float f[CW];
#pragma unroll
          for (int c = 0; c < CW; c += 2)
            ffma2(f[c], f[c + 1], __uint_as_float(sv[c]), __uint_as_float(sv[c + 1]), sl2, sl2, nmb, nmb);
#pragma unroll
          for (int c = 0; c < CW; c += 2) {
            if (((c >> 1) & 7) >= 8 - EMU / 2) {
              ex2_poly2(f[c], f[c + 1], f[c], f[c + 1]);
            } else {
              f[c] = ex2(f[c]);
              f[c + 1] = ex2(f[c + 1]);
            }
          }
#pragma unroll
          for (int c = 0; c < CW; c += 2) {
            pk_all[c / 2] = pack2<F16>(f[c], f[c + 1]);
            if constexpr (!C::ONES) { ls0 += f[c]; ls1 += f[c + 1]; }
          }
        } else
#endif
#pragma unroll
        for (int c0 = 0; c0 < CW; c0 += PW) {
          // three passes over PW columns (scale, exponentiate, pack) so no
          // MUFU result is consumed right after it is issued (in-order issue)
          float xv[PW], pv[PW];
          uint32_t pk_local[C::SEP ? 1 : PW / 2];
          uint32_t* pk = C::SEP ? pk_all + c0 / 2 : pk_local;
#pragma unroll
          for (int c = 0; c < PW; c += 2)
            ffma2(xv[c], xv[c + 1], __uint_as_float(sv[c0 + c]), __uint_as_float(sv[c0 + c + 1]), sl2, sl2, nmb,
                  nmb);
#pragma unroll
          for (int c = 0; c < PW; c += 2) {
            if (((c >> 1) & 7) >= 8 - EMU / 2) {
              ex2_poly2(pv[c], pv[c + 1], xv[c], xv[c + 1]);   // FMA/ALU pipes
            } else {
              pv[c] = ex2(xv[c]);                              // MUFU
              pv[c + 1] = ex2(xv[c + 1]);
            }
          }
#pragma unroll
          for (int c = 0; c < PW; c += 2) {
            pk[c / 2] = pack2<F16>(pv[c], pv[c + 1]);
            if constexpr (!C::ONES) { ls0 += pv[c]; ls1 += pv[c + 1]; }
          }
          if constexpr (!C::SEP) {
            if (c0 == 0) before_p_store();
            if constexpr (PW == 32) tmem_st_x16(tPb + c0 / 2, pk);
            else tmem_st_x8(tPb + c0 / 2, pk);
          }
        }
        TSF_STAMP(p, warp, 7 * i + 4);
        if constexpr (C::SEP) {
          // ping-pong: hand the MUFU to the other tile's warps as soon as the
          // exponentials are done, before waiting for PV_t(G-1) and storing P
          if (pingpong) named_bar_arrive(2 - t, 256 * SPLIT);
          before_p_store();
#pragma unroll
          for (int c0 = 0; c0 < CW; c0 += PW) {
            if constexpr (PW == 32) tmem_st_x16(tPb + c0 / 2, pk_all + c0 / 2);
            else tmem_st_x8(tPb + c0 / 2, pk_all + c0 / 2);
          }
        } else {
          if (pingpong) named_bar_arrive(2 - t, 256 * SPLIT);
        }
        l_run += ls0 + ls1;
        TSF_STAMP(p, warp, 7 * i + 5);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[C::SEP ? t : b]);
        TSF_STAMP(p, warp, 7 * i + 6);
      }

      if (k < 256) TSF_STAMP(p, warp, 512 + 2 * k + 1);  // last P handed, epilogue next
      // ---- epilogue of item k: this warp's OCOLS columns of its rows ----
      mbar_wait(&o_done[t], k & 1);
      tc_fence_after();
      float o[OCOLS];
#pragma unroll
      for (int c = 0; c < OCOLS; c += 32) tmem_ld_x32(tOrow + hf * OCOLS + c, reinterpret_cast<uint32_t*>(o + c));
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
      if constexpr (EPI == EPI_OUT16 && SPLIT == 1) {
        if (p.lse != nullptr && l_idx < L) {  // backward recompute: row statistics
          const long long li = ((long long)gb * p.A + ga) * p.lse_pitch + l_idx;
          p.lse[li] = m_run + log2f(l_run);
          if (p.dO != nullptr) {
            const long long off = (long long)l_idx * p.osL + (long long)ga * p.osA + (long long)gb * p.osB;
            const uint4* dp = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.dO) + off);
            float acc = 0.f;
#pragma unroll
            for (int u = 0; u < OCOLS / 8; ++u) {
              const uint4 w = dp[u];
              const float2 a0 = unpack2<false>(w.x), a1 = unpack2<false>(w.y), a2 = unpack2<false>(w.z),
                           a3 = unpack2<false>(w.w);
              acc += o[8 * u] * a0.x + o[8 * u + 1] * a0.y + o[8 * u + 2] * a1.x + o[8 * u + 3] * a1.y +
                     o[8 * u + 4] * a2.x + o[8 * u + 5] * a2.y + o[8 * u + 6] * a3.x + o[8 * u + 7] * a3.y;
            }
            p.drow[li] = acc / l_run;
          }
        }
      }
      bool staged = false;
      if constexpr (C::EPI_STAGE > 0) {
        if (p.P > 1 && RES_SMEM) {
          // distributed temporal stage: X_t rows staged per warp, then written
          // to their owner ranks (frame l belongs to rank l / Kc) UPR lanes per row
          staged = true;
          uint8_t* stw = sEpi + warp * (32 * 2 * D);
          const bool ok = l_idx < L;
          int dst = 0;
          long long off = 0;
          if (ok) {
            dst = l_idx / p.Kc;
            off = (long long)(l_idx - dst * p.Kc) * p.osL + (long long)ga * p.osA + (long long)(gb + p.b_off) * p.osB;
            report_nonfinite(p, epilogue_row_stage<D, 128, 32>(o, 1.0f / l_run, sQ + (k % C::QST) * C::Q_BYTES + t * C::Q_TILE, row, stw,
                                           lane));
          }
          __syncwarp();
          constexpr int UPR = 2 * D / 16;  // 16-byte units per row
          constexpr int RPI = 32 / UPR;    // rows per warp store
#pragma unroll
          for (int j = 0; j < 32 / RPI; ++j) {
            const int r = j * RPI + (int)lane / UPR, u = (int)lane % UPR;
            const int rd = __shfl_sync(0xffffffffu, dst, r);
            const long long ro = __shfl_sync(0xffffffffu, off, r);
            const int rok = __shfl_sync(0xffffffffu, (int)ok, r);
            if (rok)
              *reinterpret_cast<uint4*>(static_cast<__half*>(p.peer_out[rd]) + ro + 8 * u) = tile_row_u4<D, 32>(stw, r, u);
          }
          __syncwarp();  // the staging tile is rewritten at the next item
        }
      }
      if (l_idx < L && !staged) {
        const long long in_off = (long long)l_idx * p.sL + (long long)ga * p.sA + (long long)gb * p.sB;
        constexpr int NU = OCOLS / 8;
        if (EPI == EPI_BLOCK_T && p.P > 1) {
          // distributed temporal stage: frame l_idx belongs to rank l_idx / Kc
          const int dst = l_idx / p.Kc;
          AttnParams q = p;
          q.o = p.peer_out[dst];
          const long long off = (long long)(l_idx - dst * p.Kc) * p.osL + (long long)ga * p.osA +
                                (long long)(gb + p.b_off) * p.osB;
          if (RES_SMEM_OK && RES_SMEM)
            report_nonfinite(p, epilogue_row<D, 128, EPI, NU>(q, o, 1.0f / l_run, off,
                                          sQ + (k % C::QST) * C::Q_BYTES + t * C::Q_TILE, row, hf * NU));
          else
            report_nonfinite(p, epilogue_row_g<D, EPI, NU>(q, o, 1.0f / l_run, off, in_off, hf * NU));
        } else if (RES_SMEM_OK && RES_SMEM) {
          const long long off = (long long)l_idx * p.osL + (long long)ga * p.osA + (long long)gb * p.osB;
          report_nonfinite(p, epilogue_row<D, 128, EPI, NU>(p, o, 1.0f / l_run, off,
                                        sQ + (k % C::QST) * C::Q_BYTES + t * C::Q_TILE, row, hf * NU));
        } else {
          const long long off = (long long)l_idx * p.osL + (long long)ga * p.osA + (long long)gb * p.osB;
          report_nonfinite(p, epilogue_row_g<D, EPI, NU>(p, o, 1.0f / l_run, off, in_off, hf * NU));
        }
      }
      if (RES_SMEM) {  // this warp's rows of Q_t (item k) read: the next Q may load
        __syncwarp();
        if (lane == 0) mbar_arrive(&q_empty[k % C::QST]);
      }
    }  // items
    if (pingpong && t == 0 && my_items > 0) named_bar_sync(1, 256 * SPLIT);  // consume tile 1's last turn
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
      // (converting the next item's Q between K tiles, instead of at the item
      // boundary, measured neutral at C5 and perturbed the kernel's code: removed)
      for (int k = 0; k < my_items; ++k) {
        const int qs = k % C::QST;
        mbar_wait(&q_full[qs], (k / C::QST) & 1);
        convert_tile(sQ + qs * C::Q_BYTES, 128);
        convert_tile(sQ + qs * C::Q_BYTES + C::Q_TILE, 128);
        if (lane == 0) mbar_arrive(&q_conv[qs]);
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
