// Flash (online-softmax) attention for long sequences (L > 128): spatial
// attention over N tokens of each frame (C2-C5) and temporal attention over
// K = 1024 frames (C5).  Tensor-core bound: 4 d L^2 flops per group against
// 8 d L bytes.
//
// One CTA owns two 128-row query tiles of one group and streams the group's
// K/V in 128-row tiles through an NST-deep TMA ring shared by both query tiles
// (halves K/V smem/L2 traffic per flop).  Each KV tile is consumed in two
// 64-column sub-steps.  Per query tile t the S accumulator is double-buffered
// in TMEM (buffers at columns 128 t + {0, 64}); P_t(i) (16-bit pairs, 32
// columns) overwrites the upper half of the buffer S_t(i) came from, after it
// has been read into registers.  The MMA warp issues, per sub-step i and tile
// t: O_t += P_t(i) V(i), then S_t(i+2) into the buffer just released (the
// tensor pipe executes in order), so while a softmax warpgroup works on S_t(i)
// the next S_t(i+1) is already resident and the tensor core works on the other
// tile and on S_t(i+2).  O0, O1 live at columns 256 and 256 + OW, OW = D (+16
// l columns when D <= 64).
//
// Online softmax in the log2 domain with conditional rescaling: the running
// max only moves (and O_t is rescaled in TMEM) when a row max grows by more
// than RESCALE_LOG2; O/l is exact either way because l is accumulated against
// the same stale max.
//
// Softmax denominator: for D <= 64 the MMA warp also multiplies P_t by a
// column of ones (an N=16 MMA into the l columns after O_t), so l is the exact
// fp32 sum of the rounded P and the softmax warps spend no ALU on it; for
// D = 128 (TMEM full) the warps sum the rounded P themselves.
//
// exp2: EMU of every 16 exponentials per row go to a polynomial on the FMA/ALU
// pipes (ex2_poly2) instead of MUFU, which alone caps d = 64 attention near
// half of tensor peak (16 ex2/clk/SM vs 4d MMA flops per score).
//
// Warp roles (384 threads): warps 0-3 softmax of tile 0, warps 4-7 softmax of
// tile 1 (thread owns TMEM lane = tile row), warp 8 TMA producer, warps 9 and
// 10 MMA issuers of tile 0 and tile 1 (independent, so one tile's issue never
// waits for the other tile's softmax; warp 9 owns TMEM), warp 11 converts bf16
// tiles to fp16 in the block's temporal stage (otherwise idle; it completes
// the third warpgroup so setmaxnreg can move registers to the softmax warps).  In the block
// modes q = k = v, so one TMA tile per stage serves as K (K-major view for
// QK^T) and V (MN-major view for PV).
#pragma once
#include "sm100.cuh"
#include "attn_common.cuh"

namespace tsf {

constexpr float RESCALE_LOG2 = 8.0f;

// SPLIT = warps per tile row: 1, or 2 (d = 64: each warp of a pair takes 32 of
// a sub-step's 64 columns, row maxima exchanged through shared memory) to put
// four softmax warps on every SM sub-partition.
template <int D, int EPI, int NST, int SPLIT = 1, int SUB = 64>
struct FlashCfg {
  static constexpr int SWB = (2 * D < 128) ? 2 * D : 128;
  static constexpr int CH = SWB / 2;
  static constexpr int NCH = D / CH;
  static constexpr int CHUNK_BYTES = 128 * SWB;
  static constexpr int TILE_BYTES = NCH * CHUNK_BYTES;  // 128 x D 16-bit
  static constexpr int Q_BYTES = 2 * TILE_BYTES;
  static constexpr bool SHARED = EpiTraits<EPI>::SHARED;  // block: K_j = V_j (one tile per stage)
  static constexpr int STAGE_BYTES = (SHARED ? 1 : 2) * TILE_BYTES;  // K (+ V)
  // l via an MMA against a ones column: off.  Every tcgen05.mma (M=128, K=16)
  // costs >= 44 cycles whatever its N (tools/ubench5.cu), so the N=16 ones MMA
  // cost as much tensor time as the PV MMA itself; l is summed by the softmax
  // threads instead (FADD2 on the fp32 P before rounding).
  // l via the PV MMA itself (d = 64): the ones column is a second MN atom of
  // the V operand (descriptor LBO points from the V tile to a 128-row tile of
  // ones), so one N = d + 16 MMA produces O and l = P 1 (+~8% PV time).
  // (A separate N=16 MMA cost as much as the PV MMA: every tcgen05.mma is
  // >= 44 cycles; summing P on the FMA pipe competes with the softmax.)
  static constexpr bool ONES = (D == 64);
  static constexpr int ONES_BYTES = ONES ? 128 * SWB : 0;
  static constexpr int XMAX_BYTES = (SPLIT > 1) ? 2 * 2 * 2 * 128 * 4 : 0;  // [tile][half][parity][row]
  static constexpr int SMEM = Q_BYTES + NST * STAGE_BYTES + ONES_BYTES + XMAX_BYTES + 1024 + 256;
  static_assert(SMEM <= 227 * 1024, "shared memory");
  // SUB = KV columns per sub-step: 64 (S double-buffered per tile, N=64 QK^T
  // MMAs) or 128 (one S buffer per tile, N=128 QK^T MMAs: full-rate
  // instructions, but S(i+1) is issued only after PV(i) has consumed P(i))
  static_assert(SUB == 64 || SUB == 128, "sub-step width");
  static constexpr int NBUF = 128 / SUB;                  // S buffers per tile
  static constexpr int LA = NBUF;                         // S look-ahead in sub-steps
  static constexpr int NSW = 8 * SPLIT;                    // softmax warps
  static constexpr int W_TMA = NSW, W_MMA0 = NSW + 1, W_MMA1 = NSW + 2, W_CONV = NSW + 3;
  static constexpr int THREADS = 32 * (NSW + 4);          // whole warpgroups (setmaxnreg is per warpgroup)
  // setmaxnreg must balance: registers the producer warpgroup releases
  // (launch count - 56) x 128 >= what the softmax warpgroups gain.  Launch
  // counts: 168 (384 threads), 96 (640 threads).
  static constexpr int REG_SOFTMAX = (SPLIT == 1) ? 224 : 104, REG_PRODUCER = 56;
  static_assert(SPLIT == 1 || D == 64, "column split: d = 64");
  static constexpr uint32_t OW = ONES ? D + 16 : D;
  // S buffers: tile t, buffer b at column 128 t + 64 b (64 fp32 columns); P
  // (64 16-bit values = 32 columns) overwrites the buffer's upper half.
  static constexpr uint32_t COL_O0 = 256, COL_O1 = 256 + OW;
  static_assert(COL_O1 + OW <= 512, "TMEM budget");
};

template <int D, int EPI, int NST, int EMU, int SPLIT, int SUB>
__global__ void __launch_bounds__(32 * (8 * SPLIT + 4), 1)
attn_flash_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                  const __grid_constant__ CUtensorMap tv, const AttnParams p) {
  using C = FlashCfg<D, EPI, NST, SPLIT, SUB>;
  constexpr int NBUF = C::NBUF, LA = C::LA;
  // sub-step i: S buffer b(i), barrier parity ph(i) (each buffer completes once per NBUF sub-steps)
  auto bufi = [](int i) { return (NBUF == 2) ? (i & 1) : 0; };
  auto phase = [](int i) { return (NBUF == 2) ? ((i >> 1) & 1) : (i & 1); };
  constexpr bool F16 = EpiTraits<EPI>::F16;
  constexpr bool CONVERT = EpiTraits<EPI>::CONVERT;
  constexpr bool SHARED = C::SHARED;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                        // Q0 | Q1
  uint8_t* sKV = smem + C::Q_BYTES;          // NST x (K | V)
  uint8_t* sOnes = sKV + NST * C::STAGE_BYTES;
  float* xmax = reinterpret_cast<float*>(sOnes + C::ONES_BYTES);  // SPLIT > 1: partial row maxima
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOnes + C::ONES_BYTES + C::XMAX_BYTES);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;               // [NST]
  uint64_t* v_full = k_full + NST;           // [NST]
  uint64_t* kv_empty = v_full + NST;         // [NST]
  uint64_t* s_full = kv_empty + NST;         // [2 tiles][2 buffers]
  uint64_t* p_full = s_full + 4;             // [2 tiles][2 buffers]
  uint64_t* o_full = p_full + 4;             // [2] one phase per PV sub-step
  uint64_t* o_done = o_full + 2;             // [2] last PV of the item retired (one phase per item)
  uint64_t* o_empty = o_done + 2;            // [2] epilogue read O -> next item's PV may overwrite
  uint64_t* q_empty = o_empty + 2;           // last QK^T of the item retired -> next Q may load
  uint64_t* q_conv = q_empty + 1;            // converter warp -> MMA (CONVERT only)
  uint64_t* kv_conv = q_conv + 1;            // [NST]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(kv_conv + NST);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int L = p.L, nkv = p.nkv;
  const int nsub = (L + SUB - 1) / SUB;  // SUB-column sub-steps (128 / SUB per 128-row KV tile)
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
      mbar_init(&kv_empty[s], 2);  // one commit from each tile's MMA issuer
      mbar_init(&kv_conv[s], 1);
    }
    mbar_init(q_conv, 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4 * SPLIT);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&o_full[t], 1);
      mbar_init(&o_done[t], 1);
      mbar_init(&o_empty[t], 4 * SPLIT);
    }
    mbar_init(q_empty, 2);
    fence_barrier_init();
  }
  if (warp == C::W_MMA0) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  // registers (setmaxnreg, per role branch): softmax warpgroups 224/thread,
  // producer warpgroup (TMA, MMA, 2 converter warps) 56/thread
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
        if (k > 0) mbar_wait(q_empty, (k - 1) & 1);
        mbar_arrive_expect_tx(q_full, C::Q_BYTES);
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int c = 0; c < C::NCH; ++c)
            tma_load_4d(sQ + t * C::TILE_BYTES + c * C::CHUNK_BYTES, &tq, q_full, c * C::CH,
                        qp * 256 + t * 128, ga, gb);
        for (int j = 0; j < nkv; ++j, ++g) {
          const int s = g % NST;
          if (g >= NST) mbar_wait(&kv_empty[s], ((g / NST) - 1) & 1);
          uint8_t* sk = sKV + s * C::STAGE_BYTES;
          mbar_arrive_expect_tx(&k_full[s], C::TILE_BYTES);
#pragma unroll
          for (int c = 0; c < C::NCH; ++c)
            tma_load_4d(sk + c * C::CHUNK_BYTES, &tk, &k_full[s], c * C::CH, j * 128, ga, gb);
          if constexpr (!SHARED) {
            mbar_arrive_expect_tx(&v_full[s], C::TILE_BYTES);
#pragma unroll
            for (int c = 0; c < C::NCH; ++c)
              tma_load_4d(sk + C::TILE_BYTES + c * C::CHUNK_BYTES, &tv, &v_full[s], c * C::CH, j * 128, ga, gb);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == C::W_MMA0 || warp == C::W_MMA1) {
    // ===================== MMA issuers: one per query tile =====================
    reg_dealloc<C::REG_PRODUCER>();
    // FLASH_ONE_ISSUER: warp W_MMA0 issues both tiles in sub-step order
    // (PV_0(i), S_0(i+LA), PV_1(i), S_1(i+LA)): the tensor pipe then finishes
    // tile 0's work before tile 1's, which keeps the two softmax warpgroups
    // half a period apart.  Otherwise one issuer per tile (their MMAs
    // interleave in the pipe).
    const bool one = (p.flags & FLASH_ONE_ISSUER) != 0;
    const int t_self = warp - C::W_MMA0;
    const int t_lo = one ? 0 : t_self, t_hi = one ? 1 : t_self;
    if (!(one && t_self == 1) && elect_one()) {
      constexpr uint32_t idesc_qk = make_idesc(128, SUB, 0, 0, F16);
      constexpr uint32_t idesc_pv = make_idesc(128, C::OW, 0, 1, F16);
      constexpr uint32_t swz = (C::SWB == 128) ? SWZ_128B : SWZ_64B;
      const uint32_t q_addr = smem_u32(sQ);
      // S_t(i) = Q_t K_{rows 64i..64i+63}^T  -> S buffer (t, i % 2)
      // i: sub-step within the item, G: global sub-step (buffers/parities), g0: global index of the item's first KV tile
      auto issue_s = [&](int t, int i, int G, int g0) {
        const int j = g0 + i * SUB / 128, half = (i * SUB) % 128;
        const uint32_t ka = smem_u32(sKV + (j % NST) * C::STAGE_BYTES) + half * C::SWB;
        const uint32_t qa = q_addr + t * C::TILE_BYTES;
        const uint32_t dS = tmem + 128 * t + SUB * bufi(G);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k * 16 / C::CH) * C::CHUNK_BYTES + (k * 16 % C::CH) * 2;
          mma_ss(dS, make_sdesc(qa + off, 16, 8 * C::SWB, swz), make_sdesc(ka + off, 16, 8 * C::SWB, swz),
                 idesc_qk, k > 0);
        }
        mma_commit(&s_full[2 * t + bufi(G)]);
      };
      // O_t += P_t(i) V_{rows 64i..64i+63} (+ l_t += P_t(i) 1)
      auto issue_pv = [&](int t, int i, int G, int g0) {
        const int j = g0 + i * SUB / 128, half = (i * SUB) % 128;
        const uint32_t va = smem_u32(sKV + (j % NST) * C::STAGE_BYTES + (SHARED ? 0 : C::TILE_BYTES)) +
                            half * C::SWB;
        const uint32_t aP = tmem + 128 * t + SUB * bufi(G) + SUB / 2;
        // second MN atom of the B operand: the next V chunk (d = 128) or the ones tile
        const uint32_t vlbo = C::ONES ? smem_u32(sOnes) - va : (uint32_t)C::CHUNK_BYTES;
        const uint32_t dO = tmem + (t ? C::COL_O1 : C::COL_O0);
#pragma unroll
        for (int k = 0; k < SUB / 16; ++k) {
          const uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
          mma_ts(dO, aP + 8 * k, make_sdesc(va + k * 16 * C::SWB, vlbo, 8 * C::SWB, swz), idesc_pv, acc);
        }
        mma_commit(&o_full[t]);
        if (i == nsub - 1) mma_commit(&o_done[t]);
      };

      // K tile j (and, separately, V tile j) of stage j % NST usable
      auto wait_k = [&](int j) {
        if constexpr (CONVERT) mbar_wait(&kv_conv[j % NST], (j / NST) & 1);
        else mbar_wait(&k_full[j % NST], (j / NST) & 1);
      };
      auto wait_v = [&](int j) {
        if constexpr (!SHARED) mbar_wait(&v_full[j % NST], (j / NST) & 1);
        else wait_k(j);
      };
      constexpr int SPT = 128 / SUB;  // sub-steps per KV tile
      int G0 = 0, g0 = 0;             // global sub-step / KV tile index of the item's start
      for (int k = 0; k < my_items; ++k, G0 += nsub, g0 += nkv) {
        if constexpr (CONVERT) mbar_wait(q_conv, k & 1);
        else mbar_wait(q_full, k & 1);
        wait_k(g0);
        tc_fence_after();
        for (int i = 0; i < LA && i < nsub; ++i)
          for (int t = t_lo; t <= t_hi; ++t) {
            issue_s(t, i, G0 + i, g0);
            if (i == nsub - 1) mma_commit(q_empty);   // Q no longer read once this retires
          }
        for (int i = 0; i < nsub; ++i) {
          const int G = G0 + i, j = g0 + i / SPT;
          if (i % SPT == 0) wait_v(j);
          const bool last_of_tile = (i % SPT == SPT - 1) || i == nsub - 1;
          const bool more = i + LA < nsub;
          if (more && (i + LA) % SPT == 0) wait_k(g0 + (i + LA) / SPT);
          for (int t = t_lo; t <= t_hi; ++t) {
            mbar_wait(&p_full[2 * t + bufi(G)], phase(G));
            TSF_STAMP(p, C::W_MMA0 + t, 2 * i);
            tc_fence_after();
            if (i == 0 && k > 0) {  // the epilogue of the previous item has read O_t
              mbar_wait(&o_empty[t], (k - 1) & 1);
              tc_fence_after();
            }
            issue_pv(t, i, G, g0);
            if (last_of_tile) mma_commit(&kv_empty[j % NST]);  // K_j/V_j free once both tiles' MMAs retire
            if (more) {
              issue_s(t, i + LA, G + LA, g0);  // reuses buffer b(G) after PV_t(G) (same issuer: in order)
              if (i + LA == nsub - 1) mma_commit(q_empty);
            }
            TSF_STAMP(p, C::W_MMA0 + t, 2 * i + 1);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < C::NSW) {
    // ===================== softmax warps =====================
    reg_alloc<C::REG_SOFTMAX>();
    constexpr int CW = SUB / SPLIT;                            // sub-step columns per warp
    const int t = warp / (4 * SPLIT);                          // query tile
    const int hf = (warp >> 2) % SPLIT;                        // column half (SPLIT = 2)
    const int c_off = CW * hf;
    const uint32_t row = (warp & 3) * 32 + lane;               // tile row == TMEM lane
    const uint32_t lane_base = ((warp & 3) * 32) << 16;
    const uint32_t tSrow = tmem + lane_base + 128 * t;
    const uint32_t tOrow = tmem + lane_base + (t ? C::COL_O1 : C::COL_O0);
    const float sl2 = p.scale_log2;
    const bool pingpong = (p.flags & FLASH_PINGPONG) != 0;
    int G0 = 0;
    for (int k = 0; k < my_items; ++k, G0 += nsub) {
    int qp, ga, gb;
    item_coords(k, qp, ga, gb);
    float m_run = -INFINITY;  // running max, log2-scaled units
    float l_run = 0.f;        // used when !ONES

    for (int i = 0; i < nsub; ++i) {
      const int G = G0 + i;
      const uint32_t tSb = tSrow + SUB * bufi(G);
      TSF_STAMP(p, warp, 6 * i + 0);
      mbar_wait(&s_full[2 * t + bufi(G)], phase(G));
      TSF_STAMP(p, warp, 6 * i + 1);
      tc_fence_after();
      uint32_t sv[CW];
#pragma unroll
      for (int c = 0; c < CW; c += 32) tmem_ld_x32(tSb + c_off + c, sv + c);
      tmem_wait_ld();
      TSF_STAMP(p, warp, 6 * i + 2);
      const int valid = L - i * SUB - c_off;  // columns >= valid are beyond the sequence
      if (valid < CW) {
#pragma unroll
        for (int c = 0; c < CW; ++c) sv[c] = (c < valid) ? sv[c] : 0xFF800000u;  // -inf
      }
      // row max: 4 independent FMNMX3 chains
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < CW; c += 8)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          m4[q] = max3(m4[q], __uint_as_float(sv[c + 2 * q]), __uint_as_float(sv[c + 2 * q + 1]));
      float mx = max3(m4[0], m4[1], fmaxf(m4[2], m4[3]));
      if constexpr (SPLIT > 1) {
        // combine with the partner warp's half of the row (parity-buffered slots)
        xmax[((t * 2 + hf) * 2 + (G & 1)) * 128 + row] = mx;
        named_bar_sync(3 + t * 4 + (warp & 3), 64);
        mx = fmaxf(mx, xmax[((t * 2 + (1 - hf)) * 2 + (G & 1)) * 128 + row]);
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
          if (NBUF == 2) mbar_wait(&o_full[t], (G - 1) & 1);  // NBUF == 1: S(i) was issued after PV(i-1)
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < D / SPLIT; c += 32) {   // this warp's share of O's columns
            uint32_t ov[32];
            tmem_ld_x32(tOrow + hf * (D / SPLIT) + c, ov);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
            tmem_st_x32(tOrow + hf * (D / SPLIT) + c, ov);
          }
          if (C::ONES && hf == 0) {
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
      if (pingpong && !(t == 0 && G == 0)) named_bar_sync(1 + t, 256 * SPLIT);
      // every exponential depends on nmb: the fence keeps them below the barrier
      const float nmb = reg_fence(-m_run);
      float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < CW; c0 += 32) {
        // three passes over 32 columns (scale, exponentiate, pack) so no
        // MUFU result is consumed right after it is issued (in-order issue)
        float xv[32], pv[32];
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 32; c += 2)
          ffma2(xv[c], xv[c + 1], __uint_as_float(sv[c0 + c]), __uint_as_float(sv[c0 + c + 1]), sl2, sl2, nmb, nmb);
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
        tmem_st_x16(tSb + SUB / 2 + (c_off + c0) / 2, pk);
      }
      if (pingpong) named_bar_arrive(2 - t, 256 * SPLIT);
      float lsum = ls0 + ls1;
      if constexpr (SPLIT > 1 && !C::ONES) {
        // the row's other half: partial sums through the same parity slots
        // (after the max exchange above the partner has consumed them)
        named_bar_sync(3 + t * 4 + (warp & 3), 64);
        xmax[((t * 2 + hf) * 2 + (G & 1)) * 128 + row] = lsum;
        named_bar_sync(3 + t * 4 + (warp & 3), 64);
        lsum += xmax[((t * 2 + (1 - hf)) * 2 + (G & 1)) * 128 + row];
      }
      l_run += lsum;
      TSF_STAMP(p, warp, 6 * i + 4);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[2 * t + bufi(G)]);
      TSF_STAMP(p, warp, 6 * i + 5);
    }

    // ---- epilogue of item k ----
    mbar_wait(&o_done[t], k & 1);
    tc_fence_after();
    constexpr int DW = D / SPLIT;  // output columns of this warp
    float o[DW];
#pragma unroll
    for (int c = 0; c < DW; c += 32) tmem_ld_x32(tOrow + hf * DW + c, reinterpret_cast<uint32_t*>(o + c));
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
        epilogue_row_g<D, EPI, DW / 8>(q, o, 1.0f / l_run, off, in_off, hf * DW / 8);
      } else {
        const long long off = (long long)l_idx * p.osL + (long long)ga * p.osA + (long long)gb * p.osB;
        epilogue_row_g<D, EPI, DW / 8>(p, o, 1.0f / l_run, off, in_off, hf * DW / 8);
      }
    }
    }  // items
    if (pingpong && t == 0 && my_items > 0) named_bar_sync(1, 256 * SPLIT);  // consume tile 1's last turn
  } else {
    // ===================== converter warp (block temporal stage) =====================
    reg_dealloc<C::REG_PRODUCER>();
    if constexpr (CONVERT) {
      // bf16 tiles from TMA -> fp16 in place (rows are whole 16-byte units, so
      // the swizzle does not matter); 32 threads, one row-chunk unit at a time
      constexpr int UPR = 2 * D / 16;  // 16-byte units per row
      constexpr int UPC = C::SWB / 16;
      const uint32_t ct = threadIdx.x - 32 * C::W_CONV;
      auto convert_tile = [&](uint8_t* tile) {
        constexpr int PER = 128 * UPR / 32;   // units per lane (32 at d = 64)
        constexpr int BATCH = 8;              // loads in flight per lane
        static_assert(PER % BATCH == 0, "conversion batching");
#pragma unroll 1
        for (int b0 = 0; b0 < PER; b0 += BATCH) {
          uint4 w[BATCH];
          uint8_t* ptr[BATCH];
#pragma unroll
          for (int k = 0; k < BATCH; ++k) {
            const uint32_t i = ct + 32 * (b0 + k);
            const uint32_t row = i / UPR, u = i % UPR;
            ptr[k] = tile + (u / UPC) * C::CHUNK_BYTES + row * C::SWB + (u % UPC) * 16;
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
      int g = 0;
      for (int k = 0; k < my_items; ++k) {
        mbar_wait(q_full, k & 1);
        convert_tile(sQ);
        convert_tile(sQ + C::TILE_BYTES);
        if (lane == 0) mbar_arrive(q_conv);
        for (int j = 0; j < nkv; ++j, ++g) {
          const int s = g % NST;
          mbar_wait(&k_full[s], (g / NST) & 1);
          convert_tile(sKV + s * C::STAGE_BYTES);
          if (lane == 0) mbar_arrive(&kv_conv[s]);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == C::W_MMA0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace tsf
