// Backward pass of one attention stage (the training the
// paper reports for TimeSformer, PAPER.md P:159-163 / P:509).  For every group
// (a temporal (n, h) or spatial (t, h) sequence of L tokens):
//
//   P = softmax(s Q K^T),  dV = P^T dO,  dP = dO V^T,  dS = P (dP - D),
//   dQ = s dS K,  dK = s dS^T Q,       D_i = sum_e O_ie dO_ie,  s = 1/sqrt(d)
//
// with P recomputed from the forward's row statistic lse2 = log2 sum 2^(s q.k log2e)
// (flash forward, AttnParams.lse).  One CTA owns a 128-key tile of one group
// and walks the group's 128-query tiles (FlashAttention-2 order, transposed):
//
//   MMA  S^T  = K Q_i^T      (TMEM, keys = lanes)        A = K, B = Q_i   (K-major)
//   MMA  dP^T = V dO_i^T     (TMEM)                       A = V, B = dO_i  (K-major)
//   softmax warps (thread = key row): P^T = 2^(S^T s log2e - lse2), dS^T =
//        P^T (dP^T - D); bf16 P^T over S^T, bf16 dS^T over dP^T (TMEM) and
//        into a shared-memory tile (the A operand of the dQ MMA)
//   MMA  dV += P^T dO_i      A = P^T (TMEM), B = dO_i (MN-major)
//   MMA  dK += dS^T Q_i      A = dS^T (TMEM), B = Q_i (MN-major)
//   MMA  dQ_i = dS K         A = dS (smem, MN-major), B = K (MN-major) -> TMEM;
//        the softmax warps (thread = query row) add s dQ_i into an
//        fp32 dQ accumulator with vector reductions (red.global.add.v4.f32)
//   end: dK (times s) and dV rows -> bf16.
//
// TMEM (512 columns): S^T / P^T [0,128) | dP^T / dS^T [128,256) |
// dK [256, 256+d) | dV [256+d, 256+2d) | dQ_i [256+2d, 256+3d) (d <= 64; at
// d = 128 dQ_i goes over S^T).  bf16 operands (the training precision of the
// paper), fp32 accumulation.  d in {32, 64, 128}.
//
// Warps (192 threads): 0-3 softmax / dQ / epilogue, 4 TMA producer, 5 MMA.
#pragma once
#include "sm100.cuh"
#include "attn_common.cuh"

namespace tsf {

struct BwdParams {
  int L, A, B;                 // sequence length, group dims
  long long sL, sA, sB;        // element strides of q, k, v, dO, dK, dV, dQacc (same layout)
  const float* lse;            // [A*B][lse_pitch] group-major, log2 units
  const float* drow;           // [A*B][lse_pitch]
  int lse_pitch;               // >= ceil(L / 128) * 128
  float scale;                 // 1 / sqrt(d)
  float scale_log2;            // log2(e) / sqrt(d)
  float* dq;                   // fp32 accumulator (zeroed by the host)
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  int nkt, nqt;                // 128-row key / query tiles per group
  // PACKED (L <= 128): one 128-row tile holds G = Ab * Bb whole groups (group-
  // major rows, as the forward's packed kernel); keys and queries of a group
  // are in the same tile, so the row statistics are computed in the kernel
  int Ab, Bb, tiles_a;
  int flags;                   // diagnostics: 1 = skip the dQ reductions (timing only, wrong dq)
};

TSF_DEV void bulk_load_1d(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
TSF_DEV void red_add_v4(float* gaddr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(gaddr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

template <int D>
struct BwdCfg {
  static constexpr int SWB = (2 * D < 128) ? 2 * D : 128;
  static constexpr int CH = SWB / 2;
  static constexpr int NCH = D / CH;
  static constexpr int CHUNK = 128 * SWB;                 // one column chunk of a 128-row tile
  static constexpr int TILE = NCH * CHUNK;                // 128 x D bf16
  static constexpr int STAGE = 2 * TILE + 2 * 512;        // Q_i, dO_i, lse2_i, D_i
  static constexpr int NST = (D == 128) ? 1 : 2;          // d = 128: 64 KB tiles, one stage fits
  static constexpr int DS_BYTES = 128 * 128 * 2;          // dS, MN-major A operand (2 chunks of 64 queries)
  static constexpr int SMEM = 2 * TILE + NST * STAGE + DS_BYTES + 256 + 1024;
  // dQ_i gets its own columns when they fit (d <= 64); at d = 128 (S^T | dP^T |
  // dK | dV = 512 columns) it overwrites S^T after the dV MMAs have read P^T
  static constexpr bool DQ_OWN = (256 + 3 * D <= 512);
  static constexpr uint32_t COL_S = 0, COL_DP = 128, COL_DK = 256, COL_DV = 256 + D,
                            COL_DQ = DQ_OWN ? 256 + 2 * D : 0;
  static_assert(256 + 2 * D <= 512, "TMEM: S^T | dP^T | dK | dV");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

template <int D, bool PACKED>
__global__ void __launch_bounds__(192, 1)
attn_bwd_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
                const BwdParams p) {
  using C = BwdCfg<D>;
  constexpr int NST = C::NST;
  constexpr uint32_t swz = (C::SWB == 128) ? SWZ_128B : SWZ_64B;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + C::TILE;
  uint8_t* sSt = smem + 2 * C::TILE;                      // NST stages
  uint8_t* sDS = sSt + NST * C::STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sDS + C::DS_BYTES);
  uint64_t* kv_full = bars;
  uint64_t* st_full = bars + 1;          // [NST]
  uint64_t* st_empty = bars + 1 + NST;   // [NST]
  uint64_t* s_full = bars + 1 + 2 * NST;
  uint64_t* p_full = s_full + 1;         // 4 softmax warps
  uint64_t* dq_full = s_full + 2;
  uint64_t* dq_empty = s_full + 3;       // 4 warps
  uint64_t* dkv_full = s_full + 4;
  uint64_t* st0_full = s_full + 5;       // PACKED: row statistics phase (S, P handed, O)
  uint64_t* p0_full = s_full + 6;
  uint64_t* o0_full = s_full + 7;
  uint64_t* stats_done = s_full + 8;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_full + 9);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int kt = PACKED ? 0 : blockIdx.x % p.nkt;
  const int grp = PACKED ? 0 : blockIdx.x / p.nkt;
  const int ga = grp % p.A, gb = grp / p.A;
  const int nq = PACKED ? 1 : p.nqt;
  // PACKED: tile coordinates and rows in use; row r is position r % L of group r / L
  const int a0 = PACKED ? (int)(blockIdx.x % p.tiles_a) * p.Ab : 0;
  const int b0 = PACKED ? (int)(blockIdx.x / p.tiles_a) * p.Bb : 0;
  const int Gt = PACKED ? p.Ab * p.Bb : 1;
  const int rows_used = PACKED ? p.L * Gt : 128;
  // element offset of tile row r (PACKED: its own group; else the CTA's group)
  auto row_off = [&](int r, int tile0) -> long long {
    if constexpr (PACKED) {
      const int g = r / p.L, l = r - g * p.L;
      return (long long)l * p.sL + (long long)(a0 + g % p.Ab) * p.sA + (long long)(b0 + g / p.Ab) * p.sB;
    } else {
      return (long long)(tile0 + r) * p.sL + (long long)ga * p.sA + (long long)gb * p.sB;
    }
  };
  if constexpr (PACKED) {
    // rows >= rows_used are never written by TMA: zero all tiles once
    if (rows_used < 128) {
      for (uint32_t i = threadIdx.x; i < (2 * C::TILE + NST * C::STAGE) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
      fence_proxy_async_smem();
    }
  }

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < NST; ++s) {
      mbar_init(&st_full[s], 1);
      mbar_init(&st_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 4);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 4);
    mbar_init(dkv_full, 1);
    mbar_init(st0_full, 1);
    mbar_init(p0_full, 4);
    mbar_init(o0_full, 1);
    mbar_init(stats_done, 4);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 4) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      const uint32_t tile_bytes = PACKED ? (uint32_t)(C::CH * 2 * rows_used * C::NCH) : (uint32_t)C::TILE;
      mbar_arrive_expect_tx(kv_full, 2 * tile_bytes);
#pragma unroll
      for (int c = 0; c < C::NCH; ++c) {
        if constexpr (PACKED) {
          tma_load_4d(sK + c * C::CHUNK, &tk, kv_full, c * C::CH, 0, a0, b0);
          tma_load_4d(sV + c * C::CHUNK, &tv, kv_full, c * C::CH, 0, a0, b0);
        } else {
          tma_load_4d(sK + c * C::CHUNK, &tk, kv_full, c * C::CH, kt * 128, ga, gb);
          tma_load_4d(sV + c * C::CHUNK, &tv, kv_full, c * C::CH, kt * 128, ga, gb);
        }
      }
      const long long lbase = (long long)grp * p.lse_pitch;
      for (int i = 0; i < nq; ++i) {
        const int s = i % NST;
        if (i >= NST) mbar_wait_sleep(&st_empty[s], ((i / NST) - 1) & 1);
        uint8_t* st = sSt + s * C::STAGE;
        if constexpr (PACKED) {  // statistics are computed in the kernel
          mbar_arrive_expect_tx(&st_full[s], 2 * tile_bytes);
#pragma unroll
          for (int c = 0; c < C::NCH; ++c) {
            tma_load_4d(st + c * C::CHUNK, &tq, &st_full[s], c * C::CH, 0, a0, b0);
            tma_load_4d(st + C::TILE + c * C::CHUNK, &tdo, &st_full[s], c * C::CH, 0, a0, b0);
          }
        } else {
          mbar_arrive_expect_tx(&st_full[s], C::STAGE);
#pragma unroll
          for (int c = 0; c < C::NCH; ++c) {
            tma_load_4d(st + c * C::CHUNK, &tq, &st_full[s], c * C::CH, i * 128, ga, gb);
            tma_load_4d(st + C::TILE + c * C::CHUNK, &tdo, &st_full[s], c * C::CH, i * 128, ga, gb);
          }
          bulk_load_1d(st + 2 * C::TILE, p.lse + lbase + i * 128, 512, &st_full[s]);
          bulk_load_1d(st + 2 * C::TILE + 512, p.drow + lbase + i * 128, 512, &st_full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ===================== MMA issuer =====================
    if (elect_one()) {
      constexpr uint32_t id_kk = make_idesc(128, 128, 0, 0, false);   // S^T, dP^T: both K-major
      constexpr uint32_t id_tn = make_idesc(128, D, 0, 1, false);     // dV, dK: A TMEM, B MN-major
      constexpr uint32_t id_nn = make_idesc(128, D, 1, 1, false);     // dQ: A, B MN-major
      const uint32_t ka = smem_u32(sK), va = smem_u32(sV), dsa = smem_u32(sDS);
      mbar_wait_sleep(kv_full, 0);
      if constexpr (PACKED) {
        // statistics phase: S = Q K^T (queries = lanes), then O = P V
        constexpr uint32_t id_pv = make_idesc(128, D, 0, 1, false);
        mbar_wait_sleep(&st_full[0], 0);
        tc_fence_after();
        const uint32_t qa = smem_u32(sSt);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k * 16 / C::CH) * C::CHUNK + (k * 16 % C::CH) * 2;
          mma_ss(tmem + C::COL_S, make_sdesc(qa + off, 16, 8 * C::SWB, swz), make_sdesc(ka + off, 16, 8 * C::SWB, swz),
                 id_kk, k > 0);
        }
        mma_commit(st0_full);
        mbar_wait(p0_full, 0);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k)
          mma_ts(tmem + C::COL_DP, tmem + C::COL_S + 8 * k,
                 make_sdesc(va + k * 16 * C::SWB, C::CHUNK, 8 * C::SWB, swz), id_pv, k > 0);
        mma_commit(o0_full);
        mbar_wait(stats_done, 0);
        tc_fence_after();
      }
      for (int i = 0; i < nq; ++i) {
        const int s = i % NST;
        mbar_wait_sleep(&st_full[s], (i / NST) & 1);
        if (!C::DQ_OWN && i > 0) mbar_wait(dq_empty, (i - 1) & 1);   // S^T region: dQ_(i-1) read
        tc_fence_after();
        const uint32_t qa = smem_u32(sSt + s * C::STAGE), doa = qa + C::TILE;
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k * 16 / C::CH) * C::CHUNK + (k * 16 % C::CH) * 2;
          mma_ss(tmem + C::COL_S, make_sdesc(ka + off, 16, 8 * C::SWB, swz), make_sdesc(qa + off, 16, 8 * C::SWB, swz),
                 id_kk, k > 0);
        }
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k * 16 / C::CH) * C::CHUNK + (k * 16 % C::CH) * 2;
          mma_ss(tmem + C::COL_DP, make_sdesc(va + off, 16, 8 * C::SWB, swz),
                 make_sdesc(doa + off, 16, 8 * C::SWB, swz), id_kk, k > 0);
        }
        mma_commit(s_full);
        mbar_wait(p_full, i & 1);
        tc_fence_after();
        // dV += P^T dO_i, dK += dS^T Q_i   (K = 128 queries in steps of 16; B MN-major)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          mma_ts(tmem + C::COL_DV, tmem + C::COL_S + 8 * k,
                 make_sdesc(doa + k * 16 * C::SWB, C::CHUNK, 8 * C::SWB, swz), id_tn, (i > 0 || k > 0) ? 1u : 0u);
          mma_ts(tmem + C::COL_DK, tmem + C::COL_DP + 8 * k,
                 make_sdesc(qa + k * 16 * C::SWB, C::CHUNK, 8 * C::SWB, swz), id_tn, (i > 0 || k > 0) ? 1u : 0u);
        }
        // dQ_i = dS K   (M = 128 queries, K = 128 keys; A = dS in smem, MN-major,
        // 2 chunks of 64 queries; B = K tile, MN-major) -> its own columns, so the
        // next tile's S^T / dP^T MMAs need not wait for the dQ_i readout
        if (C::DQ_OWN && i > 0) {
          mbar_wait(dq_empty, (i - 1) & 1);
          tc_fence_after();
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
          mma_ss(tmem + C::COL_DQ, make_sdesc(dsa + k * 16 * 128, 128 * 128, 8 * 128, SWZ_128B),
                 make_sdesc(ka + k * 16 * C::SWB, C::CHUNK, 8 * C::SWB, swz), id_nn, k > 0);
        mma_commit(dq_full);
        mma_commit(&st_empty[s]);
      }
      mma_commit(dkv_full);
    }
    __syncwarp();
  } else {
    // ===================== softmax / dQ / epilogue (warps 0-3) =====================
    const uint32_t r = warp * 32 + lane;                    // TMEM lane
    const uint32_t lane_base = (warp * 32) << 16;
    // PACKED: a row is real if it is inside the box and its group's b < B (the
    // last tile along B may be partial: TMA zero-fills it, nothing is stored)
    const bool key_ok = PACKED ? ((int)r < rows_used && b0 + ((int)r / p.L) / p.Ab < p.B)
                               : kt * 128 + (int)r < p.L;
    const float sl2 = p.scale_log2;
    // PACKED: this row's group occupies columns [glo, glo + L) of the tile
    const int glo = PACKED ? ((int)r / p.L) * p.L : 0;
    if constexpr (PACKED) {
      // ---- row statistics (thread = query row r): lse2 = m + log2 l, D = O . dO ----
      float* lse_s = reinterpret_cast<float*>(sSt + 2 * C::TILE);
      float* dr_s = reinterpret_cast<float*>(sSt + 2 * C::TILE + 512);
      mbar_wait(st0_full, 0);
      tc_fence_after();
      float m = -INFINITY;
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t sv[32];
        tmem_ld_x32(tmem + lane_base + C::COL_S + c0, sv);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const bool ok = key_ok && c0 + c >= glo && c0 + c < glo + p.L;
          m = ok ? fmaxf(m, __uint_as_float(sv[c])) : m;
        }
      }
      const float mb = (m == -INFINITY) ? 0.f : m * sl2;
      float l = 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t sv[32], pp[16];
        tmem_ld_x32(tmem + lane_base + C::COL_S + c0, sv);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          float pr[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const bool ok = key_ok && c0 + c + e >= glo && c0 + c + e < glo + p.L;
            pr[e] = ok ? ex2(fmaf(__uint_as_float(sv[c + e]), sl2, -mb)) : 0.f;
            l += pr[e];
          }
          pp[c / 2] = pack2<false>(pr[0], pr[1]);
        }
        tmem_st_x16(tmem + lane_base + C::COL_S + c0 / 2, pp);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p0_full);
      lse_s[r] = mb + log2f(l > 0.f ? l : 1.f);
      mbar_wait(o0_full, 0);
      tc_fence_after();
      float dacc = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t ov[32];
        tmem_ld_x32(tmem + lane_base + C::COL_DP + c0, ov);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint4 w = tile_row_u4<D, 128>(sSt + C::TILE, r, c0 / 8 + u);   // dO row r
          const float2 a0 = unpack2<false>(w.x), a1 = unpack2<false>(w.y), a2 = unpack2<false>(w.z),
                       a3 = unpack2<false>(w.w);
          const float* o8 = reinterpret_cast<const float*>(ov) + 8 * u;
          dacc += o8[0] * a0.x + o8[1] * a0.y + o8[2] * a1.x + o8[3] * a1.y + o8[4] * a2.x + o8[5] * a2.y +
                  o8[6] * a3.x + o8[7] * a3.y;
        }
      }
      dr_s[r] = key_ok && l > 0.f ? dacc / l : 0.f;
      tc_fence_before();
      named_bar_sync(1, 128);                                // lse / D of every row visible
      if (lane == 0) mbar_arrive(stats_done);
    }
    for (int i = 0; i < nq; ++i) {
      const int s = i % NST;
      const uint8_t* st = sSt + s * C::STAGE;
      const float* lse = reinterpret_cast<const float*>(st + 2 * C::TILE);
      const float* dr = reinterpret_cast<const float*>(st + 2 * C::TILE + 512);
      const int qvalid = PACKED ? rows_used : p.L - i * 128;  // queries >= qvalid are padding
      mbar_wait(s_full, i & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t sv[32], dv[32];
        tmem_ld_x32(tmem + lane_base + C::COL_S + c0, sv);
        tmem_ld_x32(tmem + lane_base + C::COL_DP + c0, dv);
        tmem_wait_ld();
        uint32_t pp[16], dd[16];
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          float pr[2], dsr[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int q = c0 + c + e;
            const bool ok = key_ok && q < qvalid && (!PACKED || (q >= glo && q < glo + p.L));
            const float pv = ok ? ex2(fmaf(__uint_as_float(sv[c + e]), sl2, -lse[q])) : 0.f;
            pr[e] = pv;
            dsr[e] = ok ? pv * (__uint_as_float(dv[c + e]) - dr[q]) : 0.f;
          }
          pp[c / 2] = pack2<false>(pr[0], pr[1]);
          dd[c / 2] = pack2<false>(dsr[0], dsr[1]);
        }
        tmem_st_x16(tmem + lane_base + C::COL_S + c0 / 2, pp);
        tmem_st_x16(tmem + lane_base + C::COL_DP + c0 / 2, dd);
        // dS (query-contiguous rows of this key) into the MN-major A tile of the dQ MMA
        uint8_t* chunk = sDS + (c0 / 64) * (128 * 128);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t unit = (uint32_t)((c0 % 64) / 8 + u);
          *reinterpret_cast<uint4*>(chunk + r * 128 + ((unit ^ (r & 7u)) << 4)) =
              make_uint4(dd[4 * u], dd[4 * u + 1], dd[4 * u + 2], dd[4 * u + 3]);
        }
      }
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      // dQ_i rows (thread = query row): s dQ into the fp32 accumulator
      mbar_wait(dq_full, i & 1);
      tc_fence_after();
      const bool q_in = PACKED ? key_ok : i * 128 + (int)r < p.L;
      const long long qoff = row_off((int)r, i * 128);
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t qv[32];
        tmem_ld_x32(tmem + lane_base + C::COL_DQ + c0, qv);
        tmem_wait_ld();
        if (q_in && !(p.flags & 1)) {
          float* dst = p.dq + qoff + c0;
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            red_add_v4(dst + e, p.scale * __uint_as_float(qv[e]), p.scale * __uint_as_float(qv[e + 1]),
                       p.scale * __uint_as_float(qv[e + 2]), p.scale * __uint_as_float(qv[e + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_empty);
    }
    // ---- dK, dV rows of this key tile ----
    mbar_wait(dkv_full, 0);
    tc_fence_after();
    const long long off = row_off((int)r, kt * 128);
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t kv[32], vv[32];
      tmem_ld_x32(tmem + lane_base + C::COL_DK + c0, kv);
      tmem_ld_x32(tmem + lane_base + C::COL_DV + c0, vv);
      tmem_wait_ld();
      if (key_ok) {
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
          uint4 wk, wv;
          wk.x = pack2<false>(p.scale * __uint_as_float(kv[e]), p.scale * __uint_as_float(kv[e + 1]));
          wk.y = pack2<false>(p.scale * __uint_as_float(kv[e + 2]), p.scale * __uint_as_float(kv[e + 3]));
          wk.z = pack2<false>(p.scale * __uint_as_float(kv[e + 4]), p.scale * __uint_as_float(kv[e + 5]));
          wk.w = pack2<false>(p.scale * __uint_as_float(kv[e + 6]), p.scale * __uint_as_float(kv[e + 7]));
          wv.x = pack2<false>(__uint_as_float(vv[e]), __uint_as_float(vv[e + 1]));
          wv.y = pack2<false>(__uint_as_float(vv[e + 2]), __uint_as_float(vv[e + 3]));
          wv.z = pack2<false>(__uint_as_float(vv[e + 4]), __uint_as_float(vv[e + 5]));
          wv.w = pack2<false>(__uint_as_float(vv[e + 6]), __uint_as_float(vv[e + 7]));
          *reinterpret_cast<uint4*>(p.dk + off + c0 + e) = wk;
          *reinterpret_cast<uint4*>(p.dv + off + c0 + e) = wv;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// Elementwise helpers of the block backward (HBM-bound, 16-byte vectors).
// out_f32 = a + b + c + d (fp32 a; bf16 b, c; fp32 d accumulator), and its bf16 copy.
__global__ void __launch_bounds__(256) sum4_kernel(const float* __restrict__ a, const float* __restrict__ dq,
                                                   const __nv_bfloat16* __restrict__ dk,
                                                   const __nv_bfloat16* __restrict__ dv, float* __restrict__ out,
                                                   __nv_bfloat16* __restrict__ out_bf16, long long n8) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
    const float4 a0 = reinterpret_cast<const float4*>(a)[2 * i], a1 = reinterpret_cast<const float4*>(a)[2 * i + 1];
    const float4 q0 = reinterpret_cast<const float4*>(dq)[2 * i], q1 = reinterpret_cast<const float4*>(dq)[2 * i + 1];
    const uint4 kb = reinterpret_cast<const uint4*>(dk)[i], vb = reinterpret_cast<const uint4*>(dv)[i];
    const uint32_t ku[4] = {kb.x, kb.y, kb.z, kb.w}, vu[4] = {vb.x, vb.y, vb.z, vb.w};
    float f[8] = {a0.x + q0.x, a0.y + q0.y, a0.z + q0.z, a0.w + q0.w, a1.x + q1.x, a1.y + q1.y, a1.z + q1.z, a1.w + q1.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 k2 = unpack2<false>(ku[e]), v2 = unpack2<false>(vu[e]);
      f[2 * e] += k2.x + v2.x;
      f[2 * e + 1] += k2.y + v2.y;
    }
    reinterpret_cast<float4*>(out)[2 * i] = make_float4(f[0], f[1], f[2], f[3]);
    reinterpret_cast<float4*>(out)[2 * i + 1] = make_float4(f[4], f[5], f[6], f[7]);
    if (out_bf16)
      reinterpret_cast<uint4*>(out_bf16)[i] =
          make_uint4(pack2<false>(f[0], f[1]), pack2<false>(f[2], f[3]), pack2<false>(f[4], f[5]), pack2<false>(f[6], f[7]));
  }
}

// out (bf16) = bf16(a_bf16 + b_bf16) and (optionally) fp32 -> bf16 of c
__global__ void __launch_bounds__(256) add_bf16_kernel(const __nv_bfloat16* __restrict__ a,
                                                       const __nv_bfloat16* __restrict__ b,
                                                       __nv_bfloat16* __restrict__ out, long long n8) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
    const uint4 x = reinterpret_cast<const uint4*>(a)[i], y = reinterpret_cast<const uint4*>(b)[i];
    const uint32_t xu[4] = {x.x, x.y, x.z, x.w}, yu[4] = {y.x, y.y, y.z, y.w};
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 p = unpack2<false>(xu[e]), q = unpack2<false>(yu[e]);
      o[e] = pack2<false>(p.x + q.x, p.y + q.y);
    }
    reinterpret_cast<uint4*>(out)[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

__global__ void __launch_bounds__(256) f32_to_bf16_kernel(const float* __restrict__ a, __nv_bfloat16* __restrict__ out,
                                                          long long n8) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
    const float4 a0 = reinterpret_cast<const float4*>(a)[2 * i], a1 = reinterpret_cast<const float4*>(a)[2 * i + 1];
    reinterpret_cast<uint4*>(out)[i] = make_uint4(pack2<false>(a0.x, a0.y), pack2<false>(a0.z, a0.w),
                                                  pack2<false>(a1.x, a1.y), pack2<false>(a1.z, a1.w));
  }
}

}  // namespace tsf
