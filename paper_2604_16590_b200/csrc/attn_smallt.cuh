// Short-window temporal stage of the block (SURVEY 8(a) rows a1-a5 for
// K in {4, 8, 16, 32}, d = 64): X_t = x + T(x, x, x)
// "temporal attention at each spatial location", stored fp16 (G8),
// optionally scattered straight into the owning ranks' frame shards (row a5,
// fused exchange).
//
// At these K a group's attention is a K x K x 64 contraction -- 4K flop per
// 128-byte row -- so the stage is purely HBM-bound (C2: 134 MB at >= 17 us
// against ~1 GFLOP).  The tcgen05 streaming kernel (attn_stream.cuh) moves
// every tile through a chain of six roles (TMA, converter, QK issuer,
// softmax, PV issuer, epilogue) and its throughput is set by that chain's
// latency with two TMEM slots.  Here every warp does the whole
// chain for its rows in registers, so the only pipeline is the memory one:
//
//   thread 0      keeps NS = 4 x 32 KB input tiles in flight (one 4-D TMA
//                 box per tile: d x K frames x Ab x Bb groups, SWIZZLE_128B,
//                 group-major rows) and issues the tile's output TMA store(s)
//   warps         16 for K <= 16 (one 16-row unit each per tile), 8 for K = 32
//                 (one 32-row group each); per 16-row m-tile: ldmatrix x -> registers, bf16 -> fp16
//                 (exact for |x| < 65504), S = X X^T with mma.sync m16n8k16
//                 (fp32 accumulate; the key fragments ARE the query
//                 fragments, q = k = v = x), block-diagonal softmax in
//                 registers (exact max, one pass: all K keys are present),
//                 P fp16 (unnormalised, l summed from the rounded P), O =
//                 P X (ldmatrix.trans for V), X_t = x + O / l (the residual
//                 is the query fragment again), fp16,
//                 stmatrix into a staging tile laid out per destination rank
//
// The contraction is tiny and register-resident, so the legacy warp-level
// MMA is the right unit here: the tensor pipe is < 5% busy either way and
// what matters is that no role waits on another (K-small
// temporal kernel).
//
// Variants (A/B, profiles/r07/smallt): TSF_SMALLT_WARPS=8; TSF_SMALLT_BULK=1
// (1-D bulk copies per frame into a padded frame-major ring instead of the
// 4-D boxes: slower, 33 vs 31 us at C2 and 0.95 vs 0.54 ms at C3).
//
// Rows of a tile: group-major, row R = gi * L + l (gi = bb * Ab + ab, l the
// frame).  A warp unit is 16 rows (L <= 16: 16 / L whole groups, block-
// diagonal mask) or 32 rows (L = 32: one group, two m-tiles, 32 keys).
#pragma once
#include "attn_common.cuh"

namespace tsf {

constexpr int SMALLT_NO_MATH = 32;  // diagnostics: memory pipeline only (timing, wrong results)

template <int L, int W, bool BULK>
struct SmallTCfg {
  static_assert(L == 4 || L == 8 || L == 16 || L == 32, "window");
  static_assert(W == 8 || (W == 16 && L <= 16), "warps");
  static constexpr int ROWS = 256;               // rows per tile (group x frame)
  static constexpr int G = ROWS / L;             // groups per full tile
  static constexpr int U = L < 16 ? 16 : L;      // rows per warp unit
  static constexpr int MT = U / 16;              // m16 tiles per unit
  static constexpr int KEYS = L < 16 ? 16 : L;   // key columns per unit
  static constexpr int NU = ROWS / U;            // units per tile
  static constexpr int WARPS = W;                // 8, or 16 for L <= 16 (one unit per warp)
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int NS = 4;                   // input ring depth
  static constexpr int TILE = ROWS * 128;        // bytes: 256 rows x 64 x 16-bit
  // BULK layout: frame-major, frame l's G rows contiguous (one 1-D bulk copy per
  // frame), frames FS = G * 128 + 16 bytes apart so that the 8 rows of one
  // ldmatrix / stmatrix (8 frames of a group) fall in 8 different bank groups
  static constexpr int FS = G * 128 + 16;
  static constexpr int STAGE = BULK ? ((L * FS + 1023) / 1024) * 1024 : TILE;
  static constexpr int SMEM = 1024 + NS * STAGE + 2 * STAGE + 64;
};

TSF_DEV uint32_t bf16x2_to_f16x2(uint32_t w) {
  const float lo = __uint_as_float(w << 16), hi = __uint_as_float(w & 0xffff0000u);
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
TSF_DEV uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
TSF_DEV void ldsm_x4(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
TSF_DEV void ldsm_x4_t(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
TSF_DEV void stsm_x4(uint32_t addr, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(r0), "r"(r1),
               "r"(r2), "r"(r3)
               : "memory");
}
// D += A B, m16n8k16, fp16 operands, fp32 accumulators
TSF_DEV void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// byte offset of 16-byte chunk c of row R in a SWIZZLE_128B tile (1024-byte aligned base)
TSF_DEV uint32_t swz(uint32_t R, uint32_t c) { return R * 128u + ((c ^ (R & 7u)) << 4); }

// 1-D bulk copies (contiguous bytes, multiples of 16)
TSF_DEV void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
TSF_DEV void bulk_store(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<uint64_t>(dst)),
               "r"(src), "r"(bytes)
               : "memory");
}

template <int L, int W, bool BULK>
__global__ void __launch_bounds__(SmallTCfg<L, W, BULK>::THREADS, 1)
attn_smallt_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap to,
                   const __grid_constant__ PeerMaps pm, const AttnParams p) {
  using C = SmallTCfg<L, W, BULK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* in_buf = base;
  uint8_t* out_buf = base + C::NS * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(out_buf + 2 * C::STAGE);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int Ab = p.Ab, Bb = p.Bb, gt = Ab * Bb;        // groups in this launch's tiles
  const int P = p.P, Kc = L / P;                        // destination ranks, frames per rank
  const uint32_t in_bytes = (uint32_t)gt * L * 128u;
  const int valid_units = gt * L / C::U;                // host guarantees gt * L % U == 0
  const float sc = p.scale_log2;
  // BULK: tiles are G consecutive groups of the frame plane (group = h + A * n)
  const long long gtot = (long long)p.A * p.B;
  const __nv_bfloat16* xg = static_cast<const __nv_bfloat16*>(p.res);
  // row R = gi * L + l of a tile -> byte offset of its 16-byte chunk c in a stage / staging buffer
  auto in_off = [&](uint32_t R, uint32_t c) -> uint32_t {
    if constexpr (BULK) return (R % L) * C::FS + (R / L) * 128u + c * 16u;
    else return swz(R, c);
  };
  auto issue_load = [&](int tile_, int s_) {
    if constexpr (BULK) {
      const long long g0 = (long long)tile_ * C::G;
      const uint32_t gv = (uint32_t)min((long long)C::G, gtot - g0);
      mbar_arrive_expect_tx(&full[s_], gv * L * 128u);
      const uint32_t dst = smem_u32(in_buf + s_ * C::STAGE);
      for (int l = 0; l < L; ++l) bulk_load(dst + l * C::FS, xg + l * p.sL + g0 * 64, gv * 128u, &full[s_]);
    } else {
      mbar_arrive_expect_tx(&full[s_], in_bytes);
      tma_load_4d(in_buf + s_ * C::STAGE, &tx, &full[s_], 0, 0, (tile_ % p.tiles_a) * Ab, (tile_ / p.tiles_a) * Bb);
    }
  };

  if (tid == 0) {
    for (int s = 0; s < C::NS; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    tma_prefetch_desc(&tx);
    tma_prefetch_desc(P == 1 ? &to : &pm.m[0]);
  }
  __syncthreads();
  const int ntiles = p.num_tiles;
  if (tid == 0) {
    for (int s = 0; s < C::NS; ++s) {
      const int tile = blockIdx.x + s * gridDim.x;
      if (tile >= ntiles) break;
      issue_load(tile, s);
    }
  }
  uint32_t nf = 0;
  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it % C::NS, ob = it & 1;
    mbar_wait(&full[s], (uint32_t)(it / C::NS) & 1u);
    if (tid == 0 && it >= 2) bulk_wait_read1();          // the store of tile it-2 has read staging[ob]
    const uint32_t xin = smem_u32(in_buf + s * C::STAGE);
    const uint32_t xout = smem_u32(out_buf + ob * C::STAGE);
    int units = valid_units;
    uint32_t gv = 0;
    if constexpr (BULK) {
      // a short last tile: zero the rows of the groups that complete its last unit
      // (a stale non-finite row would reach valid rows of the unit through 0 * inf)
      const long long g0 = (long long)tile * C::G;
      gv = (uint32_t)min((long long)C::G, gtot - g0);
      const uint32_t gvr = ((gv * L + C::U - 1) / C::U) * C::U / L;
      units = (int)(gvr * L / C::U);
      for (uint32_t i = tid; i < (gvr - gv) * L * 8u; i += C::THREADS) {
        const uint32_t gi = gv + i / (L * 8u), l = (i / 8u) % L, c = i % 8u;
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(xin + l * C::FS + gi * 128u + c * 16u), "r"(0u)
                     : "memory");
      }
    }
    __syncthreads();
#pragma unroll 1
    for (int u = warp; u < ((p.flags & SMALLT_NO_MATH) ? 0 : units); u += C::WARPS) {
      // ---- x fragments (A operand, row-major 16 x 64 per m-tile), bf16 and fp16
      uint32_t xa[C::MT][4][4], xh[C::MT][4][4];
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t R = u * C::U + mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
          ldsm_x4(xa[mt][kk], xin + in_off(R, kk * 2 + (lane >> 4)));
#pragma unroll
          for (int i = 0; i < 4; ++i) xh[mt][kk][i] = bf16x2_to_f16x2(xa[mt][kk][i]);
        }
      // ---- S = X X^T: key n-tile nt = rows 8 nt .. 8 nt + 7 of the unit, whose
      // B fragments are the A fragments of m-tile nt / 2 (half nt & 1)
      float sacc[C::MT][C::KEYS / 8][4];
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < C::KEYS / 8; ++nt) {
          sacc[mt][nt][0] = sacc[mt][nt][1] = sacc[mt][nt][2] = sacc[mt][nt][3] = 0.f;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma16816(sacc[mt][nt], xh[mt][kk], xh[nt >> 1][kk][nt & 1], xh[nt >> 1][kk][(nt & 1) + 2]);
        }
      // ---- softmax per row (rows g and g + 8 of each m-tile), block-diagonal below 16.
      // P is rounded to fp16 unnormalised (<= 1) and l summed from the ROUNDED
      // values, so the weights applied by the MMA sum to exactly l (as in the
      // tcgen05 kernels, where l comes from the PV MMA); O is scaled by 1/l below.
      uint32_t pa[C::MT][C::KEYS / 16][4];
      float inv[C::MT][2];
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt) {
        float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < C::KEYS / 8; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int key = nt * 8 + 2 * t + e;
            if (L >= 16 || (g / L == key / L)) m0 = fmaxf(m0, sacc[mt][nt][e]);
            if (L >= 16 || ((g + 8) / L == key / L)) m1 = fmaxf(m1, sacc[mt][nt][2 + e]);
          }
        m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
        m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 2));
        m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
        m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 2));
        const float b0 = -m0 * sc, b1 = -m1 * sc;
#pragma unroll
        for (int nt = 0; nt < C::KEYS / 8; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int key = nt * 8 + 2 * t + e;
            sacc[mt][nt][e] = (L >= 16 || (g / L == key / L)) ? ex2(fmaf(sacc[mt][nt][e], sc, b0)) : 0.f;
            sacc[mt][nt][2 + e] =
                (L >= 16 || ((g + 8) / L == key / L)) ? ex2(fmaf(sacc[mt][nt][2 + e], sc, b1)) : 0.f;
          }
        float l0 = 0.f, l1 = 0.f;
#pragma unroll
        for (int kb = 0; kb < C::KEYS / 16; ++kb) {
          pa[mt][kb][0] = pack_f16x2(sacc[mt][2 * kb][0], sacc[mt][2 * kb][1]);
          pa[mt][kb][1] = pack_f16x2(sacc[mt][2 * kb][2], sacc[mt][2 * kb][3]);
          pa[mt][kb][2] = pack_f16x2(sacc[mt][2 * kb + 1][0], sacc[mt][2 * kb + 1][1]);
          pa[mt][kb][3] = pack_f16x2(sacc[mt][2 * kb + 1][2], sacc[mt][2 * kb + 1][3]);
          float2 f;
          f = __half22float2(*reinterpret_cast<const __half2*>(&pa[mt][kb][0])); l0 += f.x + f.y;
          f = __half22float2(*reinterpret_cast<const __half2*>(&pa[mt][kb][2])); l0 += f.x + f.y;
          f = __half22float2(*reinterpret_cast<const __half2*>(&pa[mt][kb][1])); l1 += f.x + f.y;
          f = __half22float2(*reinterpret_cast<const __half2*>(&pa[mt][kb][3])); l1 += f.x + f.y;
        }
        l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
        l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
        inv[mt][0] = 1.f / l0;
        inv[mt][1] = 1.f / l1;
      }
      // ---- O = P X (B fragments of 16 keys x 16 columns by ldmatrix.trans)
      float oacc[C::MT][8][4];
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) oacc[mt][nt][0] = oacc[mt][nt][1] = oacc[mt][nt][2] = oacc[mt][nt][3] = 0.f;
#pragma unroll
      for (int kb = 0; kb < C::KEYS / 16; ++kb)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          uint32_t vb[4];
          const uint32_t R = u * C::U + kb * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
          ldsm_x4_t(vb, xin + in_off(R, jj * 2 + (lane >> 4)));
#pragma unroll
          for (int i = 0; i < 4; ++i) vb[i] = bf16x2_to_f16x2(vb[i]);
#pragma unroll
          for (int mt = 0; mt < C::MT; ++mt) {
            mma16816(oacc[mt][2 * jj], pa[mt][kb], vb[0], vb[1]);
            mma16816(oacc[mt][2 * jj + 1], pa[mt][kb], vb[2], vb[3]);
          }
        }
      // ---- X_t = x + O (x = the A fragments: n-tile nt <-> k-step nt / 2, half nt & 1),
      // fp16, stmatrix into the staging tile of the row's destination rank
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt) {
        uint32_t w[8][2];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          const uint32_t r0 = xa[mt][nt >> 1][(nt & 1) * 2], r1 = xa[mt][nt >> 1][(nt & 1) * 2 + 1];
          w[nt][0] = pack_f16x2(fmaf(oacc[mt][nt][0], inv[mt][0], __uint_as_float(r0 << 16)),
                                fmaf(oacc[mt][nt][1], inv[mt][0], __uint_as_float(r0 & 0xffff0000u)));
          w[nt][1] = pack_f16x2(fmaf(oacc[mt][nt][2], inv[mt][1], __uint_as_float(r1 << 16)),
                                fmaf(oacc[mt][nt][3], inv[mt][1], __uint_as_float(r1 & 0xffff0000u)));
          nf |= f16x2_nonfinite_bits(w[nt][0]) | f16x2_nonfinite_bits(w[nt][1]);
        }
        // staging row of this lane's stmatrix address: tile row R = (gi, l) ->
        // destination r = l / Kc, row gi * Kc + l % Kc of its sub-tile (each sub-tile
        // G * Kc rows, a multiple of 8, so every sub-tile base is 1024-byte aligned)
        const uint32_t R = u * C::U + mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        if constexpr (BULK) {  // same frame-major layout as the input; frame l goes to rank l / Kc
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            stsm_x4(xout + in_off(R, jj * 2 + (lane >> 4)), w[2 * jj][0], w[2 * jj][1], w[2 * jj + 1][0],
                    w[2 * jj + 1][1]);
        } else {
          const uint32_t gi = R / L, l = R % L;
          const uint32_t r = l / Kc, Rs = gi * Kc + l % Kc;
          const uint32_t sub = xout + r * (uint32_t)(C::G * Kc * 128);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            stsm_x4(sub + swz(Rs, jj * 2 + (lane >> 4)), w[2 * jj][0], w[2 * jj][1], w[2 * jj + 1][0],
                    w[2 * jj + 1][1]);
        }
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      if constexpr (BULK) {
        // frame l's G rows are contiguous in X_t (and in rank l / Kc's frame shard)
        const long long g0 = (long long)tile * C::G;
        for (int l = 0; l < L; ++l) {
          __half* dst = P == 1 ? static_cast<__half*>(p.o) + l * p.osL + g0 * 64
                               : static_cast<__half*>(p.peer_out[l / Kc]) + (l % Kc) * p.osL +
                                     ((long long)p.b_off * p.A + g0) * 64;
          bulk_store(dst, xout + l * C::FS, gv * 128u);
        }
      } else {
        const int ca = (tile % p.tiles_a) * Ab, cb = (tile / p.tiles_a) * Bb;
        if (P == 1) {
          tma_store_4d(&to, out_buf + ob * C::STAGE, 0, 0, ca, cb);
        } else {
          for (int r = 0; r < P; ++r)
            tma_store_4d(&pm.m[r], out_buf + ob * C::STAGE + r * (C::G * Kc * 128), 0, 0, ca, cb);
        }
      }
      bulk_commit();
      const int next = tile + C::NS * gridDim.x;
      if (next < ntiles) issue_load(next, s);
    }
  }
  if (tid == 0) bulk_wait0();
  report_nonfinite(p, nf);
}

}  // namespace tsf
