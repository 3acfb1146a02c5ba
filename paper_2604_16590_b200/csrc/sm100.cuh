// sm_100a primitives: mbarrier, TMA (cp.async.bulk.tensor), tcgen05 (MMA, TMEM
// alloc/ld/st, commit), UMMA shared-memory and instruction descriptors.
//
// Only inline PTX; no CUTLASS/CuTe.  Descriptor bit layouts follow the PTX ISA
// "tcgen05 matrix descriptors" (shared memory descriptor: start>>4 in [0,14),
// LBO>>4 in [16,30), SBO>>4 in [32,46), version=1 at bit 46, swizzle mode in
// [61,64)) and the instruction descriptor for kind::f16 (c_format [4,6),
// a_format [7,10), b_format [10,13), a_major bit 15, b_major bit 16,
// N>>3 in [17,23), M>>4 in [24,29)).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

#define TSF_DEV __device__ __forceinline__

namespace tsf {

// ----------------------------------------------------------------------------
// generic helpers
// ----------------------------------------------------------------------------
TSF_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
TSF_DEV uint32_t warp_id() { return threadIdx.x >> 5; }
TSF_DEV uint32_t lane_id() { return threadIdx.x & 31; }

TSF_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

TSF_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 3-input max (FMNMX3, sm_100+)
TSF_DEV float max3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// 2^x on a packed fp16 pair (one MUFU op for two values)
TSF_DEV uint32_t ex2_f16x2(uint32_t x) {
  uint32_t y;
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

// Packed fp32x2 FMA (FFMA2, sm_100+): (x0, x1) = (a0*b0 + c0, a1*b1 + c1)
TSF_DEV void ffma2(float& x0, float& x1, float a0, float a1, float b0, float b1, float c0, float c1) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.ftz.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(x0), "=f"(x1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}

// Packed fp32x2 add (FADD2): (a0, a1) += (b0, b1)
TSF_DEV void add2(float& a0, float& a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb;\n\t"
      "mov.b64 ra, {%0, %1};\n\tmov.b64 rb, {%2, %3};\n\t"
      "add.rn.ftz.f32x2 ra, ra, rb;\n\tmov.b64 {%0, %1}, ra;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(b0), "f"(b1));
}

// 2^x for a pair on the FMA/ALU pipes (no MUFU), x <= 0: Cody-Waite split
// x = i + f, f in [0, 1), 2^f by a degree-3 polynomial with p(0) = 1 (minimax
// in relative error, max 8.6e-5: below the 2^-9 / 2^-12 rounding that P gets
// as bf16 / fp16), 2^i added into the exponent field.  Inputs are clamped at
// -126 (their weight is < 2^-126 of the row max).
TSF_DEV void ex2_poly2(float& y0, float& y1, float x0, float x1) {
  // p(f) = 1 + c1 f + c2 f^2 + c3 f^3; c1 = 0.69511634 (0x3F31F325),
  // c2 = 0.22764700 (0x3E691C4C), c3 = 0.07706520 (0x3D9DD45C): Lawson
  // iteration for the minimax relative error (tools/fit_exp2.py).
  asm("{\n\t.reg .b64 rx, rr, rb, rf, rp, c1, c2, c3, one;\n\t"
      ".reg .f32 a0, a1, b0, b1;\n\t.reg .b32 i0, i1, q0, q1;\n\t"
      "max.ftz.f32 a0, %2, 0fC2FC0000;\n\tmax.ftz.f32 a1, %3, 0fC2FC0000;\n\t"
      "mov.b64 rx, {a0, a1};\n\t"
      "mov.b64 rb, {0f4B400000, 0f4B400000};\n\t"
      "add.rm.ftz.f32x2 rr, rx, rb;\n\t"          // floor(x) in the low mantissa bits
      "sub.rn.ftz.f32x2 rf, rr, rb;\n\t"
      "sub.rn.ftz.f32x2 rf, rx, rf;\n\t"          // f = x - floor(x) in [0, 1)
      "mov.b64 c3, {0f3D9DD45C, 0f3D9DD45C};\n\t"
      "mov.b64 c2, {0f3E691C4C, 0f3E691C4C};\n\t"
      "mov.b64 c1, {0f3F31F325, 0f3F31F325};\n\t"
      "mov.b64 one, {0f3F800000, 0f3F800000};\n\t"
      "fma.rn.ftz.f32x2 rp, rf, c3, c2;\n\t"
      "fma.rn.ftz.f32x2 rp, rp, rf, c1;\n\t"
      "fma.rn.ftz.f32x2 rp, rp, rf, one;\n\t"
      "mov.b64 {i0, i1}, rr;\n\tmov.b64 {q0, q1}, rp;\n\t"
      "shl.b32 i0, i0, 23;\n\tshl.b32 i1, i1, 23;\n\t"
      "add.s32 q0, q0, i0;\n\tadd.s32 q1, q1, i1;\n\t"
      "mov.b32 %0, q0;\n\tmov.b32 %1, q1;\n\t}"
      : "=f"(y0), "=f"(y1)
      : "f"(x0), "f"(x1));
}

template <uint32_t R>
TSF_DEV void reg_alloc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(R)); }
template <uint32_t R>
TSF_DEV void reg_dealloc() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(R)); }

TSF_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// Register fence: the value is "redefined" by a volatile asm, so arithmetic
// that consumes it cannot be scheduled above earlier volatile asm (barriers).
TSF_DEV float reg_fence(float x) {
  asm volatile("" : "+f"(x));
  return x;
}
TSF_DEV void named_bar_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ----------------------------------------------------------------------------
// mbarrier
// ----------------------------------------------------------------------------
TSF_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
TSF_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
TSF_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
TSF_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// Wait until the phase with the given parity has completed.
TSF_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TSF_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TSF_WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Non-blocking test: has the phase with the given parity completed?
TSF_DEV bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Producer-side wait: try_wait with a suspend-time hint, so a waiting TMA/MMA
// warp sleeps until the phase completes instead of spinning on issue slots
// the softmax warps of its sub-partition need.
TSF_DEV void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TSF_WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
      "@!p bra TSF_WAITS_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ----------------------------------------------------------------------------
// TMA
// ----------------------------------------------------------------------------
TSF_DEV void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
TSF_DEV void tma_load_4d(void* smem_dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                         int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

TSF_DEV void tma_load_2d(void* smem_dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// shared -> global tensor store (bulk group), and its completion waits
TSF_DEV void tma_store_4d(const CUtensorMap* m, const void* smem_src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
TSF_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
TSF_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
TSF_DEV void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
TSF_DEV void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
TSF_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ----------------------------------------------------------------------------
// tcgen05: TMEM allocation
// ----------------------------------------------------------------------------
template <uint32_t NCOLS>
TSF_DEV void tmem_alloc(uint32_t* smem_holder) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_holder)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
TSF_DEV void tmem_dealloc(uint32_t taddr) {  // whole warp (the allocating one)
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}
TSF_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
TSF_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// ----------------------------------------------------------------------------
// tcgen05: MMA (kind::f16, bf16 x bf16 -> fp32), one issuing thread
// ----------------------------------------------------------------------------
// D[tmem] (+)= A[smem] * B[smem]
TSF_DEV void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]
TSF_DEV void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive (once) on an mbarrier when all prior tcgen05 async ops of this thread complete.
TSF_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Instruction descriptor, kind::f16: A/B both bf16 (f16 = false) or both fp16
// (f16 = true), fp32 D, M x N, majors (0 = K-major, 1 = MN-major).
__host__ __device__ constexpr uint32_t make_idesc(uint32_t M, uint32_t N, uint32_t a_major, uint32_t b_major,
                                                  bool f16) {
  return (1u << 4)                          // D format F32
         | ((f16 ? 0u : 1u) << 7)           // A format F16 / BF16
         | ((f16 ? 0u : 1u) << 10)          // B format F16 / BF16
         | (a_major << 15) | (b_major << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// Swizzle modes (descriptor bits 61-63)
enum : uint32_t { SWZ_NONE = 0, SWZ_128B = 2, SWZ_64B = 4, SWZ_32B = 6 };

// Shared memory matrix descriptor.
TSF_DEV uint64_t make_sdesc(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t swz) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  d |= (uint64_t)swz << 61;
  return d;
}

// ----------------------------------------------------------------------------
// tcgen05: TMEM <-> registers.  32x32b shape: warp w (w%4 = quadrant) reads
// lanes [32*(w%4), 32*(w%4)+32), thread i gets lane 32*(w%4)+i, N columns.
// ----------------------------------------------------------------------------
TSF_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
TSF_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

#define TSF_R8(b) "=r"(r[b + 0]), "=r"(r[b + 1]), "=r"(r[b + 2]), "=r"(r[b + 3]), \
                  "=r"(r[b + 4]), "=r"(r[b + 5]), "=r"(r[b + 6]), "=r"(r[b + 7])
#define TSF_W8(b) "r"(r[b + 0]), "r"(r[b + 1]), "r"(r[b + 2]), "r"(r[b + 3]), \
                  "r"(r[b + 4]), "r"(r[b + 5]), "r"(r[b + 6]), "r"(r[b + 7])

TSF_DEV void tmem_ld_x8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : TSF_R8(0)
               : "r"(taddr));
}
TSF_DEV void tmem_ld_x16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : TSF_R8(0), TSF_R8(8)
      : "r"(taddr));
}
TSF_DEV void tmem_ld_x32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : TSF_R8(0), TSF_R8(8), TSF_R8(16), TSF_R8(24)
      : "r"(taddr));
}
TSF_DEV void tmem_st_x8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), TSF_W8(0)
               : "memory");
}
TSF_DEV void tmem_st_x16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      TSF_W8(0), TSF_W8(8)
      : "memory");
}
TSF_DEV void tmem_st_x32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      TSF_W8(0), TSF_W8(8), TSF_W8(16), TSF_W8(24)
      : "memory");
}
#undef TSF_R8
#undef TSF_W8

}  // namespace tsf
