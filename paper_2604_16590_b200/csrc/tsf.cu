// libtsf.so: C ABI (include/tsf.h) over the sm_100a kernels.
//
// Host side only: validation, TMA tensor maps, kernel selection and launch,
// workspace, NCCL all-to-all for the distributed block, stage timing.
#include "../../include/tsf.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "attn_flash.cuh"
#include "attn_packed.cuh"
#include "attn_stream.cuh"
#include "attn_smallt.cuh"
#include "attn_flash3.cuh"
#include "gemm.cuh"
#include "attn_bwd.cuh"
#include "layout.cuh"

using namespace tsf;

struct StageRec {
  int stage;
  cudaEvent_t e0, e1;
};

struct tsf_handle {
  int K = 0, N = 0, H = 0, d = 0;
  int rank = 0, world = 1;
  int device = 0, num_sms = 148;
  ncclComm_t comm = nullptr;
  // workspace (device)
  __half* xt = nullptr;    // X_t = x + T(x) in fp16, [K, N/P, H, d]
  __half* rxt = nullptr;   // dist: all-to-all receive [P][K/P][N/P][H][d] (also reshard scratch)
  __half* uxt = nullptr;   // dist: unpacked frame shard [K/P][N][H][d]
  __nv_bfloat16* xdev = nullptr;                 // host API staging, slot 0
  float* ydev = nullptr;
  __nv_bfloat16* xdev2 = nullptr;                // slot 1 (tsf_spacetime_block_host_batch, n >= 2)
  float* ydev2 = nullptr;
  std::string err;
  int launches = 0;
  bool timing = false;
  std::vector<StageRec> recs;
  std::vector<cudaEvent_t> event_pool;
  unsigned long long* trace = nullptr;  // TSF_TRACE builds only
  // distributed block: X_t is exchanged in nchunk head chunks on comm_stream
  // while the spatial stage of earlier chunks runs (X_t layout [c][K][N/P][H/c][d])
  int nchunk = 1;
  cudaStream_t comm_stream = nullptr;
  std::vector<cudaEvent_t> ev_t, ev_a;
  // fused exchange: every rank's frame-shard X_t buffers mapped here through
  // CUDA IPC; the temporal kernel stores X_t rows straight into them.  Two
  // buffers used on alternate calls (ubuf[0] = uxt): a rank's next temporal
  // stage may write a peer's buffer while that peer's spatial stage still
  // reads the other one; the all-reduce of the call in between orders reuse.
  __half* ubuf[2] = {};
  void* peer_buf[2][MAX_PEERS] = {};
  int fparity = 0;
  int fchunks = 1;                       // head chunks of the fused pipeline (TSF_FUSED_CHUNKS)
  std::vector<cudaEvent_t> ev_f;         // [fchunks + 1]
  bool fused = false;
  int* d_flag = nullptr;        // 1-int NCCL all-reduce = cross-rank barrier
  // peer-memory barrier of the fused exchange (TSF_PEER_BARRIER, default on):
  // a 1 KB flag area after each rank's ubuf[0] (IPC-mapped with it); rank r's
  // slot s holds the epoch rank s last announced to r
  unsigned int* peer_flags[MAX_PEERS] = {};
  unsigned int bar_epoch = 0;
  bool peer_barrier = false;
  PeerMaps pm{};                // per-destination output maps of the current launch
  bool use_pm = false;
  // host API (single GPU): the spatial stage runs in frame chunks and each
  // chunk's y copy to the host overlaps the next chunk's compute
  cudaStream_t copy_stream = nullptr;     // device -> host
  cudaStream_t h2d_stream = nullptr;      // host -> device
  std::vector<cudaEvent_t> ev_h;         // [HOST_CHUNKS + 1 + 6]: chunk ends, D2H end, per slot: x in, x used, y out
  // small device scratch allocated before the (collective) communicator init:
  // [0] 1-int all-reduce barrier, [16] agreement flag, [256..] IPC handle all-gather
  char* scratch = nullptr;
  bool comm_dead = false;                // aborted by tsf_sync's timeout
  // non-finite X_t flag (host-mapped, written by the temporal epilogue)
  volatile unsigned int* nf_host = nullptr;
  unsigned int* nf_dev = nullptr;
  // one-GPU simulation of `world` ranks (tsf_create_sim): xt / rxt / uxt hold
  // every virtual rank's buffer back to back; sim_mode 1 = NCCL byte plan with
  // device copies in place of send/recv, 2 = fused scatter
  bool sim = false;
  // full-block activation workspace (tsf_full_block), allocated on first use
  void* fb = nullptr;
  size_t fb_bytes = 0;
  // backward workspace (tsf_*_bwd), allocated on first use
  void* bw = nullptr;
  size_t bw_bytes = 0;
  // backward recompute: row statistics requested from the next flash forward
  float* st_lse = nullptr;
  float* st_drow = nullptr;
  const void* st_dO = nullptr;
  int st_pitch = 0;
};
constexpr int HOST_CHUNKS = 4;

// Output routing of the distributed temporal stage (run_attention).
struct DistOut {
  int P, Kc, rank, Nl;
  void* const* peers;   // every rank's frame-shard buffer (this call's parity, head-chunk offset applied)
};

static thread_local std::string g_create_err;
extern "C" void tsf_destroy(tsf_handle* h);
extern "C" tsf_status tsf_sync(tsf_handle* h, void* stream, int timeout_ms);

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
static tsf_status fail(tsf_handle* h, tsf_status s, const std::string& msg) {
  if (h) h->err = msg;
  else g_create_err = msg;
  return s;
}
#define TSF_CUDA(h, call)                                                                          \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      return fail(h, TSF_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));          \
  } while (0)
#define TSF_NCCL(h, call)                                                                          \
  do {                                                                                             \
    ncclResult_t r_ = (call);                                                                      \
    if (r_ != ncclSuccess)                                                                         \
      return fail(h, TSF_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_));          \
  } while (0)

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

// A sequence view of a [*, *, H, d] bf16 tensor (see attn_common.cuh).
struct View {
  int L, A, B;
  long long sL, sA, sB;  // element strides
};

static View temporal_view(int K, int Nl, int H, int d) {  // groups (h, n), axis t
  return View{K, H, Nl, (long long)Nl * H * d, (long long)d, (long long)H * d};
}
static View spatial_view(int Kl, int N, int H, int d) {  // groups (h, t), axis n
  return View{N, H, Kl, (long long)H * d, (long long)d, (long long)N * H * d};
}

// 4-D tensor map (d, L, A, B) with box (CH, boxL, boxA, boxB).
static tsf_status make_map(tsf_handle* h, CUtensorMap* m, const void* base, int d, const View& v, int boxL, int boxA,
                           int boxB, bool f16) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return fail(h, TSF_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  const int swb = (2 * d < 128) ? 2 * d : 128;
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)v.L, (cuuint64_t)v.A, (cuuint64_t)v.B};
  cuuint64_t strides[3] = {(cuuint64_t)v.sL * 2, (cuuint64_t)v.sA * 2, (cuuint64_t)v.sB * 2};
  cuuint32_t box[4] = {(cuuint32_t)(swb / 2), (cuuint32_t)boxL, (cuuint32_t)boxA, (cuuint32_t)boxB};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[256];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d): dims %llu %llu %llu %llu box %u %u %u %u", (int)r,
             (unsigned long long)dims[0], (unsigned long long)dims[1], (unsigned long long)dims[2],
             (unsigned long long)dims[3], box[0], box[1], box[2], box[3]);
    return fail(h, TSF_ERR_CUDA, buf);
  }
  return TSF_OK;
}

// ---------------------------------------------------------------------------
// stage timing
// ---------------------------------------------------------------------------
static cudaEvent_t pool_event(tsf_handle* h) {
  if (!h->event_pool.empty()) {
    cudaEvent_t e = h->event_pool.back();
    h->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
// NVTX range per stage (host-side enqueue span; a no-op unless a tool such as
// nsys or ncu is attached) plus, with tsf_set_timing, CUDA events on the stream.
static const char* const kStageName[] = {"tsf.temporal", "tsf.spatial", "tsf.exchange", "tsf.copy",
                                         "tsf.transpose", "tsf.joint", "tsf.storm", "tsf.gemm_ln", "tsf.backward"};
struct StageTimer {
  tsf_handle* h;
  cudaStream_t s;
  int stage;
  cudaEvent_t e0 = nullptr;
  bool open = true;
  StageTimer(tsf_handle* h_, cudaStream_t s_, int st) : h(h_), s(s_), stage(st) {
    nvtxRangePushA(kStageName[st]);
    if (h->timing) {
      e0 = pool_event(h);
      cudaEventRecord(e0, s);
    }
  }
  void done() {
    if (open) {
      nvtxRangePop();
      open = false;
    }
    if (e0) {
      cudaEvent_t e1 = pool_event(h);
      cudaEventRecord(e1, s);
      h->recs.push_back({stage, e0, e1});
      e0 = nullptr;
    }
  }
  ~StageTimer() {
    if (open) nvtxRangePop();
  }
};

// ---------------------------------------------------------------------------
// kernel launch
// ---------------------------------------------------------------------------
template <typename KernelT, typename... Maps>
static tsf_status launch(tsf_handle* h, KernelT kern, int grid, int threads, int smem, cudaStream_t st,
                         const AttnParams& p, const Maps&... maps) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return fail(h, TSF_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  kern<<<grid, threads, smem, st>>>(maps..., p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(h, TSF_ERR_CUDA, std::string("attention launch: ") + cudaGetErrorString(e));
  h->launches++;
  return TSF_OK;
}

template <int D, int WIN, int EPI, bool SHARED>
static tsf_status launch_packed_t(tsf_handle* h, cudaStream_t st, const CUtensorMap& mq, const CUtensorMap& mk,
                                  const CUtensorMap& mv, const CUtensorMap& mo, const AttnParams& p) {
  constexpr int NST = SHARED ? 4 : 2;
  using C = PackedCfg<D, WIN, EPI, SHARED, NST>;
  const int smem = h->use_pm ? C::SMEM_DIST : C::SMEM;
  const int per_sm = (C::TCOLS == 256 && 2 * smem <= 227 * 1024) ? 2 : 1;
  int grid = h->num_sms * per_sm;
  if (grid > p.num_tiles) grid = p.num_tiles;
  return launch(h, attn_packed_kernel<D, WIN, EPI, SHARED, NST>, grid, C::THREADS, smem, st, p, mq, mk, mv, mo,
                h->pm);
}

// Flash kernel K/V tile rows (= score tile columns): d = 64 uses 96 (three
// rotating score buffers fit TMEM next to O + l); otherwise 128.  TSF_SUB
// (64 | 96 | 128) overrides for d = 64 experiments.
static int flash_sub(int d) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("TSF_SUB");
    env = e ? atoi(e) : -1;
  }
  if (d != 64) return 128;
  if (env == 64 || env == 96 || env == 128) return env;
  return 96;
}

// Softmax warps per score row in the d = 64 flash kernel (1 | 2): TSF_SPLIT
// overrides the default for experiments.
static int flash_split() {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("TSF_SPLIT");
    env = e ? atoi(e) : -1;
  }
  return env == 2 ? 2 : 1;  // 2: measured slower at C2 (the row-max exchange serialises the pair)
}

template <int D, int EPI, int EMU, int SUB>
static tsf_status launch_flash_sub(tsf_handle* h, cudaStream_t st, const CUtensorMap& mq, const CUtensorMap& mk,
                                   const CUtensorMap& mv, const AttnParams& p) {
  constexpr bool SH = EpiTraits<EPI>::SHARED;
  constexpr int NST = SH ? ((D == 128) ? 4 : 8) : ((D == 128) ? 2 : 4);
  const long long items = (long long)p.n_qpairs * p.A * p.B;
  if (items > 0x7fffffffLL) return fail(h, TSF_ERR_CONFIG, "too many work items");
  AttnParams pp = p;
  pp.num_items = (int)items;
  static int flags_env = -1;
  if (flags_env < 0) {
    const char* g = getenv("TSF_FLASH_FLAGS");  // FLASH_PINGPONG (off: measured slower with rotating buffers)
    flags_env = g ? atoi(g) : 0;
  }
  pp.flags = flags_env;
  // persistent: one CTA per SM, each loops over work items
  const long long grid = items < h->num_sms ? items : h->num_sms;
  if constexpr (FlashCfg<D, EPI, NST, SUB>::SEP && FlashCfg<D, EPI, NST, SUB>::ONES) {
    if (flash_split() == 2) {
      using C = FlashCfg<D, EPI, NST, SUB, 2>;
      return launch(h, attn_flash_kernel<D, EPI, NST, EMU, SUB, 2>, (int)grid, C::THREADS, C::SMEM, st, pp, mq, mk,
                    mv);
    }
  }
  using C = FlashCfg<D, EPI, NST, SUB, 1>;
  return launch(h, attn_flash_kernel<D, EPI, NST, EMU, SUB, 1>, (int)grid, C::THREADS, C::SMEM, st, pp, mq, mk, mv);
}

template <int D, int EPI, int EMU>
static tsf_status launch_flash_emu(tsf_handle* h, cudaStream_t st, const CUtensorMap& mq, const CUtensorMap& mk,
                                   const CUtensorMap& mv, const AttnParams& p) {
  if constexpr (D == 64) {
    switch (flash_sub(D)) {
      case 64: return launch_flash_sub<D, EPI, EMU, 64>(h, st, mq, mk, mv, p);
      case 128: return launch_flash_sub<D, EPI, EMU, 128>(h, st, mq, mk, mv, p);
      default: return launch_flash_sub<D, EPI, EMU, 96>(h, st, mq, mk, mv, p);
    }
  }
  return launch_flash_sub<D, EPI, EMU, 128>(h, st, mq, mk, mv, p);
}

// exp2 emulation share (of 16) for the d = 64 flash kernel: TSF_EMU overrides
// the default for experiments.  (ex2.approx.f16x2 lowers to two scalar
// MUFU.EX2.F16 + PRMT on sm_100a, so fp16 P gains nothing from it; both
// precisions use fp32 MUFU ex2 with part of the exps on the FMA pipe.)
static int emu_setting(int d, int epi) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("TSF_EMU");
    env = e ? atoi(e) : -1;
  }
  if (d != 64) return 0;
  if (env >= 0) return env;
  return epi == EPI_OUT16 ? 6 : 4;
}

template <int D, int EPI>
static tsf_status launch_flash_t(tsf_handle* h, cudaStream_t st, const CUtensorMap& mq, const CUtensorMap& mk,
                                 const CUtensorMap& mv, const AttnParams& p) {
  if constexpr (D == 64) {
    switch (emu_setting(D, EPI)) {
      case 4: return launch_flash_emu<D, EPI, 4>(h, st, mq, mk, mv, p);
      case 6: return launch_flash_emu<D, EPI, 6>(h, st, mq, mk, mv, p);
      case 8: return launch_flash_emu<D, EPI, 8>(h, st, mq, mk, mv, p);
      default: break;
    }
  }
  return launch_flash_emu<D, EPI, 0>(h, st, mq, mk, mv, p);
}

// Streaming block temporal stage (attn_stream.cuh): d in {32, 64}, window 32 / 64.
// TSF_STREAM=0 selects the older one-slot packed kernel (A/B measurements).
static bool use_stream(int d, int win) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("TSF_STREAM");
    env = e ? atoi(e) : 1;
  }
  return env != 0 && (d == 32 || d == 64) && (win == 32 || win == 64);
}

// Short-window temporal kernel (attn_smallt.cuh): d = 64, K in {4, 8, 16, 32}.
// TSF_SMALLT=0 selects the tcgen05 stream kernel instead (A/B measurements).
static bool use_smallt(int d, int L) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("TSF_SMALLT");
    env = e ? atoi(e) : 1;
  }
  return env != 0 && d == 64 && (L == 4 || L == 8 || L == 16 || L == 32);
}

// TMEM slots of the stream kernel: TSF_STREAM_SLOTS = 2 | 4.  Four slots (S, P, O
// aliased in 128 columns) measured no faster at C2 (34.7 vs 34.3 us, profiles/r07/traces,
// trace 1831 vs 1773 cycles per tile): the stage is not limited by tiles in flight.
static int stream_slots() {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("TSF_STREAM_SLOTS");
    env = e ? atoi(e) : 2;
  }
  return env == 4 ? 4 : 2;
}

template <int D, int WIN, int NS>
static tsf_status launch_stream_ns(tsf_handle* h, cudaStream_t st, const CUtensorMap& mx, const CUtensorMap& mo,
                                   const AttnParams& p) {
  constexpr int NST = 8;
  using C = StreamCfg<D, WIN, NST, NS>;
  int grid = h->num_sms;
  if (grid > p.num_tiles) grid = p.num_tiles;
  if constexpr (WIN == 32) {  // compact softmax for the short windows (C1 K = 4, C2 K = 8, C2 at P = 2 K = 16)
    switch (p.L) {
      case 4: return launch(h, attn_stream_kernel<D, WIN, NST, 4, NS>, grid, C::THREADS, C::SMEM, st, p, mx, mo, h->pm);
      case 8: return launch(h, attn_stream_kernel<D, WIN, NST, 8, NS>, grid, C::THREADS, C::SMEM, st, p, mx, mo, h->pm);
      case 16: return launch(h, attn_stream_kernel<D, WIN, NST, 16, NS>, grid, C::THREADS, C::SMEM, st, p, mx, mo, h->pm);
      default: break;
    }
  }
  return launch(h, attn_stream_kernel<D, WIN, NST, 0, NS>, grid, C::THREADS, C::SMEM, st, p, mx, mo, h->pm);
}

template <int D, int WIN>
static tsf_status launch_stream_t(tsf_handle* h, cudaStream_t st, const CUtensorMap& mx, const CUtensorMap& mo,
                                  const AttnParams& p) {
  if constexpr (D <= 64 && WIN <= 64) {
    if constexpr (D == 64) {  // the four-slot A/B variant is built for d = 64 only
      if (stream_slots() == 4) return launch_stream_ns<D, WIN, 4>(h, st, mx, mo, p);
    }
    return launch_stream_ns<D, WIN, 2>(h, st, mx, mo, p);
  }
  return fail(h, TSF_ERR_UNSUPPORTED, "stream kernel shape");
}

template <int D, int EPI, bool SHARED>
static tsf_status dispatch_packed_win(tsf_handle* h, int win, cudaStream_t st, const CUtensorMap& mq,
                                      const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mo,
                                      const AttnParams& p) {
  if constexpr (EPI == EPI_BLOCK_T && D <= 64) {
    if (use_stream(D, win)) {
      if (win == 32) return launch_stream_t<D, 32>(h, st, mq, mo, p);
      return launch_stream_t<D, 64>(h, st, mq, mo, p);
    }
  }
  switch (win) {
    case 32: return launch_packed_t<D, 32, EPI, SHARED>(h, st, mq, mk, mv, mo, p);
    case 64: return launch_packed_t<D, 64, EPI, SHARED>(h, st, mq, mk, mv, mo, p);
    default: return launch_packed_t<D, 128, EPI, SHARED>(h, st, mq, mk, mv, mo, p);
  }
}

template <int D>
static tsf_status dispatch_d(tsf_handle* h, bool packed, int win, int epi, cudaStream_t st, const CUtensorMap& mq,
                             const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mo,
                             const AttnParams& p) {
  if (packed) {
    switch (epi) {
      case EPI_OUT16: return dispatch_packed_win<D, EPI_OUT16, false>(h, win, st, mq, mk, mv, mo, p);
      case EPI_BLOCK_T: return dispatch_packed_win<D, EPI_BLOCK_T, true>(h, win, st, mq, mk, mv, mo, p);
      default: return dispatch_packed_win<D, EPI_BLOCK_S, true>(h, win, st, mq, mk, mv, mo, p);
    }
  }
  switch (epi) {
    case EPI_OUT16: return launch_flash_t<D, EPI_OUT16>(h, st, mq, mk, mv, p);
    case EPI_BLOCK_T: return launch_flash_t<D, EPI_BLOCK_T>(h, st, mq, mk, mv, p);
    default: return launch_flash_t<D, EPI_BLOCK_S>(h, st, mq, mk, mv, p);
  }
}

// Attention over one view: q/k/v (q == k == v for the block stages).  The
// output (o or y) uses the strides of `ov` (default: the input view's).
// One-query-tile-per-CTA flash kernel, three CTAs per SM (attn_flash3.cuh):
// d = 64, spatial block stage and the standalone calls.  TSF_FLASH3=0 selects
// the two-tile kernel (attn_flash.cuh) for A/B measurements.
static bool use_flash3(int d, int epi) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("TSF_FLASH3");
    env = e ? atoi(e) : 0;
  }
  return env != 0 && d == 64 && (epi == EPI_BLOCK_S || epi == EPI_OUT16);
}
static int flash3_cps() {  // CTAs per SM (TSF_F3CTAS: 3 | 4)
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("TSF_F3CTAS");
    env = e ? atoi(e) : 3;
  }
  return env == 4 ? 4 : 3;
}

template <int EPI, int EMU, int CPS>
static tsf_status launch_flash3_cps(tsf_handle* h, cudaStream_t st, const CUtensorMap& mq, const CUtensorMap& mk,
                                    const CUtensorMap& mv, const AttnParams& p) {
  constexpr bool SH = EpiTraits<EPI>::SHARED;
  constexpr int NST = CPS == 4 ? (SH ? 3 : 2) : (SH ? 6 : 4);
  using C = Flash3Cfg<64, EPI, NST>;
  const long long items = (long long)p.n_qpairs * p.A * p.B;
  if (items > 0x7fffffffLL) return fail(h, TSF_ERR_CONFIG, "too many work items");
  AttnParams pp = p;
  pp.num_items = (int)items;
  const long long cap = (long long)CPS * h->num_sms;
  return launch(h, attn_flash3_kernel<64, EPI, NST, EMU, CPS>, (int)(items < cap ? items : cap), C::THREADS, C::SMEM,
                st, pp, mq, mk, mv);
}

// flash3 is an A/B variant (off by default): one exp split (EMU = 4), 3 or 4 CTAs per SM
template <int EPI>
static tsf_status launch_flash3(tsf_handle* h, cudaStream_t st, const CUtensorMap& mq, const CUtensorMap& mk,
                                const CUtensorMap& mv, const AttnParams& p) {
  if (flash3_cps() == 4) return launch_flash3_cps<EPI, 4, 4>(h, st, mq, mk, mv, p);
  return launch_flash3_cps<EPI, 4, 3>(h, st, mq, mk, mv, p);
}

// Flash kernel with fixed tile / exp settings for the secondary calls: joint
// attention with a block or causal mask (tsf_joint_attn, MASK = 1) and the
// STORM epilogues (tsf_storm_attn), bf16 operands and P.
template <int D, int EPI, int MASK>
static tsf_status launch_flash_fixed(tsf_handle* h, cudaStream_t st, const CUtensorMap& mq, const CUtensorMap& mk,
                                     const CUtensorMap& mv, const AttnParams& p) {
  constexpr int SUB = (D == 64) ? 96 : 128, EMU = (D == 64) ? 6 : 0;
  constexpr bool SH = EpiTraits<EPI>::SHARED;
  constexpr int NST = SH ? ((D == 128) ? 4 : 8) : ((D == 128) ? 2 : 4);
  using C = FlashCfg<D, EPI, NST, SUB, 1>;
  const long long items = (long long)p.n_qpairs * p.A * p.B;
  if (items > 0x7fffffffLL) return fail(h, TSF_ERR_CONFIG, "too many work items");
  AttnParams pp = p;
  pp.num_items = (int)items;
  pp.flags = 0;
  const long long grid = items < h->num_sms ? items : h->num_sms;
  return launch(h, attn_flash_kernel<D, EPI, NST, EMU, SUB, 1, MASK>, (int)grid, C::THREADS, C::SMEM, st, pp, mq,
                mk, mv);
}

template <int D>
static tsf_status launch_flash_special(tsf_handle* h, int epi, int mask, cudaStream_t st, const CUtensorMap& mq,
                                       const CUtensorMap& mk, const CUtensorMap& mv, const AttnParams& p) {
  if (mask) return launch_flash_fixed<D, EPI_OUT16, 1>(h, st, mq, mk, mv, p);
  if (epi == EPI_OUT16) return launch_flash_fixed<D, EPI_OUT16, 0>(h, st, mq, mk, mv, p);
  if (epi == EPI_STORM_X) return launch_flash_fixed<D, EPI_STORM_X, 0>(h, st, mq, mk, mv, p);
  return launch_flash_fixed<D, EPI_STORM_S, 0>(h, st, mq, mk, mv, p);
}

static tsf_status run_attention(tsf_handle* h, const View& v, const void* q, const void* k, const void* vv, int epi,
                                void* o, float* y, cudaStream_t st, const View* ov = nullptr,
                                const DistOut* dist = nullptr, int mask = 0, const View* kvv = nullptr,
                                float gate = 0.f) {
  if (!ov) ov = &v;
  h->use_pm = false;
  const int d = h->d;
  if ((long long)v.A * v.B == 0 || v.L == 0) return TSF_OK;
  AttnParams p{};
  p.L = v.L; p.A = v.A; p.B = v.B;
  p.sL = v.sL; p.sA = v.sA; p.sB = v.sB;
  p.osL = ov->sL; p.osA = ov->sA; p.osB = ov->sB;
  p.P = 1;
  if (dist) {  // EPI_BLOCK_T rows of frame l go to rank l / Kc, frame shard [Kc][N][H][d]
    p.P = dist->P;
    p.Kc = dist->Kc;
    p.b_off = dist->rank * dist->Nl;
    for (int r = 0; r < dist->P; ++r) p.peer_out[r] = dist->peers[r];
    p.osL = (long long)h->N * h->H * h->d;
    p.osA = h->d;
    p.osB = (long long)h->H * h->d;
  }
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d));
  p.o = o;
  p.y = y;
  p.res = q;  // the block's residual input (q = k = v there)
  p.nonfinite = h->nf_dev;
#ifdef TSF_TRACE
  if (!h->trace) {
    cudaMalloc(&h->trace, 32 * TRACE_PER_WARP * sizeof(unsigned long long));
    cudaMemset(h->trace, 0, 32 * TRACE_PER_WARP * sizeof(unsigned long long));
  }
  p.trace = h->trace;
#endif
  const bool f16 = (epi == EPI_BLOCK_S);  // X_t lives in fp16; x (BLOCK_T) arrives bf16
  const bool special = mask != 0 || epi == EPI_STORM_X || epi == EPI_STORM_S ||
                       h->st_lse != nullptr;  // flash kernel, fixed settings
  p.lse = h->st_lse;
  p.drow = h->st_drow;
  p.dO = h->st_dO;
  p.lse_pitch = h->st_pitch;
  const bool packed = v.L <= 128 && !special;
  if (packed && epi == EPI_BLOCK_T && use_smallt(d, v.L) && v.sB == (long long)v.A * v.sA && v.sA == d) {
    // 256-row tiles of G = 256 / L whole groups (Ab heads x Bb tokens), every warp
    // unit (16 or 32 rows) either fully inside the tile or skipped
    const int G = 256 / v.L;
    int Ab = 1;
    for (int a = 1; a <= G && a <= v.A; ++a)
      if (v.A % a == 0) Ab = a;
    int Bb = G / Ab;
    if (Bb > v.B) Bb = v.B;
    const int unit = v.L < 16 ? 16 : v.L;
    if ((Ab * Bb * v.L) % unit == 0) {
      p.Ab = Ab; p.Bb = Bb;
      p.tiles_a = v.A / Ab;
      const long long tiles = (long long)p.tiles_a * ((v.B + Bb - 1) / Bb);
      if (tiles > 0x7fffffffLL) return fail(h, TSF_ERR_CONFIG, "too many tiles");
      p.num_tiles = (int)tiles;
      CUtensorMap mx, mo;
      memset(&mo, 0, sizeof mo);
      tsf_status s;
      if ((s = make_map(h, &mx, q, d, v, v.L, Ab, Bb, false)) != TSF_OK) return s;
      if (dist) {
        for (int r = 0; r < dist->P; ++r) {
          const View pv{dist->Kc, v.A, dist->Nl, p.osL, p.osA, p.osB};
          const void* base = static_cast<const __half*>(dist->peers[r]) + (size_t)dist->rank * dist->Nl * h->H * d;
          if ((s = make_map(h, &h->pm.m[r], base, d, pv, dist->Kc, Ab, Bb, true)) != TSF_OK) return s;
        }
      } else if ((s = make_map(h, &mo, o, d, *ov, v.L, Ab, Bb, true)) != TSF_OK) {
        return s;
      }
      if (getenv("TSF_SMALLT_NOMATH")) p.flags |= SMALLT_NO_MATH;
      int grid = h->num_sms;
      if (grid > p.num_tiles) grid = p.num_tiles;
      static int warps = -1, bulk = -1;
      if (warps < 0) {
        const char* e = getenv("TSF_SMALLT_WARPS");
        warps = (e && atoi(e) == 8) ? 8 : 16;
        e = getenv("TSF_SMALLT_BULK");
        bulk = e ? atoi(e) != 0 : 0;
      }
      // (the output's groups must be contiguous per frame too: X_t [K, N, H, d] or the
      // peers' frame shards)
      const bool use_bulk = bulk && (dist || (ov->sA == d && ov->sB == (long long)v.A * d));
      if (use_bulk) {
        // tiles of G consecutive groups of the frame plane, one 1-D copy per frame
        const long long nt = ((long long)v.A * v.B + G - 1) / G;
        if (nt > 0x7fffffffLL) return fail(h, TSF_ERR_CONFIG, "too many tiles");
        p.num_tiles = (int)nt;
        p.Ab = G; p.Bb = 1;  // (gt = G: every unit of a full tile is valid)
        grid = h->num_sms < p.num_tiles ? h->num_sms : p.num_tiles;
      }
#define TSF_SMALLT_LAUNCH(LL, WW, BB)                                                                        \
  launch(h, attn_smallt_kernel<LL, WW, BB>, grid, SmallTCfg<LL, WW, BB>::THREADS, SmallTCfg<LL, WW, BB>::SMEM, st, p, \
         mx, mo, h->pm)
#define TSF_SMALLT_W(LL, BB) (warps == 8 ? TSF_SMALLT_LAUNCH(LL, 8, BB) : TSF_SMALLT_LAUNCH(LL, 16, BB))
      switch (v.L) {
        case 4: return use_bulk ? TSF_SMALLT_W(4, true) : TSF_SMALLT_W(4, false);
        case 8: return use_bulk ? TSF_SMALLT_W(8, true) : TSF_SMALLT_W(8, false);
        case 16: return use_bulk ? TSF_SMALLT_W(16, true) : TSF_SMALLT_W(16, false);
        default: return use_bulk ? TSF_SMALLT_LAUNCH(32, 8, true) : TSF_SMALLT_LAUNCH(32, 8, false);
      }
#undef TSF_SMALLT_W
#undef TSF_SMALLT_LAUNCH
    }
  }
  p.mask_mode = mask;
  p.mask_n = h->N;
  if (!kvv) kvv = &v;  // keys / values: the query view unless cross-attention
  p.Lk = kvv->L;
  p.gate = gate;
  int win = 128;
  CUtensorMap mq, mk, mv, mo;
  memset(&mo, 0, sizeof mo);
  tsf_status s;
  if (packed) {
    const int G = 128 / v.L;
    int Ab = 1;
    for (int a = 1; a <= G && a <= v.A; ++a)
      if (v.A % a == 0) Ab = a;
    int Bb = G / Ab;
    if (Bb > v.B) Bb = v.B;
    p.Ab = Ab; p.Bb = Bb;
    p.tiles_a = v.A / Ab;
    const long long tiles = (long long)p.tiles_a * ((v.B + Bb - 1) / Bb);
    if (tiles > 0x7fffffffLL) return fail(h, TSF_ERR_CONFIG, "too many tiles");
    p.num_tiles = (int)tiles;
    win = (32 % v.L == 0) ? 32 : (64 % v.L == 0) ? 64 : 128;
    if ((s = make_map(h, &mq, q, d, v, v.L, Ab, Bb, f16)) != TSF_OK) return s;
    if ((s = make_map(h, &mk, k, d, v, v.L, Ab, Bb, f16)) != TSF_OK) return s;
    if ((s = make_map(h, &mv, vv, d, v, v.L, Ab, Bb, f16)) != TSF_OK) return s;
    // output map (16-bit outputs): bf16 for the standalone calls, fp16 X_t for the block
    if (!dist && epi != EPI_BLOCK_S && (s = make_map(h, &mo, o, d, *ov, v.L, Ab, Bb, epi == EPI_BLOCK_T)) != TSF_OK)
      return s;
    if (dist) {
      // one map per destination rank over its frame shard, restricted to this
      // rank's token range: dims (d, Kc, H, N/P), base + rank * (N/P) * H * d
      if ((dist->Kc * Ab * Bb) % 8 != 0 || v.L * Ab * Bb > 128)
        return fail(h, TSF_ERR_UNSUPPORTED, "fused exchange needs (K/P) * groups-per-tile % 8 == 0");
      for (int r = 0; r < dist->P; ++r) {
        const View pv{dist->Kc, v.A, dist->Nl, p.osL, p.osA, p.osB};
        const void* base = static_cast<const __half*>(dist->peers[r]) + (size_t)dist->rank * dist->Nl * h->H * d;
        if ((s = make_map(h, &h->pm.m[r], base, d, pv, dist->Kc, Ab, Bb, true)) != TSF_OK) return s;
      }
      h->use_pm = true;
    }
  } else {
    const bool f3 = !special && use_flash3(d, epi);
    p.n_qpairs = f3 ? (v.L + 127) / 128 : (v.L + 255) / 256;   // flash3: 128-row query tiles
    const int sub = f3 ? 64 : special ? ((d == 64) ? 96 : 128) : flash_sub(d);  // K/V tile rows
    p.nkv = (kvv->L + sub - 1) / sub;
    if ((s = make_map(h, &mq, q, d, v, 128, 1, 1, f16)) != TSF_OK) return s;
    if ((s = make_map(h, &mk, k, d, *kvv, sub, 1, 1, f16)) != TSF_OK) return s;
    if ((s = make_map(h, &mv, vv, d, *kvv, sub, 1, 1, f16)) != TSF_OK) return s;
    if (f3) return epi == EPI_BLOCK_S ? launch_flash3<EPI_BLOCK_S>(h, st, mq, mk, mv, p)
                                      : launch_flash3<EPI_OUT16>(h, st, mq, mk, mv, p);
    if (special) {
      switch (d) {
        case 32: return launch_flash_special<32>(h, epi, mask, st, mq, mk, mv, p);
        case 64: return launch_flash_special<64>(h, epi, mask, st, mq, mk, mv, p);
        default: return launch_flash_special<128>(h, epi, mask, st, mq, mk, mv, p);
      }
    }
  }
  switch (d) {
    case 32: return dispatch_d<32>(h, packed, win, epi, st, mq, mk, mv, mo, p);
    case 64: return dispatch_d<64>(h, packed, win, epi, st, mq, mk, mv, mo, p);
    default: return dispatch_d<128>(h, packed, win, epi, st, mq, mk, mv, mo, p);
  }
}

static int grid_for(tsf_handle* h, long long work_items) {
  long long g = (work_items + 255) / 256;
  const long long cap = (long long)h->num_sms * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// ---------------------------------------------------------------------------
// validation
// ---------------------------------------------------------------------------
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
static bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  const char *x = (const char*)a, *y = (const char*)b;
  return x < y + nb && y < x + na;
}

static tsf_status check_ptrs(tsf_handle* h, std::initializer_list<const void*> ins, const void* out, size_t in_bytes,
                             size_t out_bytes) {
  if (!out || !aligned16(out)) return fail(h, TSF_ERR_CONFIG, "output pointer null or not 16-byte aligned");
  for (const void* p : ins) {
    if (!p || !aligned16(p)) return fail(h, TSF_ERR_CONFIG, "input pointer null or not 16-byte aligned");
    if (overlap(p, in_bytes, out, out_bytes)) return fail(h, TSF_ERR_CONFIG, "output overlaps an input");
  }
  return TSF_OK;
}

static tsf_status check_device(tsf_handle* h, int* dev, int* sms) {
  TSF_CUDA(h, cudaGetDevice(dev));
  cudaDeviceProp prop;
  TSF_CUDA(h, cudaGetDeviceProperties(&prop, *dev));
  if (prop.major != 10 || prop.minor != 0)
    return fail(h, TSF_ERR_UNSUPPORTED, "device is not sm_100 (B200): compute capability " +
                                            std::to_string(prop.major) + "." + std::to_string(prop.minor));
  *sms = prop.multiProcessorCount;
  return TSF_OK;
}

static tsf_status check_shape(int K, int N, int H, int d, int world) {
  if (K < 1 || N < 1 || H < 1) return fail(nullptr, TSF_ERR_CONFIG, "K, N, H must be >= 1");
  if (d != 32 && d != 64 && d != 128) return fail(nullptr, TSF_ERR_UNSUPPORTED, "d must be 32, 64 or 128");
  if (world < 1) return fail(nullptr, TSF_ERR_CONFIG, "world must be >= 1");
  if (K % world || N % world) return fail(nullptr, TSF_ERR_CONFIG, "K and N must be divisible by the world size");
  if ((long long)K * N * H * d >= (1LL << 40)) return fail(nullptr, TSF_ERR_CONFIG, "tensor too large");
  return TSF_OK;
}

// flag area of the peer barrier: 1 KB after a frame-shard buffer of El halves
constexpr size_t FLAG_AREA_BYTES = 1024;
static size_t flag_area_off(size_t El) { return (El * sizeof(__half) + 255) & ~size_t(255); }
static size_t flag_area_halfs(size_t El) { return (flag_area_off(El) + FLAG_AREA_BYTES) / sizeof(__half); }

static tsf_status alloc_workspace(tsf_handle* h) {
  // token-shard elements (times the virtual ranks of a simulated handle)
  const size_t El = (size_t)h->K * (h->N / h->world) * h->H * h->d * (h->sim ? h->world : 1);
  auto a = [&](__half** p, size_t n) -> bool {
    return cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(__half)) == cudaSuccess;
  };
  bool ok = a(&h->xt, El);
  if (ok && h->world > 1) ok = a(&h->rxt, El) && a(&h->uxt, h->sim ? El : flag_area_halfs(El));
  if (ok && h->world > 1 && !h->sim)
    ok = cudaMemset(reinterpret_cast<char*>(h->uxt) + flag_area_off(El), 0, FLAG_AREA_BYTES) == cudaSuccess;
  if (ok && h->world > 1 && !h->sim)
    ok = cudaMalloc(reinterpret_cast<void**>(&h->scratch), 256 + (size_t)h->world * 2 * sizeof(cudaIpcMemHandle_t)) ==
         cudaSuccess;
  if (ok) {
    unsigned int* hp = nullptr;
    // [0] non-finite X_t, [1] peer-barrier timeout
    ok = cudaHostAlloc(reinterpret_cast<void**>(&hp), 2 * sizeof(unsigned int), cudaHostAllocMapped) == cudaSuccess;
    if (ok) {
      hp[0] = hp[1] = 0u;
      h->nf_host = hp;
      ok = cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->nf_dev), hp, 0) == cudaSuccess;
    }
  }
  if (!ok) {
    cudaGetLastError();
    return fail(nullptr, TSF_ERR_NOMEM, "workspace cudaMalloc failed");
  }
  return TSF_OK;
}

static void free_workspace(tsf_handle* h) {
  for (void* p : {(void*)h->xt, (void*)h->rxt, (void*)h->uxt, (void*)h->xdev, (void*)h->ydev, (void*)h->xdev2,
                  (void*)h->ydev2, (void*)h->scratch, h->fb, h->bw})
    if (p) cudaFree(p);
  if (h->nf_host) cudaFreeHost(const_cast<unsigned int*>(h->nf_host));
  h->xt = h->rxt = h->uxt = nullptr;
  h->xdev = h->xdev2 = nullptr;
  h->ydev = h->ydev2 = nullptr;
  h->scratch = nullptr;
  h->nf_host = nullptr;
  h->fb = nullptr;
  h->bw = nullptr;
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

tsf_status tsf_create(int K, int N, int H, int d, tsf_handle** out) {
  if (!out) return fail(nullptr, TSF_ERR_CONFIG, "out is null");
  *out = nullptr;
  tsf_status s = check_shape(K, N, H, d, 1);
  if (s != TSF_OK) return s;
  tsf_handle* h = new tsf_handle();
  h->K = K; h->N = N; h->H = H; h->d = d;
  if ((s = check_device(nullptr, &h->device, &h->num_sms)) != TSF_OK || (s = alloc_workspace(h)) != TSF_OK) {
    free_workspace(h);
    delete h;
    return s;
  }
  *out = h;
  return TSF_OK;
}

tsf_status tsf_get_unique_id(void* id128) {
  if (!id128) return fail(nullptr, TSF_ERR_CONFIG, "id128 is null");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, TSF_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  memcpy(id128, &id, sizeof id);
  return TSF_OK;
}

tsf_status tsf_create_dist(int K, int N, int H, int d, const void* id128, int rank, int world, tsf_handle** out) {
  if (!out || !id128) return fail(nullptr, TSF_ERR_CONFIG, "null argument");
  *out = nullptr;
  tsf_status s = check_shape(K, N, H, d, world);
  if (s != TSF_OK) return s;
  if (rank < 0 || rank >= world) return fail(nullptr, TSF_ERR_CONFIG, "rank out of range");
  tsf_handle* h = new tsf_handle();
  h->K = K; h->N = N; h->H = H; h->d = d;
  h->rank = rank; h->world = world;
  // everything the setup below needs on the device (workspace, the barrier
  // int, the agreement flag, the IPC-handle exchange buffer) is allocated
  // BEFORE the collective communicator init
  if ((s = check_device(nullptr, &h->device, &h->num_sms)) != TSF_OK || (s = alloc_workspace(h)) != TSF_OK) {
    free_workspace(h);
    delete h;
    return s;
  }
  if (world > 1) {
    ncclUniqueId id;
    memcpy(&id, id128, sizeof id);
    ncclResult_t r = ncclCommInitRank(&h->comm, world, id, rank);
    if (r != ncclSuccess) {
      h->comm = nullptr;
      tsf_destroy(h);
      return fail(nullptr, TSF_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    // head chunks of the NCCL fallback path (exchange / spatial overlap):
    // TSF_NCHUNK, default 1 (chunking measured slower at P = 2: NCCL's kernels
    // and the spatial kernel compete for SMs)
    int nc = 1;
    if (const char* e = getenv("TSF_NCHUNK")) nc = atoi(e);
    if (nc < 1) nc = 1;
    while (nc > 1 && H % nc) --nc;
    h->nchunk = nc;
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    if (cudaStreamCreateWithPriority(&h->comm_stream, cudaStreamNonBlocking, hi_prio) != cudaSuccess) {
      tsf_destroy(h);
      return fail(nullptr, TSF_ERR_CUDA, "comm stream creation failed");
    }
    h->ev_t.resize(nc);
    h->ev_a.resize(nc);
    for (int c = 0; c < nc; ++c) {
      cudaEventCreateWithFlags(&h->ev_t[c], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&h->ev_a[c], cudaEventDisableTiming);
    }
    h->d_flag = reinterpret_cast<int*>(h->scratch);
    int* d_ok = reinterpret_cast<int*>(h->scratch + 16);
    char* dh = h->scratch + 256;
    cudaStream_t cs = h->comm_stream;
    // every rank takes part in every collective below, whatever its local
    // outcome, so the sequence of collectives is identical on all ranks
    auto agree = [&](bool local_ok) -> bool {  // all-reduce (min) of the local outcome
      int v = local_ok ? 1 : 0;
      if (cudaMemcpy(d_ok, &v, sizeof v, cudaMemcpyHostToDevice) != cudaSuccess) v = 0;
      if (ncclAllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, h->comm, cs) != ncclSuccess ||
          cudaStreamSynchronize(cs) != cudaSuccess || cudaMemcpy(&v, d_ok, sizeof v, cudaMemcpyDeviceToHost) != cudaSuccess)
        return false;
      return v == 1;
    };
    // fused exchange: all-gather the IPC handles of every rank's two
    // frame-shard X_t buffers and map them (TSF_FUSED_EXCHANGE=0 disables it
    // on every rank: the environment is the job's)
    const char* fe = getenv("TSF_FUSED_EXCHANGE");
    const bool want = world <= MAX_PEERS && !(fe && atoi(fe) == 0);
    if (want) {
      const size_t El = (size_t)h->K * (h->N / world) * h->H * h->d;
      h->ubuf[0] = h->uxt;
      cudaIpcMemHandle_t mine[2];
      memset(mine, 0, sizeof mine);
      bool ok = cudaMalloc(reinterpret_cast<void**>(&h->ubuf[1]), flag_area_halfs(El) * sizeof(__half)) == cudaSuccess &&
                cudaIpcGetMemHandle(&mine[0], h->ubuf[0]) == cudaSuccess &&
                cudaIpcGetMemHandle(&mine[1], h->ubuf[1]) == cudaSuccess;
      cudaGetLastError();
      ok = cudaMemcpy(dh + rank * sizeof mine, mine, sizeof mine, cudaMemcpyHostToDevice) == cudaSuccess && ok;
      bool fused = agree(ok);
      if (fused) {
        std::vector<cudaIpcMemHandle_t> all(2 * world);
        bool ok2 = ncclAllGather(dh + rank * sizeof mine, dh, sizeof mine, ncclUint8, h->comm, cs) == ncclSuccess &&
                   cudaStreamSynchronize(cs) == cudaSuccess &&
                   cudaMemcpy(all.data(), dh, (size_t)world * sizeof mine, cudaMemcpyDeviceToHost) == cudaSuccess;
        for (int p = 0; ok2 && p < world; ++p)
          for (int b = 0; ok2 && b < 2; ++b) {
            if (p == rank) h->peer_buf[b][p] = h->ubuf[b];
            else ok2 = cudaIpcOpenMemHandle(&h->peer_buf[b][p], all[2 * p + b], cudaIpcMemLazyEnablePeerAccess) ==
                       cudaSuccess;
          }
        cudaGetLastError();
        fused = agree(ok2);
      }
      if (!fused) {  // close whatever was opened; fall back to the NCCL path
        for (int b = 0; b < 2; ++b)
          for (int p = 0; p < world && p < MAX_PEERS; ++p) {
            if (h->peer_buf[b][p] && p != rank) cudaIpcCloseMemHandle(h->peer_buf[b][p]);
            h->peer_buf[b][p] = nullptr;
          }
      }
      if (fused) {
        for (int p = 0; p < world; ++p)
          h->peer_flags[p] =
              reinterpret_cast<unsigned int*>(static_cast<char*>(h->peer_buf[0][p]) + flag_area_off(El));
        const char* pb = getenv("TSF_PEER_BARRIER");
        h->peer_barrier = !(pb && atoi(pb) == 0);
      }
      int fc = 1;
      if (const char* e = getenv("TSF_FUSED_CHUNKS")) fc = atoi(e);
      if (fc < 1 || h->H % fc) fc = 1;
      h->fchunks = fc;
      h->ev_f.resize(fc + 1);
      for (auto& e : h->ev_f) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      h->fused = fused;
    }
  }
  *out = h;
  return TSF_OK;
}

tsf_status tsf_create_sim(int K, int N, int H, int d, int P, int exchange_mode, tsf_handle** out) {
  if (!out) return fail(nullptr, TSF_ERR_CONFIG, "out is null");
  *out = nullptr;
  if (P < 2 || P > MAX_PEERS) return fail(nullptr, TSF_ERR_CONFIG, "simulated world size must be in [2, 8]");
  if (exchange_mode != 1 && exchange_mode != 2) return fail(nullptr, TSF_ERR_CONFIG, "exchange_mode must be 1 or 2");
  tsf_status s = check_shape(K, N, H, d, P);
  if (s != TSF_OK) return s;
  tsf_handle* h = new tsf_handle();
  h->K = K; h->N = N; h->H = H; h->d = d;
  h->world = P;
  h->sim = true;
  if ((s = check_device(nullptr, &h->device, &h->num_sms)) != TSF_OK || (s = alloc_workspace(h)) != TSF_OK) {
    free_workspace(h);
    delete h;
    return s;
  }
  h->fused = exchange_mode == 2;
  *out = h;
  return TSF_OK;
}

void tsf_destroy(tsf_handle* h) {
  if (!h) return;
  if (h->comm) {
    ncclResult_t async_err = ncclSuccess;
    ncclCommGetAsyncError(h->comm, &async_err);
    if (async_err != ncclSuccess) ncclCommAbort(h->comm);
    else ncclCommDestroy(h->comm);
  }
  for (auto& r : h->recs) { cudaEventDestroy(r.e0); cudaEventDestroy(r.e1); }
  for (int b = 0; b < 2; ++b)
    for (int p = 0; p < h->world && p < MAX_PEERS; ++p)
      if (h->peer_buf[b][p] && p != h->rank) cudaIpcCloseMemHandle(h->peer_buf[b][p]);
  if (h->ubuf[1]) cudaFree(h->ubuf[1]);
  for (auto e : h->ev_f) cudaEventDestroy(e);
  for (auto e : h->ev_t) cudaEventDestroy(e);
  for (auto e : h->ev_a) cudaEventDestroy(e);
  if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
  for (auto e : h->ev_h) cudaEventDestroy(e);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  if (h->h2d_stream) cudaStreamDestroy(h->h2d_stream);
  for (auto e : h->event_pool) cudaEventDestroy(e);
  free_workspace(h);
  if (h->trace) cudaFree(h->trace);
  delete h;
}

const char* tsf_last_error(const tsf_handle* h) { return h ? h->err.c_str() : g_create_err.c_str(); }

int tsf_last_launch_count(const tsf_handle* h) { return h ? h->launches : 0; }

int tsf_exchange_mode(const tsf_handle* h) {
  if (!h) return -1;
  if (h->world <= 1) return 0;
  return h->fused ? 2 : 1;
}

int tsf_world_size(const tsf_handle* h) { return h ? h->world : -1; }

tsf_status tsf_set_timing(tsf_handle* h, int enable) {
  if (!h) return fail(nullptr, TSF_ERR_CONFIG, "null handle");
  for (auto& r : h->recs) { h->event_pool.push_back(r.e0); h->event_pool.push_back(r.e1); }
  h->recs.clear();
  h->timing = enable != 0;
  return TSF_OK;
}

tsf_status tsf_stage_ms(tsf_handle* h, int stage, float* total_ms, int* n_records) {
  if (!h || !total_ms) return fail(h, TSF_ERR_CONFIG, "null argument");
  float tot = 0.f;
  int n = 0;
  for (auto& r : h->recs) {
    if (r.stage != stage) continue;
    TSF_CUDA(h, cudaEventSynchronize(r.e1));
    float ms = 0.f;
    TSF_CUDA(h, cudaEventElapsedTime(&ms, r.e0, r.e1));
    tot += ms;
    ++n;
  }
  *total_ms = tot;
  if (n_records) *n_records = n;
  return TSF_OK;
}

tsf_status tsf_temporal_attn(tsf_handle* h, const tsf_bf16* q, const tsf_bf16* k, const tsf_bf16* v, tsf_bf16* o,
                             void* stream) {
  if (!h) return fail(nullptr, TSF_ERR_CONFIG, "null handle");
  h->launches = 0;
  const int Nl = h->N / h->world;
  const size_t bytes = (size_t)h->K * Nl * h->H * h->d * 2;
  tsf_status s = check_ptrs(h, {q, k, v}, o, bytes, bytes);
  if (s != TSF_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  StageTimer tm(h, st, 0);
  s = run_attention(h, temporal_view(h->K, Nl, h->H, h->d), q, k, v, EPI_OUT16, o, nullptr, st);
  tm.done();
  return s;
}

tsf_status tsf_spatial_attn(tsf_handle* h, const tsf_bf16* q, const tsf_bf16* k, const tsf_bf16* v, tsf_bf16* o,
                            void* stream) {
  if (!h) return fail(nullptr, TSF_ERR_CONFIG, "null handle");
  h->launches = 0;
  const int Kl = h->K / h->world;
  const size_t bytes = (size_t)Kl * h->N * h->H * h->d * 2;
  tsf_status s = check_ptrs(h, {q, k, v}, o, bytes, bytes);
  if (s != TSF_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  StageTimer tm(h, st, 1);
  s = run_attention(h, spatial_view(Kl, h->N, h->H, h->d), q, k, v, EPI_OUT16, o, nullptr, st);
  tm.done();
  return s;
}

tsf_status tsf_joint_attn(tsf_handle* h, const tsf_bf16* q, const tsf_bf16* k, const tsf_bf16* v, tsf_bf16* o,
                          int mask, void* stream) {
  if (!h) return fail(nullptr, TSF_ERR_CONFIG, "null handle");
  h->launches = 0;
  if (mask < TSF_MASK_NONE || mask > TSF_MASK_CAUSAL_FRAMES) return fail(h, TSF_ERR_CONFIG, "unknown mask");
  if (h->world != 1) return fail(h, TSF_ERR_UNSUPPORTED, "joint attention runs on single-GPU handles");
  if ((long long)h->K * h->N > 0x7fffffffLL) return fail(h, TSF_ERR_CONFIG, "K * N too large");
  const size_t bytes = (size_t)h->K * h->N * h->H * h->d * 2;
  tsf_status s = check_ptrs(h, {q, k, v}, o, bytes, bytes);
  if (s != TSF_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  // all K*N tokens as one sequence per head: [K, N, H, d] = [1, K*N, H, d]
  const View jv{h->K * h->N, h->H, 1, (long long)h->H * h->d, (long long)h->d, (long long)h->K * h->N * h->H * h->d};
  StageTimer tm(h, st, 5);
  static int split = -1;
  if (split < 0) {
    const char* e = getenv("TSF_CAUSAL_SPLIT");
    split = e ? atoi(e) != 0 : 1;
  }
  if (mask == TSF_MASK_CAUSAL_FRAMES && split && h->N > 128) {
    // causal frames [t' <= t]: the queries of frame t attend exactly to the first
    // (t + 1) N tokens, so frame t is an unmasked attention of its N queries over
    // that key prefix -- K launches doing K (K + 1) / 2 frames of keys instead of
    // one masked launch visiting all K^2 (the flash kernel's separate key length)
    const size_t frame = (size_t)h->N * h->H * h->d;
    const View qv{h->N, h->H, 1, (long long)h->H * h->d, (long long)h->d, (long long)frame};
    for (int t = 0; t < h->K && s == TSF_OK; ++t) {
      const View kv{(t + 1) * h->N, h->H, 1, (long long)h->H * h->d, (long long)h->d, (long long)h->K * frame};
      s = run_attention(h, qv, reinterpret_cast<const __nv_bfloat16*>(q) + t * frame, k, v, EPI_OUT16,
                        reinterpret_cast<__nv_bfloat16*>(o) + t * frame, nullptr, st, nullptr, nullptr, 0, &kv);
    }
  } else {
    s = run_attention(h, jv, q, k, v, EPI_OUT16, o, nullptr, st, nullptr, nullptr, mask);
  }
  tm.done();
  return s;
}

tsf_status tsf_storm_attn(tsf_handle* h, const tsf_bf16* u, const tsf_bf16* ctx, int M, double sigma,
                          double sigma_data, float* y, void* stream) {
  if (!h) return fail(nullptr, TSF_ERR_CONFIG, "null handle");
  h->launches = 0;
  if (M < 1) return fail(h, TSF_ERR_CONFIG, "M must be >= 1");
  if (!(sigma_data > 0.0) || !(sigma >= 0.0) || !std::isfinite(sigma))
    return fail(h, TSF_ERR_CONFIG, "need sigma >= 0 (finite) and sigma_data > 0");
  if (h->world != 1) return fail(h, TSF_ERR_UNSUPPORTED, "STORM attention runs on single-GPU handles");
  const int B = h->K, N = h->N, H = h->H, d = h->d;
  const size_t ubytes = (size_t)B * N * H * d * 2, cbytes = (size_t)B * M * H * d * 2, ybytes = (size_t)B * N * H * d * 4;
  tsf_status s = check_ptrs(h, {u}, y, ubytes, ybytes);
  if (s != TSF_OK) return s;
  if ((s = check_ptrs(h, {ctx}, y, cbytes, ybytes)) != TSF_OK) return s;
  const double g = sigma * sigma / (sigma * sigma + sigma_data * sigma_data);  // noise gate (reading G18)
  cudaStream_t st = (cudaStream_t)stream;
  const View vu = spatial_view(B, N, H, d);                                    // groups (h, b), axis n
  const View vc{M, H, B, (long long)H * d, (long long)d, (long long)M * H * d};  // groups (h, b), axis m
  StageTimer tm(h, st, 6);
  // y = u + g Cross(u, ctx, ctx)  then  y += (1 - g) Self(u, u, u)
  s = run_attention(h, vu, u, ctx, ctx, EPI_STORM_X, nullptr, y, st, nullptr, nullptr, 0, &vc, (float)g);
  if (s == TSF_OK) s = run_attention(h, vu, u, u, u, EPI_STORM_S, nullptr, y, st, nullptr, nullptr, 0, nullptr, (float)(1.0 - g));
  tm.done();
  return s;
}

// ---------------------------------------------------------------------------
// Backward (NEXT-2): forward recompute with row statistics, the key-tile
// backward kernel (attn_bwd.cuh), small elementwise kernels.
// ---------------------------------------------------------------------------
}  // extern "C"

static tsf_status bwd_workspace(tsf_handle* h, size_t need) {
  if (h->bw_bytes >= need) return TSF_OK;
  if (h->bw) cudaFree(h->bw);
  h->bw = nullptr;
  h->bw_bytes = 0;
  if (cudaMalloc(&h->bw, need) != cudaSuccess) {
    cudaGetLastError();
    return fail(h, TSF_ERR_NOMEM, "backward workspace cudaMalloc failed");
  }
  h->bw_bytes = need;
  return TSF_OK;
}

// Gradients of one attention stage over view v (q, k, v, dO bf16 with the
// view's strides): dq accumulated in fp32 (dqacc, zeroed here), dk / dv bf16.
// Workspace: o (bf16, E elements) and the row statistics (lse, drow).
static tsf_status stage_bwd(tsf_handle* h, const View& v, const void* q, const void* k, const void* vv,
                            const void* dO, float* dqacc, __nv_bfloat16* dk, __nv_bfloat16* dv, __nv_bfloat16* o_ws,
                            float* lse, float* drow, cudaStream_t st) {
  const int d = h->d;
  const int nt = (v.L + 127) / 128;
  const int pitch = nt * 128;
  const size_t E0 = (size_t)v.L * v.A * v.B * d;  // elements of the viewed (contiguous) tensor
  if (v.L <= 128) {
    // packed: G = 128 / L whole groups per tile, row statistics computed in the
    // kernel (no forward recompute), one launch
    const int G = 128 / v.L;
    int Ab = 1;
    for (int a = 1; a <= G && a <= v.A; ++a)
      if (v.A % a == 0) Ab = a;
    int Bb = G / Ab;
    if (Bb > v.B) Bb = v.B;
    CUtensorMap mq, mk, mv, mdo;
    tsf_status s;
    if ((s = make_map(h, &mq, q, d, v, v.L, Ab, Bb, false)) != TSF_OK) return s;
    if ((s = make_map(h, &mk, k, d, v, v.L, Ab, Bb, false)) != TSF_OK) return s;
    if ((s = make_map(h, &mv, vv, d, v, v.L, Ab, Bb, false)) != TSF_OK) return s;
    if ((s = make_map(h, &mdo, dO, d, v, v.L, Ab, Bb, false)) != TSF_OK) return s;
    TSF_CUDA(h, cudaMemsetAsync(dqacc, 0, E0 * sizeof(float), st));
    BwdParams bp{};
    bp.L = v.L; bp.A = v.A; bp.B = v.B;
    bp.sL = v.sL; bp.sA = v.sA; bp.sB = v.sB;
    bp.scale = (float)(1.0 / std::sqrt((double)d));
    bp.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d));
    bp.dq = dqacc; bp.dk = dk; bp.dv = dv;
    bp.nkt = 1; bp.nqt = 1;
    bp.Ab = Ab; bp.Bb = Bb; bp.tiles_a = v.A / Ab;
    const long long grid = (long long)bp.tiles_a * ((v.B + Bb - 1) / Bb);
    if (grid > 0x7fffffffLL) return fail(h, TSF_ERR_CONFIG, "too many backward tiles");
    auto go = [&](auto kern, int smem) -> tsf_status {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return fail(h, TSF_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      kern<<<(int)grid, 192, smem, st>>>(mq, mk, mv, mdo, bp);
      e = cudaGetLastError();
      if (e != cudaSuccess) return fail(h, TSF_ERR_CUDA, std::string("backward launch: ") + cudaGetErrorString(e));
      h->launches++;
      return TSF_OK;
    };
    if (d == 32) return go(attn_bwd_kernel<32, true>, BwdCfg<32>::SMEM);
    if (d == 128) return go(attn_bwd_kernel<128, true>, BwdCfg<128>::SMEM);
    return go(attn_bwd_kernel<64, true>, BwdCfg<64>::SMEM);
  }
  // 1. forward recompute with lse2 and D = rowsum(O dO)
  h->st_lse = lse;
  h->st_drow = drow;
  h->st_dO = dO;
  h->st_pitch = pitch;
  tsf_status s = run_attention(h, v, q, k, vv, EPI_OUT16, o_ws, nullptr, st);
  h->st_lse = nullptr;
  h->st_drow = nullptr;
  h->st_dO = nullptr;
  h->st_pitch = 0;
  if (s != TSF_OK) return s;
  // 2. the key-tile backward
  TSF_CUDA(h, cudaMemsetAsync(dqacc, 0, E0 * sizeof(float), st));
  CUtensorMap mq, mk, mv, mdo;
  if ((s = make_map(h, &mq, q, d, v, 128, 1, 1, false)) != TSF_OK) return s;
  if ((s = make_map(h, &mk, k, d, v, 128, 1, 1, false)) != TSF_OK) return s;
  if ((s = make_map(h, &mv, vv, d, v, 128, 1, 1, false)) != TSF_OK) return s;
  if ((s = make_map(h, &mdo, dO, d, v, 128, 1, 1, false)) != TSF_OK) return s;
  BwdParams bp{};
  bp.L = v.L; bp.A = v.A; bp.B = v.B;
  bp.sL = v.sL; bp.sA = v.sA; bp.sB = v.sB;
  bp.lse = lse; bp.drow = drow; bp.lse_pitch = pitch;
  bp.scale = (float)(1.0 / std::sqrt((double)d));
  bp.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d));
  bp.dq = dqacc; bp.dk = dk; bp.dv = dv;
  bp.nkt = nt; bp.nqt = nt;
  if (const char* e = getenv("TSF_BWD_FLAGS")) bp.flags = atoi(e);
  const long long grid = (long long)nt * v.A * v.B;
  if (grid > 0x7fffffffLL) return fail(h, TSF_ERR_CONFIG, "too many backward tiles");
  auto go = [&](auto kern, int smem) -> tsf_status {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return fail(h, TSF_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    kern<<<(int)grid, 192, smem, st>>>(mq, mk, mv, mdo, bp);
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(h, TSF_ERR_CUDA, std::string("backward launch: ") + cudaGetErrorString(e));
    h->launches++;
    return TSF_OK;
  };
  if (d == 32) return go(attn_bwd_kernel<32, false>, BwdCfg<32>::SMEM);
  if (d == 128) return go(attn_bwd_kernel<128, false>, BwdCfg<128>::SMEM);
  return go(attn_bwd_kernel<64, false>, BwdCfg<64>::SMEM);
}

static int ew_grid(tsf_handle* h, long long n) {
  long long g = (n + 255) / 256;
  const long long cap = (long long)h->num_sms * 8;
  return (int)(g < 1 ? 1 : g > cap ? cap : g);
}

// one stage's public backward: bf16 dq / dk / dv
static tsf_status stage_bwd_public(tsf_handle* h, int axis, const tsf_bf16* q, const tsf_bf16* k, const tsf_bf16* v,
                                   const tsf_bf16* dO, tsf_bf16* dq, tsf_bf16* dk, tsf_bf16* dv, void* stream) {
  if (!h) return fail(nullptr, TSF_ERR_CONFIG, "null handle");
  h->launches = 0;
  // distributed (and simulated) handles: the rank's own shard, like the forward
  // stage calls -- temporal on the token shard [K, N/P, H, d], spatial on the
  // frame shard [K/P, N, H, d]; both are local (no exchange)
  const int Nl = h->N / h->world, Kl = h->K / h->world;
  const size_t E = (size_t)(axis == 0 ? h->K : Kl) * (axis == 0 ? Nl : h->N) * h->H * h->d;
  for (const void* o : {(const void*)dq, (const void*)dk, (const void*)dv}) {
    tsf_status s = check_ptrs(h, {q, k, v, dO}, o, E * 2, E * 2);
    if (s != TSF_OK) return s;
  }
  if (overlap(dq, E * 2, dk, E * 2) || overlap(dq, E * 2, dv, E * 2) || overlap(dk, E * 2, dv, E * 2))
    return fail(h, TSF_ERR_CONFIG, "gradient outputs overlap");
  const View vw = axis == 0 ? temporal_view(h->K, Nl, h->H, h->d) : spatial_view(Kl, h->N, h->H, h->d);
  const size_t groups = (size_t)vw.A * vw.B, pitch = (size_t)((vw.L + 127) / 128) * 128;
  const size_t need = E * 2 + E * 4 + 2 * groups * pitch * 4 + 1024;
  tsf_status s = bwd_workspace(h, need);
  if (s != TSF_OK) return s;
  char* b = static_cast<char*>(h->bw);
  __nv_bfloat16* o_ws = reinterpret_cast<__nv_bfloat16*>(b);
  float* dqacc = reinterpret_cast<float*>(b + ((E * 2 + 255) & ~size_t(255)));
  float* lse = dqacc + E;
  float* drow = lse + groups * pitch;
  cudaStream_t st = (cudaStream_t)stream;
  StageTimer tm(h, st, 8);
  s = stage_bwd(h, vw, q, k, v, dO, dqacc, reinterpret_cast<__nv_bfloat16*>(dk), reinterpret_cast<__nv_bfloat16*>(dv),
                o_ws, lse, drow, st);
  if (s == TSF_OK) {
    f32_to_bf16_kernel<<<ew_grid(h, (long long)(E / 8)), 256, 0, st>>>(dqacc, reinterpret_cast<__nv_bfloat16*>(dq),
                                                                       (long long)(E / 8));
    h->launches++;
    if (cudaGetLastError() != cudaSuccess) s = fail(h, TSF_ERR_CUDA, "dq conversion launch failed");
  }
  tm.done();
  return s;
}

extern "C" {

tsf_status tsf_temporal_attn_bwd(tsf_handle* h, const tsf_bf16* q, const tsf_bf16* k, const tsf_bf16* v,
                                 const tsf_bf16* dO, tsf_bf16* dq, tsf_bf16* dk, tsf_bf16* dv, void* stream) {
  return stage_bwd_public(h, 0, q, k, v, dO, dq, dk, dv, stream);
}

tsf_status tsf_spatial_attn_bwd(tsf_handle* h, const tsf_bf16* q, const tsf_bf16* k, const tsf_bf16* v,
                                const tsf_bf16* dO, tsf_bf16* dq, tsf_bf16* dk, tsf_bf16* dv, void* stream) {
  return stage_bwd_public(h, 1, q, k, v, dO, dq, dk, dv, stream);
}

}  // extern "C"

extern "C" {
static tsf_status check_comm(tsf_handle* h);
}
static tsf_status reshard_gen(tsf_handle* h, int dir, const void* in, void* out, int elem_bytes, void* scratch,
                              cudaStream_t st);

// Distributed block backward (P > 1, real or simulated ranks), the exchange
// reversed: x token shard -> X_t token shard (temporal forward, local) -> X_t
// frame shard (T2S) -> spatial backward on the frame shard with dy -> dX_t
// frame shard (fp32) -> dX_t token shard (S2T, fp32 bytes) -> temporal
// backward on the token shard -> dx token shard.  Simulated handles take every
// rank's shards stacked, as tsf_spacetime_block does.
static tsf_status block_bwd_dist(tsf_handle* h, const tsf_bf16* x, const float* dy, float* dx, cudaStream_t st) {
  const int P = h->world, Nl = h->N / P, Kl = h->K / P, H = h->H, d = h->d;
  const int V = h->sim ? P : 1;
  const size_t Es = (size_t)h->K * Nl * H * d;   // one rank's token shard = frame shard elements
  const View vt = temporal_view(h->K, Nl, H, d), vs = spatial_view(Kl, h->N, H, d);
  const size_t pt = (size_t)((vt.L + 127) / 128) * 128 * vt.A * vt.B, ps = (size_t)((vs.L + 127) / 128) * 128 * vs.A * vs.B;
  const size_t pmax = pt > ps ? pt : ps;
  // per handled rank: o_ws | xtb_tok | xtb_fr | dyb | dxtb | dk | dv (bf16) | dqacc | dxt_fr | dxt_tok | scratch (fp32)
  const size_t per = 7 * Es * 2 + 4 * Es * 4;
  const size_t need = V * per + 2 * pmax * 4 + 4096;
  tsf_status s = bwd_workspace(h, need);
  if (s != TSF_OK) return s;
  char* base = static_cast<char*>(h->bw);
  auto bfp = [&](int slot) { return reinterpret_cast<__nv_bfloat16*>(base + (size_t)slot * V * Es * 2); };
  __nv_bfloat16 *o_ws = bfp(0), *xtb_tok = bfp(1), *xtb_fr = bfp(2), *dyb = bfp(3), *dxtb = bfp(4), *dk = bfp(5),
                *dv = bfp(6);
  float* f32 = reinterpret_cast<float*>(base + 7 * V * Es * 2);
  float *dqacc = f32, *dxt_fr = f32 + V * Es, *dxt_tok = f32 + 2 * V * Es, *scratch = f32 + 3 * V * Es;
  float* lse = f32 + 4 * V * Es;
  float* drow = lse + pmax;
  const long long n8 = (long long)(Es / 8);
  const int g = ew_grid(h, n8);
  // X_t token shard of every handled rank, then to frame shards
  for (int r = 0; r < V; ++r) {
    if ((s = run_attention(h, vt, x + r * Es, x + r * Es, x + r * Es, EPI_OUT16, o_ws + r * Es, nullptr, st)) != TSF_OK)
      return s;
    add_bf16_kernel<<<g, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(x) + r * Es, o_ws + r * Es,
                                       xtb_tok + r * Es, n8);
    h->launches++;
  }
  TSF_CUDA(h, cudaGetLastError());
  if ((s = check_comm(h)) != TSF_OK) return s;
  if ((s = reshard_gen(h, TSF_T2S, xtb_tok, xtb_fr, 2, scratch, st)) != TSF_OK) return s;
  // spatial backward on each frame shard
  for (int r = 0; r < V; ++r) {
    f32_to_bf16_kernel<<<g, 256, 0, st>>>(dy + r * Es, dyb + r * Es, n8);
    h->launches++;
    const __nv_bfloat16* xf = xtb_fr + r * Es;
    if ((s = stage_bwd(h, vs, xf, xf, xf, dyb + r * Es, dqacc + r * Es, dk + r * Es, dv + r * Es, o_ws + r * Es, lse,
                       drow, st)) != TSF_OK)
      return s;
    sum4_kernel<<<g, 256, 0, st>>>(dy + r * Es, dqacc + r * Es, dk + r * Es, dv + r * Es, dxt_fr + r * Es, nullptr, n8);
    h->launches++;
  }
  TSF_CUDA(h, cudaGetLastError());
  // dX_t back to token shards (fp32 bytes, bit-exact)
  if ((s = reshard_gen(h, TSF_S2T, dxt_fr, dxt_tok, 4, scratch, st)) != TSF_OK) return s;
  // temporal backward on each token shard
  for (int r = 0; r < V; ++r) {
    f32_to_bf16_kernel<<<g, 256, 0, st>>>(dxt_tok + r * Es, dxtb + r * Es, n8);
    h->launches++;
    const tsf_bf16* xr = x + r * Es;
    if ((s = stage_bwd(h, vt, xr, xr, xr, dxtb + r * Es, dqacc + r * Es, dk + r * Es, dv + r * Es, o_ws + r * Es, lse,
                       drow, st)) != TSF_OK)
      return s;
    sum4_kernel<<<g, 256, 0, st>>>(dxt_tok + r * Es, dqacc + r * Es, dk + r * Es, dv + r * Es, dx + r * Es, nullptr, n8);
    h->launches++;
  }
  TSF_CUDA(h, cudaGetLastError());
  return TSF_OK;
}

extern "C" {

tsf_status tsf_spacetime_block_bwd(tsf_handle* h, const tsf_bf16* x, const float* dy, float* dx, void* stream) {
  if (!h) return fail(nullptr, TSF_ERR_CONFIG, "null handle");
  h->launches = 0;
  if (h->world != 1) {
    const size_t Eall = (size_t)h->K * (h->N / h->world) * h->H * h->d * (h->sim ? h->world : 1);
    tsf_status s = check_ptrs(h, {x}, dx, Eall * 2, Eall * 4);
    if (s != TSF_OK) return s;
    if ((s = check_ptrs(h, {dy}, dx, Eall * 4, Eall * 4)) != TSF_OK) return s;
    if ((s = check_comm(h)) != TSF_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    StageTimer tm(h, st, 8);
    s = block_bwd_dist(h, x, dy, dx, st);
    tm.done();
    return s;
  }
  const size_t E = (size_t)h->K * h->N * h->H * h->d;
  tsf_status s = check_ptrs(h, {x}, dx, E * 2, E * 4);
  if (s != TSF_OK) return s;
  if ((s = check_ptrs(h, {dy}, dx, E * 4, E * 4)) != TSF_OK) return s;
  const View vt = temporal_view(h->K, h->N, h->H, h->d), vs = spatial_view(h->K, h->N, h->H, h->d);
  const size_t pt = (size_t)((vt.L + 127) / 128) * 128 * vt.A * vt.B, ps = (size_t)((vs.L + 127) / 128) * 128 * vs.A * vs.B;
  const size_t pmax = pt > ps ? pt : ps;
  // o_ws | xtb | dyb | dxtb | dk | dv (bf16, E each) | dqacc | dxt (fp32, E each) | lse | drow
  const size_t need = 6 * E * 2 + 2 * E * 4 + 2 * pmax * 4 + 4096;
  if ((s = bwd_workspace(h, need)) != TSF_OK) return s;
  __nv_bfloat16* o_ws = static_cast<__nv_bfloat16*>(h->bw);
  __nv_bfloat16* xtb = o_ws + E;
  __nv_bfloat16* dyb = xtb + E;
  __nv_bfloat16* dxtb = dyb + E;
  __nv_bfloat16* dk = dxtb + E;
  __nv_bfloat16* dv = dk + E;
  float* dqacc = reinterpret_cast<float*>(dv + E);
  float* dxt = dqacc + E;
  float* lse = dxt + E;
  float* drow = lse + pmax;
  cudaStream_t st = (cudaStream_t)stream;
  const long long n8 = (long long)(E / 8);
  const int g = ew_grid(h, n8);
  int total = 0;
  auto count = [&]() { total += h->launches; h->launches = 0; };
  StageTimer tm(h, st, 8);
  // X_t = x + T(x, x, x) (bf16), dy -> bf16
  if ((s = run_attention(h, vt, x, x, x, EPI_OUT16, o_ws, nullptr, st)) != TSF_OK) return s;
  count();
  add_bf16_kernel<<<g, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(x), o_ws, xtb, n8);
  f32_to_bf16_kernel<<<g, 256, 0, st>>>(dy, dyb, n8);
  total += 2;
  TSF_CUDA(h, cudaGetLastError());
  // spatial stage: dX_t = dy + dq + dk + dv of S at X_t
  if ((s = stage_bwd(h, vs, xtb, xtb, xtb, dyb, dqacc, dk, dv, o_ws, lse, drow, st)) != TSF_OK) return s;
  count();
  sum4_kernel<<<g, 256, 0, st>>>(dy, dqacc, dk, dv, dxt, dxtb, n8);
  total++;
  TSF_CUDA(h, cudaGetLastError());
  // temporal stage: dx = dX_t + dq + dk + dv of T at x
  if ((s = stage_bwd(h, vt, x, x, x, dxtb, dqacc, dk, dv, o_ws, lse, drow, st)) != TSF_OK) return s;
  count();
  sum4_kernel<<<g, 256, 0, st>>>(dxt, dqacc, dk, dv, dx, nullptr, n8);
  total++;
  TSF_CUDA(h, cudaGetLastError());
  tm.done();
  h->launches = total;
  return TSF_OK;
}

// ---------------------------------------------------------------------------
// Full divided block (NEXT-1): LayerNorm, tcgen05 GEMMs with fused epilogues,
// and the attention kernels on strided q / k / v views of the QKV output.
// ---------------------------------------------------------------------------
}  // extern "C"
static tsf_status make_map2d(tsf_handle* h, CUtensorMap* m, const void* base, long long rows, long long cols,
                             int box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return fail(h, TSF_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(h, TSF_ERR_CUDA, "cuTensorMapEncodeTiled (GEMM) failed: " + std::to_string((int)r));
  return TSF_OK;
}

template <int BN, int EPI>
static tsf_status launch_gemm(tsf_handle* h, cudaStream_t st, const CUtensorMap& ma, const CUtensorMap& mw,
                              const GemmParams& p) {
  using C = GemmCfg<BN>;
  const int tiles = p.tiles_m * p.tiles_n;
  cudaError_t e = cudaFuncSetAttribute(gemm_kernel<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return fail(h, TSF_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  gemm_kernel<BN, EPI><<<tiles < h->num_sms ? tiles : h->num_sms, 192, C::SMEM, st>>>(ma, mw, p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(h, TSF_ERR_CUDA, std::string("GEMM launch: ") + cudaGetErrorString(e));
  h->launches++;
  return TSF_OK;
}

// C[M, N] = A[M, K] W[N, K]^T + bias (+ epilogue); N % 128 == 0, K % 64 == 0
static tsf_status gemm(tsf_handle* h, cudaStream_t st, int epi, const void* A, const void* W, const float* bias,
                       const void* res, void* Cout, long long M, int N, int K) {
  if (N % 128 || K % 64) return fail(h, TSF_ERR_UNSUPPORTED, "GEMM needs N % 128 == 0 and K % 64 == 0");
  const int BN = (N % 256 == 0) ? 256 : 128;
  CUtensorMap ma, mw;
  tsf_status s;
  if ((s = make_map2d(h, &ma, A, M, K, 128)) != TSF_OK) return s;
  if ((s = make_map2d(h, &mw, W, N, K, BN)) != TSF_OK) return s;
  GemmParams p{};
  p.M = (int)M; p.N = N; p.K = K;
  p.bias = bias; p.res = res; p.c = Cout; p.ldc = N;
  p.tiles_m = (int)((M + 127) / 128);
  p.tiles_n = N / BN;
  StageTimer tm(h, st, 7);
  if (BN == 256) {
    switch (epi) {
      case GEPI_BIAS_BF16: s = launch_gemm<256, GEPI_BIAS_BF16>(h, st, ma, mw, p); break;
      case GEPI_GELU_BF16: s = launch_gemm<256, GEPI_GELU_BF16>(h, st, ma, mw, p); break;
      case GEPI_RES_F32: s = launch_gemm<256, GEPI_RES_F32>(h, st, ma, mw, p); break;
      default: s = launch_gemm<256, GEPI_RESB_F32>(h, st, ma, mw, p); break;
    }
  } else {
    switch (epi) {
      case GEPI_BIAS_BF16: s = launch_gemm<128, GEPI_BIAS_BF16>(h, st, ma, mw, p); break;
      case GEPI_GELU_BF16: s = launch_gemm<128, GEPI_GELU_BF16>(h, st, ma, mw, p); break;
      case GEPI_RES_F32: s = launch_gemm<128, GEPI_RES_F32>(h, st, ma, mw, p); break;
      default: s = launch_gemm<128, GEPI_RESB_F32>(h, st, ma, mw, p); break;
    }
  }
  tm.done();
  return s;
}

template <typename IN>
static tsf_status layer_norm(tsf_handle* h, cudaStream_t st, const IN* x, const float* g, const float* b,
                             __nv_bfloat16* y, long long rows, int D) {
  const int blocks = (int)((rows + 7) / 8);
  const int need = (D + 255) / 256;  // 8-element chunks per lane
  StageTimer tm(h, st, 7);
  if (need <= 1) layernorm_kernel<IN, 1><<<blocks, 256, 0, st>>>(x, g, b, y, rows, D);
  else if (need <= 2) layernorm_kernel<IN, 2><<<blocks, 256, 0, st>>>(x, g, b, y, rows, D);
  else if (need <= 4) layernorm_kernel<IN, 4><<<blocks, 256, 0, st>>>(x, g, b, y, rows, D);
  else if (need <= 8) layernorm_kernel<IN, 8><<<blocks, 256, 0, st>>>(x, g, b, y, rows, D);
  else if (need <= 16) layernorm_kernel<IN, 16><<<blocks, 256, 0, st>>>(x, g, b, y, rows, D);
  else layernorm_kernel<IN, 32><<<blocks, 256, 0, st>>>(x, g, b, y, rows, D);
  tm.done();
  TSF_CUDA(h, cudaGetLastError());
  h->launches++;
  return TSF_OK;
}

extern "C" {
tsf_status tsf_full_block(tsf_handle* h, const tsf_block_weights* w, const tsf_bf16* x, float* y, void* stream) {
  if (!h) return fail(nullptr, TSF_ERR_CONFIG, "null handle");
  h->launches = 0;
  if (!w) return fail(h, TSF_ERR_CONFIG, "null weights");
  if (h->world != 1) return fail(h, TSF_ERR_UNSUPPORTED, "the full block runs on single-GPU handles");
  const int K = h->K, N = h->N, H = h->H, d = h->d, D = H * d, F = w->F;
  const long long T = (long long)K * N;
  if (D % 128 || D > 8192 || F < 128 || F % 128) return fail(h, TSF_ERR_UNSUPPORTED, "need D = H*d % 128 == 0 (<= 8192) and F % 128 == 0");
  const void* ptrs[] = {w->ln_t_g, w->ln_t_b, w->w_qkv_t, w->b_qkv_t, w->w_o_t, w->b_o_t, w->ln_s_g, w->ln_s_b,
                        w->w_qkv_s, w->b_qkv_s, w->w_o_s, w->b_o_s, w->ln_m_g, w->ln_m_b, w->w_1, w->b_1, w->w_2, w->b_2};
  for (const void* p : ptrs)
    if (!p || !aligned16(p)) return fail(h, TSF_ERR_CONFIG, "weight pointer null or not 16-byte aligned");
  tsf_status s = check_ptrs(h, {x}, y, (size_t)T * D * 2, (size_t)T * D * 4);
  if (s != TSF_OK) return s;
  // workspace: hb bf16 [T, D] | qkv bf16 [T, 3D] | o bf16 [T, D] | m bf16 [T, F] | xt fp32 [T, D] | xs fp32 [T, D]
  const size_t need = (size_t)T * (2 * D + 6 * D + 2 * D + 2 * (size_t)F + 4 * D + 4 * D) + 4 * 256;
  if (h->fb_bytes < need) {
    if (h->fb) cudaFree(h->fb);
    h->fb = nullptr;
    h->fb_bytes = 0;
    if (cudaMalloc(&h->fb, need) != cudaSuccess) {
      cudaGetLastError();
      return fail(h, TSF_ERR_NOMEM, "full-block workspace cudaMalloc failed");
    }
    h->fb_bytes = need;
  }
  auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
  char* base = static_cast<char*>(h->fb);
  __nv_bfloat16* hb = reinterpret_cast<__nv_bfloat16*>(base);
  __nv_bfloat16* qkv = reinterpret_cast<__nv_bfloat16*>(base + al((size_t)T * D * 2));
  __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<char*>(qkv) + al((size_t)T * 3 * D * 2));
  __nv_bfloat16* m = reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<char*>(o) + al((size_t)T * D * 2));
  float* xt = reinterpret_cast<float*>(reinterpret_cast<char*>(m) + al((size_t)T * F * 2));
  float* xsp = xt + T * D;
  cudaStream_t st = (cudaStream_t)stream;
  const int launches_before = 0;
  (void)launches_before;
  int total = 0;
  auto count = [&]() { total += h->launches; h->launches = 0; };
  const long long D3 = 3LL * D;
  // views of q / k / v inside the QKV output [K, N, 3D] (head h at columns h d of each third)
  const View qt{K, H, N, (long long)N * D3, (long long)d, D3};            // temporal: axis t, groups (h, n)
  const View qs{N, H, K, D3, (long long)d, (long long)N * D3};            // spatial: axis n, groups (h, t)
  const View ot = temporal_view(K, N, H, d), os = spatial_view(K, N, H, d);
  // ---- temporal stage ----
  if ((s = layer_norm(h, st, reinterpret_cast<const __nv_bfloat16*>(x), w->ln_t_g, w->ln_t_b, hb, T, D)) != TSF_OK) return s;
  count();
  if ((s = gemm(h, st, GEPI_BIAS_BF16, hb, w->w_qkv_t, w->b_qkv_t, nullptr, qkv, T, 3 * D, D)) != TSF_OK) return s;
  count();
  {
    StageTimer tm(h, st, 0);
    s = run_attention(h, qt, qkv, qkv + D, qkv + 2 * D, EPI_OUT16, o, nullptr, st, &ot);
    tm.done();
    if (s != TSF_OK) return s;
    count();
  }
  if ((s = gemm(h, st, GEPI_RESB_F32, o, w->w_o_t, w->b_o_t, x, xt, T, D, D)) != TSF_OK) return s;
  count();
  // ---- spatial stage ----
  if ((s = layer_norm(h, st, xt, w->ln_s_g, w->ln_s_b, hb, T, D)) != TSF_OK) return s;
  count();
  if ((s = gemm(h, st, GEPI_BIAS_BF16, hb, w->w_qkv_s, w->b_qkv_s, nullptr, qkv, T, 3 * D, D)) != TSF_OK) return s;
  count();
  {
    StageTimer tm(h, st, 1);
    s = run_attention(h, qs, qkv, qkv + D, qkv + 2 * D, EPI_OUT16, o, nullptr, st, &os);
    tm.done();
    if (s != TSF_OK) return s;
    count();
  }
  if ((s = gemm(h, st, GEPI_RES_F32, o, w->w_o_s, w->b_o_s, xt, xsp, T, D, D)) != TSF_OK) return s;
  count();
  // ---- MLP ----
  if ((s = layer_norm(h, st, xsp, w->ln_m_g, w->ln_m_b, hb, T, D)) != TSF_OK) return s;
  count();
  if ((s = gemm(h, st, GEPI_GELU_BF16, hb, w->w_1, w->b_1, nullptr, m, T, F, D)) != TSF_OK) return s;
  count();
  if ((s = gemm(h, st, GEPI_RES_F32, m, w->w_2, w->b_2, xsp, y, T, D, F)) != TSF_OK) return s;
  count();
  h->launches = total;
  return TSF_OK;
}

// ---------------------------------------------------------------------------
// Distributed block pieces.  The multi-process path (one rank per GPU) and the
// one-GPU simulation of P ranks (tsf_create_sim) run the SAME pieces: the same
// run_attention calls (output routing, per-destination tensor maps, kernels),
// the same byte plan and unpack kernel.  Only the transport differs: NCCL
// send/recv and CUDA IPC peer pointers vs device copies and local buffers.
// ---------------------------------------------------------------------------

// Temporal stage of rank `rank` with the fused exchange: X_t rows go straight
// into every rank's frame shard (peers[r]); vin is the rank's token-shard view
// (all heads, or one head chunk).
// Cross-rank barrier of the fused exchange over peer memory (replaces the 1-int
// NCCL all-reduce, ~16-36 us, on the step's critical path).  Thread r announces
// `epoch` in peer r's slot for this rank (release, system scope: the temporal
// kernel that stored X_t rows into the peers ran before this one on the
// stream), then waits (acquire) until peer r has announced it here.  Bounded:
// after ~10 s a missing peer sets err (host-mapped), reported by tsf_sync.
struct PeerFlags {
  unsigned int* f[MAX_PEERS];
};
__global__ void peer_barrier_kernel(const PeerFlags pf, int rank, int P, unsigned int epoch, unsigned int* err) {
  const int r = threadIdx.x;
  if (r < P) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pf.f[r] + rank), "r"(epoch) : "memory");
  }
  if (r < P) {
    const unsigned int* mine = pf.f[rank] + r;
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      unsigned int v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if ((int)(v - epoch) >= 0) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 10000000000ull) {  // 10 s
        *reinterpret_cast<volatile unsigned int*>(err) = 1u;
        break;
      }
      __nanosleep(64);
    }
  }
}

static tsf_status peer_barrier(tsf_handle* h, cudaStream_t st) {
  PeerFlags pf{};
  for (int r = 0; r < h->world && r < MAX_PEERS; ++r) pf.f[r] = h->peer_flags[r];
  peer_barrier_kernel<<<1, 32, 0, st>>>(pf, h->rank, h->world, ++h->bar_epoch, h->nf_dev + 1);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(h, TSF_ERR_CUDA, std::string("peer barrier launch: ") + cudaGetErrorString(e));
  h->launches++;
  return TSF_OK;
}

static tsf_status temporal_fused(tsf_handle* h, const View& vin, const tsf_bf16* x, int rank, void* const* peers,
                                 cudaStream_t st) {
  const DistOut dist{h->world, h->K / h->world, rank, h->N / h->world, peers};
  StageTimer tm(h, st, 0);
  tsf_status s = run_attention(h, vin, x, x, x, EPI_BLOCK_T, nullptr, nullptr, st, nullptr, &dist);
  tm.done();
  return s;
}

// NCCL-path temporal stage of head chunk c: X_t token shard chunk
// [K][N/P][Hc][d] into xt (rank-local).
static tsf_status temporal_tokens(tsf_handle* h, const tsf_bf16* x, __half* xt, int c, cudaStream_t st) {
  const int nc = h->nchunk, Hc = h->H / nc, K = h->K, Nl = h->N / h->world, H = h->H, d = h->d;
  const size_t chunk_elems = (size_t)K * Nl * Hc * d;
  const View vin{K, Hc, Nl, (long long)Nl * H * d, (long long)d, (long long)H * d};
  const View vout{K, Hc, Nl, (long long)Nl * Hc * d, (long long)d, (long long)Hc * d};
  const tsf_bf16* xc = x + (size_t)c * Hc * d;
  StageTimer tm(h, st, 0);
  tsf_status s = run_attention(h, vin, xc, xc, xc, EPI_BLOCK_T, xt + c * chunk_elems, nullptr, st, &vout);
  tm.done();
  return s;
}

// Byte plan of the exchange of head chunk c: chunk c of X_t is
// [K][N/P][Hc][d]; its frames [p K/P, (p+1) K/P) (contiguous, peer_bytes)
// go to peer p, which stores them at slot `rank` of its receive buffer
// [P][K/P][N/P][Hc][d].  Untyped bytes: bit-exact.
static size_t exchange_peer_bytes(const tsf_handle* h) {
  return (size_t)(h->K / h->world) * (h->N / h->world) * (h->H / h->nchunk) * h->d * 2;
}
static size_t chunk_elems(const tsf_handle* h) {
  return (size_t)h->K * (h->N / h->world) * (h->H / h->nchunk) * h->d;
}
static tsf_status exchange_chunk(tsf_handle* h, int c, cudaStream_t cs) {  // NCCL transport
  const int P = h->world;
  const size_t peer_bytes = exchange_peer_bytes(h);
  const char* src = reinterpret_cast<const char*>(h->xt + c * chunk_elems(h));
  char* dst = reinterpret_cast<char*>(h->rxt + c * chunk_elems(h));
  TSF_NCCL(h, ncclGroupStart());
  for (int p = 0; p < P; ++p) {
    TSF_NCCL(h, ncclSend(src + p * peer_bytes, peer_bytes, ncclUint8, p, h->comm, cs));
    TSF_NCCL(h, ncclRecv(dst + p * peer_bytes, peer_bytes, ncclUint8, p, h->comm, cs));
  }
  TSF_NCCL(h, ncclGroupEnd());
  return TSF_OK;
}
// The same byte plan with device copies between the simulated ranks'
// buffers (base[r] = rank r's buffer, El elements apart).
static tsf_status exchange_sim(tsf_handle* h, const __half* src_base, __half* dst_base, size_t stride_elems,
                               size_t src_off, size_t dst_off, size_t peer_bytes, cudaStream_t st) {
  const int P = h->world;
  for (int r = 0; r < P; ++r)
    for (int p = 0; p < P; ++p) {
      const char* src = reinterpret_cast<const char*>(src_base + r * stride_elems + src_off) + p * peer_bytes;
      char* dst = reinterpret_cast<char*>(dst_base + p * stride_elems + dst_off) + r * peer_bytes;
      TSF_CUDA(h, cudaMemcpyAsync(dst, src, peer_bytes, cudaMemcpyDeviceToDevice, st));
    }
  return TSF_OK;
}

// receive buffer [P][K/P][N/P][Hc][d] of chunk c -> frame shard [K/P][N][Hc][d]
static tsf_status unpack_chunk(tsf_handle* h, const __half* rxt, __half* uxt, int c, cudaStream_t st) {
  const int P = h->world, Kc = h->K / P, Nc = h->N / P, Hc = h->H / h->nchunk;
  const int vecs = Hc * h->d * 2 / 16;
  const long long items = (long long)P * Kc * Nc * vecs;
  reshard_perm_kernel<true><<<grid_for(h, items), 256, 0, st>>>((const uint4*)(rxt + c * chunk_elems(h)),
                                                                (uint4*)(uxt + c * chunk_elems(h)), nullptr,
                                                                nullptr, P, Kc, Nc, vecs);
  TSF_CUDA(h, cudaGetLastError());
  h->launches++;
  return TSF_OK;
}

// Spatial stage of a frame shard: u = X_t [K/P][N][H][d] (chunk layout
// [c][K/P][N][Hc][d] when `chunked`), y fp32 [K/P][N][H][d].
static tsf_status spatial_shard(tsf_handle* h, const __half* u, float* y, int nc, int c, bool chunked,
                                cudaStream_t st) {
  const int Kl = h->K / h->world, N = h->N, H = h->H, d = h->d, Hc = H / nc;
  const View vy{N, Hc, Kl, (long long)H * d, (long long)d, (long long)N * H * d};
  const View vs = chunked ? View{N, Hc, Kl, (long long)Hc * d, (long long)d, (long long)N * Hc * d} : vy;
  const __half* uc = u + (chunked ? c * chunk_elems(h) : (size_t)c * Hc * d);
  StageTimer tm(h, st, 1);
  tsf_status s = run_attention(h, vs, uc, uc, uc, EPI_BLOCK_S, nullptr, y + (size_t)c * Hc * d, st, &vy);
  tm.done();
  return s;
}

static tsf_status check_comm(tsf_handle* h) {
  if (h->world <= 1 || h->sim) return TSF_OK;
  if (h->comm_dead || !h->comm) return fail(h, TSF_ERR_NCCL, "communicator aborted (tsf_sync timeout or error)");
  ncclResult_t ae = ncclSuccess;
  if (ncclCommGetAsyncError(h->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
    return fail(h, TSF_ERR_NCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(ae));
  return TSF_OK;
}

// One-GPU simulation of the distributed block: x = the P token shards back
// to back ([P][K][N/P][H][d]), y = the P frame shards back to back
// ([P][K/P][N][H][d] = [K][N][H][d]).
static tsf_status block_sim(tsf_handle* h, const tsf_bf16* x, float* y, cudaStream_t st) {
  const int P = h->world, Nl = h->N / P, Kl = h->K / P, H = h->H, d = h->d;
  const size_t El = (size_t)h->K * Nl * H * d;            // token shard = frame shard elements
  const size_t Ey = (size_t)Kl * h->N * H * d;
  tsf_status s = TSF_ERR_UNSUPPORTED;
  if (h->fused) {
    void* peers[MAX_PEERS];
    for (int r = 0; r < P; ++r) peers[r] = h->uxt + r * El;
    for (int r = 0; r < P; ++r) {
      s = temporal_fused(h, temporal_view(h->K, Nl, H, d), x + r * El, r, peers, st);
      if (s != TSF_OK) break;
    }
    if (s == TSF_OK) {
      for (int r = 0; r < P && s == TSF_OK; ++r) s = spatial_shard(h, h->uxt + r * El, y + r * Ey, 1, 0, false, st);
      return s;
    }
    if (s != TSF_ERR_UNSUPPORTED) return s;
  }
  // NCCL byte plan (one head chunk), device copies as the transport
  for (int r = 0; r < P; ++r)
    if ((s = temporal_tokens(h, x + r * El, h->xt + r * El, 0, st)) != TSF_OK) return s;
  {
    StageTimer tm(h, st, 2);
    if ((s = exchange_sim(h, h->xt, h->rxt, El, 0, 0, exchange_peer_bytes(h), st)) != TSF_OK) return s;
    tm.done();
  }
  for (int r = 0; r < P; ++r) {
    if ((s = unpack_chunk(h, h->rxt + r * El, h->uxt + r * El, 0, st)) != TSF_OK) return s;
    if ((s = spatial_shard(h, h->uxt + r * El, y + r * Ey, 1, 0, true, st)) != TSF_OK) return s;
  }
  return TSF_OK;
}

tsf_status tsf_spacetime_block(tsf_handle* h, const tsf_bf16* x, float* y, void* stream) {
  if (!h) return fail(nullptr, TSF_ERR_CONFIG, "null handle");
  h->launches = 0;
  const int P = h->world, Nl = h->N / P, Kl = h->K / P;
  const int V = h->sim ? P : 1;  // a simulated handle takes every virtual rank's shard
  const size_t in_bytes = (size_t)h->K * Nl * h->H * h->d * 2 * V;
  const size_t out_bytes = (size_t)Kl * h->N * h->H * h->d * 4 * V;
  tsf_status s = check_ptrs(h, {x}, y, in_bytes, out_bytes);
  if (s != TSF_OK) return s;
  if ((s = check_comm(h)) != TSF_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (P == 1) {
    // temporal stage: X_t = x + T(x, x, x), stored fp16
    {
      StageTimer tm(h, st, 0);
      s = run_attention(h, temporal_view(h->K, Nl, h->H, h->d), x, x, x, EPI_BLOCK_T, h->xt, nullptr, st);
      tm.done();
      if (s != TSF_OK) return s;
    }
    // spatial stage: y = X_t + S(X_t, X_t, X_t)
    StageTimer tm(h, st, 1);
    s = run_attention(h, spatial_view(Kl, h->N, h->H, h->d), h->xt, h->xt, h->xt, EPI_BLOCK_S, nullptr, y, st);
    tm.done();
    return s;
  }
  if (h->sim) return block_sim(h, x, y, st);
  if (h->fused) {
    // Fused exchange: the temporal kernel writes X_t rows straight into the
    // owning rank's frame shard (CUDA IPC + NVLink TMA/plain stores), a 1-int
    // NCCL all-reduce orders every rank's stores before any spatial read.
    // With fchunks > 1 the heads are split into chunks: temporal(c) + its
    // all-reduce run on the comm stream, spatial(c) on `st` after them, so the
    // NVLink stores of chunk c+1 overlap the spatial stage of chunk c.
    const int par = h->fparity, nc = h->fchunks, H = h->H, d = h->d, Hc = H / nc;
    const __half* u = h->ubuf[par];
    auto peers_of = [&](int c, void** out) {
      for (int r = 0; r < P; ++r) out[r] = static_cast<__half*>(h->peer_buf[par][r]) + (size_t)c * Hc * d;
    };
    if (nc == 1) {
      void* peers[MAX_PEERS];
      peers_of(0, peers);
      s = temporal_fused(h, temporal_view(h->K, Nl, H, d), x, h->rank, peers, st);
      if (s == TSF_OK) {
        StageTimer tm(h, st, 2);
        if (h->peer_barrier) {
          if ((s = peer_barrier(h, st)) != TSF_OK) return s;
        } else {
          TSF_NCCL(h, ncclAllReduce(h->d_flag, h->d_flag, 1, ncclInt32, ncclSum, h->comm, st));
        }
        tm.done();
        s = spatial_shard(h, u, y, 1, 0, false, st);
        if (s == TSF_OK) h->fparity ^= 1;
        return s;
      }
      if (s != TSF_ERR_UNSUPPORTED) return s;
    } else {
      cudaStream_t cs = h->comm_stream;
      TSF_CUDA(h, cudaEventRecord(h->ev_f[nc], st));  // x ready
      TSF_CUDA(h, cudaStreamWaitEvent(cs, h->ev_f[nc], 0));
      const View vin{h->K, Hc, Nl, (long long)Nl * H * d, (long long)d, (long long)H * d};
      for (int c = 0; c < nc && s == TSF_OK; ++c) {
        void* peers[MAX_PEERS];
        peers_of(c, peers);
        s = temporal_fused(h, vin, x + (size_t)c * Hc * d, h->rank, peers, cs);
        if (s != TSF_OK) break;
        StageTimer tm(h, cs, 2);
        TSF_NCCL(h, ncclAllReduce(h->d_flag, h->d_flag, 1, ncclInt32, ncclSum, h->comm, cs));
        tm.done();
        TSF_CUDA(h, cudaEventRecord(h->ev_f[c], cs));
      }
      if (s == TSF_OK) {
        for (int c = 0; c < nc && s == TSF_OK; ++c) {
          TSF_CUDA(h, cudaStreamWaitEvent(st, h->ev_f[c], 0));
          s = spatial_shard(h, u, y, nc, c, false, st);
        }
        if (s == TSF_OK) h->fparity ^= 1;
        return s;
      }
      // the comm stream must not run ahead of a fallback on `st`
      TSF_CUDA(h, cudaEventRecord(h->ev_f[nc], cs));
      TSF_CUDA(h, cudaStreamWaitEvent(st, h->ev_f[nc], 0));
      if (s != TSF_ERR_UNSUPPORTED) return s;
    }
    // shapes the fused scatter cannot tile: fall through to the NCCL path
  }
  // Distributed: head-chunk pipeline.  temporal(c) for all chunks on `st`;
  // exchange(c) on the comm stream after temporal(c); unpack(c) + spatial(c)
  // on `st` after exchange(c), so exchange(c+1) overlaps spatial(c).
  const int nc = h->nchunk;
  for (int c = 0; c < nc; ++c) {
    if ((s = temporal_tokens(h, x, h->xt, c, st)) != TSF_OK) return s;
    TSF_CUDA(h, cudaEventRecord(h->ev_t[c], st));
  }
  for (int c = 0; c < nc; ++c) {
    TSF_CUDA(h, cudaStreamWaitEvent(h->comm_stream, h->ev_t[c], 0));
    StageTimer tm(h, h->comm_stream, 2);
    s = exchange_chunk(h, c, h->comm_stream);
    tm.done();
    if (s != TSF_OK) return s;
    TSF_CUDA(h, cudaEventRecord(h->ev_a[c], h->comm_stream));
  }
  for (int c = 0; c < nc; ++c) {
    TSF_CUDA(h, cudaStreamWaitEvent(st, h->ev_a[c], 0));
    if ((s = unpack_chunk(h, h->rxt, h->uxt, c, st)) != TSF_OK) return s;
    if ((s = spatial_shard(h, h->uxt, y, nc, c, true, st)) != TSF_OK) return s;
  }
  return TSF_OK;
}

// one staging slot (device x, y) of the host calls: both or neither allocated
static tsf_status host_slot(tsf_handle* h, __nv_bfloat16** x, float** y, size_t in_bytes, size_t out_bytes) {
  if (*x && *y) return TSF_OK;
  if (!*x && cudaMalloc(x, in_bytes) != cudaSuccess) *x = nullptr;
  if (*x && !*y && cudaMalloc(y, out_bytes) != cudaSuccess) *y = nullptr;
  if (!*x || !*y) {  // a half-done allocation is undone
    if (*x) cudaFree(*x);
    *x = nullptr;
    cudaGetLastError();
    return fail(h, TSF_ERR_NOMEM, "staging cudaMalloc failed");
  }
  return TSF_OK;
}

static tsf_status host_batch_enqueue(tsf_handle* h, const tsf_bf16* const* x_host, float* const* y_host, int n,
                                     void* stream) {
  if (!h) return fail(nullptr, TSF_ERR_CONFIG, "null handle");
  if (n < 0 || (n > 0 && (!x_host || !y_host))) return fail(h, TSF_ERR_CONFIG, "need n >= 0 and pointer arrays");
  for (int i = 0; i < n; ++i)
    if (!x_host[i] || !y_host[i]) return fail(h, TSF_ERR_CONFIG, "null host buffer");
  if (n == 0) return TSF_OK;
  const int P = h->world, Nl = h->N / P, Kl = h->K / P;
  const int V = h->sim ? P : 1;
  const size_t in_bytes = (size_t)h->K * Nl * h->H * h->d * 2 * V;
  const size_t out_bytes = (size_t)Kl * h->N * h->H * h->d * 4 * V;
  tsf_status s = host_slot(h, &h->xdev, &h->ydev, in_bytes, out_bytes);
  if (s == TSF_OK && n > 1) s = host_slot(h, &h->xdev2, &h->ydev2, in_bytes, out_bytes);
  if (s != TSF_OK) return s;
  if (!h->copy_stream) {
    TSF_CUDA(h, cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
    TSF_CUDA(h, cudaStreamCreateWithFlags(&h->h2d_stream, cudaStreamNonBlocking));
    h->ev_h.resize(HOST_CHUNKS + 1 + 6);
    for (auto& e : h->ev_h) TSF_CUDA(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t* ev_chunk = h->ev_h.data();                 // [HOST_CHUNKS]
  cudaEvent_t ev_done = h->ev_h[HOST_CHUNKS];
  cudaEvent_t* ev_in = h->ev_h.data() + HOST_CHUNKS + 1;  // [2] x of slot b on the device
  cudaEvent_t* ev_used = ev_in + 2;                       // [2] the block has read x of slot b
  cudaEvent_t* ev_out = ev_in + 4;                        // [2] y of slot b is on the host
  // Pipeline over two device slots (item i uses slot i & 1):
  //   h2d_stream:  H2D x_i  (after the block of item i-2 has read the slot)
  //   stream:      block i  (after H2D x_i and after D2H y_{i-2} has drained the slot)
  //   copy_stream: D2H y_i  (single GPU: per frame chunk, as soon as the chunk is computed)
  // so H2D of item i+1 and D2H of item i run concurrently in the two PCIe directions and
  // the blocks hide behind them.  Every cross-stream wait is issued right after the record
  // it refers to, so reusing the events across items is exact.
  TSF_CUDA(h, cudaEventRecord(ev_done, st));              // prior work on `stream` before any staging reuse
  TSF_CUDA(h, cudaStreamWaitEvent(h->h2d_stream, ev_done, 0));
  TSF_CUDA(h, cudaStreamWaitEvent(h->copy_stream, ev_done, 0));
  for (int i = 0; i < n; ++i) {
    const int b = i & 1;
    __nv_bfloat16* xd = b ? h->xdev2 : h->xdev;
    float* yd = b ? h->ydev2 : h->ydev;
    if (i >= 2) TSF_CUDA(h, cudaStreamWaitEvent(h->h2d_stream, ev_used[b], 0));
    {
      StageTimer tm(h, h->h2d_stream, 3);
      TSF_CUDA(h, cudaMemcpyAsync(xd, x_host[i], in_bytes, cudaMemcpyHostToDevice, h->h2d_stream));
      tm.done();
    }
    TSF_CUDA(h, cudaEventRecord(ev_in[b], h->h2d_stream));
    TSF_CUDA(h, cudaStreamWaitEvent(st, ev_in[b], 0));
    if (i >= 2) TSF_CUDA(h, cudaStreamWaitEvent(st, ev_out[b], 0));
    if (P == 1 && h->K >= 2) {
      // temporal stage whole (it needs every frame of a token), then the spatial
      // stage in frame chunks: chunk c's y goes to the host on copy_stream while
      // chunk c+1 computes (y is frame-major, so a chunk is contiguous)
      h->launches = 0;
      {
        StageTimer tm(h, st, 0);
        s = run_attention(h, temporal_view(h->K, h->N, h->H, h->d), xd, xd, xd, EPI_BLOCK_T, h->xt, nullptr, st);
        tm.done();
        if (s != TSF_OK) return s;
      }
      TSF_CUDA(h, cudaEventRecord(ev_used[b], st));
      const int nch = h->K < HOST_CHUNKS ? h->K : HOST_CHUNKS;
      const size_t frame = (size_t)h->N * h->H * h->d;
      int f0 = 0;
      for (int c = 0; c < nch; ++c) {
        const int f1 = (int)(((long long)h->K * (c + 1)) / nch);
        {
          StageTimer tm(h, st, 1);
          s = run_attention(h, spatial_view(f1 - f0, h->N, h->H, h->d), h->xt + f0 * frame, h->xt + f0 * frame,
                            h->xt + f0 * frame, EPI_BLOCK_S, nullptr, yd + f0 * frame, st);
          tm.done();
          if (s != TSF_OK) return s;
        }
        TSF_CUDA(h, cudaEventRecord(ev_chunk[c], st));
        TSF_CUDA(h, cudaStreamWaitEvent(h->copy_stream, ev_chunk[c], 0));
        TSF_CUDA(h, cudaMemcpyAsync(y_host[i] + f0 * frame, yd + f0 * frame, (f1 - f0) * frame * sizeof(float),
                                    cudaMemcpyDeviceToHost, h->copy_stream));
        f0 = f1;
      }
    } else {
      s = tsf_spacetime_block(h, reinterpret_cast<const tsf_bf16*>(xd), yd, st);
      if (s != TSF_OK) return s;
      TSF_CUDA(h, cudaEventRecord(ev_used[b], st));
      TSF_CUDA(h, cudaStreamWaitEvent(h->copy_stream, ev_used[b], 0));
      StageTimer tm(h, h->copy_stream, 3);
      TSF_CUDA(h, cudaMemcpyAsync(y_host[i], yd, out_bytes, cudaMemcpyDeviceToHost, h->copy_stream));
      tm.done();
    }
    TSF_CUDA(h, cudaEventRecord(ev_out[b], h->copy_stream));
  }
  TSF_CUDA(h, cudaEventRecord(ev_done, h->copy_stream));
  TSF_CUDA(h, cudaStreamWaitEvent(st, ev_done, 0));       // `stream` completes after the last D2H
  TSF_CUDA(h, cudaEventRecord(ev_in[0], h->h2d_stream));  // ... and after the last H2D (the next call's slots)
  TSF_CUDA(h, cudaStreamWaitEvent(st, ev_in[0], 0));
  return tsf_sync(h, st, 0);
}

tsf_status tsf_spacetime_block_host_batch(tsf_handle* h, const tsf_bf16* const* x_host, float* const* y_host, int n,
                                          void* stream) {
  const tsf_status s = host_batch_enqueue(h, x_host, y_host, n, stream);
  if (s != TSF_OK && h) {
    // an error mid-batch: copies already queued on the two copy streams may still
    // read x_host / write y_host -- drain them before the caller gets control back
    if (h->h2d_stream) cudaStreamSynchronize(h->h2d_stream);
    if (h->copy_stream) cudaStreamSynchronize(h->copy_stream);
    cudaGetLastError();
  }
  return s;
}

tsf_status tsf_spacetime_block_host(tsf_handle* h, const tsf_bf16* x_host, float* y_host, void* stream) {
  if (!h) return fail(nullptr, TSF_ERR_CONFIG, "null handle");
  if (!x_host || !y_host) return fail(h, TSF_ERR_CONFIG, "null host buffer");
  return tsf_spacetime_block_host_batch(h, &x_host, &y_host, 1, stream);
}

tsf_status tsf_sync(tsf_handle* h, void* stream, int timeout_ms) {
  if (!h) return fail(nullptr, TSF_ERR_CONFIG, "null handle");
  cudaStream_t st = (cudaStream_t)stream;
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) return fail(h, TSF_ERR_CUDA, std::string("stream: ") + cudaGetErrorString(e));
    tsf_status s = check_comm(h);
    if (s != TSF_OK) return s;
    if (timeout_ms > 0) {
      const double ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      if (ms > timeout_ms) {
        if (h->comm && !h->sim) {  // a peer is gone or hung: abort so the stream drains
          ncclCommAbort(h->comm);
          h->comm = nullptr;
          h->comm_dead = true;
        }
        return fail(h, TSF_ERR_NCCL, "tsf_sync: timeout after " + std::to_string(timeout_ms) + " ms");
      }
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  if (h->nf_host && h->nf_host[1]) {
    h->nf_host[1] = 0u;
    return fail(h, TSF_ERR_NCCL, "fused-exchange peer barrier timed out (a peer rank stopped)");
  }
  if (h->nf_host && *h->nf_host) {
    *h->nf_host = 0u;
    return fail(h, TSF_ERR_NUMERIC,
                "non-finite X_t: |x + T(x)| exceeded the fp16 range of the block intermediate (or x was not finite)");
  }
  return TSF_OK;
}

}  // extern "C"

// The exchange's byte plan for any element size: rank r's shard is shard_bytes;
// its block p (peer_bytes) goes to rank p, which stores it at slot r.  Real
// ranks: one grouped NCCL send/recv round on `st`; simulated ranks (stacked
// shards): device copies.
static tsf_status exchange_bytes(tsf_handle* h, const char* src, char* dst, size_t shard_bytes, size_t peer_bytes,
                                 cudaStream_t st) {
  const int P = h->world;
  if (h->sim) {
    for (int r = 0; r < P; ++r)
      for (int p = 0; p < P; ++p)
        TSF_CUDA(h, cudaMemcpyAsync(dst + p * shard_bytes + r * peer_bytes, src + r * shard_bytes + p * peer_bytes,
                                    peer_bytes, cudaMemcpyDeviceToDevice, st));
    return TSF_OK;
  }
  TSF_NCCL(h, ncclGroupStart());
  for (int p = 0; p < P; ++p) {
    TSF_NCCL(h, ncclSend(src + p * peer_bytes, peer_bytes, ncclUint8, p, h->comm, st));
    TSF_NCCL(h, ncclRecv(dst + p * peer_bytes, peer_bytes, ncclUint8, p, h->comm, st));
  }
  TSF_NCCL(h, ncclGroupEnd());
  return TSF_OK;
}

// Token shard <-> frame shard of a [K, N, H, d] tensor of elem_bytes-sized
// elements (untyped, bit-exact).  scratch: one shard per rank handled.
static tsf_status reshard_gen(tsf_handle* h, int dir, const void* in, void* out, int elem_bytes, void* scratch,
                              cudaStream_t st) {
  const int P = h->world, Kc = h->K / P, Nc = h->N / P;
  const size_t shard = (size_t)h->K * Nc * h->H * h->d * elem_bytes, peer = shard / P;
  const int vecs = h->H * h->d * elem_bytes / 16;
  const long long items = (long long)P * Kc * Nc * vecs;
  const int V = h->sim ? P : 1;
  const char* cin = static_cast<const char*>(in);
  char* cout = static_cast<char*>(out);
  char* sc = static_cast<char*>(scratch);
  tsf_status s;
  if (dir == TSF_T2S) {
    // send frames [p Kc, (p+1) Kc) of the token shard (contiguous); receive
    // [P][Kc][Nc] blocks, unpack to [Kc][N]
    if ((s = exchange_bytes(h, cin, sc, shard, peer, st)) != TSF_OK) return s;
    for (int r = 0; r < V; ++r) {
      reshard_perm_kernel<true><<<grid_for(h, items), 256, 0, st>>>((const uint4*)(sc + r * shard),
                                                                    (uint4*)(cout + r * shard), nullptr, nullptr, P,
                                                                    Kc, Nc, vecs);
      h->launches++;
    }
  } else {
    // pack [Kc][N] -> [P][Kc][Nc], send block p to peer p; the received
    // blocks [P][Kc][Nc] are exactly the token shard [K][Nc]
    for (int r = 0; r < V; ++r) {
      reshard_perm_kernel<false><<<grid_for(h, items), 256, 0, st>>>((const uint4*)(cin + r * shard),
                                                                     (uint4*)(sc + r * shard), nullptr, nullptr, P,
                                                                     Kc, Nc, vecs);
      h->launches++;
    }
    TSF_CUDA(h, cudaGetLastError());
    if ((s = exchange_bytes(h, sc, cout, shard, peer, st)) != TSF_OK) return s;
  }
  TSF_CUDA(h, cudaGetLastError());
  return TSF_OK;
}

extern "C" {

tsf_status tsf_reshard(tsf_handle* h, int dir, const tsf_bf16* in, tsf_bf16* out, void* stream) {
  if (!h) return fail(nullptr, TSF_ERR_CONFIG, "null handle");
  if (dir != TSF_T2S && dir != TSF_S2T) return fail(h, TSF_ERR_CONFIG, "bad direction");
  h->launches = 0;
  const int P = h->world, Kc = h->K / P, Nc = h->N / P;
  const size_t bytes = (size_t)h->K * Nc * h->H * h->d * 2;  // same size both ways (one rank)
  tsf_status s = check_ptrs(h, {in}, out, bytes * (h->sim ? P : 1), bytes * (h->sim ? P : 1));
  if (s != TSF_OK) return s;
  if ((s = check_comm(h)) != TSF_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  StageTimer tm(h, st, 2);
  if (P == 1) {
    TSF_CUDA(h, cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, st));
    tm.done();
    return TSF_OK;
  }
  s = reshard_gen(h, dir, in, out, 2, h->rxt, st);
  tm.done();
  return s;
}

#ifdef TSF_TRACE
// Diagnostics only (not in tsf.h): copy the clock64 stamps of CTA 0 of the last
// traced launch (16 warps x TRACE_PER_WARP entries).
int tsf_trace_read(tsf_handle* h, unsigned long long* host, int n) {
  if (!h || !h->trace) return -1;
  const int cap = 32 * TRACE_PER_WARP;
  if (n > cap) n = cap;
  cudaMemcpy(host, h->trace, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaMemset(h->trace, 0, cap * sizeof(unsigned long long));
  return n;
}
#endif

tsf_status tsf_transpose(tsf_handle* h, int A, int B, const tsf_bf16* in, tsf_bf16* out, void* stream) {
  if (!h) return fail(nullptr, TSF_ERR_CONFIG, "null handle");
  if (A < 1 || B < 1) return fail(h, TSF_ERR_CONFIG, "A, B must be >= 1");
  h->launches = 0;
  const size_t bytes = (size_t)A * B * h->H * h->d * 2;
  tsf_status s = check_ptrs(h, {in}, out, bytes, bytes);
  if (s != TSF_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  const int vecs = h->H * h->d * 2 / 16;
  StageTimer tm(h, st, 4);
  static int variant = -1;
  if (variant < 0) {
    const char* e = getenv("TSF_TRANSPOSE");
    variant = e ? atoi(e) : 1;
  }
  if (variant == 1)
    transpose_rows_ilp_kernel<<<grid_for(h, ((long long)A * B * vecs + 3) / 4), 256, 0, st>>>(
        (const uint4*)in, (uint4*)out, A, B, vecs);
  else
    transpose_rows_kernel<<<grid_for(h, (long long)A * B * vecs), 256, 0, st>>>((const uint4*)in, (uint4*)out,
                                                                                 nullptr, nullptr, A, B, vecs);
  TSF_CUDA(h, cudaGetLastError());
  tm.done();
  h->launches++;
  return TSF_OK;
}

}  // extern "C"
