/*
 * tsf.h -- C ABI of libtsf.so: TimeSformer-style factorized ("divided")
 * space-time attention on NVIDIA B200 (sm_100a).
 *
 * What it computes (Sec. I): "temporal attention at each
 * spatial location ... followed by spatial attention at each time frame",
 * per-layer cost O(K^2 N + K N^2) (Fig. 1 caption, Table I), in
 * place of joint attention over all K*N tokens.  A token is one
 * spatial patch of one frame; K frames x N tokens per frame.
 *
 * Layout.  Every tensor is row-major [K, N, H, d] (frames, tokens per frame,
 * heads, head dim; d fastest), contiguous, in device memory unless the
 * function name ends in _host.  bf16 tensors are passed as tsf_bf16 (the raw
 * 16-bit pattern, e.g. torch.bfloat16 storage).  The softmax scale is
 * 1/sqrt(d) (reading G4); there are no projections (reading G1).
 *
 * Ownership.  The caller owns every input/output buffer; they must be
 * 16-byte aligned and outputs must not overlap inputs.  The handle owns its
 * workspace (allocated in tsf_create*, no allocation in the call path except
 * the one-time staging buffers of tsf_spacetime_block_host) and, for
 * distributed handles, its NCCL communicator.
 *
 * Streams.  `stream` is a cudaStream_t (NULL = legacy default stream).  All
 * calls are asynchronous on that stream, except tsf_spacetime_block_host which
 * synchronises it before returning.  A handle is not thread-safe; use one
 * handle per stream.  Results are deterministic: the same inputs give the same
 * bits on every run.
 *
 * Errors.  Arguments are validated synchronously before anything is enqueued;
 * no exception crosses the ABI.  tsf_last_error() describes the last failure
 * of a handle (or of handle creation when called with NULL).
 */
#ifndef TSF_H_
#define TSF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef uint16_t tsf_bf16;            /* bf16 bit pattern */
typedef struct tsf_handle tsf_handle; /* opaque */

typedef enum {
  TSF_OK = 0,
  TSF_ERR_CONFIG = 2,      /* bad size, null/misaligned/aliased pointer, K%P or N%P != 0 */
  TSF_ERR_NUMERIC = 3,     /* non-finite block intermediate X_t (fp16 overflow or non-finite x), see tsf_sync */
  TSF_ERR_UNSUPPORTED = 4, /* d not in {32, 64, 128}, or device is not sm_100 */
  TSF_ERR_CUDA = 5,        /* CUDA runtime/driver failure (launch, copy, tensor map) */
  TSF_ERR_NCCL = 6,        /* NCCL failure, or a peer rank stopped (fused-exchange barrier timeout) */
  TSF_ERR_NOMEM = 7        /* workspace allocation failed */
} tsf_status;

enum { TSF_T2S = 0, TSF_S2T = 1 }; /* reshard directions */

/* masks of tsf_joint_attn over the flattened tokens (t, n) -> t*N + n */
enum {
  TSF_MASK_NONE = 0,          /* global attention over all K*N tokens (Table I "ViT (global)" P:73) */
  TSF_MASK_TEMPORAL = 1,      /* [n' == n]: equals tsf_temporal_attn (block-mask check, pin I1) */
  TSF_MASK_SPATIAL = 2,       /* [t' == t]: equals tsf_spatial_attn (pin I1) */
  TSF_MASK_CAUSAL_FRAMES = 3  /* [t' <= t]: causal in time, global in space (SURVEY NEXT-4 variant;
                                 the paper's temporal context is non-causal) */
};

/* Create a single-GPU handle for a [K, N, H, d] layer on the current CUDA
 * device.  K, N, H >= 1; d in {32, 64, 128}.  Allocates the block workspace
 * (X_t in fp16, 2*K*N*H*d bytes). */
tsf_status tsf_create(int K, int N, int H, int d, tsf_handle** out);

/* Temporal attention ("at each spatial location"): for every (n, h),
 *   o[t,n,h,:] = sum_t' softmax_t'(<q[t,n,h,:], k[t',n,h,:]> / sqrt(d)) v[t',n,h,:].
 * q, k, v, o: bf16 [K, Nl, H, d] with Nl = N (single GPU) or N/P (distributed
 * handle: the rank's token shard).  Accumulation in fp32; o rounded to bf16. */
tsf_status tsf_temporal_attn(tsf_handle* h, const tsf_bf16* q, const tsf_bf16* k, const tsf_bf16* v,
                             tsf_bf16* o, void* stream);

/* Spatial attention ("at each time frame"): for every (t, h),
 *   o[t,n,h,:] = sum_n' softmax_n'(<q[t,n,h,:], k[t,n',h,:]> / sqrt(d)) v[t,n',h,:].
 * q, k, v, o: bf16 [Kl, N, H, d] with Kl = K or K/P (the rank's frame shard). */
tsf_status tsf_spatial_attn(tsf_handle* h, const tsf_bf16* q, const tsf_bf16* k, const tsf_bf16* v,
                            tsf_bf16* o, void* stream);

/* Joint (global) attention over all L = K*N tokens of each head -- the
 * O((K N)^2) regime the factorization avoids (Table I):
 *   o[i,h,:] = sum_j softmax_j(<q[i,h,:], k[j,h,:]> / sqrt(d) + M[i,j]) v[j,h,:],
 * i, j over the flattened tokens (t, n) -> t*N + n, M = 0 where the mask
 * allows and -inf elsewhere (mask = TSF_MASK_*).  Every score is computed
 * (masked tiles are not skipped: this is the cost the factorization removes);
 * with TSF_MASK_TEMPORAL / _SPATIAL the result equals the factorized stages
 * (a GPU-side block-mask check).  q, k, v, o: bf16 [K, N, H, d]; fp32
 * accumulation; o rounded to bf16.  Single-GPU handles only
 * (TSF_ERR_UNSUPPORTED otherwise); K*N < 2^31. */
tsf_status tsf_joint_attn(tsf_handle* h, const tsf_bf16* q, const tsf_bf16* k, const tsf_bf16* v, tsf_bf16* o,
                          int mask, void* stream);

/* STORM per-layer attention (sec. IV-B):
 * spatial self-attention on the current state plus cross-attention to M
 * compressed history tokens, mixed by the noise gate g(sigma), identity
 * projections (reading G1):
 *   y[b] = u[b] + (1 - g) S(u[b], u[b], u[b]) + g C(u[b], ctx[b], ctx[b]),
 *   g = sigma^2 / (sigma^2 + sigma_data^2)   (reading G18),
 * S = softmax attention over the N tokens of u[b] (per head), C = attention of
 * those N queries over the M context tokens of ctx[b] (per head), scale
 * 1/sqrt(d).  The handle's K is the number B of independent states.
 * u: bf16 [K, N, H, d]; ctx: bf16 [K, M, H, d], M >= 1; y: fp32 [K, N, H, d].
 * bf16 operands and P, fp32 accumulation; y must not overlap u or ctx.
 * sigma >= 0 and finite, sigma_data > 0 (else TSF_ERR_CONFIG).  Two launches
 * (cross writes y, self adds into it).  Single-GPU handles only. */
tsf_status tsf_storm_attn(tsf_handle* h, const tsf_bf16* u, const tsf_bf16* ctx, int M, double sigma,
                          double sigma_data, float* y, void* stream);

/* Parameters of the full TimeSformer divided block (tsf_full_block), device
 * pointers.  D = H*d, F = MLP hidden size.  Weights bf16 in the [out, in]
 * layout (nn.Linear), biases and LayerNorm gains/shifts fp32. */
typedef struct {
  const float* ln_t_g; const float* ln_t_b;          /* [D]: pre-LN of the temporal stage */
  const tsf_bf16* w_qkv_t; const float* b_qkv_t;     /* [3D, D], [3D]: rows q | k | v */
  const tsf_bf16* w_o_t; const float* b_o_t;         /* [D, D], [D] */
  const float* ln_s_g; const float* ln_s_b;          /* spatial stage, same shapes */
  const tsf_bf16* w_qkv_s; const float* b_qkv_s;
  const tsf_bf16* w_o_s; const float* b_o_s;
  const float* ln_m_g; const float* ln_m_b;          /* [D]: pre-LN of the MLP */
  const tsf_bf16* w_1; const float* b_1;             /* [F, D], [F] */
  const tsf_bf16* w_2; const float* b_2;             /* [D, F], [D] */
  int F;
} tsf_block_weights;

/* Full TimeSformer divided space-time block (the layers around
 * the factorized attention of P:64, reading G21 in DESIGN.md):
 *   (q,k,v) = split(LN_t(x) Wqkv_t^T + b);   X_t = x + T(q,k,v) Wo_t^T + bo_t
 *   (q,k,v) = split(LN_s(X_t) Wqkv_s^T + b); X_s = X_t + S(q,k,v) Wo_s^T + bo_s
 *   y = X_s + GELU(LN_m(X_s) W1^T + b1) W2^T + b2
 * x: bf16 [K, N, H, d] (= [K*N, D] tokens); y: fp32 [K, N, H, d].  Residual
 * stream fp32; LN outputs, q/k/v, attention outputs and the GELU output bf16;
 * every GEMM bf16 x bf16 -> fp32 on tcgen05 with the bias / GELU / residual
 * fused into its epilogue; attention = the tsf_temporal_attn /
 * tsf_spatial_attn kernels reading q, k, v in place from the QKV GEMM output.
 * Needs D % 128 == 0, F % 128 == 0, D <= 8192; single-GPU handles.  The
 * first call allocates the activation workspace (~2*T*(4D + F) bytes + 8*T*D
 * for T = K*N tokens), kept until tsf_destroy. */
tsf_status tsf_full_block(tsf_handle* h, const tsf_block_weights* w, const tsf_bf16* x, float* y, void* stream);

/* Backward of the attention stages (the paper's TimeSformer
 * numbers are training runs).  For the forward
 * o = softmax(s q k^T) v of tsf_temporal_attn / tsf_spatial_attn (s = 1/sqrt d)
 * and the output gradient dO:
 *   dv = P^T dO,  dS = P (dO v^T - rowsum(dO o)),  dq = s dS k,  dk = s dS^T q.
 * P is recomputed (a forward pass that also yields the row statistics), then
 * one kernel per 128-key tile accumulates dk, dv in TMEM and adds dq into an
 * fp32 buffer.  All tensors bf16 [K, N, H, d]; fp32 accumulation; outputs must
 * not overlap inputs or each other.  d in {32, 64, 128}.  On a distributed
 * (or simulated) handle the call acts on the rank's own shard, like the
 * forward stage calls: temporal on the token shard [K, N/P, H, d], spatial on
 * the frame shard [K/P, N, H, d]; no exchange.  dq is summed with fp32 atomic
 * adds across key tiles, so results can differ run to run in the last bits
 * (G22).  Workspace allocated on first use. */
tsf_status tsf_temporal_attn_bwd(tsf_handle* h, const tsf_bf16* q, const tsf_bf16* k, const tsf_bf16* v,
                                 const tsf_bf16* dO, tsf_bf16* dq, tsf_bf16* dk, tsf_bf16* dv, void* stream);
tsf_status tsf_spatial_attn_bwd(tsf_handle* h, const tsf_bf16* q, const tsf_bf16* k, const tsf_bf16* v,
                                const tsf_bf16* dO, tsf_bf16* dq, tsf_bf16* dk, tsf_bf16* dv, void* stream);

/* Backward of tsf_spacetime_block: dx (fp32) for x (bf16) and dy (fp32).
 * Single GPU: all [K, N, H, d].  Distributed handle: x and dx are the rank's
 * token shard [K, N/P, H, d], dy its frame shard [K/P, N, H, d], and the
 * exchange runs in reverse (X_t token -> frame shard, then dX_t frame ->
 * token shard as fp32 bytes); simulated handles take all shards stacked.
 * Collective on distributed handles.  Gradient:   dX_t = dy + (dq + dk + dv of S at X_t),  dx = dX_t + (dq + dk +
 * dv of T at x)  (q = k = v in each stage).  X_t is recomputed in bf16 (the
 * training precision; the forward keeps it in fp16, reading G8), so dx
 * carries bf16-level error (tests: rel-L2 <= 1e-2).  dx fp32. */
tsf_status tsf_spacetime_block_bwd(tsf_handle* h, const tsf_bf16* x, const float* dy, float* dx, void* stream);

/* Divided space-time block, temporal then spatial ("followed by"), with
 * identity projections and residual weight 1 (readings G1, G5):
 *   X_t = x + T(x, x, x);   y = X_t + S(X_t, X_t, X_t).
 * x: bf16.  y: fp32.  X_t is kept in fp16 (11-bit mantissa, reading G8): the
 * spatial stage's MMAs read it (with fp16 P) and the residual adds it.
 * Range: |X_t| must stay below 65504 (fp16), e.g. |x| < 32752.  The temporal
 * epilogue checks every stored X_t element; a non-finite one (overflow, or a
 * non-finite x) sets the handle's flag, reported as TSF_ERR_NUMERIC by the next
 * tsf_sync (and by tsf_spacetime_block_host, which synchronises).  y is then
 * not meaningful.
 * Single GPU: x, y are [K, N, H, d].  Distributed: x is the token shard
 * [K, N/P, H, d], y the frame shard [K/P, N, H, d]; X_t is resharded between
 * the stages bit-exactly: by default the temporal kernel stores its rows
 * straight into the owning ranks' frame shards over NVLink (CUDA IPC) and a
 * peer-memory barrier orders the stores before the spatial stage; NCCL byte
 * send/recv plus an unpack kernel where that is unavailable
 * (TSF_FUSED_EXCHANGE=0, or shapes the fused scatter does not cover). */
tsf_status tsf_spacetime_block(tsf_handle* h, const tsf_bf16* x, float* y, void* stream);

/* Same as tsf_spacetime_block with HOST buffers (pinned memory recommended):
 * copies x host->device, runs the block, copies y device->host and
 * synchronises `stream`.  Staging buffers (and, single GPU, a copy stream)
 * are allocated on first use.  Single GPU: the spatial stage runs in up to 4
 * frame chunks and each chunk's y is copied out while the next one computes;
 * the result is bitwise the device call's. */
tsf_status tsf_spacetime_block_host(tsf_handle* h, const tsf_bf16* x_host, float* y_host, void* stream);

/* n independent blocks from HOST buffers: y_host[i] = block(x_host[i]) for
 * i < n, each pair shaped as in tsf_spacetime_block_host (pinned memory
 * needed for overlap).  Pipelined through two device staging slots (allocated
 * on first use, 2 x (x + y) bytes): the host->device copy of x_{i+1}, the
 * block of item i and the device->host copy of y_i run concurrently (separate
 * copy streams, one per PCIe direction), so a batch costs about
 * max(H2D, D2H) per item instead of their sum.  Returns after `stream` has
 * synchronised (all y_host written); host buffers must stay valid until then.
 * Each y_host[i] is bitwise what tsf_spacetime_block_host gives for
 * x_host[i].  n = 0 is a no-op; a null array or element is TSF_ERR_CONFIG.
 * On any error the call returns only after the copies it queued have drained
 * (the host buffers are free again); a non-finite X_t in any item is
 * TSF_ERR_NUMERIC, as for tsf_spacetime_block_host.
 * Collective on distributed handles (every rank passes the same n). */
tsf_status tsf_spacetime_block_host_batch(tsf_handle* h, const tsf_bf16* const* x_host, float* const* y_host, int n,
                                          void* stream);

/* Wait for `stream` and report what the asynchronous work found:
 *   TSF_ERR_NUMERIC  a block since the last tsf_sync stored a non-finite X_t
 *                    (the flag is cleared);
 *   TSF_ERR_NCCL     (distributed handles) NCCL reported an asynchronous error
 *                    while waiting, or timeout_ms > 0 elapsed first: then the
 *                    communicator is aborted (a dead or hung peer cannot hang
 *                    this rank forever) and later collective calls on h fail;
 *                    or the fused exchange's peer-memory barrier waited 10 s
 *                    for a peer that never arrived (the ranks' barrier epochs
 *                    are then out of step: destroy the handle);
 *   TSF_ERR_CUDA     the stream reported a CUDA error.
 * timeout_ms <= 0 waits without a limit.  Polls the stream (no blocking sync). */
tsf_status tsf_sync(tsf_handle* h, void* stream, int timeout_ms);

/* Release the workspace (and the NCCL communicator of a distributed handle;
 * aborted instead of destroyed if it reports an asynchronous error). */
void tsf_destroy(tsf_handle* h);

/* ---- distributed (one process per GPU, NCCL over NVLink/NVSwitch) ---- */

/* Fill id128 (128 bytes) with a new NCCL unique id.  Call on rank 0 and
 * broadcast the bytes to the other ranks (the Python binding uses the torch
 * process group). */
tsf_status tsf_get_unique_id(void* id128);

/* Collective over `world` ranks: create a distributed handle on the current
 * device.  Requires K % world == 0 and N % world == 0. */
tsf_status tsf_create_dist(int K, int N, int H, int d, const void* id128, int rank, int world,
                           tsf_handle** out);

/* One-GPU simulation of P ranks (validation of the distributed path without P
 * GPUs; BASELINE.json north_star: "the all-to-all reshard must be bit-exact").
 * The handle runs every virtual rank's share of the distributed block on the
 * current device with the same code as tsf_create_dist handles: the same
 * kernels, output routing and per-destination tensor maps, the same byte plan
 * and unpack kernel.  Only the transport differs: the ranks' buffers are local
 * and device copies stand in for NCCL send/recv.  exchange_mode: 1 = NCCL byte
 * plan (send/recv + unpack), 2 = fused scatter (the temporal kernel stores X_t
 * rows into every rank's frame shard).  2 <= P <= 8, K % P == N % P == 0.
 * On such a handle the calls take ALL virtual ranks' shards back to back:
 *   tsf_spacetime_block: x = [P][K][N/P][H][d] (rank r's token shard at
 *     r*K*(N/P)*H*d), y = [P][K/P][N][H][d] (= the full frame-major [K,N,H,d]);
 *   tsf_reshard: the same stacking of token and frame shards.
 * tsf_temporal_attn / tsf_spatial_attn act on one shard (rank 0's shapes). */
tsf_status tsf_create_sim(int K, int N, int H, int d, int P, int exchange_mode, tsf_handle** out);

/* Reshard a bf16 tensor between the two shardings (pure data movement,
 * bit-exact): TSF_T2S: in = token shard [K, N/P, H, d] -> out = frame shard
 * [K/P, N, H, d]; TSF_S2T: the inverse.  Collective over all ranks. */
tsf_status tsf_reshard(tsf_handle* h, int dir, const tsf_bf16* in, tsf_bf16* out, void* stream);

/* ---- layout kernels (HBM-bound, 16-byte vectors) ---- */

/* Frame-major <-> token-major transpose of a bf16 [A, B, H, d] tensor into
 * [B, A, H, d] (A = K, B = N for frame->token; swap for the inverse).  The
 * attention kernels read both orders directly through TMA views, so the block
 * never needs it; it is exported for callers whose data is token-major. */
tsf_status tsf_transpose(tsf_handle* h, int A, int B, const tsf_bf16* in, tsf_bf16* out, void* stream);

/* ---- introspection ---- */

/* Last error message of h (or of the last failed create when h is NULL). */
const char* tsf_last_error(const tsf_handle* h);

/* Number of kernels the last tsf_* compute call launched (bench accounting). */
int tsf_last_launch_count(const tsf_handle* h);

/* How a distributed handle moves X_t between the stages: 0 single GPU (no
 * exchange), 1 NCCL grouped send/recv + unpack kernel, 2 fused NVLink scatter
 * (the temporal kernel stores rows into every rank's frame shard through CUDA
 * IPC mappings; a 1-int NCCL all-reduce orders the stores).  Shapes the fused
 * scatter cannot tile use mode 1 per call.  Returns -1 for NULL. */
int tsf_exchange_mode(const tsf_handle* h);

/* Number of ranks of h (1 single GPU; P distributed or simulated); -1 for NULL. */
int tsf_world_size(const tsf_handle* h);

/* Stage timing with CUDA events recorded on the call's stream around each
 * stage's kernel(s).  tsf_set_timing(h, 1) starts recording (clearing earlier
 * records), 0 stops.  tsf_stage_ms synchronises on the recorded events and
 * returns the summed milliseconds and the number of recorded launches of
 * stage 0 = temporal attention, 1 = spatial attention, 2 = reshard
 * (all-to-all + unpack), 3 = host<->device copies, 4 = tsf_transpose,
 * 5 = tsf_joint_attn, 6 = tsf_storm_attn, 7 = tsf_full_block GEMMs and
 * LayerNorms (its attention kernels are recorded as stages 0 and 1),
 * 8 = the backward calls. */
tsf_status tsf_set_timing(tsf_handle* h, int enable);
tsf_status tsf_stage_ms(tsf_handle* h, int stage, float* total_ms, int* n_records);

#ifdef __cplusplus
}
#endif
#endif /* TSF_H_ */
