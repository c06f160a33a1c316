/* mux.h — C ABI of libmux: MuxTune's spatially multiplexed LoRA linear layer
 * (arXiv 2603.02885) on B200 (sm_100a).
 *
 * Citations: P:n = PAPER.md line n (the paper's LaTeX source).
 *
 * Operations
 *   mux_pack_chunks  chunk-based data alignment, P:833-843 (§3.5): per-task
 *                    packing of sequences, partition of packs into
 *                    equal power-of-two chunks with KV-reuse dependency links
 *                    (P:837-838), chunk size rule.
 *   mux_pack_apply   gathers token-major rows into the packed row layout
 *                    (the "Dispatch" sub-module), zero-filling pad rows.
 *   mux_linear_fwd   BaseOp forward spatially batched over all segments,
 *                    Eq. 1, plus each segment's LoRA adapter
 *                    (north_star:  Y_t += s_t (X_t A_t^T) B_t^T ), fused
 *                    "horizontally" per hTask.
 *   mux_linear_bwd   BaseOp backward Eq. 2 plus the LoRA chain
 *                    rule: dX = dY W + s_t (dY B_t) A_t, dA_t, dB_t; no
 *                    backbone weight gradient (frozen backbone).
 *   Decoder-block ops around the linears (NEXT-3; LLaMA, the backbones of
 *   the paper's workloads):
 *   mux_pack_row_start  per packed row, the first row of its sequence
 *   mux_attn_fwd/bwd    causal attention inside packed sequences: the chunk
 *                       dependency "KV cache reuse in causal attention"
 *                       (Fig. alignment), masked per sequence
 *
 *   mux_rope            rotary position embedding at in-sequence positions
 *   mux_rmsnorm_fwd/bwd, mux_swiglu_fwd/bwd, mux_add (residual)
 *
 * Conventions (all functions)
 *   - Pointers are DEVICE pointers unless marked [host].  The caller owns
 *     every buffer; the library never allocates, frees or synchronizes.
 *   - Every call only enqueues work on `stream` (graph-capturable: no host
 *     reads of device data) and returns.
 *   - Outputs are overwritten (beta = 0), inputs never written, outputs must
 *     not alias inputs.
 *   - Host-side validation runs before any launch: on failure nothing is
 *     launched, outputs are untouched, the status is returned and
 *     mux_last_error() holds a thread-local message.
 *   - Layouts: row-major.  X [max_rows, K], W [N, K] (nn.Linear.weight),
 *     A_t [rank, K] (PEFT lora_A.weight), B_t [N, rank] (lora_B.weight),
 *     Y [max_rows, N], Hs [max_rows, r_cap], dY [max_rows, N], dX [max_rows, K].
 *   - bf16 storage, fp32 accumulation; Hs/Gs are rounded to bf16; dA/dB fp32.
 *   - A segment is the contiguous row range [seg_off[s], seg_off[s+1]) owned
 *     by adapter seg_task[s]; several segments may share an adapter (its
 *     gradients are then summed over all of them).
 */
#ifndef MUX_H_
#define MUX_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime.h>

#if defined(__GNUC__)
#define MUX_API __attribute__((visibility("default")))
#else
#define MUX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* bf16 tensors are passed as raw 16-bit patterns (bit-compatible with CUDA's
 * __nv_bfloat16 and torch.bfloat16), so the header is plain C. */
typedef uint16_t mux_bf16;

#define MUX_MAX_SEGMENTS 64   /* per linear call (kernel parameter block <= 32 KB) */
#define MUX_MAX_ADAPTERS 64
#define MUX_RS_MAX_WORLD 8    /* ranks of a fused reduce-scatter (one 8-GPU NVSwitch box) */
#define MUX_MAX_RANK 64        /* LoRA ranks up to 64 in the paper's workloads */
#define MUX_MAX_SLICES 4       /* column slices of one fused projection (q|k|v, gate|up) */
#define MUX_MAX_ROWS 524288    /* max_rows of a linear call (the workspace's fixed row-block flag region) */
#define MUX_MAX_ADAPTER_SLOTS 96  /* num_adapters * num_slices per call (kernel parameter block) */

typedef enum {
  MUX_OK = 0,
  MUX_ERR_INVALID_ARGUMENT = 1,
  MUX_ERR_UNSUPPORTED = 2,
  MUX_ERR_INSUFFICIENT_BUFFER = 3,
  MUX_ERR_CUDA = 4
} mux_status;

/* Thread-local message describing the last non-OK status of this thread. */
MUX_API const char* mux_last_error(void);

/* Library version string, e.g. "mux 0.1 sm_100a". */
MUX_API const char* mux_version(void);

/* ------------------------------------------------------------------ packing */

/* Written by mux_pack_chunks (device struct).
 *   chunk_size   c actually used (P:843 rule or the caller's value)
 *   num_chunks   chunks emitted; total_rows = num_chunks * c = seg_off[M]
 *   num_packs    packs over all tasks
 *   valid_rows   sum of sequence lengths (effective tokens)
 *   zero_pad_rows  rows the zero-pad-to-global-max strategy would execute
 *                (num_seqs * max length, reported for comparison)
 *   overflow     0 = ok; bit 1: total_rows > max_rows; bit 2: num_chunks >
 *                max_chunks; bit 4: invalid device data (a length < 1 or a
 *                capacity below a task's longest sequence).  When nonzero
 *                nothing but this struct is written. */
typedef struct {
  int32_t chunk_size, num_chunks, num_packs, total_rows, valid_rows, zero_pad_rows, overflow;
} mux_pack_info;

/* [host] Worst-case packed rows for a call (every sequence alone in its own
 * pack and rounded up to the largest possible chunk): lets the caller size
 * max_rows without reading device data.  chunk_size_or_max = the explicit
 * chunk size, or an upper bound on the rule's result (e.g. max capacity). */
MUX_API int64_t mux_pack_bound_rows(int64_t total_tokens, int32_t num_seqs, int32_t chunk_size_or_max);

/* Bytes of device workspace mux_pack_chunks needs. */
MUX_API size_t mux_pack_workspace_size(int32_t num_tasks, int32_t num_seqs);

/* Chunk-based alignment of one hTask.
 *   num_tasks M >= 1, num_seqs >= 0                             [host]
 *   task_seq_off [M+1]  CSR over seq_len, task-major caller order; a task may be empty
 *   seq_len [num_seqs]  each >= 1
 *   pack_capacity [M]   per-task pack capacity >= the task's longest sequence,
 *                       or NULL = round_up(max(max len_t, c), c)
 *   chunk_size          [host] 0 = rule of P:843: c = max(chunk_min, 2^{min_s v2(len_s)});
 *                       else a power of two >= 64
 *   chunk_min           [host] power of two >= 64 ("minimum threshold (typically 64)")
 *   max_rows, max_chunks [host] capacities of row_src and of the chunk table
 * Packing (reading Q5 in DESIGN.md): first-fit decreasing per task, sequences
 * visited by (length desc, index asc), each into the lowest-index pack with
 * room; chunks numbered task-major, then pack-creation order; row of chunk =
 * id * c; seg_off[t] = first row of task t.
 * Outputs: seg_off [M+1]; seq_row [num_seqs] (packed row of each sequence's
 * token 0); chunk_task/chunk_pack/chunk_valid/chunk_dep [max_chunks] (dep =
 * previous chunk of the same pack, -1 = none: the KV-reuse link of P:838);
 * row_src [max_rows] (source token index, token = concatenation of sequences
 * in (task, caller) order; -1 = pad or unused); info.
 * Errors: MUX_ERR_INVALID_ARGUMENT (host-checkable arguments),
 * MUX_ERR_INSUFFICIENT_BUFFER (workspace too small), MUX_ERR_CUDA.
 * Device-data problems are reported in info->overflow (see above). */
MUX_API mux_status mux_pack_chunks(int32_t num_tasks, int32_t num_seqs,
                           const int32_t* task_seq_off, const int32_t* seq_len,
                           const int32_t* pack_capacity, int32_t chunk_size, int32_t chunk_min,
                           int32_t max_rows, int32_t max_chunks,
                           int32_t* seg_off, int32_t* seq_row,
                           int32_t* chunk_task, int32_t* chunk_pack, int32_t* chunk_valid,
                           int32_t* chunk_dep, int32_t* row_src, mux_pack_info* info,
                           void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* Dispatch: dst[r, :] = src[row_src[r], :] if row_src[r] >= 0 else 0, for
 * r < max_rows.  src [num_tokens, cols], dst [max_rows, cols] bf16;
 * cols a multiple of 8, pointers 16-byte aligned.  Indices >= num_tokens
 * are treated as pad (0). */
MUX_API mux_status mux_pack_apply(int32_t max_rows, int32_t cols, int32_t num_tokens,
                          const int32_t* row_src, const mux_bf16* src,
                          mux_bf16* dst, cudaStream_t stream);

/* ------------------------------------------------------------------ linear */

/* One adapter (task) of a linear layer.  [host] array; the pointers inside
 * are device pointers. */
typedef struct {
  const mux_bf16* A;  /* [rank, K] row-major (lora_A.weight) */
  const mux_bf16* B;  /* [N, rank] row-major (lora_B.weight) */
  float* dA;               /* [rank, K] fp32, overwritten by bwd; NULL = skip */
  float* dB;               /* [N, rank] fp32, overwritten by bwd; NULL = skip */
  int32_t rank;            /* 0 (no adapter on this layer) .. 64 */
  int32_t ldb;             /* leading dimension (elements) of B: 0 = rank; must be a
                              multiple of 8 (16-byte rows for TMA), so ranks that are
                              not multiples of 8 need a padded B (columns >= rank are
                              never read).  dB is always [N, rank] contiguous. */
  float scale;             /* s_t (LoRA alpha_t / rank_t, computed by the caller) */
} mux_adapter;

/* Bytes of device workspace mux_linear_fwd / mux_linear_bwd need.  The
 * workspace must be zero-filled once before its first use; it may then be
 * reused by any number of calls on the same stream, with any max_rows <=
 * MUX_MAX_ROWS and r_cap (it carries a fixed-size region of per-row-block
 * shrink flags that every launch leaves reset, and an epoch-tagged stream-K
 * flag set, so no per-call reset is needed), but must not be shared by calls
 * that can run concurrently. */
MUX_API size_t mux_linear_workspace_size(int32_t num_segs, int32_t max_rows, int32_t K, int32_t N,
                                 int32_t r_cap);

/* Forward (Eq. 1 + LoRA).  For every row i of segment s, t = seg_task[s]:
 *   Y[i,:]  = X[i,:] W^T + s_t (X[i,:] A_t^T) B_t^T
 *   Hs[i,j] = bf16(s_t * X[i,:] A_t[j,:]^T) for j < rank_t, 0 for rank_t <= j < r_cap
 * Arguments
 *   num_segs S (1..64) [host]; seg_off [S+1] device, non-decreasing, every
 *   entry a multiple of 64 (mux_pack_chunks guarantees it; the host cannot
 *   check device data without a sync: a -DMUX_DEBUG_CHECKS build checks it on
 *   the device and traps), seg_off[S] <=
 *   max_rows; seg_task [S] [host] adapter index per segment;
 *   num_adapters (1..64), adapters [host];
 *   K, N multiples of 8 (e.g. 11008/8 = 1376 for an 8-way tensor-parallel shard);
 *   r_cap in {16,32,48,64} >= every rank;
 *   X [max_rows, K] (pad rows inside segments must be 0: then Y's pad rows are 0);
 *   W [N, K]; Y [max_rows, N]; Hs [max_rows, r_cap] or NULL (inference: kept
 *   in the workspace).  Rows >= seg_off[S] of Y/Hs are not written.
 * Errors: MUX_ERR_INVALID_ARGUMENT (shape, alignment (16 B), rank/scale,
 * index checks), MUX_ERR_INSUFFICIENT_BUFFER, MUX_ERR_CUDA. */
MUX_API mux_status mux_linear_fwd(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                          int32_t num_adapters, const mux_adapter* adapters,
                          int32_t max_rows, int32_t K, int32_t N, int32_t r_cap,
                          const mux_bf16* X, const mux_bf16* W,
                          mux_bf16* Y, mux_bf16* Hs,
                          void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* Forward with the shrink supplied by the caller (tensor parallelism, SURVEY
 * §8(e)): Y[i,:] = X[i,:] W^T + Hs[i,:] B_t^T for rows i of segment s,
 * t = seg_task[s] — the same as mux_linear_fwd except that Hs [max_rows, r_cap]
 * is an INPUT (bf16, columns >= rank_t zero, e.g. from mux_linear_shrink on
 * each rank's own rows, then all-gathered) and no shrink tiles run.  With the
 * Hs of mux_linear_fwd, Y is bit-identical to mux_linear_fwd's.  Arguments and
 * errors as mux_linear_fwd; Hs must be non-NULL and 16-byte aligned. */
MUX_API mux_status mux_linear_fwd_hs(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                          int32_t num_adapters, const mux_adapter* adapters,
                          int32_t max_rows, int32_t K, int32_t N, int32_t r_cap,
                          const mux_bf16* X, const mux_bf16* W, mux_bf16* Y, const mux_bf16* Hs,
                          void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* Shrink only, over a row range: Hs[i,j] = bf16(s_t * X[i,:] A_t[j,:]^T)
 * (0 for rank_t <= j < r_cap) for the pair row blocks overlapping packed rows
 * [row_begin, row_end) — the per-rank part of a column-parallel forward under
 * sequence parallelism (each rank shrinks only the rows it owns; the Hs rows,
 * T x r_cap, are then all-gathered instead of every rank recomputing all of
 * them inside mux_linear_fwd).  Values equal mux_linear_fwd's Hs bit for bit.
 * row_begin a multiple of 256; row_end a multiple of 256 or >= max_rows; rows
 * outside the range or >= seg_off[S] are not written.  Arguments as
 * mux_linear_fwd without W/Y (N still sizes the adapters' B_t); Hs output
 * non-NULL.  Errors as mux_linear_fwd. */
MUX_API mux_status mux_linear_shrink(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                          int32_t num_adapters, const mux_adapter* adapters,
                          int32_t max_rows, int32_t K, int32_t N, int32_t r_cap,
                          const mux_bf16* X, int32_t row_begin, int32_t row_end, mux_bf16* Hs,
                          void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* Backward (Eq. 2 + LoRA chain rule).  For rows i of segment s, t = seg_task[s]:
 *   Gs[i,j]  = bf16(s_t * dY[i,:] B_t[:,j])                 (workspace)
 *   dX[i,:]  = dY[i,:] W + Gs[i,:] A_t                      (NULL = skip)
 *   dA_t     = sum over t's rows of Gs[i,:]^T X[i,:]         fp32 [rank, K]
 *   dB_t     = sum over t's rows of dY[i,:]^T Hs[i,:]        fp32 [N, rank]
 * Hs is the forward's output.  A task with no rows gets dA = dB = 0.
 * Arguments as in mux_linear_fwd; dY [max_rows, N] (pad rows may be nonzero:
 * they reach only dX's pad rows). */
MUX_API mux_status mux_linear_bwd(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                          int32_t num_adapters, const mux_adapter* adapters,
                          int32_t max_rows, int32_t K, int32_t N, int32_t r_cap,
                          const mux_bf16* dY, const mux_bf16* X,
                          const mux_bf16* W, const mux_bf16* Hs,
                          mux_bf16* dX,
                          void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* The two halves of mux_linear_bwd, for callers that overlap them on two
 * streams (the HBM-bound adapter gradients of layer l run in the tail of the
 * tensor-bound dX GEMM of layer l-1):
 *   MUX_BWD_DX     the fused GEMM: Gs into the workspace and dX (dX may be NULL)
 *   MUX_BWD_GRADS  dA_t, dB_t from X, dY, Hs and the Gs that MUX_BWD_DX left in
 *                  the SAME workspace; must run after it (stream order or an
 *                  event), and nothing may reuse that workspace in between.
 * Arguments as mux_linear_bwd; part 1 + part 2 == mux_linear_bwd bit for bit. */
#define MUX_BWD_DX 1
#define MUX_BWD_GRADS 2
MUX_API mux_status mux_linear_bwd_part(int32_t part, int32_t num_segs, const int32_t* seg_off,
                                       const int32_t* seg_task, int32_t num_adapters, const mux_adapter* adapters,
                                       int32_t max_rows, int32_t K, int32_t N, int32_t r_cap, const mux_bf16* dY,
                                       const mux_bf16* X, const mux_bf16* W, const mux_bf16* Hs, mux_bf16* dX,
                                       void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* ---------------------------------------------------------------------------
 * Fused GEMM -> reduce-scatter for tensor parallelism (NEXT-1:
 * the row-parallel forward Y = sum_p X_p W_p^T and the column-parallel dX =
 * sum_p dY_p W_p both end in a reduce-scatter over rows).  Instead of writing
 * a local partial and calling a collective, the fused GEMM's epilogue stores
 * every output tile straight into the receive slot of the rank that owns the
 * tile's rows (peer memory over NVLink), tile by tile as the GEMM runs;
 * mux_rs_reduce on the owner then sums the `world` slots.  Rows are owned in
 * contiguous blocks of rows_per_rank (a multiple of 256; world *
 * rows_per_rank == max_rows).  Each rank allocates, once, a receive buffer of
 * world * rows_per_rank * cols bf16 and a flag block of mux_rs_flags_elems()
 * zeroed uint64, and every rank gets all ranks' pointers (e.g. by CUDA IPC or
 * symmetric memory).  seq numbers the calls (1, 2, ...) and is the same on
 * all ranks: a GEMM waits until every owner has reduced call seq - 1 before
 * overwriting its slot, and publishes call seq when its last tile landed;
 * mux_rs_reduce waits for all sources' call seq, then acknowledges.  Both are
 * stream-ordered (no host synchronisation).
 * Waits on another rank's flag (here and in the all-gather below) give up
 * after MUX_PEER_TIMEOUT_S seconds (environment, read once per process;
 * default 600, 0 = never) by trapping, which the caller sees as a sticky
 * CUDA error: rank skew (a checkpoint or an eval on one rank) is normal, only
 * a protocol bug never completes.  Waits inside one GPU keep an 8 s watchdog.
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t world;                                  /* 1 .. MUX_RS_MAX_WORLD */
  int32_t rank;                                   /* this rank */
  int32_t rows_per_rank;                          /* multiple of 256 */
  uint64_t seq;                                   /* > 0, increasing per call */
  mux_bf16* recv[MUX_RS_MAX_WORLD];               /* rank d's receive buffer [world][rows_per_rank][cols] */
  unsigned long long* flags[MUX_RS_MAX_WORLD];    /* rank d's flag block [mux_rs_flags_elems(world)] */
} mux_rs;
MUX_API size_t mux_rs_flags_elems(int32_t world);
/* forward of a row-parallel layer: mux_linear_fwd with Y replaced by the fused reduce-scatter */
MUX_API mux_status mux_linear_fwd_rs(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                                     int32_t num_adapters, const mux_adapter* adapters, int32_t max_rows,
                                     int32_t K, int32_t N, int32_t r_cap, const mux_bf16* X, const mux_bf16* W,
                                     mux_bf16* Hs, const mux_rs* rs, void* workspace, size_t workspace_bytes,
                                     cudaStream_t stream);
/* dX GEMM of a column-parallel layer (mux_linear_bwd_part(MUX_BWD_DX) with dX reduce-scattered);
 * the adapter gradients follow with mux_linear_bwd_part(MUX_BWD_GRADS) on the same workspace */
MUX_API mux_status mux_linear_bwd_dx_rs(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                                        int32_t num_adapters, const mux_adapter* adapters, int32_t max_rows,
                                        int32_t K, int32_t N, int32_t r_cap, const mux_bf16* dY,
                                        const mux_bf16* X, const mux_bf16* W, const mux_bf16* Hs,
                                        const mux_rs* rs, void* workspace, size_t workspace_bytes,
                                        cudaStream_t stream);
/* owner side: out[rows_per_rank, cols] = sum over sources of their slots (fp32, ascending source order) */
MUX_API mux_status mux_rs_reduce(const mux_rs* rs, int32_t cols, mux_bf16* out, int64_t ldo, cudaStream_t stream);

/* ---------------------------------------------------------------------------
 * All-gather -> GEMM for tensor parallelism (the column-parallel forward's
 * AG(X) and the row-parallel backward's AG(dY)).  Every
 * rank pushes its own rows into every rank's gather buffer with the copy
 * engines (mux_ag_push: no SMs, so it runs under the GEMMs) and signals each
 * destination with a stream memory write; the fused GEMM's TMA producer waits
 * on a row block's owner flag just before its first load of those rows, so
 * the GEMM starts on whatever rows have landed (its own at once) while the
 * rest are in flight.  The gather buffer stays valid until the caller
 * releases it (mux_ag_release, e.g. after the backward that re-reads X),
 * which allows the owners to push the next call's rows.
 * mux_ag has mux_rs's fields: recv[d] = rank d's gather buffer
 * [world * rows_per_rank][cols] (the full A operand on rank d), flags[d] =
 * rank d's flag block [mux_rs_flags_elems(world)], zeroed once. */
typedef mux_rs mux_ag;
MUX_API mux_status mux_ag_push(const mux_ag* ag, const mux_bf16* rows, int64_t ld, int32_t cols,
                               cudaStream_t stream);
MUX_API mux_status mux_ag_release(const mux_ag* ag, cudaStream_t stream);
/* mux_linear_fwd with X = ag->recv[ag->rank], each row block read once it has landed */
MUX_API mux_status mux_linear_fwd_ag(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                                     int32_t num_adapters, const mux_adapter* adapters, int32_t max_rows,
                                     int32_t K, int32_t N, int32_t r_cap, const mux_ag* ag, const mux_bf16* W,
                                     mux_bf16* Y, mux_bf16* Hs, void* workspace, size_t workspace_bytes,
                                     cudaStream_t stream);
/* mux_linear_bwd with dY = ag->recv[ag->rank] */
MUX_API mux_status mux_linear_bwd_ag(int32_t num_segs, const int32_t* seg_off, const int32_t* seg_task,
                                     int32_t num_adapters, const mux_adapter* adapters, int32_t max_rows,
                                     int32_t K, int32_t N, int32_t r_cap, const mux_ag* ag, const mux_bf16* X,
                                     const mux_bf16* W, const mux_bf16* Hs, mux_bf16* dX, void* workspace,
                                     size_t workspace_bytes, cudaStream_t stream);

/* ---------------------------------------------------------------------------
 * Fused projections with one adapter per column slice (q|k|v, gate|up).
 * P:296 names "attaching adapters to the fused qkv projection" as what keeps
 * per-projection LoRA from running on one fused backbone op; here the backbone
 * W = [W_0; W_1; ...] (rows = output columns) runs as ONE GEMM while every
 * task keeps an independent adapter (A_{t,s}, B_{t,s}, rank, scale) on each
 * slice s = output columns [col_off[s], col_off[s+1]).  By definition this is
 * num_slices independent LoRA linears sharing X, computed together:
 *   fwd:  Y[i, slice s] = X[i,:] W_s^T + s_{t,s} (X[i,:] A_{t,s}^T) B_{t,s}^T
 *         Hs[i, s*r_cap + j] = bf16(s_{t,s} X[i,:] A_{t,s}[j,:]^T)   (Hs [max_rows, S*r_cap])
 *   bwd:  Gs_s = bf16(s_{t,s} dY[i, slice s] B_{t,s})
 *         dX[i,:] = dY[i,:] W + sum_s Gs_s[i,:] A_{t,s}
 *         dA_{t,s} = sum over t's rows Gs_s^T X;  dB_{t,s} = sum dY[:, slice s]^T Hs_s
 * With num_slices = 1 (or slices = NULL) every op equals the per-call entry
 * points above bit for bit.  Adapters are indexed task-major:
 * adapters[t * num_slices + s]; B_{t,s} is [col_off[s+1] - col_off[s], rank]
 * (leading dimension ldb) and dB_{t,s} likewise; rank 0 = no adapter on that
 * slice.  Within one task, a non-finite value in one slice's adapter can reach
 * that task's other slices where a 256-column output tile straddles two
 * slices (the kernel multiplies it by the zero rows outside the slice); it
 * never reaches another task's rows.
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t num_slices;                    /* 1 .. MUX_MAX_SLICES */
  int32_t col_off[MUX_MAX_SLICES + 1];   /* 0 = col_off[0] < ... < col_off[S] = N, multiples of 8 */
} mux_slices;

typedef enum {
  MUX_OP_FWD = 1,        /* mux_linear_fwd (rs != NULL: mux_linear_fwd_rs; ag != NULL: mux_linear_fwd_ag) */
  MUX_OP_FWD_HS = 2,     /* mux_linear_fwd_hs (Hs is the input) */
  MUX_OP_SHRINK = 3,     /* mux_linear_shrink over [row_begin, row_end) */
  MUX_OP_BWD = 4,        /* mux_linear_bwd (ag != NULL: mux_linear_bwd_ag) */
  MUX_OP_BWD_DX = 5,     /* mux_linear_bwd_part(MUX_BWD_DX) (rs != NULL: mux_linear_bwd_dx_rs) */
  MUX_OP_BWD_GRADS = 6,  /* mux_linear_bwd_part(MUX_BWD_GRADS) */
  MUX_OP_SHRINK_BWD = 7  /* Gs[i, s*r_cap + j] = bf16(s_{t,s} dY[i, slice s] B_{t,s}[:, j]) for the pair row
                            blocks overlapping [row_begin, row_end) into Gs (no X, W, Hs): the per-rank
                            part of a row-parallel backward whose Gs rows are then all-gathered */
} mux_linear_op;

/* All arguments of one linear call; fields an op does not use are ignored
 * (set them to 0/NULL).  Pointers as in the per-op entry points. */
typedef struct {
  int32_t op;                        /* mux_linear_op */
  int32_t num_segs;
  const int32_t* seg_off;            /* device [num_segs + 1] */
  const int32_t* seg_task;           /* [host] [num_segs] task index */
  int32_t num_adapters;              /* tasks (1..64); num_adapters * num_slices <= MUX_MAX_ADAPTER_SLOTS */
  const mux_adapter* adapters;       /* [host] [num_adapters * num_slices], task-major */
  const mux_slices* slices;          /* [host] NULL = one slice over all N columns */
  int32_t max_rows, K, N, r_cap;     /* r_cap: per slice, >= every rank */
  const mux_bf16* X;                 /* [max_rows, K] (fwd input; bwd: for dA) */
  const mux_bf16* W;                 /* [N, K] */
  const mux_bf16* dY;                /* [max_rows, N] (bwd) */
  mux_bf16* Y;                       /* [max_rows, N] (fwd output) */
  mux_bf16* Hs;                      /* [max_rows, S * r_cap]: fwd/shrink output (fwd: NULL = workspace),
                                        fwd_hs / bwd input */
  mux_bf16* dX;                      /* [max_rows, K] (bwd output, NULL = skip) */
  int32_t row_begin, row_end;        /* MUX_OP_SHRINK row range */
  const mux_rs* rs;                  /* optional fused reduce-scatter (FWD, BWD_DX) */
  const mux_ag* ag;                  /* optional fused all-gather (FWD: X, BWD: dY) */
  void* workspace;                   /* >= mux_linear_workspace_size(num_segs, max_rows, K, N, S * r_cap) */
  size_t workspace_bytes;
  cudaStream_t stream;
  mux_bf16* Gs;                      /* [max_rows, S * r_cap] backward: NULL = in the workspace; else the
                                        output of MUX_OP_SHRINK_BWD, or the given Gs of BWD / BWD_DX /
                                        BWD_GRADS (then no shrink tiles run; e.g. all-gathered rows) */
} mux_linear_args;

/* One linear call described by `a` (the per-op entry points above are this
 * with slices = NULL).  Errors as mux_linear_fwd, plus MUX_ERR_INVALID_ARGUMENT
 * for an unknown op, a bad slice table or too many adapter slots. */
MUX_API mux_status mux_linear(const mux_linear_args* a);

/* ---------------------------------------------------------------------------
 * Collectives reduced / broadcast inside the NVSwitch (NVLink SHARP, "NVLS";
 * NEXT-1: the paper offloads the overlapped collectives to NVLink
 * SHARP so they need only ~8 CTAs).  The caller (e.g. with the CUDA driver's
 * cuMulticastCreate / cuMulticastBindMem; paper_2603_02885_b200/nvls.py)
 * gives every rank one copy of a symmetric buffer of world * rows_per_rank *
 * cols bf16 and of a flag block of mux_nvls_flags_elems() zeroed uint64, both
 * also bound to a multicast object: uc_* = this rank's copy, mc_* = the
 * multicast address.  seq numbers the calls on one mux_nvls (1, 2, ...), the
 * same on all ranks; ctas = CTAs used (0 = 16).  Waits on other ranks obey
 * MUX_PEER_TIMEOUT_S.  Errors: MUX_ERR_INVALID_ARGUMENT, MUX_ERR_CUDA.
 *
 * mux_nvls_reduce_scatter: every rank has written its partial [world *
 *   rows_per_rank, cols] into uc_buf (stream order: e.g. mux_linear_fwd with Y
 *   = uc_buf); out [rows_per_rank, cols] (row stride ldo) = the sum over ranks
 *   of their copies' rows [rank * rows_per_rank, ...), read with
 *   multimem.ld_reduce (summed in the switch, fp32 accumulation).  Returns
 *   (in stream order) once every rank has read every copy, so uc_buf may be
 *   rewritten by the next call.
 * mux_nvls_all_gather: rows [rows_per_rank, cols] (row stride ld) are stored
 *   once to the multicast address (multimem.st): afterwards every rank's uc_buf
 *   holds all ranks' rows.  Waits for the previous call's mux_nvls_release
 *   on every rank before storing.
 * mux_nvls_release: this rank is done reading uc_buf of the last all-gather.
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t world;                   /* 1 .. MUX_RS_MAX_WORLD */
  int32_t rank;
  int32_t rows_per_rank;
  uint64_t seq;                    /* > 0, increasing per call */
  mux_bf16* uc_buf;                /* this rank's copy [world * rows_per_rank][cols] (16-byte aligned) */
  mux_bf16* mc_buf;                /* multicast address of the buffer */
  unsigned long long* uc_flags;    /* this rank's copy of the flag block */
  unsigned long long* mc_flags;    /* multicast address of the flag block */
} mux_nvls;
MUX_API size_t mux_nvls_flags_elems(void);
MUX_API mux_status mux_nvls_reduce_scatter(const mux_nvls* nv, int32_t cols, mux_bf16* out, int64_t ldo,
                                           int32_t ctas, cudaStream_t stream);
MUX_API mux_status mux_nvls_all_gather(const mux_nvls* nv, const mux_bf16* rows, int64_t ld, int32_t cols,
                                       int32_t ctas, cudaStream_t stream);
MUX_API mux_status mux_nvls_release(const mux_nvls* nv, cudaStream_t stream);

/* ---------------------------------------------------------------------------
 * Decoder-block ops (NEXT-3).  Row-major bf16 matrices with an explicit row
 * stride `ld*` in ELEMENTS (a multiple of 8: 16-byte rows), so q/k/v or
 * gate/up can be column slices of one fused projection output.  fp32 math.
 * Errors: MUX_ERR_INVALID_ARGUMENT (sizes, strides, 16-byte alignment),
 * MUX_ERR_INSUFFICIENT_BUFFER, MUX_ERR_CUDA.
 * ------------------------------------------------------------------------- */

/* row_start[r] for r < max_rows: the first packed row of row r's sequence,
 * -1 for pad rows.  seq_len [num_seqs] and seq_row [num_seqs] are the
 * mux_pack_chunks inputs/outputs (a sequence occupies rows
 * [seq_row[s], seq_row[s] + seq_len[s]) of its pack). */
MUX_API mux_status mux_pack_row_start(int32_t num_seqs, const int32_t* seq_len, const int32_t* seq_row,
                                      int32_t max_rows, int32_t* row_start, cudaStream_t stream);

/* Causal attention inside packed sequences, per head h (kv head h / (H/Hkv)):
 *   o[r,h,:] = sum_{j = row_start[r]..r} softmax_j(scale <q[r,h,:], k[j,hk,:]>) v[j,hk,:]
 *   lse[r,h] = log sum_j exp(scale <q, k>)   (fp32 [rows, H]; -inf, o = 0 for pad rows)
 * q [rows, H*128] (row stride ldq), k, v [rows, Hkv*128]; head dim 128;
 * H % Hkv == 0.  Warp-level tensor-core MMAs, flash-style (S never in HBM). */
MUX_API mux_status mux_attn_fwd(int32_t rows, int32_t heads, int32_t kv_heads, int32_t head_dim,
                                const mux_bf16* q, int64_t ldq, const mux_bf16* k, int64_t ldk,
                                const mux_bf16* v, int64_t ldv, const int32_t* row_start, float scale,
                                mux_bf16* o, int64_t ldo, float* lse, cudaStream_t stream);

/* Gradients of the above for upstream dO: dq [rows, H*128], dk, dv
 * [rows, Hkv*128] (overwritten; pad rows 0).  Deterministic (no atomics).
 * workspace: >= mux_attn_workspace_size(rows, heads) bytes, no zeroing needed. */
MUX_API size_t mux_attn_workspace_size(int32_t rows, int32_t heads);
MUX_API mux_status mux_attn_bwd(int32_t rows, int32_t heads, int32_t kv_heads, int32_t head_dim,
                                const mux_bf16* dO, int64_t lddo, const mux_bf16* q, int64_t ldq,
                                const mux_bf16* k, int64_t ldk, const mux_bf16* v, int64_t ldv,
                                const mux_bf16* o, int64_t ldo, const float* lse, const int32_t* row_start,
                                float scale, mux_bf16* dq, int64_t lddq, mux_bf16* dk, int64_t lddk,
                                mux_bf16* dv, int64_t lddv, void* workspace, size_t workspace_bytes,
                                cudaStream_t stream);

/* Rotary position embedding, IN PLACE on x [rows, heads*head_dim] (stride ld):
 * pairs (i, i + d/2) of each head rotated by pos * base^(-2i/d), pos =
 * r - row_start[r] (inverse != 0: by the negative angle = the backward).
 * Pad rows (row_start -1) untouched.  head_dim a multiple of 16. */
MUX_API mux_status mux_rope(int32_t rows, int32_t heads, int32_t head_dim, mux_bf16* x, int64_t ld,
                            const int32_t* row_start, float base, int32_t inverse, cudaStream_t stream);

/* RMSNorm with the pre-norm residual stream fused in (w is frozen backbone: no dw).
 * fwd: xs = x + res (bf16; written to xsum) when res != NULL, else xs = x;
 *      y = xs / sqrt(mean(xs^2) + eps) * w.   res and xsum may be NULL (plain RMSNorm).
 * bwd: g = dy + dy2 + dy3 (dy2, dy3 may be NULL: the gradients of the linears that
 *      read the normalised output, summed here), dx = d rmsnorm(x)/dx^T (g * w)
 *      + resid (resid may be NULL: the residual path's gradient).
 * All [rows, dim] with row strides in elements; w [dim]; dim % 8 == 0. */
MUX_API mux_status mux_rmsnorm_fwd(int32_t rows, int32_t dim, const mux_bf16* x, int64_t ldx, const mux_bf16* res,
                                   int64_t ldres, mux_bf16* xsum, int64_t ldxs, const mux_bf16* w, float eps,
                                   mux_bf16* y, int64_t ldy, cudaStream_t stream);
MUX_API mux_status mux_rmsnorm_bwd(int32_t rows, int32_t dim, const mux_bf16* dy, int64_t lddy,
                                   const mux_bf16* dy2, int64_t lddy2, const mux_bf16* dy3, int64_t lddy3,
                                   const mux_bf16* x, int64_t ldx, const mux_bf16* w, float eps,
                                   const mux_bf16* resid, int64_t ldres, mux_bf16* dx, int64_t lddx,
                                   cudaStream_t stream);

/* SwiGLU h = silu(g) * u; backward dg = dh u s (1 + g (1 - s)), du = dh silu(g),
 * s = sigmoid(g).  All [rows, dim], dim % 8 == 0. */
MUX_API mux_status mux_swiglu_fwd(int32_t rows, int32_t dim, const mux_bf16* g, int64_t ldg, const mux_bf16* u,
                                  int64_t ldu, mux_bf16* h, int64_t ldh, cudaStream_t stream);
MUX_API mux_status mux_swiglu_bwd(int32_t rows, int32_t dim, const mux_bf16* dh, int64_t lddh, const mux_bf16* g,
                                  int64_t ldg, const mux_bf16* u, int64_t ldu, mux_bf16* dg, int64_t lddg,
                                  mux_bf16* du, int64_t lddu, cudaStream_t stream);

/* Residual add y = a + b (fp32 add, bf16 out); y may alias a or b.  [rows, dim], dim % 8 == 0. */
MUX_API mux_status mux_add(int32_t rows, int32_t dim, const mux_bf16* a, int64_t lda, const mux_bf16* b,
                           int64_t ldb, mux_bf16* y, int64_t ldy, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* MUX_H_ */
