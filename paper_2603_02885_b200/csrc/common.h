// common.h — kernel parameter blocks shared by the host ABI (mux_abi.cu) and
// the kernels.  Product code only; nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

#include "../../include/mux.h"
#include <cuda_bf16.h>

namespace mux {

// ---- fused linear GEMM (mux_linear_fwd / the dX part of mux_linear_bwd)
// A work tile is computed by a CTA pair (cluster of 2, tcgen05 cta_group::2):
// 256 rows (128 per CTA = TMEM lanes) x 256 output columns (each CTA stages
// half of the B operand), reduction in k-blocks of 64.
constexpr int kBM = 128;        // rows per CTA
constexpr int kPairRows = 256;  // rows per pair tile (MMA M = 256)
constexpr int kBN = 256;        // output columns per tile (TMEM columns per accumulator)
// Reduction depth per pipeline stage: 64 (6 stages) for the forward kernel,
// 128 (3 stages) for the backward dX kernel (measured best for each,
// profiles/r01_gemm_ab_bk.jsonl).  Both keep 192 KB of operands in flight.
#ifndef MUX_BWD_BK
#define MUX_BWD_BK 128   // A/B builds: 64 (then 6 stages)
#endif
template <bool kBwd>
struct GemmCfg {
  static constexpr int kBK = kBwd ? MUX_BWD_BK : 64;
  static constexpr int kKSub = kBK / 64;  // 128 B swizzle rows (64 bf16) per stage row
  static constexpr int kStages = kBwd ? (MUX_BWD_BK == 64 ? 6 : 3) : 6;
};
constexpr int kRowQuarter = 64; // segment granularity inside a pair tile (chunk minimum)
constexpr int kSideN = 128;     // N of the shrink MMA (rank padded to 64 in CTA 0's half)
constexpr int kSkMaxClusters = 120;          // stream-K range table in shared memory (misc area)
constexpr int kSkSlotFloats = 2 * 4 * 256 * 32;  // one cluster's partial 256 x 256 fp32 tile

constexpr int kMaxCarrySlots = 32;

struct GemmParams {
  // A operand of the main product: X (fwd) / dY (bwd): dims {Kred, rows}, box {64, 128}
  CUtensorMap map_a;
  // backbone W [N, K]: dims {K, N}, box {64, 64}
  CUtensorMap map_w;
  // side tensor Hs (fwd) / Gs (bwd): dims {r_cap, rows}, box {64, 128}
  CUtensorMap map_side;
  // output Y (fwd) / dX (bwd): dims {Nout, rows}, box {64, 32} (TMA store)
  CUtensorMap map_out;
  // per adapter slot (task t, column slice s: slot t * num_slices + s):
  // A_{t,s} dims {K, rank} box {64, 64};  B_{t,s} dims {rank, slice width} box {64, 64}.
  // A rank-0 slot holds a copy of another slot's maps (read only out of bounds: zero fill).
  CUtensorMap map_lora_a[MUX_MAX_ADAPTER_SLOTS];
  CUtensorMap map_lora_b[MUX_MAX_ADAPTER_SLOTS];
  // carrier shrink operand per adapter (carry = 1, one slice, <= kMaxCarrySlots adapters):
  // fwd A_t dims {K, rank} box {64, 8} (128 B swizzle, K-major);
  // bwd B_t dims {rank, N} box {16, 128} (32 B swizzle: the MMA's N = rank is contiguous, MN-major)
  CUtensorMap map_shrink[kMaxCarrySlots];
  const int32_t* seg_off;        // device [num_segs + 1]
  __nv_bfloat16* side_out;       // Hs / Gs [max_rows, num_slices * r_cap] (slice s: columns s * r_cap ..)
  __nv_bfloat16* out;            // Y / dX [max_rows, nout] (direct-store epilogue variant)
  unsigned long long* flags;     // [ceil(max_rows/256)] shrink-published counters (workspace, zeroed once;
                                 // the last CTA of every launch resets them)
  unsigned long long* epoch;     // workspace launch epoch; bumped by the last CTA to finish
  unsigned int* done;            // CTAs finished in this launch (reset by the last one)
  int32_t num_segs;
  int32_t max_rows;
  int32_t kred;                  // reduction length of the main product (K fwd, N bwd)
  int32_t nout;                  // output columns (N fwd, K bwd)
  int32_t r_cap;                 // per slice
  int32_t num_slices;            // column slices of the fwd output (1 = plain linear)
  int32_t slice_off[MUX_MAX_SLICES + 1];  // fwd output columns of each slice (bwd: reduction columns)
  int32_t has_main;              // 0: only the shrink (side) tiles, over row blocks [side_m_lo, side_m_hi)
  int32_t has_side;              // 0: no side tiles, Hs given (mux_linear_fwd_hs)
  int32_t side_m_lo, side_m_hi;  // shrink-only launches: pair row-block range
  int32_t side_first;            // 1: all side tiles before the main tiles (short reductions)
  int32_t group_m;               // raster band: pair row-blocks sharing a sweep over W tiles
  int32_t group_n;               // > 0: column bands of group_n output blocks instead (W-resident raster)
  int32_t carry;                 // 1: shrink on carrier main tiles, no side tiles (gemm.cu), from map_shrink;
                                 // 2: also when one carrier per row block spans several waves
  unsigned long long* dbg;       // MUX_PROFILE builds only: wait-cycle counters (see gemm.cu)
  // Fused reduce-scatter output (tensor parallel, mux_linear_*_rs): rs_world > 0 sends each
  // output tile straight to the rank that owns its rows (rs_rows per rank, contiguous blocks):
  // map_out_rs[d] = rank d's receive slot for this rank ([rs_rows, nout], box {64, 32}).
  // Handshake (all values = the call's sequence number rs_seq): before its first store the
  // epilogue waits rs_ack[d] >= rs_seq - 1 (rank d reduced the previous call); after the last
  // store the last CTA sets rs_ready[d] = rs_seq on every rank d.
  int32_t rs_world;
  int32_t rs_rows;
  unsigned long long rs_seq;
  const unsigned long long* rs_ack;          // this rank's ack flags [rs_world] (written by the dests)
  unsigned long long* rs_ready[MUX_RS_MAX_WORLD];  // rank d's ready flag for this source (peer)
  CUtensorMap map_out_rs[MUX_RS_MAX_WORLD];
  // Fused all-gather input (tensor parallel, mux_linear_*_ag): the A operand (X or dY) is the
  // local gather buffer that every rank pushes its own rows into (copy engines, mux_ag_push);
  // before loading a row block the producer waits until ag_flags[owner] >= ag_seq.
  int32_t ag_world;
  int32_t ag_rows;
  unsigned long long ag_seq;
  const unsigned long long* ag_flags;
  unsigned long long peer_wait_ns;  // limit of a wait on another rank's flag (0 = none; ptx.cuh)
  // Stream-K schedule of the main tiles (sk = 1, chosen on the host where whole tiles leave the last
  // round of clusters half idle, e.g. 512-column tensor-parallel shards; see gemm.cu): cluster c's
  // first piece of a split tile is a partial accumulator in sk_part slot c, published on sk_flags[c].
  int32_t sk;
  int32_t sk_side_cost_x4;          // a shrink tile's k-block, in quarters of a main k-block (balance)
  unsigned long long* sk_flags;     // [kSkMaxClusters] epoch-tagged (workspace)
  float* sk_part;                   // [kSkMaxClusters][2 CTAs][4 warps][256 cols][32 lanes] fp32
  int32_t seg_adapter[MUX_MAX_SEGMENTS];  // task of the segment
  int32_t seg_rank[MUX_MAX_SEGMENTS];     // max rank over the task's slots (0: no adapter at all)
  int32_t slot_rank[MUX_MAX_ADAPTER_SLOTS];
  float slot_scale[MUX_MAX_ADAPTER_SLOTS];
};

// a __grid_constant__ kernel parameter block is limited to 32764 bytes
static_assert(sizeof(GemmParams) <= 32764, "GemmParams exceeds the kernel parameter limit");

// ---- segmented adapter gradients (dA_t, dB_t)
constexpr int kGradBM = 128;     // output rows per unit (k for dA, n for dB)
constexpr int kGradBK = 128;     // tokens per pipeline stage
constexpr int kGradStages = 4;   // at most (fewer when a dA unit stages several Gs boxes: grad.cu)

struct GradParams {
  CUtensorMap map_x;    // X  dims {K, rows} box {64, 128}
  CUtensorMap map_dy;   // dY dims {N, rows} box {64, 128}
  CUtensorMap map_hs;   // Hs dims {r_cap, rows} box {64, 128}
  CUtensorMap map_gs;   // Gs dims {r_cap, rows} box {64, 128}
  const int32_t* seg_off;
  int32_t num_segs;
  int32_t K, N, r_cap;
  int32_t num_tasks;                       // adapters with rank > 0 and a gradient to write
  int32_t units_a;                         // ceil(K/128) dA units per task (0 if no task wants dA)
  int32_t units_b;                         // ceil(N/128)
  uint64_t task_segs[MUX_MAX_ADAPTERS];    // bit s set: segment s belongs to the task
  // CUDA-core kernel (grad_simt.cu): one launch per column slice, one slot per task
  int32_t task_rank[MUX_MAX_ADAPTERS];
  float* task_dA[MUX_MAX_ADAPTERS];
  float* task_dB[MUX_MAX_ADAPTERS];
  // tcgen05 kernel (grad.cu): every column slice of a fused projection in one launch.  map_dy spans
  // all N columns, map_hs / map_gs all S * r_cap side columns.  A dA unit (task, 128 k) stages nb_a
  // 64-column Gs boxes and issues one MMA of N = 64 nb_a per 16 tokens (X read once for all slices);
  // dB unit u of a task belongs to slice s with b_units_off[s] <= u < b_units_off[s + 1].
  int32_t num_slices;
  int32_t slice_off[MUX_MAX_SLICES + 1];
  int32_t b_units_off[MUX_MAX_SLICES + 1];
  int32_t nb_a;                            // ceil(S * r_cap / 64) <= 4
  int32_t stages;                          // pipeline stages (stage_bytes each)
  uint32_t stage_bytes;
  int32_t slot_rank[MUX_MAX_ADAPTER_SLOTS];  // slot = (compacted task) * S + slice
  float* slot_dA[MUX_MAX_ADAPTER_SLOTS];
  float* slot_dB[MUX_MAX_ADAPTER_SLOTS];
};
static_assert(sizeof(GradParams) <= 32764, "GradParams exceeds the kernel parameter limit");

// ---- causal attention forward on tcgen05 (attn_tc.cu)
struct AttnTcParams {
  CUtensorMap map_q;  // q [R, H*128]: box {64 cols, 128 rows}, 128 B swizzle
  CUtensorMap map_k;  // k [R, Hkv*128]: box {64 cols, 64 rows}
  CUtensorMap map_v;  // v [R, Hkv*128]
  const int32_t* row_start;
  __nv_bfloat16* o;
  long long ldo;
  float* lse;
  int R, H, Hkv;
  float scale_log2;
};

// ---- causal attention backward on tcgen05 (attn_bwd_tc.cu); boxes {64 cols, rows}
struct AttnBwdTcParams {
  CUtensorMap map_q128, map_do128;  // dQ kernel: 128-row query tiles
  CUtensorMap map_k64, map_v64;     // dQ kernel: 64-row key tiles
  CUtensorMap map_k128, map_v128;   // dK/dV kernel: 128-row key tiles
  CUtensorMap map_q64, map_do64;    // dK/dV kernel: 64-row query tiles
  const int32_t* row_start;
  const float* lse;                 // [R, H]
  const float* D;                   // [R, H] rowsum(dO * O)
  __nv_bfloat16* dq;
  long long lddq;
  __nv_bfloat16* dk;
  long long lddk;
  __nv_bfloat16* dv;
  long long lddv;
  int R, H, Hkv;
  float scale_log2, scale;
};

// ---- receive side of the fused GEMM -> reduce-scatter (rs.cu)
struct RsReduceParams {
  int world, rank, rows, cols;
  unsigned long long seq;
  const uint4* recv;                      // this rank's receive buffer [world][rows][cols]
  unsigned long long* flags;              // this rank's flag block
  unsigned long long* ack[MUX_RS_MAX_WORLD];  // rank s's ack slot for this rank (peer)
  uint4* out;                             // [rows, cols], row stride ldo8 * 8 elements
  long long ldo8;
  unsigned long long peer_wait_ns;        // limit of the wait for the sources' ready flags (0 = none)
};

}  // namespace mux

// library-internal (hidden) helpers defined in mux_abi.cu, shared by the other ABI translation units
mux_status mux_set_error(mux_status st, const char* msg);   // thread-local mux_last_error() message
unsigned long long mux_peer_wait_ns();                       // MUX_PEER_TIMEOUT_S in ns (0 = none)
